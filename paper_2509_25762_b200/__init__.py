"""B200-native OPPO PPO-RLHF step (arXiv 2509.25762), behind a C ABI.

The product is ``liboppo.so`` (C++ host scheduler + sm_100a CUDA engine);
this package is the thin Python binding used by the tests and bench.
"""
from . import abi  # noqa: F401
from ._lib import ConfigError, InputError, InternalError, OppoError, lib  # noqa: F401
