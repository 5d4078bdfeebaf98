import json
import os
import sys

# as bench.py: the engine's device-side chunk hand-off requires eager kernel loading
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_vectors.json")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running")


@pytest.fixture(scope="session")
def golden():
    with open(GOLDEN) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def live_ref():
    """The compiled reference (oracle/_ref), or skip when it is not built here."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref/librlpipe_ref.so not built")
    R.ref()
    return R


def config_from_dict(d):
    from paper_2509_25762_b200 import abi
    cfg = abi.RunConfig()
    for k, v in d.items():
        if k == "chunk_candidates":
            for i, x in enumerate(v):
                cfg.chunk_candidates[i] = x
            continue
        if isinstance(v, dict):
            sub = getattr(cfg, k)
            for k2, v2 in v.items():
                if isinstance(v2, list):
                    arr = getattr(sub, k2)
                    for i, x in enumerate(v2):
                        arr[i] = x
                else:
                    setattr(sub, k2, v2)
        else:
            setattr(cfg, k, v)
    return cfg
