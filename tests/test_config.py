"""JSON config schema parity: paper_2509_25762_b200.config
against rlpipe::load_config_text / config_echo / task_fingerprint /
baseline() (config.cpp:75-420) — the committed vectors of
tests/golden/make_config_golden.py, and random configs against the live
compiled reference where oracle/_ref is built (this container)."""
import copy
import json
import os
import random

import pytest

from oracle import ref as R
from paper_2509_25762_b200 import abi
from paper_2509_25762_b200 import config as K

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "config_vectors.json")


def ours(text):
    try:
        c = K.load_config_text(text)
    except K.ConfigError as e:
        return dict(ok=False, error=str(e))
    return dict(ok=True, echo=K.config_echo(c), baseline_echo=K.config_echo(K.baseline(c)),
                fingerprint=K.task_fingerprint(c), error="")


def _canon(echo):
    return json.dumps(json.loads(echo), indent=2)


def check(text, ref):
    got = ours(text)
    assert got["ok"] == ref["ok"], (text, got.get("error"), ref["error"])
    if ref["ok"]:
        # key order, values and number types of the echo; the layout is
        # compared through a re-dump because the nlohmann copy this image
        # builds the reference with (cudnn_frontend's) prints integer arrays
        # inline, where stock nlohmann 3.11.3 (and config_echo) use one line
        # per element.  The fingerprint hashes the compact dump: exact.
        assert _canon(got["echo"]) == _canon(ref["echo"]), text
        assert _canon(got["baseline_echo"]) == _canon(ref["baseline_echo"]), text
        assert got["fingerprint"] == ref["fingerprint"], text
    elif ref["error"].startswith("config is not valid JSON: "):
        assert got["error"].startswith("config is not valid JSON: ")  # parser text differs
    else:
        assert got["error"] == ref["error"], text


def _cases():
    with open(GOLDEN) as f:
        return json.load(f)["cases"]


@pytest.mark.parametrize("case", _cases(), ids=lambda c: c["text"][:40])
def test_config_golden_vectors(case):
    check(case["text"], case)


def test_defaults_match_the_c_abi_defaults():
    """RunConfig{} restated in config.defaults() equals oppo_run_config_default."""
    a = K.to_run_config(K.defaults())
    from paper_2509_25762_b200 import scheduler as S
    b = S.default_config()
    for name, _ in abi.RunConfig._fields_:
        va, vb = getattr(a, name), getattr(b, name)
        if name in ("latency", "lengths", "ppo"):
            for f, _t in type(va)._fields_:
                x, y = getattr(va, f), getattr(vb, f)
                if hasattr(x, "__len__"):
                    x, y = list(x), list(y)
                assert x == y, (name, f)
        elif hasattr(va, "__len__"):
            assert list(va) == list(vb), name
        else:
            assert va == vb, name


def test_to_run_config_carries_every_field():
    c = K.load_config_text(_cases()[2]["text"])  # the cfg2-shaped config
    rc = K.to_run_config(c)
    assert (rc.mode, rc.steps, rc.batch_size, rc.prompt_len) == (abi.RUN_TRAIN, 40, 256, 128)
    assert (rc.delta_init, rc.delta_max, rc.controller, rc.window, rc.delta_inc) == (26, 64, 1, 4, 2)
    assert (rc.chunk_size, rc.schedule_mode, rc.vocab, rc.target_token) == (64, 0, 16, 3)
    assert (rc.lengths.kind, rc.lengths.cap, rc.lengths.sigma_log) == (1, 1024, 1.0)
    assert (rc.latency.prefill_per_token, rc.latency.count_prompt_in_prefill) == (0, 0)
    assert rc.ppo.lambda_ == 0.95 and rc.reward_bias == -0.125


def test_extension_blocks():
    text = json.dumps({"steps": 3, "model": {"actor": "0.5b", "reward": {"n_layers": 2, "d_model": 128}},
                       "gpu": {"dtype": "bf16", "scorer_sms": 64, "carry": "token"}})
    with pytest.raises(K.ConfigError, match="unknown key 'model'"):
        K.load_config_text(text)  # the reference schema rejects them
    c = K.load_config_text(text, extended=True)
    assert c["model"]["actor"] == "0.5b" and c["gpu"]["scorer_sms"] == 64
    assert K.task_fingerprint(c) == K.task_fingerprint(K.load_config_text('{"steps": 3}'))
    with pytest.raises(K.ConfigError, match="gpu.dtype"):
        K.load_config_text('{"gpu": {"dtype": "fp8"}}', extended=True)


def _mutations(rng, base):
    """Random edits of a valid config: values of other JSON types, out-of-range
    numbers, unknown keys, deleted blocks."""
    weird = [None, True, False, 0, -1, 3, 2.5, -0.5, 1e-7, 1e20, "x", "streamed", [], [1, 2], [[5, 1.0]], {}]
    c = copy.deepcopy(base)
    for _ in range(rng.randint(1, 3)):
        block = rng.choice(list(c.keys()) + ["nope"])
        if block == "nope":
            c[rng.choice(["nope", "extra"])] = rng.choice(weird)
        elif isinstance(c[block], dict) and c[block] and rng.random() < 0.8:
            key = rng.choice(list(c[block].keys()) + ["bogus"])
            c[block][key] = rng.choice(weird)
        elif rng.random() < 0.3:
            del c[block]
        else:
            c[block] = rng.choice(weird)
    return c


@pytest.mark.skipif(not R.available(), reason="oracle/_ref not built (no /root/reference)")
def test_random_configs_against_live_reference():
    base = json.loads(_cases()[2]["text"])  # the cfg2-shaped config
    rng = random.Random(2509)
    for _ in range(1500):
        text = json.dumps(_mutations(rng, base))
        check(text, R.ref_load_config(text))


def test_bench_workload_from_config_matches_cfg2():
    """configs/cfg2.json (reference schema + model/gpu blocks) drives bench.py
    --config with exactly the RunConfig of the built-in cfg2 workload."""
    import importlib.util
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    spec = importlib.util.spec_from_file_location("bench", os.path.join(root, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    wl = bench.workload_from_config(os.path.join(root, "configs", "cfg2.json"))
    a, b = bench.make_cfg(wl), bench.make_cfg(bench.WORKLOADS["cfg2"])
    assert bytes(a) == bytes(b)
    assert bytes(bench.make_cfg(wl, True)) == bytes(bench.make_cfg(bench.WORKLOADS["cfg2"], True))
    assert (wl["batch"], wl["chunk"], wl["delta"], wl["scorer_sms"]) == (256, 64, 26, 56)
