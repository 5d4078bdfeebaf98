"""Run-output compatibility: steps_<seed>.csv, tuner_<seed>.csv
and summary.json written by paper_2509_25762_b200.outputs from this build's
step loop are identical to the reference's write_outputs (driver.cpp:248-350)
for the same configuration (lockstep latency model, where the two loops make
identical decisions), byte for byte for the CSVs and key for key for the
summary (task_fingerprint excepted: it hashes the reference's JSON config echo).
"""
import json

import pytest

from paper_2509_25762_b200 import abi, outputs
from paper_2509_25762_b200 import scheduler as S


def _cfg(tune):
    return S.default_config(
        mode=abi.RUN_SIMULATE, steps=40, batch_size=6, prompt_len=4, delta_init=3, delta_min=0,
        delta_max=6, controller=abi.DELTA_EQ4, window=3, chunk_size=8,
        schedule_mode=abi.MODE_STREAMED, tune_chunks=int(tune), chunk_candidates=[4, 8, 16],
        retune_period=10, lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=3.0,
        lengths_sigma_log=0.8, lengths_cap=64, latency_decode_per_token=1,
        latency_prefill_per_token=0, latency_reward_residual=0,
        latency_placement=abi.PLACE_DISAGGREGATED, proxy_kind=1, proxy_value=0.1,
        proxy_ramp_steps=20, proxy_ramp_scale=0.7)


@pytest.mark.parametrize("tune", [False, True])
def test_outputs_match_reference_writer(live_ref, tmp_path, tune):
    cfg = _cfg(tune)
    seeds = [1, 7]
    ref_dir, our_dir = tmp_path / "ref", tmp_path / "ours"
    live_ref.write_outputs(cfg, seeds, ref_dir)
    base = S.baseline(cfg)
    runs, bases = [], []
    for sd in seeds:
        recs, _ = S.run_seed_logical(cfg, sd)
        runs.append(dict(seed=sd, records=recs, complete=True, error=""))
        brecs, _ = S.run_seed_logical(base, sd)
        bases.append(dict(seed=sd, records=brecs, complete=True, error=""))
    outputs.write_outputs(cfg, runs, bases, our_dir)
    for sd in seeds:
        assert (our_dir / f"steps_{sd}.csv").read_text() == (ref_dir / f"steps_{sd}.csv").read_text()
        if tune:
            assert (our_dir / f"tuner_{sd}.csv").read_text() == (ref_dir / f"tuner_{sd}.csv").read_text()
    a = json.loads((our_dir / "summary.json").read_text())
    b = json.loads((ref_dir / "summary.json").read_text())
    a.pop("task_fingerprint")
    b.pop("task_fingerprint")
    assert list(a.keys()) == list(b.keys())
    assert _close(a, b)


def _close(a, b):
    if isinstance(a, dict):
        assert a.keys() == b.keys()
        return all(_close(a[k], b[k]) for k in a)
    if isinstance(a, list):
        assert len(a) == len(b)
        return all(_close(x, y) for x, y in zip(a, b))
    if isinstance(a, float) or isinstance(b, float):
        assert abs(a - b) <= 1e-12 * max(1.0, abs(b)), (a, b)
        return True
    assert a == b, (a, b)
    return True
