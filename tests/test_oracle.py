"""Pins the C restatement (oracle/oppo_oracle.c) before it is trusted as a checker:
against the golden vectors of the compiled reference and, where it is built
here, against the live reference (oracle/_ref)."""
import random

import pytest

from conftest import config_from_dict
from oracle import oracle as O
from paper_2509_25762_b200 import abi
from paper_2509_25762_b200 import scheduler as S


def test_oracle_rng_and_lengths_match_golden(golden):
    g = golden["rng"]
    assert [str(x) for x in O.rng_draws(1, "lengths", 8)] == g["lengths_u64"]
    assert O.rng_draws(1, "lengths", 9, "normal") == g["lengths_normal"]
    for case in golden["lengths"]:
        d = abi.LengthDist()
        d.kind = case["kind"]
        for k, v in case["params"].items():
            if k == "table":
                d.table_n = len(v)
                for i, (ln, w) in enumerate(v):
                    d.table_len[i], d.table_w[i] = ln, w
            else:
                setattr(d, k, v)
        assert O.sample_lengths(d, case["seed"], 200) == case["draws"]


def test_oracle_lockstep_steps_match_golden(golden):
    lat = abi.Latency(1, 0, 0, 0, 0, abi.PLACE_DISAGGREGATED, 1)
    for case in golden["lockstep_steps"]:
        arr = S.seq_array(case["states"])
        outs, led = O.run_step(arr, len(case["states"]), case["chunk"], case["mode"], lat,
                               case["stop_after"])
        assert [list(o.as_tuple()) for o in outs] == case["outcomes"]
        assert [led.wall, led.busy_generation, led.busy_scoring, led.work_generation,
                led.work_scoring] == case["ledger"]


def test_oracle_runs_match_golden(golden):
    for run in golden["runs"]:
        cfg = config_from_dict(run["config"])
        recs, sel = O.run_seed(cfg, run["seed"])
        assert [list(r) for r in recs] == [[r[1], r[2], r[3], r[4]] for r in run["records"]], run["name"]
        assert sel == run["selected"], run["name"]


def test_oracle_ppo_math_matches_golden(golden):
    for c in golden["gae"]:
        got = O.gae(c["rewards"], c["values"], c["gamma"], c["lambda"])
        assert got == c["adv"]  # same operation order: bit-identical
    for c in golden["clipped"]:
        offs = c["offsets"]
        adv = []
        for i in range(len(offs) - 1):
            T = offs[i + 1] - offs[i]
            r = [0.0] * T
            r[-1] = c["rewards"][i]
            adv += O.gae(r, c["values"][offs[i] + i:offs[i + 1] + i + 1], c["gamma"], c["lambda"])
        obj, _ = O.ppo_clip(c["new_lp"], c["old_lp"], adv, c["eps"])
        assert abs(obj - c["objective"]) <= 1e-12 * max(1, abs(c["objective"]))


def _rand_states(rng, n, chunk):
    out = []
    for i in range(n):
        L = rng.randint(1, 90)
        g = rng.choice([0, 0, rng.randint(0, L)])
        p = rng.randint(0, g) if g else 0
        out.append(dict(id=i * 5 + rng.randint(0, 4), prompt_len=rng.randint(1, 9), target_len=L,
                        generated=g, prefilled_tokens=p, chunks_emitted=(g + chunk - 1) // chunk,
                        chunks_prefilled=(p + chunk - 1) // chunk, scored=0))
    return out


def test_oracle_general_des_matches_live_reference(live_ref):
    """Every latency model (colocated/disaggregated, switch/transfer/residual costs)."""
    rng = random.Random(11)
    for trial in range(400):
        chunk = rng.choice([1, 2, 5, 16, 40])
        n = rng.randint(1, 10)
        states = _rand_states(rng, n, chunk)
        arr = S.seq_array(states)
        lat = abi.Latency(rng.randint(0, 6), rng.randint(0, 6), rng.randint(0, 20),
                          rng.randint(0, 9), rng.randint(0, 9), rng.choice([0, 1]),
                          rng.choice([0, 1]))
        mode = rng.choice([0, 1])
        stop = rng.choice([0, 1, rng.randint(1, n), n + 1])
        ro, rl = live_ref.run_step(arr, n, chunk, mode, lat, stop)
        oo, ol = O.run_step(arr, n, chunk, mode, lat, stop)
        assert [o.as_tuple() for o in oo] == [o.as_tuple() for o in ro], trial
        assert (ol.wall, ol.busy_generation, ol.busy_scoring, ol.work_generation,
                ol.work_scoring) == (rl.wall, rl.busy_generation, rl.busy_scoring,
                                     rl.work_generation, rl.work_scoring), trial


def test_token_granularity_product_matches_oracle():
    """north_star carry mode (no reference counterpart): the product's logical
    clock vs the oracle's credit_partial rule, step by step and over whole runs."""
    rng = random.Random(5)
    lat = abi.Latency(1, 0, 0, 0, 0, abi.PLACE_DISAGGREGATED, 1)
    for trial in range(300):
        chunk = rng.choice([1, 3, 8, 16, 64])
        n = rng.randint(1, 12)
        states = _rand_states(rng, n, chunk)
        mode = rng.choice([0, 1])
        stop = rng.randint(1, n)
        po, pl = S.plan_step(states, chunk, mode, stop, abi.CARRY_TOKEN)
        oo, ol = O.run_step(S.seq_array(states), n, chunk, mode, lat, stop, credit_partial=True)
        assert [o.as_tuple() for o in po] == [o.as_tuple() for o in oo], trial
        assert (pl.wall, pl.work_generation, pl.busy_generation) == \
               (ol.wall, ol.work_generation, ol.busy_generation), trial
    for trial in range(40):
        cfg = S.default_config(steps=8, batch_size=rng.randint(2, 32), prompt_len=4,
                               delta_init=3, delta_max=6, chunk_size=rng.choice([4, 16, 64]),
                               schedule_mode=rng.choice([0, 1]), carry_granularity=abi.CARRY_TOKEN,
                               latency_decode_per_token=1, latency_prefill_per_token=0,
                               latency_reward_residual=0, latency_placement=1,
                               lengths_kind=abi.LEN_LOGNORMAL, lengths_mu_log=4.0,
                               lengths_sigma_log=1.0, lengths_cap=512)
        recs, sel = S.run_seed_logical(cfg, trial)
        orecs, osel = O.run_seed(cfg, trial)
        assert [(r.wall_ticks, r.finished, r.deferred, r.delta) for r in recs] == orecs
        assert sel == osel
