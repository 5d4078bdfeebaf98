"""Run outputs in the reference's formats, so the reference's
``compare_runs`` (driver.cpp:418-452) can read GPU runs:

* ``steps_<seed>.csv``  — columns and number formats of write_steps_csv
  (driver.cpp:248-263);
* ``tuner_<seed>.csv``  — write_tuner_csv (driver.cpp:265-272), rows rebuilt
  from the step records by replaying the tuner (chunking.cpp:73-100);
* ``summary.json``      — the keys of write_outputs (driver.cpp:276-350), in the
  same order, aggregates as finalize_aggregates (driver.cpp:34-60).

For GPU runs ``wall_ticks`` is the logical-clock wall of the step (the
reference's unit); the measured device time is written to a side column file
``steps_<seed>_us.csv`` so the reference CSV stays byte-compatible.
"""
import json
import os

from . import abi
from . import scheduler as S


def _g9(x):
    return "%.9g" % x


def steps_csv(records):
    out = ["step,wall_ticks,finished,deferred,delta,controller_stat,mean_reward,"
           "util_generation,util_scoring,max_deferrals"]
    for r in records:
        stat = _g9(r.controller_stat) if r.has_controller_stat else ""
        out.append(f"{r.step},{r.wall_ticks},{r.finished},{r.deferred},{r.delta},{stat},"
                   f"{_g9(r.mean_reward)},{r.util_generation:.6f},{r.util_scoring:.6f},"
                   f"{r.max_deferrals}")
    return "\n".join(out) + "\n"


def tuner_rows(cfg, records, measure="wall"):
    """(step, candidate, measurement, chosen) for every exploration step."""
    cands = [cfg.chunk_candidates[i] for i in range(cfg.n_candidates)]
    if not cands:
        return []
    order = sorted(set(cands))  # make_tuner dedupes the candidates (chunking.cpp:61-71)
    meas, steps = [], []
    for r in records:
        slot = r.step % cfg.retune_period
        if slot < len(order):  # exploration step (chunking.cpp:102-107)
            m = float(r.wall_ticks) if measure == "wall" else float(r.step_us)
            meas.append((r.chunk_size, m))
            steps.append(r.step)
    chosen = S.tuner_replay(order, cfg.retune_period, meas)
    return [(s, c, m, ch) for s, (c, m), ch in zip(steps, meas, chosen)]


def tuner_csv(rows):
    out = ["step,candidate,mean_ticks,chosen"]
    out += [f"{s},{c},{_g9(m)},{ch}" for s, c, m, ch in rows]
    return "\n".join(out) + "\n"


def _aggregates(records):
    a = dict(total_wall_ticks=0, mean_step_ticks=0.0, final_reward=0.0, mean_util_generation=0.0,
             mean_util_scoring=0.0, delta_final=0, delta_mean=0.0, delta_lo=0, delta_hi=0)
    if not records:
        return a
    n = len(records)
    a["total_wall_ticks"] = sum(r.wall_ticks for r in records)
    a["mean_step_ticks"] = a["total_wall_ticks"] / n
    a["mean_util_generation"] = sum(r.util_generation for r in records) / n
    a["mean_util_scoring"] = sum(r.util_scoring for r in records) / n
    a["delta_mean"] = sum(r.delta for r in records) / n
    a["delta_lo"] = min(r.delta for r in records)
    a["delta_hi"] = max(r.delta for r in records)
    a["delta_final"] = records[-1].delta
    tail = max(1, n // 10)
    a["final_reward"] = sum(r.mean_reward for r in records[n - tail:]) / tail
    return a


def summary(cfg, runs, baselines, fingerprint=""):
    """runs / baselines: lists of dict(seed, records, complete, error)."""
    mode = {abi.RUN_SIMULATE: "simulate", abi.RUN_TRAIN: "train"}.get(cfg.mode, "tune")
    ag = [_aggregates(r["records"]) for r in runs]
    bg = [_aggregates(b["records"]) for b in baselines]
    complete = all(r["complete"] for r in runs)
    error = ""
    for r in runs:
        if not r["complete"]:
            error = r["error"]
    n = len(runs)
    speed = 1.0
    if n and len(bg) == n:
        if all(a["mean_step_ticks"] > 0 for a in ag):
            speed = sum(b["mean_step_ticks"] / a["mean_step_ticks"] for a, b in zip(ag, bg)) / n
    d = {"schema_version": 1, "mode": mode, "task_fingerprint": fingerprint,
         "seeds": [r["seed"] for r in runs], "steps_requested": cfg.steps, "complete": complete,
         "error": error,
         "final_reward": sum(a["final_reward"] for a in ag) / n if n else 0.0,
         "mean_step_ticks": sum(a["mean_step_ticks"] for a in ag) / n if n else 0.0,
         "speedup_vs_baseline": speed}
    ug = sum(a["mean_util_generation"] for a in ag) / n if n else 0.0
    us = sum(a["mean_util_scoring"] for a in ag) / n if n else 0.0
    d["utilization"] = {"generation": ug, "scoring": us}
    d["delta_stats"] = {"initial": cfg.delta_init,
                        "min": min((a["delta_lo"] for a in ag), default=0),
                        "max": max((a["delta_hi"] for a in ag), default=0),
                        "mean": sum(a["delta_mean"] for a in ag) / n if n else 0.0,
                        "final": ag[-1]["delta_final"] if ag else 0}
    per = []
    for i, (r, a) in enumerate(zip(runs, ag)):
        row = {"seed": r["seed"], "complete": r["complete"], "steps_recorded": len(r["records"]),
               "final_reward": a["final_reward"], "mean_step_ticks": a["mean_step_ticks"],
               "total_wall_ticks": a["total_wall_ticks"], "mean_util_generation": a["mean_util_generation"],
               "mean_util_scoring": a["mean_util_scoring"]}
        row["speedup_vs_baseline"] = (bg[i]["mean_step_ticks"] / a["mean_step_ticks"]
                                      if i < len(bg) and a["mean_step_ticks"] > 0 else 1.0)
        per.append(row)
    d["per_seed"] = per
    return d


def write_outputs(cfg, runs, baselines, out_dir, fingerprint=""):
    """write_outputs (driver.cpp:276-350) for runs produced by this package."""
    os.makedirs(out_dir, exist_ok=True)
    tune = cfg.mode == abi.RUN_TUNE or cfg.tune_chunks
    for r in runs:
        with open(os.path.join(out_dir, f"steps_{r['seed']}.csv"), "w") as f:
            f.write(steps_csv(r["records"]))
        if any(x.step_us > 0 for x in r["records"]):
            with open(os.path.join(out_dir, f"steps_{r['seed']}_us.csv"), "w") as f:
                f.write("step,step_us,update_us,chunk_size\n")
                for x in r["records"]:
                    f.write(f"{x.step},{x.step_us:.3f},{x.update_us:.3f},{x.chunk_size}\n")
        if tune:
            with open(os.path.join(out_dir, f"tuner_{r['seed']}.csv"), "w") as f:
                f.write(tuner_csv(tuner_rows(cfg, r["records"])))
    with open(os.path.join(out_dir, "summary.json"), "w") as f:
        f.write(json.dumps(summary(cfg, runs, baselines, fingerprint), indent=2) + "\n")
