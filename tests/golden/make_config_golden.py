"""Generates tests/golden/config_vectors.json from the COMPILED REFERENCE
(oracle/_ref/librlpipe_ref.so): for each JSON config text below, what
rlpipe::load_config_text accepts or rejects (the ConfigError message), the
config_echo of the parsed RunConfig and of its baseline(), and
RunConfig::task_fingerprint.  Run in the build container:
    python tests/golden/make_config_golden.py
(JSON config schema parity; checked by tests/test_config.py.)"""
import json
import os
import sys

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), "..", ".."))
sys.path.insert(0, ROOT)

from oracle import ref as R  # noqa: E402

OUT = os.path.join(os.path.dirname(__file__), "config_vectors.json")

CFG2 = {
    "mode": "train", "steps": 40, "seeds": [1, 2, 3], "out_dir": "runs/cfg2",
    "batch": {"size": 256, "prompt_len": 128},
    "delta": {"init": 26, "min": 0, "max": 64, "controller": "alg1", "window": 4, "inc": 2, "dec": 1},
    "chunk": {"size": 64, "mode": "streamed"},
    "latency": {"decode_per_token": 1, "prefill_per_token": 0, "reward_residual": 0,
                "placement": "disaggregated", "count_prompt_in_prefill": False},
    "lengths": {"kind": "lognormal", "mu_log": 5.0, "sigma_log": 1.0, "cap": 1024},
    "ppo": {"gamma": 1.0, "lambda": 0.95, "clip_epsilon": 0.2, "learning_rate": 0.001,
            "value_learning_rate": 0.0001, "vocab": 16, "target_token": 3, "reward_scale": 2.5,
            "reward_bias": -0.125},
}

CASES = [
    "{}",
    '{"preset": "paper"}',
    json.dumps(CFG2),
    json.dumps(dict(CFG2, mode="tune", chunk={"size": 32, "tune": True, "candidates": [16, 32, 64],
                                              "retune_period": 9})),
    '{"lengths": {"kind": "empirical", "cap": 512, "table": [[12, 0.5], [300, 2], [512, 1e-3]]}}',
    '{"lengths": {"kind": "two_point", "fast_len": 50, "slow_len": 900, "p_slow": 0.125, "cap": 1000}}',
    '{"sgd": {"dim": 3, "mu": 0.25, "lipschitz": 2.0, "eta": 0.4, "noise": "outward",'
    ' "eigenvalues": [0.25, 1.0, 2.0], "iterations": 123456789012}}',
    '{"reward_proxy": {"kind": "ramp", "value": 0.5, "ramp_scale": 3.0, "ramp_steps": 7},'
    ' "debug": {"fail_after_step": 5}}',
    # nlohmann get<T> coercions: float -> int (truncation), bool -> int, int -> double
    '{"steps": 2.7, "batch": {"size": true, "prompts": 1e3}, "ppo": {"gamma": 1, "clip_epsilon": 1}}',
    '{"seeds": [7, 18446744073709551615, 0], "latency": {"chunk_switch_cost": 3, "transfer_per_chunk": 2,'
    ' "placement": "colocated"}}',
    '{"ppo": {"learning_rate": 1e-05, "value_learning_rate": 1e-4, "reward_bias": 1e16,'
    ' "reward_scale": 123456.789}, "lengths": {"kind": "lognormal", "mu_log": -0.5, "sigma_log": 0.0}}',
    # schema errors (collected, one ConfigError)
    '{"stepz": 3, "batch": {"sizes": 1}, "delta": {"controller": "pid"}}',
    '{"steps": "ten", "mode": 3, "chunk": {"tune": 1}, "seeds": 5}',
    '{"schema_version": 2, "preset": "huge"}',
    '{"preset": 7, "lengths": {"table": [[1]]}}',
    '{"batch": 5, "delta": [1, 2], "chunk": null}',
    '{"out_dir": 3, "sgd": {"noise": "gaussian", "eigenvalues": "flat"}}',
    # validate() errors
    '{"delta": {"init": 5, "min": 4, "max": 2}}',
    '{"steps": 0, "seeds": [], "batch": {"size": 0, "prompt_len": 0}, "delta": {"window": 0, "inc": 0}}',
    '{"chunk": {"size": 0, "retune_period": 0}}',
    '{"chunk": {"tune": true, "candidates": [], "retune_period": 1}}',
    '{"chunk": {"tune": true, "candidates": [8, 0, 16], "retune_period": 2}}',
    '{"ppo": {"vocab": 20, "target_token": 25}}',
    '{"ppo": {"vocab": 4, "target_token": -1, "gamma": 1.5}}',
    '{"latency": {"decode_per_token": -1}}',
    '{"lengths": {"cap": 0}}',
    '{"lengths": {"kind": "two_point", "fast_len": 0}}',
    '{"lengths": {"kind": "two_point", "slow_len": 5000}}',
    '{"lengths": {"kind": "two_point", "p_slow": 1.5}}',
    '{"lengths": {"kind": "lognormal", "sigma_log": -1}}',
    '{"lengths": {"kind": "empirical"}}',
    '{"lengths": {"kind": "empirical", "cap": 10, "table": [[11, 1.0]]}}',
    '{"lengths": {"kind": "empirical", "table": [[10, -1.0]]}}',
    '{"lengths": {"kind": "empirical", "table": [[10, 0.0]]}}',
    '{"ppo": {"lambda": -0.1}}',
    '{"ppo": {"clip_epsilon": 0}}',
    '{"ppo": {"learning_rate": 0}}',
    '{"ppo": {"value_learning_rate": -1}}',
    '{"sgd": {"dim": 0}}',
    '{"sgd": {"mu": 2.0}}',
    '{"sgd": {"eta": 0.95}}',
    '{"sgd": {"d_max": -1}}',
    '{"sgd": {"iterations": -5}}',
    '{"sgd": {"initial_distance_sq": 0}}',
    '{"sgd": {"dim": 2, "eigenvalues": [0.5]}}',
    '{"sgd": {"dim": 2, "eigenvalues": [0.5, 3.0]}}',
    '{"delta": {"min": -1, "max": -2, "init": -1}, "ppo": {"gamma": -1}, "lengths": {"cap": -3}}',
    # not JSON / not an object
    "[1, 2]",
    "{x",
    '"config"',
]


def main():
    vecs = []
    for text in CASES:
        r = R.ref_load_config(text)
        vecs.append(dict(text=text, **r))
    with open(OUT, "w") as f:
        json.dump({"source": "oracle/_ref/librlpipe_ref.so (rlpipe::load_config_text, config_echo, "
                             "RunConfig::task_fingerprint, RunConfig::baseline)",
                   "cases": vecs}, f, indent=1)
        f.write("\n")
    print(f"{len(vecs)} cases -> {OUT}")


if __name__ == "__main__":
    main()
