"""bench.py contract checks that need no GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_reference_arm_never_maps_liboppo():
    """--impl reference times the reference's own CPU path (oracle/_ref) and
    must not load the product library (its RunConfig comes from the reference)."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    code = ("import sys, runpy; sys.argv=['bench.py','--impl','reference','--steps','1','--warmup','0'];"
            "runpy.run_path('bench.py', run_name='__main__');"
            "m=open('/proc/self/maps').read(); print('MAPPED', 'liboppo.so' in m, 'librlpipe_ref' in m)")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=300, env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.strip().splitlines()
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert lines[-1] == "MAPPED False True"


def test_reference_default_config_matches_product_default():
    """The reference-built RunConfig{} equals liboppo's oppo_run_config_default
    (the two arms run the same workload definition)."""
    from oracle import ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built")
    from paper_2509_25762_b200 import scheduler as S
    a, b = R.default_config(batch_size=256, chunk_size=64), S.default_config(batch_size=256, chunk_size=64)
    assert bytes(a) == bytes(b)
    assert bytes(R.baseline_config(a)) == bytes(S.baseline(b))


def test_gpus_flag_spawns_one_rank_per_gpu():
    """`bench.py --gpus N` outside torchrun launches N ranks itself with the
    torchrun environment (127.0.0.1 rendezvous); rank 0 reports n_gpus=N and
    global_batch=N*B."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "3", "--dry-run-ranks"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300,
                         env={k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")})
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["n_gpus"] == 3 and line["global_batch"] == 3 * 256
    assert sorted(tuple(r) for r in line["ranks"]) == [(0, 0), (1, 1), (2, 2)]
