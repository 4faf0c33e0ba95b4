"""bench.py plumbing on CPU: the --gpus N self-launch and the shared config object."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_bench_gpus_flag_launches_that_many_ranks():
    """`python bench.py --gpus 2` (no torchrun) re-launches itself as 2 ranks
    and the ranks agree on the world size (gloo, 127.0.0.1)."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing"],
                         capture_output=True, text=True, timeout=240, env=env)
    assert res.returncode == 0, res.stderr[-2000:]
    line = [ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1]
    out = json.loads(line)
    assert out["n_gpus"] == 2 and out["gpus_arg"] == 2 and out["rank_sum"] == 1.0


def test_bench_refuses_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="1", RANK="0")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing"],
                         capture_output=True, text=True, timeout=120, env=env)
    assert res.returncode != 0 and "WORLD_SIZE=1" in (res.stderr + res.stdout)


def test_both_arms_share_the_config_object():
    import bench
    from paper_2201_12324_b200 import workloads
    wl = workloads.cfg4(n=512, m=256)
    cfg = bench.workload_config(wl)
    assert cfg == bench.workload_config(wl)
    assert "parallelism" not in cfg and cfg["workload"].startswith("cfg4")
    saved = sys.argv
    sys.argv = ["bench.py"]
    try:
        args = bench.parse()
    finally:
        sys.argv = saved
    assert args.config == 4 and args.gpus == 1  # headline: the largest single-GPU config
