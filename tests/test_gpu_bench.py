"""bench.py's JSON contract on the GPU (small config, few steps): the keys the
driver reads, a native library actually loaded, roofline / e2e / cpu_baseline
present and the reference arm on the same config object."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _line(args):
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                         text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-3000:]
    return json.loads([ln for ln in res.stdout.splitlines() if ln.startswith("{")][-1])


def test_bench_line_contract():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    d = _line(["--config", "1", "--steps", "3", "--warmup", "3"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "clocks", "gpu_launches", "e2e",
              "roofline", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] >= 3 and d["value"] > 0
    assert d["gpu_launches"] >= 3  # one persistent launch per cfg1 solve
    assert set(d["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert set(d["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert 0 < d["roofline"]["frac"] < 1.5
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["run"]["tolerance_converged"] and d["run"]["tolerance_iterations"] == 40
    ref = _line(["--impl", "reference", "--config", "1", "--steps", "1", "--warmup", "0"])
    assert ref["impl"] == "reference" and ref["config"] == d["config"]
    assert ref["e2e"]["h2d_bytes_per_step"] == 0 and ref["cpu_baseline"]["value"] == ref["value"]
