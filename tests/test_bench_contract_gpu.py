"""bench.py's output contract on the GPU (the driver parses it): one JSON line with the keys
the task fixes, a positive throughput, the roofline object for the headline kernel and the
clocks record, from a short run without sub-records or CPU baseline."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_json_line():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "1", "--warmup", "3",
                          "--no-sub", "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    b = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "clocks", "roofline"):
        assert k in b, k
    assert b["value"] > 0 and b["n_gpus"] == 1 and b["steps"] == 1 and b["warmup"] == 3
    assert b["config"]["workload"].startswith("cfg5")
    assert b["gpu_launches"] > 0
    r = b["roofline"]
    assert r["bound"] in ("hbm", "tensor", "alu") and 0 < r["frac"] <= 1.5 and r["peak"] > 0
    e = b["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
