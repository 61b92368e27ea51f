"""bench.py's reference arm on CPU (config A): one JSON line with the driver's
keys, and a config dict identical to the one the GPU arm prints for the same
workload (the driver compares the two arms' configs)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref")),
                    reason="oracle/_ref (the reference's compiled kernels) not built")
def test_reference_arm_line_and_config():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "A",
                          "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    sys.path.insert(0, ROOT)
    import bench
    coords, off, k, n_bins, scaling, _ = bench.workload("A", 0, 1)
    n, dd = coords.shape
    gpu_cfg = bench.config_keys("A", n, dd, k, n_bins, 1 if scaling == "weak" else 64, True)
    assert d["config"] == gpu_cfg
