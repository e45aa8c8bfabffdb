"""bench.py on CPU: the reference arm (the driver runs it at round end) prints
one JSON line with the contract's keys; the GPU arm's host helpers."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "t8", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "s" and d["higher_is_better"] is False
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] == 1
    assert d["e2e"] == {"value": d["value"], "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert d["gmres"]["converged"] is True
    for k in ("metric", "n_gpus", "steps", "warmup", "ms_per_step", "scaling", "vs_baseline", "dtype", "data",
              "config"):
        assert k in d


def test_phase_rooflines_helper():
    sys.path.insert(0, ROOT)
    import bench
    from types import SimpleNamespace as NS
    tim = {"sample_entries": 1e6, "sample_ms": 1.0, "pivot_lu_visits": 2e6, "pivot_lu_ms": 2.0,
           "dense_front_ms": 1.0}
    recs = [NS(path="dense", n_pivot=10, front_size=30), NS(path="structured", n_pivot=100, front_size=200)]
    r = bench.phase_rooflines(tim, recs, 6000.0, 30.0, 0.5, 1e9)
    assert abs(r["sample"]["achieved"] - 16.0) < 1e-9        # 16 MB in 1 ms = 16 GB/s
    assert abs(r["pivot_lu"]["achieved"] - 8.0) < 1e-9       # 16 MB in 2 ms
    dense = (2 / 3) * 1000 + 2 * 100 * 20 + 2 * 10 * 400
    assert abs(r["dense_front"]["achieved"] - dense / 1e-3 / 1e12) < 1e-15
    assert abs(r["apply"]["achieved"] - 2000.0) < 1e-9
