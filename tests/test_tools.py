"""The measurement tools around the hot path.

* CPU: the performance model (paper Eqs. 12-15, NEXT-4) re-instantiated from
  the committed round-2 probe and measurement files reproduces its table: the
  per-kernel costs of the iteration as built and the 8-GPU projections.
* GPU: `bench.py` prints ONE JSON line carrying every key of the bench contract
  (metric, value, roofline, cpu_baseline, e2e, clocks, gpu_launches, ...).
"""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MDIR = os.path.join(ROOT, "profiles", "r02_model")


def test_perf_model_reinstantiates(tmp_path):
    out = tmp_path / "model.md"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "perf_model.py"), "model",
                        os.path.join(MDIR, "probe.json"), MDIR, str(out)],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    text = out.read_text()
    # the iteration as built in round 2: operator + p update 88 B, update + x 57 B per point
    assert "Ax+p (116, 88.0)" in text and "cg_update+x (10, 57.0)" in text
    rows = {}
    for line in text.splitlines():
        cells = [c.strip() for c in line.strip().strip("|").split("|")]
        if len(cells) >= 5 and cells[0] == "8":
            rows.setdefault("8", []).append(cells)
    # weak C2, strong C3, strong C4: one 8-GPU row each
    assert len(rows["8"]) == 3
    c4_cal_eff = float(rows["8"][2][4])
    assert 0.8 <= c4_cal_eff <= 1.0   # calibrated C4 projection at 8 GPUs (DESIGN 7.2: 0.958)


@pytest.mark.gpu
def test_bench_contract_line():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", "5", "--warmup",
                        "3", "--no-c3"], capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "cpu_baseline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 5 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["higher_is_better"] is True and d["scaling"] == "weak"
    rf = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in rf, k
    assert rf["bound"] == "hbm" and 0.3 < rf["frac"] < 1.2
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] > 0 and cb["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0 and "sm_mhz" in d["clocks"]
    assert d["config"]["workload"].startswith("C2")
