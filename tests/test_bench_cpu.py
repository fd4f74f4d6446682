"""bench.py host logic on CPU: the reference arm's JSON line (the contract keys,
run as a subprocess on the smallest config) and the algorithmic counts the
metric divides by (N_theta P (1 + 3 (n - 1)) pixel-angle updates
per ROI, n n_FGP P FGP pixel-iterations)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "C1", "--steps", "1",
                        "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert "workload" in line["config"]


def test_algorithmic_counts():
    import bench
    import synth
    cfg = synth.config("C4")
    # two full 256 x 256 tiles and one clipped to 100 x 256 (rect rows: [.., .., r0, r1, c0, c1])
    rects = [(0, 0, 0, 256, 0, 256), (0, 0, 0, 256, 0, 256), (0, 0, 156, 256, 0, 256)]
    upd, fgp, ptot = bench.algorithmic_counts(cfg, rects, 200)
    P = 2 * 256 * 256 + 100 * 256
    assert ptot == P
    assert upd == cfg.n_angles * P * (1 + 3 * 199)
    assert fgp == P * 200 * cfg.n_fgp
    box = synth.config("C5")
    _, fgp_box, _ = bench.algorithmic_counts(box, rects, 500)
    assert fgp_box == 0.0
