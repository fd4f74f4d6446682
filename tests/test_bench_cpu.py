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


def test_self_launch_spawns_world_ranks():
    """`bench.py --gpus N` without WORLD_SIZE re-executes itself under
    torch.distributed.run with N ranks (rendezvous at 127.0.0.1); checked with
    the gloo self-test: one JSON line from rank 0 with n_gpus = N."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--selftest"], cwd=ROOT, capture_output=True,
                       text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["rank_sum"] == 1.0 and line["master_addr"] == "127.0.0.1"


def test_reference_arm_under_two_ranks_prints_once():
    """The reference arm launched for N = 2: rank 0 alone runs the oracle and
    prints; the other rank exits 0 without work."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--impl", "reference", "--config", "C1",
                        "--steps", "1", "--warmup", "0"], cwd=ROOT, capture_output=True, text=True, timeout=600,
                       env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1 and json.loads(lines[0])["impl"] == "reference"


def test_executed_updates_count():
    """gray_s_executed: per iteration 2..n one A and one A^T per ROI, plus one
    x_s backprojection per 64 x 64 block the extended ROIs meet, every iteration."""
    import bench
    import synth
    cfg = synth.config("C4")
    rects = [(0, 0, 0, 256, 0, 256), (128, 128, 0, 256, 0, 256)]      # overlapping 4x4-block squares
    exe = bench.executed_updates(cfg, rects, 10)
    blocks = 16 + 16 - 4                                                 # their union: 28 blocks of 64 x 64
    assert exe == cfg.n_angles * (2.0 * 2 * 256 * 256 * 9 + blocks * 64 * 64 * 10)
