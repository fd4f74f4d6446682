"""The N > 1 path of bench.py on a one-GPU box (-m gpu): `--gpus 2` self-launches
two ranks (torch.distributed.run, 127.0.0.1), LT_BENCH_FUNCTIONAL=1 puts both on
cuda:0 with gloo, and the run must partition the ROIs, build the slot tables,
combine through the peer-memory stitch (CUDA IPC between the two processes) or
the all-gather, reduce the timings over ranks and print ONE line with n_gpus 2.
A functional check of the multi-rank code only: its timings are not measurements."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("combine", ["peer", "nccl"])
def test_bench_two_ranks_functional(combine):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    env["LT_BENCH_FUNCTIONAL"] = "1"
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "1",
                        "--no-cpu-baseline", "--config", "C1", "--combine", combine],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["gpu_launches"] > 0
    assert ("peer" in line["combine"]) == (combine == "peer")
