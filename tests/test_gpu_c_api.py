"""The C-ABI from plain C (-m gpu): examples/c_api_demo.c is compiled with gcc
against include/loctomo.h and the in-tree library (no Python in the path),
runs a C2-shaped local nonneg SIRT on a sinogram file and writes the combined
image; it must equal the Python binding's solve + combine bitwise (same
library, same launches) and the oracle's stitched cores to 1e-3."""
import math
import os
import subprocess

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_api_demo(tmp_path, orc):
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as lt
    exe = str(tmp_path / "c_api_demo")
    so = os.path.join(ROOT, "paper_1604_02292_b200", "_loctomo.so")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(ROOT, "examples", "c_api_demo.c"), so, "-L", "/usr/local/cuda/lib64",
                           "-lcudart", "-Wl,-rpath,/usr/local/cuda/lib64",
                           "-Wl,-rpath," + os.path.dirname(so), "-o", exe, "-lm"])
    cfg = synth.config("C2")
    inp = synth.make_inputs("C2")
    n_iter = 12
    sino_f = tmp_path / "sino.f32"
    img_f = tmp_path / "image.f32"
    inp.sino.astype(np.float32).tofile(sino_f)
    args = [exe, str(cfg.n), str(cfg.n_angles), str(cfg.n_det), str(cfg.radius), str(cfg.margin), str(n_iter),
            str(sino_f), str(img_f)] + [str(int(v)) for v in inp.centres.reshape(-1)]
    r = subprocess.run(args, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    assert "kernels launched" in r.stdout
    img_c = np.fromfile(img_f, dtype=np.float32).reshape(cfg.n, cfg.n)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
    plan.filter_bank()
    cores = plan.sirt_solve(torch.from_numpy(inp.sino).cuda(), 0.0, math.inf)
    img_py = plan.combine_rois(cores).cpu().numpy()
    assert np.array_equal(img_c, img_py)
    ref = orc.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, inp.centres, cfg.radius, cfg.margin,
                       n_iter, mode="box")
    ref_img = orc.stitch(cfg.n, inp.centres, cfg.radius, ref)
    assert float(np.linalg.norm(img_c - ref_img) / np.linalg.norm(ref_img)) <= 1e-3
