"""Measured max relL2 of GPU ROI cores vs the fp64 oracle per config (the
numbers behind BASELINE.md §4's parity column): C1 and C2 as configured (every
ROI), C3 (6 seeded ROIs, SIRT and TV, as configured), C4 and C5 in bench.py's
full-batch launch configuration with n = 3 (8 / 6 sampled ROIs)."""
import math, sys
sys.path.insert(0, '.')
import numpy as np
import torch
import synth, oracle
import paper_1604_02292_b200 as lt

def relerr(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))

def run(name, n_iter=None, sample=None, modes=None):
    cfg = synth.config(name); inp = synth.make_inputs(name)
    n_iter = n_iter or cfg.n_iter
    modes = modes or (["tv"] if "tv" in cfg.solver else ["box"])
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
    plan.filter_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    idx = np.arange(len(inp.centres)) if sample is None else np.asarray(sample)
    out = []
    for mode in modes:
        got = (plan.tv_solve(sino, cfg.lam, cfg.n_fgp) if mode == "tv" else plan.sirt_solve(sino, 0.0, math.inf)).cpu().numpy()
        ref = oracle.pipeline(inp.sino.astype(np.float64), inp.angles, cfg.n, inp.centres[idx], cfg.radius, cfg.margin,
                              n_iter, mode=mode, lam=cfg.lam, n_fgp=cfg.n_fgp)
        errs = [relerr(got[int(np.nonzero(plan.local_rois == g)[0][0])], ref[k]) for k, g in enumerate(idx)]
        out.append(f"{mode} max relL2 {max(errs):.2e} over {len(idx)} ROIs, n = {n_iter}")
    print(name, "; ".join(out), flush=True)

oracle.build()
run("C1")
run("C2")
run("C3", sample=np.arange(6), modes=["box", "tv"])
run("C4", n_iter=3, sample=[0, 15, 240, 255, 7, 100, 136, 200])
run("C5", n_iter=3, sample=[0, 31, 992, 1023, 500, 529])
