"""Small solves that exercise every kernel family and launch shape, for
compute-sanitizer (memcheck / racecheck / synccheck), VERDICT r01 item 7.

  C1  one 40^2 ROI: SIRT + TV (16-row FGP clusters), project / backproject, combine
  C2  16 seeded 128^2 ROIs: TV (32-row 4-CTA clusters), Haar prior, combine, metrics
  T1  one 256^2 ROI of a 1024^2 / 512-angle geometry: truncated-data padding, the
      band-split forward projector + k_fp_join, the angle-split backprojector
      (stage 1 / 2 partials), 16-CTA FGP clusters
  P   64 ROIs of the C4 geometry (256^2 tiles): the persistent 8-CTA FGP with
      cp.async prefetch of the next tile and mbarrier re-initialisation per tile
Usage: python tools/sanitize_cases.py C1|C2|T1|P
"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1604_02292_b200 as lt  # noqa: E402


def main(case):
    torch.cuda.set_device(0)
    if case in ("C1", "C2"):
        cfg = synth.config(case)
        inp = synth.make_inputs(case)
        plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 3)
        plan.filter_bank()
        sino = torch.from_numpy(inp.sino).cuda()
        c1 = plan.sirt_solve(sino, 0.0, math.inf)
        c2 = plan.tv_solve(sino, 0.05, 5)
        plan.combine(c2, plan.local_rois)
        plan.combine_rois(c2)
        if case == "C1":
            x = torch.rand(cfg.n, cfg.n, device="cuda")
            plan.project(x, roi=0); plan.backproject(sino, roi=0); plan.project(x); plan.backproject(sino)
            lt.fgp_batch(torch.rand(3, 37, 53, device="cuda"), 0.1, 7)
        else:
            plan.haar_solve(sino, 0.02, 4)
            lt.metrics(c1, c2)
        print(case, "ok", float(c2.abs().sum()))
    elif case == "T1":
        cfg = synth.config("T1")
        inp = synth.make_inputs("T1")
        plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, 2)
        plan.filter_bank()
        sino = lt.pad_truncated(torch.from_numpy(inp.sino_trunc).cuda(), cfg.n_det)
        c = plan.tv_solve(sino, 0.05, 4)
        plan.sirt_solve(sino, 0.0, math.inf)
        print(case, "ok", float(c.abs().sum()))
    elif case == "P":
        cfg = synth.config("C4")
        inp = synth.make_inputs("C4")
        cen = inp.centres[np.arange(0, 256, 4)]
        plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, cen, cfg.radius, cfg.margin, 2)
        plan.filter_bank()
        c = plan.tv_solve(torch.from_numpy(inp.sino).cuda(), 0.05, 3)
        print(case, "ok", float(c.abs().sum()))
    torch.cuda.synchronize()


if __name__ == "__main__":
    main(sys.argv[1])
