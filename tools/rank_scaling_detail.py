"""Strong-scaling projection on one GPU: for world = 1, 2, 4, 8 time every
rank's share of the C4 batch (Plan(rank, world): its ROIs, its x_s blocks)
as a solve on this GPU; the slowest rank bounds the N-GPU step (the combine
over NVLink is not included).  Projected ROI solves/s = R / max_rank(t)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import synth
import paper_1604_02292_b200 as lt
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
worlds = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
inp = synth.make_inputs(cfg)
sino = torch.from_numpy(inp.sino).cuda()
bank = None
for world in worlds:
    times = []
    for rank in range(world):
        plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter,
                       rank=rank, world=world)
        if bank is None:
            plan.filter_bank(); bank = plan.get_bank()
        else:
            plan.set_bank(bank)
        solve = (lambda: plan.tv_solve(sino, cfg.lam, cfg.n_fgp)) if "tv" in cfg.solver else \
                (lambda: plan.sirt_solve(sino, 0.0, float("inf")))
        solve(); torch.cuda.synchronize()
        e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
        e0.record()
        for _ in range(2): solve()
        e1.record(); torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 2)
        del plan
    t = max(times)
    print("  ranks ms", [round(v, 1) for v in times]); print(f"{cfg.name} world={world}: rank step ms min {min(times):.1f} max {t:.1f} -> projected "
          f"{cfg.n_roi / (t / 1e3):.1f} ROI solves/s ({cfg.n_roi / (t / 1e3) / world:.1f} per GPU)", flush=True)
