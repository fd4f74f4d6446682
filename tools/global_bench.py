"""Time the GLOBAL solvers (a10 and NEXT-4(iii)) on a config's full grid:
box-SIRT, FISTA-TV (FGP prox) and Chambolle-Pock TV, n iterations each."""
import math, sys
sys.path.insert(0, '.')
import torch
import synth
import paper_1604_02292_b200 as lt
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C2")
nit = int(sys.argv[2]) if len(sys.argv) > 2 else 50
inp = synth.make_inputs(cfg)
plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres[:1], cfg.radius, cfg.margin, 2)
s = torch.from_numpy(inp.sino).cuda()
mu = cfg.lam * cfg.n_angles * cfg.n_det
def t(f):
    f(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record(); f(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
print(f"{cfg.name} global, {nit} iterations: box-SIRT {t(lambda: plan.global_sirt(s, nit, 0.0, math.inf)):.1f} ms, "
      f"FISTA-TV {t(lambda: plan.global_tv(s, nit, cfg.lam, cfg.n_fgp)):.1f} ms, "
      f"Chambolle-Pock {t(lambda: plan.global_cp(s, nit, mu)):.1f} ms")
