"""Quick timing probe of the C4 workload phases (not the bench contract)."""
import sys, time, math
import numpy as np, torch
sys.path.insert(0, '.')
import synth
import paper_1604_02292_b200 as lt

cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
n_iter = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.n_iter
inp = synth.make_inputs(cfg, noise=True)
plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
sino = torch.from_numpy(inp.sino).cuda()
def t(f):
    torch.cuda.synchronize(); e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record(); f(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
print("bank ms", t(plan.filter_bank))
print("bank ms (2nd)", t(plan.filter_bank))
pc, c = plan.disc_correct(sino)
print("disc ms", t(lambda: plan.disc_correct(sino)))
print("conv ms", t(lambda: plan.conv_cache(pc)))
if "tv" in cfg.solver:
    print("tv solve ms", t(lambda: plan.tv_solve(sino, cfg.lam, cfg.n_fgp)))
print("sirt solve ms", t(lambda: plan.sirt_solve(sino, 0.0, math.inf)))
img = torch.rand(cfg.n, cfg.n, device='cuda')
print("global FP ms", t(lambda: plan.project(img)))
s = plan.project(img)
print("global BP ms", t(lambda: plan.backproject(s)))
x = torch.rand(plan.R, 2*plan.h, 2*plan.h, device='cuda')
print("fgp batch ms", t(lambda: lt.fgp_batch(x, 0.05, 100)))
