"""Time one rank shard's C4-like solve on this GPU (env: SH_WORLD, SH_RANK, SH_NITER; the library's
LT_* switches apply).  Prints ms per solve and a checksum of the cores."""
import os, sys
sys.path.insert(0, '.')
import torch
import synth
import paper_1604_02292_b200 as lt
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
inp = synth.make_inputs(cfg)
world, rank = int(os.environ.get("SH_WORLD", "1")), int(os.environ.get("SH_RANK", "0"))
n_iter = int(os.environ.get("SH_NITER", str(cfg.n_iter)))
plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter, rank=rank, world=world)
plan.filter_bank()
sino = torch.from_numpy(inp.sino).cuda()
solve = (lambda: plan.tv_solve(sino, cfg.lam, cfg.n_fgp)) if "tv" in cfg.solver else \
        (lambda: plan.sirt_solve(sino, 0.0, float("inf")))
c = solve(); torch.cuda.synchronize()
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
reps = int(os.environ.get("SH_REPS", "3"))
e0.record()
for _ in range(reps): c = solve()
e1.record(); torch.cuda.synchronize()
print(f"{cfg.name} w{world} r{rank} R={plan.R} n={n_iter}: "
      f"{e0.elapsed_time(e1) / reps:.2f} ms/solve  sum={float(c.double().sum()):.6f}", flush=True)
