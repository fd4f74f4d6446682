"""Host-side cost of one C4 solve call (launch returns vs device completion):
the e2e number syncs every step, so host launch latency is exposed there."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
import synth
import paper_1604_02292_b200 as lt
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
inp = synth.make_inputs(cfg)
plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
plan.filter_bank()
sino = torch.from_numpy(inp.sino).cuda()
for _ in range(2):
    plan.tv_solve(sino, cfg.lam, cfg.n_fgp)
torch.cuda.synchronize()
for _ in range(3):
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    t0 = time.perf_counter(); e0.record()
    plan.tv_solve(sino, cfg.lam, cfg.n_fgp)
    t1 = time.perf_counter(); e1.record()
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"host launch {1e3*(t1-t0):.2f} ms, wall {1e3*(t2-t0):.2f} ms, device {e0.elapsed_time(e1):.2f} ms")
