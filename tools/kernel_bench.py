"""Per-kernel timing inside a C4 solve on one stream (LT_SPLIT=1), CUDA events
per launch class (lt_timing)."""
import os, sys
os.environ.setdefault("LT_SPLIT", "1")
sys.path.insert(0, '.')
import torch
import synth
import paper_1604_02292_b200 as lt
cfg = synth.config(sys.argv[1] if len(sys.argv) > 1 else "C4")
inp = synth.make_inputs(cfg, noise=True)
n_iter = int(os.environ.get('KB_NITER', '6'))
plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter,
               rank=int(os.environ.get('KB_RANK', '0')), world=int(os.environ.get('KB_WORLD', '1')))
plan.filter_bank()
sino = torch.from_numpy(inp.sino).cuda()
plan.tv_solve(sino, cfg.lam, cfg.n_fgp)
torch.cuda.synchronize()
lt.timing_enable(True)
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
e0.record()
cores = plan.tv_solve(sino, cfg.lam, cfg.n_fgp)
e1.record()
torch.cuda.synchronize()
t = lt.timing_read()
lt.timing_enable(False)
print(f"solve {n_iter} it: {e0.elapsed_time(e1):.2f} ms;", {k: (round(v[0] / max(v[1], 1), 3), v[1]) for k, v in t.items()})
os.makedirs("/tmp/lt_ab", exist_ok=True)
torch.save(cores.cpu(), f"/tmp/lt_ab/cores_{os.environ.get('TAG', 'x')}.pt")
