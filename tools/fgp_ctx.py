"""FGP in context vs standalone: per-launch FGP time inside a C4 tv_solve
(LT_SPLIT=1 -> one stream, no overlap) vs lt_fgp_batch on random and on the
solve's own v data, and on denormal-scaled data."""
import os, sys
os.environ.setdefault("LT_SPLIT", "1")
sys.path.insert(0, '.')
import torch
import synth
import paper_1604_02292_b200 as lt
cfg = synth.config("C4")
inp = synth.make_inputs(cfg, noise=True)
n_iter = 6
plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter)
plan.filter_bank()
sino = torch.from_numpy(inp.sino).cuda()
plan.tv_solve(sino, cfg.lam, cfg.n_fgp)
torch.cuda.synchronize()
lt.timing_enable(True)
plan.tv_solve(sino, cfg.lam, cfg.n_fgp)
torch.cuda.synchronize()
t = lt.timing_read()
lt.timing_enable(False)
print("in solve:", {k: (round(v[0] / max(v[1], 1), 3), v[1]) for k, v in t.items()})
def bench(x, tag):
    for _ in range(2): lt.fgp_batch(x, cfg.lam, cfg.n_fgp)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(3): lt.fgp_batch(x, cfg.lam, cfg.n_fgp)
    e1.record(); torch.cuda.synchronize()
    print(f"fgp_batch {tag}: {e0.elapsed_time(e1)/3:.3f} ms for {x.shape[0]} tiles")
x = torch.rand(plan.R, 256, 256, device='cuda')
bench(x, "rand")
bench(x[:128].contiguous(), "rand 128")
bench(x * 1e-36, "rand*1e-36 (denormal range)")
v = plan.get_ext()
print("ext stats", float(v.abs().max()), float(v.abs().mean()))
bench(v.contiguous(), "solve output")
