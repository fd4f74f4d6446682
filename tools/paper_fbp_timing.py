"""The paper's one timing of its local method (BASELINE.md
§1): a single filtered local backprojection FBP_L(p, u_n) of a 256 x 256 local
part of a 1024 x 1024 grid, 1024 (here 1025, odd for the filter centring)
detectors, 512 angles -- 28 ms per local reconstruction on a GTX TITAN Z with
ASTRA.  Here: the conv of every angle row with u_n (one filter of the bank,
lt_conv_cache computes all n) is timed separately from the ROI backprojection
W_L^T (lt_backproject on the 256 x 256 ROI)."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import synth
import paper_1604_02292_b200 as lt

n, na, nd, n_iter = 1024, 512, 1025, 200
ang = synth.angles_for(na)
cfg = synth.Config(90, "paper-fbp", n, na, np.pi, nd, "poisson", 1e4, 1, 128, 0, "centre", n_iter, "sirt", 0.0, 1, 8, 0)
inp = synth.make_inputs(cfg)
cen = np.array([[n // 2, n // 2]], dtype=np.int32)
plan = lt.Plan(n, ang, nd, cen, 128, 0, n_iter)
plan.filter_bank()
sino = torch.from_numpy(inp.sino).cuda()
pc = plan.disc_correct(sino)[0] if isinstance(plan.disc_correct(sino), tuple) else plan.disc_correct(sino)
def timeit(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
t_conv_all = timeit(lambda: plan.conv_cache(pc), 5)
t_bp = timeit(lambda: plan.backproject(sino, roi=0))
print(f"conv cache, all {n_iter} filters: {t_conv_all:.3f} ms (one filter ~{t_conv_all / n_iter * 1e3:.1f} us)")
print(f"ROI backprojection W_L^T (256 x 256, 512 angles): {t_bp * 1e3:.1f} us")
print(f"FBP_L(p, u_n) per local reconstruction ~ {t_bp + t_conv_all / n_iter:.3f} ms (paper: 28 ms on a GTX TITAN Z)")
