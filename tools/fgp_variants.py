"""FGP kernel variants: time on C4-shaped tiles (256 x 256^2, 100 iterations)
and check against the fp64 oracle on full and clipped tile shapes.
Run once per variant (the library reads LT_FGP2_CFG once)."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1604_02292_b200 as lt
import oracle
tag = f"cfg={os.environ.get('LT_FGP2_CFG', '-')}"
torch.manual_seed(0)
x = torch.rand(256, 256, 256, device='cuda')
for _ in range(2): lt.fgp_batch(x, 0.05, 100)
torch.cuda.synchronize()
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
e0.record()
for _ in range(5): y = lt.fgp_batch(x, 0.05, 100)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"{tag}: fgp 256 x 256^2 x 100 it: {ms:.3f} ms = {256*65536*100/ms/1e6:.1f} Gpix-it/s")
errs = []
for (h, w) in [(256, 256), (192, 256), (256, 192), (200, 177), (40, 40), (128, 128), (33, 250)]:
    xs = torch.rand(3, h, w, device='cuda') * 2 - 0.5
    ys = lt.fgp_batch(xs, 0.07, 37)
    for t in range(3):
        ref = oracle.fgp(xs[t].double().cpu().numpy(), 0.07, 37)
        errs.append(np.linalg.norm(ys[t].double().cpu().numpy() - ref) / np.linalg.norm(ref))
print(f"{tag}: max relerr vs oracle over shapes = {max(errs):.3e}")
