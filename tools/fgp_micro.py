"""Microbenchmark: FGP batch on C4-shaped tiles (256 x 256x256, 100 iterations)."""
import sys, os, shutil, importlib
sys.path.insert(0, '.')
import torch
so = sys.argv[1] if len(sys.argv) > 1 else None
if so:
    shutil.copy(so, 'paper_1604_02292_b200/_loctomo.so')
import paper_1604_02292_b200 as lt
x = torch.rand(256, 256, 256, device='cuda')
for _ in range(2): lt.fgp_batch(x, 0.05, 100)
torch.cuda.synchronize()
e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
e0.record()
for _ in range(5): y = lt.fgp_batch(x, 0.05, 100)
e1.record(); torch.cuda.synchronize()
print(so, "fgp 256x256^2 x100 it: %.3f ms" % (e0.elapsed_time(e1) / 5))
import numpy as np, oracle
ref = oracle.fgp(x[3].double().cpu().numpy(), 0.05, 100)
print("relerr", np.linalg.norm(y[3].double().cpu().numpy() - ref) / np.linalg.norm(ref))
