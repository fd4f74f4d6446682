"""FGP latency on a few 256x256 tiles (single-ROI workloads: T1): time per
100 FGP iterations with the default launch shape and with LT_FGP2_CFG."""
import os, sys
sys.path.insert(0, '.')
import torch
import paper_1604_02292_b200 as lt
tag = os.environ.get('LT_FGP2_CFG', 'auto')
for nt in (1, 2, 4, 7, 8, 12, 15, 16):
    x = torch.rand(nt, 256, 256, device='cuda')
    for _ in range(3): lt.fgp_batch(x, 0.05, 100)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(10): lt.fgp_batch(x, 0.05, 100)
    e1.record(); torch.cuda.synchronize()
    print(f"cfg={tag} tiles={nt}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us per 100 FGP iterations")
