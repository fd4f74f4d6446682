"""FGP time vs cluster size: same pixel count (256 x 256^2), tiles of H x 256
(H = 32..256), so the effect of the cross-CTA (DSMEM) chain is isolated."""
import os, sys
sys.path.insert(0, '.')
import torch
import paper_1604_02292_b200 as lt
tag = f"cfg={os.environ.get('LT_FGP2_CFG', '-')}"
for H in (32, 64, 128, 256):
    x = torch.rand(256 * 256 // H, H, 256, device='cuda')
    for _ in range(2): lt.fgp_batch(x, 0.05, 100)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(3): lt.fgp_batch(x, 0.05, 100)
    e1.record(); torch.cuda.synchronize()
    print(f"{tag} H={H:4d} tiles={x.shape[0]:5d}: {e0.elapsed_time(e1)/3:.3f} ms")
