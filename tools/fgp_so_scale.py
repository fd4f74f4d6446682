"""Time lt_fgp_batch of an alternative library build (argv[1], copied over the
in-tree .so in a scratch copy of the package) on H x 256 tiles (timing experiments)."""
import os, sys, shutil, tempfile
src = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tmp = tempfile.mkdtemp()
shutil.copytree(os.path.join(src, "paper_1604_02292_b200"), os.path.join(tmp, "paper_1604_02292_b200"))
if len(sys.argv) > 1:
    shutil.copy(sys.argv[1], os.path.join(tmp, "paper_1604_02292_b200", "_loctomo.so"))
sys.path.insert(0, tmp)
import torch
import paper_1604_02292_b200 as lt
for H in (32, 256):
    x = torch.rand(256 * 256 // H, H, 256, device='cuda')
    for _ in range(2): lt.fgp_batch(x, 0.05, 100)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(3): lt.fgp_batch(x, 0.05, 100)
    e1.record(); torch.cuda.synchronize()
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'in-tree'} H={H}: {e0.elapsed_time(e1)/3:.3f} ms")
