python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python -m pytest tests -m gpu -x -q -k "fgp or tv or C1 or fuzz or boundary" 2>&1 | tail -2
python - <<'PY'
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
import paper_1604_02292_b200 as lt
for h, w in ((40, 40), (64, 64), (33, 61)):
    x = torch.rand(32, h, w, device='cuda')
    lt.fgp_batch(x, 0.05, 100); torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(10): lt.fgp_batch(x, 0.05, 100)
    e1.record(); torch.cuda.synchronize()
    print(h, w, "fgp_batch 32 tiles x 100 it:", round(e0.elapsed_time(e1) / 10 * 1000, 1), "us")
PY
