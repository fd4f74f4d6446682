"""CUDA-graph replay of the local iteration loop: identical results to the
eager launches (LT_GRAPH=0 in a subprocess) and the C1 solve time either way."""
import math, os, subprocess, sys
sys.path.insert(0, '.')
import numpy as np, torch
import synth
import paper_1604_02292_b200 as lt
inp = synth.make_inputs("C1")
s = torch.from_numpy(inp.sino).cuda()
plan = lt.Plan(64, inp.angles, 91, inp.centres, 12, 8, 100)
plan.filter_bank()
outs = []
for mode in ("sirt", "tv"):
    f = (lambda: plan.sirt_solve(s, 0.0, math.inf)) if mode == "sirt" else (lambda: plan.tv_solve(s, 0.05, 100))
    a = f().clone(); b = f().clone()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(True); e1 = torch.cuda.Event(True)
    e0.record()
    for _ in range(10): f()
    e1.record(); torch.cuda.synchronize()
    print(f"{mode}: graph={os.environ.get('LT_GRAPH', '1')} {e0.elapsed_time(e1) / 10:.3f} ms per C1 solve; "
          f"replay == first: {bool(torch.equal(a, b))}")
    outs.append(b.cpu().numpy())
np.save(f"gpurun_out/graph_{os.environ.get('LT_GRAPH', '1')}.npy", np.stack(outs))
