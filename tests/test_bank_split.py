"""Angle-split filter bank (SURVEY §8(e) "cold bank", Alg. 1 P:L489-503 with W
split by angle rows): G ranks each project / backproject their angles, the
partial images are summed (the all-reduce) and applied, and the gathered rows
equal the single-rank bank up to fp32 summation order -- in one process with
G plans standing in for the ranks (G = 2, 3), and across two processes on one
GPU with a real gloo all-reduce and all-gather through dist.filter_bank_split."""
import math
import os
import socket

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lt():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as m
    return m


def _plan(lt, n_iter=12):
    cfg = synth.config("C2")
    inp = synth.make_inputs("C2")
    return cfg, inp, lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres[:2], cfg.radius, cfg.margin, n_iter)


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.mark.parametrize("world", [2, 3])
def test_bank_split_in_one_process(lt, world):
    from paper_1604_02292_b200 import dist as ltd
    cfg, inp, ref_plan = _plan(lt)
    ref_plan.filter_bank()
    ref = ref_plan.get_bank().cpu().numpy()
    plans = [_plan(lt)[2] for _ in range(world)]
    na, n, nit = ref_plan.n_angles, ref_plan.n, ref_plan.n_iter
    ranges = [ltd.angle_range(na, g, world) for g in range(world)]
    for p, (a0, a1) in zip(plans, ranges):
        p.bank_split_begin(a0, a1)
    parts = [torch.empty(n * n, device="cuda") for _ in range(world)]
    for k in range(nit):
        last = k + 1 == nit
        for p, t in zip(plans, parts):
            p.bank_split_step(k, None if last else t)
        if not last:
            red = torch.stack(parts).sum(0)          # the all-reduce (test harness)
            for p in plans:
                p.bank_split_apply(red)
    rows = [p.get_bank()[:, a0:a1] for p, (a0, a1) in zip(plans, ranges)]
    got = torch.cat(rows, dim=1).cpu().numpy()
    assert got.shape == ref.shape
    assert relerr(got, ref) <= 1e-5
    for k in (0, nit // 2, nit - 1):
        assert relerr(got[k], ref[k]) <= 1e-5, k
    # the installed split bank drives a solve exactly like the single-rank one
    plans[0].set_bank(torch.from_numpy(got).cuda())
    sino = torch.from_numpy(inp.sino).cuda()
    a = plans[0].sirt_solve(sino, 0.0, math.inf).cpu().numpy()
    b = ref_plan.sirt_solve(sino, 0.0, math.inf).cpu().numpy()
    assert relerr(a, b) <= 1e-5


def test_bank_split_rejects(lt):
    _, _, p = _plan(lt)
    with pytest.raises(Exception):
        p.bank_split_step(0, torch.empty(p.n * p.n, device="cuda"))      # begin not called
    with pytest.raises(Exception):
        p.bank_split_begin(5, 5)
    with pytest.raises(Exception):
        p.bank_split_begin(0, p.n_angles + 1)


def _free_port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as lt
    from paper_1604_02292_b200 import dist as ltd
    torch.cuda.set_device(0)
    _, _, plan = _plan(lt)
    # gloo moves host tensors: the all-reduce / all-gather go through pinned copies
    def reduce(t):
        h = t.cpu(); dist.all_reduce(h); t.copy_(h)
    def gather(mine):
        sizes = [ltd.angle_range(plan.n_angles, g, world) for g in range(world)]
        cap = max(b - a for a, b in sizes)
        slot = torch.zeros((mine.shape[0], cap, mine.shape[2]))
        slot[:, :mine.shape[1]] = mine.cpu()
        slots = [torch.empty_like(slot) for _ in range(world)]
        dist.all_gather(slots, slot)
        return [slots[g][:, :b - a].cuda() for g, (a, b) in enumerate(sizes)]
    ltd.filter_bank_split(plan, reduce=reduce, gather=gather)
    got = plan.get_bank().cpu().numpy()
    _, _, ref_plan = _plan(lt)
    ref_plan.filter_bank()
    ref = ref_plan.get_bank().cpu().numpy()
    q.put((rank, relerr(got, ref)))
    dist.barrier()
    dist.destroy_process_group()


def test_bank_split_two_processes():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs: p.start()
    res = dict(q.get(timeout=180) for _ in range(2))
    for p in procs: p.join(timeout=60)
    assert set(res) == {0, 1}
    assert max(res.values()) <= 1e-5, res


@pytest.mark.parametrize("world,lo,hi", [(2, 0.0, math.inf), (3, -math.inf, math.inf), (4, 0.0, 0.02)])
def test_global_sirt_split_in_one_process(lt, world, lo, hi):
    """Angle-split GLOBAL box-SIRT: G plans standing
    in for the ranks, partials summed by the harness, equals lt_global_sirt."""
    cfg, inp, ref_plan = _plan(lt)
    sino = torch.from_numpy(inp.sino).cuda()
    n_iter = 8
    ref = ref_plan.global_sirt(sino, n_iter, lo, hi).cpu().numpy()
    from paper_1604_02292_b200 import dist as ltd
    plans = [_plan(lt)[2] for _ in range(world)]
    n = ref_plan.n
    for g, p in enumerate(plans):
        p.global_split_begin(*ltd.angle_range(p.n_angles, g, world))
    parts = [torch.empty(n * n, device="cuda") for _ in range(world)]
    for _ in range(n_iter):
        for p, t in zip(plans, parts):
            p.global_split_step(sino, t)
        red = torch.stack(parts).sum(0)
        for p in plans:
            p.global_split_apply(red, lo, hi)
    outs = [p.global_split_result().cpu().numpy() for p in plans]
    for o in outs:
        assert relerr(o, ref) <= 1e-5
        assert np.array_equal(o, outs[0])              # every rank holds the same image
    if lo == 0.0:
        assert outs[0].min() >= 0.0


def test_global_sirt_split_single_rank_helper(lt):
    """dist.global_sirt_split without a process group (world 1) = lt_global_sirt."""
    from paper_1604_02292_b200 import dist as ltd
    cfg, inp, plan = _plan(lt)
    sino = torch.from_numpy(inp.sino).cuda()
    a = ltd.global_sirt_split(plan, sino, 5).cpu().numpy()
    b = plan.global_sirt(sino, 5).cpu().numpy()
    assert relerr(a, b) <= 1e-6
