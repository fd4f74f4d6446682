"""Combine over peer memory (lt_combine_peers): the stitch kernel
reading every rank's core buffer in place equals the all-gather + stitch path
bitwise -- in one process with several local buffers standing in for the
ranks, and across two processes on one GPU through real CUDA IPC handles."""
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


def _setup(lt, world):
    cfg = synth.config("C2")
    cen = synth.roi_centres(cfg)
    lists = []
    for r in range(world):
        plan = lt.Plan(cfg.n, synth.angles_for(8), cfg.n_det, cen, cfg.radius, cfg.margin, 1, rank=r, world=world,
                       bind=False)
        lists.append(list(plan.local_rois))
    from paper_1604_02292_b200 import dist as ltd
    spr = ltd.slots_per_rank(lists)
    table = ltd.slot_table(lists, spr)
    side = 2 * cfg.radius
    rng = np.random.default_rng(7)
    cores = [torch.from_numpy(rng.random((spr, side, side)).astype(np.float32)).cuda() for _ in range(world)]
    return cfg, cen, spr, table, cores


@pytest.mark.parametrize("world", [1, 3])
def test_peer_combine_equals_gather_combine(lt, world):
    cfg, cen, spr, table, cores = _setup(lt, world)
    plan = lt.Plan(cfg.n, synth.angles_for(8), cfg.n_det, cen, cfg.radius, cfg.margin, 1, rank=0, world=world)
    ref = plan.combine(torch.cat(cores), table)
    got = plan.combine_peers([c.data_ptr() for c in cores], spr, table)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)


def _free_port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    return port


def _ipc_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as lt
    from paper_1604_02292_b200 import dist as ltd
    torch.cuda.set_device(0)
    cfg, cen, spr, table, cores = _setup(lt, world)
    plan = lt.Plan(cfg.n, synth.angles_for(8), cfg.n_det, cen, cfg.radius, cfg.margin, 1, rank=rank, world=world)
    mine = cores[rank].clone()                    # this rank's buffer (same content on both sides)
    pc = ltd.PeerCombine(plan, mine, table, spr)
    img = pc.combine(torch.empty(cfg.n, cfg.n, device="cuda"))
    ref = plan.combine(torch.cat(cores), table)
    torch.cuda.synchronize()
    q.put((rank, bool(torch.equal(img, ref))))
    dist.barrier()
    pc.close()
    dist.destroy_process_group()


def test_peer_combine_two_processes_ipc():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs: p.start()
    res = dict(q.get(timeout=120) for _ in range(2))
    for p in procs: p.join(timeout=60)
    assert res == {0: True, 1: True}
