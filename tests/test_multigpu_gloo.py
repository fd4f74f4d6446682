"""World-size-2 gloo tests of the multi-GPU host logic (-m "not gpu"):
LPT partition + slot table + all-gather layout reproduce the single-process
combine exactly (the stitch here is the oracle's, fed through the gathered
slot layout; the device stitch kernel is covered by the GPU parity tests)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _fake_core(g, side):
    # deterministic core content for global ROI g (any function of g works)
    ii, jj = np.meshgrid(np.arange(side), np.arange(side), indexing="ij")
    return (np.sin(0.37 * g + 0.11 * ii) + 0.01 * jj + g).astype(np.float32)


def _worker(rank, world, port, cfg_name, result_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as lt
    from paper_1604_02292_b200 import dist as ltd
    cfg = synth.config(cfg_name)
    cen = synth.roi_centres(cfg)
    plan = lt.Plan(cfg.n, synth.angles_for(8), cfg.n_det, cen, cfg.radius, cfg.margin, 1,
                   rank=rank, world=world, bind=False)
    spr, table = ltd.setup_combine(plan)
    side = 2 * cfg.radius
    block = torch.zeros(spr, side, side)
    for q, g in enumerate(plan.local_rois):
        block[q] = torch.from_numpy(_fake_core(int(g), side))
    gathered = ltd.gather_cores(block)
    if rank == 0:
        result_q.put((table, gathered.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("cfg_name", ["C2", "C4"])
def test_gloo_world2_gather_and_combine(orc, cfg_name):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg_name, q)) for r in range(world)]
    for p in procs:
        p.start()
    table, gathered = q.get(timeout=300)
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    cfg = synth.config(cfg_name)
    cen = synth.roi_centres(cfg)
    side = 2 * cfg.radius
    # every ROI exactly once
    used = table[table >= 0]
    assert sorted(used.tolist()) == list(range(len(cen)))
    # gathered slots carry the right cores
    for s, g in enumerate(table):
        if g >= 0:
            assert np.array_equal(gathered[s], _fake_core(int(g), side))
    # combine through the slot layout == single-process combine
    order = np.argsort(used, kind="stable")
    cores_by_roi = gathered[np.nonzero(table >= 0)[0][order]].astype(np.float64)
    ref_cores = np.stack([_fake_core(g, side) for g in range(len(cen))]).astype(np.float64)
    assert np.array_equal(cores_by_roi, ref_cores)
    img = orc.stitch(cfg.n, cen, cfg.radius, cores_by_roi)
    assert np.array_equal(img, orc.stitch(cfg.n, cen, cfg.radius, ref_cores))


def test_slot_table_and_partition_balance():
    from paper_1604_02292_b200 import dist as ltd
    import paper_1604_02292_b200 as lt
    cfg = synth.config("C5")
    cen = synth.roi_centres(cfg)
    for world in (2, 4, 8):
        lists = []
        for r in range(world):
            plan = lt.Plan(cfg.n, synth.angles_for(4), cfg.n_det, cen, cfg.radius, cfg.margin, 1,
                           rank=r, world=world, bind=False)
            lists.append(list(plan.local_rois))
        spr = ltd.slots_per_rank(lists)
        t = ltd.slot_table(lists, spr)
        assert sorted(t[t >= 0].tolist()) == list(range(len(cen)))
        assert max(len(l) for l in lists) <= spr


@pytest.mark.parametrize("na", [1, 7, 64, 180, 256])
def test_angle_split_ranges_partition(na):
    """The angle-split bank's rank ranges are contiguous, disjoint, cover
    [0, N_theta) and differ in size by at most one."""
    from paper_1604_02292_b200.dist import angle_range
    for world in range(1, 9):
        rs = [angle_range(na, g, world) for g in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == na
        assert all(rs[g][1] == rs[g + 1][0] for g in range(world - 1))
        sizes = [b - a for a, b in rs]
        assert max(sizes) - min(sizes) <= 1
