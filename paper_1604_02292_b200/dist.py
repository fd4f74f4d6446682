"""Multi-GPU combine plumbing: ROIs are partitioned by
``lt_roi_setup(rank, world)``; each rank solves its ROIs, the cores are
all-gathered into fixed slots (the largest local count of any rank, ROI-index
ordered within a rank) and every rank stitches the same image with ``lt_stitch_slots``
(ascending global ROI order => bitwise identical for every world size).
``Plan.combine_rois`` + ``NcclComm`` do the same inside the library
(lt_combine_rois: its own NCCL communicator and in-place all-gather).

torch.distributed provides the collective (NCCL on GPUs; gloo works for the
CPU tests of this host logic).  No arithmetic of the method lives here.
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np
import torch


def slots_per_rank(local_lists: Sequence[Sequence[int]]) -> int:
    """Slots per rank of the all-gather: the largest local ROI count (the
    cost-balanced partition gives cheap clipped ROIs to some ranks, so counts differ)."""
    return max(1, max(len(lst) for lst in local_lists))


def slot_table(local_lists: Sequence[Sequence[int]], slots_per_rank: int) -> np.ndarray:
    """Global ROI index of every gathered slot (-1 = empty)."""
    world = len(local_lists)
    out = np.full(world * slots_per_rank, -1, dtype=np.int32)
    for g, lst in enumerate(local_lists):
        if len(lst) > slots_per_rank:
            raise ValueError(f"rank {g} holds {len(lst)} ROIs > {slots_per_rank} slots")
        out[g * slots_per_rank:g * slots_per_rank + len(lst)] = np.asarray(lst, dtype=np.int32)
    return out


def exchange_local_lists(local_rois: Sequence[int], group=None) -> List[List[int]]:
    import torch.distributed as dist
    world = dist.get_world_size(group)
    lists: List = [None] * world
    dist.all_gather_object(lists, [int(v) for v in local_rois], group=group)
    return lists


def gather_cores(cores_slots: torch.Tensor, group=None, out: torch.Tensor = None) -> torch.Tensor:
    """All-gather this rank's padded slot block [slots_per_rank, side, side]
    into [world * slots_per_rank, side, side] (rank-major)."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if out is None:
        out = torch.empty((world * cores_slots.shape[0],) + tuple(cores_slots.shape[1:]),
                          dtype=cores_slots.dtype, device=cores_slots.device)
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, cores_slots.contiguous(), group=group)
    else:
        parts = list(out.chunk(world, dim=0))
        dist.all_gather(parts, cores_slots.contiguous(), group=group)
    return out


def setup_combine(plan, group=None) -> Tuple[int, np.ndarray]:
    """(slots_per_rank, slot -> global ROI table) for a plan of this rank: the
    ranks' local lists are exchanged and must equal the partition the library
    computed on every rank (lt_plan_slot_table)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    lists = exchange_local_lists(plan.local_rois, group) if world > 1 else [list(plan.local_rois)]
    spr = slots_per_rank(lists)
    table = slot_table(lists, spr)
    if getattr(plan, "world", world) == world:
        spr_lib, table_lib = plan.slot_table()
        if spr_lib != spr or not np.array_equal(table_lib, table):
            raise RuntimeError("exchanged ROI lists differ from the library's partition")
    return spr, table


def angle_range(n_angles: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous angle rows [a0, a1) of one rank for the angle-split bank."""
    return rank * n_angles // world, (rank + 1) * n_angles // world


def filter_bank_split(plan, group=None, reduce=None, gather=None) -> None:
    """Cold filter bank on all ranks by angle split:
    each rank projects / backprojects its angle rows (lt_bank_split_step), the
    per-step partial images are all-reduced (NCCL / gloo: the only exchange),
    the sum is applied in the kernels (lt_bank_split_apply), and finally every
    rank's bank rows are all-gathered and installed with lt_set_bank.
    ``reduce(t)`` / ``gather(rows) -> list`` override the collectives (tests)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if reduce is None:
        reduce = (lambda t: dist.all_reduce(t, group=group)) if world > 1 else (lambda t: None)
    na, n, nd, nit = plan.n_angles, plan.n, plan.n_det, plan.n_iter
    a0, a1 = angle_range(na, rank, world)
    plan.bank_split_begin(a0, a1)
    part = torch.empty(n * n, dtype=torch.float32, device=plan.device)
    for k in range(nit):
        last = k + 1 == nit
        plan.bank_split_step(k, None if last else part)
        if not last:
            reduce(part)
            plan.bank_split_apply(part)
    bank = plan.get_bank()
    mine = bank[:, a0:a1, :].contiguous()
    if gather is None and world == 1:
        rows = [mine]
    elif gather is None:
        # equal-size slots (the largest share), then each rank's rows cut out
        sizes = [angle_range(na, g, world) for g in range(world)]
        cap = max(b - a for a, b in sizes)
        slot = torch.zeros((nit, cap, nd), dtype=torch.float32, device=plan.device)
        slot[:, :a1 - a0] = mine
        slots = [torch.empty_like(slot) for _ in range(world)]
        dist.all_gather(slots, slot, group=group)
        rows = [slots[g][:, :b - a] for g, (a, b) in enumerate(sizes)]
    else:
        rows = gather(mine)
    plan.set_bank(torch.cat(rows, dim=1).contiguous(), key=plan.bank_key)


def global_sirt_split(plan, sino: torch.Tensor, n_iter: int, lo: float = 0.0, hi: float = float("inf"),
                      group=None, reduce=None) -> torch.Tensor:
    """GLOBAL box-SIRT on all ranks by angle split: per iteration
    each rank forms its residual rows and partial backprojection
    (lt_global_split_step), the N x N partials are all-reduced, and the clamped
    update is applied in a kernel (lt_global_split_apply).  Every rank ends with
    the same image.  ``reduce(t)`` overrides the all-reduce (tests)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if reduce is None:
        reduce = (lambda t: dist.all_reduce(t, group=group)) if world > 1 else (lambda t: None)
    a0, a1 = angle_range(plan.n_angles, rank, world)
    plan.global_split_begin(a0, a1)
    part = torch.empty(plan.n * plan.n, dtype=torch.float32, device=plan.device)
    for _ in range(n_iter):
        plan.global_split_step(sino, part)
        reduce(part)
        plan.global_split_apply(part, lo, hi)
    return plan.global_split_result()


class PeerCombine:
    """Combine over NVLink peer memory (lt_combine_peers): every rank's core
    buffer [slots_per_rank, 2r, 2r] is mapped into every other rank with CUDA
    IPC once; each combine then reads the peers' cores in place inside the
    stitch kernel (no all-gather copy).  Ordering: the solves of all ranks
    complete before any stitch (stream sync + barrier), and every stitch
    completes before any rank overwrites its buffer (sync + barrier again)."""

    def __init__(self, plan, cores: torch.Tensor, slot_roi: np.ndarray, spr: int, group=None):
        import torch.distributed as dist
        import paper_1604_02292_b200 as lt
        self.plan, self.cores, self.slot_roi, self.spr, self.group = plan, cores, slot_roi, spr, group
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self._opened = []
        if self.world == 1:
            self.ptrs = [cores.data_ptr()]
            return
        # the IPC handle names the whole cudaMalloc segment of torch's caching
        # allocator: torch reports the storage's offset inside it (_share_cuda_);
        # add the tensor's offset inside the storage.  Every step that can fail
        # is followed by a collective agreement, so either every rank uses the
        # peer path or every rank raises (and the caller falls back together).
        try:
            seg_off = int(cores.untyped_storage()._share_cuda_()[3])
            info = (lt.ipc_handle(cores), seg_off + cores.storage_offset() * cores.element_size())
        except Exception:
            info = None
        infos: List = [None] * self.world
        dist.all_gather_object(infos, info, group=group)
        if any(i is None for i in infos):
            raise RuntimeError("CUDA IPC handle unavailable on some rank")
        self.ptrs = []
        ok = True
        for g, i in enumerate(infos):
            if g == self.rank:
                self.ptrs.append(cores.data_ptr())
                continue
            try:
                p = lt.ipc_open(i[0])
                self._opened.append(p)
                self.ptrs.append(p + i[1])
            except Exception:
                ok = False
                break
        flags: List = [None] * self.world
        dist.all_gather_object(flags, ok, group=group)
        if not all(flags):
            self.close()
            raise RuntimeError("CUDA IPC mapping failed on some rank")

    def combine(self, out: torch.Tensor) -> torch.Tensor:
        import torch.distributed as dist
        if self.world > 1:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)
        self.plan.combine_peers(self.ptrs, self.spr, self.slot_roi, out=out)
        if self.world > 1:
            torch.cuda.current_stream().synchronize()
            dist.barrier(group=self.group)
        return out

    def close(self):
        import paper_1604_02292_b200 as lt
        for p in self._opened:
            lt.ipc_close(p)
        self._opened = []
