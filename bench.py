#!/usr/bin/env python
"""Benchmark of the local-tomography hot path (BASELINE.json metric).

Step = one pass of the whole hot path over one synthetic C4 batch:
disc pre-correction (a2) + convolution cache (a4) + n = 200 local FISTA-TV
iterations on every ROI (a5-a8: Joseph FP, fused two-sinogram BP + update,
cluster FGP + momentum) + crop (a9) + combine into one N x N image (a9/e:
NCCL all-gather of the cores when N > 1, stitch kernel).  The filter bank
(a3, Alg. 1) depends only on the geometry and is computed once before the
timed region ("subsequent applications"); its time is
reported as bank_ms.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C4]
Multi-GPU: one rank per GPU, either launched by torchrun (WORLD_SIZE set) or,
for `--gpus N` without WORLD_SIZE, by this script itself (it re-executes
under torch.distributed.run with N local ranks and rendezvous at 127.0.0.1);
ROIs are partitioned across ranks (strong scaling of one image), timing = max
over ranks, one JSON line from rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import platform
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "ROI solves/sec and A+A^T Gray/s (ray-pixel updates/s) vs HBM roofline, 1–8 GPU"
UNIT = "ROI solves/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--prior", default="config", choices=["config", "haar", "exterior"],
                    help="haar: NEXT-2 Haar-wavelet l1 prior (FISTA, 4 levels, lambda 0.02) instead of the config's; "
                         "exterior: NEXT-4(ii) exterior-subtraction box-SIRT (the prior art) for comparison")
    ap.add_argument("--combine", default="peer", choices=["peer", "nccl", "library"],
                    help="N > 1: stitch reading the peers' cores over NVLink (CUDA IPC, one kernel), torch's NCCL "
                         "all-gather + stitch, or the library-owned lt_combine_rois (its own NCCL communicator)")
    ap.add_argument("--bank", default="local", choices=["local", "split"],
                    help="N > 1: every rank computes the whole filter bank (no communication), or the "
                         "angle-split cold bank (rank g owns N_theta/N angles, NCCL all-reduce of the N x N "
                         "partial image per Alg. 1 step, all-gather of the bank rows); reported as bank_ms")
    ap.add_argument("--xs-exact", action="store_true",
                    help="NEXT-4(i): x_s^k from the global SIRT iterate instead of the filtered backprojection")
    ap.add_argument("--selftest", action="store_true",
                    help="launcher self-test (no GPU): every rank joins a gloo group, rank 0 prints the world size")
    return ap.parse_args()


def free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args) -> int:
    """`--gpus N` without WORLD_SIZE: run this script under torch.distributed.run
    with N local ranks (one per GPU), rendezvous at 127.0.0.1; rank 0 prints
    the JSON line, the launcher returns the ranks' exit status."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", str(max(1, (os.cpu_count() or 1)))))
    return subprocess.run(cmd, env=env).returncode


def selftest():
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo")
    world, rank = dist.get_world_size(), dist.get_rank()
    t = torch.tensor([float(rank)])
    dist.all_reduce(t)
    if rank == 0:
        print(json.dumps({"selftest": True, "n_gpus": world, "rank_sum": float(t.item()),
                          "master_addr": os.environ.get("MASTER_ADDR")}), flush=True)
    dist.destroy_process_group()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return d, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback"


MICRO_PEAKS = os.path.join("profiles", "r02", "peaks_micro.json")


def sm_peaks():
    """Measured SM-side ceilings (tools/peaks_micro.cu run on a B200, committed
    under profiles/): shared-memory crossbar bytes/s of a conflict-free LDS.64
    stream and FP32 FMA flops/s, over all SMs.  None when not measured."""
    try:
        with open(os.path.join(ROOT, MICRO_PEAKS)) as f:
            return json.load(f)
    except Exception:
        return None


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        time.sleep(0.1)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[2 + k].lower() == "active"})
        loaded = [s for s in sm if s > 0.5 * max(sm)] if sm else []
        return {"sm_mhz": statistics.median(loaded) if loaded else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows)}


# --------------------------------------------------------------------------- work counts
def algorithmic_counts(cfg, plan_rects, n_iter):
    """Pixel-angle updates of one step (A+A^T Gray), FGP pixel-iterations."""
    P = [(r[3] - r[2]) * (r[5] - r[4]) for r in plan_rects]
    Ptot = float(sum(P))
    # iteration 1: y = 0 -> one A^T (of b_1); iterations 2..n: A y, A^T b_k, A^T s
    updates = cfg.n_angles * Ptot * (1 + 3 * (n_iter - 1))
    fgp_px_it = Ptot * n_iter * cfg.n_fgp if "tv" in cfg.solver else 0.0
    return updates, fgp_px_it, Ptot


def executed_updates(cfg, plan_rects, n_iter, block=64):
    """Pixel-angle updates the kernels actually execute in one step: per
    iteration 2..n one W_{L'} y and one W_{L'}^T s per ROI (valid pixels), and
    per iteration 1..n ONE global x_s backprojection over the 64 x 64 image
    blocks the extended ROIs meet (shared by overlapping ROIs)."""
    P = float(sum((r[3] - r[2]) * (r[5] - r[4]) for r in plan_rects))
    nb = (cfg.n + block - 1) // block
    need = np.zeros((nb, nb), dtype=bool)
    for row0, col0, vr0, vr1, vc0, vc1 in plan_rects:
        r0, r1, c0, c1 = row0 + vr0, row0 + vr1, col0 + vc0, col0 + vc1
        need[r0 // block:(r1 - 1) // block + 1, c0 // block:(c1 - 1) // block + 1] = True
    xs_pix = 0.0
    for by, bx in zip(*np.nonzero(need)):
        xs_pix += (min(cfg.n, (by + 1) * block) - by * block) * (min(cfg.n, (bx + 1) * block) - bx * block)
    return cfg.n_angles * (2.0 * P * (n_iter - 1) + xs_pix * n_iter)


# FP32 operations per unit, DESIGN.md §Roofline (counted from the formulas, not the SASS)
FGP_FLOPS_PER_PX_IT = 21.0      # z (5) + two dual steps with clip (10) + momentum (6)
JOSEPH_FLOPS_PER_UPDATE = 8.0   # hat weight (2 FMA-equivalents) + 2 taps x FMA, per pixel-angle
FP_SMEM_BYTES_PER_STEP = 8.0    # forward projector: one staged (S, D) fp32 pair read per ray-line step


HAAR_LAM, HAAR_LEVELS = 0.02, 4


def solve_mode(cfg, args) -> str:
    if args.prior in ("haar", "exterior"):
        return args.prior
    return "tv" if "tv" in cfg.solver else "sirt"


def config_dict(cfg, args, world: int) -> dict:
    """The workload description both arms print (same metric, unit, config)."""
    mode = solve_mode(cfg, args)
    sweep = cfg.layout == "sweep"
    return {"workload": f"{cfg.name}: {cfg.n}x{cfg.n}, {cfg.n_angles} angles, {cfg.n_det} det, "
                        f"{cfg.n_roi} ROIs r={cfg.radius} m={cfg.margin}, {mode}, n={cfg.n_iter}"
                        + (f", lambda={cfg.lam}, n_fgp={cfg.n_fgp}" if mode == "tv" and not sweep
                           else f", n_fgp={cfg.n_fgp}" if mode == "tv" else "")
                        + (f", Haar l1 lambda={HAAR_LAM}, levels={HAAR_LEVELS}, FISTA" if mode == "haar" else "")
                        + (f", truncated to {cfg.n_trunc} central bins" if cfg.n_trunc else "")
                        + (", x_s = global SIRT iterate (exact)" if args.xs_exact else "")
                        + (f", lambda sweep: {synth.SWEEP_ROIS} ROIs x {synth.SWEEP_LAMBDAS} lambdas in "
                           "[1e-3, 1], MSE+SSIM vs ground truth" if sweep else ""),
            "global_batch_rois": cfg.n_roi, "parallelism": f"roi-shard x{world}",
            "l2": "inputs larger than L2 (conv cache 417 MB + ROI state), no flush",
            "bank": "warm (per-geometry precompute, excluded)"}


def run_ours(args, cfg):
    import torch
    import paper_1604_02292_b200 as lt

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    # LT_BENCH_FUNCTIONAL=1: every rank on cuda:0 with gloo -- a functional check of
    # the N > 1 code path (partition, slot tables, peer / library combine, max-over-
    # ranks timing) on a one-GPU box; its timings are NOT measurements
    functional = os.environ.get("LT_BENCH_FUNCTIONAL") == "1"
    dev_index = 0 if functional else local_rank
    torch.cuda.set_device(dev_index)
    dist = None
    if world > 1:
        import torch.distributed as dist
        if functional:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    red_dev = "cpu" if functional else "cuda"     # gloo reduces host tensors

    def allreduce(vals, op_max=True, dtype=None):
        t = torch.tensor(vals, device=red_dev, dtype=dtype or torch.float32)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op_max else dist.ReduceOp.SUM)
        return [float(v) for v in t.cpu()]

    inp = synth.make_inputs(cfg)
    n_iter = cfg.n_iter
    mode = solve_mode(cfg, args)
    plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, n_iter, rank=rank, world=world,
                   xs_exact=args.xs_exact)
    rects, _, _ = plan.tables()
    # per-geometry precompute (outside the timed region)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if args.bank == "split" and world > 1:
        from paper_1604_02292_b200 import dist as ltd
        ltd.filter_bank_split(plan)
    else:
        plan.filter_bank()
    torch.cuda.synchronize()
    bank_ms = (time.perf_counter() - t0) * 1e3

    # truncated-data workloads (T1, NEXT-3) measure only the central bins: the
    # step pads them on the GPU (lt_pad_truncated) before the solve
    trunc = bool(cfg.n_trunc)
    sino_host = torch.from_numpy(inp.sino_trunc if trunc else inp.sino).pin_memory()
    sino_in = sino_host.cuda()
    sino = lt.pad_truncated(sino_in, cfg.n_det) if trunc else sino_in
    side = 2 * cfg.radius
    from paper_1604_02292_b200 import dist as ltd
    if world > 1:
        spr, slot_roi = ltd.setup_combine(plan)
    else:
        spr, slot_roi = plan.R, np.asarray(plan.local_rois, dtype=np.int32)
    cores = torch.zeros(spr, side, side, device="cuda")
    image = torch.empty(cfg.n, cfg.n, device="cuda")
    gathered = torch.empty(world * spr, side, side, device="cuda") if world > 1 else None
    peer = None
    ncomm = None
    if world > 1 and args.combine == "library" and not functional:
        ncomm = lt.NcclComm.from_process_group()
    if world > 1 and args.combine == "peer":
        try:
            peer = ltd.PeerCombine(plan, cores, slot_roi, spr)
        except Exception as e:   # e.g. no CUDA IPC between these devices: NCCL all-gather instead
            print(f"peer combine unavailable ({e}); using the NCCL all-gather", file=sys.stderr)
            peer = None

    # lambda-sweep workloads (L1, NEXT-1): every ROI carries its own lambda; the
    # step scores each core against the ground truth (MSE, SSIM) instead of combining
    sweep = cfg.layout == "sweep"
    lam_arg = cfg.lam
    scores = {}
    if sweep:
        lam_arg = synth.sweep_lambdas(cfg)[plan.local_rois]
        truth = synth.raster(inp.shapes, cfg.n)
        r_ = cfg.radius
        tc = np.stack([truth[c[0] - r_:c[0] + r_, c[1] - r_:c[1] + r_] for c in inp.centres[plan.local_rois]])
        truth_cores = torch.from_numpy(tc.astype(np.float32)).cuda()

    def step():
        out = cores[:plan.R]
        if trunc:
            lt.pad_truncated(sino_in, cfg.n_det, out=sino)
        if mode == "tv":
            plan.tv_solve(sino, lam_arg, cfg.n_fgp, out=out)
        elif mode == "haar":
            plan.haar_solve(sino, HAAR_LAM, HAAR_LEVELS, out=out)
        elif mode == "exterior":
            plan.exterior_solve(sino, 0.0, math.inf, out=out)
        else:
            plan.sirt_solve(sino, 0.0, math.inf, out=out)
        if sweep:
            scores["mse"], scores["ssim"] = lt.metrics(out, truth_cores)
            return
        combine_step()

    def combine_step():
        if peer is not None:
            peer.combine(image)                            # stitch reading the peers' cores over NVLink
        elif ncomm is not None:
            plan.combine_rois(cores[:plan.R], ncomm, out=image)   # lt_combine_rois: in-place ncclAllGather + stitch
        elif world > 1:
            ltd.gather_cores(cores, out=gathered)          # NCCL all-gather over NVLink
            plan.combine(gathered, slot_roi, out=image)
        else:
            plan.combine(cores[:plan.R], slot_roi, out=image)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    n_launch0 = lt.launch_count()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    # the timed region: K steps exactly as a user runs them (no per-kernel
    # instrumentation: per-launch events would add launch latency and disable
    # the CUDA-graph replay of small batches)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(args.steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    elapsed_ms = ev0.elapsed_time(ev1)
    n_launch = lt.launch_count() - n_launch0
    # per-kernel CUDA events on each kernel's own stream: the same K steps
    # again with lt_timing on (the roofline's average launch durations)
    lt.timing_enable(True)
    lt.timing_read()
    ei0 = torch.cuda.Event(enable_timing=True)
    ei1 = torch.cuda.Event(enable_timing=True)
    ei0.record()
    for _ in range(args.steps):
        step()
    ei1.record()
    torch.cuda.synchronize()
    instr_ms = ei0.elapsed_time(ei1)
    ktimes = lt.timing_read()
    lt.timing_enable(False)
    # the combine (a9 / e) alone, reported separately; part of every step above
    combine_ms = None
    if not sweep:
        if dist:
            dist.barrier()
        ec0 = torch.cuda.Event(enable_timing=True)
        ec1 = torch.cuda.Event(enable_timing=True)
        ec0.record()
        for _ in range(5):
            combine_step()
        ec1.record()
        torch.cuda.synchronize()
        combine_ms = ec0.elapsed_time(ec1) / 5
        if dist:
            combine_ms = allreduce([combine_ms])[0]
    clk = clocks.stop()
    if dist:
        elapsed_ms, instr_ms = allreduce([elapsed_ms, instr_ms])

    # e2e: same step through the host-buffer C-ABI entry (pinned H2D + solve + combine + D2H)
    image_host = torch.empty(cfg.n, cfg.n, dtype=torch.float32).pin_memory()
    if sweep:
        score_host = torch.empty(2, plan.R, dtype=torch.float64).pin_memory()

        def e2e_step():
            sino_in.copy_(sino_host, non_blocking=True)
            step()
            score_host[0].copy_(scores["mse"], non_blocking=True)
            score_host[1].copy_(scores["ssim"], non_blocking=True)
            torch.cuda.synchronize()
    elif world == 1 and not trunc and mode not in ("haar", "exterior"):
        def e2e_step():
            plan.solve_host(mode, sino_host, cfg.lam if mode == "tv" else 0.0,
                            0.0 if mode == "tv" else math.inf, cfg.n_fgp, image_host)
    else:
        def e2e_step():
            sino_in.copy_(sino_host, non_blocking=True)
            step()
            image_host.copy_(image, non_blocking=True)
            torch.cuda.synchronize()
    e2e_step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    e_steps = max(1, min(args.steps, 3))
    for _ in range(e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e_steps
    if dist:
        e2e_ms = allreduce([e2e_ms])[0]

    # global counts
    upd_local, fgp_local, Ptot_local = algorithmic_counts(cfg, rects, n_iter)
    exe_local = executed_updates(cfg, rects, n_iter) if not args.xs_exact and mode in ("tv", "sirt", "haar") else None
    if dist:
        upd, fgp_pi, exe_sum = allreduce([upd_local, fgp_local, exe_local or 0.0], op_max=False, dtype=torch.float64)
        exe = exe_sum if exe_local is not None else None
    else:
        upd, fgp_pi, exe = upd_local, fgp_local, exe_local
    ms_per_step = elapsed_ms / args.steps
    value = cfg.n_roi / (ms_per_step / 1e3)
    if rank != 0:
        if dist:
            if peer is not None:
                dist.barrier()
                peer.close()
                dist.barrier()
            if ncomm is not None:
                ncomm.close()
            dist.destroy_process_group()
        return None

    pk, pk_src = peaks()
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    alu_derived = 148 * 128 * 2 * sm_max * 1e6 / 1e12          # FP32 lanes x FMA, DESIGN.md §Roofline
    smem_derived = 148 * 128 * sm_max * 1e6 / 1e9              # shared-memory crossbar, 128 B/clk/SM
    mp = sm_peaks()
    if mp:
        alu_peak_tflops = max(float(mp["ffma_tflops"]), float(mp["ffma2_tflops"]))
        smem_peak_gbs = float(mp["smem_lds64_gbs"])
        alu_src = (f"measured: FP32 FMA stream over all SMs, {MICRO_PEAKS} (tools/peaks_micro.cu); "
                   f"derived 148 x 128 lanes x 2 x {sm_max:.0f} MHz = {alu_derived:.1f}")
        smem_src = (f"measured: conflict-free LDS.64 stream over all SMs, {MICRO_PEAKS} (tools/peaks_micro.cu); "
                    f"derived 148 x 128 B/clk x {sm_max:.0f} MHz = {smem_derived:.0f}")
    else:
        alu_peak_tflops, smem_peak_gbs = alu_derived, smem_derived
        alu_src = f"derived: 148 SM x 128 FP32 lanes x 2 x {sm_max:.0f} MHz ({pk_src} clock)"
        smem_src = f"derived: 148 SM x 128 B/clk shared-memory crossbar x {sm_max:.0f} MHz ({pk_src} clock)"
    nA = cfg.n_angles * Ptot_local          # pixel-angle updates of one A or A^T over all local ROIs
    # Joseph ray-line steps of one W_{L'} over all local ROIs: per angle c_a P
    # (a line of w valid pixels is crossed by c_a w rays, c_a = max(|cos|, |sin|))
    c_sum = float(np.sum(np.maximum(np.abs(np.cos(inp.angles)), np.abs(np.sin(inp.angles)))))
    fp_steps = c_sum * Ptot_local
    traffic_all = {}
    for rnd in ("r02", "r01"):   # dram__bytes_read.sum + dram__bytes_write.sum per launch, latest committed ncu capture
        try:
            with open(os.path.join(ROOT, "profiles", rnd, "traffic.json")) as f:
                traffic_all = json.load(f)
            break
        except Exception:
            traffic_all = {}

    def roofline_of(cls):
        """Roofline entry of one main-stream kernel class."""
        ms, n = ktimes[cls]
        if n == 0 or ms <= 0:
            return None
        avg_ms = ms / n
        kname = {"fgp": "k_fgp2", "fp": "k_fp_roi2", "bp": "k_bp_roi"}[cls]
        if cls == "fgp":
            if mode in ("haar", "exterior"):
                return None      # the Haar prox is a few flops per pixel: not a roofline kernel
            work = fgp_local * args.steps * FGP_FLOPS_PER_PX_IT / n
            ent = {"bound": "alu", "peak": round(alu_peak_tflops, 1), "unit": "TFLOP/s",
                   "achieved": work / (avg_ms / 1e3) / 1e12,
                   "work_per_unit": f"{FGP_FLOPS_PER_PX_IT:g} FP32 flops per pixel-iteration",
                   "peak_source": alu_src}
        elif cls == "fp":        # one W_{L'} y per iteration 2..n; one (S, D) pair (8 B) per ray-line step
            work = FP_SMEM_BYTES_PER_STEP * fp_steps * (n_iter - 1) * args.steps / n
            ent = {"bound": "smem", "peak": round(smem_peak_gbs, 1), "unit": "GB/s",
                   "achieved": work / (avg_ms / 1e3) / 1e9,
                   "work_per_unit": f"{FP_SMEM_BYTES_PER_STEP:g} B of staged (S, D) pairs per Joseph ray-line step",
                   "peak_source": smem_src}
        else:                    # W_{L'}^T s of iterations 2..n (iteration 1 has s = 0: no gather)
            work = JOSEPH_FLOPS_PER_UPDATE * nA * (n_iter - 1) * args.steps / n
            ent = {"bound": "alu", "peak": round(alu_peak_tflops, 1), "unit": "TFLOP/s",
                   "achieved": work / (avg_ms / 1e3) / 1e12,
                   "work_per_unit": f"{JOSEPH_FLOPS_PER_UPDATE:g} FP32 flops per pixel-angle update",
                   "peak_source": alu_src}
        traffic, traffic_src = None, None
        busy = None
        if kname in traffic_all:   # the capture's launches cover all R ROIs; scale to this run's launch size
            tj = traffic_all[kname]
            traffic = float(tj["dram_bytes_per_launch"]) * (plan.R / float(tj.get("rois_per_launch", plan.R)))
            traffic_src = tj["source"]
            # how busy the binding unit itself is in the same capture (ncu): the
            # shared-memory / L1 data path for the FP, the FP32 pipe for BP / FGP
            if all(k_ in tj for k_ in ("issue_pct", "fma_pipe_pct", "l1tex_pct")):
                busy = {"issue_pct": tj["issue_pct"], "fma_pipe_pct": tj["fma_pipe_pct"],
                        "l1tex_pct": tj["l1tex_pct"], "source": tj["source"]}
        ent["achieved"] = round(ent["achieved"], 3)
        # the HBM fraction (reported although the path is SM-bound)
        hbm = float(pk.get("hbm_gbs") or 0.0)
        ent["hbm_frac"] = round(traffic / (avg_ms / 1e3) / 1e9 / hbm, 4) if traffic and hbm > 0 else None
        ent.update({"kernel": kname, "frac": round(ent["achieved"] / ent["peak"], 4), "traffic": traffic,
                    "unit_busy_ncu": busy,
                    "traffic_unit": "DRAM bytes per launch", "traffic_source": traffic_src,
                    "avg_launch_ms": round(avg_ms, 4), "launches": n,
                    "share_of_step": round(ms / instr_ms, 3)})
        return ent

    rooflines = {c: roofline_of(c) for c in ("fp", "bp", "fgp")}
    rooflines = {c: v for c, v in rooflines.items() if v is not None}
    # dominant kernel class over the timed region (rank 0's main stream; the x_s
    # backprojection "xs" runs on a side stream, overlapped: reported per class only)
    if rooflines:
        dom = max(rooflines, key=lambda c: ktimes[c][0])
        roofline = {k: rooflines[dom][k] for k in ("bound", "achieved", "peak", "unit", "frac", "traffic")}
        roofline.update({k: v for k, v in rooflines[dom].items() if k not in roofline})
    else:   # (N > 1 with fewer ROIs than ranks: rank 0 may own none and launch no roofline kernel)
        roofline = {"bound": None, "achieved": None, "peak": None, "unit": None, "frac": None, "traffic": None,
                    "note": "rank 0 launched none of the roofline kernels (it owns no ROI)"}
    kshare = {k: {"ms_per_step": round(v[0] / args.steps, 3), "launches_per_step": v[1] // args.steps}
              for k, v in ktimes.items()}
    cpu = None
    if not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, budget_s=20.0, mode=mode)
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(cfg, args, world),
        "combine": ("peer-memory stitch (CUDA IPC over NVLink, one kernel)" if peer is not None else
                    "lt_combine_rois (library-owned NCCL all-gather + stitch)" if ncomm is not None else
                    "NCCL all-gather + stitch" if world > 1 else "local stitch"),
        "gray_s": round(upd / (ms_per_step / 1e3) / 1e9, 2),
        "gray_s_note": "method-defined count: N_theta P (1 + 3 (n-1)) per ROI; gray_s_executed counts what the "
                       "kernels execute (x_s once per 64x64 image block per iteration, shared by overlapping ROIs)",
        "gray_s_executed": None if exe is None else round(exe / (ms_per_step / 1e3) / 1e9, 2),
        "fgp_gpix_it_s": round(fgp_pi / (ms_per_step / 1e3) / 1e9, 2),
        "bank_ms": round(bank_ms, 2),
        "combine_ms": None if combine_ms is None else round(combine_ms, 3),
        "bank_mode": ("angle-split (NCCL all-reduce per Alg. 1 step)" if args.bank == "split" and world > 1
                      else "local (every rank computes the whole bank)"),
        "kernels": kshare,
        "kernel_timing": {"pass": "the same K steps again with per-launch CUDA events on each kernel's stream "
                                  "(lt_timing; eager launches)",
                          "ms_per_step": round(instr_ms / args.steps, 3)},
        "gpu_launches": int(n_launch),
        "e2e": {"value": round(cfg.n_roi / (e2e_ms / 1e3), 3), "unit": UNIT,
                "h2d_bytes_per_step": int(sino_host.numel() * 4),
                "d2h_bytes_per_step": int(2 * plan.R * 8 if sweep else cfg.n * cfg.n * 4),
                "ms_per_step": round(e2e_ms, 3)},
        "roofline": roofline,
        "rooflines": rooflines,
        "hbm_peak_gbs": pk.get("hbm_gbs"),
        "clocks": clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if dist:
        if peer is not None:        # unmap the peers' buffers before any rank frees its own
            dist.barrier()
            peer.close()
            dist.barrier()
        if ncomm is not None:
            ncomm.close()
        dist.destroy_process_group()
    return line


# --------------------------------------------------------------------------- oracle (CPU)
def cpu_model() -> str:
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def oracle_sample(cfg, n_iter_sample=2, n_conv_k=1, n_rois=16, mode=None):
    """Time the fp64 oracle on a bounded sample of the same workload and
    extrapolate to the full step: disc (whole) + conv cache
    (n_conv_k of the n filters, x n / n_conv_k) + a seeded sample of n_rois ROIs
    for iterations 1..n_iter_sample, extrapolated linearly to n iterations and
    to all ROIs by valid extended-pixel count (the oracle's per-ROI cost is
    proportional to it).  Iteration 1 has y = 0 (its projection of y is
    skipped by the oracle's zero test), so the extrapolation favours the oracle."""
    import oracle
    inp = synth.make_inputs(cfg)
    p = inp.sino.astype(np.float64)
    n = cfg.n
    t0 = time.perf_counter()
    pc, c, _, _ = oracle.disc(p, inp.angles, n)
    t_disc = time.perf_counter() - t0
    rng = np.random.default_rng(0)
    fake_bank = rng.standard_normal((n_conv_k, cfg.n_angles, cfg.n_det))
    t0 = time.perf_counter()
    oracle.conv_cache(fake_bank, pc)
    t_conv = (time.perf_counter() - t0) * cfg.n_iter / n_conv_k
    R = cfg.n_roi
    pick = np.sort(synth.seeded_rng(cfg.cfg_id, 3).choice(R, size=min(n_rois, R), replace=False))
    rects = oracle.roi_rects(n, inp.centres, cfg.radius, cfg.margin)
    valid = (rects[:, 5] - rects[:, 4]).astype(np.float64) * (rects[:, 7] - rects[:, 6])
    bconv = rng.standard_normal((n_iter_sample, cfg.n_angles, cfg.n_det)) * 1e-3
    mode = {"sirt": "box", "tv": "tv", "haar": "haar", "exterior": "box",
            None: "tv" if "tv" in cfg.solver else "box"}[mode]
    t0 = time.perf_counter()
    oracle.local_solve(n, inp.angles, cfg.n_det, bconv, inp.centres[pick], cfg.radius, cfg.margin, mode=mode,
                       lam=HAAR_LAM if mode == "haar" else cfg.lam, n_fgp=cfg.n_fgp, disc_c=c, use_disc=True,
                       levels=HAAR_LEVELS)
    t_rois = time.perf_counter() - t0
    scale_iter = cfg.n_iter / n_iter_sample
    scale_pix = float(valid.sum() / valid[pick].sum())
    total = t_disc + t_conv + t_rois * scale_iter * scale_pix
    sample = (f"disc (full) + conv cache {n_conv_k}/{cfg.n_iter} filters (x{cfg.n_iter / n_conv_k:g}) + "
              f"{len(pick)} seeded ROIs {pick.tolist()[:16]} x iterations 1-{n_iter_sample} of {cfg.n_iter} "
              f"(x{scale_iter:g} iterations, x{scale_pix:.2f} by valid extended pixels for all {R} ROIs); "
              f"measured {t_disc:.2f}+{t_conv * n_conv_k / cfg.n_iter:.2f}+{t_rois:.2f} s")
    return R / total, sample, oracle.get_threads()


def cpu_baseline(cfg, budget_s=20.0, mode=None):
    try:
        v, sample, cores = oracle_sample(cfg, mode=mode)
        out = {"value": round(v, 6), "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
               "nproc": os.cpu_count(), "cpu_model": cpu_model()}
        if cfg.n <= 512:        # small configs also single-threaded
            import oracle
            oracle.set_threads(1)
            try:
                v1, _, _ = oracle_sample(cfg, mode=mode)
            finally:
                oracle.set_threads(cores)
            out["single_thread_value"] = round(v1, 6)
        return out
    except Exception as e:  # report, never fake
        return {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle", "sample": f"failed: {e}"}


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return None
    import oracle
    for _ in range(args.warmup):
        oracle_sample(cfg, mode=solve_mode(cfg, args))
    vals = []
    t0 = time.perf_counter()
    sample = ""
    for _ in range(args.steps):
        v, sample, cores = oracle_sample(cfg, mode=solve_mode(cfg, args))
        vals.append(v)
    wall = time.perf_counter() - t0
    value = statistics.median(vals)
    line = {"metric": METRIC, "value": round(value, 6), "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(cfg.n_roi / value * 1e3, 1), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": dict(config_dict(cfg, args, 1),
                           reference="fp64 CPU oracle (the paper has no code), extrapolated from a bounded sample"),
            "cpu_baseline": {"value": round(value, 6), "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
                             "sample": sample, "nproc": os.cpu_count(), "cpu_model": cpu_model()},
            "e2e": {"value": round(value, 6), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": round(wall, 1)}
    print(json.dumps(line), flush=True)
    return line


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))
    if args.selftest:
        selftest()
        return
    cfg = synth.config(args.config)
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_ours(args, cfg)


if __name__ == "__main__":
    main()
