"""GPU parity at the configs' FULL sizes and STATED iteration counts (-m gpu).

The north star asks for "full solves within 1e-3 relative L2 after the stated
iteration count" (BASELINE.json; the paper's 200 outer x 100 FGP iterations,
PAPER.md L796-798).  The fp64 oracle's filter bank at these sizes takes minutes
to hours, so its results on sampled ROIs are precomputed by
tests/golden/make_oracle_refs.py (which calls only oracle/ and synth/) into
tests/golden/oracle_ref/<cfg>.npz.  Each test runs the GPU path exactly as
bench.py launches it -- the full ROI batch of the config in one plan -- and
compares the sampled ROIs:

  C3  1024^2, 32 angles over [0, 2pi/3), 64 seeded ROIs, n = 300, box AND TV
  C4  2048^2, 180 angles, 256-ROI tiling, FISTA-TV n = 200, n_FGP = 100 (the bench workload)
  C5  4096^2, 256 angles, 1024-ROI tiling, nonneg SIRT n = 500

plus the filter bank u_k (<= 1e-4) and the convolution cache b_k at
k in {1, n/2, n} on sampled angle rows, and the disc value c.  With
LT_PARITY_REPORT=<path> every measured relL2 is appended to a JSON-lines file
(profiles/r02/parity_full_iterations.jsonl).
"""
import json
import math
import os

import numpy as np
import pytest

import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REF_DIR = os.path.join(os.path.dirname(__file__), "golden", "oracle_ref")


def relerr(a, b):
    a = np.asarray(a, dtype=np.float64); b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def report(**kw):
    path = os.environ.get("LT_PARITY_REPORT")
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(kw) + "\n")


def load_ref(name):
    path = os.path.join(REF_DIR, f"{name}.npz")
    assert os.path.exists(path), f"{path} missing: run tests/golden/make_oracle_refs.py {name}"
    z = np.load(path)
    ref = {k: z[k] for k in z.files}
    ref["meta"] = json.loads(str(ref["meta"]))
    return ref


@pytest.fixture(scope="module")
def lt():
    import __graft_entry__
    __graft_entry__.build()
    import paper_1604_02292_b200 as m
    assert torch.cuda.is_available()
    return m


_PLANS = {}


def plan_for(lt, name):
    """One plan per config (the full ROI batch, as bench.py builds it) with its bank."""
    if name not in _PLANS:
        _PLANS.clear()                     # one large workspace at a time
        torch.cuda.empty_cache()
        cfg = synth.config(name)
        inp = synth.make_inputs(name)
        plan = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter)
        plan.filter_bank()
        _PLANS[name] = (cfg, inp, plan)
    return _PLANS[name]


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_inputs_match_the_reference_run(name):
    """The seeded inputs regenerate (to fp32 rounding) what the oracle run used."""
    ref = load_ref(name)
    inp = synth.make_inputs(name)
    assert relerr(inp.sino[ref["angles_idx"]], ref["sino_rows"]) <= 1e-6


def check_bank_conv_disc(lt, name):
    """Alg. 1 filters u_k at k = 1, n/2, n on sampled angle rows
    <= 1e-4; disc c <= 1e-5; b_k = C_{u_k} p_c of the
    GPU's own bank and p_c <= 1e-4 (bank and convolution errors combined)."""
    ref = load_ref(name)
    cfg, inp, plan = plan_for(lt, name)
    ks, aidx = ref["ks"], ref["angles_idx"]
    bank = plan.get_bank()
    for j, k in enumerate(ks):
        got = bank[int(k) - 1][torch.as_tensor(aidx, device=bank.device)].cpu().double().numpy()
        e = relerr(got, ref["bank_rows"][j])
        report(config=name, what="bank u_k", k=int(k), relL2=e, tol=1e-4)
        assert e <= 1e-4, (name, int(k), e)
    del bank
    pc, c = plan.disc_correct(torch.from_numpy(inp.sino).cuda())
    ec = abs(float(c.cpu()[0]) - float(ref["disc_c"])) / abs(float(ref["disc_c"]))
    report(config=name, what="disc c", relerr=ec, tol=1e-5)
    assert ec <= 1e-5
    conv = plan.conv_cache(pc)
    for j, k in enumerate(ks):
        got = conv[int(k) - 1][torch.as_tensor(aidx, device=conv.device)].cpu().double().numpy()
        e = relerr(got, ref["conv_rows"][j])
        report(config=name, what="conv b_k", k=int(k), relL2=e, tol=1e-4)
        assert e <= 1e-4, (name, int(k), e)
    del conv
    torch.cuda.empty_cache()


def check_full_solve(lt, name, mode):
    """Full local solve of the whole ROI batch at the stated n (and n_FGP = 100
    for TV), disc on, lambda = 0.05; every sampled ROI core <= 1e-3 relL2
    against the oracle (north star; Alg. 2, Alg. 3)."""
    ref = load_ref(name)
    cfg, inp, plan = plan_for(lt, name)
    assert ref["meta"]["n_iter"] == cfg.n_iter == plan.n_iter
    sino = torch.from_numpy(inp.sino).cuda()
    if mode == "box":
        cores = plan.sirt_solve(sino, 0.0, math.inf)
    else:
        cores = plan.tv_solve(sino, cfg.lam, cfg.n_fgp)
    torch.cuda.synchronize()
    want = ref[f"cores_{mode}"]
    errs = []
    for k, g in enumerate(ref["rois"]):
        q = int(np.nonzero(plan.local_rois == g)[0][0])
        errs.append(relerr(cores[q].cpu().double().numpy(), want[k]))
    report(config=name, what=f"{mode} solve cores", n_iter=cfg.n_iter, n_fgp=cfg.n_fgp if mode == "tv" else None,
           rois=[int(v) for v in ref["rois"]], relL2=errs, max_relL2=max(errs), tol=1e-3)
    assert max(errs) <= 1e-3, (name, mode, errs)
    assert torch.isfinite(cores).all()


# ordered per config, so each config's plan and bank are built once
CASES = [("C3", "bank"), ("C3", "box"), ("C3", "tv"), ("C4", "bank"), ("C4", "tv"), ("C4", "shards"),
         ("C5", "bank"), ("C5", "box"), ("C5", "shards")]


@pytest.mark.parametrize("name,what", CASES)
def test_full_size_stated_iterations(lt, name, what):
    if what == "bank":
        check_bank_conv_disc(lt, name)
    elif what == "shards":
        check_rank_shards(lt, name, worlds=(2, 8) if name == "C4" else (8,))
    else:
        check_full_solve(lt, name, what)


def check_rank_shards(lt, name, worlds=(2, 8)):
    """The multi-GPU partition (every local
    reconstruction is independent): each rank's shard of the ROI batch, solved
    as its own plan in the launch shapes a rank of an N-GPU run takes (C4 on 8
    GPUs: ~32 ROIs -- 24-angle forward-projector CTAs under one wave, 3 FGP
    cluster waves), at the stated n and n_FGP, reproduces the oracle on every
    sampled ROI the shard holds (<= 1e-3)."""
    ref = load_ref(name)
    cfg, inp, plan = plan_for(lt, name)
    bank = plan.get_bank()
    sino = torch.from_numpy(inp.sino).cuda()
    rois = [int(g) for g in ref["rois"]]
    for world in worlds:
        seen = set()
        for rank in range(world):
            sp = lt.Plan(cfg.n, inp.angles, cfg.n_det, inp.centres, cfg.radius, cfg.margin, cfg.n_iter,
                         rank=rank, world=world)
            hits = [k for k, g in enumerate(rois) if g in set(int(v) for v in sp.local_rois)]
            if not hits:
                del sp
                continue
            sp.set_bank(bank)
            if "tv" in cfg.solver:
                cores = sp.tv_solve(sino, cfg.lam, cfg.n_fgp)
                want = ref["cores_tv"]
            else:
                cores = sp.sirt_solve(sino, 0.0, math.inf)
                want = ref["cores_box"]
            errs = []
            for k in hits:
                q = int(np.nonzero(sp.local_rois == rois[k])[0][0])
                errs.append(relerr(cores[q].cpu().double().numpy(), want[k]))
                seen.add(k)
            report(config=name, what="rank shard solve cores", world=world, rank=rank, local_rois=int(sp.R),
                   rois=[rois[k] for k in hits], relL2=errs, max_relL2=max(errs), tol=1e-3)
            assert max(errs) <= 1e-3, (name, world, rank, errs)
            del sp, cores
        assert seen == set(range(len(rois)))      # the shards cover every sampled ROI
    del bank
    torch.cuda.empty_cache()
