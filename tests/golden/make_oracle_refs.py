"""Writes tests/golden/oracle_ref/<cfg>.npz: fp64 ORACLE results for the
BASELINE.json configs at their full sizes and stated iteration counts, on
sampled ROIs, for the GPU parity tests (tests/test_gpu_full_iterations.py).

Calls only oracle/ (the fp64 CPU oracle) and synth/ (seeded inputs).  The
stored values are therefore expected values "written by a committed script
that calls only oracle/": the oracle's filter bank at these sizes costs
minutes (C4: 200 Alg. 1 iterations on 2048^2 x 180 angles) to hours (C5: 500
on 4096^2 x 256), too long to recompute inside a GPU test run.

Per config it stores:
  cores          [S, 2r, 2r]   oracle.local_solve cores of the sampled ROIs
                               (Alg. 2 box / Alg. 3 TV), per mode
  bank_rows      [3, A, N_d]   u_k at k in {1, n/2, n} for the sampled angles (Alg. 1)
  conv_rows      [3, A, N_d]   b_k = C_{u_k} p_c at the same k and angles
  disc_c                       the disc gray value c
  sino_rows      [A, N_d]      the fp32 input sinogram rows at the sampled angles
                               (the test checks synth regenerates the same input)
  rois, angles_idx, ks, meta   (what was sampled, the oracle source hash, timings)

Run (CPU only, OMP threads = all cores):
    python tests/golden/make_oracle_refs.py C3 C4 C5
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
import synth   # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "oracle_ref")

# sampled ROIs: corners, edges and interior of the tilings; spread seeded ROIs for C3
SAMPLES = {
    "C3": [0, 9, 21, 33, 47, 63],
    "C4": [0, 15, 240, 255, 7, 112, 136, 200],
    "C5": [0, 31, 992, 1023, 16, 496, 529, 700],
}
MODES = {"C3": ["box", "tv"], "C4": ["tv"], "C5": ["box"]}


def sampled_angles(na):
    return np.unique(np.round(np.linspace(0, na - 1, 8)).astype(int))


def main(names):
    os.makedirs(OUT, exist_ok=True)
    src_hash = hashlib.sha256(open(os.path.join(ROOT, "oracle", "loctomo_oracle.c"), "rb").read()).hexdigest()
    for name in names:
        cfg = synth.config(name)
        inp = synth.make_inputs(name)
        n, nd, na, nk = cfg.n, cfg.n_det, cfg.n_angles, cfg.n_iter
        p = inp.sino.astype(np.float64)
        sample = np.array(SAMPLES[name])
        aidx = sampled_angles(na)
        ks = np.array([1, nk // 2, nk])
        tm = {}
        t0 = time.time()
        pc, c, _, _ = oracle.disc(p, inp.angles, n)
        tm["disc_s"] = time.time() - t0
        t0 = time.time()
        bank = oracle.filter_bank(n, inp.angles, nd, nk)
        tm["bank_s"] = time.time() - t0
        print(f"{name}: bank {tm['bank_s']:.0f} s", flush=True)
        bank_rows = np.stack([bank[k - 1][aidx] for k in ks])
        t0 = time.time()
        b = np.empty_like(bank)
        for k in range(nk):
            b[k] = oracle.convolve(bank[k], pc)
        tm["conv_s"] = time.time() - t0
        print(f"{name}: conv cache {tm['conv_s']:.0f} s", flush=True)
        del bank
        conv_rows = np.stack([b[k - 1][aidx] for k in ks])
        out = dict(bank_rows=bank_rows, conv_rows=conv_rows, disc_c=np.float64(c),
                   sino_rows=inp.sino[aidx], rois=sample, angles_idx=aidx, ks=ks)
        for mode in MODES[name]:
            t0 = time.time()
            cores = oracle.local_solve(n, inp.angles, nd, b, inp.centres[sample], cfg.radius, cfg.margin,
                                       mode=mode, lo=0.0, hi=np.inf, lam=cfg.lam, n_fgp=cfg.n_fgp,
                                       disc_c=c, use_disc=True)
            tm[f"solve_{mode}_s"] = time.time() - t0
            print(f"{name}: {mode} solve of {len(sample)} ROIs {tm[f'solve_{mode}_s']:.0f} s", flush=True)
            out[f"cores_{mode}"] = cores
        meta = dict(config=name, n_iter=nk, lam=cfg.lam, n_fgp=cfg.n_fgp, radius=cfg.radius, margin=cfg.margin,
                    oracle_c_sha256=src_hash, threads=oracle.get_threads(), timings=tm,
                    script="tests/golden/make_oracle_refs.py")
        out["meta"] = np.array(json.dumps(meta))
        np.savez_compressed(os.path.join(OUT, f"{name}.npz"), **out)
        print(f"{name}: written ({json.dumps(tm)})", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C3", "C4", "C5"])
