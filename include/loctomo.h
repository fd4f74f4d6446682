/*
 * loctomo.h -- C-ABI of the B200-native local tomography library
 * (local approximation of regularized iterative reconstruction,
 *  Pelt & Batenburg, arXiv 1604.02292; "P:Lnnn" = PAPER.md line).
 *
 * Conventions (V1-V4):
 *  - image: N x N fp32, row-major, row i = 0 at the top; pixel centre
 *    x_j = j - (N-1)/2, y_i = (N-1)/2 - i.
 *  - sinogram: [N_theta][N_d] fp32, bin centre t_d = d - (N_d-1)/2.
 *  - W: Joseph interpolation, W[(a,d),(i,j)] = hat((t_d - t_ij)/c_a)/c_a,
 *    c_a = max(|cos|,|sin|); W^T is its exact transpose.
 *  - alpha = 1/(N_theta N_d).
 *  - ROI: square core of half-side `radius` around integer pixel-corner
 *    centre (row, col); extended ROI L' = core padded by `margin` and clipped
 *    to the grid.
 *
 * Memory: every pointer named d_* is a DEVICE pointer owned by the caller
 * (the Python binding allocates with torch); h_* pointers are HOST memory,
 * read (or written) only during the call.  The library never allocates
 * device memory: all scratch lives in the caller-provided workspace bound
 * with lt_plan_bind_workspace.  `stream` is a cudaStream_t (NULL = legacy
 * default stream); all device work is stream-ordered and asynchronous
 * unless stated otherwise.
 *
 * Errors: LT_OK = 0; LT_ERR_RUNTIME = 1 (CUDA failure); LT_ERR_INVALID = 2
 * (argument violates the contract; detected on the host before any launch,
 * no partial output).  lt_last_error() returns a thread-local message.
 * Results are deterministic: no atomics, fixed summation orders.
 * A plan keeps the solve state in its workspace: calls on one plan must be
 * stream-ordered (one stream at a time); different plans are independent.
 */
#ifndef LOCTOMO_H
#define LOCTOMO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LT_OK 0
#define LT_ERR_RUNTIME 1
#define LT_ERR_INVALID 2

/* flags for lt_roi_setup */
#define LT_DISC_ON 1   /* disc pre-correction, default on */
#define LT_XS_EXACT 2  /* x_s^k = M_{L'} (global SIRT iterate k) instead of
                        * FBP_L(p_c, u_k) + cD (removes approximation 1 of P:L625-630, so a
                        * ROI covering the grid reproduces the global solve, pins P9/P10); the
                        * SIRT iterate is advanced once per iteration on the full grid (shared by
                        * all ROIs), no filter bank, conv cache or disc is used */
#define LT_GUARD_BANDS 4 /* debug: a canary band after every workspace region (more workspace),
                          * checked by lt_guard_check -- detects out-of-bounds device writes */

typedef struct lt_plan lt_plan;

/* Plan a batch of local reconstructions (host only; no device work).
 *  n, n_angles, n_det: N, N_theta, N_d.  n_det must be odd
 *      (filter centring, A3).
 *  angles: host, n_angles radians, strictly increasing in [0, pi).
 *  n_roi, center_row, center_col: host, the ROI core centres (integer pixel
 *      corners); every core must lie inside the grid.
 *  radius (>= 1), margin (>= 0): core half-side r and padding m.
 *  n_iter (>= 1): outer iterations n; the filter bank holds u_1..u_n.
 *  rank, world: this process's share of the ROIs (the ROIs in raster order
 *      cut into world contiguous runs of balanced cost); world = 1
 *      for a single GPU.
 *  out: receives the plan.  Returns LT_ERR_INVALID on any violation. */
int lt_roi_setup(int32_t n, int32_t n_angles, int32_t n_det, const double* angles,
                 int32_t n_roi, const int32_t* center_row, const int32_t* center_col,
                 int32_t radius, int32_t margin, int32_t n_iter, int32_t flags,
                 int32_t rank, int32_t world, lt_plan** out);

/* Bytes of device workspace the plan needs (tables, filter bank, convolution
 * cache, per-ROI state). */
int64_t lt_plan_workspace_bytes(const lt_plan* plan);

/* Bind a device workspace of >= lt_plan_workspace_bytes bytes (256-byte
 * aligned) and upload the geometry tables (synchronous on `stream`). */
int lt_plan_bind_workspace(lt_plan* plan, void* d_ws, int64_t bytes, void* stream);

/* Local ROI count on this rank and their global ROI indices (host array of
 * lt_plan_local_count entries). */
int32_t lt_plan_local_count(const lt_plan* plan);
int lt_plan_local_rois(const lt_plan* plan, int32_t* h_global_idx);

/* Host copies of the plan's ROI tables (for tests and tooling):
 * h_rects [local_count][6] = tile row0, col0 (global coords of the extended
 * square's top-left pixel), valid rect vr0, vr1, vc0, vc1 (tile-local);
 * h_d0 [local_count][N_theta] = first detector bin of each ROI's window;
 * *h_wwin = window width W(h) = 2 ceil((2h-1)/sqrt2) + 4 (V4).
 * Any pointer may be NULL. */
int lt_plan_tables(const lt_plan* plan, int32_t* h_rects, int32_t* h_d0, int32_t* h_wwin);

/* Alg. 1: compute every filter u_k, k = 1..n, into the
 * workspace; also caches W D for the disc correction.  Geometry-only. */
int lt_filter_bank(lt_plan* plan, void* stream);

/* Angle-split Alg. 1 for a cold bank on G ranks (P:L489-503 with
 * W = [W_0; ...; W_{G-1}] split by angle rows): rank g owns angles [a0, a1).
 *   lt_bank_split_begin: c = e_c (the centred impulse, reading A5) in the plan's
 *     global image; records [a0, a1).  Errors: 2 if the range is empty or
 *     outside [0, n_angles).
 *   lt_bank_split_step(k): v_g = W_g c; bank rows u_k[a] = u_{k-1}[a] + alpha v_g[a]
 *     for a in [a0, a1) (rows of other angles untouched); for k < n_iter - 1 also
 *     d_partial = W_g^T v_g, a plain row-major N x N device image (caller-owned).
 *     Errors: 2 if begin was not called, k outside [0, n_iter), d_partial null
 *     when needed, or the geometry needs the single-pass projector (tiles wider
 *     than the tiled projector's band).
 *   lt_bank_split_apply: c <- c - alpha d_reduced, d_reduced = sum over ranks of
 *     the partials (the caller's all-reduce, N x N device image).
 * Steps must be issued in order k = 0, 1, ... with apply between steps.  After
 * step n_iter - 1 the plan holds its own rows of every u_k (lt_get_bank returns
 * them, the other rows unspecified); the caller gathers the other ranks' rows
 * and installs the full bank with lt_set_bank. */
int lt_bank_split_begin(lt_plan* plan, int32_t a0, int32_t a1, void* stream);
int lt_bank_split_step(lt_plan* plan, int32_t k, float* d_partial, void* stream);
int lt_bank_split_apply(lt_plan* plan, const float* d_reduced, void* stream);

/* Filter-bank reuse and persistence ("the needed filters ... can be precomputed
 * for a certain projection geometry").
 *  lt_bank_key: 64-bit key of what u_k depends on -- N, the angles (bits),
 *    N_d, alpha, the projector and the impulse rule (readings V2, A5); NOT
 *    n_iter (u_k does not depend on n).  0 for a null plan.
 *  lt_set_bank: install a bank [n_iter][N_theta][N_d] fp32 (device, caller-owned,
 *    copied on `stream`) computed for the geometry with key `key`.  Errors: 2 if
 *    the key differs from lt_bank_key(plan), null pointers, unbound plan.
 *  lt_get_bank: copy the plan's bank out (same layout).
 *  lt_save_bank / lt_load_bank: the bank to / from a file (header: magic
 *    "LTBANK01", key, N, N_theta, N_d, n_iter, alpha; then fp32 u_1..u_n).  Both
 *    synchronous on `stream`; save writes `path`.tmp then renames.  load accepts
 *    a file with n' >= n_iter filters (uses the first n_iter).  Errors: 2 for a
 *    non-bank file, another geometry (key / sizes / alpha) or too few filters;
 *    1 for I/O failures. */
uint64_t lt_bank_key(const lt_plan* plan);
int lt_set_bank(lt_plan* plan, const float* d_bank, uint64_t key, void* stream);
int lt_save_bank(const lt_plan* plan, const char* path, void* stream);
int lt_load_bank(lt_plan* plan, const char* path, void* stream);

/* Angle-split GLOBAL box-SIRT on G ranks (SURVEY §8(e), P:L382-396 with W split
 * by angle rows), the same pattern as the split bank:
 *   lt_global_split_begin: x = 0 in the plan's global image; this rank owns
 *     angles [a0, a1) (errors: 2 if empty or outside [0, n_angles)).
 *   lt_global_split_step: r_g = p_g - W_g x on its angles (d_sino: the full
 *     N_theta x N_d sinogram, device) and d_partial = W_g^T r_g, a row-major
 *     N x N device image (caller-owned).
 *   lt_global_split_apply: x <- clamp(x + alpha d_reduced, lo, hi), d_reduced =
 *     the sum of all ranks' partials (the caller's all-reduce).
 *   lt_global_split_result: d_img (N x N, device) = x.
 * Errors: 2 if begin was not called, null pointers, lo > hi. */
int lt_global_split_begin(lt_plan* plan, int32_t a0, int32_t a1, void* stream);
int lt_global_split_step(lt_plan* plan, const float* d_sino, float* d_partial, void* stream);
int lt_global_split_apply(lt_plan* plan, const float* d_reduced, float lo, float hi, void* stream);
int lt_global_split_result(lt_plan* plan, float* d_img, void* stream);
int lt_get_bank(const lt_plan* plan, float* d_bank, void* stream);

/* Forward projection.  roi = -1: full grid, d_img N x N -> d_sino N_theta x N_d
 * (W x).  roi >= 0 (local index): W M_{L'} x, the ROI's extended
 * region only; d_sino is the full sinogram (zero where W_{L'} is). */
int lt_project(const lt_plan* plan, int32_t roi, const float* d_img, float* d_sino, void* stream);

/* Backprojection.  roi = -1: W^T s on the full grid; roi >= 0: M_{L'} W^T s
 * (P:L251), d_img is N x N and zero outside L'. */
int lt_backproject(const lt_plan* plan, int32_t roi, const float* d_sino, float* d_img, void* stream);

/* Disc pre-correction: d_pc = p - c W D, c minimizes the
 * zero-frequency l2 norm; *d_c (device, 1 float) receives c.  Needs
 * lt_filter_bank (or lt_set_bank + this computing W D on first use). */
int lt_disc_correct(lt_plan* plan, const float* d_sino, float* d_pc, float* d_c, void* stream);

/* Convolution cache b_k = C_{u_k} p_c for k = 1..n into the
 * workspace; lt_get_conv copies it out ([n][N_theta][N_d]). */
int lt_conv_cache(lt_plan* plan, const float* d_pc, void* stream);
int lt_get_conv(const lt_plan* plan, float* d_out, void* stream);

/* Local box-constrained SIRT (Alg. 2 with d of P:L538-546) on every local
 * ROI: disc (if LT_DISC_ON) -> conv cache -> n iterations -> crop.
 * d_sino: N_theta x N_d.  lo <= hi (use +INFINITY for "nonneg" SIRT).
 * d_cores: [local_count][2r][2r]. */
int lt_sirt_solve(lt_plan* plan, const float* d_sino, float lo, float hi, float* d_cores, void* stream);

/* Local FISTA-TV (Alg. 3, FISTA update per DESIGN.md A12, FGP prox A13/A14).
 * lambda >= 0, 1 <= n_fgp <= 4096; extended ROI side 2h <= 256. */
int lt_tv_solve(lt_plan* plan, const float* d_sino, float lambda, int32_t n_fgp, float* d_cores, void* stream);

/* Extended-ROI results of the last solve: [local_count][2h][2h], the valid
 * part top-left aligned, zeros elsewhere (for stage-wise parity). */
int lt_get_ext(const lt_plan* plan, float* d_ext, void* stream);

/* Combine ("combined ... by tiling"; A19):
 * d_image (N x N, device) = the mean of the cores covering each pixel, summed in
 * ascending global ROI order, 0 where no core covers -- on EVERY rank.
 *  d_cores: this rank's cores [local_count][2r][2r] (lt_sirt_solve / lt_tv_solve).
 *  nccl_comm: an ncclComm_t of the plan's `world` ranks with this process at the
 *    plan's `rank` (lt_nccl_comm_init); may be NULL when world == 1.
 * For world > 1 the cores go into fixed slots of the largest local count
 * (lt_plan_slot_table; the partition is the same on every rank, so no table is
 * exchanged), one in-place ncclAllGather runs on `stream`, then the stitch
 * kernel: the image is bitwise identical for every world size.  All ranks must
 * call it (collective).  Errors: 2 null pointers, missing communicator for
 * world > 1, communicator size / rank different from the plan's; 1 CUDA or
 * NCCL failures (including NCCL not loadable). */
int lt_combine_rois(const lt_plan* plan, const float* d_cores, float* d_image, void* nccl_comm, void* stream);

/* NCCL communicator for lt_combine_rois (created with
 * ncclCommInitRank after the unique id is exchanged, e.g. by
 * torch.distributed.broadcast of the LT_NCCL_ID_BYTES bytes from rank 0).
 * lt_nccl_comm_init binds the communicator to the CURRENT device (set it
 * first).  The library resolves NCCL from libnccl.so.2 at first use. */
#define LT_NCCL_ID_BYTES 128
int lt_nccl_get_unique_id(void* h_id);
int lt_nccl_comm_init(int32_t world, int32_t rank, const void* h_id, void** comm);
int lt_nccl_comm_destroy(void* comm);

/* The partition's slot table: h_slot_roi[world * spr] = the global ROI index of
 * rank g's q-th local ROI at g * spr + q (-1 = empty); *h_spr = spr = the
 * largest local count.  Either pointer may be NULL (query spr first). */
int lt_plan_slot_table(const lt_plan* plan, int32_t* h_slot_roi, int32_t* h_spr);

/* Stitch already-gathered cores (the stitch step of lt_combine_rois without the
 * collective, e.g. after the caller's own all-gather): d_image (N x N) = mean of
 * the cores covering each pixel in ascending global ROI order, 0 where uncovered.
 * d_cores_all: [n_slots][2r][2r]; h_slot_roi: host, the global ROI index of each
 * slot (-1 = empty). */
int lt_stitch_slots(const lt_plan* plan, const float* d_cores_all, int32_t n_slots,
                    const int32_t* h_slot_roi, float* d_image, void* stream);

/* LT_GUARD_BANDS plans only: synchronizes `stream`, then compares every canary
 * band with its fill pattern: *h_damaged = the number of damaged bands (0 =
 * every band intact), *h_bad_offset (nullable) = the workspace byte offset of
 * the first damaged byte (-1 if none).  Errors: 2 for a plan without guard
 * bands, unbound or a null h_damaged; 1 on a CUDA error. */
int lt_guard_check(const lt_plan* plan, int32_t* h_damaged, int64_t* h_bad_offset, void* stream);

/* Window width W(h) = 2 ceil((2h-1)/sqrt2) + 4 of an extended half-side h
 * (V4): the detector bins every ROI window holds per angle. */
int32_t lt_window_width(int32_t h);

/* Combine over peer memory (the all-gather and the stitch in one
 * kernel): like lt_stitch_slots, but slot s of the gathered layout is read in
 * place from rank s / slots_per_rank's core buffer, h_peer_cores[rank]
 * (a host array of `world` <= 64 DEVICE pointers valid in this process: the
 * own buffer and the others' buffers mapped with lt_ipc_open_handle, read over
 * NVLink), at index s % slots_per_rank ([slots_per_rank][2r][2r] each).
 * h_slot_roi: the global ROI of each of the world * slots_per_rank slots
 * (-1 = empty).  The caller orders the peers' solves before this call (e.g. a
 * stream sync + process-group barrier) and this call before the peers
 * overwrite their buffers.  Same image, bitwise, as lt_stitch_slots on the
 * all-gathered cores (the peer-memory counterpart of lt_combine_rois, used by
 * bench.py for N > 1).  Errors (2): null pointers, world outside 1..64. */
int lt_combine_peers(const lt_plan* plan, const float* const* h_peer_cores, int32_t world, int32_t slots_per_rank,
                     const int32_t* h_slot_roi, float* d_image, void* stream);

/* CUDA IPC for lt_combine_peers: the 64-byte handle of a device allocation
 * (h_handle: host buffer of 64 bytes), opening a peer's handle in this process
 * (peer access over NVLink enabled lazily) and closing it. */
int lt_ipc_get_handle(const void* d_ptr, void* h_handle);
int lt_ipc_open_handle(const void* h_handle, void** d_ptr);
int lt_ipc_close(void* d_ptr);

/* End-to-end entry with HOST buffers (pinned recommended): copies h_sino in,
 * runs lt_sirt_solve (mode 0) or lt_tv_solve (mode 1), combines this rank's
 * cores into h_image (N x N).  Synchronous. */
int lt_solve_host(lt_plan* plan, int32_t mode, const float* h_sino, float p0, float p1,
                  int32_t n_fgp, float* h_image, void* stream);

/* Global solvers the method approximates: box-SIRT
 * (eq. sirtbox) and FISTA-TV on the full grid, from 0. */
int lt_global_sirt(lt_plan* plan, const float* d_sino, int32_t n_iter, float lo, float hi,
                   float* d_img, void* stream);
int lt_global_tv(lt_plan* plan, const float* d_sino, int32_t n_iter, float lambda, int32_t n_fgp,
                 float* d_img, void* stream);

/* Exterior subtraction (the prior art of P:L140-146,
 * "subtracting simulated projections of a global reconstruction outside the
 * region of interest from the acquired projections"), for comparison with the
 * paper's method: the global reconstruction is xg = W^T C_{u_n} p_c + c D (FBP
 * with the SIRT filter of Alg. 1, eq. sfbp, disc per the plan's
 * flags; needs the filter bank), then for every local ROI box-SIRT on its
 * extended rect L' (eq. sirtbox, n_iter iterations from 0) with the data
 * p - W M_F xg.  d_cores as lt_sirt_solve.  Errors (2): lo > hi, null
 * pointers, no bank. */
int lt_exterior_solve(lt_plan* plan, const float* d_sino, float lo, float hi, float* d_cores, void* stream);

/* Chambolle-Pock primal-dual TV solver with diagonal (row / column sum)
 * preconditioning on the full grid (the north
 * star's literal "TV-regularized primal-dual solver"; P:L351-353 names
 * primal-dual methods; global only, since it is not a "SIRT step +
 * correction" method): minimises 1/2 ||W x - p||^2 +
 * mu ||grad x||_1 (anisotropic, Neumann; mu = lambda / alpha gives the
 * objective of lt_global_tv, reading A14), from x = 0, n_iter iterations.
 * d_img: N x N.  Errors (2): n_iter < 1, mu < 0 or NaN, null pointers. */
int lt_global_cp(lt_plan* plan, const float* d_sino, int32_t n_iter, float mu, float* d_img, void* stream);

/* FGP TV prox (Beck & Teboulle) on `count` independent h x w
 * images (d_in/d_out: count x h x w), same kernel the TV solve uses
 * (h, w <= 256). */
int lt_fgp_batch(int32_t h, int32_t w, int32_t count, const float* d_in, float lambda,
                 int32_t n_fgp, float* d_out, void* stream);

/* Local reconstruction with the Haar-wavelet l1 prior (
 * g(x) = ||Bx||_1 in a Haar basis; eq. sirtista, solved
 * with FISTA as in the paper, or ISTA when momentum = 0): Alg. 3
 * with the FGP replaced by x = B^{-1} P_lambda(B v), B the orthonormal 2D Haar
 * transform with `levels` levels and P_lambda the symmetric soft threshold of
 * every coefficient.  0 <= levels <= 5; every local ROI's
 * extended rectangle (after clipping) must have both sides divisible by
 * 2^levels, else error 2.  d_cores as lt_tv_solve. */
int lt_haar_solve(lt_plan* plan, const float* d_sino, float lambda, int32_t levels, int32_t momentum,
                  float* d_cores, void* stream);

/* Lambda sweep (P:L789-795 tune lambda per reconstruction,
 * P:L1116-1120 "the same ... for many different parameter values"): the local
 * FISTA-TV solve of lt_tv_solve with lambda = h_lambdas[q] (host array, one
 * value >= 0 per LOCAL ROI q, in lt_plan_local_rois order) — every ROI of the
 * plan may be the same region repeated with another lambda; the ROIs share the
 * filter bank, the conv cache and the global x_s backprojection.  Errors as
 * lt_tv_solve, plus 2 for a negative or NaN lambda. */
int lt_tv_solve_lambdas(lt_plan* plan, const float* d_sino, const float* h_lambdas, int32_t n_fgp,
                        float* d_cores, void* stream);

/* Quality inside the ROI: for each of `count`
 * image pairs (d_x[i], d_ref[i], each h x w row-major, device) d_mse[i] =
 * mean (x - ref)^2 and d_ssim[i] = mean SSIM (Wang et al. 2004: 11 x 11
 * Gaussian window with sigma 1.5, weights normalised, K1 = 0.01, K2 = 0.03,
 * population moments, mean over the window positions inside the image — 0
 * when h or w < 11) with dynamic range L = data_range if > 0, else
 * max(ref_i) - min(ref_i).  d_mse, d_ssim: device double[count].  Errors (2):
 * count < 0, h or w < 1, null pointers. */
int lt_metrics(const float* d_x, const float* d_ref, int32_t count, int32_t h, int32_t w, float data_range,
               double* d_mse, double* d_ssim, void* stream);

/* One-dimensional Nelder-Mead ("using the Nelder-Mead method")
 * minimising f(t, ctx) over t in [t_lo, t_hi] (the caller's t, e.g. log10 of
 * lambda): initial simplex {mid, mid + 0.5}, reflection 1, expansion 2,
 * contraction 1/2, shrink 1/2, every trial point clamped into the bounds, at
 * most `budget` evaluations (the 2 initial ones included).  Host-only and
 * deterministic; writes the best evaluated point and value and the number of
 * evaluations.  Errors (2): null f/outputs, t_lo >= t_hi, budget < 3. */
int lt_nelder_mead_1d(double (*f)(double, void*), void* ctx, double t_lo, double t_hi, int32_t budget,
                      double* t_best, double* f_best, int32_t* n_eval);

/* Truncated projection data ("simply
 * padding the acquired data", constant padding P:L1148): each of the
 * n_angles rows of d_in (n_trunc measured central bins, row-major
 * [n_angles][n_trunc]) is extended on both sides with its edge value to n_det
 * bins, centred: d_out[a][d] = d_in[a][clamp(d - (n_det - n_trunc)/2, 0,
 * n_trunc - 1)] ([n_angles][n_det]).  The result is an ordinary sinogram of the
 * plan's geometry.  Errors (2): n_angles < 1, n_trunc < 1, n_det < n_trunc,
 * n_det - n_trunc odd (no centred padding), null pointers. */
int lt_pad_truncated(const float* d_in, int32_t n_angles, int32_t n_trunc, int32_t n_det, float* d_out,
                     void* stream);

/* Number of kernels this library has launched so far (process-wide). */
int64_t lt_launch_count(void);

/* Per-kernel-class device timing (bench.py's roofline): when enabled, every
 * launch of the Joseph forward (class 0), ROI / global-iteration
 * backprojection (1), FGP (2), convolution (3) and block-listed global x_s
 * backprojection (4, the side-stream M_{L'} W^T b_k of Alg. 3) kernels is
 * bracketed by CUDA events recorded on its launch stream.  lt_timing_read
 * synchronizes on the recorded events, writes the summed milliseconds and
 * launch counts per class (host arrays of 5) and clears the records.  Timing
 * disables the CUDA-graph replay of the local iterations. */
void lt_timing_enable(int32_t on);
int lt_timing_read(double* h_ms, int64_t* h_count);

void lt_plan_destroy(lt_plan* plan);
const char* lt_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LOCTOMO_H */
