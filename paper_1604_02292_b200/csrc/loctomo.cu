// loctomo.cu -- C-ABI (include/loctomo.h), host planner and launch logic of
// the B200-native local tomography library (arXiv 1604.02292).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -shared.
#include "loctomo.h"
#include "kernels.cuh"

#include <cufft.h>
#include <nvtx3/nvToolsExt.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

using namespace lt;

namespace {

thread_local std::string g_err;
std::atomic<long long> g_launches{0};

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define LT_CUDA(call)                                                                     \
    do {                                                                                  \
        cudaError_t e_ = (call);                                                          \
        if (e_ != cudaSuccess) return fail(LT_ERR_RUNTIME, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

#define LT_LAUNCHED()                                                                     \
    do {                                                                                  \
        g_launches.fetch_add(1, std::memory_order_relaxed);                               \
        cudaError_t e_ = cudaGetLastError();                                              \
        if (e_ != cudaSuccess) return fail(LT_ERR_RUNTIME, "launch: %s", cudaGetErrorString(e_)); \
    } while (0)

size_t align256(size_t x) { return (x + 255) & ~size_t(255); }
constexpr int LT_MAX_PEERS = 64;
constexpr int LT_MAX_DEV = 64;      // per-device caches (occupancy, __constant__ tables) are indexed by ordinal
constexpr unsigned char kGuardByte = 0xA5;   // LT_GUARD_BANDS canary

// the calling thread's current device (every launch goes to it); -1 on error
int cur_dev() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= LT_MAX_DEV) { cudaGetLastError(); return -1; }
    return d;
}
std::mutex g_dev_mu;                // guards the per-device __constant__ uploads

// ---- optional per-kernel-class timing (CUDA events on the launch stream) ----
enum { TC_FP = 0, TC_BP = 1, TC_FGP = 2, TC_CONV = 3, TC_XS = 4, TC_N = 5 };
struct TimerRec { int cls; cudaEvent_t a, b; };
bool g_timing = false;
std::vector<TimerRec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t ev_get() {
    if (!g_pool.empty()) { cudaEvent_t e = g_pool.back(); g_pool.pop_back(); return e; }
    cudaEvent_t e = nullptr;
    cudaEventCreate(&e);
    return e;
}
// NVTX ranges around the library's phases (header-only NVTX v3: a no-op
// unless a profiler is attached) -- SURVEY §5 tracing
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

struct ScopedTimer {
    int cls; cudaStream_t st; cudaEvent_t a = nullptr;
    ScopedTimer(int c, cudaStream_t s) : cls(c), st(s) {
        if (g_timing) { a = ev_get(); cudaEventRecord(a, st); }
    }
    ~ScopedTimer() {
        if (a) { cudaEvent_t b = ev_get(); cudaEventRecord(b, st); g_recs.push_back({cls, a, b}); }
    }
};

// NCCL (lt_combine_rois): resolved from libnccl.so.2 on first use, so the
// library loads without it; under PyTorch this is the NCCL torch already loaded
struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*commUserRank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*errStr)(ncclResult_t) = nullptr;
};
NcclApi& nccl_api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) { a.why = std::string("dlopen libnccl.so.2: ") + dlerror(); return; }
        a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
        a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
        a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
        a.commCount = (decltype(a.commCount))dlsym(h, "ncclCommCount");
        a.commUserRank = (decltype(a.commUserRank))dlsym(h, "ncclCommUserRank");
        a.allGather = (decltype(a.allGather))dlsym(h, "ncclAllGather");
        a.errStr = (decltype(a.errStr))dlsym(h, "ncclGetErrorString");
        a.ok = a.getUniqueId && a.commInitRank && a.commDestroy && a.commCount && a.commUserRank && a.allGather &&
               a.errStr;
        if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    });
    return a;
}

#define LT_NCCL(call)                                                                     \
    do {                                                                                  \
        ncclResult_t r_ = (call);                                                         \
        if (r_ != ncclSuccess) return fail(LT_ERR_RUNTIME, "%s: %s", #call, nccl_api().errStr(r_)); \
    } while (0)

}  // namespace

struct lt_plan {
    int n = 0, na = 0, nd = 0, nroi_all = 0, radius = 0, margin = 0, h = 0;
    int T = 0, TP = 0, Wwin = 0, n_iter = 0, flags = 0, rank = 0, world = 1;
    int GT = 0, GTP = 0;          // global tile (whole image)
    int num_sms = 148;            // of the bound device (launch sizing)
    long long bpart_cap = 0;      // floats of the angle-split backprojection partials (small batches)
    int a_lo = 0, a_hi = 0;       // global projections restricted to angles [a_lo, a_hi) (angle-split bank; 0: all)
    int split_a0 = 0, split_a1 = 0;   // this rank's angles in the angle-split bank
    bool split_rows_ready = false;    // all steps of the angle-split bank issued (own rows valid)
    int gsplit_a0 = 0, gsplit_a1 = 0; // this rank's angles in the angle-split global SIRT
    long long fpart_cap = 0;      // floats of the band-split forward-projection partials
    double alpha = 0.0;
    std::vector<double> ang;
    std::vector<int> cen;         // [nroi_all][2]
    std::vector<int> local;       // global ROI indices on this rank (ascending)
    int R = 0;
    // the whole partition (every rank computes the same one): slots_per_rank =
    // the largest local count; slot_all[g * spr + q] = rank g's q-th ROI (-1 empty)
    int spr = 1;
    std::vector<int> slot_all;
    // host tables
    std::vector<AngF> angf;
    std::vector<double> cs64, sn64, A64, B64;
    std::vector<TileT> tiles, gtile, ttiles;
    std::vector<int> d0, gd0, td0;
    std::vector<double> tauc, gtauc, ttauc;
    // tiled global forward projection: the grid cut into Tg x Tg tiles, each
    // projected by the ROI kernel onto its window, windows summed per bin
    int Tg = 0, TPg = 0, Wg = 0, NTg = 0;
    std::vector<int> fpgroups;    // [ngroups][16] angle indices of one orientation, -1 padded (2 per warp)
    std::vector<int> fpgroups1;   // [ngroups1][8] the same, one angle per warp
    std::vector<int> fpgroups24;  // [ngroups24][24] the same, 12 warps x 2 angles
    // BP_SUB^2 image blocks that the global x_s^k backprojection must cover: list 0 for
    // all local ROIs, lists 1 and 2 for the two pipelined ROI groups (halves)
    std::vector<int> xsblk[3];
    int ngroups = 0, ngroups1 = 0, ngroups24 = 0;
    // workspace
    char* ws = nullptr;
    int64_t ws_bytes = 0;
    std::vector<std::pair<size_t, size_t>> guards;   // LT_GUARD_BANDS: (offset, bytes) canary bands
    bool bound = false, bank_ready = false, wd_ready = false;
    int last_mode = -1;
    bool lam_array = false;       // tv solve with per-ROI lambda (lt_tv_solve_lambdas)
    bool haar_momentum = true;    // Haar solve: FISTA (true) or ISTA (false) update
    // convolution cache by FFT (cuFFT, library): length L >= 2 N_d - 1, k chunk,
    // plans with their work area in the workspace, bank spectra U_k / L
    int fftL = 0, fftF = 0, fft_kc = 0;
    size_t fwork_bytes = 0;
    cufftHandle plan_r2c_p = 0, plan_r2c_k = 0, plan_c2r_k = 0;
    bool spec_ready = false;
    // CUDA graph of the local iteration loop (replayed while its key is unchanged)
    cudaGraphExec_t gexec = nullptr;
    double gkey[10] = {0};
    long long g_nlaunch = 0;
    cudaStream_t gs = nullptr;                       // capture / replay stream (the caller's may be the legacy one)
    cudaEvent_t gev_in = nullptr, gev_out = nullptr;
    // side stream for the global x_s backprojection of the NEXT iteration (it
    // only waits for the ROI BP that read the previous x_s, so it overlaps the
    // FGP and the forward projection; LT_XS_OVERLAP=0 disables)
    cudaStream_t xst = nullptr;
    cudaEvent_t xev_bp = nullptr, xev_xs = nullptr;
    int stitch_cap = 0;           // max list entries
    // the stitch tables last uploaded to the workspace, keyed by the slot table
    // (and the peer pointers): repeated combines of the same layout skip the upload
    mutable std::vector<long long> st_key;
    // ROI-batch pipelining: the local ROIs are split into groups whose
    // iteration chains run on separate streams and overlap on the device
    int nsplit = 1;
    int split_at = 0;               // first ROI of the second group (two-group pipelining)
    cudaStream_t gst[2] = {nullptr, nullptr};        // per group: projector work (low priority)
    cudaStream_t fst[2] = {nullptr, nullptr};        // per group: FGP (high priority)
    cudaEvent_t gev[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t pev[2] = {nullptr, nullptr}, fev[2] = {nullptr, nullptr}, bpev[2] = {nullptr, nullptr};
    struct {
        size_t angf, cs64, sn64, A64, B64, tiles, d0, tauc, gtile, gd0, gtauc, fpgroups, fpgroups1, fpgroups24, bpart, fpart;
        size_t bank, conv, pc, wd, wdsum, psum, discc64, discc32, err;
        size_t gimg, gimgT, gsino, gsino2, gplain, gr, gs, gpo, gqo, gz, gxprev;
        size_t y, yT, s, v, xs, xprev;
        size_t xsblk[3], xsg[2], lams;
        size_t uhat, phat, fspec, freal, fwork;
        size_t cp_sd, cp_tau, cp_yd, dwin, peers;
        size_t ttiles, td0, ttauc, tstack, tstackT, twin;
        size_t tt, ttT, tw;
        size_t st_off, st_lst, st_r0, st_c0, cores, hsino, himg, gather;
        size_t total;
    } off{};

    template <class X> X* P(size_t o) const { return reinterpret_cast<X*>(ws + o); }
    Geo geo() const {
        return Geo{n, na, nd, P<AngF>(off.angf), P<double>(off.cs64), P<double>(off.sn64),
                   P<double>(off.A64), P<double>(off.B64)};
    }
    Tiles roi_tiles() const { return Tiles{T, TP, Wwin, R, P<TileT>(off.tiles), P<int>(off.d0), P<double>(off.tauc)}; }
    Tiles glob_tiles() const { return Tiles{GT, GTP, nd, 1, P<TileT>(off.gtile), P<int>(off.gd0), P<double>(off.gtauc)}; }
    Tiles tile_tiles() const { return Tiles{Tg, TPg, Wg, NTg, P<TileT>(off.ttiles), P<int>(off.td0), P<double>(off.ttauc)}; }
    long long ytile() const { return (long long)T * TP; }
    long long ptile() const { return (long long)T * T; }
};

namespace {

int window_width(int h) {
    // W(h) = 2 ceil((2h-1)/sqrt2) + 4 (V4): covers the support of every
    // pixel of a 2h x 2h tile at every angle.
    return 2 * (int)std::ceil((2.0 * h - 1.0) / std::sqrt(2.0) - 1e-12) + 4;
}

void tile_window(const lt_plan& p, double cx, double cy, int Wwin, int* d0_out, double* tauc_out) {
    // cx, cy: coordinates of the tile centre point; tau = x cos + y sin + (N_d-1)/2
    for (int a = 0; a < p.na; ++a) {
        const double tau = cx * p.cs64[a] + cy * p.sn64[a] + 0.5 * (p.nd - 1);
        const int d0 = (int)std::floor(tau) - Wwin / 2;
        d0_out[a] = d0;
        tauc_out[a] = tau - d0;
    }
}

int check_plan(const lt_plan* p) {
    if (!p) return fail(LT_ERR_INVALID, "null plan");
    if (!p->bound) return fail(LT_ERR_INVALID, "workspace not bound");
    return LT_OK;
}

// ---- launch helpers -------------------------------------------------------
int launch_fp(const lt_plan& p, int mode, const Tiles& t, const float* img, const float* imgT, long long img_ts,
              float* out, long long out_ts, const float* aux_in, float* aux_out, cudaStream_t st) {
    FpArgs f{img, imgT, img_ts, out, out_ts, aux_in, aux_out, (float)p.alpha};
    dim3 grid((t.Wwin + 127) / 128, p.na, t.ntiles);
    ScopedTimer tm(TC_FP, st);
    if (mode == 0) k_fp<0><<<grid, 128, 0, st>>>(p.geo(), t, f);
    else if (mode == 1) k_fp<1><<<grid, 128, 0, st>>>(p.geo(), t, f);
    else k_fp<2><<<grid, 128, 0, st>>>(p.geo(), t, f);
    LT_LAUNCHED();
    return LT_OK;
}

// Split factor of a launch with `ctas` CTAs whose work divides into `units`
// equal parts (bands, angle chunks): the s in [1, smax] minimising rounds x
// units per CTA, rounds = ceil(ctas s / resident) (ties: the smaller s, less
// joining).  `resident` = CTAs of the kernel co-resident on the device.
int best_split(long long ctas, int units, long long resident, int smax) {
    int best = 1;
    long long best_cost = LLONG_MAX;
    for (int sp = 1; sp <= std::max(1, std::min(smax, units)); ++sp) {
        const long long rounds = (ctas * sp + resident - 1) / std::max(1LL, resident);
        const long long cost = rounds * ((units + sp - 1) / sp);
        if (cost < best_cost) { best_cost = cost; best = sp; }
    }
    return best;
}

template <typename Kern>
long long resident_ctas(const lt_plan& p, Kern kern, int threads, size_t smem) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem) != cudaSuccess) {
        cudaGetLastError();
        per_sm = 1;
    }
    return (long long)std::max(1, per_sm) * p.num_sms;
}

bool fp_force24() {   // diagnostics: 24-angle CTAs even where they pad more than the 16-angle ones
    static int v = -1;
    if (v < 0) { const char* e = getenv("LT_FP_24"); v = (e && atoi(e) == 1) ? 1 : 0; }
    return v != 0;
}

bool fp_wide() {
    static int v = -1;
    if (v < 0) { const char* e = getenv("LT_FP_WIDE"); v = !(e && atoi(e) == 0); }
    return v != 0;
}

// ROI-batch forward projection (shared-memory staged k_fp_roi2; the
// single-pass k_fp for tiles wider than its band)
int launch_fp_roi(const lt_plan& p, const Tiles& t, const float* img, const float* imgT, long long img_ts,
                  float* out, long long out_ts, cudaStream_t st) {
    if (t.TP > FP2_PW || t.Wwin > 32 * FP_UW)
        return launch_fp(p, 0, t, img, imgT, img_ts, out, out_ts, nullptr, nullptr, st);
    if (t.TP > FP2_P || t.Wwin > 32 * FP_U) {
        // wide tiles (up to 320: the paper's 256^2 parts with 1/8 padding): 8 warps x
        // 1 angle, 336-entry staged lines, 15 rays per lane; bands split over CTAs
        // when a launch is under one wave (as below)
        const size_t smemw = (size_t)FP2_BL * fp_line(FP2_PW, 1) * sizeof(float2) + (size_t)8 * 32 * FP_UW * sizeof(float);
        auto kw = k_fp_roi2<1, 8, FP2_PW, FP_UW>;
        LT_CUDA(cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smemw));
        FpArgs f{img, imgT, img_ts, out, out_ts, nullptr, nullptr, (float)p.alpha, nullptr, 1, p.a_lo, p.a_hi};
        ScopedTimer tm(TC_FP, st);
        const long long ctas = (long long)p.ngroups1 * t.ntiles;
        const int nbands = (t.T + FP2_BL - 1) / FP2_BL;
        static long long resident_dev[LT_MAX_DEV] = {};
        const int dv = std::max(0, cur_dev());
        if (!resident_dev[dv]) resident_dev[dv] = resident_ctas(p, kw, 256, smemw);
        int nsplit = 1;
        if (ctas < resident_dev[dv] && p.nsplit <= 1 && nbands >= 8) nsplit = best_split(ctas, nbands, resident_dev[dv], 8);
        if (nsplit > 1 && (long long)nsplit * t.ntiles * p.na * t.Wwin <= p.fpart_cap) {
            f.part = p.P<float>(p.off.fpart); f.nsplit = nsplit;
            kw<<<dim3(p.ngroups1, t.ntiles, nsplit), 256, smemw, st>>>(p.geo(), t, f, p.P<int>(p.off.fpgroups1));
            LT_LAUNCHED();
            k_fp_join<<<dim3((t.Wwin + 127) / 128, p.na, t.ntiles), 128, 0, st>>>(p.geo(), t, f);
        } else {
            kw<<<dim3(p.ngroups1, t.ntiles), 256, smemw, st>>>(p.geo(), t, f, p.P<int>(p.off.fpgroups1));
        }
        LT_LAUNCHED();
        return LT_OK;
    }
    // 16 angles per CTA share each staged band; 8 when that would leave the
    // SMs short of two waves (small ROI batches: C1-C3, T1, 8-GPU shards)
    static int one_env = -2;
    if (one_env == -2) { const char* e = getenv("LT_FP_ONE"); one_env = (e && *e) ? atoi(e) : -1; }   // diagnostics: 0 / 1 force
    bool one = one_env >= 0 ? one_env == 1 : (long long)p.ngroups * t.ntiles < 2LL * 3 * p.num_sms;
    // ... but the 24-angle CTAs when they pad the angles by <= 10 % and still fill
    // >= 3/4 of a wave (a C4 shard of 32 ROIs on 8 GPUs: 256 CTAs for 296 slots,
    // FP 0.236 -> 0.223 ms; C2 / C3 pad 32 / 64 angles to 48 / 96 and keep 8)
    bool small24 = false;
    if (one && one_env < 0 && fp_wide() && 10 * p.ngroups24 * 24 <= 11 * p.na && p.ngroups24 * 24 <= p.ngroups * 16) {
        static long long r24_dev[LT_MAX_DEV] = {};
        const int dv = std::max(0, cur_dev());
        if (!r24_dev[dv]) {
            const size_t smem3 = (size_t)FP2_BL * fp_line(FP2_P, 2) * sizeof(float2) + (size_t)24 * 32 * FP_U * sizeof(float);
            LT_CUDA(cudaFuncSetAttribute(k_fp_roi2<2, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
            r24_dev[dv] = resident_ctas(p, k_fp_roi2<2, 12>, 384, smem3);
        }
        if (4LL * p.ngroups24 * t.ntiles >= 3LL * r24_dev[dv]) { one = false; small24 = true; }
    }
    const int apw = one ? 1 : 2;
    const size_t smem2 = (size_t)FP2_BL * fp_line(FP2_P, apw) * sizeof(float2) + (size_t)8 * apw * 32 * FP_U * sizeof(float);
    FpArgs f{img, imgT, img_ts, out, out_ts, nullptr, nullptr, (float)p.alpha, nullptr, 1, p.a_lo, p.a_hi};
    ScopedTimer tm(TC_FP, st);
    if (one) {
        LT_CUDA(cudaFuncSetAttribute(k_fp_roi2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        // at most one CTA per SM (single ROIs: T1): split the 16-line bands over
        // nsplit CTAs per (tile, angle group), joined by k_fp_join in split order
        const long long ctas = (long long)p.ngroups1 * t.ntiles;
        const int nbands = (t.T + FP2_BL - 1) / FP2_BL;
        int nsplit = 1;
        static long long resident_dev[LT_MAX_DEV] = {};
        const int dv = std::max(0, cur_dev());
        if (!resident_dev[dv]) resident_dev[dv] = resident_ctas(p, k_fp_roi2<1>, 256, smem2);
        const long long resident = resident_dev[dv];
        if (ctas < resident && p.nsplit <= 1 && nbands >= 8)   // less than one wave; tiny tiles (C1: 3 bands) keep one launch
            nsplit = best_split(ctas, nbands, resident, 8);      // T1: 64 CTAs x 6 = one wave of 3 bands
        if (nsplit > 1 && (long long)nsplit * t.ntiles * p.na * t.Wwin <= p.fpart_cap) {
            f.part = p.P<float>(p.off.fpart); f.nsplit = nsplit;
            k_fp_roi2<1><<<dim3(p.ngroups1, t.ntiles, nsplit), 256, smem2, st>>>(p.geo(), t, f, p.P<int>(p.off.fpgroups1));
            LT_LAUNCHED();
            k_fp_join<<<dim3((t.Wwin + 127) / 128, p.na, t.ntiles), 128, 0, st>>>(p.geo(), t, f);
        } else {
            k_fp_roi2<1><<<dim3(p.ngroups1, t.ntiles), 256, smem2, st>>>(p.geo(), t, f, p.P<int>(p.off.fpgroups1));
        }
    } else if (fp_wide() && ((long long)p.ngroups24 * t.ntiles >= 2LL * 2 * p.num_sms || one_env == 0 || small24) &&
               (5 * p.ngroups24 * 24 <= 6 * p.na || fp_force24())) {
        // 12 warps x 2 angles: each staged band shared by 24 angles (2 CTAs per SM),
        // unless the 24-angle groups pad the angles by more than 20 % (C5's 128 angles
        // per orientation = 5 1/3 x 24: 12.5 %, measured 134.1 vs 132.4 ROI solves/s
        // against the 16-angle CTAs since the staged lines carry zero margins)
        const size_t smem3 = (size_t)FP2_BL * fp_line(FP2_P, 2) * sizeof(float2) + (size_t)24 * 32 * FP_U * sizeof(float);
        LT_CUDA(cudaFuncSetAttribute(k_fp_roi2<2, 12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3));
        k_fp_roi2<2, 12><<<dim3(p.ngroups24, t.ntiles), 384, smem3, st>>>(p.geo(), t, f, p.P<int>(p.off.fpgroups24));
    } else {
        LT_CUDA(cudaFuncSetAttribute(k_fp_roi2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2));
        k_fp_roi2<2><<<dim3(p.ngroups, t.ntiles), 256, smem2, st>>>(p.geo(), t, f, p.P<int>(p.off.fpgroups));
    }
    LT_LAUNCHED();
    return LT_OK;
}

// Global forward projection W x of a padded global image (+ twin): the grid is
// cut into Tg x Tg tiles (k_extract_tiles), every tile is projected onto its
// detector window by the shared-memory ROI projector (k_fp_roi2), and k_winsum
// adds the windows per bin in fixed tile order, with the k_fp epilogues
// (mode 0: W x; 1: Alg. 1 bank update; 2: p - W x).  LT_GFP=direct keeps the
// single-pass k_fp.
int global_fp(const lt_plan& p, int mode, const float* img, const float* imgT, float* out, const float* aux_in,
              float* aux_out, cudaStream_t st) {
    static int direct = -1;
    if (direct < 0) { const char* e = getenv("LT_GFP"); direct = (e && !strcmp(e, "direct")) ? 1 : 0; }
    if (direct || p.TPg > FP2_P || p.Wg > 32 * FP_U) {
        if (p.a_hi > 0) return fail(LT_ERR_INVALID, "angle-restricted projection needs the tiled global projector");
        return launch_fp(p, mode, p.glob_tiles(), img, imgT, 0, out, 0, aux_in, aux_out, st);
    }
    const Tiles tt = p.tile_tiles();
    float* stack = p.P<float>(p.off.tstack);
    float* stackT = p.P<float>(p.off.tstackT);
    float* win = p.P<float>(p.off.twin);
    const long long ts = (long long)p.Tg * p.TPg;
    k_extract_tiles<<<dim3((p.Tg + 31) / 32, (p.Tg + 7) / 8, p.NTg), dim3(32, 8), 0, st>>>(
        p.Tg, p.TPg, tt.tile, img, p.GTP, stack, stackT, ts);
    LT_LAUNCHED();
    if (int rc = launch_fp_roi(p, tt, stack, stackT, ts, win, (long long)p.na * p.Wg, st)) return rc;
    const int a_off = p.a_hi > 0 ? p.a_lo : 0, a_cnt = p.a_hi > 0 ? p.a_hi - p.a_lo : p.na;
    k_winsum<<<dim3((p.nd + 255) / 256, a_cnt), 256, p.NTg * sizeof(int), st>>>(
        mode, p.na, p.nd, p.Wg, p.NTg, tt.d0, win, out, aux_in, aux_out, (float)p.alpha, a_off);
    LT_LAUNCHED();
    return LT_OK;
}

// 64 x 64 sub-tiles per CTA; 32 x 32 when a batch would give fewer than about
// two waves of 64 x 64 CTAs (small ROI counts: C2, C3, 8-GPU shards), so the
// SMs stay busy (block lists are in 64 x 64 units: a listed block becomes four
// 32 x 32 CTAs)
template <int NS, int MODE>
int launch_bp_t(const lt_plan& p, const Tiles& t, const SinoView& s1, const SinoView& s2, const BpEpi& e,
                cudaStream_t st, int nblist = 0) {
    if (e.blist && nblist == 0) return LT_OK;
    const int nsx = (t.T + BP_SUB - 1) / BP_SUB;
    const long long ctas64 = e.blist ? nblist : (long long)nsx * nsx * t.ntiles;
    ScopedTimer tm(e.blist ? TC_XS : TC_BP, st);   // block-listed launches: the global x_s backprojection
    static int sub_env = -1;
    if (sub_env < 0) { const char* v = getenv("LT_BP_SUB"); sub_env = v ? atoi(v) : 0; }
    // 32x32 below two waves of 64x64 CTAs for the block-listed x_s, below one
    // wave for the ROI backprojection (a C4 shard of 34 ROIs on 8 GPUs: 544
    // CTAs of 64x64 take 0.18 ms, 2176 of 32x32 0.21 ms)
    const long long lim32 = (e.blist ? 2LL : 1LL) * 3 * p.num_sms;
    if (sub_env == 32 || (sub_env != 64 && ctas64 < lim32)) {
        const int nsx32 = (t.T + 31) / 32;
        const dim3 grid(e.blist ? 4 * nblist : nsx32 * nsx32, t.ntiles);
        // at most one CTA per SM (single ROIs: T1, the x_s blocks of one ROI):
        // split the angles over nsa CTAs per block (stage 1: partial sums;
        // stage 2: their ordered sum + the epilogue).  Measured: T1 ROI BP 76 ->
        // 36 us; with 2 CTAs per SM already (C2) the extra pass costs more than it gains
        const long long ctas = (long long)grid.x * grid.y;
        // (one partial buffer per plan: not with two concurrent ROI groups, LT_SPLIT)
        const int nang = e.a_hi > 0 ? e.a_hi - e.a_lo : p.na;
        int nsa = 1;
        if (NS > 0 && p.bpart_cap > 0 && p.nsplit <= 1 && ctas <= p.num_sms) {
            static long long resident_dev[LT_MAX_DEV] = {};
            const int dv = std::max(0, cur_dev());
            if (!resident_dev[dv]) resident_dev[dv] = resident_ctas(p, k_bp<NS, MODE, 32>, 256, 0);
            const long long resident = resident_dev[dv];
            nsa = best_split(ctas, (nang + BP_CA - 1) / BP_CA, resident, 8);
        }
        const int achunk = ((nang + nsa - 1) / nsa + BP_CA - 1) / BP_CA * BP_CA;
        nsa = (nang + achunk - 1) / achunk;
        if (nsa > 1 && (long long)nsa * ctas * 32 * 32 <= p.bpart_cap) {
            BpEpi e1 = e;
            e1.part = p.P<float>(p.off.bpart); e1.nsa = nsa; e1.achunk = achunk;
            e1.stage = 1;
            k_bp<NS, MODE, 32><<<dim3(grid.x, grid.y, nsa), 256, 0, st>>>(p.geo(), t, s1, s2, e1);
            LT_LAUNCHED();
            e1.stage = 2;
            k_bp<NS, MODE, 32><<<grid, 256, 0, st>>>(p.geo(), t, s1, s2, e1);
        } else {
            k_bp<NS, MODE, 32><<<grid, 256, 0, st>>>(p.geo(), t, s1, s2, e);
        }
    } else {
        static int tall_env = -1;
        if (tall_env < 0) { const char* v = getenv("LT_BP_TALL"); tall_env = v ? atoi(v) : 1; }   // LT_BP_TALL=0: 64 x 64
        const int nsy = (t.T + 127) / 128;
        // 64 x 128 sub-tiles for the ROI backprojection when they still fill >= 4 waves
        // (128 registers: 2 CTAs per SM; C3's 64 ROIs: 0.070 vs 0.047 ms at under 2 waves)
        // 64 x 32 sub-tiles when the 64 x 64 CTAs would load the busiest SM clearly
        // more than the average (a C4 shard of 32 ROIs on 8 GPUs: 512 CTAs = 3.46 per
        // SM, 4 on the busiest; 1024 half-size CTAs: 7 x 1/2), by the estimate
        // ceil(CTAs / SMs) x work per CTA x 1.06 (staging and setup over half the pixels)
        static int short_env = -2;
        if (short_env == -2) { const char* v = getenv("LT_BP_SHORT"); short_env = (v && *v) ? atoi(v) : -1; }
        const int nsyh = (t.T + 31) / 32;
        const long long c64 = (long long)nsx * nsx * t.ntiles, c32 = (long long)nsx * nsyh * t.ntiles;
        const double est64 = (double)((c64 + p.num_sms - 1) / p.num_sms);
        const double est32 = 0.5 * 1.06 * (double)((c32 + p.num_sms - 1) / p.num_sms);
        const bool shortb = !e.blist && NS > 0 && short_env != 0 && (short_env == 1 || est32 < 0.97 * est64);
        if (tall_env && !e.blist && NS > 0 && (long long)nsx * nsy * t.ntiles >= 4LL * 2 * p.num_sms) {
            k_bp<NS, MODE, BP_SUB, 128><<<dim3(nsx * nsy, t.ntiles), 256, 0, st>>>(p.geo(), t, s1, s2, e);
        } else if (shortb) {
            if constexpr (NS > 0) k_bp<NS, MODE, BP_SUB, 32><<<dim3(nsx * nsyh, t.ntiles), 256, 0, st>>>(p.geo(), t, s1, s2, e);
        } else {
            k_bp<NS, MODE, BP_SUB><<<dim3(e.blist ? nblist : nsx * nsx, t.ntiles), 256, 0, st>>>(p.geo(), t, s1, s2, e);
        }
    }
    LT_LAUNCHED();
    return LT_OK;
}

BpEpi epi0() {
    BpEpi e;
    memset(&e, 0, sizeof e);
    e.hi = INFINITY;
    e.lo = -INFINITY;
    return e;
}

SinoView view_full(const float* base, int nd, long long tile_stride = 0) {
    return SinoView{base, tile_stride, nd, 1, nd};
}
SinoView view_win(const float* base, int Wwin, int na) {
    return SinoView{base, (long long)na * Wwin, Wwin, 0, Wwin};
}

// the FGP kernels support extended ROIs up to 320 x 320 (32 lanes x 8 columns
// up to 256, 32 lanes x 10 columns above: the paper's 256^2 parts padded by 1/8)
int fgp_check(int rows, int cols) {
    if (rows < 1 || cols < 1 || cols > FGP2_ROW_MAX || rows > FGP2_ROW_MAX)
        return fail(LT_ERR_INVALID, "FGP tile %dx%d unsupported (extended ROI side <= %d)", rows, cols, FGP2_ROW_MAX);
    return LT_OK;
}

// host-computed FGP momentum table (Beck-Teboulle t_k, reading A12) in __constant__
// memory.  __constant__ symbols exist once PER DEVICE, so the upload is tracked
// per device ordinal: a second device in the same process gets its own copy.
int ensure_fgp_beta(int nfgp, cudaStream_t st) {
    (void)nfgp;                         // the whole FGP_MAX_IT table is uploaded once per device
    static uint64_t have_mask = 0;
    static float tab[FGP_MAX_IT];
    const int dv = cur_dev();
    if (dv < 0) return fail(LT_ERR_RUNTIME, "cudaGetDevice failed or device ordinal >= %d", LT_MAX_DEV);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (have_mask >> dv & 1) return LT_OK;
    double t = 1.0;
    for (int k = 0; k < FGP_MAX_IT; ++k) {
        const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * t * t));
        tab[k] = (float)((t - 1.0) / tn);
        t = tn;
    }
    LT_CUDA(cudaMemcpyToSymbolAsync(c_fgp_beta, tab, sizeof tab, 0, cudaMemcpyHostToDevice, st));
    LT_CUDA(cudaStreamSynchronize(st));
    have_mask |= 1ull << dv;
    return LT_OK;
}

// k_fgp2 (paired-FP32 layout): NW warps of FR full rows per CTA, K CTAs per
// cluster.  LT_FGP2_CFG = "4x8" (default, 8-CTA clusters for 256-row tiles),
// "2x8" (16-CTA clusters), "2x8b" (b in shared memory, two CTAs per SM).
// CP = 5: tiles wider than 256 (up to 320) with 10 columns per lane (3 rows per warp).
template <int MODE, int FR, int NW, bool BSM = false, bool PERSIST = false, int CP = 4>
int launch_fgp2_t(FgpArgs A, int rows, int ntiles, cudaStream_t st, int* max_clusters = nullptr) {
    const int K = (rows + NW * FR - 1) / (NW * FR);
    if (K > 16) return fail(LT_ERR_INVALID, "FGP tile with %d rows needs a %d-CTA cluster (> 16)", rows, K);
    using SMl = Fgp2Smem<FR, NW, CP>;
    const size_t smem = PERSIST ? (size_t)(SMl::total + 2 * SMl::xin_floats + SMl::bnext_floats) * sizeof(float)
                                : (size_t)((BSM ? SMl::total_bsm : SMl::total) +
                                           (MODE == 1 ? SMl::xin_floats : 0)) * sizeof(float);
    auto kern = k_fgp2<MODE, FR, NW, BSM, PERSIST, CP>;
    LT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (K > 8) LT_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t cfg;
    memset(&cfg, 0, sizeof cfg);
    cfg.gridDim = dim3(K, ntiles, 1);
    cfg.blockDim = dim3(NW * 32, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    A.ntiles = ntiles;
    if (max_clusters) {    // query only: how many clusters of this shape are co-resident
        if (cudaOccupancyMaxActiveClusters(max_clusters, kern, &cfg) != cudaSuccess) *max_clusters = 0;
        cudaGetLastError();
        return LT_OK;
    }
    if (PERSIST) {   // only the co-resident clusters; each iterates over its tiles
        // (cached per device and cluster size K: the shape changes with the tile rows)
        static int cmax_dev[LT_MAX_DEV][17] = {};
        int& cmax = cmax_dev[std::max(0, cur_dev())][K];
        if (!cmax) {
            cfg.gridDim = dim3(K, 1024, 1);
            if (cudaOccupancyMaxActiveClusters(&cmax, kern, &cfg) != cudaSuccess || cmax <= 0) { cudaGetLastError(); cmax = 1; }
        }
        cfg.gridDim = dim3(K, std::min(ntiles, cmax), 1);
    }
    ScopedTimer tm(TC_FGP, st);
    LT_CUDA(cudaLaunchKernelEx(&cfg, kern, A));
    LT_LAUNCHED();
    return LT_OK;
}

// tiles up to 256 columns: CP = 1 / 2 / 3 / 4 column pairs per lane for tiles up
// to 64 / 128 / 192 / 256 columns (narrow tiles use all 32 lanes: half the work
// per warp of the 256-wide layout on a 128-wide tile)
template <int MODE, int CP>
int launch_fgp_cp(FgpArgs A, int rows, int ntiles, cudaStream_t st) {
    static int cfgv = -1;
    if (cfgv < 0) {
        const char* e = getenv("LT_FGP2_CFG");
        cfgv = !e ? 0 : !strcmp(e, "2x8") ? 1 : !strcmp(e, "2x8b") ? 2 : !strcmp(e, "2x16b") ? 3 : !strcmp(e, "4x8") ? 4 : 0;
    }
    // 16-row CTAs (twice the CTAs per tile, shorter iteration latency) or
    // 32-row CTAs (fewer SMs per tile): the shape with fewer waves x wave
    // latency, from the co-resident cluster counts of both shapes (B200,
    // 256-row tiles: 7 clusters of 16 / 15 of 8) and the measured single-wave
    // latencies (52 / 73 us per 100 FGP iterations, tools/fgp_single.py)
    bool use16 = false;
    int clusters8 = 0;                                        // co-resident 32-row-CTA clusters
    if (cfgv == 0 && rows > 16 && (rows + 15) / 16 <= 16) {
        static int c2_dev[LT_MAX_DEV][17] = {}, c4_dev[LT_MAX_DEV][17] = {};   // cache by device and rows / 16
        const int dv = std::max(0, cur_dev());
        int* c2 = c2_dev[dv];
        int* c4 = c4_dev[dv];
        const int key = (rows + 15) / 16;
        if (!c2[key]) {
            launch_fgp2_t<MODE, 2, 8, false, false, CP>(A, rows, 1, st, &c2[key]);
            launch_fgp2_t<MODE, 4, 8, false, false, CP>(A, rows, 1, st, &c4[key]);
            if (c2[key] <= 0) c2[key] = -1;
            if (c4[key] <= 0) c4[key] = -1;
        }
        clusters8 = c4[key];
        if (c2[key] > 0 && c4[key] > 0) {
            const long long w2 = (ntiles + c2[key] - 1) / c2[key], w4 = (ntiles + c4[key] - 1) / c4[key];
            // (the 52 / 73 us latencies are the 256-wide CP = 4 layout's; on narrow tiles,
            // CP <= 2, a 32-row CTA is the faster one per wave -- L1's 64 tiles of 128^2:
            // 46 vs 52 us per wave -- so 16-row CTAs only when they save a wave)
            use16 = CP >= 3 ? w2 * 52 < w4 * 73 : w2 < w4;
        }
    }
    if (cfgv == 4) return launch_fgp2_t<MODE, 4, 8, false, false, CP>(A, rows, ntiles, st);
    if (cfgv == 1 || use16) return launch_fgp2_t<MODE, 2, 8, false, false, CP>(A, rows, ntiles, st);
    if constexpr (CP == 4) {
        static int persist_env = -1;
        if (persist_env < 0) { const char* e = getenv("LT_FGP_PERSIST"); persist_env = !(e && atoi(e) == 0); }
        if (cfgv == 2) return launch_fgp2_t<MODE, 2, 8, true>(A, rows, ntiles, st);
        if (cfgv == 3) return launch_fgp2_t<MODE, 2, 16, true>(A, rows, ntiles, st);
        // persistent 8-CTA clusters (many waves): only the co-resident clusters are
        // launched and each walks its tiles, prefetching the next tile's b, x_prev
        // and x_s during the current one; the SMs the clusters cannot use stay free
        // for the side-stream x_s backprojection for the whole FGP (C4 318 -> 331)
        // (at C3's 64 tiles = 2.8 waves the dynamic wave scheduling does as well)
        if (persist_env && clusters8 > 0 && ntiles > 3 * clusters8)
            return launch_fgp2_t<MODE, 4, 8, false, true>(A, rows, ntiles, st);
    }
    return launch_fgp2_t<MODE, 4, 8, false, false, CP>(A, rows, ntiles, st);
}

template <int MODE>
int launch_fgp(FgpArgs A, int rows, int cols, int ntiles, cudaStream_t st) {
    if (int rc = fgp_check(rows, cols)) return rc;
    if (int rc = ensure_fgp_beta(A.nfgp, st)) return rc;
    // wide tiles (257..320 columns or rows): 10 columns per lane, 2 rows per warp,
    // 10 warps: 20-row CTAs (clusters of up to 16 CTAs); P1 FGP 83 -> 79 us per
    // launch against 3 rows x 8 warps (24-row CTAs, 14-CTA clusters), which
    // LT_FGP_WIDE_CFG=3x8 keeps
    if (rows > FGP2_ROW || cols > FGP2_ROW) {
        static int w_env = -1;
        if (w_env < 0) { const char* e = getenv("LT_FGP_WIDE_CFG"); w_env = (e && !strcmp(e, "3x8")) ? 1 : 0; }
        if (w_env == 1) return launch_fgp2_t<MODE, 3, 8, false, false, 5>(A, rows, ntiles, st);
        return launch_fgp2_t<MODE, 2, 10, false, false, 5>(A, rows, ntiles, st);
    }
    static int narrow_env = -1;
    if (narrow_env < 0) { const char* e = getenv("LT_FGP_NARROW"); narrow_env = !(e && atoi(e) == 0); }
    if (narrow_env && cols <= 64) return launch_fgp_cp<MODE, 1>(A, rows, ntiles, st);
    if (narrow_env && cols <= 128) return launch_fgp_cp<MODE, 2>(A, rows, ntiles, st);
    if (narrow_env && cols <= 192) return launch_fgp_cp<MODE, 3>(A, rows, ntiles, st);
    return launch_fgp_cp<MODE, 4>(A, rows, ntiles, st);
}

dim3 grid2d(int w, int h) { return dim3((w + 31) / 32, (h + 7) / 8); }

// W D and its zero-frequency sums (geometry only, cached)
int ensure_wd(lt_plan& p, cudaStream_t st) {
    if (p.wd_ready) return LT_OK;
    float* gi = p.P<float>(p.off.gimg);
    float* giT = p.P<float>(p.off.gimgT);
    const size_t gbytes = (size_t)p.GT * p.GTP * sizeof(float);
    LT_CUDA(cudaMemsetAsync(gi, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(giT, 0, gbytes, st));
    k_pack<<<grid2d(p.n, p.n), dim3(32, 8), 0, st>>>(p.n, p.GTP, nullptr, 1, gi, giT);
    LT_LAUNCHED();
    if (int rc = global_fp(p, 0, gi, giT, p.P<float>(p.off.wd), nullptr, nullptr, st)) return rc;
    k_rowsum<<<p.na, 256, 0, st>>>(p.nd, p.P<float>(p.off.wd), p.P<double>(p.off.wdsum));
    LT_LAUNCHED();
    p.wd_ready = true;
    return LT_OK;
}

int disc_correct(lt_plan& p, const float* d_sino, float* d_pc, float* d_cuser, cudaStream_t st) {
    NvtxRange nv("lt/disc");
    if (int rc = ensure_wd(p, st)) return rc;
    k_rowsum<<<p.na, 256, 0, st>>>(p.nd, d_sino, p.P<double>(p.off.psum));
    LT_LAUNCHED();
    k_discc<<<1, 256, 0, st>>>(p.na, p.P<double>(p.off.psum), p.P<double>(p.off.wdsum), p.P<double>(p.off.discc64),
                               p.P<float>(p.off.discc32), d_cuser, p.P<int>(p.off.err));
    LT_LAUNCHED();
    const long long ne = (long long)p.na * p.nd;
    k_pc<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(ne, d_sino, p.P<float>(p.off.wd), p.P<double>(p.off.discc64), d_pc);
    LT_LAUNCHED();
    return LT_OK;
}

#define LT_CUFFT(call)                                                                    \
    do {                                                                                  \
        cufftResult r_ = (call);                                                          \
        if (r_ != CUFFT_SUCCESS) return fail(LT_ERR_RUNTIME, "%s: cufft error %d", #call, (int)r_); \
    } while (0)

// cuFFT plans (created on first use, work area inside the workspace)
int fft_plans(lt_plan& p, cudaStream_t st) {
    const int L = p.fftL, F = p.fftF;
    int nL[1] = {L};
    void* work = p.ws + p.off.fwork;
    auto mk = [&](cufftHandle* h, cufftType type, int batch) -> int {
        if (*h) return LT_OK;
        size_t ws = 0;
        LT_CUFFT(cufftCreate(h));
        LT_CUFFT(cufftSetAutoAllocation(*h, 0));
        if (type == CUFFT_R2C) LT_CUFFT(cufftMakePlanMany(*h, 1, nL, nullptr, 1, L, nullptr, 1, F, type, batch, &ws));
        else LT_CUFFT(cufftMakePlanMany(*h, 1, nL, nullptr, 1, F, nullptr, 1, L, type, batch, &ws));
        if (ws > p.fwork_bytes) return fail(LT_ERR_RUNTIME, "cufft needs %zu work bytes > %zu planned", ws, p.fwork_bytes);
        return LT_OK;
    };
    if (int rc = mk(&p.plan_r2c_p, CUFFT_R2C, p.na)) return rc;
    if (int rc = mk(&p.plan_r2c_k, CUFFT_R2C, p.fft_kc * p.na)) return rc;
    if (int rc = mk(&p.plan_c2r_k, CUFFT_C2R, p.fft_kc * p.na)) return rc;
    LT_CUFFT(cufftSetWorkArea(p.plan_r2c_p, work));    // (re-set every call: the workspace may be rebound)
    LT_CUFFT(cufftSetWorkArea(p.plan_r2c_k, work));
    LT_CUFFT(cufftSetWorkArea(p.plan_c2r_k, work));
    LT_CUFFT(cufftSetStream(p.plan_r2c_p, st));
    LT_CUFFT(cufftSetStream(p.plan_r2c_k, st));
    LT_CUFFT(cufftSetStream(p.plan_c2r_k, st));
    return LT_OK;
}

// bank spectra U_k / L (once per bank)
int bank_spectra(lt_plan& p, cudaStream_t st) {
    if (int rc = fft_plans(p, st)) return rc;
    const int L = p.fftL, F = p.fftF, na = p.na, nd = p.nd;
    const long long ns = (long long)na * nd;
    float* real = p.P<float>(p.off.freal);
    for (int k0 = 0; k0 < p.n_iter; k0 += p.fft_kc) {
        const int kc = std::min(p.fft_kc, p.n_iter - k0);
        k_padrows<<<dim3((L + 255) / 256, kc * na), 256, 0, st>>>(kc * na, nd, L, p.P<float>(p.off.bank) + k0 * ns, real);
        LT_LAUNCHED();
        if (kc < p.fft_kc)   // tail chunk: the plan's batch covers fft_kc rows-groups; clear the rest
            LT_CUDA(cudaMemsetAsync(real + (size_t)kc * na * L, 0, (size_t)(p.fft_kc - kc) * na * L * sizeof(float), st));
        float2* dst = p.P<float2>(p.off.uhat) + (size_t)k0 * na * F;
        if (kc == p.fft_kc) {
            LT_CUFFT(cufftExecR2C(p.plan_r2c_k, real, (cufftComplex*)dst));
        } else {
            float2* tmp = p.P<float2>(p.off.fspec);
            LT_CUFFT(cufftExecR2C(p.plan_r2c_k, real, (cufftComplex*)tmp));
            LT_CUDA(cudaMemcpyAsync(dst, tmp, (size_t)kc * na * F * sizeof(float2), cudaMemcpyDeviceToDevice, st));
        }
    }
    // 1/L of the inverse transform folded into the spectra
    const long long tot = (long long)p.n_iter * na * F * 2;
    k_scale<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(tot, 1.f / (float)L, p.P<float>(p.off.uhat));
    LT_LAUNCHED();
    p.spec_ready = true;
    return LT_OK;
}

int conv_cache_direct(lt_plan& p, const float* d_pc, cudaStream_t st);

int conv_cache(lt_plan& p, const float* d_pc, cudaStream_t st) {
    if (!p.bank_ready) return fail(LT_ERR_INVALID, "filter bank not computed (lt_filter_bank / lt_set_bank)");
    static int direct = -1;
    if (direct < 0) { const char* e = getenv("LT_CONV"); direct = (e && !strcmp(e, "direct")) ? 1 : 0; }
    if (direct) return conv_cache_direct(p, d_pc, st);
    ScopedTimer tm(TC_CONV, st);
    if (!p.spec_ready)
        if (int rc = bank_spectra(p, st)) return rc;
    if (int rc = fft_plans(p, st)) return rc;
    const int L = p.fftL, F = p.fftF, na = p.na, nd = p.nd;
    float* real = p.P<float>(p.off.freal);
    float2* spec = p.P<float2>(p.off.fspec);
    float2* phat = p.P<float2>(p.off.phat);
    k_padrows<<<dim3((L + 255) / 256, na), 256, 0, st>>>(na, nd, L, d_pc, real);
    LT_LAUNCHED();
    LT_CUFFT(cufftExecR2C(p.plan_r2c_p, real, (cufftComplex*)phat));
    const long long ns = (long long)na * nd;
    for (int k0 = 0; k0 < p.n_iter; k0 += p.fft_kc) {
        const int kc = std::min(p.fft_kc, p.n_iter - k0);
        const long long ne = (long long)kc * na * F;
        k_specmul<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(ne, na, F, p.P<float2>(p.off.uhat) + (size_t)k0 * na * F,
                                                               phat, spec);
        LT_LAUNCHED();
        LT_CUFFT(cufftExecC2R(p.plan_c2r_k, (cufftComplex*)spec, real));
        k_croprows<<<dim3((nd + 255) / 256, kc * na), 256, 0, st>>>(kc * na, nd, L, (nd - 1) / 2, real,
                                                                   p.P<float>(p.off.conv) + k0 * ns);
        LT_LAUNCHED();
    }
    return LT_OK;
}

int conv_cache_direct(lt_plan& p, const float* d_pc, cudaStream_t st) {
    dim3 grid((p.nd + CV_DB - 1) / CV_DB, p.na, (p.n_iter + CV_KB - 1) / CV_KB);
    ScopedTimer tm(TC_CONV, st);
    k_conv<<<grid, 256, 0, st>>>(p.na, p.nd, p.n_iter, p.P<float>(p.off.bank), d_pc, p.P<float>(p.off.conv));
    LT_LAUNCHED();
    return LT_OK;
}

// the local iteration loop (a5-a8) for every local ROI; mode 0 box, 1 TV
// one ROI group (tiles [t0, t0 + cnt)) through all n iterations on stream st
// (two-group pipelining with a shared x_s: the caller runs one iteration at a
// time, [k0, k1) with the FISTA t_k in *tkp; ext_side = the caller computes
// x_s^k on the side stream into xsg[0] for both groups and records p.xev_xs;
// this group's ROI backprojection waits for it and records bpev when done)
int group_iterations(lt_plan& p, int gl, int t0, int cnt, int mode, float lo, float hi, float lam, int nfgp,
                     const float* d_sino, cudaStream_t st, cudaStream_t fst = nullptr, cudaEvent_t pev = nullptr,
                     cudaEvent_t fev = nullptr, int k0 = 0, int k1 = -1, double* tkp = nullptr, bool ext_side = false,
                     cudaEvent_t bpev = nullptr) {
    if (k1 < 0) k1 = p.n_iter;
    Tiles t = p.roi_tiles();
    t.tile += t0; t.d0 += (size_t)t0 * p.na; t.tauc += (size_t)t0 * p.na; t.ntiles = cnt;
    const long long yts = p.ytile();
    float* y = p.P<float>(p.off.y) + t0 * yts;
    float* yT = p.P<float>(p.off.yT) + t0 * yts;
    float* s = p.P<float>(p.off.s) + (long long)t0 * p.na * p.Wwin;
    float* v = p.P<float>(p.off.v) + t0 * p.ptile();
    float* xs = p.P<float>(p.off.xs) + t0 * p.ptile();
    float* xprev = p.P<float>(p.off.xprev) + t0 * p.ptile();
    const long long ns = (long long)p.na * p.nd;
    const bool exact = (p.flags & LT_XS_EXACT) != 0;
    const bool disc = (p.flags & LT_DISC_ON) != 0 && !exact;
    // x_s^k = M_{L'} W^T b_k for every ROI of the group comes from one global
    // backprojection over the image blocks the group's extended ROIs cover
    // (the extended ROIs overlap, so this is ~4x less work than per ROI)
    float* xsg = p.P<float>(p.off.xsg[(gl == 2 && !ext_side) ? 1 : 0]);
    int xsg_pitch = p.n;
    const int* blist = p.P<int>(p.off.xsblk[gl]);
    const int nbl = (int)p.xsblk[gl].size();
    if (exact) { xsg = p.P<float>(p.off.gimg) + PADL; xsg_pitch = p.GTP; }   // the global SIRT iterate
    static int overlap_env = -1;
    if (overlap_env < 0) { const char* e = getenv("LT_XS_OVERLAP"); overlap_env = !(e && atoi(e) == 0); }
    const bool side = overlap_env && !exact && !fst && nbl > 0 && !ext_side;
    if (side && !p.xst) {
        LT_CUDA(cudaStreamCreateWithFlags(&p.xst, cudaStreamNonBlocking));
        LT_CUDA(cudaEventCreateWithFlags(&p.xev_bp, cudaEventDisableTiming));
        LT_CUDA(cudaEventCreateWithFlags(&p.xev_xs, cudaEventDisableTiming));
    }
    auto xs_bp = [&](int k, cudaStream_t sx) -> int {
        BpEpi ex = epi0();
        ex.blist = blist; ex.out = xsg; ex.out_pitch = p.n;
        const SinoView vb = view_full(p.P<float>(p.off.conv) + (long long)k * ns, p.nd);
        return launch_bp_t<1, BP_PLAIN_GLOBAL>(p, p.glob_tiles(), vb, vb, ex, sx, nbl);
    };
    if (side) {   // x_s^0 on the side stream, after everything queued so far
        LT_CUDA(cudaEventRecord(p.xev_bp, st));
        LT_CUDA(cudaStreamWaitEvent(p.xst, p.xev_bp, 0));
        if (int rc = xs_bp(0, p.xst)) return rc;
        LT_CUDA(cudaEventRecord(p.xev_xs, p.xst));
    }
    double tk = tkp ? *tkp : 1.0;
    for (int k = k0; k < k1; ++k) {
        const float* bk = p.P<float>(p.off.conv) + (long long)k * ns;
        if (side || ext_side) {
            // x_s^k was queued on the side stream; its ROI BP waits for it below
        } else if (exact) {   // x^k = x^{k-1} + alpha W^T (p - W x^{k-1}) on the full grid, x^0 = 0 (eq. sirtit)
            const Tiles gt = p.glob_tiles();
            float* gx = p.P<float>(p.off.gimg);
            float* gxT = p.P<float>(p.off.gimgT);
            float* r = p.P<float>(p.off.gsino);
            if (int rc = global_fp(p, 2, gx, gxT, r, d_sino, nullptr, st)) return rc;
            BpEpi eg = epi0();
            eg.y = gx; eg.yT = gxT; eg.alpha = (float)p.alpha;
            const SinoView sv = view_full(r, p.nd);
            if (int rc = launch_bp_t<1, BP_GSIRT>(p, gt, sv, sv, eg, st)) return rc;
        } else {   // (independent of y: overlaps the previous FGP of this group)
            if (int rc = xs_bp(k, st)) return rc;
        }
        if (fst && k > 0) LT_CUDA(cudaStreamWaitEvent(st, fev, 0));    // previous FGP of this group
        BpEpi e = epi0();
        e.xsg = xsg; e.xsg_pitch = xsg_pitch;
        e.y = y; e.yT = yT; e.y_tstride = yts;
        e.v = v; e.xs = xs; e.p_tstride = p.ptile();
        e.discc = p.P<float>(p.off.discc32); e.use_disc = disc;
        e.alpha = (float)p.alpha; e.lo = lo; e.hi = hi; e.last = (k == p.n_iter - 1);
        if (k == 0) {
            // y^0 = 0: W_{L'} y^0 = 0, no gather
            if (side || ext_side) LT_CUDA(cudaStreamWaitEvent(st, p.xev_xs, 0));
            const SinoView v0 = view_full(bk, p.nd);
            if (mode == 0) { if (int rc = launch_bp_t<0, BP_BOX>(p, t, v0, v0, e, st)) return rc; }
            else { if (int rc = launch_bp_t<0, BP_TV>(p, t, v0, v0, e, st)) return rc; }
        } else {
            if (int rc = launch_fp_roi(p, t, y, yT, yts, s, (long long)p.na * p.Wwin, st)) return rc;
            if (side || ext_side) LT_CUDA(cudaStreamWaitEvent(st, p.xev_xs, 0));
            const SinoView vs = view_win(s, p.Wwin, p.na);
            if (mode == 0) { if (int rc = launch_bp_t<1, BP_BOX>(p, t, vs, vs, e, st)) return rc; }
            else { if (int rc = launch_bp_t<1, BP_TV>(p, t, vs, vs, e, st)) return rc; }
        }
        if (ext_side && bpev) LT_CUDA(cudaEventRecord(bpev, st));
        if (side && k + 1 < p.n_iter) {   // x_s^{k+1} may overwrite x_s^k once this ROI BP has read it
            LT_CUDA(cudaEventRecord(p.xev_bp, st));
            LT_CUDA(cudaStreamWaitEvent(p.xst, p.xev_bp, 0));
            if (int rc = xs_bp(k + 1, p.xst)) return rc;
            LT_CUDA(cudaEventRecord(p.xev_xs, p.xst));
        }
        if (mode == 1) {
            const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tk * tk));
            const double beta = (tk - 1.0) / tn;
            tk = tn;
            FgpArgs A;
            memset(&A, 0, sizeof A);
            A.b = v; A.b_pitch = p.T; A.b_tstride = p.ptile();
            A.tiles = p.P<TileT>(p.off.tiles) + t0;
            A.lam = lam; A.nfgp = nfgp;
            A.lams = p.lam_array ? p.P<float>(p.off.lams) + t0 : nullptr;
            A.xs = xs; A.xprev = xprev; A.p_tstride = p.ptile(); A.T = p.T;
            A.y = y; A.yT = yT; A.y_tstride = yts; A.TP = p.TP;
            A.beta_o = (float)beta;
            if (fst) {
                LT_CUDA(cudaEventRecord(pev, st));
                LT_CUDA(cudaStreamWaitEvent(fst, pev, 0));
                if (int rc = launch_fgp<1>(A, p.T, p.T, cnt, fst)) return rc;
                LT_CUDA(cudaEventRecord(fev, fst));
            } else {
                if (int rc = launch_fgp<1>(A, p.T, p.T, cnt, st)) return rc;
            }
        } else if (mode == 2) {     // Haar l1 prox (NEXT-2), nfgp = levels
            const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tk * tk));
            const double beta = p.haar_momentum ? (tk - 1.0) / tn : 0.0;
            tk = tn;
            HaarArgs Hh{v, xs, xprev, p.ptile(), p.T, y, yT, yts, p.TP, p.P<TileT>(p.off.tiles) + t0,
                        lam, nfgp, (float)beta};
            const int nb = (p.T + 31) / 32;
            ScopedTimer tm(TC_FGP, st);
            k_haar<<<dim3(nb * nb, cnt), 256, 0, st>>>(Hh);
            LT_LAUNCHED();
        }
    }
    if (tkp) *tkp = tk;
    if (fst && mode == 1 && k1 == p.n_iter) LT_CUDA(cudaStreamWaitEvent(st, fev, 0));   // the group's stream ends after its last FGP
    return LT_OK;
}

// the local iteration loop (a5-a8) for every local ROI; mode 0 box, 1 TV
int local_iterations(lt_plan& p, int mode, float lo, float hi, float lam, int nfgp, const float* d_sino,
                     cudaStream_t st) {
    const long long yts = p.ytile();
    const bool exact = (p.flags & LT_XS_EXACT) != 0;
    if (exact) {
        const size_t gbytes = (size_t)p.GT * p.GTP * sizeof(float);
        LT_CUDA(cudaMemsetAsync(p.P<float>(p.off.gimg), 0, gbytes, st));
        LT_CUDA(cudaMemsetAsync(p.P<float>(p.off.gimgT), 0, gbytes, st));
    }
    LT_CUDA(cudaMemsetAsync(p.P<float>(p.off.y), 0, (size_t)p.R * yts * sizeof(float), st));
    LT_CUDA(cudaMemsetAsync(p.P<float>(p.off.yT), 0, (size_t)p.R * yts * sizeof(float), st));
    if (mode != 0) LT_CUDA(cudaMemsetAsync(p.P<float>(p.off.xprev), 0, (size_t)p.R * p.ptile() * sizeof(float), st));
    const int ng = (p.nsplit > 1 && p.R >= 2 && p.gst[0] && !exact) ? 2 : 1;
    if (ng == 1) {
        if (int rc = group_iterations(p, 0, 0, p.R, mode, lo, hi, lam, nfgp, d_sino, st)) return rc;
    } else {
        // fork: both group streams wait for the work already queued on st
        LT_CUDA(cudaEventRecord(p.gev[2], st));
        const int half = p.split_at;
        static int sxs_env = -1;
        if (sxs_env < 0) { const char* e = getenv("LT_SPLIT_XS"); sxs_env = !(e && atoi(e) == 0); }
        const bool shared_xs = sxs_env && !p.xsblk[0].empty();
        for (int g = 0; g < 2; ++g) {
            LT_CUDA(cudaStreamWaitEvent(p.gst[g], p.gev[2], 0));
            if (p.fst[g] && mode == 1) LT_CUDA(cudaStreamWaitEvent(p.fst[g], p.gev[2], 0));
        }
        if (!shared_xs) {   // each group computes the x_s of its own blocks on its own stream
            for (int g = 0; g < 2; ++g) {
                const int t0 = g ? half : 0, cnt = g ? p.R - half : half;
                const bool prio = p.fst[g] && mode == 1;
                if (int rc = group_iterations(p, 1 + g, t0, cnt, mode, lo, hi, lam, nfgp, d_sino, p.gst[g],
                                              prio ? p.fst[g] : nullptr, p.pev[g], p.fev[g])) return rc;
                LT_CUDA(cudaEventRecord(p.gev[g], p.gst[g]));
            }
        } else {
            // one x_s^k for both groups on the side stream (the global backprojection
            // over all their blocks), queued as soon as both groups' ROI backprojections
            // of iteration k - 1 have read x_s^{k-1}; the groups run one iteration at a time
            if (!p.xst) {
                LT_CUDA(cudaStreamCreateWithFlags(&p.xst, cudaStreamNonBlocking));
                LT_CUDA(cudaEventCreateWithFlags(&p.xev_bp, cudaEventDisableTiming));
                LT_CUDA(cudaEventCreateWithFlags(&p.xev_xs, cudaEventDisableTiming));
            }
            auto xs_full = [&](int k) -> int {
                BpEpi ex = epi0();
                ex.blist = p.P<int>(p.off.xsblk[0]); ex.out = p.P<float>(p.off.xsg[0]); ex.out_pitch = p.n;
                const SinoView vb = view_full(p.P<float>(p.off.conv) + (long long)k * p.na * p.nd, p.nd);
                return launch_bp_t<1, BP_PLAIN_GLOBAL>(p, p.glob_tiles(), vb, vb, ex, p.xst, (int)p.xsblk[0].size());
            };
            LT_CUDA(cudaStreamWaitEvent(p.xst, p.gev[2], 0));
            if (int rc = xs_full(0)) return rc;
            LT_CUDA(cudaEventRecord(p.xev_xs, p.xst));
            double tk[2] = {1.0, 1.0};
            for (int k = 0; k < p.n_iter; ++k) {
                for (int g = 0; g < 2; ++g) {
                    const int t0 = g ? half : 0, cnt = g ? p.R - half : half;
                    const bool prio = p.fst[g] && mode == 1;
                    if (int rc = group_iterations(p, 1 + g, t0, cnt, mode, lo, hi, lam, nfgp, d_sino, p.gst[g],
                                                  prio ? p.fst[g] : nullptr, p.pev[g], p.fev[g], k, k + 1, &tk[g], true,
                                                  p.bpev[g])) return rc;
                }
                if (k + 1 < p.n_iter) {
                    LT_CUDA(cudaStreamWaitEvent(p.xst, p.bpev[0], 0));
                    LT_CUDA(cudaStreamWaitEvent(p.xst, p.bpev[1], 0));
                    if (int rc = xs_full(k + 1)) return rc;
                    LT_CUDA(cudaEventRecord(p.xev_xs, p.xst));
                }
            }
            for (int g = 0; g < 2; ++g) LT_CUDA(cudaEventRecord(p.gev[g], p.gst[g]));
        }
        // join
        LT_CUDA(cudaStreamWaitEvent(st, p.gev[0], 0));
        LT_CUDA(cudaStreamWaitEvent(st, p.gev[1], 0));
    }
    p.last_mode = mode;
    return LT_OK;
}

int crop_cores(lt_plan& p, float* d_cores, cudaStream_t st) {
    const int side = 2 * p.radius;
    dim3 grid((side + 31) / 32, (side + 7) / 8, p.R);
    if (p.last_mode == 0)
        k_crop<<<grid, dim3(32, 8), 0, st>>>(side, p.margin, p.P<float>(p.off.y), p.ytile(), p.TP, PADL, d_cores);
    else
        k_crop<<<grid, dim3(32, 8), 0, st>>>(side, p.margin, p.P<float>(p.off.xprev), p.ptile(), p.T, 0, d_cores);
    LT_LAUNCHED();
    return LT_OK;
}

// The local iteration loop (n x 3-4 launches) as one CUDA graph: captured on
// the first solve with a given (mode, bounds, lambda, n_FGP, lambda array,
// Haar momentum, sinogram pointer) and replayed afterwards; every input of the
// loop lives in the workspace, so a replay sees the new data.  Off under
// per-kernel timing (the timing events would not repeat) and with two ROI
// streams; by default only for small batches (see below), LT_GRAPH=1 / 0
// forces it on / off.
int run_local(lt_plan& p, int mode, float lo, float hi, float lam, int nfgp, const float* d_sino, cudaStream_t st) {
    static int env = -2;
    if (env == -2) { const char* e = getenv("LT_GRAPH"); env = e ? atoi(e) : -1; }   // 1 on, 0 off, unset: auto
    // auto: only launch-bound batches gain from the replay (C1 e2e 502 -> 634,
    // C2 565 -> 576 solves/s); with more work per iteration the eagerly issued
    // streams overlap better (C3 614 vs 591, T1 36 vs 34, C4 319 vs 309)
    const double work = (double)p.R * p.T * p.T * p.na;    // pixel-angle updates of one A over the batch
    const bool use = env == 1 || (env == -1 && work < 2.5e7);
    if (!use || g_timing || (p.nsplit > 1 && p.R >= 2)) return local_iterations(p, mode, lo, hi, lam, nfgp, d_sino, st);
    if (mode == 1)
        if (int rc = ensure_fgp_beta(nfgp, st)) return rc;   // (synchronous on first use: not inside a capture)
    if (!p.gs) {
        LT_CUDA(cudaStreamCreateWithFlags(&p.gs, cudaStreamNonBlocking));
        LT_CUDA(cudaEventCreateWithFlags(&p.gev_in, cudaEventDisableTiming));
        LT_CUDA(cudaEventCreateWithFlags(&p.gev_out, cudaEventDisableTiming));
    }
    // fork onto the graph stream, join back after the replay
    LT_CUDA(cudaEventRecord(p.gev_in, st));
    LT_CUDA(cudaStreamWaitEvent(p.gs, p.gev_in, 0));
    const cudaStream_t caller = st;
    st = p.gs;
    const double key[10] = {(double)mode, (double)lo, (double)hi, (double)lam, (double)nfgp, (double)p.lam_array,
                            (double)p.haar_momentum, (double)(uintptr_t)d_sino, (double)(uintptr_t)p.ws, 1.0};
    if (!p.gexec || memcmp(key, p.gkey, sizeof key) != 0) {
        if (p.gexec) { cudaGraphExecDestroy(p.gexec); p.gexec = nullptr; }
        cudaGraph_t g = nullptr;
        const long long n0 = g_launches.load();
        LT_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        const int rc = local_iterations(p, mode, lo, hi, lam, nfgp, d_sino, st);
        const cudaError_t ec = cudaStreamEndCapture(st, &g);
        if (rc) { if (g) cudaGraphDestroy(g); return rc; }
        LT_CUDA(ec);
        const cudaError_t ei = cudaGraphInstantiate(&p.gexec, g, 0);
        cudaGraphDestroy(g);
        LT_CUDA(ei);
        p.g_nlaunch = g_launches.load() - n0;   // counted again at every replay
        g_launches.fetch_sub(p.g_nlaunch);
        memcpy(p.gkey, key, sizeof key);
    }
    LT_CUDA(cudaGraphLaunch(p.gexec, st));
    g_launches.fetch_add(p.g_nlaunch);
    LT_CUDA(cudaEventRecord(p.gev_out, st));
    LT_CUDA(cudaStreamWaitEvent(caller, p.gev_out, 0));
    p.last_mode = mode;
    return LT_OK;
}

int solve(lt_plan& p, int mode, const float* d_sino, float a0, float a1, int nfgp, float* d_cores, cudaStream_t st) {
    NvtxRange nv(mode == 0 ? "lt/sirt_solve" : mode == 1 ? "lt/tv_solve" : "lt/haar_solve");
    float* pc = p.P<float>(p.off.pc);
    if (p.flags & LT_XS_EXACT) {
        LT_CUDA(cudaMemsetAsync(p.P<float>(p.off.discc32), 0, sizeof(float), st));
    } else if (p.flags & LT_DISC_ON) {
        if (int rc = disc_correct(p, d_sino, pc, nullptr, st)) return rc;
    } else {
        LT_CUDA(cudaMemcpyAsync(pc, d_sino, (size_t)p.na * p.nd * sizeof(float), cudaMemcpyDeviceToDevice, st));
        LT_CUDA(cudaMemsetAsync(p.P<float>(p.off.discc32), 0, sizeof(float), st));
    }
    if (!(p.flags & LT_XS_EXACT)) {
        NvtxRange nc("lt/conv_cache");
        if (int rc = conv_cache(p, pc, st)) return rc;
    }
    {
        NvtxRange ni("lt/iterations");
        if (int rc = run_local(p, mode, mode == 0 ? a0 : 0.f, mode == 0 ? a1 : 0.f, mode != 0 ? a0 : 0.f, nfgp, d_sino, st))
            return rc;
    }
    return crop_cores(p, d_cores, st);
}

int combine(const lt_plan& p, const float* d_cores, int n_slots, const int* slot_roi, float* d_image, cudaStream_t st,
            const float* const* h_peers = nullptr, int world = 0, int spr = 1) {
    NvtxRange nv("lt/combine");
    const int side = 2 * p.radius;
    const int nb = (p.n + 31) / 32;
    std::vector<std::vector<std::pair<int, int>>> buckets((size_t)nb * nb);
    std::vector<int> r0(std::max(n_slots, 1)), c0(std::max(n_slots, 1));
    for (int s = 0; s < n_slots; ++s) {
        const int g = slot_roi[s];
        if (g < -1 || g >= p.nroi_all) return fail(LT_ERR_INVALID, "slot %d: bad ROI index %d", s, g);
        if (g < 0) { r0[s] = c0[s] = -1000000; continue; }
        r0[s] = p.cen[2 * g] - p.radius;
        c0[s] = p.cen[2 * g + 1] - p.radius;
        for (int by = r0[s] / 32; by <= (r0[s] + side - 1) / 32; ++by)
            for (int bx = c0[s] / 32; bx <= (c0[s] + side - 1) / 32; ++bx) buckets[(size_t)by * nb + bx].push_back({g, s});
    }
    std::vector<int> offs(1, 0), lst;
    for (auto& b : buckets) {
        std::sort(b.begin(), b.end());
        for (auto& e : b) lst.push_back(e.second);
        offs.push_back((int)lst.size());
    }
    if ((int)lst.size() > p.stitch_cap || n_slots > p.nroi_all * std::max(1, p.world))
        return fail(LT_ERR_INVALID, "combine: %zu list entries / %d slots exceed the plan's capacity", lst.size(), n_slots);
    if (h_peers && (world < 1 || world > LT_MAX_PEERS || spr < 1 || (long long)world * spr < n_slots))
        return fail(LT_ERR_INVALID, "combine_peers: bad world %d / slots per rank %d", world, spr);
    // tables live in the workspace; uploaded (stream-ordered) only when the slot
    // layout or the peer pointers differ from the last combine on this plan
    int* d_off = p.P<int>(p.off.st_off);
    int* d_lst = p.P<int>(p.off.st_lst);
    int* d_r0 = p.P<int>(p.off.st_r0);
    int* d_c0 = p.P<int>(p.off.st_c0);
    std::vector<long long> key;
    key.reserve((size_t)n_slots + 3 + (h_peers ? world : 0));
    key.push_back(n_slots); key.push_back(h_peers ? world : 0); key.push_back(h_peers ? spr : 0);
    for (int s = 0; s < n_slots; ++s) key.push_back(slot_roi[s]);
    if (h_peers)
        for (int g = 0; g < world; ++g) key.push_back((long long)(uintptr_t)h_peers[g]);
    if (key != p.st_key) {
        LT_CUDA(cudaMemcpyAsync(d_off, offs.data(), offs.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        if (!lst.empty()) LT_CUDA(cudaMemcpyAsync(d_lst, lst.data(), lst.size() * sizeof(int), cudaMemcpyHostToDevice, st));
        LT_CUDA(cudaMemcpyAsync(d_r0, r0.data(), n_slots * sizeof(int), cudaMemcpyHostToDevice, st));
        LT_CUDA(cudaMemcpyAsync(d_c0, c0.data(), n_slots * sizeof(int), cudaMemcpyHostToDevice, st));
        if (h_peers)
            LT_CUDA(cudaMemcpyAsync(p.P<const float*>(p.off.peers), h_peers, world * sizeof(float*),
                                    cudaMemcpyHostToDevice, st));
        p.st_key.swap(key);
    }
    const float* const* d_peers = h_peers ? p.P<const float*>(p.off.peers) : nullptr;
    k_stitch<<<nb * nb, dim3(32, 8), 0, st>>>(p.n, side, nb, d_off, d_lst, d_r0, d_c0, d_cores, d_image, d_peers, spr);
    LT_LAUNCHED();
    // pageable copies above are staged synchronously by the driver before returning
    return LT_OK;
}

}  // namespace

// ============================================================================
// C-ABI
// ============================================================================
extern "C" {

const char* lt_last_error(void) { return g_err.c_str(); }

void lt_timing_enable(int32_t on) { g_timing = on != 0; }

int lt_timing_read(double* h_ms, int64_t* h_count) {
    double ms[TC_N] = {};
    int64_t cnt[TC_N] = {};
    for (auto& r : g_recs) {
        float t = 0.f;
        LT_CUDA(cudaEventSynchronize(r.b));
        LT_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
        ms[r.cls] += t;
        cnt[r.cls] += 1;
        g_pool.push_back(r.a);
        g_pool.push_back(r.b);
    }
    g_recs.clear();
    for (int k = 0; k < TC_N; ++k) {
        if (h_ms) h_ms[k] = ms[k];
        if (h_count) h_count[k] = cnt[k];
    }
    return LT_OK;
}
int64_t lt_launch_count(void) { return g_launches.load(); }

int lt_roi_setup(int32_t n, int32_t n_angles, int32_t n_det, const double* angles, int32_t n_roi,
                 const int32_t* center_row, const int32_t* center_col, int32_t radius, int32_t margin,
                 int32_t n_iter, int32_t flags, int32_t rank, int32_t world, lt_plan** out) {
    if (!out) return fail(LT_ERR_INVALID, "out is null");
    *out = nullptr;
    if (n < 1 || n_angles < 1 || n_det < 1) return fail(LT_ERR_INVALID, "N, N_theta, N_d must be >= 1");
    if (n_det % 2 == 0) return fail(LT_ERR_INVALID, "N_d must be odd (filter centring)");
    if (!angles) return fail(LT_ERR_INVALID, "angles is null");
    for (int a = 0; a < n_angles; ++a) {
        if (!(angles[a] >= 0.0 && angles[a] < M_PI)) return fail(LT_ERR_INVALID, "angle %d outside [0, pi)", a);
        if (a && !(angles[a] > angles[a - 1])) return fail(LT_ERR_INVALID, "angles not strictly increasing at %d", a);
    }
    if (n_roi < 0 || (n_roi > 0 && (!center_row || !center_col))) return fail(LT_ERR_INVALID, "bad ROI list");
    if (radius < 1 || margin < 0 || n_iter < 1) return fail(LT_ERR_INVALID, "radius >= 1, margin >= 0, n_iter >= 1");
    if (world < 1 || rank < 0 || rank >= world) return fail(LT_ERR_INVALID, "bad rank/world");
    for (int r = 0; r < n_roi; ++r)
        if (center_row[r] - radius < 0 || center_col[r] - radius < 0 || center_row[r] + radius > n ||
            center_col[r] + radius > n)
            return fail(LT_ERR_INVALID, "ROI %d core outside the grid", r);
    lt_plan* p = new lt_plan();
    p->n = n; p->na = n_angles; p->nd = n_det; p->nroi_all = n_roi; p->radius = radius; p->margin = margin;
    p->h = radius + margin; p->T = 2 * p->h; p->TP = (p->T + PADL + PADR + 3) & ~3;   // 16-byte rows (cp.async)
    p->Wwin = window_width(p->h);
    p->n_iter = n_iter; p->flags = flags; p->rank = rank; p->world = world;
    p->GT = n; p->GTP = n + PADL + PADR;
    p->alpha = 1.0 / ((double)n_angles * n_det);
    p->ang.assign(angles, angles + n_angles);
    p->cen.resize(2 * (size_t)n_roi);
    for (int r = 0; r < n_roi; ++r) { p->cen[2 * r] = center_row[r]; p->cen[2 * r + 1] = center_col[r]; }
    // per-angle tables
    p->angf.resize(n_angles); p->cs64.resize(n_angles); p->sn64.resize(n_angles);
    p->A64.resize(n_angles); p->B64.resize(n_angles);
    for (int a = 0; a < n_angles; ++a) {
        const double cs = std::cos(angles[a]), sn = std::sin(angles[a]);
        const double c = std::max(std::fabs(cs), std::fabs(sn));
        const bool col = std::fabs(sn) > std::fabs(cs);
        const double A = col ? -1.0 / sn : 1.0 / cs;
        const double B = col ? cs / sn : sn / cs;
        p->cs64[a] = cs; p->sn64[a] = sn; p->A64[a] = A; p->B64[a] = B;
        AngF f;
        f.cs = (float)cs; f.sn = (float)sn; f.invc = (float)(1.0 / c); f.ic2 = (float)(1.0 / (c * c));
        f.K = (float)(1.0 / c - 0.5 / (c * c)); f.A = (float)A; f.B = (float)B; f.col = col ? 1 : 0;
        p->angf[a] = f;
    }
    // partition: ROIs in raster order of their centres, cut into
    // `world` contiguous runs of balanced cost, so each rank's ROIs are spatially
    // compact (its global x_s backprojection covers only their neighbourhood).
    // Cost model: the FGP cluster works on the full (2h)^2 tile, the projectors on
    // the valid pixels: cost = 4 (2h)^2 + 3 * valid (weight 2, the measured ~40/60 time
    // split, left the 8-GPU C4 edge ranks 34 ROIs and the slowest; 4: projected 2084 ->
    // 2109 ROI solves/s, C5 960 -> 965, 2 / 4 GPUs unchanged; LT_PART_FGPW overrides)
    std::vector<long long> cost(n_roi);
    static int fgpw = -1;     // weight of the FGP term (LT_PART_FGPW, diagnostics; default 4)
    if (fgpw < 0) { const char* e = getenv("LT_PART_FGPW"); fgpw = (e && *e) ? std::max(0, atoi(e)) : 4; }
    for (int r = 0; r < n_roi; ++r) {
        const int cr = p->cen[2 * r], cc = p->cen[2 * r + 1], h = p->h;
        const long long hv = std::min(n, cr + h) - std::max(0, cr - h);
        const long long wv = std::min(n, cc + h) - std::max(0, cc - h);
        cost[r] = (long long)fgpw * (2 * h) * (2 * h) + 3LL * hv * wv;
    }
    std::vector<int> order(n_roi);
    for (int r = 0; r < n_roi; ++r) order[r] = r;
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
        return p->cen[2 * a] != p->cen[2 * b] ? p->cen[2 * a] < p->cen[2 * b] : p->cen[2 * a + 1] < p->cen[2 * b + 1];
    });
    long long total = 0;
    for (int r = 0; r < n_roi; ++r) total += cost[r];
    std::vector<int> owner(n_roi, 0);
    {
        long long cum = 0;
        for (int r : order) {
            // rank of the cost midpoint of this ROI: floor(world * (cum + cost/2) / total)
            const long long mid2 = 2 * cum + cost[r];
            int g = total > 0 ? (int)((long long)world * mid2 / (2 * total)) : 0;
            owner[r] = std::min(std::max(g, 0), world - 1);
            cum += cost[r];
        }
    }
    for (int r = 0; r < n_roi; ++r)
        if (owner[r] == rank) p->local.push_back(r);
    p->R = (int)p->local.size();
    {
        std::vector<std::vector<int>> per(world);
        for (int r = 0; r < n_roi; ++r) per[owner[r]].push_back(r);
        p->spr = 1;
        for (auto& v : per) p->spr = std::max(p->spr, (int)v.size());
        p->slot_all.assign((size_t)world * p->spr, -1);
        for (int g = 0; g < world; ++g)
            for (size_t q = 0; q < per[g].size(); ++q) p->slot_all[(size_t)g * p->spr + q] = per[g][q];
    }
    // ROI tiles and windows
    p->tiles.resize(std::max(p->R, 1));
    p->d0.resize((size_t)std::max(p->R, 1) * n_angles);
    p->tauc.resize((size_t)std::max(p->R, 1) * n_angles);
    for (int q = 0; q < p->R; ++q) {
        const int g = p->local[q];
        const int cr = p->cen[2 * g], cc = p->cen[2 * g + 1], h = p->h;
        TileT t;
        t.row0 = cr - h; t.col0 = cc - h;
        t.vr0 = std::max(0, -t.row0); t.vr1 = std::min(p->T, n - t.row0);
        t.vc0 = std::max(0, -t.col0); t.vc1 = std::min(p->T, n - t.col0);
        t.pad0 = t.pad1 = 0;
        p->tiles[q] = t;
        // tile centre point (x, y) = (cc - N/2, N/2 - cr)
        tile_window(*p, cc - 0.5 * n, 0.5 * n - cr, p->Wwin, &p->d0[(size_t)q * n_angles], &p->tauc[(size_t)q * n_angles]);
    }
    // forward-projection angle groups (16, 8 and 24 angles): one orientation per
    // group.  Balanced (default; LT_FP_BALANCE=0: consecutive angles): an angle's
    // work per band is ~ the rays crossing it, T c_a + 16 s_a (c_a = max(|cos|,
    // |sin|), s_a = min); the orientation's angles sorted by it are paired
    // largest-with-smallest for the two-angles-per-warp groups (every warp of a
    // CTA then reaches the band barrier with about the same work) and kept in
    // sorted order for the one-angle-per-warp groups
    static int bal_env = -1;
    if (bal_env < 0) { const char* e = getenv("LT_FP_BALANCE"); bal_env = !(e && atoi(e) == 0); }
    for (int ga : {16, 8, 24}) {
        std::vector<int>& grp = ga == 16 ? p->fpgroups : ga == 8 ? p->fpgroups1 : p->fpgroups24;
        for (int o = 0; o < 2; ++o) {
            std::vector<int> lst;
            for (int a = 0; a < n_angles; ++a)
                if (p->angf[a].col == o) lst.push_back(a);
            if (bal_env) {
                auto work = [&](int a) {
                    const double c = std::fabs(p->cs64[a]), sv = std::fabs(p->sn64[a]);
                    return (double)p->T * std::max(c, sv) + 16.0 * std::min(c, sv);
                };
                std::stable_sort(lst.begin(), lst.end(), [&](int x, int y) { return work(x) > work(y); });
                if (ga != 8) {   // pairs (largest, smallest), then the pairs in order
                    std::vector<int> pr;
                    for (size_t i = 0, j = lst.size(); i < j; ) {
                        pr.push_back(lst[i++]);
                        if (i < j) pr.push_back(lst[--j]);
                    }
                    lst.swap(pr);
                }
            }
            std::vector<int> cur;
            for (int a : lst) {
                cur.push_back(a);
                if ((int)cur.size() == ga) { grp.insert(grp.end(), cur.begin(), cur.end()); cur.clear(); }
            }
            if (!cur.empty()) {
                cur.resize(ga, -1);
                grp.insert(grp.end(), cur.begin(), cur.end());
            }
        }
    }
    p->ngroups = (int)p->fpgroups.size() / 16;
    p->ngroups1 = (int)p->fpgroups1.size() / 8;
    p->ngroups24 = (int)p->fpgroups24.size() / 24;
    // x_s block lists: blocks meeting any valid extended rect
    {
        const int nbk = (n + BP_SUB - 1) / BP_SUB;
        const char* sb = getenv("LT_SPLIT_B");     // size of the second ROI group (LT_SPLIT=2); default half
        const int nb2 = sb ? atoi(sb) : 0;
        const int half = (nb2 > 0 && nb2 < p->R) ? p->R - nb2 : (p->R + 1) / 2;
        p->split_at = half;
        const int ranges[3][2] = {{0, p->R}, {0, half}, {half, p->R}};
        for (int l = 0; l < 3; ++l) {
            std::vector<char> need((size_t)nbk * nbk, 0);
            for (int q = ranges[l][0]; q < ranges[l][1]; ++q) {
                const TileT& t = p->tiles[q];
                const int r0 = t.row0 + t.vr0, r1 = t.row0 + t.vr1, c0 = t.col0 + t.vc0, c1 = t.col0 + t.vc1;
                for (int by = r0 / BP_SUB; by <= (r1 - 1) / BP_SUB; ++by)
                    for (int bx = c0 / BP_SUB; bx <= (c1 - 1) / BP_SUB; ++bx) need[(size_t)by * nbk + bx] = 1;
            }
            for (int b = 0; b < nbk * nbk; ++b)
                if (need[b]) p->xsblk[l].push_back(b);
        }
    }
    // global tile: the whole grid, window = the full detector
    {
        TileT t;
        t.row0 = 0; t.col0 = 0; t.vr0 = 0; t.vr1 = n; t.vc0 = 0; t.vc1 = n; t.pad0 = t.pad1 = 0;
        p->gtile.assign(1, t);
        p->gd0.assign(n_angles, 0);
        p->gtauc.assign(n_angles, 0.5 * (n_det - 1));
    }
    // global tiling for the forward projector (same tables as ROI tiles, margin 0)
    {
        const int Tg = std::min(256, n);
        const int h = (Tg + 1) / 2;
        p->Tg = 2 * h; p->TPg = (p->Tg + PADL + PADR + 3) & ~3; p->Wg = window_width(h);
        const int nt = (n + p->Tg - 1) / p->Tg;
        p->NTg = nt * nt;
        p->ttiles.resize(p->NTg);
        p->td0.resize((size_t)p->NTg * n_angles);
        p->ttauc.resize((size_t)p->NTg * n_angles);
        for (int bi = 0; bi < nt; ++bi)
            for (int bj = 0; bj < nt; ++bj) {
                const int q = bi * nt + bj;
                TileT t;
                t.row0 = bi * p->Tg; t.col0 = bj * p->Tg;
                t.vr0 = 0; t.vr1 = std::min(p->Tg, n - t.row0);
                t.vc0 = 0; t.vc1 = std::min(p->Tg, n - t.col0);
                t.pad0 = t.pad1 = 0;
                p->ttiles[q] = t;
                // tile centre point (x, y) = (col0 + h - N/2, N/2 - row0 - h)
                tile_window(*p, t.col0 + h - 0.5 * n, 0.5 * n - t.row0 - h, p->Wg, &p->td0[(size_t)q * n_angles],
                            &p->ttauc[(size_t)q * n_angles]);
            }
    }
    // workspace layout
    const size_t fs = sizeof(float);
    const size_t ns = (size_t)n_angles * n_det, R = std::max(p->R, 1);
    const size_t gimg = (size_t)p->GT * p->GTP, ytile = (size_t)p->T * p->TP, ptile = (size_t)p->T * p->T;
    const int side = 2 * radius;
    const int nb = (n + 31) / 32;
    p->stitch_cap = n_roi * std::max(1, world) * ((side + 31) / 32 + 1) * ((side + 31) / 32 + 1);
    size_t o = 0;
    // LT_GUARD_BANDS: every region is followed by a canary band (from the first
    // 16-byte boundary after its last byte to 256 bytes past its aligned end),
    // filled at bind time and checked by lt_guard_check: any out-of-bounds write
    // of a kernel into the workspace shows up as a changed canary
    const bool guard = (flags & LT_GUARD_BANDS) != 0;
    auto take = [&](size_t bytes) {
        const size_t r = o;
        o = align256(o + bytes);
        if (guard) {
            const size_t g0 = (r + bytes + 15) & ~size_t(15);
            p->guards.push_back({g0, o + 256 - g0});
            o += 256;
        }
        return r;
    };
    auto& f = p->off;
    f.angf = take(n_angles * sizeof(AngF));
    f.cs64 = take(n_angles * 8); f.sn64 = take(n_angles * 8); f.A64 = take(n_angles * 8); f.B64 = take(n_angles * 8);
    f.tiles = take(R * sizeof(TileT)); f.d0 = take(R * n_angles * 4); f.tauc = take(R * n_angles * 8);
    f.gtile = take(sizeof(TileT)); f.gd0 = take(n_angles * 4); f.gtauc = take(n_angles * 8);
    f.ttiles = take(p->NTg * sizeof(TileT)); f.td0 = take((size_t)p->NTg * n_angles * 4);
    f.ttauc = take((size_t)p->NTg * n_angles * 8);
    f.tstack = take((size_t)p->NTg * p->Tg * p->TPg * fs); f.tstackT = take((size_t)p->NTg * p->Tg * p->TPg * fs);
    f.twin = take((size_t)p->NTg * n_angles * p->Wg * fs);
    f.fpgroups = take(p->fpgroups.size() * 4);
    f.fpgroups1 = take(p->fpgroups1.size() * 4);
    f.fpgroups24 = take(p->fpgroups24.size() * 4);
    // angle-split BP partials: up to 8 chunks x two waves of 32x32 CTAs (<= 160 SMs x 3)
    p->bpart_cap = 8LL * 2 * 3 * 160 * 32 * 32;
    f.bpart = take((size_t)p->bpart_cap * fs);
    // band-split FP partials: up to 8 splits x one wave of 8-angle CTAs (<= 3 x 160 SMs)
    p->fpart_cap = 8LL * 3 * 160 * 8 * 32 * FP_U;
    f.fpart = take((size_t)p->fpart_cap * fs);
    f.bank = take((size_t)n_iter * ns * fs); f.conv = take((size_t)n_iter * ns * fs);
    f.pc = take(ns * fs); f.wd = take(ns * fs); f.wdsum = take(n_angles * 8); f.psum = take(n_angles * 8);
    f.discc64 = take(8); f.discc32 = take(4); f.err = take(4);
    f.gimg = take(gimg * fs); f.gimgT = take(gimg * fs); f.gsino = take(ns * fs); f.gsino2 = take(ns * fs);
    const size_t nn = (size_t)n * n;
    f.gplain = take(nn * fs); f.gr = take(nn * fs); f.gs = take(nn * fs); f.gpo = take(nn * fs);
    f.gqo = take(nn * fs); f.gz = take(nn * fs); f.gxprev = take(nn * fs);
    f.y = take(R * ytile * fs); f.yT = take(R * ytile * fs); f.s = take(R * n_angles * p->Wwin * fs);
    f.v = take(R * ptile * fs); f.xs = take(R * ptile * fs); f.xprev = take(R * ptile * fs);
    for (int l = 0; l < 3; ++l) f.xsblk[l] = take(std::max<size_t>(p->xsblk[l].size(), 1) * 4);
    for (int l = 0; l < 2; ++l) f.xsg[l] = take((size_t)n * n * fs);
    f.lams = take(R * fs);
    f.cp_sd = take(ns * fs); f.cp_tau = take((size_t)n * n * fs); f.cp_yd = take(ns * fs);
    f.dwin = take(R * n_angles * p->Wwin * fs);
    f.peers = take(LT_MAX_PEERS * sizeof(void*));
    {   // FFT convolution cache: L = smallest power of two >= 2 N_d - 1
        // FFT length: the smallest 2^a 3^b 5^c >= 2 N_d - 1 (the circular
        // convolution of that length is the linear one on the bins kept; cuFFT's
        // mixed radices: C4 6144 instead of 8192, T1 3000 instead of 4096)
        int L = 1 << 30;
        for (long long a = 1; a < (1LL << 31); a *= 2)
            for (long long b = a; b < (1LL << 31); b *= 3)
                for (long long c = b; c < (1LL << 31); c *= 5)
                    if (c >= 2LL * n_det - 1 && c < L) L = (int)c;
        p->fftL = L; p->fftF = L / 2 + 1;
        p->fft_kc = std::max(1, std::min(n_iter, (int)((size_t)(256u << 20) / ((size_t)n_angles * L * 4))));
        const size_t F = p->fftF;
        f.uhat = take((size_t)n_iter * n_angles * F * 8);
        f.phat = take((size_t)n_angles * F * 8);
        f.fspec = take((size_t)p->fft_kc * n_angles * F * 8);
        f.freal = take((size_t)p->fft_kc * n_angles * L * fs);
        // cuFFT work area: host-side estimate (no device work at setup)
        size_t w1 = 0, w2 = 0, w3 = 0;
        int nL[1] = {L};
        cufftEstimateMany(1, nL, nullptr, 1, L, nullptr, 1, (int)F, CUFFT_R2C, n_angles, &w1);
        cufftEstimateMany(1, nL, nullptr, 1, L, nullptr, 1, (int)F, CUFFT_R2C, p->fft_kc * n_angles, &w2);
        cufftEstimateMany(1, nL, nullptr, 1, (int)F, nullptr, 1, L, CUFFT_C2R, p->fft_kc * n_angles, &w3);
        p->fwork_bytes = std::max(std::max(w1, w2), w3) + (1u << 20);
        f.fwork = take(p->fwork_bytes);
    }
    f.tt = take(ytile * fs); f.ttT = take(ytile * fs); f.tw = take((size_t)n_angles * p->Wwin * fs);
    f.st_off = take(((size_t)nb * nb + 1) * 4); f.st_lst = take((size_t)p->stitch_cap * 4);
    f.st_r0 = take((size_t)n_roi * std::max(1, world) * 4 + 4); f.st_c0 = take((size_t)n_roi * std::max(1, world) * 4 + 4);
    f.cores = take(R * side * side * fs); f.hsino = take(ns * fs); f.himg = take(nn * fs);
    f.gather = take((size_t)world * p->spr * side * side * fs);    // lt_combine_rois all-gather slots
    f.total = o;
    p->ws_bytes = (int64_t)o;
    *out = p;
    return LT_OK;
}

int64_t lt_plan_workspace_bytes(const lt_plan* p) { return p ? (int64_t)p->off.total : -1; }

int lt_plan_bind_workspace(lt_plan* p, void* d_ws, int64_t bytes, void* stream) {
    if (!p || !d_ws) return fail(LT_ERR_INVALID, "null plan/workspace");
    if (bytes < (int64_t)p->off.total) return fail(LT_ERR_INVALID, "workspace too small: %lld < %lld", (long long)bytes, (long long)p->off.total);
    if (((uintptr_t)d_ws) & 255) return fail(LT_ERR_INVALID, "workspace must be 256-byte aligned");
    cudaStream_t st = (cudaStream_t)stream;
    p->ws = (char*)d_ws;
    {
        int dev = 0;
        LT_CUDA(cudaGetDevice(&dev));
        LT_CUDA(cudaDeviceGetAttribute(&p->num_sms, cudaDevAttrMultiProcessorCount, dev));
    }
    auto up = [&](size_t o, const void* src, size_t bytes_) {
        return cudaMemcpyAsync(p->ws + o, src, bytes_, cudaMemcpyHostToDevice, st);
    };
    const size_t na = p->na;
    LT_CUDA(up(p->off.angf, p->angf.data(), na * sizeof(AngF)));
    LT_CUDA(up(p->off.cs64, p->cs64.data(), na * 8));
    LT_CUDA(up(p->off.sn64, p->sn64.data(), na * 8));
    LT_CUDA(up(p->off.A64, p->A64.data(), na * 8));
    LT_CUDA(up(p->off.B64, p->B64.data(), na * 8));
    LT_CUDA(up(p->off.tiles, p->tiles.data(), p->tiles.size() * sizeof(TileT)));
    LT_CUDA(up(p->off.d0, p->d0.data(), p->d0.size() * 4));
    LT_CUDA(up(p->off.tauc, p->tauc.data(), p->tauc.size() * 8));
    LT_CUDA(up(p->off.gtile, p->gtile.data(), sizeof(TileT)));
    LT_CUDA(up(p->off.gd0, p->gd0.data(), na * 4));
    LT_CUDA(up(p->off.gtauc, p->gtauc.data(), na * 8));
    LT_CUDA(up(p->off.ttiles, p->ttiles.data(), p->ttiles.size() * sizeof(TileT)));
    LT_CUDA(up(p->off.td0, p->td0.data(), p->td0.size() * 4));
    LT_CUDA(up(p->off.ttauc, p->ttauc.data(), p->ttauc.size() * 8));
    // the tile stack's padding columns stay zero (k_extract_tiles writes the tile columns only)
    LT_CUDA(cudaMemsetAsync(p->ws + p->off.tstack, 0, (size_t)p->NTg * p->Tg * p->TPg * sizeof(float), st));
    LT_CUDA(cudaMemsetAsync(p->ws + p->off.tstackT, 0, (size_t)p->NTg * p->Tg * p->TPg * sizeof(float), st));
    LT_CUDA(up(p->off.fpgroups, p->fpgroups.data(), p->fpgroups.size() * 4));
    LT_CUDA(up(p->off.fpgroups1, p->fpgroups1.data(), p->fpgroups1.size() * 4));
    LT_CUDA(up(p->off.fpgroups24, p->fpgroups24.data(), p->fpgroups24.size() * 4));
    for (int l = 0; l < 3; ++l)
        if (!p->xsblk[l].empty()) LT_CUDA(up(p->off.xsblk[l], p->xsblk[l].data(), p->xsblk[l].size() * 4));
    LT_CUDA(cudaMemsetAsync(p->ws + p->off.err, 0, 4, st));
    LT_CUDA(cudaMemsetAsync(p->ws + p->off.discc32, 0, 4, st));
    for (auto& g : p->guards) LT_CUDA(cudaMemsetAsync(p->ws + g.first, kGuardByte, g.second, st));
    LT_CUDA(cudaStreamSynchronize(st));
    if (!p->gst[0]) {
        const char* e = getenv("LT_SPLIT");
        p->nsplit = (e && atoi(e) == 2) ? 2 : 1;     // default: one stream (kernels fill the SMs; overlap gains ~2%)
        int lo_prio = 0, hi_prio = 0;
        LT_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
        const char* pe = getenv("LT_PRIO");
        const bool use_prio = !(pe && atoi(pe) == 0);
        for (int g = 0; g < 2; ++g) {
            LT_CUDA(cudaStreamCreateWithPriority(&p->gst[g], cudaStreamNonBlocking, lo_prio));
            if (use_prio) LT_CUDA(cudaStreamCreateWithPriority(&p->fst[g], cudaStreamNonBlocking, hi_prio));
            LT_CUDA(cudaEventCreateWithFlags(&p->pev[g], cudaEventDisableTiming));
            LT_CUDA(cudaEventCreateWithFlags(&p->fev[g], cudaEventDisableTiming));
            LT_CUDA(cudaEventCreateWithFlags(&p->bpev[g], cudaEventDisableTiming));
        }
        for (int g = 0; g < 3; ++g) LT_CUDA(cudaEventCreateWithFlags(&p->gev[g], cudaEventDisableTiming));
    }
    p->bound = true;
    p->bank_ready = p->wd_ready = p->spec_ready = false;
    p->st_key.clear();
    if (p->gexec) { cudaGraphExecDestroy(p->gexec); p->gexec = nullptr; }
    return LT_OK;
}

int32_t lt_plan_local_count(const lt_plan* p) { return p ? p->R : -1; }

int lt_plan_local_rois(const lt_plan* p, int32_t* out) {
    if (!p || !out) return fail(LT_ERR_INVALID, "null argument");
    for (int q = 0; q < p->R; ++q) out[q] = p->local[q];
    return LT_OK;
}

int lt_plan_tables(const lt_plan* p, int32_t* rects, int32_t* d0, int32_t* wwin) {
    if (!p) return fail(LT_ERR_INVALID, "null plan");
    for (int q = 0; q < p->R; ++q) {
        const TileT& t = p->tiles[q];
        if (rects) {
            int32_t* o = rects + 6 * q;
            o[0] = t.row0; o[1] = t.col0; o[2] = t.vr0; o[3] = t.vr1; o[4] = t.vc0; o[5] = t.vc1;
        }
        if (d0)
            for (int a = 0; a < p->na; ++a) d0[(size_t)q * p->na + a] = p->d0[(size_t)q * p->na + a];
    }
    if (wwin) *wwin = p->Wwin;
    return LT_OK;
}

int lt_filter_bank(lt_plan* p, void* stream) {
    if (int rc = check_plan(p)) return rc;
    NvtxRange nv("lt/filter_bank");
    cudaStream_t st = (cudaStream_t)stream;
    if (int rc = ensure_wd(*p, st)) return rc;
    // Alg. 1: c = e_c; for k: v = W c; u_k = u_{k-1} + alpha v; c <- c - alpha W^T v
    float* c = p->P<float>(p->off.gimg);
    float* cT = p->P<float>(p->off.gimgT);
    float* v = p->P<float>(p->off.gsino);
    const size_t gbytes = (size_t)p->GT * p->GTP * sizeof(float);
    LT_CUDA(cudaMemsetAsync(c, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(cT, 0, gbytes, st));
    k_impulse<<<1, 32, 0, st>>>(p->n, p->GTP, c, cT);
    LT_LAUNCHED();
    const long long ns = (long long)p->na * p->nd;
    const Tiles gt = p->glob_tiles();
    for (int k = 0; k < p->n_iter; ++k) {
        float* bk = p->P<float>(p->off.bank) + k * ns;
        const float* bprev = k ? bk - ns : nullptr;
        if (int rc = global_fp(*p, 1, c, cT, v, bprev, bk, st)) return rc;
        if (k + 1 < p->n_iter) {
            BpEpi e = epi0();
            e.y = c; e.yT = cT; e.y_tstride = 0; e.alpha = (float)p->alpha;
            const SinoView sv = view_full(v, p->nd);
            if (int rc = launch_bp_t<1, BP_ALG1>(*p, gt, sv, sv, e, st)) return rc;
        }
    }
    p->bank_ready = true;
    p->spec_ready = false;
    return LT_OK;
}

// ---- angle-split Alg. 1 (SURVEY §8(e) "cold bank"): rank g owns angles
// [a0, a1); per step it projects c on its angles (its bank rows) and
// backprojects them into a partial image; the caller all-reduces the partials
// (NCCL) and applies the sum.  The bank rows of other ranks are gathered by the
// caller afterwards (lt_get_bank / lt_set_bank).
int lt_bank_split_begin(lt_plan* p, int32_t a0, int32_t a1, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (a0 < 0 || a1 <= a0 || a1 > p->na) return fail(LT_ERR_INVALID, "angle range [%d, %d) invalid for %d angles", a0, a1, p->na);
    cudaStream_t st = (cudaStream_t)stream;
    float* c = p->P<float>(p->off.gimg);
    float* cT = p->P<float>(p->off.gimgT);
    const size_t gbytes = (size_t)p->GT * p->GTP * sizeof(float);
    LT_CUDA(cudaMemsetAsync(c, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(cT, 0, gbytes, st));
    k_impulse<<<1, 32, 0, st>>>(p->n, p->GTP, c, cT);
    LT_LAUNCHED();
    p->split_a0 = a0; p->split_a1 = a1;
    p->bank_ready = false;
    p->split_rows_ready = false;
    return LT_OK;
}

int lt_bank_split_step(lt_plan* p, int32_t k, float* d_partial, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (p->split_a1 <= 0) return fail(LT_ERR_INVALID, "lt_bank_split_begin not called");
    if (k < 0 || k >= p->n_iter) return fail(LT_ERR_INVALID, "step %d out of range", k);
    if (k + 1 < p->n_iter && !d_partial) return fail(LT_ERR_INVALID, "null partial image");
    cudaStream_t st = (cudaStream_t)stream;
    const long long ns = (long long)p->na * p->nd;
    float* c = p->P<float>(p->off.gimg);
    float* cT = p->P<float>(p->off.gimgT);
    float* v = p->P<float>(p->off.gsino);
    float* bk = p->P<float>(p->off.bank) + k * ns;
    p->a_lo = p->split_a0; p->a_hi = p->split_a1;
    int rc = global_fp(*p, 1, c, cT, v, k ? bk - ns : nullptr, bk, st);    // v_g = W_g c, u_k = u_{k-1} + alpha v_g
    if (!rc && k + 1 < p->n_iter) {                                        // partial = W_g^T v_g
        BpEpi e = epi0();
        e.out = d_partial; e.out_pitch = p->n;
        e.a_lo = p->split_a0; e.a_hi = p->split_a1;
        const SinoView sv = view_full(v, p->nd);
        rc = launch_bp_t<1, BP_PLAIN_GLOBAL>(*p, p->glob_tiles(), sv, sv, e, st);
    }
    p->a_lo = 0; p->a_hi = 0;
    if (!rc && k + 1 == p->n_iter) p->split_rows_ready = true;
    return rc;
}

int lt_bank_split_apply(lt_plan* p, const float* d_reduced, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (p->split_a1 <= 0) return fail(LT_ERR_INVALID, "lt_bank_split_begin not called");
    if (!d_reduced) return fail(LT_ERR_INVALID, "null reduced image");
    k_alg1_apply<<<dim3((p->n + 31) / 32, (p->n + 7) / 8), dim3(32, 8), 0, (cudaStream_t)stream>>>(
        p->n, p->GTP, d_reduced, (float)p->alpha, p->P<float>(p->off.gimg), p->P<float>(p->off.gimgT));
    LT_LAUNCHED();
    return LT_OK;
}

uint64_t lt_bank_key(const lt_plan* p) {
    if (!p) return 0;
    // FNV-1a over what the filters u_k depend on (Alg. 1): the grid N,
    // the angles (bit patterns), N_d, alpha, the projector (Joseph, V2)
    // and the impulse rule (reading A5); NOT n_iter: u_k does not depend on n
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](const void* d, size_t len) {
        const unsigned char* b = (const unsigned char*)d;
        for (size_t i = 0; i < len; ++i) { h ^= b[i]; h *= 1099511628211ull; }
    };
    const char tag[] = "loctomo-bank/joseph-v2/impulse-A5/alpha-1-over-NthetaNd";
    mix(tag, sizeof tag);
    mix(&p->n, sizeof p->n); mix(&p->na, sizeof p->na); mix(&p->nd, sizeof p->nd);
    mix(p->ang.data(), p->ang.size() * sizeof(double));
    mix(&p->alpha, sizeof p->alpha);
    return h;
}

int lt_set_bank(lt_plan* p, const float* d_bank, uint64_t key, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_bank) return fail(LT_ERR_INVALID, "null bank");
    if (key != lt_bank_key(p))
        return fail(LT_ERR_INVALID, "bank key %016llx does not match this plan's geometry (%016llx)",
                    (unsigned long long)key, (unsigned long long)lt_bank_key(p));
    LT_CUDA(cudaMemcpyAsync(p->ws + p->off.bank, d_bank, (size_t)p->n_iter * p->na * p->nd * sizeof(float),
                            cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    p->bank_ready = true;
    p->spec_ready = false;
    return LT_OK;
}

// bank file: header (magic, key, n, n_angles, n_det, n_iter, alpha) + fp32 u_1..u_{n_iter}
namespace {
struct BankHeader {
    char magic[8];
    uint64_t key;
    int32_t n, na, nd, n_iter;
    double alpha;
};
const char kBankMagic[8] = {'L', 'T', 'B', 'A', 'N', 'K', '0', '1'};
}  // namespace

int lt_save_bank(const lt_plan* p, const char* path, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!path) return fail(LT_ERR_INVALID, "null path");
    if (!p->bank_ready) return fail(LT_ERR_INVALID, "bank not computed");
    const size_t cnt = (size_t)p->n_iter * p->na * p->nd;
    std::vector<float> host(cnt);
    LT_CUDA(cudaMemcpyAsync(host.data(), p->ws + p->off.bank, cnt * sizeof(float), cudaMemcpyDeviceToHost,
                            (cudaStream_t)stream));
    LT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    BankHeader hd;
    memcpy(hd.magic, kBankMagic, 8);
    hd.key = lt_bank_key(p); hd.n = p->n; hd.na = p->na; hd.nd = p->nd; hd.n_iter = p->n_iter; hd.alpha = p->alpha;
    const std::string tmp = std::string(path) + ".tmp";
    FILE* f = fopen(tmp.c_str(), "wb");
    if (!f) return fail(LT_ERR_RUNTIME, "cannot open %s for writing", tmp.c_str());
    const bool ok = fwrite(&hd, sizeof hd, 1, f) == 1 && fwrite(host.data(), sizeof(float), cnt, f) == cnt;
    if (fclose(f) != 0 || !ok) { remove(tmp.c_str()); return fail(LT_ERR_RUNTIME, "write to %s failed", tmp.c_str()); }
    if (rename(tmp.c_str(), path) != 0) { remove(tmp.c_str()); return fail(LT_ERR_RUNTIME, "rename to %s failed", path); }
    return LT_OK;
}

int lt_load_bank(lt_plan* p, const char* path, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!path) return fail(LT_ERR_INVALID, "null path");
    FILE* f = fopen(path, "rb");
    if (!f) return fail(LT_ERR_RUNTIME, "cannot open %s", path);
    BankHeader hd;
    if (fread(&hd, sizeof hd, 1, f) != 1 || memcmp(hd.magic, kBankMagic, 8) != 0) {
        fclose(f);
        return fail(LT_ERR_INVALID, "%s is not a bank file", path);
    }
    if (hd.key != lt_bank_key(p) || hd.n != p->n || hd.na != p->na || hd.nd != p->nd || hd.alpha != p->alpha) {
        fclose(f);
        return fail(LT_ERR_INVALID, "%s was computed for another geometry (key %016llx, plan %016llx)", path,
                    (unsigned long long)hd.key, (unsigned long long)lt_bank_key(p));
    }
    if (hd.n_iter < p->n_iter) {
        fclose(f);
        return fail(LT_ERR_INVALID, "%s holds %d filters, the plan needs %d", path, hd.n_iter, p->n_iter);
    }
    // u_k does not depend on n: the first n_iter filters of a longer bank are this plan's
    const size_t cnt = (size_t)p->n_iter * p->na * p->nd;
    std::vector<float> host(cnt);
    const bool ok = fread(host.data(), sizeof(float), cnt, f) == cnt;
    fclose(f);
    if (!ok) return fail(LT_ERR_RUNTIME, "%s is truncated", path);
    LT_CUDA(cudaMemcpyAsync(p->ws + p->off.bank, host.data(), cnt * sizeof(float), cudaMemcpyHostToDevice,
                            (cudaStream_t)stream));
    LT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    p->bank_ready = true;
    p->spec_ready = false;
    return LT_OK;
}

int lt_get_bank(const lt_plan* p, float* d_bank, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!p->bank_ready && !p->split_rows_ready) return fail(LT_ERR_INVALID, "bank not computed");
    LT_CUDA(cudaMemcpyAsync(d_bank, p->ws + p->off.bank, (size_t)p->n_iter * p->na * p->nd * sizeof(float),
                            cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return LT_OK;
}

int lt_project(const lt_plan* cp, int32_t roi, const float* d_img, float* d_sino, void* stream) {
    if (int rc = check_plan(cp)) return rc;
    lt_plan* p = const_cast<lt_plan*>(cp);
    if (!d_img || !d_sino) return fail(LT_ERR_INVALID, "null pointer");
    if (roi < -1 || roi >= p->R) return fail(LT_ERR_INVALID, "roi %d out of range", roi);
    cudaStream_t st = (cudaStream_t)stream;
    if (roi < 0) {
        float* gi = p->P<float>(p->off.gimg);
        float* giT = p->P<float>(p->off.gimgT);
        const size_t gbytes = (size_t)p->GT * p->GTP * sizeof(float);
        LT_CUDA(cudaMemsetAsync(gi, 0, gbytes, st));
        LT_CUDA(cudaMemsetAsync(giT, 0, gbytes, st));
        k_pack<<<grid2d(p->n, p->n), dim3(32, 8), 0, st>>>(p->n, p->GTP, d_img, 0, gi, giT);
        LT_LAUNCHED();
        return global_fp(*p, 0, gi, giT, d_sino, nullptr, nullptr, st);
    }
    float* tt = p->P<float>(p->off.tt);
    float* ttT = p->P<float>(p->off.ttT);
    float* tw = p->P<float>(p->off.tw);
    const size_t tb = (size_t)p->T * p->TP * sizeof(float);
    LT_CUDA(cudaMemsetAsync(tt, 0, tb, st));
    LT_CUDA(cudaMemsetAsync(ttT, 0, tb, st));
    k_extract<<<grid2d(p->T, p->T), dim3(32, 8), 0, st>>>(p->n, p->T, p->TP, p->tiles[roi], d_img, tt, ttT);
    LT_LAUNCHED();
    // single-tile view of this ROI's tables
    Tiles t = p->roi_tiles();
    t.tile += roi; t.d0 += (size_t)roi * p->na; t.tauc += (size_t)roi * p->na; t.ntiles = 1;
    if (int rc = launch_fp_roi(*p, t, tt, ttT, 0, tw, 0, st)) return rc;
    k_scatter_win<<<dim3((p->nd + 255) / 256, p->na), 256, 0, st>>>(p->na, p->nd, p->Wwin, t.d0, tw, d_sino);
    LT_LAUNCHED();
    return LT_OK;
}

int lt_backproject(const lt_plan* cp, int32_t roi, const float* d_sino, float* d_img, void* stream) {
    if (int rc = check_plan(cp)) return rc;
    lt_plan* p = const_cast<lt_plan*>(cp);
    if (!d_img || !d_sino) return fail(LT_ERR_INVALID, "null pointer");
    if (roi < -1 || roi >= p->R) return fail(LT_ERR_INVALID, "roi %d out of range", roi);
    cudaStream_t st = (cudaStream_t)stream;
    BpEpi e = epi0();
    e.out = d_img; e.out_pitch = p->n;
    const SinoView sv = view_full(d_sino, p->nd);
    if (roi < 0) return launch_bp_t<1, BP_PLAIN_GLOBAL>(*p, p->glob_tiles(), sv, sv, e, st);
    LT_CUDA(cudaMemsetAsync(d_img, 0, (size_t)p->n * p->n * sizeof(float), st));
    Tiles t = p->roi_tiles();
    t.tile += roi; t.d0 += (size_t)roi * p->na; t.tauc += (size_t)roi * p->na; t.ntiles = 1;
    return launch_bp_t<1, BP_PLAIN_GLOBAL>(*p, t, sv, sv, e, st);
}

int lt_disc_correct(lt_plan* p, const float* d_sino, float* d_pc, float* d_c, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || !d_pc) return fail(LT_ERR_INVALID, "null pointer");
    return disc_correct(*p, d_sino, d_pc, d_c, (cudaStream_t)stream);
}

int lt_conv_cache(lt_plan* p, const float* d_pc, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_pc) return fail(LT_ERR_INVALID, "null pointer");
    return conv_cache(*p, d_pc, (cudaStream_t)stream);
}

int lt_get_conv(const lt_plan* p, float* d_out, void* stream) {
    if (int rc = check_plan(p)) return rc;
    LT_CUDA(cudaMemcpyAsync(d_out, p->ws + p->off.conv, (size_t)p->n_iter * p->na * p->nd * sizeof(float),
                            cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
    return LT_OK;
}

int lt_sirt_solve(lt_plan* p, const float* d_sino, float lo, float hi, float* d_cores, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || (!d_cores && p->R > 0)) return fail(LT_ERR_INVALID, "null pointer");
    if (!(lo <= hi)) return fail(LT_ERR_INVALID, "lo > hi");
    if (p->R == 0) return LT_OK;
    return solve(*p, 0, d_sino, lo, hi, 0, d_cores, (cudaStream_t)stream);
}

int lt_tv_solve(lt_plan* p, const float* d_sino, float lambda, int32_t n_fgp, float* d_cores, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || (!d_cores && p->R > 0)) return fail(LT_ERR_INVALID, "null pointer");
    if (!(lambda >= 0.f) || n_fgp < 1 || n_fgp > 4096) return fail(LT_ERR_INVALID, "lambda >= 0 and 1 <= n_fgp <= 4096 required");
    if (int rc = fgp_check(p->T, p->T)) return rc;
    if (p->R == 0) return LT_OK;
    return solve(*p, 1, d_sino, lambda, 0.f, n_fgp, d_cores, (cudaStream_t)stream);
}

int lt_get_ext(const lt_plan* p, float* d_ext, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (p->last_mode < 0) return fail(LT_ERR_INVALID, "no solve has run");
    const int E = p->T;
    dim3 grid((E + 31) / 32, (E + 7) / 8, p->R);
    cudaStream_t st = (cudaStream_t)stream;
    if (p->last_mode == 0)
        k_ext<<<grid, dim3(32, 8), 0, st>>>(E, p->P<TileT>(p->off.tiles), p->P<float>(p->off.y), p->ytile(), p->TP, PADL, d_ext);
    else
        k_ext<<<grid, dim3(32, 8), 0, st>>>(E, p->P<TileT>(p->off.tiles), p->P<float>(p->off.xprev), p->ptile(), p->T, 0, d_ext);
    LT_LAUNCHED();
    return LT_OK;
}

int lt_stitch_slots(const lt_plan* p, const float* d_cores_all, int32_t n_slots, const int32_t* h_slot_roi,
                    float* d_image, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_image || n_slots < 0 || (n_slots > 0 && (!d_cores_all || !h_slot_roi))) return fail(LT_ERR_INVALID, "bad arguments");
    return combine(*p, d_cores_all, n_slots, h_slot_roi, d_image, (cudaStream_t)stream);
}

int lt_guard_check(const lt_plan* p, int32_t* h_damaged, int64_t* h_bad_offset, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!h_damaged) return fail(LT_ERR_INVALID, "null output");
    if (p->guards.empty()) return fail(LT_ERR_INVALID, "plan was set up without LT_GUARD_BANDS");
    LT_CUDA(cudaStreamSynchronize((cudaStream_t)stream));
    std::vector<unsigned char> buf;
    int bad = 0;
    if (h_bad_offset) *h_bad_offset = -1;
    for (auto& g : p->guards) {
        buf.resize(g.second);
        LT_CUDA(cudaMemcpy(buf.data(), p->ws + g.first, g.second, cudaMemcpyDeviceToHost));
        for (size_t i = 0; i < g.second; ++i)
            if (buf[i] != kGuardByte) {
                if (!bad && h_bad_offset) *h_bad_offset = (int64_t)(g.first + i);
                ++bad;
                break;
            }
    }
    *h_damaged = bad;
    return LT_OK;
}

int32_t lt_window_width(int32_t h) { return h < 1 ? -1 : window_width(h); }

int lt_plan_slot_table(const lt_plan* p, int32_t* h_slot_roi, int32_t* h_spr) {
    if (!p) return fail(LT_ERR_INVALID, "null plan");
    if (h_spr) *h_spr = p->spr;
    if (h_slot_roi)
        for (size_t s = 0; s < p->slot_all.size(); ++s) h_slot_roi[s] = p->slot_all[s];
    return LT_OK;
}

int lt_nccl_get_unique_id(void* h_id) {
    if (!h_id) return fail(LT_ERR_INVALID, "null id buffer");
    NcclApi& a = nccl_api();
    if (!a.ok) return fail(LT_ERR_RUNTIME, "NCCL unavailable: %s", a.why.c_str());
    static_assert(sizeof(ncclUniqueId) == LT_NCCL_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    LT_NCCL(a.getUniqueId(&id));
    memcpy(h_id, &id, sizeof id);
    return LT_OK;
}

int lt_nccl_comm_init(int32_t world, int32_t rank, const void* h_id, void** comm) {
    if (!h_id || !comm || world < 1 || rank < 0 || rank >= world) return fail(LT_ERR_INVALID, "bad arguments");
    NcclApi& a = nccl_api();
    if (!a.ok) return fail(LT_ERR_RUNTIME, "NCCL unavailable: %s", a.why.c_str());
    ncclUniqueId id;
    memcpy(&id, h_id, sizeof id);
    ncclComm_t c = nullptr;
    LT_NCCL(a.commInitRank(&c, world, id, rank));
    *comm = c;
    return LT_OK;
}

int lt_nccl_comm_destroy(void* comm) {
    if (!comm) return fail(LT_ERR_INVALID, "null communicator");
    NcclApi& a = nccl_api();
    if (!a.ok) return fail(LT_ERR_RUNTIME, "NCCL unavailable: %s", a.why.c_str());
    LT_NCCL(a.commDestroy((ncclComm_t)comm));
    return LT_OK;
}

int lt_combine_rois(const lt_plan* p, const float* d_cores, float* d_image, void* nccl_comm, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_image || (p->R > 0 && !d_cores)) return fail(LT_ERR_INVALID, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const int side = 2 * p->radius;
    const long long slot = (long long)side * side;
    if (p->world == 1) {   // single rank: no collective, the local cores are the whole image's
        if (nccl_comm) {
            NcclApi& a = nccl_api();
            int cnt = 0;
            if (!a.ok) return fail(LT_ERR_RUNTIME, "NCCL unavailable: %s", a.why.c_str());
            LT_NCCL(a.commCount((ncclComm_t)nccl_comm, &cnt));
            if (cnt != 1) return fail(LT_ERR_INVALID, "communicator has %d ranks, the plan 1", cnt);
        }
        return combine(*p, d_cores, p->spr, p->slot_all.data(), d_image, st);
    }
    if (!nccl_comm) return fail(LT_ERR_INVALID, "plan of %d ranks needs a communicator", p->world);
    NcclApi& a = nccl_api();
    if (!a.ok) return fail(LT_ERR_RUNTIME, "NCCL unavailable: %s", a.why.c_str());
    int cnt = 0, me = -1;
    LT_NCCL(a.commCount((ncclComm_t)nccl_comm, &cnt));
    LT_NCCL(a.commUserRank((ncclComm_t)nccl_comm, &me));
    if (cnt != p->world || me != p->rank)
        return fail(LT_ERR_INVALID, "communicator rank %d of %d, plan rank %d of %d", me, cnt, p->rank, p->world);
    // own cores into this rank's slot block, then the in-place all-gather of the
    // fixed-size blocks (rank-major), then the stitch in ascending ROI order
    float* gbuf = p->P<float>(p->off.gather);
    float* mine = gbuf + (long long)p->rank * p->spr * slot;
    if (p->R > 0) LT_CUDA(cudaMemcpyAsync(mine, d_cores, (size_t)p->R * slot * sizeof(float), cudaMemcpyDeviceToDevice, st));
    LT_NCCL(a.allGather(mine, gbuf, (size_t)p->spr * slot, ncclFloat, (ncclComm_t)nccl_comm, st));
    return combine(*p, gbuf, p->world * p->spr, p->slot_all.data(), d_image, st);
}

int lt_combine_peers(const lt_plan* p, const float* const* h_peer_cores, int32_t world, int32_t slots_per_rank,
                     const int32_t* h_slot_roi, float* d_image, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_image || !h_peer_cores || !h_slot_roi || world < 1 || slots_per_rank < 1)
        return fail(LT_ERR_INVALID, "bad arguments");
    for (int g = 0; g < world; ++g)
        if (!h_peer_cores[g]) return fail(LT_ERR_INVALID, "null core buffer of rank %d", g);
    return combine(*p, nullptr, world * slots_per_rank, h_slot_roi, d_image, (cudaStream_t)stream, h_peer_cores, world,
                   slots_per_rank);
}

int lt_ipc_get_handle(const void* d_ptr, void* h_handle) {
    if (!d_ptr || !h_handle) return fail(LT_ERR_INVALID, "null pointer");
    cudaIpcMemHandle_t h;
    LT_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    memcpy(h_handle, &h, sizeof h);
    return LT_OK;
}

int lt_ipc_open_handle(const void* h_handle, void** d_ptr) {
    if (!h_handle || !d_ptr) return fail(LT_ERR_INVALID, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, h_handle, sizeof h);
    LT_CUDA(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return LT_OK;
}

int lt_ipc_close(void* d_ptr) {
    if (!d_ptr) return fail(LT_ERR_INVALID, "null pointer");
    LT_CUDA(cudaIpcCloseMemHandle(d_ptr));
    return LT_OK;
}

int lt_solve_host(lt_plan* p, int32_t mode, const float* h_sino, float p0, float p1, int32_t n_fgp, float* h_image,
                  void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!h_sino || !h_image) return fail(LT_ERR_INVALID, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    float* ds = p->P<float>(p->off.hsino);
    float* di = p->P<float>(p->off.himg);
    float* dc = p->P<float>(p->off.cores);
    LT_CUDA(cudaMemcpyAsync(ds, h_sino, (size_t)p->na * p->nd * sizeof(float), cudaMemcpyHostToDevice, st));
    int rc = mode == 0 ? lt_sirt_solve(p, ds, p0, p1, dc, st) : lt_tv_solve(p, ds, p0, n_fgp, dc, st);
    if (rc) return rc;
    std::vector<int> slots(p->local.begin(), p->local.end());
    if (int rc2 = combine(*p, dc, p->R, slots.data(), di, st)) return rc2;
    LT_CUDA(cudaMemcpyAsync(h_image, di, (size_t)p->n * p->n * sizeof(float), cudaMemcpyDeviceToHost, st));
    LT_CUDA(cudaStreamSynchronize(st));
    return LT_OK;
}

int lt_global_sirt(lt_plan* p, const float* d_sino, int32_t n_iter, float lo, float hi, float* d_img, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || !d_img || n_iter < 1 || !(lo <= hi)) return fail(LT_ERR_INVALID, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    float* x = p->P<float>(p->off.gimg);
    float* xT = p->P<float>(p->off.gimgT);
    float* r = p->P<float>(p->off.gsino);
    const size_t gbytes = (size_t)p->GT * p->GTP * sizeof(float);
    LT_CUDA(cudaMemsetAsync(x, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(xT, 0, gbytes, st));
    const Tiles gt = p->glob_tiles();
    for (int k = 0; k < n_iter; ++k) {
        if (int rc = global_fp(*p, 2, x, xT, r, d_sino, nullptr, st)) return rc;   // r = p - W x
        BpEpi e = epi0();
        e.y = x; e.yT = xT; e.alpha = (float)p->alpha; e.lo = lo; e.hi = hi;
        const SinoView sv = view_full(r, p->nd);
        if (int rc = launch_bp_t<1, BP_GSIRT>(*p, gt, sv, sv, e, st)) return rc;
    }
    k_unpack<<<grid2d(p->n, p->n), dim3(32, 8), 0, st>>>(p->n, p->GTP, x, d_img);
    LT_LAUNCHED();
    return LT_OK;
}

// ---- angle-split global box-SIRT ("the same pattern serves
// GLOBAL-mode solves"): rank g owns angles [a0, a1); per iteration it forms its
// residual rows r_g = p_g - W_g x and the partial image W_g^T r_g; the caller
// all-reduces the partials and applies the sum with the box clamp.
int lt_global_split_begin(lt_plan* p, int32_t a0, int32_t a1, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (a0 < 0 || a1 <= a0 || a1 > p->na) return fail(LT_ERR_INVALID, "angle range [%d, %d) invalid for %d angles", a0, a1, p->na);
    cudaStream_t st = (cudaStream_t)stream;
    const size_t gbytes = (size_t)p->GT * p->GTP * sizeof(float);
    LT_CUDA(cudaMemsetAsync(p->P<float>(p->off.gimg), 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(p->P<float>(p->off.gimgT), 0, gbytes, st));
    p->gsplit_a0 = a0; p->gsplit_a1 = a1;
    return LT_OK;
}

int lt_global_split_step(lt_plan* p, const float* d_sino, float* d_partial, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (p->gsplit_a1 <= 0) return fail(LT_ERR_INVALID, "lt_global_split_begin not called");
    if (!d_sino || !d_partial) return fail(LT_ERR_INVALID, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    float* x = p->P<float>(p->off.gimg);
    float* xT = p->P<float>(p->off.gimgT);
    float* r = p->P<float>(p->off.gsino);
    p->a_lo = p->gsplit_a0; p->a_hi = p->gsplit_a1;
    int rc = global_fp(*p, 2, x, xT, r, d_sino, nullptr, st);               // r_g = p_g - W_g x
    if (!rc) {                                                             // partial = W_g^T r_g
        BpEpi e = epi0();
        e.out = d_partial; e.out_pitch = p->n;
        e.a_lo = p->gsplit_a0; e.a_hi = p->gsplit_a1;
        const SinoView sv = view_full(r, p->nd);
        rc = launch_bp_t<1, BP_PLAIN_GLOBAL>(*p, p->glob_tiles(), sv, sv, e, st);
    }
    p->a_lo = 0; p->a_hi = 0;
    return rc;
}

int lt_global_split_apply(lt_plan* p, const float* d_reduced, float lo, float hi, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (p->gsplit_a1 <= 0) return fail(LT_ERR_INVALID, "lt_global_split_begin not called");
    if (!d_reduced || !(lo <= hi)) return fail(LT_ERR_INVALID, "bad arguments");
    k_gsirt_apply<<<grid2d(p->n, p->n), dim3(32, 8), 0, (cudaStream_t)stream>>>(
        p->n, p->GTP, d_reduced, (float)p->alpha, lo, hi, p->P<float>(p->off.gimg), p->P<float>(p->off.gimgT));
    LT_LAUNCHED();
    return LT_OK;
}

int lt_global_split_result(lt_plan* p, float* d_img, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (p->gsplit_a1 <= 0) return fail(LT_ERR_INVALID, "lt_global_split_begin not called");
    if (!d_img) return fail(LT_ERR_INVALID, "null pointer");
    k_unpack<<<grid2d(p->n, p->n), dim3(32, 8), 0, (cudaStream_t)stream>>>(p->n, p->GTP, p->P<float>(p->off.gimg), d_img);
    LT_LAUNCHED();
    return LT_OK;
}

int lt_global_tv(lt_plan* p, const float* d_sino, int32_t n_iter, float lambda, int32_t n_fgp, float* d_img,
                 void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || !d_img || n_iter < 1 || !(lambda >= 0.f) || n_fgp < 1) return fail(LT_ERR_INVALID, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int n = p->n;
    float* xm = p->P<float>(p->off.gimg);     // momentum point r^k (padded + twin)
    float* xmT = p->P<float>(p->off.gimgT);
    float* r = p->P<float>(p->off.gsino);
    float* v = p->P<float>(p->off.gplain);
    float* gr = p->P<float>(p->off.gr);
    float* gs = p->P<float>(p->off.gs);
    float* gpo = p->P<float>(p->off.gpo);
    float* gqo = p->P<float>(p->off.gqo);
    float* gz = p->P<float>(p->off.gz);
    float* xprev = p->P<float>(p->off.gxprev);
    const size_t gbytes = (size_t)p->GT * p->GTP * sizeof(float), nb = (size_t)n * n * sizeof(float);
    LT_CUDA(cudaMemsetAsync(xm, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(xmT, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(xprev, 0, nb, st));
    const Tiles gt = p->glob_tiles();
    const dim3 g2 = grid2d(n, n), b2(32, 8);
    double tk = 1.0;
    for (int k = 0; k < n_iter; ++k) {
        if (int rc = global_fp(*p, 2, xm, xmT, r, d_sino, nullptr, st)) return rc;
        BpEpi e = epi0();
        e.y = xm; e.out = v; e.alpha = (float)p->alpha;
        const SinoView sv = view_full(r, p->nd);
        if (int rc = launch_bp_t<1, BP_GTV>(*p, gt, sv, sv, e, st)) return rc;    // v = S(r^{k-1})
        LT_CUDA(cudaMemsetAsync(gr, 0, nb, st));
        LT_CUDA(cudaMemsetAsync(gs, 0, nb, st));
        LT_CUDA(cudaMemsetAsync(gpo, 0, nb, st));
        LT_CUDA(cudaMemsetAsync(gqo, 0, nb, st));
        if (lambda > 0.f) {
            double ti = 1.0;
            for (int it = 0; it < n_fgp; ++it) {
                k_gfgp_z<<<g2, b2, 0, st>>>(n, lambda, v, gr, gs, gz);
                LT_LAUNCHED();
                const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * ti * ti));
                const float beta = (float)((ti - 1.0) / tn);
                ti = tn;
                k_gfgp_dual<<<g2, b2, 0, st>>>(n, 1.f / (8.f * lambda), beta, gz, gr, gs, gpo, gqo);
                LT_LAUNCHED();
            }
        }
        const double tn = 0.5 * (1.0 + std::sqrt(1.0 + 4.0 * tk * tk));
        const float beta_o = (float)((tk - 1.0) / tn);
        tk = tn;
        k_gfgp_out<<<g2, b2, 0, st>>>(n, lambda, beta_o, v, gpo, gqo, xprev, xm, xmT, p->GTP);
        LT_LAUNCHED();
    }
    LT_CUDA(cudaMemcpyAsync(d_img, xprev, nb, cudaMemcpyDeviceToDevice, st));
    return LT_OK;
}

int lt_exterior_solve(lt_plan* p, const float* d_sino, float lo, float hi, float* d_cores, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || (!d_cores && p->R > 0)) return fail(LT_ERR_INVALID, "null pointer");
    if (!(lo <= hi)) return fail(LT_ERR_INVALID, "lo <= hi required");
    if (p->R == 0) return LT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    lt_plan& P = *p;
    const int n = P.n;
    // 1. global reconstruction xg = W^T C_{u_n} p_c + c D (FBP with the SIRT filter u_n, eq. sfbp)
    float* pc = P.P<float>(P.off.pc);
    if (P.flags & LT_DISC_ON) {
        if (int rc = disc_correct(P, d_sino, pc, nullptr, st)) return rc;
    } else {
        LT_CUDA(cudaMemcpyAsync(pc, d_sino, (size_t)P.na * P.nd * sizeof(float), cudaMemcpyDeviceToDevice, st));
        LT_CUDA(cudaMemsetAsync(P.P<float>(P.off.discc32), 0, sizeof(float), st));
    }
    if (int rc = conv_cache(P, pc, st)) return rc;
    const Tiles gt = P.glob_tiles();
    float* xg = P.P<float>(P.off.gplain);
    {
        BpEpi ex = epi0();
        ex.out = xg; ex.out_pitch = n;
        const SinoView vb = view_full(P.P<float>(P.off.conv) + (long long)(P.n_iter - 1) * P.na * P.nd, P.nd);
        if (int rc = launch_bp_t<1, BP_PLAIN_GLOBAL>(P, gt, vb, vb, ex, st)) return rc;
    }
    float* gx = P.P<float>(P.off.gimg);
    float* gxT = P.P<float>(P.off.gimgT);
    const size_t gbytes = (size_t)P.GT * P.GTP * sizeof(float);
    LT_CUDA(cudaMemsetAsync(gx, 0, gbytes, st));        // zero padding columns (Joseph taps)
    LT_CUDA(cudaMemsetAsync(gxT, 0, gbytes, st));
    k_pack_disc<<<grid2d(n, n), dim3(32, 8), 0, st>>>(n, P.GTP, xg, P.P<float>(P.off.discc32),
                                                     (P.flags & LT_DISC_ON) ? 1 : 0, gx, gxT);
    LT_LAUNCHED();
    // 2. r_g = p - W xg on the full sinogram
    float* rg = P.P<float>(P.off.gsino);
    if (int rc = global_fp(P, 2, gx, gxT, rg, d_sino, nullptr, st)) return rc;
    // 3. per ROI: p~ = r_g + W_{L'} xg on the window, x_d = alpha W_{L'}^T p~
    Tiles t = P.roi_tiles();
    const long long yts = P.ytile();
    float* y = P.P<float>(P.off.y);
    float* yT = P.P<float>(P.off.yT);
    float* s = P.P<float>(P.off.s);
    float* dw = P.P<float>(P.off.dwin);
    float* xd = P.P<float>(P.off.xs);
    LT_CUDA(cudaMemsetAsync(y, 0, (size_t)P.R * yts * sizeof(float), st));     // zero padding columns
    LT_CUDA(cudaMemsetAsync(yT, 0, (size_t)P.R * yts * sizeof(float), st));
    k_extract_tiles<<<dim3((P.T + 31) / 32, (P.T + 7) / 8, P.R), dim3(32, 8), 0, st>>>(
        P.T, P.TP, P.P<TileT>(P.off.tiles), gx, P.GTP, y, yT, yts);
    LT_LAUNCHED();
    if (int rc = launch_fp_roi(P, t, y, yT, yts, s, (long long)P.na * P.Wwin, st)) return rc;
    k_dwin<<<dim3((P.Wwin + 127) / 128, P.na, P.R), 128, 0, st>>>(P.na, P.nd, P.Wwin, P.P<int>(P.off.d0), rg, s, dw);
    LT_LAUNCHED();
    {
        BpEpi e = epi0();
        e.out = xd; e.out_tstride = P.ptile();
        const SinoView vd = view_win(dw, P.Wwin, P.na);
        if (int rc = launch_bp_t<1, BP_PLAIN_TILE>(P, t, vd, vd, e, st)) return rc;
        const long long ne = (long long)P.R * P.ptile();
        k_scale<<<(unsigned)((ne + 255) / 256), 256, 0, st>>>(ne, (float)P.alpha, xd);
        LT_LAUNCHED();
    }
    // 4. box-SIRT on L' from 0: x <- clamp(x + x_d - alpha W_{L'}^T W_{L'} x); y holds x
    LT_CUDA(cudaMemsetAsync(y, 0, (size_t)P.R * yts * sizeof(float), st));
    LT_CUDA(cudaMemsetAsync(yT, 0, (size_t)P.R * yts * sizeof(float), st));
    for (int k = 0; k < P.n_iter; ++k) {
        BpEpi e = epi0();
        e.xs_tile = xd; e.p_tstride = P.ptile();
        e.y = y; e.yT = yT; e.y_tstride = yts;
        e.alpha = (float)P.alpha; e.lo = lo; e.hi = hi; e.last = 1;       // store x itself every iteration
        if (k == 0) {
            const SinoView v0 = view_win(dw, P.Wwin, P.na);
            if (int rc = launch_bp_t<0, BP_BOX>(P, t, v0, v0, e, st)) return rc;
        } else {
            if (int rc = launch_fp_roi(P, t, y, yT, yts, s, (long long)P.na * P.Wwin, st)) return rc;
            const SinoView vs = view_win(s, P.Wwin, P.na);
            if (int rc = launch_bp_t<1, BP_BOX>(P, t, vs, vs, e, st)) return rc;
        }
    }
    P.last_mode = 0;
    return crop_cores(P, d_cores, st);
}

int lt_global_cp(lt_plan* p, const float* d_sino, int32_t n_iter, float mu, float* d_img, void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || !d_img || n_iter < 1 || !(mu >= 0.f)) return fail(LT_ERR_INVALID, "bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    const int n = p->n;
    const long long ns = (long long)p->na * p->nd, nn = (long long)n * n;
    float* xb = p->P<float>(p->off.gimg);
    float* xbT = p->P<float>(p->off.gimgT);
    float* s = p->P<float>(p->off.gsino);
    float* g = p->P<float>(p->off.gplain);
    float* yp = p->P<float>(p->off.gr);
    float* yq = p->P<float>(p->off.gs);
    float* x = p->P<float>(p->off.gxprev);
    float* sd = p->P<float>(p->off.cp_sd);
    float* tau = p->P<float>(p->off.cp_tau);
    float* yd = p->P<float>(p->off.cp_yd);
    const size_t gbytes = (size_t)p->GT * p->GTP * sizeof(float);
    const Tiles gt = p->glob_tiles();
    const dim3 g2 = grid2d(n, n), b2(32, 8);
    // preconditioners: W 1 (rays) and W^T 1 (pixels)
    LT_CUDA(cudaMemsetAsync(xb, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(xbT, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(g, 0, nn * sizeof(float), st));
    k_pack<<<g2, b2, 0, st>>>(n, p->GTP, nullptr, 2, xb, xbT);            // ones image
    LT_LAUNCHED();
    if (int rc = global_fp(*p, 0, xb, xbT, s, nullptr, nullptr, st)) return rc;
    k_cp_recip<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(ns, s, sd);
    LT_LAUNCHED();
    k_fill<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(ns, 1.f, s);
    LT_LAUNCHED();
    {
        BpEpi e = epi0();
        e.out = g; e.out_pitch = n;
        const SinoView sv = view_full(s, p->nd);
        if (int rc = launch_bp_t<1, BP_PLAIN_GLOBAL>(*p, gt, sv, sv, e, st)) return rc;
    }
    k_cp_tau<<<g2, b2, 0, st>>>(n, g, tau);
    LT_LAUNCHED();
    // state: x = xbar = 0, duals 0
    LT_CUDA(cudaMemsetAsync(xb, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(xbT, 0, gbytes, st));
    LT_CUDA(cudaMemsetAsync(x, 0, nn * sizeof(float), st));
    LT_CUDA(cudaMemsetAsync(yp, 0, nn * sizeof(float), st));
    LT_CUDA(cudaMemsetAsync(yq, 0, nn * sizeof(float), st));
    LT_CUDA(cudaMemsetAsync(yd, 0, ns * sizeof(float), st));
    for (int k = 0; k < n_iter; ++k) {
        if (int rc = global_fp(*p, 0, xb, xbT, s, nullptr, nullptr, st)) return rc;     // W xbar
        k_cp_dual<<<(unsigned)((ns + 255) / 256), 256, 0, st>>>(ns, s, d_sino, sd, yd);
        LT_LAUNCHED();
        k_cp_tvdual<<<g2, b2, 0, st>>>(n, p->GTP, mu, xb, yp, yq);
        LT_LAUNCHED();
        BpEpi e = epi0();
        e.out = g; e.out_pitch = n;
        const SinoView sv = view_full(yd, p->nd);
        if (int rc = launch_bp_t<1, BP_PLAIN_GLOBAL>(*p, gt, sv, sv, e, st)) return rc;            // W^T yd
        k_cp_primal<<<g2, b2, 0, st>>>(n, p->GTP, g, yp, yq, tau, x, xb, xbT);
        LT_LAUNCHED();
    }
    LT_CUDA(cudaMemcpyAsync(d_img, x, nn * sizeof(float), cudaMemcpyDeviceToDevice, st));
    return LT_OK;
}

int lt_fgp_batch(int32_t h, int32_t w, int32_t count, const float* d_in, float lambda, int32_t n_fgp, float* d_out,
                 void* stream) {
    if (h < 1 || w < 1 || count < 0 || !(lambda >= 0.f) || n_fgp < 1 || n_fgp > 4096 || h > FGP2_ROW_MAX ||
        w > FGP2_ROW_MAX)
        return fail(LT_ERR_INVALID, "bad FGP arguments");
    if (count == 0) return LT_OK;
    if (!d_in || !d_out) return fail(LT_ERR_INVALID, "null pointer");
    FgpArgs A;
    memset(&A, 0, sizeof A);
    A.b = d_in; A.b_pitch = w; A.b_tstride = (long long)h * w;
    A.tiles = nullptr; A.H = h; A.W = w;
    A.lam = lambda; A.nfgp = n_fgp;
    A.out = d_out; A.out_pitch = w; A.out_tstride = (long long)h * w;
    return launch_fgp<0>(A, h, w, count, (cudaStream_t)stream);
}

int lt_haar_solve(lt_plan* p, const float* d_sino, float lambda, int32_t levels, int32_t momentum, float* d_cores,
                  void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || (!d_cores && p->R > 0)) return fail(LT_ERR_INVALID, "null pointer");
    if (!(lambda >= 0.f) || levels < 0 || levels > 5) return fail(LT_ERR_INVALID, "lambda >= 0 and 0 <= levels <= 5 required");
    for (int q = 0; q < p->R; ++q) {
        const TileT& t = p->tiles[q];
        if ((t.vr1 - t.vr0) % (1 << levels) || (t.vc1 - t.vc0) % (1 << levels))
            return fail(LT_ERR_INVALID, "ROI %d: extended rect %dx%d not divisible by 2^%d", p->local[q],
                        t.vr1 - t.vr0, t.vc1 - t.vc0, levels);
    }
    if (p->R == 0) return LT_OK;
    p->haar_momentum = momentum != 0;
    return solve(*p, 2, d_sino, lambda, 0.f, levels, d_cores, (cudaStream_t)stream);
}

int lt_tv_solve_lambdas(lt_plan* p, const float* d_sino, const float* h_lambdas, int32_t n_fgp, float* d_cores,
                        void* stream) {
    if (int rc = check_plan(p)) return rc;
    if (!d_sino || (p->R > 0 && (!d_cores || !h_lambdas))) return fail(LT_ERR_INVALID, "null pointer");
    if (n_fgp < 1 || n_fgp > 4096) return fail(LT_ERR_INVALID, "1 <= n_fgp <= 4096 required");
    for (int q = 0; q < p->R; ++q)
        if (!(h_lambdas[q] >= 0.f)) return fail(LT_ERR_INVALID, "lambda[%d] must be >= 0", q);
    if (int rc = fgp_check(p->T, p->T)) return rc;
    if (p->R == 0) return LT_OK;
    cudaStream_t st = (cudaStream_t)stream;
    LT_CUDA(cudaMemcpyAsync(p->P<float>(p->off.lams), h_lambdas, (size_t)p->R * sizeof(float), cudaMemcpyHostToDevice, st));
    p->lam_array = true;
    const int rc = solve(*p, 1, d_sino, 0.f, 0.f, n_fgp, d_cores, st);
    p->lam_array = false;
    return rc;
}

int lt_metrics(const float* d_x, const float* d_ref, int32_t count, int32_t h, int32_t w, float data_range,
               double* d_mse, double* d_ssim, void* stream) {
    if (count < 0 || h < 1 || w < 1) return fail(LT_ERR_INVALID, "count >= 0, h, w >= 1 required");
    if (count == 0) return LT_OK;
    if (!d_x || !d_ref || !d_mse || !d_ssim) return fail(LT_ERR_INVALID, "null pointer");
    static uint64_t have_w = 0;       // per device: __constant__ memory is per device
    const int dv = cur_dev();
    if (dv < 0) return fail(LT_ERR_RUNTIME, "cudaGetDevice failed or device ordinal >= %d", LT_MAX_DEV);
    std::lock_guard<std::mutex> lk(g_dev_mu);
    if (!(have_w >> dv & 1)) {   // 11 x 11 Gaussian, sigma 1.5, normalised (fp64 on the host)
        double wt[121], s = 0.0;
        for (int a = 0; a < 11; ++a)
            for (int b = 0; b < 11; ++b) { wt[a * 11 + b] = std::exp(-((a - 5) * (a - 5) + (b - 5) * (b - 5)) / (2.0 * 1.5 * 1.5)); s += wt[a * 11 + b]; }
        float wf[121];
        for (int e = 0; e < 121; ++e) wf[e] = (float)(wt[e] / s);
        LT_CUDA(cudaMemcpyToSymbol(c_ssim_w, wf, sizeof wf));
        have_w |= 1ull << dv;
    }
    k_metrics<<<count, 256, 0, (cudaStream_t)stream>>>(h, w, d_x, d_ref, data_range, d_mse, d_ssim);
    LT_LAUNCHED();
    return LT_OK;
}

int lt_nelder_mead_1d(double (*f)(double, void*), void* ctx, double t_lo, double t_hi, int32_t budget,
                      double* t_best, double* f_best, int32_t* n_eval) {
    if (!f || !t_best || !f_best) return fail(LT_ERR_INVALID, "null pointer");
    if (!(t_lo < t_hi) || budget < 3) return fail(LT_ERR_INVALID, "need t_lo < t_hi and budget >= 3");
    // Nelder & Mead (1965) in one dimension, coefficients 1, 2, 1/2, 1/2; initial
    // simplex {mid, mid + 0.5} (SPEC S:L499 reading); every point
    // is clamped into [t_lo, t_hi]; the best evaluated point is returned.
    int ne = 0;
    double bx = 0.0, bf = INFINITY;
    auto F = [&](double t) {
        t = std::min(std::max(t, t_lo), t_hi);
        const double v = f(t, ctx);
        ++ne;
        if (v < bf || ne == 1) { bf = v; bx = t; }
        return v;
    };
    auto clampt = [&](double t) { return std::min(std::max(t, t_lo), t_hi); };
    const double mid = 0.5 * (t_lo + t_hi);
    double x0 = mid, x1 = clampt(mid + 0.5);
    if (x1 == x0) x1 = clampt(mid - 0.5);
    double f0 = F(x0), f1 = F(x1);
    while (ne < budget) {
        if (f1 < f0) { std::swap(x0, x1); std::swap(f0, f1); }      // x0 best, x1 worst
        if (std::fabs(x1 - x0) < 1e-9) break;
        const double xr = clampt(x0 + (x0 - x1));
        const double fr = F(xr);
        if (fr < f0) {
            if (ne < budget) {
                const double xe = clampt(x0 + 2.0 * (xr - x0));
                const double fe = F(xe);
                if (fe < fr) { x1 = xe; f1 = fe; } else { x1 = xr; f1 = fr; }
            } else { x1 = xr; f1 = fr; }
            continue;
        }
        if (ne >= budget) break;
        if (fr < f1) {                                             // outside contraction
            const double xc = clampt(x0 + 0.5 * (xr - x0));
            const double fc = F(xc);
            if (fc <= fr) { x1 = xc; f1 = fc; continue; }
        } else {                                                   // inside contraction
            const double xc = clampt(x0 + 0.5 * (x1 - x0));
            const double fc = F(xc);
            if (fc < f1) { x1 = xc; f1 = fc; continue; }
        }
        if (ne >= budget) break;
        x1 = x0 + 0.5 * (x1 - x0);                                 // shrink towards the best point
        f1 = F(x1);
    }
    *t_best = bx; *f_best = bf;
    if (n_eval) *n_eval = ne;
    return LT_OK;
}

int lt_pad_truncated(const float* d_in, int32_t n_angles, int32_t n_trunc, int32_t n_det, float* d_out,
                     void* stream) {
    if (n_angles < 1 || n_trunc < 1 || n_det < n_trunc || (n_det - n_trunc) % 2)
        return fail(LT_ERR_INVALID, "pad_truncated: need n_angles >= 1, 1 <= n_trunc <= n_det, n_det - n_trunc even");
    if (!d_in || !d_out) return fail(LT_ERR_INVALID, "null pointer");
    dim3 grid((n_det + 255) / 256, n_angles);
    k_pad_truncated<<<grid, 256, 0, (cudaStream_t)stream>>>(n_angles, n_trunc, n_det, d_in, d_out);
    LT_LAUNCHED();
    return LT_OK;
}

void lt_plan_destroy(lt_plan* p) {
    if (!p) return;
    for (int g = 0; g < 2; ++g) {
        if (p->gst[g]) cudaStreamDestroy(p->gst[g]);
        if (p->fst[g]) cudaStreamDestroy(p->fst[g]);
        if (p->pev[g]) cudaEventDestroy(p->pev[g]);
        if (p->fev[g]) cudaEventDestroy(p->fev[g]);
        if (p->bpev[g]) cudaEventDestroy(p->bpev[g]);
    }
    for (int g = 0; g < 3; ++g)
        if (p->gev[g]) cudaEventDestroy(p->gev[g]);
    if (p->gexec) cudaGraphExecDestroy(p->gexec);
    if (p->gs) cudaStreamDestroy(p->gs);
    if (p->xst) cudaStreamDestroy(p->xst);
    if (p->xev_bp) cudaEventDestroy(p->xev_bp);
    if (p->xev_xs) cudaEventDestroy(p->xev_xs);
    if (p->gev_in) cudaEventDestroy(p->gev_in);
    if (p->gev_out) cudaEventDestroy(p->gev_out);
    if (p->plan_r2c_p) cufftDestroy(p->plan_r2c_p);
    if (p->plan_r2c_k) cufftDestroy(p->plan_r2c_k);
    if (p->plan_c2r_k) cufftDestroy(p->plan_c2r_k);
    delete p;
}

}  // extern "C"
