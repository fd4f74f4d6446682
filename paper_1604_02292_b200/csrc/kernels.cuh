// kernels.cuh -- sm_100a kernels of the local tomography hot path.
//
// Notation follows PAPER.md (arXiv 1604.02292) and DESIGN.md:
//   W   Joseph projector, W[(a,d),(i,j)] = hat((t_d - t_ij)/c_a)/c_a      (V2)
//   "tile"  = a square block of pixels processed as one unit: the extended
//             ROI L' of one local reconstruction, or the
//             whole N x N grid for the global operators (Alg. 1, a10).
//   "window" = the contiguous run of detector bins that a tile can reach at
//             one angle (V4); W_{L'} is evaluated only there.
//
// Layouts (DESIGN.md §Data layout):
//   padded tile image  [tile][T][TP], data at columns PADL..PADL+T-1, two-sided
//                      zero padding so Joseph taps never need bounds checks.
//                      Every padded image has a transposed twin (lines = columns)
//                      so column-driven angles march contiguous memory too.
//   plain tile image   [tile][T][T]
//   window sinogram    [tile][N_theta][Wwin]
//   sinogram           [N_theta][N_d]
#pragma once
#include <cuda_runtime.h>
#include <cooperative_groups.h>
#include <stdint.h>
#include <type_traits>

namespace lt {
namespace cg = cooperative_groups;

constexpr int PADL = 4;           // left zero padding of padded tile rows
constexpr int PADR = 4;           // right zero padding
constexpr float MAGICF = 12582912.0f;   // 1.5 * 2^23: x + MAGICF rounds x to an integer in the low mantissa bits
constexpr int MAGICI = 0x4B400000;

struct AngF {       // per-angle constants (fp32), 32 B
    float cs, sn;   // cos, sin
    float invc;     // 1/c, c = max(|cos|,|sin|)
    float ic2;      // 1/c^2
    float K;        // 1/c - 0.5/c^2  (hat weights in the magic-floor form)
    float A, B;     // Joseph marching: pos(w, l) = Lc + (w - tau_c) A + (l - Lc) B
    int col;        // 1 = column-driven (|sin| > |cos|): march columns on the transposed image
};

struct TileT {      // per tile, tile-local coordinates
    int row0, col0;           // global coords of tile pixel (0,0) (negative if clipped)
    int vr0, vr1, vc0, vc1;   // valid rectangle (inside the grid), half-open
    int pad0, pad1;
};

struct Geo {
    int n, na, nd;
    const AngF* ang;
    const double* cs64;
    const double* sn64;
    const double* A64;
    const double* B64;
};

struct Tiles {
    int T, TP, Wwin, ntiles;
    const TileT* tile;
    const int* d0;          // [tile][na] window start (global bin index)
    const double* tauc;     // [tile][na] bin coordinate of the tile centre relative to d0
};

struct SinoView {           // element (tile r, angle a, window bin w)
    const float* base;
    long long tile_stride;  // elements between tiles (0 = shared sinogram)
    int row_stride;         // elements between angles
    int use_d0;             // 1: index = d0[r][a] + w (full sinogram); 0: index = w (window sinogram)
    int len;                // valid index range [0, len)
};

__device__ __forceinline__ float sv_fetch(const SinoView& s, const int* d0, int na, int r, int a, int w) {
    const int idx = (s.use_d0 ? __ldg(d0 + r * na + a) : 0) + w;
    if (idx < 0 || idx >= s.len) return 0.f;
    return __ldg(s.base + (long long)r * s.tile_stride + (long long)a * s.row_stride + idx);
}

// ---------------------------------------------------------------------------
// Forward projection W_{L'} (ray driven, Joseph).  One thread = one ray
// (tile r, angle a, window bin w).  The ray marches the lines (rows for
// row-driven angles, columns via the transposed image otherwise) that its
// footprint can touch inside the valid rectangle, interpolating linearly
// between the two neighbouring pixel centres (V2).
// Coordinates: the ray position is re-anchored in fp64 every 32 lines, so
// the fp32 offsets stay < 34 pixels.
// MODE 0: out[r][a][w] = (W y)   (zero for bins outside [0, N_d))
// MODE 1: Alg. 1 step: out = v = W c; bank_k = bank_{k-1} + alpha v
// MODE 2: residual: out = p - W x  (global SIRT, eq. sirtit)
// ---------------------------------------------------------------------------
struct FpArgs {
    const float* img;       // padded images, row-driven source
    const float* imgT;      // transposed twin
    long long img_tstride;  // elements between tiles
    float* out;             // [tile][na][Wwin]
    long long out_tstride;
    const float* aux_in;    // MODE 1: bank_{k-1} (nullable); MODE 2: p
    float* aux_out;         // MODE 1: bank_k
    float alpha;
    // k_fp_roi2 band split (single ROIs): CTA z marches bands z, z + nsplit, ...
    // and writes raw ray sums to part [z][tile][na][Wwin]; k_fp_join sums them
    float* part; int nsplit;
    int a_lo, a_hi;         // k_fp_roi2: only angles [a_lo, a_hi) (a_hi <= 0: all; angle-split filter bank)
};

template <int MODE>
__global__ void __launch_bounds__(128) k_fp(Geo g, Tiles t, FpArgs f) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int a = blockIdx.y, r = blockIdx.z;
    if (w >= t.Wwin) return;
    const int na = g.na;
    const int d = __ldg(t.d0 + r * na + a) + w;
    float acc = 0.f;
    const AngF an = g.ang[a];
    if (d >= 0 && d < g.nd) {
        const TileT ti = t.tile[r];
        const int lv0 = an.col ? ti.vc0 : ti.vr0, lv1 = an.col ? ti.vc1 : ti.vr1;
        const int pv0 = an.col ? ti.vr0 : ti.vc0, pv1 = an.col ? ti.vr1 : ti.vc1;
        const double Lc = 0.5 * (t.T - 1);
        const double A = g.A64[a], B = g.B64[a];
        const double Pw = Lc + ((double)w - t.tauc[r * na + a]) * A;   // position at the centre line
        int la, lb;
        if (fabs(B) < 1e-12) {
            const bool hit = (Pw > pv0 - 1.0) && (Pw < (double)pv1);
            la = hit ? lv0 : 0;
            lb = hit ? lv1 : 0;
        } else {
            double l1 = Lc + ((pv0 - 1.0) - Pw) / B, l2 = Lc + ((double)pv1 - Pw) / B;
            if (l1 > l2) { const double tmp = l1; l1 = l2; l2 = tmp; }
            la = max(lv0, (int)floor(l1));
            lb = min(lv1, (int)ceil(l2) + 1);
        }
        const float* base = (an.col ? f.imgT : f.img) + (long long)r * f.img_tstride + PADL;
        const float Bf = an.B;
        for (int l = la; l < lb; l += 32) {
            const double p0 = Pw + ((double)l - Lc) * B;
            const double fb = floor(p0);
            const int ib = (int)fb;
            const float f0 = (float)(p0 - fb) - 0.5f;     // -0.5: magic rounding gives floor
            const int cnt = min(32, lb - l);
            const float* rowp = base + (long long)l * t.TP + ib;
            #pragma unroll 4
            for (int i = 0; i < cnt; ++i) {
                const float tt = fmaf((float)i, Bf, f0);
                const float rm = tt + MAGICF;
                const int m = __float_as_int(rm) - MAGICI;
                const float gg = tt - (rm - MAGICF);        // in [-0.5, 0.5]; frac = gg + 0.5
                const float* q = rowp + (long long)i * t.TP + m;
                const float v0 = __ldg(q), v1 = __ldg(q + 1);
                const float sum = v0 + v1, dif = v1 - v0;
                acc = fmaf(0.5f, sum, acc);
                acc = fmaf(gg, dif, acc);
            }
        }
        acc *= an.invc;
    }
    const long long o = (long long)r * f.out_tstride + (long long)a * t.Wwin + w;
    if (MODE == 0) {
        f.out[o] = acc;
    } else if (MODE == 1) {
        f.out[o] = acc;
        const float prev = f.aux_in ? f.aux_in[(long long)a * g.nd + w] : 0.f;
        f.aux_out[(long long)a * g.nd + w] = fmaf(f.alpha, acc, prev);
    } else {
        const float pv = (d >= 0 && d < g.nd) ? f.aux_in[(long long)a * g.nd + d] : 0.f;
        f.out[o] = pv - acc;
    }
}

constexpr int FP_APW_MAX = 2;          // angles per warp of the ROI forward projector (1 for small batches)
constexpr int FP_GA = 8 * FP_APW_MAX;  // angles per CTA at the default 2 per warp (they share each staged band)
constexpr int FP_U = 12;     // rays per lane: window width <= 32 * FP_U

// keeps ptxas from re-materialising a folded address bias (a mov it cannot see through)
__device__ __forceinline__ unsigned opaque_u32(unsigned x) {
    unsigned y;
    asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x));
    return y;
}

// ---------------------------------------------------------------------------
// k_fp_roi2: W_{L'} for a batch of ROI tiles, built for the sm_100 FP32
// datapath and the shared-memory crossbar:
//  * the band is staged as interpolation pairs (S[m], D[m]) = (v[m] + v[m+1],
//    v[m+1] - v[m]) (one 64-bit entry per pixel, built once per band and shared
//    by the CTA's 8 angles), so a Joseph step is one LDS.64 and two FP ops:
//    2 * lerp(v, pos) = S[m] + g D[m], g = 2 (pos - m) - 1;
//  * the position / index / fraction arithmetic runs on line pairs (FFMA2, FADD2);
//  * per band each warp visits only the rays that cross the band's valid
//    pixels (the range is computed in fp64), not the whole window.
// Staging: the next band's raw lines are prefetched into registers while the
// current band is marched, then transformed into the single (S, D) buffer.
// ---------------------------------------------------------------------------
constexpr int FP2_BL = 16;       // lines per band
constexpr int FP2_P = 272;       // (S, D) entries per staged line (>= T + PADL + PADR)
constexpr int FP2_CPT = (FP2_P / 4 + 15) / 16;  // float4 chunks per thread per band (16 threads per line)

template <bool CLAMP>
__device__ __forceinline__ float fp2_band_ray(unsigned rowbase_, float f0, float Bf, float lo, float hi) {
    const unsigned rowbase = __shfl_sync(0xffffffffu, rowbase_, threadIdx.x & 31);
    float acc = 0.f;
    #pragma unroll
    for (int i = 0; i < FP2_BL; i += 2) {
        float2 tt = make_float2(fmaf((float)i, Bf, f0), fmaf((float)(i + 1), Bf, f0));   // immediates
        if (CLAMP) {
            tt.x = fminf(fmaxf(tt.x, lo), hi);
            tt.y = fminf(fmaxf(tt.y, lo), hi);
        }
        const float2 rm = __fadd2_rn(tt, make_float2(MAGICF, MAGICF));           // round(tt) in the low bits
        const float2 k2 = __ffma2_rn(rm, make_float2(-2.f, -2.f), make_float2(2.f * MAGICF, 2.f * MAGICF));   // -2 round(tt)
        const float2 g = __ffma2_rn(tt, make_float2(2.f, 2.f), k2);             // 2 (tt - round(tt)) in [-1, 1]
        // (shift + add: LEA on the ALU pipe, not IMAD on the FMA pipe)
        const unsigned a0 = rowbase + ((unsigned)__float_as_int(rm.x) << 3);
        const unsigned a1 = rowbase + ((unsigned)__float_as_int(rm.y) << 3);
        float s0, d0, s1, d1;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(s0), "=f"(d0) : "r"(a0 + (unsigned)(i * FP2_P * 8)));
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(s1), "=f"(d1) : "r"(a1 + (unsigned)((i + 1) * FP2_P * 8)));
        acc = fmaf(g.x, d0, acc + s0);
        acc = fmaf(g.y, d1, acc + s1);
    }
    return acc;
}

template <int FP_APW>
__global__ void __launch_bounds__(256, 3) k_fp_roi2(Geo g, Tiles t, FpArgs f, const int* __restrict__ groups) {
    constexpr int FP_GA = 8 * FP_APW;
    extern __shared__ float4 smf4[];
    float2* sd = reinterpret_cast<float2*>(smf4);                 // [FP2_BL][FP2_P] (S, D), entry 0 = pixel -PADL
    float* sacc = reinterpret_cast<float*>(sd + FP2_BL * FP2_P);  // [FP_GA][32 * FP_U] per-ray accumulators
    const int r = blockIdx.y, grp = blockIdx.x;
    const int na = g.na, T = t.T, TP = t.TP, Wwin = t.Wwin;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int a0 = groups[grp * FP_GA];
    auto in_range = [&](int a) { return a >= 0 && (f.a_hi <= 0 || (a >= f.a_lo && a < f.a_hi)); };
    {   // a group with no angle in the requested range has nothing to do
        bool any = false;
        for (int q = 0; q < FP_GA; ++q) any |= in_range(groups[grp * FP_GA + q]);
        if (!any) return;
    }
    const int col = g.ang[a0].col;
    const TileT ti = t.tile[r];
    const int lv0 = col ? ti.vc0 : ti.vr0, lv1 = col ? ti.vc1 : ti.vr1;
    const int pv0 = col ? ti.vr0 : ti.vc0, pv1 = col ? ti.vr1 : ti.vc1;
    const double Lc = 0.5 * (T - 1);
    const float* src = (col ? f.imgT : f.img) + (long long)r * f.img_tstride;
    for (int e = threadIdx.x; e < FP_GA * 32 * FP_U; e += 256) sacc[e] = 0.f;

    // staging map (no division): thread = (line tid / 16, chunks c4 = tid % 16 + 16 u)
    const int q4 = TP / 4;                        // float4 chunks per raw line
    const int sline = threadIdx.x >> 4, sc0 = threadIdx.x & 15;
    float4 raw[FP2_CPT];
    float nxt[FP2_CPT];
    auto fetch = [&](int l0) {                    // raw lines l0.. of the band into registers
        const bool lok = l0 + sline < T;
        const float* rp0 = src + (long long)(l0 + sline) * TP;
        #pragma unroll
        for (int u = 0; u < FP2_CPT; ++u) {
            const int c4 = sc0 + 16 * u;
            raw[u] = make_float4(0.f, 0.f, 0.f, 0.f);
            nxt[u] = 0.f;
            if (lok && c4 < q4) {
                raw[u] = __ldg(reinterpret_cast<const float4*>(rp0 + c4 * 4));
                if (c4 + 1 < q4) nxt[u] = __ldg(rp0 + c4 * 4 + 4);
            }
        }
    };
    auto transform = [&]() {                      // registers -> (S, D) buffer
        #pragma unroll
        for (int u = 0; u < FP2_CPT; ++u) {
            const int c4 = sc0 + 16 * u;
            if (c4 < q4) {
                const float4 v = raw[u];
                float4* dst = reinterpret_cast<float4*>(sd + sline * FP2_P + c4 * 4);
                dst[0] = make_float4(v.x + v.y, v.y - v.x, v.y + v.z, v.z - v.y);
                dst[1] = make_float4(v.z + v.w, v.w - v.z, v.w + nxt[u], nxt[u] - v.w);
            }
        }
    };
    const int nsplit = f.nsplit > 1 ? f.nsplit : 1;
    const int lbeg = (lv0 / FP2_BL) * FP2_BL + (int)blockIdx.z * FP2_BL, lstep = nsplit * FP2_BL;
    if (lbeg < lv1) { fetch(lbeg); transform(); }
    __syncthreads();
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sd + PADL);     // entry of pixel 0
    for (int l0 = lbeg; l0 < lv1; l0 += lstep) {
        const bool more = l0 + lstep < lv1;
        if (more) fetch(l0 + lstep);
        #pragma unroll 1
        for (int j = 0; j < FP_APW; ++j) {
            const int a = groups[grp * FP_GA + warp * FP_APW + j];    // this warp's angle j (-1: idle)
            if (!in_range(a)) continue;
            const double A = g.A64[a], B = g.B64[a];
            const double tauc = t.tauc[r * na + a];
            const int d0 = __ldg(t.d0 + r * na + a);
            const float Bf = (float)B;
            float* acc = sacc + (warp * FP_APW + j) * (32 * FP_U);
            // rays with a detector bin: w in [wv0, wv1)
            const int wv0 = max(0, -d0), wv1 = min(Wwin, g.nd - d0);
            // rays meeting the valid pixels (pv0 - 1, pv1) on some line of the band
            const double P0 = Lc - tauc * A + ((double)l0 - Lc) * B;           // p(w, l0) = P0 + w A
            const double P1 = P0 + (double)(FP2_BL - 1) * B;                   // p(w, l0 + 15) = P1 + w A
            const double ia = 1.0 / A;
            const double e1 = (pv0 - 1.0 - P0) * ia, e2 = (pv1 - P0) * ia;
            const double e3 = (pv0 - 1.0 - P1) * ia, e4 = (pv1 - P1) * ia;
            const int wlo = max(wv0, (int)floor(fmin(fmin(e1, e2), fmin(e3, e4))) - 1);
            const int whi = min(wv1, (int)ceil(fmax(fmax(e1, e2), fmax(e3, e4))) + 2);
            const float Af = (float)A;
            const float Bl = (float)((FP2_BL - 1) * B);
            for (int wb = wlo; wb < whi; wb += 32) {
                const int w = wb + lane;
                const bool ray = w < whi;
                // position (pixel index) on line l0: fp64 anchor at the group's
                // middle ray, fp32 offset |(lane - 16) A| <= 23 px
                const double pc = P0 + (double)(wb + 16) * A;
                const double fbc = floor(pc);
                const float pos = fmaf((float)(lane - 16), Af, (float)(pc - fbc));
                const float fl = floorf(pos);
                const int ib = ray ? (int)fbc + (int)fl : 0;
                const float f0 = ray ? (pos - fl) - 0.5f : -0.5f;
                const float Bu = ray ? Bf : 0.f;
                const float pa = (float)ib + f0 + 0.5f, pe = pa + Bl;
                const bool safe = !ray || (fminf(pa, pe) >= -3.f && fmaxf(pa, pe) <= (float)T + 1.5f);
                const unsigned rowbase = sbase + 8u * (unsigned)(ib - MAGICI);
                float v;
                if (__all_sync(0xffffffffu, safe)) {
                    v = fp2_band_ray<false>(rowbase, f0, Bu, 0.f, 0.f);
                } else {
                    const float lo = (float)(-3 - ib) - 0.5f, hi = (float)(T + 2 - ib) - 0.5f;
                    v = fp2_band_ray<true>(rowbase, f0, Bu, lo, hi);
                }
                if (ray) acc[w] += v;
            }
        }
        __syncthreads();
        if (more) transform();
        __syncthreads();
    }
    for (int j = 0; j < FP_APW; ++j) {
        const int a = groups[grp * FP_GA + warp * FP_APW + j];
        if (!in_range(a)) continue;
        const int d0 = __ldg(t.d0 + r * na + a);
        const float* acc = sacc + (warp * FP_APW + j) * (32 * FP_U);
        if (nsplit > 1) {
            float* dst = f.part + (((long long)blockIdx.z * gridDim.y + r) * na + a) * Wwin;
            for (int w = lane; w < Wwin; w += 32) dst[w] = acc[w];
            continue;
        }
        const float sc = 0.5f * g.ang[a].invc;        // (S + g D) = 2 lerp
        for (int w = lane; w < Wwin; w += 32) {
            const int d = d0 + w;
            f.out[(long long)r * f.out_tstride + (long long)a * Wwin + w] = (d >= 0 && d < g.nd) ? acc[w] * sc : 0.f;
        }
    }
}

// the band-split partial ray sums of k_fp_roi2, summed in split order
__global__ void k_fp_join(Geo g, Tiles t, FpArgs f) {
    const int r = blockIdx.z, a = blockIdx.y, w = blockIdx.x * blockDim.x + threadIdx.x;
    const int na = g.na, Wwin = t.Wwin;
    if (w >= Wwin) return;
    float sum = 0.f;
    for (int z = 0; z < f.nsplit; ++z) sum += f.part[(((long long)z * gridDim.z + r) * na + a) * Wwin + w];
    const int d = __ldg(t.d0 + r * na + a) + w;
    f.out[(long long)r * f.out_tstride + (long long)a * Wwin + w] = (d >= 0 && d < g.nd) ? sum * (0.5f * g.ang[a].invc) : 0.f;
}

// ---------------------------------------------------------------------------
// Backprojection M_{L'} W^T (pixel driven, exact transpose of k_fp) with the
// fused solver epilogues.  CTA = (tile r, 64x64 sub-tile); thread = 2 x 8
// pixels (columns lane, lane + 32; 8 consecutive rows).  Per chunk of CA angles the CTA stages, for each angle, the
// SW-bin sub-window of the source sinogram that its sub-tile can reach, as
// tap pairs (v[m], v[m+1]) / c (one conflict-free LDS.64 per pixel-angle: a
// warp's 32 pixels of one row reach at most 33 consecutive bins).  The window
// is staged one warp per angle row (coalesced loads, pairs via shuffles).  The hat
// weights (V2) become hat(u / c) = sat(1 - |u| / c), computed on the
// fp32 pair datapath for two pixels at a time.
// Anchors: tau at the sub-tile centre in fp64, fp32 positions relative to the
// window centre (|.| <= 48 bins).
// NS = 0: no gather (y = 0 at k = 1), NS = 1: one sinogram.
// ---------------------------------------------------------------------------
constexpr int BP_CA = 32;   // angles per staged chunk
constexpr int BP_SUB = 64;  // default sub-tile side (pixels); 32 for small ROI batches

enum BpMode {
    BP_PLAIN_TILE = 0,   // out plain [tile][T][T]  (stage-wise parity, lt_backproject)
    BP_PLAIN_GLOBAL = 1, // out N x N at the tile's global position
    BP_BOX = 2,          // Alg. 2 with the box correction
    BP_TV = 3,           // Alg. 3 lines 4-5: v = x_s + x_L - alpha W^T W x_L; keep x_s
    BP_ALG1 = 4,         // Alg. 1: c <- c - alpha W^T v (padded image + twin)
    BP_GSIRT = 5,        // global box-SIRT: x <- clamp(x + alpha W^T r)
    BP_GTV = 6           // global FISTA-TV: v = x + alpha W^T r (plain N x N)
};

struct BpEpi {
    const int* blist;                                      // sub-tile list (nullable: all sub-tiles of the tile)
    const float* xsg; int xsg_pitch;                       // global x_s^k = W^T b_k image (BOX/TV)
    const float* xs_tile;                                  // nullable: per-tile x_s [tile][T][T] (p_tstride) instead
    float* out; long long out_tstride; int out_pitch;     // plain outputs
    float* y; float* yT; long long y_tstride;              // padded tile images (state)
    float* v; float* xs; long long p_tstride;              // plain [T][T] (TV)
    const float* discc; int use_disc;                      // disc gray value (device)
    float alpha, lo, hi; int last;
    // angle split for small batches: stage 1 = CTA z gathers angles
    // [z achunk, (z + 1) achunk) into part (CTA-local layout, no epilogue);
    // stage 2 = the same grid sums the nsa partials in order, then the epilogue
    float* part; int nsa, stage, achunk;
    int a_lo, a_hi;        // only angles [a_lo, a_hi) (a_hi <= 0: all; angle-split filter bank)
};

template <int NS, int MODE, int SUB = BP_SUB>
__global__ void __launch_bounds__(256) k_bp(Geo g, Tiles t, SinoView s1, SinoView s2, BpEpi e) {
    static_assert(NS == 0 || NS == 1, "one gathered sinogram at most");
    static_assert(SUB == 64 || SUB == 32, "64x64 (2 columns x 8 rows per thread) or 32x32 (1 x 4) sub-tiles");
    constexpr int COLS = SUB / 32;                // columns per thread (32 apart)
    constexpr int BP_PR = SUB * SUB / (256 * COLS);   // rows per thread
    constexpr int BP_SW = SUB == 64 ? 96 : 64;        // window bins (>= (SUB-1) sqrt2 + 4, a multiple of 32)
    __shared__ float2 sw[BP_CA][BP_SW];          // (v[m], v[m+1]) / c_a, m relative to the window centre
    __shared__ float4 sa[BP_CA];                 // (cos, sin, K' = 1 - 1/(2c), 1/c)
    __shared__ float sanch[BP_CA];

    const int r = blockIdx.y;
    const int T = t.T, na = g.na;
    const int nsx = (T + SUB - 1) / SUB;
    int sty, stx;
    if (e.blist && SUB == 32) {     // block list in 64x64 units: four 32x32 CTAs per listed block
        const int nsx64 = (T + 63) / 64;
        const int b = __ldg(e.blist + (blockIdx.x >> 2));
        const int by = b / nsx64, bx = b - by * nsx64;
        sty = 2 * by + ((blockIdx.x >> 1) & 1);
        stx = 2 * bx + (blockIdx.x & 1);
    } else {
        const int sub = e.blist ? __ldg(e.blist + blockIdx.x) : (int)blockIdx.x;
        sty = sub / nsx; stx = sub - sty * nsx;
    }
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const int pj0 = stx * SUB + lane;                  // columns pj0, pj0 + 32
    const int pi0 = sty * SUB + wq * BP_PR;            // rows pi0 .. pi0 + BP_PR - 1
    const double Lc = 0.5 * (T - 1);
    const double hs = 0.5 * (SUB - 1);
    const double dxc = stx * SUB + hs - Lc, dyc = sty * SUB + hs - Lc;
    const float dx = (float)lane - (float)hs, dy0 = (float)(wq * BP_PR) - (float)hs;

    // angles this CTA gathers (all, or one chunk of an angle-split stage 1; none in stage 2)
    const int alo = e.a_hi > 0 ? e.a_lo : 0, ahi = e.a_hi > 0 ? min(e.a_hi, na) : na;
    const int az0 = e.stage == 1 ? alo + (int)blockIdx.z * e.achunk : alo;
    const int az1 = e.stage == 1 ? min(ahi, az0 + e.achunk) : ahi;
    const bool gather = NS > 0 && e.stage != 2;
    float2 acc[COLS][BP_PR];                      // (left-tap, right-tap) partial sums per pixel
    #pragma unroll
    for (int h = 0; h < COLS; ++h)
        #pragma unroll
        for (int p = 0; p < BP_PR; ++p) acc[h][p] = make_float2(0.f, 0.f);
    // Staging, software-pipelined: the next chunk's window bins are loaded into
    // registers (warp = angle row, BP_CA / 8 rows per warp) while the current
    // chunk is gathered, then written as pairs between two barriers.
    constexpr int RPW = BP_CA / 8, NV = BP_SW / 32 + 1;
    float pv[RPW][NV];
    auto window_start = [&](int a, double& tc) {
        tc = t.tauc[r * na + a] + dxc * g.cs64[a] - dyc * g.sn64[a];
        return (int)floor(tc) - BP_SW / 2;                       // window bins sub0 .. sub0 + BP_SW
    };
    auto prefetch = [&](int a0n) {
        const int can = min(BP_CA, az1 - a0n);
        #pragma unroll
        for (int qq = 0; qq < RPW; ++qq) {
            const int q = wq + 8 * qq, a = a0n + q;
            double tc;
            const int sub0 = q < can ? window_start(a, tc) : 0;
            const int off = q < can ? (s1.use_d0 ? __ldg(t.d0 + r * na + a) : 0) + sub0 : 0;
            const float* rowp = s1.base + (long long)r * s1.tile_stride + (long long)(q < can ? a : 0) * s1.row_stride;
            #pragma unroll
            for (int u = 0; u < NV; ++u) {
                const int idx = off + lane + 32 * u;
                pv[qq][u] = (q < can && idx >= 0 && idx < s1.len && lane + 32 * u <= BP_SW) ? __ldg(rowp + idx) : 0.f;
            }
        }
    };
    if (gather && az0 < az1) prefetch(az0);
    for (int a0 = az0; a0 < (gather ? az1 : az0); a0 += BP_CA) {
        const int ca = min(BP_CA, az1 - a0);
        __syncthreads();
        #pragma unroll
        for (int qq = 0; qq < RPW; ++qq) {
            const int q = wq + 8 * qq;
            if (q >= ca) continue;
            const int a = a0 + q;
            double tc;
            const int sub0 = window_start(a, tc);
            const AngF an = g.ang[a];
            if (lane == 0) {
                sanch[q] = (float)(tc - (double)(sub0 + BP_SW / 2)) - 0.5f;
                sa[q] = make_float4(an.cs, an.sn, 1.f - 0.5f * an.invc, an.invc);
            }
            #pragma unroll
            for (int u = 0; u < BP_SW / 32; ++u) {
                float nx = __shfl_down_sync(0xffffffffu, pv[qq][u], 1);
                const float nx0 = __shfl_sync(0xffffffffu, pv[qq][u + 1], 0);
                if (lane == 31) nx = nx0;
                sw[q][lane + 32 * u] = make_float2(pv[qq][u] * an.invc, nx * an.invc);
            }
        }
        __syncthreads();
        if (a0 + BP_CA < az1) prefetch(a0 + BP_CA);
        // entry of bin m (relative to the window centre) at swbase + 8 (m + MAGIC bits)
        const unsigned swbase = opaque_u32((unsigned)__cvta_generic_to_shared(&sw[0][BP_SW / 2]) - 8u * (unsigned)MAGICI);
        #pragma unroll 1
        for (int q = 0; q < ca; ++q) {
            const float4 A4 = sa[q];
            const float t00 = fmaf(dx, A4.x, fmaf(-dy0, A4.y, sanch[q]));   // column pj0, row pi0
            const unsigned rowb = opaque_u32(swbase + (unsigned)(q * BP_SW * 8));
            #pragma unroll
            for (int h = 0; h < COLS; ++h) {
                const float t0 = h ? fmaf(32.f, A4.x, t00) : t00;
                #pragma unroll
                for (int p = 0; p < BP_PR; p += 2) {
                    // positions of pixels p, p+1 (one row apart): tt = t0 - p sin
                    const float2 tt = __ffma2_rn(make_float2(-(float)p, -(float)(p + 1)), make_float2(A4.y, A4.y),
                                                 make_float2(t0, t0));
                    const float2 rm = __fadd2_rn(tt, make_float2(MAGICF, MAGICF));
                    const float2 kk = __fadd2_rn(rm, make_float2(-MAGICF, -MAGICF));   // round(tt), exact
                    const float2 gg = __fadd2_rn(tt, make_float2(-kk.x, -kk.y));
                    unsigned ad0, ad1;
                    asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(ad0) : "r"(__float_as_int(rm.x)), "r"(rowb));
                    asm("mad.lo.u32 %0, %1, 8, %2;" : "=r"(ad1) : "r"(__float_as_int(rm.y)), "r"(rowb));
                    float2 b0, b1;
                    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(b0.x), "=f"(b0.y) : "r"(ad0));
                    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(b1.x), "=f"(b1.y) : "r"(ad1));
                    // hat weights of the left / right bin: sat(K' -/+ gg / c) (FFMA.SAT, full-rate scalar FP32;
                    // an FFMA2 + FMNMX form measured slower: FMNMX runs at half rate on the ALU pipe)
                    const float2 w0 = make_float2(__saturatef(fmaf(-gg.x, A4.w, A4.z)), __saturatef(fmaf(gg.x, A4.w, A4.z)));
                    const float2 w1 = make_float2(__saturatef(fmaf(-gg.y, A4.w, A4.z)), __saturatef(fmaf(gg.y, A4.w, A4.z)));
                    acc[h][p] = __ffma2_rn(w0, b0, acc[h][p]);
                    acc[h][p + 1] = __ffma2_rn(w1, b1, acc[h][p + 1]);
                }
            }
        }
    }
    const TileT ti = t.tile[r];
    const int n = g.n;
    #pragma unroll
    for (int h = 0; h < COLS; ++h) {
    const int pj = pj0 + 32 * h;
    float g1[BP_PR];
    #pragma unroll
    for (int p = 0; p < BP_PR; ++p) g1[p] = acc[h][p].x + acc[h][p].y;
    if (SUB == 32 && e.stage != 0) {   // angle split (32x32 launches only): partial sums per CTA-local pixel
        const long long ctas = (long long)gridDim.x * gridDim.y;
        const long long cta = (long long)blockIdx.y * gridDim.x + blockIdx.x;
        const int loc = (wq * BP_PR) * SUB + lane + 32 * h;
        if (e.stage == 1) {
            float* dst = e.part + ((long long)blockIdx.z * ctas + cta) * (SUB * SUB) + loc;
            #pragma unroll
            for (int p = 0; p < BP_PR; ++p) dst[p * SUB] = g1[p];
            continue;
        }
        #pragma unroll
        for (int p = 0; p < BP_PR; ++p) {
            float sum = 0.f;
            for (int z = 0; z < e.nsa; ++z) sum += e.part[((long long)z * ctas + cta) * (SUB * SUB) + loc + p * SUB];
            g1[p] = sum;
        }
    }

    // ---- epilogue ------------------------------------------------------------
    if (MODE == BP_BOX || MODE == BP_TV) {
        const float discc = e.use_disc ? *e.discc : 0.f;
        // loads of all four pixels first, then the stores
        float yv[BP_PR], xsv[BP_PR];
        bool valid[BP_PR];
        #pragma unroll
        for (int p = 0; p < BP_PR; ++p) {
            const int i = pi0 + p, j = pj;
            valid[p] = i < T && j < T && i >= ti.vr0 && i < ti.vr1 && j >= ti.vc0 && j < ti.vc1;
            yv[p] = 0.f; xsv[p] = 0.f;
            if (valid[p]) {
                float dval = 0.f;
                if (e.use_disc) {
                    const int gi = ti.row0 + i, gj = ti.col0 + j;
                    const int u = 2 * gj - n + 1, v = 2 * gi - n + 1;   // 2x, 2y of the pixel centre
                    dval = (u * u + v * v <= n * n) ? discc : 0.f;      // D: centred disc, diameter N
                }
                // x_s^k = M_{L'} W^T b_k + c D: the global backprojection, read at this pixel
                // (exterior-subtraction mode: the per-ROI alpha W_{L'}^T p~, no disc term)
                xsv[p] = e.xs_tile ? __ldg(e.xs_tile + (long long)r * e.p_tstride + (long long)i * T + j)
                                   : __ldg(e.xsg + (long long)(ti.row0 + i) * e.xsg_pitch + (ti.col0 + j)) + dval;
                yv[p] = e.y[(long long)r * e.y_tstride + (long long)i * t.TP + PADL + j];
            }
        }
        #pragma unroll
        for (int p = 0; p < BP_PR; ++p) {
            const int i = pi0 + p, j = pj;
            if (i >= T || j >= T) continue;
            float val = 0.f;
            if (valid[p]) {
                const float wts = NS >= 1 ? g1[p] : 0.f;                // (W_{L'}^T W_{L'} y)_j
                const float S = xsv[p] + yv[p] - e.alpha * wts;         // S(x^{k-1}) split
                if (MODE == BP_BOX) {
                    const float x = fminf(fmaxf(S, e.lo), e.hi);         // eq. sirtbox
                    val = e.last ? x : x - xsv[p];                       // y^k = clamp(S) - x_s^k
                } else {
                    val = S;
                }
            }
            if (MODE == BP_BOX) {
                e.y[(long long)r * e.y_tstride + (long long)i * t.TP + PADL + j] = val;
                e.yT[(long long)r * e.y_tstride + (long long)j * t.TP + PADL + i] = val;
            } else {
                const long long pl = (long long)r * e.p_tstride + (long long)i * T + j;
                e.v[pl] = val;
                e.xs[pl] = xsv[p];
            }
        }
        continue;
    }
    #pragma unroll
    for (int p = 0; p < BP_PR; ++p) {
        const int i = pi0 + p, j = pj;
        if (i >= T || j >= T) continue;
        const bool valid = i >= ti.vr0 && i < ti.vr1 && j >= ti.vc0 && j < ti.vc1;
        const long long pp = (long long)r * e.y_tstride + (long long)i * t.TP + PADL + j;
        const long long pt = (long long)r * e.y_tstride + (long long)j * t.TP + PADL + i;
        if (MODE == BP_PLAIN_TILE) {
            e.out[(long long)r * e.out_tstride + (long long)i * T + j] = valid ? g1[p] : 0.f;
        } else if (MODE == BP_PLAIN_GLOBAL) {
            if (valid) e.out[(long long)(ti.row0 + i) * e.out_pitch + (ti.col0 + j)] = g1[p];
        } else if (MODE == BP_ALG1) {
            const float c = valid ? e.y[pp] - e.alpha * g1[p] : 0.f;
            e.y[pp] = c;
            e.yT[pt] = c;
        } else if (MODE == BP_GSIRT) {
            const float x = valid ? fminf(fmaxf(e.y[pp] + e.alpha * g1[p], e.lo), e.hi) : 0.f;
            e.y[pp] = x;
            e.yT[pt] = x;
        } else if (MODE == BP_GTV) {
            if (valid) e.out[(long long)i * T + j] = e.y[pp] + e.alpha * g1[p];
        }
    }
    }
}

// ---------------------------------------------------------------------------
// FGP TV prox (Beck & Teboulle, named at P:L661-663; A13/A14),
// anisotropic, Neumann boundary on each tile's valid rectangle, fused with
// the FISTA update of Alg. 3 (lines 7-9, corrected per A12): arguments, the
// momentum table and the cluster (DSMEM / mbarrier) helpers of k_fgp2.
// ---------------------------------------------------------------------------

struct FgpArgs {
    const float* b; int b_pitch; long long b_tstride;   // input image(s)
    const TileT* tiles;                                 // valid rect per tile (nullable: whole H x W)
    int H, W;                                           // when tiles == nullptr
    float lam; int nfgp;
    const float* lams;                                  // nullable: per-tile lambda (lambda sweep, NEXT-1)
    float* out; int out_pitch; long long out_tstride;   // MODE 0
    // FISTA epilogue (MODE 1)
    const float* xs; float* xprev; long long p_tstride; int T;
    float* y; float* yT; long long y_tstride; int TP;
    float beta_o;
};

__device__ __forceinline__ float clip1(float v) { return fminf(1.f, fmaxf(-1.f, v)); }

// FGP momentum coefficients beta_k = (t_k - 1)/t_{k+1}, t_0 = 1,
// t_{k+1} = (1 + sqrt(1 + 4 t_k^2))/2 (Beck & Teboulle), computed on the host in fp64
constexpr int FGP_MAX_IT = 4096;
__constant__ float c_fgp_beta[FGP_MAX_IT];

// DSMEM push with transaction-count completion (sm_90+): a producer stores one
// float into a neighbour CTA's shared memory and the bytes complete on the
// neighbour's mbarrier; the consumer waits on its own mbarrier (acquire).
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ unsigned mapa(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f32(unsigned remote, float v, unsigned remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];"
                 ::"r"(remote), "f"(v), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(bar), "r"(parity) : "memory");
}

// ---------------------------------------------------------------------------
// k_fgp2: the FGP TV prox + FISTA epilogue, laid out for the sm_100
// paired FP32 datapath (FFMA2 / FADD2: two fp32 lanes per instruction).
//
// Warp w of CTA k owns FR full rows (rows (k*NW + w)*FR ...) of the tile, 256
// columns wide; lane l owns the 8 consecutive columns 8l..8l+7 of each row, as
// four column pairs.  Vertical neighbours are the same lane (aligned pairs ->
// paired instructions); the horizontal neighbour across a lane boundary comes
// by one warp shuffle per row and direction.  Rows crossing warps go through
// shared memory, rows crossing CTAs through DSMEM (st.async + mbarrier), as in
// k_fgp.  Per pixel-iteration ~8 issue slots (k_fgp: ~30).
//
// Masks (A13, Neumann boundary on the valid rectangle H_v x W_v):
// p exists for rows i < H_v - 1 (warp-uniform per row), q for columns
// j < W_v - 1 (per-column step register).  Pixels outside the valid rectangle
// carry finite garbage that no valid pixel reads.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2s(float s) { return make_float2(s, s); }
// row storage in shared memory: column 8l + c of a 256-wide row at
// (c >> 2) * 128 + 4l + (c & 3), so each lane moves its octet as two
// conflict-free 128-bit accesses
__device__ __forceinline__ void row_st(float* row, int lane, const float2 (&v)[4]) {
    reinterpret_cast<float4*>(row)[lane] = make_float4(v[0].x, v[0].y, v[1].x, v[1].y);
    reinterpret_cast<float4*>(row + 128)[lane] = make_float4(v[2].x, v[2].y, v[3].x, v[3].y);
}
__device__ __forceinline__ void row_ld(const float* row, int lane, float2 (&v)[4]) {
    const float4 a = reinterpret_cast<const float4*>(row)[lane];
    const float4 b = reinterpret_cast<const float4*>(row + 128)[lane];
    v[0] = make_float2(a.x, a.y); v[1] = make_float2(a.z, a.w);
    v[2] = make_float2(b.x, b.y); v[3] = make_float2(b.z, b.w);
}
// the same through 32-bit shared-window addresses (loop-invariant bases, no
// generic-to-shared conversion inside the iteration loop)
__device__ __forceinline__ void row_st_s(unsigned row, int lane, const float2 (&v)[4]) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(row + 16u * lane),
                 "f"(v[0].x), "f"(v[0].y), "f"(v[1].x), "f"(v[1].y) : "memory");
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(row + 512u + 16u * lane),
                 "f"(v[2].x), "f"(v[2].y), "f"(v[3].x), "f"(v[3].y) : "memory");
}
__device__ __forceinline__ void row_ld_s(unsigned row, int lane, float2 (&v)[4]) {
    float a0, a1, a2, a3, b0, b1, b2, b3;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3) : "r"(row + 16u * lane) : "memory");
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(b0), "=f"(b1), "=f"(b2), "=f"(b3) : "r"(row + 512u + 16u * lane) : "memory");
    v[0] = make_float2(a0, a1); v[1] = make_float2(a2, a3);
    v[2] = make_float2(b0, b1); v[3] = make_float2(b2, b3);
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_v4(unsigned remote, float4 v, unsigned remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                 ::"r"(remote), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void row_push(unsigned remote_row, int lane, const float2 (&v)[4], unsigned remote_bar) {
    st_async_v4(remote_row + 16u * lane, make_float4(v[0].x, v[0].y, v[1].x, v[1].y), remote_bar);
    st_async_v4(remote_row + 512u + 16u * lane, make_float4(v[2].x, v[2].y, v[3].x, v[3].y), remote_bar);
}

constexpr int FGP2_ROW = 256;     // columns per warp row (32 lanes x 8)
// producer / consumer named barriers between two neighbouring warps (ids 1..15; 0 = __syncthreads)
__device__ __forceinline__ void bar_arrive2(int id) { asm volatile("bar.arrive %0, 64;" ::"r"(id) : "memory"); }
__device__ __forceinline__ void bar_sync2(int id) { asm volatile("bar.sync %0, 64;" ::"r"(id) : "memory"); }
#ifndef FGP_NAMED_BARS
#define FGP_NAMED_BARS 0          // 1: named-barrier hand-over (measured slower: 1.35 vs 1.26 ms, C4 tiles)
#endif
#ifndef FGP_PAIR_SLEFT
#define FGP_PAIR_SLEFT 0           // 1: paired left-neighbour term (measured: no gain)
#endif
#ifndef FGP_HALO_PREFETCH
#define FGP_HALO_PREFETCH 0       // 1: halo rows loaded at the phase start (255 registers; measured slower: 1.59 ms)
#endif
#ifndef FGP_BAR_LATE
#define FGP_BAR_LATE 0            // 1: barrier before each halo row (measured slower: 1.30 vs 1.26 ms)
#endif
#ifndef FGP_HALO_LAST
#define FGP_HALO_LAST 1           // rows that read a halo are computed last in their phase
#endif
template <int V> struct Parity { __device__ __forceinline__ operator int() const { return V; } };

template <int FR, int NW>
struct Fgp2Smem {
    // halo rows, one slot per warp and parity, so every warp reads its halo
    // from the same place whichever warp or CTA wrote it:
    //   hr[par][j]: the r row above warp j (j = 0: pushed by the CTA above over
    //               DSMEM; j > 0: the last row of warp j - 1)
    //   hz[par][j]: the z row below warp j - 1 (j < NW: the first row of warp j;
    //               j = NW: pushed by the CTA below)
    // slots never written keep their initial value (r: the shifted zero 1/2, z: 0)
    static constexpr int bars = 0;                             // 4 x u64: r from above [2], z from below [2]
    static constexpr int hr = 8;                               // [2][NW + 1][256]
    static constexpr int hz = hr + 2 * (NW + 1) * FGP2_ROW;    // [2][NW + 1][256]
    static constexpr int hp = hz + 2 * (NW + 1) * FGP2_ROW;    // [NW][256] last p row (epilogue)
    static constexpr int bsm = hp + NW * FGP2_ROW;             // [NW][FR][256] b (BSM variant)
    static constexpr int total = bsm;
    static constexpr int total_bsm = bsm + NW * FR * FGP2_ROW;
    // MODE 1: [NW][FR][2][256] xprev and x_s rows, fetched with cp.async at
    // kernel start (they are inputs the FGP loop never touches) and read by the epilogue
    static constexpr int xin_floats = NW * FR * 2 * FGP2_ROW;
};
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}

// BSM: b (read once per iteration) lives in shared memory instead of registers,
// so the kernel fits 128 registers and two CTAs (two tiles) share an SM: one
// tile's halo latency is hidden behind the other tile's arithmetic.
template <int MODE, int FR, int NW, bool BSM>
__global__ void __launch_bounds__(NW * 32, (BSM && NW <= 8) ? 2 : 1) k_fgp2(FgpArgs A) {
    using SM = Fgp2Smem<FR, NW>;
    extern __shared__ __align__(16) float sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int K = (int)cl.num_blocks();
    const int kr = (int)cl.block_rank();
    const int tile = blockIdx.y;
    int vr0 = 0, vc0 = 0, Hv = A.H, Wv = A.W;
    if (A.tiles) {
        const TileT ti = A.tiles[tile];
        vr0 = ti.vr0; vc0 = ti.vc0; Hv = ti.vr1 - ti.vr0; Wv = ti.vc1 - ti.vc0;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i0 = (kr * NW + w) * FR;          // first row of this warp (valid-rectangle coordinates)
    const int x0 = lane * 8;                    // first column of this lane
    const bool has_up = kr > 0, has_dn = kr < K - 1;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + SM::bars);
    float* hp = sm + SM::hp;
    for (int e = threadIdx.x; e < SM::hp - SM::hr; e += NW * 32)
        sm[SM::hr + e] = SM::hr + e >= SM::hz ? 0.f : 0.5f;   // z halos start at 0, dual halos at the shifted zero 1/2
    if (threadIdx.x == 0) {
        for (int q_ = 0; q_ < 4; ++q_) mbar_init(smem_u32(bars + q_), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    float2 breg[BSM ? 1 : FR][4], r[FR][4], s[FR][4], p[FR][4], q[FR][4], z[FR][4];
    float* bs = sm + SM::bsm + (w * FR) * FGP2_ROW;          // this warp's b rows (BSM)
    auto bget = [&](int k, float2 (&v)[4]) {
        if constexpr (BSM) {
            row_ld(bs + k * FGP2_ROW, lane, v);
        } else {
            #pragma unroll
            for (int c2 = 0; c2 < 4; ++c2) v[c2] = breg[k][c2];
        }
    };
    const float* bsrc = A.b + (long long)tile * A.b_tstride + (long long)vr0 * A.b_pitch + vc0;
    // 16-byte loads when the rows are 16-byte aligned and the lane's 8 columns are valid
    const bool vec_b = ((reinterpret_cast<uintptr_t>(bsrc) | ((uintptr_t)A.b_pitch << 2)) & 15) == 0 && x0 + 8 <= Wv;
    #pragma unroll
    for (int k = 0; k < FR; ++k) {
        const int i = i0 + k;
        float2 bv[4];
        const float* brow = bsrc + (long long)i * A.b_pitch + x0;
        if (vec_b && i < Hv) {
            const float4 u0 = __ldg(reinterpret_cast<const float4*>(brow));
            const float4 u1 = __ldg(reinterpret_cast<const float4*>(brow) + 1);
            bv[0] = make_float2(u0.x, u0.y); bv[1] = make_float2(u0.z, u0.w);
            bv[2] = make_float2(u1.x, u1.y); bv[3] = make_float2(u1.z, u1.w);
        } else {
            #pragma unroll
            for (int c2 = 0; c2 < 4; ++c2) {
                const int x = x0 + 2 * c2;
                const bool rv = i < Hv;
                bv[c2] = make_float2((rv && x < Wv) ? __ldg(brow + 2 * c2) : 0.f,
                                     (rv && x + 1 < Wv) ? __ldg(brow + 2 * c2 + 1) : 0.f);
            }
        }
        #pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) {
            if constexpr (!BSM) breg[k][c2] = bv[c2];
            r[k][c2] = f2s(0.5f); s[k][c2] = f2s(0.5f); p[k][c2] = f2s(0.5f); q[k][c2] = f2s(0.5f);
        }
        if constexpr (BSM) row_st(bs + k * FGP2_ROW, lane, bv);
    }
    // FISTA state for the epilogue: asynchronous copies into shared memory now,
    // consumed after the FGP loop (each lane reads back only its own columns)
    float* xin = sm + (BSM ? SM::total_bsm : SM::total) + (w * FR) * 2 * FGP2_ROW;
    const bool vec_p = ((vc0 | A.T) & 3) == 0;
    if constexpr (MODE == 1) {
        #pragma unroll
        for (int k = 0; k < FR; ++k) {
            const int i = i0 + k;
            if (i >= Hv) continue;
            const long long prow = (long long)tile * A.p_tstride + (long long)(vr0 + i) * A.T + vc0 + x0;
            float* dx = xin + k * 2 * FGP2_ROW + x0;
            #pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (vec_p && x0 + 4 * h + 3 < Wv) {
                    cp_async16(dx + 4 * h, A.xprev + prow + 4 * h);
                    cp_async16(dx + FGP2_ROW + 4 * h, A.xs + prow + 4 * h);
                } else {
                    #pragma unroll
                    for (int c = 4 * h; c < 4 * h + 4; ++c)
                        if (x0 + c < Wv) {
                            cp_async4(dx + c, A.xprev + prow + c);
                            cp_async4(dx + FGP2_ROW + c, A.xs + prow + c);
                        }
                }
            }
        }
    }
    const float lam = A.lams ? __ldg(A.lams + tile) : A.lam;
    const float lam2 = 2.f * lam;               // L(p, q) = 2 L(p', q')
    const float gam = lam > 0.f ? 1.f / (16.f * lam) : 0.f;
    // q step per column (0 where q does not exist: j >= W_v - 1)
    float gq[8];
    #pragma unroll
    for (int c = 0; c < 8; ++c) gq[c] = (x0 + c < Wv - 1) ? gam : 0.f;
    float2 gq2[4];
    #pragma unroll
    for (int c2 = 0; c2 < 4; ++c2) gq2[c2] = make_float2(gq[2 * c2], gq[2 * c2 + 1]);
    cl.sync();
    const unsigned up_rank = has_up ? kr - 1 : kr, dn_rank = has_dn ? kr + 1 : kr;
    constexpr unsigned RB = FGP2_ROW * 4u;             // bytes per staged row
    constexpr unsigned PS = (NW + 1) * RB;             // bytes per parity of hr / hz
    const unsigned s_hr = smem_u32(sm + SM::hr), s_hz = smem_u32(sm + SM::hz);
    // this warp's halo slots: r from above, z from below (read); r / z it publishes (written)
    const unsigned up_slot = s_hr + w * RB, dn_slot = s_hz + (w + 1) * RB;
    const unsigned rem_rx_r = mapa(s_hr, dn_rank);                 // my last warp's r row -> slot 0 of the CTA below
    const unsigned rem_bar_r = mapa(smem_u32(bars + 0), dn_rank);
    const unsigned rem_rx_z = mapa(s_hz + NW * RB, up_rank);       // my first warp's z row -> slot NW of the CTA above
    const unsigned rem_bar_z = mapa(smem_u32(bars + 2), up_rank);
    const unsigned my_r_slot = s_hr + (w + 1) * RB, my_z_slot = s_hz + w * RB;
    constexpr unsigned row_bytes = FGP2_ROW * 4;
    const int nit = lam > 0.f ? A.nfgp : 0;
    const unsigned bar0 = smem_u32(bars);
    const float2 nl2 = f2s(-lam2);
    // p step per row of this warp (0 where p does not exist: i >= H_v - 1)
    float gp[FR];
    #pragma unroll
    for (int k = 0; k < FR; ++k) gp[k] = (i0 + k < Hv - 1) ? gam : 0.f;

    // Halo hand-over between the warps of the CTA: NBAR (NW <= 8, with the halo
    // rows computed last): producer / consumer named barriers per warp pair,
    // so a warp waits only for the neighbour whose row it reads, and only
    // before that row; otherwise a CTA barrier after each phase.  Parity cb is
    // compile-time, so every halo address is loop invariant.
    constexpr bool NBAR = FGP_HALO_LAST && NW <= 8 && FGP_NAMED_BARS;
    // BAR_LATE: the CTA barrier sits right before each phase's halo row instead
    // of at the phase end (same count; the segments between barriers balance)
    constexpr bool BAR_LATE = FGP_HALO_LAST && !NBAR && FGP_BAR_LATE;
    auto fgp_iter = [&](int it, auto cbv) {
        const int cb = cbv, pb = cb ^ 1;
        if (lane == 0) {   // the consuming warp arms its DSMEM receive buffers
            if (w == NW - 1 && has_dn) mbar_expect_tx(bar0 + 16 + 8 * cb, row_bytes);   // z row of it, from below
            if (w == 0 && has_up) mbar_expect_tx(bar0 + 8 * cb, row_bytes);             // r row of it, from above
        }
        // ---- phase A: z = b - lam2 L(r, s); row 0 first (its upper neighbour
        // may come from another warp or CTA) and publish it at once
        // halo rows published before the last barrier: loaded now, used last
        // (the DSMEM rows wait on their mbarrier first, at the halo row)
        constexpr bool PRE = FGP_HALO_LAST && !NBAR && !BAR_LATE && FGP_HALO_PREFETCH;
        const bool up_local = !(w == 0 && has_up);
        float2 rpre[4];
        if constexpr (PRE) { if (up_local) row_ld_s(up_slot + pb * PS, lane, rpre); }
        #pragma unroll
        for (int kk = 0; kk < FR; ++kk) {
            const int k = FGP_HALO_LAST ? (kk + 1) % FR : kk;     // halo row 0 last: 1, ..., FR-1, 0
            float2 rup[4];
            if (k > 0) {
                #pragma unroll
                for (int c2 = 0; c2 < 4; ++c2) rup[c2] = r[k - 1][c2];
            } else {
                if constexpr (BAR_LATE) __syncthreads();   // every warp has published its r row of it - 1
                // slot of parity pb: written in iteration it - 1 (still 1/2 at it = 0)
                if (PRE && up_local) {
                    #pragma unroll
                    for (int c2 = 0; c2 < 4; ++c2) rup[c2] = rpre[c2];
                } else {
                    if (w == 0 && has_up && it > 0) mbar_wait(bar0 + 8 * pb, ((it - 1) >> 1) & 1);
                    if constexpr (NBAR) { if (w > 0 && it > 0) bar_sync2(NW + w - 1); }   // r row of warp w - 1
                    row_ld_s(up_slot + pb * PS, lane, rup);
                }
            }
            float sl = __shfl_up_sync(0xffffffffu, s[k][3].y, 1);
            if (lane == 0) sl = 0.5f;
            // z = b - lam2 (r - rup) - lam2 s + lam2 s_left
            float2 t[4], bk[4];
            bget(k, bk);
            #pragma unroll
            for (int c2 = 0; c2 < 4; ++c2) {
                t[c2] = f2fma(nl2, f2sub(r[k][c2], rup[c2]), bk[c2]);
                t[c2] = f2fma(nl2, s[k][c2], t[c2]);
            }
#if FGP_PAIR_SLEFT
            // the left neighbours (s_{j-1}, s_j) as an aligned register pair (two
            // moves) so the last term is one FFMA2 instead of two scalar FFMAs
            {
                const float2 l2 = f2s(lam2);
                z[k][0] = f2fma(l2, make_float2(sl, s[k][0].x), t[0]);
                #pragma unroll
                for (int c2 = 1; c2 < 4; ++c2) z[k][c2] = f2fma(l2, make_float2(s[k][c2 - 1].y, s[k][c2].x), t[c2]);
            }
#else
            z[k][0].x = fmaf(lam2, sl, t[0].x);
            z[k][0].y = fmaf(lam2, s[k][0].x, t[0].y);
            #pragma unroll
            for (int c2 = 1; c2 < 4; ++c2) {
                z[k][c2].x = fmaf(lam2, s[k][c2 - 1].y, t[c2].x);
                z[k][c2].y = fmaf(lam2, s[k][c2].x, t[c2].y);
            }
#endif
            if (k == 0) {
                if (w == 0 && has_up) row_push(rem_rx_z + cb * PS, lane, z[0], rem_bar_z + cb * 8);
                if (w > 0) row_st_s(my_z_slot + cb * PS, lane, z[0]);
                if constexpr (NBAR) { if (w > 0) bar_arrive2(w); }           // z row -> warp w - 1
            }
        }
        if constexpr (!NBAR && !BAR_LATE) __syncthreads();
        // ---- phase B: dual ascent, projection on [0, 1] (shifted), FGP momentum;
        // last row first and publish it
        const float beta = c_fgp_beta[it];
        const float2 beta2 = f2s(beta);
        const bool dn_local = !(w == NW - 1 && has_dn);
        float2 zpre[4];
        if constexpr (PRE) { if (dn_local) row_ld_s(dn_slot + cb * PS, lane, zpre); }
        #pragma unroll
        for (int kk = 0; kk < FR; ++kk) {
            const int k = FGP_HALO_LAST ? kk : (kk + FR - 1) % FR;   // halo row FR-1 last: 0, ..., FR-1
            float2 zb[4];
            if (k < FR - 1) {
                #pragma unroll
                for (int c2 = 0; c2 < 4; ++c2) zb[c2] = z[k + 1][c2];
            } else {
                if constexpr (BAR_LATE) __syncthreads();   // every warp has published its z row of it
                if (PRE && dn_local) {
                    #pragma unroll
                    for (int c2 = 0; c2 < 4; ++c2) zb[c2] = zpre[c2];
                } else {
                    if (w == NW - 1 && has_dn) mbar_wait(bar0 + 16 + 8 * cb, (it >> 1) & 1);
                    if constexpr (NBAR) { if (w < NW - 1) bar_sync2(w + 1); }     // z row of warp w + 1
                    row_ld_s(dn_slot + cb * PS, lane, zb);
                }
            }
            const float zr = __shfl_down_sync(0xffffffffu, z[k][0].x, 1);   // lane 31: masked by gq
            const float gpk = gp[k];
            const float2 gp2 = f2s(gpk);
            #pragma unroll
            for (int c2 = 0; c2 < 4; ++c2) {
                // p' = sat(r + g (z - z_below)), q' = sat(s + g (z - z_right))
                const float2 tp = f2fma(gp2, z[k][c2], r[k][c2]);
                const float2 tq = f2fma(gq2[c2], z[k][c2], s[k][c2]);
                const float zrx = z[k][c2].y;
                const float zry = c2 < 3 ? z[k][c2 + 1].x : zr;
                float2 pn, qn;
                pn.x = __saturatef(fmaf(-gpk, zb[c2].x, tp.x));
                pn.y = __saturatef(fmaf(-gpk, zb[c2].y, tp.y));
                qn.x = __saturatef(fmaf(-gq[2 * c2], zrx, tq.x));
                qn.y = __saturatef(fmaf(-gq[2 * c2 + 1], zry, tq.y));
                r[k][c2] = f2fma(beta2, f2sub(pn, p[k][c2]), pn);
                s[k][c2] = f2fma(beta2, f2sub(qn, q[k][c2]), qn);
                p[k][c2] = pn;
                q[k][c2] = qn;
            }
            if (k == FR - 1) {
                if (w == NW - 1 && has_dn) row_push(rem_rx_r + cb * PS, lane, r[FR - 1], rem_bar_r + cb * 8);
                if (w < NW - 1) row_st_s(my_r_slot + cb * PS, lane, r[FR - 1]);
                if constexpr (NBAR) { if (w < NW - 1 && it + 1 < nit) bar_arrive2(NW + w); }   // r row -> warp w + 1
            }
        }
        if constexpr (!NBAR && !BAR_LATE) __syncthreads();
    };
    {
        int it = 0;
        for (; it + 1 < nit; it += 2) {
            fgp_iter(it, Parity<0>{});
            fgp_iter(it + 1, Parity<1>{});
        }
        if (it < nit) fgp_iter(it, Parity<0>{});
    }

    // ---- x = b - lam2 L(p', q'), then the epilogue
    row_st(hp + w * FGP2_ROW, lane, p[FR - 1]);
    cl.sync();
    float2 pup0[4];
    if (w > 0) row_ld(hp + (w - 1) * FGP2_ROW, lane, pup0);
    else if (has_up) row_ld(cl.map_shared_rank(hp, kr - 1) + (NW - 1) * FGP2_ROW, lane, pup0);
    else {
        #pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) pup0[c2] = f2s(0.5f);
    }
    // the neighbour's halo row has been read: arrive now, wait at exit (keeps
    // shared memory alive until every neighbour has read its halo)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if constexpr (MODE == 1) cp_async_commit_wait_all();
    const bool vec_y = (vc0 & 3) == 0;                  // y rows: PADL + vc0 + x0, TP % 4 == 0
    const bool vec_yT = FR == 4 && (vr0 & 3) == 0;      // yT columns: PADL + vr0 + i0 + k
    float xall[FR][8];
    #pragma unroll
    for (int k = 0; k < FR; ++k) {
        const int i = i0 + k;
        float ql = __shfl_up_sync(0xffffffffu, q[k][3].y, 1);
        if (lane == 0) ql = 0.5f;
        float2 bk[4];
        bget(k, bk);
        #pragma unroll
        for (int c2 = 0; c2 < 4; ++c2) {
            const float2 pu = k > 0 ? p[k - 1][c2] : pup0[c2];
            const float qlx = c2 > 0 ? q[k][c2 - 1].y : ql;
            xall[k][2 * c2] = bk[c2].x - lam2 * (p[k][c2].x + q[k][c2].x - pu.x - qlx);
            xall[k][2 * c2 + 1] = bk[c2].y - lam2 * (p[k][c2].y + q[k][c2].y - pu.y - q[k][c2].x);
        }
        if (i >= Hv) continue;
        if constexpr (MODE == 0) {
            #pragma unroll
            for (int c = 0; c < 8; ++c)
                if (x0 + c < Wv) A.out[(long long)tile * A.out_tstride + (long long)i * A.out_pitch + x0 + c] = xall[k][c];
        } else {
            const int ti_ = vr0 + i;
            const long long prow = (long long)tile * A.p_tstride + (long long)ti_ * A.T + vc0 + x0;
            float* yrow = A.y + (long long)tile * A.y_tstride + (long long)ti_ * A.TP + PADL + vc0 + x0;
            const float* sx = xin + k * 2 * FGP2_ROW + x0;
            float xp[8], xsv[8];
            *reinterpret_cast<float4*>(xp) = *reinterpret_cast<const float4*>(sx);
            *reinterpret_cast<float4*>(xp + 4) = *reinterpret_cast<const float4*>(sx + 4);
            *reinterpret_cast<float4*>(xsv) = *reinterpret_cast<const float4*>(sx + FGP2_ROW);
            *reinterpret_cast<float4*>(xsv + 4) = *reinterpret_cast<const float4*>(sx + FGP2_ROW + 4);
            float yv[8];
            #pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float x = xall[k][c];
                const float rr = x + A.beta_o * (x - xp[c]);          // FISTA extrapolation (A12)
                yv[c] = rr - xsv[c];                                  // x_L^k = r - x_s^k
            }
            #pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (x0 + 4 * h + 3 < Wv && vec_p) {
                    *reinterpret_cast<float4*>(A.xprev + prow + 4 * h) =
                        make_float4(xall[k][4 * h], xall[k][4 * h + 1], xall[k][4 * h + 2], xall[k][4 * h + 3]);
                } else {
                    #pragma unroll
                    for (int c = 4 * h; c < 4 * h + 4; ++c)
                        if (x0 + c < Wv) A.xprev[prow + c] = xall[k][c];
                }
                if (x0 + 4 * h + 3 < Wv && vec_y) {
                    *reinterpret_cast<float4*>(yrow + 4 * h) = make_float4(yv[4 * h], yv[4 * h + 1], yv[4 * h + 2], yv[4 * h + 3]);
                } else {
                    #pragma unroll
                    for (int c = 4 * h; c < 4 * h + 4; ++c)
                        if (x0 + c < Wv) yrow[c] = yv[c];
                }
            }
            if (vec_yT) {
                // the warp's FR = 4 rows are consecutive: the transposed copy of
                // column c is one 16-byte store per lane, written after the last row
                #pragma unroll
                for (int c = 0; c < 8; ++c) xall[k][c] = yv[c];
            } else {
                float* ycol = A.yT + (long long)tile * A.y_tstride + (long long)(vc0 + x0) * A.TP + PADL + ti_;
                #pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (x0 + c < Wv) ycol[(long long)c * A.TP] = yv[c];
            }
        }
    }
    if constexpr (MODE == 1) {
        if (vec_yT && i0 < Hv) {
            float* ycol = A.yT + (long long)tile * A.y_tstride + (long long)(vc0 + x0) * A.TP + PADL + vr0 + i0;
            if (i0 + 3 < Hv) {
                #pragma unroll
                for (int c = 0; c < 8; ++c)
                    if (x0 + c < Wv)
                        *reinterpret_cast<float4*>(ycol + (long long)c * A.TP) =
                            make_float4(xall[0][c], xall[FR > 1 ? 1 : 0][c], xall[FR > 2 ? 2 : 0][c], xall[FR > 3 ? 3 : 0][c]);
            } else {
                #pragma unroll
                for (int c = 0; c < 8; ++c)
                    #pragma unroll
                    for (int k = 0; k < FR; ++k)
                        if (x0 + c < Wv && i0 + k < Hv) ycol[(long long)c * A.TP + k] = xall[k][c];
            }
        }
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");

}

// ---------------------------------------------------------------------------
// Convolution cache b_k = C_{u_k} p_c, direct form
//   b_k(a,d) = sum_j u_k(a,j) p_c(a, d - j + d_c)
// CTA = (angle a, 8 consecutive k, 256 consecutive d); thread = one d, 8 k.
// Products in fp32, each 512-tap chunk summed in fp32 and added into an fp64
// accumulator (bounds the fp32 error of the N_d-long sums).
// ---------------------------------------------------------------------------
constexpr int CV_KB = 8, CV_DB = 256, CV_JB = 512;

__global__ void __launch_bounds__(256) k_conv(int na, int nd, int nk, const float* __restrict__ bank,
                                              const float* __restrict__ pc, float* __restrict__ outb) {
    __shared__ float4 su[CV_JB][CV_KB / 4];
    __shared__ float sp[CV_DB + CV_JB];
    const int a = blockIdx.y;
    const int k0 = blockIdx.z * CV_KB;
    const int d0 = blockIdx.x * CV_DB;
    const int dcen = (nd - 1) / 2;
    const int d = d0 + threadIdx.x;
    double accd[CV_KB];
    #pragma unroll
    for (int q = 0; q < CV_KB; ++q) accd[q] = 0.0;
    for (int j0 = 0; j0 < nd; j0 += CV_JB) {
        __syncthreads();
        for (int el = threadIdx.x; el < CV_JB * CV_KB; el += blockDim.x) {
            const int jj = el % CV_JB, q = el / CV_JB;
            const int j = j0 + jj, k = k0 + q;
            float v = 0.f;
            if (j < nd && k < nk) v = bank[((long long)k * na + a) * nd + j];
            reinterpret_cast<float*>(&su[jj][0])[q] = v;
        }
        // p index m = d - j + dcen, for d in [d0, d0+DB), j in [j0, j0+JB):
        // m in (d0 - j0 - JB + dcen, d0 - j0 + DB - 1 + dcen]; store sp[x] = p[mbase + x]
        const int mbase = d0 - j0 - CV_JB + 1 + dcen;
        for (int x = threadIdx.x; x < CV_DB + CV_JB; x += blockDim.x) {
            const int m = mbase + x;
            sp[x] = (m >= 0 && m < nd) ? pc[(long long)a * nd + m] : 0.f;
        }
        __syncthreads();
        float acc[CV_KB];
        #pragma unroll
        for (int q = 0; q < CV_KB; ++q) acc[q] = 0.f;
        const int jn = min(CV_JB, nd - j0);
        // m - mbase = (d - j + dcen) - mbase = threadIdx.x + (JB - 1) - jj
        const float* pp = sp + threadIdx.x + CV_JB - 1;
        #pragma unroll 4
        for (int jj = 0; jj < jn; ++jj) {
            const float pv = pp[-jj];
            const float4 u0 = su[jj][0], u1 = su[jj][1];
            acc[0] = fmaf(u0.x, pv, acc[0]); acc[1] = fmaf(u0.y, pv, acc[1]);
            acc[2] = fmaf(u0.z, pv, acc[2]); acc[3] = fmaf(u0.w, pv, acc[3]);
            acc[4] = fmaf(u1.x, pv, acc[4]); acc[5] = fmaf(u1.y, pv, acc[5]);
            acc[6] = fmaf(u1.z, pv, acc[6]); acc[7] = fmaf(u1.w, pv, acc[7]);
        }
        #pragma unroll
        for (int q = 0; q < CV_KB; ++q) accd[q] += (double)acc[q];
    }
    if (d < nd) {
        #pragma unroll
        for (int q = 0; q < CV_KB; ++q)
            if (k0 + q < nk) outb[((long long)(k0 + q) * na + a) * nd + d] = (float)accd[q];
    }
}

// ---------------------------------------------------------------------------
// Convolution cache by FFT (same b_k as k_conv; the linear convolution of
// rows zero-padded to L >= 2 N_d - 1 is the circular one of length L):
//   k_padrows:  dst[r][0..L) = (src[r][0..nd), 0, ...)
//   k_specmul:  S[kk][a][f] = U[k0+kk][a][f] * P[a][f]  (U already scaled by 1/L)
//   k_croprows: b[k0+kk][a][d] = c[kk][a][d + d_c], d < N_d
// ---------------------------------------------------------------------------
__global__ void k_fill(long long n, float v, float* __restrict__ x) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) x[e] = v;
}

__global__ void k_scale(long long n, float s, float* __restrict__ x) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) x[e] *= s;
}

__global__ void k_padrows(int nrows, int nd, int L, const float* __restrict__ src, float* __restrict__ dst) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (c >= L || r >= nrows) return;
    dst[(long long)r * L + c] = c < nd ? src[(long long)r * nd + c] : 0.f;
}

__global__ void k_specmul(long long nk_rows_f, int na, int F, const float2* __restrict__ U, const float2* __restrict__ P,
                          float2* __restrict__ S) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= nk_rows_f) return;
    const long long row = e / F;
    const int f = (int)(e - row * F);
    const int a = (int)(row % na);
    const float2 u = U[e], q = P[(long long)a * F + f];
    S[e] = make_float2(fmaf(u.x, q.x, -u.y * q.y), fmaf(u.x, q.y, u.y * q.x));
}

__global__ void k_croprows(int nrows, int nd, int L, int dc, const float* __restrict__ c, float* __restrict__ b) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x, r = blockIdx.y;
    if (d >= nd || r >= nrows) return;
    b[(long long)r * nd + d] = c[(long long)r * L + d + dc];
}

// ---------------------------------------------------------------------------
// Small kernels: disc raster, zero-frequency sums, disc gray value, p_c,
// image (un)packing, crop, extended-ROI export, stitch.
// ---------------------------------------------------------------------------
// padded image + twin from a plain N x N image (src nullable: disc raster D, P:L726-727;
// disc = 2: the all-ones image)
__global__ void k_pack(int n, int TP, const float* __restrict__ src, int disc, float* __restrict__ img,
                       float* __restrict__ imgT) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    float v;
    if (disc == 2) {
        v = 1.f;
    } else if (disc) {
        const int u = 2 * j - n + 1, w = 2 * i - n + 1;
        v = (u * u + w * w <= n * n) ? 1.f : 0.f;
    } else {
        v = src[(long long)i * n + j];
    }
    img[(long long)i * TP + PADL + j] = v;
    imgT[(long long)j * TP + PADL + i] = v;
}

// one block per angle: fixed-order fp64 reduction of a sinogram row
__global__ void k_rowsum(int nd, const float* __restrict__ s, double* __restrict__ out) {
    __shared__ double red[256];
    const int a = blockIdx.x;
    double acc = 0.0;
    for (int d = threadIdx.x; d < nd; d += blockDim.x) acc += (double)s[(long long)a * nd + d];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st) red[threadIdx.x] += red[threadIdx.x + st];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[a] = red[0];
}

// c = sum_a P_a D_a / sum_a D_a^2  (least squares on the zero-frequency components)
__global__ void k_discc(int na, const double* __restrict__ P, const double* __restrict__ D,
                        double* __restrict__ c64, float* __restrict__ c32, float* __restrict__ cuser, int* err) {
    __shared__ double rn[256], rd[256];
    double num = 0.0, den = 0.0;
    for (int a = threadIdx.x; a < na; a += blockDim.x) { num += P[a] * D[a]; den += D[a] * D[a]; }
    rn[threadIdx.x] = num; rd[threadIdx.x] = den;
    __syncthreads();
    for (int st = 128; st > 0; st >>= 1) {
        if (threadIdx.x < st) { rn[threadIdx.x] += rn[threadIdx.x + st]; rd[threadIdx.x] += rd[threadIdx.x + st]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const double c = rd[0] > 0.0 ? rn[0] / rd[0] : 0.0;
        *c64 = c; *c32 = (float)c;
        if (cuser) *cuser = (float)c;
        if (!(rd[0] > 0.0)) *err = 1;
    }
}

__global__ void k_pc(long long ne, const float* __restrict__ p, const float* __restrict__ wd,
                     const double* __restrict__ c64, float* __restrict__ pc) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < ne) pc[e] = (float)((double)p[e] - *c64 * (double)wd[e]);
}

// core crop: cores[r][i][j] = src[r][(m+i)][(m+j)] (src padded or plain)
__global__ void k_crop(int side, int m, const float* __restrict__ src, long long s_tstride, int s_pitch,
                       int s_off, float* __restrict__ cores) {
    const int r = blockIdx.z;
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= side || j >= side) return;
    cores[((long long)r * side + i) * side + j] =
        src[(long long)r * s_tstride + (long long)(m + i) * s_pitch + s_off + m + j];
}

// extended export: ext[r][i][j] = src[r][vr0+i][vc0+j] for the valid rect, 0 elsewhere
__global__ void k_ext(int E, const TileT* tiles, const float* __restrict__ src, long long s_tstride,
                      int s_pitch, int s_off, float* __restrict__ ext) {
    const int r = blockIdx.z;
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= E || j >= E) return;
    const TileT ti = tiles[r];
    float v = 0.f;
    if (i < ti.vr1 - ti.vr0 && j < ti.vc1 - ti.vc0)
        v = src[(long long)r * s_tstride + (long long)(ti.vr0 + i) * s_pitch + s_off + ti.vc0 + j];
    ext[((long long)r * E + i) * E + j] = v;
}

// ROI extraction for lt_project(roi): padded tile + twin of M_{L'} x
__global__ void k_extract(int n, int T, int TP, TileT ti, const float* __restrict__ img,
                          float* __restrict__ t, float* __restrict__ tT) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= T || j >= T) return;
    const bool valid = i >= ti.vr0 && i < ti.vr1 && j >= ti.vc0 && j < ti.vc1;
    const float v = valid ? img[(long long)(ti.row0 + i) * n + ti.col0 + j] : 0.f;
    t[(long long)i * TP + PADL + j] = v;
    tT[(long long)j * TP + PADL + i] = v;
}

// ---------------------------------------------------------------------------
// Quality metrics inside the ROI (DESIGN.md
// §11 reading M1): per image pair (x, g) of h x w,
//   MSE  = mean (x - g)^2,
//   SSIM = mean over the valid positions (window inside the image) of
//          (2 mu_x mu_g + C1)(2 s_xg + C2) / ((mu_x^2 + mu_g^2 + C1)(s_x^2 + s_g^2 + C2))
//   (Wang et al. 2004: 11 x 11 Gaussian window, sigma 1.5, normalised weights;
//   C1 = (0.01 L)^2, C2 = (0.03 L)^2, L = max g - min g unless given).
// One CTA per image; fp64 accumulation of the means.
// ---------------------------------------------------------------------------
__constant__ float c_ssim_w[121];

__global__ void __launch_bounds__(256) k_metrics(int h, int w, const float* __restrict__ x, const float* __restrict__ g,
                                                 float range, double* __restrict__ mse, double* __restrict__ ssim) {
    __shared__ double red[256];
    __shared__ float smin[256], smax[256];
    const int img = blockIdx.x;
    const float* xi = x + (long long)img * h * w;
    const float* gi = g + (long long)img * h * w;
    const int n = h * w;
    double se = 0.0;
    float lo = INFINITY, hi = -INFINITY;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const double d = (double)xi[e] - (double)gi[e];
        se += d * d;
        lo = fminf(lo, gi[e]); hi = fmaxf(hi, gi[e]);
    }
    red[threadIdx.x] = se; smin[threadIdx.x] = lo; smax[threadIdx.x] = hi;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            red[threadIdx.x] += red[threadIdx.x + s];
            smin[threadIdx.x] = fminf(smin[threadIdx.x], smin[threadIdx.x + s]);
            smax[threadIdx.x] = fmaxf(smax[threadIdx.x], smax[threadIdx.x + s]);
        }
        __syncthreads();
    }
    const double L = range > 0.f ? (double)range : (double)smax[0] - (double)smin[0];
    const double C1 = (0.01 * L) * (0.01 * L), C2 = (0.03 * L) * (0.03 * L);
    if (threadIdx.x == 0) mse[img] = red[0] / n;
    __syncthreads();
    const int vh = h - 10, vw = w - 10;
    double acc = 0.0;
    for (int e = threadIdx.x; e < vh * vw; e += blockDim.x) {
        const int i = e / vw, j = e - i * vw;
        double mx = 0.0, mg = 0.0, xx = 0.0, gg = 0.0, xg = 0.0;
        for (int a = 0; a < 11; ++a)
            for (int b = 0; b < 11; ++b) {
                const double wt = c_ssim_w[a * 11 + b];
                const double xv = xi[(i + a) * w + j + b], gv = gi[(i + a) * w + j + b];
                mx += wt * xv; mg += wt * gv;
                xx += wt * xv * xv; gg += wt * gv * gv; xg += wt * xv * gv;
            }
        const double vx = xx - mx * mx, vg = gg - mg * mg, cxg = xg - mx * mg;
        acc += (2.0 * mx * mg + C1) * (2.0 * cxg + C2) / ((mx * mx + mg * mg + C1) * (vx + vg + C2));
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = 128; s > 0; s >>= 1) {
        if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
    }
    if (threadIdx.x == 0) ssim[img] = vh > 0 && vw > 0 ? red[0] / ((double)vh * vw) : 0.0;
}

// ---------------------------------------------------------------------------
// Haar-wavelet l1 prox + FISTA update (eq. sirtista
// P:L397-409 with the paper's FISTA for the l1 penalties):
//   x = B^{-1} P_lam(B v) on each tile's valid rectangle, then
//   r = x + beta_o (x - x_prev), y = r - x_s, x_prev = x   (Alg. 3, A12).
// B: orthonormal 2D Haar with `levels` <= 5 levels (2^levels divides the
// valid sizes), in place: level l (stride s = 2^l) maps each 2x2 group of
// approximation samples (a b; c d) to ((a+b+c+d), (a-b+c-d), (a+b-c-d),
// (a-b-c+d)) / 2.  The transform is block-local (2^levels-pixel blocks), so a
// CTA owns a 32 x 32 region in shared memory; every coefficient is soft
// thresholded (symmetric, A15).  HBM-bound: reads v, x_s, x_prev, writes
// x_prev, y, y^T once.
// ---------------------------------------------------------------------------
struct HaarArgs {
    const float* v; const float* xs; float* xprev; long long p_tstride; int T;
    float* y; float* yT; long long y_tstride; int TP;
    const TileT* tiles;
    float lam; int levels; float beta_o;
};

__global__ void __launch_bounds__(256) k_haar(HaarArgs A) {
    __shared__ float sx[32][33];
    const int tile = blockIdx.y;
    const TileT ti = A.tiles[tile];
    const int Hv = ti.vr1 - ti.vr0, Wv = ti.vc1 - ti.vc0;
    const int nbx = (A.T + 31) / 32;
    const int by = blockIdx.x / nbx, bx = blockIdx.x - by * nbx;
    const int i0 = by * 32, j0 = bx * 32;              // region origin in valid-rect coordinates
    if (i0 >= Hv || j0 >= Wv) return;
    const long long pbase = (long long)tile * A.p_tstride;
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int e = threadIdx.x + 256 * u, i = e >> 5, j = e & 31;
        const bool ok = i0 + i < Hv && j0 + j < Wv;
        sx[i][j] = ok ? __ldcs(A.v + pbase + (long long)(ti.vr0 + i0 + i) * A.T + ti.vc0 + j0 + j) : 0.f;
    }
    __syncthreads();
    auto level = [&](int s) {
        const int ng = 32 / (2 * s);                        // groups per row of the region
        for (int e = threadIdx.x; e < ng * ng; e += 256) {
            const int gi = (e / ng) * 2 * s, gj = (e % ng) * 2 * s;
            const float a = sx[gi][gj], b = sx[gi][gj + s], c = sx[gi + s][gj], d = sx[gi + s][gj + s];
            sx[gi][gj] = 0.5f * (a + b + c + d);
            sx[gi][gj + s] = 0.5f * (a - b + c - d);
            sx[gi + s][gj] = 0.5f * (a + b - c - d);
            sx[gi + s][gj + s] = 0.5f * (a - b - c + d);
        }
        __syncthreads();
    };
    for (int l = 0; l < A.levels; ++l) level(1 << l);
    for (int e = threadIdx.x; e < 1024; e += 256) {
        const int i = e >> 5, j = e & 31;
        const float c = sx[i][j], m = fabsf(c) - A.lam;
        sx[i][j] = m > 0.f ? copysignf(m, c) : 0.f;
    }
    __syncthreads();
    for (int l = A.levels - 1; l >= 0; --l) level(1 << l);
    float xpv[4], xsv[4];                                             // all loads in flight first
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int e = threadIdx.x + 256 * u, i = e >> 5, j = e & 31;
        const bool ok = i0 + i < Hv && j0 + j < Wv;
        const long long pl = pbase + (long long)(ti.vr0 + i0 + i) * A.T + ti.vc0 + j0 + j;
        xpv[u] = ok ? __ldcs(A.xprev + pl) : 0.f;
        xsv[u] = ok ? __ldcs(A.xs + pl) : 0.f;
    }
    #pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int e = threadIdx.x + 256 * u, i = e >> 5, j = e & 31;
        if (i0 + i >= Hv || j0 + j >= Wv) continue;
        const int ti_ = ti.vr0 + i0 + i, tj = ti.vc0 + j0 + j;
        const long long pl = pbase + (long long)ti_ * A.T + tj;
        const float x = sx[i][j];
        const float rr = x + A.beta_o * (x - xpv[u]);                 // FISTA extrapolation (A12)
        const float yv = rr - xsv[u];                                 // x_L^k = r - x_s^k
        A.xprev[pl] = x;
        A.y[(long long)tile * A.y_tstride + (long long)ti_ * A.TP + PADL + tj] = yv;
        sx[i][j] = yv;                                                // own element: no race
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 1024; e += 256) {                  // y^T through shared memory (coalesced)
        const int j = e >> 5, i = e & 31;
        if (i0 + i >= Hv || j0 + j >= Wv) continue;
        const int ti_ = ti.vr0 + i0 + i, tj = ti.vc0 + j0 + j;
        A.yT[(long long)tile * A.y_tstride + (long long)tj * A.TP + PADL + ti_] = sx[i][j];
    }
}

// truncated data, edge-constant centred padding: one thread per output bin
__global__ void k_pad_truncated(int na, int nt, int nd, const float* __restrict__ in, float* __restrict__ out) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x, a = blockIdx.y;
    if (d >= nd) return;
    const int j = min(max(d - (nd - nt) / 2, 0), nt - 1);
    out[(long long)a * nd + d] = __ldg(in + (long long)a * nt + j);
}

// exterior subtraction (NEXT-4(ii)) helpers
// padded image + twin of x + c D (D: centred disc of diameter N; disc value read from the device)
__global__ void k_pack_disc(int n, int TP, const float* __restrict__ src, const float* __restrict__ discc, int use_disc,
                            float* __restrict__ img, float* __restrict__ imgT) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    float v = src[(long long)i * n + j];
    if (use_disc) {
        const int u = 2 * j - n + 1, w = 2 * i - n + 1;
        if (u * u + w * w <= n * n) v += *discc;
    }
    img[(long long)i * TP + PADL + j] = v;
    imgT[(long long)j * TP + PADL + i] = v;
}
// every tile's padded image + twin = M_{L'} of a padded global image
__global__ void k_extract_tiles(int T, int TP, const TileT* __restrict__ tiles, const float* __restrict__ g, int GTP,
                                float* __restrict__ y, float* __restrict__ yT, long long y_tstride) {
    const int r = blockIdx.z;
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= T || j >= T) return;
    const TileT ti = tiles[r];
    const bool valid = i >= ti.vr0 && i < ti.vr1 && j >= ti.vc0 && j < ti.vc1;
    const float v = valid ? g[(long long)(ti.row0 + i) * GTP + PADL + ti.col0 + j] : 0.f;
    y[(long long)r * y_tstride + (long long)i * TP + PADL + j] = v;
    yT[(long long)r * y_tstride + (long long)j * TP + PADL + i] = v;
}
// per-ROI window data p~ = (p - W xg)[window] + W_{L'} xg   (= p - W M_F xg on the window)
__global__ void k_dwin(int na, int nd, int Wwin, const int* __restrict__ d0, const float* __restrict__ rg,
                       const float* __restrict__ s, float* __restrict__ dw) {
    const int w = blockIdx.x * blockDim.x + threadIdx.x, a = blockIdx.y, r = blockIdx.z;
    if (w >= Wwin) return;
    const int d = d0[r * na + a] + w;
    const long long o = ((long long)r * na + a) * Wwin + w;
    dw[o] = (d >= 0 && d < nd) ? rg[(long long)a * nd + d] + s[o] : 0.f;
}

// global forward projection from tile windows: out[a][d] = sum over tiles (fixed
// order) of win[t][a][d - d0[t][a]] where inside the window; epilogues as k_fp
// (mode 1: out = v, aux_out = aux_in + alpha v; mode 2: out = aux_in - v)
__global__ void k_winsum(int mode, int na, int nd, int Wwin, int ntiles, const int* __restrict__ d0,
                         const float* __restrict__ win, float* __restrict__ out, const float* __restrict__ aux_in,
                         float* __restrict__ aux_out, float alpha, int a_off) {
    extern __shared__ int sd0[];
    const int a = blockIdx.y + a_off;
    for (int t = threadIdx.x; t < ntiles; t += blockDim.x) sd0[t] = d0[t * na + a];
    __syncthreads();
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= nd) return;
    float acc = 0.f;
    for (int t = 0; t < ntiles; ++t) {
        const int w = d - sd0[t];
        if (w >= 0 && w < Wwin) acc += __ldg(win + ((long long)t * na + a) * Wwin + w);
    }
    const long long o = (long long)a * nd + d;
    if (mode == 2) {
        out[o] = aux_in[o] - acc;
    } else {
        out[o] = acc;
        if (mode == 1) aux_out[o] = fmaf(alpha, acc, aux_in ? aux_in[o] : 0.f);
    }
}

// angle-split Alg. 1: c <- c - alpha (sum over ranks of W_g^T v_g),
// on the padded image and its transposed twin
__global__ void k_alg1_apply(int n, int GTP, const float* __restrict__ red, float alpha, float* c, float* cT) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= n || j >= n) return;
    const float u = alpha * red[(long long)i * n + j];
    c[(long long)i * GTP + PADL + j] -= u;
    cT[(long long)j * GTP + PADL + i] -= u;
}

// angle-split global box-SIRT: x <- clamp(x + alpha sum_g W_g^T r_g, lo, hi)
__global__ void k_gsirt_apply(int n, int GTP, const float* __restrict__ red, float alpha, float lo, float hi,
                              float* x, float* xT) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x, i = blockIdx.y * blockDim.y + threadIdx.y;
    if (i >= n || j >= n) return;
    const long long o = (long long)i * GTP + PADL + j;
    const float v = fminf(fmaxf(fmaf(alpha, red[(long long)i * n + j], x[o]), lo), hi);
    x[o] = v;
    xT[(long long)j * GTP + PADL + i] = v;
}

// window -> full sinogram (zero outside the window)
__global__ void k_scatter_win(int na, int nd, int Wwin, const int* __restrict__ d0,
                              const float* __restrict__ win, float* __restrict__ sino) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x, a = blockIdx.y;
    if (d >= nd) return;
    const int w = d - d0[a];
    sino[(long long)a * nd + d] = (w >= 0 && w < Wwin) ? win[(long long)a * Wwin + w] : 0.f;
}

// combine: CTA per 32x32 image block, fixed ascending-ROI order (A19).
// peers == nullptr: slot s is cores[s]; else slot s lives in rank s / spr's
// core buffer (peers[rank], a local or CUDA-IPC-mapped NVLink peer pointer)
// at index s % spr: the all-gather and the stitch in one pass over peer memory.
__global__ void k_stitch(int n, int side, int nbx, const int* __restrict__ lst_off, const int* __restrict__ lst,
                         const int* __restrict__ slot_r0, const int* __restrict__ slot_c0,
                         const float* __restrict__ cores, float* __restrict__ img,
                         const float* const* __restrict__ peers = nullptr, int spr = 1) {
    const int bx = blockIdx.x % nbx, by = blockIdx.x / nbx;
    const int j = bx * 32 + threadIdx.x;
    const int beg = lst_off[blockIdx.x], end = lst_off[blockIdx.x + 1];
    for (int ii = threadIdx.y; ii < 32; ii += blockDim.y) {
        const int i = by * 32 + ii;
        if (i >= n || j >= n) continue;
        float sum = 0.f; int cnt = 0;
        for (int q = beg; q < end; ++q) {
            const int s = lst[q];
            const int li = i - slot_r0[s], lj = j - slot_c0[s];
            if (li >= 0 && li < side && lj >= 0 && lj < side) {
                const float* c = peers ? peers[s / spr] + (long long)(s % spr) * side * side
                                       : cores + (long long)s * side * side;
                sum += c[(long long)li * side + lj];
                ++cnt;
            }
        }
        img[(long long)i * n + j] = cnt ? sum / (float)cnt : 0.f;
    }
}

// global FGP (a10 FISTA-TV on the full grid): one launch per phase, state in HBM
__global__ void k_gfgp_z(int n, float lam, const float* __restrict__ b, const float* __restrict__ r,
                         const float* __restrict__ s, float* __restrict__ z) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    const long long o = (long long)i * n + j;
    const float rup = i > 0 ? r[o - n] : 0.f, sl = j > 0 ? s[o - 1] : 0.f;
    z[o] = b[o] - lam * (r[o] + s[o] - rup - sl);
}
__global__ void k_gfgp_dual(int n, float gam, float beta, const float* __restrict__ z, float* __restrict__ r,
                            float* __restrict__ s, float* __restrict__ po, float* __restrict__ qo) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    const long long o = (long long)i * n + j;
    const float zc = z[o];
    const float pn = i < n - 1 ? clip1(r[o] + gam * (zc - z[o + n])) : 0.f;
    const float qn = j < n - 1 ? clip1(s[o] + gam * (zc - z[o + 1])) : 0.f;
    r[o] = pn + beta * (pn - po[o]); s[o] = qn + beta * (qn - qo[o]);
    po[o] = pn; qo[o] = qn;
}
__global__ void k_gfgp_out(int n, float lam, float beta_o, const float* __restrict__ b,
                           const float* __restrict__ po, const float* __restrict__ qo,
                           float* __restrict__ xprev, float* __restrict__ rm, float* __restrict__ rmT, int TP) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    const long long o = (long long)i * n + j;
    const float pup = i > 0 ? po[o - n] : 0.f, ql = j > 0 ? qo[o - 1] : 0.f;
    const float x = b[o] - lam * (po[o] + qo[o] - pup - ql);
    const float r = x + beta_o * (x - xprev[o]);
    xprev[o] = x;
    rm[(long long)i * TP + PADL + j] = r;
    rmT[(long long)j * TP + PADL + i] = r;
}

// ---------------------------------------------------------------------------
// Chambolle-Pock TV with diagonal preconditioning (NEXT-4(iii); oracle
// or_global_cp): data dual, TV dual and primal steps on the full grid.
// ---------------------------------------------------------------------------
// sd = 1 / (W 1) per ray (0 where the ray misses the grid)
__global__ void k_cp_recip(long long n, const float* __restrict__ w1, float* __restrict__ sd) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) sd[e] = w1[e] > 0.f ? 1.f / w1[e] : 0.f;
}
// tau = 1 / (W^T 1 + number of forward-difference terms touching the pixel)
__global__ void k_cp_tau(int n, const float* __restrict__ wt1, float* __restrict__ tau) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    const int terms = (i < n - 1) + (i > 0) + (j < n - 1) + (j > 0);
    tau[(long long)i * n + j] = 1.f / (wt1[(long long)i * n + j] + (float)terms);
}
// yd <- (yd + sd (W xbar - p)) / (1 + sd)
__global__ void k_cp_dual(long long n, const float* __restrict__ wx, const float* __restrict__ p,
                          const float* __restrict__ sd, float* __restrict__ yd) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < n) yd[e] = fmaf(sd[e], wx[e] - p[e], yd[e]) / (1.f + sd[e]);
}
// (yp, yq) <- clip_[-mu, mu]((yp, yq) + grad xbar / 2); xbar padded [n][TP] at PADL
__global__ void k_cp_tvdual(int n, int TP, float mu, const float* __restrict__ xb, float* __restrict__ yp,
                            float* __restrict__ yq) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    const long long o = (long long)i * n + j;
    const float* xr = xb + (long long)i * TP + PADL + j;
    const float dx = i < n - 1 ? xr[TP] - xr[0] : 0.f;
    const float dy = j < n - 1 ? xr[1] - xr[0] : 0.f;
    yp[o] = i < n - 1 ? fminf(mu, fmaxf(-mu, fmaf(0.5f, dx, yp[o]))) : 0.f;
    yq[o] = j < n - 1 ? fminf(mu, fmaxf(-mu, fmaf(0.5f, dy, yq[o]))) : 0.f;
}
// x' = x - tau (W^T yd + grad^T (yp, yq)); xbar = 2 x' - x (padded + twin); x = x'
__global__ void k_cp_primal(int n, int TP, const float* __restrict__ g, const float* __restrict__ yp,
                            const float* __restrict__ yq, const float* __restrict__ tau, float* __restrict__ x,
                            float* __restrict__ xb, float* __restrict__ xbT) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    const long long o = (long long)i * n + j;
    const float gt = -(yp[o] + yq[o]) + (i > 0 ? yp[o - n] : 0.f) + (j > 0 ? yq[o - 1] : 0.f);
    const float xo = x[o];
    const float xn = xo - tau[o] * (g[o] + gt);
    x[o] = xn;
    const float b = 2.f * xn - xo;
    xb[(long long)i * TP + PADL + j] = b;
    xbT[(long long)j * TP + PADL + i] = b;
}

__global__ void k_unpack(int n, int TP, const float* __restrict__ img, float* __restrict__ out) {
    const int j = blockIdx.x * 32 + threadIdx.x, i = blockIdx.y * 8 + threadIdx.y;
    if (i >= n || j >= n) return;
    out[(long long)i * n + j] = img[(long long)i * TP + PADL + j];
}

__global__ void k_impulse(int n, int TP, float* img, float* imgT) {
    // e_c (A5): 2x2 average of the central pixels for even N, centre pixel for odd N
    if (threadIdx.x != 0) return;
    if (n % 2) {
        const int m = n / 2;
        img[(long long)m * TP + PADL + m] = 1.f; imgT[(long long)m * TP + PADL + m] = 1.f;
    } else {
        const int m = n / 2;
        for (int di = -1; di <= 0; ++di)
            for (int dj = -1; dj <= 0; ++dj) {
                img[(long long)(m + di) * TP + PADL + m + dj] = 0.25f;
                imgT[(long long)(m + dj) * TP + PADL + m + di] = 0.25f;
            }
    }
}

}  // namespace lt
