// projectors.cuh -- Joseph forward projectors (k_fp, k_fp_roi2, k_fp_join) and the backprojector with its fused epilogues (k_bp)
// (part of kernels.cuh; notation and layouts: see kernels.cuh and DESIGN.md)
#pragma once
#include "common.cuh"

namespace lt {

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
#ifndef FP_BLN
#define FP_BLN 16
#endif
constexpr int FP2_BL = FP_BLN;   // lines per band
#ifndef FP_LEAN
#define FP_LEAN 1   // line positions by FFMA2 pairs; per-ray-group anchors by fp64 increments and magic rounding
#endif
constexpr int FP2_P = 272;       // (S, D) entries per staged line (>= T + PADL + PADR)
constexpr int FP2_PW = 336;      // wide tiles (T <= 328 - PADL - PADR = 320): entries per staged line
constexpr int FP_UW = 15;        // wide tiles: rays per lane (window W(160) = 456 <= 32 * 15)
constexpr int FP2_CPT = (FP2_P / 4 + 15) / 16;  // float4 chunks per thread per band (16 threads per line)
#ifndef FP_XPAD
#define FP_XPAD 16     // zero (S, D) entries staged on each side of a line (0: the round-1/2 layout)
#endif
// With FP_XPAD >= 16 every ray the band visits stays inside its staged line
// (positions reach at most 15 |B| + 2 A + 1 < 19 px beyond the valid pixels:
// PADL + FP_XPAD zero pixels on the left, >= PADR + FP_XPAD on the right), so
// the clamped ray variant (FMNMX per step) is no longer needed for the rays
// near the tile edges; the results are bitwise the same (zeros either way).
// Only the two-angles-per-warp kernels (C4 / C5 batches) take the margins: the
// one-angle-per-warp kernel of small batches measured slower with them (L1 FP
// 0.062 -> 0.068 ms per launch) and keeps the clamped edge groups.
__host__ __device__ constexpr int fp_line(int sp, int apw) { return sp + 2 * (apw == 2 ? FP_XPAD : 0); }   // staged entries per line
#ifndef FP_STAGE64
#define FP_STAGE64 1   // staging by 8-byte pixel pairs: each STS.128 of a half-warp covers 256 contiguous bytes
#endif
constexpr int FP2_CPT2 = (FP2_P / 2 + 15) / 16; // float2 chunks per thread per band (FP_STAGE64)

#ifndef FP_PIPE
#define FP_PIPE 1      // the loads of the next line pair issued before the current pair is consumed
#endif                 // (C4 FP 1.427 -> 1.417 ms, bitwise identical; ray addresses by mad.lo: no change)
template <bool CLAMP, int SP = FP2_P>
__device__ __forceinline__ float fp2_band_ray(unsigned rowbase_, float f0, float Bf, float lo, float hi) {
    const unsigned rowbase = __shfl_sync(0xffffffffu, rowbase_, threadIdx.x & 31);
    float acc = 0.f;
#if FP_LEAN
    const float2 B2 = make_float2(Bf, Bf), f01 = make_float2(f0, f0 + Bf);
#endif
    auto addr_g = [&](int i, unsigned& a0, unsigned& a1, float2& g) {
#if FP_LEAN
        float2 tt = __ffma2_rn(B2, make_float2((float)i, (float)i), f01);          // lines i, i + 1: one FFMA2
#else
        float2 tt = make_float2(fmaf((float)i, Bf, f0), fmaf((float)(i + 1), Bf, f0));   // immediates
#endif
        if (CLAMP) {
            tt.x = fminf(fmaxf(tt.x, lo), hi);
            tt.y = fminf(fmaxf(tt.y, lo), hi);
        }
        const float2 rm = __fadd2_rn(tt, make_float2(MAGICF, MAGICF));           // round(tt) in the low bits
        const float2 k2 = __ffma2_rn(rm, make_float2(-2.f, -2.f), make_float2(2.f * MAGICF, 2.f * MAGICF));   // -2 round(tt)
        g = __ffma2_rn(tt, make_float2(2.f, 2.f), k2);                          // 2 (tt - round(tt)) in [-1, 1]
        a0 = rowbase + ((unsigned)__float_as_int(rm.x) << 3);
        a1 = rowbase + ((unsigned)__float_as_int(rm.y) << 3);
    };
#if FP_PIPE
    unsigned a0, a1;
    float2 g;
    addr_g(0, a0, a1, g);
    float s0, d0, s1, d1;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(s0), "=f"(d0) : "r"(a0));
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(s1), "=f"(d1) : "r"(a1 + (unsigned)(SP * 8)));
    #pragma unroll
    for (int i = 0; i < FP2_BL; i += 2) {
        float ns0 = 0.f, nd0 = 0.f, ns1 = 0.f, nd1 = 0.f;
        float2 ng = g;
        if (i + 2 < FP2_BL) {
            unsigned b0, b1;
            addr_g(i + 2, b0, b1, ng);
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(ns0), "=f"(nd0) : "r"(b0 + (unsigned)((i + 2) * SP * 8)));
            asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(ns1), "=f"(nd1) : "r"(b1 + (unsigned)((i + 3) * SP * 8)));
        }
        acc = fmaf(g.x, d0, acc + s0);
        acc = fmaf(g.y, d1, acc + s1);
        s0 = ns0; d0 = nd0; s1 = ns1; d1 = nd1; g = ng;
    }
#else
    #pragma unroll
    for (int i = 0; i < FP2_BL; i += 2) {
        unsigned a0, a1;
        float2 g;
        addr_g(i, a0, a1, g);
        float s0, d0, s1, d1;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(s0), "=f"(d0) : "r"(a0 + (unsigned)(i * SP * 8)));
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(s1), "=f"(d1) : "r"(a1 + (unsigned)((i + 1) * SP * 8)));
        acc = fmaf(g.x, d0, acc + s0);
        acc = fmaf(g.y, d1, acc + s1);
    }
#endif
    return acc;
}

// (a double-buffered band -- one CTA barrier per band, the transform off the
// critical path -- measured no faster: C4 FP 1.431 vs 1.425 ms; not kept)
// SP, SU: staged entries per line and rays per lane (FP2_P, FP_U; FP2_PW, FP_UW for
// tiles wider than 256)
template <int FP_APW, int NWARP = 8, int SP = FP2_P, int SU = FP_U>
__global__ void __launch_bounds__(NWARP * 32, NWARP == 8 ? 3 : 2) k_fp_roi2(Geo g, Tiles t, FpArgs f,
                                                                            const int* __restrict__ groups) {
    constexpr int FP_GA = NWARP * FP_APW;       // angles per CTA (they share each staged band)
    constexpr int FP2_P = SP, FP_U = SU;
    constexpr int FP_XP = FP_APW == 2 ? FP_XPAD : 0;   // zero entries on each side of a staged line
    constexpr int SPX = fp_line(SP, FP_APW);            // staged entries per line
    constexpr int FP2_CPT = (FP2_P / 4 + 15) / 16, FP2_CPT2 = (FP2_P / 2 + 15) / 16;
    extern __shared__ float4 smf4[];
    float2* sd = reinterpret_cast<float2*>(smf4);                 // [FP2_BL][SPX] (S, D), entry 0 = pixel -PADL - FP_XP
    float* sacc = reinterpret_cast<float*>(sd + FP2_BL * SPX);    // [FP_GA][32 * FP_U] per-ray accumulators
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
    for (int e = threadIdx.x; e < FP_GA * 32 * FP_U; e += NWARP * 32) sacc[e] = 0.f;
    if constexpr (FP_XP > 0) {   // the zero margins of every staged line (never overwritten by the staging):
        // FP_XP entries before and after the raw line (entries past them are never read)
        const int rb = FP_XP + TP;               // first entry after the raw line
        for (int e = threadIdx.x; e < FP2_BL * 2 * FP_XP; e += NWARP * 32) {
            const int l = e / (2 * FP_XP), k = e - l * 2 * FP_XP;
            sd[l * SPX + (k < FP_XP ? k : rb + (k - FP_XP))] = make_float2(0.f, 0.f);
        }
    }

    const int q4 = TP / 4;                        // float4 chunks per raw line
    const int q2 = TP / 2;                        // float2 chunks per raw line
#if FP_STAGE64
    // every thread stages: TPL = (threads / 16) threads per line (16 or 24),
    // thread = (line tid / TPL, pixel pairs c2 = tid % TPL + TPL u): entry pair
    // (2 c2, 2 c2 + 1) is one 16-byte store, a line's threads write contiguous bytes
    constexpr int TPL = NWARP * 32 / FP2_BL;
    constexpr int CPT2 = (FP2_P / 2 + TPL - 1) / TPL;
    const int sline = (int)threadIdx.x / TPL, sc0 = (int)threadIdx.x - sline * TPL;
    float2 raw[CPT2];
    float nxt[CPT2];
    auto fetch = [&](int l0) {
        const bool lok = sline < FP2_BL && l0 + sline < T;
        const float* rp0 = src + (long long)(l0 + sline) * TP;
        #pragma unroll
        for (int u = 0; u < CPT2; ++u) {
            const int c2 = sc0 + TPL * u;
            raw[u] = make_float2(0.f, 0.f);
            nxt[u] = 0.f;
            if (lok && c2 < q2) {
                raw[u] = __ldg(reinterpret_cast<const float2*>(rp0 + c2 * 2));
                if (c2 + 1 < q2) nxt[u] = __ldg(rp0 + c2 * 2 + 2);
            }
        }
    };
    auto transform = [&]() {
        #pragma unroll
        for (int u = 0; u < CPT2; ++u) {
            const int c2 = sc0 + TPL * u;
            if (sline < FP2_BL && c2 < q2) {
                const float2 v = raw[u];
                *reinterpret_cast<float4*>(sd + sline * SPX + FP_XP + c2 * 2) =
                    make_float4(v.x + v.y, v.y - v.x, v.y + nxt[u], nxt[u] - v.y);
            }
        }
    };
#else
    const int sline = threadIdx.x >> 4, sc0 = threadIdx.x & 15;   // (threads 256.. of a 12-warp CTA do not stage)
    float4 raw[FP2_CPT];
    float nxt[FP2_CPT];
    auto fetch = [&](int l0) {                    // raw lines l0.. of the band into registers
        const bool lok = sline < FP2_BL && l0 + sline < T;
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
            if (sline < FP2_BL && c4 < q4) {
                const float4 v = raw[u];
                float4* dst = reinterpret_cast<float4*>(sd + sline * SPX + FP_XP + c4 * 4);
                dst[0] = make_float4(v.x + v.y, v.y - v.x, v.y + v.z, v.z - v.y);
                dst[1] = make_float4(v.z + v.w, v.w - v.z, v.w + nxt[u], nxt[u] - v.w);
            }
        }
    };
#endif
    const int nsplit = f.nsplit > 1 ? f.nsplit : 1;
    const int lbeg = (lv0 / FP2_BL) * FP2_BL + (int)blockIdx.z * FP2_BL, lstep = nsplit * FP2_BL;
    if (lbeg < lv1) { fetch(lbeg); transform(); }
    __syncthreads();
#if FP_LEAN
    const unsigned sbase = opaque_u32((unsigned)__cvta_generic_to_shared(sd + FP_XP + PADL));   // entry of pixel 0 (kept in a register)
#else
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(sd + FP_XP + PADL);     // entry of pixel 0
#endif
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
#if FP_LEAN
            const unsigned acc_s = opaque_u32((unsigned)__cvta_generic_to_shared(acc));   // (no per-group address rebuild)
#endif
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
#if FP_LEAN
            constexpr double MAGICD = 6755399441055744.0;      // 1.5 * 2^52: x + MAGICD rounds x in the low bits
            double pc = P0 + (double)(wlo + 16) * A;           // fp64 anchor of the first group, + 32 A per group
            const double A32 = 32.0 * A;
#endif
            for (int wb = wlo; wb < whi; wb += 32) {
                const int w = wb + lane;
                const bool ray = w < whi;
                // position (pixel index) on line l0: fp64 anchor at the group's
                // middle ray, fp32 offset |(lane - 16) A| <= 23 px
#if FP_LEAN
                const double rmd = pc + MAGICD;                 // round(pc) in the low bits
                const double frd = pc - (rmd - MAGICD);         // in [-1/2, 1/2]
                pc += A32;
                const float pos = fmaf((float)(lane - 16), Af, (float)frd);
                const float rmf = pos + MAGICF;                 // a nearest integer of pos (any integer near pos will do)
                const float fl = rmf - MAGICF;
                const int ib = ray ? (int)__double2loint(rmd) + (__float_as_int(rmf) - MAGICI) : 0;
                const float f0 = ray ? (pos - fl) - 0.5f : -0.5f;
#else
                const double pc = P0 + (double)(wb + 16) * A;
                const double fbc = floor(pc);
                const float pos = fmaf((float)(lane - 16), Af, (float)(pc - fbc));
                const float fl = floorf(pos);
                const int ib = ray ? (int)fbc + (int)fl : 0;
                const float f0 = ray ? (pos - fl) - 0.5f : -0.5f;
#endif
                const float Bu = ray ? Bf : 0.f;
                const float pa = (float)ib + f0 + 0.5f, pe = pa + Bl;
                // inside the zeroed / staged entries (pixels -PADL - FP_XP .. TP - PADL + FP_XP - 1), one pixel to spare
                // (FP_XP = 0: the round-2 bounds, pixels -3 .. T + 1.5 of the raw line)
                const bool safe = !ray || (FP_XP > 0 ? (fminf(pa, pe) >= (float)(1 - PADL - FP_XP) &&
                                                        fmaxf(pa, pe) <= (float)(TP - PADL + FP_XP - 3))
                                                     : (fminf(pa, pe) >= -3.f && fmaxf(pa, pe) <= (float)T + 1.5f));
                const unsigned rowbase = sbase + 8u * (unsigned)(ib - MAGICI);
                float v;
                if (__all_sync(0xffffffffu, safe)) {
                    v = fp2_band_ray<false, SPX>(rowbase, f0, Bu, 0.f, 0.f);
                } else {
                    const float lo = (float)(-3 - ib) - 0.5f, hi = (float)(T + 2 - ib) - 0.5f;
                    v = fp2_band_ray<true, SPX>(rowbase, f0, Bu, lo, hi);
                }
#if FP_LEAN
                if (ray) {
                    float o;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(acc_s + 4u * (unsigned)w) : "memory");
                    asm volatile("st.shared.f32 [%0], %1;" ::"r"(acc_s + 4u * (unsigned)w), "f"(o + v) : "memory");
                }
#else
                if (ray) acc[w] += v;
#endif
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
#ifndef BP_PAIR_WEIGHTS
#define BP_PAIR_WEIGHTS 0   // 1: FFMA2 + lower clamp (FMNMX) weights (measured slower: BP 1.19 vs 0.96 ms avg)
#endif
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

// SUBH: sub-tile height (SUB wide): 64 x 128 sub-tiles give each thread 2 x 16
// pixels, so the per-angle setup is spread over twice the pixels
template <int NS, int MODE, int SUB = BP_SUB, int SUBH = SUB>
__global__ void __launch_bounds__(256) k_bp(Geo g, Tiles t, SinoView s1, SinoView s2, BpEpi e) {
    static_assert(NS == 0 || NS == 1, "one gathered sinogram at most");
    static_assert((SUB == 64 && (SUBH == 32 || SUBH == 64 || SUBH == 128)) || (SUB == 32 && SUBH == 32),
                  "64x32 / 64x64 / 64x128 (2 columns x 4 / 8 / 16 rows per thread) or 32x32 (1 x 4) sub-tiles");
    constexpr int COLS = SUB / 32;                // columns per thread (32 apart)
    constexpr int BP_PR = SUB * SUBH / (256 * COLS);  // rows per thread
    // window bins (unit bin spacing): centred on the sub-tile centre's projection, half-width
    // >= max |u - u_c| + 2 = sqrt(((SUB-1)/2)^2 + ((SUBH-1)/2)^2) + 2 (46.5 / 72.9 / 37.1 / 23.9 of 48 / 80 / 48 / 32),
    // a multiple of 32 (64 x 32 sub-tiles take the 64 x 64 window)
    constexpr int BP_SW = SUB == 64 ? (SUBH == 128 ? 160 : 96) : 64;
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
    const int pi0 = sty * SUBH + wq * BP_PR;           // rows pi0 .. pi0 + BP_PR - 1
    const double Lc = 0.5 * (T - 1);
    const double hsx = 0.5 * (SUB - 1), hsy = 0.5 * (SUBH - 1);
    const double dxc = stx * SUB + hsx - Lc, dyc = sty * SUBH + hsy - Lc;
    const float dx = (float)lane - (float)hsx, dy0 = (float)(wq * BP_PR) - (float)hsy;

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
#if BP_PAIR_WEIGHTS
                    // (K' - u, K' + u) as one FFMA2, clamped at 0 only (K' + |u| <= 1 exactly)
                    const float2 icp = make_float2(-A4.w, A4.w), kk2 = make_float2(A4.z, A4.z);
                    float2 w0 = __ffma2_rn(icp, make_float2(gg.x, gg.x), kk2);
                    float2 w1 = __ffma2_rn(icp, make_float2(gg.y, gg.y), kk2);
                    w0 = make_float2(fmaxf(w0.x, 0.f), fmaxf(w0.y, 0.f));
                    w1 = make_float2(fmaxf(w1.x, 0.f), fmaxf(w1.y, 0.f));
#else
                    const float2 w0 = make_float2(__saturatef(fmaf(-gg.x, A4.w, A4.z)), __saturatef(fmaf(gg.x, A4.w, A4.z)));
                    const float2 w1 = make_float2(__saturatef(fmaf(-gg.y, A4.w, A4.z)), __saturatef(fmaf(gg.y, A4.w, A4.z)));
#endif
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

}  // namespace lt
