// fgp.cuh -- FGP TV prox + FISTA update on thread-block clusters (k_fgp2) and its DSMEM / mbarrier helpers
// (part of kernels.cuh; notation and layouts: see kernels.cuh and DESIGN.md)
#pragma once
#include "common.cuh"

namespace lt {

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
    int ntiles;             // persistent launch: tiles blockIdx.y, + gridDim.y, ... < ntiles
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
#ifndef FGP_OPAQUE
#define FGP_OPAQUE 1   // loop-invariant shared addresses kept in registers (not rematerialised from SR_CgaCtaId)
#endif
#ifndef FGP_KEEP4
#define FGP_KEEP4 1    // CP = 4: 0 none, 1 the mbarrier base only (1.267 -> 1.261 ms), 2 all (1.273; tools/ab_fgpkeep4.sh)
#endif
// K: keep x in a register (an opaque move).  Measured (tools/ab_fgpkeep2.sh, FGP per
// launch): C3 (CP = 3) 0.188 -> 0.178 ms, P1 (CP = 5) 0.079 -> 0.077, but C4 (CP = 4,
// 232 -> 228 registers) 1.271 -> 1.276, so the CP = 4 kernel leaves it to ptxas
template <bool K>
__device__ __forceinline__ unsigned keep_u32(unsigned x) {
    if constexpr (K && FGP_OPAQUE) asm volatile("mov.b32 %0, %0;" : "+r"(x));
    return x;
}
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
// Warp w of CTA k owns FR full rows (rows (k*NW + w)*FR ...) of the tile,
// 64*CP columns wide; lane l owns the 2*CP consecutive columns 2CP*l .. of each
// row, as CP column pairs (CP = 4: 256-wide tiles; CP = 5: 320-wide tiles,
// the paper's 256^2 local parts with 1/8 padding).  Vertical
// neighbours are the same lane (aligned pairs -> paired instructions); the
// horizontal neighbour across a lane boundary comes by one warp shuffle per
// row and direction.  Rows crossing warps go through shared memory, rows
// crossing CTAs through DSMEM (st.async + mbarrier).
//
// Masks (A13, Neumann boundary on the valid rectangle H_v x W_v):
// p exists for rows i < H_v - 1 (warp-uniform per row), q for columns
// j < W_v - 1 (per-column step register).  Pixels outside the valid rectangle
// carry finite garbage that no valid pixel reads.
// (Measured slower in round 1 and removed: named-barrier hand-over between
// warps, a paired left-neighbour term, halo prefetch at the phase start, a
// barrier before each halo row.)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 f2s(float s) { return make_float2(s, s); }

// Staged row layout (shared memory), CP column pairs per lane: pairs 2h, 2h+1
// of lane l as one float4 at h*128 + 4l (h < CP/2), an odd last pair as a
// float2 at (CP/2)*128 + 2l -- every access of a warp is conflict free.
template <int CP> struct RowL {
    static constexpr int ROW = 64 * CP;            // floats per staged row
    static constexpr int NQ = CP / 2;              // float4 chunks per lane
    static constexpr bool ODD = (CP & 1) != 0;     // one float2 chunk
};
template <int CP>
__device__ __forceinline__ void row_st(float* row, int lane, const float2 (&v)[CP]) {
    #pragma unroll
    for (int h = 0; h < CP / 2; ++h)
        reinterpret_cast<float4*>(row + 128 * h)[lane] = make_float4(v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y);
    if constexpr (CP & 1) reinterpret_cast<float2*>(row + 128 * (CP / 2))[lane] = v[CP - 1];
}
template <int CP>
__device__ __forceinline__ void row_ld(const float* row, int lane, float2 (&v)[CP]) {
    #pragma unroll
    for (int h = 0; h < CP / 2; ++h) {
        const float4 a = reinterpret_cast<const float4*>(row + 128 * h)[lane];
        v[2 * h] = make_float2(a.x, a.y); v[2 * h + 1] = make_float2(a.z, a.w);
    }
    if constexpr (CP & 1) v[CP - 1] = reinterpret_cast<const float2*>(row + 128 * (CP / 2))[lane];
}
// the same through 32-bit shared-window addresses (loop-invariant bases, no
// generic-to-shared conversion inside the iteration loop)
template <int CP>
__device__ __forceinline__ void row_st_s(unsigned row, int lane, const float2 (&v)[CP]) {
    #pragma unroll
    for (int h = 0; h < CP / 2; ++h)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(row + 512u * h + 16u * lane),
                     "f"(v[2 * h].x), "f"(v[2 * h].y), "f"(v[2 * h + 1].x), "f"(v[2 * h + 1].y) : "memory");
    if constexpr (CP & 1)
        asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(row + 512u * (CP / 2) + 8u * lane),
                     "f"(v[CP - 1].x), "f"(v[CP - 1].y) : "memory");
}
template <int CP>
__device__ __forceinline__ void row_ld_s(unsigned row, int lane, float2 (&v)[CP]) {
    #pragma unroll
    for (int h = 0; h < CP / 2; ++h) {
        float a0, a1, a2, a3;
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3)
                     : "r"(row + 512u * h + 16u * lane) : "memory");
        v[2 * h] = make_float2(a0, a1); v[2 * h + 1] = make_float2(a2, a3);
    }
    if constexpr (CP & 1) {
        float a0, a1;
        asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(a0), "=f"(a1) : "r"(row + 512u * (CP / 2) + 8u * lane)
                     : "memory");
        v[CP - 1] = make_float2(a0, a1);
    }
}
// a lane's 2*CP consecutive columns of a naturally laid out shared row (8-byte aligned)
template <int CP>
__device__ __forceinline__ void row_ld_nat(const float* p, float2 (&v)[CP]) {
    if constexpr (CP % 2 == 0) {
        #pragma unroll
        for (int h = 0; h < CP / 2; ++h) {
            const float4 a = reinterpret_cast<const float4*>(p)[h];
            v[2 * h] = make_float2(a.x, a.y); v[2 * h + 1] = make_float2(a.z, a.w);
        }
    } else {
        #pragma unroll
        for (int c2 = 0; c2 < CP; ++c2) v[c2] = reinterpret_cast<const float2*>(p)[c2];
    }
}
__device__ __forceinline__ void mbar_arrive(unsigned bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void st_async_v4(unsigned remote, float4 v, unsigned remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1, %2, %3, %4}, [%5];"
                 ::"r"(remote), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(remote_bar) : "memory");
}
__device__ __forceinline__ void st_async_v2(unsigned remote, float2 v, unsigned remote_bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f32 [%0], {%1, %2}, [%3];"
                 ::"r"(remote), "f"(v.x), "f"(v.y), "r"(remote_bar) : "memory");
}
template <int CP>
__device__ __forceinline__ void row_push(unsigned remote_row, int lane, const float2 (&v)[CP], unsigned remote_bar) {
    #pragma unroll
    for (int h = 0; h < CP / 2; ++h)
        st_async_v4(remote_row + 512u * h + 16u * lane, make_float4(v[2 * h].x, v[2 * h].y, v[2 * h + 1].x, v[2 * h + 1].y),
                    remote_bar);
    if constexpr (CP & 1) st_async_v2(remote_row + 512u * (CP / 2) + 8u * lane, v[CP - 1], remote_bar);
}

constexpr int FGP2_ROW = 256;     // columns per warp row of the CP = 4 kernel (32 lanes x 8)
constexpr int FGP2_ROW_MAX = 320; // widest tile (CP = 5)
template <int V> struct Parity { __device__ __forceinline__ operator int() const { return V; } };

template <int FR, int NW, int CP = 4>
struct Fgp2Smem {
    static constexpr int ROW = RowL<CP>::ROW;
    // halo rows, one slot per warp and parity, so every warp reads its halo
    // from the same place whichever warp or CTA wrote it:
    //   hr[par][j]: the r row above warp j (j = 0: pushed by the CTA above over
    //               DSMEM; j > 0: the last row of warp j - 1)
    //   hz[par][j]: the z row below warp j - 1 (j < NW: the first row of warp j;
    //               j = NW: pushed by the CTA below)
    // slots never written keep their initial value (r: the shifted zero 1/2, z: 0)
    static constexpr int bars = 0;                             // 4 x u64: r from above [2], z from below [2]
    static constexpr int hr = 8;                               // [2][NW + 1][ROW]
    static constexpr int hz = hr + 2 * (NW + 1) * ROW;         // [2][NW + 1][ROW]
    static constexpr int hp = hz + 2 * (NW + 1) * ROW;         // [NW][ROW] last p row (epilogue)
    static constexpr int bsm = hp + NW * ROW;                  // [NW][FR][ROW] b (BSM variant)
    static constexpr int total = bsm;
    static constexpr int total_bsm = bsm + NW * FR * ROW;
    // MODE 1: [NW][FR][2][ROW] xprev and x_s rows, fetched with cp.async at
    // kernel start (they are inputs the FGP loop never touches) and read by the epilogue
    static constexpr int xin_floats = NW * FR * 2 * ROW;
    // persistent launch: [NW][FR][ROW] b of the cluster's next tile (cp.async)
    static constexpr int bnext_floats = NW * FR * ROW;
};
__device__ __forceinline__ void mbar_inval(unsigned bar) {
    asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(void* sdst, const void* gsrc) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sdst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_all;" ::: "memory");
}
// a lane's 2*CP columns [x0, x0 + 2CP) of a global row into shared memory by
// cp.async: 16-byte chunks (CP even, 16-byte aligned source), 8-byte chunks
// (CP odd, 8-byte aligned), else per float; columns >= wv are not copied
template <int CP>
__device__ __forceinline__ void cp_async_cols(float* dst, const float* src, int x0, int wv, bool vec) {
    if constexpr (CP % 2 == 0) {
        #pragma unroll
        for (int h = 0; h < CP / 2; ++h) {
            if (vec && x0 + 4 * h + 3 < wv) {
                cp_async16(dst + 4 * h, src + 4 * h);
            } else {
                #pragma unroll
                for (int c = 4 * h; c < 4 * h + 4; ++c)
                    if (x0 + c < wv) cp_async4(dst + c, src + c);
            }
        }
    } else {
        #pragma unroll
        for (int c2 = 0; c2 < CP; ++c2) {
            if (vec && x0 + 2 * c2 + 1 < wv) {
                cp_async8(dst + 2 * c2, src + 2 * c2);
            } else {
                #pragma unroll
                for (int c = 2 * c2; c < 2 * c2 + 2; ++c)
                    if (x0 + c < wv) cp_async4(dst + c, src + c);
            }
        }
    }
}
// store a lane's 2*CP values to a global row (16- / 8-byte stores when aligned)
template <int CP>
__device__ __forceinline__ void st_cols(float* dst, const float* v, int x0, int wv, bool vec) {
    if constexpr (CP % 2 == 0) {
        #pragma unroll
        for (int h = 0; h < CP / 2; ++h) {
            if (vec && x0 + 4 * h + 3 < wv) {
                *reinterpret_cast<float4*>(dst + 4 * h) = make_float4(v[4 * h], v[4 * h + 1], v[4 * h + 2], v[4 * h + 3]);
            } else {
                #pragma unroll
                for (int c = 4 * h; c < 4 * h + 4; ++c)
                    if (x0 + c < wv) dst[c] = v[c];
            }
        }
    } else {
        #pragma unroll
        for (int c2 = 0; c2 < CP; ++c2) {
            if (vec && x0 + 2 * c2 + 1 < wv) {
                *reinterpret_cast<float2*>(dst + 2 * c2) = make_float2(v[2 * c2], v[2 * c2 + 1]);
            } else {
                #pragma unroll
                for (int c = 2 * c2; c < 2 * c2 + 2; ++c)
                    if (x0 + c < wv) dst[c] = v[c];
            }
        }
    }
}

// BSM: b (read once per iteration) lives in shared memory instead of registers,
// so the kernel fits 128 registers and two CTAs (two tiles) share an SM: one
// tile's halo latency is hidden behind the other tile's arithmetic.
// PERSIST: the grid holds only as many clusters as are co-resident; each
// cluster iterates over the tiles blockIdx.y, + gridDim.y, ... and fetches the
// next tile's b, x_prev and x_s by cp.async while iterating the current one.
template <int MODE, int FR, int NW, bool BSM, bool PERSIST = false, int CP = 4>
__global__ void __launch_bounds__(NW * 32, (BSM && NW <= 8) ? 2 : 1) k_fgp2(FgpArgs A) {
    static_assert(!(PERSIST && BSM), "persistent launch keeps b in registers");
    static_assert(CP >= 1 && CP <= 5, "64-, 128-, 192-, 256- or 320-wide tiles");
    using SM = Fgp2Smem<FR, NW, CP>;
    constexpr int ROW = SM::ROW;
    constexpr int NC = 2 * CP;                  // columns per lane
    extern __shared__ __align__(16) float sm[];
    cg::cluster_group cl = cg::this_cluster();
    const int K = (int)cl.num_blocks();
    const int kr = (int)cl.block_rank();
    const int tile_end = PERSIST ? A.ntiles : (int)blockIdx.y + 1;
    int tcount = 0;
    for (int tile = blockIdx.y; tile < tile_end; tile += gridDim.y, ++tcount) {
    int vr0 = 0, vc0 = 0, Hv = A.H, Wv = A.W;
    if (A.tiles) {
        const TileT ti = A.tiles[tile];
        vr0 = ti.vr0; vc0 = ti.vc0; Hv = ti.vr1 - ti.vr0; Wv = ti.vc1 - ti.vc0;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int i0 = (kr * NW + w) * FR;          // first row of this warp (valid-rectangle coordinates)
    const int x0 = lane * NC;                   // first column of this lane
    const bool has_up = kr > 0, has_dn = kr < K - 1;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(sm + SM::bars);
    float* hp = sm + SM::hp;
    for (int e = threadIdx.x; e < SM::hp - SM::hr; e += NW * 32)
        sm[SM::hr + e] = SM::hr + e >= SM::hz ? 0.f : 0.5f;   // z halos start at 0, dual halos at the shifted zero 1/2
    if (threadIdx.x == 0) {
        for (int q_ = 0; q_ < 4; ++q_) {
            if (PERSIST && tcount > 0) mbar_inval(smem_u32(bars + q_));   // (every transfer of the last tile landed)
            mbar_init(smem_u32(bars + q_), 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    float2 breg[BSM ? 1 : FR][CP], r[FR][CP], s[FR][CP], p[FR][CP], q[FR][CP], z[FR][CP];
    float* bs = sm + SM::bsm + (w * FR) * ROW;               // this warp's b rows (BSM)
    auto bget = [&](int k, float2 (&v)[CP]) {
        if constexpr (BSM) {
            row_ld<CP>(bs + k * ROW, lane, v);
        } else {
            #pragma unroll
            for (int c2 = 0; c2 < CP; ++c2) v[c2] = breg[k][c2];
        }
    };
    const float* bsrc = A.b + (long long)tile * A.b_tstride + (long long)vr0 * A.b_pitch + vc0;
    // vector loads when the rows are aligned (16 bytes for CP = 4, 8 for CP = 5)
    // and the lane's columns are valid
    constexpr unsigned VAL = CP % 2 == 0 ? 15u : 7u;
    const bool vec_b = ((reinterpret_cast<uintptr_t>(bsrc) | ((uintptr_t)A.b_pitch << 2)) & VAL) == 0 && x0 + NC <= Wv;
    float* bnext = sm + SM::total + 2 * SM::xin_floats + (w * FR) * ROW;   // (PERSIST layout)
    if (PERSIST && tcount > 0) cp_async_commit_wait_all();   // this tile's b, x_prev, x_s (prefetched)
    #pragma unroll
    for (int k = 0; k < FR; ++k) {
        const int i = i0 + k;
        float2 bv[CP];
        const float* brow = bsrc + (long long)i * A.b_pitch + x0;
        if (PERSIST && tcount > 0) {
            row_ld_nat<CP>(bnext + k * ROW + x0, bv);
        } else if (vec_b && i < Hv) {
            if constexpr (CP % 2 == 0) {
                #pragma unroll
                for (int h = 0; h < CP / 2; ++h) {
                    const float4 u0 = __ldg(reinterpret_cast<const float4*>(brow) + h);
                    bv[2 * h] = make_float2(u0.x, u0.y); bv[2 * h + 1] = make_float2(u0.z, u0.w);
                }
            } else {
                #pragma unroll
                for (int c2 = 0; c2 < CP; ++c2) bv[c2] = __ldg(reinterpret_cast<const float2*>(brow) + c2);
            }
        } else {
            #pragma unroll
            for (int c2 = 0; c2 < CP; ++c2) {
                const int x = x0 + 2 * c2;
                const bool rv = i < Hv;
                bv[c2] = make_float2((rv && x < Wv) ? __ldg(brow + 2 * c2) : 0.f,
                                     (rv && x + 1 < Wv) ? __ldg(brow + 2 * c2 + 1) : 0.f);
            }
        }
        #pragma unroll
        for (int c2 = 0; c2 < CP; ++c2) {
            if constexpr (!BSM) breg[k][c2] = bv[c2];
            r[k][c2] = f2s(0.5f); s[k][c2] = f2s(0.5f); p[k][c2] = f2s(0.5f); q[k][c2] = f2s(0.5f);
        }
        if constexpr (BSM) row_st<CP>(bs + k * ROW, lane, bv);
    }
    // FISTA state for the epilogue: asynchronous copies into shared memory now,
    // consumed after the FGP loop (each lane reads back only its own columns)
    float* xin = sm + (BSM ? SM::total_bsm : SM::total) + (PERSIST ? (tcount & 1) * SM::xin_floats : 0) +
                 (w * FR) * 2 * ROW;
    const bool vec_p = CP % 2 == 0 ? ((vc0 | A.T) & 3) == 0 : ((vc0 | A.T) & 1) == 0;
    if (MODE == 1 && !(PERSIST && tcount > 0)) {
        #pragma unroll
        for (int k = 0; k < FR; ++k) {
            const int i = i0 + k;
            if (i >= Hv) continue;
            const long long prow = (long long)tile * A.p_tstride + (long long)(vr0 + i) * A.T + vc0 + x0;
            float* dx = xin + k * 2 * ROW + x0;
            cp_async_cols<CP>(dx, A.xprev + prow, x0, Wv, vec_p);
            cp_async_cols<CP>(dx + ROW, A.xs + prow, x0, Wv, vec_p);
        }
    }
    const float lam = A.lams ? __ldg(A.lams + tile) : A.lam;
    const float lam2 = 2.f * lam;               // L(p, q) = 2 L(p', q')
    const float gam = lam > 0.f ? 1.f / (16.f * lam) : 0.f;
    // q step per column (0 where q does not exist: j >= W_v - 1)
    float gq[NC];
    #pragma unroll
    for (int c = 0; c < NC; ++c) gq[c] = (x0 + c < Wv - 1) ? gam : 0.f;
    float2 gq2[CP];
    #pragma unroll
    for (int c2 = 0; c2 < CP; ++c2) gq2[c2] = make_float2(gq[2 * c2], gq[2 * c2 + 1]);
    cl.sync();
    if constexpr (PERSIST) {   // the cluster's next tile: b, x_prev, x_s into shared memory now
        const int tn = tile + (int)gridDim.y;
        if (tn < tile_end) {
            int nvr0 = 0, nvc0 = 0, nHv = A.H, nWv = A.W;
            if (A.tiles) {
                const TileT tn_ = A.tiles[tn];
                nvr0 = tn_.vr0; nvc0 = tn_.vc0; nHv = tn_.vr1 - tn_.vr0; nWv = tn_.vc1 - tn_.vc0;
            }
            const float* nb = A.b + (long long)tn * A.b_tstride + (long long)nvr0 * A.b_pitch + nvc0;
            const bool nvec_b = ((reinterpret_cast<uintptr_t>(nb) | ((uintptr_t)A.b_pitch << 2)) & VAL) == 0;
            float* nxin = sm + SM::total + ((tcount + 1) & 1) * SM::xin_floats + (w * FR) * 2 * ROW;
            const bool nvec_p = CP % 2 == 0 ? ((nvc0 | A.T) & 3) == 0 : ((nvc0 | A.T) & 1) == 0;
            #pragma unroll
            for (int k = 0; k < FR; ++k) {
                const int i = i0 + k;
                float* db = bnext + k * ROW + x0;
                const float* brow = nb + (long long)i * A.b_pitch + x0;
                if (i < nHv) {
                    cp_async_cols<CP>(db, brow, x0, nWv, nvec_b);
                    #pragma unroll
                    for (int c = 0; c < NC; ++c)
                        if (x0 + c >= nWv) db[c] = 0.f;
                } else {
                    #pragma unroll
                    for (int c = 0; c < NC; ++c) db[c] = 0.f;
                }
                if (MODE == 1 && i < nHv) {
                    const long long prow = (long long)tn * A.p_tstride + (long long)(nvr0 + i) * A.T + nvc0 + x0;
                    float* dx = nxin + k * 2 * ROW + x0;
                    cp_async_cols<CP>(dx, A.xprev + prow, x0, nWv, nvec_p);
                    cp_async_cols<CP>(dx + ROW, A.xs + prow, x0, nWv, nvec_p);
                }
            }
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
    }
    const unsigned up_rank = has_up ? kr - 1 : kr, dn_rank = has_dn ? kr + 1 : kr;
    constexpr unsigned RB = ROW * 4u;                  // bytes per staged row
    constexpr unsigned PS = (NW + 1) * RB;             // bytes per parity of hr / hz
    const unsigned s_hr = smem_u32(sm + SM::hr), s_hz = smem_u32(sm + SM::hz);
    // this warp's halo slots: r from above, z from below (read); r / z it publishes (written)
    const unsigned up_slot = keep_u32<CP != 4 || FGP_KEEP4 >= 2>(s_hr + w * RB), dn_slot = keep_u32<CP != 4 || FGP_KEEP4 >= 2>(s_hz + (w + 1) * RB);
    const unsigned rem_rx_r = mapa(s_hr, dn_rank);                 // my last warp's r row -> slot 0 of the CTA below
    const unsigned rem_bar_r = mapa(smem_u32(bars + 0), dn_rank);
    const unsigned rem_rx_z = mapa(s_hz + NW * RB, up_rank);       // my first warp's z row -> slot NW of the CTA above
    const unsigned rem_bar_z = mapa(smem_u32(bars + 2), up_rank);
    const unsigned my_r_slot = keep_u32<CP != 4 || FGP_KEEP4 >= 2>(s_hr + (w + 1) * RB), my_z_slot = keep_u32<CP != 4 || FGP_KEEP4 >= 2>(s_hz + w * RB);
    constexpr unsigned row_bytes = ROW * 4;
    const int nit = lam > 0.f ? A.nfgp : 0;
    const unsigned bar0 = keep_u32<CP != 4 || FGP_KEEP4 >= 1>(smem_u32(bars));
    const float2 nl2 = f2s(-lam2);
    // p step per row of this warp (0 where p does not exist: i >= H_v - 1)
    float gp[FR];
    #pragma unroll
    for (int k = 0; k < FR; ++k) gp[k] = (i0 + k < Hv - 1) ? gam : 0.f;

    // Two CTA barriers per iteration (one after each phase); the rows that read
    // a halo are computed last in their phase, so the halo's DSMEM transfer and
    // the neighbour warps' work overlap the interior rows.  Parity cb is
    // compile-time, so every halo address is loop invariant.
    auto fgp_iter = [&](int it, auto cbv) {
        const int cb = cbv, pb = cb ^ 1;
        if (lane == 0) {   // the consuming warp arms its DSMEM receive buffers
            if (w == NW - 1 && has_dn) mbar_expect_tx(bar0 + 16 + 8 * cb, row_bytes);   // z row of it, from below
            if (w == 0 && has_up) mbar_expect_tx(bar0 + 8 * cb, row_bytes);             // r row of it, from above
        }
        // ---- phase A: z = b - lam2 L(r, s); halo row 0 last: 1, ..., FR-1, 0
        #pragma unroll
        for (int kk = 0; kk < FR; ++kk) {
            const int k = (kk + 1) % FR;
            float2 rup[CP];
            if (k > 0) {
                #pragma unroll
                for (int c2 = 0; c2 < CP; ++c2) rup[c2] = r[k - 1][c2];
            } else {
                // slot of parity pb: written in iteration it - 1 (still 1/2 at it = 0)
                if (w == 0 && has_up && it > 0) mbar_wait(bar0 + 8 * pb, ((it - 1) >> 1) & 1);
                row_ld_s<CP>(up_slot + pb * PS, lane, rup);
            }
            float sl = __shfl_up_sync(0xffffffffu, s[k][CP - 1].y, 1);
            if (lane == 0) sl = 0.5f;
            // z = b - lam2 (r - rup) - lam2 s + lam2 s_left
            float2 t[CP], bk[CP];
            bget(k, bk);
            #pragma unroll
            for (int c2 = 0; c2 < CP; ++c2) {
                t[c2] = f2fma(nl2, f2sub(r[k][c2], rup[c2]), bk[c2]);
                t[c2] = f2fma(nl2, s[k][c2], t[c2]);
            }
            z[k][0].x = fmaf(lam2, sl, t[0].x);
            z[k][0].y = fmaf(lam2, s[k][0].x, t[0].y);
            #pragma unroll
            for (int c2 = 1; c2 < CP; ++c2) {
                z[k][c2].x = fmaf(lam2, s[k][c2 - 1].y, t[c2].x);
                z[k][c2].y = fmaf(lam2, s[k][c2].x, t[c2].y);
            }
            if (k == 0) {
                if (w == 0 && has_up) row_push<CP>(rem_rx_z + cb * PS, lane, z[0], rem_bar_z + cb * 8);
                if (w > 0) row_st_s<CP>(my_z_slot + cb * PS, lane, z[0]);
            }
        }
        __syncthreads();
        // ---- phase B: dual ascent, projection on [0, 1] (shifted), FGP momentum;
        // halo row FR-1 last: 0, ..., FR-1
        const float beta = c_fgp_beta[it];
        const float2 beta2 = f2s(beta);
        #pragma unroll
        for (int k = 0; k < FR; ++k) {
            float2 zb[CP];
            if (k < FR - 1) {
                #pragma unroll
                for (int c2 = 0; c2 < CP; ++c2) zb[c2] = z[k + 1][c2];
            } else {
                if (w == NW - 1 && has_dn) mbar_wait(bar0 + 16 + 8 * cb, (it >> 1) & 1);
                row_ld_s<CP>(dn_slot + cb * PS, lane, zb);
            }
            const float zr = __shfl_down_sync(0xffffffffu, z[k][0].x, 1);   // lane 31: masked by gq
            const float gpk = gp[k];
            const float2 gp2 = f2s(gpk);
            #pragma unroll
            for (int c2 = 0; c2 < CP; ++c2) {
                // p' = sat(r + g (z - z_below)), q' = sat(s + g (z - z_right))
                const float2 tp = f2fma(gp2, z[k][c2], r[k][c2]);
                const float2 tq = f2fma(gq2[c2], z[k][c2], s[k][c2]);
                const float zrx = z[k][c2].y;
                const float zry = c2 < CP - 1 ? z[k][c2 + 1].x : zr;
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
                if (w == NW - 1 && has_dn) row_push<CP>(rem_rx_r + cb * PS, lane, r[FR - 1], rem_bar_r + cb * 8);
                if (w < NW - 1) row_st_s<CP>(my_r_slot + cb * PS, lane, r[FR - 1]);
            }
        }
        __syncthreads();
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
    row_st<CP>(hp + w * ROW, lane, p[FR - 1]);
    cl.sync();
    float2 pup0[CP];
    if (w > 0) row_ld<CP>(hp + (w - 1) * ROW, lane, pup0);
    else if (has_up) row_ld<CP>(cl.map_shared_rank(hp, kr - 1) + (NW - 1) * ROW, lane, pup0);
    else {
        #pragma unroll
        for (int c2 = 0; c2 < CP; ++c2) pup0[c2] = f2s(0.5f);
    }
    // the neighbour's halo row has been read: arrive now, wait at exit (keeps
    // shared memory alive until every neighbour has read its halo)
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
    if constexpr (MODE == 1) cp_async_commit_wait_all();
    const bool vec_y = CP % 2 == 0 ? (vc0 & 3) == 0 : (vc0 & 1) == 0;   // y rows: PADL + vc0 + x0, TP % 4 == 0
    const bool vec_yT = FR == 4 && (vr0 & 3) == 0;      // yT columns: PADL + vr0 + i0 + k
    float xall[FR][NC];
    #pragma unroll
    for (int k = 0; k < FR; ++k) {
        const int i = i0 + k;
        float ql = __shfl_up_sync(0xffffffffu, q[k][CP - 1].y, 1);
        if (lane == 0) ql = 0.5f;
        float2 bk[CP];
        bget(k, bk);
        #pragma unroll
        for (int c2 = 0; c2 < CP; ++c2) {
            const float2 pu = k > 0 ? p[k - 1][c2] : pup0[c2];
            const float qlx = c2 > 0 ? q[k][c2 - 1].y : ql;
            xall[k][2 * c2] = bk[c2].x - lam2 * (p[k][c2].x + q[k][c2].x - pu.x - qlx);
            xall[k][2 * c2 + 1] = bk[c2].y - lam2 * (p[k][c2].y + q[k][c2].y - pu.y - q[k][c2].x);
        }
        if (i >= Hv) continue;
        if constexpr (MODE == 0) {
            #pragma unroll
            for (int c = 0; c < NC; ++c)
                if (x0 + c < Wv) A.out[(long long)tile * A.out_tstride + (long long)i * A.out_pitch + x0 + c] = xall[k][c];
        } else {
            const int ti_ = vr0 + i;
            const long long prow = (long long)tile * A.p_tstride + (long long)ti_ * A.T + vc0 + x0;
            float* yrow = A.y + (long long)tile * A.y_tstride + (long long)ti_ * A.TP + PADL + vc0 + x0;
            const float* sx = xin + k * 2 * ROW + x0;
            float xp[NC], xsv[NC];
            #pragma unroll
            for (int c2 = 0; c2 < CP; ++c2) {
                const float2 a = *reinterpret_cast<const float2*>(sx + 2 * c2);
                const float2 b = *reinterpret_cast<const float2*>(sx + ROW + 2 * c2);
                xp[2 * c2] = a.x; xp[2 * c2 + 1] = a.y; xsv[2 * c2] = b.x; xsv[2 * c2 + 1] = b.y;
            }
            float yv[NC];
            #pragma unroll
            for (int c = 0; c < NC; ++c) {
                const float x = xall[k][c];
                const float rr = x + A.beta_o * (x - xp[c]);          // FISTA extrapolation (A12)
                yv[c] = rr - xsv[c];                                  // x_L^k = r - x_s^k
            }
            st_cols<CP>(A.xprev + prow, xall[k], x0, Wv, vec_p);
            st_cols<CP>(yrow, yv, x0, Wv, vec_y);
            if (vec_yT) {
                // the warp's FR = 4 rows are consecutive: the transposed copy of
                // column c is one 16-byte store per lane, written after the last row
                #pragma unroll
                for (int c = 0; c < NC; ++c) xall[k][c] = yv[c];
            } else {
                float* ycol = A.yT + (long long)tile * A.y_tstride + (long long)(vc0 + x0) * A.TP + PADL + ti_;
                #pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (x0 + c < Wv) ycol[(long long)c * A.TP] = yv[c];
            }
        }
    }
    if constexpr (MODE == 1) {
        if (vec_yT && i0 < Hv) {
            float* ycol = A.yT + (long long)tile * A.y_tstride + (long long)(vc0 + x0) * A.TP + PADL + vr0 + i0;
            if (i0 + 3 < Hv) {
                #pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (x0 + c < Wv)
                        *reinterpret_cast<float4*>(ycol + (long long)c * A.TP) =
                            make_float4(xall[0][c], xall[FR > 1 ? 1 : 0][c], xall[FR > 2 ? 2 : 0][c], xall[FR > 3 ? 3 : 0][c]);
            } else {
                #pragma unroll
                for (int c = 0; c < NC; ++c)
                    #pragma unroll
                    for (int k = 0; k < FR; ++k)
                        if (x0 + c < Wv && i0 + k < Hv) ycol[(long long)c * A.TP + k] = xall[k][c];
            }
        }
    }
    asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
    }   // tile loop
}

}  // namespace lt
