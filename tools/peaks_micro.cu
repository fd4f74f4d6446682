// peaks_micro.cu -- measured SM-side ceilings for the roofline of the path's
// kernels ("measure the SMEM crossbar and FFMA peaks on the box"):
//   * shared-memory crossbar: conflict-free LDS.64 / LDS.128 streams (every warp
//     reads 32 consecutive 8- / 16-byte entries: 2 / 4 wavefronts of 128 B),
//     bytes delivered per second over all SMs;
//   * FP32 pipe: FFMA (scalar) and FFMA2 (paired) with 8 independent chains per
//     thread, 2 flops per lane-FMA, over all SMs.
// Each kernel runs on every SM with 2048 threads per SM, timed by CUDA events
// (best of 5 after a warm-up).  Prints one JSON object.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/peaks_micro tools/peaks_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ long long g_cycles;

template <int VEC>
__global__ void __launch_bounds__(256) k_lds(float* out, int iters) {
    __shared__ __align__(16) float buf[8192];        // 32 KB
    for (int e = threadIdx.x; e < 8192; e += blockDim.x) buf[e] = (float)e * 1e-6f;
    __syncthreads();
    const long long c0 = clock64();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // warp w streams rows of 32 entries of VEC floats (conflict-free), 8 rows per iteration
    const unsigned base = (unsigned)__cvta_generic_to_shared(buf) + (unsigned)(lane * VEC * 4);
    const unsigned rowb = 32u * VEC * 4;                          // bytes per row
    const unsigned nrows = 8192u * 4u / rowb;                     // rows in the buffer
    float2 acc[8];
    #pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = make_float2(0.f, 0.f);
    unsigned row = (unsigned)warp;
    for (int i = 0; i < iters; ++i) {
        const unsigned a = base + (row % (nrows - 8)) * rowb;
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (VEC == 2) {
                float2 v;
                asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a + u * rowb));
                acc[u] = __fadd2_rn(acc[u], v);
            } else {
                float4 v;
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                             : "r"(a + u * rowb));
                acc[u] = __fadd2_rn(acc[u], __fadd2_rn(make_float2(v.x, v.y), make_float2(v.z, v.w)));
            }
        }
        row += 8;
    }
    float s = 0.f;
    #pragma unroll
    for (int u = 0; u < 8; ++u) s += acc[u].x + acc[u].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) g_cycles = clock64() - c0;
}

template <bool PAIRED>
__global__ void __launch_bounds__(256) k_ffma(float* out, int iters, float b, float c) {
    const long long c0 = clock64();
    float2 a[8];
    #pragma unroll
    for (int u = 0; u < 8; ++u) a[u] = make_float2(threadIdx.x * 1e-3f + u, u * 0.5f);
    const float2 b2 = make_float2(b, b), c2 = make_float2(c, c);
    for (int i = 0; i < iters; ++i) {
        #pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (PAIRED) {
                a[u] = __ffma2_rn(a[u], b2, c2);
            } else {
                a[u].x = fmaf(a[u].x, b, c);
                a[u].y = fmaf(a[u].y, b, c);
            }
        }
    }
    float s = 0.f;
    #pragma unroll
    for (int u = 0; u < 8; ++u) s += a[u].x + a[u].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (blockIdx.x == 0 && threadIdx.x == 0) g_cycles = clock64() - c0;
}

template <class F>
int best_of(F launch, float* best_ms, long long* cycles) {
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    launch();
    CK(cudaDeviceSynchronize());
    *best_ms = 1e30f;
    for (int r = 0; r < 5; ++r) {
        CK(cudaEventRecord(e0));
        launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (ms < *best_ms) { *best_ms = ms; CK(cudaMemcpyFromSymbol(cycles, g_cycles, sizeof(long long))); }
    }
    CK(cudaGetLastError());
    return 0;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int threads = 256;
    // exactly one wave of each kernel (CTA 0's clock64 span = the kernel's)
    int occ_lds = 0, occ_fma = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_lds, k_lds<4>, threads, 0));
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_fma, k_ffma<true>, threads, 0));
    const int ctas_lds = sms * occ_lds, ctas_fma = sms * occ_fma;
    const int ctas = ctas_lds > ctas_fma ? ctas_lds : ctas_fma;
    float* out = nullptr;
    CK(cudaMalloc(&out, (size_t)ctas * threads * sizeof(float)));
    const int it_lds = 1 << 13, it_fma = 1 << 13;
    float ms64, ms128, msf, msf2;
    long long cy64, cy128, cyf, cyf2;
    if (best_of([&] { k_lds<2><<<ctas_lds, threads>>>(out, it_lds); }, &ms64, &cy64)) return 1;
    if (best_of([&] { k_lds<4><<<ctas_lds, threads>>>(out, it_lds); }, &ms128, &cy128)) return 1;
    if (best_of([&] { k_ffma<false><<<ctas_fma, threads>>>(out, it_fma, 0.999f, 1e-4f); }, &msf, &cyf)) return 1;
    if (best_of([&] { k_ffma<true><<<ctas_fma, threads>>>(out, it_fma, 0.999f, 1e-4f); }, &msf2, &cyf2)) return 1;
    const double nl = (double)ctas_lds * threads, nf = (double)ctas_fma * threads;
    const double b64 = nl * it_lds * 8 * 8, b128 = nl * it_lds * 8 * 16;              // bytes delivered
    const double fl = nf * it_fma * 8 * 2 * 2;                                        // 16 lane-FMAs x 2 flops
    // clock: cycles of CTA 0 over the kernel time (CTA 0 spans ~the whole kernel: one wave)
    printf("{\"device_sms\": %d, \"ctas_lds\": %d, \"ctas_fma\": %d, \"threads_per_cta\": %d,\n", sms, ctas_lds,
           ctas_fma, threads);
    // per SM-clock at the B200's 1965 MHz max SM clock (MEASURED_PEAKS.json)
    const double clk = 1965e6 * sms;
    printf(" \"smem_lds64_gbs\": %.1f, \"smem_lds64_B_per_clk_per_sm_at_1965MHz\": %.1f,\n",
           b64 / (ms64 * 1e6), b64 / (ms64 * 1e-3) / clk);
    printf(" \"smem_lds128_gbs\": %.1f, \"smem_lds128_B_per_clk_per_sm_at_1965MHz\": %.1f,\n",
           b128 / (ms128 * 1e6), b128 / (ms128 * 1e-3) / clk);
    printf(" \"ffma_tflops\": %.2f, \"ffma_flops_per_clk_per_sm_at_1965MHz\": %.1f,\n",
           fl / (msf * 1e9), fl / (msf * 1e-3) / clk);
    printf(" \"ffma2_tflops\": %.2f, \"ffma2_flops_per_clk_per_sm_at_1965MHz\": %.1f,\n",
           fl / (msf2 * 1e9), fl / (msf2 * 1e-3) / clk);
    printf(" \"how\": \"tools/peaks_micro.cu: one full wave (occupancy-sized grid) of %d-thread CTAs, best of 5 "
           "(CUDA events); LDS: conflict-free 32-entry rows, 8 independent loads per iteration; FFMA: 8 independent "
           "chains per thread\"}\n", threads);
    return 0;
}
