// Microbenchmark: warp-shuffle vs shared-memory load throughput per SM (B200).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_shfl(float* out, int iters) {
    float a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
    for (int i = 0; i < iters; ++i) {
        a += __shfl_down_sync(0xffffffffu, a, 1);
        b += __shfl_down_sync(0xffffffffu, b, 1);
        c += __shfl_down_sync(0xffffffffu, c, 1);
        d += __shfl_down_sync(0xffffffffu, d, 1);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_lds(float* out, int iters) {
    __shared__ float s[1024];
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) s[e] = e;
    __syncthreads();
    float a = 0, b = 0, c = 0, d = 0;
    int i0 = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) {
        a += s[(i0 + i) & 1023];
        b += s[(i0 + i + 32) & 1023];
        c += s[(i0 + i + 64) & 1023];
        d += s[(i0 + i + 96) & 1023];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
__global__ void k_lds64(float* out, int iters) {
    __shared__ float2 s[1024];
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) s[e] = make_float2(e, e);
    __syncthreads();
    float a = 0, b = 0, c = 0, d = 0;
    int i0 = threadIdx.x & 31;
    for (int i = 0; i < iters; ++i) {
        float2 x = s[(i0 + i) & 1023], y = s[(i0 + i + 32) & 1023];
        a += x.x; b += x.y; c += y.x; d += y.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a + b + c + d;
}
int main() {
    float* o; cudaMalloc(&o, 148 * 8 * 256 * 4);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 14;
    for (int k = 0; k < 3; ++k) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (k == 0) k_shfl<<<148 * 8, 256>>>(o, iters);
            if (k == 1) k_lds<<<148 * 8, 256>>>(o, iters);
            if (k == 2) k_lds64<<<148 * 8, 256>>>(o, iters);
            cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            const double warp_ops = 148.0 * 8 * 8 * iters * (k == 2 ? 2 : 4);
            if (rep) printf("%s: %.3f ms, %.2f warp-ops per SM per ns -> %.2f per SM-clock @1.965GHz\n",
                            k == 0 ? "SHFL" : k == 1 ? "LDS.32" : "LDS.64", ms, warp_ops / 148 / (ms * 1e6),
                            warp_ops / 148 / (ms * 1e6) / 1.965);
        }
    }
    return 0;
}
