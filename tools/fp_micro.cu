// FP32 pipe microbenchmark (sm_100a): issue rate of FFMA, FFMA.SAT, FFMA2,
// FADD2 and mixes, for W warps per SM sub-partition.  Diagnostic for k_fgp2.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int NCH = 8;       // independent chains per thread
constexpr int IT = 16384;
template <int KIND>
__global__ void kern(float* out, long long* cyc, float a, float b) {
    float2 x[NCH];
    float y[NCH];
    for (int c = 0; c < NCH; ++c) { x[c % NCH] = make_float2(threadIdx.x * 1e-3f + c, c * 0.5f); y[c % NCH] = c * 0.25f + threadIdx.x * 1e-3f; }
    const float2 a2 = make_float2(a, a), b2 = make_float2(b, b);
    long long t0 = clock64();
    #pragma unroll 1
    for (int i = 0; i < IT; ++i) {
        #pragma unroll
        for (int c = 0; c < 4 * NCH; ++c) {
            if (KIND == 0) { y[c % NCH] = fmaf(y[c % NCH], a, b); }                               // FFMA
            if (KIND == 1) { y[c % NCH] = __saturatef(fmaf(y[c % NCH], a, b)); }                  // FFMA.SAT
            if (KIND == 2) { x[c % NCH] = __ffma2_rn(x[c % NCH], a2, b2); }                       // FFMA2
            if (KIND == 3) { x[c % NCH] = __fadd2_rn(x[c % NCH], b2); }                           // FADD2
            if (KIND == 4) { x[c % NCH] = __ffma2_rn(x[c % NCH], a2, b2); y[c % NCH] = __saturatef(fmaf(y[c % NCH], a, b)); }   // mix 1:1
            if (KIND == 5) { y[c % NCH] = fmaxf(y[c % NCH] * a, b); }                             // FMUL + FMNMX
            if (KIND == 6) { unsigned u = __float_as_uint(y[c % NCH]); u = (u ^ 0x1234u) + (unsigned)c; y[c % NCH] = __uint_as_float(u); }   // LOP3 + IADD3 (-> IADD3/LOP3)
            if (KIND == 7) { unsigned u = __float_as_uint(y[c % NCH]); u = (u >> 3) + (u << 5); y[c % NCH] = __uint_as_float(u); }   // SHF + LEA
            if (KIND == 8) { unsigned u = __float_as_uint(y[c % NCH]); u = (u & 0x7FFFFFu) | 0x3F800000u; y[c % NCH] = __saturatef(fmaf(__uint_as_float(u + 0x100u), a, b)); }   // LOP3 + IADD + FFMA.SAT
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    float s = 0.f;
    for (int c = 0; c < NCH; ++c) s += x[c].x + x[c].y + y[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int KIND>
void run(const char* name, float* d, long long* dc, int nsm) {
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int w : {1, 2, 4, 8}) {
        const int threads = 128 * w;      // w warps per SMSP
        for (int r = 0; r < 3; ++r) kern<KIND><<<nsm, threads>>>(d, dc, 0.999f, 0.001f);
        cudaEventRecord(e0);
        kern<KIND><<<nsm, threads>>>(d, dc, 0.999f, 0.001f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
        long long hc[1024]; cudaMemcpy(hc, dc, nsm * sizeof(long long), cudaMemcpyDeviceToHost);
        double cyc = 0; for (int i = 0; i < nsm; ++i) cyc += hc[i]; cyc /= nsm;
        const double ninst = (double)IT * 4 * NCH * (KIND == 4 ? 2 : KIND == 5 ? 2 : KIND >= 6 ? 2 : 1) * w;   // per SMSP (warp-instr)
        printf("%-10s warps/SMSP=%d: %.3f ms, %.0f cyc (%.0f MHz), %.3f warp-inst/clk/SMSP\n", name, w, ms, cyc, cyc / (ms * 1e3), ninst / cyc);
    }
}
int main() {
    int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* d; cudaMalloc(&d, nsm * 1024 * sizeof(float)); long long* dc; cudaMalloc(&dc, 1024 * sizeof(long long));
    run<0>("FFMA", d, dc, nsm); run<1>("FFMA.SAT", d, dc, nsm); run<2>("FFMA2", d, dc, nsm);
    run<3>("FADD2", d, dc, nsm); run<4>("FFMA2+SAT", d, dc, nsm); run<5>("FMUL+FMNMX", d, dc, nsm);
    run<6>("LOP3+IADD", d, dc, nsm); run<7>("SHF+LEA", d, dc, nsm); run<8>("LOP+ADD+SAT", d, dc, nsm);
    return 0;
}
