/* c_api_demo.c -- the C-ABI (include/loctomo.h) used from plain C, no Python:
 * plan a batch of local reconstructions, bind a cudaMalloc'ed workspace,
 * compute the filter bank (Alg. 1), run the local nonneg SIRT
 * (Alg. 2) on a sinogram read from a raw float32 file, combine the
 * cores into one image (lt_combine_rois; one rank, no
 * communicator) and write it as raw float32.
 *
 * Build: gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_demo.c \
 *          paper_1604_02292_b200/_loctomo.so -L /usr/local/cuda/lib64 -lcudart \
 *          -Wl,-rpath,/usr/local/cuda/lib64 -Wl,-rpath,$PWD/paper_1604_02292_b200 -o c_api_demo
 * Run:   ./c_api_demo N N_theta N_d radius margin n_iter sino.f32 image.f32 row col [row col ...]
 *        (angles theta_a = a pi / N_theta; exit code 0 on success)
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime.h>

#include "loctomo.h"

#define CHECK_LT(call)                                                              \
    do {                                                                            \
        int rc_ = (call);                                                           \
        if (rc_ != LT_OK) {                                                         \
            fprintf(stderr, "%s failed (%d): %s\n", #call, rc_, lt_last_error());   \
            return 1;                                                               \
        }                                                                           \
    } while (0)
#define CHECK_CUDA(call)                                                            \
    do {                                                                            \
        cudaError_t e_ = (call);                                                    \
        if (e_ != cudaSuccess) {                                                    \
            fprintf(stderr, "%s: %s\n", #call, cudaGetErrorString(e_));             \
            return 1;                                                               \
        }                                                                           \
    } while (0)

int main(int argc, char** argv) {
    if (argc < 11 || (argc - 9) % 2) {
        fprintf(stderr, "usage: %s N N_theta N_d radius margin n_iter sino.f32 image.f32 row col [row col ...]\n", argv[0]);
        return 2;
    }
    const int n = atoi(argv[1]), na = atoi(argv[2]), nd = atoi(argv[3]);
    const int radius = atoi(argv[4]), margin = atoi(argv[5]), n_iter = atoi(argv[6]);
    const int n_roi = (argc - 9) / 2;
    double* angles = (double*)malloc(sizeof(double) * na);
    int32_t* rows = (int32_t*)malloc(sizeof(int32_t) * n_roi);
    int32_t* cols = (int32_t*)malloc(sizeof(int32_t) * n_roi);
    for (int a = 0; a < na; ++a) angles[a] = a * M_PI / na;
    for (int q = 0; q < n_roi; ++q) { rows[q] = atoi(argv[9 + 2 * q]); cols[q] = atoi(argv[10 + 2 * q]); }

    float* h_sino = (float*)malloc(sizeof(float) * (size_t)na * nd);
    FILE* f = fopen(argv[7], "rb");
    if (!f || fread(h_sino, sizeof(float), (size_t)na * nd, f) != (size_t)na * nd) { fprintf(stderr, "bad sinogram\n"); return 1; }
    fclose(f);

    lt_plan* plan = NULL;
    CHECK_LT(lt_roi_setup(n, na, nd, angles, n_roi, rows, cols, radius, margin, n_iter, LT_DISC_ON, 0, 1, &plan));
    const int64_t ws_bytes = lt_plan_workspace_bytes(plan);
    void* d_ws = NULL;
    CHECK_CUDA(cudaMalloc(&d_ws, (size_t)ws_bytes));                 /* 256-byte aligned */
    cudaStream_t st;
    CHECK_CUDA(cudaStreamCreate(&st));
    CHECK_LT(lt_plan_bind_workspace(plan, d_ws, ws_bytes, st));
    CHECK_LT(lt_filter_bank(plan, st));

    const int R = lt_plan_local_count(plan), side = 2 * radius;
    float *d_sino = NULL, *d_cores = NULL, *d_image = NULL;
    CHECK_CUDA(cudaMalloc((void**)&d_sino, sizeof(float) * (size_t)na * nd));
    CHECK_CUDA(cudaMalloc((void**)&d_cores, sizeof(float) * (size_t)(R > 0 ? R : 1) * side * side));
    CHECK_CUDA(cudaMalloc((void**)&d_image, sizeof(float) * (size_t)n * n));
    CHECK_CUDA(cudaMemcpyAsync(d_sino, h_sino, sizeof(float) * (size_t)na * nd, cudaMemcpyHostToDevice, st));
    CHECK_LT(lt_sirt_solve(plan, d_sino, 0.0f, INFINITY, d_cores, st));
    CHECK_LT(lt_combine_rois(plan, d_cores, d_image, NULL, st));

    float* h_image = (float*)malloc(sizeof(float) * (size_t)n * n);
    CHECK_CUDA(cudaMemcpyAsync(h_image, d_image, sizeof(float) * (size_t)n * n, cudaMemcpyDeviceToHost, st));
    CHECK_CUDA(cudaStreamSynchronize(st));
    f = fopen(argv[8], "wb");
    if (!f || fwrite(h_image, sizeof(float), (size_t)n * n, f) != (size_t)n * n) { fprintf(stderr, "cannot write image\n"); return 1; }
    fclose(f);
    printf("c_api_demo: %d ROIs, %lld workspace bytes, %lld kernels launched\n", R, (long long)ws_bytes,
           (long long)lt_launch_count());

    lt_plan_destroy(plan);
    cudaFree(d_ws); cudaFree(d_sino); cudaFree(d_cores); cudaFree(d_image);
    cudaStreamDestroy(st);
    free(angles); free(rows); free(cols); free(h_sino); free(h_image);
    return 0;
}
