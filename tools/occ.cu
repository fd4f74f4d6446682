// max active clusters for the FGP configurations (diagnostic)
#include "../paper_1604_02292_b200/csrc/kernels.cuh"
#include <cstdio>
using namespace lt;
template <int FR, int NT>
void q(int K, int G, int ntw, size_t smem) {
    auto kern = k_fgp<1, FR, NT>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(K, 256, 1); cfg.blockDim = dim3(ntw, G, 1); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    printf("FR=%d NT=%d K=%d G=%d smem=%zu: max active clusters %d (%s) -> %d SMs\n", FR, NT, K, G, smem, n, cudaGetErrorString(e), n * K);
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("%s SMs=%d\n", p.name, p.multiProcessorCount);
    q<8, 512>(16, 2, 256, 40000);
    q<8, 1024>(8, 4, 256, 130000);
    q<16, 256>(16, 1, 256, 30000);
    q<8, 512>(8, 2, 256, 40000);
    q<8, 512>(4, 2, 256, 40000);
    q<8, 512>(2, 2, 256, 40000);
    return 0;
}
