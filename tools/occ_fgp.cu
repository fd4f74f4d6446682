// max active clusters of the k_fgp2 configurations (diagnostic: how many SMs
// a cluster launch can keep busy, given the GPC sizes)
#include "../paper_1604_02292_b200/csrc/kernels.cuh"
#include <cstdio>
using namespace lt;
template <int FR, int NW, bool BSM>
void q(int K) {
    auto kern = k_fgp2<1, FR, NW, BSM>;
    const size_t smem = (size_t)(BSM ? Fgp2Smem<FR, NW>::total_bsm : Fgp2Smem<FR, NW>::total) * sizeof(float);
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(K, 256, 1); cfg.blockDim = dim3(NW * 32, 1, 1); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1]; attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = K; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    printf("FR=%d NW=%d BSM=%d K=%d smem=%zu: max active clusters %d (%s) -> %d CTAs\n", FR, NW, (int)BSM, K, smem, n,
           cudaGetErrorString(e), n * K);
}
int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("%s SMs=%d\n", p.name, p.multiProcessorCount);
    q<4, 8, false>(8);
    q<4, 8, false>(4);
    q<4, 8, false>(2);
    q<2, 8, false>(16);
    q<2, 8, false>(8);
    q<2, 8, true>(16);
    q<2, 8, true>(8);
    q<2, 16, true>(8);
    return 0;
}
