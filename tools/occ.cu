// occ.cu — cluster occupancy of the fused kernels (measurement tool):
// cudaOccupancyMaxActiveClusters for the launch shapes engine.cu uses.
#include <cstdio>
#include <cstdlib>
#include "kernels_pc.cuh"
using namespace plbm;

template <class K>
void report(const char* name, K kern, int nt, int smem, int cl) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (getenv("CARVEOUT")) cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, atoi(getenv("CARVEOUT")));
    if (cl > 8) cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cl * 1000);
    cfg.blockDim = dim3(nt);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg);
    int blocks = -1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kern, nt, smem);
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, kern);
    printf("  regs %d static smem %zu max dyn %d\n", fa.numRegs, fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes);
    printf("%-28s cluster %2d: max active clusters %4d (= %4d CTAs; %d CTAs/SM x 148 = %d)  %s\n", name, cl, n,
           n * cl, blocks, blocks * 148, cudaGetErrorString(e));
}

int main() {
    {   // the half-tile kernel at cluster sizes 2 / 4 / 8 (what quarter / half / whole tiles would pack)
        auto kh = k_main_pc<32, 2, 1, 256, true, false, AA_OFF, 2>;
        for (int cl : {1, 2, 4, 8}) report("k_main_pc<32,2,NH=2> as", kh, 256, PcCfg<32, 2, 1, 256, 2>::SMEM, cl);
    }
    report("k_main_pc<32,2,1>", k_main_pc<32, 2, 1, 256>, 256, PcCfg<32, 2, 1>::SMEM, PcCfg<32, 2, 1>::CL);
    report("k_main_pc<32,1,1>", k_main_pc<32, 1, 1, 256>, 256, PcCfg<32, 1, 1>::SMEM, PcCfg<32, 1, 1>::CL);
    report("k_main_pc<32,3,1>", k_main_pc<32, 3, 1, 256>, 256, PcCfg<32, 3, 1>::SMEM, PcCfg<32, 3, 1>::CL);
    report("k_main_pc<16,2,1>", k_main_pc<16, 2, 1, 256>, 256, PcCfg<16, 2, 1>::SMEM, PcCfg<16, 2, 1>::CL);
    return 0;
}
