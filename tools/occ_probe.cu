#include <cstdio>
#include <cuda_runtime.h>
__global__ void __cluster_dims__(2,1,1) __launch_bounds__(256,1) k(float* p){ extern __shared__ float s[]; if (p) p[threadIdx.x] = s[threadIdx.x]; }
int main(){
  for (int smem : {100*1024, 150*1024, 200*1024, 216*1024, 227*1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(148); cfg.blockDim = dim3(256); cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute a[1]; a[0].id = cudaLaunchAttributeClusterDimension; a[0].val.clusterDim.x = 2; a[0].val.clusterDim.y = 1; a[0].val.clusterDim.z = 1;
    cfg.attrs = a; cfg.numAttrs = 1;
    int n = -1; cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
    printf("smem %d KB: max active 2-CTA clusters %d (%s)\n", smem/1024, n, cudaGetErrorString(e));
  }
  int v; cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, 0); printf("SMs %d\n", v);
}
