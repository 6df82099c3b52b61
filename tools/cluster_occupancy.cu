// cluster_occupancy.cu — how many SMs can clusters of 2 / 4 / 8 CTAs (one ~200 KB CTA per SM) occupy
// on this B200?  GPC granularity decides whether a 4-CTA cluster (two cta_group::2 pairs sharing an
// operand by TMA multicast) loses SMs against the 2-CTA pairs the GEMMs use.  Prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/cluster_occupancy tools/cluster_occupancy.cu
#include <cuda_runtime.h>
#include <stdio.h>

__global__ void k(int* p) { if (p) p[blockIdx.x] = 1; }

int main() {
  const int smem = 200 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  printf("{\"sms\": %d", sms);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(cs * 64);
    cfg.blockDim = dim3(320);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int n = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&n, (void*)k, &cfg);
    printf(", \"cluster%d\": {\"max_active_clusters\": %d, \"sms_used\": %d, \"err\": \"%s\"}", cs, n, n * cs,
           cudaGetErrorString(e));
  }
  printf("}\n");
  return 0;
}
