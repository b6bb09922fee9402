// How many clusters of a stage-kernel-shaped launch can be co-resident on this GPU?
// (cudaOccupancyMaxActiveClusters for 3-CTA clusters, 384 threads, 56 registers, 67 KB smem)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -maxrregcount 56 -o cluster_occ cluster_occ.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(384, 3) dummy(float* out) {
  extern __shared__ float sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (out) out[blockIdx.x] = sm[(threadIdx.x + 1) % 384];
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int smem_kb : {60, 67, 72}) {
    for (int csize : {1, 2, 3, 4}) {
      const size_t smem = (size_t)smem_kb * 1024;
      cudaFuncSetAttribute(dummy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaFuncSetAttribute(dummy, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(csize * 1000);
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = csize;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, dummy, &cfg);
      printf("smem %d KB cluster %d: max active clusters %d (%d CTAs; %d SMs x 3 = %d) %s\n", smem_kb, csize, n,
             n * csize, sms, sms * 3, cudaGetErrorString(e));
    }
  }
  return 0;
}
