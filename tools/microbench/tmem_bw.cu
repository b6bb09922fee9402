// TMEM read bandwidth microbenchmark (B200): W warps per CTA, one CTA per SM, each warp
// streams tcgen05.ld.32x32b.x16 from its lane quadrant; prints bytes / SM clock.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_bw tmem_bw.cu && /tmp/tmem_bw
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void bw(int iters, unsigned long long* cyc, uint32_t* sink, int lds_per_wait) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"((uint32_t)__cvta_generic_to_shared(&slot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = slot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(16 * (warp >> 2) % 512);
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t r[16];
    for (int k = 0; k < lds_per_wait; ++k) {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(tmem + (uint32_t)((k * 16 + it * 64) % 448)));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      for (int j = 0; j < 16; ++j) acc += r[j];
    }
  }
  const long long t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) cyc[blockIdx.x * 32 + warp] = (unsigned long long)(t1 - t0);
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(slot), "r"(512) : "memory");
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* cyc;
  uint32_t* sink;
  cudaMalloc(&cyc, nsm * 32 * 8);
  cudaMalloc(&sink, nsm * 1024 * 4);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    bw<<<nsm, warps * 32>>>(iters, cyc, sink, 1);
    cudaDeviceSynchronize();
    unsigned long long h[32 * 256];
    cudaMemcpy(h, cyc, nsm * 32 * 8, cudaMemcpyDeviceToHost);
    unsigned long long mx = 0;
    for (int w = 0; w < warps; ++w) mx = h[w] > mx ? h[w] : mx;
    const double bytes = (double)warps * iters * 32 * 16 * 4;
    printf("warps=%2d  cycles=%llu  TMEM read %.1f B/clk/SM  (%s)\n", warps, mx, bytes / mx,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
