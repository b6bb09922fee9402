// Is a 32x32->64 IMAD.WIDE (no accumulate) cheaper than IMAD.HI for the high word? (B200: no)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o wide wide.cu && ./wide
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#define CH 8
__device__ __forceinline__ uint32_t hi_wide_ptx(uint32_t a, uint32_t b) {
  uint64_t r;
  asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
  return (uint32_t)(r >> 32);
}
__device__ __forceinline__ uint32_t hi_wide_ptx2(uint32_t a, uint32_t b) {
  uint32_t lo, hi;
  asm volatile("{ .reg .u64 t; mul.wide.u32 t, %2, %3; mov.b64 {%0, %1}, t; }" : "=r"(lo), "=r"(hi) : "r"(a), "r"(b));
  return hi;
}
template <int K>
__global__ void k(uint64_t* out, int iters, uint32_t b) {
  uint32_t a = threadIdx.x * 2654435761u;
  uint32_t c[CH];
  uint64_t w[CH];
  for (int i = 0; i < CH; ++i) c[i] = a + i, w[i] = a ^ i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (K == 0) c[i] = __umulhi(c[i], b) + a;                          // IMAD.HI
      if (K == 1) c[i] = hi_wide_ptx(c[i], b) + a;                       // mul.wide asm volatile
      if (K == 2) c[i] = hi_wide_ptx2(c[i], b) + a;
      if (K == 3) { uint64_t r = (uint64_t)c[i] * b; c[i] = (uint32_t)r ^ (uint32_t)(r >> 32); }  // wide, both halves
      if (K == 4) w[i] += (uint64_t)(uint32_t)w[i] * b;                   // wide + 64-bit acc
      if (K == 5) { uint64_t r = (uint64_t)(uint32_t)w[i] * b; w[i] = r + (w[i] >> 7); }  // wide noacc + separate add?
      if (K == 6) c[i] = c[i] * b + a;                                   // IMAD
    }
  uint64_t s = 0;
  for (int i = 0; i < CH; ++i) s += c[i] + w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename F>
void run(const char* name, F kern, uint64_t* buf) {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  kern<<<blocks, threads>>>(buf, 16, 0x9E3779B9u);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(buf, iters, 0x9E3779B9u);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms = 0; cudaEventElapsedTime(&ms, e0, e1);
  const double thr_iters = (double)blocks * threads * iters;
  const double clks = ms * 1e-3 * clk * 1e3;
  printf("%-26s %8.3f ms  warp-clk per op per SMSP %.2f\n", name, ms, clks * sms * 4 / (thr_iters * CH / 32));
}
int main() {
  uint64_t* buf; cudaMalloc(&buf, 148 * 8 * 256 * 8);
  run("imad.hi", k<0>, buf);
  run("mul.wide asm hi", k<1>, buf);
  run("mul.wide asm2 hi", k<2>, buf);
  run("wide both halves", k<3>, buf);
  run("wide + acc", k<4>, buf);
  run("wide noacc + shr-add", k<5>, buf);
  run("imad", k<6>, buf);
  return 0;
}
