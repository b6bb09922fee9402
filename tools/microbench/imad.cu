// Integer-multiply pipe costs on B200 (fmaheavy) and whether the FP64 pipe overlaps them.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o imad imad.cu && ./imad
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
template <int K>
__global__ void k_int(uint64_t* out, int iters, uint32_t b) {
  uint32_t a = threadIdx.x * 2654435761u;
  uint32_t c[CH];
  uint64_t w[CH];
  for (int i = 0; i < CH; ++i) c[i] = a + i, w[i] = a ^ i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (K == 0) c[i] = c[i] * b + a;                         // IMAD
      if (K == 1) c[i] = __umulhi(c[i], b) + a;                // IMAD.HI
      if (K == 2) w[i] += (uint64_t)(uint32_t)w[i] * b;        // IMAD.WIDE.U32 + 64-bit acc
      if (K == 3) w[i] = (uint64_t)((uint32_t)w[i] ^ a) * b;   // IMAD.WIDE.U32 (no acc) + LOP
      if (K == 4) c[i] = c[i] * b + (c[i] >> 3);               // IMAD + SHF (alu)
    }
  uint64_t s = 0;
  for (int i = 0; i < CH; ++i) s += c[i] + w[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// IMAD.WIDE chains interleaved with independent DFMA chains
template <int ND>
__global__ void k_mix(uint64_t* out, int iters, uint32_t b) {
  uint32_t a = threadIdx.x * 2654435761u;
  uint64_t w[CH];
  double d[CH];
  for (int i = 0; i < CH; ++i) w[i] = a ^ i, d[i] = a * 1e-9 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      w[i] += (uint64_t)(uint32_t)w[i] * b;
#pragma unroll
      for (int j = 0; j < ND; ++j) d[i] = fma(d[i], 1.0000001, 0.5);
    }
  uint64_t s = 0;
  for (int i = 0; i < CH; ++i) s += w[i] + (uint64_t)d[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F>
void run(const char* name, F kern, uint64_t* buf, double ops_per_iter) {
  int sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  kern<<<blocks, threads>>>(buf, 16, 0x9E3779B9u);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(buf, iters, 0x9E3779B9u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double thr_iters = (double)blocks * threads * iters;
  const double clks = ms * 1e-3 * clk * 1e3;
  printf("%-22s %8.3f ms  %7.1f iters(x%d)/clk/SM  -> warp-clk per unit per SMSP %.2f\n", name, ms,
         thr_iters * CH / clks / sms, CH, clks * sms * 4 / (thr_iters * CH / 32) / ops_per_iter);
}

int main() {
  uint64_t* buf;
  cudaMalloc(&buf, 148 * 8 * 256 * 8);
  run("imad", k_int<0>, buf, 1);
  run("imad.hi", k_int<1>, buf, 1);
  run("imad.wide+acc", k_int<2>, buf, 1);
  run("imad.wide(noacc)+lop", k_int<3>, buf, 1);
  run("imad+shf", k_int<4>, buf, 1);
  run("wide + 0 dfma", k_mix<0>, buf, 1);
  run("wide + 1 dfma", k_mix<1>, buf, 1);
  run("wide + 2 dfma", k_mix<2>, buf, 1);
  run("wide + 4 dfma", k_mix<4>, buf, 1);
  return 0;
}
