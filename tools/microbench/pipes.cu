// Pipe-throughput microbenchmark (B200): DFMA vs IMAD.WIDE.U32 vs 64-bit mulhi, per SM per clock.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0000001, c[8];
  for (int i = 0; i < 8; ++i) c[i] = a + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fma(c[i], b, a);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_imadw(uint64_t* out, int iters) {
  uint32_t a = threadIdx.x * 2654435761u, b = 0x9E3779B9u;
  uint64_t c[8];
  for (int i = 0; i < 8; ++i) c[i] = a + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] += (uint64_t)((uint32_t)c[i] ^ a) * b;
  uint64_t s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mulhi64(uint64_t* out, int iters) {
  uint64_t a = threadIdx.x * 0x9E3779B97F4A7C15ull, b = 0xD1B54A32D192ED03ull, c[8];
  for (int i = 0; i < 8; ++i) c[i] = a + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = __umul64hi(c[i], b) + c[i];
  uint64_t s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0000001f, c[8];
  for (int i = 0; i < 8; ++i) c[i] = a + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = fmaf(c[i], b, a);
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_frnd(double* out, int iters) {
  double a = threadIdx.x * 1e-3 + 0.3, c[8];
  for (int i = 0; i < 8; ++i) c[i] = a + i * 0.37;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = rint(c[i]) + 0.3;  // FRND.F64 + DADD
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dadd(double* out, int iters) {
  double a = threadIdx.x * 1e-3 + 0.3, c[8];
  for (int i = 0; i < 8; ++i) c[i] = a + i * 0.37;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = __dadd_rn(c[i], a);
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// exact FP64 modular multiply, rint vs magic-constant rounding (ops counted as 1 mulmod)
__global__ void k_mm_rint(double* out, int iters) {
  const double p = 1125899906826241.0, w = 987654321098765.0, wp = w / p;
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1000.0 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double h = __dmul_rn(c[i], w), l = __fma_rn(c[i], w, -h);
      const double q = rint(__dmul_rn(c[i], wp));
      c[i] = __dadd_rn(__fma_rn(-q, p, h), l);
    }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mm_magic(double* out, int iters) {
  const double p = 1125899906826241.0, w = 987654321098765.0, wp = w / p, mg = 6755399441055744.0;
  double c[8];
  for (int i = 0; i < 8; ++i) c[i] = threadIdx.x * 1000.0 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const double h = __dmul_rn(c[i], w), l = __fma_rn(c[i], w, -h);
      const double q = __dadd_rn(__fma_rn(c[i], wp, mg), -mg);
      c[i] = __dadd_rn(__fma_rn(-q, p, h), l);
    }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename F, typename T>
void run(const char* name, F kern, T* buf, int ops_per_iter_thread) {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int blocks = sms * 8, threads = 256, iters = 4096;
  kern<<<blocks, threads>>>(buf, 16);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<blocks, threads>>>(buf, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = (double)blocks * threads * iters * ops_per_iter_thread;
  const double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
  printf("%-10s %8.3f ms  %8.1f ops/clk/SM (at %d MHz nominal)\n", name, ms, per_sm_clk, clk / 1000);
}

int main() {
  void* buf;
  cudaMalloc(&buf, 148 * 8 * 256 * 8);
  run("dfma", k_dfma, (double*)buf, 8);
  run("ffma", k_ffma, (float*)buf, 8);
  run("imad.wide", k_imadw, (uint64_t*)buf, 8);
  run("mulhi64", k_mulhi64, (uint64_t*)buf, 8);
  run("frnd+dadd", k_frnd, (double*)buf, 8);
  run("dadd", k_dadd, (double*)buf, 8);
  run("mm_rint", k_mm_rint, (double*)buf, 8);
  run("mm_magic", k_mm_magic, (double*)buf, 8);
  return 0;
}
