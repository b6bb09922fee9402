// Ciphertext-block wire codec on the device (reference pkg/src/sfhr/wire.py:99-124,
// 208-254): the raw ROUND_REQ payload is copied to the GPU in
// one transfer and unpacked there into the (k, npow, 2, N) upload layout with the
// reference's < 2^53 range check on every lane (padding included); packed outputs are
// laid out as the zero-padded (count, 2, M) block body straight from device memory.
// Block bodies sit at arbitrary byte offsets (each block ends with a 1-byte gamma tag),
// so every lane is assembled from three aligned u32 words with funnel shifts.
#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/sfhr_b200.h"

namespace sfhr {

__global__ void wire_unpack_kernel(const uint32_t* __restrict__ raw, const int64_t* __restrict__ body_off,
                                   int npow, int M, int N, uint64_t* __restrict__ out, int* err) {
  const int64_t r = blockIdx.x;  // (chunk j, power q, component c)
  const int64_t j = r / (2 * npow), qc = r - j * 2 * npow;
  const int64_t B = body_off[j] + qc * (int64_t)M * 8;  // byte offset of lane 0
  const uint32_t* src = raw + (B >> 2);
  const uint32_t sh = (uint32_t)(B & 3) * 8;
  uint64_t* dst = out + r * N;
  int bad = 0;
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    const uint32_t w0 = src[2 * i], w1 = src[2 * i + 1], w2 = sh ? src[2 * i + 2] : 0u;
    const uint64_t v = (uint64_t)__funnelshift_r(w0, w1, sh) | ((uint64_t)__funnelshift_r(w1, w2, sh) << 32);
    bad |= v >= (1ull << 53);
    if (i < N) dst[i] = v;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(err, 1);
}

__global__ void wire_pack_kernel(const uint64_t* __restrict__ rows, int M, int N, uint64_t* __restrict__ body) {
  const int64_t r = blockIdx.x;  // (pack, component)
  for (int i = threadIdx.x; i < M; i += blockDim.x) body[r * M + i] = i < N ? rows[r * N + i] : 0ull;
}

}  // namespace sfhr

extern "C" {

int sfhr_wire_unpack(const uint8_t* payload, const int64_t* body_offsets, int64_t k, int npow, int M, int N,
                     uint64_t* out, int* err, void* stream) {
  if (k < 0 || npow < 1 || M < N || N < 1) return SFHR_EINVAL;
  if (k == 0) return SFHR_OK;
  sfhr::wire_unpack_kernel<<<(unsigned)(k * npow * 2), 256, 0, (cudaStream_t)stream>>>(
      reinterpret_cast<const uint32_t*>(payload), body_offsets, npow, M, N, out, err);
  return cudaGetLastError() == cudaSuccess ? SFHR_OK : SFHR_ECUDA;
}

int sfhr_wire_pack(const uint64_t* rows, int64_t count, int M, int N, uint64_t* body, void* stream) {
  if (count < 0 || M < N || N < 1) return SFHR_EINVAL;
  if (count == 0) return SFHR_OK;
  sfhr::wire_pack_kernel<<<(unsigned)(count * 2), 256, 0, (cudaStream_t)stream>>>(rows, M, N, body);
  return cudaGetLastError() == cudaSuccess ? SFHR_OK : SFHR_ECUDA;
}

}  // extern "C"
