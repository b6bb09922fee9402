// Standalone RNS negacyclic NTT over ~50-bit primes (BASELINE.json configs[1],
// SURVEY.md §8(d)-B): forward / inverse transforms of batches of (L, N) u64
// residue polynomials modulo X^N + 1, N = 2^10 .. 2^16, L <= 32 limbs.
//
// There is no counterpart in the reference (it has no power-of-two rings,
// SURVEY.md §0); this is the north star's "RNS NTT/iNTT" primitive, checked
// by self-consistency (inverse o forward = id, NTT convolution = schoolbook)
// and bit-exactly against the plain-C oracle in oracle/ntt_ref.c.
//
// Algorithm: merged-twiddle Cooley-Tukey forward (natural order in,
// bit-reversed out; twiddles psi^brv(k)) and Gentleman-Sande inverse with Shoup
// multiplication (w' = floor(w 2^64 / p)).  Primes are < 2^50, so the 14 spare
// bits of a u64 let the butterflies run without range corrections (forward:
// values < (2 log2 N + 1) p; inverse: sums reduced once per radix-16 pass);
// residues are fully reduced at the boundary.
//
// One HBM pass per transform: a polynomial is split over a thread-block
// CLUSTER of C = max(1, N / 8192) CTAs, each holding a contiguous chunk of
// <= 8192 residues in shared memory.  The log2(C) stages whose butterflies
// cross chunks are done in registers straight from / to global memory (each
// thread owns the C residues at one chunk offset) and exchanged through
// distributed shared memory; the remaining stages run in radix-16 register
// passes over the CTA's chunk.
#include <cooperative_groups.h>

#include <cstdint>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "../../include/sfhr_b200.h"

namespace cg = cooperative_groups;

namespace sfhr {
namespace ntt {

constexpr int CHUNK_MAX = 8192;  // residues per CTA
constexpr int EPT = 16;          // residues per thread in a local pass
#ifndef NTT_MINB
#define NTT_MINB 2
#endif

struct Tables {
  const uint64_t* w;    // [L][N] psi^brv(k) (forward), k >= 1 used
  const uint64_t* ws;   // [L][N] Shoup companions
  const uint64_t* wi;   // [L][N] psi^-brv(k) (inverse); wi[0] = N^-1
  const uint64_t* wis;  // [L][N]
  const uint64_t* p;    // [L]
  const uint64_t* mu;   // [L] floor(2^64 / p)
};

__device__ __forceinline__ uint64_t shoup(uint64_t x, uint64_t w, uint64_t ws, uint64_t p) {
  const uint64_t q = __umul64hi(x, ws);
  return x * w - q * p;  // in [0, 2p) for any x < 2^64
}

// forward CT butterfly without range corrections: Shoup accepts any 64-bit Y and
// returns t in [0, 2p), so an input bound X, Y < k p gives outputs < (k + 2) p.
// After the 16 stages of N = 2^16 every value is < 33 p < 2^56 (p < 2^50 is
// enforced by the planner), and one final reduction brings it to [0, p).
__device__ __forceinline__ void ct_bfly(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t ws, uint64_t p) {
  const uint64_t t = shoup(Y, w, ws, p);
  const uint64_t x = X;
  X = x + t;
  Y = x + (2 * p - t);
}
// inverse GS butterfly with lazy sums: X, Y < M (M a multiple of p) -> X' = X + Y < 2M,
// Y' in [0, 2p); a local pass reduces once at its end
__device__ __forceinline__ void gs_bfly_lazy(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t ws, uint64_t p,
                                             uint64_t M) {
  const uint64_t x = X, y = Y;
  X = x + y;
  Y = shoup(x + M - y, w, ws, p);
}
__device__ __forceinline__ uint64_t barrett2(uint64_t x, uint64_t p, uint64_t mu) {
  return x - __umul64hi(x, mu) * p;  // x < 2^63 -> [0, 2p)
}
// inverse GS butterfly, inputs/outputs in [0, 2p)
__device__ __forceinline__ void gs_bfly(uint64_t& X, uint64_t& Y, uint64_t w, uint64_t ws, uint64_t p) {
  const uint64_t p2 = 2 * p;
  const uint64_t x = X, y = Y;
  uint64_t s = x + y;
  X = s >= p2 ? s - p2 : s;
  Y = shoup(x - y + p2, w, ws, p);
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }  // one pad word per 16 (bank spread)

// Twiddles of one radix-2^r sub-butterfly: for the pass's stage st (global stage
// s0 + st, distance d = D >> st) the 2^st groups it touches are
// g = B0 / (2d) + t, t < 2^st (B0 = global start of its 2D block), i.e. the
// entries k = 2^(s0+st) + (B0 >> (log2 D + 1 - st)) + t.  They do not depend on
// the data, so each pass loads all of them (2^r - 1 pairs) before touching smem.

// local forward passes over a chunk (global position of element 0 = c0), stages with
// distance chunk/2 .. 1; s0 = global stage index of the first local stage
template <int LOGC>
__device__ __forceinline__ void fwd_local(uint64_t* sm, int64_t c0, int s0, const uint64_t* w, const uint64_t* ws,
                                          uint64_t p) {
  constexpr int CH = 1 << LOGC;
  int done = 0;
  // first pass takes LOGC % 4 stages (if any), the rest are radix-16
#pragma unroll
  for (int pass = 0; pass < (LOGC + 3) / 4; ++pass) {
    const int r = (pass == 0 && (LOGC % 4)) ? (LOGC % 4) : 4;
    const int logD = LOGC - done - 1;           // log2 distance of the pass's first stage
    const int D = 1 << logD;
    const int inner = D >> (r - 1);             // stride between the 2^r elements
    const int per = EPT >> r;                   // independent sub-butterflies per thread
    uint64_t v[EPT];
    int base[EPT >> 1];
    uint64_t tw[EPT >> 1][15], tws[EPT >> 1][15];
#pragma unroll
    for (int h = 0; h < per; ++h) {
      const int id = threadIdx.x * per + h;
      const int b = id / inner, j = id - b * inner;
      base[h] = b * 2 * D + j;
      const int64_t B0 = c0 + (int64_t)b * 2 * D;
#pragma unroll
      for (int st = 0; st < r; ++st) {
        const int64_t k0 = ((int64_t)1 << (s0 + done + st)) + (B0 >> (logD + 1 - st));
#pragma unroll
        for (int t = 0; t < (1 << st); ++t) {
          tw[h][(1 << st) - 1 + t] = __ldg(w + k0 + t);
          tws[h][(1 << st) - 1 + t] = __ldg(ws + k0 + t);
        }
      }
#pragma unroll
      for (int lo = 0; lo < (1 << r); ++lo) v[h * (1 << r) + lo] = sm[pad(base[h] + lo * inner)];
    }
#pragma unroll
    for (int st = 0; st < r; ++st) {
      const int half = (1 << r) >> (st + 1);    // distance in lo units
#pragma unroll
      for (int h = 0; h < per; ++h) {
#pragma unroll
        for (int lo = 0; lo < (1 << r); ++lo) {
          if (lo & half) continue;
          const int t = (1 << st) - 1 + (lo >> (r - st));
          ct_bfly(v[h * (1 << r) + lo], v[h * (1 << r) + lo + half], tw[h][t], tws[h][t], p);
        }
      }
    }
#pragma unroll
    for (int h = 0; h < per; ++h)
#pragma unroll
      for (int lo = 0; lo < (1 << r); ++lo) sm[pad(base[h] + lo * inner)] = v[h * (1 << r) + lo];
    __syncthreads();
    done += r;
  }
}

// local inverse passes: stages with distance 1 .. chunk/2 (global stage index s0 + LOGC - 1 .. s0)
template <int LOGC>
__device__ __forceinline__ void inv_local(uint64_t* sm, int64_t c0, int s0, const uint64_t* w, const uint64_t* ws,
                                          uint64_t p, uint64_t mu) {
  int done = 0;  // stages done, counted from distance 1 upwards
#pragma unroll
  for (int pass = 0; pass < (LOGC + 3) / 4; ++pass) {
    const int r = (pass == (LOGC + 3) / 4 - 1 && (LOGC % 4)) ? (LOGC % 4) : 4;
    const int Dmin = 1 << done;               // distance of the pass's first (smallest) stage
    const int logD = done + r - 1;            // log2 of the largest distance in the pass
    const int D = 1 << logD;
    const int inner = Dmin;
    const int per = EPT >> r;
    uint64_t v[EPT];
    int base[EPT >> 1];
    uint64_t tw[EPT >> 1][15], tws[EPT >> 1][15];
#pragma unroll
    for (int h = 0; h < per; ++h) {
      const int id = threadIdx.x * per + h;
      const int b = id / inner, j = id - b * inner;
      base[h] = b * 2 * D + j;
      const int64_t B0 = c0 + (int64_t)b * 2 * D;
      // stage with distance D >> u (u = r-1-st) has 2^u groups in the block
#pragma unroll
      for (int u = 0; u < r; ++u) {
        const int s = s0 + LOGC - 1 - (done + r - 1 - u);
        const int64_t k0 = ((int64_t)1 << s) + (B0 >> (logD + 1 - u));
#pragma unroll
        for (int t = 0; t < (1 << u); ++t) {
          tw[h][(1 << u) - 1 + t] = __ldg(w + k0 + t);
          tws[h][(1 << u) - 1 + t] = __ldg(ws + k0 + t);
        }
      }
#pragma unroll
      for (int lo = 0; lo < (1 << r); ++lo) v[h * (1 << r) + lo] = sm[pad(base[h] + lo * inner)];
    }
#pragma unroll
    for (int st = 0; st < r; ++st) {
      const int half = 1 << st;
      const int u = r - 1 - st;
#pragma unroll
      for (int h = 0; h < per; ++h) {
#pragma unroll
        for (int lo = 0; lo < (1 << r); ++lo) {
          if (lo & half) continue;
          const int t = (1 << u) - 1 + (lo >> (st + 1));
          // inputs of stage st are < 2^(st+1) p (sums double, Shoup outputs < 2p)
          gs_bfly_lazy(v[h * (1 << r) + lo], v[h * (1 << r) + lo + half], tw[h][t], tws[h][t], p,
                       p << (st + 1));
        }
      }
    }
#pragma unroll
    for (int h = 0; h < per; ++h)
#pragma unroll
      for (int lo = 0; lo < (1 << r); ++lo)
        sm[pad(base[h] + lo * inner)] = barrett2(v[h * (1 << r) + lo], p, mu);
    __syncthreads();
    done += r;
  }
}

__device__ __forceinline__ uint64_t reduce4(uint64_t x, uint64_t p) {
  if (x >= 2 * p) x -= 2 * p;
  if (x >= p) x -= p;
  return x;
}
// x < 2^63 -> x mod p, with mu = floor(2^64 / p)
__device__ __forceinline__ uint64_t reduce_full(uint64_t x, uint64_t p, uint64_t mu) {
  uint64_t r = x - __umul64hi(x, mu) * p;  // [0, 2p)
  return r >= p ? r - p : r;
}

// grid: (batch * L) clusters of C CTAs; data (batch, L, N) u64
template <int LOGN, int LOGCL>
__global__ void __launch_bounds__((1 << (LOGN - LOGCL)) / EPT, NTT_MINB) ntt_fwd_kernel(uint64_t* data, int L, Tables t) {
  constexpr int C = 1 << LOGCL, LOGC = LOGN - LOGCL, CH = 1 << LOGC, NT = CH / EPT;
  extern __shared__ __align__(16) uint64_t sm[];
  const int64_t poly = blockIdx.x / C;
  const int c = (int)(blockIdx.x % C);
  const int limb = (int)(poly % L);
  const uint64_t p = t.p[limb];
  const uint64_t* w = t.w + (size_t)limb * ((size_t)1 << LOGN);
  const uint64_t* ws = t.ws + (size_t)limb * ((size_t)1 << LOGN);
  uint64_t* x = data + poly * ((int64_t)1 << LOGN);
  if (C == 1) {
    for (int i = threadIdx.x; i < CH; i += NT) sm[pad(i)] = x[i];
    __syncthreads();
  } else {
    // cross-chunk stages 0 .. LOGCL-1: this CTA owns chunk offsets [c*CH/C, (c+1)*CH/C)
    cg::cluster_group cluster = cg::this_cluster();
    // every peer must be running before its shared memory is written: arrive now,
    // wait just before the first remote store
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    bool waited = false;
    for (int o = c * (CH / C) + threadIdx.x; o < (c + 1) * (CH / C); o += NT) {
      uint64_t v[C];
#pragma unroll
      for (int q = 0; q < C; ++q) v[q] = x[(int64_t)q * CH + o];
#pragma unroll
      for (int s = 0; s < LOGCL; ++s) {
        const int half = C >> (s + 1);
#pragma unroll
        for (int q = 0; q < C; ++q) {
          if (q & half) continue;
          const int g = q >> (LOGCL - s);
          const int k = (1 << s) + g;
          ct_bfly(v[q], v[q + half], __ldg(w + k), __ldg(ws + k), p);
        }
      }
      if (!waited) {
        asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
        waited = true;
      }
#pragma unroll
      for (int q = 0; q < C; ++q) cluster.map_shared_rank(sm, q)[pad(o)] = v[q];
    }
    if (!waited) asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    cluster.sync();
  }
  fwd_local<LOGC>(sm, (int64_t)c * CH, LOGCL, w, ws, p);
  uint64_t* xo = x + (int64_t)c * CH;
  const uint64_t mu = t.mu[limb];
  for (int i = threadIdx.x; i < CH; i += NT) xo[i] = reduce_full(sm[pad(i)], p, mu);
}

template <int LOGN, int LOGCL>
__global__ void __launch_bounds__((1 << (LOGN - LOGCL)) / EPT, NTT_MINB) ntt_inv_kernel(uint64_t* data, int L, Tables t) {
  constexpr int C = 1 << LOGCL, LOGC = LOGN - LOGCL, CH = 1 << LOGC, NT = CH / EPT;
  extern __shared__ __align__(16) uint64_t sm[];
  const int64_t poly = blockIdx.x / C;
  const int c = (int)(blockIdx.x % C);
  const int limb = (int)(poly % L);
  const uint64_t p = t.p[limb];
  const uint64_t* w = t.wi + (size_t)limb * ((size_t)1 << LOGN);
  const uint64_t* ws = t.wis + (size_t)limb * ((size_t)1 << LOGN);
  const uint64_t ninv = __ldg(w), ninvs = __ldg(ws);  // wi[0] = N^-1
  uint64_t* x = data + poly * ((int64_t)1 << LOGN);
  const uint64_t* xi = x + (int64_t)c * CH;
  for (int i = threadIdx.x; i < CH; i += NT) {
    const uint64_t v = xi[i];
    sm[pad(i)] = v >= p ? v - p : v;  // tolerate inputs in [0, 2p)
  }
  __syncthreads();
  inv_local<LOGC>(sm, (int64_t)c * CH, LOGCL, w, ws, p, t.mu[limb]);
  if (C == 1) {
    for (int i = threadIdx.x; i < CH; i += NT) x[i] = reduce4(shoup(sm[pad(i)], ninv, ninvs, p), p);
  } else {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    for (int o = c * (CH / C) + threadIdx.x; o < (c + 1) * (CH / C); o += NT) {
      uint64_t v[C];
#pragma unroll
      for (int q = 0; q < C; ++q) v[q] = cluster.map_shared_rank(sm, q)[pad(o)];
#pragma unroll
      for (int s = LOGCL - 1; s >= 0; --s) {
        const int half = C >> (s + 1);
#pragma unroll
        for (int q = 0; q < C; ++q) {
          if (q & half) continue;
          const int g = q >> (LOGCL - s);
          const int k = (1 << s) + g;
          gs_bfly(v[q], v[q + half], __ldg(w + k), __ldg(ws + k), p);
        }
      }
#pragma unroll
      for (int q = 0; q < C; ++q) x[(int64_t)q * CH + o] = reduce4(shoup(v[q], ninv, ninvs, p), p);
    }
    cluster.sync();  // peers may still read this CTA's chunk
  }
}

// ---------------------------------------------------------------------------
// host: primes, tables, launch

uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) { return (uint64_t)((unsigned __int128)a * b % m); }
uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
  uint64_t r = 1;
  a %= m;
  while (e) {
    if (e & 1) r = mulmod(r, a, m);
    a = mulmod(a, a, m);
    e >>= 1;
  }
  return r;
}
bool is_prime(uint64_t n) {
  if (n < 2) return false;
  for (uint64_t q : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull})
    if (n % q == 0) return n == q;
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) d >>= 1, ++s;
  for (uint64_t a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull}) {
    uint64_t x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int i = 1; i < s && comp; ++i) {
      x = mulmod(x, x, n);
      if (x == n - 1) comp = false;
    }
    if (comp) return false;
  }
  return true;
}
int brv(int x, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1) << (bits - 1 - i);
  return r;
}
uint64_t shoup_of(uint64_t w, uint64_t p) { return (uint64_t)(((unsigned __int128)w << 64) / p); }

}  // namespace ntt
}  // namespace sfhr

using namespace sfhr::ntt;

struct sfhr_ntt_plan {
  int logn = 0, L = 0, device = 0;
  std::vector<uint64_t> primes, w, ws, wi, wis;  // host copies
  uint64_t* d_tab = nullptr;                     // [5][...] device copy
  Tables t{};
};

namespace {
thread_local std::string g_ntt_err;
int nfail(int code, const std::string& m) {
  g_ntt_err = m;
  return code;
}

template <int LOGN, int LOGCL>
cudaError_t launch_one(bool fwd, uint64_t* data, int64_t polys, int L, const Tables& t, cudaStream_t st) {
  constexpr int C = 1 << LOGCL, CH = 1 << (LOGN - LOGCL), NT = CH / EPT;
  const size_t smem = (size_t)(CH + CH / 16) * 8;
  auto kern = fwd ? ntt_fwd_kernel<LOGN, LOGCL> : ntt_inv_kernel<LOGN, LOGCL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(polys * C), 1, 1);
  cfg.blockDim = dim3(NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = C;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, data, L, t);
}

cudaError_t launch(bool fwd, int logn, uint64_t* data, int64_t polys, int L, const Tables& t, cudaStream_t st) {
  switch (logn) {
    case 10: return launch_one<10, 0>(fwd, data, polys, L, t, st);
    case 11: return launch_one<11, 0>(fwd, data, polys, L, t, st);
    case 12: return launch_one<12, 0>(fwd, data, polys, L, t, st);
    case 13: return launch_one<13, 0>(fwd, data, polys, L, t, st);
    case 14: return launch_one<14, 1>(fwd, data, polys, L, t, st);
    case 15: return launch_one<15, 2>(fwd, data, polys, L, t, st);
    case 16: return launch_one<16, 3>(fwd, data, polys, L, t, st);
    default: return cudaErrorInvalidValue;
  }
}
}  // namespace

extern "C" {

int sfhr_ntt_plan_create(int logn, int L, int prime_bits, int device, sfhr_ntt_plan** out) {
  if (!out) return nfail(SFHR_EINVAL, "null output");
  if (logn < 10 || logn > 16) return nfail(SFHR_EINVAL, "log2 N must be in [10, 16]");
  if (L < 1 || L > 32) return nfail(SFHR_EINVAL, "limb count must be in [1, 32]");
  // the lazy forward butterflies keep values below (2 log2 N + 1) p < 2^56 (see ct_bfly)
  if (prime_bits < 30 || prime_bits > 50) return nfail(SFHR_EINVAL, "prime bits must be in [30, 50]");
  auto* P = new sfhr_ntt_plan();
  P->logn = logn;
  P->L = L;
  P->device = device;
  const uint64_t N = 1ull << logn, twoN = 2 * N;
  // largest primes p = 1 (mod 2N) below 2^prime_bits
  for (uint64_t k = ((1ull << prime_bits) - 1) / twoN; k > 0 && (int)P->primes.size() < L; --k) {
    const uint64_t p = k * twoN + 1;
    if (p < (1ull << prime_bits) && is_prime(p)) P->primes.push_back(p);
  }
  if ((int)P->primes.size() < L) {
    delete P;
    return nfail(SFHR_EINVAL, "not enough NTT primes");
  }
  P->w.assign(L * N, 0);
  P->ws.assign(L * N, 0);
  P->wi.assign(L * N, 0);
  P->wis.assign(L * N, 0);
  for (int i = 0; i < L; ++i) {
    const uint64_t p = P->primes[i];
    uint64_t psi = 0;  // primitive 2N-th root: psi^N = -1
    for (uint64_t g = 2; g < p && !psi; ++g) {
      const uint64_t c = powmod(g, (p - 1) / twoN, p);
      if (powmod(c, N, p) == p - 1) psi = c;
    }
    const uint64_t psii = powmod(psi, p - 2, p);
    std::vector<uint64_t> pw(N), pwi(N);
    pw[0] = pwi[0] = 1;
    for (uint64_t e = 1; e < N; ++e) {
      pw[e] = mulmod(pw[e - 1], psi, p);
      pwi[e] = mulmod(pwi[e - 1], psii, p);
    }
    for (uint64_t k = 0; k < N; ++k) {
      const int e = brv((int)k, logn);
      const uint64_t a = pw[e], b = pwi[e];
      P->w[i * N + k] = a;
      P->ws[i * N + k] = shoup_of(a, p);
      P->wi[i * N + k] = b;
      P->wis[i * N + k] = shoup_of(b, p);
    }
    const uint64_t ninv = powmod(N % p, p - 2, p);
    P->wi[i * N] = ninv;  // slot 0 is unused by the butterflies
    P->wis[i * N] = shoup_of(ninv, p);
  }
  if (device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    const size_t words = (size_t)4 * L * N + 2 * L;
    cudaError_t e = cudaMalloc(&P->d_tab, words * 8);
    uint64_t* d = P->d_tab;
    if (e == cudaSuccess) e = cudaMemcpy(d, P->w.data(), L * N * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + L * N, P->ws.data(), L * N * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + 2 * L * N, P->wi.data(), L * N * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + 3 * L * N, P->wis.data(), L * N * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + 4 * L * N, P->primes.data(), L * 8, cudaMemcpyHostToDevice);
    std::vector<uint64_t> mus(L);
    for (int i = 0; i < L; ++i) mus[i] = (uint64_t)(((unsigned __int128)1 << 64) / P->primes[i]);
    if (e == cudaSuccess) e = cudaMemcpy(d + 4 * L * N + L, mus.data(), L * 8, cudaMemcpyHostToDevice);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
      cudaFree(P->d_tab);
      delete P;
      return nfail(SFHR_ECUDA, std::string("ntt tables: ") + cudaGetErrorString(e));
    }
    P->t = Tables{d, d + L * N, d + 2 * L * N, d + 3 * L * N, d + 4 * L * N, d + 4 * L * N + L};
  }
  *out = P;
  return SFHR_OK;
}

int sfhr_ntt_plan_destroy(sfhr_ntt_plan* P) {
  if (!P) return SFHR_OK;
  if (P->d_tab) cudaFree(P->d_tab);
  delete P;
  return SFHR_OK;
}

int sfhr_ntt_plan_primes(const sfhr_ntt_plan* P, uint64_t* primes, int n) {
  if (!P || !primes) return nfail(SFHR_EINVAL, "null argument");
  for (int i = 0; i < n && i < P->L; ++i) primes[i] = P->primes[i];
  return SFHR_OK;
}

int sfhr_ntt_plan_tables(const sfhr_ntt_plan* P, uint64_t* w, uint64_t* wi) {
  if (!P) return nfail(SFHR_EINVAL, "null argument");
  const size_t n = (size_t)P->L << P->logn;
  if (w) std::memcpy(w, P->w.data(), n * 8);
  if (wi) std::memcpy(wi, P->wi.data(), n * 8);
  return SFHR_OK;
}

static int ntt_run(bool fwd, const sfhr_ntt_plan* P, uint64_t* data, int64_t batch, void* stream) {
  if (!P || !data) return nfail(SFHR_EINVAL, "null argument");
  if (P->device < 0) return nfail(SFHR_EINVAL, "planning-only NTT plan (device -1) cannot compute");
  if (batch < 0) return nfail(SFHR_EINVAL, "negative batch");
  if (batch == 0) return SFHR_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  if (prev != P->device) cudaSetDevice(P->device);
  cudaError_t e = launch(fwd, P->logn, data, batch * P->L, P->L, P->t, (cudaStream_t)stream);
  if (prev != P->device) cudaSetDevice(prev);
  if (e != cudaSuccess) return nfail(SFHR_ECUDA, std::string("ntt kernel: ") + cudaGetErrorString(e));
  return SFHR_OK;
}

int sfhr_ntt_forward(const sfhr_ntt_plan* P, uint64_t* data, int64_t batch, void* stream) {
  return ntt_run(true, P, data, batch, stream);
}
int sfhr_ntt_inverse(const sfhr_ntt_plan* P, uint64_t* data, int64_t batch, void* stream) {
  return ntt_run(false, P, data, batch, stream);
}
const char* sfhr_ntt_last_error(void) { return g_ntt_err.c_str(); }

}  // extern "C"
