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
// bit-reversed out; twiddles psi^brv(k)) and Gentleman-Sande inverse.  The
// modular arithmetic runs on the FP64 pipe: residues (< 2^50) are exact integers
// in doubles, x w mod p = (h + l) - rint(x w/p) p with the FMA error-free product
// h + l (see mulmod_d; exact for |x| < 2^52), values kept below 4p by a rounding
// reduction every two stages; u64 residues in and out, fully reduced.
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
#ifndef NTT_EPT
#define NTT_EPT 16
#endif
constexpr int EPT = NTT_EPT;     // residues per thread in a local pass
#ifndef NTT_MINB
#define NTT_MINB 2
#endif
// every global / remote load of a thread's cross-chunk work and of its final chunk pass issued
// before the first use (the loops were latency-serialised: one round trip per iteration)
// (bit 0: forward cross-chunk loads, for clusters of <= 2^NTT_FWD_PRE_MAXCL CTAs; bit 1: forward
// final pass; bit 2: inverse final pass (C = 1); bit 3: inverse cross-chunk DSMEM loads, for
// clusters of >= 2^NTT_INV_PRE_MINCL CTAs -- below those sizes the 16 prefetched values per
// thread cost more in registers than the latency they hide)
#ifndef NTT_BATCH_IO
#define NTT_BATCH_IO 1
#endif
// A/B knob: the next local pass's twiddles prefetched into L1 while the current pass runs (their
// L2 latency stalls the first butterfly of a pass); measured 1-7 % slower (the prefetch
// instructions and address math cost more issue slots than the latency they hide), so off
#ifndef NTT_TW_PREFETCH
#define NTT_TW_PREFETCH 0
#endif
#ifndef NTT_FWD_PRE_MAXCL
#define NTT_FWD_PRE_MAXCL 2
#endif
#ifndef NTT_INV_PRE_MINCL
#define NTT_INV_PRE_MINCL 3
#endif

struct Tables {
  const double* w;     // [L][N] psi^brv(k) (forward), k >= 1 used, exact integers
  const double* wp;    // [L][N] w / p (rounded)
  const double* wi;    // [L][N] psi^-brv(k) (inverse); wi[0] = N^-1
  const double* wip;   // [L][N]
  const uint64_t* p;   // [L]
};

// Modular arithmetic on the FP64 pipe (B200: ~60 DFMA/clk/SM vs ~7 64-bit mulhi/clk/SM).
// Residues are exact integers held in doubles, |x| < 2^52 (primes < 2^50, values < 4p).
// mulmod: h + l = x w exactly (FMA error-free product), q = rint(x w/p) is within 1.5
// of x w / p, and h - q p is an integer below 2^53, so fma(-q, p, h) is exact and
// r = x w - q p exactly, |r| <= 1.5 p.  (Intrinsics keep the compiler from contracting.)
__device__ __forceinline__ double mulmod_d(double x, double w, double wp, double p) {
  const double h = __dmul_rn(x, w);
  const double l = __fma_rn(x, w, -h);
  const double q = rint(__dmul_rn(x, wp));
  return __dadd_rn(__fma_rn(-q, p, h), l);
}
// |x| < 2^52 -> x mod p in [-p/2, p/2] (up to rounding of x / p)
__device__ __forceinline__ double red_d(double x, double p, double pinv) {
  return __fma_rn(-rint(__dmul_rn(x, pinv)), p, x);
}
__device__ __forceinline__ uint64_t to_residue(double x, double p, double pinv) {
  double r = red_d(x, p, pinv);
  if (r < 0.0) r = __dadd_rn(r, p);
  return (uint64_t)r;
}
// forward CT butterfly: |X|, |Y| < B -> |X'|, |Y'| < B + 1.5 p
__device__ __forceinline__ void ct_bfly(double& X, double& Y, double w, double wp, double p) {
  const double t = mulmod_d(Y, w, wp, p);
  const double x = X;
  X = __dadd_rn(x, t);
  Y = __dsub_rn(x, t);
}
// inverse GS butterfly: X' = X + Y, Y' = (X - Y) w
__device__ __forceinline__ void gs_bfly(double& X, double& Y, double w, double wp, double p) {
  const double x = X, y = Y;
  X = __dadd_rn(x, y);
  Y = mulmod_d(__dsub_rn(x, y), w, wp, p);
}

__device__ __forceinline__ int pad(int i) { return i + (i >> 4); }  // one pad word per 16 (bank spread)

// The 2^st twiddles of one sub-butterfly stage are consecutive and 2^st-aligned in the table:
// 16-byte vector loads, and only w is loaded.  Its Shoup companion w / p is formed in registers
// as w * (1/p) (two roundings instead of one: x * wp stays within 1.5 of x w / p for the
// |x| < 2p inputs the passes feed mulmod_d, so the quotient is off by at most 2 and every
// intermediate stays far below 2^52; the final residues are exact either way).
// (K is a constant after the callers' loops unroll)
__device__ __forceinline__ void load_twiddles(int K, double* tw, const double* src) {
  if (K == 1) {
    tw[0] = __ldg(src);
  } else {
#pragma unroll
    for (int t = 0; t < 8; t += 2) {
      if (t >= K) break;
      const double2 q = __ldg(reinterpret_cast<const double2*>(src + t));
      tw[t] = q.x;
      tw[t + 1] = q.y;
    }
  }
}

// Twiddles of one radix-2^r sub-butterfly: for the pass's stage st (global stage
// s0 + st, distance d = D >> st) the 2^st groups it touches are
// g = B0 / (2d) + t, t < 2^st (B0 = global start of its 2D block), i.e. the
// entries k = 2^(s0+st) + (B0 >> (log2 D + 1 - st)) + t.  They do not depend on
// the data, so each pass loads all of them (2^r - 1 pairs) before touching smem.
// Range discipline: every pass reduces on load and after its second stage, so no
// value exceeds 0.5 p + 2 * 1.5 p < 4 p < 2^52.

__device__ __forceinline__ void prefetch_l1(const void* a) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(a));
}
// L1 prefetch of the twiddle groups forward pass `pass` of fwd_local will load (same addresses)
template <int LOGC>
__device__ __forceinline__ void fwd_tw_prefetch(int pass, int64_t c0, int s0, const double* w) {
  int done = 0;
#pragma unroll
  for (int q = 0; q < (LOGC + 3) / 4; ++q) {
    if (q == pass) break;
    done += (q == 0 && (LOGC % 4)) ? (LOGC % 4) : 4;
  }
  const int r = (pass == 0 && (LOGC % 4)) ? (LOGC % 4) : 4;
  const int logD = LOGC - done - 1, D = 1 << logD, inner = D >> (r - 1), per = EPT >> r;
#pragma unroll
  for (int h = 0; h < per; ++h) {
    const int id = threadIdx.x * per + h;
    const int b = id / inner;
    const int64_t B0 = c0 + (int64_t)b * 2 * D;
#pragma unroll
    for (int st = 0; st < r; ++st)
      prefetch_l1(w + ((int64_t)1 << (s0 + done + st)) + (B0 >> (logD + 1 - st)));
  }
}
// the same for inverse pass `pass` of inv_local
template <int LOGC>
__device__ __forceinline__ void inv_tw_prefetch(int pass, int64_t c0, int s0, const double* w) {
  constexpr int NP = (LOGC + 3) / 4;
  int done = 0;
#pragma unroll
  for (int q = 0; q < NP; ++q) {
    if (q == pass) break;
    done += (q == NP - 1 && (LOGC % 4)) ? (LOGC % 4) : 4;
  }
  const int r = (pass == NP - 1 && (LOGC % 4)) ? (LOGC % 4) : 4;
  const int logD = done + r - 1, D = 1 << logD, inner = 1 << done, per = EPT >> r;
#pragma unroll
  for (int h = 0; h < per; ++h) {
    const int id = threadIdx.x * per + h;
    const int b = id / inner;
    const int64_t B0 = c0 + (int64_t)b * 2 * D;
#pragma unroll
    for (int u = 0; u < r; ++u) {
      const int sg = s0 + LOGC - 1 - (done + r - 1 - u);
      prefetch_l1(w + ((int64_t)1 << sg) + (B0 >> (logD + 1 - u)));
    }
  }
}

// local forward passes over a chunk (global position of element 0 = c0), stages with
// distance chunk/2 .. 1; s0 = global stage index of the first local stage
template <int LOGC>
__device__ __forceinline__ void fwd_local(double* sm, int64_t c0, int s0, const double* w, const double* wp,
                                          double p, double pinv) {
  int done = 0;
  // first pass takes LOGC % 4 stages (if any), the rest are radix-16
#pragma unroll
  for (int pass = 0; pass < (LOGC + 3) / 4; ++pass) {
    const int r = (pass == 0 && (LOGC % 4)) ? (LOGC % 4) : 4;
    const int logD = LOGC - done - 1;           // log2 distance of the pass's first stage
    const int D = 1 << logD;
    const int inner = D >> (r - 1);             // stride between the 2^r elements
    const int per = EPT >> r;                   // independent sub-butterflies per thread
    double v[EPT];
    int base[EPT >> 1];
    double tw[EPT >> 1][15];
#pragma unroll
    for (int h = 0; h < per; ++h) {
      const int id = threadIdx.x * per + h;
      const int b = id / inner, j = id - b * inner;
      base[h] = b * 2 * D + j;
      const int64_t B0 = c0 + (int64_t)b * 2 * D;
#pragma unroll
      for (int st = 0; st < r; ++st) {
        const int64_t k0 = ((int64_t)1 << (s0 + done + st)) + (B0 >> (logD + 1 - st));
        load_twiddles(1 << st, tw[h] + (1 << st) - 1, w + k0);
      }
      // passes of >= 3 stages reduce after their second stage and store values below ~2p, and the
      // cross-chunk stages / raw input are below ~2p too, so only the short (r <= 2) passes
      // reduce on load: two CT stages from 2p stay below ~5p < 2^53 (see load_twiddles)
#pragma unroll
      for (int lo = 0; lo < (1 << r); ++lo) {
        const double x = sm[pad(base[h] + lo * inner)];
        v[h * (1 << r) + lo] = r <= 2 ? red_d(x, p, pinv) : x;
      }
    }
    if (NTT_TW_PREFETCH && pass + 1 < (LOGC + 3) / 4) fwd_tw_prefetch<LOGC>(pass + 1, c0, s0, w);
#pragma unroll
    for (int st = 0; st < r; ++st) {
      const int half = (1 << r) >> (st + 1);    // distance in lo units
#pragma unroll
      for (int h = 0; h < per; ++h) {
        double twp[8];  // w / p of this stage's twiddles (see load_twiddles)
#pragma unroll
        for (int t = 0; t < (1 << st); ++t) twp[t] = __dmul_rn(tw[h][(1 << st) - 1 + t], pinv);
#pragma unroll
        for (int lo = 0; lo < (1 << r); ++lo) {
          if (lo & half) continue;
          const int t = (1 << st) - 1 + (lo >> (r - st));
          ct_bfly(v[h * (1 << r) + lo], v[h * (1 << r) + lo + half], tw[h][t], twp[lo >> (r - st)], p);
        }
      }
      if (st == 1 && r > 2) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = red_d(v[e], p, pinv);
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
__device__ __forceinline__ void inv_local(double* sm, int64_t c0, int s0, const double* w, const double* wp,
                                          double p, double pinv) {
  int done = 0;  // stages done, counted from distance 1 upwards
#pragma unroll
  for (int pass = 0; pass < (LOGC + 3) / 4; ++pass) {
    const int r = (pass == (LOGC + 3) / 4 - 1 && (LOGC % 4)) ? (LOGC % 4) : 4;
    const int Dmin = 1 << done;               // distance of the pass's first (smallest) stage
    const int logD = done + r - 1;            // log2 of the largest distance in the pass
    const int D = 1 << logD;
    const int inner = Dmin;
    const int per = EPT >> r;
    double v[EPT];
    int base[EPT >> 1];
    double tw[EPT >> 1][15];
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
        load_twiddles(1 << u, tw[h] + (1 << u) - 1, w + k0);
      }
      // GS stages double X: a pass of >= 3 stages reduces after its second and stores values
      // below ~1.6p, so two more stages from there stay below ~5p < 2^53 without reducing on load
#pragma unroll
      for (int lo = 0; lo < (1 << r); ++lo) {
        const double x = sm[pad(base[h] + lo * inner)];
        v[h * (1 << r) + lo] = r <= 2 ? red_d(x, p, pinv) : x;
      }
    }
    if (NTT_TW_PREFETCH && pass + 1 < (LOGC + 3) / 4) inv_tw_prefetch<LOGC>(pass + 1, c0, s0, w);
#pragma unroll
    for (int st = 0; st < r; ++st) {
      const int half = 1 << st;
      const int u = r - 1 - st;
#pragma unroll
      for (int h = 0; h < per; ++h) {
        double twp[8];
#pragma unroll
        for (int t = 0; t < (1 << u); ++t) twp[t] = __dmul_rn(tw[h][(1 << u) - 1 + t], pinv);
#pragma unroll
        for (int lo = 0; lo < (1 << r); ++lo) {
          if (lo & half) continue;
          const int t = (1 << u) - 1 + (lo >> (st + 1));
          gs_bfly(v[h * (1 << r) + lo], v[h * (1 << r) + lo + half], tw[h][t], twp[lo >> (st + 1)], p);
        }
      }
      if (st == 1 && r > 2) {
#pragma unroll
        for (int e = 0; e < EPT; ++e) v[e] = red_d(v[e], p, pinv);
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

// grid: (batch * L) clusters of C CTAs; data (batch, L, N) u64
template <int LOGN, int LOGCL>
__global__ void __launch_bounds__((1 << (LOGN - LOGCL)) / EPT, NTT_MINB) ntt_fwd_kernel(uint64_t* data, int L, Tables t) {
  constexpr int C = 1 << LOGCL, LOGC = LOGN - LOGCL, CH = 1 << LOGC, NT = CH / EPT;
  extern __shared__ __align__(16) double sm[];
  const int64_t poly = blockIdx.x / C;
  const int c = (int)(blockIdx.x % C);
  const int limb = (int)(poly % L);
  const double p = (double)t.p[limb], pinv = 1.0 / p;
  const double* w = t.w + (size_t)limb * ((size_t)1 << LOGN);
  const double* wp = t.wp + (size_t)limb * ((size_t)1 << LOGN);
  uint64_t* x = data + poly * ((int64_t)1 << LOGN);
  if (NTT_TW_PREFETCH) fwd_tw_prefetch<LOGC>(0, (int64_t)c * CH, LOGCL, w);
  if (C == 1) {
    uint64_t in[EPT];  // all loads in flight before the first shared store
#pragma unroll
    for (int e = 0; e < EPT; ++e) in[e] = x[threadIdx.x + e * NT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) sm[pad(threadIdx.x + e * NT)] = (double)in[e];
    __syncthreads();
  } else {
    // cross-chunk stages 0 .. LOGCL-1: this CTA owns chunk offsets [c*CH/C, (c+1)*CH/C)
    cg::cluster_group cluster = cg::this_cluster();
    // every peer must be running before its shared memory is written: arrive now,
    // wait just before the first remote store
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    bool waited = false;
    constexpr int IT = (CH / C) / NT;  // o-iterations per thread (EPT / C)
    constexpr bool kPre = (NTT_BATCH_IO & 1) && LOGCL <= NTT_FWD_PRE_MAXCL && IT * C <= EPT;
    uint64_t pre[kPre ? IT * C : 1];
    if constexpr (kPre) {
#pragma unroll
      for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int q = 0; q < C; ++q) pre[it * C + q] = x[(int64_t)q * CH + c * (CH / C) + threadIdx.x + it * NT];
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int o = c * (CH / C) + threadIdx.x + it * NT;
      double v[C];
#pragma unroll
      for (int q = 0; q < C; ++q) {
        if constexpr (kPre) v[q] = (double)pre[it * C + q];
        else v[q] = (double)x[(int64_t)q * CH + o];
      }
#pragma unroll
      for (int s = 0; s < LOGCL; ++s) {
        const int half = C >> (s + 1);
#pragma unroll
        for (int q = 0; q < C; ++q) {
          if (q & half) continue;
          const int g = q >> (LOGCL - s);
          const int k = (1 << s) + g;
          ct_bfly(v[q], v[q + half], __ldg(w + k), __ldg(wp + k), p);
        }
        if (s == 1) {
#pragma unroll
          for (int q = 0; q < C; ++q) v[q] = red_d(v[q], p, pinv);
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
  fwd_local<LOGC>(sm, (int64_t)c * CH, LOGCL, w, wp, p, pinv);
  uint64_t* xo = x + (int64_t)c * CH;
  if (NTT_BATCH_IO & 2) {
    double o[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) o[e] = sm[pad(threadIdx.x + e * NT)];
#pragma unroll
    for (int e = 0; e < EPT; ++e) xo[threadIdx.x + e * NT] = to_residue(o[e], p, pinv);
  } else {
    for (int i = threadIdx.x; i < CH; i += NT) xo[i] = to_residue(sm[pad(i)], p, pinv);
  }
}

template <int LOGN, int LOGCL>
__global__ void __launch_bounds__((1 << (LOGN - LOGCL)) / EPT, NTT_MINB) ntt_inv_kernel(uint64_t* data, int L, Tables t) {
  constexpr int C = 1 << LOGCL, LOGC = LOGN - LOGCL, CH = 1 << LOGC, NT = CH / EPT;
  extern __shared__ __align__(16) double sm[];
  const int64_t poly = blockIdx.x / C;
  const int c = (int)(blockIdx.x % C);
  const int limb = (int)(poly % L);
  const uint64_t pu = t.p[limb];
  const double p = (double)pu, pinv = 1.0 / p;
  const double* w = t.wi + (size_t)limb * ((size_t)1 << LOGN);
  const double* wp = t.wip + (size_t)limb * ((size_t)1 << LOGN);
  const double ninv = __ldg(w), ninvp = __ldg(wp);  // wi[0] = N^-1
  uint64_t* x = data + poly * ((int64_t)1 << LOGN);
  if (NTT_TW_PREFETCH) inv_tw_prefetch<LOGC>(0, (int64_t)c * CH, LOGCL, w);
  const uint64_t* xi = x + (int64_t)c * CH;
  {
    uint64_t in[EPT];  // all loads in flight before the first shared store
#pragma unroll
    for (int e = 0; e < EPT; ++e) in[e] = xi[threadIdx.x + e * NT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const uint64_t v = in[e];
      sm[pad(threadIdx.x + e * NT)] = (double)(v >= pu ? v - pu : v);  // tolerate inputs in [0, 2p)
    }
  }
  __syncthreads();
  inv_local<LOGC>(sm, (int64_t)c * CH, LOGCL, w, wp, p, pinv);
  if (C == 1) {
    if (NTT_BATCH_IO & 4) {
      double o[EPT];
#pragma unroll
      for (int e = 0; e < EPT; ++e) o[e] = sm[pad(threadIdx.x + e * NT)];
#pragma unroll
      for (int e = 0; e < EPT; ++e)
        x[threadIdx.x + e * NT] = to_residue(mulmod_d(red_d(o[e], p, pinv), ninv, ninvp, p), p, pinv);
    } else {
      for (int i = threadIdx.x; i < CH; i += NT)
        x[i] = to_residue(mulmod_d(red_d(sm[pad(i)], p, pinv), ninv, ninvp, p), p, pinv);
    }
  } else {
    cg::cluster_group cluster = cg::this_cluster();
    cluster.sync();
    constexpr int IT = (CH / C) / NT;  // o-iterations per thread (EPT / C)
    constexpr bool kPre = (NTT_BATCH_IO & 8) && LOGCL >= NTT_INV_PRE_MINCL && IT * C <= EPT;
    double pre[kPre ? IT * C : 1];
    if constexpr (kPre) {
#pragma unroll
      for (int it = 0; it < IT; ++it)
#pragma unroll
        for (int q = 0; q < C; ++q)
          pre[it * C + q] = cluster.map_shared_rank(sm, q)[pad(c * (CH / C) + threadIdx.x + it * NT)];
    }
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      const int o = c * (CH / C) + threadIdx.x + it * NT;
      double v[C];
#pragma unroll
      for (int q = 0; q < C; ++q) {
        if constexpr (kPre) v[q] = red_d(pre[it * C + q], p, pinv);
        else v[q] = red_d(cluster.map_shared_rank(sm, q)[pad(o)], p, pinv);
      }
#pragma unroll
      for (int s = LOGCL - 1; s >= 0; --s) {
        const int half = C >> (s + 1);
#pragma unroll
        for (int q = 0; q < C; ++q) {
          if (q & half) continue;
          const int g = q >> (LOGCL - s);
          const int k = (1 << s) + g;
          gs_bfly(v[q], v[q + half], __ldg(w + k), __ldg(wp + k), p);
        }
        if (s == LOGCL - 2) {
#pragma unroll
          for (int q = 0; q < C; ++q) v[q] = red_d(v[q], p, pinv);
        }
      }
#pragma unroll
      for (int q = 0; q < C; ++q)
        x[(int64_t)q * CH + o] = to_residue(mulmod_d(v[q], ninv, ninvp, p), p, pinv);
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

}  // namespace ntt
}  // namespace sfhr

using namespace sfhr::ntt;

struct sfhr_ntt_plan {
  int logn = 0, L = 0, device = 0;
  std::vector<uint64_t> primes, w, wi;   // host copies (integers)
  std::vector<double> wd, wpd, wid, wipd;  // device tables: value and value / p
  void* d_tab = nullptr;
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
  const size_t smem = (size_t)(CH + CH / 16) * sizeof(double);
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
  // the FP64 butterflies keep residues below 4p < 2^52 (see mulmod_d)
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
  P->wi.assign(L * N, 0);
  P->wd.assign(L * N, 0);
  P->wpd.assign(L * N, 0);
  P->wid.assign(L * N, 0);
  P->wipd.assign(L * N, 0);
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
      P->wi[i * N + k] = b;
    }
    const uint64_t ninv = powmod(N % p, p - 2, p);
    P->wi[i * N] = ninv;  // slot 0 is unused by the butterflies
    for (uint64_t k = 0; k < N; ++k) {
      P->wd[i * N + k] = (double)P->w[i * N + k];
      P->wpd[i * N + k] = (double)P->w[i * N + k] / (double)p;
      P->wid[i * N + k] = (double)P->wi[i * N + k];
      P->wipd[i * N + k] = (double)P->wi[i * N + k] / (double)p;
    }
  }
  if (device >= 0) {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    const size_t words = (size_t)4 * L * N + L;
    cudaError_t e = cudaMalloc(&P->d_tab, words * 8);
    double* d = static_cast<double*>(P->d_tab);
    if (e == cudaSuccess) e = cudaMemcpy(d, P->wd.data(), L * N * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + L * N, P->wpd.data(), L * N * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + 2 * L * N, P->wid.data(), L * N * 8, cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMemcpy(d + 3 * L * N, P->wipd.data(), L * N * 8, cudaMemcpyHostToDevice);
    uint64_t* dp = reinterpret_cast<uint64_t*>(d + 4 * L * N);
    if (e == cudaSuccess) e = cudaMemcpy(dp, P->primes.data(), L * 8, cudaMemcpyHostToDevice);
    cudaSetDevice(prev);
    if (e != cudaSuccess) {
      cudaFree(P->d_tab);
      delete P;
      return nfail(SFHR_ECUDA, std::string("ntt tables: ") + cudaGetErrorString(e));
    }
    P->t = Tables{d, d + L * N, d + 2 * L * N, d + 3 * L * N, dp};
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
  if (!P) return nfail(SFHR_EINVAL, "null plan");
  if (batch == 0) return SFHR_OK;  // an empty batch may come with a null data pointer
  if (!data) return nfail(SFHR_EINVAL, "null data");
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
