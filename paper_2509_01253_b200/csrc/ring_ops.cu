// Gather-style ring kernels: automorphism, tower merge, partial extraction,
// and the grouped ciphertext x plaintext linear map.  All are HBM/L2-bound
// integer kernels: coalesced along the coefficient axis, one 64-bit lane per
// thread, mod-2^53 wrap arithmetic.
#include <cstdlib>

#include "sfhr_common.cuh"
#include "sfhr_kernels.h"

namespace sfhr {

// ---------------------------------------------------------------------------
// automorphism + fold: out[k] = v[s1]*[s1<N] - v[s2]*[s2<N]
// with s1 = k*d^-1, s2 = (N + k mod n1)*d^-1 (mod M)   (reference ring.py:101-130)

__global__ void automorphism_kernel(const __grid_constant__ RingConst rc, uint32_t dinv,
                                    const uint64_t* __restrict__ in, uint64_t* __restrict__ out) {
  const int64_t rc_row = blockIdx.x;  // (b, comp)
  const uint64_t* v = in + rc_row * rc.N;
  uint64_t* o = out + rc_row * rc.N;
  for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < rc.N; k += gridDim.y * blockDim.x) {
    const uint32_t km = fastmod((uint32_t)k, rc.n1, rc.magicN1);
    const uint32_t s1 = fastmod((uint32_t)k * dinv, rc.M, rc.magicM);
    const uint32_t s2 = fastmod((uint32_t)(rc.N + km) * dinv, rc.M, rc.magicM);
    uint64_t r = s1 < (uint32_t)rc.N ? v[s1] : 0ull;
    if (s2 < (uint32_t)rc.N) r -= v[s2];
    o[k] = r & QMASK;
  }
}

cudaError_t launch_automorphism(const RingConst& rc, uint32_t dinv, const uint64_t* in,
                                uint64_t* out, int64_t B, cudaStream_t st) {
  if (B == 0) return cudaSuccess;
  dim3 grid((unsigned)(B * 2), (rc.N + 255) / 256);
  automorphism_kernel<<<grid, 256, 0, st>>>(rc, dinv, in, out);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// tower merge (reference tracepack.py:307-316 with ring.py:77-84)

template <int MEM>
__global__ void merge_kernel(const __grid_constant__ RingConst rc, const uint64_t* __restrict__ in,
                             uint64_t* __restrict__ out, int members, int rest, int stride) {
  const int64_t orow = blockIdx.x;          // (g, r)
  const int comp = blockIdx.z;
  const int64_t g = orow / rest;
  const int r = (int)(orow - g * rest);
  const int N = rc.N, M = rc.M;
  const int nm = MEM ? MEM : members;
  const int st = (int)((uint32_t)stride % (uint32_t)M);  // member a rotates by a * st (mod M)
  for (int k = blockIdx.y * blockDim.x + threadIdx.x; k < N; k += gridDim.y * blockDim.x) {
    const int km = (int)fastmod((uint32_t)k, rc.n1, rc.magicN1);
    uint64_t t1[MEM ? MEM : 1], t2[MEM ? MEM : 1];
    uint64_t acc = 0;
    // all members' loads are issued before any is consumed (MEM is the compile-time count)
    int e = 0;
#pragma unroll
    for (int a = 0; a < (MEM ? MEM : 1); ++a) {
      const uint64_t* v = in + ((g * nm + a) * (int64_t)rest + r) * 2 * N + (int64_t)comp * N;
      if (a) {
        e += st;
        if (e >= M) e -= M;
      }
      int s1 = k - e;
      if (s1 < 0) s1 += M;
      int s2 = N + km - e;
      if (s2 < 0) s2 += M;
      t1[a] = s1 < N ? v[s1] : 0ull;
      t2[a] = s2 < N ? v[s2] : 0ull;
    }
    if (MEM) {
#pragma unroll
      for (int a = 0; a < (MEM ? MEM : 1); ++a) acc += t1[a] - t2[a];
    } else {
      for (int a = 0; a < nm; ++a) {
        const uint64_t* v = in + ((g * nm + a) * (int64_t)rest + r) * 2 * N + (int64_t)comp * N;
        const int e = (int)(((int64_t)a * stride) % M);
        int s1 = k - e;
        if (s1 < 0) s1 += M;
        int s2 = N + km - e;
        if (s2 < 0) s2 += M;
        uint64_t t = s1 < N ? v[s1] : 0ull;
        if (s2 < N) t -= v[s2];
        acc += t;
      }
    }
    out[orow * 2 * N + (int64_t)comp * N + k] = acc & QMASK;
  }
}

cudaError_t launch_merge(const RingConst& rc, const uint64_t* in, uint64_t* out, int64_t G,
                         int members, int rest, int stride, cudaStream_t st) {
  if (G == 0) return cudaSuccess;
  dim3 grid((unsigned)(G * rest), (rc.N + 255) / 256, 2);
  switch (members) {  // t - 1 or t members: 2..7 for the production rings
    case 2: merge_kernel<2><<<grid, 256, 0, st>>>(rc, in, out, members, rest, stride); break;
    case 3: merge_kernel<3><<<grid, 256, 0, st>>>(rc, in, out, members, rest, stride); break;
    case 4: merge_kernel<4><<<grid, 256, 0, st>>>(rc, in, out, members, rest, stride); break;
    case 5: merge_kernel<5><<<grid, 256, 0, st>>>(rc, in, out, members, rest, stride); break;
    case 6: merge_kernel<6><<<grid, 256, 0, st>>>(rc, in, out, members, rest, stride); break;
    case 7: merge_kernel<7><<<grid, 256, 0, st>>>(rc, in, out, members, rest, stride); break;
    default: merge_kernel<0><<<grid, 256, 0, st>>>(rc, in, out, members, rest, stride); break;
  }
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// partial-trace extraction (reference tracepack.py:118-154):
//   row_i = fold( sum_d cu * (ct_d[x] - ct_d[x - c_i n1 d]) ),  x = (i d + m) mod M

__global__ void extract_kernel(const __grid_constant__ RingConst rc, const __grid_constant__ ExtractArgs a) {
  const int64_t g = blockIdx.x;
  const int j = (int)(g / rc.N);
  const int i = (int)(g - (int64_t)j * rc.N);
  const int N = rc.N, M = rc.M, n1 = rc.n1;
  const int ci = a.cvec[i];
  for (int lane = blockIdx.y * blockDim.x + threadIdx.x; lane < 2 * N; lane += gridDim.y * blockDim.x) {
    const int comp = lane >= N;
    const int k = lane - comp * N;
    const uint32_t km = fastmod((uint32_t)k, n1, rc.magicN1);
    uint64_t acc = 0;
    for (int q = 0; q < a.npow; ++q) {
      const uint32_t d = a.exps[q];
      const uint64_t* ct = a.power + (((int64_t)j * a.npow + q) * 2 + comp) * N;
      const uint32_t id = fastmod((uint32_t)i * d, M, rc.magicM);
      const uint32_t sh = fastmod((uint32_t)(ci * n1) * d, M, rc.magicM);
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t x = id + (h ? (uint32_t)(N + km) : (uint32_t)k);
        x = x >= (uint32_t)M ? x - M : x;
        x = x >= (uint32_t)M ? x - M : x;
        uint32_t y = x + M - sh;
        y = y >= (uint32_t)M ? y - M : y;
        uint64_t t = x < (uint32_t)N ? __ldg(ct + x) : 0ull;
        if (y < (uint32_t)N) t -= __ldg(ct + y);
        acc = h ? acc - t : acc + t;
      }
    }
    a.rows[g * 2 * N + lane] = (acc * a.cu) & QMASK;
  }
}

// Row-tiled variant: one CTA per (chunk, EX_ROWS consecutive coefficients), the chunk's
// power ciphertexts staged once in shared memory (zero beyond N, so the reference's
// masked reads become plain reads), per-(row, power) rotation offsets precomputed, every
// thread producing 2N / EX_THREADS lanes of each row.  HBM-write-bound.
constexpr int EX_ROWS = 32;
constexpr int EX_THREADS = 512;
constexpr int EX_MAXPOW = 8;

__global__ void __launch_bounds__(EX_THREADS) extract_tiled_kernel(const __grid_constant__ RingConst rc,
                                                                   const __grid_constant__ ExtractArgs a) {
  extern __shared__ __align__(16) uint64_t sp[];  // [npow][2][M]
  __shared__ uint32_t sid[EX_ROWS][EX_MAXPOW], ssh[EX_ROWS][EX_MAXPOW];
  const int N = rc.N, M = rc.M, n1 = rc.n1;
  const int rblocks = (N + EX_ROWS - 1) / EX_ROWS;
  const int j = (int)(blockIdx.x / rblocks), rb = (int)(blockIdx.x % rblocks);
  const int i0 = rb * EX_ROWS;
  const int64_t g0 = (int64_t)j * N + i0;
  if (g0 >= a.E) return;
  const int nrows = (int)min((int64_t)min(EX_ROWS, N - i0), a.E - g0);
  const int np = a.npow;
  const uint64_t* src = a.power + (int64_t)j * np * 2 * N;
  for (int idx = threadIdx.x; idx < np * 2 * M; idx += EX_THREADS) {
    const int qc = idx / M, x = idx - qc * M;
    sp[idx] = x < N ? src[(int64_t)qc * N + x] : 0ull;
  }
  for (int t = threadIdx.x; t < nrows * np; t += EX_THREADS) {
    const int r = t / np, q = t - r * np;
    const uint32_t d = a.exps[q];
    sid[r][q] = fastmod((uint32_t)(i0 + r) * d, M, rc.magicM);
    ssh[r][q] = fastmod((uint32_t)(a.cvec[i0 + r] * n1) * d, M, rc.magicM);
  }
  __syncthreads();
  // lanes outer (their component / fold offsets are row-invariant), rows inner
  for (int lane = threadIdx.x; lane < 2 * N; lane += EX_THREADS) {
    const int comp = lane >= N;
    const uint32_t k = (uint32_t)(lane - comp * N);
    const uint32_t kf = (uint32_t)N + fastmod(k, n1, rc.magicN1);  // folded position N + (k mod n1)
    uint64_t* dst = a.rows + g0 * 2 * N + lane;
    for (int r = 0; r < nrows; ++r) {
      uint64_t acc = 0;
      for (int q = 0; q < np; ++q) {
        const uint64_t* ct = sp + (2 * q + comp) * M;
        const uint32_t id = sid[r][q], sh = ssh[r][q];
        uint32_t x0 = id + k, x1 = id + kf;  // both < 2M
        x0 = x0 >= (uint32_t)M ? x0 - M : x0;
        x1 = x1 >= (uint32_t)M ? x1 - M : x1;
        const uint32_t y0 = x0 >= sh ? x0 - sh : x0 + M - sh;
        const uint32_t y1 = x1 >= sh ? x1 - sh : x1 + M - sh;
        acc += (ct[x0] - ct[y0]) - (ct[x1] - ct[y1]);
      }
      dst[(int64_t)r * 2 * N] = (acc * a.cu) & QMASK;
    }
  }
}

size_t extract_tiled_smem(const RingConst& rc, int npow) { return (size_t)npow * 2 * rc.M * 8; }

// Offset-table variant (up to 6 powers).  Row i needs, per power d, (ct[x0] - ct[x0 - s]) -
// (ct[x1] - ct[x1 - s]) at x0 = i d + k, x1 = i d + N + (k mod n1), s = c_i n1 d (mod M).  c_i
// is constant over long runs of rows, so per distinct c of the CTA's row tile each power is
// staged once as the DIFFERENCE array D[x] = cu (ct[x mod M] - ct[(x - s) mod M]) (ct = 0 at
// indices >= N), extended to length M + N so that both reads are D[o + k] / D[o' + k mod n1]
// with per-(row, power) offsets o = i d, o' = i d + N precomputed once, no modular index
// arithmetic per element.  A thread owns the t - 1 lanes f + n1 m of a component, which share
// the folded read D[o' + f]: 1 + 1 / (t - 1) shared loads per (output, power).  When both components of
// all powers do not fit in shared memory (SPLIT) the CTA stages one component at a time.
// M^-1 (cu) is folded into the staged values: (sum +-ct) cu = sum +-(ct cu) mod 2^64.
constexpr int EXX_MAXPOW = 6;
#ifndef SFHR_EXX_ROWS
#define SFHR_EXX_ROWS 16
#endif
constexpr int EXX_ROWS = SFHR_EXX_ROWS;  // rows per CTA (A/B on B200: 16 > 8 > 32)
constexpr size_t EXX_SMEM_MAX = 220 * 1024;  // dynamic part; static tables (<= 7 KB) take the rest of 227 KB

// SPLIT kernels hold one CTA per SM: twice the threads and more rows per staging of the powers
template <bool SPLIT> struct ExxGeo {
  static constexpr int THREADS = SPLIT ? 1024 : EX_THREADS;
#ifndef SFHR_EXX_SPLIT_MULT
#define SFHR_EXX_SPLIT_MULT 2  // A/B (ResNet-18 extraction ms): 16 rows 6.34, 32 rows 5.48, 64 rows 5.67, 128 rows 7.13
#endif
  static constexpr int ROWS = SPLIT ? SFHR_EXX_SPLIT_MULT * EXX_ROWS : EXX_ROWS;
};

template <int NP, bool SPLIT, int LPT>
__global__ void __launch_bounds__(ExxGeo<SPLIT>::THREADS) extract_ext_kernel(const __grid_constant__ RingConst rc,
                                                                             const __grid_constant__ ExtractArgs a) {
  constexpr int EXX_ROWS = ExxGeo<SPLIT>::ROWS, EX_THREADS = ExxGeo<SPLIT>::THREADS;
  extern __shared__ __align__(16) uint64_t se[];  // [SPLIT ? 1 : 2][NP][M + N] difference arrays
  __shared__ uint2 soff[EXX_ROWS][NP];            // byte offsets x0 = i d, x1 = i d + N (mod M)
  __shared__ int srow_c[EXX_ROWS], scv[EXX_ROWS], sncv;
  __shared__ uint32_t ssh[NP];
  const int N = rc.N, M = rc.M, n1 = rc.n1, L = M + N;
  const int rblocks = (N + EXX_ROWS - 1) / EXX_ROWS;
  const int j = (int)(blockIdx.x / rblocks), rb = (int)(blockIdx.x % rblocks);
  const int i0 = rb * EXX_ROWS;
  const int64_t g0 = (int64_t)j * N + i0;
  if (g0 >= a.E) return;
  const int nrows = (int)min((int64_t)min(EXX_ROWS, N - i0), a.E - g0);
  const uint64_t* src = a.power + (int64_t)j * NP * 2 * N;  // [NP][2][N]
  const uint64_t cu = a.cu;
  for (int t = threadIdx.x; t < nrows * NP; t += EX_THREADS) {
    const int r = t / NP, q = t - r * NP;
    const uint32_t id = fastmod((uint32_t)(i0 + r) * a.exps[q], M, rc.magicM);
    const uint32_t x1 = id + (uint32_t)N >= (uint32_t)M ? id + N - M : id + N;
    soff[r][q] = make_uint2(8 * (q * L + id), 8 * (q * L + x1));
  }
  for (int r = threadIdx.x; r < nrows; r += EX_THREADS) srow_c[r] = a.cvec[i0 + r];
  __syncthreads();
  if (threadIdx.x == 0) {  // distinct c_i of the tile (c_i is constant over runs of n1 rows)
    int n = 0;
    for (int r = 0; r < nrows; ++r) {
      bool seen = false;
      for (int u = 0; u < n; ++u) seen |= scv[u] == srow_c[r];
      if (!seen) scv[n++] = srow_c[r];
    }
    sncv = n;
  }
  __syncthreads();
  const char* sb = reinterpret_cast<const char*>(se);
  const int ncv = sncv;
#pragma unroll 1
  for (int ci = 0; ci < ncv; ++ci) {
    const int c = scv[ci];
#pragma unroll 1
    for (int part = 0; part < (SPLIT ? 2 : 1); ++part) {
      if (threadIdx.x < NP) ssh[threadIdx.x] = fastmod((uint32_t)(c * n1) * a.exps[threadIdx.x], M, rc.magicM);
      __syncthreads();  // shifts visible; every thread is done with the previous staging
      // staged layout [comp (SPLIT: this part's only)][q][L]: D[x] = cu (ct[x mod M] - ct[(x - sh_q) mod M])
      const int ncomp = SPLIT ? 1 : 2;
      for (int idx = threadIdx.x; idx < ncomp * NP * L; idx += EX_THREADS) {
        const int cq = idx / L, x = idx - cq * L;
        const int comp = SPLIT ? part : cq / NP, q = cq - (cq / NP) * NP;
        const uint32_t xm = x >= M ? x - M : x, sh = ssh[q];
        const uint32_t y = xm >= sh ? xm - sh : xm + M - sh;
        const uint64_t* s = src + ((int64_t)q * 2 + comp) * N;
        const uint64_t v = (xm < (uint32_t)N ? s[xm] : 0ull) - (y < (uint32_t)N ? s[y] : 0ull);
        se[idx] = v * cu;
      }
      __syncthreads();
      // work item = (component, fold position f < n1): the t-1 lanes k = f + n1 m of a row share
      // the folded read D[i d + N + f], loaded once per (row, power)
      const int w1 = (SPLIT ? 1 : 2) * n1;
      for (int w = threadIdx.x; w < w1; w += EX_THREADS) {
        const int comp = SPLIT ? part : (w >= n1);
        const int f = w - (SPLIT ? 0 : comp) * n1;
        const char* ek = sb + 8 * ((SPLIT ? 0 : comp * NP * L) + f);
        uint64_t* dst = a.rows + g0 * 2 * N + (int64_t)comp * N + f;
        auto row = [&](int r) {
          uint64_t fold = 0, acc[LPT];
#pragma unroll
          for (int m = 0; m < LPT; ++m) acc[m] = 0;
#pragma unroll
          for (int q = 0; q < NP; ++q) {
            const uint2 o = soff[r][q];
            fold += *reinterpret_cast<const uint64_t*>(ek + o.y);
#pragma unroll
            for (int m = 0; m < LPT; ++m) acc[m] += *reinterpret_cast<const uint64_t*>(ek + o.x + 8 * m * n1);
          }
#pragma unroll
          for (int m = 0; m < LPT; ++m) dst[(int64_t)r * 2 * N + m * n1] = (acc[m] - fold) & QMASK;
        };
        if (ncv == 1) {  // the common case: one c_i for the whole tile, no per-row test
#pragma unroll 2
          for (int r = 0; r < nrows; ++r) row(r);
        } else {
#pragma unroll 2
          for (int r = 0; r < nrows; ++r)
            if (srow_c[r] == c) row(r);
        }
      }
    }
  }
}

// Many-power variant (gamma = 2: 42 powers at b = 12, 20 at b = 16).  The row terms of every
// power are summed in registers: one CTA per (chunk, component, tile of EXM_ROWS rows inside one
// run of n1 rows, where c_i = i / n1 + 1 is constant).  Powers stream through shared memory: the
// raw component arrives by bulk copy two powers ahead and is turned into the same M^-1-scaled
// difference array as extract_ext_kernel (double-buffered: power q + 1 is staged while q is
// accumulated); every output lane is written once.
#ifndef SFHR_EXM_ROWS
#define SFHR_EXM_ROWS 8
#endif
constexpr int EXM_ROWS = SFHR_EXM_ROWS;
template <int T> struct ExmGeo {  // production rows: t = 7 (alpha 4), 5 (alpha 5), 3 (alpha 7)
  static constexpr int N1 = T == 7 ? 343 : T == 5 ? 625 : 729;
  static constexpr int THREADS = (N1 + 31) / 32 * 32;
};

// Thread f < n1 owns the t-1 lanes k = f + n1 m of its component; they share the folded position
// N + (k mod n1) = N + f, so per (row, power) the folded term D[i d + N + f] is loaded once and
// summed separately (subtracted at the end): 1 + 1 / (t - 1) shared loads and one 64-bit add per
// output lane and power.
template <int T>
__global__ void __launch_bounds__(ExmGeo<T>::THREADS, 1) extract_many_kernel(const __grid_constant__ RingConst rc,
                                                                            const __grid_constant__ ExtractArgs a) {
  constexpr int N1 = ExmGeo<T>::N1, THREADS = ExmGeo<T>::THREADS, LPT = T - 1;
  // shared: [2][M + N] difference arrays, [2][M] raw power components (zero beyond N), 2 mbarriers
  extern __shared__ __align__(16) uint64_t sd[];
  __shared__ uint2 soff[2][EXM_ROWS];  // per staged power: offsets i d, i d + N (mod M)
  __shared__ __align__(8) uint64_t sbar[2];
  const int N = rc.N, M = rc.M, L = M + N;
  const int RS = (M + 1) & ~1;  // raw buffer stride (16-byte aligned bulk-copy destinations)
  uint64_t* raw = sd + 2 * ((L + 1) & ~1);
  constexpr int tiles_per_run = (N1 + EXM_ROWS - 1) / EXM_ROWS;
  int64_t b = blockIdx.x;
  const int tile = (int)(b % tiles_per_run);
  b /= tiles_per_run;
  const int run = (int)(b % (T - 1));
  b /= T - 1;
  const int comp = (int)(b & 1);
  const int j = (int)(b >> 1);
  const int i0 = run * N1 + tile * EXM_ROWS;
  const int i1 = min(run * N1 + N1, i0 + EXM_ROWS);
  const int64_t g0 = (int64_t)j * N + i0;
  if (g0 >= a.E) return;
  const int nrows = (int)min((int64_t)(i1 - i0), a.E - g0);
  const int c = a.cvec[i0];  // constant over the run
  const uint64_t cu = a.cu;
  const uint64_t* src = a.power + (int64_t)j * a.npow * 2 * N + (int64_t)comp * N;  // power q at + q 2N
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&sbar[0]);
  const int f = threadIdx.x;
  const bool act = f < N1;

  // raw components arrive by bulk copy (TMA engine, no registers), two powers ahead
  auto fetch = [&](int q) {
    const uint32_t bar = bar0 + 8u * (q & 1);
    const uint32_t bytes = (uint32_t)N * 8u;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(raw + (q & 1) * RS)),
                 "l"(src + (int64_t)q * 2 * N), "r"(bytes), "r"(bar)
                 : "memory");
  };
  auto wait_raw = [&](int q) {
    const uint32_t bar = bar0 + 8u * (q & 1), parity = (uint32_t)((q >> 1) & 1);
    uint32_t done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
                   " selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done)
                   : "r"(bar), "r"(parity)
                   : "memory");
  };
  // difference array of power q from its raw component: D[x] = cu (ct[x mod M] - ct[(x - s) mod M])
  auto stage = [&](int q, int buf) {
    const uint32_t d = a.exps[q];
    const uint32_t sh = fastmod((uint32_t)(c * N1) * d, M, rc.magicM);
    const uint64_t* rw = raw + (q & 1) * RS;
    uint64_t* D = sd + buf * L;
    for (int x = threadIdx.x; x < L; x += THREADS) {
      const uint32_t xm = x >= M ? x - M : x;
      const uint32_t y = xm >= sh ? xm - sh : xm + M - sh;
      D[x] = (rw[xm] - rw[y]) * cu;
    }
    if (threadIdx.x < EXM_ROWS) {
      const uint32_t id = fastmod((uint32_t)(i0 + threadIdx.x) * d, M, rc.magicM);
      soff[buf][threadIdx.x] = make_uint2(id, id + (uint32_t)N >= (uint32_t)M ? id + N - M : id + N);
    }
  };

  for (int x = N + threadIdx.x; x < M; x += THREADS) raw[x] = raw[RS + x] = 0ull;  // zero tails
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bar0 + 8u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    fetch(0);
    if (a.npow > 1) fetch(1);
  }

  uint64_t acc[EXM_ROWS][LPT], accf[EXM_ROWS];
#pragma unroll
  for (int r = 0; r < EXM_ROWS; ++r) {
    accf[r] = 0;
#pragma unroll
    for (int l = 0; l < LPT; ++l) acc[r][l] = 0;
  }

  wait_raw(0);
  stage(0, 0);
  __syncthreads();
  if (threadIdx.x == 0 && a.npow > 2) fetch(2);  // raw buffer 0 is free again
  for (int q = 0; q < a.npow; ++q) {
    if (q + 1 < a.npow) {  // overlaps the accumulation below
      wait_raw(q + 1);
      stage(q + 1, (q + 1) & 1);
    }
    if (act) {
      const char* Db = reinterpret_cast<const char*>(sd + (q & 1) * L);
#pragma unroll
      for (int r = 0; r < EXM_ROWS; ++r) {
        const uint2 o = soff[q & 1][r];
        const char* p0 = Db + 8u * (o.x + f);
        accf[r] += *reinterpret_cast<const uint64_t*>(Db + 8u * (o.y + f));
#pragma unroll
        for (int l = 0; l < LPT; ++l) acc[r][l] += *reinterpret_cast<const uint64_t*>(p0 + 8 * l * N1);
      }
    }
    __syncthreads();
    if (threadIdx.x == 0 && q + 3 < a.npow) fetch(q + 3);  // raw buffer (q + 1) & 1 is free
  }
  if (act) {
    uint64_t* dst = a.rows + g0 * 2 * N + (int64_t)comp * N + f;
#pragma unroll
    for (int r = 0; r < EXM_ROWS; ++r)
      if (r < nrows)
#pragma unroll
        for (int l = 0; l < LPT; ++l) dst[(int64_t)r * 2 * N + l * N1] = (acc[r][l] - accf[r]) & QMASK;
  }
}

static size_t exm_smem(const RingConst& rc) {  // [2][M + N] difference arrays + [2][M] raw components
  return (size_t)(2 * ((rc.M + rc.N + 1) & ~1) + 2 * ((rc.M + 1) & ~1)) * 8;
}

template <int T>
static cudaError_t launch_many(const RingConst& rc, const ExtractArgs& a, cudaStream_t st) {
  const size_t smem = exm_smem(rc);
  cudaError_t e = cudaFuncSetAttribute(extract_many_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t tiles = (int64_t)((ExmGeo<T>::N1 + EXM_ROWS - 1) / EXM_ROWS) * (T - 1);
  const int64_t grid = (int64_t)a.k_chunks * 2 * tiles;
  extract_many_kernel<T><<<(unsigned)grid, ExmGeo<T>::THREADS, smem, st>>>(rc, a);
  return cudaGetLastError();
}

template <int NP, int LPT>
static cudaError_t launch_ext_t(const RingConst& rc, const ExtractArgs& a, cudaStream_t st) {
  const size_t both = (size_t)2 * NP * (rc.M + rc.N) * 8;
  const bool split = both > EXX_SMEM_MAX;
  const size_t smem = split ? both / 2 : both;
  const auto kern = split ? extract_ext_kernel<NP, true, LPT> : extract_ext_kernel<NP, false, LPT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int rows = split ? ExxGeo<true>::ROWS : ExxGeo<false>::ROWS;
  const int threads = split ? ExxGeo<true>::THREADS : ExxGeo<false>::THREADS;
  const int rblocks = (rc.N + rows - 1) / rows;
  kern<<<(unsigned)(a.k_chunks * rblocks), threads, smem, st>>>(rc, a);
  return cudaGetLastError();
}

template <int NP>
static cudaError_t launch_ext(const RingConst& rc, const ExtractArgs& a, cudaStream_t st) {
  switch (rc.t) {  // lanes per fold position: t - 1
    case 3: return launch_ext_t<NP, 2>(rc, a, st);
    case 5: return launch_ext_t<NP, 4>(rc, a, st);
    case 7: return launch_ext_t<NP, 6>(rc, a, st);
    default: return cudaErrorInvalidValue;
  }
}

// powers from which the many-power kernel takes over (SFHR_EXM_MIN_POW for A/B).  A/B on B200:
// ResNet-20 b = 12 gamma = 1 (6 powers) extraction 7.90 -> 6.22 ms per inference; b = 16 gamma = 1
// (4 powers) unchanged (ResNet-18 73.9 vs 73.7 ms), so the offset-table kernel keeps < 6 powers
static int exm_min_pow() {
  static const int v = [] {
    const char* e = getenv("SFHR_EXM_MIN_POW");
    return e ? atoi(e) : 6;
  }();
  return v;
}

cudaError_t launch_extract(const RingConst& rc, const ExtractArgs& a, cudaStream_t st) {
  if (a.E == 0) return cudaSuccess;
  if (a.npow >= exm_min_pow() && !getenv("SFHR_EXTRACT_TILED") && exm_smem(rc) <= 200 * 1024) {
    if (rc.t == 7 && rc.alpha == 4) return launch_many<7>(rc, a, st);
    if (rc.t == 5 && rc.alpha == 5) return launch_many<5>(rc, a, st);
    if (rc.t == 3 && rc.alpha == 7) return launch_many<3>(rc, a, st);
  }
  // SFHR_EXTRACT_TILED=1 forces the general kernels (the tests compare both paths)
  if (a.npow >= 1 && a.npow <= EXX_MAXPOW && (size_t)a.npow * (rc.M + rc.N) * 8 <= EXX_SMEM_MAX &&
      !getenv("SFHR_EXTRACT_TILED")) {
    switch (a.npow) {
      case 1: return launch_ext<1>(rc, a, st);
      case 2: return launch_ext<2>(rc, a, st);
      case 3: return launch_ext<3>(rc, a, st);
      case 4: return launch_ext<4>(rc, a, st);
      case 5: return launch_ext<5>(rc, a, st);
      default: return launch_ext<6>(rc, a, st);
    }
  }
  const size_t smem = extract_tiled_smem(rc, a.npow);
  if (a.npow <= EX_MAXPOW && smem <= 200 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(extract_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    const int rblocks = (rc.N + EX_ROWS - 1) / EX_ROWS;
    extract_tiled_kernel<<<(unsigned)(a.k_chunks * rblocks), EX_THREADS, smem, st>>>(rc, a);
    return cudaGetLastError();
  }
  dim3 grid((unsigned)a.E, (2 * rc.N + 255) / 256);
  extract_kernel<<<grid, 256, 0, st>>>(rc, a);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// grouped linear map over ciphertext rows (reference model.py:384-429):
// exact mod 2^53 via a 31/22-bit operand split: w*x = w*x_lo + (w*x_hi) 2^31,
// the high product only matters mod 2^22, so a 32-bit accumulator suffices.

constexpr int RPG = 16;     // rows per group
constexpr int LCHUNK = 256; // columns staged in shared memory per chunk
constexpr int LTHREADS = 128;

__device__ __forceinline__ void mac16(uint64_t (&lo)[RPG], uint32_t (&hi)[RPG], const int4* w4, uint64_t x) {
  const int64_t xl = (int64_t)(x & 0x7fffffffull);
  const uint32_t xh = (uint32_t)(x >> 31);
#pragma unroll
  for (int q = 0; q < RPG / 4; ++q) {
    const int4 v = w4[q];
    lo[4 * q + 0] += (uint64_t)((int64_t)v.x * xl);
    hi[4 * q + 0] += (uint32_t)v.x * xh;
    lo[4 * q + 1] += (uint64_t)((int64_t)v.y * xl);
    hi[4 * q + 1] += (uint32_t)v.y * xh;
    lo[4 * q + 2] += (uint64_t)((int64_t)v.z * xl);
    hi[4 * q + 2] += (uint32_t)v.z * xh;
    lo[4 * q + 3] += (uint64_t)((int64_t)v.w * xl);
    hi[4 * q + 3] += (uint32_t)v.w * xh;
  }
}

__global__ void __launch_bounds__(LTHREADS) linear_kernel(const __grid_constant__ RingConst rc,
                                                          const __grid_constant__ LinearArgs a) {
  __shared__ int64_t colp[LCHUNK];                 // physical row offset (row * lanes) or -1
  __shared__ __align__(16) int32_t wsm[LCHUNK * RPG];
  const int64_t g = blockIdx.x;
  const int64_t W2 = a.lanes;
  const int64_t lane = (int64_t)blockIdx.y * blockDim.x + threadIdx.x;
  const bool act = lane < W2;
  const int32_t* gr = a.groups + 6 * g;
  const int c0 = gr[0], nc = gr[1], w0 = gr[2], r0 = gr[3], nr = gr[4], per = gr[5];
  uint64_t lo[RPG];
  uint32_t hi[RPG];
#pragma unroll
  for (int r = 0; r < RPG; ++r) { lo[r] = 0; hi[r] = 0; }

  if (!per) {
    for (int cb = 0; cb < nc; cb += LCHUNK) {
      const int cn = min(LCHUNK, nc - cb);
      __syncthreads();
      for (int k = threadIdx.x; k < cn; k += blockDim.x) {
        const int col = __ldg(a.cols + c0 + cb + k);
        colp[k] = col < 0 ? -1 : (a.in_map ? __ldg(a.in_map + col) : (int64_t)col) * W2;
      }
      const int4* wsrc = reinterpret_cast<const int4*>(a.weights + w0 + (int64_t)cb * RPG);
      int4* wdst = reinterpret_cast<int4*>(wsm);
      for (int k = threadIdx.x; k < cn * (RPG / 4); k += blockDim.x) wdst[k] = __ldg(wsrc + k);
      __syncthreads();
      if (act) {
        int k = 0;
        for (; k + 4 <= cn; k += 4) {
          uint64_t x[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int64_t off = colp[k + u];
            x[u] = off >= 0 ? __ldg(a.in + off + lane) : 0ull;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u)
            mac16(lo, hi, reinterpret_cast<const int4*>(wsm + (k + u) * RPG), x[u]);
        }
        for (; k < cn; ++k) {
          const int64_t off = colp[k];
          const uint64_t x = off >= 0 ? __ldg(a.in + off + lane) : 0ull;
          mac16(lo, hi, reinterpret_cast<const int4*>(wsm + k * RPG), x);
        }
      }
    }
  } else if (act) {
#pragma unroll
    for (int r = 0; r < RPG; ++r) {
      if (r < nr) {
        for (int c = 0; c < nc; ++c) {
          const int col = __ldg(a.cols + c0 + r * nc + c);
          if (col < 0) continue;
          const int64_t src = a.in_map ? __ldg(a.in_map + col) : col;
          const uint64_t x = __ldg(a.in + src * W2 + lane);
          const int wt = __ldg(a.weights + w0 + c * RPG + r);
          lo[r] += (uint64_t)((int64_t)wt * (int64_t)(x & 0x7fffffffull));
          hi[r] += (uint32_t)wt * (uint32_t)(x >> 31);
        }
      }
    }
  }
  if (!act) return;

#pragma unroll
  for (int r = 0; r < RPG; ++r) {
    if (r < nr) {
      const int o = __ldg(a.rows + r0 + r);
      if (a.ex_ptr) {
        const int e0 = __ldg(a.ex_ptr + o), e1 = __ldg(a.ex_ptr + o + 1);
        for (int e = e0; e < e1; ++e) {
          const int col = __ldg(a.ex_col + e);
          const int64_t src = a.round_map ? __ldg(a.round_map + col) : col;
          const uint64_t x = __ldg(a.round_in + src * W2 + lane);
          const int wt = __ldg(a.ex_w + e);
          lo[r] += (uint64_t)((int64_t)wt * (int64_t)(x & 0x7fffffffull));
          hi[r] += (uint32_t)wt * (uint32_t)(x >> 31);
        }
      }
      uint64_t v = lo[r] + ((uint64_t)hi[r] << 31);
      if (a.bias && lane >= a.body_off) v += (uint64_t)__ldg(a.bias + o) * __ldg(a.unit + (lane - a.body_off));
      const int64_t dst = a.out_map ? __ldg(a.out_map + o) : o;
      a.out[dst * W2 + lane] = v & QMASK;
    }
  }
}

cudaError_t launch_linear(const RingConst& rc, const LinearArgs& a, cudaStream_t st) {
  if (a.G == 0) return cudaSuccess;
  dim3 grid((unsigned)a.G, (unsigned)((a.lanes + LTHREADS - 1) / LTHREADS));
  linear_kernel<<<grid, LTHREADS, 0, st>>>(rc, a);
  return cudaGetLastError();
}

}  // namespace sfhr
