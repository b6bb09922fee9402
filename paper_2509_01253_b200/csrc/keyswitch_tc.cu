// Tensor-core forward key switch (sm_100a, tcgen05 kind::i8), ring row t = 7
// (M = 7^4, N = 2058, the b = 12 presets).
//
// Semantics: for every input row x and each of the stage's representatives
// (automorphism d_r, key set K_r), the NTT-domain accumulators
//     A = sum_r sum_i NTT(dig_i(aut_r(x.a))) * NTT(K_r[i].a)      (same for B / .b)
// modulo each CRT prime -- exactly what ks_stage_kernel's forward part
// computes (reference tracepack.py:268-285, crypto.py:288-323, 400-464).  The
// CUDA-core kernel then runs in its acc_in mode for the inverse transforms,
// CRT mod 2^53 and the identity / body terms (keyswitch.cu).
//
// The Phi_M-NTT of a digit polynomial is two batched small matrix products
// over Z_p (derivation and a bit-level model: tests/tc_model.py):
//   coefficient c = j*343 + m1*49 + m0, output (o, k1), o = 7 (r-1) + k0,
//   evaluation point omega^(r + 7 k0 + 49 k1):
//   pass A   z[o | m0] = sum_{j,m1} W_A[o][(j,m1)] d[c]       (42 x 42, per m0)
//   twiddle  y[o | m0] = z[o | m0] omega^((r + 7 k0) m0)
//   pass B   A[o, k1]  = sum_{m0} omega^(49 k1 m0) y[o | m0]   (49 x 49, per o)
// Each pass is an exact u8 x u8 -> s32 GEMM over byte planes with the data
// planes folded into K (constant rows C[plane][.] = 256^plane W mod p), so the
// four per-byte-plane accumulators of the constants combine as l + 2^16 h
// (l = D0 + 256 D1, h = D2 + 256 D3) and ONE Montgomery REDC against the pair
// (x R, 2^16 x R) reduces and multiplies (by the twiddle after pass A, by the key
// spectrum after pass B).  Digits enter with an offset (unsigned planes); an
// extra K row of ones carries the correction.
//
// One CTA = one CRT prime, persistent over row pairs; warp-specialised:
//   warps 0-15  E_B: pass-B accumulators -> MAC with the key spectra (keys
//               prefetched into registers before the wait), NTT-domain sums
//               over reps and digits kept in TMEM, written once per row pair
//   warps 16-19 E_A: pass-A accumulators -> twiddle -> byte planes of the
//               pass-B operand (MN-major, 128B swizzle) in shared memory
//   warps 20-26 producers: automorphism gather + balanced digits of both rows
//               -> byte planes of the pass-A operand
//   warp 27     MMA issuer (tcgen05.mma, commits to mbarriers), TMEM owner
// TMEM: pass A [0, 176), accumulators [176, 288), pass-B k1-halves [288, 400), [400, 512).
#include <cstring>
#include <vector>

#include "sfhr_common.cuh"
#include "sfhr_kernels.h"
#include "tc_ptx.cuh"

namespace sfhr {

namespace tc7 {

constexpr int T = 7, M = 2401, N = 2058, N1 = 343;
constexpr int SA = 42, SB = 49;        // pass sizes (outputs o / inputs (j, m1) and m0 / k1)
constexpr int KA = 96;                 // pass-A K rows: 2 planes x 42 + ones row, padded to 3 x 32
constexpr int NAO = 44;                // pass-A columns per constant byte plane
constexpr int NA = 4 * NAO;            // 176
constexpr int KB = 224;                // pass-B K rows: 4 planes x 49, padded to 7 x 32
constexpr int KBH = 28;                // pass-B columns per plane and k1-half
constexpr int NBH = 4 * KBH;           // 112
constexpr int K1H = 25;                // k1 in half 0: [0, 25), half 1: [25, 49)
constexpr int AA_BYTES = KA * 128;     // 12288 per digit tile
constexpr int AB_BYTES = KB * 128;     // 28672 per buffer
constexpr int BA_BYTES = KA * NA;      // 16896
constexpr int BB_BYTES = KB * NBH;     // 25088 per half
constexpr int TWS = 43;                // twiddle table row stride (uint2), bank-conflict free
constexpr int TW_BYTES = SB * TWS * 8; // 16856
constexpr int TAB_BYTES = BA_BYTES + 2 * BB_BYTES + ((TW_BYTES + 15) & ~15);  // per prime
constexpr int XA_BYTES = 2 * N * 8;    // digits kernel: both rows' mask components
constexpr int EB_WARPS = 16;           // E_B: 4 lane quadrants x 2 k1-halves x 2 parts ([0,12), [12,25|24))
constexpr int EA_WARPS = 8;            // E_A: 4 lane quadrants x 2 output halves
constexpr int LOAD_WARP = EB_WARPS + EA_WARPS;
constexpr int MMA_WARP = LOAD_WARP + 1;
constexpr int NTHREADS = (MMA_WARP + 1) * 32;  // 26 warps: 7 per SMSP leaves 72 registers
// TMEM columns: pass A, the NTT-domain accumulators (a / b, k1-half h at +28h), pass-B halves
constexpr uint32_t COL_A = 0, COL_ACC_A = 176, COL_ACC_B = 232, COL_B0 = 288, COL_B1 = 400;
constexpr int NBARS = 14;
constexpr int DIG_THREADS = 256;       // digits kernel block

// byte address of (K row k, M lane m) in an MN-major 128B-swizzled u8 operand tile
__device__ __forceinline__ uint32_t swz(uint32_t tile, int k, int m) {
  return tile + (uint32_t)(k * 128 + ((((m >> 4) ^ (k & 7)) << 4) | (m & 15)));
}

struct Smem {
  int aa, ab, ba, bb, tw, bars, tslot, total;
  __host__ __device__ static Smem make(int L) {
    Smem s;
    s.aa = 0;                          // two sets of L pass-A operand tiles (double-buffered reps)
    s.ab = s.aa + 2 * L * AA_BYTES;
    s.ba = s.ab + 2 * AB_BYTES;
    s.bb = s.ba + BA_BYTES;
    s.tw = s.bb + 2 * BB_BYTES;
    s.bars = s.tw + ((TW_BYTES + 15) & ~15);
    s.tslot = s.bars + NBARS * 8;
    s.total = s.tslot + 16 + 1024;  // + alignment slack for the 1024-B swizzle atoms
    return s;
  }
};

enum { AA_FULL0, AA_FULL1, AA_EMPTY0, AA_EMPTY1, TA_FULL, TA_EMPTY, AB_FULL0, AB_FULL1, AB_EMPTY0, AB_EMPTY1,
       TB_FULL0, TB_FULL1, TB_EMPTY0, TB_EMPTY1 };

// debug timeline (CTA 0 only): role 0 producers, 1 MMA, 2 E_A, 3 E_B; events appended in order
__device__ __forceinline__ void trace(const TcFwdArgs& a, int role, int& n, bool leader) {
  if (a.trace && blockIdx.x == 0 && leader && n < TC_TRACE_N) a.trace[role * TC_TRACE_N + n] = clock64();
  ++n;
}

template <int L>
__global__ void __launch_bounds__(NTHREADS, 1)
    fwd_kernel(const __grid_constant__ RingConst rc, const __grid_constant__ TcFwdArgs a) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int prime = (int)(blockIdx.x / a.cpp), slot = (int)(blockIdx.x % a.cpp);
  const PrimeConst& pc = rc.pc[prime];
  const uint32_t p = pc.p, pinv = pc.pinv, mu = pc.mu;
  const int64_t npairs = (a.B + 1) / 2;

  const uint32_t raw = su32(smem_raw);
  unsigned char* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const Smem S = Smem::make(L);
  const uint32_t aa = su32(sm + S.aa), ab = su32(sm + S.ab), ba = su32(sm + S.ba), bb = su32(sm + S.bb);
  const uint2* tw = reinterpret_cast<const uint2*>(sm + S.tw);
  const uint32_t bars = su32(sm + S.bars);
  auto bar = [&](int i) { return bars + 8u * (uint32_t)i; };
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + S.tslot);

  // ---- setup: constant operands of this prime ----
  {
    const uint4* src = reinterpret_cast<const uint4*>(a.tabs + (size_t)prime * TAB_BYTES);
    uint4* dst = reinterpret_cast<uint4*>(sm + S.ba);  // BA | BB0 | BB1 | TW are contiguous
    for (int k = tid; k < TAB_BYTES / 16; k += NTHREADS) dst[k] = src[k];
  }
  if (tid == 0) {
    // arrivals per phase: epilogue warps, or one tcgen05.commit / expect_tx
    for (int i = 0; i < NBARS; ++i)
      mbar_init(bar(i), (i == TA_EMPTY || i == AB_FULL0 || i == AB_FULL1) ? (uint32_t)EA_WARPS
                        : (i == TB_EMPTY0 || i == TB_EMPTY1) ? (uint32_t)(EB_WARPS / 2) : 1u);  // per k1-half
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)),
                 "r"(512)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == LOAD_WARP) {
    // ------------------------------ loader: pass-A operand tiles of each rep (digits kernel) ------------------------------
    // the L digit tiles of (row pair, rep) are contiguous in the workspace: one bulk copy per rep
    // into the rep's buffer (two buffers, so the next rep streams in while this one is multiplied)
    uint32_t gr = 0;
    int tn = 0;
    if (lane == 0) {
      for (int64_t rp = slot; rp < npairs; rp += a.cpp) {
        for (int r = 0; r < a.nreps; ++r, ++gr) {
          const uint32_t b = gr & 1;
          mbar_wait_sleep(bar(AA_EMPTY0 + b), ((gr >> 1) & 1) ^ 1);
          trace(a, 0, tn, true);
          const uint32_t bytes = (uint32_t)(L * AA_BYTES);
          mbar_expect_tx(bar(AA_FULL0 + b), bytes);
          bulk_copy(aa + b * bytes, a.tiles + ((size_t)rp * a.nreps + r) * bytes, bytes, bar(AA_FULL0 + b));
        }
      }
    }
    __syncwarp();
  } else if (warp == MMA_WARP) {
    // ------------------------------ MMA issuer ------------------------------
    constexpr uint32_t idescA = (2u << 4) | (1u << 15) | ((uint32_t)(NA >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t idescB = (2u << 4) | (1u << 15) | ((uint32_t)(NBH >> 3) << 17) | ((128u >> 4) << 24);
    constexpr uint32_t kbA = (NA / 8) * 128, kbB = (NBH / 8) * 128;  // bytes per 16-row K block of B
    uint32_t g = 0, gr = 0;
    int tn = 0;
    auto issueB = [&](uint32_t gb) {
      const uint32_t buf = gb & 1;
      mbar_wait_sleep(bar(AB_FULL0 + buf), (gb >> 1) & 1);
      for (int h = 0; h < 2; ++h) {
        mbar_wait_sleep(bar(TB_EMPTY0 + h), (gb & 1) ^ 1);
        tc_fence_after();
        if (lane == 0) {
#pragma unroll
          for (int j = 0; j < KB / 32; ++j) {
            const uint64_t ad = sdesc(ab + buf * AB_BYTES + j * 4096, 16, 1024, 2);
            const uint64_t bd = sdesc(bb + h * BB_BYTES + 2 * j * kbB, kbB, 128, 0);
            mma_i8(tmem + (h ? COL_B1 : COL_B0), ad, bd, idescB, j > 0 ? 1u : 0u);
          }
          mma_commit(bar(TB_FULL0 + h));
        }
        __syncwarp();
      }
      if (lane == 0) mma_commit(bar(AB_EMPTY0 + buf));
      __syncwarp();
      trace(a, 1, tn, lane == 0);
    };
    for (int64_t rp = slot; rp < npairs; rp += a.cpp) {
      for (int r = 0; r < a.nreps; ++r, ++gr) {
        for (int i = 0; i < L; ++i, ++g) {
          const uint32_t ab_set = gr & 1;  // pass-A operand buffer of this rep
          if (i == 0) {
            if (g > 0) issueB(g - 1);  // before waiting on the next rep's operand tiles
            mbar_wait_sleep(bar(AA_FULL0 + ab_set), (gr >> 1) & 1);
          }
          mbar_wait_sleep(bar(TA_EMPTY), (g & 1) ^ 1);
          tc_fence_after();
          if (lane == 0) {
#pragma unroll
            for (int j = 0; j < KA / 32; ++j) {
              const uint64_t ad = sdesc(aa + (ab_set * L + i) * AA_BYTES + j * 4096, 16, 1024, 2);
              const uint64_t bd = sdesc(ba + 2 * j * kbA, kbA, 128, 0);
              mma_i8(tmem + COL_A, ad, bd, idescA, j > 0 ? 1u : 0u);
            }
            mma_commit(bar(TA_FULL));
            if (i == L - 1) mma_commit(bar(AA_EMPTY0 + ab_set));
          }
          __syncwarp();
          trace(a, 1, tn, lane == 0);
          if (i > 0) issueB(g - 1);
        }
      }
    }
    if (g > 0) issueB(g - 1);
  } else if (warp >= EB_WARPS && warp < LOAD_WARP) {
    // ------------------------------ E_A: pass A -> twiddle -> pass-B operand ------------------------------
    const int q = warp & 3, h = (warp - EB_WARPS) >> 2;
    const int s = q >> 1;
    const int m0 = (q & 1) ? 25 + lane : lane;
    const bool valid = (q & 1) ? lane < 24 : lane < 25;
    const uint2* twr = tw + (valid ? m0 : 0) * TWS;
    const uint32_t trow = tmem + ((uint32_t)(32 * q) << 16) + COL_A;
    uint32_t g = 0;
    int tn = 0;
    for (int64_t rp = slot; rp < npairs; rp += a.cpp) {
      for (int r = 0; r < a.nreps; ++r) {
        for (int i = 0; i < L; ++i, ++g) {
          const uint32_t buf = g & 1;
          mbar_wait_sleep(bar(TA_FULL), g & 1);
          tc_fence_after();
          trace(a, 2, tn, tid == EB_WARPS * 32);
          mbar_wait_sleep(bar(AB_EMPTY0 + buf), ((g >> 1) & 1) ^ 1);
          const uint32_t dst = ab + buf * AB_BYTES;
          {  // outputs o = 21 h + [0, 21) -> pass-B lanes 64 s + 32 h + [0, 21)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              uint32_t w[4][8];
#pragma unroll
              for (int pl = 0; pl < 4; ++pl) tmem_ld8(trow + (uint32_t)(pl * NAO + 21 * h + 8 * c), w[pl]);
              tmem_wait_ld();
              if (c == 2) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(bar(TA_EMPTY));
              }
              uint32_t y[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                const int o = 21 * h + 8 * c + u;
                const uint32_t lo = w[0][u] + (w[1][u] << 8), hi = w[2][u] + (w[3][u] << 8);
                const uint2 t2 = twr[o < SA ? o : 0];
                y[u] = redc((uint64_t)lo * t2.x + (uint64_t)hi * t2.y, p, pinv);
              }
              if (valid) {
                const uint32_t a0 = __byte_perm(y[0], y[1], 0x5140), b0 = __byte_perm(y[0], y[1], 0x7362);
                const uint32_t c0 = __byte_perm(y[2], y[3], 0x5140), d0 = __byte_perm(y[2], y[3], 0x7362);
                const uint32_t a1 = __byte_perm(y[4], y[5], 0x5140), b1 = __byte_perm(y[4], y[5], 0x7362);
                const uint32_t c1 = __byte_perm(y[6], y[7], 0x5140), d1 = __byte_perm(y[6], y[7], 0x7362);
                const int mlane = 64 * s + 32 * h + 8 * c;
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(swz(dst, 0 * SB + m0, mlane)),
                             "r"(__byte_perm(a0, c0, 0x5410)), "r"(__byte_perm(a1, c1, 0x5410)) : "memory");
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(swz(dst, 1 * SB + m0, mlane)),
                             "r"(__byte_perm(a0, c0, 0x7632)), "r"(__byte_perm(a1, c1, 0x7632)) : "memory");
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(swz(dst, 2 * SB + m0, mlane)),
                             "r"(__byte_perm(b0, d0, 0x5410)), "r"(__byte_perm(b1, d1, 0x5410)) : "memory");
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(swz(dst, 3 * SB + m0, mlane)),
                             "r"(__byte_perm(b0, d0, 0x7632)), "r"(__byte_perm(b1, d1, 0x7632)) : "memory");
              }
            }
          }
          fence_proxy_async();
          __syncwarp();
          if (lane == 0) mbar_arrive(bar(AB_FULL0 + buf));
          trace(a, 2, tn, tid == EB_WARPS * 32);
        }
      }
    }
  } else if (warp < EB_WARPS) {
    // ------------------------------ E_B: pass B -> key MAC -> accumulators ------------------------------
    const int q = warp & 3, h = warp >> 3, part = (warp >> 2) & 1;
    const int s = q >> 1;
    const int o = (q & 1) ? 21 + lane : lane;
    const bool valid = lane < 21;
    const int nk = h ? SB - K1H : K1H;  // 25 / 24 k1 values of this half; this warp: [12 part, ...)
    constexpr int KP = 13;              // keys per warp (12 or 13)
    const int c0 = part ? 3 : 0;
    const uint32_t lane_base = tmem + ((uint32_t)(32 * q) << 16);
    const uint32_t trow = lane_base + (h ? COL_B1 : COL_B0);
    const uint32_t acc_a_col = lane_base + COL_ACC_A + 28 * h, acc_b_col = lane_base + COL_ACC_B + 28 * h;
    uint32_t g = 0;
    int tn = 0;
    for (int64_t rp = slot; rp < npairs; rp += a.cpp) {
      const int64_t row = 2 * rp + s;
      for (int r = 0; r < a.nreps; ++r) {
        for (int i = 0; i < L; ++i, ++g) {
          // this step's key spectra (one 8-byte pair per k1), in flight while pass B runs
          const uint2* kt = a.keys[r] + ((size_t)(i * rc.np + prime) * SB + K1H * h + 12 * part) * SA + (valid ? o : 0);
          uint2 kv[KP];
#pragma unroll
          for (int k = 0; k < KP; ++k) kv[k] = 12 * part + k < nk ? __ldg(kt + (size_t)k * SA) : make_uint2(0, 0);
          const bool first = r == 0 && i == 0, last = r == a.nreps - 1 && i == L - 1;
          trace(a, 3, tn, tid == 0);
          mbar_wait_sleep(bar(TB_FULL0 + h), g & 1);
          tc_fence_after();
          trace(a, 3, tn, tid == 0);
          uint32_t* dst = a.acc + ((size_t)(row < a.B ? row : 0) * rc.np + prime) * 2 * N;
          const int32_t* oi = a.old_idx + (valid ? o : 0) * SB + K1H * h;
          const bool write = last && valid && row < a.B;
#pragma unroll
          for (int cc = 0; cc < 4; ++cc) {  // chunks of 4 k1: part 0 -> [0, 12), part 1 -> [12, 28)
            const int c = c0 + cc;
            if (!part && cc == 3) break;
            uint32_t w[4][4], ca[4], cb[4];
#pragma unroll
            for (int pl = 0; pl < 4; ++pl) tmem_ld4(trow + (uint32_t)(pl * KBH + 4 * c), w[pl]);
            if (!first) {
              tmem_ld4(acc_a_col + 4 * c, ca);
              tmem_ld4(acc_b_col + 4 * c, cb);
            }
            tmem_wait_ld();
            if (cc == (part ? 3 : 2)) {
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(bar(TB_EMPTY0 + h));
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int k = 4 * c + u, kk = 4 * cc + u;  // k1 - 25 h, key slot
              const uint32_t lo = w[0][u] + (w[1][u] << 8), hi = w[2][u] + (w[3][u] << 8);
              const uint32_t v = redc(((uint64_t)hi << 16) + lo, p, pinv);  // (A value) R^-1, < 2p
              const uint2 kk2 = kv[kk < KP ? kk : 0];
              uint32_t xa = redc((uint64_t)v * kk2.x, p, pinv);
              uint32_t xb = redc((uint64_t)v * kk2.y, p, pinv);
              if (!first) {
                xa += ca[u];
                xb += cb[u];
              }
              if (i == L - 1) {  // per rep: back to [0, 2p) so reps * digits terms stay below 2^32
                xa -= __umulhi(xa, mu) * p;
                xb -= __umulhi(xb, mu) * p;
              }
              ca[u] = xa;
              cb[u] = xb;
              if (write && k < nk) {  // last step of the pair: out to the CUDA-core kernel's NTT order
                const int pos = __ldg(oi + k);
                dst[pos] = xa;
                dst[N + pos] = xb;
              }
            }
            if (!last) {
              tmem_st4(acc_a_col + 4 * c, ca);
              tmem_st4(acc_b_col + 4 * c, cb);
            }
          }
          if (!last) tmem_wait_st();
          trace(a, 3, tn, tid == 0);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == MMA_WARP)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512) : "memory");
}

// Digits kernel: the pass-A operand tiles of every (row pair, rep, digit), already in the UMMA
// MN-major 128B-swizzled layout (K row kk, lane m at kk * 128 + ((m / 16) ^ (kk % 8)) * 16 + m % 16).
// K rows: plane 0 / 1 (low / high byte of digit + offset) of input q = j * 7 + m1 at q / 42 + q,
// row 84 all ones (offset correction), rows 85..95 zero.  Lane 64 s + (m0 < 25 ? m0 : m0 + 7) holds
// coefficient j * 343 + m1 * 49 + m0 of row s of the pair (other lanes zero).  One CTA per row
// pair, all reps: the automorphism gather (reference ring.py:101-130) reads the two staged rows,
// digits are the reference's balanced decomposition (crypto.py:288-323).
template <int L>
__global__ void __launch_bounds__(DIG_THREADS)
    digits_kernel(const __grid_constant__ RingConst rc, const __grid_constant__ TcFwdArgs a) {
  __shared__ __align__(16) uint64_t xs[2 * N];
  const int64_t rp = blockIdx.x;
  const int64_t row0 = 2 * rp;
  const int nrows = a.B - row0 < 2 ? (int)(a.B - row0) : 2;
  for (int s = 0; s < 2; ++s) {
    const uint4* src = reinterpret_cast<const uint4*>(a.in + (row0 + s) * 2 * (int64_t)N);
    uint4* dst = reinterpret_cast<uint4*>(xs + s * N);
    for (int k = threadIdx.x; k < N / 2; k += DIG_THREADS)
      dst[k] = s < nrows ? src[k] : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const uint32_t magic = rc.magicM;
  for (int r = 0; r < a.nreps; ++r) {
    const uint32_t dinv = a.dinv[r];
    unsigned char* tiles = a.tiles + ((size_t)rp * a.nreps + r) * L * AA_BYTES;
    // constant rows 84..95 of each digit tile
    for (int k = threadIdx.x; k < L * 12 * 8; k += DIG_THREADS) {
      const int i = k / 96, rr = 84 + (k % 96) / 8, c = k % 8;
      const uint32_t v = rr == 84 ? 0x01010101u : 0u;
      *reinterpret_cast<uint4*>(tiles + i * AA_BYTES + rr * 128 + c * 16) = make_uint4(v, v, v, v);
    }
    // work item (q, chunk c): 16 lanes of K rows q (plane 0) and 42 + q (plane 1) in every digit tile
    for (int it = threadIdx.x; it < SA * 8; it += DIG_THREADS) {
      const int q = it >> 3, c = it & 7;
      const int s = c >> 2, cc = c & 3;
      const int j = q / 7, m1 = q - 7 * j;
      uint32_t lo[L][4], hi[L][4];
#pragma unroll
      for (int i = 0; i < L; ++i)
#pragma unroll
        for (int w = 0; w < 4; ++w) lo[i][w] = hi[i][w] = 0u;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int ln = 16 * cc + u;
        const int m0 = ln < 32 ? ln : ln - 7;
        const bool lane_ok = ln < 32 ? m0 < 25 : ln < 56;
        if (!lane_ok) continue;
        uint64_t y = 0;
        if (s < nrows) {
          const uint32_t m = (uint32_t)(m1 * SB + m0);
          const uint32_t s1 = fastmod((uint32_t)(j * N1 + (int)m) * dinv, M, magic);
          const uint32_t s2 = fastmod((uint32_t)(N + m) * dinv, M, magic);
          const uint64_t* xr = xs + s * N;
          const uint64_t v1 = s1 < (uint32_t)N ? xr[s1] : 0ull;
          const uint64_t v2 = s2 < (uint32_t)N ? xr[s2] : 0ull;
          y = (v1 - v2) & QMASK;
        }
        int dg[L];
        decompose<L>(y, dg, rc);
#pragma unroll
        for (int i = 0; i < L; ++i) {
          const uint32_t ev = (uint32_t)(dg[i] + a.off);
          lo[i][u >> 2] |= (ev & 255u) << (8 * (u & 3));
          hi[i][u >> 2] |= (ev >> 8) << (8 * (u & 3));
        }
      }
      const int chunk = 4 * s + cc;  // 16-byte chunk of the 128-lane K row
#pragma unroll
      for (int i = 0; i < L; ++i) {
        unsigned char* t = tiles + i * AA_BYTES;
        *reinterpret_cast<uint4*>(t + q * 128 + ((chunk ^ (q & 7)) << 4)) =
            make_uint4(lo[i][0], lo[i][1], lo[i][2], lo[i][3]);
        const int kh = SA + q;
        *reinterpret_cast<uint4*>(t + kh * 128 + ((chunk ^ (kh & 7)) << 4)) =
            make_uint4(hi[i][0], hi[i][1], hi[i][2], hi[i][3]);
      }
    }
  }
}

// key spectra (CUDA-core kernel layout, K^ R mod p) -> per (slot, digit, prime) [k1][o] uint2
// (Ka R, Kb R) = K^ R^2 mod p in the tensor-core output order (E_B: REDC(REDC(value) * K R^2) = value * K^)
__global__ void keys_kernel(const __grid_constant__ RingConst rc, const uint32_t* spectra, int nslots,
                            const int32_t* old_idx, uint2* out) {
  const int64_t total = (int64_t)nslots * rc.l * rc.np * SB * SA;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    const int o = (int)(e % SA);
    int64_t r = e / SA;
    const int k1 = (int)(r % SB);
    r /= SB;
    const int pr = (int)(r % rc.np);
    r /= rc.np;
    const int i = (int)(r % rc.l);
    const int64_t slot = r / rc.l;
    const uint32_t p = rc.pc[pr].p;
    const uint64_t R = rc.pc[pr].rmod;
    const int f = old_idx[o * SB + k1];
    const int pos = (f % T) * rc.nitems + f / T;  // thread-owned layout of the spectra
    const uint32_t* base = spectra + (size_t)slot * rc.l * 2 * rc.np * N;
    const uint64_t ka = base[((size_t)(i * 2 + 0) * rc.np + pr) * N + pos];
    const uint64_t kb = base[((size_t)(i * 2 + 1) * rc.np + pr) * N + pos];
    out[e] = make_uint2((uint32_t)(ka * R % p), (uint32_t)(kb * R % p));
  }
}

}  // namespace tc7

// ---------------------------------------------------------------------------
// host side

static uint64_t tc_powmod(uint64_t b, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  b %= m;
  while (e) {
    if (e & 1) r = (unsigned __int128)r * b % m;
    b = (unsigned __int128)b * b % m;
    e >>= 1;
  }
  return r;
}

bool tc_supported(const RingConst& rc) { return rc.t == 7 && rc.alpha == 4 && (rc.l == 2 || rc.l == 3); }

size_t tc_table_bytes(const RingConst& rc) { return (size_t)rc.np * tc7::TAB_BYTES; }

int tc_digit_offset(const RingConst& rc) {
  const int D = rc.D;
  return (D & (D - 1)) == 0 ? D / 2 - 1 : D / 2;
}

// canonical K-major (no swizzle) byte offset of element (k, n) in a [K][Ncols] u8 operand
static size_t kmaj(int k, int n, int ncols) {
  return ((size_t)(k / 16) * (ncols / 8) + n / 8) * 128 + (n % 8) * 16 + (k % 16);
}

void tc_build_tables(const RingConst& rc, const uint32_t* twid, int twid_stride_words, uint8_t* tabs,
                     int32_t* old_idx) {
  using namespace tc7;
  const int off = tc_digit_offset(rc);
  for (int pr = 0; pr < rc.np; ++pr) {
    const uint64_t p = rc.pc[pr].p;
    const uint64_t R = (1ull << 32) % p;
    const uint64_t Rinv = tc_powmod(R, p - 2, p);
    const uint64_t omega = (uint64_t)twid[(size_t)pr * twid_stride_words + 1] * Rinv % p;
    std::vector<uint64_t> pw(M);
    pw[0] = 1;
    for (int e = 1; e < M; ++e) pw[e] = (unsigned __int128)pw[e - 1] * omega % p;
    uint8_t* base = tabs + (size_t)pr * TAB_BYTES;
    std::memset(base, 0, TAB_BYTES);
    uint8_t* BA = base;
    uint8_t* BB = base + BA_BYTES;
    uint32_t* TW = reinterpret_cast<uint32_t*>(base + BA_BYTES + 2 * BB_BYTES);
    // pass A: rows (plane, q = j*7 + m1) and the ones row; columns b * 44 + o
    for (int o = 0; o < SA; ++o) {
      const int r = o / 7 + 1, k0 = o % 7;
      uint64_t rowsum = 0;
      for (int qq = 0; qq < SA; ++qq) {
        const int j = qq / 7, m1 = qq % 7;
        const uint64_t w = pw[((uint64_t)N1 * r * j + (uint64_t)SB * m1 * (r + 7 * k0)) % M];
        rowsum = (rowsum + w) % p;
        for (int plane = 0; plane < 2; ++plane) {
          const uint64_t c = plane ? (w << 8) % p : w;
          for (int b = 0; b < 4; ++b) BA[kmaj(plane * SA + qq, b * NAO + o, NA)] = (uint8_t)(c >> (8 * b));
        }
      }
      const uint64_t corr = (p - (uint64_t)off % p * rowsum % p) % p;
      for (int b = 0; b < 4; ++b) BA[kmaj(2 * SA, b * NAO + o, NA)] = (uint8_t)(corr >> (8 * b));
      // twiddles omega^((r + 7 k0) m0) * R, and * 2^16
      for (int m0 = 0; m0 < SB; ++m0) {
        const uint64_t tv = pw[((uint64_t)(r + 7 * k0) * m0) % M] * R % p;
        TW[2 * (m0 * TWS + o)] = (uint32_t)tv;
        TW[2 * (m0 * TWS + o) + 1] = (uint32_t)((tv << 16) % p);
      }
    }
    // pass B: rows (plane, m0), columns (half h) b * 28 + (k1 - 25 h)
    for (int k1 = 0; k1 < SB; ++k1) {
      const int h = k1 >= K1H, kl = k1 - K1H * h;
      for (int m0 = 0; m0 < SB; ++m0) {
        const uint64_t w = pw[((uint64_t)49 * k1 * m0) % M];
        for (int plane = 0; plane < 4; ++plane) {
          const uint64_t c = (w << (8 * plane)) % p;
          for (int b = 0; b < 4; ++b)
            BB[h * BB_BYTES + kmaj(plane * SB + m0, b * KBH + kl, NBH)] = (uint8_t)(c >> (8 * b));
        }
      }
    }
  }
  // NTT-domain position of (o, k1) in the CUDA-core kernel's order: block r-1, digit-reversed k
  for (int o = 0; o < SA; ++o)
    for (int k1 = 0; k1 < SB; ++k1) {
      const int r = o / 7 + 1, k = o % 7 + 7 * k1;
      const int rev = (k % 7) * 49 + ((k / 7) % 7) * 7 + k / 49;
      old_idx[o * SB + k1] = (r - 1) * N1 + rev;
    }
}

size_t tc_fwd_smem_bytes(int L) { return (size_t)tc7::Smem::make(L).total; }

size_t tc_tile_bytes(const RingConst& rc, int64_t rows, int nreps) {
  return (size_t)((rows + 1) / 2) * nreps * rc.l * tc7::AA_BYTES;
}

cudaError_t launch_tc_fwd(const RingConst& rc, const TcFwdArgs& a, cudaStream_t st) {
  if (a.B <= 0 || a.nreps <= 0) return cudaSuccess;
  {
    const unsigned pairs = (unsigned)((a.B + 1) / 2);
    if (rc.l == 3)
      tc7::digits_kernel<3><<<pairs, tc7::DIG_THREADS, 0, st>>>(rc, a);
    else
      tc7::digits_kernel<2><<<pairs, tc7::DIG_THREADS, 0, st>>>(rc, a);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const size_t smem = tc_fwd_smem_bytes(rc.l);
  const int64_t npairs = (a.B + 1) / 2;
  TcFwdArgs b = a;
  static int nsm = 0;  // per process: one device model
  static cudaError_t attr = [&] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaError_t e = cudaFuncSetAttribute(tc7::fwd_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tc_fwd_smem_bytes(3));
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(tc7::fwd_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)tc_fwd_smem_bytes(2));
    return e;
  }();
  if (attr != cudaSuccess) return attr;
  const int per_prime = nsm / rc.np;
  b.cpp = (int)(npairs < per_prime ? npairs : per_prime);
  const dim3 grid((unsigned)(b.cpp * rc.np));
  if (rc.l == 3)
    tc7::fwd_kernel<3><<<grid, tc7::NTHREADS, smem, st>>>(rc, b);
  else
    tc7::fwd_kernel<2><<<grid, tc7::NTHREADS, smem, st>>>(rc, b);
  return cudaGetLastError();
}

cudaError_t launch_tc_keys(const RingConst& rc, const uint32_t* spectra, int nslots, const int32_t* old_idx,
                           uint2* out, cudaStream_t st) {
  if (nslots <= 0) return cudaSuccess;
  tc7::keys_kernel<<<256, 256, 0, st>>>(rc, spectra, nslots, old_idx, out);
  return cudaGetLastError();
}

size_t tc_keys_bytes(const RingConst& rc, int nslots) {
  return (size_t)nslots * rc.l * rc.np * tc7::SB * tc7::SA * 8;
}

}  // namespace sfhr
