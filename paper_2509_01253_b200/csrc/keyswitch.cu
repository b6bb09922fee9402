// Fused hoisted key-switch stage kernel (sm_100a).
//
// Semantics (reference pkg/src/sfhr/tracepack.py:268-285 with
// crypto.py:288-323, 400-464): for each input row x = (a, b) and the stage's
// switched representatives r_1..r_T (automorphism index d_r, key set K_r):
//
//   y_r          = aut_{d_r}(x)                          (ring.py:101-130)
//   dig_{r,i}    = balanced base-D digit i of y_r.a       (crypto.py:288-323)
//   A            = sum_r sum_i dig_{r,i} * K_r[i].a  mod Phi_M
//   B            = sum_r sum_i dig_{r,i} * K_r[i].b  mod Phi_M
//   out.a        = [identity] * x.a - A                  (mod 2^53)
//   out.b        = [identity] * x.b + sum_r y_r.b - B    (mod 2^53)
//
// which is acc = x + sum_r KS_r(aut_r(x)) for a stage, and the plain
// switch_batch (one rep, d_r = 1, no identity term) otherwise.
//
// Device design: one thread-block CLUSTER per row, one CTA per CRT prime.
// Per rep, a CTA
//   A. gathers aut_{d_r}(x.a) from the row staged in shared memory and
//      decomposes every coefficient into its l balanced digits (balanced over
//      all N coefficients), lifted mod p into the l transform buffers;
//   B. runs the first Phi_M-NTT step in place, then the radix-t DIF stages of
//      all l digit transforms together (one barrier per stage);
//   C. computes the last (span-1) butterflies in registers and multiply-
//      accumulates them against the precomputed key spectra (thread-owned
//      layout => coalesced) into NTT-domain accumulators in shared memory.
// Reps are summed in the NTT domain, so a row needs only 2 inverse
// transforms per prime.  The CTAs of the cluster then exchange residues
// through distributed shared memory and each reconstructs a 1/NP slice of
// the row by explicit CRT mod 2^53.
#include <cooperative_groups.h>

#include "sfhr_common.cuh"
#include "sfhr_kernels.h"

#ifndef SFHR_FUSED_FIRST_STEP
#define SFHR_FUSED_FIRST_STEP 1
#endif
// row prologue by bulk copies (one elected thread, one mbarrier) instead of a 16-byte
// load/store loop per thread: the mask and the twiddle tables arrive in one round trip
#ifndef SFHR_STAGE_BULK
#define SFHR_STAGE_BULK 1
#endif
// L2 CRT path: the body x.b is bulk-copied into the dead accumulator region while the inverse
// transforms run, and the identity term reads the staged mask, so the last arriver's body
// gathers and identity loads hit shared memory instead of global
#ifndef SFHR_BODY_STAGE
#define SFHR_BODY_STAGE 1
#endif

namespace cg = cooperative_groups;

namespace sfhr {

// ---------------------------------------------------------------------------
// geometry: compile-time when the tower height A is a template argument

__host__ __device__ __forceinline__ constexpr int cpow(int b, int e) {
  int r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

template <int T, int A>
struct Geo {
  const int alpha, M, n1, N, nitems;
  __device__ __forceinline__ explicit Geo(const RingConst& rc)
      : alpha(A ? A : rc.alpha),
        M(A ? cpow(T, A) : rc.M),
        n1(A ? cpow(T, A - 1) : rc.n1),
        N(A ? cpow(T, A - 1) * (T - 1) : rc.N),
        nitems(A ? cpow(T, A - 1) * (T - 1) / T : rc.nitems) {}
};

#ifndef SFHR_T7_THREADS
#define SFHR_T7_THREADS 384
#endif
#ifndef SFHR_T5_THREADS
#define SFHR_T5_THREADS 512
#endif
#ifndef SFHR_T5_MINBLOCKS
#define SFHR_T5_MINBLOCKS 2
#endif
#ifndef SFHR_T7_MINBLOCKS
#define SFHR_T7_MINBLOCKS 3
#endif
template <int T>
struct StageLaunch {
  static constexpr int kThreads = T == 7 ? SFHR_T7_THREADS : T == 5 ? SFHR_T5_THREADS : 512;
  static constexpr int kMinBlocks = T == 7 ? SFHR_T7_MINBLOCKS : T == 5 ? SFHR_T5_MINBLOCKS : 2;
};

// block size: the launch-bound constant for the compile-time geometries (stage_threads launches
// them with exactly kThreads), so block-strided loops have compile-time trip counts.  At t = 7
// (56-register cap) the compiler would unroll them into ~1 KB of spills, so there they stay
// rolled (SFHR_T7_LOOP); SFHR_BDIM_T7=0 keeps blockDim.x for t = 7
#ifndef SFHR_BDIM_T7
#define SFHR_BDIM_T7 1
#endif
// with the constant stride at t = 7 the block-strided loops are kept rolled (the unrolled ones spill)
#if SFHR_BDIM_T7
#define SFHR_T7_LOOP _Pragma("unroll 1")
#else
#define SFHR_T7_LOOP
#endif
// the flat mid-stage loops (t = 7) -- A/B knob SFHR_T7_MID_UNROLL2: unrolled by 2
#if SFHR_BDIM_T7 && SFHR_T7_MID_UNROLL2
#define SFHR_T7_MID_LOOP _Pragma("unroll 2")
#else
#define SFHR_T7_MID_LOOP SFHR_T7_LOOP
#endif
// x mod M: a constant division for the compile-time geometries (SFHR_CT_MOD; -0.1 %)
#ifndef SFHR_CT_MOD
#define SFHR_CT_MOD 1
#endif
template <int T, int A>
__device__ __forceinline__ uint32_t mod_m(uint32_t x, const RingConst& rc) {
  if constexpr (A != 0 && SFHR_CT_MOD) return x % (uint32_t)cpow(T, A);
  else return fastmod(x, (uint32_t)rc.M, rc.magicM);
}
template <int T, int A>
__device__ __forceinline__ int bdim() {
  return A && (T != 7 || SFHR_BDIM_T7) ? StageLaunch<T>::kThreads : (int)blockDim.x;
}

// ---------------------------------------------------------------------------
// small DFT helper (constants come from the __grid_constant__ parameter block
// at compile-time offsets -> uniform-register operands of IMAD.WIDE.U32)

// Barrett step to [0, 2p) (A/B knob: the 32-bit-multiply form bred or umulhi by floor(2^32 / p))
#ifndef SFHR_BRED
#define SFHR_BRED 1
#endif
__device__ __forceinline__ uint32_t bar(uint32_t y, const PrimeConst& pc) {
  return SFHR_BRED ? bred(y, pc.p, pc.bc) : y - __umulhi(y, pc.mu) * pc.p;
}

template <int T>
__device__ __forceinline__ void dft_t(const uint32_t (&x)[T], uint32_t (&y)[T],
                                      const uint32_t (&Z)[MAXT][MAXT], uint32_t p, uint32_t pinv) {
#pragma unroll
  for (int k = 0; k < T; ++k) {
    uint64_t s = 0;
#pragma unroll
    for (int m = 0; m < T; ++m) s += (uint64_t)x[m] * Z[k][m];
    y[k] = redc(s, p, pinv);
  }
}

// Symmetric-pair radix-t DFT.  With a_m = x_m + x_{t-m} and b_m = x_m - x_{t-m}
// (m = 1..H, H = (t-1)/2), P_k = sum_m a_m c_km and Q_k = sum_m b_m s_km
// (c, s = (zeta^km +- zeta^-km) / 2):  y_k = x_0 + P_k + Q_k, y_{t-k} = x_0 + P_k - Q_k
// (signs of Q swapped for the inverse), so 2 H^2 products replace t^2 (18 vs 49
// at t = 7).  Inputs in [0, 2p); y_0 returned in [0, 2p); y_k in [0, 6p), or in
// [0, 2p) when RED.  Ranges (checked by the planner): 4 H p < 2^32, 2 t p < 2^32.
template <int T, bool INV, bool RED>
__device__ __forceinline__ void dft_sym(const uint32_t (&x)[T], uint32_t (&y)[T], const PrimeConst& pc) {
  constexpr int H = (T - 1) / 2;
  const uint32_t p = pc.p, pinv = pc.pinv, p2 = 2 * p, mu = pc.mu;
  uint32_t a[H], b[H];
  uint32_t y0 = x[0];
#pragma unroll
  for (int m = 1; m <= H; ++m) {
    a[m - 1] = x[m] + x[T - m];
    b[m - 1] = x[m] + p2 - x[T - m];
    y0 += a[m - 1];
  }
  y[0] = bar(y0, pc);
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    uint64_t sp = 0, sq = 0;
#pragma unroll
    for (int m = 1; m <= H; ++m) {
      sp += (uint64_t)a[m - 1] * pc.hc[k - 1][m - 1];
      sq += (uint64_t)b[m - 1] * pc.hs[k - 1][m - 1];
    }
    const uint32_t P = redc(sp, p, pinv), Q = redc(sq, p, pinv);
    const uint32_t t0 = x[0] + P;
    uint32_t u = t0 + Q, v = t0 + p2 - Q;
    if (RED) {
      u = bar(u, pc);
      v = bar(v, pc);
    }
    y[k] = INV ? v : u;
    y[T - k] = INV ? u : v;
  }
}

#ifndef SFHR_SYM_DFT
#define SFHR_SYM_DFT 1
#endif
#ifndef SFHR_WINO7
#define SFHR_WINO7 1
#endif
#ifndef SFHR_WINO5
#define SFHR_WINO5 1
#endif
#ifndef SFHR_WINO7_INV1
#define SFHR_WINO7_INV1 1
#endif
// the two single-product Rader terms (M0 = S mu, R2 = Tm rho) as Shoup products: IMAD.HI + 2 IMAD
// against IMAD.WIDE + IMAD + IMAD.HI (plan.cpp bounds both by 2p)
#ifndef SFHR_WINO_SHOUP
#define SFHR_WINO_SHOUP 1
#endif
#ifndef SFHR_WINO_KARA
#define SFHR_WINO_KARA 0
#endif
// the 2x2 blocks of the Rader DFTs: g = [[a00, a01], [a10, a00]] (A0, A1), h likewise with b,
// Karatsuba (3 IMAD.WIDE per pair instead of 4; operand ranges unchanged, see WinoConst)
__device__ __forceinline__ void wino_g(int32_t A0, int32_t A1, const WinoConst& w, uint32_t p, uint32_t pinv,
                                       uint32_t& g0, uint32_t& g1) {
  if (SFHR_WINO_KARA) {
    const int64_t P = (int64_t)(A0 - A1) * w.a00;
    g0 = redc((uint64_t)((int64_t)w.kG + P + (int64_t)A1 * w.ka01), p, pinv);
    g1 = redc((uint64_t)((int64_t)w.kG - P + (int64_t)A0 * w.ka10), p, pinv);
  } else {
    g0 = redc((uint64_t)((int64_t)w.kG + (int64_t)A0 * w.a00 + (int64_t)A1 * w.a01), p, pinv);
    g1 = redc((uint64_t)((int64_t)w.kG + (int64_t)A0 * w.a10 + (int64_t)A1 * w.a00), p, pinv);
  }
}
__device__ __forceinline__ void wino_h(int32_t C0, int32_t C1, const WinoConst& w, uint32_t p, uint32_t pinv,
                                       uint32_t& h0, uint32_t& h1) {
  if (SFHR_WINO_KARA) {
    const int64_t P = (int64_t)(C0 + C1) * w.b00;
    h0 = redc((uint64_t)((int64_t)w.kG + P + (int64_t)C1 * w.kb01), p, pinv);
    h1 = redc((uint64_t)((int64_t)w.kG + P + (int64_t)C0 * w.kb10), p, pinv);
  } else {
    h0 = redc((uint64_t)((int64_t)w.kG + (int64_t)C0 * w.b00 + (int64_t)C1 * w.b01), p, pinv);
    h1 = redc((uint64_t)((int64_t)w.kG + (int64_t)C0 * w.b10 + (int64_t)C1 * w.b00), p, pinv);
  }
}
__device__ __forceinline__ uint32_t wino_m0(uint32_t S, const WinoConst& w, uint32_t p, uint32_t pinv) {
  return SFHR_WINO_SHOUP ? shoup_mul(S, make_uint2(w.mu_w, w.mu_q), p) : redc((uint64_t)S * w.mu, p, pinv);
}
__device__ __forceinline__ uint32_t wino_r2(int32_t Tm, const WinoConst& w, uint32_t p, uint32_t pinv) {
  return SFHR_WINO_SHOUP ? shoup_mul((uint32_t)(Tm + (int32_t)w.toff), make_uint2(w.rho_w, w.rho_q), p)
                         : redc((uint64_t)((int64_t)w.kT + (int64_t)Tm * w.rho), p, pinv);
}
// lazy ranges (A/B knobs): inverse DFT outputs that feed a twiddle multiply stay unreduced
// (the next stage Barrett-reduces only its x_0); the last forward stage feeds the key MAC
// unreduced when l >= 3 (one REDC + Barrett per accumulator instead of one Barrett per digit)
#ifndef SFHR_LAZY_INV
#define SFHR_LAZY_INV 1
#endif
#ifndef SFHR_LAZY_MAC
#define SFHR_LAZY_MAC 1
#endif

// Rader/Winograd radix-7 DFT (constants and range proof: plan.cpp build_wino7).  The integer
// multiply (fmaheavy) pipe bounds the stage kernel, so products are what to save: 10 IMAD.WIDE
// + 6 REDC against 18 + 6 for dft_sym; the reconstruction adds run on the ALU pipe.
// Inputs in [0, 2p); y_0 returned in [0, 2p), y_k < 2^32 (or [0, 2p) when RED).
template <bool INV, bool RED>
__device__ __forceinline__ void dft_wino7(const uint32_t (&x)[7], uint32_t (&y)[7], const PrimeConst& pc) {
  const WinoConst& w = pc.wino[INV ? 1 : 0];
  const uint32_t p = pc.p, pinv = pc.pinv, mu = pc.mu;
  // v_j = x_{5^j mod 7}
  const uint32_t v0 = x[1], v1 = x[5], v2 = x[4], v3 = x[6], v4 = x[2], v5 = x[3];
  const uint32_t p03 = v0 + v3, p14 = v1 + v4, p25 = v2 + v5;                       // [0, 4p)
  const int32_t d03 = (int32_t)(v0 - v3), d14 = (int32_t)(v1 - v4), d25 = (int32_t)(v2 - v5);  // (-2p, 2p)
  const uint32_t S = p03 + p14 + p25;                                               // V(1)
  const int32_t Tm = d03 - d14 + d25;                                               // V(-1)
  const int32_t A0 = (int32_t)(p03 - p25), A1 = (int32_t)(p14 - p25);               // V mod X^2+X+1
  const int32_t C0 = d03 - d25, C1 = d14 + d25;                                     // V mod X^2-X+1
  const uint32_t M0 = wino_m0(S, w, p, pinv);
  const uint32_t R2 = wino_r2(Tm, w, p, pinv);
  uint32_t g0, g1, h0, h1;
  wino_g(A0, A1, w, p, pinv, g0, g1);
  wino_h(C0, C1, w, p, pinv, h0, h1);
  // z_i = x_0 + M0 + (-1)^i R2 + g_{i mod 3} +- h_{i mod 3} (g_2 = -g_0 - g_1, h_2 = h_1 - h_0,
  // h negated for i >= 3), mod 2^32 arithmetic whose true values are non-negative
  const uint32_t X0 = x[0] + M0, Xp = X0 + R2, Xm = X0 - R2;
  const uint32_t gs = g0 + g1, hd = h1 - h0;
  uint32_t z[6];
  z[0] = Xp + g0 + h0;
  z[1] = Xm + w.k1p + g1 + h1;
  z[2] = Xp + w.k3p - gs + hd;
  z[3] = Xm + w.k2p + g0 - h0;
  z[4] = Xp + w.k4p + g1 - h1;
  z[5] = Xm + w.k5p - gs - hd;
  const uint32_t y0 = x[0] + S;
  y[0] = bar(y0, pc);
  // outputs y_{3^i mod 7}
  constexpr int kout[6] = {1, 3, 2, 6, 4, 5};
#pragma unroll
  for (int i = 0; i < 6; ++i) y[kout[i]] = RED ? bar(z[i], pc) : z[i];
}

// forward DFT whose k >= 1 outputs are multiplied by twiddles next (lazy [0, 6p) ok)
// Inverse first step of the t = 7 transform (plan.cpp build_wino7_invfirst): with Y the inverse
// 7-point DFT of (0, C_1..C_6), out_j = s (Y_j - Y_6) = sum_r C_r g[j][r]; the Winograd form of
// Y_j - Y_6 drops M0 and needs 10 products instead of the matrix's 36.  Inputs C < 2p; outputs
// in [0, p) (the CRT-weighted residues).
__device__ __forceinline__ void inv_first7(const uint32_t (&C)[6], uint32_t (&o)[6], const PrimeConst& pc) {
  const WinoConst& w = pc.wino[2];
  const uint32_t p = pc.p, pinv = pc.pinv, mu = pc.mu;
  // v_j = c_{5^j mod 7} with c_r = C[r - 1]
  const uint32_t v0 = C[0], v1 = C[4], v2 = C[3], v3 = C[5], v4 = C[1], v5 = C[2];
  const uint32_t p03 = v0 + v3, p14 = v1 + v4, p25 = v2 + v5;
  const int32_t d03 = (int32_t)(v0 - v3), d14 = (int32_t)(v1 - v4), d25 = (int32_t)(v2 - v5);
  const uint32_t S = p03 + p14 + p25;
  const int32_t Tm = d03 - d14 + d25;
  const int32_t A0 = (int32_t)(p03 - p25), A1 = (int32_t)(p14 - p25);
  const int32_t C0 = d03 - d25, C1 = d14 + d25;
  const uint32_t S7 = wino_m0(S, w, p, pinv);  // 7 s S / 6
  const uint32_t R2 = wino_r2(Tm, w, p, pinv);
  uint32_t g0, g1, h0, h1;
  wino_g(A0, A1, w, p, pinv, g0, g1);
  wino_h(C0, C1, w, p, pinv, h0, h1);
  uint32_t z[6];
  z[0] = S7 + R2 + h0 + w.k1p - g0;
  z[1] = 2 * (R2 + h0);
  z[2] = 2 * R2 + h1 + w.k2p - 2 * g0 - g1;
  z[3] = g1 + h1 + h0 + w.k3p - g0;
  z[4] = 2 * R2 + g1 + h0 + w.k4p - h1 - g0;
  z[5] = 2 * h0 + w.k5p - 2 * g0 - g1 - h1;
#pragma unroll
  for (int j = 0; j < 6; ++j) o[j] = fully(bar(z[j], pc), p);
}

// Rader radix-5 DFT (plan.cpp build_wino5): 6 IMAD.WIDE + 4 REDC against 8 + 4 for dft_sym.
// Inputs in [0, 2p); y_0 in [0, 2p), y_k < 2^32 (or [0, 2p) when RED).
template <bool INV, bool RED>
__device__ __forceinline__ void dft_wino5(const uint32_t (&x)[5], uint32_t (&y)[5], const PrimeConst& pc) {
  const WinoConst& w = pc.wino[INV ? 1 : 0];
  const uint32_t p = pc.p, pinv = pc.pinv, mu = pc.mu;
  const uint32_t v0 = x[1], v1 = x[3], v2 = x[4], v3 = x[2];  // v_j = x_{3^j mod 5}
  const uint32_t S = v0 + v1 + v2 + v3;
  const int32_t Tm = (int32_t)(v0 - v1 + v2 - v3);  // V(-1), (-4p, 4p)
  const int32_t A0 = (int32_t)(v0 - v2), A1 = (int32_t)(v1 - v3);  // V mod X^2 + 1
  const uint32_t M0 = wino_m0(S, w, p, pinv);
  const uint32_t R2 = wino_r2(Tm, w, p, pinv);
  uint32_t g0, g1;
  wino_g(A0, A1, w, p, pinv, g0, g1);
  const uint32_t X0 = x[0] + M0, Xp = X0 + R2, Xm = X0 - R2;
  uint32_t z[4];
  z[0] = Xp + g0;
  z[1] = Xm + w.k1p + g1;
  z[2] = Xp + w.k2p - g0;
  z[3] = Xm + w.k3p - g1;
  const uint32_t y0 = x[0] + S;
  y[0] = bar(y0, pc);
  constexpr int kout[4] = {1, 2, 4, 3};  // outputs y_{2^i mod 5}
#pragma unroll
  for (int i = 0; i < 4; ++i) y[kout[i]] = RED ? bar(z[i], pc) : z[i];
}

template <int T>
__device__ __forceinline__ void dft_fwd_tw(const uint32_t (&x)[T], uint32_t (&y)[T], const PrimeConst& pc) {
  if constexpr (T == 7 && SFHR_WINO7) dft_wino7<false, false>(x, y, pc);
  else if constexpr (T == 5 && SFHR_WINO5) dft_wino5<false, false>(x, y, pc);
  else if (SFHR_SYM_DFT) dft_sym<T, false, false>(x, y, pc);
  else dft_t<T>(x, y, pc.z, pc.p, pc.pinv);
}
// forward / inverse DFT with every output in [0, 2p)
template <int T>
__device__ __forceinline__ void dft_fwd_red(const uint32_t (&x)[T], uint32_t (&y)[T], const PrimeConst& pc) {
  if constexpr (T == 7 && SFHR_WINO7) dft_wino7<false, true>(x, y, pc);
  else if constexpr (T == 5 && SFHR_WINO5) dft_wino5<false, true>(x, y, pc);
  else if (SFHR_SYM_DFT) dft_sym<T, false, true>(x, y, pc);
  else dft_t<T>(x, y, pc.z, pc.p, pc.pinv);
}
template <int T>
__device__ __forceinline__ void dft_inv_red(const uint32_t (&x)[T], uint32_t (&y)[T], const PrimeConst& pc) {
  if constexpr (T == 7 && SFHR_WINO7) dft_wino7<true, true>(x, y, pc);
  else if constexpr (T == 5 && SFHR_WINO5) dft_wino5<true, true>(x, y, pc);
  else if (SFHR_SYM_DFT) dft_sym<T, true, true>(x, y, pc);
  else dft_t<T>(x, y, pc.zi, pc.p, pc.pinv);
}
// inverse DFT whose k >= 1 outputs are only ever multiplied by a twiddle next (y_0 in [0, 2p),
// y_k < 2^32): every consumer either Montgomery-multiplies an input (any a < 2^32 keeps
// a * bm < p 2^32) or Barrett-reduces it first (the x_0 of the next inverse stage)
template <int T>
__device__ __forceinline__ void dft_inv_lazy(const uint32_t (&x)[T], uint32_t (&y)[T], const PrimeConst& pc) {
  if constexpr (T == 7 && SFHR_WINO7) dft_wino7<true, false>(x, y, pc);
  else if constexpr (T == 5 && SFHR_WINO5) dft_wino5<true, false>(x, y, pc);
  else if (SFHR_SYM_DFT) dft_sym<T, true, false>(x, y, pc);
  else dft_t<T>(x, y, pc.zi, pc.p, pc.pinv);
}
template <int T>
__device__ __forceinline__ void dft_inv(const uint32_t (&x)[T], uint32_t (&y)[T], const PrimeConst& pc) {
  if (SFHR_LAZY_INV) dft_inv_lazy<T>(x, y, pc);
  else dft_inv_red<T>(x, y, pc);
}

__device__ __forceinline__ uint32_t lift_signed(int d, uint32_t p) {
  return d < 0 ? (uint32_t)(d + (int)p) : (uint32_t)d;
}

// bulk-copy helpers (cp.async.bulk completes on an mbarrier; sizes and addresses are 16-byte
// multiples: rows are 2N u64 with N even, the twiddle rows are padded to 4 words)
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void row_bulk(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(dst),
               "l"(src), "r"(bytes), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void row_bar_expect(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void row_bar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  }
}

// ---------------------------------------------------------------------------
// transform building blocks over nb buffers of N words each (block-wide)

// forward first step, in place: buf[q-1][m] = omega^{q m} sum_{j<T-1} zeta^{q j} buf[j][m]
template <int T, int A, int PR>
__device__ __forceinline__ void fwd_first_step(uint32_t* buf, int nb, const RingConst& rc,
                                               const uint32_t* wt) {
  const PrimeConst& pc = rc.pc[PR];
  const Geo<T, A> g(rc);
  for (int w = threadIdx.x; w < g.n1 * nb; w += bdim<T, A>()) {
    const int i = w / g.n1, m = w - i * g.n1;
    uint32_t* v = buf + i * g.N + m;
    uint32_t vals[T - 1];
#pragma unroll
    for (int j = 0; j < T - 1; ++j) vals[j] = v[j * g.n1];
#pragma unroll
    for (int q = 1; q < T; ++q) {
      uint64_t s = 0;
#pragma unroll
      for (int j = 0; j < T - 1; ++j) s += (uint64_t)vals[j] * pc.z[q][j];
      v[(q - 1) * g.n1] = mont_mul(redc(s, pc.p, pc.pinv), wt[q * m], pc.p, pc.pinv);
    }
  }
  __syncthreads();
}

// digits of the key MAC loop: unrolled at t = 7 (the next digit's key-spectrum loads issue during
// this digit's DFT: ResNet-20 stage -2.6 %, no spills), rolled at t = 3 / 5 (+2.9 % at t = 5).
// SFHR_MAC_UNROLL = 0: rolled everywhere
#ifndef SFHR_MAC_UNROLL
#define SFHR_MAC_UNROLL 1
#endif
template <int T, int L>
constexpr int kMacUnroll = SFHR_MAC_UNROLL && T == 7 ? L : 1;

// lazy MAC pays off from three digits on (one Barrett per accumulator vs one per digit)
template <int L>
constexpr bool kLazyMac = SFHR_LAZY_MAC && L >= 3;

// mid-stage work order: item-major (one item's index math for all digit buffers) for t <= 5
template <int T>
constexpr bool kItemMajor = T <= 5;

#ifndef SFHR_SHOUP_MID
#define SFHR_SHOUP_MID 1
#endif
// twiddles loaded before the item's DFT instead of between its stores (the compiler cannot hoist
// shared loads above stores to the transform buffer it cannot prove disjoint): the LDS latency
// overlaps the DFT instead of stalling the twiddle multiplies
#ifndef SFHR_TW_EARLY
#define SFHR_TW_EARLY 1
#endif

// forward DIF stages s = 0 .. alpha-3 (all but the last, span > 1).  SH: twiddles from the Shoup
// pairs sh[e / t] (every mid-stage exponent is a multiple of t) instead of the Montgomery table
template <int T, int A, int PR, bool SH = false, int SKIP = 0>
__device__ __forceinline__ void fwd_mid_stages(uint32_t* buf, int nb, const RingConst& rc,
                                               const uint32_t* wt, const uint2* sh = nullptr) {
  const PrimeConst& pc = rc.pc[PR];
  const Geo<T, A> g(rc);
  const int nsub = g.n1 / T;
#pragma unroll
  for (int s = 0; s < (A ? A - 2 - SKIP : 16); ++s) {
    if (!A && s >= g.alpha - 2 - SKIP) break;
    const int L = A ? cpow(T, A - 2 - s) : nsub / cpow(T, s);
    const int step = g.M / (T * L);
    const int stepT = step / T;  // exact: L <= n1 / T
    auto item = [&](uint32_t* v, const int j) {
      const int e1 = step * j;
      uint32_t x[T], y[T];
      if constexpr (SH && SFHR_TW_EARLY) {
        const int es = stepT * j;  // e1 / t
        uint2 tw[T];
#pragma unroll
        for (int k = 1; k < T; ++k) tw[k] = sh[es * k];
#pragma unroll
        for (int m = 0; m < T; ++m) x[m] = v[m * L];
        dft_fwd_tw<T>(x, y, pc);
        v[0] = y[0];
#pragma unroll
        for (int k = 1; k < T; ++k) v[k * L] = shoup_mul(y[k], tw[k], pc.p);
        return;
      }
#pragma unroll
      for (int m = 0; m < T; ++m) x[m] = v[m * L];
      dft_fwd_tw<T>(x, y, pc);
      v[0] = y[0];
      if constexpr (SH) {
        const int es = stepT * j;  // e1 / t
#pragma unroll
        for (int k = 1; k < T; ++k) v[k * L] = shoup_mul(y[k], sh[es * k], pc.p);
      } else {
#pragma unroll
        for (int k = 1; k < T; ++k) v[k * L] = mont_mul(y[k], wt[e1 * k], pc.p, pc.pinv);
      }
    };
    if constexpr (kItemMajor<T>) {
      // item-major, buffers inner: position and twiddle exponent computed once for all nb
      // transforms (A/B on B200: t = 5 stage kernel -6 %; t = 7 +3 %, so t = 7 stays flat)
      for (int it = threadIdx.x; it < g.nitems; it += bdim<T, A>()) {
        const int sub = it / nsub, rem = it - sub * nsub;
        const int b = rem / L, j = rem - b * L;
        const int off = sub * g.n1 + b * T * L + j;
#pragma unroll 1
        for (int q = 0; q < nb; ++q) item(buf + q * g.N + off, j);
      }
    } else {
      // w = q nitems + sub nsub + b L + j; with N = (T-1) n1 the buffer offset
      // q N + sub n1 + b T L + j is P n1 + r + b (T-1) L for P = w / nsub, r = w mod nsub
      // (two constant divisions instead of three; none at the first stage, where L = nsub)
      SFHR_T7_MID_LOOP
      for (int w = threadIdx.x; w < g.nitems * nb; w += bdim<T, A>()) {
        const int P = w / nsub, r = w - P * nsub;
        const int b = L == nsub ? 0 : r / L, j = r - b * L;
        item(buf + P * g.n1 + r + b * (T - 1) * L, j);
      }
    }
    __syncthreads();
  }
}

// The last mid stage (span L = T) fused with the last stage + key MAC (SFHR_FUSE_LAST_MID): a
// group of T lanes of one warp owns a T x T block of every digit transform -- its T mid-stage
// items (offset j, stride T), then, after a __syncwarp, its T MAC items (rows of the block) --
// so no CTA barrier separates the two phases.  Shoup twiddles loaded ahead (SH + TW_EARLY form).
// Measured slower on B200 (ResNet-20 stage 109.95 vs 105.79 ms: the mid-stage items run on 11
// of 12 warps with 28 of 32 lanes instead of all 384 threads, and spills grow), so off.
#ifndef SFHR_FUSE_LAST_MID
#define SFHR_FUSE_LAST_MID 0
#endif
template <int T, int A, int PR>
__device__ __forceinline__ void fwd_last_mid_item(uint32_t* v, const int j, const RingConst& rc, const uint2* sh) {
  const PrimeConst& pc = rc.pc[PR];
  const Geo<T, A> g(rc);
  const int es = g.M / (T * T * T) * j;  // (step / t) j with step = M / t^2
  uint2 tw[T];
#pragma unroll
  for (int k = 1; k < T; ++k) tw[k] = sh[es * k];
  uint32_t x[T], y[T];
#pragma unroll
  for (int m = 0; m < T; ++m) x[m] = v[m * T];
  dft_fwd_tw<T>(x, y, pc);
  v[0] = y[0];
#pragma unroll
  for (int k = 1; k < T; ++k) v[k * T] = shoup_mul(y[k], tw[k], pc.p);
}

// inverse DIT stages s = alpha-3 .. 0 (the span-1 stage is undone in registers)
template <int T, int A, int PR, bool SH = false>
__device__ __forceinline__ void inv_mid_stages(uint32_t* buf, int nb, const RingConst& rc,
                                               const uint32_t* wt, const uint2* sh = nullptr) {
  const PrimeConst& pc = rc.pc[PR];
  const Geo<T, A> g(rc);
  const int nsub = g.n1 / T;
#pragma unroll
  for (int si = 0; si < (A ? A - 2 : 16); ++si) {
    if (!A && si >= g.alpha - 2) break;
    const int L = cpow(T, si + 1);
    const int step = g.M / (T * L);
    const int stepT = step / T;
    auto item = [&](uint32_t* v, const int j) {
      const int e1 = step * j;
      uint32_t z[T], x[T];
      // lazy: v[0] is some earlier stage's unreduced output (< 2^32)
      z[0] = SFHR_LAZY_INV ? bar(v[0], pc) : v[0];
      if constexpr (SH) {
        const int es = stepT * j;  // omega^(M - e1 k) = sh[n1 - es k]
#pragma unroll
        for (int k = 1; k < T; ++k) z[k] = shoup_mul(v[k * L], sh[g.n1 - es * k], pc.p);
      } else {
#pragma unroll
        for (int k = 1; k < T; ++k) z[k] = mont_mul(v[k * L], wt[g.M - e1 * k], pc.p, pc.pinv);
      }
      dft_inv<T>(z, x, pc);
#pragma unroll
      for (int m = 0; m < T; ++m) v[m * L] = x[m];
    };
    if constexpr (kItemMajor<T>) {
      for (int it = threadIdx.x; it < g.nitems; it += bdim<T, A>()) {
        const int sub = it / nsub, rem = it - sub * nsub;
        const int b = rem / L, j = rem - b * L;
        const int off = sub * g.n1 + b * T * L + j;
#pragma unroll 1
        for (int q = 0; q < nb; ++q) item(buf + q * g.N + off, j);
      }
    } else {
      // w = q nitems + sub nsub + b L + j; with N = (T-1) n1 the buffer offset
      // q N + sub n1 + b T L + j is P n1 + r + b (T-1) L for P = w / nsub, r = w mod nsub
      // (two constant divisions instead of three; none at the first stage, where L = nsub)
      SFHR_T7_MID_LOOP
      for (int w = threadIdx.x; w < g.nitems * nb; w += bdim<T, A>()) {
        const int P = w / nsub, r = w - P * nsub;
        const int b = L == nsub ? 0 : r / L, j = r - b * L;
        item(buf + P * g.n1 + r + b * (T - 1) * L, j);
      }
    }
    __syncthreads();
  }
}

// inverse first step: untwist + (t-1)x(t-1) solve, writes CRT-weighted y_i in [0, p)
template <int T, int A, int PR>
__device__ __forceinline__ void inv_first_step(uint32_t* buf, int nb, const RingConst& rc,
                                               const uint32_t* wt) {
  const PrimeConst& pc = rc.pc[PR];
  const Geo<T, A> g(rc);
  auto untwist = [&](const int w) {
    const int q = w / g.n1, m = w - q * g.n1;
    uint32_t* v = buf + q * g.N + m;
    uint32_t C[T - 1];
#pragma unroll
    for (int r = 1; r < T; ++r) C[r - 1] = mont_mul(v[(r - 1) * g.n1], wt[g.M - r * m], pc.p, pc.pinv);
    if constexpr (T == 7 && SFHR_WINO7 && SFHR_WINO7_INV1) {
      uint32_t o[6];
      inv_first7(C, o, pc);
#pragma unroll
      for (int j = 0; j < 6; ++j) v[j * g.n1] = o[j];
    } else {
#pragma unroll
      for (int j = 0; j < T - 1; ++j) {
        uint64_t s = 0;
#pragma unroll
        for (int r = 0; r < T - 1; ++r) s += (uint64_t)C[r] * pc.g[j][r];
        v[j * g.n1] = fully(redc(s, pc.p, pc.pinv), pc.p);
      }
    }
  };
  if constexpr (T == 7) {
    SFHR_T7_LOOP
    for (int w = threadIdx.x; w < g.n1 * nb; w += bdim<T, A>()) untwist(w);
  } else {
    for (int w = threadIdx.x; w < g.n1 * nb; w += bdim<T, A>()) untwist(w);
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// the fused stage kernel

struct SmemLayout {
  uint64_t* xa;   // (N,) staged mask component of the row
  uint32_t* wt;   // (M+1,) Montgomery twiddles of this CTA's prime
  uint2* sh;      // (n1+1,) Shoup pairs of the exponents t i (mid-stage twiddles)
  uint32_t* acc;  // (2, N) NTT-domain accumulators, summed over reps
  uint32_t* buf;  // (nb, N) transform buffers
};

// the mask buffer doubles as the CRT receive buffer [np][2][per] u32 (per = ceil(N / np))
// (32-bit arithmetic: a 64-bit division by the runtime np cost ~2 % of the kernel's instructions)
__host__ __device__ __forceinline__ size_t xa_region_bytes(const RingConst& rc) {
  const unsigned per = ((unsigned)rc.N + (unsigned)rc.np - 1u) / (unsigned)rc.np;
  const unsigned recv = (unsigned)rc.np * 2u * per * 4u, mask = (unsigned)rc.N * 8u;
  return (size_t)(((recv > mask ? recv : mask) + 15u) & ~15u);
}

__device__ __forceinline__ SmemLayout carve(unsigned char* smem, const RingConst& rc) {
  SmemLayout s;
  s.xa = reinterpret_cast<uint64_t*>(smem);
  s.wt = reinterpret_cast<uint32_t*>(smem + xa_region_bytes(rc));
  s.sh = reinterpret_cast<uint2*>(s.wt + twid_stride(rc.M));
  s.acc = s.wt + twid_stride(rc.M) + shoup_stride(rc.n1);
  s.buf = s.acc + 2 * rc.N;
  return s;
}

// CRT primes of the compile-time (production) geometries: the planner gives 3 for every preset
// row; launch_stage takes the A != 0 specialisation only when rc.np matches, so the stage
// kernel's per-CTA divisions by np and the shared-memory carve-up fold to constants
constexpr int kProdNP = 3;
template <int T, int A>
__device__ __forceinline__ int stage_np(const RingConst& rc) { return A ? kProdNP : rc.np; }

// gadget base of the preset rows by (t, alpha, l): b=8 (512, 3); b=12
// (4096, 3) at gamma = 0 and (2^16, 2) above; b=16 (310, 5) / (310, 4).  0: runtime gadget.
// launch_stage takes the A != 0 specialisation only when rc.D matches
template <int T, int A, int L>
__host__ __device__ constexpr int prod_gadget_D() {
  return !A ? 0
         : T == 7 && A == 4 ? (L == 3 ? 4096 : L == 2 ? 65536 : 0)
         : T == 5 && A == 5 ? (L == 5 || L == 4 ? 310 : 0)
         : T == 3 && A == 7 ? (L == 3 ? 512 : 0)
         : 0;
}
__host__ __device__ constexpr int ilog2c(int v) { return v <= 1 ? 0 : 1 + ilog2c(v / 2); }

// balanced digits with the gadget as compile-time constants when the geometry fixes it
template <int T, int A, int L>
__device__ __forceinline__ void decompose_t(uint64_t y, int (&dg)[L], const RingConst& rc) {
  constexpr int DC = prod_gadget_D<T, A, L>();
  if constexpr (DC == 0) {
    decompose<L>(y, dg, rc);
  } else if constexpr ((DC & (DC - 1)) == 0) {
    constexpr int w = ilog2c(DC), shift = 53 - w * L;
    uint64_t u = (y + (1ull << (shift - 1))) >> shift;
    int carry = 0;
#pragma unroll
    for (int i = L - 1; i >= 0; --i) {
      const int x = (int)(u & (uint64_t)(DC - 1)) + carry;
      u >>= w;
      carry = x > (DC >> 1);
      dg[i] = carry ? x - DC : x;
    }
  } else {
    long long r = (long long)y;
    if (y > (1ull << 52)) r -= (1ll << 53);
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const long long prod = r * DC;
      const long long d = (prod + (1ll << 52)) >> 53;
      dg[i] = (int)d;
      r = prod - d * (1ll << 53);
    }
  }
}

template <int T, int A>
__device__ __forceinline__ SmemLayout carve_t(unsigned char* smem, const RingConst& rc) {
  const Geo<T, A> g(rc);
  const unsigned np = (unsigned)stage_np<T, A>(rc);
  const unsigned per = ((unsigned)g.N + np - 1u) / np;
  const unsigned recv = np * 2u * per * 4u, mask = (unsigned)g.N * 8u;
  const unsigned xa = ((recv > mask ? recv : mask) + 15u) & ~15u;
  SmemLayout s;
  s.xa = reinterpret_cast<uint64_t*>(smem);
  s.wt = reinterpret_cast<uint32_t*>(smem + xa);
  s.sh = reinterpret_cast<uint2*>(s.wt + twid_stride(g.M));
  s.acc = s.wt + twid_stride(g.M) + shoup_stride(g.n1);
  s.buf = s.acc + 2 * g.N;
  return s;
}

// bulk-copy completion state of a CTA across its rows: bar_mask completes the row prologue (or
// the previous row's prefetch of this row's mask), bar_body the body copy of the L2 CRT path
struct RowSync {
  uint32_t bar_mask, bar_body;
  uint32_t ph_mask, ph_body;  // parity of the next phase to wait for
  bool prefetched;            // this row's mask was issued by the previous row
};

#ifndef SFHR_PREFETCH_NEXT
#define SFHR_PREFETCH_NEXT 1
#endif

template <int T, int A, int L, int PR>
__device__ __forceinline__ void stage_row(const RingConst& rc, const StageArgs& a, unsigned char* smem,
                                          const int64_t row, const bool stage_twiddles, RowSync& sync,
                                          const int64_t next_row = -1, const int split = 0) {
  const PrimeConst& pc = rc.pc[PR];
  const uint32_t p = pc.p, pinv = pc.pinv, mu = pc.mu;
  const Geo<T, A> g(rc);
  const int N = g.N, n1 = g.n1, M = g.M;
  SmemLayout S = carve_t<T, A>(smem, rc);
  const int np = stage_np<T, A>(rc);
  const size_t crw = ((size_t)np * 2 * N + 31) & ~(size_t)31;  // crt_row_words
  const uint64_t* xin = a.in + row * 2 * (int64_t)N;
  uint64_t* xout = a.out + row * 2 * (int64_t)N;
  cg::cluster_group cluster = cg::this_cluster();

  // stage x.a (16-byte loads) and the twiddle table; detect an all-zero row
  // (the body is only read when the mask is all zero, which is rare)
  int nz = 0;
  __shared__ int last_s;
  const uint32_t row_bar = sync.bar_mask;
  if (SFHR_STAGE_BULK) {
    // the CTA's first row initialises the barriers; the copies are issued before the CTA barrier
    // that publishes the init, so they overlap it
    if (threadIdx.x == 0 && stage_twiddles) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sync.bar_mask) : "memory");
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(sync.bar_body) : "memory");
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    }
    if (threadIdx.x == 0 && !sync.prefetched) {
      const uint32_t xb = (uint32_t)N * 8u;
      const uint32_t wb = stage_twiddles ? (uint32_t)twid_stride(M) * 4u : 0u;
      const uint32_t hb = stage_twiddles && SFHR_SHOUP_MID ? (uint32_t)shoup_stride(n1) * 4u : 0u;
      row_bar_expect(row_bar, xb + wb + hb);
      row_bulk(smem_addr(S.xa), xin, xb, row_bar);
      if (wb) row_bulk(smem_addr(S.wt), a.twid + (size_t)PR * twid_stride(M), wb, row_bar);
      if (hb)
        row_bulk(smem_addr(S.sh), a.twid + (size_t)np * twid_stride(M) + (size_t)PR * shoup_stride(n1), hb,
                 row_bar);
    }
    if (stage_twiddles) __syncthreads();  // the barriers' init is visible
    row_bar_wait(row_bar, sync.ph_mask);
    sync.ph_mask ^= 1u;
    sync.prefetched = false;
    const uint4* src = reinterpret_cast<const uint4*>(S.xa);
    for (int c = threadIdx.x; c < N / 2; c += bdim<T, A>()) {
      const uint4 v = src[c];
      nz |= (v.x | v.y | v.z | v.w) != 0;
    }
  } else {
    const uint4* src = reinterpret_cast<const uint4*>(xin);  // rows are 16-byte aligned (N even)
    uint4* dst = reinterpret_cast<uint4*>(S.xa);
    for (int c = threadIdx.x; c < N / 2; c += bdim<T, A>()) {
      const uint4 v = src[c];
      dst[c] = v;
      nz |= (v.x | v.y | v.z | v.w) != 0;
    }
  }
  if (stage_twiddles && !SFHR_STAGE_BULK) {
    const uint4* wsrc = reinterpret_cast<const uint4*>(a.twid + (size_t)PR * twid_stride(M));
    uint4* wdst = reinterpret_cast<uint4*>(S.wt);
    for (int k = threadIdx.x; k < twid_stride(M) / 4; k += bdim<T, A>()) wdst[k] = wsrc[k];
    if (SFHR_SHOUP_MID) {
      const uint4* hsrc = reinterpret_cast<const uint4*>(a.twid + (size_t)np * twid_stride(M) +
                                                         (size_t)PR * shoup_stride(n1));
      uint4* hdst = reinterpret_cast<uint4*>(S.sh);
      for (int k = threadIdx.x; k < shoup_stride(n1) / 4; k += bdim<T, A>()) hdst[k] = hsrc[k];
    }
  }
  int live = __syncthreads_or(nz);
  if (!live) {
    for (int k = threadIdx.x; k < N; k += bdim<T, A>()) nz |= xin[N + k] != 0;
    live = __syncthreads_or(nz);
  }
  const int per = (N + np - 1) / np;
  const int k0 = PR * per, k1 = min(N, k0 + per);
  // this cluster's representatives (all of them unless the launch splits them, acc_out); the
  // split launch counts its own reps, so the acc_in launch that sums the partials does not
  const int nsp = a.acc_out && a.nsplit > 1 ? a.nsplit : 1;
  const int rb = split * a.nreps / nsp, re = (split + 1) * a.nreps / nsp;
  const bool counts = !(a.acc_in && a.nsplit > 1);
  if (!live) {
    if (!a.acc_out)
      for (int k = k0 + threadIdx.x; k < k1; k += bdim<T, A>()) {
        xout[k] = 0;
        xout[N + k] = 0;
      }
    if (PR == 0 && threadIdx.x == 0 && a.counter && !a.skip_zero && counts)
      atomicAdd(a.counter, (unsigned long long)(re - rb));
    return;  // uniform across the cluster: every CTA saw the same row
  }
  if (PR == 0 && threadIdx.x == 0 && a.counter && counts) atomicAdd(a.counter, (unsigned long long)(re - rb));

  const int item = threadIdx.x;
  const bool owner = item < g.nitems;

  if (a.acc_in) {
    // NTT-domain accumulators come from the tensor-core forward kernel (keyswitch_tc.cu) or
    // from the nsplit partial sums of a representative-split launch (each < 2 p reps_s: the
    // total stays below 2 p nreps, as in one pass)
    const int parts = a.nsplit > 1 ? a.nsplit : 1;
    uint4* dst = reinterpret_cast<uint4*>(S.acc);
    for (int c = threadIdx.x; c < N / 2; c += bdim<T, A>()) {  // 2N u32 = N/2 uint4
      uint4 v = make_uint4(0, 0, 0, 0);
      for (int q = 0; q < parts; ++q) {
        const uint4 w = reinterpret_cast<const uint4*>(a.acc_in + (((size_t)row * parts + q) * np + PR) * 2 * N)[c];
        v.x += w.x;
        v.y += w.y;
        v.z += w.z;
        v.w += w.w;
      }
      dst[c] = v;
    }
    if (!a.independent) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    __syncthreads();
  }
  for (int r = rb; r < (a.acc_in ? rb : re); ++r) {
    const uint32_t dinv = a.dinv[r];
#if SFHR_FUSED_FIRST_STEP
    // ---- A+B fused: per column m, gather the T-1 coefficients j*n1+m of
    // aut(x.a), decompose them (carry chain, all digits), and run the first
    // transform step for every digit straight from registers ----
    {
      const uint32_t step1 = mod_m<T, A>((uint32_t)n1 * dinv, rc);
      auto column = [&](const int m) {
        const uint32_t s2 = mod_m<T, A>((uint32_t)(N + m) * dinv, rc);
        const uint64_t v2 = s2 < (uint32_t)N ? S.xa[s2] : 0ull;
        uint32_t s1 = mod_m<T, A>((uint32_t)m * dinv, rc);
        int dg[L][T - 1];
        uint32_t tw[T];  // first-step twists omega^(q m), shared by the l digit transforms
        if (SFHR_TW_EARLY) {
#pragma unroll
          for (int q = 1; q < T; ++q) tw[q] = S.wt[q * m];
        }
#pragma unroll
        for (int j = 0; j < T - 1; ++j) {
          const uint64_t v1 = s1 < (uint32_t)N ? S.xa[s1] : 0ull;
          int d[L];
          decompose_t<T, A, L>((v1 - v2) & QMASK, d, rc);
#pragma unroll
          for (int i = 0; i < L; ++i) dg[i][j] = d[i];
          s1 += step1;
          if (s1 >= (uint32_t)M) s1 -= M;
        }
#pragma unroll
        for (int i = 0; i < L; ++i) {
          uint32_t vals[T - 1];
#pragma unroll
          for (int j = 0; j < T - 1; ++j) vals[j] = lift_signed(dg[i][j], p);
          uint32_t* o = S.buf + i * N + m;
#if SFHR_SYM_DFT
          uint32_t xv[T], yq[T];
#pragma unroll
          for (int j = 0; j < T - 1; ++j) xv[j] = vals[j];
          xv[T - 1] = 0;
          dft_fwd_tw<T>(xv, yq, pc);
#pragma unroll
          for (int q = 1; q < T; ++q) o[(q - 1) * n1] = mont_mul(yq[q], SFHR_TW_EARLY ? tw[q] : S.wt[q * m], p, pinv);
#else
#pragma unroll
          for (int q = 1; q < T; ++q) {
            uint64_t s = 0;
#pragma unroll
            for (int j = 0; j < T - 1; ++j) s += (uint64_t)vals[j] * pc.z[q][j];
            o[(q - 1) * n1] = mont_mul(redc(s, p, pinv), S.wt[q * m], p, pinv);
          }
#endif
        }
      };
      if constexpr (T == 7) {
        SFHR_T7_LOOP
        for (int m = threadIdx.x; m < n1; m += bdim<T, A>()) column(m);
      } else {
        for (int m = threadIdx.x; m < n1; m += bdim<T, A>()) column(m);
      }
      __syncthreads();
    }
#else
    // ---- A: automorphism gather + digits of every coefficient ----
    for (int k = threadIdx.x; k < N; k += bdim<T, A>()) {
      const uint32_t km = (uint32_t)(k % n1);
      const uint32_t s1 = fastmod((uint32_t)k * dinv, M, rc.magicM);
      const uint32_t s2 = fastmod((uint32_t)(N + km) * dinv, M, rc.magicM);
      uint64_t y = s1 < (uint32_t)N ? S.xa[s1] : 0ull;
      if (s2 < (uint32_t)N) y -= S.xa[s2];
      int dg[L];
      decompose_t<T, A, L>(y & QMASK, dg, rc);
#pragma unroll
      for (int i = 0; i < L; ++i) S.buf[i * N + k] = lift_signed(dg[i], p);
    }
    __syncthreads();
    // ---- B: first step + mid stages of the l digit transforms ----
    fwd_first_step<T, A, PR>(S.buf, L, rc, S.wt);
#endif
    // the mask is dead after the last rep's gathers: prefetch the CTA's next row into it
    if (SFHR_STAGE_BULK && SFHR_PREFETCH_NEXT && next_row >= 0 && r == re - 1 && a.crt_scratch && !a.acc_out) {
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads of S.xa before
        row_bar_expect(sync.bar_mask, (uint32_t)N * 8u);
        row_bulk(smem_addr(S.xa), a.in + next_row * 2 * (int64_t)N, (uint32_t)N * 8u, sync.bar_mask);
      }
      sync.prefetched = true;
    }
    constexpr bool kFuse = SFHR_FUSE_LAST_MID && T == 7 && A >= 3 && SFHR_SHOUP_MID && SFHR_TW_EARLY &&
                           !kItemMajor<T>;
    fwd_mid_stages<T, A, PR, SFHR_SHOUP_MID, kFuse ? 1 : 0>(S.buf, L, rc, S.wt, S.sh);
#ifdef SFHR_T7_THREADS
    static_assert(!kFuse || A != 4 || SFHR_T7_THREADS >= 352, "the fused MAC needs 42 groups of 7 lanes");
#endif
    int mac_item = item;
    bool mac_owner = owner;
    if constexpr (kFuse) {
      constexpr int GPW = 32 / T;  // groups per warp
      const int lane = threadIdx.x & 31, grp = (threadIdx.x >> 5) * GPW + lane / T, j = lane % T;
      mac_owner = lane < GPW * T && grp < g.nitems / T;
      mac_item = grp * T + j;
      if (mac_owner) {
#pragma unroll 1
        for (int i = 0; i < L; ++i) fwd_last_mid_item<T, A, PR>(S.buf + i * N + grp * T * T + j, j, rc, S.sh);
      }
      __syncwarp();
    }
    // the staged mask is dead after the last rep's gathers: tell the peers they may push
    // their CRT residues into it (the matching wait precedes our own pushes)
    if (r == a.nreps - 1 && !a.independent) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    // ---- C: last stage (span 1) in registers, MAC against the key spectra ----
    if (mac_owner) {
      const int item = mac_item;
      const uint32_t* ks = a.spec[r];
      uint64_t ta[T], tb[T];
#pragma unroll
      for (int k = 0; k < T; ++k) ta[k] = tb[k] = 0;
#pragma unroll(kMacUnroll<T, L>)
      for (int i = 0; i < L; ++i) {
        const uint32_t* v = S.buf + i * N + item * T;
        uint32_t x[T], yv[T];
#pragma unroll
        for (int m = 0; m < T; ++m) x[m] = v[m];
        if constexpr (kLazyMac<L>) dft_fwd_tw<T>(x, yv, pc);  // y_k < 2^32
        else dft_fwd_red<T>(x, yv, pc);
        const uint32_t* ka = ks + ((size_t)(i * 2 + 0) * np + PR) * N + item;
        const uint32_t* kb = ks + ((size_t)(i * 2 + 1) * np + PR) * N + item;
#pragma unroll
        for (int k = 0; k < T; ++k) {
          ta[k] += (uint64_t)yv[k] * __ldg(ka + k * g.nitems);
          tb[k] += (uint64_t)yv[k] * __ldg(kb + k * g.nitems);
        }
      }
      // L products of (<2p)(<p) < p 2^32 (p < 2^31/L): one REDC each; sum over reps < 2 reps p.
      // Lazy MAC: L products of (<2^32)(<p) < L p 2^32 (< 2^64): the REDC lands in (0, (L+1) p)
      // (< 2^32), one Barrett step brings it to [0, 2p)
      uint32_t* aa = S.acc + item * T;
      uint32_t* ab = S.acc + N + item * T;
#pragma unroll
      for (int k = 0; k < T; ++k) {
        uint32_t ra = redc(ta[k], p, pinv), rb2 = redc(tb[k], p, pinv);
        if constexpr (kLazyMac<L>) {
          ra = bar(ra, pc);
          rb2 = bar(rb2, pc);
        }
        aa[k] = r > rb ? aa[k] + ra : ra;
        ab[k] = r > rb ? ab[k] + rb2 : rb2;
      }
    }
    __syncthreads();
  }

  if (a.acc_out) {  // representative split: hand this cluster's partial sums to the acc_in launch
    uint4* dst = reinterpret_cast<uint4*>(
        a.acc_out + (((size_t)row * (a.nsplit > 1 ? a.nsplit : 1) + split) * np + PR) * 2 * N);
    const uint4* src = reinterpret_cast<const uint4*>(S.acc);
    for (int c = threadIdx.x; c < N / 2; c += bdim<T, A>()) dst[c] = src[c];
    return;
  }

  // ---- inverse transforms of the two accumulators (buffers 0: a, 1: b) ----
  if (owner) {
    uint32_t za[T], zb[T], xa[T], xb[T];
#pragma unroll
    for (int k = 0; k < T; ++k) {
      const uint32_t va = S.acc[item * T + k], vb = S.acc[N + item * T + k];
      za[k] = bar(va, pc);  // -> [0, 2p)
      zb[k] = bar(vb, pc);
    }
    dft_inv<T>(za, xa, pc);
    dft_inv<T>(zb, xb, pc);
#pragma unroll
    for (int m = 0; m < T; ++m) {
      S.buf[item * T + m] = xa[m];
      S.buf[N + item * T + m] = xb[m];
    }
  }
  __syncthreads();
  // the accumulators are dead: stage the body x.b (N u64 = the 2N u32 of S.acc) behind the
  // inverse transforms (every CTA waits for it before it exits: the copy targets its smem)
  constexpr bool kBodyStage = SFHR_BODY_STAGE && SFHR_STAGE_BULK;
  const bool body_staged = kBodyStage && a.crt_scratch != nullptr;
  if (body_staged && threadIdx.x == 0) {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic reads of S.acc before
    row_bar_expect(sync.bar_body, (uint32_t)N * 8u);
    row_bulk(smem_addr(S.acc), xin + N, (uint32_t)N * 8u, sync.bar_body);
  }
  inv_mid_stages<T, A, PR, SFHR_SHOUP_MID>(S.buf, 2, rc, S.wt, S.sh);
  inv_first_step<T, A, PR>(S.buf, 2, rc, S.wt);
  const uint64_t* xbs = reinterpret_cast<const uint64_t*>(S.acc);  // staged body (body_staged)

  // body term x.b + sum_r aut_r(x.b) of coefficient k, gathered from global
  auto body_sum = [&](const int k) -> uint64_t {
    uint64_t bsum = a.identity ? xin[N + k] : 0ull;
    const uint32_t kmod = (uint32_t)(k % n1);
#if SFHR_BODY_UNROLL
    // every rep's two gathers in flight before the first add (the loop was latency-serialised)
    uint64_t g1[SFHR_BODY_UNROLL], g2[SFHR_BODY_UNROLL];
    for (int r0 = 0; r0 < a.nreps; r0 += SFHR_BODY_UNROLL) {
#pragma unroll
      for (int u = 0; u < SFHR_BODY_UNROLL; ++u) {
        g1[u] = g2[u] = 0ull;
        if (r0 + u < a.nreps) {
          const uint32_t dinv = a.dinv[r0 + u];
          const uint32_t s1 = fastmod((uint32_t)k * dinv, M, rc.magicM);
          const uint32_t s2 = fastmod((uint32_t)(N + kmod) * dinv, M, rc.magicM);
          if (s1 < (uint32_t)N) g1[u] = xin[N + s1];
          if (s2 < (uint32_t)N) g2[u] = xin[N + s2];
        }
      }
#pragma unroll
      for (int u = 0; u < SFHR_BODY_UNROLL; ++u) bsum += g1[u] - g2[u];
    }
#else
    for (int r = 0; r < a.nreps; ++r) {
      const uint32_t dinv = a.dinv[r];
      const uint32_t s1 = fastmod((uint32_t)k * dinv, M, rc.magicM);
      const uint32_t s2 = fastmod((uint32_t)(N + kmod) * dinv, M, rc.magicM);
      uint64_t v = s1 < (uint32_t)N ? xin[N + s1] : 0ull;
      if (s2 < (uint32_t)N) v -= xin[N + s2];
      bsum += v;
    }
#endif
    return bsum;
  };
  // explicit CRT of coefficient k from the np CRT-weighted residues (ya_i, yb_i)
  auto crt_out = [&](const int k, const uint32_t* ya, const uint32_t* yb, const uint64_t bsum,
                     const bool xa_staged = false) {
    uint64_t ua = 0, ub = 0;
    double fa = 0.0, fb = 0.0;
#pragma unroll
    for (int i = 0; i < MAXNP; ++i) {
      if (i < np) {
        ua += (uint64_t)ya[i] * rc.pc[i].q_mod64;
        ub += (uint64_t)yb[i] * rc.pc[i].q_mod64;
        fa += (double)ya[i] * rc.pc[i].inv_p;
        fb += (double)yb[i] * rc.pc[i].inv_p;
      }
    }
    const uint64_t Av = ua - (uint64_t)__double2ll_rn(fa) * rc.P_mod64;
    const uint64_t Bv = ub - (uint64_t)__double2ll_rn(fb) * rc.P_mod64;
    xout[k] = ((a.identity ? (xa_staged ? S.xa[k] : xin[k]) : 0ull) - Av) & QMASK;
    xout[N + k] = (bsum - Bv) & QMASK;
  };

  if (a.crt_scratch) {
    // ---- CRT through L2 (independent CTAs, no cluster): every CTA stores its residues of the
    // whole row, and the last of the row's np CTAs to arrive (device-scope counter) combines
    // them, adds the body term and writes the row; the others exit at once ----
    uint32_t* rs = a.crt_scratch + (size_t)row * crw;
    {
      uint4* mine = reinterpret_cast<uint4*>(rs + (size_t)PR * 2 * N);
      const uint4* src = reinterpret_cast<const uint4*>(S.buf);
      for (int c = threadIdx.x; c < N / 2; c += bdim<T, A>()) mine[c] = src[c];  // 2N u32
    }
    // release: the barrier orders the CTA's stores before thread 0's gpu-scope fence (cumulative)
    __syncthreads();
    if (threadIdx.x == 0) {
      // acq_rel: releases this CTA's residues and, for the last arriver, acquires the peers'
      unsigned old;
      asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(old) : "l"(a.crt_cnt + row) : "memory");
      last_s = old == (unsigned)(np - 1);
    }
    __syncthreads();
    if (body_staged) {  // every CTA: the copy targets its smem
      row_bar_wait(sync.bar_body, sync.ph_body);
      sync.ph_body ^= 1u;
    }
    if (!last_s) return;
    // staged body term x.b + sum_r aut_r(x.b) of coefficient k (shared-memory gathers)
    auto body_sum_s = [&](const int k) -> uint64_t {
      uint64_t bsum = a.identity ? xbs[k] : 0ull;
      const uint32_t kmod = (uint32_t)(k % n1);
      for (int r = 0; r < a.nreps; ++r) {
        const uint32_t dinv = a.dinv[r];
        const uint32_t s1 = fastmod((uint32_t)k * dinv, M, rc.magicM);
        const uint32_t s2 = fastmod((uint32_t)(N + kmod) * dinv, M, rc.magicM);
        uint64_t v = s1 < (uint32_t)N ? xbs[s1] : 0ull;
        if (s2 < (uint32_t)N) v -= xbs[s2];
        bsum += v;
      }
      return bsum;
    };
    for (int k = threadIdx.x; k < N; k += bdim<T, A>()) {
      uint32_t ya[MAXNP], yb[MAXNP];
#pragma unroll
      for (int i = 0; i < MAXNP; ++i) {
        if (i < np) {
          ya[i] = i == PR ? S.buf[k] : __ldcg(rs + (size_t)i * 2 * N + k);
          yb[i] = i == PR ? S.buf[N + k] : __ldcg(rs + (size_t)i * 2 * N + N + k);
        }
      }
      crt_out(k, ya, yb, body_staged ? body_sum_s(k) : body_sum(k), body_staged && !sync.prefetched);
    }
    __syncthreads();
    // the row's residues are dead: drop their L2 lines without writing them back
    for (int w = threadIdx.x * 32; w < crw; w += bdim<T, A>() * 32)
      asm volatile("discard.global.L2 [%0], 128;" ::"l"(rs + w) : "memory");
    return;
  }

  // ---- body term of this CTA's slice, into the (now free) accumulator region while the
  // other CTAs of the cluster finish ----
  uint64_t* bsum_s = reinterpret_cast<uint64_t*>(S.acc);  // (k1 - k0) u64 <= N u64
  for (int k = k0 + threadIdx.x; k < k1; k += bdim<T, A>()) bsum_s[k - k0] = body_sum(k);

  // ---- explicit CRT across the cluster through distributed shared memory (push) ----
  // every CTA stores its residues of each peer's slice into that peer's (dead) mask
  // buffer; one release/acquire cluster barrier later each CTA owns all np residues of
  // its slice locally, so no CTA reads a peer's memory and none must wait for peers to exit
  asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");  // peers' masks are dead
  {
    uint32_t* recv = reinterpret_cast<uint32_t*>(S.xa);
    for (int q = 0; q < np; ++q) {
      uint32_t* dst = cluster.map_shared_rank(recv, q) + (size_t)PR * 2 * per;
      const int q0 = q * per, q1 = min(N, q0 + per);
      for (int k = q0 + threadIdx.x; k < q1; k += bdim<T, A>()) {
        dst[k - q0] = S.buf[k];
        dst[per + k - q0] = S.buf[N + k];
      }
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
  asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
  const uint32_t* recv = reinterpret_cast<const uint32_t*>(S.xa);
  for (int k = k0 + threadIdx.x; k < k1; k += bdim<T, A>()) {
    uint32_t ya[MAXNP], yb[MAXNP];
#pragma unroll
    for (int i = 0; i < MAXNP; ++i) {
      if (i < np) {
        ya[i] = recv[(size_t)i * 2 * per + (k - k0)];
        yb[i] = recv[(size_t)i * 2 * per + per + (k - k0)];
      }
    }
    crt_out(k, ya, yb, bsum_s[k - k0]);
  }
}

#ifndef SFHR_BODY_UNROLL
#define SFHR_BODY_UNROLL 0
#endif
#ifndef SFHR_ROWS_PER_CLUSTER
#define SFHR_ROWS_PER_CLUSTER 1
#endif

// a cluster processes SFHR_ROWS_PER_CLUSTER consecutive rows (twiddles staged once)
template <int T, int A, int L, int PR>
__device__ void stage_body(const RingConst& rc, const StageArgs& a, unsigned char* smem, const int64_t item) {
  __shared__ __align__(8) uint64_t bars[2];
  RowSync sync{smem_addr(&bars[0]), smem_addr(&bars[1]), 0u, 0u, false};  // init: first stage_row
  if (a.acc_out && a.nsplit > 1) {  // representative split: item = (row, split)
    const unsigned r = (unsigned)item / (unsigned)a.nsplit;
    stage_row<T, A, L, PR>(rc, a, smem, r, true, sync, -1, (int)((unsigned)item - r * (unsigned)a.nsplit));
    return;
  }
  const int64_t row0 = item * SFHR_ROWS_PER_CLUSTER;
  for (int rr = 0; rr < SFHR_ROWS_PER_CLUSTER; ++rr) {
    if (row0 + rr >= a.B) break;  // uniform across the cluster
    if (rr > 0) __syncthreads();  // the previous row's last shared-memory reads are done
    const int64_t next = rr + 1 < SFHR_ROWS_PER_CLUSTER && row0 + rr + 1 < a.B ? row0 + rr + 1 : -1;
    stage_row<T, A, L, PR>(rc, a, smem, row0 + rr, rr == 0, sync, next);
  }
}


template <int T, int A, int L>
__global__ void __launch_bounds__(StageLaunch<T>::kThreads, StageLaunch<T>::kMinBlocks)
    ks_stage_kernel(const __grid_constant__ RingConst rc, const __grid_constant__ StageArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int np = stage_np<T, A>(rc);
  // item = row (or (row, split) of a representative-split launch) and the CTA's CRT prime
  int64_t item = blockIdx.x / np;
  unsigned rank;
  if (!a.independent) {
    rank = cg::this_cluster().block_rank();
  } else if (a.group > 0) {
    // prime-major groups of `group` items: the CTAs resident at any time run one or two of the
    // np prime specialisations of this kernel, not all of them (instruction-cache footprint)
    // (32-bit: the grid has < 2^31 CTAs; 64-bit divisions here cost ~1 % of the instructions)
    const unsigned nitems = (unsigned)(a.acc_out && a.nsplit > 1
                                           ? a.B * a.nsplit
                                           : (a.B + SFHR_ROWS_PER_CLUSTER - 1) / SFHR_ROWS_PER_CLUSTER);
    const unsigned per_group = (unsigned)a.group * (unsigned)np;
    const unsigned g = blockIdx.x / per_group, base = g * (unsigned)a.group;
    const unsigned gc = nitems - base < (unsigned)a.group ? nitems - base : (unsigned)a.group;
    const unsigned within = blockIdx.x - g * per_group;
    rank = within / gc;
    item = base + (within - rank * gc);
  } else {
    rank = blockIdx.x % np;
  }
  switch (rank) {
    case 0: stage_body<T, A, L, 0>(rc, a, smem, item); break;
    case 1: stage_body<T, A, L, 1>(rc, a, smem, item); break;
    case 2: stage_body<T, A, L, 2>(rc, a, smem, item); break;
    default: stage_body<T, A, L, 3>(rc, a, smem, item); break;
  }
}

// ---------------------------------------------------------------------------
// key spectra precompute: forward transform of (centered) key polynomials,
// times R, stored in the thread-owned layout [k * nitems + item].
// One CTA per (slot, digit, comp, prime); runs once per registered key set.

template <int T, int PR>
__device__ void spectra_body(const RingConst& rc, const SpecArgs a, unsigned char* smem, int job) {
  const PrimeConst& pc = rc.pc[PR];
  const int N = rc.N;
  SmemLayout S = carve(smem, rc);
  const uint64_t* src = a.keys + (size_t)job * N;  // job = (slot*l + i)*2 + c
  for (int k = threadIdx.x; k <= rc.M; k += blockDim.x) S.wt[k] = a.twid[(size_t)PR * twid_stride(rc.M) + k];
  for (int k = threadIdx.x; k < N; k += blockDim.x) {
    const uint64_t v = src[k] & QMASK;
    long long c = (long long)v;
    if (v >= (1ull << 52)) c -= (1ll << 53);
    long long r = c % (long long)pc.p;
    if (r < 0) r += pc.p;
    S.buf[k] = (uint32_t)r;
  }
  __syncthreads();
  fwd_first_step<T, 0, PR>(S.buf, 1, rc, S.wt);
  fwd_mid_stages<T, 0, PR>(S.buf, 1, rc, S.wt);
  for (int it = threadIdx.x; it < rc.nitems; it += blockDim.x) {
    uint32_t x[T], y[T];
#pragma unroll
    for (int m = 0; m < T; ++m) x[m] = S.buf[it * T + m];
    dft_t<T>(x, y, pc.z, pc.p, pc.pinv);
    uint32_t* dst = a.out + ((size_t)job * rc.np + PR) * N + it;
#pragma unroll
    for (int k = 0; k < T; ++k) dst[k * rc.nitems] = fully(mont_mul(y[k], pc.r2, pc.p, pc.pinv), pc.p);
  }
}

template <int T>
__global__ void __launch_bounds__(512) ks_spectra_kernel(const __grid_constant__ RingConst rc,
                                                         const __grid_constant__ SpecArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int job = blockIdx.x / rc.np;
  const int pr = blockIdx.x % rc.np;
  switch (pr) {
    case 0: spectra_body<T, 0>(rc, a, smem, job); break;
    case 1: spectra_body<T, 1>(rc, a, smem, job); break;
    case 2: spectra_body<T, 2>(rc, a, smem, job); break;
    default: spectra_body<T, 3>(rc, a, smem, job); break;
  }
}

// ---------------------------------------------------------------------------
// launchers

#if !defined(SFHR_KS_T)
size_t stage_smem_bytes(const RingConst& rc) {
  const int nb = rc.l > 2 ? rc.l : 2;
  return xa_region_bytes(rc) + (size_t)(twid_stride(rc.M) + shoup_stride(rc.n1)) * 4 +
         (size_t)(2 + nb) * rc.N * 4;
}

int stage_threads(const RingConst& rc) {
  const int cap = rc.t == 7 ? StageLaunch<7>::kThreads : rc.t == 5 ? StageLaunch<5>::kThreads
                                                                    : StageLaunch<3>::kThreads;
  const int need = ((rc.nitems + 31) / 32) * 32;
  const bool production = (rc.t == 7 && rc.alpha == 4) || (rc.t == 5 && rc.alpha == 5) ||
                          (rc.t == 3 && rc.alpha == 7);
  if (production && cap >= need) return cap;  // the tuned block size of the compile-time geometry
  // enough threads for one pass over the n1 first-step columns when they fit
  const int want = ((rc.n1 + 31) / 32) * 32;
  return want <= cap ? (want > need ? want : need) : need;
}
#endif

template <int T, int A, int L>
static cudaError_t launch_stage_tal(const RingConst& rc, const StageArgs& a, cudaStream_t st) {
  auto kern = ks_stage_kernel<T, A, L>;
  const size_t smem = stage_smem_bytes(rc);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  const int64_t clusters = a.acc_out && a.nsplit > 1 ? a.B * a.nsplit
                                                     : (a.B + SFHR_ROWS_PER_CLUSTER - 1) / SFHR_ROWS_PER_CLUSTER;
  cfg.gridDim = dim3((unsigned)(clusters * rc.np), 1, 1);
  cfg.blockDim = dim3(stage_threads(rc), 1, 1);
  // the compile-time geometries stride their loops by the launch-bound block size (bdim)
  if (A && cfg.blockDim.x != (unsigned)StageLaunch<T>::kThreads) return cudaErrorInvalidConfiguration;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = rc.np;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = a.independent ? 0 : 1;
  return cudaLaunchKernelEx(&cfg, kern, rc, a);
}

// One translation unit per (t, l) (build.py compiles this file with
// -DSFHR_KS_T=t -DSFHR_KS_L=l) keeps the template fan-out compiling in parallel.
#define SFHR_KS_DECL(T, L) \
  cudaError_t launch_stage_t##T##_l##L(const RingConst& rc, const StageArgs& a, cudaStream_t st)
#define SFHR_KS_DECL_ALL(T) SFHR_KS_DECL(T, 1); SFHR_KS_DECL(T, 2); SFHR_KS_DECL(T, 3); \
  SFHR_KS_DECL(T, 4); SFHR_KS_DECL(T, 5);
SFHR_KS_DECL_ALL(3)
SFHR_KS_DECL_ALL(5)
SFHR_KS_DECL_ALL(7)

#if defined(SFHR_KS_T) && defined(SFHR_KS_L)
#define SFHR_CAT2(a, b, c, d) a##b##c##d
#define SFHR_CAT(a, b, c, d) SFHR_CAT2(a, b, c, d)
// the production rows get a compile-time tower height; everything else is generic
cudaError_t SFHR_CAT(launch_stage_t, SFHR_KS_T, _l, SFHR_KS_L)(const RingConst& rc, const StageArgs& a,
                                                              cudaStream_t st) {
  constexpr int T = SFHR_KS_T, L = SFHR_KS_L;
  constexpr int A = T == 7 ? 4 : T == 5 ? 5 : 7;
  if (rc.alpha == A && rc.np == kProdNP && rc.D == prod_gadget_D<T, A, L>())
    return launch_stage_tal<T, A, L>(rc, a, st);
  return launch_stage_tal<T, 0, L>(rc, a, st);
}
#else

#define SFHR_KS_CASES(T)                              \
  switch (rc.l) {                                     \
    case 1: return launch_stage_t##T##_l1(rc, a, st); \
    case 2: return launch_stage_t##T##_l2(rc, a, st); \
    case 3: return launch_stage_t##T##_l3(rc, a, st); \
    case 4: return launch_stage_t##T##_l4(rc, a, st); \
    case 5: return launch_stage_t##T##_l5(rc, a, st); \
    default: return cudaErrorInvalidValue;            \
  }

cudaError_t launch_stage(const RingConst& rc, const StageArgs& a, cudaStream_t st) {
  if (a.B == 0 || a.nreps == 0) return cudaSuccess;
  if (rc.t == 7) SFHR_KS_CASES(7)
  if (rc.t == 5) SFHR_KS_CASES(5)
  if (rc.t == 3) SFHR_KS_CASES(3)
  return cudaErrorInvalidValue;
}

template <int T>
static cudaError_t launch_spec_t(const RingConst& rc, const SpecArgs& a, int njobs, cudaStream_t st) {
  auto kern = ks_spectra_kernel<T>;
  const size_t smem = stage_smem_bytes(rc);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int nt = stage_threads(rc) < 512 ? stage_threads(rc) : 512;  // ks_spectra_kernel launch bound
  kern<<<njobs * rc.np, nt, smem, st>>>(rc, a);
  return cudaGetLastError();
}

cudaError_t launch_spectra(const RingConst& rc, const SpecArgs& a, int njobs, cudaStream_t st) {
  if (njobs == 0) return cudaSuccess;
  switch (rc.t) {
    case 3: return launch_spec_t<3>(rc, a, njobs, st);
    case 5: return launch_spec_t<5>(rc, a, njobs, st);
    case 7: return launch_spec_t<7>(rc, a, njobs, st);
    default: return cudaErrorInvalidValue;
  }
}

#endif  // SFHR_KS_T

}  // namespace sfhr
