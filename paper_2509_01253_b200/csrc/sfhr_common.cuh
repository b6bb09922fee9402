// Shared definitions for the sm_100a Safhire server kernels.
//
// Ciphertext rows are (2, N) little-endian uint64 torus numerators mod
// q = 2^53 (reference pkg/src/sfhr/params.py:14-16); every integer op on them
// is uint64 wrap followed by & QMASK (reference ring.py:1-9).
//
// The key-switch convolution is done exactly over NP <= 4 word-size primes
// p_i = 1 (mod M) (p_i < 2^31 / max(t, l)) with a "Phi_M-NTT": evaluation of
// degree-<N polynomials at the N primitive M-th roots of unity, followed by
// explicit CRT mod 2^53.  Arithmetic is 32-bit Montgomery with R = 2^32; data
// is kept lazily in [0, 2p), constants fully reduced in [0, p).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sfhr {

constexpr int MAXT = 7;     // largest supported ring prime t (3, 5, 7)
constexpr int MAXNP = 4;    // CRT primes
constexpr int MAXL = 5;     // gadget depth
constexpr int MAXREPS = 8;  // switched automorphisms per stage (t-1 <= 6)
constexpr uint64_t QMASK = (1ull << 53) - 1;

// Rader/Winograd radix-7 DFT (keyswitch.cu dft_wino7): the 6 nonzero inputs, reordered by
// powers of the generator 3, form a length-6 cyclic convolution with the roots; it is split by
// X^6 - 1 = (X - 1)(X + 1)(X^2 + X + 1)(X^2 - X + 1) into 10 products (vs 18 for the symmetric
// pairs).  Constants in Montgomery form, signed ones centred in (-p/2, p/2); offsets keep every
// REDC input and output sum non-negative and below 2^32 (bounds checked by the planner)
struct WinoConst {
  uint64_t kT, kG;      // multiples of p added to the signed R2 / g / h accumulations
  uint32_t mu;          // W(1) / 6 * R in [0, p) (times the unsigned S)
  int32_t rho;          // W(-1) / 6 * R
  int32_t a00, a01, a10, b00, b01, b10;  // (X^2 + X + 1) / (X^2 - X + 1) parts, / 6, * R
  uint32_t k1p, k2p, k3p, k4p, k5p;      // output-sum offsets (multiples of p)
  // Shoup forms of the two single-product terms (M0 = S mu, R2 = (Tm + toff) rho): plain
  // constants and floor(c 2^32 / p); toff = multiple of p making the signed Tm non-negative
  uint32_t mu_w, mu_q, rho_w, rho_q, toff;
  uint32_t pad0, pad1;
  // Karatsuba forms of the 2x2 blocks (3 products instead of 4 per pair, same ranges):
  // g0 = a00 (A0 - A1) + ka01 A1, g1 = -a00 (A0 - A1) + ka10 A0  (ka01 = a01 + a00, ka10 = a10 + a00)
  // h0 = b00 (C0 + C1) + kb01 C1, h1 = b00 (C0 + C1) + kb10 C0   (kb01 = b01 - b00, kb10 = b10 - b00)
  int32_t ka01, ka10, kb01, kb10;
};

struct PrimeConst {
  uint32_t p;      // NTT prime, p = 1 mod M, p < 2^31 / max(t, l)
  uint32_t pinv;   // p^-1 mod 2^32
  uint32_t mu;     // floor(2^32 / p)
  uint32_t r2;     // 2^64 mod p   (to enter Montgomery form)
  uint32_t rmod;   // 2^32 mod p
  uint32_t z[MAXT][MAXT];   // zeta^(k m) * R mod p, zeta = omega^(M/t)
  uint32_t zi[MAXT][MAXT];  // zeta^(-k m) * R mod p
  uint32_t g[MAXT][MAXT];   // inverse first step [j][r-1]: (zeta^(-rj) - zeta^r) / M * Qinv * R
  uint32_t hc[MAXT / 2][MAXT / 2];  // symmetric DFT: (zeta^(km) + zeta^(-km)) / 2 * R, k, m = 1..(t-1)/2
  uint32_t hs[MAXT / 2][MAXT / 2];  //                (zeta^(km) - zeta^(-km)) / 2 * R
  uint64_t q_mod64;         // (P / p) mod 2^64
  double inv_p;             // 1.0 / p
  WinoConst wino[3];        // t = 7: forward, inverse, inverse first step (t = 5: [0], [1])
  uint32_t bc;              // floor(2^33 / p): Barrett step with 32-bit multiplies only (bred)
  uint32_t pad_bc;
};

struct RingConst {
  int t, alpha, M, N, n1, nitems;   // nitems = N / t
  int np;                            // CRT primes in use
  int l, D, dlog2, shift;            // gadget; dlog2 = -1 for odd D
  uint32_t magicM;                   // floor(2^32 / M)
  uint32_t magicN1;                  // floor(2^32 / n1)
  uint64_t P_mod64;                  // prod p_i mod 2^64
  uint64_t decM[MAXL];               // pow2 gadget: carry threshold of digit i (balanced lower part max)
  uint64_t decDp[MAXL];              // odd gadget: D^(i+1)
  PrimeConst pc[MAXNP];
};

// row stride (u32 words) of the [np][M+1] twiddle table, padded for 16-byte loads
#ifdef __CUDACC__
__host__ __device__
#endif
inline constexpr int twid_stride(int M) { return (M + 4) & ~3; }

// Shoup twiddle pairs (w, floor(w 2^32 / p)) of the exponents t i, i = 0..n1 (= M / t): every
// mid-stage twiddle exponent is a multiple of t.  Row stride in u32 words, after the np rows of
// the Montgomery table in the same allocation
#ifdef __CUDACC__
__host__ __device__
#endif
inline constexpr int shoup_stride(int n1) { return (2 * (n1 + 1) + 3) & ~3; }

#ifdef __CUDACC__
// x < p * 2^32  ->  x * 2^-32 mod p, in (0, 2p)
__device__ __forceinline__ uint32_t redc(uint64_t x, uint32_t p, uint32_t pinv) {
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  uint32_t m = lo * pinv;
  return hi - __umulhi(m, p) + p;
}

// x < 2^63  ->  x * 2^-32 mod p, in [0, 2p)
__device__ __forceinline__ uint32_t redc_wide(uint64_t x, uint32_t p, uint32_t pinv, uint32_t mu) {
  uint32_t lo = (uint32_t)x, hi = (uint32_t)(x >> 32);
  uint32_t m = lo * pinv;
  uint32_t r = hi - __umulhi(m, p) + p;
  return r - __umulhi(r, mu) * p;
}

// a in [0, 2p), bm = b*R mod p  ->  a*b mod p in (0, 2p)
__device__ __forceinline__ uint32_t mont_mul(uint32_t a, uint32_t bm, uint32_t p, uint32_t pinv) {
  return redc((uint64_t)a * bm, p, pinv);
}

// Barrett step to [0, 2p) for any y < 2^32 with two low multiplies instead of IMAD.HI + IMAD:
// q = ((y >> 16) bc) >> 17 with bc = floor(2^33 / p) satisfies y / p - 1/2 - 2^16 / p < q <= y / p
// (needs 2^18 <= p < 2^31; the product stays below 2^49 / p < 2^32), so y - q p is in [0, 2p)
__device__ __forceinline__ uint32_t bred(uint32_t y, uint32_t p, uint32_t bc) {
  const uint32_t q = ((y >> 16) * bc) >> 17;
  return y - q * p;
}

// Shoup: x < 2^32, wq = (w, floor(w 2^32 / p)), w < p  ->  x w mod p in [0, 2p)
// (IMAD.HI + 2 IMAD against IMAD.WIDE + IMAD + IMAD.HI for a Montgomery twiddle)
__device__ __forceinline__ uint32_t shoup_mul(uint32_t x, uint2 wq, uint32_t p) {
  const uint32_t q = __umulhi(x, wq.y);
  return x * wq.x - q * p;
}

// [0, 2p) -> [0, p)
__device__ __forceinline__ uint32_t fully(uint32_t a, uint32_t p) { return a >= p ? a - p : a; }

// x mod M for x < 2^32 using magic = floor(2^32 / M)
__device__ __forceinline__ uint32_t fastmod(uint32_t x, uint32_t M, uint32_t magic) {
  uint32_t r = x - __umulhi(x, magic) * M;
  return r >= M ? r - M : r;
}

// balanced base-D digits of y < 2^53 (reference crypto.py:288-323), all at once
template <int L>
__device__ __forceinline__ void decompose(uint64_t y, int (&dg)[L], const RingConst& rc) {
  if (rc.dlog2 >= 0) {
    const int w = rc.dlog2, D = rc.D;
    uint64_t u = (y + (1ull << (rc.shift - 1))) >> rc.shift;
    int carry = 0;
#pragma unroll
    for (int i = L - 1; i >= 0; --i) {
      const int x = (int)(u & (uint64_t)(D - 1)) + carry;
      u >>= w;
      carry = x > (D >> 1);
      dg[i] = carry ? x - D : x;
    }
  } else {
    const long long D = rc.D;
    long long r = (long long)y;
    if (y > (1ull << 52)) r -= (1ll << 53);
#pragma unroll
    for (int i = 0; i < L; ++i) {
      const long long prod = r * D;
      const long long d = (prod + (1ll << 52)) >> 53;
      dg[i] = (int)d;
      r = prod - d * (1ll << 53);
    }
  }
}

#endif  // __CUDACC__

}  // namespace sfhr
