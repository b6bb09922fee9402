// Host-side planning for a ring row: NTT primes, Montgomery constants,
// explicit-CRT constants, twiddle tables, the two-term dual basis, and the
// tower/pack schedule.  Pure C++ (no CUDA calls).
#include "plan.h"

#include <cmath>
#include <initializer_list>
#include <cstring>
#include <stdexcept>
#include <string>

namespace sfhr {

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
  return (uint64_t)((unsigned __int128)a * b % m);
}
static uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
  uint64_t r = 1 % m;
  a %= m;
  while (e) {
    if (e & 1) r = mulmod(r, a, m);
    a = mulmod(a, a, m);
    e >>= 1;
  }
  return r;
}
static bool is_prime_u32(uint64_t n) {
  if (n < 2) return false;
  for (uint64_t p : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull, 19ull, 23ull, 29ull, 31ull, 37ull})
    if (n % p == 0) return n == p;
  uint64_t d = n - 1;
  int s = 0;
  while (!(d & 1)) { d >>= 1; ++s; }
  for (uint64_t a : {2ull, 3ull, 5ull, 7ull, 11ull, 13ull, 17ull}) {
    uint64_t x = powmod(a, d, n);
    if (x == 1 || x == n - 1) continue;
    bool comp = true;
    for (int r = 1; r < s; ++r) {
      x = mulmod(x, x, n);
      if (x == n - 1) { comp = false; break; }
    }
    if (comp) return false;
  }
  return true;
}
static bool small_prime(int n) {
  if (n < 2) return false;
  for (int k = 2; k * k <= n; ++k)
    if (n % k == 0) return false;
  return true;
}
static std::vector<int> factor_multiset(int n) {
  std::vector<int> f;
  for (int k = 2; k * k <= n; ++k)
    while (n % k == 0) { f.push_back(k); n /= k; }
  if (n > 1) f.push_back(n);
  return f;
}
static int primitive_root_small(int t) {
  auto fs = factor_multiset(t - 1);
  for (int g = 2; g < t; ++g) {
    bool ok = true;
    for (int f : fs)
      if (powmod(g, (t - 1) / f, t) == 1) { ok = false; break; }
    if (ok) return g;
  }
  throw std::invalid_argument("no primitive root");
}
static uint64_t inv_mod(uint64_t a, uint64_t m) {  // m prime
  return powmod(a, m - 2, m);
}
static int64_t inv_mod_any(int64_t a, int64_t m) {  // gcd(a, m) = 1
  int64_t g = m, x = 0, x1 = 1, aa = ((a % m) + m) % m;
  while (aa) {
    int64_t q = g / aa;
    int64_t t = g - q * aa; g = aa; aa = t;
    t = x - q * x1; x = x1; x1 = t;
  }
  return ((x % m) + m) % m;
}

// Shoup form (plain constant, floor(c 2^32 / p)) of c in [0, p)
static void shoup_pair(uint64_t c, uint64_t p, uint32_t& w, uint32_t& q) {
  w = (uint32_t)(c % p);
  q = (uint32_t)(((uint64_t)w << 32) / p);
}

// Tr(zeta_M^k) over Q (reference dual.py:18-27)
static long long tr_zeta(long long k, int t, int alpha) {
  long long M = 1, n1 = 1;
  for (int i = 0; i < alpha; ++i) M *= t;
  n1 = M / t;
  k %= M;
  if (k < 0) k += M;
  if (k == 0) return n1 * (t - 1);
  return (k % n1 == 0) ? -n1 : 0;
}

// Rader/Winograd radix-7 DFT constants and range offsets (keyswitch.cu dft_wino7).  With
// v_j = x_{5^j mod 7} and w_c = z^(3^c), y_{3^i} - x_0 = (v (*) w)_i (cyclic, length 6); the
// product is computed from its residues mod X - 1 (W(1) = -1), X + 1, X^2 + X + 1 and
// X^2 - X + 1 and reconstructed with 6 L^-1 (entries +-1, +-2; the 1/6 folded into constants,
// as is an optional output scale s).  Every bound below assumes inputs < 2p and is checked, so a
// prime that would overflow throws.  Returns the REDC output bounds of M0, R2 and g / h.
struct Wino7Bounds {
  long double M0, R2, G;
};
static Wino7Bounds wino7_consts(WinoConst& k, uint64_t z, uint64_t scale, uint64_t p) {
  const uint64_t R32 = 1ull << 32, Rm = R32 % p;
  const uint64_t i6 = mulmod(inv_mod(6 % p, p), scale % p, p);
  auto cen = [&](uint64_t v) -> int32_t {  // Montgomery form, centred
    const uint64_t m = mulmod(v % p, Rm, p);
    return m > p / 2 ? (int32_t)((int64_t)m - (int64_t)p) : (int32_t)m;
  };
  auto sub = [&](uint64_t a, uint64_t b) { return (a + p - b % p) % p; };
  const long double X = 2.0L * p, ch = (long double)((p - 1) / 2), two32 = 4294967296.0L;
  const long double Smax = 6.0L * X, Tmax = 3.0L * X, Amax = 2.0L * X;
  uint64_t w[6];
  for (int c = 0, g = 1; c < 6; ++c, g = g * 3 % 7) w[c] = powmod(z, (uint64_t)g, p);
  const uint64_t B0 = sub((w[0] + w[3]) % p, (w[2] + w[5]) % p), B1 = sub((w[1] + w[4]) % p, (w[2] + w[5]) % p);
  const uint64_t D0 = sub((w[0] + w[5]) % p, (w[3] + w[2]) % p), D1 = sub((w[1] + w[2]) % p, (w[4] + w[5]) % p);
  uint64_t W1 = 0, Wm = 0;
  for (int c = 0; c < 6; ++c) {
    W1 = (W1 + w[c]) % p;
    Wm = (c & 1) ? sub(Wm, w[c]) : (Wm + w[c]) % p;
  }
  std::memset(&k, 0, sizeof(k));
  k.mu = (uint32_t)mulmod(mulmod(W1, i6, p), Rm, p);
  k.rho = cen(mulmod(Wm, i6, p));
  shoup_pair(mulmod(W1, i6, p), p, k.mu_w, k.mu_q);
  shoup_pair(mulmod(Wm, i6, p), p, k.rho_w, k.rho_q);
  k.toff = (uint32_t)(6 * p);  // Tm in (-3X, 3X) = (-6p, 6p)
  k.a00 = cen(mulmod(sub(2 * B0 % p, B1), i6, p));
  k.a01 = cen(mulmod(sub(0, (B0 + B1) % p), i6, p));
  k.a10 = cen(mulmod(sub(2 * B1 % p, B0), i6, p));
  k.b00 = cen(mulmod((2 * D0 + D1) % p, i6, p));
  k.b01 = cen(mulmod(sub(D0, D1), i6, p));
  k.b10 = cen(mulmod((D0 + 2 * D1) % p, i6, p));
  auto cadd = [&](int32_t a, int32_t b) {  // centred Montgomery constants a + b, re-centred
    int64_t v = ((int64_t)a + b) % (int64_t)p;
    if (v > (int64_t)(p / 2)) v -= p;
    if (v < -(int64_t)(p / 2)) v += p;
    return (int32_t)v;
  };
  k.ka01 = cadd(k.a01, k.a00);
  k.ka10 = cadd(k.a10, k.a00);
  k.kb01 = cadd(k.b01, -k.b00);
  k.kb10 = cadd(k.b10, -k.b00);
  // REDC(x) <= floor(x / 2^32) + p; signed sums offset by a multiple of p
  auto up = [&](long double v) { return (uint64_t)std::ceil(v / (long double)p) * p; };
  k.kT = up(Tmax * ch);
  k.kG = up(2.0L * Amax * ch);
  if (X + Smax >= two32 || 2.0L * Tmax >= two32)
    throw std::invalid_argument("NTT prime too large for the radix-7 DFT ranges");
  // M0 and R2 may come from the Shoup forms (keyswitch.cu SFHR_WINO_SHOUP): bound them by 2p
  const long double M0 = std::floor(Smax * (p - 1) / two32) + p, R2 = std::floor(((long double)k.kT + Tmax * ch) / two32) + p;
  return {std::max(M0, X), std::max(R2, X), std::floor(((long double)k.kG + 2.0L * Amax * ch) / two32) + p};
}

static uint32_t up_p(long double v, uint64_t p) { return (uint32_t)((uint64_t)std::ceil(v / (long double)p) * p); }

static void check32(std::initializer_list<long double> maxima) {
  for (long double v : maxima)
    if (v >= 4294967296.0L) throw std::invalid_argument("NTT prime too large for the radix-7 Winograd DFT ranges");
}

// forward (wino[0]) and inverse (wino[1]) radix-7 DFTs
static void build_wino7(PrimeConst& pc, uint64_t zeta, uint64_t p) {
  const long double X = 2.0L * p;
  for (int dir = 0; dir < 2; ++dir) {
    WinoConst& k = pc.wino[dir];
    const Wino7Bounds b = wino7_consts(k, dir ? inv_mod(zeta, p) : zeta, 1, p);
    const long double R2 = b.R2, G = b.G;
    k.k1p = up_p(R2, p);
    k.k2p = up_p(R2 + G, p);
    k.k3p = up_p(3.0L * G, p);
    k.k4p = up_p(G, p);
    k.k5p = up_p(R2 + 3.0L * G, p);
    const long double X0 = X + b.M0;
    check32({X0 + R2 + 2 * G, X0 + k.k1p + 2 * G, X0 + R2 + k.k3p + G, X0 + k.k2p + G, X0 + R2 + k.k4p + G,
             X0 + k.k5p + G});
  }
}

// inverse first step (wino[2], keyswitch.cu inv_first7): out_j = s (Y_j - Y_6), j < 6, where Y is
// the inverse 7-point DFT of (0, C_1..C_6) and s = Qinv / M (the CRT weight; pc.g's matrix is
// s (zeta^-rj - zeta^r)).  Constants scaled by s; mu holds 7 s / 6 (out_0 = 7 s S / 6 + ...),
// k1p..k5p offset out_0, out_2, out_3, out_4, out_5.
static void build_wino7_invfirst(PrimeConst& pc, uint64_t zeta, uint64_t s, uint64_t p) {
  WinoConst& k = pc.wino[2];
  const Wino7Bounds b = wino7_consts(k, inv_mod(zeta, p), s, p);
  const uint64_t Rm = (1ull << 32) % p;
  k.mu = (uint32_t)mulmod(mulmod(mulmod(7, inv_mod(6, p), p), s, p), Rm, p);
  shoup_pair(mulmod(mulmod(7, inv_mod(6, p), p), s, p), p, k.mu_w, k.mu_q);
  const long double R2 = b.R2, G = b.G, S7 = b.M0;
  k.k1p = up_p(G, p);
  k.k2p = up_p(3.0L * G, p);
  k.k3p = up_p(G, p);
  k.k4p = up_p(2.0L * G, p);
  k.k5p = up_p(4.0L * G, p);
  check32({S7 + R2 + G + k.k1p, 2 * R2 + 2 * G, 2 * R2 + 2 * G + k.k2p, 3 * G + k.k3p, 2 * R2 + 2 * G + k.k4p,
           3 * G + k.k5p});
}

// Rader radix-5 DFT constants (keyswitch.cu dft_wino5): v_j = x_{3^j mod 5}, w_c = zeta^(2^c),
// y_{2^i} - x_0 = (v (*) w)_i (cyclic, length 4) through X^4 - 1 = (X - 1)(X + 1)(X^2 + 1):
// 6 products instead of 8.  Fields of WinoConst: mu = W(1)/4, rho = W(-1)/4, a00 = B0/2,
// a01 = -B1/2, a10 = B1/2 (B = W mod X^2 + 1); k1p..k3p offsets of z1..z3.
static void build_wino5(PrimeConst& pc, uint64_t zeta, uint64_t p) {
  const uint64_t R32 = 1ull << 32, Rm = R32 % p;
  const uint64_t i4 = inv_mod(4 % p, p), i2 = inv_mod(2 % p, p);
  auto cen = [&](uint64_t v) -> int32_t {
    const uint64_t m = mulmod(v % p, Rm, p);
    return m > p / 2 ? (int32_t)((int64_t)m - (int64_t)p) : (int32_t)m;
  };
  auto sub = [&](uint64_t a, uint64_t b) { return (a + p - b % p) % p; };
  const long double X = 2.0L * p, ch = (long double)((p - 1) / 2), two32 = 4294967296.0L;
  for (int dir = 0; dir < 2; ++dir) {
    const uint64_t z = dir ? inv_mod(zeta, p) : zeta;
    uint64_t w[4];
    for (int c = 0, g = 1; c < 4; ++c, g = g * 2 % 5) w[c] = powmod(z, (uint64_t)g, p);
    const uint64_t B0 = sub(w[0], w[2]), B1 = sub(w[1], w[3]);
    const uint64_t W1 = (w[0] + w[1] + w[2] + w[3]) % p, Wm = sub((w[0] + w[2]) % p, (w[1] + w[3]) % p);
    WinoConst& k = pc.wino[dir];
    std::memset(&k, 0, sizeof(k));
    k.mu = (uint32_t)mulmod(mulmod(W1, i4, p), Rm, p);
    k.rho = cen(mulmod(Wm, i4, p));
    shoup_pair(mulmod(W1, i4, p), p, k.mu_w, k.mu_q);
    shoup_pair(mulmod(Wm, i4, p), p, k.rho_w, k.rho_q);
    k.toff = (uint32_t)(4 * p);  // Tm in (-2X, 2X)
    k.a00 = cen(mulmod(B0, i2, p));
    k.a01 = cen(mulmod(sub(0, B1), i2, p));
    k.a10 = cen(mulmod(B1, i2, p));
    auto cadd = [&](int32_t a, int32_t b) {
      int64_t v = ((int64_t)a + b) % (int64_t)p;
      if (v > (int64_t)(p / 2)) v -= p;
      if (v < -(int64_t)(p / 2)) v += p;
      return (int32_t)v;
    };
    k.ka01 = cadd(k.a01, k.a00);
    k.ka10 = cadd(k.a10, k.a00);
    auto up = [&](long double v) { return (uint64_t)std::ceil(v / (long double)p) * p; };
    k.kT = up(2.0L * X * ch);
    // |a00 (A0 - A1)| + |ka A| < (2X + X) ch (Karatsuba form; the direct form needs 2 X ch)
    k.kG = up(3.0L * X * ch);
    // (bounded by 2p: M0 and R2 may come from the Shoup forms)
    const long double M0 = std::max(std::floor(4.0L * X * (p - 1) / two32) + p, X);
    const long double R2 = std::max(std::floor(((long double)k.kT + 2.0L * X * ch) / two32) + p, X);
    const long double G = std::floor(((long double)k.kG + 3.0L * X * ch) / two32) + p;
    k.k1p = (uint32_t)up(R2);
    k.k2p = (uint32_t)up(G);
    k.k3p = (uint32_t)up(R2 + G);
    const long double X0 = X + M0;
    const long double zmax[4] = {X0 + R2 + G, X0 + k.k1p + G, X0 + R2 + k.k2p, X0 + k.k3p};
    for (long double v : zmax)
      if (v >= two32) throw std::invalid_argument("NTT prime too large for the radix-5 Rader DFT ranges");
  }
}

Plan make_plan(int t, int alpha, int p_bits, int D, int l, int gamma, int beta) {
  if (t < 3 || !small_prime(t)) throw std::invalid_argument("t must be an odd prime >= 3");
  if (t != 3 && t != 5 && t != 7) throw std::invalid_argument("device kernels support t in {3, 5, 7}");
  if (alpha < 2) throw std::invalid_argument("device kernels need alpha >= 2");
  if (p_bits < 8 || p_bits > 16) throw std::invalid_argument("p must be a power of two between 2^8 and 2^16");
  if (D < 2 || l < 1) throw std::invalid_argument("need D >= 2 and l >= 1");
  if (l > MAXL) throw std::invalid_argument("gadget depth l > 5 unsupported on device");
  if (gamma < 0 || gamma > 2) throw std::invalid_argument("extraction level gamma must be 0, 1 or 2");
  const int beta_eff = beta ? beta : alpha - 1;
  if (beta_eff < 1 || beta_eff > alpha - 1)
    throw std::invalid_argument("packing level beta must satisfy 1 <= beta <= alpha-1");

  Plan P;
  RingConst& rc = P.rc;
  std::memset(&rc, 0, sizeof(rc));
  rc.t = t;
  rc.alpha = alpha;
  long long M = 1;
  for (int i = 0; i < alpha; ++i) M *= t;
  rc.M = (int)M;
  rc.n1 = (int)(M / t);
  rc.N = rc.n1 * (t - 1);
  rc.nitems = rc.N / t;
  rc.l = l;
  rc.D = D;
  // D^l <= q
  {
    long double lg = l * std::log2((long double)D);
    if (lg > 53.0L + 1e-12L) throw std::invalid_argument("D^l must not exceed q");
  }
  if ((D & (D - 1)) == 0) {
    int w = 0;
    while ((1 << w) < D) ++w;
    rc.dlog2 = w;
    rc.shift = 53 - w * l;
    if (rc.shift < 1) throw std::invalid_argument("gadget with D^l == q unsupported");
  } else {
    if (D > 1024) throw std::invalid_argument("non-power-of-two base must be <= 1024");
    rc.dlog2 = -1;
    rc.shift = 0;
  }
  {
    const int cap = t == 7 ? 320 : 512;  // StageLaunch<T>::kThreads (keyswitch.cu)
    if (((rc.nitems + 31) / 32) * 32 > cap)
      throw std::invalid_argument("ring too large for one CTA per row on this device path");
  }
  // per-digit closed forms of the balanced decomposition (see keyswitch.cu digit_i)
  for (int i = 0; i < l; ++i) {
    unsigned __int128 Mi = 0, pw = 1;
    for (int k = l - 1; k > i; --k) {
      Mi += (unsigned __int128)(D / 2) * pw;
      pw *= (unsigned __int128)D;
    }
    rc.decM[i] = (uint64_t)Mi;
    unsigned __int128 dp = 1;
    for (int k = 0; k <= i; ++k) dp *= (unsigned __int128)D;
    rc.decDp[i] = (uint64_t)dp;
  }
  rc.magicM = (uint32_t)((1ull << 32) / (uint64_t)rc.M);
  rc.magicN1 = (uint32_t)((1ull << 32) / (uint64_t)rc.n1);

  P.p_bits = p_bits;
  P.gamma = gamma;
  P.beta = beta_eff;
  P.pack_factor = 1;
  for (int i = 0; i < beta_eff - 1; ++i) P.pack_factor *= t;
  P.pack_factor *= (t - 1);

  // ---- schedule (reference tracepack.py:179-201, 288-326) ----
  {
    int g = primitive_root_small(t);
    long long stride = 1;
    for (int ell : factor_multiset(t - 1)) {
      std::vector<uint32_t> ch;
      for (int u = 0; u < ell; ++u) ch.push_back((uint32_t)powmod(g, stride * u, M));
      P.chains.push_back(ch);
      stride *= ell;
    }
    for (int j = 1; j < alpha; ++j) {
      std::vector<uint32_t> reps;
      long long tj = 1;
      for (int i = 0; i < j; ++i) tj *= t;
      for (int i = 0; i < t; ++i) reps.push_back((uint32_t)((1 + i * tj) % M));
      P.reps_above.push_back(reps);
    }
  }
  int maxreps = t - 1;
  for (auto& ch : P.chains) maxreps = std::max(maxreps, (int)ch.size() - 1);
  if (maxreps > MAXREPS) throw std::invalid_argument("too many representatives per stage");

  // ---- NTT primes: p = 1 mod M, p < 2^31 / max(t, l) ----
  const uint64_t limit = ((1ull << 31) - 1) / (uint64_t)std::max(t, l);
  // worst-case |coefficient| of one stage's NTT-domain sum, centered keys:
  //   maxreps * 2 (fold) * l * N * ceil(D/2) * 2^52
  const long double bound_bits = std::log2((long double)maxreps * 2.0L * l * rc.N *
                                           (long double)((D + 1) / 2)) + 52.0L;
  std::vector<uint64_t> primes;
  long double pbits = 0;
  for (uint64_t k = (limit - 1) / (uint64_t)M; k > 0 && (int)primes.size() < MAXNP; --k) {
    uint64_t p = k * (uint64_t)M + 1;
    if (p >= limit || !is_prime_u32(p)) continue;
    primes.push_back(p);
    pbits += std::log2((long double)p);
    if (pbits >= bound_bits + 1.5L) break;
  }
  if (pbits < bound_bits + 1.5L) throw std::invalid_argument("no CRT prime set large enough for this gadget");
  rc.np = (int)primes.size();
  P.bound_bits = (double)bound_bits;
  P.crt_bits = (double)pbits;
  // accumulator headroom: each rep adds one REDC output (< 2p) to a u32
  if (2.0L * maxreps * (long double)primes[0] >= 4294967296.0L)
    throw std::invalid_argument("NTT-domain accumulator would overflow 32 bits");
  P.shrink = 0;

  uint64_t Pmod = 1;
  for (uint64_t p : primes) Pmod *= p;
  rc.P_mod64 = Pmod;
  // [np][twid_stride(M)] Montgomery powers, then [np][shoup_stride(n1)] Shoup pairs
  P.twid.assign((size_t)rc.np * (twid_stride(M) + shoup_stride(M / t)), 0);
  const uint64_t R32 = 1ull << 32;
  for (int i = 0; i < rc.np; ++i) {
    const uint64_t p = primes[i];
    PrimeConst& pc = rc.pc[i];
    pc.p = (uint32_t)p;
    uint32_t inv = 1;
    for (int it = 0; it < 5; ++it) inv *= 2u - (uint32_t)p * inv;  // Newton: p^-1 mod 2^32
    pc.pinv = inv;
    pc.mu = (uint32_t)(R32 / p);
    pc.bc = (uint32_t)((R32 << 1) / p);
    if (p < (1ull << 18)) throw std::invalid_argument("NTT prime below 2^18 (bred range)");
    pc.rmod = (uint32_t)(R32 % p);
    pc.r2 = (uint32_t)mulmod(R32 % p, R32 % p, p);
    uint64_t omega = 0;
    for (uint64_t x = 2; x < p; ++x) {
      uint64_t w = powmod(x, (p - 1) / M, p);
      if (powmod(w, M / t, p) != 1) { omega = w; break; }
    }
    if (!omega) throw std::runtime_error("no primitive M-th root");
    const uint64_t Rm = R32 % p;
    auto mont = [&](uint64_t v) { return (uint32_t)mulmod(v % p, Rm, p); };
    const uint64_t zeta = powmod(omega, M / t, p);
    for (int k = 0; k < t; ++k)
      for (int m = 0; m < t; ++m) {
        pc.z[k][m] = mont(powmod(zeta, (uint64_t)((k * m) % t), p));
        pc.zi[k][m] = mont(powmod(zeta, (uint64_t)((t - (k * m) % t) % t), p));
      }
    // symmetric-pair DFT constants (keyswitch.cu dft_sym): a_m = x_m + x_{t-m} < 4p and
    // sum_m a_m c_km over (t-1)/2 terms must stay below p 2^32; y_0 < 2tp below 2^32
    {
      const int H = (t - 1) / 2;
      if (4.0L * H * (long double)p >= 4294967296.0L || 2.0L * t * (long double)p >= 4294967296.0L)
        throw std::invalid_argument("NTT prime too large for the symmetric DFT ranges");
      const uint64_t inv2 = (p + 1) / 2;
      for (int k = 1; k <= H; ++k)
        for (int m = 1; m <= H; ++m) {
          const uint64_t zp = powmod(zeta, (uint64_t)((k * m) % t), p);
          const uint64_t zm = powmod(zeta, (uint64_t)((t - (k * m) % t) % t), p);
          pc.hc[k - 1][m - 1] = mont(mulmod((zp + zm) % p, inv2, p));
          pc.hs[k - 1][m - 1] = mont(mulmod((zp + p - zm) % p, inv2, p));
        }
    }
    if (t == 7) build_wino7(pc, zeta, p);
    if (t == 5) build_wino5(pc, zeta, p);
    // CRT: Q_i = P / p_i, Qinv = Q_i^-1 mod p_i
    uint64_t qmod64 = 1, qmodp = 1;
    for (int j = 0; j < rc.np; ++j)
      if (j != i) {
        qmod64 *= primes[j];
        qmodp = mulmod(qmodp, primes[j] % p, p);
      }
    pc.q_mod64 = qmod64;
    pc.inv_p = 1.0 / (double)p;
    const uint64_t qinv = inv_mod(qmodp, p);
    const uint64_t minv = inv_mod((uint64_t)M % p, p);
    if (t == 7) build_wino7_invfirst(pc, zeta, mulmod(minv, qinv, p), p);
    for (int j = 0; j < t - 1; ++j)
      for (int r = 1; r < t; ++r) {
        uint64_t a = powmod(zeta, (uint64_t)((t - (r * j) % t) % t), p);
        uint64_t b = powmod(zeta, (uint64_t)(r % t), p);
        uint64_t v = (a + p - b) % p;
        v = mulmod(mulmod(v, minv, p), qinv, p);
        pc.g[j][r - 1] = mont(v);
      }
    uint64_t w = 1;
    uint32_t* sh = P.twid.data() + (size_t)rc.np * twid_stride(M) + (size_t)i * shoup_stride(M / t);
    for (long long e = 0; e <= M; ++e) {
      const uint64_t we = e == M ? 1 : w;
      P.twid[(size_t)i * twid_stride(M) + e] = mont(we);
      if (e % t == 0) {
        sh[2 * (e / t)] = (uint32_t)we;
        sh[2 * (e / t) + 1] = (uint32_t)((we << 32) / p);
      }
      w = mulmod(w, omega, p);
    }
  }

  // ---- dual basis two-term forms (reference dual.py:108-166) ----
  P.e1.assign(rc.N, 0);
  P.e2.assign(rc.N, 0);
  P.cvec.assign(rc.N, 0);
  const int n1 = rc.n1, N = rc.N;
  for (int i = 0; i < N; ++i) {
    const long long a = (M - i) % M;
    const int first = i / n1 + 1;
    bool found = false;
    std::vector<int> cands = {first};
    for (int c = 1; c < t; ++c)
      if (c != first) cands.push_back(c);
    for (int c : cands) {
      const long long b = (a + (long long)c * n1) % M;
      bool ok = true;
      for (int j = i % n1; j < N && ok; j += n1) {
        long long pr = tr_zeta(j + a, t, alpha) - tr_zeta(j + b, t, alpha);
        ok = pr == (j == i ? M : 0);
      }
      if (ok) {
        P.e1[i] = (int32_t)a;
        P.e2[i] = (int32_t)b;
        P.cvec[i] = c;
        found = true;
        break;
      }
    }
    if (!found) throw std::runtime_error("dual basis index has no two-term form");
  }
  const long long pmod = 1ll << p_bits;
  long long u = inv_mod_any(M % pmod, pmod);
  P.inv_m_mod_p = u;
  const long long cu = u > pmod / 2 ? u - pmod : u;
  P.cu = (uint64_t)(int64_t)cu;
  return P;
}

uint32_t inv_mod_M(const Plan& P, uint32_t d) {
  const long long M = P.rc.M;
  if (std::gcd((long long)d % M, M) != 1) throw std::invalid_argument("automorphism index not coprime with M");
  return (uint32_t)inv_mod_any((long long)d % M, M);
}

}  // namespace sfhr
