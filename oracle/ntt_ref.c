/* CPU oracle for the standalone RNS negacyclic NTT (BASELINE configs[1]).
 *
 * TEST INFRASTRUCTURE ONLY: used by tests/ and bench.py's cpu_baseline leg as
 * the checker, never by the product path.  The reference (arxiv 2509.01253,
 * pkg/src/sfhr) has no power-of-two ring or RNS NTT, so
 * this restates the textbook algorithm the north star names and is pinned by
 * self-consistency instead of reference vectors ("parity unpinned" for this
 * primitive): inverse(forward(x)) = x and NTT-domain products = the schoolbook
 * negacyclic convolution.
 *
 * Conventions (shared with csrc/ntt64.cu): psi = g^((p-1)/2N) for the smallest
 * g >= 2 with psi^N = -1; forward = merged-twiddle Cooley-Tukey with
 * W[k] = psi^brv(k), natural order in, bit-reversed order out; inverse =
 * Gentleman-Sande with psi^-brv(k) and the N^-1 scaling.
 *
 *   gcc -O2 -shared -fPIC oracle/ntt_ref.c -o oracle/libntt_ref.so
 */
#include <stdint.h>
#include <stdlib.h>

typedef unsigned __int128 u128;

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t p) { return (uint64_t)((u128)a * b % p); }

static uint64_t powmod(uint64_t a, uint64_t e, uint64_t p) {
  uint64_t r = 1;
  a %= p;
  while (e) {
    if (e & 1) r = mulmod(r, a, p);
    a = mulmod(a, a, p);
    e >>= 1;
  }
  return r;
}

static unsigned brv(unsigned x, int bits) {
  unsigned r = 0;
  for (int i = 0; i < bits; ++i) r |= ((x >> i) & 1u) << (bits - 1 - i);
  return r;
}

uint64_t ntt_ref_psi(uint64_t p, int logn) {
  const uint64_t N = 1ull << logn;
  for (uint64_t g = 2; g < p; ++g) {
    const uint64_t c = powmod(g, (p - 1) / (2 * N), p);
    if (powmod(c, N, p) == p - 1) return c;
  }
  return 0;
}

void ntt_ref_forward(uint64_t* x, int logn, uint64_t p) {
  const uint64_t N = 1ull << logn, psi = ntt_ref_psi(p, logn);
  for (uint64_t m = 1, d = N >> 1; m < N; m <<= 1, d >>= 1) {
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t w = powmod(psi, brv((unsigned)(m + i), logn), p);
      for (uint64_t j = 2 * i * d; j < 2 * i * d + d; ++j) {
        const uint64_t u = x[j], v = mulmod(x[j + d], w, p);
        x[j] = (u + v) % p;
        x[j + d] = (u + p - v) % p;
      }
    }
  }
}

void ntt_ref_inverse(uint64_t* x, int logn, uint64_t p) {
  const uint64_t N = 1ull << logn, psi = ntt_ref_psi(p, logn);
  const uint64_t psii = powmod(psi, p - 2, p);
  for (uint64_t m = N >> 1, d = 1; m >= 1; m >>= 1, d <<= 1) {
    for (uint64_t i = 0; i < m; ++i) {
      const uint64_t w = powmod(psii, brv((unsigned)(m + i), logn), p);
      for (uint64_t j = 2 * i * d; j < 2 * i * d + d; ++j) {
        const uint64_t u = x[j], v = x[j + d];
        x[j] = (u + v) % p;
        x[j + d] = mulmod((u + p - v) % p, w, p);
      }
    }
    if (m == 1) break;
  }
  const uint64_t ninv = powmod(N % p, p - 2, p);
  for (uint64_t j = 0; j < N; ++j) x[j] = mulmod(x[j], ninv, p);
}

/* c = a * b mod (X^n + 1, p), schoolbook */
void ntt_ref_negacyclic(const uint64_t* a, const uint64_t* b, uint64_t* c, int n, uint64_t p) {
  for (int k = 0; k < n; ++k) c[k] = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const uint64_t t = mulmod(a[i], b[j], p);
      const int k = i + j;
      if (k < n) c[k] = (c[k] + t) % p;
      else c[k - n] = (c[k - n] + p - t) % p;
    }
}

void ntt_ref_pointwise(const uint64_t* a, const uint64_t* b, uint64_t* c, int64_t n, uint64_t p) {
  for (int64_t k = 0; k < n; ++k) c[k] = mulmod(a[k], b[k], p);
}
