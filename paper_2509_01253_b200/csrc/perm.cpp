// Keyed permutation sigma_r, bit-exact with the reference's
// confidentiality.derive_permutation (pkg/src/sfhr/confidentiality.py:27-76):
//   session_key = BLAKE2b-256(session_id; key = master_seed)
//   round_key   = BLAKE2b-256(le32(round); key = session_key)
//   word stream = BLAKE2b-512(le64(counter); key = round_key), 8 LE words/block
//   uniform_int(bound): rejection below 2^64 - (2^64 mod (bound+1))
//   Fisher-Yates over i = size-1 .. 1 with j = uniform_int(i)
// BLAKE2b is implemented from RFC 7693.
#include <cstdint>
#include <cstring>
#include <stdexcept>

namespace sfhr {
namespace {

constexpr uint64_t IV[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                            0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                            0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
constexpr uint8_t SIGMA[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

inline uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }
inline uint64_t load64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

struct Blake2b {
  uint64_t h[8];
  uint64_t t0 = 0, t1 = 0;
  uint8_t buf[128];
  size_t fill = 0;
  size_t outlen;

  Blake2b(size_t outlen_, const uint8_t* key, size_t keylen) : outlen(outlen_) {
    if (outlen == 0 || outlen > 64 || keylen > 64) throw std::invalid_argument("blake2b parameters");
    for (int i = 0; i < 8; ++i) h[i] = IV[i];
    h[0] ^= 0x01010000ULL ^ ((uint64_t)keylen << 8) ^ outlen;
    std::memset(buf, 0, sizeof(buf));
    if (keylen) {
      update(key, keylen);
      fill = 128;  // key block is a full (zero-padded) block
    }
  }
  void compress(bool last) {
    uint64_t v[16], m[16];
    for (int i = 0; i < 16; ++i) m[i] = load64(buf + 8 * i);
    for (int i = 0; i < 8; ++i) { v[i] = h[i]; v[i + 8] = IV[i]; }
    v[12] ^= t0;
    v[13] ^= t1;
    if (last) v[14] = ~v[14];
#define G(a, b, c, d, x, y)             \
  do {                                  \
    v[a] = v[a] + v[b] + (x);           \
    v[d] = rotr(v[d] ^ v[a], 32);       \
    v[c] = v[c] + v[d];                 \
    v[b] = rotr(v[b] ^ v[c], 24);       \
    v[a] = v[a] + v[b] + (y);           \
    v[d] = rotr(v[d] ^ v[a], 16);       \
    v[c] = v[c] + v[d];                 \
    v[b] = rotr(v[b] ^ v[c], 63);       \
  } while (0)
    for (int r = 0; r < 12; ++r) {
      const uint8_t* s = SIGMA[r];
      G(0, 4, 8, 12, m[s[0]], m[s[1]]);
      G(1, 5, 9, 13, m[s[2]], m[s[3]]);
      G(2, 6, 10, 14, m[s[4]], m[s[5]]);
      G(3, 7, 11, 15, m[s[6]], m[s[7]]);
      G(0, 5, 10, 15, m[s[8]], m[s[9]]);
      G(1, 6, 11, 12, m[s[10]], m[s[11]]);
      G(2, 7, 8, 13, m[s[12]], m[s[13]]);
      G(3, 4, 9, 14, m[s[14]], m[s[15]]);
    }
#undef G
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
  }
  void update(const uint8_t* in, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      if (fill == 128) {
        t0 += 128;
        if (t0 < 128) ++t1;
        compress(false);
        fill = 0;
      }
      buf[fill++] = in[i];
    }
  }
  void final(uint8_t* out) {
    t0 += fill;
    if (t0 < fill) ++t1;
    std::memset(buf + fill, 0, 128 - fill);
    compress(true);
    for (size_t i = 0; i < outlen; ++i) out[i] = (uint8_t)(h[i / 8] >> (8 * (i % 8)));
  }
};

void blake2b(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen, const uint8_t* key,
             size_t keylen) {
  Blake2b s(outlen, key, keylen);
  s.update(in, inlen);
  s.final(out);
}

struct PrfStream {
  uint8_t key[32];
  uint64_t ctr = 0;
  uint64_t words[8];
  int pos = 8;
  uint64_t next() {
    if (pos == 8) {
      uint8_t c[8], blk[64];
      for (int i = 0; i < 8; ++i) c[i] = (uint8_t)(ctr >> (8 * i));
      blake2b(blk, 64, c, 8, key, 32);
      ++ctr;
      for (int i = 0; i < 8; ++i) words[i] = load64(blk + 8 * i);
      pos = 0;
    }
    return words[pos++];
  }
  uint64_t uniform(uint64_t bound) {
    const unsigned __int128 two64 = (unsigned __int128)1 << 64;
    const unsigned __int128 span = (unsigned __int128)bound + 1;
    const unsigned __int128 limit = two64 - (two64 % span);
    for (;;) {
      uint64_t u = next();
      if ((unsigned __int128)u < limit) return (uint64_t)((unsigned __int128)u % span);
    }
  }
};

}  // namespace

void blake2b_public(uint8_t* out, size_t outlen, const uint8_t* in, size_t inlen, const uint8_t* key,
                    size_t keylen) {
  blake2b(out, outlen, in, inlen, key, keylen);
}

void derive_permutation(const uint8_t* seed, int seed_len, const uint8_t* sid, int sid_len,
                        uint32_t round_no, int64_t size, int64_t* out) {
  if (size < 1) throw std::invalid_argument("permutation size must be >= 1");
  for (int64_t i = 0; i < size; ++i) out[i] = i;
  if (round_no == 0) return;
  uint8_t skey[32], rkey[32], rb[4];
  blake2b(skey, 32, sid, (size_t)sid_len, seed, (size_t)seed_len);
  for (int i = 0; i < 4; ++i) rb[i] = (uint8_t)(round_no >> (8 * i));
  blake2b(rkey, 32, rb, 4, skey, 32);
  PrfStream s;
  std::memcpy(s.key, rkey, 32);
  for (int64_t i = size - 1; i > 0; --i) {
    const int64_t j = (int64_t)s.uniform((uint64_t)i);
    const int64_t tmp = out[i];
    out[i] = out[j];
    out[j] = tmp;
  }
}

}  // namespace sfhr
