// Internal kernel interfaces (not part of the public C-ABI; see include/sfhr_b200.h).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "sfhr_common.cuh"

namespace sfhr {

struct StageArgs {
  const uint64_t* in;     // (B, 2, N)
  uint64_t* out;          // (B, 2, N), may not alias in
  int64_t B;
  int nreps;              // switched representatives (identity excluded)
  int identity;           // 1: stage (acc = x + ...), 0: plain switch_batch
  int skip_zero;          // zero rows are not counted
  int shrink;             // reduce 64-bit accumulators after every rep
  uint32_t dinv[MAXREPS]; // d^-1 mod M of each rep's automorphism (1 = none)
  const uint32_t* spec[MAXREPS];  // key spectra of each rep: [l][2][np][N]
  const uint32_t* twid;   // [np][twid_stride(M)] omega^e * R mod p (e <= M)
  unsigned long long* counter;    // live-row switch counter (may be null)
  // tensor-core forward path: NTT-domain accumulators already summed over reps and digits
  // ([B][np][2][N] u32, old NTT order, any value < 2^32) -> the kernel only runs the
  // inverse transforms, CRT and identity / body terms
  const uint32_t* acc_in;
  // representative split (latency of small launches): with acc_out set, cluster (row, s) of a
  // grid of B * nsplit clusters runs reps [s nreps / nsplit, (s + 1) nreps / nsplit) and writes
  // its NTT-domain accumulators to acc_out [B][nsplit][np][2][N]; an acc_in launch with the same
  // nsplit then sums the partials (0 or 1: one set)
  uint32_t* acc_out;
  int nsplit;
  // independent CTAs (no cluster launch; the CTA's prime is blockIdx % np): set for acc_out
  // launches (no CRT) and for the L2 CRT: each CTA stores its residues of the row in
  // crt_scratch [B][crt_row_words] and the last of the row's CTAs (crt_cnt [B], zeroed by the
  // host) combines them
  int independent;
  uint32_t* crt_scratch;
  unsigned* crt_cnt;
  int group;  // independent CTAs: items per prime-major group (0: prime = blockIdx % np)
};
// u32 words of one row's CRT residues in the L2 CRT scratch (np x 2 x N, 128-byte lines)
inline __host__ __device__ size_t crt_row_words(const RingConst& rc) {
  return ((size_t)rc.np * 2 * rc.N + 31) & ~(size_t)31;
}

struct SpecArgs {
  const uint64_t* keys;   // (jobs, N) key polynomials, job = (slot*l + i)*2 + c
  uint32_t* out;          // (jobs, np, N) thread-owned layout
  const uint32_t* twid;
};

// tensor-core forward key switch (keyswitch_tc.cu), ring row t = 7, l in {2, 3}
struct TcFwdArgs {
  const uint64_t* in;           // (B, 2, N) rows
  int64_t B;
  int nreps;
  uint32_t dinv[MAXREPS];       // as StageArgs
  const uint2* keys[MAXREPS];   // per rep: [l][np][49][42] (Ka, Kb) = K^ R^2 mod p
  const uint8_t* tabs;          // per prime constant operands (tc_table_bytes)
  const int32_t* old_idx;       // [42][49] position of (o, k1) in the CUDA-core kernel's NTT order
  uint32_t* acc;                // (B, np, 2, N) NTT-domain accumulators out
  unsigned char* tiles;         // workspace: pass-A operand tiles [pair][rep][l] (tc_tile_bytes)
  int off;                      // digit offset (tc_digit_offset)
  int cpp;                      // CTAs per prime (set by the launcher)
  long long* trace;             // debug (SFHR_TC_TRACE): CTA 0's role event clocks, [4 roles][TC_TRACE_N]
};
constexpr int TC_TRACE_N = 512;
bool tc_supported(const RingConst& rc);
size_t tc_table_bytes(const RingConst& rc);
int tc_digit_offset(const RingConst& rc);
void tc_build_tables(const RingConst& rc, const uint32_t* twid, int twid_stride_words, uint8_t* tabs,
                     int32_t* old_idx);
size_t tc_fwd_smem_bytes(int L);
size_t tc_tile_bytes(const RingConst& rc, int64_t rows, int nreps);
size_t tc_keys_bytes(const RingConst& rc, int nslots);
cudaError_t launch_tc_fwd(const RingConst& rc, const TcFwdArgs& a, cudaStream_t st);
cudaError_t launch_tc_keys(const RingConst& rc, const uint32_t* spectra, int nslots, const int32_t* old_idx,
                           uint2* out, cudaStream_t st);

size_t stage_smem_bytes(const RingConst& rc);
int stage_threads(const RingConst& rc);
cudaError_t launch_stage(const RingConst& rc, const StageArgs& a, cudaStream_t st);
cudaError_t launch_spectra(const RingConst& rc, const SpecArgs& a, int njobs, cudaStream_t st);

// ---- elementwise ring ops (ring_ops.cu) ----

// out[b] = aut_d(in[b]) for (B, 2, N) batches (reference ring.py:124-130)
cudaError_t launch_automorphism(const RingConst& rc, uint32_t dinv, const uint64_t* in,
                                uint64_t* out, int64_t B, cudaStream_t st);

// merge: out[g][r] = sum_a X^(a*stride) * in[g][a*rest + r]   (tracepack.py:307-316)
cudaError_t launch_merge(const RingConst& rc, const uint64_t* in, uint64_t* out, int64_t G,
                         int members, int rest, int stride, cudaStream_t st);

struct ExtractArgs {
  const uint64_t* power;   // (k_chunks, npow, 2, N) in ascending exponent order
  uint32_t exps[64];       // (npow,) exponents
  const int32_t* cvec;     // (N,) dual ratio_len c_i
  uint64_t* rows;          // (E, 2, N), row j*N + i
  int64_t E;
  int k_chunks, npow;
  uint64_t cu;             // centered M^-1 mod p as uint64
};
cudaError_t launch_extract(const RingConst& rc, const ExtractArgs& a, cudaStream_t st);

struct LinearArgs {
  const uint64_t* in;        // pass input rows
  const int64_t* in_map;     // optional: physical row of pass-input column (first pass)
  const uint64_t* round_in;  // round input rows (for extras)
  const int64_t* round_map;  // physical row of round-input column
  uint64_t* out;             // output rows
  const int64_t* out_map;    // optional: physical output row of canonical row
  const int32_t* groups;     // (G, 6)
  const int32_t* cols;
  const int32_t* weights;    // blocks [ncols][16]
  const int32_t* rows;       // canonical output row per group row
  const int32_t* ex_ptr;     // optional CSR extras (out_len + 1)
  const int32_t* ex_col;
  const int32_t* ex_w;
  const int64_t* bias;       // optional (out_len,)
  const uint64_t* unit;      // bias unit payload (lanes - body_off,)
  int64_t G;
  int64_t lanes;             // u64 lanes per row (2N for ciphertext rows)
  int64_t body_off;          // first body lane (N)
};
cudaError_t launch_linear(const RingConst& rc, const LinearArgs& a, cudaStream_t st);

// tensor-core (tcgen05 kind::i8) variant over tile groups (linear_mma.cu)
struct LinearMmaArgs {
  CUtensorMap tm_in;         // TMA maps over the pass input / round input rows (use_tma)
  CUtensorMap tm_rin;
  int use_tma;               // 1: taps gathered by tile::gather4 TMA (rows known), 0: cp.async
  int64_t in_rows, rin_rows;
  const uint64_t* in;
  const int64_t* in_map;
  const uint64_t* round_in;
  const int64_t* round_map;
  uint64_t* out;
  const int64_t* out_map;
  const int32_t* tiles;      // (T, 8): cols_off, K_pad, w_off (bytes), rows_off, nrows, N_pad, 0, 0
  const int32_t* tcols;      // K_pad taps per tile: >= 0 pass-input row, -1 zero, <= -2 round-input row -(v+2)
  const int32_t* trows;      // canonical output rows per tile
  const uint8_t* tw;         // packed s8 B operands (UMMA K-major, no swizzle)
  const int64_t* bias;
  const uint64_t* unit;
  int64_t T;
  int64_t lanes;
  int64_t body_off;
  int mt_per_cta;            // 128-byte M-tiles per CTA
};
size_t linear_mma_smem_bytes(int Np, int Kp);
size_t linear_mma_b_resident_bytes();
cudaError_t launch_linear_mma(const LinearMmaArgs& a, int max_np, int max_kp, cudaStream_t st);

}  // namespace sfhr
