/*
 * sfhr_b200 — C-ABI of the B200-native Safhire server hot path.
 *
 * Plain pointers and sizes only.  Unless stated otherwise, ciphertext
 * buffers are DEVICE pointers to little-endian uint64 arrays laid out exactly
 * like the reference's numpy batches: (rows, 2, N) C-contiguous, values < 2^53
 * (reference pkg/src/sfhr/crypto.py:404-406, tracepack.py:118-123).  Every
 * call that launches work takes a cudaStream_t passed as `void* stream`
 * (NULL = legacy default stream) and is asynchronous on it.
 *
 * Return codes map onto the reference's exception types in the Python shim
 * (paper_2509_01253_b200/_native.py):
 *   SFHR_EINVAL -> ValueError, SFHR_EKEY -> KeyError, SFHR_EMODEL -> ModelError,
 *   SFHR_ECUDA/SFHR_ENOMEM -> RuntimeError.  sfhr_last_error() returns the
 *   message of the calling thread's last failure.
 *
 * Thread safety: a context may be used from several host threads; calls are
 * serialised per context by an internal mutex (the reference runs one thread
 * per TCP connection, transport.py:136-156).
 */
#ifndef SFHR_B200_H
#define SFHR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  SFHR_OK = 0,
  SFHR_EINVAL = 1,
  SFHR_EKEY = 2,
  SFHR_ECUDA = 3,
  SFHR_EMODEL = 4,
  SFHR_ENOMEM = 5
};

typedef struct sfhr_ctx sfhr_ctx;
typedef struct sfhr_key sfhr_key;

/* Ring row + gadget + levels.  device = -1 creates a planning-only context
 * (no GPU required; compute entry points then return SFHR_EINVAL).  Replaces the parameter plumbing of
 * SchemeParams / KeySwitchEngine.__init__ (reference params.py:117-164,
 * crypto.py:370-382); validates like RingParams/GadgetParams/SchemeParams.
 * Uploads NTT twiddles to `device`. */
int sfhr_ctx_create(int t, int alpha, int p_bits, int D, int l, int gamma, int beta,
                    int device, sfhr_ctx** out);
int sfhr_ctx_destroy(sfhr_ctx* ctx);

/* info[0..]: M, N, n1, np (CRT primes), pack_factor, beta_eff, shrink,
 * inv_m_mod_p, cu (as int64), primes[0..np), bound_bits*1000, crt_bits*1000.
 * Returns the number of entries written (<= n). */
int sfhr_ctx_info(const sfhr_ctx* ctx, int64_t* info, int n);

/* Debug/verification: copy the device constant block (RingConst, size
 * sfhr_ringconst_bytes()) and the [np][(M + 4) & ~3] Montgomery twiddle table
 * (rows padded to a multiple of 4 words; entries 0..M used). */
size_t sfhr_ringconst_bytes(void);
int sfhr_ctx_debug_tables(const sfhr_ctx* ctx, void* ringconst, size_t rc_bytes, uint32_t* twid,
                          size_t twid_words);

/* Two-term dual basis (reference dual.py:108-166): host arrays of length N. */
int sfhr_ctx_dual(const sfhr_ctx* ctx, int32_t* e1, int32_t* e2, int32_t* ratio_len);

/* Register a key-switching key set.  Replaces KeySwitchEngine's spectra cache
 * (reference crypto.py:384-398) as built by ServerEngine.register_client
 * (protocol.py:182-194).  idx: host array of nidx automorphism indices;
 * ksk: DEVICE (nidx, l, 2, N) uint64, keys[idx[s]][i].a / .b. */
int sfhr_register_ksk(sfhr_ctx* ctx, const uint32_t* idx, int nidx, const uint64_t* ksk,
                      void* stream, sfhr_key** out);
int sfhr_key_destroy(sfhr_key* key);

/* KeySwitchEngine.automorphism_batch (reference crypto.py:400-402). */
int sfhr_automorphism_batch(sfhr_ctx* ctx, uint32_t d, const uint64_t* in, uint64_t* out,
                            int64_t B, void* stream);

/* KeySwitchEngine.switch_batch (reference crypto.py:404-421): `in` is the
 * already-automorphed batch.  counter (DEVICE u64, may be NULL) is increased
 * by the number of switched rows (live rows only when skip_zero).  in and out
 * must not alias and must be 16-byte aligned (SFHR_EINVAL otherwise). */
int sfhr_keyswitch_batch(sfhr_ctx* ctx, const sfhr_key* key, uint32_t d, const uint64_t* in,
                         uint64_t* out, int64_t B, int skip_zero,
                         unsigned long long* counter, void* stream);

/* tracepack._apply_stage_batch (reference tracepack.py:268-285):
 * out = in + sum_{rep in reps[1:]} KS_rep(aut_rep(in)).  reps: host array
 * (reps[0] must be 1).  in and out must not alias and must be 16-byte
 * aligned. */
int sfhr_stage_batch(sfhr_ctx* ctx, const sfhr_key* key, const uint32_t* reps, int nreps,
                     const uint64_t* in, uint64_t* out, int64_t B, int skip_zero,
                     unsigned long long* counter, void* stream);

/* tracepack.partial_extract for k_chunks bundles + ServerEngine._extract
 * concatenation (reference tracepack.py:118-154, protocol.py:282-294).
 * power: DEVICE (k_chunks, npow, 2, N), exponents ascending; exps: host
 * array; rows: DEVICE (E, 2, N), row j*N + i = coefficient i of chunk j. */
int sfhr_extract(sfhr_ctx* ctx, const uint64_t* power, const uint32_t* exps, int npow,
                 int k_chunks, int64_t E, uint64_t* rows, void* stream);

/* One pass of the lowered round map (reference model.py:384-429 semantics;
 * see paper_2509_01253_b200/model.py LinearPass).  All pointers DEVICE. */
typedef struct {
  const uint64_t* in;        /* pass input rows */
  const int64_t* in_map;     /* optional physical row of each pass-input column */
  const uint64_t* round_in;  /* round input rows (residual extras) */
  const int64_t* round_map;  /* optional physical row of each round-input column */
  uint64_t* out;             /* output rows */
  const int64_t* out_map;    /* optional physical output row per canonical row */
  const int32_t* groups;     /* (n_groups, 6) */
  int64_t n_groups;
  const int32_t* cols;
  const int32_t* weights;    /* [ncols][16] blocks */
  const int32_t* rows;
  const int32_t* ex_ptr;     /* optional CSR extras */
  const int32_t* ex_col;
  const int32_t* ex_w;
  const int64_t* bias;       /* optional */
  const uint64_t* unit;      /* (N,) bias unit payload, tracepack.py:157-172 */
  int64_t lanes;             /* u64 lanes per row; 0 = 2N (ciphertext rows) */
  int64_t body_off;          /* first lane receiving bias*unit (N for ciphertext rows) */
  /* Optional tensor-core tile groups (tcgen05 kind::i8; |w| <= 127): output
   * rows of consecutive shared-column groups merged into tiles of <= 256 rows,
   * their residual extras folded in as taps (the CSR extras above then apply
   * only to the groups, which must exclude the tile rows). */
  const int32_t* mma_tiles;  /* (n_mma_tiles, 8): cols_off, K_pad, w_off, rows_off, nrows, N_pad, 0, 0 */
  int64_t n_mma_tiles;
  const int32_t* mma_cols;   /* K_pad taps per tile: >= 0 pass-input row, -1 zero, <= -2 round-input row -(v+2) */
  const int32_t* mma_rows;   /* canonical output row of each tile row */
  const uint8_t* mma_w;      /* packed s8 weights, UMMA K-major no-swizzle core matrices */
  int32_t mma_max_np, mma_max_kp;  /* largest N_pad / K_pad over the tiles */
  /* Row counts of `in` / `round_in`; when given (> 0) the tensor-core tiles gather their
   * taps with TMA (tile::gather4 over a 2-D tensor map) instead of per-thread cp.async. */
  int64_t in_rows, round_in_rows;
} sfhr_linear_desc;
int sfhr_linear_pass(sfhr_ctx* ctx, const sfhr_linear_desc* desc, void* stream);
/* sizeof(sfhr_linear_desc), for binding-layout checks */
size_t sfhr_linear_desc_bytes(void);
/* Largest s8 weight operand (bytes, N_pad * K_pad) the tensor-core linear kernel keeps
 * resident in shared memory; larger tile groups stream their weights per pipeline stage.
 * The host tiler (linear.split_mma_tiles) merges groups only below this size. */
size_t sfhr_mma_b_resident_bytes(void);

/* ServerEngine._pack / tracepack.pack_rows + fast_pack (reference
 * protocol.py:296-321, tracepack.py:288-348) for n_groups zero-padded groups
 * of pack_factor rows.  rows (DEVICE, n_groups*F rows) is used as scratch and
 * clobbered; workspace: sfhr_pack_workspace_bytes(); packs: DEVICE
 * (n_groups, 2, N).  counter (DEVICE u64) += key switches (live rows only
 * when skip_zero, as ServerEngine._pack does). */
size_t sfhr_pack_workspace_bytes(const sfhr_ctx* ctx, int64_t n_groups);
int sfhr_pack(sfhr_ctx* ctx, const sfhr_key* key, uint64_t* rows, int64_t n_groups,
              uint64_t* packs, void* workspace, size_t workspace_bytes, int skip_zero,
              unsigned long long* counter, void* stream);

/* confidentiality.derive_permutation (reference confidentiality.py:27-76),
 * bit-exact: blake2b keyed tree + counter-mode PRF + descending Fisher-Yates.
 * Host-only; out: host int64[size]. */
int sfhr_derive_permutation(const uint8_t* master_seed, int seed_len, const uint8_t* session_id,
                            int sid_len, uint32_t round_no, int64_t size, int64_t* out);

/* Tensor-core forward key switch (keyswitch_tc.cu; ring row t = 7, l in {2, 3}): the
 * constant operands the library builds for each CRT prime (planning-only contexts too),
 * for host-side verification against tests/tc_model.py.  tabs: sfhr_tc_table_bytes()
 * bytes; old_idx: 42 * 49 int32.  sfhr_ctx_set_tc(ctx, k): stage launches with >= k switched
 * representatives use the tensor-core forward (k = 0: never, i.e. the CUDA-core forward of
 * ks_stage_kernel everywhere, the default: measured faster on B200); SFHR_TC_MIN_REPS=k sets
 * the default of new contexts.
 * sfhr_ctx_tc_enabled returns the current k. */
size_t sfhr_tc_table_bytes(const sfhr_ctx* ctx);
int sfhr_ctx_tc_tables(const sfhr_ctx* ctx, uint8_t* tabs, size_t tab_bytes, int32_t* old_idx);
int sfhr_ctx_tc_enabled(const sfhr_ctx* ctx);
int sfhr_ctx_set_tc(sfhr_ctx* ctx, int enable);

const char* sfhr_last_error(void);

/* Number of CUDA kernels this library has launched (process-wide counter). */
unsigned long long sfhr_launch_count(void);

/* Live kernel timing: when enabled, every key-switch stage launch is
 * bracketed by CUDA events on its stream; collect() waits for them and
 * returns the summed device time, algorithmic bytes (rows * 32 N) and count. */
int sfhr_profile_enable(sfhr_ctx* ctx, int enable);
int sfhr_profile_collect(sfhr_ctx* ctx, double* total_ms, long long* total_bytes, long long* launches);


/* ---- standalone RNS negacyclic NTT (BASELINE configs[1]; no reference
 * counterpart).  Residues are (batch, L, N) u64 on the
 * DEVICE, each limb reduced mod its ~prime_bits-bit prime p = 1 (mod 2N).
 * Forward: natural order in, bit-reversed out; inverse takes that order back
 * and includes the N^-1 scaling.  In place. */
typedef struct sfhr_ntt_plan sfhr_ntt_plan;
int sfhr_ntt_plan_create(int log2n, int L, int prime_bits, int device, sfhr_ntt_plan** out);
int sfhr_ntt_plan_destroy(sfhr_ntt_plan* plan);
int sfhr_ntt_plan_primes(const sfhr_ntt_plan* plan, uint64_t* primes, int n);
/* host copies of the [L][N] forward (psi^brv(k)) and inverse twiddles (inverse slot 0 = N^-1) */
int sfhr_ntt_plan_tables(const sfhr_ntt_plan* plan, uint64_t* w, uint64_t* wi);
int sfhr_ntt_forward(const sfhr_ntt_plan* plan, uint64_t* data, int64_t batch, void* stream);
int sfhr_ntt_inverse(const sfhr_ntt_plan* plan, uint64_t* data, int64_t batch, void* stream);
const char* sfhr_ntt_last_error(void);


/* ---- device ciphertext-block wire codec (reference wire.py:99-124, 208-254) ----
 * payload: DEVICE copy of a ROUND_REQ payload (4-byte aligned base, readable for 4
 * bytes past its end); body_offsets: DEVICE (k,) byte offsets of each chunk's block
 * body (after its 8-byte block header).  Writes out (k, npow, 2, N) u64 (lanes N..M-1 dropped) and
 * sets *err (DEVICE int, caller-zeroed) to 1 when any lane, padding included, is >= 2^53
 * (the reference's "torus numerator out of range"). */
int sfhr_wire_unpack(const uint8_t* payload, const int64_t* body_offsets, int64_t k, int npow, int M, int N,
                     uint64_t* out, int* err, void* stream);
/* rows (count, 2, N) DEVICE -> body (count, 2, M) DEVICE, zero-padded lanes (encode_block body) */
int sfhr_wire_pack(const uint64_t* rows, int64_t count, int M, int N, uint64_t* body, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SFHR_B200_H */
