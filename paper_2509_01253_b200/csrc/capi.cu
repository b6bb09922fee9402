// extern "C" boundary of libsfhr_b200.so (declared in include/sfhr_b200.h).
// Host orchestration of the pack schedule lives here; all compute is in the
// kernels of keyswitch.cu / ring_ops.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/sfhr_b200.h"
#include "plan.h"
#include "sfhr_kernels.h"

namespace sfhr {
void derive_permutation(const uint8_t* seed, int seed_len, const uint8_t* sid, int sid_len,
                        uint32_t round_no, int64_t size, int64_t* out);
}

using namespace sfhr;

struct ProfRec {
  cudaEvent_t a, b;
  long long bytes;
};

struct sfhr_ctx {
  Plan plan;
  int device = 0;
  bool prof = false;                 // time every stage launch with CUDA events
  std::vector<ProfRec> prof_recs;    // pending (unresolved) records
  std::vector<cudaEvent_t> ev_pool;  // recycled events
  uint32_t* twid = nullptr;  // [np][twid_stride(M)]
  int32_t* cvec = nullptr;   // [N]
  // tensor-core forward key switch (keyswitch_tc.cu): constant operands per prime and the
  // NTT-order map; null when the ring row has no tensor-core path or SFHR_TC=0
  uint8_t* tc_tabs = nullptr;
  int32_t* tc_oldidx = nullptr;
  int tc_min_reps = 0;       // stage launches with >= this many switched reps take the tensor-core
                             // path (0: never; sfhr_ctx_set_tc)
  uint32_t* tc_ws = nullptr;  // NTT-domain accumulator workspace (grow-only), last used on ...
  size_t tc_ws_bytes = 0;
  cudaEvent_t tc_ws_free = nullptr;  // ... the stream position recorded here
  uint32_t* crt_ws = nullptr;  // L2 CRT residues + row counters (grow-only), same protocol
  size_t crt_ws_bytes = 0;
  cudaEvent_t crt_ws_free = nullptr;
  std::mutex mu;
};

struct sfhr_key {
  sfhr_ctx* ctx = nullptr;
  std::map<uint32_t, int> slot;  // d -> slot
  uint32_t* spectra = nullptr;   // [nidx][l][2][np][N]
  size_t slot_words = 0;
  mutable uint2* tc_keys = nullptr;  // [nidx][l][np][49][42] tensor-core MAC operands, built on first use
  int nidx = 0;
};

namespace {
thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};  // kernels launched through this library
const bool g_debug_sync = std::getenv("SFHR_DEBUG_SYNC") != nullptr;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}
int cuda_fail(cudaError_t e, const char* where) {
  return fail(SFHR_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call, where)                          \
  do {                                           \
    cudaError_t _e = (call);                     \
    if (_e != cudaSuccess) return cuda_fail(_e, where); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

// 2-D TMA map over (rows, lanes) u64 rows: box = 16 lanes x 1 row, 128B swizzle (the UMMA A layout),
// out-of-bounds rows / lanes zero-filled.  cuTensorMapEncodeTiled comes from the driver entry point.
bool make_row_map(CUtensorMap* m, const void* base, int64_t rows, int64_t lanes) {
  using Fn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                          const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                          CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static Fn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<Fn>(p);
  });
  if (!fn || !base || rows <= 0 || rows > 0x7ffffffe || lanes <= 0) return false;
  const cuuint64_t dims[2] = {(cuuint64_t)lanes, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)lanes * 8};
  const cuuint32_t box[2] = {16, 1};
  const cuuint32_t estr[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int key_slot(const sfhr_key* key, uint32_t d) {
  const uint32_t M = (uint32_t)key->ctx->plan.rc.M;
  auto it = key->slot.find(d % M);
  if (it == key->slot.end()) return -1;
  return it->second;
}

// Clusters per row of a representative-split launch: enough to give ~SFHR_REP_SPLIT clusters per
// SM when a launch has few rows (default 1; 0 disables)
int rep_split(int nreps, int64_t B) {
  static const int enabled = [] {
    const char* e = std::getenv("SFHR_REP_SPLIT");
    return e ? std::atoi(e) : 1;
  }();
  static int nsm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  }
  if (!enabled || nreps < 2 || B <= 0) return 1;
  const int64_t want = (int64_t)enabled * nsm / B;
  return (int)std::max<int64_t>(1, std::min<int64_t>(nreps, want));
}

// grow-only device workspace; a call waits (stream-ordered) for the previous user recorded on
// its event
int grow_workspace(uint32_t*& buf, size_t& have, cudaEvent_t& ev, size_t bytes, cudaStream_t st, uint32_t** out) {
  if (!ev) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "workspace event");
  if (bytes > have) {  // grow (rare): wait for the last user before freeing
    CK(cudaEventSynchronize(ev), "workspace sync");
    cudaFree(buf);
    buf = nullptr;
    have = 0;
    CK(cudaMalloc(reinterpret_cast<void**>(&buf), bytes), "workspace alloc");
    have = bytes;
  }
  CK(cudaStreamWaitEvent(st, ev, 0), "workspace wait");  // a previous caller's stream
  *out = buf;
  return SFHR_OK;
}

// the context's accumulator workspace, shared by the tensor-core and representative-split paths
int workspace(sfhr_ctx* ctx, size_t bytes, cudaStream_t st, uint32_t** out) {
  return grow_workspace(ctx->tc_ws, ctx->tc_ws_bytes, ctx->tc_ws_free, bytes, st, out);
}

// Stage launches finish with the explicit CRT of each row over its np prime CTAs.  Default
// (SFHR_STAGE_CLUSTER unset or 0): independent CTAs and a CRT through L2 (crt_scratch, last
// arriver); SFHR_STAGE_CLUSTER=1: the CTAs of a row form a thread-block cluster and exchange
// residues through distributed shared memory.  Clusters of 3 CTAs leave 4 % of the CTA slots
// of a B200 unusable (cudaOccupancyMaxActiveClusters: 142 x 3 of 148 x 3) and make every CTA
// wait for its slowest peer.
bool stage_clusters() {
  static const bool on = [] {
    const char* e = std::getenv("SFHR_STAGE_CLUSTER");
    return e && std::atoi(e) != 0;
  }();
  return on;
}

// items per prime-major CTA group of an independent stage launch (SFHR_STAGE_GROUP; default
// 444 = one wave of b = 12 CTAs on 148 SMs)
int stage_group() {
  static const int v = [] {
    const char* e = std::getenv("SFHR_STAGE_GROUP");
    return e ? std::atoi(e) : 444;
  }();
  return v;
}

// launches with fewer rows than this keep the cluster CRT: they are latency bound, and the L2
// CRT's last arriver serialises the whole row's CRT (SFHR_CRT_MIN_ROWS, default one row per SM)
int64_t crt_min_rows() {
  static const int64_t v = [] {
    const char* e = std::getenv("SFHR_CRT_MIN_ROWS");
    if (e) return (int64_t)std::atoll(e);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return (int64_t)nsm;
  }();
  return v;
}

// launch a stage (or the acc_in tail of a split / tensor-core stage) with the configured CRT;
// rows go in equal chunks of at most CRT_CHUNK_ROWS (scratch <= 1.6 GB at b = 12; its lines are
// discarded from L2 after use, so it costs address space, not HBM traffic)
constexpr int64_t CRT_CHUNK_ROWS = 32768;
int launch_stage_crt(sfhr_ctx* ctx, const StageArgs& a, cudaStream_t st, const char* what) {
  const RingConst& rc = ctx->plan.rc;
  if (stage_clusters() || a.B < crt_min_rows()) {
    CK(launch_stage(rc, a, st), what);
    return SFHR_OK;
  }
  const size_t row_words = crt_row_words(rc);
  const int64_t nch = (a.B + CRT_CHUNK_ROWS - 1) / CRT_CHUNK_ROWS;
  const int64_t chunk = (a.B + nch - 1) / nch;
  const size_t scratch_bytes = (size_t)chunk * row_words * 4;
  uint32_t* ws = nullptr;
  if (const int rc_ = grow_workspace(ctx->crt_ws, ctx->crt_ws_bytes, ctx->crt_ws_free,
                                     scratch_bytes + (size_t)chunk * 4, st, &ws))
    return rc_;
  unsigned* cnt = reinterpret_cast<unsigned*>(ws + (size_t)chunk * row_words);
  const int parts = a.nsplit > 1 ? a.nsplit : 1;
  for (int64_t r0 = 0; r0 < a.B; r0 += chunk) {
    StageArgs c = a;
    c.B = std::min<int64_t>(chunk, a.B - r0);
    c.in = a.in + r0 * 2 * rc.N;
    c.out = a.out + r0 * 2 * rc.N;
    if (a.acc_in) c.acc_in = a.acc_in + (size_t)r0 * parts * rc.np * 2 * rc.N;
    c.independent = 1;
    c.crt_scratch = ws;
    c.crt_cnt = cnt;
    // prime-major groups only for launches of several waves: in a short launch they push every
    // row's last arriver (the CRT) to the end of the launch
    c.group = c.B >= 4 * (int64_t)stage_group() ? stage_group() : 0;
    CK(cudaMemsetAsync(cnt, 0, (size_t)c.B * 4, st), "CRT counters");
    CK(launch_stage(rc, c, st), what);
    if (r0) ++g_launches;  // the callers count one launch per stage
  }
  CK(cudaEventRecord(ctx->crt_ws_free, st), "CRT workspace release");
  return SFHR_OK;
}

int64_t tc_chunk_rows() {
  static const int64_t rows = [] {
    const char* e = std::getenv("SFHR_TC_CHUNK");
    const long long v = e ? std::atoll(e) : 0;
    return (int64_t)(v > 0 ? v : 2048);
  }();
  return rows;
}

// The tensor-core forward (keyswitch_tc.cu) is bit-exact but measured slower than the CUDA-core
// forward on B200 (ResNet-20 stage kernel 132 -> 141 ms with it on 6-rep stages,
// 24 -> 32 ms at gamma = 1), so it is opt-in: SFHR_TC_MIN_REPS=k (or sfhr_ctx_set_tc) routes
// stage launches with >= k switched representatives through it.
int tc_default_min_reps() {
  const char* e = std::getenv("SFHR_TC_MIN_REPS");
  const int v = e ? std::atoi(e) : 0;
  return v > 0 ? v : 0;
}

int run_stage(sfhr_ctx* ctx, const sfhr_key* key, const uint32_t* reps, int nreps, int identity,
              const uint64_t* in, uint64_t* out, int64_t B, int skip_zero,
              unsigned long long* counter, cudaStream_t st) {
  const Plan& P = ctx->plan;
  StageArgs a;
  std::memset(&a, 0, sizeof(a));
  a.in = in;
  a.out = out;
  a.B = B;
  a.identity = identity;
  a.skip_zero = skip_zero;
  a.shrink = P.shrink;
  a.twid = ctx->twid;
  a.counter = counter;
  int ns = 0;
  for (int r = 0; r < nreps; ++r) {
    const uint32_t d = reps[r] % (uint32_t)P.rc.M;
    if (identity && r == 0) {
      if (d != 1) return fail(SFHR_EINVAL, "stage representatives must start with the identity");
      continue;
    }
    if (ns >= MAXREPS) return fail(SFHR_EINVAL, "too many representatives in one stage");
    const int s = key_slot(key, d);
    if (s < 0) return fail(SFHR_EKEY, "key-switch key set has no index " + std::to_string(d));
    a.spec[ns] = key->spectra + (size_t)s * key->slot_words;
    a.dinv[ns] = identity ? inv_mod_M(P, d) : 1u;
    ++ns;
  }
  a.nreps = ns;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (ctx->prof && ns > 0 && B > 0) {
    for (cudaEvent_t* e : {&e0, &e1}) {
      if (!ctx->ev_pool.empty()) {
        *e = ctx->ev_pool.back();
        ctx->ev_pool.pop_back();
      } else {
        CK(cudaEventCreate(e), "event create");
      }
    }
    CK(cudaEventRecord(e0, st), "event record");
  }
  if (ns == 0) {
    if (in != out) CK(cudaMemcpyAsync(out, in, (size_t)B * 2 * P.rc.N * 8, cudaMemcpyDeviceToDevice, st), "stage copy");
    return SFHR_OK;
  }
  const bool use_tc = ctx->tc_min_reps > 0 && ctx->tc_tabs && key->nidx > 0 && ns >= ctx->tc_min_reps;
  if (use_tc && !key->tc_keys) {  // the tensor-core MAC operands of this key set, on first use
    CK(cudaMalloc(reinterpret_cast<void**>(&key->tc_keys), tc_keys_bytes(P.rc, key->nidx)), "tc key alloc");
    CK(launch_tc_keys(P.rc, key->spectra, key->nidx, ctx->tc_oldidx, key->tc_keys, st), "tc key kernel");
    ++g_launches;
  }
  if (use_tc) {
    // tensor-core forward (NTT-domain accumulators) + the CUDA-core kernel's inverse / CRT tail,
    // in chunks whose accumulators (49 KB per row at b = 12) stay L2-sized
    TcFwdArgs f;
    std::memset(&f, 0, sizeof(f));
    f.nreps = ns;
    f.tabs = ctx->tc_tabs;
    f.old_idx = ctx->tc_oldidx;
    f.off = tc_digit_offset(P.rc);
    for (int r = 0; r < ns; ++r) {
      f.dinv[r] = a.dinv[r];
      f.keys[r] = key->tc_keys + (size_t)(a.spec[r] - key->spectra) / key->slot_words *
                                     (tc_keys_bytes(P.rc, 1) / sizeof(uint2));
    }
    // chunks: the operand tiles of a chunk (nreps * l * 6 KB per row) stay L2-sized
    const int64_t per_row_tiles = (int64_t)tc_tile_bytes(P.rc, 2, ns) / 2;
    int64_t chunk = std::min<int64_t>(tc_chunk_rows(), std::max<int64_t>(2, (64ll << 20) / per_row_tiles));
    chunk &= ~1ll;
    const size_t acc_bytes = (size_t)std::min<int64_t>(B, chunk) * P.rc.np * 2 * P.rc.N * 4;
    const size_t tile_bytes = tc_tile_bytes(P.rc, std::min<int64_t>(B, chunk), ns);
    const size_t ws_bytes = ((acc_bytes + 1023) & ~(size_t)1023) + tile_bytes;
    uint32_t* acc = nullptr;
    if (const int rc_ = workspace(ctx, ws_bytes, st, &acc)) return rc_;
    f.tiles = reinterpret_cast<unsigned char*>(ctx->tc_ws) + ((acc_bytes + 1023) & ~(size_t)1023);
    for (int64_t r0 = 0; r0 < B; r0 += chunk) {
      const int64_t nb = std::min<int64_t>(chunk, B - r0);
      f.in = in + r0 * 2 * P.rc.N;
      f.B = nb;
      f.acc = acc;
      static const bool tc_trace = std::getenv("SFHR_TC_TRACE") != nullptr;
      std::vector<long long> trace_host;
      if (tc_trace) {
        CK(cudaMallocAsync(reinterpret_cast<void**>(&f.trace), 4 * TC_TRACE_N * 8, st), "trace alloc");
        CK(cudaMemsetAsync(f.trace, 0, 4 * TC_TRACE_N * 8, st), "trace memset");
      }
      CK(launch_tc_fwd(P.rc, f, st), "tensor-core key-switch kernel");
      if (tc_trace) {  // debug timeline of CTA 0 (SFHR_TC_TRACE=1), one line per role
        trace_host.resize(4 * TC_TRACE_N);
        CK(cudaMemcpyAsync(trace_host.data(), f.trace, trace_host.size() * 8, cudaMemcpyDeviceToHost, st), "trace copy");
        CK(cudaStreamSynchronize(st), "trace sync");
        CK(cudaFree(f.trace), "trace free");
        f.trace = nullptr;
        long long t0 = trace_host[0];
        for (long long v : trace_host) if (v && v < t0) t0 = v;
        std::fprintf(stderr, "[tc-trace] B=%lld nreps=%d\n", (long long)nb, ns);
        for (int role = 0; role < 4; ++role) {
          std::fprintf(stderr, "[tc-trace] role %d:", role);
          for (int k = 0; k < TC_TRACE_N; ++k) {
            const long long v = trace_host[role * TC_TRACE_N + k];
            if (!v) break;
            std::fprintf(stderr, " %lld", v - t0);
          }
          std::fprintf(stderr, "\n");
        }
      }
      StageArgs t = a;
      t.in = in + r0 * 2 * P.rc.N;
      t.out = out + r0 * 2 * P.rc.N;
      t.B = nb;
      t.acc_in = acc;
      if (const int rc_ = launch_stage_crt(ctx, t, st, "stage kernel (inverse / CRT)")) return rc_;
      g_launches += 3;
    }
    CK(cudaEventRecord(ctx->tc_ws_free, st), "tc workspace release");
    --g_launches;  // counted once below (digits + tensor-core forward + inverse per chunk)
  } else if (const int split = rep_split(ns, B); split > 1) {
    // few rows (late tower stages, small models): the representatives of a row are spread over
    // `split` clusters whose NTT-domain partial sums the second launch adds before the inverse
    const size_t ws_bytes = (size_t)B * split * P.rc.np * 2 * P.rc.N * 4;
    uint32_t* ws = nullptr;
    if (const int rc_ = workspace(ctx, ws_bytes, st, &ws)) return rc_;
    StageArgs s1 = a;
    s1.acc_out = ws;
    s1.nsplit = split;
    s1.independent = 1;  // no CRT in this half: its CTAs never talk to each other
    s1.group = B * split >= 4 * (int64_t)stage_group() ? stage_group() : 0;
    CK(launch_stage(P.rc, s1, st), "stage kernel (representative split)");
    StageArgs s2 = a;
    s2.acc_in = ws;
    s2.nsplit = split;
    if (const int rc_ = launch_stage_crt(ctx, s2, st, "stage kernel (inverse / CRT)")) return rc_;
    CK(cudaEventRecord(ctx->tc_ws_free, st), "workspace release");
    ++g_launches;
  } else {
    if (const int rc_ = launch_stage_crt(ctx, a, st, "stage kernel")) return rc_;
  }
  if (g_debug_sync) {  // SFHR_DEBUG_SYNC=1: locate a faulting launch
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) {
      std::fprintf(stderr, "[sfhr] stage kernel failed: B=%lld nreps=%d identity=%d in=%p out=%p: %s\n",
                   (long long)B, a.nreps, identity, (const void*)in, (void*)out, cudaGetErrorString(e));
      return cuda_fail(e, "stage kernel (debug sync)");
    }
  }
  ++g_launches;
  if (e0) {
    CK(cudaEventRecord(e1, st), "event record");
    ctx->prof_recs.push_back({e0, e1, (long long)B * 32LL * P.rc.N});
  }
  return SFHR_OK;
}
}  // namespace

extern "C" {

const char* sfhr_last_error(void) { return g_err.c_str(); }

unsigned long long sfhr_launch_count(void) { return g_launches.load(); }

int sfhr_profile_enable(sfhr_ctx* ctx, int enable) {
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  ctx->prof = enable != 0;
  return SFHR_OK;
}

int sfhr_profile_collect(sfhr_ctx* ctx, double* total_ms, long long* total_bytes, long long* launches) {
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  double ms = 0;
  long long by = 0, n = 0;
  for (auto& r : ctx->prof_recs) {
    CK(cudaEventSynchronize(r.b), "event sync");
    float t = 0;
    CK(cudaEventElapsedTime(&t, r.a, r.b), "event elapsed");
    ms += t;
    by += r.bytes;
    ++n;
    ctx->ev_pool.push_back(r.a);
    ctx->ev_pool.push_back(r.b);
  }
  ctx->prof_recs.clear();
  if (total_ms) *total_ms = ms;
  if (total_bytes) *total_bytes = by;
  if (launches) *launches = n;
  return SFHR_OK;
}

int sfhr_ctx_create(int t, int alpha, int p_bits, int D, int l, int gamma, int beta, int device,
                    sfhr_ctx** out) {
  if (!out) return fail(SFHR_EINVAL, "null output pointer");
  sfhr_ctx* ctx = new (std::nothrow) sfhr_ctx();
  if (!ctx) return fail(SFHR_ENOMEM, "out of host memory");
  try {
    ctx->plan = make_plan(t, alpha, p_bits, D, l, gamma, beta);
  } catch (const std::exception& e) {
    delete ctx;
    return fail(SFHR_EINVAL, e.what());
  }
  ctx->device = device;
  if (device < 0) {  // planning-only context (no GPU needed): info/dual/debug tables
    *out = ctx;
    return SFHR_OK;
  }
  DeviceGuard g(device);
  const Plan& P = ctx->plan;
  cudaError_t e = cudaMalloc(&ctx->twid, P.twid.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->twid, P.twid.data(), P.twid.size() * 4, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&ctx->cvec, P.cvec.size() * 4);
  if (e == cudaSuccess) e = cudaMemcpy(ctx->cvec, P.cvec.data(), P.cvec.size() * 4, cudaMemcpyHostToDevice);
  const char* tc_env = std::getenv("SFHR_TC");
  ctx->tc_min_reps = tc_supported(P.rc) && !(tc_env && tc_env[0] == '0') ? tc_default_min_reps() : 0;
  if (e == cudaSuccess && tc_supported(P.rc)) {
    std::vector<uint8_t> tabs(tc_table_bytes(P.rc));
    std::vector<int32_t> oi(42 * 49);
    tc_build_tables(P.rc, P.twid.data(), twid_stride(P.rc.M), tabs.data(), oi.data());
    e = cudaMalloc(&ctx->tc_tabs, tabs.size());
    if (e == cudaSuccess) e = cudaMemcpy(ctx->tc_tabs, tabs.data(), tabs.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&ctx->tc_oldidx, oi.size() * 4);
    if (e == cudaSuccess) e = cudaMemcpy(ctx->tc_oldidx, oi.data(), oi.size() * 4, cudaMemcpyHostToDevice);
  }
  if (e != cudaSuccess) {
    cudaFree(ctx->twid);
    cudaFree(ctx->cvec);
    cudaFree(ctx->tc_tabs);
    cudaFree(ctx->tc_oldidx);
    delete ctx;
    return cuda_fail(e, "ctx create");
  }
  *out = ctx;
  return SFHR_OK;
}

int sfhr_ctx_destroy(sfhr_ctx* ctx) {
  if (!ctx) return SFHR_OK;
  if (ctx->device < 0) {
    delete ctx;
    return SFHR_OK;
  }
  DeviceGuard g(ctx->device);
  for (auto& r : ctx->prof_recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  cudaFree(ctx->twid);
  cudaFree(ctx->cvec);
  cudaFree(ctx->tc_tabs);
  cudaFree(ctx->tc_oldidx);
  if (ctx->tc_ws_free) cudaEventSynchronize(ctx->tc_ws_free);
  cudaFree(ctx->tc_ws);
  if (ctx->tc_ws_free) cudaEventDestroy(ctx->tc_ws_free);
  if (ctx->crt_ws_free) cudaEventSynchronize(ctx->crt_ws_free);
  cudaFree(ctx->crt_ws);
  if (ctx->crt_ws_free) cudaEventDestroy(ctx->crt_ws_free);
  delete ctx;
  return SFHR_OK;
}

int sfhr_ctx_info(const sfhr_ctx* ctx, int64_t* info, int n) {
  if (!ctx || !info) return -1;
  const Plan& P = ctx->plan;
  std::vector<int64_t> v = {P.rc.M, P.rc.N, P.rc.n1, P.rc.np, P.pack_factor, P.beta, P.shrink,
                            P.inv_m_mod_p, (int64_t)P.cu};
  for (int i = 0; i < P.rc.np; ++i) v.push_back(P.rc.pc[i].p);
  v.push_back((int64_t)(P.bound_bits * 1000));
  v.push_back((int64_t)(P.crt_bits * 1000));
  int k = std::min<int>(n, (int)v.size());
  for (int i = 0; i < k; ++i) info[i] = v[i];
  return k;
}

int sfhr_ctx_debug_tables(const sfhr_ctx* ctx, void* ringconst, size_t rc_bytes, uint32_t* twid,
                          size_t twid_words) {
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  const Plan& P = ctx->plan;
  if (rc_bytes != sizeof(RingConst)) return fail(SFHR_EINVAL, "RingConst size mismatch");
  std::memcpy(ringconst, &P.rc, sizeof(RingConst));
  if (twid) std::memcpy(twid, P.twid.data(), std::min(twid_words, P.twid.size()) * 4);
  return SFHR_OK;
}

int sfhr_ctx_tc_tables(const sfhr_ctx* ctx, uint8_t* tabs, size_t tab_bytes, int32_t* old_idx) {
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  const Plan& P = ctx->plan;
  if (!tc_supported(P.rc)) return fail(SFHR_EINVAL, "ring row has no tensor-core key-switch path");
  if (tab_bytes != tc_table_bytes(P.rc)) return fail(SFHR_EINVAL, "tensor-core table size mismatch");
  tc_build_tables(P.rc, P.twid.data(), twid_stride(P.rc.M), tabs, old_idx);
  return SFHR_OK;
}

size_t sfhr_tc_table_bytes(const sfhr_ctx* ctx) {
  return ctx && tc_supported(ctx->plan.rc) ? tc_table_bytes(ctx->plan.rc) : 0;
}

int sfhr_ctx_tc_enabled(const sfhr_ctx* ctx) { return ctx && ctx->tc_tabs ? ctx->tc_min_reps : 0; }

int sfhr_ctx_set_tc(sfhr_ctx* ctx, int min_reps) {
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  if (min_reps < 0) return fail(SFHR_EINVAL, "negative representative threshold");
  if (min_reps && !ctx->tc_tabs) return fail(SFHR_EINVAL, "ring row has no tensor-core key-switch path");
  ctx->tc_min_reps = min_reps;
  return SFHR_OK;
}

size_t sfhr_ringconst_bytes(void) { return sizeof(RingConst); }

size_t sfhr_linear_desc_bytes(void) { return sizeof(sfhr_linear_desc); }
size_t sfhr_mma_b_resident_bytes(void) { return sfhr::linear_mma_b_resident_bytes(); }

int sfhr_ctx_dual(const sfhr_ctx* ctx, int32_t* e1, int32_t* e2, int32_t* ratio_len) {
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  const Plan& P = ctx->plan;
  std::memcpy(e1, P.e1.data(), P.e1.size() * 4);
  std::memcpy(e2, P.e2.data(), P.e2.size() * 4);
  std::memcpy(ratio_len, P.cvec.data(), P.cvec.size() * 4);
  return SFHR_OK;
}

int sfhr_register_ksk(sfhr_ctx* ctx, const uint32_t* idx, int nidx, const uint64_t* ksk, void* stream,
                      sfhr_key** out) {
  if (ctx && ctx->device < 0) return fail(SFHR_EINVAL, "planning-only context (device -1) cannot compute");
  if (!ctx || !out || (nidx > 0 && (!idx || !ksk))) return fail(SFHR_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const Plan& P = ctx->plan;
  const RingConst& rc = P.rc;
  sfhr_key* key = new (std::nothrow) sfhr_key();
  if (!key) return fail(SFHR_ENOMEM, "out of host memory");
  key->ctx = ctx;
  for (int s = 0; s < nidx; ++s) {
    const uint32_t d = idx[s] % (uint32_t)rc.M;
    if (std::gcd((long long)d, (long long)rc.M) != 1) {
      delete key;
      return fail(SFHR_EINVAL, "key-switch index " + std::to_string(d) + " not coprime with M");
    }
    key->slot[d] = s;
  }
  key->slot_words = (size_t)rc.l * 2 * rc.np * rc.N;
  const size_t bytes = (size_t)std::max(nidx, 1) * key->slot_words * 4;
  cudaError_t e = cudaMalloc(&key->spectra, bytes);
  if (e != cudaSuccess) {
    delete key;
    return cuda_fail(e, "ksk spectra alloc");
  }
  SpecArgs a;
  a.keys = ksk;
  a.out = key->spectra;
  a.twid = ctx->twid;
  e = launch_spectra(rc, a, nidx * rc.l * 2, (cudaStream_t)stream);
  if (nidx) ++g_launches;
  key->nidx = nidx;
  if (e != cudaSuccess) {
    cudaFree(key->spectra);
    delete key;
    return cuda_fail(e, "ksk spectra kernel");
  }
  *out = key;
  return SFHR_OK;
}

int sfhr_key_destroy(sfhr_key* key) {
  if (!key) return SFHR_OK;
  DeviceGuard g(key->ctx->device);
  cudaFree(key->spectra);
  cudaFree(key->tc_keys);
  delete key;
  return SFHR_OK;
}

int sfhr_automorphism_batch(sfhr_ctx* ctx, uint32_t d, const uint64_t* in, uint64_t* out, int64_t B,
                            void* stream) {
  if (ctx && ctx->device < 0) return fail(SFHR_EINVAL, "planning-only context (device -1) cannot compute");
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  uint32_t dinv;
  try {
    dinv = inv_mod_M(ctx->plan, d);
  } catch (const std::exception& ex) {
    return fail(SFHR_EINVAL, ex.what());
  }
  CK(launch_automorphism(ctx->plan.rc, dinv, in, out, B, (cudaStream_t)stream), "automorphism kernel");
  if (B) ++g_launches;
  return SFHR_OK;
}

int sfhr_keyswitch_batch(sfhr_ctx* ctx, const sfhr_key* key, uint32_t d, const uint64_t* in, uint64_t* out,
                         int64_t B, int skip_zero, unsigned long long* counter, void* stream) {
  if (ctx && ctx->device < 0) return fail(SFHR_EINVAL, "planning-only context (device -1) cannot compute");
  if (!ctx || !key) return fail(SFHR_EINVAL, "null argument");
  if (B == 0) return SFHR_OK;
  if (in == out) return fail(SFHR_EINVAL, "in and out must not alias");
  // the stage kernel bulk-copies rows into shared memory (cp.async.bulk: 16-byte granules)
  if (((uintptr_t)in | (uintptr_t)out) & 15) return fail(SFHR_EINVAL, "in and out must be 16-byte aligned");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  uint32_t reps[1] = {d};
  return run_stage(ctx, key, reps, 1, 0, in, out, B, skip_zero, counter, (cudaStream_t)stream);
}

int sfhr_stage_batch(sfhr_ctx* ctx, const sfhr_key* key, const uint32_t* reps, int nreps, const uint64_t* in,
                     uint64_t* out, int64_t B, int skip_zero, unsigned long long* counter, void* stream) {
  if (ctx && ctx->device < 0) return fail(SFHR_EINVAL, "planning-only context (device -1) cannot compute");
  if (!ctx || !key || !reps || nreps < 1) return fail(SFHR_EINVAL, "bad argument");
  if (B == 0) return SFHR_OK;
  if (in == out) return fail(SFHR_EINVAL, "in and out must not alias");
  // the stage kernel bulk-copies rows into shared memory (cp.async.bulk: 16-byte granules)
  if (((uintptr_t)in | (uintptr_t)out) & 15) return fail(SFHR_EINVAL, "in and out must be 16-byte aligned");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  try {
    return run_stage(ctx, key, reps, nreps, 1, in, out, B, skip_zero, counter, (cudaStream_t)stream);
  } catch (const std::exception& ex) {
    return fail(SFHR_EINVAL, ex.what());
  }
}

int sfhr_extract(sfhr_ctx* ctx, const uint64_t* power, const uint32_t* exps, int npow, int k_chunks, int64_t E,
                 uint64_t* rows, void* stream) {
  if (ctx && ctx->device < 0) return fail(SFHR_EINVAL, "planning-only context (device -1) cannot compute");
  if (!ctx) return fail(SFHR_EINVAL, "null context");
  const Plan& P = ctx->plan;
  if (E < 0 || E > (int64_t)k_chunks * P.rc.N) return fail(SFHR_EINVAL, "row count exceeds chunk capacity");
  if (npow < 1 || npow > 64) return fail(SFHR_EINVAL, "bad power count");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  ExtractArgs a;
  std::memset(&a, 0, sizeof(a));
  a.power = power;
  for (int q = 0; q < npow; ++q) a.exps[q] = exps[q] % (uint32_t)P.rc.M;
  a.cvec = ctx->cvec;
  a.rows = rows;
  a.E = E;
  a.k_chunks = k_chunks;
  a.npow = npow;
  a.cu = P.cu;
  CK(launch_extract(P.rc, a, (cudaStream_t)stream), "extract kernel");
  if (E) ++g_launches;
  return SFHR_OK;
}

int sfhr_linear_pass(sfhr_ctx* ctx, const sfhr_linear_desc* d, void* stream) {
  if (ctx && ctx->device < 0) return fail(SFHR_EINVAL, "planning-only context (device -1) cannot compute");
  if (!ctx || !d) return fail(SFHR_EINVAL, "null argument");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  LinearArgs a;
  a.in = d->in;
  a.in_map = d->in_map;
  a.round_in = d->round_in;
  a.round_map = d->round_map;
  a.out = d->out;
  a.out_map = d->out_map;
  a.groups = d->groups;
  a.cols = d->cols;
  a.weights = d->weights;
  a.rows = d->rows;
  a.ex_ptr = d->ex_ptr;
  a.ex_col = d->ex_col;
  a.ex_w = d->ex_w;
  a.bias = d->bias;
  a.unit = d->unit;
  a.G = d->n_groups;
  a.lanes = d->lanes ? d->lanes : 2 * (int64_t)ctx->plan.rc.N;
  a.body_off = d->lanes ? d->body_off : ctx->plan.rc.N;
  if (a.lanes > 65535LL * 128) return fail(SFHR_EINVAL, "too many lanes per row");
  CK(launch_linear(ctx->plan.rc, a, (cudaStream_t)stream), "linear kernel");
  if (a.G) ++g_launches;
  if (d->n_mma_tiles > 0) {
    if (!d->mma_tiles || !d->mma_cols || !d->mma_rows || !d->mma_w)
      return fail(SFHR_EINVAL, "incomplete tensor-core tile description");
    LinearMmaArgs m;
    std::memset(&m, 0, sizeof(m));
    m.in = a.in;
    m.in_map = a.in_map;
    m.round_in = a.round_in;
    m.round_map = a.round_map;
    m.out = a.out;
    m.out_map = a.out_map;
    m.tiles = d->mma_tiles;
    m.tcols = d->mma_cols;
    m.trows = d->mma_rows;
    m.tw = d->mma_w;
    m.bias = a.bias;
    m.unit = a.unit;
    m.T = d->n_mma_tiles;
    m.lanes = a.lanes;
    m.body_off = a.body_off;
    // M-tiles per CTA: enough CTAs to fill the GPU several times, <= 16 tiles so the
    // column slice all tile groups of a wave touch stays L2-resident
    const int64_t n_mt = (a.lanes + 15) / 16;
    int64_t per = (m.T * n_mt + 148 * 8 - 1) / (148 * 8);
    per = per < 1 ? 1 : (per > 16 ? 16 : per);
    const int64_t chunks = (n_mt + per - 1) / per;
    m.mt_per_cta = (int)((n_mt + chunks - 1) / chunks);
    m.in_rows = d->in_rows;
    m.rin_rows = d->round_in_rows;
    m.use_tma = 0;
    if (d->in_rows > 0 && a.lanes % 2 == 0) {
      const bool rin_ok = d->round_in_rows > 0 && a.round_in;
      if (make_row_map(&m.tm_in, a.in, d->in_rows, a.lanes) &&
          make_row_map(&m.tm_rin, rin_ok ? a.round_in : a.in, rin_ok ? d->round_in_rows : d->in_rows, a.lanes))
        m.use_tma = 1;
    }
    CK(launch_linear_mma(m, d->mma_max_np, d->mma_max_kp, (cudaStream_t)stream), "linear tensor-core kernel");
    ++g_launches;
  }
  return SFHR_OK;
}

size_t sfhr_pack_workspace_bytes(const sfhr_ctx* ctx, int64_t n_groups) {
  if (!ctx) return 0;
  return (size_t)n_groups * ctx->plan.pack_factor * 2 * ctx->plan.rc.N * 8;
}

int sfhr_pack(sfhr_ctx* ctx, const sfhr_key* key, uint64_t* rows, int64_t G, uint64_t* packs, void* ws,
              size_t ws_bytes, int skip_zero, unsigned long long* counter, void* stream) {
  if (ctx && ctx->device < 0) return fail(SFHR_EINVAL, "planning-only context (device -1) cannot compute");
  if (!ctx || !key) return fail(SFHR_EINVAL, "null argument");
  if (G == 0) return SFHR_OK;
  if (ws_bytes < sfhr_pack_workspace_bytes(ctx, G)) return fail(SFHR_EINVAL, "pack workspace too small");
  std::lock_guard<std::mutex> lk(ctx->mu);
  DeviceGuard g(ctx->device);
  const Plan& P = ctx->plan;
  const RingConst& rc = P.rc;
  cudaStream_t st = (cudaStream_t)stream;
  uint64_t* cur = rows;
  uint64_t* oth = (uint64_t*)ws;
  int64_t per = P.pack_factor;  // rows per group at the current level
  auto stage = [&](const std::vector<uint32_t>& reps) -> int {
    int rc_ = run_stage(ctx, key, reps.data(), (int)reps.size(), 1, cur, oth, G * per, skip_zero, counter, st);
    if (rc_ == SFHR_OK) std::swap(cur, oth);
    return rc_;
  };
  const int t = rc.t, gamma = P.gamma, beta = P.beta;
  try {
    if (gamma == 0)
      for (auto& ch : P.chains)
        if (int e = stage(ch)) return e;
    long long tj = 1;
    for (int j = 1; j <= beta; ++j) {
      tj *= t;
      const int members = j == 1 ? t - 1 : t;
      const int rest = (int)(per / members);
      CK(launch_merge(rc, cur, oth, G, members, rest, (int)(rc.M / tj), st), "merge kernel");
      ++g_launches;
      std::swap(cur, oth);
      per = rest;
      if (j <= beta - 1 && j >= std::max(gamma, 1))
        if (int e = stage(P.reps_above[j - 1])) return e;
    }
    for (int j = beta; j < rc.alpha; ++j)
      if (j >= std::max(gamma, 1))
        if (int e = stage(P.reps_above[j - 1])) return e;
  } catch (const std::exception& ex) {
    return fail(SFHR_EINVAL, ex.what());
  }
  CK(cudaMemcpyAsync(packs, cur, (size_t)G * 2 * rc.N * 8, cudaMemcpyDeviceToDevice, st), "pack copy");
  return SFHR_OK;
}

int sfhr_derive_permutation(const uint8_t* seed, int seed_len, const uint8_t* sid, int sid_len, uint32_t round_no,
                            int64_t size, int64_t* out) {
  try {
    derive_permutation(seed, seed_len, sid, sid_len, round_no, size, out);
  } catch (const std::exception& ex) {
    return fail(SFHR_EINVAL, ex.what());
  }
  return SFHR_OK;
}

}  // extern "C"
