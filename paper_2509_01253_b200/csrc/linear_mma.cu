// Tensor-core grouped linear map over ciphertext rows (reference
// pkg/src/sfhr/model.py:384-429 semantics): out[o] = sum_k W[o,k] * in[col_k]
// mod 2^53, exact, on the 5th-generation tensor cores (tcgen05.mma kind::i8).
//
// The trick that makes a 53-bit modular MAC a plain int8 GEMM with no operand
// transposition: view every u64 lane of an input row as its 8 little-endian
// bytes.  With the byte-lanes of one 128-byte row slice on the MMA's M axis
// (A operand MN-major: a tap's 128 contiguous bytes are one K-row of A), the
// taps on K and the output rows of a tile group on N (B = s8 weights,
// K-major), the accumulator D[m = 8u + j][o] = sum_k W[o,k] * byte_j(in_k[u])
// is an exact s32 (|W| <= 127, K * 127 * 255 < 2^31), and
//     out[o][u] = sum_j D[8u + j][o] << 8j   (mod 2^64, then & (2^53 - 1))
// is the exact reference result.  Byte 7 of a lane is always 0 (values
// < 2^53), so 7/8 of the tensor work is useful.
//
// Per CTA: one tile group (<= 256 output rows sharing one column list; the
// residual skip rows are folded in as extra taps with identity weights) over a
// contiguous range of 128-byte M-tiles.  Warp-specialised pipeline: 4 producer
// warps gather the K taps of each stage with cp.async (16 B, zero-fill for
// padding taps and row tails) straight into the 128B-swizzled canonical layout
// and arrive on the stage's mbarrier when their copies land; one MMA warp
// issues the MMAs (K = 32 each) into a double-buffered TMEM accumulator and
// commits to per-stage / per-accumulator mbarriers; 4 epilogue warps
// (tcgen05.ld -> per-warp smem transpose -> byte recombination, bias*unit,
// sigma_r scatter) drain tile t-1 while tile t is being gathered and multiplied.
#include "sfhr_common.cuh"
#include "sfhr_kernels.h"
#include "tc_ptx.cuh"

namespace sfhr {

namespace {

constexpr int EPI_WARPS = 4;              // TMEM lanes 0-127
// cp.async gather threads per CTA: a template parameter, chosen per launch from the widest tile
// (A/B on B200, linear ms per inference: ResNet-20 (N <= 64, up to 4 CTAs/SM) 7.4 with 128 vs 8.0
// with 256; ResNet-18 (N up to 256, 1-2 CTAs/SM by TMEM) 14.0 with 128 vs 12.7 with 256)
template <int PRODUCERS>
constexpr int mma_threads() { return EPI_WARPS * 32 + PRODUCERS + 32; }
constexpr int KC = 64;                    // taps per pipeline stage (2 MMAs)
#ifndef SFHR_MMA_NSTAGE
#define SFHR_MMA_NSTAGE 4
#endif
constexpr int NSTAGE = SFHR_MMA_NSTAGE;  // pipeline depth (bytes in flight bound the gather rate)
constexpr int STAGE_BYTES = KC * 128;     // 8 KB of A per stage
#ifndef SFHR_B_RESIDENT_KB
#define SFHR_B_RESIDENT_KB 168  // A/B on B200 (linear ms per inference): ResNet-18 14.41 at 96 KB, 14.01 at 168; ResNet-34 343 -> 329
#endif
constexpr int B_RESIDENT_MAX = SFHR_B_RESIDENT_KB * 1024;  // larger weight operands are streamed with each stage
constexpr int MMA_SMEM_CAP = 226 * 1024;                  // per-CTA carve-up limit (227 KB opt-in)
constexpr int EP_COLS = 16;               // accumulator columns per epilogue chunk

}  // namespace

// byte offsets of the dynamic shared-memory carve-up (host and device agree)
struct MmaSmem {
  int ring, stage, bstage, b, ep, colp, odst, obias, bars, tslot, total;
  bool stream;  // B streamed per stage (stage = A 8 KB + B chunk Np x 64 B) instead of resident
  // B resident when it is at most B_RESIDENT_MAX and the whole carve-up fits MMA_SMEM_CAP
  __host__ __device__ static MmaSmem make(int Np, int Kp) {
    MmaSmem r = layout(Np, Kp, false);
    if (Np * Kp > B_RESIDENT_MAX || r.total > MMA_SMEM_CAP) r = layout(Np, Kp, true);
    return r;
  }
  __host__ __device__ static MmaSmem layout(int Np, int Kp, bool stream) {
    MmaSmem s;
    s.stream = stream;
    s.ring = 0;
    s.bstage = s.stream ? Np * KC : 0;
    s.stage = STAGE_BYTES + s.bstage;  // multiple of 1024 (Np % 16 == 0)
    s.b = s.ring + NSTAGE * s.stage;
    s.ep = s.b + (s.stream ? 0 : ((Np * Kp + 127) & ~127));
    s.colp = s.ep + EPI_WARPS * EP_COLS * 32 * 4;
    s.odst = s.colp + Kp * 8;
    s.obias = s.odst + Np * 8;
    s.bars = s.obias + Np * 8;
    s.tslot = s.bars + (2 * NSTAGE + 4) * 8;
    s.total = s.tslot + 16 + 1024;  // + alignment slack for the 1024-B swizzle atoms
    return s;
  }
};

// Warp roles: 0-3 epilogue (TMEM lanes 32w..32w+31), then PRODUCERS / 32 producer warps
// (cp.async gathers, one mbarrier arrival per thread per stage), then the MMA issuer.
template <int PRODUCERS>
__global__ void __launch_bounds__(mma_threads<PRODUCERS>()) linear_mma_kernel(const __grid_constant__ LinearMmaArgs a) {
  constexpr int MMA_THREADS = mma_threads<PRODUCERS>();
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int tg = (int)(blockIdx.x % a.T);
  const int chunk = (int)(blockIdx.x / a.T);
  const int32_t* td = a.tiles + 8 * (int64_t)tg;
  const int c0 = td[0], Kp = td[1], w0 = td[2], r0 = td[3], nr = td[4], Np = td[5];
  const int64_t lanes = a.lanes;
  const int64_t rowbytes = lanes * 8;
  const int n_mt = (int)((lanes + 15) / 16);
  const int mt0 = chunk * a.mt_per_cta;
  const int mt1 = min(n_mt, mt0 + a.mt_per_cta);
  if (mt0 >= mt1) return;

  const uint32_t raw = su32(smem_raw);
  unsigned char* sm = smem_raw + (((raw + 1023u) & ~1023u) - raw);
  const MmaSmem L = MmaSmem::make(Np, Kp);
  const uint32_t ring = su32(sm + L.ring), bsm = su32(sm + L.b);
  const int SB = L.stage;  // bytes per pipeline stage
  const unsigned char** colp = reinterpret_cast<const unsigned char**>(sm + L.colp);
  int64_t* odst = reinterpret_cast<int64_t*>(sm + L.odst);
  int64_t* obias = reinterpret_cast<int64_t*>(sm + L.obias);
  // barriers: full[NSTAGE] (128 producer arrivals), empty[NSTAGE] (MMA commit),
  // acc_full[2] (MMA commit), acc_empty[2] (4 epilogue warps)
  const uint32_t bars = su32(sm + L.bars);
  const uint32_t full0 = bars, empty0 = bars + 8 * NSTAGE, accf0 = bars + 16 * NSTAGE, acce0 = accf0 + 16;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + L.tslot);
  const uint32_t ncols = 2 * Np <= 32 ? 32 : 2 * Np <= 64 ? 64 : 2 * Np <= 128 ? 128 : 2 * Np <= 256 ? 256 : 512;

  // ---- setup: B operand (weights), tap row pointers, output row maps, barriers, TMEM ----
  const unsigned char* wsrc = a.tw + w0;
  if (!L.stream)
    for (int i = tid; i < Np * Kp / 16; i += MMA_THREADS) cp16(bsm + 16 * i, wsrc + 16 * i, 16);
  cp_commit();
  const unsigned char* in8 = reinterpret_cast<const unsigned char*>(a.in);
  const unsigned char* rin8 = reinterpret_cast<const unsigned char*>(a.round_in);
  int2* trow = reinterpret_cast<int2*>(sm + L.colp);  // TMA mode: (row, map) per tap, same slot
  for (int k = tid; k < Kp && a.use_tma; k += MMA_THREADS) {
    const int col = a.tcols[c0 + k];
    int2 e = make_int2(0x7fffffff, 0);  // zero tap: out-of-bounds row, zero-filled by the TMA
    if (col >= 0) e = make_int2((int)(a.in_map ? a.in_map[col] : (int64_t)col), 0);
    else if (col <= -2) e = make_int2((int)(a.round_map ? a.round_map[-(col + 2)] : (int64_t)(-(col + 2))), 1);
    trow[k] = e;
  }
  for (int k = tid; k < Kp && !a.use_tma; k += MMA_THREADS) {
    const int col = a.tcols[c0 + k];
    const unsigned char* p = nullptr;
    if (col >= 0) {
      p = in8 + (a.in_map ? a.in_map[col] : (int64_t)col) * rowbytes;
    } else if (col <= -2) {  // folded residual extra: a row of the ROUND input
      const int rc = -(col + 2);
      p = rin8 + (a.round_map ? a.round_map[rc] : (int64_t)rc) * rowbytes;
    }
    colp[k] = p;
  }
  for (int o = tid; o < Np; o += MMA_THREADS) {
    if (o < nr) {
      const int r = a.trows[r0 + o];
      obias[o] = a.bias ? a.bias[r] : 0;
      odst[o] = (a.out_map ? a.out_map[r] : (int64_t)r) * lanes;  // element offset of the output row
    } else {
      obias[o] = 0;
      odst[o] = -1;
    }
  }
  if (tid == 0) {
    for (int i = 0; i < NSTAGE; ++i) {
      mbar_init(full0 + 8 * i, a.use_tma ? 1 : PRODUCERS);
      mbar_init(empty0 + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(accf0 + 8 * i, 1);
      mbar_init(acce0 + 8 * i, EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(su32(tslot)),
                 "r"(ncols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
  }
  cp_wait<0>();
  fence_proxy_async();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int nkc = (Kp + KC - 1) / KC;

  if (a.use_tma && warp == EPI_WARPS) {
    // ---------------- TMA producer warp: tile::gather4 per 4 taps, spread over the lanes ----------------
    int stage = 0;
    uint32_t phase = 0;
    for (int mt = mt0; mt < mt1; ++mt) {
      for (int kc = 0; kc < nkc; ++kc) {
        mbar_wait(empty0 + 8 * stage, phase ^ 1);
        const int ntaps = min(KC, Kp - kc * KC);  // multiple of 32
        const int nkb = ntaps / 16;
        const uint32_t bbytes = L.stream ? (uint32_t)(nkb * (Np / 8) * 128) : 0u;
        const uint32_t full = full0 + 8 * stage;
        if (lane == 0) mbar_expect_tx(full, (uint32_t)ntaps * 128u + bbytes);
        __syncwarp();
        const uint32_t dst = ring + stage * SB;
        const int2* tr = trow + kc * KC;
        const int g = 4 * lane;  // <= 16 lanes active (KC = 64 taps)
        if (g < ntaps) {
          // a group of 4 taps never mixes the two inputs (host pads the pass-input taps to 4)
          const int2 e0 = tr[g], e1 = tr[g + 1], e2 = tr[g + 2], e3 = tr[g + 3];
          const int which = e0.y | e1.y | e2.y | e3.y;
          tma_gather4(dst + g * 128, which ? &a.tm_rin : &a.tm_in, mt * 16, e0.x, e1.x, e2.x, e3.x, full);
        }
        if (L.stream && lane == 31)
          bulk_copy(dst + STAGE_BYTES, wsrc + (size_t)kc * (KC / 16) * (Np / 8) * 128, bbytes, full);
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (!a.use_tma && warp >= EPI_WARPS && warp < EPI_WARPS + PRODUCERS / 32) {
    // ---------------- producers ----------------
    const int pt = tid - EPI_WARPS * 32;
    const int c = pt & 7, tb = pt >> 3;          // 16-byte chunk, first tap (taps tb + 16 i)
    const uint32_t dst_lane = (uint32_t)(tb * 128 + ((c ^ (tb & 7)) << 4));
    int stage = 0;
    uint32_t phase = 0;
    for (int mt = mt0; mt < mt1; ++mt) {
      const int64_t off = (int64_t)mt * 128 + c * 16;
      const uint32_t nbytes = off < rowbytes ? 16u : 0u;
      for (int kc = 0; kc < nkc; ++kc) {
        mbar_wait(empty0 + 8 * stage, phase ^ 1);
        const int ntaps = min(KC, Kp - kc * KC);
        const unsigned char* const* cp = colp + kc * KC;
        const uint32_t dst = ring + stage * SB + dst_lane;
        if (L.stream && pt == 0) {  // this stage's B chunk (contiguous K blocks 4kc.. of the packed
          // [K/16][N/8][8][16] weights): one bulk copy on the stage's barrier, tx counted before
          // this thread's own arrival so the phase cannot complete without it
          const int kb0 = kc * (KC / 16), nkb = min(KC, Kp - kc * KC) / 16;
          const uint32_t bbytes = (uint32_t)(nkb * (Np / 8) * 128);
          mbar_add_tx(full0 + 8 * stage, bbytes);
          bulk_copy(ring + stage * SB + STAGE_BYTES, wsrc + (size_t)kb0 * (Np / 8) * 128, bbytes, full0 + 8 * stage);
        }
        constexpr int TSTRIDE = PRODUCERS / 8;  // taps covered by one sweep of the producers
#pragma unroll
        for (int i = 0; i < KC / TSTRIDE; ++i) {
          const int tap = tb + TSTRIDE * i;
          if (tap < ntaps) {
            const unsigned char* rp = cp[tap];
            cp16(dst + i * TSTRIDE * 128, rp ? rp + off : in8, rp ? nbytes : 0u);
          }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(full0 + 8 * stage)
                     : "memory");
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == EPI_WARPS + PRODUCERS / 32) {
    // ---------------- MMA issuer ----------------
    // kind::i8, D = s32, A = u8 (MN-major), B = s8 (K-major), M = 128, N = Np
    const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | (1u << 15) | ((uint32_t)(Np >> 3) << 17) |
                           ((128u >> 4) << 24);
    const uint32_t b_kblock = (uint32_t)(Np / 8) * 128;  // bytes per 16-byte K block of B
    int stage = 0;
    uint32_t phase = 0;
    for (int mtl = 0; mtl < mt1 - mt0; ++mtl) {
      const int buf = mtl & 1;
      mbar_wait(acce0 + 8 * buf, (uint32_t)(((mtl >> 1) & 1) ^ 1));
      tc_fence_after();
      for (int kc = 0; kc < nkc; ++kc) {
        mbar_wait(full0 + 8 * stage, phase);
        tc_fence_after();
        if (lane == 0) {
          const int nmma = min(KC, Kp - kc * KC) / 32;
          for (int j = 0; j < nmma; ++j) {
            const uint64_t ad = sdesc(ring + stage * SB + j * 4096, 16, 1024, 2);
            const uint64_t bd = L.stream
                                    ? sdesc(ring + stage * SB + STAGE_BYTES + 2 * j * b_kblock, b_kblock, 128, 0)
                                    : sdesc(bsm + ((kc * KC + j * 32) >> 4) * b_kblock, b_kblock, 128, 0);
            mma_i8(tmem + (uint32_t)(buf * Np), ad, bd, idesc, (kc > 0 || j > 0) ? 1u : 0u);
          }
          mma_commit(empty0 + 8 * stage);
          if (kc == nkc - 1) mma_commit(accf0 + 8 * buf);
        }
        __syncwarp();
        if (++stage == NSTAGE) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp < EPI_WARPS) {
    // ---------------- epilogue ----------------
    int32_t* ep = reinterpret_cast<int32_t*>(sm + L.ep) + warp * (EP_COLS * 32);
    for (int mtl = 0; mtl < mt1 - mt0; ++mtl) {
      const int buf = mtl & 1;
      mbar_wait(accf0 + 8 * buf, (uint32_t)((mtl >> 1) & 1));
      tc_fence_after();
      const int64_t lane0 = (int64_t)(mt0 + mtl) * 16 + warp * 4;  // this warp's 4 u64 lanes
      const int64_t ln = lane0 + (lane & 3);                         // this thread's lane (both h)
      const bool lane_ok = ln < lanes;
      const uint64_t unitv = (a.bias && lane_ok && ln >= a.body_off) ? a.unit[ln - a.body_off] : 0ull;
      for (int cc = 0; cc < Np; cc += EP_COLS) {
        uint32_t r[16];
        tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(buf * Np + cc), r);
#pragma unroll
        for (int j = 0; j < 16; ++j) ep[j * 32 + lane] = (int32_t)r[j];
        __syncwarp();
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int idx = lane + 32 * h;
          const int cl = idx >> 2, u = idx & 3;
          const int o = cc + cl;
          if (o < nr && lane_ok) {
            const int4* p = reinterpret_cast<const int4*>(ep + cl * 32 + u * 8);
            const int4 x0 = p[0], x1 = p[1];
            uint64_t v = sx(x0.x) + (sx(x0.y) << 8) + (sx(x0.z) << 16) + (sx(x0.w) << 24) +
                         (sx(x1.x) << 32) + (sx(x1.y) << 40) + (sx(x1.z) << 48) + (sx(x1.w) << 56);
            v += (uint64_t)obias[o] * unitv;
            a.out[odst[o] + ln] = v & QMASK;
          }
        }
        __syncwarp();
      }
      tc_fence_before();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(acce0 + 8 * buf) : "memory");
    }
  }

  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols) : "memory");
}

size_t linear_mma_b_resident_bytes() { return (size_t)B_RESIDENT_MAX; }

size_t linear_mma_smem_bytes(int Np, int Kp) {
  // worst case over the tiles of a launch (N_pad <= Np, K_pad <= Kp): the streamed layout of
  // (Np, Kp) and any resident layout (B <= B_RESIDENT_MAX) with the same colp / row tables
  const MmaSmem s = MmaSmem::layout(Np, Kp, true);
  const size_t bres = (size_t)Np * Kp < (size_t)B_RESIDENT_MAX ? (size_t)Np * Kp : (size_t)B_RESIDENT_MAX;
  size_t resident = (size_t)NSTAGE * STAGE_BYTES + ((bres + 127) & ~(size_t)127) + (s.total - s.ep);
  if (resident > (size_t)MMA_SMEM_CAP) resident = MMA_SMEM_CAP;  // larger resident layouts stream
  return s.total > resident ? (size_t)s.total : resident;
}

cudaError_t launch_linear_mma(const LinearMmaArgs& a, int max_np, int max_kp, cudaStream_t st) {
  if (a.T == 0) return cudaSuccess;
  if (max_np < 16 || max_np > 256 || (max_np & 15) || (max_kp & 31) || a.lanes <= 0 || (a.lanes & 1))
    return cudaErrorInvalidValue;
  size_t smem = linear_mma_smem_bytes(max_np, max_kp);
  // keep resident CTAs x TMEM columns <= 512 (otherwise tcgen05.alloc would serialise)
  const int ncols = 2 * max_np <= 32 ? 32 : 2 * max_np <= 64 ? 64 : 2 * max_np <= 128 ? 128 : 2 * max_np <= 256 ? 256 : 512;
  const size_t floor_bytes = (size_t)(228 * 1024) / (size_t)(512 / ncols + 1) + 1024;
  if (smem < floor_bytes) smem = floor_bytes;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = max_np >= 128
                      ? cudaFuncSetAttribute(linear_mma_kernel<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)
                      : cudaFuncSetAttribute(linear_mma_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t n_mt = (a.lanes + 15) / 16;
  const int64_t chunks = (n_mt + a.mt_per_cta - 1) / a.mt_per_cta;
  const int64_t grid = chunks * a.T;
  if (grid > 0x7fffffffLL) return cudaErrorInvalidValue;
  if (max_np >= 128)
    linear_mma_kernel<256><<<(unsigned)grid, mma_threads<256>(), smem, st>>>(a);
  else
    linear_mma_kernel<128><<<(unsigned)grid, mma_threads<128>(), smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace sfhr
