// gemm.cu — K4/K5/K6: the W6A16 linear on tcgen05 (gemm.py:65-94 CGQ path).
//
//   Y[n, m] = S[n] * sum_k V[n, k] * X[m, k]
//
// exactly the reference's CGQ algorithm (raw code values V = value_table[c],
// row scale applied once after the fp32 accumulation, gemm.py:84-88), up to
// fp32 summation order.  V is rebuilt in registers by the hardware e3m2
// converter from the tile layout (common.cuh); the paper's bias-shift
// identity compose[c] * (S * 2^12) == V * S (dequant.py:33-69) means the same
// result as the folded-scale formulation, bit for bit per element.
//
// Work decomposition: stream-K.  The (tile, k-step) iteration space — tiles of
// 128 weight rows x BN batch columns, k-steps of kKStep x 128 k — is split
// into `gridDim.x` contiguous, equal ranges, one per persistent CTA.  A range
// is a sequence of segments (tile, k-range): at most a partial tail of its
// first tile ("B"), whole tiles, and a partial head of its last tile ("A").
// A tile cut between CTAs is finished by whichever contributor arrives last,
// summing the contributors' fp32 partials in a fixed order (deterministic).
// Each CTA runs its partial segments FIRST (A, then B, then the whole tiles):
// every contributor of a cut tile reaches it early, so the cross-CTA fixups
// overlap the whole-tile work instead of forming the kernel's tail.
//
// Per CTA (1 per SM, 768 threads), warp-specialised:
//   warp 16     W producer: per stage one 1-D bulk copy of the stage's
//               consecutive 12288-B weight tiles (evict-first); starts at
//               once, before the preceding kernel finishes (PDL).
//   warp 17     X producer: 2-D TMA boxes of X (64 k x BN rows, 128-B
//               swizzle; rows >= M, k >= K read 0) after griddepcontrol.wait.
//   warps 0-15  dequant (DQ): all 16 warps on every stage; warp w owns TMEM
//               lane group w % 4 (tcgen05.st restriction) and a 64-weight
//               (kKStep 2) or 32-weight (kKStep 1) piece of each row: LDS of
//               the tile layout -> FP6->FP16 rebuild (hardware e3m2
//               converter + spare-bit gather) -> tcgen05.st into the stage's
//               TMEM A slot (128 lanes = weight rows, 64 columns of half2
//               per 128-k tile).  The A ring is kASlots (>= 3) deep, so the
//               dequant of stage i overlaps the MMAs of stages i-1, i-2.
//   warps 18-19 MMA issuers (2 for N <= 64, alternate stages, one
//               accumulator each): tcgen05.mma.kind::f16, A in TMEM ("TS"),
//               B = X from SMEM, D (fp32, 128 x BN) in TMEM.
//   warps 20-23 epilogue: tcgen05.ld D (accumulators summed in fixed order)
//               -> x S -> Y, or the stream-K partial/fixup.
// Pipelines: W ring full/empty (W producer <-> DQ), X ring (X producer <->
// MMA commit), TMEM-A ring afull/aempty (DQ <-> MMA commit), TMEM-D ring
// dfull/dempty (MMA <-> epilogue).  Every ring slot is always consumed by
// the same party in stage order, so no parity wait can skip a phase (the X
// ring is even-sized: issuer i & 1 owns the stages of its parity).
#include <stdlib.h>

#include <mutex>

#include "../../paper_2312_08583_b200/csrc/common.cuh"

namespace lpqt {

constexpr int kNumDqWarps = 16;
constexpr int kNumEpiWarps = 4;
constexpr int kMaxMmaWarps = 2;
constexpr int kWarpTmaW = kNumDqWarps;       // weight-tile producer
constexpr int kWarpTmaX = kNumDqWarps + 1;   // activation producer
constexpr int kWarpMma0 = kNumDqWarps + 2;
constexpr int kWarpEpi0 = kWarpMma0 + kMaxMmaWarps;
constexpr int kThreads = (kWarpEpi0 + kNumEpiWarps) * 32;  // 768
constexpr int kAColsPerBuf = kTileK / 2;  // 64 columns of packed half2
constexpr int kTmemCols = 512;
constexpr int kSmemBudget = 200 * 1024;
constexpr int64_t kMaxCounters = 65536;   // stream-K tile counters (256 KiB)

struct GemmArgs {
  const uint8_t* tiles;
  const uint16_t* scales;
  void* y;
  float* partials;    // [gridDim.x][2][128][BN] fp32 (first / last segment of each CTA)
  int* counters;      // [tiles] k-steps contributed so far (self-resetting)
  long long* trace;   // LPQT_TRACE builds only: per-CTA %globaltimer stamps
  int64_t ldy;
  int64_t total;      // tiles * ksteps: the stream-K iteration space
  int M, N;
  int k_tiles, ksteps, n_tiles, m_tiles;
  int y_dtype, y_layout;
  ShiftMuls sm;       // 2^26, 2^28, 2^30: right shifts on the FMA pipe (common.cuh)
};

template <int BN>
struct Cfg {
  static constexpr int kKStep = BN <= 32 ? 2 : 1;           // 128-k tiles per pipeline stage
  static constexpr int kXTileBytes = BN * kTileK * 2;       // X for one tile: two SW128 blocks
  // Two smem rings per stage index: W (weight tiles, released by the DQ warps
  // as soon as their words are consumed) and X (activations, released by the
  // MMA commit), each fed by its own producer warp.
  static constexpr int kWStageBytes = kKStep * kTileBytes;
  static constexpr int kXStageBytes = kKStep * kXTileBytes;
  static constexpr int kXStages = BN <= 64 ? 6 : (BN <= 128 ? 4 : 2);
  static constexpr int kWStagesRaw = (kSmemBudget - kXStages * kXStageBytes) / kWStageBytes;
  static constexpr int kWStages = (kWStagesRaw > 12 ? 12 : kWStagesRaw) & ~1;  // even: see kASlots
  static constexpr int kStages = kWStages;                  // reported by the plan
  static constexpr int kDBufs = BN <= 128 ? 2 : 1;
  // MMA issue: at small N a tcgen05.mma executes in ~9 cycles (measured,
  // tools/mma_bench.cu) while its single-lane issue sequence (R2UR/VOTEU/
  // UTCHMMA) takes several times that, so two warps issue alternate stages,
  // each into its own accumulator; the epilogue sums the accumulators in a
  // fixed order.  Prefill MMAs (N >= 128) are long enough for one issuer.
  static constexpr int kMmaWarps = BN <= 64 ? 2 : 1;
  static constexpr int kNAcc = kMmaWarps;
  static constexpr int kDCols = BN * kNAcc;
  // TMEM: D buffers at the top, the rest is the A ring (64 columns per tile)
  static constexpr int kACols = kTmemCols - kDBufs * kDCols;
  // slots of kKStep tiles; even, so every slot is always filled by the same
  // dequant group (groups take alternate stages)
  static constexpr int kASlots = ((kACols / kAColsPerBuf) / kKStep) & ~1;
  // dequant work split: 16 warps = 4 TMEM lane groups x 4 pieces per row
  static constexpr int kDqWeights = kKStep * 32;            // weights per thread per stage
  static constexpr int kBarBytes = 8 * (2 * kWStages + 2 * kXStages + 2 * kASlots + 2 * kDBufs) + 16;
  static constexpr int kSmemBytes = kXStages * kXStageBytes + kWStages * kWStageBytes + kBarBytes + 1024;
  static_assert(kWStages >= 2 && kXStages >= 2, "pipeline too shallow");
  static_assert(kMmaWarps == 1 || kXStages % 2 == 0, "X ring slots must keep their issuer");
  static_assert(kSmemBytes <= 227 * 1024, "shared memory");
  static_assert(kASlots >= 2, "A ring too shallow");
  static_assert(kMmaWarps <= kMaxMmaWarps, "MMA issuers");
};

#ifdef LPQT_TRACE
// per-CTA %globaltimer stamps: trace[cta * 24 + ev]
#define CTA_STAMP(ev)                                                   \
  do {                                                                  \
    if (a.trace && blockIdx.x < 256) {                                  \
      uint64_t gt;                                                      \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));            \
      a.trace[blockIdx.x * 24 + (ev)] = (long long)gt;                  \
    }                                                                   \
  } while (0)
// per-stage clock64 events of CTA 0: trace[kTraceEv + ev * 64 + stage]
#define TRACE(ev, i)                                                          \
  do {                                                                        \
    if (a.trace && blockIdx.x == 0 && (i) < 64 && lane == 0)                  \
      a.trace[kTraceEv + (ev) * 64 + (i)] = clock64();                       \
  } while (0)
#define WTRACE(ev, i)                                                                     \
  do {                                                                                    \
    if (a.trace && blockIdx.x == 0 && (i) < 64 && lane == 0)                              \
      a.trace[kTraceWarp + (warp * 3 + (ev)) * 64 + (i)] = clock64();                    \
  } while (0)
#else
#define WTRACE(ev, i) \
  do {                \
  } while (0)
#define CTA_STAMP(ev) \
  do {                \
  } while (0)
#define TRACE(ev, i) \
  do {               \
  } while (0)
#endif
constexpr int kTraceEv = 256 * 24;
constexpr int kTraceWarp = kTraceEv + 12 * 64;   // [dq warp 16][3 events][64 stages] of CTA 0
constexpr int kTraceLen = kTraceWarp + 16 * 3 * 64;

// ---- stream-K geometry ----------------------------------------------------------
__device__ __forceinline__ int64_t sk_begin(const GemmArgs& a, int c) {
  return (int64_t)c * a.total / (int64_t)gridDim.x;
}
// CTA whose range holds global k-step position p
__device__ __forceinline__ int sk_cta_of(const GemmArgs& a, int64_t p) {
  return static_cast<int>(((p + 1) * (int64_t)gridDim.x - 1) / a.total);
}

// This CTA's local work order over its range [beg, end): piece A (the
// partial head of the last tile, nA k-steps from pA), piece B (the partial
// tail of the first tile, nB k-steps from beg), then the rest from c0 in
// global order (whole tiles, or the single partial segment of a range inside
// one tile).
struct Order {
  int64_t beg, pA, c0;
  int nA, nB, n;
};

__device__ __forceinline__ Order make_order(const GemmArgs& a, int64_t beg, int64_t end) {
  Order o{beg, 0, beg, 0, 0, static_cast<int>(end - beg)};
#ifdef LPQT_EXP_NATURAL_ORDER
  return o;
#endif
  if (end <= beg) return o;
  const int64_t ks = a.ksteps;
  const int64_t t_first = beg / ks, t_last = (end - 1) / ks;
  if (t_first == t_last) return o;
  if (end % ks != 0) {
    o.pA = t_last * ks;
    o.nA = static_cast<int>(end - o.pA);
  }
  if (beg % ks != 0) {
    o.nB = static_cast<int>((t_first + 1) * ks - beg);
    o.c0 = (t_first + 1) * ks;
  }
  return o;
}
__device__ __forceinline__ int64_t order_pos(const Order& o, int i) {
  if (i < o.nA) return o.pA + i;
  if (i < o.nA + o.nB) return o.beg + (i - o.nA);
  return o.c0 + (i - o.nA - o.nB);
}

// Walks the local order one stage at a time; divides only at piece starts.
struct OrderIter {
  int i, t, kk;  // local stage index, tile, k-step inside the tile
  __device__ __forceinline__ void seek(const GemmArgs& a, const Order& o, int i_) {
    i = i_;
    const int64_t p = order_pos(o, i);
    t = static_cast<int>(p / a.ksteps);
    kk = static_cast<int>(p - (int64_t)t * a.ksteps);
  }
  __device__ __forceinline__ void next(const GemmArgs& a, const Order& o) {
    ++i;
    if (i == o.nA || i == o.nA + o.nB) {
      if (i < o.n) seek(a, o, i);
    } else if (++kk == a.ksteps) {
      kk = 0;
      ++t;
    }
  }
};

struct Seg {
  int tile, ks0, ks1;  // k-steps [ks0, ks1) of `tile`
  int i0;              // local stage index of k-step ks0
  bool full;           // the whole tile (no other contributor)
  int pidx;            // partial slot: 0 = tile holding the range's start, 1 = the last tile
};

// next segment of the local order (segments never straddle a piece or tile)
__device__ __forceinline__ bool seg_next(const GemmArgs& a, const Order& o, int& i, Seg& sg) {
  if (i >= o.n) return false;
  const int64_t p = order_pos(o, i);
  const int t = static_cast<int>(p / a.ksteps);
  const int s0 = static_cast<int>(p - (int64_t)t * a.ksteps);
  const int piece_end = i < o.nA ? o.nA : (i < o.nA + o.nB ? o.nA + o.nB : o.n);
  const int len = min(piece_end - i, a.ksteps - s0);
  sg.tile = t;
  sg.ks0 = s0;
  sg.ks1 = s0 + len;
  sg.i0 = i;
  sg.full = (s0 == 0 && len == a.ksteps);
  sg.pidx = (o.beg >= (int64_t)t * a.ksteps) ? 0 : 1;
  i += len;
  return true;
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void store_y(const GemmArgs& a, int n, int m, float v) {
  if (n >= a.N || m >= a.M) return;
  const int64_t off = a.y_layout == LPQT_Y_NM ? (int64_t)n * a.ldy + m : (int64_t)m * a.ldy + n;
  if (a.y_dtype == LPQT_F32) {
    static_cast<float*>(a.y)[off] = v;
  } else if (a.y_dtype == LPQT_F16) {
    static_cast<__half*>(a.y)[off] = __float2half_rn(v);
  } else {
    static_cast<__nv_bfloat16*>(a.y)[off] = __float2bfloat16_rn(v);
  }
}

// Sum the first `nacc` accumulators over 16 columns [c0, c0+16) (fixed order).
template <int BN>
__device__ __forceinline__ void load_acc16(uint32_t t_d, int c0, int q0, int nacc, float (&acc)[16]) {
  uint32_t v[16];
  tmem_ld_x16(t_d + q0 * BN + c0, v);
  tmem_wait_ld();
#pragma unroll
  for (int j = 0; j < 16; ++j) acc[j] = __uint_as_float(v[j]);
#pragma unroll 1
  for (int q = q0 + 1; q < q0 + nacc; ++q) {
    tmem_ld_x16(t_d + q * BN + c0, v);
    tmem_wait_ld();
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] += __uint_as_float(v[j]);
  }
}

// Dequant piece of one thread: kKStep 2 -> 64 weights (3 x LDS.128 of the
// tile layout), kKStep 1 -> 32 weights (LDS.128 + LDS.64).  `src` points at
// the thread's (row, k-half) slot of the tile (common.cuh tile geometry).
template <int KSTEP>
struct DqPiece {
  uint32_t w[KSTEP * 6];
  __device__ __forceinline__ void load(uint32_t src, int grp) {
    if constexpr (KSTEP == 2) {
      const uint4 q0 = lds128_u32(src), q1 = lds128_u32(src + kTileN * 16), q2 = lds128_u32(src + 2 * kTileN * 16);
      w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w; w[4] = q1.x; w[5] = q1.y;
      w[6] = q1.z; w[7] = q1.w; w[8] = q2.x; w[9] = q2.y; w[10] = q2.z; w[11] = q2.w;
    } else {
      if (grp == 0) {
        const uint4 q0 = lds128_u32(src);
        const uint2 q1 = lds64_u32(src + kTileN * 16);
        w[0] = q0.x; w[1] = q0.y; w[2] = q0.z; w[3] = q0.w; w[4] = q1.x; w[5] = q1.y;
      } else {
        const uint2 q1 = lds64_u32(src + kTileN * 16 + 8);
        const uint4 q2 = lds128_u32(src + 2 * kTileN * 16);
        w[0] = q1.x; w[1] = q1.y; w[2] = q2.x; w[3] = q2.y; w[4] = q2.z; w[5] = q2.w;
      }
    }
  }
  // FP6 -> FP16 rebuild of the piece into KSTEP * 16 half2 registers
  __device__ __forceinline__ void rebuild(uint32_t (&r)[KSTEP * 16], const ShiftMuls& sm) const {
    fp6x32_cvt_f16x32_fma(w, r, sm);
    if constexpr (KSTEP == 2) fp6x32_cvt_f16x32_fma(w + 6, r + 16, sm);
  }
};

template <int KSTEP>
__device__ __forceinline__ void tmem_st_piece(uint32_t taddr, const uint32_t (&r)[KSTEP * 16]) {
  if constexpr (KSTEP == 2) {
    tmem_st_x32(taddr, r);
  } else {
    tmem_st_x16(taddr, r);
  }
}

// RAGGED: k_tiles % kKStep != 0, so the last k-step of every tile holds one
// tile (only possible for kKStep 2; LLaMA/StarCoder K are multiples of 256).
template <int BN, bool RAGGED>
__global__ void __launch_bounds__(kThreads, 1)
    w6a16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmArgs a) {
  using C = Cfg<BN>;
  // The dynamic shared window starts 1024-aligned (as CUTLASS also assumes
  // for SW128 operands; checked below), so every address is a constant offset
  // from the symbol and needs no runtime re-derivation.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  uint8_t* smem_x = smem;                                     // kXStages x kXStageBytes (1024-aligned)
  uint8_t* smem_w = smem + C::kXStages * C::kXStageBytes;     // kWStages x kWStageBytes
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem_w + C::kWStages * C::kWStageBytes);
  uint64_t* empty_w = full_w + C::kWStages;
  uint64_t* full_x = empty_w + C::kWStages;
  uint64_t* empty_x = full_x + C::kXStages;
  uint64_t* afull = empty_x + C::kXStages;
  uint64_t* aempty = afull + C::kASlots;
  uint64_t* dfull = aempty + C::kASlots;
  uint64_t* dempty = dfull + C::kDBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + C::kDBufs);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    CTA_STAMP(0);
    if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 descriptors need 1024-B alignment
  }
  const Order ord = make_order(a, sk_begin(a, blockIdx.x), sk_begin(a, blockIdx.x + 1));
  const int n_st = ord.n;

  // Setup.  The W producer initialises every mbarrier and starts streaming
  // weight tiles at once (weights never depend on the preceding kernel, see
  // LPQT_LAUNCH_PDL); the other warps meet on named barrier 2 (the producer
  // only arrives), so the TMEM allocation overlaps the first weight loads.
  if (warp == kWarpTmaW) {
    if (lane == 0) {
      for (int s = 0; s < C::kWStages; ++s) {
        mbar_init(&full_w[s], 1);
        mbar_init(&empty_w[s], kNumDqWarps / 2);  // the dequant group owning the slot
      }
      for (int s = 0; s < C::kXStages; ++s) {
        mbar_init(&full_x[s], 1);
        mbar_init(&empty_x[s], 1);  // MMA commit
      }
      for (int b = 0; b < C::kASlots; ++b) {
        mbar_init(&afull[b], kNumDqWarps / 2);
        mbar_init(&aempty[b], 1);   // MMA commit
      }
      for (int d = 0; d < C::kDBufs; ++d) {
        mbar_init(&dfull[d], C::kMmaWarps);
        mbar_init(&dempty[d], kNumEpiWarps);
      }
      fence_mbar_init();
      pdl_launch_dependents();  // the next kernel may queue for this SM as soon as it frees
    }
    __syncwarp();
    named_bar_arrive(2, kThreads);
  } else {
    if (warp == kWarpMma0) {
      tmem_alloc(tmem_slot, kTmemCols);
      tmem_relinquish();
    }
    if (warp == kWarpTmaX && lane == 0) prefetch_tmap(&tmap_x);
    tc_fence_before();
    named_bar_sync(2, kThreads);
    tc_fence_after();
  }
  // warp-uniform (not read by the W producer, which may pass before the alloc)
  const uint32_t tmem_base = warp == kWarpTmaW ? 0u : __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const uint32_t tmem_d0 = tmem_base + C::kACols;                       // D buffers above the A ring
  if (threadIdx.x == 0) {
    CTA_STAMP(1);
#ifdef LPQT_TRACE
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (a.trace && blockIdx.x < 256) a.trace[blockIdx.x * 24 + 7] = smid;
#endif
  }

  // Register split (launch: 768 x 80): each role's warpgroup re-sizes its
  // registers on entry — dequant 88, producer/MMA 48, epilogue 64
  // (4 x 128 x 88 + 128 x 48 + 128 x 64 <= 768 x 80).
  if (warp == kWarpTmaW || warp == kWarpTmaX) {
    // ------------------------------------------------------------ producers
    setmaxnreg_dec<48>();
    const bool is_w = (warp == kWarpTmaW);
    if (!is_w) pdl_wait();  // X is the preceding kernel's output
    if (!is_w && lane == 0) CTA_STAMP(13);
    const uint64_t pol = l2_evict_first_policy();
    OrderIter oi;
    if (n_st > 0) oi.seek(a, ord, 0);
    for (int it = 0; it < n_st; ++it, oi.next(a, ord)) {
      const int kt = oi.kk * C::kKStep;
      const int nt = min(C::kKStep, a.k_tiles - kt);
      const int n_tile = oi.t / a.m_tiles, m_tile = oi.t - n_tile * a.m_tiles;
      if (is_w) {
        const int s = it % C::kWStages;
        mbar_wait(&empty_w[s], ((it / C::kWStages) & 1) ^ 1);
        TRACE(0, it);
        const uint8_t* src = a.tiles + ((int64_t)n_tile * a.k_tiles + kt) * kTileBytes;
        const uint32_t bytes = static_cast<uint32_t>(nt * kTileBytes);
        const uint32_t e = elect_one();
        mbar_arrive_expect_tx_if(e, &full_w[s], bytes);
        bulk_g2s_if(e, smem_w + s * C::kWStageBytes, src, bytes, &full_w[s], pol);
      } else {
        const int s = it % C::kXStages;
        mbar_wait(&empty_x[s], ((it / C::kXStages) & 1) ^ 1);
        uint8_t* xs = smem_x + s * C::kXStageBytes;
        const uint32_t e = elect_one();
        mbar_arrive_expect_tx_if(e, &full_x[s], static_cast<uint32_t>(nt * C::kXTileBytes));
        for (int j = 0; j < nt; ++j) {
          tma_load_2d_if(e, xs + j * C::kXTileBytes, &tmap_x, &full_x[s], (kt + j) * kTileK, m_tile * BN);
          tma_load_2d_if(e, xs + j * C::kXTileBytes + BN * 128, &tmap_x, &full_x[s], (kt + j) * kTileK + 64,
                         m_tile * BN);
        }
      }
    }
    if (is_w && lane == 0) CTA_STAMP(2);
  } else if (warp < kNumDqWarps) {
    // ------------------------------------------------------------ dequant
    // Two groups of 8 warps take alternate stages (one group's barrier waits
    // overlap the other's ALU work); in a group warp w owns TMEM lane group
    // w % 4 (rows 32 (w % 4) ..) and, for kKStep 2, tile tl = (w / 4) % 2 of
    // the stage (its whole 128-k row: two 64-weight segments), for kKStep 1
    // k-half tl of the stage's tile.
    setmaxnreg_inc<88>();
    constexpr int KS = C::kKStep;
    constexpr int kSegs = KS == 2 ? 2 : 1;
    const int lg = warp & 3, grp = warp >> 3, tl = (warp >> 2) & 1;
    const int row = lg * 32 + lane;
    const uint32_t w_src = smem_u32(smem_w) + static_cast<uint32_t>(row * 16 + (KS == 2 ? tl * kTileBytes
                                                                                         : tl * 3 * kTileN * 16));
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) +
                            static_cast<uint32_t>(KS == 2 ? tl * kAColsPerBuf : tl * 32);
    const uint32_t fw0 = smem_u32(full_w), ew0 = smem_u32(empty_w);
    const uint32_t af0 = smem_u32(afull), ae0 = smem_u32(aempty);
    const ShiftMuls sm = a.sm;
    // the group's stages are i = grp, grp + 2, ...: cursors step by two slots
    struct Cur {
      uint32_t idx, ph;
      __device__ __forceinline__ void adv2(uint32_t n) {
        idx += 2;
        if (idx >= n) {
          idx -= n;
          ph ^= 1u;
        }
      }
    };
    Cur wc{static_cast<uint32_t>(grp), 0u};   // W ring
    Cur ac{static_cast<uint32_t>(grp), 0u};   // A ring
    OrderIter oi;
    if (RAGGED && grp < n_st) oi.seek(a, ord, grp);
    auto nt_next = [&]() -> int {  // tiles of the group's next stage, then advance two stages
      if constexpr (!RAGGED) {
        return KS;
      } else {
        const int nt = min(KS, a.k_tiles - oi.kk * KS);
        oi.next(a, ord);
        oi.next(a, ord);
        return nt;
      }
    };
    uint32_t q[kSegs][6 * 2];
    auto load_words = [&](int nt) {
      mbar_wait_u32(fw0 + 8 * wc.idx, wc.ph);
      if (KS == 1 || tl < nt) {
        const uint32_t src = w_src + wc.idx * C::kWStageBytes;
#pragma unroll
        for (int h = 0; h < kSegs; ++h) {
          const uint32_t sh = src + h * 3 * kTileN * 16;
          const uint4 v0 = lds128_u32(sh), v1 = lds128_u32(sh + kTileN * 16), v2 = lds128_u32(sh + 2 * kTileN * 16);
          q[h][0] = v0.x; q[h][1] = v0.y; q[h][2] = v0.z; q[h][3] = v0.w; q[h][4] = v1.x; q[h][5] = v1.y;
          q[h][6] = v1.z; q[h][7] = v1.w; q[h][8] = v2.x; q[h][9] = v2.y; q[h][10] = v2.z; q[h][11] = v2.w;
        }
      }
    };
    int nt_cur = 0;
    if (grp < n_st) {
      nt_cur = nt_next();
      load_words(nt_cur);
    }
    if (warp == 0 && lane == 0) CTA_STAMP(12);
    for (int i = grp; i < n_st; i += 2) {
      if (warp == 0) TRACE(1, i);
      mbar_wait_u32(ae0 + 8 * ac.idx, ac.ph ^ 1u);
      if (warp == 0) TRACE(2, i);
      WTRACE(0, i);
      tc_fence_after();
      if (KS == 1 || tl < nt_cur) {
        const uint32_t ta = t_lane + ac.idx * (KS * kAColsPerBuf);
#pragma unroll
        for (int h = 0; h < kSegs; ++h) {
          uint32_t r[32];
          fp6x32_cvt_f16x32_fma(q[h], r, sm);
          fp6x32_cvt_f16x32_fma(q[h] + 6, r + 16, sm);
          tmem_st_x32(ta + h * 32, r);
        }
      }
      if (warp == 0) TRACE(3, i);
      WTRACE(1, i);
      // the stage's words are consumed: hand the W slot back to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(ew0 + 8 * wc.idx);
      wc.adv2(C::kWStages);
      // prefetch the group's next stage while the TMEM stores drain
      if (i + 2 < n_st) {
        const int ntn = nt_next();
        load_words(ntn);
        nt_cur = ntn;
      }
      if (warp == 0) TRACE(4, i);
      tmem_wait_st();
      if (warp == 0) TRACE(5, i);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(af0 + 8 * ac.idx);
      ac.adv2(C::kASlots);
      WTRACE(2, i);
    }
    if (warp == 0 && lane == 0) CTA_STAMP(3);
  } else if (warp < kWarpEpi0) {
    // ------------------------------------------------------------ MMA issue
    setmaxnreg_dec<48>();
    // issuer mw takes the local stages of parity mw into accumulator mw; a
    // one-stage segment leaves one issuer without work: it then arrives on
    // dfull without a commit, and the epilogue sums only the accumulators
    // that were written.
    const int mw = warp - kWarpMma0;
    if (mw < C::kMmaWarps) {
      constexpr uint32_t idesc = idesc_f16_m128(BN);
      int i = 0;
      Seg sg;
      int lu = 0;
      while (seg_next(a, ord, i, sg)) {
        const int d = lu % C::kDBufs;
        const uint32_t dph = (lu / C::kDBufs) & 1;
        mbar_wait(&dempty[d], dph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_d0 + d * C::kDCols + mw * BN;
        const int ks_first = sg.ks0 + (C::kMmaWarps == 2 ? ((mw - sg.i0) & 1) : 0);
        for (int ks = ks_first; ks < sg.ks1; ks += C::kMmaWarps) {
          const int it = sg.i0 + (ks - sg.ks0);
          const int kt = ks * C::kKStep;
          const int nt = min(C::kKStep, a.k_tiles - kt);
          const int s = it % C::kXStages;
          const int slot = it % C::kASlots;
          mbar_wait(&full_x[s], (it / C::kXStages) & 1);
          if (it == mw && lane == 0) CTA_STAMP(14);
          TRACE(7, it);
          mbar_wait(&afull[slot], (it / C::kASlots) & 1);
          TRACE(8, it);
          tc_fence_after();
          const uint32_t e = elect_one();
          // descriptor of X block 0 of this stage; every other operand is a
          // compile-time offset from it (start address field = addr >> 4)
          const uint64_t bd0 = sdesc_kmajor_sw128(smem_u32(smem_x + s * C::kXStageBytes));
          const uint32_t bd_lo = static_cast<uint32_t>(bd0), bd_hi = static_cast<uint32_t>(bd0 >> 32);
          const uint32_t ta = tmem_base + slot * (C::kKStep * kAColsPerBuf);
          const bool first = (ks == ks_first);
#pragma unroll
          for (int t = 0; t < C::kKStep; ++t) {
            if (t < nt) {
#pragma unroll
              for (int j = 0; j < kTileK / 16; ++j) {
                const uint32_t off = (t * C::kXTileBytes + (j >> 2) * (BN * 128) + (j & 3) * 32) >> 4;
                const bool init = first && t == 0 && j == 0;
                mma_f16_ts_if(e, d_tmem, ta + t * kAColsPerBuf + j * 8, bd_lo + off, bd_hi, idesc,
                              init ? 0u : 1u);
              }
            }
          }
          tc_commit_if(e, &empty_x[s]);
          tc_commit_if(e, &aempty[slot]);
          TRACE(9, it);
        }
        if (ks_first < sg.ks1) {
          tc_commit_elect(&dfull[d]);
        } else if (lane == 0) {
          mbar_arrive(&dfull[d]);  // no MMA of this issuer in the segment
        }
        ++lu;
      }
      if (mw == 0 && lane == 0) CTA_STAMP(4);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    setmaxnreg_dec<64>();
    pdl_wait();  // Y / workspace writes: the preceding grid must be complete
    const int lg = warp & 3;
    const int rr = lg * 32 + lane;  // row inside the 128-row tile (= TMEM lane)
    const uint32_t t_lane = tmem_d0 + (static_cast<uint32_t>(lg * 32) << 16);
    int i = 0;
    Seg sg;
    int lu = 0;
    while (seg_next(a, ord, i, sg)) {
      const int d = lu % C::kDBufs;
      const uint32_t dph = (lu / C::kDBufs) & 1;
      const int n_tile = sg.tile / a.m_tiles, m_tile = sg.tile % a.m_tiles;
      const int n = n_tile * kTileN + rr;
      const int m0 = m_tile * BN;
      const float fs = n < a.N ? __half2float(__ushort_as_half(a.scales[n])) : 0.f;
      const uint32_t t_d = t_lane + d * C::kDCols;
      // accumulators written for this segment: both issuers when it spans >= 2
      // stages, else only the issuer of the single stage's parity
      const int nacc = min(C::kNAcc, sg.ks1 - sg.ks0);
      const int q0 = (nacc < C::kNAcc) ? (sg.i0 & 1) : 0;
      const bool last_seg = i >= n_st;
      mbar_wait(&dfull[d], dph);
      if (last_seg && warp == kWarpEpi0 && lane == 0) CTA_STAMP(8);
      tc_fence_after();
      if (sg.full) {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float acc[16];
          load_acc16<BN>(t_d, c0, q0, nacc, acc);
          if (c0 + 16 >= BN) {  // last chunk read: hand the D buffer back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&dempty[d]);
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) store_y(a, n, m0 + c0 + j, acc[j] * fs);
        }
      } else {
        float* part = a.partials + (((int64_t)blockIdx.x * 2 + sg.pidx) * kTileN + rr) * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float acc[16];
          load_acc16<BN>(t_d, c0, q0, nacc, acc);
          if (c0 + 16 >= BN) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&dempty[d]);
          }
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            __stcg(reinterpret_cast<float4*>(part + c0 + j), make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
          }
        }
        // publish: CTA barrier, then one gpu-scope acq_rel atomic (release our
        // partial, acquire the other contributors' partials if we are last)
        named_bar_sync(1, kNumEpiWarps * 32);
        if (last_seg && warp == kWarpEpi0 && lane == 0) CTA_STAMP(9);
        if (warp == kWarpEpi0 && lane == 0) {
          const int k_done = sg.ks1 - sg.ks0;
          const int prev = atom_add_acq_rel_gpu(&a.counters[sg.tile], k_done);
          *last_flag = (prev + k_done == a.ksteps) ? 1 : 0;
        }
        named_bar_sync(1, kNumEpiWarps * 32);
        if (last_seg && warp == kWarpEpi0 && lane == 0) CTA_STAMP(10);
        if (*last_flag) {
          const int64_t p_first = (int64_t)sg.tile * a.ksteps;
          const int c_first = sk_cta_of(a, p_first);
          const int c_last = sk_cta_of(a, p_first + a.ksteps - 1);
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float acc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = 0.f;
            // contributors in k order (fixed summation order: deterministic);
            // kFix of them are loaded at once so their L2 round trips overlap
            constexpr int kFix = 2;
#pragma unroll 1
            for (int cb = c_first; cb <= c_last; cb += kFix) {
              float4 v[kFix][4];
#pragma unroll
              for (int u = 0; u < kFix; ++u) {
                const int c = cb + u;
                if (c <= c_last) {
                  const int idx = (sk_begin(a, c) >= p_first) ? 0 : 1;
                  const float4* src =
                      reinterpret_cast<const float4*>(a.partials + (((int64_t)c * 2 + idx) * kTileN + rr) * BN + c0);
#pragma unroll
                  for (int j = 0; j < 4; ++j) v[u][j] = __ldcg(src + j);
                } else {
#pragma unroll
                  for (int j = 0; j < 4; ++j) v[u][j] = make_float4(0.f, 0.f, 0.f, 0.f);
                }
              }
#pragma unroll
              for (int u = 0; u < kFix; ++u) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  acc[4 * j + 0] += v[u][j].x;
                  acc[4 * j + 1] += v[u][j].y;
                  acc[4 * j + 2] += v[u][j].z;
                  acc[4 * j + 3] += v[u][j].w;
                }
              }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) store_y(a, n, m0 + c0 + j, acc[j] * fs);
          }
          if (warp == kWarpEpi0 && lane == 0) a.counters[sg.tile] = 0;
          if (last_seg && warp == kWarpEpi0 && lane == 0) CTA_STAMP(11);
        }
        named_bar_sync(1, kNumEpiWarps * 32);
      }
      ++lu;
    }
    if (warp == kWarpEpi0 && lane == 0) CTA_STAMP(5);
  }

  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) CTA_STAMP(6);
  if (warp == kWarpMma0) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// host side: plan, tensor map, launch
// ---------------------------------------------------------------------------
struct Plan {
  int bn, grid, n_tiles, m_tiles, k_tiles, ksteps, stages, smem, kstep;
  int64_t tiles, total, ws_bytes, counters_bytes;
  bool partials;
};

static int pick_bn(int64_t M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128) return 128;
  return 256;
}

template <int BN>
static void cfg_of(Plan& p) {
  p.stages = Cfg<BN>::kStages;
  p.smem = Cfg<BN>::kSmemBytes;
  p.kstep = Cfg<BN>::kKStep;
}

static int num_sms() {
  static int sms = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  });
  return sms;
}

// split_k == 0: one persistent CTA per SM over the whole stream-K space.
// split_k  > 0: about split_k CTAs per tile (testing / tuning hook).
static Plan make_plan(int64_t M, int64_t N, int64_t K, int split_k, int sms) {
  Plan p{};
  p.bn = pick_bn(M);
  switch (p.bn) {
    case 16: cfg_of<16>(p); break;
    case 32: cfg_of<32>(p); break;
    case 64: cfg_of<64>(p); break;
    case 128: cfg_of<128>(p); break;
    default: cfg_of<256>(p); break;
  }
  p.n_tiles = static_cast<int>((N + kTileN - 1) / kTileN);
  p.m_tiles = static_cast<int>((M + p.bn - 1) / p.bn);
  p.k_tiles = static_cast<int>((K + kTileK - 1) / kTileK);
  p.ksteps = (p.k_tiles + p.kstep - 1) / p.kstep;
  p.tiles = (int64_t)p.n_tiles * p.m_tiles;
  p.total = p.tiles * p.ksteps;
  int64_t g = split_k > 0 ? p.tiles * split_k : sms;
  if (g > p.total) g = p.total;
  if (p.tiles > kMaxCounters) g = p.tiles;  // one whole tile per CTA: no counters needed
  if (g < 1) g = 1;
  p.grid = static_cast<int>(g);
  // partial tiles exist unless every CTA range is a whole number of tiles
  p.partials = !(p.total % g == 0 && (p.total / g) % p.ksteps == 0);
  if (p.partials) {
    p.counters_bytes = kMaxCounters * 4;  // fixed region, zeroed once, self-resetting
    p.ws_bytes = p.counters_bytes + (int64_t)p.grid * 2 * kTileN * p.bn * 4;
  }
  return p;
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

#ifdef LPQT_TRACE
static long long* trace_buffer() {
  static long long* buf = nullptr;
  if (!buf) {
    cudaMalloc(&buf, kTraceLen * sizeof(long long));
    cudaMemset(buf, 0, kTraceLen * sizeof(long long));
  }
  return buf;
}
#endif

template <int BN, bool RAGGED>
static int launch_impl(const Plan& p, const GemmArgs& args, const uint16_t* Xt, int64_t ldx, int64_t M,
                       cudaStream_t stream, int flags) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return LPQT_E_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(ldx), static_cast<cuuint64_t>(M)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BN)};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(Xt), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return LPQT_E_INVALID_INPUT;
  auto kern = w6a16_tcgen05_kernel<BN, RAGGED>;
  constexpr int smem = Cfg<BN>::kSmemBytes;
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  });
  if (attr_err != cudaSuccess) return LPQT_E_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(p.grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (flags & LPQT_LAUNCH_PDL) ? 1 : 0;
  if (cudaLaunchKernelEx(&cfg, kern, map, args) != cudaSuccess) return LPQT_E_CUDA;
  note_launch();
  return check_launch();
}

template <int BN>
static int launch(const Plan& p, const GemmArgs& args, const uint16_t* Xt, int64_t ldx, int64_t M,
                  cudaStream_t stream, int flags) {
  if constexpr (Cfg<BN>::kKStep > 1) {
    if (p.k_tiles % Cfg<BN>::kKStep != 0) return launch_impl<BN, true>(p, args, Xt, ldx, M, stream, flags);
  }
  return launch_impl<BN, false>(p, args, Xt, ldx, M, stream, flags);
}

}  // namespace lpqt

using namespace lpqt;

extern "C" {

#ifdef LPQT_TRACE
int lpqt_trace_dump(long long* host) {
  cudaDeviceSynchronize();
  return cudaMemcpy(host, trace_buffer(), kTraceLen * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess
             ? 0
             : -1;
}
#endif

int lpqt_w6a16_plan_ex(int64_t M, int64_t N, int64_t K, int split_k, int flags, int* out, int n_out) {
  int v[4];
  const int st = lpqt_w6a16_plan(M, N, K, split_k, &v[0], &v[1], &v[2], &v[3]);
  for (int i = 0; i < n_out; ++i) out[i] = i < 4 ? v[i] : 0;
  return st;
}

int64_t lpqt_w6a16_workspace_bytes(int64_t M, int64_t N, int64_t K, int split_k) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  return make_plan(M, N, K, split_k, num_sms()).ws_bytes;
}

// Reports the plan: block_n = MMA N, splits = max CTAs sharing one tile
// (stream-K), grid = CTAs, stages = smem pipeline depth.
int lpqt_w6a16_plan(int64_t M, int64_t N, int64_t K, int split_k, int* block_n, int* splits, int* grid, int* stages) {
  if (M <= 0 || N <= 0 || K <= 0) return LPQT_E_SHAPE;
  const Plan p = make_plan(M, N, K, split_k, num_sms());
  if (block_n) *block_n = p.bn;
  if (splits) {
    const int64_t per = p.total / p.grid;  // k-steps per CTA (floor)
    *splits = p.partials ? static_cast<int>((p.ksteps + (per > 0 ? per : 1) - 1) / (per > 0 ? per : 1) + 1) : 1;
  }
  if (grid) *grid = p.grid;
  if (stages) *stages = p.stages;
  return LPQT_OK;
}

int lpqt_w6a16_linear(const uint8_t* tiles, const uint16_t* scales, const uint16_t* Xt, int64_t ldx, int64_t M,
                      int64_t N, int64_t K, void* Y, int y_dtype, int y_layout, int64_t ldy, int split_k,
                      void* workspace, int64_t workspace_bytes, void* stream) {
  return lpqt_w6a16_linear_ex(tiles, scales, Xt, ldx, M, N, K, Y, y_dtype, y_layout, ldy, split_k, workspace,
                              workspace_bytes, 0, stream);
}

int lpqt_w6a16_linear_ex(const uint8_t* tiles, const uint16_t* scales, const uint16_t* Xt, int64_t ldx, int64_t M,
                         int64_t N, int64_t K, void* Y, int y_dtype, int y_layout, int64_t ldy, int split_k,
                         void* workspace, int64_t workspace_bytes, int flags, void* stream) {
  flags &= LPQT_LAUNCH_PDL;
  if (M < 0 || N < 0 || K < 0) return LPQT_E_SHAPE;
  if (M == 0 || N == 0) return LPQT_OK;
  if (K == 0) return LPQT_E_SHAPE;  // callers zero-fill (gemm.py:74-75)
  if (ldx < K || ldx % 8 != 0 || (reinterpret_cast<uintptr_t>(Xt) & 15)) return LPQT_E_SHAPE;
  if (y_dtype != LPQT_F32 && y_dtype != LPQT_F16 && y_dtype != LPQT_BF16) return LPQT_E_UNSUPPORTED;
  if (y_layout != LPQT_Y_NM && y_layout != LPQT_Y_MN) return LPQT_E_UNSUPPORTED;
  if (y_layout == LPQT_Y_NM ? ldy < M : ldy < N) return LPQT_E_SHAPE;
  if (split_k < 0) return LPQT_E_INVALID_INPUT;
  if (N > (int64_t)1 << 30 || M > (int64_t)1 << 30 || K > (int64_t)1 << 30) return LPQT_E_SHAPE;
  const Plan p = make_plan(M, N, K, split_k, num_sms());
  if (p.ws_bytes > 0 && (workspace == nullptr || workspace_bytes < p.ws_bytes)) return LPQT_E_WORKSPACE;
  GemmArgs args{};
#ifdef LPQT_TRACE
  args.trace = trace_buffer();
#endif
  args.tiles = tiles;
  args.scales = scales;
  args.y = Y;
  args.counters = static_cast<int*>(workspace);
  args.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + p.counters_bytes);
  args.ldy = ldy;
  args.total = p.total;
  args.M = static_cast<int>(M);
  args.N = static_cast<int>(N);
  args.k_tiles = p.k_tiles;
  args.ksteps = p.ksteps;
  args.n_tiles = p.n_tiles;
  args.m_tiles = p.m_tiles;
  args.y_dtype = y_dtype;
  args.y_layout = y_layout;
  args.sm = ShiftMuls{1u << 26, 1u << 28, 1u << 30};
  cudaStream_t st = as_stream(stream);
  switch (p.bn) {
    case 16: return launch<16>(p, args, Xt, ldx, M, st, flags);
    case 32: return launch<32>(p, args, Xt, ldx, M, st, flags);
    case 64: return launch<64>(p, args, Xt, ldx, M, st, flags);
    case 128: return launch<128>(p, args, Xt, ldx, M, st, flags);
    default: return launch<256>(p, args, Xt, ldx, M, st, flags);
  }
}

}  // extern "C"
