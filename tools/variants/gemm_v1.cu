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
// into `gridDim.x` contiguous, equal ranges, one per persistent CTA.  A CTA's
// range is a sequence of segments (tile, k-range); whole tiles store Y
// directly, a tile cut between CTAs (at most the first and last segment of a
// range) is finished by whichever contributor arrives last, summing the
// contributors' fp32 partials in a fixed order (deterministic).
//
// Per CTA (1 per SM, 736 threads), warp-specialised:
//   warp 16     TMA producer: per stage one 1-D bulk copy of the stage's
//               consecutive 12288-B weight tiles (evict-first) + 2-D TMA boxes
//               of X (64 k x BN rows, 128-B swizzle; rows >= M, k >= K read 0).
//   warps 0-15  dequant (DQ), two groups on alternate stages: LDS.128 of the
//               thread's weight row -> FP6->FP16 rebuild (hardware e3m2
//               converter + spare-bit gather) -> tcgen05.st into a TMEM A slot
//               (128 lanes = weight rows, 64 columns of half2 per 128-k tile);
//               software-pipelined: the next stage's words load while the
//               stores drain.
//   warps 17-18 MMA issuers (2 for N <= 64, alternate stages, one
//               accumulator each): tcgen05.mma.kind::f16, A in TMEM ("TS"),
//               B = X from SMEM, D (fp32, 128 x BN) in TMEM.
//   warps 19-22 epilogue: tcgen05.ld D (accumulators summed in fixed order)
//               -> x S*2^12 -> Y, or the stream-K partial/fixup.
// Pipelines: smem ring full/empty (TMA <-> DQ+MMA), TMEM-A ring afull/aempty
// (DQ <-> MMA), TMEM-D ring dfull/dempty (MMA <-> epilogue).  The producer and
// MMA warps run warp-converged and issue through elect.sync-predicated PTX so
// the uniform-datapath instructions (UBLKCP/UTMALDG/UTCHMMA) need no per-issue
// lane waterfall.
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
  long long* trace;   // LPQT_TRACE builds only: [cta][16 events][64] clock64 stamps
  int64_t ldy;
  int64_t total;      // tiles * ksteps: the stream-K iteration space
  int M, N;
  int k_tiles, ksteps, n_tiles, m_tiles;
  int y_dtype, y_layout;
};

template <int BN>
struct Cfg {
  static constexpr int kKStep = BN <= 32 ? 2 : 1;           // 128-k tiles per pipeline stage
  static constexpr int kXTileBytes = BN * kTileK * 2;       // X for one tile: two SW128 blocks
  // Two smem rings per stage index: W (weight tiles, released by the DQ warps
  // as soon as their LDS are done) and X (activations, released by the MMA
  // commit), each fed by its own producer warp, so weight prefetch depth does
  // not wait on MMA completion.  Ring sizes are even: DQ groups (and the two
  // MMA issuers) own alternate stages, so every slot of every ring is always
  // consumed by the same party and each parity wait observes every phase of
  // its barrier (an odd ring would let a consumer skip a phase and pass on a
  // stale parity).
  static constexpr int kWStageBytes = kKStep * kTileBytes;
  static constexpr int kXStageBytes = kKStep * kXTileBytes;
  static constexpr int kXStages = BN <= 64 ? 6 : (BN <= 128 ? 4 : 2);
  static constexpr int kWStagesRaw = (kSmemBudget - kXStages * kXStageBytes) / kWStageBytes;
  static constexpr int kWStages = (kWStagesRaw > 8 ? 8 : kWStagesRaw) & ~1;
  static constexpr int kStages = kWStages;                  // reported by the plan
  static constexpr int kDBufs = BN <= 128 ? 2 : 1;
  // MMA issue: at small N a tcgen05.mma executes in ~9 cycles (measured,
  // tools/mma_bench.cu) while its single-lane issue sequence (R2UR/VOTEU/
  // UTCHMMA) takes several times that, so two warps issue alternate stages of
  // a segment, each into its own accumulator; the epilogue sums the
  // accumulators in a fixed order.  Prefill MMAs (N >= 128) are long enough
  // for one issuer.
  static constexpr int kMmaWarps = BN <= 64 ? 2 : 1;
  static constexpr int kNAcc = kMmaWarps;
  static constexpr int kDCols = BN * kNAcc;
  // TMEM: D buffers at the top, the rest is the A ring (64 columns per tile)
  static constexpr int kACols = kTmemCols - kDBufs * kDCols;
  static constexpr int kASlots = ((kACols / kAColsPerBuf) / kKStep) & ~1;   // slots of kKStep tiles
  static constexpr int kBarBytes = 8 * (2 * kWStages + 2 * kXStages + 2 * kASlots + 2 * kDBufs) + 16;
  static constexpr int kSmemBytes = kXStages * kXStageBytes + kWStages * kWStageBytes + kBarBytes + 1024;
  static_assert(kWStages >= 2 && kXStages >= 2, "pipeline too shallow");
  static_assert(kSmemBytes <= 227 * 1024, "shared memory");
  static_assert(kASlots >= 2, "A ring too shallow");
  static_assert(kMmaWarps <= kMaxMmaWarps, "MMA issuers");
};

#ifdef LPQT_TRACE
#define TRACE(ev, i)                                                                       \
  do {                                                                                     \
    if (a.trace && (i) < 64 && lane == 0 && (blockIdx.x == 0 || blockIdx.x == 77) &&      \
        ((ev) < 2 || (ev) > 7 || warp == 0) && ((ev) != 9 || warp == kWarpEpi0)) {          \
      a.trace[((blockIdx.x == 0 ? 0 : 1) * 16 + (ev)) * 64 + (i)] = clock64();              \
    }                                                                                      \
  } while (0)
#else
#define TRACE(ev, i) \
  do {               \
  } while (0)
#endif

// ---- stream-K geometry ----------------------------------------------------------
__device__ __forceinline__ int64_t sk_begin(const GemmArgs& a, int c) {
  return (int64_t)c * a.total / (int64_t)gridDim.x;
}
// CTA whose range holds global k-step position p
__device__ __forceinline__ int sk_cta_of(const GemmArgs& a, int64_t p) {
  return static_cast<int>(((p + 1) * (int64_t)gridDim.x - 1) / a.total);
}

struct Seg {
  int tile, ks0, ks1;  // k-steps [ks0, ks1) of `tile`
  bool full;           // the whole tile (no other contributor)
  int pidx;            // partial slot: 0 = first segment of this CTA's range, 1 = last
};

template <int KSTEP>
__device__ __forceinline__ bool seg_next(const GemmArgs& a, int64_t& pos, int64_t end, int64_t beg, Seg& sg) {
  if (pos >= end) return false;
  const int t = static_cast<int>(pos / a.ksteps);
  const int s0 = static_cast<int>(pos - (int64_t)t * a.ksteps);
  const int64_t rem = end - pos;
  const int s1 = rem < (int64_t)(a.ksteps - s0) ? s0 + static_cast<int>(rem) : a.ksteps;
  sg.tile = t;
  sg.ks0 = s0;
  sg.ks1 = s1;
  sg.full = (s0 == 0 && s1 == a.ksteps);
  sg.pidx = (beg >= (int64_t)t * a.ksteps) ? 0 : 1;
  pos += s1 - s0;
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

// One thread's 64-weight row segment: 3 x LDS.128 (tile layout, common.cuh)
__device__ __forceinline__ void lds_row64(const uint8_t* src, uint4 (&q)[3]) {
  q[0] = lds128(src);
  q[1] = lds128(src + kTileN * 16);
  q[2] = lds128(src + 2 * kTileN * 16);
}
// ... -> 32 half2 of composed binary16 (k ascending)
__device__ __forceinline__ void dq_row64(const uint4 (&q)[3], uint32_t (&r)[32]) {
  const uint32_t w0[6] = {q[0].x, q[0].y, q[0].z, q[0].w, q[1].x, q[1].y};
  const uint32_t w1[6] = {q[1].z, q[1].w, q[2].x, q[2].y, q[2].z, q[2].w};
  fp6x32_cvt_f16x32(w0, r);
  fp6x32_cvt_f16x32(w1, r + 16);
}

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    w6a16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmArgs a) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
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
  const int64_t beg = sk_begin(a, blockIdx.x);
  const int64_t end = sk_begin(a, blockIdx.x + 1);

  if (warp == kWarpTmaW) {
    if (lane == 0) {
      for (int s = 0; s < C::kWStages; ++s) {
        mbar_init(&full_w[s], 1);
        mbar_init(&empty_w[s], kNumDqWarps / 2);
      }
      for (int s = 0; s < C::kXStages; ++s) {
        mbar_init(&full_x[s], 1);
        mbar_init(&empty_x[s], 1);
      }
      for (int b = 0; b < C::kASlots; ++b) {
        mbar_init(&afull[b], kNumDqWarps / 2);
        mbar_init(&aempty[b], 1);
      }
      for (int d = 0; d < C::kDBufs; ++d) {
        mbar_init(&dfull[d], C::kMmaWarps);
        mbar_init(&dempty[d], kNumEpiWarps);
      }
      fence_mbar_init();
      pdl_launch_dependents();
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
  const uint32_t tmem_base = warp == kWarpTmaW ? 0u : __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const uint32_t tmem_d0 = tmem_base + C::kACols;                       // D buffers above the A ring

  if (warp == kWarpTmaW || warp == kWarpTmaX) {
    // ------------------------------------------------------------ producers
    // warp kWarpTmaW: one 1-D bulk copy of the stage's weight tiles (W ring);
    // warp kWarpTmaX: the stage's X boxes (X ring).
    const bool is_w = (warp == kWarpTmaW);
    if (!is_w) pdl_wait();
    const uint64_t pol = l2_evict_first_policy();
    int t = static_cast<int>(beg / a.ksteps);
    int ks = static_cast<int>(beg - (int64_t)t * a.ksteps);
    const int n_st = static_cast<int>(end - beg);
    for (int it = 0; it < n_st; ++it) {
      const int kt = ks * C::kKStep;
      const int nt = min(C::kKStep, a.k_tiles - kt);
      const int n_tile = t / a.m_tiles, m_tile = t - n_tile * a.m_tiles;
      if (is_w) {
        const int s = it % C::kWStages;
        TRACE(0, it);
        mbar_wait(&empty_w[s], ((it / C::kWStages) & 1) ^ 1);
        TRACE(1, it);
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
      if (++ks == a.ksteps) {
        ks = 0;
        ++t;
      }
    }
  } else if (warp < kNumDqWarps) {
    // ------------------------------------------------------------ dequant
    // 16 warps in two groups that take alternate stages (so one group's
    // barrier waits overlap the other's ALU work); inside a group 4 warps per
    // TMEM lane group, warp `tl` takes tile tl of the stage (kKStep == 2: the
    // whole 128-k row, 2 x (3 LDS.128 + 2 transforms + tcgen05.st)) or k-half
    // tl of the stage's single tile (kKStep == 1).
    constexpr int kSegs = C::kKStep == 2 ? 2 : 1;  // 64-weight row segments per warp per stage
    const int lg = warp & 3;
    const int row = lg * 32 + lane;
    const int grp = warp >> 3;
    const int tl = (warp >> 2) & 1;
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(lg * 32) << 16);
    const int n_st = static_cast<int>(end - beg);
    int ks_next = static_cast<int>((beg + grp) % a.ksteps);  // k-step of the group's next stage to load
    auto next_nt = [&]() {
      const int nt = min(C::kKStep, a.k_tiles - ks_next * C::kKStep);
      ks_next += 2;
      while (ks_next >= a.ksteps) ks_next -= a.ksteps;
      return nt;
    };
    auto seg_src = [&](int i, int h) {
      const uint8_t* ws = smem_w + (i % C::kWStages) * C::kWStageBytes + row * 16;
      return C::kKStep == 2 ? ws + tl * kTileBytes + h * 3 * kTileN * 16 : ws + tl * 3 * kTileN * 16;
    };
    // wait for stage i's weight tiles and load this thread's words; the slot
    // is released (empty_w) only after the words have been consumed by the
    // transform, so no refill can race the loads
    auto load_words = [&](int i, int nt, uint4 (&q)[kSegs][3]) {
      mbar_wait(&full_w[i % C::kWStages], (i / C::kWStages) & 1);
      if (C::kKStep == 1 || tl < nt) {
#pragma unroll
        for (int h = 0; h < kSegs; ++h) lds_row64(seg_src(i, h), q[h]);
      }
    };
    uint4 q[kSegs][3];
    int nt_cur = 0;
    if (grp < n_st) {
      nt_cur = next_nt();
      load_words(grp, nt_cur, q);
    }
    for (int i = grp; i < n_st; i += 2) {
      const int slot = i % C::kASlots;
      const uint32_t sph = (i / C::kASlots) & 1;
      TRACE(2, i);
      mbar_wait(&aempty[slot], sph ^ 1);
      TRACE(3, i);
      tc_fence_after();
      const uint32_t ta = t_lane + slot * C::kKStep * kAColsPerBuf;
      if (C::kKStep == 1 || tl < nt_cur) {
#pragma unroll
        for (int h = 0; h < kSegs; ++h) {
          uint32_t r[32];
          dq_row64(q[h], r);
          tmem_st_x32(C::kKStep == 2 ? ta + tl * kAColsPerBuf + h * 32 : ta + tl * 32, r);
        }
      }
      // the words of stage i are consumed (the stores read the transform's
      // registers): hand the W slot back to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_w[i % C::kWStages]);
      TRACE(4, i);
      // prefetch the group's next stage while the TMEM stores drain
      if (i + 2 < n_st) {
        const int nt_next = next_nt();
        load_words(i + 2, nt_next, q);
        TRACE(5, i);
        nt_cur = nt_next;
      }
      tmem_wait_st();
      TRACE(6, i);
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&afull[slot]);
      TRACE(7, i);
    }
  } else if (warp < kWarpEpi0) {
    // ------------------------------------------------------------ MMA issue
    // issuer mw takes the stages of global parity mw (the same stages as DQ
    // group mw) into accumulator mw; a one-stage segment leaves one issuer
    // without work: it then arrives on dfull without a commit, and the
    // epilogue sums only the accumulators that were written.
    const int mw = warp - kWarpMma0;
    if (mw < C::kMmaWarps) {
    constexpr uint32_t idesc = idesc_f16_m128(BN);
    int64_t pos = beg;
    Seg sg;
    int lu = 0;
    while (seg_next<C::kKStep>(a, pos, end, beg, sg)) {
      const int d = lu % C::kDBufs;
      const uint32_t dph = (lu / C::kDBufs) & 1;
      mbar_wait(&dempty[d], dph ^ 1);
      tc_fence_after();
      const uint32_t d_tmem = tmem_d0 + d * C::kDCols + mw * BN;
      const int64_t p0 = (int64_t)sg.tile * a.ksteps;
      const int it0 = static_cast<int>(p0 + sg.ks0 - beg);
      const int ks_first = sg.ks0 + (C::kMmaWarps == 2 ? ((mw - it0) & 1) : 0);
      for (int ks = ks_first; ks < sg.ks1; ks += C::kMmaWarps) {
        const int it = static_cast<int>(p0 + ks - beg);
        const int kt = ks * C::kKStep;
        const int nt = min(C::kKStep, a.k_tiles - kt);
        const int s = it % C::kXStages;
        const uint32_t ph = (it / C::kXStages) & 1;
        const int slot = it % C::kASlots;
        const uint32_t sph = (it / C::kASlots) & 1;
        mbar_wait(&full_x[s], ph);
        mbar_wait(&afull[slot], sph);
        TRACE(8, it);
        tc_fence_after();
        const uint32_t e = elect_one();
        // descriptor of X block 0 of this stage; every other operand is a
        // compile-time offset from it (start address field = addr >> 4)
        const uint64_t bd0 = sdesc_kmajor_sw128(smem_u32(smem_x + s * C::kXStageBytes));
        const uint32_t bd_lo = static_cast<uint32_t>(bd0), bd_hi = static_cast<uint32_t>(bd0 >> 32);
        const uint32_t ta = tmem_base + slot * C::kKStep * kAColsPerBuf;
        const bool first = (ks == ks_first);
#pragma unroll
        for (int t = 0; t < C::kKStep; ++t) {
          if (t < nt) {
#pragma unroll
            for (int j = 0; j < kTileK / 16; ++j) {
              const uint32_t off = (t * C::kXTileBytes + (j >> 2) * (BN * 128) + (j & 3) * 32) >> 4;
              const bool init = first && t == 0 && j == 0;
              mma_f16_ts_if(e, d_tmem, ta + t * kAColsPerBuf + j * 8, bd_lo + off, bd_hi, idesc, init ? 0u : 1u);
            }
          }
        }
        tc_commit_if(e, &empty_x[s]);
        tc_commit_if(e, &aempty[slot]);
        TRACE(10, it);
      }
      if (ks_first < sg.ks1) {
        tc_commit_elect(&dfull[d]);
      } else if (lane == 0) {
        mbar_arrive(&dfull[d]);  // no MMA of this issuer in the segment
      }
      ++lu;
    }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    pdl_wait();
    const int lg = warp & 3;
    const int rr = lg * 32 + lane;  // row inside the 128-row tile (= TMEM lane)
    const uint32_t t_lane = tmem_d0 + (static_cast<uint32_t>(lg * 32) << 16);
    int64_t pos = beg;
    Seg sg;
    int lu = 0;
    while (seg_next<C::kKStep>(a, pos, end, beg, sg)) {
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
      const int q0 = (nacc < C::kNAcc) ? static_cast<int>(((int64_t)sg.tile * a.ksteps + sg.ks0 - beg) & 1) : 0;
      mbar_wait(&dfull[d], dph);
      TRACE(9, lu);
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
        if (warp == kWarpEpi0 && lane == 0) {
          const int k_done = sg.ks1 - sg.ks0;
          const int prev = atom_add_acq_rel_gpu(&a.counters[sg.tile], k_done);
          *last_flag = (prev + k_done == a.ksteps) ? 1 : 0;
        }
        named_bar_sync(1, kNumEpiWarps * 32);
        if (*last_flag) {
          const int64_t p_first = (int64_t)sg.tile * a.ksteps;
          const int c_first = sk_cta_of(a, p_first);
          const int c_last = sk_cta_of(a, p_first + a.ksteps - 1);
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float acc[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) acc[j] = 0.f;
#pragma unroll 1
            for (int c = c_first; c <= c_last; ++c) {  // contributor order == k order
              const int idx = (sk_begin(a, c) >= p_first) ? 0 : 1;
              const float* src = a.partials + (((int64_t)c * 2 + idx) * kTileN + rr) * BN + c0;
              float4 v[4];
#pragma unroll
              for (int j = 0; j < 4; ++j) v[j] = __ldcg(reinterpret_cast<const float4*>(src) + j);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                acc[4 * j + 0] += v[j].x;
                acc[4 * j + 1] += v[j].y;
                acc[4 * j + 2] += v[j].z;
                acc[4 * j + 3] += v[j].w;
              }
            }
#pragma unroll
            for (int j = 0; j < 16; ++j) store_y(a, n, m0 + c0 + j, acc[j] * fs);
          }
          if (warp == kWarpEpi0 && lane == 0) a.counters[sg.tile] = 0;
        }
        named_bar_sync(1, kNumEpiWarps * 32);
      }
      ++lu;
    }
  }

  tc_fence_before();
  __syncthreads();
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
    cudaMalloc(&buf, 2 * 16 * 64 * sizeof(long long));
    cudaMemset(buf, 0, 2 * 16 * 64 * sizeof(long long));
  }
  return buf;
}
#endif

template <int BN>
static int launch(const Plan& p, const GemmArgs& args, const uint16_t* Xt, int64_t ldx, int64_t M,
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
  auto kern = w6a16_tcgen05_kernel<BN>;
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

}  // namespace lpqt

using namespace lpqt;

extern "C" {

#ifdef LPQT_TRACE
int lpqt_trace_dump(long long* host) {
  cudaDeviceSynchronize();
  return cudaMemcpy(host, trace_buffer(), 2 * 16 * 64 * sizeof(long long), cudaMemcpyDeviceToHost) == cudaSuccess
             ? 0
             : -1;
}
#endif

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
