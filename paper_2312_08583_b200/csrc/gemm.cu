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
// Output tiles are 128 weight rows x BN batch columns; the contraction runs
// over "stages" of kKStep 128-k weight tiles.  Two work schedules:
//
//  * stream-K (SK): the (tile, k-step) space is cut into gridDim.x equal
//    contiguous ranges, one per persistent CTA (1 per SM).  A tile cut
//    between CTAs is finished by whichever contributor arrives last (global
//    fp32 partials + an acq_rel tile counter), summing the partials in a fixed
//    order.  Perfect balance; the cross-CTA fixups cost global round trips.
//    Used when there are many tiles (prefill, big N).
//  * cluster split-K (CSK): CTAs form clusters of C (C <= 8); cluster j
//    takes tiles j, j + #clusters, ... ("rounds"), and rank r of the cluster
//    contracts k-tiles [r KT / C, (r + 1) KT / C) of each.  The C partial
//    accumulators of a tile meet in shared memory over DSMEM: every
//    non-reducer stages its fp32 partial in its own smem and signals the
//    round's reducer (rank round % C) through a cluster-scope mbarrier; the
//    reducer reads the partials with ld.shared::cluster, sums them in rank
//    order (deterministic), scales and stores Y, and hands the staging
//    buffers back.  No global atomics, no L2 round trips on the tail.  Used
//    for decode when the tile count is small.
//
// Per CTA (768 threads), warp-specialised:
//   warp 16     W producer: per stage one 1-D bulk copy of the stage's
//               consecutive 12288-B weight tiles (evict-first); starts at
//               once, before the preceding kernel finishes (PDL).
//   warp 17     X producer: 2-D TMA boxes of X (64 k x BN rows, 128-B
//               swizzle; rows >= M, k >= K read 0) after griddepcontrol.wait.
//   warps 0-15  dequant (DQ): two groups of 8 warps on alternate stages;
//               LDS of the tile layout -> FP6->FP16 rebuild (hardware e3m2
//               converter + spare-bit gather) -> tcgen05.st into the stage's
//               TMEM A slot (128 lanes = weight rows, 64 half2 columns per
//               128-k tile).
//   warps 18-19 MMA issuers (2 for N <= 64, alternate stages, one
//               accumulator each): tcgen05.mma.kind::f16, A in TMEM ("TS"),
//               B = X from SMEM, D (fp32, 128 x BN) in TMEM.
//   warps 20-23 epilogue: tcgen05.ld D (accumulators summed in fixed order)
//               -> x S -> Y, or the split-K reduction.
// Pipelines: W ring (W producer <-> DQ), X ring (X producer <-> MMA commit),
// TMEM-A ring (DQ <-> MMA commit), TMEM-D ring (MMA <-> epilogue).  Rings
// are even-sized where two parties alternate stages, so every slot is always
// consumed by the same party in stage order and no parity wait can skip a
// phase.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <type_traits>

#include "common.cuh"

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
#ifndef LPQT_SMEM_BUDGET_KB
#define LPQT_SMEM_BUDGET_KB 216
#endif
constexpr int kSmemBudget = LPQT_SMEM_BUDGET_KB * 1024;
constexpr int64_t kMaxCounters = 65536;   // stream-K tile counters (256 KiB)
constexpr int kMaxCluster = 8;

struct GemmArgs {
  const uint8_t* tiles;
  const uint16_t* scales;
  void* y;
  float* partials;    // SK: [gridDim.x][2][128][BN] fp32 (first / last segment of each CTA)
  int* counters;      // SK: [tiles] k-steps contributed so far (self-resetting)
  long long* trace;   // LPQT_TRACE builds only: per-CTA %globaltimer stamps
  int64_t ldy;
  int64_t total;      // SK: tiles * ksteps, the stream-K iteration space
  int M, N;
  int k_tiles, ksteps, n_tiles, m_tiles, tile_count;
  int y_dtype, y_layout;
  int csk_c;          // CSK: cluster size C (k-split factor)
  int n_fastest;      // tile index order: 0 = batch tile fastest, 1 = weight-row tile fastest
  int y_tma;          // Y tiles leave through the TMA tensor store (tmap_y valid)
  int dp;             // prefill (BN >= 64): whole tiles round-robin, CTA c takes c, c + grid, ...
  ShiftMuls sm;       // 2^26, 2^28, 2^30: right shifts on the FMA pipe (common.cuh)
};

// FGQ (block scales, quantizer.py FGQ x FP6; gemm.py:96-110) and INT4: the
// block parameters are re-laid out once per weight in stage order
// (lpqt_fgq_stage_params): for weight tile (row tile rt, k tile kt), the 128
// rows' f16 scale (INT4: f16 scale | f16 zero << 16) of the block holding kt,
// at ((rt * k_tiles) + kt) * kSBytes.  The W producer copies them into the
// stage next to the weight bytes (same mbarrier), so a dequant thread reads
// its row's parameter with one LDS; the rebuilt f16 weight carries the block
// scale (the binary16 dequant of dequant.py:72-79) and the epilogue applies none.
struct FgqArgs {
  const uint8_t* stage;    // stage-ordered block parameters (null: CGQ FP6, sub-tile FGQ)
  // sub-tile FGQ x FP6 (block B | 128, B % 16 == 0; decode widths): `sub` =
  // 128 / B partials per 128-k tile, each scaled in fp32 by its block's raw
  // f16 scale (row-major, `bpr` per row) read by the epilogue — gemm.py:96-110
  const uint16_t* scales;
  int sub, bpr;
};
// INT4 rebuild, 64 weights (8 words; nibble p of word w holds weight
// 8w + 2(p & 3) + (p >> 2)): OR the nibble pair into the mantissa of
// binary16 1024 (exact 1024 + level), subtract 1024 (exact), then
// level * S + Z with one binary16 rounding (HFMA2).
// (a & IMM) | c in one LOP3 (IMM the immediate, c a register: LOP3 takes one
// immediate, so two constant operands would cost a second LOP3)
template <uint32_t IMM>
__device__ __forceinline__ uint32_t and_or(uint32_t a, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a), "n"(IMM), "r"(c));
  return d;
}
// 64 INT4 levels (8 words, weight 8i + j in nibble (j >> 1) + 4 (j & 1) of
// word i) -> 32 f16x2 Z + S * level with one rounding (HFMA2 of the exact
// level).  Nibbles 0/4 and 2/6 OR into 1024.0 (0x6400: ulp 1), nibbles 1/5
// and 3/7 in place into 64.0 (0x5400: ulp 1/16), so a pair costs one LOP3,
// one HADD2 (exact: the level) and one HFMA2, plus a shift per two pairs.
__device__ __forceinline__ void int4x64_to_f16(const uint32_t (&w)[12], uint32_t (&r)[32], uint32_t s2, uint32_t z2) {
  uint32_t m1024 = 0x64006400u, m64 = 0x54005400u;
  asm volatile("" : "+r"(m1024), "+r"(m64));  // keep the magic numbers in registers
  const __half2 k1024 = __halves2half2(__ushort_as_half(0x6400u), __ushort_as_half(0x6400u));
  const __half2 k64 = __halves2half2(__ushort_as_half(0x5400u), __ushort_as_half(0x5400u));
  const __half2 S = *reinterpret_cast<const __half2*>(&s2), Z = *reinterpret_cast<const __half2*>(&z2);
#pragma unroll
  for (int i = 0; i < 8; ++i) {
#pragma unroll
    for (int hp = 0; hp < 2; ++hp) {
      const uint32_t y = w[i] >> (8 * hp);
      const uint32_t h0 = and_or<0x000F000Fu>(y, m1024), h1 = and_or<0x00F000F0u>(y, m64);
      const __half2 v0 = __hfma2(__hsub2(*reinterpret_cast<const __half2*>(&h0), k1024), S, Z);
      const __half2 v1 = __hfma2(__hsub2(*reinterpret_cast<const __half2*>(&h1), k64), S, Z);
      r[4 * i + 2 * hp] = *reinterpret_cast<const uint32_t*>(&v0);
      r[4 * i + 2 * hp + 1] = *reinterpret_cast<const uint32_t*>(&v1);
    }
  }
}
__device__ __forceinline__ void scale_f16x2(uint32_t (&r)[32], uint32_t s2) {
#pragma unroll
  for (int j = 0; j < 32; ++j) {
    __half2 v = __hmul2(*reinterpret_cast<const __half2*>(&r[j]), *reinterpret_cast<const __half2*>(&s2));
    r[j] = *reinterpret_cast<const uint32_t*>(&v);
  }
}

// Cross-launch L2 prefetch of the NEXT linear's weights (lpqt_w6a16_linear_pf):
// slice c = the first bytes the next launch's CTA c streams, derived from
// that launch's plan (total > 0: stream-K, else cluster split-K).  A separate
// kernel parameter: growing GemmArgs perturbs the epilogue's register budget.
struct L2Prefetch {
  const uint8_t* base;
  int64_t total, bytes;
  int count, ksteps, kstep, k_tiles, c, tiles;
  uint32_t chunk;
};

// WB: weight bits, 6 (FP6 e3m2 tiles, 12288 B) or 4 (INT4 tiles, 8192 B:
// [k-half 2][quad 2][row 128][16 B], nibbles pre-permuted for the
// magic-number rebuild; the INT4 comparator of SURVEY §8 f4)
#ifndef LPQT_DECODE_KSTEP
#define LPQT_DECODE_KSTEP 2  // decode (BN <= 32): 128-k tiles per stage
#endif
#ifndef LPQT_CSK32_XSTAGES
// BN 32 cluster split-K (M 17-32): 2 X stages of 16 KB leave room for 4 weight
// stages instead of 2 (next to the DSMEM staging buffers): 4096^2 / 5120^2 /
// 6144^2 12-17 % faster; stream-K at BN 32 keeps 4 X stages (2 measured 2-5 %
// slower there) (profiles/r02_abx_bn32_xstages.jsonl)
#define LPQT_CSK32_XSTAGES 2
#endif
#ifndef LPQT_BN32_ONE_YBUF
// BN 32 stream-K (M 17-32): one Y staging buffer + a 224-KB budget -> 6 weight
// stages instead of 4: 1-5.5 % faster on every 7B / 13B / 70B shape, none slower
// (profiles/r02_abx_bn32_one_ybuf.jsonl)
#define LPQT_BN32_ONE_YBUF 1
#endif
#ifndef LPQT_CSK32_ONE_YBUF
#define LPQT_CSK32_ONE_YBUF 1  // (cluster plans too: 4 -> 6 weight stages, 0-3 % faster, profiles/r02_abx_bn32_one_ybuf.jsonl)
#endif
#ifndef LPQT_BN64_XSTAGES
// BN 64 (M 33-64): 4 X stages of 16 KB; 2 X stages + 14 weight stages measured
// 3-8 % slower, 6 / 8 X stages neutral (profiles/r02_abx_bn64_stages.jsonl)
#define LPQT_BN64_XSTAGES 4
#endif
#ifndef LPQT_BN64_WCAP
#define LPQT_BN64_WCAP 12
#endif
#ifndef LPQT_TILE_RING
#define LPQT_TILE_RING 1
#endif
#ifndef LPQT_PREFILL_XSTAGES
#define LPQT_PREFILL_XSTAGES 3  // BN 192: X stages of 48 KB (W gets the rest of the budget)
#endif
#ifndef LPQT_PD_SLOTS16
#define LPQT_PD_SLOTS16 4  // FGQ per-block partial slots at BN 16 (TMEM: <= 6)
#endif
#ifndef LPQT_PD_WAIT
#define LPQT_PD_WAIT 0     // the epilogue's partial-ready wait mode (see mbar_try_wait)
#endif
// FGQ: 0 = CGQ, 1 = block scales per 128-k tile (stage-ordered), 2 = blocks of
// 16 / 32 / 64 (decode widths, FgqArgs::sub)
template <int BN, bool CSK, int WB = 6, int FGQ = 0>
struct Cfg {
  static constexpr int kTileB = WB == 6 ? kTileBytes : (WB == 5 ? kTileBytes5 : kTileN * kTileK / 2);
  // FGQ x FP6 at decode shapes (BN <= 32): "per-block partials" — every 128-k
  // weight tile's MMAs go into a fresh fp32 partial accumulator (kPSlots ring
  // in TMEM) and the epilogue adds S_block * partial in fp32, the reference's
  // FGQ order (gemm.py:96-110).  The dequant thread of each row hands its
  // block scale to the epilogue through TMEM too (kScaleCols columns, one
  // per k-tile ordinal mod 32), ordered by the same afull -> MMA -> pfull chain.
  static constexpr bool kPD = FGQ && WB == 6 && BN <= 32;
  static constexpr int kScaleCols = kPD ? 32 : 0;
  // FGQ / INT4: a stage carries its tiles' block parameters after the weights
  // (the dequant warps apply them to the rebuilt binary16 weight, or pass
  // them on to the epilogue under kPD)
  static constexpr int kSBytes = FGQ ? kTileN * (WB == 4 ? 4 : 2) : 0;
  static constexpr int kQuads = WB == 6 ? 3 : 2;             // 16-B quads per (row, k-half)
  static constexpr int kKStep = BN <= 32 ? LPQT_DECODE_KSTEP : 1;  // 128-k tiles per pipeline stage
  static constexpr int kXTileBytes = BN * kTileK * 2;       // X for one tile: two SW128 blocks
  static constexpr int kWStageBytes = kKStep * (kTileB + kSBytes);
  static constexpr int kXStageBytes = kKStep * kXTileBytes;
  // prefill (BN = 256): an X stage is 64 KB and covers ~1000 MMA cycles, so
  // three stages keep the L2 latency of X hidden (2 W stages of 12 KB suffice)
  // (native FP5 at BN 16: 4 X stages leave room for 8 W stages of 20 KB — bytes
  // in flight per SM are what bound the decode stream)
  static constexpr int kXStages =
      BN <= 16 ? (CSK || WB == 5 ? 4 : 6) : BN == 32 && CSK && WB != 5 ? LPQT_CSK32_XSTAGES : BN == 64 ? LPQT_BN64_XSTAGES : (BN <= 128 ? 4 : (BN == 192 ? LPQT_PREFILL_XSTAGES : 3));
  // CSK: two partial staging buffers of 128 x BN fp32 (rounds alternate)
  static constexpr int kStageBufBytes = CSK ? kTileN * BN * 4 : 0;
  // decode: output tiles staged in smem (two 128 x BN buffers, fp32-sized) and
  // written by the TMA tensor store, off the epilogue's critical path
  static constexpr int kYBufBytes = BN <= 32 ? kTileN * BN * 4 : 0;
  // BN 32 stream-K: ONE Y staging buffer and a 224-KB budget make room for
  // 6 weight stages instead of 4 (LPQT_BN32_ONE_YBUF)
  static constexpr bool kOneY = LPQT_BN32_ONE_YBUF && BN == 32 && (!CSK || LPQT_CSK32_ONE_YBUF) && WB == 6;
  static constexpr int kYBufs = kOneY ? 1 : 2;
  static constexpr int kBudget = BN >= 192 ? 221 * 1024 : (kOneY ? 224 * 1024 : kSmemBudget);
  static constexpr int kWStagesRaw =
      (kBudget - kXStages * kXStageBytes - 2 * kStageBufBytes - kYBufs * kYBufBytes) / kWStageBytes;
  static constexpr int kWCap = BN == 64 ? LPQT_BN64_WCAP : 12;
  static constexpr int kWStages = (kWStagesRaw > kWCap ? kWCap : kWStagesRaw) & ~1;  // even: see header
  static constexpr int kStages = kWStages;                  // reported by the plan
  // two accumulators in flight (the epilogue drains one while the next
  // tile's MMAs fill the other) up to BN 192: 2 x 192 + a 2-slot A ring = 512
  // TMEM columns; BN 256 has room for one
  static constexpr int kDBufs = BN <= 192 ? 2 : 1;
  // MMA issue: at small N a tcgen05.mma executes in ~9 cycles while its
  // single-lane issue sequence takes several times that, so two warps issue
  // alternate stages, each into its own accumulator; the epilogue sums them
  // in a fixed order.  Prefill MMAs (N >= 128) are long enough for one.
  static constexpr int kMmaWarps = BN <= 64 ? 2 : 1;
  // (per-block partials: the epilogue writes the segment's scaled sum into a
  // single D accumulator itself)
  static constexpr int kNAcc = kPD ? 1 : kMmaWarps;
  static constexpr int kDCols = BN * kNAcc;
  // per-k-tile partial accumulators (in-order drains bound every issuer's lead
  // to kPSlots ordinals, so a slot may alternate issuers without a skipped phase)
  static constexpr int kPSlots = kPD ? (BN <= 16 ? LPQT_PD_SLOTS16 : 4) : 0;
  static constexpr int kACols = kTmemCols - kDBufs * kDCols - kPSlots * BN - kScaleCols;
  // even with two MMA issuers (each slot then always belongs to the same
  // issuer, which waits on it in stage order: no parity wait can skip a
  // phase); one issuer may use every whole slot TMEM holds
  static constexpr int kASlots =
      kMmaWarps == 1 ? (kACols / kAColsPerBuf) / kKStep : ((kACols / kAColsPerBuf) / kKStep) & ~1;
  // decode (2 k-tiles per stage, 2 issuers): instead of one 2-tile slot per
  // issuer, each issuer / dequant-group pair owns a ring of 3 single-tile
  // slots used in order, so a group may write the next stage's first tile
  // while the MMAs still read the current stage's second one
  static constexpr bool kTileRing = LPQT_TILE_RING && kKStep == 2 && kMmaWarps == 2 && kACols / kAColsPerBuf >= 6;
  static constexpr int kABars = kTileRing ? 6 : kASlots;
  static constexpr int kBarCount = 2 * kWStages + 2 * kXStages + 2 * kABars + 2 * kDBufs + 5 + 2 * kPSlots;
  static constexpr int kSmemBytes = kXStages * kXStageBytes + kWStages * kWStageBytes + 2 * kStageBufBytes +
                                    kYBufs * kYBufBytes + 8 * kBarCount + 16;
  static_assert(kWStages >= 2 && kXStages >= 2, "pipeline too shallow");
  static_assert(kMmaWarps == 1 || kXStages % 2 == 0, "X ring slots must keep their issuer");
  static_assert(kSmemBytes <= 227 * 1024, "shared memory");
  static_assert(kASlots >= 2, "A ring too shallow");
  static_assert(!CSK || BN <= 32, "cluster split-K is the decode schedule");
};

#ifdef LPQT_TRACE
// per-CTA stamps: trace[cta * 32 + ev] = %clock64 (cheap, SM-local); the
// entry (ev 0) and exit (ev 6) stamps also record %globaltimer in slots 30
// and 31 so the host maps cycles to a chip-wide time axis.  (A %globaltimer
// read per stamp costs up to ~1 us and distorted dense stamp sequences.)
#define CTA_STAMP(ev)                                                   \
  do {                                                                  \
    if (a.trace && blockIdx.x < 256) {                                  \
      long long ck = clock64();                                         \
      a.trace[blockIdx.x * 32 + (ev)] = ck;                             \
      if ((ev) == 0 || (ev) == 6) {                                     \
        uint64_t gt;                                                    \
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));          \
        a.trace[blockIdx.x * 32 + ((ev) == 0 ? 30 : 31)] = (long long)gt; \
      }                                                                 \
    }                                                                   \
  } while (0)
#else
#define CTA_STAMP(ev) \
  do {                \
  } while (0)
#endif
constexpr int kTraceLen = 256 * 32;

// ---------------------------------------------------------------------------
// Work schedules.  Both present the CTA's work as a sequence of segments
// (one tile, a contiguous k-tile range [kt0, kt1), `len` stages whose local
// indices start at i0); every role walks the same sequence.
// ---------------------------------------------------------------------------
struct Seg {
  int tile, i0, len, kt0, kt1;
  bool full;  // SK: the whole tile, no other contributor
  int pidx;   // SK: partial slot (0 = tile holding the range start, 1 = last tile)
  int red;    // CSK: reducer rank of this round
};

// ---- stream-K ------------------------------------------------------------------
__device__ __forceinline__ int64_t sk_begin(const GemmArgs& a, int c) {
  return (int64_t)c * a.total / (int64_t)gridDim.x;
}
// CTA whose range holds global k-step position p
__device__ __forceinline__ int sk_cta_of(const GemmArgs& a, int64_t p) {
  return static_cast<int>(((p + 1) * (int64_t)gridDim.x - 1) / a.total);
}

// A CTA's stream-K range [beg, end) in natural order; segments never
// straddle a tile.
//
// Prefill (KS 1, a.dp): whole tiles round-robin instead — CTA c takes tiles c,
// c + grid, c + 2 grid, ... so the CTAs in flight always work on ~grid
// consecutive tiles: with the weight-row-fastest order they share one or two
// batch tiles of X, which stays in L2 (contiguous stream-K ranges would spread
// the CTAs over every batch tile at once and stream X from HBM repeatedly).
struct SkSched {
  int64_t beg;  // (the range end is beg + n: one 64-bit value kept live, not two)
  int n;
  template <int KS>
  __device__ __forceinline__ void init(const GemmArgs& a) {
    if (KS == 1 && a.dp) {
      const int c = static_cast<int>(blockIdx.x);
      n = c < a.tile_count ? ((a.tile_count - 1 - c) / static_cast<int>(gridDim.x) + 1) * a.ksteps : 0;
      beg = 0;
      return;
    }
    beg = sk_begin(a, blockIdx.x);
    n = static_cast<int>(sk_begin(a, blockIdx.x + 1) - beg);
  }
  template <int KS>
  __device__ __forceinline__ bool seg_at(const GemmArgs& a, int i, Seg& sg) const {
    if (i >= n) return false;
    if (KS == 1 && a.dp) {
      const int j = i / a.ksteps;
      sg.tile = static_cast<int>(blockIdx.x) + j * static_cast<int>(gridDim.x);
      sg.i0 = j * a.ksteps;
      sg.len = a.ksteps;
      sg.kt0 = 0;
      sg.kt1 = a.k_tiles;
      sg.full = true;
      sg.pidx = 0;
      sg.red = 0;
      return true;
    }
    const int64_t p = beg + i;
    const int t = static_cast<int>(p / a.ksteps);
    const int s0 = static_cast<int>(p - (int64_t)t * a.ksteps);
    const int rem = n - i;
    const int len = rem < a.ksteps - s0 ? rem : a.ksteps - s0;
    sg.tile = t;
    sg.i0 = i;
    sg.len = len;
    sg.kt0 = s0 * KS;
    sg.kt1 = min((s0 + len) * KS, a.k_tiles);
    sg.full = (s0 == 0 && len == a.ksteps);
    sg.pidx = (beg >= (int64_t)t * a.ksteps) ? 0 : 1;
    sg.red = 0;
    return true;
  }
};

// ---- cluster split-K ------------------------------------------------------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

struct CskSched {
  int C, rank, cid, ncl, kt0, kt1, len, rounds, n;
  __device__ __forceinline__ void init(const GemmArgs& a, int ks) {
    C = a.csk_c;
    rank = static_cast<int>(cluster_rank());
    cid = static_cast<int>(blockIdx.x) / C;
    ncl = static_cast<int>(gridDim.x) / C;
    kt0 = rank * a.k_tiles / C;
    kt1 = (rank + 1) * a.k_tiles / C;
    len = (kt1 - kt0 + ks - 1) / ks;
    rounds = cid < a.tile_count ? (a.tile_count - 1 - cid) / ncl + 1 : 0;
    n = rounds * len;
  }
  template <int KS>
  __device__ __forceinline__ bool seg_at(const GemmArgs& a, int i, Seg& sg) const {
    if (i >= n) return false;
    const int q = i / len;
    sg.tile = cid + q * ncl;
    sg.i0 = i;
    sg.len = len;
    sg.kt0 = kt0;
    sg.kt1 = kt1;
    sg.full = (C == 1);
    sg.pidx = 0;
    sg.red = q % C;
    return true;
  }
};

// Stage walker over the segment sequence (divisions only at segment starts)
template <class S, int KS>
struct StageIter {
  Seg sg;
  int s;  // stage inside the segment
  bool ok;
  __device__ __forceinline__ void start(const GemmArgs& a, const S& sc, int i) {
    ok = sc.template seg_at<KS>(a, 0, sg);
    s = 0;
    while (ok && i >= sg.i0 + sg.len) ok = sc.template seg_at<KS>(a, sg.i0 + sg.len, sg);
    if (ok) s = i - sg.i0;
  }
  __device__ __forceinline__ void next(const GemmArgs& a, const S& sc) {
    if (++s == sg.len) {
      ok = sc.template seg_at<KS>(a, sg.i0 + sg.len, sg);
      s = 0;
    }
  }
  __device__ __forceinline__ int kt() const { return sg.kt0 + s * KS; }
  __device__ __forceinline__ int nt() const { return min(KS, sg.kt1 - kt()); }
};

// Output tile t -> (weight-row tile, batch tile).  Decode and moderate
// prefill run the batch tiles of one weight tile back to back (the weight
// tile is shared in L2); when X itself outgrows L2 the weight-row tiles of
// one batch tile run back to back instead, so the X tile stays resident.
__device__ __forceinline__ void tile_nm(const GemmArgs& a, int t, int& n_tile, int& m_tile) {
  if (a.n_fastest) {
    m_tile = t / a.n_tiles;
    n_tile = t - m_tile * a.n_tiles;
  } else {
    n_tile = t / a.m_tiles;
    m_tile = t - n_tile * a.m_tiles;
  }
}

__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.add.acq_rel.gpu.s32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

__device__ __forceinline__ void red_add_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
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

// Fused all-gather, decode tiles: one Y tensor map per peer (the staged tile
// leaves by one TMA store per peer); other kernels carry an empty struct.
struct PeerMaps {
  CUtensorMap m[LPQT_MAX_PEERS];
};
struct NoPeerMaps {};
template <bool PEERS>
using PeerMapsOf = typename std::conditional<PEERS, PeerMaps, NoPeerMaps>::type;
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Fused all-gather (lpqt_w6a16_linear_gather): the same element into every
// peer's Y (each y[p] already offset to this rank's block).
__device__ __forceinline__ void store_y_peers(const GemmArgs& a, const lpqt_peer_out& po, int n, int m, float v) {
  if (n >= a.N || m >= a.M) return;
  const int64_t off = a.y_layout == LPQT_Y_NM ? (int64_t)n * a.ldy + m : (int64_t)m * a.ldy + n;
  // (static peer indices: the pointers stay in the constant bank, no local copy)
  if (a.y_dtype == LPQT_F32) {
#pragma unroll
    for (int p = 0; p < LPQT_MAX_PEERS; ++p)
      if (p < po.npeers) static_cast<float*>(po.y[p])[off] = v;
  } else if (a.y_dtype == LPQT_F16) {
    const __half h = __float2half_rn(v);
#pragma unroll
    for (int p = 0; p < LPQT_MAX_PEERS; ++p)
      if (p < po.npeers) static_cast<__half*>(po.y[p])[off] = h;
  } else {
    const __nv_bfloat16 h = __float2bfloat16_rn(v);
#pragma unroll
    for (int p = 0; p < LPQT_MAX_PEERS; ++p)
      if (p < po.npeers) static_cast<__nv_bfloat16*>(po.y[p])[off] = h;
  }
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Called by one thread per CTA after the CTA barrier that follows its
// epilogue's peer stores.  The count is a gpu-scope release (cumulative over
// the CTA's stores through bar.sync); the last CTA's acquire of it and its
// system-scope release stores of the flag carry every CTA's stores to the
// peers (the same release/acquire chain custom NVLink all-reduce barriers
// use; a per-thread fence.sc.sys cost ~10 us per launch).  Then wait for
// every peer's signal of this epoch (>= in wrapping order: a faster peer may
// already have signalled the next one) and re-arm the counter.
__device__ __forceinline__ void peer_complete(const lpqt_peer_out& po) {
  const int prev = atom_add_acq_rel_gpu(po.done, 1);
  if (prev != static_cast<int>(gridDim.x) - 1) return;
  const uint32_t* mine = nullptr;
#pragma unroll
  for (int p = 0; p < LPQT_MAX_PEERS; ++p) {
    if (p < po.npeers) st_release_sys_u32(po.flags[p] + po.rank, po.epoch);
    if (p == po.rank) mine = po.flags[p];
  }
  for (int q = 0; q < po.npeers; ++q) {
    // a peer that never launches is a caller bug: fail loudly (~10 s) rather than hang
    for (uint32_t spin = 0; static_cast<int32_t>(ld_acquire_sys_u32(mine + q) - po.epoch) < 0; ++spin) {
      if (spin > (1u << 26)) __trap();
      __nanosleep(128);
    }
  }
  *po.done = 0;
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

// Partials are read with ld.global.cg / bulk copies (L2), never through L1:
// with programmatic dependent launch an SM's L1 may still hold the same
// workspace lines from a previous launch of another shape.
// Stream-K partial tile of contributor slot `blk` (= cta * 2 + idx): 128 x BN
// fp32, stored chunk-major (float4 chunk j of row r at [j][r]): a warp's
// accesses to one chunk are 512 contiguous bytes, coalesced in global and
// conflict-free once gathered into shared memory.  BN 32 keeps rows
// contiguous (the chunk-major index math costs its epilogue registers).
template <int BN>
struct PartLayout {
  static constexpr bool kChunkMajor = BN != 32;
  static constexpr int kJStride = kChunkMajor ? kTileN : 1;  // float4 stride between chunks of a row
  __device__ __forceinline__ static int64_t f4(int64_t blk, int j, int rr) {  // float4 index
    return blk * (kTileN * BN / 4) + (kChunkMajor ? rr : rr * (BN / 4)) + (int64_t)j * kJStride;
  }
};

// ---- DSMEM / cluster primitives ----------------------------------------------------
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ float4 ld_dsmem_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
// arrive (release, cluster scope) on an mbarrier of another CTA of the cluster
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait_cluster(uint32_t addr, uint32_t parity) {
  for (uint32_t rounds = 0;; ++rounds) {  // (watchdog per round of polls, as mbar_wait_u32)
#pragma unroll
    for (int j = 0; j < LPQT_WATCHDOG_POLLS; ++j)
      if (mbar_try_wait_cluster(addr, parity)) return;
    if (rounds == (1u << 30) / LPQT_WATCHDOG_POLLS) __trap();
  }
}
__device__ __forceinline__ void cluster_arrive() {
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
}
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// ---- output tile staging (decode; the TMA store helpers are in common.cuh) ----
// 16 scaled values of output row n (tile row rr), columns m0 + c0 .. + 15,
// into the staged tile in the tensor map's box layout: Y_MN box [BN][128]
// (n fastest), Y_NM box [128][BN] (m fastest); element type = y_dtype.
template <int BN>
__device__ __forceinline__ void ystage_put(const GemmArgs& a, uint32_t buf, int rr, int c0, const float (&v)[16],
                                           float fs) {
  if (a.y_layout == LPQT_Y_NM) {
    const uint32_t row = buf + rr * BN * (a.y_dtype == LPQT_F32 ? 4 : 2) + c0 * (a.y_dtype == LPQT_F32 ? 4 : 2);
    if (a.y_dtype == LPQT_F32) {
#pragma unroll
      for (int j = 0; j < 16; j += 4)
        asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(row + j * 4), "f"(v[j] * fs),
                     "f"(v[j + 1] * fs), "f"(v[j + 2] * fs), "f"(v[j + 3] * fs)
                     : "memory");
    } else {
      uint32_t h[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (a.y_dtype == LPQT_F16) {
          const __half2 t = __floats2half2_rn(v[2 * j] * fs, v[2 * j + 1] * fs);
          h[j] = *reinterpret_cast<const uint32_t*>(&t);
        } else {
          const __nv_bfloat162 t = __floats2bfloat162_rn(v[2 * j] * fs, v[2 * j + 1] * fs);
          h[j] = *reinterpret_cast<const uint32_t*>(&t);
        }
      }
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row), "r"(h[0]), "r"(h[1]), "r"(h[2]),
                   "r"(h[3])
                   : "memory");
      asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(row + 16), "r"(h[4]), "r"(h[5]), "r"(h[6]),
                   "r"(h[7])
                   : "memory");
    }
  } else {
    if (a.y_dtype == LPQT_F32) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(buf + ((c0 + j) * kTileN + rr) * 4), "f"(v[j] * fs)
                     : "memory");
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const uint16_t hv = a.y_dtype == LPQT_F16 ? __half_as_ushort(__float2half_rn(v[j] * fs))
                                                  : __bfloat16_as_ushort(__float2bfloat16_rn(v[j] * fs));
        asm volatile("st.shared.u16 [%0], %1;" ::"r"(buf + ((c0 + j) * kTileN + rr) * 2), "h"(hv) : "memory");
      }
    }
  }
}

// RAGGED: some stage holds fewer than kKStep tiles (the last k-step of a
// tile when k_tiles % kKStep != 0, or an odd cluster split-K k-range); only
// then do the dequant warps walk the stage sequence to learn tile counts.
// RB: weight rebuild — 0 the hardware e3m2 converter (the product path);
// 1 / 2 the paper's software bias-shift / naive rebuilds x the per-row scale
// in binary16 (the ablation kernels, common.cuh fp6x32_soft_f16x32)
template <int BN, bool CSK, bool RAGGED, int FGQ = 0, int WB = 6, bool PEERS = false, int RB = 0>
__global__ void __launch_bounds__(kThreads, 1)
    w6a16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_y,
                         const GemmArgs a, const L2Prefetch pf, const FgqArgs fg,
                         const __grid_constant__ lpqt_peer_out po,
                         const __grid_constant__ PeerMapsOf<PEERS> pmaps) {
  static_assert(WB != 4 || FGQ, "INT4 weights carry per-block scales and zero points (FGQ path)");
  static_assert(WB != 5 || (!FGQ && !PEERS), "native FP5 tiles: CGQ");
  static_assert(RB == 0 || (!FGQ && WB == 6 && !PEERS), "ablation rebuilds: CGQ FP6 only");
  using C = Cfg<BN, CSK, WB, FGQ>;
  constexpr int KS = C::kKStep;
  // barrier waits: decode (BN <= 32) parks in the hardware try_wait (woken on
  // the phase flip); prefill re-polls every LPQT_WAIT_HINT_NS (measured,
  // profiles/r01_v9_abx_wait_modes.jsonl)
  constexpr int WM = BN <= 32 ? 0 : LPQT_WAIT_MODE;
  using Sched = typename std::conditional<CSK, CskSched, SkSched>::type;
  // The dynamic shared window starts 1024-aligned (as CUTLASS also assumes
  // for SW128 operands; checked below), so every address is a constant offset
  // from the symbol.
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem_x = smem_raw;                                           // kXStages x kXStageBytes
  uint8_t* smem_w = smem_x + C::kXStages * C::kXStageBytes;             // kWStages x kWStageBytes
  uint8_t* smem_stg = smem_w + C::kWStages * C::kWStageBytes;           // CSK: 2 x [BN/4][128] float4
  uint8_t* smem_y = smem_stg + 2 * C::kStageBufBytes;                  // 2 x Y tile (TMA store source)
  uint64_t* full_w = reinterpret_cast<uint64_t*>(smem_y + C::kYBufs * C::kYBufBytes);
  uint64_t* empty_w = full_w + C::kWStages;
  uint64_t* full_x = empty_w + C::kWStages;
  uint64_t* empty_x = full_x + C::kXStages;
  uint64_t* afull = empty_x + C::kXStages;
  uint64_t* aempty = afull + C::kABars;
  uint64_t* dfull = aempty + C::kABars;
  uint64_t* dempty = dfull + C::kDBufs;
  uint64_t* part_full = dempty + C::kDBufs;  // CSK [2]: this CTA's round partials from the senders
  uint64_t* stg_free = part_full + 2;        // CSK [2]: this CTA's staging buffer read by the reducer
  uint64_t* fix_bar = stg_free + 2;          // SK: partials gathered by bulk copy (last segment)
  uint64_t* pfull = fix_bar + 1;             // kPD [kPSlots]: a k-tile's partial is in TMEM
  uint64_t* pempty = pfull + C::kPSlots;     // kPD [kPSlots]: ... read by the epilogue
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pempty + C::kPSlots);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    CTA_STAMP(0);
    if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 descriptors need 1024-B alignment
  }
  Sched sc;
  if constexpr (CSK) {
    sc.init(a, KS);
  } else {
    sc.template init<KS>(a);
  }
  const int n_st = sc.n;

  // Setup.  The W producer initialises every mbarrier and starts streaming
  // weight tiles at once (weights never depend on the preceding kernel, see
  // LPQT_LAUNCH_PDL); the other warps meet on named barrier 2 (the producer
  // only arrives), so the TMEM allocation overlaps the first weight loads.
  // W producer: one stage of weight tiles (+ FGQ block parameters) into ring slot i % kWStages
  const uint64_t w_pol = (a.m_tiles > 1 && !a.n_fastest) ? l2_evict_last_policy() : l2_evict_first_policy();
  auto issue_w = [&](int i, const StageIter<Sched, KS>& it) {
    const int kt = it.kt(), nt = it.nt();
    int n_tile, m_tile;
    tile_nm(a, it.sg.tile, n_tile, m_tile);
    const int s = i % C::kWStages;
    const uint8_t* src = a.tiles + ((int64_t)n_tile * a.k_tiles + kt) * C::kTileB;
    const uint32_t bytes = static_cast<uint32_t>(nt * C::kTileB);
    const uint32_t e = elect_one();
    const uint32_t pbytes = FGQ == 2 ? 0u : static_cast<uint32_t>(nt * C::kSBytes);
    mbar_arrive_expect_tx_if(e, &full_w[s], bytes + pbytes);
    bulk_g2s_if(e, smem_w + s * C::kWStageBytes, src, bytes, &full_w[s], w_pol);
    if (FGQ && pbytes) {
      const uint8_t* sp = fg.stage + ((int64_t)n_tile * a.k_tiles + kt) * C::kSBytes;
      bulk_g2s_if(e, smem_w + s * C::kWStageBytes + KS * C::kTileB, sp, static_cast<uint32_t>(nt * C::kSBytes),
                  &full_w[s], w_pol);
    }
  };
  // (issuing the first W stages here, before the setup barrier, measured 5-12 %
  // slower: profiles/r02_abx_w_prologue.jsonl, _1_2.jsonl)
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
      for (int b = 0; b < C::kABars; ++b) {
        mbar_init(&afull[b], C::kTileRing ? kNumDqWarps / 4 : kNumDqWarps / 2);  // one tile's / stage's warps
        mbar_init(&aempty[b], 1);   // MMA commit
      }
      for (int d = 0; d < C::kDBufs; ++d) {
        mbar_init(&dfull[d], C::kMmaWarps);
        mbar_init(&dempty[d], kNumEpiWarps);
      }
      if constexpr (CSK) {
        for (int b = 0; b < 2; ++b) {
          mbar_init(&part_full[b], sc.C > 1 ? sc.C - 1 : 1);  // one remote arrive per sender
          mbar_init(&stg_free[b], 1);                         // one remote arrive by the reducer
        }
      } else {
        mbar_init(fix_bar, 1);
      }
      for (int b = 0; b < C::kPSlots; ++b) {
        mbar_init(&pfull[b], 1);
        mbar_init(&pempty[b], kNumEpiWarps);
      }
      fence_mbar_init();
      pdl_launch_dependents();  // the next kernel may queue for this SM as soon as it frees
      CTA_STAMP(19);
    }
    __syncwarp();
    named_bar_arrive(2, kThreads);
  } else {
    if (warp == kWarpMma0) {
      tmem_alloc(tmem_slot, kTmemCols);
      tmem_relinquish();
      if (lane == 0) CTA_STAMP(21);
    }
    if (warp == kWarpTmaX && lane == 0) prefetch_tmap(&tmap_x);
    tc_fence_before();
    named_bar_sync(2, kThreads);
    tc_fence_after();
  }
  // CSK: every thread arrives on the cluster barrier once its CTA's barriers
  // are initialised; the epilogue (the only remote user) waits before its
  // first DSMEM access, every other warp just before the exit sync
  if constexpr (CSK) cluster_arrive();
  // warp-uniform (not read by the W producer, which may pass before the alloc)
  const uint32_t tmem_base = warp == kWarpTmaW ? 0u : __shfl_sync(0xffffffffu, *tmem_slot, 0);
  const uint32_t tmem_d0 = tmem_base + C::kACols;                       // D buffers above the A ring
  if (threadIdx.x == 0) {
    CTA_STAMP(1);
#ifdef LPQT_TRACE
    uint32_t smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    if (a.trace && blockIdx.x < 256) a.trace[blockIdx.x * 32 + 7] = smid;
#endif
  }

  // Register split (launch: 768 x 80): each role's warpgroup re-sizes its
  // registers on entry — dequant 88, producer/MMA 48, epilogue 72
  // (4 x 128 x 88 + 128 x 48 + 128 x 72 <= 768 x 80).
  if (warp == kWarpTmaW || warp == kWarpTmaX) {
    // ------------------------------------------------------------ producers
    setmaxnreg_dec<48>();
    const bool is_w = (warp == kWarpTmaW);
    if (!is_w) pdl_wait();  // X is the preceding kernel's output
    if (!is_w && lane == 0) CTA_STAMP(13);
    // decode streams every weight byte once (evict-first); with several
    // batch tiles (prefill) the same weight tile is re-read per batch tile
    // (w_pol).
    StageIter<Sched, KS> it;
    it.start(a, sc, 0);
    for (int i = 0; i < n_st; ++i, it.next(a, sc)) {
      if (is_w) {
        const int s = i % C::kWStages;
        mbar_wait<WM>(&empty_w[s], ((i / C::kWStages) & 1) ^ 1);
        issue_w(i, it);
        if (i == 0 && lane == 0) CTA_STAMP(20);
      } else {
        const int kt = it.kt(), nt = it.nt();
        int n_tile, m_tile;
        tile_nm(a, it.sg.tile, n_tile, m_tile);
        const int s = i % C::kXStages;
        mbar_wait<WM>(&empty_x[s], ((i / C::kXStages) & 1) ^ 1);
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
    if (is_w && lane == 0) {
      CTA_STAMP(2);
      // every weight byte of this CTA is requested: hand HBM the next
      // linear's first bytes so it keeps streaming through this launch's
      // drain and the next one's start-up
      if (pf.base) {
        for (int c = blockIdx.x; c < pf.count; c += gridDim.x) {
          int64_t kt_lin;  // tile-linear k-tile index = byte offset / kTileBytes
          if (pf.total > 0) {
            const int64_t q = (int64_t)c * pf.total / pf.count;
            const int64_t t = q / pf.ksteps;
            kt_lin = t * pf.k_tiles + (q - t * pf.ksteps) * pf.kstep;
          } else {
            const int cid = c / pf.c, r = c - cid * pf.c;
            if (cid >= pf.tiles) continue;
            kt_lin = (int64_t)cid * pf.k_tiles + r * pf.k_tiles / pf.c;
          }
          const int64_t off = kt_lin * kTileBytes;
          const int64_t len = min((int64_t)pf.chunk, pf.bytes - off);
          if (len > 0) prefetch_l2_bulk(pf.base + off, static_cast<uint32_t>(len));
        }
      }
    }
  } else if (warp < kNumDqWarps) {
    // ------------------------------------------------------------ dequant
    // Two groups of 8 warps take alternate stages (one group's barrier waits
    // overlap the other's ALU work); in a group warp w owns TMEM lane group
    // w % 4 (rows 32 (w % 4) ..) and, for kKStep 2, tile tl = (w / 4) % 2 of
    // the stage (its whole 128-k row: two 64-weight segments), for kKStep 1
    // k-half tl of the stage's tile.
    setmaxnreg_inc<88>();
    if (warp == 0 && lane == 0) CTA_STAMP(22);
    constexpr int kSegs = KS == 2 ? 2 : 1;
    const int lg = warp & 3, grp = warp >> 3, tl = (warp >> 2) & 1;
    const int row = lg * 32 + lane;
    const uint32_t w_src = smem_u32(smem_w) + static_cast<uint32_t>(row * 16 + (KS == 2 ? tl * C::kTileB
                                                                                         : tl * C::kQuads * kTileN * 16));
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
    // A ring: slot grp of the 2-slot ring, or (tile ring) position tl of the
    // group's own 3-slot ring (barriers grp * 3 + idx)
    Cur ac{static_cast<uint32_t>(C::kTileRing ? tl : grp), 0u};
    const uint32_t a_bar0 = C::kTileRing ? static_cast<uint32_t>(grp * 3) : 0u;
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(lg * 32) << 16);
    StageIter<Sched, KS> it;
    if constexpr (RAGGED || RB) it.start(a, sc, grp);
    auto stage_nt = [&]() -> int {
      if constexpr (RAGGED) {
        return it.nt();
      } else {
        return KS;
      }
    };
    uint32_t q[kSegs][6 * 2];
    // WB 5: this row's mantissa words of the tile (after the 8 KB of nibble quads)
    const uint32_t m_src = smem_u32(smem_w) + static_cast<uint32_t>(kTile5Nib + row * 8 +
                                                                    (KS == 2 ? tl * C::kTileB : tl * kTileN * 8));
    uint32_t fs2 = 0;  // FGQ: this stage's block scale as f16x2
    uint32_t fz2 = 0;  // INT4: this stage's block zero point as f16x2
    // this thread's block parameter in the stage (after the KS weight tiles)
    const uint32_t s_src = smem_u32(smem_w) + KS * C::kTileB + (KS == 2 ? tl : 0) * C::kSBytes +
                           row * (WB == 4 ? 4 : 2);
    auto load_words = [&](int nt) {
      if constexpr (RB > 0) {
        // ablation: this row's scale (bias-shift: folded S * 2^12) for the stage's weight tile
        int n_tile, m_tile;
        tile_nm(a, it.sg.tile, n_tile, m_tile);
        const int n = n_tile * kTileN + row;
        const __half sc1 = n < a.N ? __ushort_as_half(__ldg(a.scales + n)) : __float2half(0.f);
        const __half f = RB == 1 ? __hmul(sc1, __float2half(4096.f)) : sc1;
        fs2 = __byte_perm(__half_as_ushort(f), 0u, 0x1010);
      }
      mbar_wait_u32<WM>(fw0 + 8 * wc.idx, wc.ph);
      if (KS == 1 || tl < nt) {
        if constexpr (FGQ) {
          if constexpr (WB == 4) {
            const uint32_t sz = lds_u32(s_src + wc.idx * C::kWStageBytes);
            fs2 = __byte_perm(sz, 0u, 0x1010);
            fz2 = __byte_perm(sz, 0u, 0x3232);
          } else {
            fs2 = __byte_perm(lds_u16(s_src + wc.idx * C::kWStageBytes), 0u, 0x1010);
          }
        }
        const uint32_t src = w_src + wc.idx * C::kWStageBytes;
#pragma unroll
        for (int h = 0; h < kSegs; ++h) {
          const uint32_t sh = src + h * C::kQuads * kTileN * 16;
          const uint4 v0 = lds128_u32(sh), v1 = lds128_u32(sh + kTileN * 16);
          q[h][0] = v0.x; q[h][1] = v0.y; q[h][2] = v0.z; q[h][3] = v0.w; q[h][4] = v1.x; q[h][5] = v1.y;
          q[h][6] = v1.z; q[h][7] = v1.w;
          if constexpr (WB == 6) {
            const uint4 v2 = lds128_u32(sh + 2 * kTileN * 16);
            q[h][8] = v2.x; q[h][9] = v2.y; q[h][10] = v2.z; q[h][11] = v2.w;
          } else if constexpr (WB == 5) {
            const uint2 mv = lds64_u32(m_src + wc.idx * C::kWStageBytes + (KS == 2 ? h * kTileN * 8 : 0));
            q[h][8] = mv.x; q[h][9] = mv.y;
          }
        }
      }
    };
    int nt_cur = 0;
    if (grp < n_st) {
      nt_cur = stage_nt();
      load_words(nt_cur);
    }
    if (warp == 0 && lane == 0) CTA_STAMP(12);
    for (int i = grp; i < n_st; i += 2) {
      // the first segment is rebuilt before the wait for the TMEM slot, so
      // half the ALU work overlaps the MMAs still reading the slot
      const bool act = KS == 1 || tl < nt_cur;
      uint32_t r[32];
      if (act) {
        if constexpr (WB == 4) {
          int4x64_to_f16(q[0], r, fs2, fz2);
        } else if constexpr (WB == 5) {
          fp5x32_cvt_f16x32(q[0], q[0][8], r, sm);
          fp5x32_cvt_f16x32(q[0] + 4, q[0][9], r + 16, sm);
        } else if constexpr (RB > 0) {
          fp6x32_soft_f16x32<RB>(q[0], r, fs2, sm);
          fp6x32_soft_f16x32<RB>(q[0] + 6, r + 16, fs2, sm);
        } else {
          fp6x32_cvt_f16x32_fma(q[0], r, sm);
          fp6x32_cvt_f16x32_fma(q[0] + 6, r + 16, sm);
          if constexpr (FGQ && !C::kPD) scale_f16x2(r, fs2);
        }
      }
      mbar_wait_u32<WM>(ae0 + 8 * (a_bar0 + ac.idx), ac.ph ^ 1u);
      tc_fence_after();
      if (act) {
        const uint32_t ta = C::kTileRing ? t_row + (a_bar0 + ac.idx) * kAColsPerBuf
                                         : t_lane + ac.idx * (KS * kAColsPerBuf);
        tmem_st_x32(ta, r);
#pragma unroll
        for (int h = 1; h < kSegs; ++h) {
          if constexpr (WB == 4) {
            int4x64_to_f16(q[h], r, fs2, fz2);
          } else if constexpr (WB == 5) {
            fp5x32_cvt_f16x32(q[h], q[h][8], r, sm);
            fp5x32_cvt_f16x32(q[h] + 4, q[h][9], r + 16, sm);
          } else if constexpr (RB > 0) {
            fp6x32_soft_f16x32<RB>(q[h], r, fs2, sm);
            fp6x32_soft_f16x32<RB>(q[h] + 6, r + 16, fs2, sm);
          } else {
            fp6x32_cvt_f16x32_fma(q[h], r, sm);
            fp6x32_cvt_f16x32_fma(q[h] + 6, r + 16, sm);
            if constexpr (FGQ && !C::kPD) scale_f16x2(r, fs2);
          }
          tmem_st_x32(ta + h * 32, r);
        }
        if constexpr (C::kPD && FGQ != 2) {
          // this row's block scale of tile ordinal q, for the epilogue (fp32)
          const uint32_t q = static_cast<uint32_t>(KS * i + (KS == 2 ? tl : 0));
          tmem_st_x1(t_row + C::kACols + C::kDBufs * C::kDCols + C::kPSlots * BN + (q & 31u),
                     __float_as_uint(__half2float(__ushort_as_half(static_cast<uint16_t>(fs2)))));
        }
      }
      // the stage's words are consumed: hand the W slot back to the producer
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(ew0 + 8 * wc.idx);
      wc.adv2(C::kWStages);
      // prefetch the group's next stage while the TMEM stores drain
      if (i + 2 < n_st) {
        if constexpr (RAGGED || RB) {
          it.next(a, sc);
          it.next(a, sc);
        }
        nt_cur = stage_nt();
        load_words(nt_cur);
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_u32(af0 + 8 * (a_bar0 + ac.idx));
      ac.adv2(C::kTileRing ? 3u : static_cast<uint32_t>(C::kASlots));
    }
    if (warp == 0 && lane == 0) CTA_STAMP(3);
    if (warp == 8 && lane == 0) CTA_STAMP(16);
  } else if (warp < kWarpEpi0) {
    // ------------------------------------------------------------ MMA issue
    // issuer mw takes the local stages of parity mw into accumulator mw; a
    // one-stage segment leaves one issuer without work: it then arrives on
    // dfull without a commit, and the epilogue sums only the accumulators
    // that were written.
    setmaxnreg_dec<48>();
    const int mw = warp - kWarpMma0;
    // sub-tile FGQ: ONE issuer takes every stage — a tile's 128 / B partials
    // would let two issuers on alternate stages run more than kPSlots
    // ordinals ahead of the in-order epilogue (parity waits could alias)
    constexpr int issuers = FGQ == 2 ? 1 : C::kMmaWarps;
    if (mw < issuers) {
      constexpr uint32_t idesc = idesc_f16_m128(BN);
      Seg sg;
      int lu = 0;
      for (int i0 = 0; sc.template seg_at<KS>(a, i0, sg); i0 += sg.len) {
        const int d = lu % C::kDBufs;
        const uint32_t dph = (lu / C::kDBufs) & 1;
        if constexpr (!C::kPD) {  // (per-block partials: the epilogue owns D)
          mbar_wait<WM>(&dempty[d], dph ^ 1);
          tc_fence_after();
        }
        const uint32_t d_tmem = tmem_d0 + d * C::kDCols + mw * BN;
        const int s_first = issuers == 2 ? ((mw - sg.i0) & 1) : 0;
        for (int s = s_first; s < sg.len; s += issuers) {
          const int it = sg.i0 + s;
          const int kt = sg.kt0 + s * KS;
          const int nt = min(KS, sg.kt1 - kt);
          const int xs = it % C::kXStages;
          const int slot = it % C::kASlots;
          mbar_wait<WM>(&full_x[xs], (it / C::kXStages) & 1);
          if (it == mw && lane == 0) CTA_STAMP(14);
          if constexpr (!C::kTileRing) mbar_wait<WM>(&afull[slot], (it / C::kASlots) & 1);
          tc_fence_after();
          const uint32_t e = elect_one();
          // descriptor of X block 0 of this stage; every other operand is a
          // compile-time offset from it (start address field = addr >> 4)
          const uint64_t bd0 = sdesc_kmajor_sw128(smem_u32(smem_x + xs * C::kXStageBytes));
          const uint32_t bd_lo = static_cast<uint32_t>(bd0), bd_hi = static_cast<uint32_t>(bd0 >> 32);
          const uint32_t ta = tmem_base + slot * (KS * kAColsPerBuf);
          const bool first = (s == s_first);
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            uint32_t ta_t = ta + t * kAColsPerBuf;
            int tb = 0;
            if constexpr (C::kTileRing) {
              // position 2 * (it >> 1) + t of this issuer's 3-slot ring
              const int pos = 2 * (it >> 1) + t, sl = pos % 3;
              tb = (it & 1) * 3 + sl;  // (the ring of the stage's dequant group)
              mbar_wait<WM>(&afull[tb], (pos / 3) & 1);
              tc_fence_after();
              ta_t = tmem_base + tb * kAColsPerBuf;
            }
            if (t < nt) {
              if constexpr (C::kPD && FGQ == 2) {
                // partial ordinal q = (KS * stage + t) * P + p: a fresh partial in
                // slot q % kPSlots for each of the tile's P = 128 / B blocks, each
                // of 8 / P MMAs of K = 16 (one issuer: ordinals in order)
                const int P = fg.sub, cpp = (kTileK / 16) / P;
                int ps = 0;
#pragma unroll
                for (int j = 0; j < kTileK / 16; ++j) {
                  const bool p0 = (j & (cpp - 1)) == 0;
                  if (p0) {
                    if (j) tc_commit_if(e, &pfull[ps]);
                    const int q = (KS * it + t) * P + j / cpp;
                    ps = q % C::kPSlots;
                    mbar_wait<WM>(&pempty[ps], ((q / C::kPSlots) & 1) ^ 1);
                    tc_fence_after();
                  }
                  const uint32_t p_tmem = tmem_d0 + C::kDBufs * C::kDCols + ps * BN;
                  const uint32_t off = (t * C::kXTileBytes + (j >> 2) * (BN * 128) + (j & 3) * 32) >> 4;
                  mma_f16_ts_if(e, p_tmem, ta_t + j * 8, bd_lo + off, bd_hi, idesc, p0 ? 0u : 1u);
                }
                tc_commit_if(e, &pfull[ps]);
              } else if constexpr (C::kPD) {
                // k-tile ordinal q = KS * stage + t: a fresh partial in slot q % kPSlots
                // (with two issuers on alternate stages each slot keeps its issuer)
                const int q = KS * it + t, ps = q % C::kPSlots;
                mbar_wait<WM>(&pempty[ps], ((q / C::kPSlots) & 1) ^ 1);
                tc_fence_after();
                const uint32_t p_tmem = tmem_d0 + C::kDBufs * C::kDCols + ps * BN;
#pragma unroll
                for (int j = 0; j < kTileK / 16; ++j) {
                  const uint32_t off = (t * C::kXTileBytes + (j >> 2) * (BN * 128) + (j & 3) * 32) >> 4;
                  mma_f16_ts_if(e, p_tmem, ta_t + j * 8, bd_lo + off, bd_hi, idesc, j == 0 ? 0u : 1u);
                }
                tc_commit_if(e, &pfull[ps]);
              } else {
#pragma unroll
                for (int j = 0; j < kTileK / 16; ++j) {
                  const uint32_t off = (t * C::kXTileBytes + (j >> 2) * (BN * 128) + (j & 3) * 32) >> 4;
                  const bool init = first && t == 0 && j == 0;
                  mma_f16_ts_if(e, d_tmem, ta_t + j * 8, bd_lo + off, bd_hi, idesc, init ? 0u : 1u);
                }
              }
            } else if constexpr (C::kPD) {
              // ragged stage (fewer than KS tiles): the missing tile's partial
              // ordinals still pass through their slots (an empty commit) so
              // every slot's phase count stays q / kPSlots — a skipped use
              // would let a later parity wait alias an old phase
              const int P = FGQ == 2 ? fg.sub : 1;
#pragma unroll 1
              for (int p = 0; p < P; ++p) {
                const int q = (KS * it + t) * P + p, ps = q % C::kPSlots;
                mbar_wait<WM>(&pempty[ps], ((q / C::kPSlots) & 1) ^ 1);
                tc_fence_after();
                tc_commit_if(e, &pfull[ps]);
              }
            }
            if constexpr (C::kTileRing) tc_commit_if(e, &aempty[tb]);  // this tile's slot is free once read
          }
          tc_commit_if(e, &empty_x[xs]);
          if constexpr (!C::kTileRing) tc_commit_if(e, &aempty[slot]);
        }
        if constexpr (!C::kPD) {
          if (s_first < sg.len) {
            tc_commit_elect(&dfull[d]);
          } else if (lane == 0) {
            mbar_arrive(&dfull[d]);  // no MMA of this issuer in the segment
          }
        }
        ++lu;
      }
      if (mw == 0 && lane == 0) CTA_STAMP(4);
      if (mw == 1 && lane == 0) CTA_STAMP(15);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    setmaxnreg_dec<72>();
    const int lg = warp & 3;
    const int rr = lg * 32 + lane;  // row inside the 128-row tile (= TMEM lane)
    // Row scales are weights (never written by the preceding kernel): the
    // first segment's is loaded before any wait, each next one a segment
    // ahead, so no global load sits on the epilogue's critical path (a cold
    // load behind the weight stream costs microseconds).
    // FGQ x FP6: the row's power-of-two factor 2^e_r (the block scales are
    // normalised by it, lpqt_fgq_stage_params); INT4 carries its scale in A
    auto scale_of = [&](const Seg& g) -> float {
      int nt, mt;
      tile_nm(a, g.tile, nt, mt);
      const int nn = nt * kTileN + rr;
      if constexpr (FGQ && WB == 6) {
        if constexpr (FGQ == 2) return nn < a.N ? 1.f : 0.f;  // (raw block scales, applied per partial)
        return nn < a.N ? __ldg(reinterpret_cast<const float*>(fg.stage + (int64_t)a.n_tiles * a.k_tiles * kTileN * 2) +
                                nn)
                        : 0.f;
      }
      if constexpr (FGQ || RB > 0) return nn < a.N ? 1.f : 0.f;  // (the scale is in A)
      return nn < a.N ? __half2float(__ushort_as_half(__ldg(a.scales + nn))) : 0.f;
    };
    Seg sg_next;
    bool have_next = sc.template seg_at<KS>(a, 0, sg_next);
    float fs_next = have_next ? scale_of(sg_next) : 0.f;
    if constexpr (CSK) cluster_wait();
    if (warp == kWarpEpi0 && lane == 0) CTA_STAMP(17);
    pdl_wait();  // Y / workspace writes: the preceding grid must be complete
    if (warp == kWarpEpi0 && lane == 0) CTA_STAMP(18);
    const uint32_t t_lane = tmem_d0 + (static_cast<uint32_t>(lg * 32) << 16);
    Seg sg;
    int lu = 0;
    // CSK, one bit per staging buffer: barrier phases to wait for, and
    // whether the buffer has been sent from before
    uint32_t pf_bits = 0u, sf_bits = 0u, sent_bits = 0u;
    // Y tiles: staged in smem and written by the TMA tensor store (decode),
    // else stored directly; ys_n counts staged tiles (buffer = ys_n & 1)
    const bool ytma = C::kYBufBytes > 0 && a.y_tma;
    int ys_n = 0;
    for (; have_next; ++lu) {
      sg = sg_next;
      const float fs = fs_next;
      have_next = sc.template seg_at<KS>(a, sg.i0 + sg.len, sg_next);
      if (have_next) fs_next = scale_of(sg_next);
      const int d = lu % C::kDBufs;
      const uint32_t dph = (lu / C::kDBufs) & 1;
      int n_tile, m_tile;
      tile_nm(a, sg.tile, n_tile, m_tile);
      const int n = n_tile * kTileN + rr;
      const int m0 = m_tile * BN;
      const uint32_t t_d = t_lane + d * C::kDCols;
      const uint32_t ybuf = smem_u32(smem_y) + (ys_n % C::kYBufs) * C::kYBufBytes;
      auto y_begin = [&]() {  // the staging buffer must have been read by its last TMA store
        if (ytma && ys_n >= C::kYBufs) {
          if (warp == kWarpEpi0 && lane == 0) bulk_wait_read<C::kYBufs - 1>();
          named_bar_sync(1, kNumEpiWarps * 32);
        }
      };
      auto y_chunk = [&](int c0, const float (&v)[16]) {
        if (ytma) {
          ystage_put<BN>(a, ybuf, rr, c0, v, fs);
        } else {
          if constexpr (PEERS && C::kYBufBytes == 0) {
            // (decode tiles always leave by the per-peer TMA stores: the host
            // refuses peer buffers the tensor maps cannot describe)
#pragma unroll 1
            for (int j = 0; j < 16; ++j) store_y_peers(a, po, n, m0 + c0 + j, v[j] * fs);
          } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) store_y(a, n, m0 + c0 + j, v[j] * fs);
          }
        }
      };
      auto y_end = [&]() {
        if (!ytma) return;
        fence_proxy_async_smem();
        named_bar_sync(1, kNumEpiWarps * 32);
        if (warp == kWarpEpi0 && lane == 0) {
          const int yc0 = a.y_layout == LPQT_Y_NM ? m_tile * BN : n_tile * kTileN;
          const int yc1 = a.y_layout == LPQT_Y_NM ? n_tile * kTileN : m_tile * BN;
          if constexpr (PEERS) {
#pragma unroll
            for (int p = 0; p < LPQT_MAX_PEERS; ++p)
              if (p < po.npeers) tma_store_2d(&pmaps.m[p], ybuf, yc0, yc1);
          } else {
            tma_store_2d(&tmap_y, ybuf, yc0, yc1);
          }
          bulk_commit();
        }
        ++ys_n;
      };
      // accumulators written for this segment: both issuers when it spans >= 2
      // stages, else only the issuer of the single stage's parity
      const int nacc = min(C::kNAcc, sg.len);
      const int q0 = (nacc < C::kNAcc) ? (sg.i0 & 1) : 0;
      const bool last_seg = sg.i0 + sg.len >= n_st;
      int64_t p_first = 0;
      int c_first = 0, c_last = 0, idx_first = 0;
      // contributors of a split tile (64-bit divisions: only when needed)
      auto contributors = [&]() {
        p_first = (int64_t)sg.tile * a.ksteps;
        c_first = sk_cta_of(a, p_first);
        c_last = sk_cta_of(a, p_first + a.ksteps - 1);
        // partial slot of contributor c: only c_first can have started its
        // range before the tile (slot 1 = its last segment); every later
        // contributor starts inside the tile (slot 0 = its first segment)
        idx_first = (sk_begin(a, c_first) >= p_first) ? 0 : 1;
      };
      // Tail reduction (BN >= 128, last segment: every X and W stage has been
      // consumed).  Contributors c_first..c_last in k order; batches of
      // kSlots partials land by bulk copy in [smem_x, smem_x + X ring + W
      // ring); the running sum lives in the other TMEM accumulator (idle: no
      // MMA follows).  Summation order = every other path's: 0 + p0 + p1 + ...
      auto tail_reduce = [&](bool own_in_tmem) {
        constexpr int kFree = C::kXStages * C::kXStageBytes + C::kWStages * C::kWStageBytes;
        constexpr int kSlots = kFree / (kTileN * BN * 4) > 0 ? kFree / (kTileN * BN * 4) : 1;
        constexpr uint32_t kPB = kTileN * BN * 4;
        const int me = static_cast<int>(blockIdx.x);
        const uint32_t t_acc = t_lane + (1 - d) * C::kDCols;   // the idle accumulator (this warp's lanes)
        const uint32_t sbase = smem_u32(smem_x) + static_cast<uint32_t>(rr * 16);
        uint32_t fph = 0;
        y_begin();
        for (int b0 = c_first; b0 <= c_last; b0 += kSlots) {
          const int b1 = min(c_last, b0 + kSlots - 1);
          if (warp == kWarpEpi0 && lane == 0) {
            uint32_t bytes = 0;
            for (int c = b0; c <= b1; ++c) bytes += (own_in_tmem && c == me) ? 0u : kPB;
            fence_proxy_async_global();  // generic-proxy partials (acquired) -> bulk-copy reads
            mbar_arrive_expect_tx(fix_bar, bytes);
            for (int c = b0; c <= b1; ++c) {
              if (own_in_tmem && c == me) continue;
              const int idx = c == c_first ? idx_first : 0;
              bulk_g2s_plain(smem_x + (c - b0) * kPB, a.partials + ((int64_t)c * 2 + idx) * (kTileN * BN), kPB,
                             fix_bar);
            }
          }
          mbar_wait<WM>(fix_bar, fph);
          fph ^= 1u;
          const bool last_batch = b1 == c_last;
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float acc[16];
            if (b0 == c_first) {
#pragma unroll
              for (int j = 0; j < 16; ++j) acc[j] = 0.f;
            } else {
              uint32_t v[16];
              tmem_ld_x16(t_acc + c0, v);
              tmem_wait_ld();
#pragma unroll
              for (int j = 0; j < 16; ++j) acc[j] = __uint_as_float(v[j]);
            }
#pragma unroll 1
            for (int c = b0; c <= b1; ++c) {
              if (own_in_tmem && c == me) {
                float own[16];
                load_acc16<BN>(t_d, c0, q0, nacc, own);
#pragma unroll
                for (int j = 0; j < 16; ++j) acc[j] += own[j];
              } else {
                const uint32_t src = sbase + (c - b0) * kPB + (c0 / 4) * kTileN * 16;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float4 v = lds128_f32(src + j * kTileN * 16);
                  acc[4 * j + 0] += v.x;
                  acc[4 * j + 1] += v.y;
                  acc[4 * j + 2] += v.z;
                  acc[4 * j + 3] += v.w;
                }
              }
            }
            if (last_batch) {
              y_chunk(c0, acc);
            } else {
              uint32_t v[16];
#pragma unroll
              for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(acc[j]);
              tmem_st_x16(t_acc + c0, v);
            }
          }
          tmem_wait_st();
          // every thread is done with this batch's slots before the next copies
          named_bar_sync(1, kNumEpiWarps * 32);
        }
        if (own_in_tmem) {  // (a published partial already handed its D buffer back)
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[d]);
        }
        y_end();
      };
      // Stream-K fixup roles (static, so nobody waits for an atomic's reply):
      // the REDUCER of a split tile is its first contributor in k order,
      // c_first — the tile's head is the END of c_first's range, so this is
      // always c_first's last segment and every other contributor's share
      // (a whole range inside the tile, or the first segment of c_last's)
      // finishes no later.  The others publish their fp32 partial and count
      // in with one release reduction (no round trip: they go on, or exit);
      // the reducer polls the tile counter after its own MMAs, then sums
      // own + partials in k order (deterministic) and stores Y.
      constexpr int kPartBytes = kTileN * BN * 4;
      bool reducer = false;
      if (!CSK && !sg.full) {
        contributors();
        reducer = c_first == static_cast<int>(blockIdx.x);
      }
      if constexpr (C::kPD) {
        // FGQ per-block partials (gemm.py:96-110): for every 128-k tile of the
        // segment, in k order, acc += S_block * partial (fp32, product and
        // sum rounded separately like the reference), then the segment's sum
        // goes to D buffer d, read below like an MMA accumulator
        float pacc[BN];
#pragma unroll
        for (int j = 0; j < BN; ++j) pacc[j] = 0.f;
        const uint32_t t_p = t_lane + C::kDBufs * C::kDCols;
        const uint32_t t_sc = t_p + C::kPSlots * BN;  // block scales, column = ordinal mod 32
#pragma unroll 1
        for (int s = 0; s < sg.len; ++s) {
          const int i = sg.i0 + s, kt = sg.kt0 + s * KS, nt = min(KS, sg.kt1 - kt);
#pragma unroll
          for (int t = 0; t < KS; ++t) {
            if (t < nt) {
              if constexpr (FGQ == 2) {
                const int P = fg.sub;
                int n_tile, m_tile;
                tile_nm(a, sg.tile, n_tile, m_tile);
                const int nn = n_tile * kTileN + rr;
#pragma unroll 1
                for (int p = 0; p < P; ++p) {
                  const int q = (KS * i + t) * P + p, ps = q % C::kPSlots, blk = (kt + t) * P + p;
                  // this row's raw block scale (the load overlaps the partial wait)
                  const float scl = nn < a.N && blk < fg.bpr
                                        ? __half2float(__ushort_as_half(__ldg(fg.scales + (int64_t)nn * fg.bpr + blk)))
                                        : 0.f;
                  mbar_wait<LPQT_PD_WAIT>(&pfull[ps], (q / C::kPSlots) & 1);
                  tc_fence_after();
#pragma unroll
                  for (int c0 = 0; c0 < BN; c0 += 16) {
                    uint32_t v[16];
                    tmem_ld_x16(t_p + ps * BN + c0, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                      pacc[c0 + j] = __fadd_rn(pacc[c0 + j], __fmul_rn(scl, __uint_as_float(v[j])));
                  }
                  tc_fence_before();
                  __syncwarp();
                  if (lane == 0) mbar_arrive(&pempty[ps]);
                }
              } else {
                const int q = KS * i + t, ps = q % C::kPSlots;
                mbar_wait<LPQT_PD_WAIT>(&pfull[ps], (q / C::kPSlots) & 1);
                tc_fence_after();
                uint32_t sv;
                tmem_ld_x1(t_sc + (q & 31), sv);
#pragma unroll
                for (int c0 = 0; c0 < BN; c0 += 16) {
                  uint32_t v[16];
                  tmem_ld_x16(t_p + ps * BN + c0, v);
                  tmem_wait_ld();
                  const float scl = __uint_as_float(sv);
#pragma unroll
                  for (int j = 0; j < 16; ++j)
                    pacc[c0 + j] = __fadd_rn(pacc[c0 + j], __fmul_rn(scl, __uint_as_float(v[j])));
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&pempty[ps]);
              }
            } else {
              // ragged stage: pass the missing tile's (empty) partial ordinals on
              const int P = FGQ == 2 ? fg.sub : 1;
#pragma unroll 1
              for (int p = 0; p < P; ++p) {
                const int q = (KS * i + t) * P + p, ps = q % C::kPSlots;
                mbar_wait<LPQT_PD_WAIT>(&pfull[ps], (q / C::kPSlots) & 1);
                tc_fence_after();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&pempty[ps]);
              }
            }
          }
        }
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t v[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(pacc[c0 + j]);
          tmem_st_x16(t_d + c0, v);
        }
        tmem_wait_st();
      } else {
        mbar_wait<WM>(&dfull[d], dph);
      }
      if (last_seg && warp == kWarpEpi0 && lane == 0) CTA_STAMP(8);
      tc_fence_after();
      if constexpr (CSK) {
        // ---- cluster split-K: reduce the C partials of this tile over DSMEM
        const int b = lu & 1;  // staging buffer / barrier of this round
        // staging layout [BN / 4][128] float4: thread rr writes column chunk
        // j at (j * 128 + rr) * 16 (conflict-free)
        const uint32_t stg = smem_u32(smem_stg) + b * C::kStageBufBytes + rr * 16;
        if (sc.C > 1 && sc.rank != sg.red) {
          // sender: wait until the reducer that read this buffer last is
          // done with it, stage the partial, signal this round's reducer
          if ((sent_bits >> b) & 1u) {
            mbar_wait_cluster(smem_u32(&stg_free[b]), (sf_bits >> b) & 1u);
            sf_bits ^= 1u << b;
          }
          sent_bits |= 1u << b;
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float acc[16];
            load_acc16<BN>(t_d, c0, q0, nacc, acc);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(stg + (c0 / 4 + j) * 128 * 16),
                           "f"(acc[4 * j]), "f"(acc[4 * j + 1]), "f"(acc[4 * j + 2]), "f"(acc[4 * j + 3])
                           : "memory");
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[d]);
          named_bar_sync(1, kNumEpiWarps * 32);
          if (warp == kWarpEpi0 && lane == 0)
            mbar_arrive_remote(mapa_shared(smem_u32(&part_full[b]), static_cast<uint32_t>(sg.red)));
        } else {
          // reducer: own partial into registers and the D buffer straight
          // back to the MMA (the reduction below must not stall the
          // pipeline), then wait for the C - 1 partials and sum in rank order
          float own[BN];
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float t16[16];
            load_acc16<BN>(t_d, c0, q0, nacc, t16);
#pragma unroll
            for (int j = 0; j < 16; ++j) own[c0 + j] = t16[j];
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&dempty[d]);
          if (sc.C > 1) {
            mbar_wait_cluster(smem_u32(&part_full[b]), (pf_bits >> b) & 1u);
            pf_bits ^= 1u << b;
          }
          y_begin();
#pragma unroll
          for (int c0 = 0; c0 < BN; c0 += 16) {
            float sum[16];
#pragma unroll
            for (int j = 0; j < 16; ++j) sum[j] = 0.f;
#pragma unroll 1
            for (int r = 0; r < sc.C; ++r) {
              if (r == sc.rank) {
#pragma unroll
                for (int j = 0; j < 16; ++j) sum[j] += own[c0 + j];
              } else {
                const uint32_t src = mapa_shared(stg + (c0 / 4) * 128 * 16, static_cast<uint32_t>(r));
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const float4 v = ld_dsmem_f4(src + j * 128 * 16);
                  sum[4 * j] += v.x;
                  sum[4 * j + 1] += v.y;
                  sum[4 * j + 2] += v.z;
                  sum[4 * j + 3] += v.w;
                }
              }
            }
            y_chunk(c0, sum);
          }
          y_end();
          if (sc.C > 1) {
            // the senders' staging buffers are read: hand them back
            named_bar_sync(1, kNumEpiWarps * 32);
            if (warp == kWarpEpi0 && lane < sc.C && lane != sc.rank)
              mbar_arrive_remote(mapa_shared(smem_u32(&stg_free[b]), static_cast<uint32_t>(lane)));
          }
        }
      } else if (sg.full) {
        y_begin();
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          float acc[16];
          load_acc16<BN>(t_d, c0, q0, nacc, acc);
          if (c0 + 16 >= BN) {  // last chunk read: hand the D buffer back to the MMA warp
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&dempty[d]);
          }
          y_chunk(c0, acc);
        }
        y_end();
      } else {
        // ---- stream-K partial tile
        if (!reducer) {
          float4* part = reinterpret_cast<float4*>(a.partials) + PartLayout<BN>::f4((int64_t)blockIdx.x * 2 + sg.pidx, 0, rr);
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
              __stcg(part + ((c0 + j) / 4) * PartLayout<BN>::kJStride, make_float4(acc[j], acc[j + 1], acc[j + 2], acc[j + 3]));
            }
          }
          // publish: CTA barrier (cumulativity over the epilogue's stores),
          // then one gpu-scope release reduction — no reply awaited
          named_bar_sync(1, kNumEpiWarps * 32);
          if (warp == kWarpEpi0 && lane == 0) {
            if (last_seg) CTA_STAMP(9);
            red_add_release_gpu(&a.counters[sg.tile], sg.len);
            if (last_seg) CTA_STAMP(10);
          }
        } else {
          // reducer: wait until the other contributors' k-steps are published
          if (warp == kWarpEpi0 && lane == 0) {
            const int others = a.ksteps - sg.len;
            for (uint32_t spin = 0; ld_acquire_gpu(&a.counters[sg.tile]) != others; ++spin) {
              if (spin > (1u << 26)) __trap();  // a contributor never published: fail loudly
              __nanosleep(32);
            }
            CTA_STAMP(10);
          }
          named_bar_sync(1, kNumEpiWarps * 32);
          if (BN >= 128 && C::kDBufs == 2) {
            tail_reduce(true);  // (own partial in TMEM, the others by bulk copy in batches)
          } else if ((int64_t)(c_last - c_first) * kPartBytes <= (int64_t)C::kWStages * C::kWStageBytes) {
            // last segment: every W stage is consumed, so the ring takes the
            // other contributors' partials in ONE round trip (one bulk copy
            // each, in flight together); own partial stays in TMEM
            if (warp == kWarpEpi0 && lane == 0) {
              fence_proxy_async_global();  // generic-proxy partials (acquired above) -> bulk-copy reads
              mbar_arrive_expect_tx(fix_bar, static_cast<uint32_t>(c_last - c_first) * kPartBytes);
              for (int c = c_first + 1; c <= c_last; ++c)
                bulk_g2s_plain(smem_w + (c - c_first - 1) * kPartBytes, a.partials + ((int64_t)c * 2) * (kTileN * BN),
                               kPartBytes, fix_bar);
            }
            y_begin();
            mbar_wait<WM>(fix_bar, 0);
            if (warp == kWarpEpi0 && lane == 0) CTA_STAMP(23);
            const uint32_t base = smem_u32(smem_w) + static_cast<uint32_t>(rr * 16);  // chunk-major rows
#pragma unroll 1
            for (int c0 = 0; c0 < BN; c0 += 16) {
              float acc[16];
              load_acc16<BN>(t_d, c0, q0, nacc, acc);
              if (c0 + 16 >= BN) {
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&dempty[d]);
              }
              // (0 + own) + p1 + p2 ...: contributors in k order
#pragma unroll
              for (int j = 0; j < 16; ++j) acc[j] = 0.f + acc[j];
#pragma unroll 1
              for (int c = 1; c <= c_last - c_first; ++c) {
                if constexpr (PartLayout<BN>::kChunkMajor) {
                  const uint32_t src = base + (c - 1) * kPartBytes + (c0 / 4) * kTileN * 16;
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const float4 v = lds128_f32(src + j * kTileN * 16);
                    acc[4 * j + 0] += v.x;
                    acc[4 * j + 1] += v.y;
                    acc[4 * j + 2] += v.z;
                    acc[4 * j + 3] += v.w;
                  }
                } else {  // rows contiguous
                  const uint32_t src = smem_u32(smem_w) + (c - 1) * kPartBytes + (rr * BN + c0) * 4;
#pragma unroll
                  for (int j = 0; j < 4; ++j) {
                    const float4 v = lds128_f32(src + j * 16);
                    acc[4 * j + 0] += v.x;
                    acc[4 * j + 1] += v.y;
                    acc[4 * j + 2] += v.z;
                    acc[4 * j + 3] += v.w;
                  }
                }
              }
              y_chunk(c0, acc);
            }
            if (warp == kWarpEpi0 && lane == 0) CTA_STAMP(24);
            y_end();
          } else {
            // many contributors (partials exceed the W ring): L2 loads in k
            // order, kFix at a time so their round trips overlap
            y_begin();
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
              for (int j = 0; j < 16; ++j) acc[j] = 0.f + acc[j];
              constexpr int kFix = BN <= 32 ? 1 : 2;  // (decode epilogue: 72 registers)
#pragma unroll 1
              for (int cb = c_first + 1; cb <= c_last; cb += kFix) {
                float4 v[kFix][4];
#pragma unroll
                for (int u = 0; u < kFix; ++u) {
                  const int c = cb + u;
                  if (c <= c_last) {
                    if constexpr (PartLayout<BN>::kChunkMajor) {
                      const float4* src = reinterpret_cast<const float4*>(a.partials) +
                                          PartLayout<BN>::f4((int64_t)c * 2, c0 / 4, rr);
#pragma unroll
                      for (int j = 0; j < 4; ++j) v[u][j] = __ldcg(src + j * PartLayout<BN>::kJStride);
                    } else {
                      const float4* src = reinterpret_cast<const float4*>(
                          a.partials + (((int64_t)c * 2) * kTileN + rr) * BN + c0);
#pragma unroll
                      for (int j = 0; j < 4; ++j) v[u][j] = __ldcg(src + j);
                    }
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
              y_chunk(c0, acc);
            }
            y_end();
          }
          // every partial is read: re-arm the counter for the next launch
          if (warp == kWarpEpi0 && lane == 0) {
            a.counters[sg.tile] = 0;
            if (last_seg) CTA_STAMP(11);
          }
        }
        named_bar_sync(1, kNumEpiWarps * 32);
      }
    }
    if (ytma && warp == kWarpEpi0 && lane == 0) {
      if constexpr (PEERS) {
        bulk_wait_all();  // the peer stores are complete before this CTA counts in
        asm volatile("fence.proxy.async.global;" ::: "memory");
      } else {
        bulk_wait_read<0>();  // smem stays valid until read
      }
    }
    if (warp == kWarpEpi0 && lane == 0) CTA_STAMP(5);
  }

  if constexpr (CSK) {
    if (warp < kWarpEpi0) cluster_wait();  // the setup phase (epilogue waited already)
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (PEERS) {
    if (threadIdx.x == 0) peer_complete(po);
  }
  // CSK: no CTA may leave while a peer can still read its staging buffer or
  // arrive on its barriers
  if constexpr (CSK) cluster_sync_all();
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
  bool csk;
  bool dp;      // prefill: whole tiles round-robin (SkSched DP mode)
  int cluster;  // CSK cluster size
  int splits;   // max CTAs contributing to one tile
  int64_t K;    // X's k extent: TMA zero-fills columns K .. ldx (W4A16 pads with Z, not 0)
};

// Prefill MMA N (M > 128).  192 keeps two accumulators in TMEM (the epilogue
// of one tile overlaps the next tile's MMAs) and its MMA time per k-tile
// (~770 cycles) still covers the 128-row dequant (~600); 256 has a single
// accumulator (the tensor pipe idles through every epilogue) and 128 is
// dequant-bound.  Measured: profiles/r01_v8_probe_prefill_bn192.txt.
#ifndef LPQT_PREFILL_BN
#define LPQT_PREFILL_BN 192
#endif
#ifndef LPQT_SK_SPLIT_WIDE
#define LPQT_SK_SPLIT_WIDE 0  // > 0: fixed cap on CTAs per tile for BN >= 64 (tuning hook)
#endif
static int pick_bn(int64_t M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128 || LPQT_PREFILL_BN == 128) return 128;
  if (LPQT_PREFILL_BN != 192) return LPQT_PREFILL_BN;
  // per 128-k step a 128-row weight tile costs ~600 cycles at N = 128 (the
  // dequant bound) and ~768 at N = 192 (the MMA bound): take the width whose
  // batch tiles cover M in the fewest cycles (M = 256: 2 x 128, not 2 x 192)
  const int64_t c128 = (M + 127) / 128 * 600, c192 = (M + 191) / 192 * 768;
  return c128 < c192 ? 128 : 192;
}

template <int BN, bool CSK>
static void cfg_of(Plan& p) {
  p.stages = Cfg<BN, CSK>::kStages;
  p.smem = Cfg<BN, CSK>::kSmemBytes;
  p.kstep = Cfg<BN, CSK>::kKStep;
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

// Co-resident clusters of c CTAs for the decode kernel (GPC packing; 1 CTA
// per SM).  Queried once per c from the driver; the fallback is a 148-SM
// B200 as measured (tools/cluster_occ.cu).
template <int BN>
static int max_clusters(int c) {
  static int cache[kMaxCluster + 1] = {0};
  static std::mutex mu;
  std::lock_guard<std::mutex> lock(mu);
  if (cache[c] > 0) return cache[c];
  static const int fallback[kMaxCluster + 1] = {0, 148, 74, 45, 33, 26, 22, 15, 15};
  int n = 0;
  auto kern = w6a16_tcgen05_kernel<BN, true, true>;
  constexpr int smem = Cfg<BN, true>::kSmemBytes;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess &&
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) == cudaSuccess) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(c * 64);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
  }
  cudaGetLastError();  // a failed query must not poison later launches
  if (n <= 0) n = fallback[c];
  cache[c] = n;
  return n;
}

static int max_clusters_bn(int bn, int c) { return bn <= 16 ? max_clusters<16>(c) : max_clusters<32>(c); }

// split_k == 0: automatic schedule.  With LPQT_SCHED_CLUSTER: cluster
// split-K with C = split_k (>= 1).  Otherwise split_k > 0 is stream-K with
// about split_k CTAs per tile (testing / tuning hooks).
static Plan make_plan(int64_t M, int64_t N, int64_t K, int split_k, int flags, int sms, bool fgq = false) {
  Plan p{};
  p.bn = pick_bn(M);
  p.n_tiles = static_cast<int>((N + kTileN - 1) / kTileN);
  p.m_tiles = static_cast<int>((M + p.bn - 1) / p.bn);
  p.K = K;
  p.k_tiles = static_cast<int>((K + kTileK - 1) / kTileK);
  p.tiles = (int64_t)p.n_tiles * p.m_tiles;
  // ---- schedule choice (decode, BN <= 32, may use cluster split-K)
  const bool csk_ok = p.bn <= 32 && p.tiles < ((int64_t)1 << 30);
  int best_c = 0;
  if (csk_ok && !(flags & LPQT_SCHED_STREAMK)) {
    if (flags & LPQT_SCHED_CLUSTER) {
      best_c = split_k > 0 ? split_k : 1;
      best_c = std::min(best_c, std::min(kMaxCluster, p.k_tiles));
    } else if (split_k == 0) {
      // Time model of one launch (us; fitted to B200 measurements of both
      // schedules on the LLaMA shapes, tools/abx.py, profiles/): a CTA
      // streams one 128x128 FP6 tile in ~0.31 us; stream-K pays ~3-6 us of
      // cross-CTA fixups on its tail when tiles are split; cluster split-K
      // ~0.7 us of DSMEM reduction per round plus ~0.5 us of cluster
      // launch/sync.  Only C <= 2 is chosen automatically (larger clusters
      // measured slower than the model predicts).
      const double tile_us = 0.31;
      const double sk_kt = (double)p.tiles * p.k_tiles / sms;  // k-tiles per CTA
      // Round 2 (stream-K with the static reducer, no atomic round trip on the
      // tail): stream-K wins once every CTA streams >= 16 k-tiles — 70B O
      // 8192 x 8192 −6 %, 7B QKV −5 % against the cluster plan, equal on the
      // rest (profiles/r02_abx_decode_schedules.jsonl); below that (7B O,
      // 4096 x 4096: 7 k-tiles per CTA) the fixups dominate and the model
      // below still picks cluster split-K.
      if (sk_kt >= 16.0) goto done_csk;
      const bool sk_partial = ((int64_t)p.tiles * p.k_tiles) % sms != 0 || p.tiles % sms != 0;
      // (a range spanning whole tiles splits each tile between two CTAs,
      // whose fixup takes the last-arriver fast path; long ranges hide part
      // of the tail)
      const double sk_tail = sk_kt >= p.k_tiles ? 2.0 : (sk_kt < 64.0 ? 6.0 : 3.0);
      double best = sk_kt * tile_us + (sk_partial ? sk_tail : 0.0);
      for (int c = 1; c <= 2 && c <= p.k_tiles; ++c) {
        const int64_t ncl = std::min<int64_t>(max_clusters_bn(p.bn, c), p.tiles);
        const int64_t rounds = (p.tiles + ncl - 1) / ncl;
        const double us = rounds * (((p.k_tiles + c - 1) / c) * tile_us + (c > 1 ? 0.7 : 0.0)) + (c > 1 ? 0.5 : 0.0);
        if (us < best) {
          best = us;
          best_c = c;
        }
      }
    }
  }
done_csk:
  if (best_c > 0) {
    p.csk = true;
    p.cluster = best_c;
    if (p.bn <= 16) {
      cfg_of<16, true>(p);
    } else {
      cfg_of<32, true>(p);
    }
    const int64_t ncl = std::min<int64_t>(max_clusters_bn(p.bn, best_c), p.tiles);
    p.grid = static_cast<int>(ncl * best_c);
    p.ksteps = (p.k_tiles + p.kstep - 1) / p.kstep;
    p.splits = best_c;
    return p;
  }
  switch (p.bn) {
    case 16: cfg_of<16, false>(p); break;
    case 32: cfg_of<32, false>(p); break;
    case 64: cfg_of<64, false>(p); break;
    case 128: cfg_of<128, false>(p); break;
    case 192: cfg_of<192, false>(p); break;
    default: cfg_of<256, false>(p); break;
  }
  p.ksteps = (p.k_tiles + p.kstep - 1) / p.kstep;
  p.total = p.tiles * p.ksteps;
  int64_t g = split_k > 0 ? p.tiles * split_k : sms;
  // BN >= 64: splitting a tile costs a 128 x BN fp32 partial round trip per
  // contributor; it pays only when each CTA still contracts >= ~24 k-tiles
  // (measured, profiles/r01_v8_abx_split_cap.jsonl: no split at K = 4096, two
  // at 8192, three at 11008, four at 28672)
  if (split_k == 0 && p.kstep == 1) {
    int64_t cap = LPQT_SK_SPLIT_WIDE > 0 ? LPQT_SK_SPLIT_WIDE : std::min(4, std::max(1, p.k_tiles / 24));
    // few tiles (tensor-parallel shards): the capped grid would leave most SMs
    // idle, so split further while every CTA keeps >= 16 k-tiles
    // (profiles/r02_probe_tp8_split.jsonl: 1280 x 8192, M = 64: 4 splits 24.6 us
    // against 2 splits 30.7 us)
    if (LPQT_SK_SPLIT_WIDE == 0 && 2 * p.tiles * cap < sms)
      cap = std::max<int64_t>(cap, std::min<int64_t>(p.k_tiles / 16, sms / p.tiles));
    if (g > p.tiles * cap) g = p.tiles * cap;
    // prefill (BN 192) tiles that fit one wave: one whole tile per CTA beats
    // spreading them over every SM (the 128 x 192 partial reduction costs
    // more than the idle SMs); at BN 128 splitting still wins
    // (profiles/r01_v14_probe_prefill_split.jsonl, _onewave_bn192.jsonl)
    // (BN 128 with several batch tiles: only when the wave is >= 3/4 full;
    // profiles/r01_v14_abx_onewave_bn128.jsonl)
    if ((p.bn >= 192 || (p.bn == 128 && p.m_tiles > 1 && 4 * p.tiles >= 3 * (int64_t)sms)) && p.tiles <= sms)
      g = p.tiles;
  }
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
  // prefill whose X outgrows L2 (see args.n_fastest): round-robin whole tiles
  // keep the CTAs in flight on consecutive tiles, sharing X in L2
  if (p.kstep == 1 && p.m_tiles > 1 && M * K * 2 > ((int64_t)40 << 20) && p.tiles >= 2 * (int64_t)sms &&
      p.tiles < ((int64_t)1 << 30) && split_k == 0 && !(flags & LPQT_SCHED_STREAMK)) {
    p.dp = true;
    p.grid = sms;
    p.partials = false;
    p.counters_bytes = 0;
    p.ws_bytes = 0;
    p.splits = 1;
    return p;
  }
  const int64_t per = p.total / p.grid;  // k-steps per CTA (floor)
  p.splits = p.partials ? static_cast<int>((p.ksteps + (per > 0 ? per : 1) - 1) / (per > 0 ? per : 1) + 1) : 1;
  return p;
}

int launch_prefill_2sm(const uint8_t* tiles, const uint16_t* scales, const uint16_t* Xt, int64_t ldx, int64_t M,
                       int64_t N, int64_t K, void* Y, int y_dtype, int y_layout, int64_t ldy, int flags,
                       int force, void* workspace, int64_t workspace_bytes, cudaStream_t stream,
                       int* grid_out, bool fgq, bool fp5);     // prefill2sm.cu
int prefill_2sm_pairs();                                       // prefill2sm.cu
double prefill_2sm_choose(int64_t M, int64_t N, int64_t K, int* bn_out, int* sk_out, int force);  // prefill2sm.cu
int64_t prefill_2sm_workspace();                                                              // prefill2sm.cu

// The CTA-pair prefill kernel (prefill2sm.cu) vs this file's single-SM one:
// per-SM cycle estimates, pair kernel ~1024 cycles per 128-k step of a
// 256 x 256 unit at ~90 % tensor-pipe efficiency, whole units per pair;
// single-SM kernel: the BN-192 / 128 step cost over 148 SMs at the measured
// ~60 % efficiency (68 % tensor-pipe activity at M = 2048, less with the
// stream-K fixups at M = 512; profiles/r02_ncu_prefill_m2048.json,
// r02_abx_pair_vs_single.jsonl).
// Automatic choice: the pair kernel from M = LPQT_PAIR_MIN_M up whenever the
// weight has an even number of 128-row tiles.  Measured on the 7B / 70B
// shapes (profiles/r02_probe_pair_vs_single_small_m.jsonl): at M = 128 / 256
// the pair kernel takes 0.55-0.85x the single-SM kernel's time (whose BN-128
// stream-K fixups of 64-KB partials dominate), and above that it wins by more.
#ifndef LPQT_PAIR_MIN_M
#define LPQT_PAIR_MIN_M 65  // (below: decode / small prefill stay single-SM)
#endif
// The pair kernel's schedule choice: split_k 0 = automatic; with
// LPQT_SCHED_PAIR, split_k 1 / 2 force whole units / whole rounds + a
// stream-K wave (testing / tuning hooks).  -1: split_k asks for the single-SM kernel.
static int pair_force(int split_k, int flags) {
  if (split_k == 0) return 0;
  return (flags & LPQT_SCHED_PAIR) && split_k <= 2 ? split_k : -1;
}
static bool use_pair_kernel(int64_t M, int64_t N, int64_t K, int flags) {
  (void)K;
  if (flags & LPQT_SCHED_SINGLE) return false;
  const int64_t n_tiles = (N + kTileN - 1) / kTileN;
  if (n_tiles % 2 != 0 || M < 17) return false;
  if (flags & LPQT_SCHED_PAIR) return true;
  return !(flags & (LPQT_SCHED_STREAMK | LPQT_SCHED_CLUSTER)) && M >= LPQT_PAIR_MIN_M;
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
// kTraceSlots trace records; launch n writes record n % kTraceSlots (graph
// captures bake the record index in at capture time)
constexpr int kTraceSlots = 16;
static long long* trace_buffer() {
  static long long* buf = nullptr;
  if (!buf) {
    cudaMalloc(&buf, (size_t)kTraceSlots * kTraceLen * sizeof(long long));
    cudaMemset(buf, 0, (size_t)kTraceSlots * kTraceLen * sizeof(long long));
  }
  return buf;
}
static int g_trace_n = 0;  // launches traced so far
static int trace_next_slot() { return g_trace_n++ % kTraceSlots; }
#endif

template <int BN, bool CSK, bool RAGGED, int FGQ = 0, int WB = 6, bool PEERS = false, int RB = 0>
static int launch_impl(const Plan& p, const GemmArgs& args, const L2Prefetch& pf, const FgqArgs& fg,
                       const uint16_t* Xt, int64_t ldx,
                       int64_t M, cudaStream_t stream, int flags, const lpqt_peer_out* peers = nullptr) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return LPQT_E_CUDA;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(p.K), static_cast<cuuint64_t>(M)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(BN)};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(Xt), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return LPQT_E_INVALID_INPUT;
  auto kern = w6a16_tcgen05_kernel<BN, CSK, RAGGED, FGQ, WB, PEERS, RB>;
  constexpr int smem = Cfg<BN, CSK, WB, FGQ>::kSmemBytes;
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
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (flags & LPQT_LAUNCH_PDL) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  if (CSK) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = p.cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  GemmArgs a2 = args;
  a2.csk_c = CSK ? p.cluster : 0;
  // Y tensor map for the TMA store epilogue (decode tiles); shapes the TMA
  // cannot describe (unaligned base / row stride) keep the direct stores
  CUtensorMap ymap;
  memset(&ymap, 0, sizeof(ymap));
  a2.y_tma = 0;
  lpqt_peer_out po;
  memset(&po, 0, sizeof(po));
  if (peers) po = *peers;
  PeerMapsOf<PEERS> pmaps;
  memset(&pmaps, 0, sizeof(pmaps));
  if (Cfg<BN, CSK, WB, FGQ>::kYBufBytes > 0) {
    const int es = args.y_dtype == LPQT_F32 ? 4 : 2;
    const CUtensorMapDataType dt = args.y_dtype == LPQT_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : args.y_dtype == LPQT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                              : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    const bool nm = args.y_layout == LPQT_Y_NM;
    const cuuint64_t ydims[2] = {static_cast<cuuint64_t>(nm ? args.M : args.N),
                                 static_cast<cuuint64_t>(nm ? args.N : args.M)};
    const cuuint64_t ystr[1] = {static_cast<cuuint64_t>(args.ldy) * es};
    const cuuint32_t ybox[2] = {static_cast<cuuint32_t>(nm ? BN : kTileN), static_cast<cuuint32_t>(nm ? kTileN : BN)};
    const bool ok = (reinterpret_cast<uintptr_t>(args.y) % 16 == 0) && (ystr[0] % 16 == 0) &&
                    ((cuuint64_t)ybox[0] * es) % 16 == 0 && (PEERS || ydims[1] > 1);
    auto encode_y = [&](void* base, CUtensorMap* out) {
      return ok && reinterpret_cast<uintptr_t>(base) % 16 == 0 &&
             enc(out, dt, 2, base, ydims, ystr, ybox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    };
    bool all = encode_y(args.y, &ymap);
    if constexpr (PEERS) {
      for (int q = 0; q < po.npeers; ++q) all = all && encode_y(po.y[q], &pmaps.m[q]);
    }
    if (all) a2.y_tma = 1;
    if (PEERS && !all) return LPQT_E_SHAPE;  // peer Y base / row stride not 16-byte aligned
  }
  if (cudaLaunchKernelEx(&cfg, kern, map, ymap, a2, pf, fg, po, pmaps) != cudaSuccess) return LPQT_E_CUDA;
  note_launch();
  return check_launch();
}

}  // namespace lpqt

using namespace lpqt;

// Schedule / stage-shape dispatch shared by the FP6 (CGQ, FGQ) and INT4 entries.
template <int FGQ, int WB, bool PEERS = false>
static int dispatch(const Plan& p, const GemmArgs& args, const L2Prefetch& pfa, const FgqArgs& fga,
                    const uint16_t* Xt, int64_t ldx, int64_t M, cudaStream_t st, int flags,
                    const lpqt_peer_out* po = nullptr) {
  bool ragged = p.k_tiles % p.kstep != 0;
  if (p.csk) {
    for (int r = 0; r < p.cluster; ++r)  // k-range of rank r must be a whole number of stages
      ragged |= ((r + 1) * p.k_tiles / p.cluster - r * p.k_tiles / p.cluster) % p.kstep != 0;
    if (p.bn <= 16)
      return ragged ? launch_impl<16, true, true, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po)
                    : launch_impl<16, true, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
    return ragged ? launch_impl<32, true, true, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po)
                  : launch_impl<32, true, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
  }
  if constexpr (FGQ == 2) {  // (sub-tile FGQ blocks: decode widths only)
    if (p.bn > 32) return LPQT_E_UNSUPPORTED;
    if (p.bn <= 16)
      return ragged ? launch_impl<16, false, true, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po)
                    : launch_impl<16, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
    return ragged ? launch_impl<32, false, true, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po)
                  : launch_impl<32, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
  }
  switch (p.bn) {
    case 16:
      return ragged ? launch_impl<16, false, true, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po)
                    : launch_impl<16, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
    case 32:
      return ragged ? launch_impl<32, false, true, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po)
                    : launch_impl<32, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
    case 64: return launch_impl<64, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
    case 128: return launch_impl<128, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
    case 192: return launch_impl<192, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
    default:
      if constexpr (FGQ) return LPQT_E_UNSUPPORTED;  // (BN 256 only by LPQT_PREFILL_BN override)
      else return launch_impl<256, false, false, FGQ, WB, PEERS>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
  }
}

// The ablation rebuilds (LPQT_REBUILD_*): decode batch tile (BN 16), CGQ FP6.
template <int RB>
static int dispatch_rebuild(const Plan& p, const GemmArgs& args, const L2Prefetch& pfa, const FgqArgs& fga,
                            const uint16_t* Xt, int64_t ldx, int64_t M, cudaStream_t st, int flags) {
  if (p.bn != 16) return LPQT_E_UNSUPPORTED;
  bool ragged = p.k_tiles % p.kstep != 0;
  if (p.csk) {
    for (int r = 0; r < p.cluster; ++r)
      ragged |= ((r + 1) * p.k_tiles / p.cluster - r * p.k_tiles / p.cluster) % p.kstep != 0;
    return ragged ? launch_impl<16, true, true, false, 6, false, RB>(p, args, pfa, fga, Xt, ldx, M, st, flags)
                  : launch_impl<16, true, false, false, 6, false, RB>(p, args, pfa, fga, Xt, ldx, M, st, flags);
  }
  return ragged ? launch_impl<16, false, true, false, 6, false, RB>(p, args, pfa, fga, Xt, ldx, M, st, flags)
                : launch_impl<16, false, false, false, 6, false, RB>(p, args, pfa, fga, Xt, ldx, M, st, flags);
}

extern "C" {

#ifdef LPQT_TRACE
int lpqt_trace_dump(long long* host) {  // the last launch's record
  cudaDeviceSynchronize();
  const int slot = (g_trace_n + kTraceSlots - 1) % kTraceSlots;
  return cudaMemcpy(host, trace_buffer() + (size_t)slot * kTraceLen, kTraceLen * sizeof(long long),
                    cudaMemcpyDeviceToHost) == cudaSuccess
             ? 0
             : -1;
}
// all kTraceSlots records (launch n -> record n % kTraceSlots); returns the
// number of launches traced so far
int lpqt_trace_dump_all(long long* host, int* n_launches) {
  cudaDeviceSynchronize();
  if (n_launches) *n_launches = g_trace_n;
  return cudaMemcpy(host, trace_buffer(), (size_t)kTraceSlots * kTraceLen * sizeof(long long),
                    cudaMemcpyDeviceToHost) == cudaSuccess
             ? 0
             : -1;
}
#endif

int64_t lpqt_w6a16_workspace_bytes(int64_t M, int64_t N, int64_t K, int split_k) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  // the largest any schedule of this shape may need (auto or forced stream-K)
  const Plan p0 = make_plan(M, N, K, split_k, 0, num_sms());
  const Plan p1 = make_plan(M, N, K, split_k, LPQT_SCHED_STREAMK, num_sms());
  // (the pair kernel's stream-K schedule: whenever the pair kernel may run)
  // (the pair kernel's stream-K wave, when its planner picks it — or split_k 2 forces it with LPQT_SCHED_PAIR)
  int pair_sk = 0;
  if ((N + kTileN - 1) / kTileN % 2 == 0 && M >= 17) {
    if (split_k == 0) prefill_2sm_choose(M, N, K, nullptr, &pair_sk, 0);
    if (split_k == 2) pair_sk = 1;
  }
  const int64_t wp = pair_sk ? prefill_2sm_workspace() : 0;
  return std::max(wp, p0.ws_bytes > p1.ws_bytes ? p0.ws_bytes : p1.ws_bytes);
}

int lpqt_w6a16_plan_ex(int64_t M, int64_t N, int64_t K, int split_k, int flags, int* out, int n_out) {
  if (M <= 0 || N <= 0 || K <= 0) return LPQT_E_SHAPE;
  if ((flags & LPQT_SCHED_STREAMK) && (flags & LPQT_SCHED_CLUSTER)) return LPQT_E_INVALID_INPUT;
  if (pair_force(split_k, flags) >= 0 && use_pair_kernel(M, N, K, flags)) {
    int bn = 256, sk = 0;
    prefill_2sm_choose(M, N, K, &bn, &sk, pair_force(split_k, flags));
    const int64_t units = ((N + kTileN - 1) / kTileN / 2) * ((M + bn - 1) / bn);
    // splits: pairs sharing one unit (stream-K cuts a unit between pairs)
    const int v[6] = {bn, sk ? 2 : 1, 2 * (int)(sk ? prefill_2sm_pairs() : std::min<int64_t>(prefill_2sm_pairs(), units)),
                      6, 3, 2};
    for (int i = 0; i < n_out && i < 6; ++i) out[i] = v[i];
    return LPQT_OK;
  }
  const Plan p = make_plan(M, N, K, split_k, flags, num_sms());
  const int v[6] = {p.bn, p.splits, p.grid, p.stages, p.csk ? 1 : (p.dp ? 2 : 0), p.csk ? p.cluster : 0};
  for (int i = 0; i < n_out && i < 6; ++i) out[i] = v[i];
  return LPQT_OK;
}

// Reports the plan: block_n = MMA N, splits = max CTAs sharing one tile,
// grid = CTAs, stages = smem pipeline depth.
int lpqt_w6a16_plan(int64_t M, int64_t N, int64_t K, int split_k, int* block_n, int* splits, int* grid, int* stages) {
  int v[4];
  const int st = lpqt_w6a16_plan_ex(M, N, K, split_k, 0, v, 4);
  if (st != LPQT_OK) return st;
  if (block_n) *block_n = v[0];
  if (splits) *splits = v[1];
  if (grid) *grid = v[2];
  if (stages) *stages = v[3];
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
  return lpqt_w6a16_linear_pf(tiles, scales, Xt, ldx, M, N, K, Y, y_dtype, y_layout, ldy, split_k, workspace,
                              workspace_bytes, flags, nullptr, stream);
}

int lpqt_w6a16_linear_pf(const uint8_t* tiles, const uint16_t* scales, const uint16_t* Xt, int64_t ldx, int64_t M,
                         int64_t N, int64_t K, void* Y, int y_dtype, int y_layout, int64_t ldy, int split_k,
                         void* workspace, int64_t workspace_bytes, int flags, const lpqt_next_linear* next,
                         void* stream) {
  return lpqt_w6a16_linear_blocks(tiles, scales, 0, Xt, ldx, M, N, K, Y, y_dtype, y_layout, ldy, split_k, workspace,
                                  workspace_bytes, flags, next, stream);
}

static int w6a16_blocks_impl(const uint8_t* tiles, const uint16_t* scales, int64_t block, const uint16_t* Xt,
                             int64_t ldx, int64_t M, int64_t N, int64_t K, void* Y, int y_dtype, int y_layout,
                             int64_t ldy, int split_k, void* workspace, int64_t workspace_bytes, int flags,
                             const lpqt_next_linear* next, void* stream, const lpqt_peer_out* po) {
  if (flags & ~(LPQT_LAUNCH_PDL | LPQT_SCHED_STREAMK | LPQT_SCHED_CLUSTER | LPQT_SCHED_SINGLE | LPQT_SCHED_PAIR |
                LPQT_REBUILD_BIAS_SHIFT | LPQT_REBUILD_NAIVE | LPQT_WEIGHTS_FP5))
    return LPQT_E_INVALID_INPUT;
  const int rebuild = (flags & LPQT_REBUILD_BIAS_SHIFT) ? 1 : ((flags & LPQT_REBUILD_NAIVE) ? 2 : 0);
  const bool fp5 = (flags & LPQT_WEIGHTS_FP5) != 0;
  if (fp5 && (rebuild || po || (block > 0 && block < K))) return LPQT_E_UNSUPPORTED;
  if ((flags & LPQT_REBUILD_BIAS_SHIFT) && (flags & LPQT_REBUILD_NAIVE)) return LPQT_E_INVALID_INPUT;
  if (rebuild && (block > 0 && block < K)) return LPQT_E_UNSUPPORTED;
  if (rebuild && (po || M > 16)) return LPQT_E_UNSUPPORTED;
  // FGQ: blocks of B columns (B = K, or block <= 0: one scale per row)
  const bool fgq = block > 0 && block < K;
  // block scales at 128-k tile granularity (stage-ordered), or — decode widths
  // (M <= 32) — blocks of 16 / 32 / 64 columns with raw row-major scales
  const bool fgq_sub = fgq && block % kTileK != 0;
  if (fgq_sub && (block % 16 != 0 || kTileK % block != 0 || M > 32)) return LPQT_E_UNSUPPORTED;
  FgqArgs fga{};
  if (fgq_sub) {
    fga.scales = scales;
    fga.sub = static_cast<int>(kTileK / block);
    fga.bpr = static_cast<int>((K + block - 1) / block);
  } else if (fgq) {
    fga.stage = reinterpret_cast<const uint8_t*>(scales);  // stage-ordered (lpqt_fgq_stage_params)
  }
  if ((flags & LPQT_SCHED_STREAMK) && (flags & LPQT_SCHED_CLUSTER)) return LPQT_E_INVALID_INPUT;
  if (M < 0 || N < 0 || K < 0) return LPQT_E_SHAPE;
  if (M == 0 || N == 0) return LPQT_OK;
  if (K == 0) return LPQT_E_SHAPE;  // callers zero-fill (gemm.py:74-75)
  if (ldx < K || ldx % 8 != 0 || (reinterpret_cast<uintptr_t>(Xt) & 15)) return LPQT_E_SHAPE;
  if (y_dtype != LPQT_F32 && y_dtype != LPQT_F16 && y_dtype != LPQT_BF16) return LPQT_E_UNSUPPORTED;
  if (y_layout != LPQT_Y_NM && y_layout != LPQT_Y_MN) return LPQT_E_UNSUPPORTED;
  if (y_layout == LPQT_Y_NM ? ldy < M : ldy < N) return LPQT_E_SHAPE;
  if (split_k < 0) return LPQT_E_INVALID_INPUT;
  if (N > (int64_t)1 << 30 || M > (int64_t)1 << 30 || K > (int64_t)1 << 30) return LPQT_E_SHAPE;
  if (!fgq_sub && !po && pair_force(split_k, flags) >= 0 && use_pair_kernel(M, N, K, flags)) {
    const int st = launch_prefill_2sm(tiles, scales, Xt, ldx, M, N, K, Y, y_dtype, y_layout, ldy, flags,
                                      pair_force(split_k, flags), workspace, workspace_bytes, as_stream(stream),
                                      nullptr, fgq, fp5);
    if (st != LPQT_E_UNSUPPORTED) return st;
  }
  Plan p = make_plan(M, N, K, split_k, flags, num_sms(), fgq);
  if (p.ws_bytes > 0 && (workspace == nullptr || workspace_bytes < p.ws_bytes)) return LPQT_E_WORKSPACE;
  GemmArgs args{};
  L2Prefetch pfa{};
#ifdef LPQT_TRACE
  args.trace = trace_buffer() + (size_t)trace_next_slot() * kTraceLen;
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
  args.tile_count = static_cast<int>(p.tiles);
  // X larger than ~1/3 of L2 (126 MB): keep each batch tile's X resident
  args.n_fastest = (p.m_tiles > 1 && M * K * 2 > (int64_t)40 << 20) ? 1 : 0;
  args.dp = p.dp ? 1 : 0;
  args.y_dtype = y_dtype;
  args.y_layout = y_layout;
  args.sm = ShiftMuls{1u << 26, 1u << 28, 1u << 30};
  if (next && next->tiles && next->M > 0 && next->N > 0 && next->K > 0 && next->bytes_per_cta >= 0) {
    // the next launch's plan tells which bytes each of its CTAs needs first
    // (decode shapes: one batch tile, tile index = weight row tile)
    if ((next->flags & LPQT_SCHED_STREAMK) && (next->flags & LPQT_SCHED_CLUSTER)) return LPQT_E_INVALID_INPUT;
    const Plan q = make_plan(next->M, next->N, next->K, next->split_k, next->flags, num_sms());
    const int64_t chunk = next->bytes_per_cta > 0 ? next->bytes_per_cta : (int64_t)64 << 10;
    if (q.m_tiles == 1) {
      pfa.base = next->tiles;
      pfa.bytes = (int64_t)q.n_tiles * q.k_tiles * kTileBytes;
      pfa.count = q.grid;
      pfa.total = q.csk ? 0 : q.total;
      pfa.ksteps = q.ksteps;
      pfa.kstep = q.kstep;
      pfa.k_tiles = q.k_tiles;
      pfa.c = q.csk ? q.cluster : 1;
      pfa.tiles = static_cast<int>(q.tiles);
      pfa.chunk = static_cast<uint32_t>(std::min<int64_t>(chunk, (int64_t)1 << 30) / 16 * 16);
    }
  }
  cudaStream_t st = as_stream(stream);
  if (fp5) {
    pfa = L2Prefetch{};  // (the next linear's bytes are located by the FP6 tile size)
    return dispatch<false, 5>(p, args, pfa, fga, Xt, ldx, M, st, flags);
  }
  if (rebuild == 1) return dispatch_rebuild<1>(p, args, pfa, fga, Xt, ldx, M, st, flags);
  if (rebuild == 2) return dispatch_rebuild<2>(p, args, pfa, fga, Xt, ldx, M, st, flags);
  if (fgq_sub) {
    if (po) return LPQT_E_UNSUPPORTED;
    return dispatch<2, 6>(p, args, pfa, fga, Xt, ldx, M, st, flags);
  }
  if (po)
    return fgq ? dispatch<true, 6, true>(p, args, pfa, fga, Xt, ldx, M, st, flags, po)
               : dispatch<false, 6, true>(p, args, pfa, fga, Xt, ldx, M, st, flags, po);
  return fgq ? dispatch<true, 6>(p, args, pfa, fga, Xt, ldx, M, st, flags)
             : dispatch<false, 6>(p, args, pfa, fga, Xt, ldx, M, st, flags);
}

int lpqt_w6a16_linear_blocks(const uint8_t* tiles, const uint16_t* scales, int64_t block, const uint16_t* Xt,
                             int64_t ldx, int64_t M, int64_t N, int64_t K, void* Y, int y_dtype, int y_layout,
                             int64_t ldy, int split_k, void* workspace, int64_t workspace_bytes, int flags,
                             const lpqt_next_linear* next, void* stream) {
  return w6a16_blocks_impl(tiles, scales, block, Xt, ldx, M, N, K, Y, y_dtype, y_layout, ldy, split_k, workspace,
                           workspace_bytes, flags, next, stream, nullptr);
}

int lpqt_w6a16_linear_gather(const uint8_t* tiles, const uint16_t* scales, int64_t block, const uint16_t* Xt,
                             int64_t ldx, int64_t M, int64_t N, int64_t K, int y_dtype, int y_layout, int64_t ldy,
                             int split_k, void* workspace, int64_t workspace_bytes, int flags,
                             const lpqt_peer_out* peers, void* stream) {
  if (!peers || peers->npeers < 1 || peers->npeers > LPQT_MAX_PEERS || peers->rank < 0 ||
      peers->rank >= peers->npeers || peers->done == nullptr)
    return LPQT_E_INVALID_INPUT;
  for (int p = 0; p < peers->npeers; ++p)
    if (peers->y[p] == nullptr || peers->flags[p] == nullptr) return LPQT_E_INVALID_INPUT;
  if (M == 0 || N == 0) return LPQT_E_SHAPE;  // every rank must launch (the barrier counts CTAs)
  return w6a16_blocks_impl(tiles, scales, block, Xt, ldx, M, N, K, peers->y[peers->rank], y_dtype, y_layout, ldy,
                           split_k, workspace, workspace_bytes, flags, nullptr, stream, peers);
}


// W4A16 (the INT4 comparator): INT4 tiles (lpqt_int4_prepack),
// per-block f16 scales and zero points (block <= 0 or >= K: one per row; else
// a multiple of 128), the rebuilt binary16 weight = Z + S * level feeds the same
// tcgen05 pipeline (stream-K / round-robin schedules).
int lpqt_w4a16_linear_blocks(const uint8_t* tiles, const uint32_t* params, int64_t block,
                             const uint16_t* Xt, int64_t ldx, int64_t M, int64_t N, int64_t K, void* Y, int y_dtype,
                             int y_layout, int64_t ldy, int split_k, void* workspace, int64_t workspace_bytes,
                             int flags, void* stream) {
  // (W4A16 always runs the single-SM kernel: LPQT_SCHED_SINGLE is accepted as a
  // no-op; there is no CTA-pair W4A16 kernel, so LPQT_SCHED_PAIR is refused)
  flags &= ~LPQT_SCHED_SINGLE;
  if (flags & ~(LPQT_LAUNCH_PDL | LPQT_SCHED_STREAMK | LPQT_SCHED_CLUSTER)) return LPQT_E_INVALID_INPUT;
  if (M < 0 || N < 0 || K < 0) return LPQT_E_SHAPE;
  if (M == 0 || N == 0) return LPQT_OK;
  if (K == 0) return LPQT_E_SHAPE;
  if (ldx < K || ldx % 8 != 0 || (reinterpret_cast<uintptr_t>(Xt) & 15)) return LPQT_E_SHAPE;
  if (y_dtype != LPQT_F32 && y_dtype != LPQT_F16 && y_dtype != LPQT_BF16) return LPQT_E_UNSUPPORTED;
  if (y_layout != LPQT_Y_NM && y_layout != LPQT_Y_MN) return LPQT_E_UNSUPPORTED;
  if (y_layout == LPQT_Y_NM ? ldy < M : ldy < N) return LPQT_E_SHAPE;
  if (split_k < 0 || params == nullptr) return LPQT_E_INVALID_INPUT;
  if ((flags & LPQT_SCHED_STREAMK) && (flags & LPQT_SCHED_CLUSTER)) return LPQT_E_INVALID_INPUT;
  if (N > (int64_t)1 << 30 || M > (int64_t)1 << 30 || K > (int64_t)1 << 30) return LPQT_E_SHAPE;
  const bool per_row = block <= 0 || block >= K;
  if (!per_row && block % kTileK != 0) return LPQT_E_UNSUPPORTED;
  const Plan p = make_plan(M, N, K, split_k, flags, num_sms(), true);
  if (p.ws_bytes > 0 && (workspace == nullptr || workspace_bytes < p.ws_bytes)) return LPQT_E_WORKSPACE;
  FgqArgs fga{};
  fga.stage = reinterpret_cast<const uint8_t*>(params);
  GemmArgs args{};
  L2Prefetch pfa{};
#ifdef LPQT_TRACE
  args.trace = trace_buffer() + (size_t)trace_next_slot() * kTraceLen;
#endif
  args.tiles = tiles;
  args.scales = nullptr;
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
  args.tile_count = static_cast<int>(p.tiles);
  args.n_fastest = (p.m_tiles > 1 && M * K * 2 > (int64_t)40 << 20) ? 1 : 0;
  args.dp = p.dp ? 1 : 0;
  args.y_dtype = y_dtype;
  args.y_layout = y_layout;
  args.sm = ShiftMuls{1u << 26, 1u << 28, 1u << 30};
  return dispatch<true, 4>(p, args, pfa, fga, Xt, ldx, M, as_stream(stream), flags);
}

}  // extern "C"
