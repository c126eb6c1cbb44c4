// prefill2sm.cu — the W6A16 GEMM at prefill batch sizes on CTA PAIRS
// (tcgen05 cta_group::2), gemm.py:65-94 CGQ.
//
// Why a second kernel: at prefill the single-SM kernel (gemm.cu, BN 192) feeds
// each 768-cycle 128 x 192 x 128 MMA step with 48 KB of X from L2 and only
// three X stages fit next to the weight ring; measured 68 % tensor-pipe
// activity at M = 2048 with the dequant warps waiting on the MMA
// (profiles/r02_ncu_prefill_m2048.json).  A CTA pair runs M = 256 x N = 256
// MMAs: each SM still dequantizes ONE 128-row weight tile per 128-k step into
// its own TMEM (A operand, "TS" MMA), but loads only HALF of the 256 batch
// columns of X (its half of B); the pair's MMA reads both halves.  Per SM and
// k step: 1024 MMA cycles against ~600 dequant cycles and 32 KB of X + 12 KB
// of weights — X per MMA cycle is half the single-SM kernel's, and four X
// stages + six weight stages fit in shared memory.
//
// Work unit: 2 weight-row tiles (one per CTA: rank r owns row tile 2p + r)
// x bn batch columns x the whole K.  Unit u -> (pair, batch tile), in groups
// of a.group pairs with the pairs fastest inside a group, so the ~P units in
// flight share a few X tiles and a few weight pairs in L2 (at M = 8192 the
// pair-fastest order over all 224 gate_up pairs re-streamed every weight pair
// once per batch tile).  Schedule over the P co-resident pairs:
//  * whole units round-robin (cluster c takes u = c, c + P, ...) for the
//    first a.dp_units units (whole rounds);
//  * stream-K over the rest (a.sk == 1): the (unit, k-tile) space of the
//    last P .. 2P - 1 units is cut into P equal contiguous ranges, so the last
//    round's idle pairs are not wasted (70B QKV at M = 512: 80 units on 74
//    pairs = 2 rounds of whole units, 1.08 rounds with the stream-K wave).  A
//    unit cut between pairs is reduced by its head's pair (the first
//    contributor in k order: the head is the END of that pair's range, so it
//    is its last segment and every other share finishes no later); each other
//    contributor's share is the first segment of its range: it publishes its
//    fp32 partial (chunk-major 128 x bn per CTA) and counts in with one
//    red.release (no reply awaited).  The reducer bulk-copies the partials
//    into its (drained) X ring one at a time and sums in k order —
//    deterministic.  Workspace: self-resetting per-(unit, rank) counters +
//    one partial slot per pair.
//
// Roles per CTA (768 threads): warps 0-15 dequant (two groups of 8 on
// alternate k steps, warp w: lane group w % 4, k-half (w / 4) % 2), warp 16
// W producer (1-D bulk copy of the CTA's 12 KB weight tile per step), warp 17
// X producer (TMA of the CTA's 128 X rows, completing on the LEADER's
// barrier), warp 18 MMA issuer (leader CTA only: tcgen05.mma.cta_group::2,
// commits multicast to both CTAs), warps 20-23 epilogue (own 128 rows x 256
// columns of D from own TMEM, x row scale, Y).  Cross-CTA hand-offs: the
// follower's dequant and epilogue warps arrive on the leader's afull /
// dempty barriers (mapa + release.cluster); its X TMA completes on the
// leader's full_x; the MMA's commits reach both CTAs' empty_x / aempty /
// dfull (multicast::cluster).
#include <string.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <type_traits>

#include "common.cuh"

namespace lpqt {
namespace p2 {

constexpr int kMaxBN = 256;              // MMA N (batch columns of a unit): a.bn, a multiple of 32 <= 256
constexpr int kHalf = kMaxBN / 2;        // X rows each CTA loads at most
constexpr int kDqWarps = 16;
constexpr int kWarpW = 16, kWarpX = 17, kWarpMma = 18, kWarpEpi0 = 20;
constexpr int kThreads = 24 * 32;
constexpr int kXStage = kHalf * kTileK * 2;   // 32 KB: two SW128 boxes of 64 k x 128 rows
constexpr int kXStages = 4;
constexpr int kWStages = 6;                   // even: the two dequant groups alternate
constexpr int kASlots = 4;                    // 64 TMEM columns each (one 128 x 128 f16 tile)
constexpr int kAColsTile = kTileK / 2;
constexpr int kDCol0 = kASlots * kAColsTile;  // D: 256 fp32 columns after the A ring
constexpr int kTmemCols = 512;
constexpr int kYChunk = 32;                   // epilogue: 32 batch columns per TMA store
constexpr int kYBuf = kYChunk * kTileN * 2;   // 8 KB staging (16-bit Y), double-buffered
// a W stage: the weight tile + (FGQ) its 128 rows' f16 block scales, stage-ordered
// (lpqt_fgq_stage_params, as in gemm.cu)
constexpr int kSParams = kTileN * 2;
constexpr int kWStageFgq = kTileBytes + kSParams;
constexpr int kSmemBytes = kXStages * kXStage + kWStages * kWStageFgq + 2 * kYBuf +
                           8 * (2 * kXStages + 2 * kWStages + 2 * kASlots + 3) + 16;
static_assert(kSmemBytes <= 227 * 1024, "shared memory");
// stream-K: one partial slot per pair and CTA, 128 rows x kMaxBN fp32 (the
// reducer stages one in its X ring)
constexpr int kPartFloats = kTileN * kMaxBN;
static_assert(kPartFloats * 4 <= kXStages * kXStage, "a partial must fit the X ring");
constexpr int64_t kCounters = 65536;  // per (unit, rank); the region gemm.cu's stream-K uses too

struct Args {
  const uint8_t* tiles;
  const uint16_t* scales;
  void* y;
  int64_t ldy;
  int M, N, k_tiles, n_tiles, m_tiles, units, n_fastest, y_dtype, y_layout;
  int bn;     // batch columns per unit (MMA N; each CTA loads bn / 2 X rows)
  int y_tma;  // 0: element stores; 1: Y[M, N] / 2: Y[N, M] staged in 8-KB chunks, TMA-stored
  int group;  // pairs per rasterization group
  int sk;     // stream-K wave over the units past dp_units
  int dp_units;    // units run whole, round-robin (a multiple of the pair count when sk)
  int64_t total;   // sk: (units - dp_units) * k_tiles
  int* counters;   // sk: [units][2] k-tiles published (self-resetting)
  float* partials; // sk: [pairs][2][kPartFloats], chunk-major float4 [bn / 4][128]
  ShiftMuls sm;
};
// FGQ block parameters: a separate kernel parameter (growing Args perturbs the
// register allocation: 24 -> 64 bytes of spills in the CGQ kernel, measured)
struct FgqP {
  const uint8_t* stage;  // stage-ordered block scales (lpqt_fgq_stage_params)
  const float* rowf;     // per-row power-of-two factors (after the stage-ordered scales)
};

// A pair's walk over its work, step i -> unit u, k tile kt: whole units
// c, c + P, ... for its first dp_n steps, then its stream-K range (from sk0)
struct Walk {
  int u, kt, i;
  __device__ __forceinline__ void set(const Args& a, int cid, int ncl, int64_t sk0, int dp_n) {
    if (i < dp_n) {
      const int ul = i / a.k_tiles;
      u = cid + ul * ncl;
      kt = i - ul * a.k_tiles;
    } else {
      const int64_t q = sk0 + (i - dp_n);
      const int64_t us = q / a.k_tiles;
      u = a.dp_units + static_cast<int>(us);
      kt = static_cast<int>(q - us * a.k_tiles);
    }
  }
  __device__ __forceinline__ void start(const Args& a, int cid, int ncl, int64_t sk0, int dp_n) {
    i = 0;
    set(a, cid, ncl, sk0, dp_n);
  }
  __device__ __forceinline__ void adv(const Args& a, int cid, int ncl, int64_t sk0, int dp_n) {
    if (++i == dp_n) {
      set(a, cid, ncl, sk0, dp_n);  // into the stream-K range
    } else if (++kt == a.k_tiles) {
      kt = 0;
      u += i < dp_n ? ncl : 1;
    }
  }
};
__device__ __forceinline__ int64_t sk_beg(const Args& a, int c, int ncl) { return (int64_t)c * a.total / ncl; }
// pair whose stream-K range holds position q
__device__ __forceinline__ int sk_pair_of(const Args& a, int64_t q, int ncl) {
  return static_cast<int>(((q + 1) * (int64_t)ncl - 1) / a.total);
}
__device__ __forceinline__ void red_release_gpu(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// arrive on a barrier of either CTA of the pair.  Default (release.cta)
// semantics: what the consumer needs ordered is TMEM (tcgen05.wait::st /
// wait::ld + tcgen05.fence::before_thread_sync precede the arrive), not
// generic memory; a release.cluster arrive costs a MEMBAR per call — measured
// 44 % of the dequant warps' stall samples (profiles/r02_ncu_pair_m2048.json).
__device__ __forceinline__ void arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ bool try_wait_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(LPQT_WAIT_HINT_NS)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void wait_cluster(uint32_t addr, uint32_t parity) {
  // (watchdog per round of polls, as mbar_wait_u32: a pipeline bug fails the launch instead of hanging)
  for (uint32_t rounds = 0;; ++rounds) {
#pragma unroll
    for (int j = 0; j < LPQT_WATCHDOG_POLLS; ++j)
      if (try_wait_cluster(addr, parity)) return;
    if (rounds == (1u << 28) / LPQT_WATCHDOG_POLLS) __trap();
  }
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// X half of this CTA into its own smem; completion counted on the leader's barrier
__device__ __forceinline__ void tma_x_2sm(uint32_t pred, uint32_t dst, const CUtensorMap* map, uint32_t mbar_cluster,
                                          int c0, int c1) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "@e cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%2, {%4, "
      "%5}], [%3];\n\t}" ::"r"(pred),
      "r"(dst), "l"(map), "r"(mbar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mma_2sm(uint32_t pred, uint32_t d_tmem, uint32_t a_tmem, uint32_t b_lo, uint32_t b_hi,
                                        uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 bd;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "mov.b64 bd, {%3, %4};\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%1], [%2], bd, %5, p;\n\t}" ::"r"(pred),
      "r"(d_tmem), "r"(a_tmem), "r"(b_lo), "r"(b_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void commit_2sm(uint32_t pred, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%1], %2;\n\t}" ::"r"(
          pred),
      "r"(smem_u32(bar)), "h"(static_cast<uint16_t>(3))
      : "memory");
}

// unit u of this cluster's sequence -> (pair, batch tile)
__device__ __forceinline__ void unit_nm(const Args& a, int u, int& pair, int& mt) {
  const int n_pairs = a.n_tiles / 2;
  if (a.n_fastest) {
    // groups of a.group pairs x all batch tiles, the group's pairs fastest
    const int gsz = a.group * a.m_tiles;
    const int g = u / gsz, r = u - g * gsz;
    const int gp = min(a.group, n_pairs - g * a.group);  // (the last group may be narrower)
    mt = r / gp;
    pair = g * a.group + (r - mt * gp);
  } else {
    pair = u / a.m_tiles;
    mt = u - pair * a.m_tiles;
  }
}

__device__ __forceinline__ void store_y(const Args& a, int n, int m, float v) {
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

// FGQ: blocks of whole 128-k tiles (stage-ordered block scales applied to the
// rebuilt binary16 weight); a separate instantiation so the CGQ code is unchanged
// WB: 6 = FP6 tiles (12 KB), 5 = native FP5 tiles (10 KB, common.cuh; CGQ)
template <bool FGQ, int WB = 6>
__global__ void __launch_bounds__(kThreads, 1)
    w6a16_prefill_2sm_kernel(const __grid_constant__ CUtensorMap tmap_x, const __grid_constant__ CUtensorMap tmap_y,
                             const Args a, const FgqP fq) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem_x = smem_raw;
  uint8_t* smem_w = smem_x + kXStages * kXStage;
  static_assert(WB == 6 || !FGQ, "FGQ FP5 streams the FP6-widened tiles");
  constexpr int kTileB = WB == 6 ? kTileBytes : kTileBytes5;
  constexpr int kWStage = FGQ ? kWStageFgq : kTileB;  // (CGQ keeps the tile stride)
  uint8_t* smem_y = smem_w + kWStages * kWStage;
  uint64_t* full_x = reinterpret_cast<uint64_t*>(smem_y + 2 * kYBuf);
  uint64_t* empty_x = full_x + kXStages;
  uint64_t* full_w = empty_x + kXStages;
  uint64_t* empty_w = full_w + kWStages;
  uint64_t* afull = empty_w + kWStages;
  uint64_t* aempty = afull + kASlots;
  uint64_t* dfull = aempty + kASlots;
  uint64_t* dempty = dfull + 1;
  uint64_t* fixb = dempty + 1;  // sk reducer: a partial landed in the X ring
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(fixb + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cta_rank();
  const bool leader = rank == 0;
  const int cid = static_cast<int>(blockIdx.x) >> 1, ncl = static_cast<int>(gridDim.x) >> 1;
  // whole units first (dp_n steps), then the stream-K range [beg, beg + n_st - dp_n)
  const int my_units = cid < a.dp_units ? (a.dp_units - 1 - cid) / ncl + 1 : 0;
  const int dp_n = my_units * a.k_tiles;
  int64_t beg = 0;
  int n_st = dp_n;
  if (a.sk) {
    beg = sk_beg(a, cid, ncl);
    n_st += static_cast<int>(sk_beg(a, cid + 1, ncl) - beg);
  }

  if (threadIdx.x == 0) {
    if (smem_u32(smem_raw) & 1023u) __trap();
    for (int s = 0; s < kXStages; ++s) {
      mbar_init(&full_x[s], 1);   // leader: its expect_tx arrival (+ both halves' bytes)
      mbar_init(&empty_x[s], 1);  // MMA commit (multicast)
    }
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(&full_w[s], 1);
      mbar_init(&empty_w[s], kDqWarps / 2);  // the dequant group owning the slot
    }
    for (int b = 0; b < kASlots; ++b) {
      mbar_init(&afull[b], 2 * (kDqWarps / 2));  // leader: both CTAs' dequant group
      mbar_init(&aempty[b], 1);                  // MMA commit (multicast)
    }
    mbar_init(dfull, 1);
    mbar_init(dempty, 2 * 4);  // leader: both CTAs' epilogue warps
    mbar_init(fixb, 1);
    fence_mbar_init();
  }
  if (warp == kWarpMma) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (warp == kWarpX && lane == 0) prefetch_tmap(&tmap_x);
  tc_fence_before();
  cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  pdl_launch_dependents();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == kWarpW || warp == kWarpX || warp == kWarpMma || warp == kWarpMma + 1) {
    setmaxnreg_dec<48>();
    if (warp == kWarpW) {
      // ------------------------------------------------ W producer (own row tile)
      const uint64_t pol = l2_evict_last_policy();  // a weight tile is re-read once per batch tile
      Walk w;
      w.start(a, cid, ncl, beg, dp_n);
      for (int i = 0; i < n_st; ++i, w.adv(a, cid, ncl, beg, dp_n)) {
        int pair, mt;
        unit_nm(a, w.u, pair, mt);
        const int s = i % kWStages;
        mbar_wait<2>(&empty_w[s], ((i / kWStages) & 1) ^ 1);
        const uint32_t e = elect_one();
        mbar_arrive_expect_tx_if(e, &full_w[s], kTileB + (FGQ ? kSParams : 0));
        if constexpr (FGQ)
          bulk_g2s_if(e, smem_w + s * kWStage + kTileBytes,
                      fq.stage + ((int64_t)(2 * pair + rank) * a.k_tiles + w.kt) * kSParams, kSParams, &full_w[s], pol);
        bulk_g2s_if(e, smem_w + s * kWStage,
                    a.tiles + ((int64_t)(2 * pair + rank) * a.k_tiles + w.kt) * kTileB, kTileB, &full_w[s], pol);
      }
    } else if (warp == kWarpX) {
      // ------------------------------------------------ X producer (own half of the batch tile)
      pdl_wait();  // X is the preceding kernel's output
      const uint32_t fx_leader = mapa(smem_u32(full_x), 0);
      Walk w;
      w.start(a, cid, ncl, beg, dp_n);
      for (int i = 0; i < n_st; ++i, w.adv(a, cid, ncl, beg, dp_n)) {
        const int kt = w.kt;
        int pair, mt;
        unit_nm(a, w.u, pair, mt);
        const int s = i % kXStages;
        mbar_wait<2>(&empty_x[s], ((i / kXStages) & 1) ^ 1);
        const uint32_t e = elect_one();
        const int half = a.bn >> 1;
        if (leader) mbar_arrive_expect_tx_if(e, &full_x[s], static_cast<uint32_t>(a.bn * kTileK * 2));
        const uint32_t dst = smem_u32(smem_x + s * kXStage);
        const int row = mt * a.bn + static_cast<int>(rank) * half;
        tma_x_2sm(e, dst, &tmap_x, fx_leader + 8 * s, kt * kTileK, row);
        tma_x_2sm(e, dst + half * 128, &tmap_x, fx_leader + 8 * s, kt * kTileK + 64, row);
      }
    } else if (warp == kWarpMma && leader) {
      // ------------------------------------------------ MMA issuer (leader only)
      const uint32_t idesc = (1u << 4) | (static_cast<uint32_t>(a.bn >> 3) << 17) |
                             (static_cast<uint32_t>(256 >> 4) << 24);
      const int half = a.bn >> 1;
      const uint32_t d_tmem = tmem_base + kDCol0;
      const uint32_t ae_bar = smem_u32(afull), dm_bar = smem_u32(dempty), fx_bar = smem_u32(full_x);
      // a segment = one unit's contiguous k range: fresh accumulator at its
      // first step, dfull committed after its last
      Walk w;
      w.start(a, cid, ncl, beg, dp_n);
      int seg = 0;
      for (int i = 0; i < n_st; ++i, w.adv(a, cid, ncl, beg, dp_n)) {
        const bool s0 = i == 0 || i == dp_n || w.kt == 0;
        if (s0) {
          wait_cluster(dm_bar, (seg & 1) ^ 1);  // both CTAs drained D
          tc_fence_after();
        }
        const int xs = i % kXStages, sl = i % kASlots;
        wait_cluster(fx_bar + 8 * xs, (i / kXStages) & 1);     // both X halves landed
        wait_cluster(ae_bar + 8 * sl, (i / kASlots) & 1);      // both A tiles rebuilt
        tc_fence_after();
        const uint32_t e = elect_one();
        const uint64_t bd0 = sdesc_kmajor_sw128(smem_u32(smem_x + xs * kXStage));
        const uint32_t bd_lo = static_cast<uint32_t>(bd0), bd_hi = static_cast<uint32_t>(bd0 >> 32);
        const uint32_t ta = tmem_base + sl * kAColsTile;
#pragma unroll
        for (int j = 0; j < kTileK / 16; ++j) {
          const uint32_t off = ((j >> 2) * (half * 128) + (j & 3) * 32) >> 4;
          mma_2sm(e, d_tmem, ta + j * 8, bd_lo + off, bd_hi, idesc, (s0 && j == 0) ? 0u : 1u);
        }
        commit_2sm(e, &empty_x[xs]);
        commit_2sm(e, &aempty[sl]);
        if (i + 1 == n_st || i + 1 == dp_n || w.kt + 1 == a.k_tiles) {
          commit_2sm(elect_one(), dfull);
          ++seg;
        }
      }
    }
  } else if (warp < kDqWarps) {
    // ------------------------------------------------ dequant (own row tile -> own TMEM A)
    setmaxnreg_inc<88>();
    const int lg = warp & 3, grp = warp >> 3, tl = (warp >> 2) & 1;
    const int row = lg * 32 + lane;
    const uint32_t w_src = smem_u32(smem_w) + static_cast<uint32_t>(row * 16 + tl * 3 * kTileN * 16);
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + static_cast<uint32_t>(tl * 32);
    const uint32_t af_leader = mapa(smem_u32(afull), 0);
    const ShiftMuls sm = a.sm;
    uint32_t q[12];
    uint32_t fs2 = 0;  // FGQ: this row's block scale (binary16 x2) of the stage's tile
    auto load = [&](int i) {
      const int s = i % kWStages;
      mbar_wait<2>(&full_w[s], (i / kWStages) & 1);
      if constexpr (FGQ) fs2 = __byte_perm(lds_u16(smem_u32(smem_w) + kTileBytes + row * 2 + s * kWStage), 0u, 0x1010);
      if constexpr (WB == 5) {  // k-half tl: nibble quads [tl][grp 0, 1][row], mantissa words [tl][row][2]
        const uint32_t base = smem_u32(smem_w) + s * kWStage;
        const uint32_t nsrc = base + static_cast<uint32_t>((tl * 2 * kTileN + row) * 16);
        const uint4 v0 = lds128_u32(nsrc), v1 = lds128_u32(nsrc + kTileN * 16);
        const uint2 mv = lds64_u32(base + kTile5Nib + static_cast<uint32_t>((tl * kTileN + row) * 8));
        q[0] = v0.x; q[1] = v0.y; q[2] = v0.z; q[3] = v0.w; q[4] = v1.x; q[5] = v1.y;
        q[6] = v1.z; q[7] = v1.w; q[8] = mv.x; q[9] = mv.y;
        return;
      }
      const uint32_t src = w_src + s * kWStage;
      const uint4 v0 = lds128_u32(src), v1 = lds128_u32(src + kTileN * 16), v2 = lds128_u32(src + 2 * kTileN * 16);
      q[0] = v0.x; q[1] = v0.y; q[2] = v0.z; q[3] = v0.w; q[4] = v1.x; q[5] = v1.y;
      q[6] = v1.z; q[7] = v1.w; q[8] = v2.x; q[9] = v2.y; q[10] = v2.z; q[11] = v2.w;
    };
    if (grp < n_st) load(grp);
    for (int i = grp; i < n_st; i += 2) {
      uint32_t r[32];
      if constexpr (WB == 5) {
        fp5x32_cvt_f16x32(q, q[8], r, sm);
        fp5x32_cvt_f16x32(q + 4, q[9], r + 16, sm);
      } else {
        fp6x32_cvt_f16x32_fma(q, r, sm);
        fp6x32_cvt_f16x32_fma(q + 6, r + 16, sm);
      }
      if constexpr (FGQ) {  // FGQ: v * S'_b in binary16 (per-row power-of-two normalised scales, as gemm.cu BN >= 64)
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const __half2 v = __hmul2(*reinterpret_cast<const __half2*>(&r[j]), *reinterpret_cast<const __half2*>(&fs2));
          r[j] = *reinterpret_cast<const uint32_t*>(&v);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_w[i % kWStages]);  // words consumed
      const int sl = i % kASlots;
      mbar_wait<2>(&aempty[sl], ((i / kASlots) & 1) ^ 1);
      tc_fence_after();
      tmem_st_x32(t_lane + sl * kAColsTile, r);
      if (i + 2 < n_st) load(i + 2);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) arrive_cluster(af_leader + 8 * sl);
    }
  } else {
    // ------------------------------------------------ epilogue (own 128 rows x bn columns)
    // (keeps the launch's 80 registers: setmaxnreg moves registers only inside the
    // CTA's allocation, 768 x 80, and the producers' 4 x 32 x 32 released by the
    // decrement above are exactly what the dequant warps' increment to 88 takes —
    // an increment here would wait forever)
    const int lg = warp & 3;
    const int rr = lg * 32 + lane;
    const uint32_t t_d = tmem_base + kDCol0 + (static_cast<uint32_t>(lg * 32) << 16);
    const uint32_t dm_leader = mapa(smem_u32(dempty), 0);
    const bool lead_thread = warp == kWarpEpi0 && lane == 0;
    int nchunk = 0;  // TMA-stored chunks so far (staging buffer = nchunk & 1)
    uint32_t fph = 0;  // fixb phase
    pdl_wait();      // Y / workspace writes: the preceding grid must be complete
    Walk w;
    w.start(a, cid, ncl, beg, dp_n);
    for (int seg = 0; w.i < n_st; ++seg) {
      const int u = w.u, kt0 = w.kt;
      const int len = min(a.k_tiles - kt0, n_st - w.i);
      w.i += len;
      w.set(a, cid, ncl, beg, dp_n);
      int pair, mt;
      unit_nm(a, u, pair, mt);
      const int n0 = (2 * pair + static_cast<int>(rank)) * kTileN, n = n0 + rr;
      // CGQ: the row scale; FGQ: the row's power-of-two factor (the block scales are in A)
      float fs;
      if constexpr (FGQ) {
        fs = n < a.N ? __ldg(fq.rowf + n) : 0.f;
      } else {
        fs = n < a.N ? __half2float(__ushort_as_half(__ldg(a.scales + n))) : 0.f;
      }
      mbar_wait<2>(dfull, seg & 1);
      tc_fence_after();
      auto d_drained = [&]() {  // D may be overwritten by the next segment's MMAs
        tc_fence_before();
        __syncwarp();
        if (lane == 0) arrive_cluster(dm_leader);
      };
      // one chunk of CW batch columns of fp32 sums -> x row scale -> Y (8 KB
      // staged: CW = 32 for 16-bit Y, 16 for f32)
      auto emit = [&](auto cw_tag, int c0, const uint32_t* v) {
        constexpr int CW = decltype(cw_tag)::value;
        const int m0 = mt * a.bn + c0;
        if (!a.y_tma) {
#pragma unroll
          for (int j = 0; j < CW; ++j) store_y(a, n, m0 + j, __uint_as_float(v[j]) * fs);
          return;
        }
        // staged chunk -> one TMA tensor store (clips m >= M, n >= N).  Y[M, N]: smem
        // [CW m][128 n] (thread rr writes column rr); Y[N, M]: smem [128 n][CW m]
        // (thread rr writes its 64-byte row with four 16-byte stores)
        const uint32_t buf = smem_u32(smem_y) + (nchunk & 1) * kYBuf;
        if (nchunk >= 2) {
          if (lead_thread) bulk_wait_read<1>();  // this buffer's previous store has read it
          named_bar_sync(1, 4 * 32);
        }
        uint32_t h[16];  // the chunk's 64 bytes of this row, packed
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if constexpr (CW == 16) {
            h[j] = __float_as_uint(__uint_as_float(v[j]) * fs);
          } else {
            const float f0 = __uint_as_float(v[2 * j]) * fs, f1 = __uint_as_float(v[2 * j + 1]) * fs;
            if (a.y_dtype == LPQT_F16) {
              const __half2 t = __floats2half2_rn(f0, f1);
              h[j] = *reinterpret_cast<const uint32_t*>(&t);
            } else {
              const __nv_bfloat162 t = __floats2bfloat162_rn(f0, f1);
              h[j] = *reinterpret_cast<const uint32_t*>(&t);
            }
          }
        }
        if (a.y_tma == 1) {
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            if constexpr (CW == 16) {
              asm volatile("st.shared.b32 [%0], %1;" ::"r"(buf + (j * kTileN + rr) * 4), "r"(h[j]) : "memory");
            } else {
              asm volatile("st.shared.u16 [%0], %1;" ::"r"(buf + (j * kTileN + rr) * 2),
                           "h"(static_cast<uint16_t>(h[j >> 1] >> (16 * (j & 1))))
                           : "memory");
            }
          }
        } else {
#pragma unroll
          for (int j = 0; j < 16; j += 4)
            asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(buf + rr * 64 + j * 4), "r"(h[j]),
                         "r"(h[j + 1]), "r"(h[j + 2]), "r"(h[j + 3])
                         : "memory");
        }
        fence_proxy_async_smem();
        named_bar_sync(1, 4 * 32);
        if (lead_thread) {
          if (a.y_tma == 1) {
            tma_store_2d(&tmap_y, buf, n0, m0);
          } else {
            tma_store_2d(&tmap_y, buf, m0, n0);
          }
          bulk_commit();
        }
        ++nchunk;
      };
      // D columns [c0, c0 + CW) of this thread's row
      auto load_d = [&](auto cw_tag, int c0, uint32_t* v) {
        constexpr int CW = decltype(cw_tag)::value;
        tmem_ld_x16(t_d + c0, *reinterpret_cast<uint32_t(*)[16]>(v));
        if constexpr (CW == 32) tmem_ld_x16(t_d + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
        tmem_wait_ld();
      };
      auto each_chunk = [&](auto&& body) {
        if (a.y_dtype == LPQT_F32) {
#pragma unroll 1
          for (int c0 = 0; c0 < a.bn; c0 += 16) body(std::integral_constant<int, 16>{}, c0);
        } else {
#pragma unroll 1
          for (int c0 = 0; c0 < a.bn; c0 += 32) body(std::integral_constant<int, 32>{}, c0);
        }
      };
      if (kt0 == 0 && len == a.k_tiles) {
        // ---- whole unit
        each_chunk([&](auto tag, int c0) {
          uint32_t v[decltype(tag)::value];
          load_d(tag, c0, v);
          if (c0 + decltype(tag)::value >= a.bn) d_drained();
          emit(tag, c0, v);
        });
      } else if (kt0 > 0) {
        // ---- stream-K share (this pair's first segment): publish the fp32
        // partial, count in, move on
        float4* part = reinterpret_cast<float4*>(a.partials + ((int64_t)cid * 2 + rank) * kPartFloats) + rr;
#pragma unroll 1
        for (int c0 = 0; c0 < a.bn; c0 += 16) {
          uint32_t v[16];
          load_d(std::integral_constant<int, 16>{}, c0, v);
          if (c0 + 16 >= a.bn) d_drained();
#pragma unroll
          for (int j = 0; j < 4; ++j)
            __stcg(part + (c0 / 4 + j) * kTileN, make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                                                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3])));
        }
        // CTA barrier (cumulativity over the epilogue's stores), then one
        // gpu-scope release reduction
        named_bar_sync(1, 4 * 32);
        if (lead_thread) red_release_gpu(&a.counters[2 * u + rank], len);
      } else {
        // ---- stream-K head (this pair's last segment): wait for the other
        // contributors, then own + p(cid + 1) + p(cid + 2) + ... in k order
        const int c_last = sk_pair_of(a, (int64_t)(u - a.dp_units) * a.k_tiles + a.k_tiles - 1, ncl);
        if (lead_thread) {
          const int others = a.k_tiles - len;
          for (uint32_t spin = 0; ld_acquire(&a.counters[2 * u + rank]) != others; ++spin) {
            if (spin > (1u << 26)) __trap();  // a contributor never published: fail loudly
            __nanosleep(64);
          }
        }
        const uint32_t pbytes = static_cast<uint32_t>(kTileN * a.bn * 4);
        const uint32_t sbase = smem_u32(smem_x) + rr * 16;
#pragma unroll 1
        for (int c = cid + 1; c <= c_last; ++c) {
          // the X ring is drained (every MMA of this last segment completed)
          if (lead_thread) {
            fence_proxy_async_global();  // acquired generic-proxy partials -> bulk-copy reads
            mbar_arrive_expect_tx(fixb, pbytes);
            bulk_g2s_plain(smem_x, a.partials + ((int64_t)c * 2 + rank) * kPartFloats, pbytes, fixb);
          }
          mbar_wait<2>(fixb, fph);
          fph ^= 1u;
          const bool last = c == c_last;
          each_chunk([&](auto tag, int c0) {
            constexpr int CW = decltype(tag)::value;
            uint32_t v[CW];
            load_d(tag, c0, v);
#pragma unroll
            for (int j = 0; j < CW / 4; ++j) {
              const float4 p = lds128_f32(sbase + (c0 / 4 + j) * kTileN * 16);
              v[4 * j + 0] = __float_as_uint(__uint_as_float(v[4 * j + 0]) + p.x);
              v[4 * j + 1] = __float_as_uint(__uint_as_float(v[4 * j + 1]) + p.y);
              v[4 * j + 2] = __float_as_uint(__uint_as_float(v[4 * j + 2]) + p.z);
              v[4 * j + 3] = __float_as_uint(__uint_as_float(v[4 * j + 3]) + p.w);
            }
            if (last) {
              if (c0 + CW >= a.bn) d_drained();
              emit(tag, c0, v);
            } else {  // running sum back into D
              tmem_st_x16(t_d + c0, *reinterpret_cast<uint32_t(*)[16]>(v));
              if constexpr (CW == 32) tmem_st_x16(t_d + c0 + 16, *reinterpret_cast<uint32_t(*)[16]>(v + 16));
            }
          });
          tmem_wait_st();
          named_bar_sync(1, 4 * 32);  // every thread is done with the staged partial
        }
        if (lead_thread) a.counters[2 * u + rank] = 0;  // every partial is read: re-arm
      }
    }
    if (lead_thread) bulk_wait_read<0>();  // staging smem stays valid until the stores read it
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers / read its TMEM
  if (warp == kWarpMma) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols) : "memory");
  }
}

}  // namespace p2

typedef CUresult (*EncodeTiledFn2)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn2 encode_fn_2sm() {
  static EncodeTiledFn2 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn2>(p);
  });
  return fn;
}

// Co-resident CTA pairs (GPC packing); queried once.
static int max_pairs() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int v = 0;
    if (cudaFuncSetAttribute(p2::w6a16_prefill_2sm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             p2::kSmemBytes) == cudaSuccess) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(2 * 64);
      cfg.blockDim = dim3(p2::kThreads);
      cfg.dynamicSmemBytes = p2::kSmemBytes;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaOccupancyMaxActiveClusters(&v, p2::w6a16_prefill_2sm_kernel<false>, &cfg) != cudaSuccess) v = 0;
    }
    cudaGetLastError();
    n = v > 0 ? v : 74;
  });
  return n;
}

int prefill_2sm_pairs() { return max_pairs(); }

// Unit width and schedule: the batch columns bn (a multiple of 32, <= 256) and
// whole units vs whole rounds + a stream-K wave that minimise the per-pair
// cycle estimate.  A k step costs max(4 bn, ~700) cycles (MMA floor M = 256
// across the pair: bn / 2 cycles per K = 16; the dequant of one 128 x 128
// tile by 16 warps: ~600 + barrier overhead) and a segment's epilogue drain
// ~32 bn.  Whole units: ceil(units / P) rounds.  Hybrid: floor(units / P) - 1
// whole rounds, then the last P + units % P units as stream-K (units * k_tiles
// / P steps per pair, each unit cut in at most a few pieces) plus a fixup
// (the publisher's partial store and the reducer's gather, ~2 drains).
// Returns the estimated cycles per SM.
// force: 0 = by the estimate, 1 = whole units only, 2 = whole rounds + stream-K wave
static double choose(int64_t M, int64_t N, int64_t K, int* bn_out, int* dp_units_out, int force = 0) {
  const int64_t n_pairs = (N + kTileN - 1) / kTileN / 2;
  const int64_t k_tiles = (K + kTileK - 1) / kTileK;
  const int64_t pairs = max_pairs();
  double best = 1e30;
  int best_bn = 256;
  int64_t best_dp = -1;  // -1: whole units only
  for (int bn = 256; bn >= 128; bn -= 32) {
    const int64_t units = n_pairs * ((M + bn - 1) / bn);
    const int64_t rounds = (units + pairs - 1) / pairs;
    const double step = std::max(4.0 * bn, 700.0), drain = 4.0 * bn * 8;
    const double t_dp = (double)rounds * (k_tiles * step + drain);
    if (force != 2 && t_dp < best * 0.98) {
      best = t_dp;
      best_bn = bn;
      best_dp = -1;
    }
    if (force == 1 || (force == 0 && units % pairs == 0) || 2 * units > p2::kCounters) continue;
    const int64_t dp_rounds = units / pairs > 0 ? units / pairs - 1 : 0;
    const int64_t sk_units = units - dp_rounds * pairs;
    const double per = (double)sk_units * k_tiles / pairs;
    if (force == 0 && per < 8.0) continue;  // (every pair streams >= 8 k steps, else the fixups dominate)
    const double t_sk = dp_rounds * (k_tiles * step + drain) + per * step + (per / k_tiles + 1.0) * drain + 2.0 * drain;
    if (t_sk < best * 0.98) {
      best = t_sk;
      best_bn = bn;
      best_dp = dp_rounds * pairs;
    }
  }
  if (bn_out) *bn_out = best_bn;
  if (dp_units_out) *dp_units_out = static_cast<int>(best_dp);
  return best;
}

double prefill_2sm_choose(int64_t M, int64_t N, int64_t K, int* bn_out, int* sk_out, int force) {
  int dp = -1;
  const double t = choose(M, N, K, bn_out, &dp, force);
  if (sk_out) *sk_out = dp >= 0;
  return t;
}

// Workspace of the stream-K schedule: the counters region (shared with
// gemm.cu's stream-K, self-resetting) + one partial slot per pair and CTA.
int64_t prefill_2sm_workspace() { return p2::kCounters * 4 + (int64_t)max_pairs() * 2 * p2::kPartFloats * 4; }

// Host launch of the pair kernel (called from gemm.cu's dispatcher; CGQ FP6,
// even number of 128-row weight tiles).  Returns LPQT_E_UNSUPPORTED when the
// shape does not fit (the caller then uses the single-SM kernel).
// scales: the f16 row scales (CGQ) or, with fgq, the stage-ordered block scales +
// row factors of lpqt_fgq_stage_params (blocks of whole 128-k tiles)
int launch_prefill_2sm(const uint8_t* tiles, const uint16_t* scales, const uint16_t* Xt, int64_t ldx, int64_t M,
                       int64_t N, int64_t K, void* Y, int y_dtype, int y_layout, int64_t ldy, int flags,
                       int force, void* workspace, int64_t workspace_bytes, cudaStream_t stream, int* grid_out,
                       bool fgq, bool fp5) {
  const int n_tiles = static_cast<int>((N + kTileN - 1) / kTileN);
  if (n_tiles % 2 != 0) return LPQT_E_UNSUPPORTED;
  EncodeTiledFn2 enc = encode_fn_2sm();
  if (!enc) return LPQT_E_CUDA;
  int bn = 256, dp_units = -1;
  choose(M, N, K, &bn, &dp_units, force);
  const int sk = dp_units >= 0;
  if (sk && (workspace == nullptr || workspace_bytes < prefill_2sm_workspace())) return LPQT_E_WORKSPACE;
  CUtensorMap map;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(K), static_cast<cuuint64_t>(M)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ldx) * 2};
  const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(bn / 2)};
  const cuuint32_t estr[2] = {1, 1};
  if (enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<uint16_t*>(Xt), dims, strides, box, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return LPQT_E_INVALID_INPUT;
  // Y with a 16-B aligned base and row stride: the TMA-store epilogue (8-KB chunks:
  // 32 batch columns of 16-bit Y or 16 of f32), Y[M, N] or Y[N, M]
  CUtensorMap ymap;
  memset(&ymap, 0, sizeof(ymap));
  int y_tma = 0;
  const int es = y_dtype == LPQT_F32 ? 4 : 2;
  const cuuint32_t cw = static_cast<cuuint32_t>(p2::kYBuf / (kTileN * es));
  if (reinterpret_cast<uintptr_t>(Y) % 16 == 0 && (ldy * es) % 16 == 0) {
    const bool mn = y_layout == LPQT_Y_MN;
    const cuuint64_t ydims[2] = {static_cast<cuuint64_t>(mn ? N : M), static_cast<cuuint64_t>(mn ? M : N)};
    const cuuint64_t ystr[1] = {static_cast<cuuint64_t>(ldy) * es};
    const cuuint32_t ybox[2] = {mn ? static_cast<cuuint32_t>(kTileN) : cw, mn ? cw : static_cast<cuuint32_t>(kTileN)};
    const CUtensorMapDataType dt = y_dtype == LPQT_F32   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                   : y_dtype == LPQT_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                         : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    if (enc(&ymap, dt, 2, Y, ydims, ystr, ybox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS)
      y_tma = mn ? 1 : 2;
  }
  p2::Args a{};
  a.tiles = tiles;
  a.scales = scales;
  p2::FgqP fq{};
  if (fgq) {
    fq.stage = reinterpret_cast<const uint8_t*>(scales);
    fq.rowf = reinterpret_cast<const float*>(fq.stage + (int64_t)n_tiles * kTileN * ((K + kTileK - 1) / kTileK) * 2);
  }
  a.y = Y;
  a.ldy = ldy;
  a.M = static_cast<int>(M);
  a.N = static_cast<int>(N);
  a.k_tiles = static_cast<int>((K + kTileK - 1) / kTileK);
  a.n_tiles = n_tiles;
  a.bn = bn;
  a.y_tma = y_tma;
  a.m_tiles = static_cast<int>((M + bn - 1) / bn);
  a.units = (n_tiles / 2) * a.m_tiles;
  a.sk = sk;
  a.dp_units = sk ? dp_units : a.units;
  a.total = (int64_t)(a.units - a.dp_units) * a.k_tiles;
  a.counters = static_cast<int*>(workspace);
  a.partials = sk ? reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + p2::kCounters * 4) : nullptr;
  // X larger than ~1/3 of L2: keep each batch tile's X resident (weight-row pairs fastest)
  a.n_fastest = (a.m_tiles > 1 && M * K * 2 > ((int64_t)40 << 20)) ? 1 : 0;
  // rasterization group: per k step the P units in flight read P / G X slices
  // (bn x 128 f16) and G weight pairs (2 x 12 KB) — least L2 -> HBM traffic at
  // G = sqrt(P x X slice / pair slice) (~14 at bn 256)
  // — a divisor of the pair count when one is within 2x of that (a narrow last
  // group would put few pairs x many X tiles in flight)
  {
    const int np = n_tiles / 2;
    const double g = std::sqrt((double)max_pairs() * bn * kTileK * 2 / (2.0 * kTileBytes));
    int best = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(np, std::llround(g))));
    double off = 1e30;
    for (int d = 1; d <= np; ++d) {
      const double o = std::fabs(std::log(d / g));
      if (np % d == 0 && o < off && o <= std::log(2.0)) {
        off = o;
        best = d;
      }
    }
    a.group = best;
  }
  a.y_dtype = y_dtype;
  a.y_layout = y_layout;
  a.sm = ShiftMuls{1u << 26, 1u << 28, 1u << 30};
  const int pairs = sk ? max_pairs() : std::min(max_pairs(), a.units);
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [] {
    attr_err = cudaFuncSetAttribute(p2::w6a16_prefill_2sm_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    p2::kSmemBytes);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(p2::w6a16_prefill_2sm_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      p2::kSmemBytes);
    if (attr_err == cudaSuccess)
      attr_err = cudaFuncSetAttribute(p2::w6a16_prefill_2sm_kernel<false, 5>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, p2::kSmemBytes);
  });
  if (attr_err != cudaSuccess) return LPQT_E_CUDA;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * pairs);
  cfg.blockDim = dim3(p2::kThreads);
  cfg.dynamicSmemBytes = p2::kSmemBytes;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  int na = 0;
  attr[na].id = cudaLaunchAttributeClusterDimension;
  attr[na].val.clusterDim.x = 2;
  attr[na].val.clusterDim.y = 1;
  attr[na].val.clusterDim.z = 1;
  ++na;
  if (flags & LPQT_LAUNCH_PDL) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (grid_out) *grid_out = 2 * pairs;
  if (fgq && fp5) return LPQT_E_UNSUPPORTED;
  const cudaError_t le = fgq   ? cudaLaunchKernelEx(&cfg, p2::w6a16_prefill_2sm_kernel<true>, map, ymap, a, fq)
                         : fp5 ? cudaLaunchKernelEx(&cfg, p2::w6a16_prefill_2sm_kernel<false, 5>, map, ymap, a, fq)
                               : cudaLaunchKernelEx(&cfg, p2::w6a16_prefill_2sm_kernel<false>, map, ymap, a, fq);
  if (le != cudaSuccess) return LPQT_E_CUDA;
  note_launch();
  return check_launch();
}

}  // namespace lpqt
