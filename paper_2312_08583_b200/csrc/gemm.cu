// gemm.cu — K4/K5/K6: the W6A16 linear on tcgen05 (gemm.py:65-94 CGQ path).
//
//   Y[n, m] = (S[n] * 2^12) * sum_k C[n, k] * X[m, k]
//
// where C holds the bias-shifted binary16 code patterns (value * 2^-12,
// dequant.py:33-43) and S * 2^12 is the folded scale (dequant.py:46-69),
// formed in an fp32 register (exact, and free of the binary16 ScaleOverflow
// limit), so the product equals the reference's S * sum_k value * x exactly
// up to fp32 summation order (power-of-two scaling commutes with rounding).
//
// One persistent, warp-specialised kernel covers decode (M <= 16, HBM-bound)
// and prefill (tensor-bound).  Per CTA (1 per SM, 448 threads):
//   warp 8      TMA producer: per stage one 1-D bulk copy of a 12288-B
//               weight tile (evict-first) + two 2-D TMA boxes of X (64 k x
//               BN rows, 128-B swizzle; rows >= M and k >= K zero-filled).
//   warps 0-7   dequant (DQ): 3 x LDS.128 per thread (its row, its 64-k half)
//               -> FP6->FP16 register rebuild -> tcgen05.st into a TMEM A
//               buffer (128 lanes = weight rows, 32 cols = 64 k).
//   warp 9      MMA issuer (one lane): tcgen05.mma.kind::f16 with A in TMEM
//               ("TS"), B = X from SMEM, D (fp32, 128 x BN) in TMEM.
//   warps 10-13 epilogue: tcgen05.ld D -> x S*2^12 (folded) -> Y, or split-K
//               partial + deterministic last-CTA reduction (fixed split order).
// Pipelines: smem ring full/empty (TMA <-> DQ+MMA), TMEM-A ring afull/aempty
// (DQ <-> MMA), TMEM-D ring dfull/dempty (MMA <-> epilogue).
#include <mutex>

#include "common.cuh"

namespace lpqt {

constexpr int kNumDqWarps = 8;
constexpr int kNumEpiWarps = 4;
constexpr int kWarpTma = 8;
constexpr int kWarpMma = 9;
constexpr int kWarpEpi0 = 10;
constexpr int kThreads = (kNumDqWarps + 2 + kNumEpiWarps) * 32;  // 448
constexpr int kABufs = 4;
constexpr int kAColsPerBuf = kTileK / 2;  // 64 columns of packed half2
constexpr int kTmemCols = 512;
constexpr int kSmemBudget = 200 * 1024;

struct GemmArgs {
  const uint8_t* tiles;
  const uint16_t* scales;
  void* y;
  float* partials;
  int* counters;
  int64_t ldy;
  int M, N;
  int k_tiles, n_tiles, m_tiles;
  int splits, kt_per_split, num_units;
  int y_dtype, y_layout;
};

template <int BN>
struct Cfg {
  static constexpr int kXStageBytes = BN * kTileK * 2;  // two SW128 blocks of BN x 128 B
  static constexpr int kStageBytes = kXStageBytes + kTileBytes;
  static constexpr int kStagesRaw = kSmemBudget / kStageBytes;
  static constexpr int kStages = kStagesRaw > 8 ? 8 : kStagesRaw;
  static constexpr int kDBufs = BN <= 128 ? 2 : 1;
  static constexpr int kBarBytes = 8 * (2 * kStages + 2 * kABufs + 2 * kDBufs) + 16;
  static constexpr int kSmemBytes = kStages * kStageBytes + kBarBytes + 1024;
  static_assert(kStages >= 2, "pipeline too shallow");
  static_assert(kABufs * kAColsPerBuf + kDBufs * BN <= kTmemCols, "TMEM over-subscribed");
};

__device__ __forceinline__ void decode_unit(const GemmArgs& a, int u, int& n_tile, int& m_tile, int& split, int& kt0,
                                            int& kt1) {
  split = u % a.splits;
  const int tile = u / a.splits;
  n_tile = tile / a.m_tiles;
  m_tile = tile % a.m_tiles;
  kt0 = split * a.kt_per_split;
  kt1 = min(a.k_tiles, kt0 + a.kt_per_split);
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

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    w6a16_tcgen05_kernel(const __grid_constant__ CUtensorMap tmap_x, const GemmArgs a) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* smem_x = smem;                                   // kStages x kXStageBytes (1024-aligned)
  uint8_t* smem_w = smem + C::kStages * C::kXStageBytes;    // kStages x 12288
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_w + C::kStages * kTileBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* afull = empty + C::kStages;
  uint64_t* aempty = afull + kABufs;
  uint64_t* dfull = aempty + kABufs;
  uint64_t* dempty = dfull + C::kDBufs;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dempty + C::kDBufs);
  volatile int* last_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kNumDqWarps + 1);
    }
    for (int b = 0; b < kABufs; ++b) {
      mbar_init(&afull[b], kNumDqWarps);
      mbar_init(&aempty[b], 1);
    }
    for (int d = 0; d < C::kDBufs; ++d) {
      mbar_init(&dfull[d], 1);
      mbar_init(&dempty[d], kNumEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == kWarpMma) {
    tmem_alloc(tmem_slot, kTmemCols);
    tmem_relinquish();
  }
  if (warp == kWarpTma && lane == 0) prefetch_tmap(&tmap_x);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const uint32_t tmem_d0 = tmem_base + kABufs * kAColsPerBuf;

  if (warp == kWarpTma) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first_policy();
      int it = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
        int n_tile, m_tile, split, kt0, kt1;
        decode_unit(a, u, n_tile, m_tile, split, kt0, kt1);
        for (int kt = kt0; kt < kt1; ++kt, ++it) {
          const int s = it % C::kStages;
          const uint32_t ph = (it / C::kStages) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], C::kStageBytes);
          bulk_g2s(smem_w + s * kTileBytes, a.tiles + ((int64_t)n_tile * a.k_tiles + kt) * kTileBytes, kTileBytes,
                   &full[s], pol);
          uint8_t* xs = smem_x + s * C::kXStageBytes;
          tma_load_2d(xs, &tmap_x, &full[s], kt * kTileK, m_tile * BN);
          tma_load_2d(xs + BN * 128, &tmap_x, &full[s], kt * kTileK + 64, m_tile * BN);
        }
      }
    }
  } else if (warp < kNumDqWarps) {
    // ------------------------------------------------------------ dequant
    const int lg = warp & 3, khalf = warp >> 2;
    const int row = lg * 32 + lane;
    const uint32_t t_lane = tmem_base + (static_cast<uint32_t>(lg * 32) << 16) + khalf * 32;
    int it = 0;
    for (int u = blockIdx.x; u < a.num_units; u += gridDim.x) {
      int n_tile, m_tile, split, kt0, kt1;
      decode_unit(a, u, n_tile, m_tile, split, kt0, kt1);
      for (int kt = kt0; kt < kt1; ++kt, ++it) {
        const int s = it % C::kStages;
        const uint32_t ph = (it / C::kStages) & 1;
        const int b = it % kABufs;
        const uint32_t bph = (it / kABufs) & 1;
        mbar_wait(&full[s], ph);
        const uint8_t* src = smem_w + s * kTileBytes + (khalf * 3 * kTileN + row) * 16;
        const uint4 q0 = lds128(src);
        const uint4 q1 = lds128(src + kTileN * 16);
        const uint4 q2 = lds128(src + 2 * kTileN * 16);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        const uint32_t w0[6] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y};
        const uint32_t w1[6] = {q1.z, q1.w, q2.x, q2.y, q2.z, q2.w};
        uint32_t r[32];
        fp6x32_to_f16x32(w0, r);
        fp6x32_to_f16x32(w1, r + 16);
        mbar_wait(&aempty[b], bph ^ 1);
        tc_fence_after();
        tmem_st_x32(t_lane + b * kAColsPerBuf, r);
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&afull[b]);
      }
    }
  } else if (warp == kWarpMma) {
    // ------------------------------------------------------------ MMA issue
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_f16_m128(BN);
      int it = 0, lu = 0;
      for (int u = blockIdx.x; u < a.num_units; u += gridDim.x, ++lu) {
        int n_tile, m_tile, split, kt0, kt1;
        decode_unit(a, u, n_tile, m_tile, split, kt0, kt1);
        const int d = lu % C::kDBufs;
        const uint32_t dph = (lu / C::kDBufs) & 1;
        mbar_wait(&dempty[d], dph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_d0 + d * BN;
        for (int kt = kt0; kt < kt1; ++kt, ++it) {
          const int s = it % C::kStages;
          const uint32_t ph = (it / C::kStages) & 1;
          const int b = it % kABufs;
          const uint32_t bph = (it / kABufs) & 1;
          mbar_wait(&full[s], ph);
          mbar_wait(&afull[b], bph);
          tc_fence_after();
          const uint32_t xs = smem_u32(smem_x + s * C::kXStageBytes);
#pragma unroll
          for (int j = 0; j < kTileK / 16; ++j) {
            const uint64_t bdesc = sdesc_kmajor_sw128(xs + (j >> 2) * (BN * 128) + (j & 3) * 32);
            mma_f16_ts(d_tmem, tmem_base + b * kAColsPerBuf + j * 8, bdesc, idesc, (kt > kt0 || j > 0) ? 1u : 0u);
          }
          tc_commit(&empty[s]);
          tc_commit(&aempty[b]);
        }
        tc_commit(&dfull[d]);
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const int lg = warp & 3;
    const int rr = lg * 32 + lane;  // row inside the 128-row tile (= TMEM lane)
    const uint32_t t_lane = tmem_d0 + (static_cast<uint32_t>(lg * 32) << 16);
    int lu = 0;
    for (int u = blockIdx.x; u < a.num_units; u += gridDim.x, ++lu) {
      int n_tile, m_tile, split, kt0, kt1;
      decode_unit(a, u, n_tile, m_tile, split, kt0, kt1);
      const int d = lu % C::kDBufs;
      const uint32_t dph = (lu / C::kDBufs) & 1;
      const int n = n_tile * kTileN + rr;
      const int m0 = m_tile * BN;
      const float fs = n < a.N ? __half2float(__ushort_as_half(a.scales[n])) * 4096.0f : 0.f;
      mbar_wait(&dfull[d], dph);
      tc_fence_after();
      if (a.splits == 1) {
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t v[16];
          tmem_ld_x16(t_lane + d * BN + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) store_y(a, n, m0 + c0 + j, __uint_as_float(v[j]) * fs);
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[d]);
      } else {
        const int tile = u / a.splits;
        float* part = a.partials + (((int64_t)tile * a.splits + split) * kTileN + rr) * BN;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 16) {
          uint32_t v[16];
          tmem_ld_x16(t_lane + d * BN + c0, v);
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            *reinterpret_cast<float4*>(part + c0 + j) = make_float4(__uint_as_float(v[j]), __uint_as_float(v[j + 1]),
                                                                    __uint_as_float(v[j + 2]), __uint_as_float(v[j + 3]));
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&dempty[d]);
        __threadfence();
        named_bar_sync(1, kNumEpiWarps * 32);
        if (warp == kWarpEpi0 && lane == 0) {
          const int prev = atomicAdd(&a.counters[tile], 1);
          *last_flag = (prev == a.splits - 1) ? 1 : 0;
        }
        named_bar_sync(1, kNumEpiWarps * 32);
        if (*last_flag) {
          __threadfence();
          const float* base = a.partials + ((int64_t)tile * a.splits * kTileN + rr) * BN;
#pragma unroll 1
          for (int c0 = 0; c0 < BN; c0 += 4) {
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int s = 0; s < a.splits; ++s) {
              const float4 p = __ldcg(reinterpret_cast<const float4*>(base + (int64_t)s * kTileN * BN + c0));
              acc.x += p.x;
              acc.y += p.y;
              acc.z += p.z;
              acc.w += p.w;
            }
            store_y(a, n, m0 + c0 + 0, acc.x * fs);
            store_y(a, n, m0 + c0 + 1, acc.y * fs);
            store_y(a, n, m0 + c0 + 2, acc.z * fs);
            store_y(a, n, m0 + c0 + 3, acc.w * fs);
          }
          if (warp == kWarpEpi0 && lane == 0) a.counters[tile] = 0;
        }
        named_bar_sync(1, kNumEpiWarps * 32);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == kWarpMma) {
    tc_fence_after();
    tmem_dealloc(tmem_base, kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// host side: plan, tensor map, launch
// ---------------------------------------------------------------------------
struct Plan {
  int bn, splits, kt_per_split, grid, num_units, n_tiles, m_tiles, k_tiles, stages, smem;
  int64_t ws_bytes, counters_bytes;
};

static int pick_bn(int64_t M) {
  if (M <= 16) return 16;
  if (M <= 32) return 32;
  if (M <= 64) return 64;
  if (M <= 128) return 128;
  return 256;
}

template <int BN>
static void cfg_of(int& stages, int& smem) {
  stages = Cfg<BN>::kStages;
  smem = Cfg<BN>::kSmemBytes;
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

static Plan make_plan(int64_t M, int64_t N, int64_t K, int split_k, int sms) {
  Plan p{};
  p.bn = pick_bn(M);
  switch (p.bn) {
    case 16: cfg_of<16>(p.stages, p.smem); break;
    case 32: cfg_of<32>(p.stages, p.smem); break;
    case 64: cfg_of<64>(p.stages, p.smem); break;
    case 128: cfg_of<128>(p.stages, p.smem); break;
    default: cfg_of<256>(p.stages, p.smem); break;
  }
  p.n_tiles = static_cast<int>((N + kTileN - 1) / kTileN);
  p.m_tiles = static_cast<int>((M + p.bn - 1) / p.bn);
  p.k_tiles = static_cast<int>((K + kTileK - 1) / kTileK);
  const int64_t tiles = (int64_t)p.n_tiles * p.m_tiles;
  int best = 1;
  if (split_k > 0) {
    best = split_k;
  } else {
    // minimise waves x (k-tiles per unit + fixed per-unit cost); the fixed
    // cost (pipeline fill + epilogue, in k-tile units) grows with the
    // partial-tile traffic of split-K.
    double best_cost = 1e30;
    const int max_s = p.k_tiles < 32 ? p.k_tiles : 32;
    for (int s = 1; s <= max_s; ++s) {
      const int per = (p.k_tiles + s - 1) / s;
      const int s_eff = (p.k_tiles + per - 1) / per;
      const int64_t units = tiles * s_eff;
      const int64_t waves = (units + sms - 1) / sms;
      const double fixed = 2.0 + (s_eff > 1 ? p.bn / 32.0 : 0.0);
      const double cost = (double)waves * (per + fixed);
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        best = s_eff;
      }
    }
  }
  if (best > p.k_tiles) best = p.k_tiles;
  if (best < 1) best = 1;
  p.kt_per_split = (p.k_tiles + best - 1) / best;
  p.splits = (p.k_tiles + p.kt_per_split - 1) / p.kt_per_split;
  p.num_units = static_cast<int>(tiles * p.splits);
  p.grid = p.num_units < sms ? p.num_units : sms;
  if (p.splits > 1) {
    p.counters_bytes = ((tiles * 4) + 255) / 256 * 256;
    p.ws_bytes = p.counters_bytes + tiles * p.splits * kTileN * p.bn * 4;
  } else {
    p.counters_bytes = 0;
    p.ws_bytes = 0;
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

template <int BN>
static int launch(const Plan& p, const GemmArgs& args, const uint16_t* Xt, int64_t ldx, int64_t M,
                  cudaStream_t stream) {
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
  static std::once_flag once;
  static cudaError_t attr_err = cudaSuccess;
  std::call_once(once, [&] {
    attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<BN>::kSmemBytes);
  });
  if (attr_err != cudaSuccess) return LPQT_E_CUDA;
  kern<<<p.grid, kThreads, Cfg<BN>::kSmemBytes, stream>>>(map, args);
  note_launch();
  return check_launch();
}

}  // namespace lpqt

using namespace lpqt;

extern "C" {

int64_t lpqt_w6a16_workspace_bytes(int64_t M, int64_t N, int64_t K, int split_k) {
  if (M <= 0 || N <= 0 || K <= 0) return 0;
  return make_plan(M, N, K, split_k, num_sms()).ws_bytes;
}

int lpqt_w6a16_plan(int64_t M, int64_t N, int64_t K, int split_k, int* block_n, int* splits, int* grid, int* stages) {
  if (M <= 0 || N <= 0 || K <= 0) return LPQT_E_SHAPE;
  const Plan p = make_plan(M, N, K, split_k, num_sms());
  if (block_n) *block_n = p.bn;
  if (splits) *splits = p.splits;
  if (grid) *grid = p.grid;
  if (stages) *stages = p.stages;
  return LPQT_OK;
}

int lpqt_w6a16_linear(const uint8_t* tiles, const uint16_t* scales, const uint16_t* Xt, int64_t ldx, int64_t M,
                      int64_t N, int64_t K, void* Y, int y_dtype, int y_layout, int64_t ldy, int split_k,
                      void* workspace, int64_t workspace_bytes, void* stream) {
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
  args.tiles = tiles;
  args.scales = scales;
  args.y = Y;
  args.counters = static_cast<int*>(workspace);
  args.partials = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + p.counters_bytes);
  args.ldy = ldy;
  args.M = static_cast<int>(M);
  args.N = static_cast<int>(N);
  args.k_tiles = p.k_tiles;
  args.n_tiles = p.n_tiles;
  args.m_tiles = p.m_tiles;
  args.splits = p.splits;
  args.kt_per_split = p.kt_per_split;
  args.num_units = p.num_units;
  args.y_dtype = y_dtype;
  args.y_layout = y_layout;
  cudaStream_t st = as_stream(stream);
  switch (p.bn) {
    case 16: return launch<16>(p, args, Xt, ldx, M, st);
    case 32: return launch<32>(p, args, Xt, ldx, M, st);
    case 64: return launch<64>(p, args, Xt, ldx, M, st);
    case 128: return launch<128>(p, args, Xt, ldx, M, st);
    default: return launch<256>(p, args, Xt, ldx, M, st);
  }
}

}  // extern "C"
