// quantize.cu — K1 (fused CGQ FP6 quantize + 4+2 pack + fold) and the
// elementwise codec kernels behind the reference API:
//   encode_rtn_array (codec.py:116-132), pack/unpack (packing.py:63-118),
//   fold_scale_array (dequant.py:61-69), dequant_{bias_shift,naive}_array
//   (dequant.py:72-86), dequantize_tensor (quantizer.py:269-299), and the
//   activation staging used by the GEMM (gemm.py:69 X -> fp16, K-major).
//
// Bit-exactness recipe: every input dtype is widened to
// double exactly, scales are S = RN_f16(peak / 28) computed as an IEEE f64
// division followed by one f64->f16 rounding (the reference's
// `(peak / 28).astype(float16)`, quantizer.py:149, :227), and codes compare
// the IEEE-rounded f64 quotient w / S against the 31 exact midpoints with the
// ties-to-even fix-up — literally the reference's arithmetic.  No fast-math.
#include "common.cuh"

namespace lpqt {

// ---- dtype loads (exact widening to double) --------------------------------
template <int DT>
__device__ __forceinline__ double load_as_double(const void* p, int64_t i);
template <>
__device__ __forceinline__ double load_as_double<LPQT_F64>(const void* p, int64_t i) {
  return static_cast<const double*>(p)[i];
}
template <>
__device__ __forceinline__ double load_as_double<LPQT_F32>(const void* p, int64_t i) {
  return static_cast<double>(static_cast<const float*>(p)[i]);
}
template <>
__device__ __forceinline__ double load_as_double<LPQT_F16>(const void* p, int64_t i) {
  return static_cast<double>(__half2float(static_cast<const __half*>(p)[i]));
}
template <>
__device__ __forceinline__ double load_as_double<LPQT_BF16>(const void* p, int64_t i) {
  return static_cast<double>(__bfloat162float(static_cast<const __nv_bfloat16*>(p)[i]));
}

// ---- RTN encode (codec.py:116-132) ------------------------------------------
// mids[i] = (g[i] + g[i+1]) / 2, exact.  idx = #{i : mids[i] <= |x|}
// (searchsorted side='right'), exact-midpoint hit with odd idx -> idx - 1,
// sign bit iff x < 0 (so -0.0 -> code 0, codec.py:130).
__device__ __forceinline__ uint32_t fp6_encode(double x, const double* __restrict__ mids) {
  const double a = fabs(x);
  int idx = 0;
#pragma unroll
  for (int step = 16; step >= 1; step >>= 1) {
    if (idx + step <= 31 && mids[idx + step - 1] <= a) idx += step;
  }
  if (idx > 0 && (idx & 1) && a == mids[idx - 1]) idx -= 1;
  return (x < 0.0 ? 0x20u : 0u) | static_cast<uint32_t>(idx);
}

__device__ __forceinline__ void load_mids(double* smem_mids) {
  for (int i = threadIdx.x; i < 32; i += blockDim.x) {
    smem_mids[i] = i < 31 ? 0.5 * (fp6_magnitude(i) + fp6_magnitude(i + 1)) : 1e300;
  }
  __syncthreads();
}

template <int DT>
__global__ void encode_kernel(const void* __restrict__ x, int64_t n, uint8_t* __restrict__ codes,
                              uint32_t* __restrict__ flags) {
  __shared__ double mids[32];
  load_mids(mids);
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = load_as_double<DT>(x, i);
    if (!isfinite(v)) {
      bad = true;
      codes[i] = 0;
      continue;
    }
    codes[i] = static_cast<uint8_t>(fp6_encode(v, mids));
  }
  if (bad) atomicOr(flags, LPQT_F_NONFINITE);
}

// ---- fast exact encode for binary16 / bfloat16 inputs ------------------------
// For w in f16 or bf16 and S a binary16 scale, the exact quotient q = |w| / S
// is never closer than 2^-15 (relative) to a grid midpoint m unless it equals
// it: w - m*S is a nonzero multiple of a granularity >= 2^-15 * m*S (w has
// <= 11 significant bits, m*S <= 15).  So RN_f32(q) lands on the same side of
// every midpoint as q (and on m exactly iff q == m), the reference's f64
// quotient does too (quantizer.py:228), and the hardware RNE conversion to
// e3m2 (cvt.rn.satfinite.e3m2x2.f32) reproduces searchsorted(mids, q, 'right')
// with the ties-to-even fix-up (codec.py:125-129): ties go to the even
// mantissa = the even grid index, and q > 26 saturates to 28 (idx 31).  The
// sign is applied separately so -0.0 -> code 0 (codec.py:130).
// f32 / f64 inputs keep the literal f64 path (fp6_encode above).
__device__ __forceinline__ uint32_t fp6_encode2_cvt_div(float w0, float w1, float S) {
  const float q0 = __fdiv_rn(fabsf(w0), S), q1 = __fdiv_rn(fabsf(w1), S);
  uint16_t r;
  asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(q1), "f"(q0));
  return static_cast<uint32_t>(r) | (w0 < 0.f ? 0x20u : 0u) | (w1 < 0.f ? 0x2000u : 0u);
}
// The same quotients without a division per element: with the row's Y =
// RN(1/S) (one __frcp_rn per row), q0 = RN(a Y), the exact residual
// R = a - S q0 (one FMA) and q = RN(q0 + R Y) (Markstein's correction) — three
// FMA-pipe ops per weight.  Pinned against the __fdiv_rn path for EVERY
// binary16 / bfloat16 weight and every binary16 scale in the quantizer's range
// (|w| <= 29 S) by lpqt_selftest_fp6_encode (tests/test_gpu_parity.py): the
// codes agree everywhere; the f32 quotients too for binary16 weights (for
// bfloat16 0.26 % differ by an ulp, none across a grid midpoint).
__device__ __forceinline__ float div_by_scale(float a, float S, float Y) {
  const float q0 = __fmul_rn(a, Y);
  const float R = __fmaf_rn(-S, q0, a);
  return __fmaf_rn(R, Y, q0);
}
__device__ __forceinline__ uint32_t fp6_encode2_cvt(float w0, float w1, float S, float Y) {
  const float q0 = div_by_scale(fabsf(w0), S, Y), q1 = div_by_scale(fabsf(w1), S, Y);
  uint16_t r;
  asm("cvt.rn.satfinite.e3m2x2.f32 %0, %1, %2;" : "=h"(r) : "f"(q1), "f"(q0));
  return static_cast<uint32_t>(r) | (w0 < 0.f ? 0x20u : 0u) | (w1 < 0.f ? 0x2000u : 0u);
}
__device__ __forceinline__ uint32_t fp6_encode2_cvt(float w0, float w1, float S) {
  return fp6_encode2_cvt(w0, w1, S, __frcp_rn(S));
}

template <int DT>
struct InTraits {
  using Acc = float;
  static constexpr bool kCvt = true;
};
template <>
struct InTraits<LPQT_F32> {
  using Acc = float;
  static constexpr bool kCvt = false;
};
template <>
struct InTraits<LPQT_F64> {
  using Acc = double;
  static constexpr bool kCvt = false;
};

// 8 consecutive elements from a 16-byte aligned address, widened exactly
template <int DT>
__device__ __forceinline__ void load8(const void* p, typename InTraits<DT>::Acc v[8]) {
  const uint4* q = static_cast<const uint4*>(p);
  if constexpr (DT == LPQT_F16 || DT == LPQT_BF16) {
    const uint4 u = __ldg(q);
    const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if constexpr (DT == LPQT_F16) {
        const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&w[i]));
        v[2 * i] = f.x;
        v[2 * i + 1] = f.y;
      } else {
        v[2 * i] = __uint_as_float(w[i] << 16);
        v[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
      }
    }
  } else if constexpr (DT == LPQT_F32) {
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const float4 f = __ldg(reinterpret_cast<const float4*>(q) + i);
      v[4 * i] = f.x, v[4 * i + 1] = f.y, v[4 * i + 2] = f.z, v[4 * i + 3] = f.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const double2 d = __ldg(reinterpret_cast<const double2*>(q) + i);
      v[2 * i] = d.x, v[2 * i + 1] = d.y;
    }
  }
}
template <int DT>
__device__ __forceinline__ typename InTraits<DT>::Acc load1(const void* p, int64_t i) {
  if constexpr (DT == LPQT_F64) return static_cast<const double*>(p)[i];
  else return static_cast<float>(load_as_double<DT>(p, i));
}
template <int DT>
__device__ __forceinline__ int elem_bytes() {
  return DT == LPQT_F64 ? 8 : DT == LPQT_F32 ? 4 : 2;
}

// 8 codes -> one u64 (byte j = code of element j)
template <int DT>
__device__ __forceinline__ uint64_t encode8(const typename InTraits<DT>::Acc v[8], float Sf, double Sd,
                                            const double* __restrict__ mids) {
  uint64_t c = 0;
  if constexpr (InTraits<DT>::kCvt) {
    const float Y = __frcp_rn(Sf);  // (hoisted out of callers' loops by the compiler when Sf is invariant)
#pragma unroll
    for (int i = 0; i < 4; ++i) c |= static_cast<uint64_t>(fp6_encode2_cvt(v[2 * i], v[2 * i + 1], Sf, Y)) << (16 * i);
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      c |= static_cast<uint64_t>(fp6_encode(static_cast<double>(v[i]) / Sd, mids)) << (8 * i);
  }
  return c;
}

template <int DT>
__device__ __forceinline__ uint32_t encode1(typename InTraits<DT>::Acc v, float S, const double* __restrict__ mids) {
  if constexpr (InTraits<DT>::kCvt) return fp6_encode2_cvt(v, 0.f, S) & 0xFFu;
  else return fp6_encode(static_cast<double>(v) / static_cast<double>(S), mids);
}

// ---- K1a: per-block scales (quantizer.py:200-201, :224-227 with the FGQ
// blocks of :91-115, _round_scales_f16 :142-153; fold dequant.py:61-69).  One
// warp per (row, block of B columns) — B = K for CGQ (one block per row) —
// scales stored row-major per block (r * bpr + j); 16-byte loads.
template <int DT>
__global__ void __launch_bounds__(256) block_scales_kernel(const void* __restrict__ W, int64_t N, int64_t K,
                                                           int64_t ldw, int64_t B, int64_t bpr, int vec,
                                                           double maxv, int bias_shift,
                                                           uint16_t* __restrict__ scales,
                                                           uint16_t* __restrict__ folded,
                                                           uint32_t* __restrict__ flags) {
  using Acc = typename InTraits<DT>::Acc;
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  uint32_t f = 0;
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < N * bpr; u += warps) {
    const int64_t r = u / bpr, j = u - r * bpr;
    const int64_t k0 = j * B, k1 = k0 + B < K ? k0 + B : K;
    const char* row = static_cast<const char*>(W) + r * ldw * elem_bytes<DT>();
    Acc peak = 0;
    bool bad = false;
    const int64_t k8 = (vec && k0 % 8 == 0) ? k0 + (k1 - k0) / 8 * 8 : k0;
    for (int64_t k = k0 + 8 * lane; k < k8; k += 256) {
      Acc v[8];
      load8<DT>(row + k * elem_bytes<DT>(), v);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        bad |= !isfinite(v[q]);
        peak = fmax(peak, fabs(v[q]));
      }
    }
    for (int64_t k = k8 + lane; k < k1; k += 32) {
      const Acc v = load1<DT>(row, k);
      bad |= !isfinite(v);
      peak = fmax(peak, fabs(v));
    }
    if (__any_sync(0xffffffffu, bad)) f |= LPQT_F_NONFINITE;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    if (lane == 0) {
      const double p = static_cast<double>(peak);
      const double raw = (p == 0.0) ? 1.0 : p / maxv;  // max_value: 28 (FP6), 24 (FP5)
      uint16_t sb = __half_as_ushort(__double2half(raw));
      if ((sb & 0x7FFFu) == 0x7C00u) f |= LPQT_F_SCALE_INF;
      if ((sb & 0x7FFFu) == 0) sb = 0x0001u;  // underflow clamps to 2^-24
      scales[u] = sb;
      if (bias_shift) {
        const double fv = static_cast<double>(__half2float(__ushort_as_half(sb))) * 4096.0;
        if (fv > 65504.0) f |= LPQT_F_FOLD_OVERFLOW;
        folded[u] = (fv > 65504.0) ? (uint16_t)0x7C00u : __half_as_ushort(__double2half(fv));
      }
    }
  }
  if (f) atomicOr(flags, f);
}

// scale of element (r, k) under B-column blocks (B = K: the row's scale)
__device__ __forceinline__ float block_scale(const uint16_t* __restrict__ scales, int64_t r, int64_t k, int64_t B,
                                             int64_t bpr) {
  return __half2float(__ushort_as_half(scales[r * bpr + k / B]));
}

__device__ __forceinline__ void load_mids_f64(double* smem_mids) {
  for (int i = threadIdx.x; i < 32; i += blockDim.x)
    smem_mids[i] = i < 31 ? 0.5 * (fp6_magnitude(i) + fp6_magnitude(i + 1)) : 1e300;
  __syncthreads();
}

// ---- K1b: codes -> canonical planes (quantizer.py:228-229, packing.py:63-90).
// Thread per 8 consecutive codes of the flat row-major stream: one u32 of
// seg4 and one u16 of seg2 (groups are 8-aligned in the flat index, so this
// holds for any K; the last group pads with code 0 like packing.py:73).
template <int DT>
__global__ void __launch_bounds__(256) encode_planes_kernel(const void* __restrict__ W, int64_t N, int64_t K,
                                                            int64_t ldw, int vec, int64_t B, int64_t bpr,
                                                            const uint16_t* __restrict__ scales,
                                                            uint8_t* __restrict__ seg4, uint8_t* __restrict__ seg2) {
  using Acc = typename InTraits<DT>::Acc;
  __shared__ double mids[32];
  if constexpr (!InTraits<DT>::kCvt) load_mids_f64(mids);
  const int64_t total = N * K, groups = (total + 7) / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = 8 * g;
    uint64_t c = 0;
    if (vec) {  // vec => K % 8 == 0 and B % 8 == 0: one row, one block
      const int64_t r = i0 / K, k = i0 - r * K;
      Acc v[8];
      load8<DT>(static_cast<const char*>(W) + (r * ldw + k) * elem_bytes<DT>(), v);
      const float s = block_scale(scales, r, k, B, bpr);
      c = encode8<DT>(v, s, static_cast<double>(s), mids);
    } else {
      int64_t r = i0 / K, k = i0 - r * K;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (i0 + j < total) {
          const Acc v = load1<DT>(W, r * ldw + k);
          c |= static_cast<uint64_t>(encode1<DT>(v, block_scale(scales, r, k, B, bpr), mids)) << (8 * j);
        }
        if (++k == K) k = 0, ++r;
      }
    }
    uint32_t s4 = 0, s2 = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint32_t cj = static_cast<uint32_t>(c >> (8 * j)) & 0x3Fu;
      s4 |= (cj >> 2) << (4 * j);
      s2 |= (cj & 3u) << (2 * j);
    }
    *reinterpret_cast<uint32_t*>(seg4 + 4 * g) = s4;
    *reinterpret_cast<uint16_t*>(seg2 + 2 * g) = static_cast<uint16_t>(s2);
  }
}

// ---- K1c: codes straight into the GEMM tile layout (no canonical planes).
// Thread per (row n < Np, 64-weight half of a 128-k tile): 8 x 16 B loads,
// 64 codes, 12 words (fp6x32 layout v2, common.cuh), 3 x 16 B stores.  Rows
// are the fastest thread index so every warp store writes 512 contiguous
// bytes of one [khalf][quad] plane.  Padding rows / columns get code 0
// (exactly what prepack writes).
__device__ __forceinline__ void pack_words_from_bytes(const uint32_t cw[8], uint32_t w[6]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    w[i] = cw[i] | (((cw[6] >> (2 * i)) & 0x03030303u) << 6);
    w[3 + i] = cw[3 + i] | (((cw[7] >> (2 * i)) & 0x03030303u) << 6);
  }
}

template <int DT>
__global__ void __launch_bounds__(256) encode_tiles_kernel(const void* __restrict__ W, int64_t N, int64_t K,
                                                           int64_t ldw, int vec, int64_t B, int64_t bpr,
                                                           const uint16_t* __restrict__ scales, int64_t Np,
                                                           int64_t k_tiles, uint8_t* __restrict__ tiles) {
  using Acc = typename InTraits<DT>::Acc;
  __shared__ double mids[32];
  if constexpr (!InTraits<DT>::kCvt) load_mids_f64(mids);
  const int64_t total = Np * k_tiles * 2;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int rr = static_cast<int>(t & 127);
    const int64_t s = t >> 7;
    const int kh = static_cast<int>(s & 1);
    const int64_t tile = s >> 1;  // rt * k_tiles + kt
    const int64_t rt = tile / k_tiles, kt = tile - rt * k_tiles;
    const int64_t n = rt * kTileN + rr, k0 = kt * kTileK + kh * 64;
    uint32_t cw[16];
    if (n < N) {
      const char* row = static_cast<const char*>(W) + n * ldw * elem_bytes<DT>();
      if (vec && k0 + 64 <= K) {  // vec => B % 8 == 0: one scale per 8 columns
        int64_t j = k0 / B, kb = (j + 1) * B;  // block of the current 8-group, its end
        float Sf = __half2float(__ushort_as_half(scales[n * bpr + j]));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          if (k0 + 8 * q >= kb) {
            ++j, kb += B;
            Sf = __half2float(__ushort_as_half(scales[n * bpr + j]));
          }
          Acc v[8];
          load8<DT>(row + (k0 + 8 * q) * elem_bytes<DT>(), v);
          const uint64_t c = encode8<DT>(v, Sf, static_cast<double>(Sf), mids);
          cw[2 * q] = static_cast<uint32_t>(c);
          cw[2 * q + 1] = static_cast<uint32_t>(c >> 32);
        }
      } else {
#pragma unroll 1
        for (int q = 0; q < 8; ++q) {
          uint64_t c = 0;
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int64_t k = k0 + 8 * q + e;
            if (k < K) c |= static_cast<uint64_t>(encode1<DT>(load1<DT>(row, k), block_scale(scales, n, k, B, bpr),
                                                                mids)) << (8 * e);
          }
          cw[2 * q] = static_cast<uint32_t>(c);
          cw[2 * q + 1] = static_cast<uint32_t>(c >> 32);
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < 16; ++i) cw[i] = 0;
    }
    uint32_t w[12];
    pack_words_from_bytes(cw, w);
    pack_words_from_bytes(cw + 8, w + 6);
    uint4* dst = reinterpret_cast<uint4*>(tiles + tile * kTileBytes) + (kh * 3) * kTileN + rr;
#pragma unroll
    for (int q = 0; q < 3; ++q) dst[q * kTileN] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
  }
}

// ---- K1 fused (CGQ, 16-B aligned rows, K % 8 == 0): one CTA per group of
// kQRows rows — phase 1: a warp per row computes the row's peak / scale /
// folded scale (block_scales_kernel's arithmetic); phase 2: the CTA encodes the
// same rows (their bytes are still in L2: the CTAs in flight hold
// <= 148 x 2 x 8 rows) into the GEMM tiles (TILES) or the canonical planes.
// DRAM traffic: the weights once + the codes, against twice + the codes for
// the two-kernel path (which stays for FGQ and unaligned rows).
constexpr int kQRows = 4;  // rows per CTA; 2 warps per row in phase 1
template <int DT, bool TILES>
__global__ void __launch_bounds__(256) quantize_fused_kernel(const void* __restrict__ W, int64_t N, int64_t K,
                                                             int64_t ldw, double maxv, int bias_shift,
                                                             uint16_t* __restrict__ scales,
                                                             uint16_t* __restrict__ folded,
                                                             uint32_t* __restrict__ flags, int64_t n_groups,
                                                             int64_t k_tiles, uint8_t* __restrict__ out4,
                                                             uint8_t* __restrict__ out2) {
  using Acc = typename InTraits<DT>::Acc;
  __shared__ double mids[32];
  __shared__ float s_scale[kQRows];
  __shared__ double s_peak[2 * kQRows];
  if constexpr (!InTraits<DT>::kCvt) load_mids_f64(mids);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t f = 0;
  for (int64_t grp = blockIdx.x; grp < n_groups; grp += gridDim.x) {
    const int64_t r0 = grp * kQRows;
    // ---- phase 1: the row scales (quantizer.py:200-201, :224-227; _round_scales_f16 :142-153; fold dequant.py:61-69)
    // 8 warps: warp 2q + h scans half h of row q; the two halves' peaks meet in
    // shared memory as doubles (exact for every input type)
    {
      const int rq = warp >> 1, h = warp & 1;
      const int64_t r = r0 + rq;
      Acc peak = 0;
      if (r < N) {
        const char* row = static_cast<const char*>(W) + r * ldw * elem_bytes<DT>();
        bool bad = false;
        for (int64_t k = 8 * (lane + 32 * h); k < K; k += 512) {
          Acc v[8];
          load8<DT>(row + k * elem_bytes<DT>(), v);
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            bad |= !isfinite(v[q]);
            peak = fmax(peak, fabs(v[q]));
          }
        }
        if (__any_sync(0xffffffffu, bad)) f |= LPQT_F_NONFINITE;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
      }
      if (lane == 0) s_peak[warp] = static_cast<double>(peak);
      __syncthreads();
      float sc = 0.f;
      if (h == 0 && r < N) {
        const double pk = fmax(s_peak[warp], s_peak[warp + 1]);
        uint16_t sb = __half_as_ushort(__double2half(pk == 0.0 ? 1.0 : pk / maxv));
        if ((sb & 0x7FFFu) == 0x7C00u) f |= LPQT_F_SCALE_INF;
        if ((sb & 0x7FFFu) == 0) sb = 0x0001u;  // underflow clamps to 2^-24
        sc = __half2float(__ushort_as_half(sb));
        if (lane == 0) {
          scales[r] = sb;
          if (bias_shift) {
            const double fv = static_cast<double>(sc) * 4096.0;
            if (fv > 65504.0) f |= LPQT_F_FOLD_OVERFLOW;
            folded[r] = (fv > 65504.0) ? (uint16_t)0x7C00u : __half_as_ushort(__double2half(fv));
          }
        }
      }
      if (h == 0 && lane == 0) s_scale[rq] = sc;
    }
    __syncthreads();
    // ---- phase 2: encode the group's rows (the bytes phase 1 just read, from L2)
    if constexpr (TILES) {
      // thread unit = (row, 64-weight half of a 128-k tile), rows fastest (encode_tiles_kernel's body)
      const int64_t units = (int64_t)kQRows * k_tiles * 2;
      for (int64_t u = threadIdx.x; u < units; u += blockDim.x) {
        const int rq = static_cast<int>(u % kQRows);
        const int64_t sk = u / kQRows;
        const int kh = static_cast<int>(sk & 1);
        const int64_t kt = sk >> 1;
        const int64_t n = r0 + rq, k0 = kt * kTileK + kh * 64;
        uint32_t cw[16];
        if (n < N) {
          const char* row = static_cast<const char*>(W) + n * ldw * elem_bytes<DT>();
          const float Sf = s_scale[rq];
          if (k0 + 64 <= K) {
#pragma unroll
            for (int q = 0; q < 8; ++q) {
              Acc v[8];
              load8<DT>(row + (k0 + 8 * q) * elem_bytes<DT>(), v);
              const uint64_t c = encode8<DT>(v, Sf, static_cast<double>(Sf), mids);
              cw[2 * q] = static_cast<uint32_t>(c);
              cw[2 * q + 1] = static_cast<uint32_t>(c >> 32);
            }
          } else {
#pragma unroll 1
            for (int q = 0; q < 8; ++q) {
              uint64_t c = 0;
              if (k0 + 8 * q < K) {  // (K % 8 == 0: whole groups of 8)
                Acc v[8];
                load8<DT>(row + (k0 + 8 * q) * elem_bytes<DT>(), v);
                c = encode8<DT>(v, Sf, static_cast<double>(Sf), mids);
              }
              cw[2 * q] = static_cast<uint32_t>(c);
              cw[2 * q + 1] = static_cast<uint32_t>(c >> 32);
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 16; ++i) cw[i] = 0;  // padding rows: code 0, as prepack writes
        }
        uint32_t w[12];
        pack_words_from_bytes(cw, w);
        pack_words_from_bytes(cw + 8, w + 6);
        const int64_t tile = (n / kTileN) * k_tiles + kt;
        uint4* dst = reinterpret_cast<uint4*>(out4 + tile * kTileBytes) + (kh * 3) * kTileN + (n % kTileN);
#pragma unroll
        for (int q = 0; q < 3; ++q) dst[q * kTileN] = make_uint4(w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
      }
    } else {
      // canonical planes: thread per 8 consecutive codes of a row (K % 8 == 0), one u32 of seg4 + one u16 of seg2
      const int64_t per_row = K / 8, units = (int64_t)kQRows * per_row;
      for (int64_t u = threadIdx.x; u < units; u += blockDim.x) {
        const int rq = static_cast<int>(u / per_row);
        const int64_t j = u - rq * per_row, n = r0 + rq;
        if (n >= N) break;  // (rows are the slow index: every later unit is past N too)
        Acc v[8];
        load8<DT>(static_cast<const char*>(W) + (n * ldw + 8 * j) * elem_bytes<DT>(), v);
        const float Sf = s_scale[rq];
        const uint64_t c = encode8<DT>(v, Sf, static_cast<double>(Sf), mids);
        uint32_t s4 = 0, s2 = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t ce = static_cast<uint32_t>(c >> (8 * e)) & 0x3Fu;
          s4 |= (ce >> 2) << (4 * e);
          s2 |= (ce & 3u) << (2 * e);
        }
        const int64_t g8 = (n * K) / 8 + j;
        *reinterpret_cast<uint32_t*>(out4 + 4 * g8) = s4;
        *reinterpret_cast<uint16_t*>(out2 + 2 * g8) = static_cast<uint16_t>(s2);
      }
    }
    __syncthreads();  // s_scale is rewritten by the next group
  }
  if (f) atomicOr(flags, f);
}

// grid of the fused quantizer: the CTAs in flight (4 per SM, 4 rows each) keep
// their rows in L2 up to K = 16384 (38 MB at K = 8192); longer rows take the
// two-kernel path (measured: fused 12-13 % faster at K = 4096 / 8192, 16 %
// slower at K = 28672; profiles/r02_quant_fused_vs_twopass.jsonl)
static int fused_grid(int64_t groups, int64_t K) {
  (void)K;
  const int64_t cap = 148 * 4;
  return static_cast<int>(groups < cap ? groups : cap);
}

// ---- self-test: the division-free quotient vs __fdiv_rn, exhaustively ------
// every positive finite binary16 scale S (block x) against every positive
// finite binary16 (dt 2) / bfloat16 (dt 3) weight a with a <= 29 S: the e3m2
// codes (and the f32 quotients) must agree bit for bit.
__global__ void selftest_encode_kernel(int bf16, unsigned long long* __restrict__ bad_codes,
                                       unsigned long long* __restrict__ bad_quot, unsigned long long* __restrict__ pairs) {
  const uint16_t sb = static_cast<uint16_t>(blockIdx.x + 1);  // 0x0001 .. 0x7BFF
  const float S = __half2float(__ushort_as_half(sb)), Y = __frcp_rn(S);
  unsigned long long nc = 0, nq = 0, np = 0;
  for (uint32_t ab = threadIdx.x; ab < (bf16 ? 0x7F80u : 0x7C00u); ab += blockDim.x) {
    const float a = bf16 ? __uint_as_float(ab << 16) : __half2float(__ushort_as_half(static_cast<uint16_t>(ab)));
    if (a > 29.f * S) continue;
    ++np;
    const float qd = __fdiv_rn(a, S), qf = div_by_scale(a, S, Y);
    nq += __float_as_uint(qd) != __float_as_uint(qf);
    nc += (fp6_encode2_cvt_div(a, -a, S) != fp6_encode2_cvt(a, -a, S, Y));
  }
  atomicAdd(bad_codes, nc);
  atomicAdd(bad_quot, nq);
  atomicAdd(pairs, np);
}

// ---- canonical pack / unpack (packing.py:63-118) --------------------------
// thread j owns seg2 byte j (codes 4j..4j+3) and seg4 bytes 2j, 2j+1; pad
// bytes are written as zero (packing.py:73, :88).
__global__ void pack_kernel(const uint8_t* __restrict__ codes, int64_t n, int64_t len4, int64_t len2,
                            uint8_t* __restrict__ seg4, uint8_t* __restrict__ seg2, uint32_t* __restrict__ flags) {
  bool bad = false;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < len2; j += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int64_t i = 4 * j + t;
      c[t] = i < n ? codes[i] : 0u;
      if (c[t] > 63u) bad = true;
    }
    seg2[j] = static_cast<uint8_t>((c[0] & 3u) | ((c[1] & 3u) << 2) | ((c[2] & 3u) << 4) | ((c[3] & 3u) << 6));
    if (2 * j < len4) seg4[2 * j] = static_cast<uint8_t>(((c[0] >> 2) & 15u) | (((c[1] >> 2) & 15u) << 4));
    if (2 * j + 1 < len4) seg4[2 * j + 1] = static_cast<uint8_t>(((c[2] >> 2) & 15u) | (((c[3] >> 2) & 15u) << 4));
  }
  if (bad) atomicOr(flags, LPQT_F_BAD_CODE);
}

__device__ __forceinline__ uint32_t canon_code(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg2,
                                               int64_t i) {
  const uint32_t hi = (seg4[i >> 1] >> (4 * (i & 1))) & 15u;
  const uint32_t lo = (seg2[i >> 2] >> (2 * (i & 3))) & 3u;
  return (hi << 2) | lo;
}

__global__ void unpack_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg2, int64_t n,
                              uint8_t* __restrict__ codes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    codes[i] = static_cast<uint8_t>(canon_code(seg4, seg2, i));
  }
}

// ---- fold (dequant.py:61-69) --------------------------------------------------
__global__ void fold_kernel(const uint16_t* __restrict__ scales, int64_t n, uint16_t* __restrict__ folded,
                            uint32_t* __restrict__ flags) {
  uint32_t f = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint16_t b = scales[i];
    const bool positive_finite = !(b & 0x8000u) && (b & 0x7FFFu) != 0 && (b & 0x7C00u) != 0x7C00u;
    if (!positive_finite) {
      f |= LPQT_F_BAD_SCALE;
      folded[i] = 0;
      continue;
    }
    const double v = static_cast<double>(__half2float(__ushort_as_half(b))) * 4096.0;
    if (v > 65504.0) {
      f |= LPQT_F_FOLD_OVERFLOW;
      folded[i] = 0x7C00u;
    } else {
      folded[i] = __half_as_ushort(__double2half(v));
    }
  }
  if (f) atomicOr(flags, f);
}

// ---- elementwise dequant (dequant.py:72-86) --------------------------------
// bias shift: compose[c] * folded, one binary16 rounding (__hmul is RN).
__global__ void dequant_bias_shift_kernel(const uint8_t* __restrict__ codes, const uint16_t* __restrict__ folded,
                                          int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const __half c = __ushort_as_half(fp6_compose_bits(codes[i]));
    out[i] = __half_as_ushort(__hmul(c, __ushort_as_half(folded[i])));
  }
}
// naive: value_f16[c] * S (value = compose * 2^12 exactly)
__global__ void dequant_naive_kernel(const uint8_t* __restrict__ codes, const uint16_t* __restrict__ scales,
                                     int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float v = __half2float(__ushort_as_half(fp6_compose_bits(codes[i]))) * 4096.0f;
    out[i] = __half_as_ushort(__hmul(__float2half_rn(v), __ushort_as_half(scales[i])));
  }
}

// ---- dequantize_tensor (quantizer.py:269-299), canonical planes -------------
// path 1 (bias_shift): compose[c] * folded[row]; path 0 (naive): value[c] * S.
// F64 output is the reference's exact f64 product; F16 output is the
// binary16 dequant of the chosen path.
template <int OUT>
__global__ void dequantize_tensor_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg2,
                                         const uint16_t* __restrict__ row_scale, int path, int64_t N, int64_t K,
                                         int64_t B, int64_t bpr, void* __restrict__ out) {
  const int64_t total = N * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = canon_code(seg4, seg2, i);
    const int64_t r = i / K, k = i - r * K;
    const __half comp = __ushort_as_half(fp6_compose_bits(c));
    const __half s = __ushort_as_half(row_scale[r * bpr + k / B]);  // the element's block (B = K: its row)
    if (OUT == LPQT_F64) {
      double v = static_cast<double>(__half2float(comp));
      if (path == 0) v *= 4096.0;
      static_cast<double*>(out)[i] = v * static_cast<double>(__half2float(s));
    } else {
      __half v = comp;
      if (path == 0) v = __float2half_rn(__half2float(comp) * 4096.0f);
      static_cast<uint16_t*>(out)[i] = __half_as_ushort(__hmul(v, s));
    }
  }
}

// ---- activation staging: X[K, M] (ldx) -> Xt[M, Kp] fp16 ---------------------
template <int DT>
__global__ void stage_activations_kernel(const void* __restrict__ X, int64_t K, int64_t M, int64_t ldx,
                                         uint16_t* __restrict__ Xt, int64_t Kp) {
  const int64_t total = M * Kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t m = i / Kp, k = i % Kp;
    __half h = __ushort_as_half(0);
    if (k < K) {
      const int64_t src = k * ldx + m;
      if (DT == LPQT_F64) h = __double2half(static_cast<const double*>(X)[src]);
      else if (DT == LPQT_F32) h = __float2half_rn(static_cast<const float*>(X)[src]);
      else if (DT == LPQT_F16) h = static_cast<const __half*>(X)[src];
      else h = __float2half_rn(__bfloat162float(static_cast<const __nv_bfloat16*>(X)[src]));
    }
    Xt[i] = __half_as_ushort(h);
  }
}


// ---------------------------------------------------------------------------
// FP5 e3m1 (codec.py FP5_E3M1: 3 exponent bits, 1 mantissa bit, bias 3, max
// 24) with the 4 + 1 split (packing.py:84-85, :112-113): seg4 holds c >> 1
// like FP6, the tail one mantissa bit per code (little-endian bit order).
// Codes are the literal f64 search (midpoints of the 16-value grid, ties to
// the even index, sign from the input).  The GEMM runs FP5 weights through
// the FP6 tile layout: every e3m1 value is the e3m2 value with mantissa m<<1.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double fp5_magnitude(int i) {
  const int e = i >> 1, m = i & 1;
  return e == 0 ? 0.125 * m : (1.0 + 0.5 * m) * ldexp(1.0, e - 3);
}
__device__ __forceinline__ void load_mids_fp5(double* smem_mids) {
  for (int i = threadIdx.x; i < 16; i += blockDim.x)
    smem_mids[i] = i < 15 ? 0.5 * (fp5_magnitude(i) + fp5_magnitude(i + 1)) : 1e300;
  __syncthreads();
}
__device__ __forceinline__ uint32_t fp5_encode(double x, const double* __restrict__ mids) {
  const double a = fabs(x);
  int idx = 0;
#pragma unroll
  for (int step = 8; step >= 1; step >>= 1) {
    if (idx + step <= 15 && mids[idx + step - 1] <= a) idx += step;
  }
  if (idx > 0 && (idx & 1) && a == mids[idx - 1]) idx -= 1;
  return (x < 0.0 ? 0x10u : 0u) | static_cast<uint32_t>(idx);
}
__device__ __forceinline__ uint32_t fp5_code(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg1,
                                             int64_t i) {
  const uint32_t hi = (seg4[i >> 1] >> (4 * (i & 1))) & 15u;
  const uint32_t lo = (seg1[i >> 3] >> (i & 7)) & 1u;
  return (hi << 1) | lo;
}
// binary16 bits of the bias-shift compose (dequant.py:33-43 with mantissa_bits 1)
__device__ __forceinline__ uint16_t fp5_compose_bits(uint32_t c) {
  return static_cast<uint16_t>(((c & 0x10u) << 11) | (((c >> 1) & 7u) << 10) | ((c & 1u) << 9));
}

template <int DT>
__global__ void fp5_encode_kernel(const void* __restrict__ x, int64_t n, uint8_t* __restrict__ codes,
                                  uint32_t* __restrict__ flags) {
  __shared__ double mids[16];
  load_mids_fp5(mids);
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = load_as_double<DT>(x, i);
    if (!isfinite(v)) {
      bad = true;
      codes[i] = 0;
      continue;
    }
    codes[i] = static_cast<uint8_t>(fp5_encode(v, mids));
  }
  if (bad) atomicOr(flags, LPQT_F_NONFINITE);
}

// thread per 8 codes: 4 bytes of seg4, 1 byte of the tail
__device__ __forceinline__ void fp5_put8(const uint32_t (&c)[8], int64_t g, int64_t len4, int64_t len1,
                                         uint8_t* __restrict__ seg4, uint8_t* __restrict__ seg1) {
  uint32_t s4 = 0, s1 = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    s4 |= ((c[j] >> 1) & 15u) << (4 * j);
    s1 |= (c[j] & 1u) << j;
  }
#pragma unroll
  for (int b = 0; b < 4; ++b)
    if (4 * g + b < len4) seg4[4 * g + b] = static_cast<uint8_t>(s4 >> (8 * b));
  if (g < len1) seg1[g] = static_cast<uint8_t>(s1);
}

__global__ void fp5_pack_kernel(const uint8_t* __restrict__ codes, int64_t n, int64_t len4, int64_t len1,
                                uint8_t* __restrict__ seg4, uint8_t* __restrict__ seg1, uint32_t* __restrict__ flags) {
  bool bad = false;
  const int64_t groups = (len4 * 2 + 7) / 8 > len1 ? (len4 * 2 + 7) / 8 : len1;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t i = 8 * g + j;
      c[j] = i < n ? codes[i] : 0u;
      if (c[j] > 31u) bad = true;
    }
    fp5_put8(c, g, len4, len1, seg4, seg1);
  }
  if (bad) atomicOr(flags, LPQT_F_BAD_CODE);
}

__global__ void fp5_unpack_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg1, int64_t n,
                                  uint8_t* __restrict__ codes) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    codes[i] = static_cast<uint8_t>(fp5_code(seg4, seg1, i));
}

// quantize_tensor minifloat branch for FP5 (quantizer.py:224-231): codes of
// W / S (f64 quotient, literal search) packed 4 + 1; thread per 8 flat codes
template <int DT>
__global__ void fp5_encode_planes_kernel(const void* __restrict__ W, int64_t N, int64_t K, int64_t ldw, int64_t B,
                                         int64_t bpr, const uint16_t* __restrict__ scales, int64_t len4, int64_t len1,
                                         uint8_t* __restrict__ seg4, uint8_t* __restrict__ seg1) {
  __shared__ double mids[16];
  load_mids_fp5(mids);
  const int64_t total = N * K, groups = (total + 7) / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = (8 * g) / K, k = 8 * g - r * K;
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c[j] = 0;
      if (8 * g + j < total) {
        const double v = load_as_double<DT>(W, r * ldw + k);
        const double S = static_cast<double>(__half2float(__ushort_as_half(scales[r * bpr + k / B])));
        c[j] = fp5_encode(v / S, mids);
      }
      if (++k == K) k = 0, ++r;
    }
    fp5_put8(c, g, len4, len1, seg4, seg1);
  }
}

// dequantize_tensor (quantizer.py:269-299) for FP5 planes, per-block scales
template <int OUT>
__global__ void fp5_dequantize_tensor_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg1,
                                             const uint16_t* __restrict__ bscale, int path, int64_t N, int64_t K,
                                             int64_t B, int64_t bpr, void* __restrict__ out) {
  const int64_t total = N * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = fp5_code(seg4, seg1, i);
    const int64_t r = i / K, k = i - r * K;
    const __half comp = __ushort_as_half(fp5_compose_bits(c));
    const __half s = __ushort_as_half(bscale[r * bpr + k / B]);
    if (OUT == LPQT_F64) {
      double v = static_cast<double>(__half2float(comp));
      if (path == 0) v *= 4096.0;
      static_cast<double*>(out)[i] = v * static_cast<double>(__half2float(s));
    } else {
      __half v = comp;
      if (path == 0) v = __float2half_rn(__half2float(comp) * 4096.0f);
      static_cast<uint16_t*>(out)[i] = __half_as_ushort(__hmul(v, s));
    }
  }
}

// elementwise binary16 dequant of FP5 codes (dequant.py:72-86)
__global__ void fp5_dequant_kernel(const uint8_t* __restrict__ codes, const uint16_t* __restrict__ scale, int path,
                                   int64_t n, uint16_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const __half comp = __ushort_as_half(fp5_compose_bits(codes[i]));
    const __half v = path == 1 ? comp : __float2half_rn(__half2float(comp) * 4096.0f);
    out[i] = __half_as_ushort(__hmul(v, __ushort_as_half(scale[i])));
  }
}


// ---------------------------------------------------------------------------
// INT4 asymmetric (quantizer.py:232-244, packing.py:121-141): per block
// zero point Z = RN_f16(min), scale S = RN_f16((max - min) / 15) (1.0 for a
// constant block, 0 -> 2^-24, inf -> InvalidInput), levels =
// clip(rint((w - Z) / S), 0, 15) in f64, two levels per byte (even index in
// the low nibble, ceil(n / 2) bytes).  The comparator path of SURVEY §8 f4.
// ---------------------------------------------------------------------------
template <int DT>
__global__ void __launch_bounds__(256) int4_block_params_kernel(const void* __restrict__ W, int64_t N, int64_t K,
                                                                int64_t ldw, int64_t B, int64_t bpr,
                                                                uint16_t* __restrict__ scales,
                                                                uint16_t* __restrict__ zeros,
                                                                uint32_t* __restrict__ flags) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  uint32_t f = 0;
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < N * bpr; u += warps) {
    const int64_t r = u / bpr, j = u - r * bpr;
    const int64_t k0 = j * B, k1 = k0 + B < K ? k0 + B : K;
    double lo = 1e308, hi = -1e308;
    bool bad = false;
    for (int64_t k = k0 + lane; k < k1; k += 32) {
      const double v = load_as_double<DT>(W, r * ldw + k);
      bad |= !isfinite(v);
      lo = fmin(lo, v);
      hi = fmax(hi, v);
    }
    if (__any_sync(0xffffffffu, bad)) f |= LPQT_F_NONFINITE;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if (lane == 0) {
      const uint16_t zb = __half_as_ushort(__double2half(lo));
      if ((zb & 0x7FFFu) == 0x7C00u) f |= LPQT_F_SCALE_INF;  // zero point overflows binary16
      const double span = hi - lo;
      uint16_t sb = __half_as_ushort(__double2half(span == 0.0 ? 1.0 : span / 15.0));
      if ((sb & 0x7FFFu) == 0x7C00u) f |= LPQT_F_SCALE_INF;
      if ((sb & 0x7FFFu) == 0) sb = 0x0001u;
      zeros[u] = zb;
      scales[u] = sb;
    }
  }
  if (f) atomicOr(flags, f);
}

__device__ __forceinline__ double h2d(uint16_t b) { return static_cast<double>(__half2float(__ushort_as_half(b))); }

template <int DT>
__global__ void int4_encode_kernel(const void* __restrict__ W, int64_t N, int64_t K, int64_t ldw, int64_t B,
                                   int64_t bpr, const uint16_t* __restrict__ scales,
                                   const uint16_t* __restrict__ zeros, int64_t len, uint8_t* __restrict__ nib) {
  const int64_t total = N * K, groups = (total + 7) / 8;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = (8 * g) / K, k = 8 * g - r * K;
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      if (8 * g + j < total) {
        const int64_t b = r * bpr + k / B;
        const double lvl = rint((load_as_double<DT>(W, r * ldw + k) - h2d(zeros[b])) / h2d(scales[b]));
        word |= static_cast<uint32_t>(fmin(fmax(lvl, 0.0), 15.0)) << (4 * j);
      }
      if (++k == K) k = 0, ++r;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (4 * g + q < len) nib[4 * g + q] = static_cast<uint8_t>(word >> (8 * q));
  }
}

__global__ void int4_pack_kernel(const uint8_t* __restrict__ lv, int64_t n, uint8_t* __restrict__ nib,
                                 uint32_t* __restrict__ flags) {
  bool bad = false;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < (n + 1) / 2;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t a = lv[2 * i], b = 2 * i + 1 < n ? lv[2 * i + 1] : 0u;
    bad |= a > 15u || b > 15u;
    nib[i] = static_cast<uint8_t>((a & 15u) | ((b & 15u) << 4));
  }
  if (bad) atomicOr(flags, LPQT_F_BAD_CODE);
}

__global__ void int4_unpack_kernel(const uint8_t* __restrict__ nib, int64_t n, uint8_t* __restrict__ lv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    lv[i] = static_cast<uint8_t>((nib[i >> 1] >> (4 * (i & 1))) & 15u);
}

// dequantize_tensor INT4 (quantizer.py:296-298): Z + S * level in f64
__global__ void int4_dequantize_kernel(const uint8_t* __restrict__ nib, const uint16_t* __restrict__ scales,
                                       const uint16_t* __restrict__ zeros, int64_t N, int64_t K, int64_t B,
                                       int64_t bpr, double* __restrict__ out) {
  const int64_t total = N * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / K, k = i - r * K, b = r * bpr + k / B;
    const double lvl = static_cast<double>((nib[i >> 1] >> (4 * (i & 1))) & 15u);
    out[i] = h2d(zeros[b]) + h2d(scales[b]) * lvl;
  }
}

}  // namespace lpqt

using namespace lpqt;

#define LPQT_DISPATCH_DT(dt, ...)                                          \
  switch (dt) {                                                            \
    case LPQT_F64: { constexpr int DT = LPQT_F64; __VA_ARGS__; } break;   \
    case LPQT_F32: { constexpr int DT = LPQT_F32; __VA_ARGS__; } break;   \
    case LPQT_F16: { constexpr int DT = LPQT_F16; __VA_ARGS__; } break;   \
    case LPQT_BF16: { constexpr int DT = LPQT_BF16; __VA_ARGS__; } break; \
    default: return LPQT_E_UNSUPPORTED;                                    \
  }

extern "C" {

int lpqt_selftest_fp6_encode(int dtype, unsigned long long* out3) {
  if (dtype != LPQT_F16 && dtype != LPQT_BF16) return LPQT_E_UNSUPPORTED;
  unsigned long long* d = nullptr;
  if (cudaMalloc(&d, 3 * sizeof(unsigned long long)) != cudaSuccess) return LPQT_E_CUDA;
  cudaMemset(d, 0, 3 * sizeof(unsigned long long));
  selftest_encode_kernel<<<0x7BFF, 256>>>(dtype == LPQT_BF16, d, d + 1, d + 2);
  note_launch();
  int rc = check_launch();
  if (cudaMemcpy(out3, d, 3 * sizeof(unsigned long long), cudaMemcpyDeviceToHost) != cudaSuccess) rc = LPQT_E_CUDA;
  cudaFree(d);
  return rc;
}

int64_t lpqt_fp6_seg4_length(int64_t n) { return ((n + 1) / 2 + 3) / 4 * 4; }
int64_t lpqt_fp6_tail_length(int64_t n) { return ((n * 2 + 7) / 8 + 3) / 4 * 4; }

int lpqt_fp6_encode_rtn(const void* x, int dtype, int64_t n, uint8_t* codes, uint32_t* dev_flags, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  const int g = grid_for(n, 256);
  LPQT_DISPATCH_DT(dtype, encode_kernel<DT><<<g, 256, 0, as_stream(stream)>>>(x, n, codes, dev_flags));
  note_launch();
  return check_launch();
}

int lpqt_fp6_pack(const uint8_t* codes, int64_t n, uint8_t* seg4, uint8_t* seg2, uint32_t* dev_flags, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  const int64_t len4 = lpqt_fp6_seg4_length(n), len2 = lpqt_fp6_tail_length(n);
  if (len2 == 0) return LPQT_OK;
  pack_kernel<<<grid_for(len2, 256), 256, 0, as_stream(stream)>>>(codes, n, len4, len2, seg4, seg2, dev_flags);
  note_launch();
  return check_launch();
}

int lpqt_fp6_unpack(const uint8_t* seg4, const uint8_t* seg2, int64_t n, uint8_t* codes, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  unpack_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(seg4, seg2, n, codes);
  note_launch();
  return check_launch();
}

int lpqt_fp6_fold_scales(const uint16_t* scales, int64_t n, uint16_t* folded, uint32_t* dev_flags, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  fold_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(scales, n, folded, dev_flags);
  note_launch();
  return check_launch();
}

int lpqt_fp6_dequant_bias_shift(const uint8_t* codes, const uint16_t* folded, int64_t n, uint16_t* out,
                                void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  dequant_bias_shift_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(codes, folded, n, out);
  note_launch();
  return check_launch();
}

int lpqt_fp6_dequant_naive(const uint8_t* codes, const uint16_t* scales, int64_t n, uint16_t* out, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  dequant_naive_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(codes, scales, n, out);
  note_launch();
  return check_launch();
}

#ifndef LPQT_FUSED_QUANT
#define LPQT_FUSED_QUANT 1
#endif
static int quantize_scales(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int64_t B, int64_t bpr,
                           int vec, int bias_shift, uint16_t* scales, uint16_t* folded, uint32_t* dev_flags,
                           cudaStream_t st, double maxv = 28.0) {
  const int64_t units = N * bpr;
  const int g = static_cast<int>((units + 7) / 8 < 148 * 8 ? (units + 7) / 8 : 148 * 8);
  LPQT_DISPATCH_DT(dtype, block_scales_kernel<DT><<<g, 256, 0, st>>>(W, N, K, ldw, B, bpr, vec, maxv, bias_shift,
                                                                      scales, folded, dev_flags));
  note_launch();
  return check_launch();
}

static int rows_vectorizable(const void* W, int64_t ldw) {
  return (reinterpret_cast<uintptr_t>(W) % 16 == 0) && (ldw % 8 == 0);
}

// block <= 0 or >= K: CGQ (one block per row)
static void block_geometry(int64_t K, int64_t block, int64_t& B, int64_t& bpr) {
  B = (block <= 0 || block >= K) ? K : block;
  bpr = (K + B - 1) / B;
}

static int check_quantize_args(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int bias_shift,
                               const uint16_t* folded) {
  (void)W;
  if (N < 0 || K < 0 || ldw < K) return LPQT_E_SHAPE;
  if (bias_shift && folded == nullptr) return LPQT_E_INVALID_INPUT;
  if (dtype < LPQT_F64 || dtype > LPQT_BF16) return LPQT_E_UNSUPPORTED;
  return LPQT_OK;
}

int lpqt_fp6_quantize_pack_blocks(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int64_t block,
                                  int bias_shift, uint16_t* scales, uint16_t* folded, uint8_t* seg4, uint8_t* seg2,
                                  uint32_t* dev_flags, void* stream) {
  int rc = check_quantize_args(W, dtype, N, K, ldw, bias_shift, folded);
  if (rc != LPQT_OK || N == 0 || K == 0) return rc;
  const cudaStream_t st = as_stream(stream);
  int64_t B, bpr;
  block_geometry(K, block, B, bpr);
  const int vec = rows_vectorizable(W, ldw);
  if (LPQT_FUSED_QUANT && bpr == 1 && vec && K % 8 == 0 && K <= 16384) {  // CGQ: one fused pass (scales + encode, W read once)
    const int64_t ng = (N + kQRows - 1) / kQRows;
    LPQT_DISPATCH_DT(dtype, (quantize_fused_kernel<DT, false><<<fused_grid(ng, K), 256, 0, st>>>(
                                W, N, K, ldw, 28.0, bias_shift, scales, folded, dev_flags, ng, 0, seg4, seg2)));
    note_launch();
    return check_launch();
  }
  rc = quantize_scales(W, dtype, N, K, ldw, B, bpr, vec, bias_shift, scales, folded, dev_flags, st);
  if (rc != LPQT_OK) return rc;
  const int64_t groups = (N * K + 7) / 8;
  const int pv = vec && (K % 8 == 0) && (B % 8 == 0);
  LPQT_DISPATCH_DT(dtype, encode_planes_kernel<DT><<<grid_for(groups, 256), 256, 0, st>>>(W, N, K, ldw, pv, B, bpr,
                                                                                         scales, seg4, seg2));
  note_launch();
  return check_launch();
}

int lpqt_fp6_quantize_pack(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int bias_shift,
                           uint16_t* scales, uint16_t* folded, uint8_t* seg4, uint8_t* seg2, uint8_t* codes_ws,
                           uint32_t* dev_flags, void* stream) {
  (void)codes_ws;  // no longer needed (ABI v1 argument)
  return lpqt_fp6_quantize_pack_blocks(W, dtype, N, K, ldw, 0, bias_shift, scales, folded, seg4, seg2, dev_flags,
                                       stream);
}

int lpqt_fp6_quantize_tiles_blocks(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int64_t block,
                                   int bias_shift, uint16_t* scales, uint16_t* folded, uint8_t* tiles,
                                   uint32_t* dev_flags, void* stream) {
  int rc = check_quantize_args(W, dtype, N, K, ldw, bias_shift, folded);
  if (rc != LPQT_OK || N == 0 || K == 0) return rc;
  if (tiles == nullptr || scales == nullptr) return LPQT_E_INVALID_INPUT;
  const cudaStream_t st = as_stream(stream);
  int64_t B, bpr;
  block_geometry(K, block, B, bpr);
  const int vec = rows_vectorizable(W, ldw);
  const int64_t Np = (N + kTileN - 1) / kTileN * kTileN, k_tiles = (K + kTileK - 1) / kTileK;
  if (LPQT_FUSED_QUANT && bpr == 1 && vec && K % 8 == 0 && K <= 16384) {  // CGQ: one fused pass (scales + encode, W read once)
    const int64_t ng = Np / kQRows;  // (padding rows get code 0)
    LPQT_DISPATCH_DT(dtype, (quantize_fused_kernel<DT, true><<<fused_grid(ng, K), 256, 0, st>>>(
                                W, N, K, ldw, 28.0, bias_shift, scales, folded, dev_flags, ng, k_tiles, tiles,
                                nullptr)));
    note_launch();
    return check_launch();
  }
  rc = quantize_scales(W, dtype, N, K, ldw, B, bpr, vec, bias_shift, scales, folded, dev_flags, st);
  if (rc != LPQT_OK) return rc;
  const int64_t threads = Np * k_tiles * 2;
  const int tv = vec && (B % 8 == 0);
  LPQT_DISPATCH_DT(dtype, encode_tiles_kernel<DT><<<grid_for(threads, 256), 256, 0, st>>>(W, N, K, ldw, tv, B, bpr,
                                                                                         scales, Np, k_tiles, tiles));
  note_launch();
  return check_launch();
}

int lpqt_fp6_quantize_tiles(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int bias_shift,
                            uint16_t* scales, uint16_t* folded, uint8_t* tiles, uint32_t* dev_flags, void* stream) {
  return lpqt_fp6_quantize_tiles_blocks(W, dtype, N, K, ldw, 0, bias_shift, scales, folded, tiles, dev_flags,
                                        stream);
}

int lpqt_fp6_dequantize_tensor_blocks(const uint8_t* seg4, const uint8_t* seg2, const uint16_t* block_scale,
                                      int path, int64_t N, int64_t K, int64_t block, void* out, int out_dtype,
                                      void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (path != 0 && path != 1) return LPQT_E_INVALID_INPUT;
  if (N * K == 0) return LPQT_OK;
  int64_t B, bpr;
  block_geometry(K, block, B, bpr);
  const int g = grid_for(N * K, 256);
  if (out_dtype == LPQT_F64) {
    dequantize_tensor_kernel<LPQT_F64><<<g, 256, 0, as_stream(stream)>>>(seg4, seg2, block_scale, path, N, K, B, bpr,
                                                                          out);
  } else if (out_dtype == LPQT_F16) {
    dequantize_tensor_kernel<LPQT_F16><<<g, 256, 0, as_stream(stream)>>>(seg4, seg2, block_scale, path, N, K, B, bpr,
                                                                          out);
  } else {
    return LPQT_E_UNSUPPORTED;
  }
  note_launch();
  return check_launch();
}

int lpqt_fp6_dequantize_tensor(const uint8_t* seg4, const uint8_t* seg2, const uint16_t* row_scale, int path,
                               int64_t N, int64_t K, void* out, int out_dtype, void* stream) {
  return lpqt_fp6_dequantize_tensor_blocks(seg4, seg2, row_scale, path, N, K, 0, out, out_dtype, stream);
}

int lpqt_stage_activations(const void* X, int dtype, int64_t K, int64_t M, int64_t ldx, uint16_t* Xt, int64_t Kp,
                           void* stream) {
  if (K < 0 || M < 0 || Kp < K || ldx < M) return LPQT_E_SHAPE;
  if (M * Kp == 0) return LPQT_OK;
  const int g = grid_for(M * Kp, 256);
  LPQT_DISPATCH_DT(dtype, stage_activations_kernel<DT><<<g, 256, 0, as_stream(stream)>>>(X, K, M, ldx, Xt, Kp));
  note_launch();
  return check_launch();
}


// ---- FP5 e3m1 (4 + 1) --------------------------------------------------------
int64_t lpqt_fp5_tail_length(int64_t n) { return ((n + 7) / 8 + 3) / 4 * 4; }

int lpqt_fp5_encode_rtn(const void* x, int dtype, int64_t n, uint8_t* codes, uint32_t* dev_flags, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  LPQT_DISPATCH_DT(dtype, fp5_encode_kernel<DT><<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(x, n, codes,
                                                                                                  dev_flags));
  note_launch();
  return check_launch();
}

int lpqt_fp5_pack(const uint8_t* codes, int64_t n, uint8_t* seg4, uint8_t* seg1, uint32_t* dev_flags, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  const int64_t len4 = lpqt_fp6_seg4_length(n), len1 = lpqt_fp5_tail_length(n);
  if (len4 == 0) return LPQT_OK;
  const int64_t groups = (len4 * 2 + 7) / 8 > len1 ? (len4 * 2 + 7) / 8 : len1;
  fp5_pack_kernel<<<grid_for(groups, 256), 256, 0, as_stream(stream)>>>(codes, n, len4, len1, seg4, seg1, dev_flags);
  note_launch();
  return check_launch();
}

int lpqt_fp5_unpack(const uint8_t* seg4, const uint8_t* seg1, int64_t n, uint8_t* codes, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  fp5_unpack_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(seg4, seg1, n, codes);
  note_launch();
  return check_launch();
}

int lpqt_fp5_quantize_pack_blocks(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int64_t block,
                                  int bias_shift, uint16_t* scales, uint16_t* folded, uint8_t* seg4, uint8_t* seg1,
                                  uint32_t* dev_flags, void* stream) {
  int rc = check_quantize_args(W, dtype, N, K, ldw, bias_shift, folded);
  if (rc != LPQT_OK || N == 0 || K == 0) return rc;
  const cudaStream_t st = as_stream(stream);
  int64_t B, bpr;
  block_geometry(K, block, B, bpr);
  rc = quantize_scales(W, dtype, N, K, ldw, B, bpr, rows_vectorizable(W, ldw), bias_shift, scales, folded, dev_flags,
                       st, 24.0);
  if (rc != LPQT_OK) return rc;
  const int64_t len4 = lpqt_fp6_seg4_length(N * K), len1 = lpqt_fp5_tail_length(N * K);
  const int64_t groups = (N * K + 7) / 8;
  LPQT_DISPATCH_DT(dtype, fp5_encode_planes_kernel<DT><<<grid_for(groups, 256), 256, 0, st>>>(
                              W, N, K, ldw, B, bpr, scales, len4, len1, seg4, seg1));
  note_launch();
  return check_launch();
}

int lpqt_fp5_dequantize_tensor_blocks(const uint8_t* seg4, const uint8_t* seg1, const uint16_t* block_scale, int path,
                                      int64_t N, int64_t K, int64_t block, void* out, int out_dtype, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (path != 0 && path != 1) return LPQT_E_INVALID_INPUT;
  if (N * K == 0) return LPQT_OK;
  int64_t B, bpr;
  block_geometry(K, block, B, bpr);
  const int g = grid_for(N * K, 256);
  if (out_dtype == LPQT_F64) {
    fp5_dequantize_tensor_kernel<LPQT_F64><<<g, 256, 0, as_stream(stream)>>>(seg4, seg1, block_scale, path, N, K, B,
                                                                              bpr, out);
  } else if (out_dtype == LPQT_F16) {
    fp5_dequantize_tensor_kernel<LPQT_F16><<<g, 256, 0, as_stream(stream)>>>(seg4, seg1, block_scale, path, N, K, B,
                                                                              bpr, out);
  } else {
    return LPQT_E_UNSUPPORTED;
  }
  note_launch();
  return check_launch();
}

int lpqt_fp5_dequant_bias_shift(const uint8_t* codes, const uint16_t* folded, int64_t n, uint16_t* out,
                                void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  fp5_dequant_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(codes, folded, 1, n, out);
  note_launch();
  return check_launch();
}

int lpqt_fp5_dequant_naive(const uint8_t* codes, const uint16_t* scales, int64_t n, uint16_t* out, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  fp5_dequant_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(codes, scales, 0, n, out);
  note_launch();
  return check_launch();
}


// ---- INT4 asymmetric (comparator path) --------------------------------------
int lpqt_int4_quantize_blocks(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int64_t block,
                              uint16_t* scales, uint16_t* zeros, uint8_t* nibbles, uint32_t* dev_flags,
                              void* stream) {
  if (N < 0 || K < 0 || ldw < K) return LPQT_E_SHAPE;
  if (dtype < LPQT_F64 || dtype > LPQT_BF16) return LPQT_E_UNSUPPORTED;
  if (N == 0 || K == 0) return LPQT_OK;
  const cudaStream_t st = as_stream(stream);
  int64_t B, bpr;
  block_geometry(K, block, B, bpr);
  const int64_t units = N * bpr;
  const int g = static_cast<int>((units + 7) / 8 < 148 * 8 ? (units + 7) / 8 : 148 * 8);
  LPQT_DISPATCH_DT(dtype, int4_block_params_kernel<DT><<<g, 256, 0, st>>>(W, N, K, ldw, B, bpr, scales, zeros,
                                                                           dev_flags));
  note_launch();
  int rc = check_launch();
  if (rc != LPQT_OK) return rc;
  const int64_t len = (N * K + 1) / 2, groups = (N * K + 7) / 8;
  LPQT_DISPATCH_DT(dtype, int4_encode_kernel<DT><<<grid_for(groups, 256), 256, 0, st>>>(W, N, K, ldw, B, bpr, scales,
                                                                                       zeros, len, nibbles));
  note_launch();
  return check_launch();
}

int lpqt_int4_pack(const uint8_t* levels, int64_t n, uint8_t* nibbles, uint32_t* dev_flags, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  int4_pack_kernel<<<grid_for((n + 1) / 2, 256), 256, 0, as_stream(stream)>>>(levels, n, nibbles, dev_flags);
  note_launch();
  return check_launch();
}

int lpqt_int4_unpack(const uint8_t* nibbles, int64_t n, uint8_t* levels, void* stream) {
  if (n < 0) return LPQT_E_SHAPE;
  if (n == 0) return LPQT_OK;
  int4_unpack_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(nibbles, n, levels);
  note_launch();
  return check_launch();
}

int lpqt_int4_dequantize_blocks(const uint8_t* nibbles, const uint16_t* scales, const uint16_t* zeros, int64_t N,
                                int64_t K, int64_t block, double* out, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N * K == 0) return LPQT_OK;
  int64_t B, bpr;
  block_geometry(K, block, B, bpr);
  int4_dequantize_kernel<<<grid_for(N * K, 256), 256, 0, as_stream(stream)>>>(nibbles, scales, zeros, N, K, B, bpr,
                                                                              out);
  note_launch();
  return check_launch();
}

}  // extern "C"
