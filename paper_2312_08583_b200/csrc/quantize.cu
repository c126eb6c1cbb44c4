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

// ---- K1: fused per-row quantize ----------------------------------------------
// One CTA per row (grid-stride): pass 1 row max|w| + finiteness, pass 2
// encode + pack.  K % 8 == 0: each thread packs 8 codes -> 4 seg4 bytes
// (one u32) + 2 seg2 bytes (one u16), rows are byte aligned.  Otherwise codes
// go to `codes_ws` and the flat pack kernel runs afterwards.
template <int DT>
__global__ void __launch_bounds__(256) quantize_rows_kernel(const void* __restrict__ W, int64_t N, int64_t K,
                                                            int64_t ldw, int bias_shift, uint16_t* __restrict__ scales,
                                                            uint16_t* __restrict__ folded, uint8_t* __restrict__ seg4,
                                                            uint8_t* __restrict__ seg2, uint8_t* __restrict__ codes_ws,
                                                            uint32_t* __restrict__ flags) {
  __shared__ double mids[32];
  __shared__ double red[8];
  __shared__ double s_scale;
  load_mids(mids);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool fused = (K % 8) == 0;
  for (int64_t r = blockIdx.x; r < N; r += gridDim.x) {
    const char* row = static_cast<const char*>(W);
    const int64_t base = r * ldw;
    // pass 1: peak (quantizer.py:225) and finiteness (quantizer.py:200)
    double peak = 0.0;
    bool bad = false;
    for (int64_t k = tid; k < K; k += blockDim.x) {
      const double v = load_as_double<DT>(row, base + k);
      if (!isfinite(v)) bad = true;
      peak = fmax(peak, fabs(v));
    }
    if (__syncthreads_or(bad)) {
      if (tid == 0) atomicOr(flags, LPQT_F_NONFINITE);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) peak = fmax(peak, __shfl_xor_sync(0xffffffffu, peak, o));
    if (lane == 0) red[wid] = peak;
    __syncthreads();
    if (tid == 0) {
      double p = red[0];
      for (int i = 1; i < (int)(blockDim.x >> 5); ++i) p = fmax(p, red[i]);
      // quantizer.py:227 + _round_scales_f16 (:142-153)
      const double raw = (p == 0.0) ? 1.0 : p / 28.0;
      __half s = __double2half(raw);
      uint16_t sb = __half_as_ushort(s);
      if ((sb & 0x7FFFu) == 0x7C00u) {
        atomicOr(flags, LPQT_F_SCALE_INF);
      }
      if ((sb & 0x7FFFu) == 0) sb = 0x0001u;  // underflow clamps to 2^-24
      scales[r] = sb;
      const double sd = static_cast<double>(__half2float(__ushort_as_half(sb)));
      if (bias_shift) {
        // dequant.py:61-69: folded = S * 2^12, overflow above 65504
        const double f = sd * 4096.0;
        if (f > 65504.0) atomicOr(flags, LPQT_F_FOLD_OVERFLOW);
        folded[r] = (f > 65504.0) ? (uint16_t)0x7C00u : __half_as_ushort(__double2half(f));
      }
      s_scale = sd;
    }
    __syncthreads();
    const double S = s_scale;
    // pass 2: codes = encode(W / S) (quantizer.py:228-229, f64 division)
    if (fused) {
      const int64_t groups = K / 8;
      for (int64_t g = tid; g < groups; g += blockDim.x) {
        uint32_t c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = fp6_encode(load_as_double<DT>(row, base + g * 8 + j) / S, mids);
        uint32_t s4 = 0, s2 = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          s4 |= (c[j] >> 2) << (4 * j);
          s2 |= (c[j] & 3u) << (2 * j);
        }
        const int64_t i0 = r * K + g * 8;
        *reinterpret_cast<uint32_t*>(seg4 + i0 / 2) = s4;
        *reinterpret_cast<uint16_t*>(seg2 + i0 / 4) = static_cast<uint16_t>(s2);
      }
    } else {
      for (int64_t k = tid; k < K; k += blockDim.x) {
        codes_ws[r * K + k] = static_cast<uint8_t>(fp6_encode(load_as_double<DT>(row, base + k) / S, mids));
      }
    }
    __syncthreads();
  }
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
                                         void* __restrict__ out) {
  const int64_t total = N * K;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t c = canon_code(seg4, seg2, i);
    const int64_t r = i / K;
    const __half comp = __ushort_as_half(fp6_compose_bits(c));
    const __half s = __ushort_as_half(row_scale[r]);
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

int lpqt_fp6_quantize_pack(const void* W, int dtype, int64_t N, int64_t K, int64_t ldw, int bias_shift,
                           uint16_t* scales, uint16_t* folded, uint8_t* seg4, uint8_t* seg2, uint8_t* codes_ws,
                           uint32_t* dev_flags, void* stream) {
  if (N < 0 || K < 0 || ldw < K) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  if (K % 8 != 0 && codes_ws == nullptr) return LPQT_E_WORKSPACE;
  if (bias_shift && folded == nullptr) return LPQT_E_INVALID_INPUT;
  const int g = static_cast<int>(N < 148 * 16 ? N : 148 * 16);
  LPQT_DISPATCH_DT(dtype, quantize_rows_kernel<DT><<<g, 256, 0, as_stream(stream)>>>(
                              W, N, K, ldw, bias_shift, scales, folded, seg4, seg2, codes_ws, dev_flags));
  note_launch();
  int st = check_launch();
  if (st != LPQT_OK || K % 8 == 0) return st;
  return lpqt_fp6_pack(codes_ws, N * K, seg4, seg2, dev_flags, stream);
}

int lpqt_fp6_dequantize_tensor(const uint8_t* seg4, const uint8_t* seg2, const uint16_t* row_scale, int path,
                               int64_t N, int64_t K, void* out, int out_dtype, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (path != 0 && path != 1) return LPQT_E_INVALID_INPUT;
  if (N * K == 0) return LPQT_OK;
  const int g = grid_for(N * K, 256);
  if (out_dtype == LPQT_F64) {
    dequantize_tensor_kernel<LPQT_F64><<<g, 256, 0, as_stream(stream)>>>(seg4, seg2, row_scale, path, N, K, out);
  } else if (out_dtype == LPQT_F16) {
    dequantize_tensor_kernel<LPQT_F16><<<g, 256, 0, as_stream(stream)>>>(seg4, seg2, row_scale, path, N, K, out);
  } else {
    return LPQT_E_UNSUPPORTED;
  }
  note_launch();
  return check_launch();
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

}  // extern "C"
