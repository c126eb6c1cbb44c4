// exact.cu — the reference's GEMM arithmetic, operation for operation, on the
// GPU (gemm.py:28-110).
//
// The tcgen05 kernel (gemm.cu) is the product path: fp16 activations, fp32
// tensor-core accumulation in its own order, equal to the reference up to
// summation order.  The reference API, however, also accepts float32 (and
// float64) activations and FGQ blocks of any width, and its own tests hold
// the result to 4 eps32 K max|W| max|X| elementwise.  These kernels cover
// exactly those calls by replaying the reference's loops: one thread per
// output element, k ascending, every product and sum rounded separately
// (__fmul_rn / __fadd_rn: numpy never contracts to FMA), so the result is
// bit-identical to the reference on the same inputs:
//
//   gemm_quantized CGQ   acc += raw[n,k] * X[k,m];  Y = S[n] * acc
//                        (INT4: + Z[n] * sum_k X[k,m])                gemm.py:81-94
//   gemm_quantized FGQ   per block b: partial = sum_{k in b} raw * X (k asc.);
//                        Y += S[n,b] * partial (INT4: + Z[n,b] * sum_b X)  gemm.py:96-110
//   gemm_dense           f32  acc += W[n,k] * X[k,m]                   gemm.py:41-51
//   gemm_reference       f64  acc += W[n,k] * X[k,m]                   gemm.py:28-38
//
// They are CUDA-core kernels (no tensor cores): the fast path for fp16
// activations is the W6A16 GEMM; these run the reference-API calls the A16
// kernel cannot reproduce within the reference's tolerance.
#include "common.cuh"

namespace lpqt {

// raw code value of a sign-magnitude minifloat (codec.py:63-82): e exponent
// bits, m mantissa bits, bias 2^(e-1) - 1; value = (1 + M/2^m) 2^(E-bias),
// subnormal (E = 0) M/2^m * 2^(1-bias); sign bit above the magnitude
__host__ __device__ inline float minifloat_value(uint32_t c, int ebits, int mbits) {
  const int bias = (1 << (ebits - 1)) - 1;
  const uint32_t mag = c & ((1u << (ebits + mbits)) - 1u);
  const int E = static_cast<int>(mag >> mbits);
  const int M = static_cast<int>(mag & ((1u << mbits) - 1u));
  const float frac = static_cast<float>(M) / static_cast<float>(1 << mbits);
  const float v = E == 0 ? ldexpf(frac, 1 - bias) : ldexpf(1.0f + frac, E - bias);
  return ((c >> (ebits + mbits)) & 1u) ? -v : v;
}

// fmt: 0 = FP6 e3m2, 1 = FP5 e3m1, 2 = INT4 level (codes = levels 0..15)
__global__ void gemm_exact_quantized_kernel(const uint8_t* __restrict__ codes, int fmt,
                                            const uint16_t* __restrict__ scales,
                                            const uint16_t* __restrict__ zeros, int64_t N, int64_t K,
                                            int64_t block, int64_t bpr, const float* __restrict__ X, int64_t M,
                                            float* __restrict__ Y) {
  __shared__ float table[64];
  if (threadIdx.x < 64) {
    const uint32_t c = threadIdx.x;
    table[c] = fmt == 0 ? minifloat_value(c, 3, 2)
                        : (fmt == 1 ? minifloat_value(c & 31u, 3, 1) : static_cast<float>(c & 15u));
  }
  __syncthreads();
  const bool int4 = fmt == 2;
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < N * M; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = o / M, m = o - n * M;
    const uint8_t* crow = codes + n * K;
    if (block <= 0) {  // CGQ: scale once after the whole row (gemm.py:81-94)
      float acc = 0.f, sx = 0.f;
      for (int64_t k = 0; k < K; ++k) {
        const float x = X[k * M + m];
        acc = __fadd_rn(acc, __fmul_rn(table[crow[k]], x));
        if (int4) sx = __fadd_rn(sx, x);
      }
      float out = __fmul_rn(__half2float(__ushort_as_half(scales[n])), acc);
      if (int4) out = __fadd_rn(out, __fmul_rn(__half2float(__ushort_as_half(zeros[n])), sx));
      Y[o] = out;
    } else {  // FGQ: block partials scaled before accumulation (gemm.py:96-110)
      float out = 0.f;
      for (int64_t b = 0; b < bpr; ++b) {
        const int64_t k0 = b * block, k1 = min(K, k0 + block);
        float part = 0.f, sx = 0.f;
        for (int64_t k = k0; k < k1; ++k) {
          const float x = X[k * M + m];
          part = __fadd_rn(part, __fmul_rn(table[crow[k]], x));
          if (int4) sx = __fadd_rn(sx, x);
        }
        float contrib = __fmul_rn(__half2float(__ushort_as_half(scales[n * bpr + b])), part);
        if (int4) contrib = __fadd_rn(contrib, __fmul_rn(__half2float(__ushort_as_half(zeros[n * bpr + b])), sx));
        out = __fadd_rn(out, contrib);
      }
      Y[o] = out;
    }
  }
}

template <typename T>
__device__ __forceinline__ T mul_rn(T a, T b);
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) { return __fmul_rn(a, b); }
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) { return __dmul_rn(a, b); }
template <typename T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }

template <typename T>
__global__ void gemm_exact_dense_kernel(const T* __restrict__ W, const T* __restrict__ X, int64_t N, int64_t K,
                                        int64_t M, T* __restrict__ Y) {
  for (int64_t o = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; o < N * M; o += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = o / M, m = o - n * M;
    T acc = T(0);
    for (int64_t k = 0; k < K; ++k) acc = add_rn<T>(acc, mul_rn<T>(W[n * K + k], X[k * M + m]));
    Y[o] = acc;
  }
}

}  // namespace lpqt

using namespace lpqt;

extern "C" {

int lpqt_gemm_exact_quantized(const uint8_t* codes, int fmt, const uint16_t* scales, const uint16_t* zeros,
                              int64_t N, int64_t K, int64_t block, const float* X, int64_t M, float* Y,
                              void* stream) {
  if (N < 0 || K < 0 || M < 0) return LPQT_E_SHAPE;
  if (fmt < 0 || fmt > 2) return LPQT_E_UNSUPPORTED;
  if (fmt == 2 && zeros == nullptr) return LPQT_E_INVALID_INPUT;
  if (N == 0 || M == 0) return LPQT_OK;
  const int64_t blk = (block > 0 && block < K) ? block : 0;
  const int64_t bpr = blk ? (K + blk - 1) / blk : 1;
  const int threads = 128;
  gemm_exact_quantized_kernel<<<grid_for(N * M, threads), threads, 0, as_stream(stream)>>>(
      codes, fmt, scales, zeros, N, K, blk, bpr, X, M, Y);
  note_launch();
  return check_launch();
}

int lpqt_gemm_exact_dense(const void* W, const void* X, int dtype, int64_t N, int64_t K, int64_t M, void* Y,
                          void* stream) {
  if (N < 0 || K < 0 || M < 0) return LPQT_E_SHAPE;
  if (dtype != LPQT_F32 && dtype != LPQT_F64) return LPQT_E_UNSUPPORTED;
  if (N == 0 || M == 0) return LPQT_OK;
  const int threads = 128;
  if (dtype == LPQT_F32) {
    gemm_exact_dense_kernel<float><<<grid_for(N * M, threads), threads, 0, as_stream(stream)>>>(
        static_cast<const float*>(W), static_cast<const float*>(X), N, K, M, static_cast<float*>(Y));
  } else {
    gemm_exact_dense_kernel<double><<<grid_for(N * M, threads), threads, 0, as_stream(stream)>>>(
        static_cast<const double*>(W), static_cast<const double*>(X), N, K, M, static_cast<double*>(Y));
  }
  note_launch();
  return check_launch();
}

}  // extern "C"
