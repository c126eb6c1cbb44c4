// prepack.cu — K2 (canonical 4+2 planes -> B200 tile layout), its inverse,
// and K3 (the standalone register transform, tiles -> binary16).
//
// The canonical planes (packing.py:63-90) are the reference's storage format
// and stay the parity artifact.  The GEMM instead streams 128x128 weight
// tiles of 12288 contiguous bytes (one 1-D bulk copy each) whose bit order is
// chosen so the in-register FP6 -> FP16 rebuild is the hardware e3m2 converter
// plus a cheap spare-bit gather (~0.8 ALU ops per weight; fp6x32_cvt_f16x32 in
// common.cuh).  K3 runs exactly that transform and multiplies by S in
// binary16: value_f16[c] * S (dequant_naive_array, dequant.py:72-79), which
// the reference proves bit-identical to the bias-shift path
// compose[c] * (S * 2^12) (dequant.py:82-86; pkg/tests/test_dequant.py:93-102).
#include "common.cuh"

namespace lpqt {

__device__ __forceinline__ uint32_t canon_code_at(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg2,
                                                  int64_t i) {
  const uint32_t hi = (seg4[i >> 1] >> (4 * (i & 1))) & 15u;
  const uint32_t lo = (seg2[i >> 2] >> (2 * (i & 3))) & 3u;
  return (hi << 2) | lo;
}

// one thread per (row n < Np, 32-weight group g < Kp/32)
__global__ void prepack_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg2, int64_t N,
                               int64_t K, int64_t Np, int64_t Kp, uint8_t* __restrict__ tiles) {
  const int64_t groups = Kp / 32, total = Np * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / groups, g = t % groups;
    uint8_t c[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t k = g * 32 + j;
      c[j] = (n < N && k < K) ? static_cast<uint8_t>(canon_code_at(seg4, seg2, n * K + k)) : 0;
    }
    uint32_t w[6];
    fp6x32_pack_words(c, w);
#pragma unroll
    for (int i = 0; i < 6; ++i) *reinterpret_cast<uint32_t*>(tiles + tile_word_addr(n, g, i, k_tiles)) = w[i];
  }
}

// K % 32 == 0 and 16-B aligned planes: a 32-weight group is 16 B of seg4 and
// 8 B of seg2 (one vector load each); rows fastest across the warp so the
// tile stores of a warp land in one [khalf][quad] plane (128 rows x 16 B)
__global__ void prepack_vec_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg2, int64_t N,
                                   int64_t K, int64_t Np, int64_t Kp, uint8_t* __restrict__ tiles) {
  const int64_t groups = Kp / 32, total = Np * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t rr = t % kTileN, rest = t / kTileN;  // rows fastest inside a 128-row tile
    const int64_t g = rest % groups, n = (rest / groups) * kTileN + rr;
    uint8_t c[32];
    if (n < N && 32 * g < K) {
      const int64_t i0 = n * K + 32 * g;
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(seg4 + i0 / 2));
      const uint2 b = __ldg(reinterpret_cast<const uint2*>(seg2 + i0 / 4));
      const uint32_t s4[4] = {a.x, a.y, a.z, a.w}, s2[2] = {b.x, b.y};
#pragma unroll
      for (int j = 0; j < 32; ++j)
        c[j] = static_cast<uint8_t>((((s4[j >> 3] >> (4 * (j & 7))) & 15u) << 2) | ((s2[j >> 4] >> (2 * (j & 15))) & 3u));
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j) c[j] = 0;
    }
    uint32_t w[6];
    fp6x32_pack_words(c, w);
#pragma unroll
    for (int i = 0; i < 6; ++i) *reinterpret_cast<uint32_t*>(tiles + tile_word_addr(n, g, i, k_tiles)) = w[i];
  }
}

__device__ __forceinline__ void load_group(const uint8_t* __restrict__ tiles, int64_t n, int64_t g, int64_t k_tiles,
                                           uint32_t w[6]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) w[i] = *reinterpret_cast<const uint32_t*>(tiles + tile_word_addr(n, g, i, k_tiles));
}

// exact inverse of prepack over the valid region -> row-major codes[N, K]
__global__ void unprepack_kernel(const uint8_t* __restrict__ tiles, int64_t N, int64_t K, int64_t Kp,
                                 uint8_t* __restrict__ codes) {
  const int64_t groups = Kp / 32, total = N * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / groups, g = t % groups;
    uint32_t w[6];
    uint8_t c[32];
    load_group(tiles, n, g, k_tiles, w);
    fp6x32_unpack_codes(w, c);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t k = g * 32 + j;
      if (k < K) codes[n * K + k] = c[j];
    }
  }
}

// K3: tiles -> out[N, K] binary16 = value_f16[c] * S[n] (the GEMM's transform)
// scales: one per (row, block of B columns), B = K for CGQ
__global__ void tiles_dequant_kernel(const uint8_t* __restrict__ tiles, const uint16_t* __restrict__ scales,
                                     int64_t N, int64_t K, int64_t Kp, int64_t B, int64_t bpr,
                                     uint16_t* __restrict__ out) {
  const int64_t groups = Kp / 32, total = N * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / groups, g = t % groups;
    uint32_t w[6], h[16];
    load_group(tiles, n, g, k_tiles, w);
    fp6x32_cvt_f16x32(w, h);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const __half2 v = *reinterpret_cast<const __half2*>(&h[j]);
      const int64_t k = g * 32 + 2 * j;
      if (k < K)
        out[n * K + k] = __half_as_ushort(__hmul(__low2half(v), __ushort_as_half(scales[n * bpr + k / B])));
      if (k + 1 < K)
        out[n * K + k + 1] =
            __half_as_ushort(__hmul(__high2half(v), __ushort_as_half(scales[n * bpr + (k + 1) / B])));
    }
  }
}


// FP5 e3m1 planes (seg4 = c >> 1, one tail bit per code) -> the FP6 tile
// layout: e3m1 code (s, e, m) is the e3m2 code (s, e, m << 1) of the same value
__global__ void prepack_fp5_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg1, int64_t N,
                                   int64_t K, int64_t Np, int64_t Kp, uint8_t* __restrict__ tiles) {
  const int64_t groups = Kp / 32, total = Np * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / groups, g = t % groups;
    uint8_t c[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t k = g * 32 + j, i = n * K + k;
      uint32_t c6 = 0;
      if (n < N && k < K) {
        const uint32_t c5 = (((seg4[i >> 1] >> (4 * (i & 1))) & 15u) << 1) | ((seg1[i >> 3] >> (i & 7)) & 1u);
        c6 = ((c5 & 0x10u) << 1) | (((c5 >> 1) & 7u) << 2) | ((c5 & 1u) << 1);
      }
      c[j] = static_cast<uint8_t>(c6);
    }
    uint32_t w[6];
    fp6x32_pack_words(c, w);
#pragma unroll
    for (int i = 0; i < 6; ++i) *reinterpret_cast<uint32_t*>(tiles + tile_word_addr(n, g, i, k_tiles)) = w[i];
  }
}


// FP5 e3m1 planes -> the native 5-bit tiles (common.cuh: 0.625 B per weight)
__global__ void prepack_fp5n_kernel(const uint8_t* __restrict__ seg4, const uint8_t* __restrict__ seg1, int64_t N,
                                    int64_t K, int64_t Np, int64_t Kp, uint8_t* __restrict__ tiles) {
  const int64_t groups = Kp / 32, total = Np * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / groups, g = t % groups;
    uint8_t c[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t k = g * 32 + j, i = n * K + k;
      c[j] = (n < N && k < K) ? static_cast<uint8_t>((((seg4[i >> 1] >> (4 * (i & 1))) & 15u) << 1) |
                                                     ((seg1[i >> 3] >> (i & 7)) & 1u))
                              : 0;
    }
    uint32_t nib[4], mw;
    fp5x32_pack_words(c, nib, mw);
#pragma unroll
    for (int i = 0; i < 4; ++i) *reinterpret_cast<uint32_t*>(tiles + tile5_word_addr(n, g, i, k_tiles)) = nib[i];
    *reinterpret_cast<uint32_t*>(tiles + tile5_word_addr(n, g, 4, k_tiles)) = mw;
  }
}

__device__ __forceinline__ void load_group5(const uint8_t* __restrict__ tiles, int64_t n, int64_t g, int64_t k_tiles,
                                            uint32_t nib[4], uint32_t& mw) {
#pragma unroll
  for (int i = 0; i < 4; ++i) nib[i] = *reinterpret_cast<const uint32_t*>(tiles + tile5_word_addr(n, g, i, k_tiles));
  mw = *reinterpret_cast<const uint32_t*>(tiles + tile5_word_addr(n, g, 4, k_tiles));
}

// native FP5 tiles -> row-major e3m1 codes[N, K]
__global__ void unprepack_fp5n_kernel(const uint8_t* __restrict__ tiles, int64_t N, int64_t K, int64_t Kp,
                                      uint8_t* __restrict__ codes) {
  const int64_t groups = Kp / 32, total = N * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / groups, g = t % groups;
    uint32_t nib[4], mw;
    uint8_t c[32];
    load_group5(tiles, n, g, k_tiles, nib, mw);
    fp5x32_unpack_codes(nib, mw, c);
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      const int64_t k = g * 32 + j;
      if (k < K) codes[n * K + k] = c[j];
    }
  }
}

// native FP5 tiles -> out[N, K] binary16 = value_f16[c] * S[n] through the GEMM's rebuild
__global__ void tiles5_dequant_kernel(const uint8_t* __restrict__ tiles, const uint16_t* __restrict__ scales,
                                      int64_t N, int64_t K, int64_t Kp, uint16_t* __restrict__ out, ShiftMuls sm) {
  const int64_t groups = Kp / 32, total = N * groups, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / groups, g = t % groups;
    uint32_t nib[4], mw, h[16];
    load_group5(tiles, n, g, k_tiles, nib, mw);
    fp5x32_cvt_f16x32(nib, mw, h, sm);
    const __half S = __ushort_as_half(scales[n]);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const __half2 v = *reinterpret_cast<const __half2*>(&h[j]);
      const int64_t k = g * 32 + 2 * j;
      if (k < K) out[n * K + k] = __half_as_ushort(__hmul(__low2half(v), S));
      if (k + 1 < K) out[n * K + k + 1] = __half_as_ushort(__hmul(__high2half(v), S));
    }
  }
}

// INT4 nibbles (row-major, two per byte, packing.py:121-129) -> INT4 tiles:
// 128 x 128 tiles of 8192 B, [k-half 2][quad 2][row 128][16 B]; word w of a
// (row, k-half) holds weights 8w .. 8w + 7 with weight 8w + j in nibble
// (j >> 1) + 4 (j & 1), the order the magic-number rebuild produces pairs in.
__global__ void prepack_int4_kernel(const uint8_t* __restrict__ nib, int64_t N, int64_t K, int64_t Np, int64_t Kp,
                                    uint8_t* __restrict__ tiles) {
  const int64_t words = Kp / 8, total = Np * words, k_tiles = Kp / kTileK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = t / words, w8 = t % words;
    uint32_t word = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t k = w8 * 8 + j;
      uint32_t lv = 0;
      if (n < N && k < K) {
        const int64_t i = n * K + k;
        lv = (nib[i >> 1] >> (4 * (i & 1))) & 15u;
      }
      word |= lv << (4 * ((j >> 1) + 4 * (j & 1)));
    }
    const int64_t kt = w8 / 16, rr = n % kTileN, rt = n / kTileN;
    const int wi = static_cast<int>(w8 % 16), khalf = wi / 8, quad = (wi % 8) / 4, wq = wi % 4;
    const int64_t off = (rt * k_tiles + kt) * (kTileN * kTileK / 2) + ((int64_t)(khalf * 2 + quad) * kTileN + rr) * 16 + wq * 4;
    *reinterpret_cast<uint32_t*>(tiles + off) = word;
  }
}


// Block parameters in GEMM stage order (FgqArgs, gemm.cu): entry
// (rt * k_tiles + kt) * 128 + r = the f16 scale (INT4: scale | zero << 16) of
// row rt * 128 + r in the block holding k tile kt; rows past N are 0.
// FP6 / FP5 (no zero points): each row's block scales are normalised by a
// power of two, S'_b = S_b * 2^-e_r with max_b S'_b in [2^10, 2^11), and
// 2^e_r (f32) is stored per row after the stage-ordered scales.  Exact
// (binary16 exponent shift) unless S_b < 2^-24 max_b S_b; the GEMM multiplies
// by 2^e_r in fp32, so the products and sums are the reference's scaled by a
// power of two (no binary16 under/overflow of v * S_b in the rebuilt weight).
__global__ void fgq_row_factor_kernel(const uint16_t* __restrict__ scales, int64_t N, int64_t Np, int64_t bpr,
                                      float* __restrict__ rowf) {
  for (int64_t n = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; n < Np; n += (int64_t)gridDim.x * blockDim.x) {
    float mx = 0.f;
    if (n < N)
      for (int64_t b = 0; b < bpr; ++b) mx = fmaxf(mx, __half2float(__ushort_as_half(scales[n * bpr + b])));
    // e = floor(log2(mx)) - 10 (mx a positive binary16 value: frexpf is exact)
    int ex = 0;
    frexpf(mx > 0.f ? mx : 1.f, &ex);  // mx = f * 2^ex, f in [0.5, 1)
    rowf[n] = ldexpf(1.f, ex - 1 - 10);
  }
}

__global__ void fgq_stage_params_kernel(const uint16_t* __restrict__ scales, const uint16_t* __restrict__ zeros,
                                        int64_t N, int64_t bpr, int64_t bkt, int64_t k_tiles, int64_t total,
                                        const float* __restrict__ rowf, void* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i % kTileN, t = i / kTileN, kt = t % k_tiles, n = (t / k_tiles) * kTileN + r;
    const int64_t b = n * bpr + kt / bkt;
    const uint32_t sc = n < N ? scales[b] : 0u;
    if (zeros) {
      static_cast<uint32_t*>(out)[i] = sc | (n < N ? static_cast<uint32_t>(zeros[b]) << 16 : 0u);
    } else {
      const float v = __half2float(__ushort_as_half(static_cast<uint16_t>(sc))) / rowf[n];  // exact: power of 2
      static_cast<uint16_t*>(out)[i] = __half_as_ushort(__float2half_rn(v));
    }
  }
}

}  // namespace lpqt

using namespace lpqt;

static inline int64_t round_up(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

extern "C" {

int64_t lpqt_fp6_tiles_bytes(int64_t N, int64_t K) {
  if (N <= 0 || K <= 0) return 0;
  return round_up(N, kTileN) / kTileN * (round_up(K, kTileK) / kTileK) * kTileBytes;
}

int lpqt_fp6_prepack(const uint8_t* seg4, const uint8_t* seg2, int64_t N, int64_t K, uint8_t* tiles, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Np = round_up(N, kTileN), Kp = round_up(K, kTileK);
  if (K % 32 == 0 && reinterpret_cast<uintptr_t>(seg4) % 16 == 0 && reinterpret_cast<uintptr_t>(seg2) % 8 == 0)
    prepack_vec_kernel<<<grid_for(Np * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(seg4, seg2, N, K, Np, Kp, tiles);
  else
    prepack_kernel<<<grid_for(Np * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(seg4, seg2, N, K, Np, Kp, tiles);
  note_launch();
  return check_launch();
}

int lpqt_fp6_unprepack(const uint8_t* tiles, int64_t N, int64_t K, uint8_t* codes, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Kp = round_up(K, kTileK);
  unprepack_kernel<<<grid_for(N * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(tiles, N, K, Kp, codes);
  note_launch();
  return check_launch();
}

int lpqt_fp6_tiles_dequant_blocks(const uint8_t* tiles, const uint16_t* scales, int64_t N, int64_t K, int64_t block,
                                  uint16_t* out, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Kp = round_up(K, kTileK);
  const int64_t B = (block <= 0 || block >= K) ? K : block, bpr = (K + B - 1) / B;
  tiles_dequant_kernel<<<grid_for(N * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(tiles, scales, N, K, Kp, B, bpr,
                                                                                     out);
  note_launch();
  return check_launch();
}

int lpqt_fp6_tiles_dequant(const uint8_t* tiles, const uint16_t* scales, int64_t N, int64_t K, uint16_t* out,
                           void* stream) {
  return lpqt_fp6_tiles_dequant_blocks(tiles, scales, N, K, 0, out, stream);
}


int lpqt_fp5_prepack(const uint8_t* seg4, const uint8_t* seg1, int64_t N, int64_t K, uint8_t* tiles, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Np = round_up(N, kTileN), Kp = round_up(K, kTileK);
  prepack_fp5_kernel<<<grid_for(Np * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(seg4, seg1, N, K, Np, Kp, tiles);
  note_launch();
  return check_launch();
}


int64_t lpqt_fp5n_tiles_bytes(int64_t N, int64_t K) {
  if (N <= 0 || K <= 0) return 0;
  return round_up(N, kTileN) / kTileN * (round_up(K, kTileK) / kTileK) * kTileBytes5;
}

int lpqt_fp5n_prepack(const uint8_t* seg4, const uint8_t* seg1, int64_t N, int64_t K, uint8_t* tiles, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Np = round_up(N, kTileN), Kp = round_up(K, kTileK);
  prepack_fp5n_kernel<<<grid_for(Np * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(seg4, seg1, N, K, Np, Kp, tiles);
  note_launch();
  return check_launch();
}

int lpqt_fp5n_unprepack(const uint8_t* tiles, int64_t N, int64_t K, uint8_t* codes, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Kp = round_up(K, kTileK);
  unprepack_fp5n_kernel<<<grid_for(N * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(tiles, N, K, Kp, codes);
  note_launch();
  return check_launch();
}

int lpqt_fp5n_tiles_dequant(const uint8_t* tiles, const uint16_t* scales, int64_t N, int64_t K, uint16_t* out,
                            void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Kp = round_up(K, kTileK);
  tiles5_dequant_kernel<<<grid_for(N * (Kp / 32), 256), 256, 0, as_stream(stream)>>>(
      tiles, scales, N, K, Kp, out, ShiftMuls{1u << 26, 1u << 28, 1u << 30});
  note_launch();
  return check_launch();
}


int64_t lpqt_int4_tiles_bytes(int64_t N, int64_t K) {
  if (N <= 0 || K <= 0) return 0;
  return round_up(N, kTileN) / kTileN * (round_up(K, kTileK) / kTileK) * (kTileN * kTileK / 2);
}

int lpqt_int4_prepack(const uint8_t* nibbles, int64_t N, int64_t K, uint8_t* tiles, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const int64_t Np = round_up(N, kTileN), Kp = round_up(K, kTileK);
  prepack_int4_kernel<<<grid_for(Np * (Kp / 8), 256), 256, 0, as_stream(stream)>>>(nibbles, N, K, Np, Kp, tiles);
  note_launch();
  return check_launch();
}


int64_t lpqt_fgq_stage_bytes(int64_t N, int64_t K, int with_zeros) {
  if (N <= 0 || K <= 0) return 0;
  const int64_t stage = round_up(N, kTileN) * (round_up(K, kTileK) / kTileK) * (with_zeros ? 4 : 2);
  return with_zeros ? stage : stage + round_up(N, kTileN) * 4;  // FP6 / FP5: + f32 row factors
}

int lpqt_fgq_stage_params(const uint16_t* scales, const uint16_t* zeros, int64_t N, int64_t K, int64_t block,
                          void* out, void* stream) {
  if (N < 0 || K < 0) return LPQT_E_SHAPE;
  if (N == 0 || K == 0) return LPQT_OK;
  const bool per_row = block <= 0 || block >= K;
  if (!per_row && block % kTileK != 0) return LPQT_E_UNSUPPORTED;
  const int64_t k_tiles = round_up(K, kTileK) / kTileK;
  const int64_t bpr = per_row ? 1 : (K + block - 1) / block;
  const int64_t bkt = per_row ? k_tiles : block / kTileK;
  const int64_t Np = round_up(N, kTileN);
  const int64_t total = Np * k_tiles;
  float* rowf = zeros ? nullptr : reinterpret_cast<float*>(static_cast<uint8_t*>(out) + total * 2);
  if (!zeros) {
    fgq_row_factor_kernel<<<grid_for(Np, 256), 256, 0, as_stream(stream)>>>(scales, N, Np, bpr, rowf);
    note_launch();
  }
  fgq_stage_params_kernel<<<grid_for(total, 256), 256, 0, as_stream(stream)>>>(scales, zeros, N, bpr, bkt, k_tiles,
                                                                               total, rowf, out);
  note_launch();
  return check_launch();
}

}  // extern "C"
