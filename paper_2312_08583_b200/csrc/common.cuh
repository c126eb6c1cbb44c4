// common.cuh — shared device helpers for liblpqt_b200 (sm_100a only).
//
// FP6 e3m2 constants and the bias-shift bit algebra follow the reference
// (codec.py:48-49, dequant.py:33-43); the PTX wrappers (mbarrier, bulk/TMA
// copies, tcgen05 alloc/mma/ld/st/commit) are the Blackwell primitives the
// W6A16 GEMM is built from.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lpqt_b200.h"

#ifndef LPQT_WAIT_HINT_NS
#define LPQT_WAIT_HINT_NS 64
#endif

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "liblpqt_b200 targets sm_100a only"
#endif

namespace lpqt {

// ---------------------------------------------------------------------------
// Host-side bookkeeping
// ---------------------------------------------------------------------------
void note_launch();           // increments the launch counter (capi.cu)
int check_launch();           // cudaGetLastError -> LPQT_OK / LPQT_E_CUDA

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(int64_t n, int threads, int64_t cap = 148 * 32) {
  int64_t g = (n + threads - 1) / threads;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return static_cast<int>(g);
}

// ---------------------------------------------------------------------------
// FP6 e3m2 scalar algebra (codec.py:63-96, dequant.py:33-43)
// ---------------------------------------------------------------------------
// magnitude grid g[i], i in 0..31 (codec.py:85-89): subnormal (E=0) i/16,
// normal (1 + M/4) * 2^(E-3).  Every value and every midpoint is a short
// binary fraction, so double comparisons against midpoints are exact.
__host__ __device__ inline double fp6_magnitude(int i) {
  const int e = i >> 2, m = i & 3;
  if (e == 0) return m * 0.0625;                   // (m/4) * 2^-2
  double v = 1.0 + m * 0.25;
  int sh = e - 3;
  return sh >= 0 ? v * (double)(1 << sh) : v / (double)(1 << (-sh));
}

// composed binary16 pattern of a code: sign<<15 | E<<10 | M<<8 (dequant.py:40)
__host__ __device__ __forceinline__ uint16_t fp6_compose_bits(uint32_t c) {
  return static_cast<uint16_t>(((c & 0x20u) << 10) | ((c & 0x1Fu) << 8));
}

// byte form used by the tile layout: s00eeemm (fp16 high byte of compose)
__host__ __device__ __forceinline__ uint32_t fp6_byteform(uint32_t c) {
  return ((c & 0x20u) << 2) | (c & 0x1Fu);
}
__host__ __device__ __forceinline__ uint32_t fp6_from_byteform(uint32_t b) {
  return ((b & 0x80u) >> 2) | (b & 0x1Fu);
}

// ---------------------------------------------------------------------------
// The register transform used by the GEMM (tile layout v2, "cvt" layout):
// 6 words of the tile layout (32 weights) -> 16 half2 of the codes' exact
// binary16 VALUES (value_table_f16, codec.py:108-113), k ascending.
//   word i (0..5), byte t: bits 0-5 = e3m2 code of weight k = 4i+t
//                          bits 6-7 = two bits of a "spare" weight
//   spare E0 (k 24..27) byte t = W0[6:7] | W1[6:7] << 2 | W2[6:7] << 4
//   spare E1 (k 28..31) byte t = W3[6:7] | W4[6:7] << 2 | W5[6:7] << 4
// The FP6 code is the OCP e3m2 encoding, so the hardware converter
// cvt.rn.f16x2.e3m2x2 (SASS F2FP.F16.E3M2.UNPACK_B, 2 weights per op, reads
// either 16-bit half, ignores container bits 6-7) does the rebuild; the
// spares cost 3 SHF + 2 LOP3 per 4.  ~0.81 ALU-pipe ops / weight, against
// ~1.19 for the bias-shift PRMT rebuild below (F2FP issues on the same
// half-rate ALU pipe as LOP3/PRMT — measured, tools/pipe_bench.cu).  The
// epilogue then scales by S (value * S == compose * S * 2^12 exactly).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cvt_e3m2x2_lo(uint32_t w) {
  uint32_t r;
  asm("{cvt.rn.f16x2.e3m2x2 %0, %1;}" : "=r"(r) : "h"(static_cast<uint16_t>(w)));
  return r;
}
__device__ __forceinline__ uint32_t cvt_e3m2x2_hi(uint32_t w) {
  uint32_t r;
  asm("{cvt.rn.f16x2.e3m2x2 %0, %1;}" : "=r"(r) : "h"(static_cast<uint16_t>(w >> 16)));
  return r;
}
// (a & M) | (b & ~M) as ONE LOP3 (ptxas splits the C form into two when it
// knows some operand bits are zero: 3 LOP3 per spare gather instead of 2)
template <uint32_t M>
__device__ __forceinline__ uint32_t lop3_sel(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(a), "r"(b), "n"(M));
  return d;
}
__device__ __forceinline__ uint32_t spare_gather(uint32_t wa, uint32_t wb, uint32_t wc) {
  const uint32_t t = lop3_sel<0x03030303u>(wa >> 6, wb >> 4);
  return lop3_sel<0x0F0F0F0Fu>(t, wc >> 2);  // bits 6-7 of each byte: don't care
}
__device__ __forceinline__ void fp6x32_cvt_f16x32(const uint32_t w[6], uint32_t out[16]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    out[2 * i] = cvt_e3m2x2_lo(w[i]);
    out[2 * i + 1] = cvt_e3m2x2_hi(w[i]);
  }
  const uint32_t e0 = spare_gather(w[0], w[1], w[2]);
  const uint32_t e1 = spare_gather(w[3], w[4], w[5]);
  out[12] = cvt_e3m2x2_lo(e0);
  out[13] = cvt_e3m2x2_hi(e0);
  out[14] = cvt_e3m2x2_lo(e1);
  out[15] = cvt_e3m2x2_hi(e1);
}
// Same rebuild with the spare-bit gather's right shifts done as IMAD.HI
// (w * 2^(32-s) >> 32) on the FMA pipe, leaving the half-rate ALU pipe the
// 16 F2FP + 4 LOP3 per 32 weights.  The multipliers come from kernel
// arguments so ptxas cannot strength-reduce them back into SHF.
struct ShiftMuls {
  uint32_t m26, m28, m30;  // 2^26, 2^28, 2^30  ->  >> 6, >> 4, >> 2
};
__device__ __forceinline__ uint32_t spare_gather_fma(uint32_t wa, uint32_t wb, uint32_t wc, const ShiftMuls& sm) {
  const uint32_t t = lop3_sel<0x03030303u>(__umulhi(wa, sm.m26), __umulhi(wb, sm.m28));
  return lop3_sel<0x0F0F0F0Fu>(t, __umulhi(wc, sm.m30));
}
__device__ __forceinline__ void fp6x32_cvt_f16x32_fma(const uint32_t w[6], uint32_t out[16], const ShiftMuls& sm) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    out[2 * i] = cvt_e3m2x2_lo(w[i]);
    out[2 * i + 1] = cvt_e3m2x2_hi(w[i]);
  }
  const uint32_t e0 = spare_gather_fma(w[0], w[1], w[2], sm);
  const uint32_t e1 = spare_gather_fma(w[3], w[4], w[5], sm);
  out[12] = cvt_e3m2x2_lo(e0);
  out[13] = cvt_e3m2x2_hi(e0);
  out[14] = cvt_e3m2x2_lo(e1);
  out[15] = cvt_e3m2x2_hi(e1);
}
// ---------------------------------------------------------------------------
// Software rebuilds on the same tile layout, for the paper's ablation
// (the FP6 kernel with vs without Bias-Shift; selected by
// LPQT_REBUILD_* launch flags, decode kernels only).  Both produce the
// binary16 dequantized weight of the reference's two dequant paths
// (dequant.py:72-86): the epilogue then applies no scale.
//   bias-shift: h16 = sign << 15 | eeemm << 8 (= value * 2^-12, dequant.py:37-41),
//               then x folded scale S * 2^12 (HMUL2, one binary16 rounding);
//   naive:      the exact binary16 value — exponent + 12 for normal codes,
//               x 2^12 for the subnormal ones (the paper's two-step cast) —
//               then x S (HMUL2).
// Both equal value_f16 * S rounded once, so the two ablation kernels give
// bit-identical Y (tests/test_dequant.py:93-102 of the reference).
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t bias_shift_x2(uint32_t w, uint32_t sel) {
  const uint32_t p = __byte_perm(w, 0u, sel);  // codes into the high bytes of the two halves
  return (p & 0x1F001F00u) | ((p << 2) & 0x80008000u);
}
__device__ __forceinline__ uint32_t naive_x2(uint32_t w, uint32_t sel) {
  const uint32_t h = bias_shift_x2(w, sel);
  const uint32_t t = (h & 0x1C001C00u) + 0x7C007C00u;    // bit 15 / 31: the exponent is non-zero
  uint32_t m;  // 0xFFFF for the normal halves: PRMT sign-replicate mode (selector msb; __byte_perm masks it off)
  asm("prmt.b32 %0, %1, 0, 0xBB99;" : "=r"(m) : "r"(t));
  const uint32_t hn = h + 0x30003000u;                   // exponent + 12 (no carry out of the field)
  const __half2 hs2 = __hmul2(*reinterpret_cast<const __half2*>(&h), __float2half2_rn(4096.f));  // subnormals x 2^12
  const uint32_t hs = *reinterpret_cast<const uint32_t*>(&hs2);
  return (hn & m) | (hs & ~m);
}
template <int RB>
__device__ __forceinline__ void fp6x32_soft_f16x32(const uint32_t w[6], uint32_t out[16], uint32_t s2,
                                                   const ShiftMuls& sm) {
  auto one = [&](uint32_t x, uint32_t sel) { return RB == 1 ? bias_shift_x2(x, sel) : naive_x2(x, sel); };
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    out[2 * i] = one(w[i], 0x1404);
    out[2 * i + 1] = one(w[i], 0x3424);
  }
  const uint32_t e0 = spare_gather_fma(w[0], w[1], w[2], sm) & 0x3F3F3F3Fu;
  const uint32_t e1 = spare_gather_fma(w[3], w[4], w[5], sm) & 0x3F3F3F3Fu;
  out[12] = one(e0, 0x1404);
  out[13] = one(e0, 0x3424);
  out[14] = one(e1, 0x1404);
  out[15] = one(e1, 0x3424);
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const __half2 v = __hmul2(*reinterpret_cast<const __half2*>(&out[j]), *reinterpret_cast<const __half2*>(&s2));
    out[j] = *reinterpret_cast<const uint32_t*>(&v);
  }
}

// FP5 native rebuild (layout above): 32 weights -> 16 half2 of the exact
// binary16 values, k ascending.  The mantissa word is split by bit parity once
// (Me = even bit positions, Mo = odd): group s shifted so its bits land on
// bit 1 of every byte then has a ZERO bit 0 (that bit comes from a position of
// the other parity), so one LOP3 (lo & 0x3C..) | (u & ~0x3C..) merges nibble
// and mantissa (bits 6-7 are ignored by the converter).  Shifts run on the
// FMA pipe (IMAD / IMAD.HI by register multipliers: sm.m26 = 2^26 etc.).
__device__ __forceinline__ uint32_t lop3_3c(uint32_t lo, uint32_t u) {
  uint32_t d;  // (lo & 0x3C3C3C3C) | (u & ~0x3C3C3C3C)
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;" : "=r"(d) : "r"(lo), "r"(u), "n"(0x3C3C3C3C));
  return d;
}
__device__ __forceinline__ void fp5x32_cvt_f16x32(const uint32_t nib[4], uint32_t mw, uint32_t out[16],
                                                  const ShiftMuls& sm) {
  const uint32_t me = mw & 0x55555555u, mo = mw & 0xAAAAAAAAu;
  const uint32_t two = sm.m26 >> 25, four = sm.m26 >> 24;  // registers: IMAD, not SHF
  uint32_t u[8];  // group s = 2i + p: mantissa of byte t at bit 8t + 1
  u[0] = me * two;                  // << 1
  u[1] = mo;                        // bit 8t + 1 already
  u[2] = me >> 1;
  u[3] = __umulhi(mo, 1u << 30);    // >> 2
  u[4] = __umulhi(me, 1u << 29);    // >> 3
  u[5] = __umulhi(mo, sm.m28);      // >> 4
  u[6] = __umulhi(me, 1u << 27);    // >> 5
  u[7] = __umulhi(mo, sm.m26);      // >> 6
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t lo = nib[i] * four, hi = __umulhi(nib[i], sm.m30);  // << 2 (even nibbles), >> 2 (odd)
    const uint32_t x0 = lop3_3c(lo, u[2 * i]), x1 = lop3_3c(hi, u[2 * i + 1]);
    out[4 * i] = cvt_e3m2x2_lo(x0);
    out[4 * i + 1] = cvt_e3m2x2_hi(x0);
    out[4 * i + 2] = cvt_e3m2x2_lo(x1);
    out[4 * i + 3] = cvt_e3m2x2_hi(x1);
  }
}

// codes of the 32 weights (inverse of fp6x32_pack_words; used by unprepack)
__host__ __device__ inline void fp6x32_unpack_codes(const uint32_t w[6], uint8_t c[32]) {
  for (int i = 0; i < 6; ++i)
    for (int t = 0; t < 4; ++t) c[4 * i + t] = static_cast<uint8_t>((w[i] >> (8 * t)) & 0x3Fu);
  for (int t = 0; t < 4; ++t) {
    const int s = 8 * t + 6;
    c[24 + t] = static_cast<uint8_t>(((w[0] >> s) & 3u) | (((w[1] >> s) & 3u) << 2) | (((w[2] >> s) & 3u) << 4));
    c[28 + t] = static_cast<uint8_t>(((w[3] >> s) & 3u) | (((w[4] >> s) & 3u) << 2) | (((w[5] >> s) & 3u) << 4));
  }
}

// ---------------------------------------------------------------------------
// Bias-shift rebuild (the paper's ALU trick, dequant.py:33-43) over the older
// "byte form" layout: word i byte t = s00eeemm of weight 4i+t, spares in bits
// 5-6.  Kept as a reference point for tools/dq_bench.cu; the GEMM uses the
// cvt layout above.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void fp6x32_to_f16x32(const uint32_t w[6], uint32_t out[16]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t q = w[i] & 0x9F9F9F9Fu;
    out[2 * i] = __byte_perm(q, 0u, 0x1404);
    out[2 * i + 1] = __byte_perm(q, 0u, 0x3424);
  }
  const uint32_t e0 = ((w[0] >> 5) & 0x03030303u) | ((w[1] >> 3) & 0x0C0C0C0Cu) |
                      ((w[2] >> 1) & 0x10101010u) | ((w[5] << 1) & 0x80808080u);
  const uint32_t e1 = ((w[3] >> 5) & 0x03030303u) | ((w[4] >> 3) & 0x0C0C0C0Cu) |
                      ((w[2] >> 2) & 0x10101010u) | ((w[5] << 2) & 0x80808080u);
  out[12] = __byte_perm(e0, 0u, 0x1404);
  out[13] = __byte_perm(e0, 0u, 0x3424);
  out[14] = __byte_perm(e1, 0u, 0x1404);
  out[15] = __byte_perm(e1, 0u, 0x3424);
}

// Byte-form layout packer (bias-shift rebuild above; dev benchmarks only).
__host__ __device__ inline void fp6x32_pack_words_byteform(const uint8_t c[32], uint32_t w[6]) {
  uint32_t b[32];
  for (int j = 0; j < 32; ++j) b[j] = fp6_byteform(c[j]);
  for (int i = 0; i < 6; ++i) {
    w[i] = b[4 * i] | (b[4 * i + 1] << 8) | (b[4 * i + 2] << 16) | (b[4 * i + 3] << 24);
  }
  for (int t = 0; t < 4; ++t) {
    const uint32_t e0 = b[24 + t], e1 = b[28 + t];
    const int s = 8 * t;
    w[0] |= ((e0 >> 0) & 3u) << (s + 5);
    w[1] |= ((e0 >> 2) & 3u) << (s + 5);
    w[2] |= ((e0 >> 4) & 1u) << (s + 5);
    w[2] |= ((e1 >> 4) & 1u) << (s + 6);
    w[3] |= ((e1 >> 0) & 3u) << (s + 5);
    w[4] |= ((e1 >> 2) & 3u) << (s + 5);
    w[5] |= ((e0 >> 7) & 1u) << (s + 6);
    w[5] |= ((e1 >> 7) & 1u) << (s + 5);
  }
}

// Tile layout v2 packer (used by prepack): 32 codes (k ascending) -> 6 words,
// inverse of fp6x32_unpack_codes / the layout read by fp6x32_cvt_f16x32.
__host__ __device__ inline void fp6x32_pack_words(const uint8_t c[32], uint32_t w[6]) {
  for (int i = 0; i < 6; ++i) {
    w[i] = (c[4 * i] & 0x3Fu) | ((c[4 * i + 1] & 0x3Fu) << 8) | ((c[4 * i + 2] & 0x3Fu) << 16) |
           ((uint32_t)(c[4 * i + 3] & 0x3Fu) << 24);
  }
  for (int t = 0; t < 4; ++t) {
    const uint32_t e0 = c[24 + t], e1 = c[28 + t];
    const int s = 8 * t + 6;
    w[0] |= (e0 & 3u) << s;
    w[1] |= ((e0 >> 2) & 3u) << s;
    w[2] |= ((e0 >> 4) & 3u) << s;
    w[3] |= (e1 & 3u) << s;
    w[4] |= ((e1 >> 2) & 3u) << s;
    w[5] |= ((e1 >> 4) & 3u) << s;
  }
}

// ---------------------------------------------------------------------------
// Tile layout geometry (shared by prepack, tiles_dequant and the GEMM)
//   tile = 128 rows x 128 k = 12288 B, stored [row_tile][k_tile]
//   inside a tile: [khalf 2][quad 3][row 128][16 B]; thread (row, khalf) owns
//   3 quads = 12 words = 64 weights = two 32-weight groups (words 0-5, 6-11).
// ---------------------------------------------------------------------------
constexpr int kTileN = 128;
constexpr int kTileK = 128;
constexpr int kTileBytes = kTileN * kTileK * 6 / 8;  // 12288

// byte offset of word wi (0..5) of the 32-weight group starting at (n, k32*32)
__host__ __device__ __forceinline__ int64_t tile_word_addr(int64_t n, int64_t g32, int wi,
                                                           int64_t k_tiles) {
  const int64_t rt = n / kTileN, rr = n % kTileN;
  const int64_t kt = g32 / 4;               // 4 groups of 32 per 128-k tile
  const int gin = static_cast<int>(g32 % 4);
  const int khalf = gin >> 1, grp = gin & 1;
  const int word = grp * 6 + wi;            // 0..11 within the (row,khalf) slot
  const int quad = word >> 2, wq = word & 3;
  return (rt * k_tiles + kt) * kTileBytes + ((int64_t)(khalf * 3 + quad) * kTileN + rr) * 16 + wq * 4;
}

// ---------------------------------------------------------------------------
// FP5 e3m1 native tiles ("4+1", packing.py:84-85's split: a 4-bit s|eee plane
// and a 1-bit mantissa plane), 0.625 B per weight.
//   tile = 128 rows x 128 k = 10240 B, stored [row_tile][k_tile];
//   inside: nibble quads [khalf 2][grp 2][row 128][16 B] (8192 B), then the
//   mantissa words [khalf 2][row 128][grp 2][4 B] (2048 B).
//   32-weight group: nibble word i (0..3) holds s|eee of weight 8i + t in
//   nibble 2t (t = 0..3) and of weight 8i + 4 + t in nibble 2t + 1; the
//   mantissa word holds m of weight 8i + 4p + t at bit 8t + 2i + p.
// Rebuild (fp5x32_cvt_f16x32): the e3m1 code (s, eee, m) is the e3m2 code
// (s, eee, m0), so per 4 weights one shift of the nibble word + one of the
// mantissa word (FMA pipe), one AND + one LOP3 build the four e3m2 bytes for
// two hardware converts (F2FP.E3M2): 16 F2FP + 16 LOP per 32 weights.
// ---------------------------------------------------------------------------
constexpr int kTileBytes5 = kTileN * kTileK * 5 / 8;  // 10240
constexpr int kTile5Nib = kTileN * kTileK / 2;         // 8192: nibble quads, then mantissa words

__host__ __device__ inline void fp5x32_pack_words(const uint8_t c[32], uint32_t nib[4], uint32_t& mw) {
  mw = 0;
  for (int i = 0; i < 4; ++i) {
    nib[i] = 0;
    for (int p = 0; p < 2; ++p)
      for (int t = 0; t < 4; ++t) {
        const uint32_t code = c[8 * i + 4 * p + t] & 0x1Fu;
        nib[i] |= (code >> 1) << (4 * (2 * t + p));
        mw |= (code & 1u) << (8 * t + 2 * i + p);
      }
  }
}
__host__ __device__ inline void fp5x32_unpack_codes(const uint32_t nib[4], uint32_t mw, uint8_t c[32]) {
  for (int i = 0; i < 4; ++i)
    for (int p = 0; p < 2; ++p)
      for (int t = 0; t < 4; ++t)
        c[8 * i + 4 * p + t] = static_cast<uint8_t>((((nib[i] >> (4 * (2 * t + p))) & 15u) << 1) |
                                                    ((mw >> (8 * t + 2 * i + p)) & 1u));
}
// byte offset of the 32-weight group g32 (k = 32 g32 ..) of row n: nibble word wi (0..3), mantissa word (wi == 4)
__host__ __device__ __forceinline__ int64_t tile5_word_addr(int64_t n, int64_t g32, int wi, int64_t k_tiles) {
  const int64_t rt = n / kTileN, rr = n % kTileN;
  const int64_t kt = g32 / 4;
  const int gin = static_cast<int>(g32 % 4);
  const int khalf = gin >> 1, grp = gin & 1;
  const int64_t base = (rt * k_tiles + kt) * kTileBytes5;
  if (wi < 4) return base + ((int64_t)(khalf * 2 + grp) * kTileN + rr) * 16 + wi * 4;
  return base + kTile5Nib + ((int64_t)khalf * kTileN + rr) * 8 + grp * 4;
}
// ---------------------------------------------------------------------------
// PTX wrappers
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// LPQT_WAIT_MODE: 0 = try_wait (HW suspend, system time limit),
// 1 = test_wait spin, 2 = try_wait with a short suspend-time hint.
#ifndef LPQT_WAIT_MODE
#define LPQT_WAIT_MODE 2
#endif
template <int MODE = LPQT_WAIT_MODE>
__device__ __forceinline__ bool mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  if constexpr (MODE == 1) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  } else if constexpr (MODE == 2) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity), "r"(LPQT_WAIT_HINT_NS)
        : "memory");
  } else {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
  }
  return ok != 0;
}
// non-blocking probe: has the phase with `parity` completed?
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
// Spin with a watchdog: a pipeline deadlock traps (the launch fails with an
// error) instead of hanging the device.
// The watchdog counts ROUNDS of 4 polls, so a poll is just try_wait + branch:
// the idle roles' polling shares the issue slots of the dequant warps, and a
// per-poll counter (+ compare + branch) cost 2-4 % of the decode launches;
// rounds of 4 polls are within 0.5 % of no watchdog at all, while 16 / 64
// unrolled polls are slower again (code size) (profiles/r02_abx_watchdog*.jsonl).
#ifndef LPQT_WATCHDOG_POLLS
#define LPQT_WATCHDOG_POLLS 4
#endif
template <int MODE = LPQT_WAIT_MODE>
__device__ __forceinline__ void mbar_wait_u32(uint32_t a, uint32_t parity) {
  for (uint32_t rounds = 0;; ++rounds) {
#pragma unroll
    for (int j = 0; j < LPQT_WATCHDOG_POLLS; ++j)
      if (mbar_try_wait<MODE>(a, parity)) return;
    if (rounds == (1u << 30) / LPQT_WATCHDOG_POLLS) __trap();
  }
}
template <int MODE = LPQT_WAIT_MODE>
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  mbar_wait_u32<MODE>(smem_u32(bar), parity);
}
__device__ __forceinline__ void mbar_arrive_u32(uint32_t a) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(a) : "memory");
}
// ring cursor: slot index + phase parity, advanced once per use
template <int N>
struct RingPos {
  uint32_t idx = 0, ph = 0;
  __device__ __forceinline__ void adv() {
    if (++idx == N) {
      idx = 0;
      ph ^= 1u;
    }
  }
};

// 1-D bulk copy global -> shared, completes tx bytes on `bar`; evict-first
// L2 policy for the streamed weight tiles.
__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_plain(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// bulk L2 prefetch (no smem, no barrier): size a multiple of 16, 16-B aligned
__device__ __forceinline__ void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// tcgen05 -------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
}
__device__ __forceinline__ void tmem_relinquish() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
// D[tmem] (+)= A[tmem] * B[smem desc]; kind::f16 (fp16 in, fp32 accumulate)
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// ---- warp-converged single-thread issue --------------------------------------
// elect.sync picks one lane; the *_if / *_elect forms execute the async op on
// that lane only, from converged code, so ptxas can keep the operands in
// uniform registers (no per-issue ELECT/R2UR.BROADCAST waterfall).
__device__ __forceinline__ uint32_t elect_one() {
  uint32_t pred;
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "selp.u32 %0, 1, 0, e;\n\t}"
      : "=r"(pred));
  return pred;
}
__device__ __forceinline__ void mbar_arrive_expect_tx_if(uint32_t pred, uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "@e mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %2;\n\t}" ::"r"(pred),
      "r"(smem_u32(bar)), "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_if(uint32_t pred, void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                            uint64_t policy) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "@e cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%1], [%2], %3, [%4], "
      "%5;\n\t}" ::"r"(pred),
      "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d_if(uint32_t pred, void* dst, const CUtensorMap* map, uint64_t* bar, int c0,
                                               int c1) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "@e cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%1], [%2, {%4, %5}], "
      "[%3];\n\t}" ::"r"(pred),
      "r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// tcgen05.mma issued by one elected lane of a converged warp
__device__ __forceinline__ void mma_f16_ts_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}
// same, with the elected-lane predicate computed once by the caller
__device__ __forceinline__ void mma_f16_ts_if(uint32_t pred, uint32_t d_tmem, uint32_t a_tmem, uint32_t b_desc_lo,
                                              uint32_t b_desc_hi, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 bd;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "mov.b64 bd, {%3, %4};\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], [%2], bd, %5, p;\n\t}" ::"r"(pred),
      "r"(d_tmem), "r"(a_tmem), "r"(b_desc_lo), "r"(b_desc_hi), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void tc_commit_if(uint32_t pred, uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "setp.ne.b32 e, %0, 0;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%1];\n\t}" ::"r"(pred),
      "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// Shared-memory matrix descriptor: K-major, 128-byte swizzle, 8-row atoms
// of 1024 B (SBO), version 1 (sm_100).
__device__ __forceinline__ uint64_t sdesc_kmajor_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr & 0x3FFFFu) >> 4);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
  d |= static_cast<uint64_t>(1) << 46;            // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;            // SWIZZLE_128B
  return d;
}

// instruction descriptor for kind::f16: A,B fp16 K-major, D fp32, M=128
__host__ __device__ constexpr uint32_t idesc_f16_m128(int n) {
  return (1u << 4) | (0u << 7) | (0u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(128 >> 4) << 24);
}

#define LPQT_R8(o) "r"(o[0]), "r"(o[1]), "r"(o[2]), "r"(o[3]), "r"(o[4]), "r"(o[5]), "r"(o[6]), "r"(o[7])
#define LPQT_W8(o) "=r"(o[0]), "=r"(o[1]), "=r"(o[2]), "=r"(o[3]), "=r"(o[4]), "=r"(o[5]), "=r"(o[6]), "=r"(o[7])

// 32 lanes x 32 consecutive 32-bit columns store (one TMEM lane per thread)
__device__ __forceinline__ void tmem_st_x32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};" ::"r"(taddr),
      LPQT_R8((r + 0)), LPQT_R8((r + 8)), LPQT_R8((r + 16)), LPQT_R8((r + 24))
      : "memory");
}
__device__ __forceinline__ void tmem_st_x16(uint32_t taddr, const uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
      "%14, %15, %16};" ::"r"(taddr),
      LPQT_R8((r + 0)), LPQT_R8((r + 8))
      : "memory");
}
__device__ __forceinline__ void tmem_st_x1(uint32_t taddr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(v) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld_x16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15}, [%16];"
      : LPQT_W8((r + 0)), LPQT_W8((r + 8))
      : "r"(taddr)
      : "memory");
}
__device__ __forceinline__ void tmem_ld_x1(uint32_t taddr, uint32_t& v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(taddr) : "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int nthreads) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Per-warpgroup register reallocation (all 4 warps of the group execute it).
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(N));
}
template <uint32_t N>
__device__ __forceinline__ void setmaxnreg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(N));
}

// Programmatic dependent launch: wait until the preceding grid on the stream
// has completed and its memory is visible (no-op without the launch
// attribute); allow the next PDL-launched grid to be scheduled.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint4 lds128_u32(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  uint16_t v;
  asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ float4 lds128_f32(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64_u32(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
__device__ __forceinline__ uint2 lds64(const void* p) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ uint4 lds128(const void* p) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(smem_u32(p)));
  return v;
}

// ---- output tiles: proxy fences + TMA tensor store from shared memory --------
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, uint32_t smem, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(map),
               "r"(smem), "r"(c0), "r"(c1)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
}  // namespace lpqt
