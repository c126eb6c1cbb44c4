// dq_bench.cu — microbenchmark of FP6->FP16 register transforms (dev tool).
//   (a) bias-shift PRMT/LOP3 transform (common.cuh fp6x32_to_f16x32)
//   (b) hardware cvt.rn.f16x2.e3m2x2 on 8-bit containers
//   (c) the GEMM's tile rebuild, a rebuild straight from the canonical 4+2
//       planes, the native FP5 rebuild and the two ablation rebuilds
// Also checks whether cvt ignores the two container bits above the 6-bit code.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/dq_bench.cu -o build/dq_bench
#include <cstdio>

#include "../paper_2312_08583_b200/csrc/common.cuh"

using namespace lpqt;

__device__ __forceinline__ uint32_t cvt_e3m2x2(uint16_t x) {
  uint32_t r;
  asm volatile("{cvt.rn.f16x2.e3m2x2 %0, %1;}\n" : "=r"(r) : "h"(x));
  return r;
}

// cvt-based transform of 32 weights: words w0..w5 hold 4 codes each in bits
// 0-5 of every byte (bits 6-7 carry the 8 spare weights' bits).
__device__ __forceinline__ void cvt32(const uint32_t w[6], uint32_t out[16]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    const uint32_t v = w[i] & 0x3F3F3F3Fu;
    out[2 * i] = cvt_e3m2x2(static_cast<uint16_t>(v));
    out[2 * i + 1] = cvt_e3m2x2(static_cast<uint16_t>(v >> 16));
  }
  const uint32_t e0 = ((w[0] >> 6) & 0x03030303u) | ((w[1] >> 4) & 0x0C0C0C0Cu) | ((w[2] >> 2) & 0x30303030u);
  const uint32_t e1 = ((w[3] >> 6) & 0x03030303u) | ((w[4] >> 4) & 0x0C0C0C0Cu) | ((w[5] >> 2) & 0x30303030u);
  out[12] = cvt_e3m2x2(static_cast<uint16_t>(e0));
  out[13] = cvt_e3m2x2(static_cast<uint16_t>(e0 >> 16));
  out[14] = cvt_e3m2x2(static_cast<uint16_t>(e1));
  out[15] = cvt_e3m2x2(static_cast<uint16_t>(e1 >> 16));
}
__device__ __forceinline__ void cvt32_nomask(const uint32_t w[6], uint32_t out[16]) {
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    out[2 * i] = cvt_e3m2x2(static_cast<uint16_t>(w[i]));
    out[2 * i + 1] = cvt_e3m2x2(static_cast<uint16_t>(w[i] >> 16));
  }
  const uint32_t e0 = ((w[0] >> 6) & 0x03030303u) | ((w[1] >> 4) & 0x0C0C0C0Cu) | ((w[2] >> 2) & 0x30303030u);
  const uint32_t e1 = ((w[3] >> 6) & 0x03030303u) | ((w[4] >> 4) & 0x0C0C0C0Cu) | ((w[5] >> 2) & 0x30303030u);
  out[12] = cvt_e3m2x2(static_cast<uint16_t>(e0));
  out[13] = cvt_e3m2x2(static_cast<uint16_t>(e0 >> 16));
  out[14] = cvt_e3m2x2(static_cast<uint16_t>(e1));
  out[15] = cvt_e3m2x2(static_cast<uint16_t>(e1 >> 16));
}

// (c) straight from the reference's canonical 4+2 planes (packing.py:63-90,
// what a TMA tensor-map stream of the planes would hand the dequant warps):
// w[0..3] = seg4 words (nibble j of word i = code >> 2 of weight 8i + j),
// w[4..5] = seg2 words (2-bit field j of word i = code & 3 of weight 16i + j).
__device__ __forceinline__ uint32_t spread_fields(uint32_t b) {  // 4 2-bit fields of byte b -> bits 0-1 of 4 bytes
  return (b | (b << 6) | (b << 12) | (b << 18)) & 0x03030303u;
}
__device__ __forceinline__ void planes32(const uint32_t w[6], uint32_t out[16]) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const uint32_t mmw = w[4 + (i >> 1)] >> (16 * (i & 1));  // fields of weights 8i .. 8i + 7
#pragma unroll
    for (int h = 0; h < 2; ++h) {  // weights 8i + 4h .. + 3
      const uint32_t p = __byte_perm(w[i], 0u, h ? 0x3322 : 0x1100);
      const uint32_t n = (p & 0x000F000Fu) | ((p >> 4) & 0x0F000F00u);  // the 4 nibbles as bytes
      const uint32_t mm = spread_fields((mmw >> (8 * h)) & 0xFFu);
      const uint32_t c = (n << 2) | mm;                                 // e3m2 codes
      out[4 * i + 2 * h] = cvt_e3m2x2(static_cast<uint16_t>(c));
      out[4 * i + 2 * h + 1] = cvt_e3m2x2(static_cast<uint16_t>(c >> 16));
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) bench(const uint32_t* in, uint32_t* out, int iters, long long* cyc,
                                                ShiftMuls sm) {
  uint32_t w[6];
#pragma unroll
  for (int i = 0; i < 6; ++i) w[i] = in[(threadIdx.x * 6 + i) & 1023];
  uint32_t acc = 0;
  __shared__ uint4 sink[2048];
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    uint32_t o[16];
#pragma unroll
    for (int g = 0; g < 4; ++g) {  // 128 weights per iteration
      if (MODE == 0) fp6x32_to_f16x32(w, o);
      else if (MODE == 1) cvt32(w, o);
      else if (MODE == 2) cvt32_nomask(w, o);
      else if (MODE == 3) fp6x32_cvt_f16x32_fma(w, o, sm);       // the GEMM's tile rebuild
      else if (MODE == 4) planes32(w, o);                        // canonical 4+2 planes
      else if (MODE == 5) fp5x32_cvt_f16x32(w, w[4], o, sm);     // native FP5 tiles (5 words)
      else if (MODE == 6) fp6x32_soft_f16x32<1>(w, o, 0x3c003c00u, sm);  // ablation: bias-shift x scale
      else fp6x32_soft_f16x32<2>(w, o, 0x3c003c00u, sm);                 // ablation: naive x scale
      // sink: 4 x STS.128 (MIO pipe, like the STTM in the GEMM)
#pragma unroll
      for (int j = 0; j < 4; ++j)
        reinterpret_cast<uint4*>(sink)[(threadIdx.x * 4 + j) & 2047] = make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
#pragma unroll
      for (int i = 0; i < 6; ++i) w[i] = w[i] * 0x9E3779B1u + g;  // defeat CSE (1 IMAD each)
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc + reinterpret_cast<uint32_t*>(sink)[threadIdx.x];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

__global__ void check_cvt(uint32_t* out) {
  // every 8-bit container value -> fp16 (low half of the f16x2)
  const int v = threadIdx.x + blockIdx.x * blockDim.x;
  if (v < 256) out[v] = cvt_e3m2x2(static_cast<uint16_t>(v)) & 0xFFFFu;
}

int main() {
  uint32_t *in, *out;
  long long* cyc;
  cudaMalloc(&in, 4096 * 4);
  cudaMalloc(&out, 148 * 512 * 4 + 4096);
  cudaMalloc(&cyc, 148 * 8);
  cudaMemset(in, 0x5A, 4096 * 4);
  const char* names[8] = {"bias-shift PRMT/LOP3 (byte form)", "cvt e3m2x2 (masked)", "cvt e3m2x2 (no mask)",
                          "GEMM tile rebuild (cvt+FMA)", "canonical 4+2 planes + cvt", "native FP5 tiles + cvt",
                          "ablation bias-shift x S", "ablation naive x S"};
  const ShiftMuls sm{1u << 26, 1u << 28, 1u << 30};
  for (int mode = 0; mode < 8; ++mode) {
    const int iters = 2000;
    for (int rep = 0; rep < 2; ++rep) {
      if (mode == 0) bench<0><<<148, 512>>>(in, out, iters, cyc, sm);
      if (mode == 1) bench<1><<<148, 512>>>(in, out, iters, cyc, sm);
      if (mode == 2) bench<2><<<148, 512>>>(in, out, iters, cyc, sm);
      if (mode == 3) bench<3><<<148, 512>>>(in, out, iters, cyc, sm);
      if (mode == 4) bench<4><<<148, 512>>>(in, out, iters, cyc, sm);
      if (mode == 5) bench<5><<<148, 512>>>(in, out, iters, cyc, sm);
      if (mode == 6) bench<6><<<148, 512>>>(in, out, iters, cyc, sm);
      if (mode == 7) bench<7><<<148, 512>>>(in, out, iters, cyc, sm);
    }
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    const double weights_per_sm = 512.0 * 128 * iters;
    printf("%-34s: %.2f weights/clk/SM (incl. 6 IMAD per 32 weights)\n", names[mode], weights_per_sm / mx);
  }
  check_cvt<<<1, 256>>>(out);
  uint32_t h[256];
  cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);
  int ignore_top = 1;
  for (int v = 0; v < 256; ++v)
    if (h[v] != h[v & 63]) ignore_top = 0;
  printf("cvt ignores container bits 6-7: %s\n", ignore_top ? "yes" : "no");
  printf("codes: 1->%04x 3->%04x 4->%04x 31->%04x 32->%04x 63->%04x 64->%04x 128->%04x\n", h[1], h[3], h[4], h[31],
         h[32], h[63], h[64], h[128]);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
