// pipe_bench.cu — which pipe does F2FP.F16.E3M2 (cvt.rn.f16x2.e3m2x2) use?
// Times 8 independent chains of (a) cvt only, (b) lop3 only, (c) both
// interleaved.  If (c) ~ max(a, b) the pipes are separate.  Dev tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/pipe_bench.cu -o build/pipe_bench
#include <cstdio>
#include <cstdint>

template <int MODE>
__global__ void __launch_bounds__(512, 1) k(uint32_t seed, int iters, uint32_t* out, long long* cyc) {
  uint32_t a0 = seed ^ threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, a4 = a0 * 9, a5 = a0 * 11, a6 = a0 * 13,
           a7 = a0 * 15;
  uint32_t b0 = a0 + 1, b1 = a1 + 1, b2 = a2 + 1, b3 = a3 + 1, b4 = a4 + 1, b5 = a5 + 1, b6 = a6 + 1, b7 = a7 + 1;
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      if (MODE == 0 || MODE == 2) {
        asm volatile(
            "{.reg .b16 l0,l1,l2,l3,l4,l5,l6,l7;\n\t"
            "mov.b32 {l0, l1}, %0; mov.b32 {l2, l3}, %1; mov.b32 {l4, l5}, %2; mov.b32 {l6, l7}, %3;\n\t"
            "cvt.rn.f16x2.e3m2x2 %0, l0; cvt.rn.f16x2.e3m2x2 %1, l2; cvt.rn.f16x2.e3m2x2 %2, l4; "
            "cvt.rn.f16x2.e3m2x2 %3, l6;}\n"
            : "+r"(a0), "+r"(a1), "+r"(a2), "+r"(a3));
        asm volatile(
            "{.reg .b16 l0,l1,l2,l3,l4,l5,l6,l7;\n\t"
            "mov.b32 {l0, l1}, %0; mov.b32 {l2, l3}, %1; mov.b32 {l4, l5}, %2; mov.b32 {l6, l7}, %3;\n\t"
            "cvt.rn.f16x2.e3m2x2 %0, l1; cvt.rn.f16x2.e3m2x2 %1, l3; cvt.rn.f16x2.e3m2x2 %2, l5; "
            "cvt.rn.f16x2.e3m2x2 %3, l7;}\n"
            : "+r"(a4), "+r"(a5), "+r"(a6), "+r"(a7));
      }
      if (MODE == 1 || MODE == 2) {
        asm volatile(
            "lop3.b32 %0, %0, %4, 0x5a5a5a5a, 0x96; lop3.b32 %1, %1, %4, 0x3c3c3c3c, 0x96;"
            "lop3.b32 %2, %2, %4, 0x0f0f0f0f, 0x96; lop3.b32 %3, %3, %4, 0x33333333, 0x96;"
            : "+r"(b0), "+r"(b1), "+r"(b2), "+r"(b3)
            : "r"(b7));
        asm volatile(
            "lop3.b32 %0, %0, %4, 0x5a5a5a5a, 0x96; lop3.b32 %1, %1, %4, 0x3c3c3c3c, 0x96;"
            "lop3.b32 %2, %2, %4, 0x0f0f0f0f, 0x96; lop3.b32 %3, %3, %4, 0x33333333, 0x96;"
            : "+r"(b4), "+r"(b5), "+r"(b6), "+r"(b7)
            : "r"(b0));
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7 ^ b0 ^ b1 ^ b2 ^ b3 ^ b4 ^ b5 ^
                                               b6 ^ b7;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const char* nm[3] = {"cvt only", "lop3 only", "cvt + lop3"};
  for (int m = 0; m < 3; ++m) {
    const int iters = 4000;
    for (int rep = 0; rep < 2; ++rep) {
      if (m == 0) k<0><<<148, 512>>>(1, iters, out, cyc);
      if (m == 1) k<1><<<148, 512>>>(1, iters, out, cyc);
      if (m == 2) k<2><<<148, 512>>>(1, iters, out, cyc);
    }
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
    // per SM: 16 warps x iters x 64 ops of each kind
    const double warp_ops = 16.0 * iters * 64;
    printf("%-12s: %.3f cycles per 64-op group per warp-slot; %.2f warp-instr/clk/SM per kind\n", nm[m],
           (double)mx / (iters * 8), warp_ops / mx);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
