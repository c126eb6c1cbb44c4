// mma_bench.cu — microbenchmark: issue rate of tcgen05.mma.kind::f16 with
// M=128 and small N, A from TMEM ("TS") or SMEM ("SS"), independent or
// dependent accumulators.  Dev tool (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_bench.cu -o build/mma_bench -lcuda
#include <cstdio>
#include <cstdlib>

#include "../paper_2312_08583_b200/csrc/common.cuh"

using namespace lpqt;

// modes: 0 = TS, 1 = SS
template <int N, int MODE, int NACC>
__global__ void __launch_bounds__(128, 1) mma_loop(int iters, long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  // zero smem operands
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = __shfl_sync(0xffffffffu, tslot, 0);
  constexpr uint32_t idesc = idesc_f16_m128(N);
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    const uint64_t bdesc = sdesc_kmajor_sw128(smem_u32(smem));             // B: N rows
    const uint64_t adesc = sdesc_kmajor_sw128(smem_u32(smem + 32 * 1024));  // A (SS): 128 rows
    const uint32_t e = elect_one();
    const uint32_t d0 = tb + 256;  // D region
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const uint32_t d = d0 + (j % NACC) * N;
        if (MODE == 0) {
          mma_f16_ts_if(e, d, tb + j * 8, static_cast<uint32_t>(bdesc) + (j & 3) * 2, static_cast<uint32_t>(bdesc >> 32),
                        idesc, 1u);
        } else {
          asm volatile(
              "{\n\t.reg .pred p, q;\n\t"
              "setp.ne.b32 q, %0, 0;\n\t"
              "setp.ne.b32 p, 1, 0;\n\t"
              "@q tcgen05.mma.cta_group::1.kind::f16 [%1], %2, %3, %4, p;\n\t}" ::"r"(e),
              "r"(d), "l"(adesc + (j & 3) * 2), "l"(bdesc + (j & 3) * 2), "r"(idesc)
              : "memory");
        }
      }
    }
    tc_commit_if(e, &bar);
    mbar_wait(&bar, 0);
    t1 = clock64();
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tb, 512);
  }
}

template <int N, int MODE, int NACC>
void run(int ctas) {
  long long* d;
  cudaMalloc(&d, sizeof(long long) * ctas);
  auto k = mma_loop<N, MODE, NACC>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int iters = 512;
  k<<<ctas, 128, 96 * 1024>>>(8, d);
  k<<<ctas, 128, 96 * 1024>>>(iters, d);
  cudaError_t err = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof(long long) * ctas, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < ctas; ++i) mx = h[i] > mx ? h[i] : mx;
  printf("%s N=%3d nacc=%d ctas=%3d: %.1f cycles/MMA  (%s)\n", MODE == 0 ? "TS" : "SS", N, NACC, ctas,
         mx / (iters * 8.0), cudaGetErrorString(err));
  cudaFree(d);
}

int main() {
  for (int ctas : {1, 148}) {
    run<16, 0, 1>(ctas);
    run<16, 0, 4>(ctas);
    run<16, 0, 8>(ctas);
    run<16, 1, 4>(ctas);
    run<32, 0, 4>(ctas);
    run<32, 1, 4>(ctas);
    run<64, 0, 2>(ctas);
    run<64, 1, 2>(ctas);
    run<128, 0, 1>(ctas);
    run<128, 1, 1>(ctas);
    run<192, 0, 1>(ctas);
    run<192, 1, 1>(ctas);
    run<256, 0, 1>(ctas);
    run<256, 1, 1>(ctas);
  }
  return 0;
}
