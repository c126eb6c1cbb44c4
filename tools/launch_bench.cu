// launch_bench.cu — microbenchmark: fixed cost of a persistent 148-CTA kernel
// shaped like the W6A16 GEMM (768 threads, ~198 KB dynamic smem, 512-column
// TMEM alloc, mbarrier init), and of a pure bulk-copy weight stream at the
// GEMM's stage size.  Dev tool (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/launch_bench.cu -o build/launch_bench -lcuda
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <vector>

#include "../paper_2312_08583_b200/csrc/common.cuh"

using namespace lpqt;

template <bool TMEM>
__global__ void __launch_bounds__(768, 1) empty_like(int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[32];
  const int warp = threadIdx.x / 32;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 32; ++i) mbar_init(&bar[i], 1);
    fence_mbar_init();
  }
  if (TMEM && warp == 18) {
    tmem_alloc(&tslot, 512);
    tmem_relinquish();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0 && sink) sink[blockIdx.x] = smem[0];
  tc_fence_before();
  __syncthreads();
  if (TMEM && warp == 18) {
    tc_fence_after();
    tmem_dealloc(__shfl_sync(0xffffffffu, tslot, 0), 512);
  }
}

// each CTA streams `per_cta` bytes of `src` through a STAGES-deep ring of
// `stage` bytes with 1-D bulk copies; one consumer warp waits + releases.
__global__ void __launch_bounds__(64, 1) stream_kernel(const uint8_t* src, int64_t per_cta, int stage, int stages,
                                                     int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const uint8_t* base = src + (int64_t)blockIdx.x * per_cta;
  const int n = static_cast<int>(per_cta / stage);
  const uint64_t pol = l2_evict_first_policy();
  if (warp == 0) {
    for (int it = 0; it < n; ++it) {
      const int s = it % stages;
      mbar_wait(&empty[s], ((it / stages) & 1) ^ 1);
      const uint32_t e = elect_one();
      mbar_arrive_expect_tx_if(e, &full[s], stage);
      bulk_g2s_if(e, smem + s * stage, base + (int64_t)it * stage, stage, &full[s], pol);
    }
  } else {
    int acc = 0;
    for (int it = 0; it < n; ++it) {
      const int s = it % stages;
      mbar_wait(&full[s], (it / stages) & 1);
      acc += smem[s * stage + lane * 4];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (lane == 0 && acc == 0x7fffffff) sink[0] = acc;
  }
}

static float time_it(cudaStream_t st, void (*fn)(cudaStream_t, void*), void* ctx, int iters, void* flush,
                     size_t flush_bytes) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  std::vector<float> ts;
  for (int i = 0; i < iters; ++i) {
    if (flush) cudaMemsetAsync(flush, i & 0xff, flush_bytes, st);
    cudaEventRecord(a, st);
    fn(st, ctx);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    ts.push_back(ms * 1000.f);
  }
  std::sort(ts.begin(), ts.end());
  return ts[ts.size() / 2];
}

struct StreamCtx {
  const uint8_t* src;
  int64_t per_cta;
  int stage, stages, grid;
  int* sink;
};

int main() {
  int* sink;
  cudaMalloc(&sink, 4096);
  const int smem_big = 198 * 1024;
  cudaFuncSetAttribute(empty_like<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big);
  cudaFuncSetAttribute(empty_like<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_big);
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaStream_t st;
  cudaStreamCreate(&st);
  void* flush;
  const size_t fb = 512ull << 20;
  cudaMalloc(&flush, fb);
  struct E {
    int smem;
    bool tmem;
  };
  for (E e : {E{smem_big, true}, E{smem_big, false}, E{0, false}, E{0, true}}) {
    auto fn = e.tmem ? +[](cudaStream_t s, void* c) {
      empty_like<true><<<148, 768, *static_cast<int*>(c), s>>>(nullptr);
    }
                     : +[](cudaStream_t s, void* c) { empty_like<false><<<148, 768, *static_cast<int*>(c), s>>>(nullptr); };
    int sm = e.smem;
    float t = time_it(st, fn, &sm, 50, nullptr, 0);
    float tf = time_it(st, fn, &sm, 50, flush, fb);
    printf("empty kernel 148x768 smem=%d tmem=%d: %.2f us (after L2 flush memset: %.2f us)\n", e.smem, e.tmem, t, tf);
  }
  // weight stream: 176 MB (70B down FP6) and 12.6 MB (7B O) over 148 CTAs
  uint8_t* src;
  const int64_t big = 180ll << 20;
  cudaMalloc(&src, big);
  cudaMemset(src, 1, big);
  for (int64_t total : {(int64_t)12582912, (int64_t)67633152, (int64_t)176160768}) {
    for (int stage : {12288, 24576, 49152}) {
      for (int stages : {2, 4, 6, 8}) {
        if ((int64_t)stage * stages > 200 * 1024) continue;
        StreamCtx c{src, (total / 148) / stage * stage, stage, stages, 148, sink};
        auto fn = +[](cudaStream_t s, void* p) {
          auto* c = static_cast<StreamCtx*>(p);
          stream_kernel<<<c->grid, 64, c->stage * c->stages, s>>>(c->src, c->per_cta, c->stage, c->stages, c->sink);
        };
        float t = time_it(st, fn, &c, 20, flush, fb);
        const double bytes = (double)c.per_cta * 148;
        printf("stream total=%.1fMB stage=%d stages=%d: %.2f us  %.0f GB/s\n", bytes / 1e6, stage, stages, t,
               bytes / t / 1e3);
      }
    }
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
