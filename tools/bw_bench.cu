// bw_bench.cu — microbenchmark: achievable HBM READ bandwidth on B200 for the
// weight-streaming pattern of the decode GEMM, by access method, and the
// kernel-to-kernel gap with and without programmatic dependent launch (PDL).
// Inputs rotate over distinct buffers (> 2x L2 per rotation), timed as CUDA
// graph replays with events.  Dev tool (not part of the library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/bw_bench.cu -o build/bw_bench -lcuda
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_2312_08583_b200/csrc/common.cuh"

using namespace lpqt;

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// (1) 1-D bulk copies through a ring; warp 0 produces, warp 1 consumes.
template <bool PDL>
__global__ void __launch_bounds__(64, 1) bulk_stream(const uint8_t* src, int64_t total, int stage, int stages,
                                                    int* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[32], empty[32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < stages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    fence_mbar_init();
  }
  __syncthreads();
  const int64_t nst = total / stage;
  const int64_t b = nst * blockIdx.x / gridDim.x, e = nst * (blockIdx.x + 1) / gridDim.x;
  const uint64_t pol = l2_evict_first_policy();
  if (warp == 0) {
    for (int64_t it = b; it < e; ++it) {
      const int i = static_cast<int>(it - b), s = i % stages;
      mbar_wait(&empty[s], ((i / stages) & 1) ^ 1);
      const uint32_t el = elect_one();
      mbar_arrive_expect_tx_if(el, &full[s], stage);
      bulk_g2s_if(el, smem + s * stage, src + it * stage, stage, &full[s], pol);
    }
  } else {
    if (PDL) pdl_wait();
    int acc = 0;
    for (int64_t it = b; it < e; ++it) {
      const int i = static_cast<int>(it - b), s = i % stages;
      mbar_wait(&full[s], (i / stages) & 1);
      acc += smem[s * stage + lane * 4];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (PDL) pdl_launch();
    if (lane == 0 && acc == 0x7fffffff) sink[0] = acc;
  }
}

// (2) plain LDG.128 grid-stride streaming, unrolled
template <int U>
__global__ void __launch_bounds__(512) ldg_stream(const uint4* src, int64_t n16, int* sink) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n16; i += U * stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(src + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
  }
  for (; i < n16; i += stride) {
    const uint4 v = __ldcs(src + i);
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

struct Run {
  const char* name;
  int64_t bytes;
  float us;
};

int main() {
  int* sink;
  cudaMalloc(&sink, 4096);
  cudaStream_t st;
  cudaStreamCreate(&st);
  const int64_t pool = 1800ll << 20;
  uint8_t* buf;
  cudaMalloc(&buf, pool);
  cudaMemset(buf, 1, pool);
  cudaFuncSetAttribute(bulk_stream<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaFuncSetAttribute(bulk_stream<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 210 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);

  auto time_graph = [&](auto launch_one, int64_t size, int reps, bool pdl) {
    // rotate over copies so every launch reads cold data
    int copies = static_cast<int>(std::max<int64_t>(2, (600ll << 20) / size + 1));
    if ((int64_t)copies * size > pool) copies = static_cast<int>(pool / size);
    cudaGraph_t g;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int r = 0; r < reps; ++r) launch_one(buf + (int64_t)(r % copies) * size, size, pdl && r > 0);
    cudaStreamEndCapture(st, &g);
    cudaGraphExec_t ge;
    if (cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
      printf("instantiate failed\n");
      return -1.f;
    }
    cudaGraphLaunch(ge, st);
    cudaGraphLaunch(ge, st);
    std::vector<float> ts;
    for (int k = 0; k < 5; ++k) {
      cudaEventRecord(e0, st);
      cudaGraphLaunch(ge, st);
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      ts.push_back(ms * 1000.f / reps);
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    std::sort(ts.begin(), ts.end());
    return ts[ts.size() / 2];
  };

  const int64_t sizes[] = {12582912, 37748736, 67633152, 176160768, 352321536, 1073741824};
  for (int64_t size : sizes) {
    for (int stage : {16384, 24576, 49152}) {
      for (int stages : {4, 8}) {
        if ((int64_t)stage * stages > 200 * 1024) continue;
        for (int cps : {1, 2}) {
          if (cps == 2 && (int64_t)stage * stages > 100 * 1024) continue;
          for (int pdl = 0; pdl < 2; ++pdl) {
            if (pdl && !(stage == 24576 && stages == 8 && cps == 1)) continue;
            auto L = [&](const uint8_t* p, int64_t sz, bool use_pdl) {
              cudaLaunchConfig_t cfg = {};
              cfg.gridDim = dim3(sms * cps);
              cfg.blockDim = dim3(64);
              cfg.dynamicSmemBytes = stage * stages;
              cfg.stream = st;
              cudaLaunchAttribute at[1];
              at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
              at[0].val.programmaticStreamSerializationAllowed = 1;
              cfg.attrs = at;
              cfg.numAttrs = use_pdl ? 1 : 0;
              if (use_pdl)
                cudaLaunchKernelEx(&cfg, bulk_stream<true>, p, sz, stage, stages, sink);
              else
                cudaLaunchKernelEx(&cfg, bulk_stream<false>, p, sz, stage, stages, sink);
            };
            const int reps = size >= (1ll << 30) ? 4 : 20;
            float us = time_graph(L, size, reps, pdl);
            printf("bulk   size=%7.1fMB stage=%5d stages=%d cta/sm=%d pdl=%d: %8.2f us/launch  %6.0f GB/s\n",
                   size / 1e6, stage, stages, cps, pdl, us, size / us / 1e3);
          }
        }
      }
    }
    for (int bps : {2, 4}) {
      auto L = [&](const uint8_t* p, int64_t sz, bool) {
        ldg_stream<4><<<sms * bps, 512, 0, st>>>(reinterpret_cast<const uint4*>(p), sz / 16, sink);
      };
      const int reps = size >= (1ll << 30) ? 4 : 20;
      float us = time_graph(L, size, reps, false);
      printf("ldg128 size=%7.1fMB blocks/sm=%d x512 unroll4:          %8.2f us/launch  %6.0f GB/s\n", size / 1e6,
             bps, us, size / us / 1e3);
    }
    fflush(stdout);
  }
  cudaError_t err = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(err));
  return 0;
}
