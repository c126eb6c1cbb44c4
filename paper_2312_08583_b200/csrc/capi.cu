// capi.cu — library-wide C ABI pieces: status strings, ABI version, the
// launch counter behind the bench's `gpu_launches` claim.
#include <atomic>

#include "common.cuh"

namespace lpqt {

static std::atomic<int64_t> g_launches{0};

void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

int check_launch() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? LPQT_OK : LPQT_E_CUDA;
}

}  // namespace lpqt

extern "C" {

const char* lpqt_strerror(int status) {
  switch (status) {
    case LPQT_OK: return "ok";
    case LPQT_E_INVALID_INPUT: return "invalid input (InvalidInput)";
    case LPQT_E_SHAPE: return "shape mismatch (ShapeError)";
    case LPQT_E_SCALE_OVERFLOW: return "folded scale exceeds binary16 range (ScaleOverflow)";
    case LPQT_E_PAYLOAD: return "payload inconsistent with code count (PayloadMismatch)";
    case LPQT_E_INVALID_CODE: return "code does not fit 6 bits (InvalidCode)";
    case LPQT_E_UNSUPPORTED: return "unsupported dtype or layout";
    case LPQT_E_WORKSPACE: return "workspace missing or too small";
    case LPQT_E_CUDA: return cudaGetErrorString(cudaPeekAtLastError());
    default: return "unknown lpqt status";
  }
}

int lpqt_abi_version(void) { return 6; }

int64_t lpqt_launch_count(void) { return lpqt::g_launches.load(std::memory_order_relaxed); }

}  // extern "C"
