// sg_common.cuh -- shared host/device helpers for libseisgpu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>

#include <nvtx3/nvToolsExt.h>

#include "seisgpu.h"

namespace sg {

extern thread_local std::string g_err;
extern std::atomic<int64_t> g_launches;

inline int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define SG_CK(x)                                                                       \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      return ::sg::fail(SG_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define SG_TRY(x)            \
  do {                       \
    int rc_ = (x);           \
    if (rc_ != SG_OK) return rc_; \
  } while (0)

// NVTX range around a C-ABI call (header-only NVTX v3: a no-op unless a
// tool such as ncu --nvtx injects itself)
struct Trace {
  explicit Trace(const char* name) { nvtxRangePushA(name); }
  ~Trace() { nvtxRangePop(); }
  Trace(const Trace&) = delete;
  Trace& operator=(const Trace&) = delete;
};

inline void count_launch(int64_t n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// Device allocations of the library.  With SG_REDZONE=1 in the environment
// every allocation carries a 64 KB guard zone of 0xFF bytes (NaN as fp32 and
// fp64) on both sides: an out-of-bounds read poisons the result with NaN, an
// out-of-bounds write is found by rz_check / at free time (sg_redzone_check).
// The library's own memcheck: compute-sanitizer is not available on the GPU
// pool this was built on.  (sg_prop.cu defines these.)
cudaError_t rz_malloc(void** p, size_t bytes);
void rz_free(void* p);

// deterministic block reduction of a double (blockDim.x multiple of 32, <= 1024)
__device__ __forceinline__ double block_sum(double v) {
  __shared__ double red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[wid] = v;
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  v = (threadIdx.x < nw) ? red[threadIdx.x] : 0.0;
  if (wid == 0) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  }
  return v;  // valid in thread 0
}

}  // namespace sg
