// Shared helpers for libhiermoe (sm_100a).  Status convention of the C-ABI:
//   0   ok
//   <0  invalid argument (Python raises ValueError), message via hm_last_error()
//   >0  CUDA error code (Python raises RuntimeError)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX3: ranges cost a null check without a tool

#define HM_API extern "C" __attribute__((visibility("default")))

namespace hm {

void set_error(const char* fmt, ...);

constexpr int kInvalid = -1;
constexpr int kOverflow = -2;     // device-side capacity/consistency flag raised
constexpr int kNotReady = -3;     // world not initialised / peers not opened

inline int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return 0;
  set_error("CUDA error %d: %s", (int)e, cudaGetErrorString(e));
  return (int)e;
}

// kernels launched by this library since load (every launch is followed by
// exactly one HM_LAUNCHED / launch_status check); read with hm_launch_count()
inline std::atomic<unsigned long long>& launch_counter() {
  static std::atomic<unsigned long long> n{0};
  return n;
}

inline int launch_status() {
  launch_counter().fetch_add(1, std::memory_order_relaxed);
  return cuda_status(cudaGetLastError());
}

inline int grid_for(int64_t work, int per_block, int max_blocks) {
  int64_t b = (work + per_block - 1) / per_block;
  if (b < 1) b = 1;
  if (b > max_blocks) b = max_blocks;
  return (int)b;
}

constexpr int kSMs = 148;

// NVTX range over one C-ABI call (SURVEY §5 tracing): nsys / ncu --nvtx show
// every dispatch / combine / FFN / planner call as a named range
struct Range {
  explicit Range(const char* name) { nvtxRangePushA(name); }
  ~Range() { nvtxRangePop(); }
  Range(const Range&) = delete;
  Range& operator=(const Range&) = delete;
};

}  // namespace hm

#define HM_RANGE(name) hm::Range _hm_nvtx_range(name)

#define HM_CHECK_ARG(cond, ...)            \
  do {                                     \
    if (!(cond)) {                         \
      hm::set_error(__VA_ARGS__);          \
      return hm::kInvalid;                 \
    }                                      \
  } while (0)

#define HM_CUDA(call)                                   \
  do {                                                  \
    int _st = hm::cuda_status(call);                    \
    if (_st) return _st;                                \
  } while (0)

#define HM_LAUNCHED()                 \
  do {                                \
    int _st = hm::launch_status();    \
    if (_st) return _st;              \
  } while (0)
