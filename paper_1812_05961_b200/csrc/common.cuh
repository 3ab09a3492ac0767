// common.cuh — shared internals of libsplatt_b200 (CUDA path only; no oracle code).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <mutex>
#include <set>
#include <utility>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/splatt_b200.h"

namespace sb {

// Internal failure carrying an ABI status; caught at the C boundary (abi.cu).
struct Error : std::runtime_error {
  splatt_status code;
  Error(splatt_status c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void fail(splatt_status c, const std::string& m) { throw Error(c, m); }

#define SB_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      ::sb::fail(e_ == cudaErrorMemoryAllocation ? SPLATT_ERR_NOMEM : SPLATT_ERR_CUDA,  \
                 std::string(#call) + ": " + cudaGetErrorString(e_));                   \
  } while (0)

#define SB_STR2_(x) #x
#define SB_STR_(x) SB_STR2_(x)
// Launch check; the message names the launch site (with CUDA_LAUNCH_BLOCKING=1 an
// asynchronous fault is then attributed to the kernel that caused it).
#define SB_CHECK_LAUNCH(ctx)                                                            \
  do {                                                                                  \
    (ctx)->kernel_launches++;                                                           \
    cudaError_t e_ = cudaGetLastError();                                                \
    if (e_ != cudaSuccess)                                                              \
      ::sb::fail(SPLATT_ERR_CUDA, std::string("kernel launch at " __FILE__ ":"         \
                                              SB_STR_(__LINE__) ": ") +                 \
                                      cudaGetErrorString(e_));                          \
  } while (0)

#define SB_REQUIRE(cond, msg) \
  do { if (!(cond)) ::sb::fail(SPLATT_ERR_BADINPUT, msg); } while (0)

// Internal leading dimension of every factor / MTTKRP buffer: ceil(R/4)*4 doubles,
// so each row is a whole number of 32-byte sectors and 256-bit loads stay aligned
// (SURVEY.md §8(a) a3).
inline int padded_ld(int R) { return (R + 3) / 4 * 4; }

inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Opt a kernel in to `bytes` of dynamic shared memory on the CURRENT device (the attribute is
// per device: a process with contexts on several GPUs must set it on each).  Once per
// (kernel, device); thread-safe (loopback ranks are threads).
inline void set_max_dynamic_smem(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  int dev = 0;
  SB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done.count({kernel, dev})) return;
  SB_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
  done.insert({kernel, dev});
}

}  // namespace sb
