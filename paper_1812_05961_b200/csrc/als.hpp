// als.hpp — CP-ALS driver and device-side COO view.
#pragma once
#include "ctx.hpp"

namespace sb {

// COO on the device (borrowed pointers; see abi.cu for the host->device upload).
struct DevCoo {
  int N = 0;
  uint64_t nnz = 0;
  uint64_t dims[SPLATT_MAX_NMODES] = {0};
  const uint32_t* ind[SPLATT_MAX_NMODES] = {nullptr};
  const double* vals = nullptr;
};

struct AlsOut {
  double* factors[SPLATT_MAX_NMODES];  // host or device, ld = R
  double* lambda;                      // host or device
  double* fit;                         // host
  int32_t* iters;                      // host
  double* fit_history;                 // host or NULL
};

// Algorithm 1 on a device COO (validated here).  init: NULL or N pointers (host or
// device, ld = R).  policy: SPLATT_CSF_ALL / ONE / TWO (ALL only when sharded).
// Throws sb::Error.
void cpd_als_device(splatt_ctx* ctx, const DevCoo& X, int R, int max_iters, double tol,
                    uint64_t seed, const double* const* init, int policy, const AlsOut& out,
                    splatt_stats* st);

// C-14 partition (host).
void host_partition(const uint64_t* w, uint64_t S, int G, uint64_t* bounds);

void nccl_unique_id(void* id128);

}  // namespace sb
