// als.hpp — CP-ALS driver and device-side COO view.
#pragma once
#include "ctx.hpp"

struct splatt_csf;

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
// prebuilt: a CSF set from splatt_csf_build (X then only supplies N, nnz and dims; no
// validation or build) or NULL.
void cpd_als_device(splatt_ctx* ctx, const DevCoo& X, int R, int max_iters, double tol,
                    uint64_t seed, const double* const* init, int policy, const AlsOut& out,
                    splatt_stats* st, const splatt_csf* prebuilt = nullptr);

// C-14 partition (host).
void host_partition(const uint64_t* w, uint64_t S, int G, uint64_t* bounds);

// P2 partition: the nonzeros of a mode in slice-major order
// (slices ascending, a slice's nonzeros in input order) are cut into G equal leaf ranges
// [k_g, k_{g+1}), k_g = floor(g nnz / G); slices may be split.  The row of a slice is owned
// by the rank holding its first nonzero; split slices are exchanged through `slots`.
struct NnzPart {
  std::vector<uint64_t> rowb;   // G+1 row bounds: rank g owns rows [rowb[g], rowb[g+1])
  std::vector<uint64_t> slots;  // the split slices (distinct, ascending): exchange slots
  // this rank's share: whole slices [full_lo, full_hi) and up to two partial slices
  uint64_t full_lo = 0, full_hi = 0;
  int npart = 0;
  uint64_t pslice[2] = {0, 0}, pa[2] = {0, 0}, pb[2] = {0, 0};  // within-slice ranks [a, b)
  int pslot[2] = {-1, -1};      // slot of each partial slice
};
void host_partition_nnz(const uint64_t* w, uint64_t S, int G, int me, NnzPart& out);

void nccl_unique_id(void* id128);

}  // namespace sb
