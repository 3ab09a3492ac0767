// mttkrp.hpp — root-mode CSF MTTKRP launcher (mttkrp.cu).
#pragma once
#include "csf.hpp"

namespace sb {

// out (out_rows x ld, ld % 4 == 0, 32-byte aligned rows) = MTTKRP of CSF `c` rooted at
// mode c.perm[0]; fac_by_mode[m] are the factors (same ld), fac_by_mode[root] unused.
// Zero-fills `out` first (rows without nonzeros are 0).  Stream-ordered on ctx.
// If tm is given, only the kernel (not the zero-fill) is timed under category `cat`.
void mttkrp_root(splatt_ctx* ctx, DevCsf& c, const double* const* fac_by_mode, double* out,
                 uint64_t out_rows, int ld, int R, EventTimer* tm = nullptr, int cat = 0);

// Algorithmic bytes of one MTTKRP over `c` at rank R (SURVEY.md §8(d) B_alg).
double mttkrp_alg_bytes(const DevCsf& c, int R);

int mttkrp_chunk_leaves(int N, int ld);

}  // namespace sb
