// mttkrp.hpp — CSF MTTKRP launcher (mttkrp.cu, kernel in mttkrp_kernel.cuh).
#pragma once
#include "csf.hpp"

namespace sb {

// out (out_rows x ld, ld % 4 == 0, 32-byte aligned rows) = MTTKRP for the mode at CSF
// level `level` of `c` (mode c.perm[level]): level 0 = ROOT traversal (owned rows),
// 1..N-2 = INTERNAL, N-1 = LEAF (atomic row updates).  fac_by_mode[m] are the factors
// (same ld); fac_by_mode[c.perm[level]] is unused.  Zero-fills `out` first (rows without
// nonzeros are 0).  Stream-ordered on ctx.  If tm is given, only the kernel (not the
// zero-fill) is timed under category `cat`.
// l1a: ROOT gather cache policy, -1 = the tree's choice (c.l1a; no_allocate if untimed),
// 0 = L1::no_allocate, 1 = L1-allocating (env SPLATT_L1_ALLOC=0/1 overrides both).
void mttkrp_level(splatt_ctx* ctx, DevCsf& c, int level, const double* const* fac_by_mode,
                  double* out, uint64_t out_rows, int ld, int R, EventTimer* tm = nullptr,
                  int cat = 0, int l1a = -1);

// Per-tree MTTKRP metadata for output level `level` (chunk table; for level > 0 the hot
// output ids), built once; mttkrp_level builds it on first use if this was not called.
// May synchronise the context stream.
void mttkrp_prepare(splatt_ctx* ctx, DevCsf& c, int level, int ld);

inline void mttkrp_root(splatt_ctx* ctx, DevCsf& c, const double* const* fac_by_mode,
                        double* out, uint64_t out_rows, int ld, int R, EventTimer* tm = nullptr,
                        int cat = 0) {
  mttkrp_level(ctx, c, 0, fac_by_mode, out, out_rows, ld, R, tm, cat);
}

// Algorithmic bytes of one MTTKRP over `c` at rank R for output level `level`
// (SURVEY.md §8(d) B_alg for level 0; DESIGN.md §4.2 for the others).
double mttkrp_alg_bytes(const DevCsf& c, int R, int level = 0);
// Compulsory bytes of one launch (tree once, referenced factor rows once, output once);
// distinct[m] = rows of mode m the tensor references (or an upper bound).
double mttkrp_min_bytes(const DevCsf& c, int R, int level, const uint64_t* distinct);

// Second-generation ROOT kernel (root2.cu): whether tree `c` runs it (N = 3, 4; non-root
// level dims < 2^28; not in deterministic mode; SPLATT_ROOT2=0 disables it), its plan, and
// its launch (acc bit 0: add into the owned rows).
bool root2_eligible(const splatt_ctx* ctx, const DevCsf& c, int ld);
void ensure_root_plan(splatt_ctx* ctx, DevCsf& c, int ld);
int root2_table_chunk();  // leaves per chunk-table entry of a tree the kernel runs
void mttkrp_root2_launch(splatt_ctx* ctx, DevCsf& c, const double* const* fac_by_mode,
                         double* out, int ld, int R, int acc);

// Leaves per ROOT/INTERNAL/LEAF work unit of tree `c` (its chunk table's granularity).
int mttkrp_chunk_leaves(const DevCsf& c);

}  // namespace sb
