// mttkrp.cu — CSF MTTKRP host entry points and the N = 3 instantiations (SURVEY.md §8(a)
// a6, §8(f) NEXT-1).  The kernel is mttkrp_kernel.cuh.
#include "mttkrp.hpp"
#include "mttkrp_kernel.cuh"

namespace sb {

#ifndef SB_MTTKRP_U
#define SB_MTTKRP_U 2
#endif
#ifndef SB_MTTKRP_MINB
#define SB_MTTKRP_MINB 3
#endif

void mttkrp_launch_n3(splatt_ctx* ctx, DevCsf& c, int D, const double* const* f, double* out,
                      int ld, int R, int chunk) {
  constexpr int U = SB_MTTKRP_U, MB = SB_MTTKRP_MINB;
  switch (D) {
    case 0: return mk::launch_g<3, 0, U, MB, true>(ctx, c, f, out, ld, R, chunk);
    case 1: return mk::launch_g<3, 1, U, MB, true>(ctx, c, f, out, ld, R, chunk);
    case 2: return mk::launch_g<3, 2, U, MB, true>(ctx, c, f, out, ld, R, chunk);
    default: fail(SPLATT_ERR_BADINPUT, "level out of range");
  }
}

// Leaves per work unit (measured on B200: c2/c4 best at 256 for N = 3, c5 at 512 for N = 4;
// shorter chunks balance better, longer ones amortise the per-chunk setup and seam rows).
#ifndef SB_MTTKRP_CHUNK3
#define SB_MTTKRP_CHUNK3 256
#endif
#ifndef SB_MTTKRP_CHUNK
#define SB_MTTKRP_CHUNK 512
#endif

int mttkrp_chunk_leaves(int N, int ld) {
  (void)ld;
  return N == 3 ? SB_MTTKRP_CHUNK3 : SB_MTTKRP_CHUNK;
}

double mttkrp_alg_bytes(const DevCsf& c, int R, int level) {
  // B_alg = CSF index/value bytes + factor-row bytes: 12 B per leaf
  // (id + value), 8 B per internal node (id + ptr), plus 8 R bytes per gathered factor
  // row — one per node of every level except the output level D and the root (root:
  // SURVEY's formula exactly) — and, for D > 0, 8 R bytes per output-row update (one
  // atomic row per level-D node; a root MTTKRP writes each owned row once, not counted).
  const int N = c.N;
  double internal = 0.0;
  for (int l = 0; l < N - 1; ++l) internal += (double)c.nodes[l];
  double rows = 0.0;
  for (int l = 0; l < N; ++l)
    if (l != level && l != 0) rows += (double)c.nodes[l];
  if (level > 0) rows += (double)c.nodes[0] + (double)c.nodes[level];
  return 12.0 * (double)c.nnz + 8.0 * internal + 8.0 * R * rows;
}

void mttkrp_level(splatt_ctx* ctx, DevCsf& c, int level, const double* const* fac_by_mode,
                  double* out, uint64_t out_rows, int ld, int R, EventTimer* tm, int cat) {
  if (ld % 4 != 0) fail(SPLATT_ERR_BADINPUT, "internal: ld must be a multiple of 4");
  if (level < 0 || level >= c.N) fail(SPLATT_ERR_BADINPUT, "internal: level out of range");
  if (tm) tm->gap();  // the zero-fill is not part of the timed kernel
  SB_CUDA(cudaMemsetAsync(out, 0, out_rows * (size_t)ld * sizeof(double), ctx->stream));
  if (c.nnz == 0) return;
  const int chunk = mttkrp_chunk_leaves(c.N, ld);
  ensure_chunk_table(ctx, c, chunk);
  if (tm) tm->begin(cat);
  switch (c.N) {
    case 3: mttkrp_launch_n3(ctx, c, level, fac_by_mode, out, ld, R, chunk); break;
    case 4: mttkrp_launch_n4(ctx, c, level, fac_by_mode, out, ld, R, chunk); break;
    default: mttkrp_launch_nx(ctx, c, level, fac_by_mode, out, ld, R, chunk); break;
  }
  if (tm) tm->end();
}

}  // namespace sb
