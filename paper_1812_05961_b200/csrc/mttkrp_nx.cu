// mttkrp_nx.cu — N = 5..8 instantiations of the CSF MTTKRP kernel (mttkrp_kernel.cuh).
// Not on any configured workload (c1-c5 are 3- and 4-mode): two lane-group widths only.
#include "mttkrp_kernel.cuh"

namespace sb {

namespace {
template <int N, int D>
void go(splatt_ctx* ctx, DevCsf& c, int level, const double* const* f, double* out, int ld,
        int R, int chunk, int acc) {
  if constexpr (D < N) {
    if (level == D) return mk::launch_g<N, D, 2, 1, false>(ctx, c, f, out, ld, R, chunk, acc);
    return go<N, D + 1>(ctx, c, level, f, out, ld, R, chunk, acc);
  } else {
    fail(SPLATT_ERR_BADINPUT, "level out of range");
  }
}
}  // namespace

void mttkrp_launch_nx(splatt_ctx* ctx, DevCsf& c, int D, const double* const* f, double* out,
                      int ld, int R, int chunk, int acc) {
  switch (c.N) {
    case 5: return go<5, 0>(ctx, c, D, f, out, ld, R, chunk, acc);
    case 6: return go<6, 0>(ctx, c, D, f, out, ld, R, chunk, acc);
    case 7: return go<7, 0>(ctx, c, D, f, out, ld, R, chunk, acc);
    case 8: return go<8, 0>(ctx, c, D, f, out, ld, R, chunk, acc);
    default: fail(SPLATT_ERR_BADINPUT, "nmodes out of range");
  }
}

}  // namespace sb
