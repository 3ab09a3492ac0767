// mttkrp_n4.cu — N = 4 instantiations of the CSF MTTKRP kernel (mttkrp_kernel.cuh).
#include "mttkrp_kernel.cuh"

namespace sb {

#ifndef SB_MTTKRP_U4
#define SB_MTTKRP_U4 2
#endif
#ifndef SB_MTTKRP_MINB4
#define SB_MTTKRP_MINB4 2
#endif

void mttkrp_launch_n4(splatt_ctx* ctx, DevCsf& c, int D, const double* const* f, double* out,
                      int ld, int R, int chunk, int acc) {
  constexpr int U = SB_MTTKRP_U4, MB = SB_MTTKRP_MINB4;
  switch (D) {
    case 0: return mk::launch_g<4, 0, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    case 1: return mk::launch_g<4, 1, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    case 2: return mk::launch_g<4, 2, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    case 3: return mk::launch_g<4, 3, U, MB, true>(ctx, c, f, out, ld, R, chunk, acc);
    default: fail(SPLATT_ERR_BADINPUT, "level out of range");
  }
}

}  // namespace sb
