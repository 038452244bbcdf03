// tu_densek_f16.cu — dense-K SpMM kernel instantiations (one compilation unit of libvenom;
// spmm_launch.cuh)
#include "spmm_launch.cuh"

namespace venom {
namespace launch {
venom_status_t densek_f16(VENOM_DENSEK_ARGS) { return run_densek_cfg<false>(M, pair, tile_t, tb, enc, p, max_ctas, s); }
}  // namespace launch
}  // namespace venom
