// tu_gather_pre_f16.cu — SpMM kernel instantiations (one compilation unit of libvenom; spmm_launch.cuh)
#include "spmm_launch.cuh"

namespace venom {
namespace launch {
venom_status_t gather_pre_f16(VENOM_GATHER_ARGS) { return run_gather<true,false>(NBg, pair, tile_t, tv, tb, te, tc, p, max_ctas, s); }
}  // namespace launch
}  // namespace venom
