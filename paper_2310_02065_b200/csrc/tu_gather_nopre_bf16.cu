// tu_gather_nopre_bf16.cu — SpMM kernel instantiations without pre-ordered metadata (one
// compilation unit of libvenom; spmm_launch.cuh)
#include "spmm_launch.cuh"

namespace venom {
namespace launch {
venom_status_t gather_nopre_bf16(VENOM_GATHER_ARGS) { return run_gather<false, true>(NBg, pair, tile_t, tv, tb, te, tc, p, max_ctas, s); }
}  // namespace launch
}  // namespace venom
