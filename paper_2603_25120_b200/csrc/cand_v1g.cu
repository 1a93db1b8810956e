// cand_v1g.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v1g, uint32_t, false, false, false)
}  // namespace dflop
