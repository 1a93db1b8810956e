// cand_v0g.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v0g, uint32_t, true, false, false)
}  // namespace dflop
