// cand_v0s.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v0s, uint32_t, true, true, false)
}  // namespace dflop
