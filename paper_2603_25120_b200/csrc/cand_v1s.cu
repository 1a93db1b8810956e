// cand_v1s.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v1s, uint32_t, false, true, false)
}  // namespace dflop
