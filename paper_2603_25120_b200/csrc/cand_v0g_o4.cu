// cand_v0g_o4.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v0g_o4, uint32_t, true, false, true)
}  // namespace dflop
