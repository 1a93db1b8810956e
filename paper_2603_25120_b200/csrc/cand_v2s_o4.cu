// cand_v2s_o4.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v2s_o4, u64, false, true, true)
}  // namespace dflop
