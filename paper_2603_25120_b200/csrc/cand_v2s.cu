// cand_v2s.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v2s, u64, false, true, false)
}  // namespace dflop
