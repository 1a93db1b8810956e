// cand_v2g.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v2g, u64, false, false, false)
}  // namespace dflop
