// cand_split.cu -- instantiation unit of the split pipeline's candidate kernel (cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_SPLIT_UNIT(plain, false)
}  // namespace dflop
