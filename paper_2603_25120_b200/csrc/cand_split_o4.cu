// cand_split_o4.cu -- the split pipeline's candidate kernel with ORDER4 (cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_SPLIT_UNIT(o4, true)
}  // namespace dflop
