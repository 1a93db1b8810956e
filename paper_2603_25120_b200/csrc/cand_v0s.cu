// cand_v0s.cu -- instantiation unit of the candidate kernel (see cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
DFLOP_CAND_UNIT(v0s, uint32_t, true, true, false)

// the split pipeline's LPT kernel (packed u32, shared-memory table)
const void* lpt_kernel_ptr(int gl) {
    switch (gl) {
        case 1: return reinterpret_cast<const void*>(&k_lpt<1>);
        case 2: return reinterpret_cast<const void*>(&k_lpt<2>);
        case 4: return reinterpret_cast<const void*>(&k_lpt<4>);
        default: return reinterpret_cast<const void*>(&k_lpt<8>);
    }
}

void lpt_launch(int gl, uint32_t grid, uint32_t cpb, size_t dyn, const CandParams& p, cudaStream_t s) {
    switch (gl) {
        case 1: k_lpt<1><<<grid, cpb * 1, dyn, s>>>(p); break;
        case 2: k_lpt<2><<<grid, cpb * 2, dyn, s>>>(p); break;
        case 4: k_lpt<4><<<grid, cpb * 4, dyn, s>>>(p); break;
        default: k_lpt<8><<<grid, cpb * 8, dyn, s>>>(p); break;
    }
}
}  // namespace dflop
