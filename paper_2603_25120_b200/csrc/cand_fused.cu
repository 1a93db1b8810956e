// cand_fused.cu -- instantiation unit of the fused pipeline kernel (cand_impl.cuh)
#include "cand_impl.cuh"

namespace dflop {
const void* fused_kernel_ptr(int gl, bool o4) { return o4 ? ptr_fused_gl<true>(gl) : ptr_fused_gl<false>(gl); }

void fused_launch(int gl, uint32_t grid, uint32_t threads, size_t dyn, const CandParams& p, const FusedParams& f,
                  cudaStream_t s) {
    if (p.order4)
        launch_fused_gl<true>(gl, grid, threads, dyn, p, f, s);
    else
        launch_fused_gl<false>(gl, grid, threads, dyn, p, f, s);
}
}  // namespace dflop
