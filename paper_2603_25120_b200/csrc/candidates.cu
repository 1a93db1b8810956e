// candidates.cu -- dispatch of the candidate kernel variants (cand_impl.cuh, cand_v*.cu).
#include "cand.cuh"

namespace dflop {

const void* cand_ptr_v0s(int gl);
void cand_launch_v0s(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v0s_o4(int gl);
void cand_launch_v0s_o4(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v0g(int gl);
void cand_launch_v0g(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v0g_o4(int gl);
void cand_launch_v0g_o4(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v1s(int gl);
void cand_launch_v1s(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v1s_o4(int gl);
void cand_launch_v1s_o4(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v1g(int gl);
void cand_launch_v1g(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v1g_o4(int gl);
void cand_launch_v1g_o4(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v2s(int gl);
void cand_launch_v2s(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v2s_o4(int gl);
void cand_launch_v2s_o4(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v2g(int gl);
void cand_launch_v2g(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* cand_ptr_v2g_o4(int gl);
void cand_launch_v2g_o4(const CandLaunch& L, const CandParams& p, cudaStream_t s);

const void* split_ptr_plain(int gl);
void split_launch_plain(const CandLaunch& L, const CandParams& p, cudaStream_t s);
const void* split_ptr_o4(int gl);
void split_launch_o4(const CandLaunch& L, const CandParams& p, cudaStream_t s);

const void* split_kernel_ptr(int gl, bool o4) { return o4 ? split_ptr_o4(gl) : split_ptr_plain(gl); }

void split_launch(const CandLaunch& L, const CandParams& p, cudaStream_t s) {
    if (p.order4)
        split_launch_o4(L, p, s);
    else
        split_launch_plain(L, p, s);
}

const void* cand_kernel_ptr(int variant, int gl, bool tbl_smem, bool o4) {
    if (o4) switch (variant) {
            case 0: return tbl_smem ? cand_ptr_v0s_o4(gl) : cand_ptr_v0g_o4(gl);
            case 1: return tbl_smem ? cand_ptr_v1s_o4(gl) : cand_ptr_v1g_o4(gl);
            default: return tbl_smem ? cand_ptr_v2s_o4(gl) : cand_ptr_v2g_o4(gl);
        }
    switch (variant) {
        case 0: return tbl_smem ? cand_ptr_v0s(gl) : cand_ptr_v0g(gl);
        case 1: return tbl_smem ? cand_ptr_v1s(gl) : cand_ptr_v1g(gl);
        default: return tbl_smem ? cand_ptr_v2s(gl) : cand_ptr_v2g(gl);
    }
}

void cand_launch(const CandLaunch& L, const CandParams& p, cudaStream_t s) {
    if (p.order4) {
        switch (L.variant) {
            case 0: L.tbl_smem ? cand_launch_v0s_o4(L, p, s) : cand_launch_v0g_o4(L, p, s); break;
            case 1: L.tbl_smem ? cand_launch_v1s_o4(L, p, s) : cand_launch_v1g_o4(L, p, s); break;
            default: L.tbl_smem ? cand_launch_v2s_o4(L, p, s) : cand_launch_v2g_o4(L, p, s); break;
        }
        return;
    }
    switch (L.variant) {
        case 0: L.tbl_smem ? cand_launch_v0s(L, p, s) : cand_launch_v0g(L, p, s); break;
        case 1: L.tbl_smem ? cand_launch_v1s(L, p, s) : cand_launch_v1g(L, p, s); break;
        default: L.tbl_smem ? cand_launch_v2s(L, p, s) : cand_launch_v2g(L, p, s); break;
    }
}

}  // namespace dflop
