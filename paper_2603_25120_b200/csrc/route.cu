// route.cu -- N4(b): the inter-model routing plan: for microbatch slot k the L_dp
// LLM data groups run buckets k * L_dp + rho (R10), so the bucket-major CSR groups of the
// assignment already list the slot's samples in (rho, sample index) order -- pos_item and
// the LLM ranges are the CSR arrays; k_route splits each slot into E_dp contiguous encoder
// ranges balanced by encoder cost (R36): a block-wide exclusive scan of e_i over the slot,
// then per boundary g the first position whose preceding cost reaches g / E_dp of the
// slot's total (binary search on the monotone prefix).  The communicator gathers encoder
// range g and scatters it over the LLM ranges (forward; reversed in the backward pass).
#include <algorithm>

#include "cand.cuh"
#include "internal.h"

namespace dflop {

__global__ void k_route_check(const uint32_t* __restrict__ assign, uint32_t n, uint32_t m, uint32_t* bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (assign[i] >= m) atomicOr(bad, 1u);
}

// one block per slot k
__global__ void __launch_bounds__(256) k_route(const uint32_t* __restrict__ cost, uint32_t n, uint32_t R, uint32_t G,
                                               const uint32_t* __restrict__ offsets, const uint32_t* __restrict__ items,
                                               u64* prefix, uint32_t* slot_off, uint32_t* enc_off, uint32_t* llm_off,
                                               u64* enc_load) {
    __shared__ u64 warp_sums[8];
    __shared__ u64 carry;
    const uint32_t k = blockIdx.x, tid = threadIdx.x, lane = tid & 31u, wid = tid >> 5;
    const uint32_t a = offsets[k * R], b = offsets[(k + 1) * R];
    u64* P = prefix + a + k;  // P[u - a] = encoder cost before position u, u in [a, b]
    for (uint32_t rho = tid; rho <= R; rho += blockDim.x) llm_off[k * (R + 1) + rho] = offsets[k * R + rho];
    if (tid == 0) {
        slot_off[k] = a;
        carry = 0;
    }
    __syncthreads();
    for (uint32_t base = a; base < b; base += blockDim.x) {
        const uint32_t u = base + tid;
        u64 e = 0;
        if (u < b) {
            const uint32_t i = items[u];
            e = (u64)cost[i] + cost[(size_t)n + i];
        }
        u64 inc = e;  // inclusive warp scan
        for (int d = 1; d < 32; d <<= 1) {
            const u64 y = __shfl_up_sync(0xFFFFFFFFu, inc, d);
            if (lane >= (uint32_t)d) inc += y;
        }
        if (lane == 31) warp_sums[wid] = inc;
        __syncthreads();
        u64 wpre = 0;
        for (uint32_t w = 0; w < wid; ++w) wpre += warp_sums[w];
        const u64 c0 = carry;
        if (u < b) P[u - a] = c0 + wpre + inc - e;
        __syncthreads();
        if (tid == blockDim.x - 1) carry = c0 + wpre + inc;
        __syncthreads();
    }
    const u64 tot = carry;
    if (tid == 0) P[b - a] = tot;
    __syncthreads();
    for (uint32_t g = tid; g <= G; g += blockDim.x) {
        uint32_t pos;
        if (g == 0) {
            pos = a;
        } else if (g == G) {
            pos = b;
        } else {  // first u in [a, b] with P(u) * G >= g * tot (P is non-decreasing, P(b) = tot)
            uint32_t lo = 0, hi = b - a;
            while (lo < hi) {
                const uint32_t mid = (lo + hi) / 2;
                if (P[mid] * G >= (u64)g * tot)
                    hi = mid;
                else
                    lo = mid + 1;
            }
            pos = a + lo;
        }
        enc_off[k * (G + 1) + g] = pos;
    }
    __syncthreads();
    if (enc_load)
        for (uint32_t g = tid; g < G; g += blockDim.x)
            enc_load[(size_t)k * G + g] = P[enc_off[k * (G + 1) + g + 1] - a] - P[enc_off[k * (G + 1) + g] - a];
}

size_t route_ws_bytes(uint32_t n, const dflop_plan* p) {
    const uint32_t m = p->n_mb * p->l_dp;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    return al(256) + al((size_t)(m + 1) * 4) + groups_ws_bytes(n, m) + al(((size_t)n + p->n_mb) * 8);
}

dflop_status route_launch(const uint32_t* cost, uint32_t n, const dflop_plan* p, const uint32_t* assign, void* ws,
                          uint32_t* pos_item, uint32_t* slot_off, uint32_t* enc_off, uint32_t* llm_off,
                          uint64_t* enc_load, cudaStream_t s) {
    const uint32_t M = p->n_mb, R = p->l_dp, G = p->e_dp, m = M * R;
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    char* w = reinterpret_cast<char*>(ws);
    uint32_t* bad = reinterpret_cast<uint32_t*>(w);
    uint32_t* offsets = reinterpret_cast<uint32_t*>(w + al(256));
    void* gws = w + al(256) + al((size_t)(m + 1) * 4);
    u64* prefix = reinterpret_cast<u64*>(w + al(256) + al((size_t)(m + 1) * 4) + groups_ws_bytes(n, m));
    cudaError_t ce = cudaMemsetAsync(bad, 0, 4, s);
    if (ce != cudaSuccess) return cuda_status(ce, "memset");
    uint32_t hbad = 0;
    if (n > 0) {
        k_route_check<<<std::min<uint32_t>((n + 255) / 256, 296), 256, 0, s>>>(assign, n, m, bad);
        count_launches(1);
        ce = cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
        if (ce != cudaSuccess) return cuda_status(ce, "route check");
        if (hbad) {
            set_error("assign holds a bucket >= m = %u", m);
            return DFLOP_ERR_INVALID_ARGUMENT;
        }
    }
    ce = groups_launch(assign, n, m, offsets, pos_item, gws, s);
    if (ce != cudaSuccess) return cuda_status(ce, "groups");
    k_route<<<M, 256, 0, s>>>(cost, n, R, G, offsets, pos_item, prefix, slot_off, enc_off, llm_off,
                             reinterpret_cast<u64*>(enc_load));
    count_launches(1);
    ce = cudaMemcpyAsync(slot_off + M, offsets + m, 4, cudaMemcpyDeviceToDevice, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    return cuda_status(ce, "route");
}

}  // namespace dflop
