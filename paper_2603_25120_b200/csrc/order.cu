// order.cu -- N4(a): microbatch-order search (R11, R35): the non-interleaved 1F1B makespan
// of a replica depends on the order of its microbatch slots; for one assignment (e.g. the
// search's winner) every LLM replica's slot order is improved independently.
//
//   k_order_sums    per-bucket sums EF, EB, LF, LB of the assignment (atomics)
//   k_order_search  one cooperative grid over all SMs, replica by replica: four start
//                   orders (identity, W ascending, W descending, valley) scored by four
//                   threads; then rounds of best-improvement pairwise swaps -- each thread
//                   simulates 1F1B (the host-built slot program, per-thread stage rings in
//                   shared memory) for its share of the swap pairs, CTA reductions and one
//                   atomicMin give the lexicographic minimum of (makespan, a, b), applied
//                   while strictly better, grid barriers between rounds
//
// Same start orders, neighbourhood and tie rules as orc_order_search (bit-exact).
#include <cooperative_groups.h>

#include <algorithm>
#include <vector>

#include "cand.cuh"
#include "internal.h"

namespace dflop {

namespace cg = cooperative_groups;

__global__ void k_order_sums(const uint32_t* __restrict__ cost, uint32_t n, const uint32_t* __restrict__ assign,
                             uint32_t m, u64* sums, uint32_t* bad) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t j = assign[i];
        if (j >= m) {
            atomicOr(bad, 1u);
            continue;
        }
        for (int r = 0; r < 4; ++r)
            atomicAdd((unsigned long long*)&sums[4 * (size_t)j + r], (unsigned long long)cost[(size_t)r * n + i]);
    }
}

struct OrderShape {
    uint32_t S, M, e_pp, l_dp, n_ops, D, rounds, threads;
};

// slot -> position in the slot array under the swap (a, b) (a == b: no swap)
DFLOP_DEV uint32_t swapped(uint32_t k, uint32_t a, uint32_t b) { return k == a ? b : (k == b ? a : k); }

// 1F1B makespan of the replica with slot k running bucket-slot ord[map(k)]
template <typename Map>
DFLOP_DEV u64 sim_order(const OrderShape& sh, const uint32_t* __restrict__ ops, const u64* sums, Map&& slot_of,
                        u64* st) {
    const uint32_t S = sh.S, D = sh.D, Dm = D - 1;
    u64* last = st;
    u64* FR = st + S;
    u64* BR = FR + S * D;
    for (uint32_t s = 0; s < S; ++s) last[s] = 0;
    for (uint32_t q = 0; q < sh.n_ops; ++q) {
        const uint32_t op = __ldg(ops + q);
        const uint32_t kind = op_kind(op), s = op_stage(op), k = op_mb(op);
        const u64* b = sums + 4 * (size_t)slot_of(k);
        const bool enc = s < sh.e_pp;
        u64 dur, dep = 0;
        if (kind == 0) {
            dur = enc ? b[0] : b[2];
            if (s > 0) dep = FR[(s - 1) * D + (k & Dm)];
        } else {
            dur = enc ? b[1] : b[3];
            dep = (s + 1 < S) ? BR[(s + 1) * D + (k & Dm)] : FR[s * D + (k & Dm)];
        }
        const u64 l0 = last[s];
        const u64 end = (l0 > dep ? l0 : dep) + dur;
        last[s] = end;
        if (kind == 0)
            FR[s * D + (k & Dm)] = end;
        else
            BR[s * D + (k & Dm)] = end;
    }
    u64 T = 0;
    for (uint32_t s = 0; s < S; ++s) T = last[s] > T ? last[s] : T;
    return T;
}

// Cooperative grid (one launch for all replicas and rounds): every CTA keeps the replica's
// slot sums and the current order in shared memory; the swap pairs of a round are spread
// over all threads of the grid, each CTA reduces its best (makespan, a, b) and one
// atomicMin on the packed key (makespan << 24 | a << 12 | b; makespan < 2^40, N_mb <= 4096
// for the grid path) picks the round's move; grid-wide barriers separate the rounds.
__global__ void k_order_search(OrderShape sh, const uint32_t* __restrict__ ops, const u64* __restrict__ sums_all,
                               uint32_t* order_out, u64* T_out, unsigned long long* keys, uint32_t* gorder) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t M = sh.M, tid = threadIdx.x, nt = blockDim.x;
    const uint32_t gtid = blockIdx.x * nt + tid, gsize = gridDim.x * nt;
    u64* sums = reinterpret_cast<u64*>(smem);                      // [M][4] of the replica (slot k)
    u64* st = sums + 4 * (size_t)M + (size_t)tid * (sh.S + 2 * sh.S * sh.D);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(sums + 4 * (size_t)M +
                                                                    (size_t)nt * (sh.S + 2 * sh.S * sh.D));
    uint32_t* ord = reinterpret_cast<uint32_t*>(red + nt);          // [M] slot -> slot index
    uint32_t* asc = ord + M;                                        // [M] slots by W ascending
    uint32_t* desc = asc + M;                                       // [M] W descending, ties by slot
    const uint32_t half = (M + 1) / 2;
    const bool all_pairs = M <= 128;
    const uint32_t n_pairs = all_pairs ? M * (M - 1) / 2 : (M - 1) * 16;
    for (uint32_t rho = 0; rho < sh.l_dp; ++rho) {
        for (uint32_t k = tid; k < M; k += nt)
            for (int r = 0; r < 4; ++r) sums[4 * k + r] = sums_all[4 * ((size_t)k * sh.l_dp + rho) + r];
        __syncthreads();
        if (tid == 0) {  // stable insertion sorts (every CTA computes the same)
            for (uint32_t k = 0; k < M; ++k) asc[k] = k;
            auto W = [&](uint32_t k) {
                const u64 E = sums[4 * k] + sums[4 * k + 1], L = sums[4 * k + 2] + sums[4 * k + 3];
                return E > L ? E : L;
            };
            for (uint32_t x = 1; x < M; ++x) {
                const uint32_t v = asc[x];
                uint32_t y = x;
                while (y > 0 && W(asc[y - 1]) > W(v)) {
                    asc[y] = asc[y - 1];
                    --y;
                }
                asc[y] = v;
            }
            uint32_t k = 0;
            for (uint32_t e = M; e > 0;) {  // runs of equal W reversed as blocks
                uint32_t s0 = e - 1;
                while (s0 > 0 && W(asc[s0 - 1]) == W(asc[e - 1])) --s0;
                for (uint32_t t = s0; t < e; ++t) desc[k++] = asc[t];
                e = s0;
            }
        }
        if (gtid == 0) keys[0] = keys[1] = keys[2] = keys[3] = ~0ull;
        __syncthreads();
        grid.sync();
        // start orders 0..3 on the first four threads of the grid: key (T << 24 | o)
        if (gtid < 4) {
            const uint32_t o = gtid;
            auto map = [&](uint32_t k) -> uint32_t {
                if (o == 0) return k;
                if (o == 1) return asc[k];
                if (o == 2) return desc[k];
                return asc[k < half ? 2 * k : 2 * (M - 1 - k) + 1];
            };
            const u64 T = sim_order(sh, ops, sums, map, st);
            atomicMin(&keys[0], (unsigned long long)((T << 24) | o));
        }
        grid.sync();
        const unsigned long long k0 = keys[0];
        const uint32_t bo = (uint32_t)(k0 & 0xFFFFFFull);
        u64 curT = k0 >> 24;
        for (uint32_t k = tid; k < M; k += nt)
            ord[k] = bo == 0 ? k : bo == 1 ? asc[k] : bo == 2 ? desc[k] : asc[k < half ? 2 * k : 2 * (M - 1 - k) + 1];
        __syncthreads();
        for (uint32_t r = 0; r < sh.rounds; ++r) {
            // three rotating key slots: round r reduces into slot r % 3 and clears the slot of
            // round r + 1, which nobody reads any more (its last readers passed round r - 1's barrier)
            const uint32_t slot = 1 + r % 3, next = 1 + (r + 1) % 3;
            unsigned long long best = ~0ull;
            for (uint32_t pidx = gtid; pidx < n_pairs; pidx += gsize) {
                uint32_t a, b;
                if (all_pairs) {  // row-major (a, b), a < b
                    a = 0;
                    uint32_t rem = pidx;
                    while (rem >= M - 1 - a) {
                        rem -= M - 1 - a;
                        ++a;
                    }
                    b = a + 1 + rem;
                } else {
                    a = pidx / 16;
                    b = a + 1 + pidx % 16;
                    if (b >= M) continue;
                }
                const u64 T = sim_order(sh, ops, sums, [&](uint32_t k) { return ord[swapped(k, a, b)]; }, st);
                const unsigned long long key = (T << 24) | ((unsigned long long)a << 12) | b;
                best = key < best ? key : best;
            }
            red[tid] = best;
            __syncthreads();
            for (uint32_t s = nt / 2; s > 0; s >>= 1) {
                if (tid < s && red[tid + s] < red[tid]) red[tid] = red[tid + s];
                __syncthreads();
            }
            if (tid == 0 && red[0] != ~0ull) atomicMin(&keys[slot], red[0]);
            if (gtid == 0) keys[next] = ~0ull;
            grid.sync();
            const unsigned long long rk = keys[slot];
            if (rk == ~0ull || (rk >> 24) >= curT) break;  // grid-uniform
            const uint32_t a = (uint32_t)(rk >> 12) & 0xFFFu, b = (uint32_t)rk & 0xFFFu;
            if (tid == 0) {
                const uint32_t t = ord[a];
                ord[a] = ord[b];
                ord[b] = t;
            }
            curT = rk >> 24;
            __syncthreads();
        }
        if (blockIdx.x == 0) {
            for (uint32_t k = tid; k < M; k += nt) order_out[(size_t)rho * M + k] = ord[k] * sh.l_dp + rho;
            if (tid == 0) T_out[rho] = curT;
        }
        grid.sync();  // the replica's keys and shared arrays are reused
    }
    (void)gorder;
}

size_t order_ws_bytes(const dflop_plan* p) {
    const size_t m = (size_t)p->n_mb * p->l_dp;
    return ((m * 4 * 8 + 255) & ~(size_t)255) + ((p->l_dp * 8 + 255) & ~(size_t)255) + 256 + 256;  // bad, keys[4]
}

dflop_status order_launch(const uint32_t* cost, uint32_t n, const dflop_plan* p, const uint32_t* assign,
                          uint32_t rounds, void* ws, uint32_t* order_out, uint64_t* T_host, cudaStream_t s) {
    const uint32_t m = p->n_mb * p->l_dp, S = p->e_pp + p->l_pp, M = p->n_mb;
    if (M > 4096) {
        set_error("order search: N_mb = %u > 4096", M);
        return DFLOP_ERR_UNSUPPORTED;
    }
    char* w = reinterpret_cast<char*>(ws);
    u64* sums = reinterpret_cast<u64*>(w);
    u64* T = reinterpret_cast<u64*>(w + (((size_t)m * 32 + 255) & ~(size_t)255));
    char* tail = reinterpret_cast<char*>(T) + (((size_t)p->l_dp * 8 + 255) & ~(size_t)255);
    uint32_t* bad = reinterpret_cast<uint32_t*>(tail);
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(tail + 256);
    cudaError_t ce = cudaMemsetAsync(sums, 0, (size_t)m * 32, s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(bad, 0, 4, s);
    if (ce != cudaSuccess) return cuda_status(ce, "memset");
    if (n > 0) {
        k_order_sums<<<std::min<uint32_t>((n + 255) / 256, 296), 256, 0, s>>>(cost, n, assign, m, sums, bad);
        count_launches(1);
    }
    SlotProgram prog;
    dflop_status st = get_slot_program(S, M, &prog);
    if (st != DFLOP_OK) return st;
    OrderShape sh{S, M, p->e_pp, p->l_dp, prog.n_ops, prog.D, rounds, 0};
    int dev = 0;
    cudaGetDevice(&dev);
    const DevAttr prop = dev_attr(dev);
    const size_t smax = prop.smem_optin;
    const size_t per_thread = (size_t)(S + 2 * S * prog.D) * 8 + 8;
    const size_t fixed = (size_t)M * 32 + (size_t)M * 12 + 64;
    uint32_t nt = 256;
    while (nt > 32 && fixed + nt * per_thread > smax) nt /= 2;
    if (fixed + nt * per_thread > smax) {
        set_error("order search: N_mb = %u, S = %u need more shared memory than %zu B", M, S, smax);
        return DFLOP_ERR_UNSUPPORTED;
    }
    sh.threads = nt;
    const size_t dyn = fixed + nt * per_thread;
    const void* fn = reinterpret_cast<const void*>(&k_order_search);
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, (int)nt, dyn);
    const uint32_t n_pairs = M <= 128 ? M * (M - 1) / 2 : (M - 1) * 16;
    uint32_t grid = std::max(1u, std::min<uint32_t>((uint32_t)std::max(1, per_sm) * prop.sms, (n_pairs + nt - 1) / nt));
    uint32_t* gorder = nullptr;
    const uint32_t* d_ops = prog.d_ops;
    void* args[] = {&sh, &d_ops, &sums, &order_out, &T, &keys, &gorder};
    ce = cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(nt), args, dyn, s);
    if (ce != cudaSuccess) return cuda_status(ce, "order search launch");
    count_launches(1);
    uint32_t hbad = 0;
    ce = cudaMemcpyAsync(T_host, T, (size_t)p->l_dp * 8, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(&hbad, bad, 4, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return cuda_status(ce, "order search");
    if (hbad) {
        set_error("assign holds a bucket >= m = %u", m);
        return DFLOP_ERR_INVALID_ARGUMENT;
    }
    return DFLOP_OK;
}

}  // namespace dflop
