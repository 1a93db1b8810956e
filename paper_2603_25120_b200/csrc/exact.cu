// exact.cu -- N3: exact C_max by parallel branch and bound (the ILP objective of
// minimise max_j max(E_j, L_j) over item -> bucket assignments).
//
//   k_exact_init    e_i, l_i in the LPT base order, the lower bound
//                   LB = max(ceil(sum e / m), ceil(sum l / m), max_i max(e_i, l_i)) and the
//                   initial incumbent (the caller's assignment, or the paper's LPT)
//   k_exact_expand  one CTA expands the search tree breadth first (first-use symmetry
//                   breaking: an item may open only the lowest unused bucket; a child is
//                   pruned when max(its max load, LB) >= incumbent) until the frontier holds
//                   enough subtrees for the GPU
//   k_exact_dfs     one thread per frontier subtree: depth-first search with an explicit
//                   stack, children in (resulting max load, j) order -- once a child is
//                   pruned all later ones are, so the level is closed; a shared incumbent
//                   key (C_max << 24 | thread) is improved with atomicMin and re-read every
//                   32 nodes; each thread has node_budget / subtrees child visits
//   k_exact_final   the winner's assignment (or the initial one), per-bucket sums and the
//                   1F1B instances of its replicas (scored by k_simulate: the "extra
//                   candidate" of SURVEY 8(f) N3)
//
// The optimum is unique as a value; the assignment returned is one optimal (or best found)
// assignment.  Subtree search: n <= kExactMaxN, m <= 32; beyond that only the bound and the
// initial incumbent are reported (proven iff they meet).
#include <algorithm>
#include <cstring>
#include <vector>

#include "cand.cuh"
#include "internal.h"

namespace dflop {

constexpr uint32_t kExactMaxN = 256;     // depth of the per-thread DFS stack
constexpr uint32_t kExactMaxM = 32;      // tried-children bit mask per level
constexpr uint32_t kExactPrefix = 24;    // deepest breadth-first level stored per node
constexpr uint32_t kExactFront = 16384;  // frontier capacity (subtrees)
constexpr uint32_t kOwnerInit = 0xFFFFFFu;

struct ExactHdr {
    unsigned long long key;   // incumbent (C_max << 24 | owner thread), owner kOwnerInit = initial
    u64 lb;
    u64 sum_e, sum_l, max_key;
    unsigned long long nodes;
    uint32_t out_of_budget;
    uint32_t n_front, depth, complete;  // frontier size / depth; complete = tree fully expanded
    uint32_t bad_init;                  // an init_assign entry >= m
    uint32_t pad;
};

struct ExactNode {
    uint8_t b[kExactPrefix];  // bucket of base-order positions 0..depth-1
    u64 curmax;
    uint32_t used;
    uint32_t pad;
};

DFLOP_DEV u64 umax64(u64 a, u64 b) { return a > b ? a : b; }

// one block: positions' (e, l), sums, LB, initial incumbent (init_assign by item, or LPT)
__global__ void __launch_bounds__(256) k_exact_init(const uint32_t* __restrict__ cost, uint32_t n, uint32_t m,
                                                    const uint32_t* __restrict__ order,
                                                    const uint32_t* __restrict__ init_assign, u64* pe, u64* pl,
                                                    uint32_t* best_by_item, ExactHdr* h) {
    __shared__ unsigned long long sE[256], sL[256];
    __shared__ unsigned long long red[3][256];
    u64 se = 0, sl = 0, mk = 0;
    for (uint32_t t = threadIdx.x; t < n; t += blockDim.x) {
        const uint32_t i = order[t];
        const u64 e = (u64)cost[i] + cost[(size_t)n + i], l = (u64)cost[2 * (size_t)n + i] + cost[3 * (size_t)n + i];
        pe[t] = e;
        pl[t] = l;
        se += e;
        sl += l;
        mk = umax64(mk, umax64(e, l));
    }
    red[0][threadIdx.x] = se;
    red[1][threadIdx.x] = sl;
    red[2][threadIdx.x] = mk;
    for (uint32_t j = threadIdx.x; j < m; j += blockDim.x) sE[j] = sL[j] = 0;
    __syncthreads();
    for (uint32_t s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            red[0][threadIdx.x] += red[0][threadIdx.x + s];
            red[1][threadIdx.x] += red[1][threadIdx.x + s];
            red[2][threadIdx.x] = umax64(red[2][threadIdx.x], red[2][threadIdx.x + s]);
        }
        __syncthreads();
    }
    const u64 SE = red[0][0], SL = red[1][0], MK = red[2][0];
    const u64 lb = umax64(umax64((SE + m - 1) / m, (SL + m - 1) / m), MK);
    if (init_assign) {
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
            uint32_t j = init_assign[i];
            if (j >= m) {
                h->bad_init = 1;
                j = 0;
            }
            best_by_item[i] = j;
            atomicAdd(&sE[j], (unsigned long long)((u64)cost[i] + cost[(size_t)n + i]));
            atomicAdd(&sL[j], (unsigned long long)((u64)cost[2 * (size_t)n + i] + cost[3 * (size_t)n + i]));
        }
    } else if (threadIdx.x < 32) {
        // the paper's LPT: lowest current max(E_j, L_j), lowest j; one warp
        const uint32_t lane = threadIdx.x;
        for (uint32_t t = 0; t < n; ++t) {
            u64 bv = ~0ull;
            uint32_t bj = 0xFFFFFFFFu;
            for (uint32_t j = lane; j < m; j += 32) {
                const u64 v = umax64(sE[j], sL[j]);
                if (v < bv) {
                    bv = v;
                    bj = j;
                }
            }
            for (int off = 16; off > 0; off >>= 1) {
                const u64 v2 = __shfl_xor_sync(0xFFFFFFFFu, bv, off);
                const uint32_t j2 = __shfl_xor_sync(0xFFFFFFFFu, bj, off);
                if (v2 < bv || (v2 == bv && j2 < bj)) {
                    bv = v2;
                    bj = j2;
                }
            }
            if (lane == 0) {
                sE[bj] += pe[t];
                sL[bj] += pl[t];
                best_by_item[order[t]] = bj;
            }
            __syncwarp();
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        u64 c = 0;
        for (uint32_t j = 0; j < m; ++j) c = umax64(c, umax64(sE[j], sL[j]));
        h->key = (c << 24) | kOwnerInit;
        h->lb = lb;
        h->sum_e = SE;
        h->sum_l = SL;
        h->max_key = MK;
        h->nodes = 0;
        h->out_of_budget = 0;
        h->n_front = 0;
        h->depth = 0;
        h->complete = 0;
    }
}

DFLOP_DEV void node_loads(const ExactNode& nd, uint32_t d, const u64* pe, const u64* pl, u64* E, u64* L,
                          uint32_t m) {
    for (uint32_t j = 0; j < m; ++j) E[j] = L[j] = 0;
    for (uint32_t t = 0; t < d; ++t) {
        E[nd.b[t]] += pe[t];
        L[nd.b[t]] += pl[t];
    }
}

// one CTA: breadth-first levels until the next one would not fit (or the prefix depth)
__global__ void __launch_bounds__(1024) k_exact_expand(uint32_t n, uint32_t m, const u64* __restrict__ pe,
                                                       const u64* __restrict__ pl, ExactNode* fa, ExactNode* fb,
                                                       uint32_t target, ExactHdr* h) {
    __shared__ uint32_t s_next, s_count, s_depth, s_done;
    const u64 lb = h->lb, inc = h->key >> 24;
    if (threadIdx.x == 0) {
        fa[0] = ExactNode{};
        s_count = 1;
        s_depth = 0;
        s_done = 0;
    }
    __syncthreads();
    ExactNode* cur = fa;
    ExactNode* nxt = fb;
    unsigned long long visits = 0;
    while (true) {
        const uint32_t d = s_depth, count = s_count;
        if (d >= n || d >= kExactPrefix || count >= target || count == 0) break;
        if (threadIdx.x == 0) s_next = 0;
        __syncthreads();
        const u64 e = pe[d], l = pl[d];
        for (uint32_t q = threadIdx.x; q < count; q += blockDim.x) {
            const ExactNode nd = cur[q];
            u64 E[kExactMaxM], L[kExactMaxM];
            node_loads(nd, d, pe, pl, E, L, m);
            const uint32_t lim = min(nd.used + 1, m);
            for (uint32_t j = 0; j < lim; ++j) {
                ++visits;
                const u64 nm = umax64(nd.curmax, umax64(E[j] + e, L[j] + l));
                if (umax64(nm, lb) >= inc) continue;
                const uint32_t at = atomicAdd(&s_next, 1u);
                if (at < kExactFront) {
                    ExactNode c = nd;
                    c.b[d] = (uint8_t)j;
                    c.curmax = nm;
                    c.used = max(nd.used, j + 1);
                    nxt[at] = c;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (s_next > kExactFront) {
                s_done = 1;  // the next level does not fit: search below the current one
            } else {
                s_count = s_next;
                s_depth = d + 1;
            }
        }
        __syncthreads();
        if (s_done) break;
        ExactNode* t = cur;
        cur = nxt;
        nxt = t;
    }
    atomicAdd(&h->nodes, visits);
    if (threadIdx.x == 0) {
        h->n_front = s_count;
        h->depth = s_depth;
        h->complete = (s_count == 0) ? 1u : 0u;  // every branch pruned: the incumbent is optimal
    }
    // the frontier must end up in fa (the DFS reads it there)
    __syncthreads();
    if (cur != fa)
        for (uint32_t q = threadIdx.x; q < s_count; q += blockDim.x) fa[q] = cur[q];
}

// one thread per frontier subtree: explicit-stack DFS below depth d0; the thread's best
// leaf goes to its own row of best_rows (no write races), the final key names the row
__global__ void __launch_bounds__(128) k_exact_dfs(uint32_t n, uint32_t m, const u64* __restrict__ pe,
                                                   const u64* __restrict__ pl, const ExactNode* __restrict__ front,
                                                   u64 budget_total, uint8_t* best_rows, ExactHdr* h) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nf = h->n_front, d0 = h->depth;
    if (tid >= nf) return;
    const u64 budget = budget_total / nf > 0 ? budget_total / nf : 1;
    const u64 lb = h->lb;
    volatile unsigned long long* vkey = &h->key;
    u64 inc = *vkey >> 24;
    const ExactNode nd = front[tid];
    u64 E[kExactMaxM], L[kExactMaxM];
    node_loads(nd, d0, pe, pl, E, L, m);
    uint32_t tried[kExactMaxN + 1];
    uint8_t choice[kExactMaxN + 1], used[kExactMaxN + 1];
    u64 cm[kExactMaxN + 1];
    uint8_t* best = best_rows + (size_t)tid * kExactMaxN;
    bool have_best = false;
    unsigned long long visits = 0;
    uint32_t t = d0;
    tried[t] = 0;
    used[t] = (uint8_t)nd.used;
    cm[t] = nd.curmax;
    while (true) {
        if (t == n) {  // leaf: its max was below the incumbent when it was entered
            const unsigned long long key = ((unsigned long long)cm[t] << 24) | tid;
            const unsigned long long old = atomicMin((unsigned long long*)&h->key, key);
            if (key < old) {
                for (uint32_t u = 0; u < d0; ++u) best[u] = nd.b[u];
                for (uint32_t u = d0; u < n; ++u) best[u] = choice[u];
                have_best = true;
                inc = cm[t];
            } else {
                inc = old >> 24;
            }
            if (inc <= lb || t == d0) break;  // meets the lower bound, or the subtree is one leaf
            --t;
            const uint32_t j = choice[t];
            E[j] -= pe[t];
            L[j] -= pl[t];
            continue;
        }
        if ((visits & 31u) == 0) inc = min(inc, (u64)(*vkey >> 24));
        // next child: the untried bucket of least (resulting max, j)
        const u64 e = pe[t], l = pl[t];
        const uint32_t lim = min((uint32_t)used[t] + 1, m);
        u64 bv = ~0ull;
        uint32_t bj = 0xFFFFFFFFu;
        for (uint32_t j = 0; j < lim; ++j) {
            if (tried[t] & (1u << j)) continue;
            const u64 v = umax64(E[j] + e, L[j] + l);
            if (v < bv) {
                bv = v;
                bj = j;
            }
        }
        bool descend = false;
        if (bj != 0xFFFFFFFFu) {
            if (visits >= budget) {
                atomicOr(&h->out_of_budget, 1u);
                break;
            }
            ++visits;
            tried[t] |= 1u << bj;
            const u64 nm = umax64(cm[t], bv);
            // children come in ascending order of bv: a pruned child closes the level
            if (umax64(nm, lb) < inc) {
                E[bj] += e;
                L[bj] += l;
                choice[t] = (uint8_t)bj;
                cm[t + 1] = nm;
                used[t + 1] = (uint8_t)max((uint32_t)used[t], bj + 1);
                ++t;
                tried[t] = 0;
                descend = true;
            }
        }
        if (!descend) {  // level exhausted or closed: backtrack
            if (t == d0) break;
            --t;
            const uint32_t j = choice[t];
            E[j] -= pe[t];
            L[j] -= pl[t];
        }
    }
    atomicAdd(&h->nodes, visits);
    (void)have_best;
}

// winner's assignment by item, per-bucket sums and the 1F1B inputs of every replica
__global__ void k_exact_final(uint32_t n, uint32_t m, const uint32_t* __restrict__ cost,
                              const uint32_t* __restrict__ order, const uint8_t* __restrict__ best_rows,
                              uint32_t* best_by_item, const ExactHdr* h, uint32_t e_pp, uint32_t l_pp,
                              uint32_t l_dp, uint32_t n_mb, u64* sums, u64* fwd, u64* bwd, uint32_t* assign) {
    const uint32_t owner = (uint32_t)(h->key & 0xFFFFFFull);
    if (owner != kOwnerInit)
        for (uint32_t t = threadIdx.x; t < n; t += blockDim.x)
            best_by_item[order[t]] = best_rows[(size_t)owner * kExactMaxN + t];
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < 4 * m; j += blockDim.x) sums[j] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        const uint32_t j = best_by_item[i];
        if (assign) assign[i] = j;
        for (int r = 0; r < 4; ++r)
            atomicAdd((unsigned long long*)&sums[4 * j + r], (unsigned long long)cost[(size_t)r * n + i]);
    }
    __syncthreads();
    // replica rho: slot k = bucket k * L_dp + rho (R10); encoder stages take (EF, EB) (R7)
    const uint32_t S = e_pp + l_pp;
    for (uint32_t x = threadIdx.x; x < l_dp * S * n_mb; x += blockDim.x) {
        const uint32_t rho = x / (S * n_mb), s = (x / n_mb) % S, k = x % n_mb;
        const uint32_t j = k * l_dp + rho;
        const bool enc = s < e_pp;
        fwd[x] = sums[4 * j + (enc ? 0 : 2)];
        bwd[x] = sums[4 * j + (enc ? 1 : 3)];
    }
}

size_t exact_ws_bytes(uint32_t n, uint32_t m, const dflop_plan* p) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t inst = (size_t)p->l_dp * (p->e_pp + p->l_pp) * p->n_mb;
    return al(sizeof(ExactHdr)) + al((size_t)n * 8) + al((size_t)n * 4) * 2 + al((size_t)n * 8) * 2 + al((size_t)kExactFront * kExactMaxN) +
           2 * al((size_t)kExactFront * sizeof(ExactNode)) + al((size_t)4 * m * 8) + 2 * al(inst * 8) +
           al((size_t)p->l_dp * 8) + al(sizeof(BalanceHeader));
}

dflop_status exact_launch(const uint32_t* cost, uint32_t n, const dflop_plan* p, uint64_t node_budget,
                          const uint32_t* init_assign, void* ws, dflop_exact_result* out, uint32_t* assign,
                          cudaStream_t s) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const uint32_t m = p->n_mb * p->l_dp, S = p->e_pp + p->l_pp;
    const size_t inst = (size_t)p->l_dp * S * p->n_mb;
    char* w = reinterpret_cast<char*>(ws);
    size_t o = 0;
    ExactHdr* h = reinterpret_cast<ExactHdr*>(w + o);        o += al(sizeof(ExactHdr));
    u64* keys = reinterpret_cast<u64*>(w + o);               o += al((size_t)n * 8);
    uint32_t* order = reinterpret_cast<uint32_t*>(w + o);    o += al((size_t)n * 4);
    uint32_t* by_item = reinterpret_cast<uint32_t*>(w + o);  o += al((size_t)n * 4);
    u64* pe = reinterpret_cast<u64*>(w + o);                 o += al((size_t)n * 8);
    u64* pl = reinterpret_cast<u64*>(w + o);                 o += al((size_t)n * 8);
    uint8_t* best_rows = reinterpret_cast<uint8_t*>(w + o);  o += al((size_t)kExactFront * kExactMaxN);
    ExactNode* fa = reinterpret_cast<ExactNode*>(w + o);     o += al((size_t)kExactFront * sizeof(ExactNode));
    ExactNode* fb = reinterpret_cast<ExactNode*>(w + o);     o += al((size_t)kExactFront * sizeof(ExactNode));
    u64* sums = reinterpret_cast<u64*>(w + o);               o += al((size_t)4 * m * 8);
    u64* fwd = reinterpret_cast<u64*>(w + o);                o += al(inst * 8);
    u64* bwd = reinterpret_cast<u64*>(w + o);                o += al(inst * 8);
    u64* ms = reinterpret_cast<u64*>(w + o);                 o += al((size_t)p->l_dp * 8);
    BalanceHeader* bh = reinterpret_cast<BalanceHeader*>(w + o);
    uint32_t* item_pos = by_item;  // scratch for the rank sort (overwritten by k_exact_init)
    cudaError_t ce = cudaMemsetAsync(bh, 0, sizeof(BalanceHeader), s);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(h, 0, sizeof(ExactHdr), s);
    if (ce != cudaSuccess) return cuda_status(ce, "memset");
    if (n > 0) {
        const uint32_t gb = std::min<uint32_t>((n + 255) / 256, 592);
        k_prep_keys<<<gb, 256, 0, s>>>(cost, n, n, bh, keys);
        order_launch_keys(keys, n, order, item_pos, s);
        count_launches(2);
    }
    k_exact_init<<<1, 256, 0, s>>>(cost, n, m, order, init_assign, pe, pl, by_item, h);
    count_launches(1);
    const bool dfs = n > 0 && n <= kExactMaxN && m <= kExactMaxM;
    if (dfs) {
        int dev = 0;
        cudaGetDevice(&dev);
        const uint32_t target = (uint32_t)std::min<int>(kExactFront / 2, dev_attr(dev).sms * 64);
        k_exact_expand<<<1, 1024, 0, s>>>(n, m, pe, pl, fa, fb, target, h);
        k_exact_dfs<<<kExactFront / 128, 128, 0, s>>>(n, m, pe, pl, fa, node_budget, best_rows, h);
        count_launches(2);
    }
    k_exact_final<<<1, 256, 0, s>>>(n, m, cost, order, best_rows, by_item, h, p->e_pp, p->l_pp, p->l_dp, p->n_mb,
                                    sums, fwd, bwd, assign);
    count_launches(1);
    SlotProgram prog;
    dflop_status st = get_slot_program(S, p->n_mb, &prog);
    if (st != DFLOP_OK) return st;
    if ((st = simulate_launch(reinterpret_cast<const uint64_t*>(fwd), reinterpret_cast<const uint64_t*>(bwd), p->l_dp, S,
                              p->n_mb, reinterpret_cast<uint64_t*>(ms), nullptr, prog, s)) != DFLOP_OK)
        return st;
    ExactHdr hh;
    std::vector<u64> hm(p->l_dp);
    ce = cudaMemcpyAsync(&hh, h, sizeof hh, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(hm.data(), ms, p->l_dp * 8, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return cuda_status(ce, "exact readback");
    if (hh.bad_init) {
        set_error("init_assign holds a bucket >= m = %u", m);
        return DFLOP_ERR_INVALID_ARGUMENT;
    }
    dflop_exact_result r;
    memset(&r, 0, sizeof r);
    r.struct_size = sizeof r;
    r.cmax = hh.key >> 24;
    r.lower_bound = hh.lb;
    r.nodes = hh.nodes;
    r.proven = (r.cmax <= hh.lb || (dfs && !hh.out_of_budget)) ? 1u : 0u;
    r.searched = dfs ? 1u : 0u;
    for (u64 v : hm) r.makespan = std::max<u64>(r.makespan, v);
    *out = r;
    return DFLOP_OK;
}

}  // namespace dflop
