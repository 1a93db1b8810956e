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
// m = 2 and m = 4 with n <= kPDMaxN use an exhaustive pair decomposition instead of the tree
// (k_pd_*: the same certificate as oracle/orc_exact_pairs, DESIGN.md section 10b N3):
//   m = 2  every subset Y holding base position 0 (Gray-code enumeration over the GPU):
//          C = max(E(Y), L(Y), E - E(Y), L - L(Y)), minimum over Y;
//   m = 4  buckets {0, 1} form X (position 0 in X), {2, 3} its complement; X's with E(X),
//          L(X) in [S - 2C0, 2C0] (C0 = incumbent - 1: no better assignment has X outside)
//          are listed, then one warp per X computes the best 2-way splits of X and of its
//          complement (Gray enumeration over the lanes); C = min over X of the larger one.
//          A list overflow splits the first kPDCap X's, tightens C0 and re-enumerates.
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

// ---------------------------------------------------------------- pair decomposition (m = 2, 4)
constexpr uint32_t kPDMaxN = 34;          // 2^33 subsets X at most
constexpr uint32_t kPDCap = 1u << 20;     // listed X's per enumeration pass
constexpr uint32_t kPDBlocks = 148 * 8, kPDThreads = 256;

struct PDHdr {
    unsigned long long best;   // (C << 24) | list index (m = 4) -- min over split X's
    unsigned long long count;  // X's in the window this pass
    u64 sum_e, sum_l;
    u64 visited;
};

// sums of the subset `mask` of base positions
DFLOP_DEV void pd_sums(const u64* pe, const u64* pl, uint32_t n, u64 mask, u64& E, u64& L) {
    E = 0;
    L = 0;
    for (uint32_t t = 0; t < n; ++t)
        if ((mask >> t) & 1ull) {
            E += pe[t];
            L += pl[t];
        }
}

// every subset holding position 0, in Gray-code order: index i -> {0} u gray(i) shifted by 1;
// m = 2: per-block minimum of (C(Y), Y) into blk[]; m = 4: X's in the window into list[]
__global__ void __launch_bounds__(kPDThreads) k_pd_enum(uint32_t n, uint32_t m, const u64* __restrict__ pe,
                                                         const u64* __restrict__ pl, u64 C0, u64* list,
                                                         PDHdr* ph, u64* blk) {
    __shared__ u64 sv[kPDThreads], sm[kPDThreads];
    const u64 SE = ph->sum_e, SL = ph->sum_l;
    const u64 loE = SE > 2 * C0 ? SE - 2 * C0 : 0, loL = SL > 2 * C0 ? SL - 2 * C0 : 0, hi = 2 * C0;
    const u64 steps = 1ull << (n - 1);
    const u64 nthr = (u64)gridDim.x * blockDim.x, tid = (u64)blockIdx.x * blockDim.x + threadIdx.x;
    const u64 chunk = (steps + nthr - 1) / nthr;
    const u64 i0 = tid * chunk, i1 = min(steps, i0 + chunk);
    u64 bv = ~0ull, bm = 0;
    if (i0 < i1) {
        u64 x = 1ull | ((i0 ^ (i0 >> 1)) << 1);
        u64 E, L;
        pd_sums(pe, pl, n, x, E, L);
        for (u64 i = i0; i < i1; ++i) {
            if (i > i0) {
                const uint32_t b = 1 + (uint32_t)__ffsll((long long)i) - 1;
                x ^= 1ull << b;
                if ((x >> b) & 1ull) {
                    E += pe[b];
                    L += pl[b];
                } else {
                    E -= pe[b];
                    L -= pl[b];
                }
            }
            if (m == 2) {
                const u64 v = umax64(umax64(E, L), umax64(SE - E, SL - L));
                if (v < bv) {
                    bv = v;
                    bm = x;
                }
            } else if (E >= loE && E <= hi && L >= loL && L <= hi) {
                const unsigned long long k = atomicAdd(&ph->count, 1ull);
                if (k < kPDCap) list[k] = x;
            }
        }
    }
    if (m == 2) {  // block minimum (value, mask)
        sv[threadIdx.x] = bv;
        sm[threadIdx.x] = bm;
        __syncthreads();
        for (uint32_t s = blockDim.x / 2; s > 0; s >>= 1) {
            if (threadIdx.x < s && (sv[threadIdx.x + s] < sv[threadIdx.x] ||
                                    (sv[threadIdx.x + s] == sv[threadIdx.x] && sm[threadIdx.x + s] < sm[threadIdx.x]))) {
                sv[threadIdx.x] = sv[threadIdx.x + s];
                sm[threadIdx.x] = sm[threadIdx.x + s];
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            blk[2 * blockIdx.x] = sv[0];
            blk[2 * blockIdx.x + 1] = sm[0];
        }
    }
}

// best 2-way split of the k items (e[], l[]) by the 32 lanes of a warp: subsets holding item 0,
// lane chunks of the Gray sequence; returns (value, mask) of the lexicographic minimum
DFLOP_DEV void pd_split_warp(const u64* e, const u64* l, uint32_t k, u64& best_v, u64& best_y) {
    const uint32_t lane = threadIdx.x & 31u;
    u64 SE = 0, SL = 0;
    for (uint32_t t = 0; t < k; ++t) {
        SE += e[t];
        SL += l[t];
    }
    const u64 steps = k ? 1ull << (k - 1) : 0ull;
    const u64 chunk = (steps + 31) / 32;
    const u64 i0 = (u64)lane * chunk, i1 = min(steps, i0 + chunk);
    u64 bv = ~0ull, by = 0;
    if (i0 < i1) {
        u64 y = 1ull | ((i0 ^ (i0 >> 1)) << 1);
        u64 E = 0, L = 0;
        for (uint32_t t = 0; t < k; ++t)
            if ((y >> t) & 1ull) {
                E += e[t];
                L += l[t];
            }
        for (u64 i = i0; i < i1; ++i) {
            if (i > i0) {
                const uint32_t b = (uint32_t)__ffsll((long long)i);  // 1 + ctz(i)
                y ^= 1ull << b;
                if ((y >> b) & 1ull) {
                    E += e[b];
                    L += l[b];
                } else {
                    E -= e[b];
                    L -= l[b];
                }
            }
            const u64 v = umax64(umax64(E, L), umax64(SE - E, SL - L));
            if (v < bv) {
                bv = v;
                by = y;
            }
        }
    }
    for (int off = 16; off > 0; off >>= 1) {
        const u64 v2 = __shfl_xor_sync(0xFFFFFFFFu, bv, off), y2 = __shfl_xor_sync(0xFFFFFFFFu, by, off);
        if (v2 < bv || (v2 == bv && y2 < by)) {
            bv = v2;
            by = y2;
        }
    }
    if (k == 0) bv = 0;
    best_v = bv;
    best_y = by;
}

// one warp per listed X: C(X) = max(split2(X), split2(complement)); atomicMin of (C << 24 | idx)
__global__ void __launch_bounds__(128) k_pd_split(uint32_t n, const u64* __restrict__ pe, const u64* __restrict__ pl,
                                                  const u64* __restrict__ list, uint32_t count, u64 inc, PDHdr* ph) {
    __shared__ u64 se[4][2][kPDMaxN], sl[4][2][kPDMaxN];
    const uint32_t w = threadIdx.x >> 5, lane = threadIdx.x & 31u;
    const uint32_t warps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t x = blockIdx.x * (blockDim.x >> 5) + w; x < count; x += warps) {
        const u64 mask = list[x];
        if (lane == 0) {
            uint32_t a = 0, b = 0;
            for (uint32_t t = 0; t < n; ++t) {
                if ((mask >> t) & 1ull) {
                    se[w][0][a] = pe[t];
                    sl[w][0][a++] = pl[t];
                } else {
                    se[w][1][b] = pe[t];
                    sl[w][1][b++] = pl[t];
                }
            }
        }
        __syncwarp();
        const uint32_t kx = (uint32_t)__popcll(mask), kc = n - kx;
        u64 v1, y1;
        pd_split_warp(se[w][0], sl[w][0], kx, v1, y1);
        const u64 cur = umax64(0, min(ph->best >> 24, inc));  // to beat: the best so far and the incumbent
        if (v1 < cur) {  // warp-uniform (v1 reduced)
            u64 v2, y2;
            pd_split_warp(se[w][1], sl[w][1], kc, v2, y2);
            const u64 v = umax64(v1, v2);
            if (lane == 0 && v < cur) atomicMin(&ph->best, (v << 24) | x);
        }
        __syncwarp();
    }
}

// the winner: m = 2 from the block minima, m = 4 from the best listed X (its splits recomputed);
// writes best_by_item and the incumbent key when it beats the initial assignment
__global__ void k_pd_final(uint32_t n, uint32_t m, const u64* __restrict__ pe, const u64* __restrict__ pl,
                           const uint32_t* __restrict__ order, const u64* __restrict__ list, const u64* __restrict__ blk,
                           uint32_t nblk, PDHdr* ph, uint32_t* best_by_item, ExactHdr* h) {
    __shared__ u64 se[2][kPDMaxN], sl[2][kPDMaxN];
    __shared__ u64 s_v, s_x, s_y1, s_y2;
    const uint32_t lane = threadIdx.x & 31u;
    if (threadIdx.x >= 32) return;
    if (m == 2) {
        u64 bv = ~0ull, bm = 0;
        for (uint32_t b = lane; b < nblk; b += 32)
            if (blk[2 * b] < bv || (blk[2 * b] == bv && blk[2 * b + 1] < bm)) {
                bv = blk[2 * b];
                bm = blk[2 * b + 1];
            }
        for (int off = 16; off > 0; off >>= 1) {
            const u64 v2 = __shfl_xor_sync(0xFFFFFFFFu, bv, off), m2 = __shfl_xor_sync(0xFFFFFFFFu, bm, off);
            if (v2 < bv || (v2 == bv && m2 < bm)) {
                bv = v2;
                bm = m2;
            }
        }
        if ((bv << 24) >> 24 == bv && bv < (h->key >> 24)) {
            for (uint32_t t = lane; t < n; t += 32) best_by_item[order[t]] = ((bm >> t) & 1ull) ? 0u : 1u;
            if (lane == 0) h->key = (bv << 24) | kOwnerInit;
        }
        return;
    }
    const unsigned long long key = ph->best;
    if ((key >> 24) >= (h->key >> 24)) return;  // nothing beat the incumbent
    const u64 mask = list[key & 0xFFFFFFull];
    if (lane == 0) {
        uint32_t a = 0, b = 0;
        for (uint32_t t = 0; t < n; ++t) {
            if ((mask >> t) & 1ull) {
                se[0][a] = pe[t];
                sl[0][a++] = pl[t];
            } else {
                se[1][b] = pe[t];
                sl[1][b++] = pl[t];
            }
        }
    }
    __syncwarp();
    const uint32_t kx = (uint32_t)__popcll(mask), kc = n - kx;
    u64 v1, y1, v2, y2;
    pd_split_warp(se[0], sl[0], kx, v1, y1);
    pd_split_warp(se[1], sl[1], kc, v2, y2);
    if (lane == 0) {
        s_v = umax64(v1, v2);
        s_x = mask;
        s_y1 = y1;
        s_y2 = y2;
    }
    __syncwarp();
    // positions of X in increasing order are X's items 0..kx-1 (same for the complement)
    if (lane == 0) {
        uint32_t a = 0, b = 0;
        for (uint32_t t = 0; t < n; ++t) {
            if ((s_x >> t) & 1ull)
                best_by_item[order[t]] = ((s_y1 >> a++) & 1ull) ? 0u : 1u;
            else
                best_by_item[order[t]] = ((s_y2 >> b++) & 1ull) ? 2u : 3u;
        }
        h->key = (s_v << 24) | kOwnerInit;
    }
}

size_t exact_ws_bytes(uint32_t n, uint32_t m, const dflop_plan* p) {
    auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
    const size_t inst = (size_t)p->l_dp * (p->e_pp + p->l_pp) * p->n_mb;
    const bool pd = (m == 2 || m == 4) && n >= 1 && n <= kPDMaxN;
    return al(sizeof(ExactHdr)) + al((size_t)n * 8) + al((size_t)n * 4) * 2 + al((size_t)n * 8) * 2 + al((size_t)kExactFront * kExactMaxN) +
           2 * al((size_t)kExactFront * sizeof(ExactNode)) + al((size_t)4 * m * 8) + 2 * al(inst * 8) +
           al((size_t)p->l_dp * 8) + al(sizeof(BalanceHeader)) +
           (pd ? al(sizeof(PDHdr)) + al((size_t)kPDCap * 8) + al((size_t)kPDBlocks * 16) : 0);
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
    BalanceHeader* bh = reinterpret_cast<BalanceHeader*>(w + o); o += al(sizeof(BalanceHeader));
    uint32_t* item_pos = by_item;  // scratch for the rank sort (overwritten by k_exact_init)
    bool h_pd_incomplete = false;
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
    // m = 2, 4 and small n: the exhaustive pair decomposition (a certificate) when its 2^(n-1)
    // subsets fit the node budget; otherwise the tree search
    const bool pd = (m == 2 || m == 4) && n >= 1 && n <= kPDMaxN && (1ull << (n - 1)) <= node_budget;
    const bool dfs = !pd && n > 0 && n <= kExactMaxN && m <= kExactMaxM;
    u64 pd_visited = 0;
    if (pd) {
        PDHdr* ph = reinterpret_cast<PDHdr*>(w + o);       o += al(sizeof(PDHdr));
        u64* list = reinterpret_cast<u64*>(w + o);          o += al((size_t)kPDCap * 8);
        u64* blk = reinterpret_cast<u64*>(w + o);           o += al((size_t)kPDBlocks * 16);
        ExactHdr hh;
        ce = cudaMemcpyAsync(&hh, h, sizeof hh, cudaMemcpyDeviceToHost, s);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
        if (ce != cudaSuccess) return cuda_status(ce, "exact init readback");
        PDHdr p0;
        memset(&p0, 0, sizeof p0);
        p0.sum_e = hh.sum_e;
        p0.sum_l = hh.sum_l;
        u64 inc = hh.key >> 24;
        p0.best = ~0ull;
        for (int pass = 0; inc > hh.lb && pass < 64; ++pass) {
            p0.count = 0;
            ce = cudaMemcpyAsync(ph, &p0, sizeof p0, cudaMemcpyHostToDevice, s);
            if (ce != cudaSuccess) return cuda_status(ce, "pd header");
            k_pd_enum<<<kPDBlocks, kPDThreads, 0, s>>>(n, m, pe, pl, inc - 1, list, ph, blk);
            count_launches(1);
            pd_visited += 1ull << (n - 1);
            if (m == 2) break;
            unsigned long long cnt = 0;
            ce = cudaMemcpyAsync(&cnt, &ph->count, 8, cudaMemcpyDeviceToHost, s);
            if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
            if (ce != cudaSuccess) return cuda_status(ce, "pd count");
            const uint32_t nx = (uint32_t)std::min<unsigned long long>(cnt, kPDCap);
            if (nx > 0) {
                k_pd_split<<<std::min<uint32_t>((nx + 3) / 4, 148 * 16), 128, 0, s>>>(n, pe, pl, list, nx, inc, ph);
                k_pd_final<<<1, 32, 0, s>>>(n, m, pe, pl, order, list, blk, kPDBlocks, ph, by_item, h);
                count_launches(2);
            }
            if (cnt <= kPDCap) break;
            // overflow: the split X's tightened the incumbent; enumerate again with it
            ce = cudaMemcpyAsync(&hh, h, sizeof hh, cudaMemcpyDeviceToHost, s);
            if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
            if (ce != cudaSuccess) return cuda_status(ce, "pd readback");
            const u64 inc2 = hh.key >> 24;
            if (inc2 >= inc) {  // no progress with the first kPDCap X's: give up (not proven)
                h_pd_incomplete = true;
                break;
            }
            inc = inc2;
            p0.best = ~0ull;
        }
        if (m == 2 && inc > hh.lb) {
            k_pd_final<<<1, 32, 0, s>>>(n, m, pe, pl, order, list, blk, kPDBlocks, ph, by_item, h);
            count_launches(1);
        }
    }
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
    r.nodes = pd ? pd_visited : hh.nodes;
    r.proven = (r.cmax <= hh.lb || (dfs && !hh.out_of_budget) || (pd && !h_pd_incomplete)) ? 1u : 0u;
    r.searched = (dfs || pd) ? 1u : 0u;
    for (u64 v : hm) r.makespan = std::max<u64>(r.makespan, v);
    *out = r;
    return DFLOP_OK;
}

}  // namespace dflop
