// protocol.cpp -- the multi-GPU candidate-sharding protocol,
// host arithmetic only (no CUDA calls), exported through the C ABI so that the exact code
// dflop_search_plans runs between its NCCL collectives is also what the world-size-2 gloo test
// (tests/test_dist_gloo.py) executes on CPU:
//
//   shard       rank g of G evaluates candidates [floor(g*K/G), floor((g+1)*K/G)); Philox
//               counters are keyed by the GLOBAL id, so the family and its winner do not
//               depend on G (P:796 is the communicator the ranks share)
//   pack        key = min(T, 2^40 - 1) << 24 | id, id < 2^24: the lexicographic minimum of
//               (T, id) is the integer minimum of the keys, ONE 8-byte MIN all-reduce (P:738's
//               argmin over candidates, R18's lowest-id tie-break)
//   owner       the rank whose shard holds the winning id broadcasts the winner (every rank
//               computes it from the reduced key)
//   select      Eq. (1) over D batches (R33): the plan p minimising
//               (sum_b T_B(b, p), p) from the reduced [P x D] key array
#include <cstring>

#include "internal.h"

using namespace dflop;

extern "C" {

dflop_status dflop_shard_range(uint32_t K, uint32_t rank, uint32_t world, uint32_t* begin, uint32_t* end) {
    if (world == 0 || rank >= world || !begin || !end) {
        set_error("dflop_shard_range: need rank < world, world >= 1, non-NULL outputs");
        return DFLOP_ERR_INVALID_ARGUMENT;
    }
    *begin = (uint32_t)(((uint64_t)K * rank) / world);
    *end = (uint32_t)(((uint64_t)K * (rank + 1)) / world);
    return DFLOP_OK;
}

uint32_t dflop_owner_of(uint32_t K, uint32_t c, uint32_t world) {
    for (uint32_t g = 0; g < world; ++g) {
        uint32_t b = 0, e = 0;
        dflop_shard_range(K, g, world, &b, &e);
        if (c >= b && c < e) return g;
    }
    return 0xFFFFFFFFu;  // c >= K: no owner
}

uint64_t dflop_pack_key(uint64_t T, uint32_t id) {
    const uint64_t tmax = (1ull << 40) - 1;
    return ((T < tmax ? T : tmax) << 24) | (uint64_t)(id & 0xFFFFFFu);
}

dflop_status dflop_select_plan(const uint64_t* keys, uint32_t P, uint32_t D, const uint32_t* batch_n,
                               uint32_t* win_p, uint64_t* objective) {
    if (!keys || !win_p || P == 0 || D == 0) {
        set_error("dflop_select_plan: keys/win_p NULL or P, D == 0");
        return DFLOP_ERR_INVALID_ARGUMENT;
    }
    uint32_t best_p = 0xFFFFFFFFu;
    uint64_t best_obj = ~0ull;
    for (uint32_t p = 0; p < P; ++p) {
        uint64_t obj = 0;
        bool ok = true;
        for (uint32_t b = 0; b < D; ++b) {
            if (batch_n && batch_n[b] == 0) continue;  // an empty batch contributes 0
            const uint64_t k = keys[(size_t)p * D + b];
            if (k == ~0ull) {  // no candidate of this (plan, batch) was evaluated
                ok = false;
                break;
            }
            obj += k >> 24;
        }
        if (objective) objective[p] = ok ? obj : ~0ull;
        if (ok && obj < best_obj) {  // strict: ties keep the lower Stage-A rank p (R18)
            best_obj = obj;
            best_p = p;
        }
    }
    *win_p = best_p;
    if (best_p == 0xFFFFFFFFu) {
        set_error("no candidate evaluated");
        return DFLOP_ERR_UNSUPPORTED;
    }
    return DFLOP_OK;
}

}  // extern "C"
