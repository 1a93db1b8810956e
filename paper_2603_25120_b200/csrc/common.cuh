// common.cuh -- device building blocks shared by the libdflop kernels (sm_100a).
// Product code: nothing here is shared with oracle/.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dflop.h"

typedef unsigned long long u64;

#define DFLOP_DEV __device__ __forceinline__

// ---------------------------------------------------------------- Philox4x32-10
// Counter-based generator (Salmon et al., SC'11): round = (hi(M1*x2)^x1^k0, lo(M1*x2),
// hi(M0*x0)^x3^k1, lo(M0*x0)), Weyl key bump between rounds.  One call per 4 words.
struct Philox4 {
    uint32_t x, y, z, w;
};

DFLOP_DEV Philox4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t lo0 = 0xD2511F53u * c0, hi0 = __umulhi(0xD2511F53u, c0);
        const uint32_t lo1 = 0xCD9E8D57u * c2, hi1 = __umulhi(0xCD9E8D57u, c2);
        const uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return Philox4{c0, c1, c2, c3};
}

// floor(u * n / 2^32)
DFLOP_DEV uint32_t mulhi32(uint32_t u, uint32_t n) { return __umulhi(u, n); }

// ---------------------------------------------------------------- fp32 grid (predict)
// A throughput grid staged in shared memory for the per-sample kernel (R3 interpolation).
// ---------------------------------------------------------------- candidate state types
// Per-sample record in LPT base-order position t: combined encoder cost e = ef + eb, LLM
// cost l = lf + lb, and the forward parts needed by the 1F1B scoring.
template <typename A>
struct __align__(16) ItemRec {
    A e, l, ef, lf;
};

// Per-bucket running sums: E_j, L_j (the ILP's stage loads) and forward parts.
template <typename A>
struct __align__(16) BucketRec {
    A E, L, EF, LF;
};

template <typename A>
struct __align__(2 * sizeof(A)) Pair2 {
    A a, b;
};

// ---------------------------------------------------------------- 1F1B slot program
// Op encoding: bit 31 = backward, bits 16..20 = stage, bits 0..15 = microbatch.
DFLOP_DEV uint32_t op_kind(uint32_t op) { return op >> 31; }
DFLOP_DEV uint32_t op_stage(uint32_t op) { return (op >> 16) & 31u; }
DFLOP_DEV uint32_t op_mb(uint32_t op) { return op & 0xFFFFu; }

// Workspace header shared by the balance kernels.
struct BalanceHeader {
    u64 sum_e, sum_l;       // totals of e_i and l_i
    u64 max_key;            // max_i max(e_i, l_i)
    u64 best_key;           // atomicMin target
    uint32_t variant;       // candidate kernel variant: 0 packed u32, 1 plain u32, 2 u64
    uint32_t shift;         // bucket-index bits of the packed variant
    uint32_t status;        // DFLOP_DEV_* bits
    uint32_t offs;          // packed variant: C << shift, C = max_ld (the LPT probe offset)
    u64 max_ld;             // max_i max(l_i - e_i, 0)
    uint32_t pad[22];
};
static_assert(sizeof(BalanceHeader) == 144, "header layout");
