#include <type_traits>
// cand_impl.cuh -- the hot kernel of the path (a3 + a4): every candidate of the seeded
// family (O6-O7) is one group of GL lanes of a warp:
//
//   order  Philox4x32-10 Fisher-Yates inside groups of G base-order positions (c >= 2)
//   LPT    per sample, the argmin over m buckets of max(E_j + e_i, L_j + l_i) (c >= 1) or of
//          the current max(E_j, L_j) (c == 0, the paper's rule); the GL lanes of the
//          group each probe m/GL buckets and reduce (value, bucket) with warp shuffles
//   refine R rounds: bottleneck bucket j*, Philox partner j', best move or swap
//   score  non-interleaved 1F1B makespan over S stages, C_max
//
// Variants (cand.cuh): packed 32-bit keys (E << s | j, L << s | j) when the provable load bound
// allows, plain 32-bit, or 64-bit sums.
//
// Memory: the per-sample records (16 B in the 32-bit variant) and the position->item map
// are staged ONCE per CTA in shared memory and shared by all candidates of the SM; each
// candidate keeps SoA bucket sums EL[m] = {E, L}, FL[m] = {EF, LF} and a scratch area in
// shared memory (per-candidate stride staggered across banks); its assignment (one byte
// per sample when m <= 255) lives in an L2-resident per-slot double buffer, written by
// the LPT/refinement leader lane and scanned with 16-byte L2 loads by the refinement.  A
// new per-slot best flips the buffer index instead of copying.
#pragma once
#include "cand.cuh"

namespace dflop {

// ---------------------------------------------------------------- helpers
template <typename A>
DFLOP_DEV A amax() {
    return (A)~(A)0;
}
template <typename A>
DFLOP_DEV A maxa(A a, A b) {
    return a > b ? a : b;
}
template <typename A>
DFLOP_DEV A shfl_x(unsigned mask, A v, int off) {
    return __shfl_xor_sync(mask, v, off);
}
// Every warp is full (blockDim is a multiple of 32) and all candidate groups of a warp run
// identical control flow, so shuffles and warp barriers use the full mask; xor offsets below
// GL keep each exchange inside its group.
constexpr unsigned FULL = 0xFFFFFFFFu;
constexpr uint32_t kNoOpDev = 0xFFFFFFFFu;  // idle stage in the level-dense 1F1B program

// Diagnostic per-phase cycle counters (built only with -DDFLOP_TIMING, libdflop_timing.so):
// 0 LPT, 1 refine j*/j', 2 refine member lists, 3 refine pairs, 4 refine reduce+apply,
// 5 1F1B score, 6 loop/bookkeeping.
struct PhaseTimer {
#ifdef DFLOP_TIMING
    unsigned long long* acc;
    unsigned long long t0;
    unsigned long long loc[8];
    DFLOP_DEV void start(unsigned long long* a) {
        acc = a;
        t0 = clock64();
        for (int k = 0; k < 8; ++k) loc[k] = 0;
    }
    DFLOP_DEV void mark(int k) {
        const unsigned long long t1 = clock64();
        loc[k] += t1 - t0;
        t0 = t1;
    }
    DFLOP_DEV void flush(bool leader) {
        if (leader && acc)
            for (int k = 0; k < 8; ++k) atomicAdd(acc + k, loc[k]);
    }
#else
    DFLOP_DEV void start(unsigned long long*) {}
    DFLOP_DEV void mark(int) {}
    DFLOP_DEV void flush(bool) {}
#endif
};

template <typename A, int GL>
DFLOP_DEV void argmin_reduce(A& v, uint32_t& j, unsigned mask) {
#pragma unroll
    for (int off = GL / 2; off > 0; off >>= 1) {
        const A v2 = shfl_x(mask, v, off);
        const uint32_t j2 = __shfl_xor_sync(mask, j, off);
        if (v2 < v || (v2 == v && j2 < j)) {
            v = v2;
            j = j2;
        }
    }
}

// (W descending, j ascending); j == UINT32_MAX marks "no bucket on this lane"
template <typename A, int GL>
DFLOP_DEV void argmax_reduce(A& w, uint32_t& j, unsigned mask) {
#pragma unroll
    for (int off = GL / 2; off > 0; off >>= 1) {
        const A w2 = shfl_x(mask, w, off);
        const uint32_t j2 = __shfl_xor_sync(mask, j, off);
        const bool take = (j2 != 0xFFFFFFFFu) && (j == 0xFFFFFFFFu || w2 > w || (w2 == w && j2 < j));
        if (take) {
            w = w2;
            j = j2;
        }
    }
}

template <typename A, int GL>
DFLOP_DEV A max_reduce(A v, unsigned mask) {
#pragma unroll
    for (int off = GL / 2; off > 0; off >>= 1) v = maxa(v, shfl_x(mask, v, off));
    return v;
}

template <typename A, int GL>
DFLOP_DEV void lexmin_reduce(A& s, uint32_t& i, uint32_t& r, unsigned mask) {
#pragma unroll
    for (int off = GL / 2; off > 0; off >>= 1) {
        const A s2 = shfl_x(mask, s, off);
        const uint32_t i2 = __shfl_xor_sync(mask, i, off);
        const uint32_t r2 = __shfl_xor_sync(mask, r, off);
        if (s2 < s || (s2 == s && (i2 < i || (i2 == i && r2 < r)))) {
            s = s2;
            i = i2;
            r = r2;
        }
    }
}

template <typename A>
DFLOP_DEV void lex_update(A& bs, uint32_t& bi, uint32_t& br, A s, uint32_t i, uint32_t r) {
    if (s < bs || (s == bs && (i < bi || (i == bi && r < br)))) {
        bs = s;
        bi = i;
        br = r;
    }
}

// Fisher-Yates permutation of the ng <= 16 positions of group g for candidate c, packed as
// nibbles (nibble t = offset placed at position t).  Words u[0], u[1], ... come from
// Philox(ctr = (g, c, 0, p)), word q of call p being u[4p+q]; step t = ng-1 .. 1 uses
// u[ng-1-t] and swaps t with mulhi32(u, t+1).
DFLOP_DEV uint64_t make_perm(uint32_t g, uint32_t c, uint32_t ng, uint32_t k0, uint32_t k1) {
    uint64_t perm = 0xFEDCBA9876543210ull;
    Philox4 w{0, 0, 0, 0};
    for (uint32_t idx = 0; idx + 1 < ng; ++idx) {
        const uint32_t q = idx & 3u;
        if (q == 0) w = philox4x32_10(g, c, 0u, idx >> 2, k0, k1);
        const uint32_t u = q == 0 ? w.x : q == 1 ? w.y : q == 2 ? w.z : w.w;
        const uint32_t t = ng - 1 - idx;
        const uint32_t r = mulhi32(u, t + 1);
        const uint64_t a = (perm >> (4 * t)) & 15ull, b = (perm >> (4 * r)) & 15ull;
        const uint64_t x = a ^ b;
        perm ^= (x << (4 * t)) | (x << (4 * r));
    }
    return perm;
}

// Warp-cooperative group permutations.  The 32/GL candidate groups of a warp walk the same
// base-order groups in lockstep, so the Philox calls of W consecutive groups of all of them
// (32/GL x W x nc calls, nc = ceil((G-1)/4)) are spread over the 32 lanes (<= 4 calls each),
// the words are exchanged with shuffles and lane u = cg*W + gg runs the Fisher-Yates of
// candidate group cg, base group g0 + gg.  Same words, same swaps as make_perm.
template <int GL>
DFLOP_DEV uint64_t batch_perms(uint32_t g0, uint32_t W, uint32_t nc, uint32_t c, uint32_t n, uint32_t G, uint32_t k0,
                               uint32_t k1) {
    constexpr uint32_t cw = 32u / GL;  // candidate groups per warp
    const uint32_t lane = threadIdx.x & 31u;
    if (cw * W == 32u) {
        // one Fisher-Yates per lane: the lane draws its own group's Philox words (no exchange)
        const uint32_t cg = lane / W, gg = lane % W;
        const uint32_t cc = __shfl_sync(FULL, c, cg * GL);
        const uint32_t start = (g0 + gg) * G;
        const uint32_t ng = start < n ? min(G, n - start) : 0u;
        uint64_t perm = 0xFEDCBA9876543210ull;
        uint32_t p32 = 0x76543210u;
        const bool narrow = G <= 8;
        if (ng == 8u && nc == 2u) {  // a full group of 8 (every preset): 7 steps, no bounds tests
            const Philox4 r0 = philox4x32_10(g0 + gg, cc, 0u, 0u, k0, k1);
            const Philox4 r1 = philox4x32_10(g0 + gg, cc, 0u, 1u, k0, k1);
            const uint32_t wq[7] = {r0.x, r0.y, r0.z, r0.w, r1.x, r1.y, r1.z};
#pragma unroll
            for (uint32_t idx = 0; idx < 7; ++idx) {
                const uint32_t tt = 7 - idx;
                const uint32_t rr = mulhi32(wq[idx], tt + 1);
                const uint32_t x = ((p32 >> (4 * tt)) ^ (p32 >> (4 * rr))) & 15u;
                p32 ^= (x << (4 * tt)) | (x << (4 * rr));
            }
            perm = 0xFEDCBA9800000000ull | p32;
            if (cc < 2) perm = 0xFEDCBA9876543210ull;
            return perm;
        }
        for (uint32_t pc = 0; pc < nc; ++pc) {
            const Philox4 r = philox4x32_10(g0 + gg, cc, 0u, pc, k0, k1);
            const uint32_t wq[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (uint32_t q = 0; q < 4; ++q) {
                const uint32_t idx = pc * 4 + q;
                if (idx + 1 < ng) {
                    const uint32_t tt = ng - 1 - idx;
                    const uint32_t rr = mulhi32(wq[q], tt + 1);
                    if (narrow) {
                        const uint32_t x = ((p32 >> (4 * tt)) ^ (p32 >> (4 * rr))) & 15u;
                        p32 ^= (x << (4 * tt)) | (x << (4 * rr));
                    } else {
                        const uint64_t a = (perm >> (4 * tt)) & 15ull, b = (perm >> (4 * rr)) & 15ull;
                        const uint64_t x = a ^ b;
                        perm ^= (x << (4 * tt)) | (x << (4 * rr));
                    }
                }
            }
        }
        if (narrow) perm = 0xFEDCBA9800000000ull | p32;
        if (cc < 2) perm = 0xFEDCBA9876543210ull;
        return perm;
    }
    const uint32_t per_cg = W * nc, tasks = cw * per_cg;
    uint32_t w[4][4];
#pragma unroll
    for (uint32_t k = 0; k < 4; ++k) {
        const uint32_t t = lane + 32u * k;
        const uint32_t cg = min(t / per_cg, cw - 1u);
        const uint32_t cc = __shfl_sync(FULL, c, cg * GL);
        w[k][0] = w[k][1] = w[k][2] = w[k][3] = 0u;
        if (t < tasks) {
            const uint32_t rem = t % per_cg, gg = rem / nc, pc = rem % nc;
            const Philox4 r = philox4x32_10(g0 + gg, cc, 0u, pc, k0, k1);
            w[k][0] = r.x;
            w[k][1] = r.y;
            w[k][2] = r.z;
            w[k][3] = r.w;
        }
        if (32u * (k + 1) >= tasks) break;  // warp-uniform
    }
    const uint32_t cg = min(lane / W, cw - 1u), gg = lane % W;
    const uint32_t cc = __shfl_sync(FULL, c, cg * GL);
    const uint32_t start = (g0 + gg) * G;
    const uint32_t ng = start < n ? min(G, n - start) : 0u;
    // the Fisher-Yates on a 32-bit word when every position of the group is < 8 (G <= 8:
    // half the shift/xor work of the 64-bit form; the high nibbles stay the identity)
    uint64_t perm = 0xFEDCBA9876543210ull;
    uint32_t p32 = 0x76543210u;
    const bool narrow = G <= 8;  // warp-uniform
    for (uint32_t pc = 0; pc < nc; ++pc) {
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q) {
            const uint32_t t = (cg * W + gg) * nc + pc;
            uint32_t word = 0;
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) {
                const uint32_t v = __shfl_sync(FULL, w[k][q], t & 31u);
                if ((t >> 5) == k) word = v;
                if (32u * (k + 1) >= tasks) break;  // warp-uniform
            }
            const uint32_t idx = pc * 4 + q;
            if (idx + 1 < ng) {
                const uint32_t tt = ng - 1 - idx;
                const uint32_t r = mulhi32(word, tt + 1);
                if (narrow) {
                    const uint32_t x = ((p32 >> (4 * tt)) ^ (p32 >> (4 * r))) & 15u;
                    p32 ^= (x << (4 * tt)) | (x << (4 * r));
                } else {
                    const uint64_t a = (perm >> (4 * tt)) & 15ull, b = (perm >> (4 * r)) & 15ull;
                    const uint64_t x = a ^ b;
                    perm ^= (x << (4 * tt)) | (x << (4 * r));
                }
            }
        }
    }
    if (narrow) perm = 0xFEDCBA9800000000ull | p32;
    if (cc < 2 || lane >= cw * W) perm = 0xFEDCBA9876543210ull;
    return perm;
}

// Pair score max(se + a, sl + b, pe - a, pl - b) of moving i (row) to j' and i' (a, b) to j*
// (O6), 32-bit: one subtraction and three fused add-max instructions
DFLOP_DEV uint32_t score4(uint32_t se, uint32_t sl, uint32_t pe, uint32_t pl, uint32_t a, uint32_t b) {
    return __viaddmax_u32(se, a, __viaddmax_u32(sl, b, __viaddmax_u32(pe, 0u - a, pl - b)));
}

// (hi << 32 | lo) as a register pair, without 64-bit arithmetic
DFLOP_DEV u64 pack64(uint32_t hi, uint32_t lo) {
    u64 r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(lo), "r"(hi));
    return r;
}

// ---------------------------------------------------------------- item table access
template <typename A, bool SM>
struct Tbl {
    const ItemRec<A>* it;
    const uint16_t* pi16;   // SM
    const uint32_t* pi32;   // !SM
    uint32_t it_s;          // SM: shared-window address of it (explicit ld.shared: no per-use
                            // generic-to-shared conversion in the LPT loop)
    DFLOP_DEV ItemRec<A> item(uint32_t pos) const {
        if (SM) return it[pos];
        if (sizeof(A) == 4) {
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(it) + pos);
            return ItemRec<A>{(A)v.x, (A)v.y, (A)v.z, (A)v.w};
        }
        const ulonglong2* q = reinterpret_cast<const ulonglong2*>(it) + 2 * (size_t)pos;
        const ulonglong2 a = __ldg(q), b = __ldg(q + 1);
        return ItemRec<A>{(A)a.x, (A)a.y, (A)b.x, (A)b.y};
    }
    DFLOP_DEV Pair2<A> el(uint32_t pos) const {
        if (SM) {
            if constexpr (sizeof(A) == 4) {
                Pair2<A> r;
                // the table is read-only after staging: no volatile, no clobber (free to schedule)
                asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.a), "=r"(r.b) : "r"(it_s + pos * 16u));
                return r;
            } else {
                return *reinterpret_cast<const Pair2<A>*>(it + pos);
            }
        }
        const ItemRec<A> r = item(pos);
        return Pair2<A>{r.e, r.l};
    }
    DFLOP_DEV uint32_t idx(uint32_t pos) const { return SM ? (uint32_t)pi16[pos] : __ldg(pi32 + pos); }
};

// load of bucket j without the packed index bits
template <typename A, bool PK>
DFLOP_DEV A unpack(A v, uint32_t sh) {
    return PK ? (A)(v >> sh) : v;
}
// the same load kept in the shifted domain (W << s) of the packed variant, whose item records
// hold e << s and l << s (k_build_items): comparisons and differences are unchanged
template <typename A, bool PK>
DFLOP_DEV A keyval(A v, uint32_t sh) {
    return PK ? (A)(v & ~((1u << sh) - 1u)) : v;
}

// shared-memory byte store / 8- and 16-byte loads at a shared-window address (the LPT's
// per-group staging of the one-byte assignment, flushed with one global store per group)
DFLOP_DEV void sts_u8(uint32_t saddr, uint32_t v) { asm volatile("st.shared.u8 [%0], %1;" ::"r"(saddr), "r"(v)); }
DFLOP_DEV uint32_t lds_u8(uint32_t saddr) {
    uint32_t v;
    asm volatile("ld.shared.u8 %0, [%1];" : "=r"(v) : "r"(saddr) : "memory");
    return v;
}
DFLOP_DEV uint2 lds_v2(uint32_t saddr) {
    uint2 v;
    asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(saddr) : "memory");
    return v;
}
DFLOP_DEV uint4 lds_v4(uint32_t saddr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(saddr)
                 : "memory");
    return v;
}

// The ng (<= 16) staged decisions of base-order group [start, start + ng) -> the assignment:
// one 8- or 16-byte store by lane 0 for full aligned groups of 8 / 16, else one byte per lane.
// Called by all lanes of the warp (start and ng are warp-uniform).
template <int GL>
DFLOP_DEV void flush_stage(uint8_t* apos, uint32_t stage_s, uint32_t start, uint32_t ng, uint32_t gl) {
    __syncwarp(FULL);
    if (ng == 8 && (start & 7u) == 0) {
        if (gl == 0) *reinterpret_cast<uint2*>(apos + start) = lds_v2(stage_s);
    } else if (ng == 16 && (start & 15u) == 0) {
        if (gl == 0) {
            if ((stage_s & 15u) == 0) {
                *reinterpret_cast<uint4*>(apos + start) = lds_v4(stage_s);
            } else {  // an 8-byte aligned stage (k_lpt with one lane per candidate)
                const uint2 lo = lds_v2(stage_s), hi = lds_v2(stage_s + 8);
                *reinterpret_cast<uint4*>(apos + start) = make_uint4(lo.x, lo.y, hi.x, hi.y);
            }
        }
    } else {
        for (uint32_t u = gl; u < ng; u += GL) apos[start + u] = (uint8_t)lds_u8(stage_s + u);
    }
    __syncwarp(FULL);
}

DFLOP_DEV void set_apos(uint8_t* apos, uint32_t pos, uint32_t j, bool wide) {
    if (wide)
        reinterpret_cast<uint16_t*>(apos)[pos] = (uint16_t)j;
    else
        apos[pos] = (uint8_t)j;
}

// Calls f(pos, j) for the entries of one 16-byte block of the assignment (16 u8 or 8 u16
// positions); padding past n holds 0xFF / 0xFFFF, never a bucket (m <= 255 / m <= 65535).
template <typename F>
DFLOP_DEV void each_entry(const uint4 v, uint32_t blk, bool wide, uint32_t m, F&& f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if (!wide) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const uint32_t j = (w[k] >> (8 * b)) & 0xFFu;
                if (j < m) f(blk * 16 + 4 * k + b, j);
            }
    } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const uint32_t j = (w[k] >> (16 * b)) & 0xFFFFu;
                if (j < m) f(blk * 8 + 2 * k + b, j);
            }
    }
}

// each_entry for a one-byte assignment with the 16 entries of the block visited from entry
// `rot` on (f(pos, j) for pos = blk*16 + (e + rot) % 16): lanes holding consecutive blocks
// then read item records 16*rot bytes apart -- distinct shared-memory banks -- instead of
// all reading the same bank (the blocks are 256 bytes of records apart)
template <typename F>
DFLOP_DEV void each_entry_rot(const uint4 v, uint32_t blk, uint32_t rot, uint32_t m, F&& f) {
    // rotate the 16 bytes right by rot (< 16) bytes: byte e of r = byte (e + rot) % 16 of v
    const uint32_t q = rot >> 2, sh = 8u * (rot & 3u);
    // words rotated by q (two select stages, no dynamic register indexing), then bytes by sh
    const bool q1 = q & 1u, q2 = q & 2u;
    const uint32_t a0 = q1 ? v.y : v.x, a1 = q1 ? v.z : v.y, a2 = q1 ? v.w : v.z, a3 = q1 ? v.x : v.w;
    const uint32_t r[4] = {q2 ? a2 : a0, q2 ? a3 : a1, q2 ? a0 : a2, q2 ? a1 : a3};
    uint32_t u[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) u[i] = __funnelshift_r(r[i], r[(i + 1) & 3], sh);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const uint32_t j = (u[k] >> (8 * b)) & 0xFFu;
            if (j < m) f(blk * 16 + ((4 * k + b + rot) & 15u), j);
        }
}

// CSR member lists of all m buckets from the assignment: cnt[j] members of bucket j at
// csr[off[j] ..], off[j+1] - off[j] = (LPT count) + sigma.  Two 16-byte L2 passes (count,
// then scatter); the list order is irrelevant (the pair search is a keyed minimum).
// With FL != null (the first build after LPT) the count pass also forms the forward sums
// FL[j] = (sum EF, sum LF) of the members (shared-memory atomics): the LPT steps then update
// only EL -- one atomic per 8 entries of a warp instead of a read-modify-write per sample.
template <typename A, int GL, bool SM, typename OT = uint32_t>
DFLOP_DEV void build_lists(const CandParams& p, const Tbl<A, SM>& T, const uint8_t* apos, bool wide, uint32_t* cnt,
                           OT* off, uint16_t* csr, uint32_t gl, Pair2<A>* FL) {
    const uint32_t m = p.m, nblk = p.apos_bytes / 16, sig = p.sigma;
    const uint4* ap = reinterpret_cast<const uint4*>(apos);
    for (uint32_t j = gl; j < m; j += GL) cnt[j] = 0;
    __syncwarp(FULL);
    if (FL) {
        auto acc = [&](uint32_t pos, uint32_t j) {
            atomicAdd(&cnt[j], 1u);
            const ItemRec<A> r = T.item(pos);
            atomicAdd(&FL[j].a, r.ef);
            atomicAdd(&FL[j].b, r.lf);
        };
        for (uint32_t b = gl; b < nblk; b += GL) {
            if (wide)
                each_entry(__ldcg(ap + b), b, true, m, acc);
            else  // the record loads of the group's lanes on distinct banks
                each_entry_rot(__ldcg(ap + b), b, gl & 15u, m, acc);
        }
    } else {
        for (uint32_t b = gl; b < nblk; b += GL)
            each_entry(__ldcg(ap + b), b, wide, m, [&](uint32_t, uint32_t j) { atomicAdd(&cnt[j], 1u); });
    }
    __syncwarp(FULL);
    // exclusive prefix of cnt[j] + sigma, GL buckets per step (coalesced when the counters
    // live in global memory); counters reset for the scatter pass
    uint32_t run = 0;
    for (uint32_t j0 = 0; j0 < m; j0 += GL) {
        const uint32_t j = j0 + gl;
        const uint32_t v = j < m ? cnt[j] + sig : 0u;
        uint32_t inc = v;
#pragma unroll
        for (int d = 1; d < GL; d <<= 1) {
            const uint32_t y = __shfl_up_sync(FULL, inc, d, GL);
            if (gl >= (uint32_t)d) inc += y;
        }
        if (j < m) {
            off[j] = (OT)(run + inc - v);
            cnt[j] = 0;
        }
        run += __shfl_sync(FULL, inc, GL - 1, GL);
    }
    if (gl == 0) off[m] = (OT)run;
    __syncwarp(FULL);
    for (uint32_t b = gl; b < nblk; b += GL)
        each_entry(__ldcg(ap + b), b, wide, m, [&](uint32_t pos, uint32_t j) {
            const uint32_t at = atomicAdd(&cnt[j], 1u);
            csr[off[j] + at] = (uint16_t)pos;
        });
    __syncwarp(FULL);
}

// FL[j] = (sum EF, sum LF) over the members of bucket j, from the assignment (when no
// refinement round runs: m == 1 or R == 0; otherwise the first build_lists forms it)
template <typename A, int GL, bool SM>
DFLOP_DEV void form_fl(const CandParams& p, const Tbl<A, SM>& T, const uint8_t* apos, bool wide, Pair2<A>* FL,
                       uint32_t gl) {
    const uint4* ap = reinterpret_cast<const uint4*>(apos);
    for (uint32_t b = gl; b < p.apos_bytes / 16; b += GL)
        each_entry(__ldcg(ap + b), b, wide, p.m, [&](uint32_t pos, uint32_t j) {
            const ItemRec<A> r = T.item(pos);
            atomicAdd(&FL[j].a, r.ef);
            atomicAdd(&FL[j].b, r.lf);
        });
    __syncwarp(FULL);
}

// Q buckets per lane (m == Q*GL), fully unrolled: two running minima of the packed keys.
// The packed buckets hold (E', L' + C') and d = e' - l' + C' (see lpt_pass): one fused add-max
// per probe, max(E' + d, L' + C') = max(E' + e', L' + l') - l' + C'.
template <int Q, int GL>
DFLOP_DEV void probe_fixed(const Pair2<uint32_t>* EL, uint32_t gl, uint32_t d, uint32_t& b0, uint32_t& b1) {
#pragma unroll
    for (uint32_t k = 0; k < Q; k += 2) {
        const Pair2<uint32_t> x = EL[gl + GL * k], y = EL[gl + GL * (k + 1)];
        b0 = min(b0, max(x.a + d, x.b));
        b1 = min(b1, max(y.a + d, y.b));
    }
}

// Two consecutive samples A, B of the (perturbed) order in one step of the packed variant
// -- exactly the sequential decisions: B's argmin is computed on the
// loads before A's update together with its runner-up; A's update only raises bucket a*, so
// if B's best b1 is not a* it stays B's argmin (ties: the packed keys carry the index), and
// if b1 = a*, B's argmin is the smaller of the runner-up and a*'s key after A's update
// (computed by a*'s owner lane and broadcast).  Halves the dependent reduction chains.
// FIX8: m == 8 * GL and a one-byte assignment (every preset); else any m (loop, bounds).
template <int GL, bool FIX8>
DFLOP_DEV void lpt_pair_step(Pair2<uint32_t>* EL, Pair2<uint32_t>* FL, uint8_t* apos, uint32_t pa, uint32_t pb,
                             const Pair2<uint32_t> ia, const Pair2<uint32_t> ib, uint32_t jmask,
                             uint32_t gl, uint32_t m, bool wide, uint32_t co, uint32_t stage_s, uint32_t start,
                             bool staged) {
    // never called for c == 0 (its probes use zero items; the single-sample loop does it)
    const uint32_t da = ia.a - ia.b + co, db = ib.a - ib.b + co;  // probe offsets (lpt_pass)
    uint32_t a0 = 0xFFFFFFFFu, a1 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu;
    if constexpr (FIX8) {
        // B's two smallest of 8 keys by a merge tree: sorted pairs, then (lo, hi) merges
        // m1 = min(lo, lo'), m2 = min(max(lo, lo'), hi, hi') -- 17 min/max instead of 24
        uint32_t lo[4], hi[4];
#pragma unroll
        for (uint32_t k = 0; k < 8; k += 2) {
            const Pair2<uint32_t> x = EL[gl + GL * k], y = EL[gl + GL * (k + 1)];
            a0 = min(a0, max(x.a + da, x.b));
            a1 = min(a1, max(y.a + da, y.b));
            const uint32_t vx = max(x.a + db, x.b), vy = max(y.a + db, y.b);
            lo[k / 2] = min(vx, vy);
            hi[k / 2] = max(vx, vy);
        }
        const uint32_t l01 = min(lo[0], lo[1]), h01 = min(max(lo[0], lo[1]), min(hi[0], hi[1]));
        const uint32_t l23 = min(lo[2], lo[3]), h23 = min(max(lo[2], lo[3]), min(hi[2], hi[3]));
        m1 = min(l01, l23);
        m2 = min(max(l01, l23), min(h01, h23));
    } else {
        // two buckets per step: B's pair sorted (lo, hi), merged into the running two smallest
        // (m1, m2) -- m2 = min(max(m1, lo), m2, hi) -- 2.5 instead of 3 min/max per bucket
        uint32_t j = gl;
        for (; j + GL < m; j += 2 * GL) {
            const Pair2<uint32_t> x = EL[j], y = EL[j + GL];
            a0 = min(a0, max(x.a + da, x.b));
            a1 = min(a1, max(y.a + da, y.b));
            const uint32_t vx = max(x.a + db, x.b), vy = max(y.a + db, y.b);
            const uint32_t lo = min(vx, vy), hi = max(vx, vy);
            m2 = min(min(max(m1, lo), m2), hi);
            m1 = min(m1, lo);
        }
        if (j < m) {
            const Pair2<uint32_t> x = EL[j];
            a0 = min(a0, max(x.a + da, x.b));
            const uint32_t vx = max(x.a + db, x.b);
            m2 = min(m2, max(m1, vx));
            m1 = min(m1, vx);
        }
    }
    uint32_t ba = min(a0, a1);
#pragma unroll
    for (int off = GL / 2; off > 0; off >>= 1) {
        ba = min(ba, __shfl_xor_sync(FULL, ba, off));
        const uint32_t o1 = __shfl_xor_sync(FULL, m1, off), o2 = __shfl_xor_sync(FULL, m2, off);
        m2 = min(max(m1, o1), min(m2, o2));  // second smallest of the two sorted pairs
        m1 = min(m1, o1);
    }
    const uint32_t ja = ba & jmask;
    const bool own_a = ((ba ^ gl) & (GL - 1)) == 0;
    // every lane of the group reads a* (one broadcast load) and evaluates B's probe of a*
    // after A itself -- no shuffle from the owner on the dependency chain
    const Pair2<uint32_t> ela = EL[ja];
    const uint32_t alt = min(m2, max(ela.a + ia.a + db, ela.b + ia.b));  // a* after A, probed by B
    const uint32_t kb = ((m1 & jmask) != ja) ? m1 : alt;
    const uint32_t jb = kb & jmask;
    const bool own_b = ((kb ^ gl) & (GL - 1)) == 0;
    // owner updates as predicated stores (no branch): FL is formed by the first build_lists;
    // the assignment byte goes to the group's shared-memory stage (flushed per base group)
    if (own_a) EL[ja] = Pair2<uint32_t>{ela.a + ia.a, ela.b + ia.b};
    const Pair2<uint32_t> elb = EL[jb];  // after A's update in program order when jb = ja (same lane)
    if (own_b) EL[jb] = Pair2<uint32_t>{elb.a + ib.a, elb.b + ib.b};
    if (FIX8 || staged) {
        if (own_a) sts_u8(stage_s + (pa - start), ja);
        if (own_b) sts_u8(stage_s + (pb - start), jb);
    } else {
        if (own_a) set_apos(apos, pa, ja, wide);
        if (own_b) set_apos(apos, pb, jb, wide);
    }
}

// lpt_pair_step for exactly Q buckets per lane (m == Q * GL, one-byte assignment, staged),
// fully unrolled: B's two smallest by sorted pairs merged four buckets at a time (the split
// pipeline's k_lpt: Q = 32 for m = 64 at GL = 2)
template <int GL, int Q>
DFLOP_DEV void lpt_pair_step_q(Pair2<uint32_t>* EL, uint32_t pa, uint32_t pb, const Pair2<uint32_t> ia,
                               const Pair2<uint32_t> ib, uint32_t jmask, uint32_t gl, uint32_t co,
                               uint32_t stage_s, uint32_t start) {
    static_assert(Q % 4 == 0, "Q buckets per lane, a multiple of 4");
    const uint32_t da = ia.a - ia.b + co, db = ib.a - ib.b + co;
    uint32_t a0 = 0xFFFFFFFFu, a1 = 0xFFFFFFFFu, m1 = 0xFFFFFFFFu, m2 = 0xFFFFFFFFu;
#pragma unroll
    for (uint32_t k = 0; k < Q; k += 4) {
        const Pair2<uint32_t> x0 = EL[gl + GL * k], x1 = EL[gl + GL * (k + 1)];
        const Pair2<uint32_t> x2 = EL[gl + GL * (k + 2)], x3 = EL[gl + GL * (k + 3)];
        a0 = min(a0, min(max(x0.a + da, x0.b), max(x1.a + da, x1.b)));
        a1 = min(a1, min(max(x2.a + da, x2.b), max(x3.a + da, x3.b)));
        const uint32_t v0 = max(x0.a + db, x0.b), v1 = max(x1.a + db, x1.b);
        const uint32_t v2 = max(x2.a + db, x2.b), v3 = max(x3.a + db, x3.b);
        const uint32_t lo01 = min(v0, v1), hi01 = max(v0, v1), lo23 = min(v2, v3), hi23 = max(v2, v3);
        const uint32_t l = min(lo01, lo23), h = min(max(lo01, lo23), min(hi01, hi23));
        m2 = min(min(max(m1, l), m2), h);
        m1 = min(m1, l);
    }
    uint32_t ba = min(a0, a1);
#pragma unroll
    for (int off = GL / 2; off > 0; off >>= 1) {
        ba = min(ba, __shfl_xor_sync(FULL, ba, off));
        const uint32_t o1 = __shfl_xor_sync(FULL, m1, off), o2 = __shfl_xor_sync(FULL, m2, off);
        m2 = min(max(m1, o1), min(m2, o2));
        m1 = min(m1, o1);
    }
    const uint32_t ja = ba & jmask;
    const bool own_a = ((ba ^ gl) & (GL - 1)) == 0;
    const Pair2<uint32_t> ela = EL[ja];
    const uint32_t alt = min(m2, max(ela.a + ia.a + db, ela.b + ia.b));
    const uint32_t kb = ((m1 & jmask) != ja) ? m1 : alt;
    const uint32_t jb = kb & jmask;
    const bool own_b = ((kb ^ gl) & (GL - 1)) == 0;
    if (own_a) EL[ja] = Pair2<uint32_t>{ela.a + ia.a, ela.b + ia.b};
    const Pair2<uint32_t> elb = EL[jb];
    if (own_b) EL[jb] = Pair2<uint32_t>{elb.a + ib.a, elb.b + ib.b};
    if (own_a) sts_u8(stage_s + (pa - start), ja);
    if (own_b) sts_u8(stage_s + (pb - start), jb);
}

// ---------------------------------------------------------------- LPT pass (R12)
// c == 0: argmin of the current max(E_j, L_j) (the paper's rule); c >= 1: argmin of the
// resulting max(E_j + e_i, L_j + l_i); lowest j on ties.
// Packed variant: during this pass bucket j holds (E_j << s | j, (L_j << s | j) + co) with
// co = C << s, C = max_i max(l_i - e_i, 0) (k_build_items), and a sample probes with
// d = e' - l' + co >= 0: max(E' + d, L' + co) = max(E' + e', L' + l') - l' + co, the same
// order over j (and the index bits) as the resulting max, without wrap-around (the variant's
// bound covers probe + C); c == 0 probes with d = co.
template <typename A, bool PK, int GL, bool SM, typename TB = Tbl<A, SM>>
DFLOP_DEV void lpt_pass(const CandParams& p, const TB& T, uint32_t c, uint32_t sh, Pair2<A>* EL,
                        Pair2<A>* FL, uint8_t* apos, uint8_t* scr, uint32_t gl, uint32_t co, bool forced) {
    const uint32_t n = p.n, m = p.m, G = p.G;
    const bool wide = p.wide != 0;  // u16 assignment when m > 255
    const A use = (c == 0) ? (A)0 : amax<A>();  // c == 0 probes the current load
    const bool pairs = __all_sync(FULL, c != 0);
    const uint32_t jmask = PK ? (1u << sh) - 1u : 0u;
    // plain 32-bit variant with lane-local packed LPT keys (k_candidates): sh = 0x100 | kb
    const uint32_t ush = (!PK && sizeof(A) == 4 && sh >= 0x100u) ? (sh & 0xFFu) : 0u;
    const bool lanepk = !PK && sizeof(A) == 4 && sh >= 0x100u;
    const uint32_t nc = (G - 1 + 3) / 4;  // Philox calls per group
    // base groups per permutation batch: every lane of the warp runs one Fisher-Yates (W = 32 /
    // candidate groups per warp) as long as the Philox words fit the 4 calls per lane of batch_perms
    const uint32_t W = nc ? max(1u, min((uint32_t)GL, 128u / ((32u / GL) * nc))) : 1u;
    const uint32_t lane = threadIdx.x & 31u, mycg = lane / GL;
    const uint32_t n_groups = (n + G - 1) / G;
    // one-byte assignments: the group's decisions are staged in the (idle) refinement scratch
    // and flushed with one 8/16-byte store per base group (flush_stage)
    const bool stg = !wide;
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(scr);
    // The first m decisions are forced when every one of the m largest items has e > 0 and
    // l > 0 (`forced`, k_candidates): at step t < m buckets 0..t-1 hold one such item each and
    // the rest are empty, so every non-empty probe -- max(E_k + e, L_k + l) with E_k, L_k > 0,
    // or the current load max(E_k, L_k) > 0 of the c = 0 rule -- is strictly above the empty
    // buckets' max(e, l) (resp. 0), and the lowest empty bucket, t, wins.  (With an item of
    // e = 0 or l = 0 among them an earlier bucket can tie the empty ones and take the sample,
    // so the shortcut is off.)  Lane gl places the forced steps of its own buckets.
    for (uint32_t g0 = 0; g0 < n_groups; g0 += W) {
      const uint64_t preg = nc ? batch_perms<GL>(g0, W, nc, c, n, G, p.seed0, p.seed1) : 0xFEDCBA9876543210ull;
      for (uint32_t gg = 0; gg < W && g0 + gg < n_groups; ++gg) {
        const uint32_t start = (g0 + gg) * G;
        const uint32_t ng = min(G, n - start);
        const uint64_t perm = nc ? __shfl_sync(FULL, preg, mycg * W + gg) : 0xFEDCBA9876543210ull;
        uint32_t t = 0;
        if (forced && start < m) {  // warp-uniform
            const uint32_t nf = min(ng, m - start);
            for (uint32_t u = (gl + GL - start % GL) % GL; u < nf; u += GL) {
                const uint32_t nib = (uint32_t)(perm >> (4 * u)) & 15u;
                const uint32_t pos = start + nib, j = start + u;  // j % GL == gl: this lane's bucket
                const Pair2<A> r = T.el(pos);
                Pair2<A> el = EL[j];
                el.a += r.a << ush;
                el.b += r.b << ush;
                EL[j] = el;
                if (stg)
                    sts_u8(stage_s + nib, j);
                else
                    set_apos(apos, pos, j, wide);
            }
            t = nf;
        }
#ifndef DFLOP_NO_LPT_PAIRS
        if constexpr (PK) {
            // two samples per step (see lpt_pair_step); the warp holding c == 0 takes the
            // single-sample loop so the pair step needs no probe mask
            if (!pairs) {
            } else if (m == 8 * GL && !wide) {
                for (; t + 1 < ng; t += 2) {
                    const uint32_t pa = start + (uint32_t)((perm >> (4 * t)) & 15ull);
                    const uint32_t pb = start + (uint32_t)((perm >> (4 * (t + 1))) & 15ull);
                    lpt_pair_step<GL, true>(reinterpret_cast<Pair2<uint32_t>*>(EL),
                                            reinterpret_cast<Pair2<uint32_t>*>(FL), apos, pa, pb, T.el(pa),
                                            T.el(pb), jmask, gl, m, false, co, stage_s, start, true);
                }
            } else if (GL == 1 && m == 64 && !wide) {
                for (; t + 1 < ng; t += 2) {
                    const uint32_t pa = start + (uint32_t)((perm >> (4 * t)) & 15ull);
                    const uint32_t pb = start + (uint32_t)((perm >> (4 * (t + 1))) & 15ull);
                    lpt_pair_step_q<GL, 64>(reinterpret_cast<Pair2<uint32_t>*>(EL), pa, pb, T.el(pa), T.el(pb),
                                            jmask, gl, co, stage_s, start);
                }
            } else if (GL <= 4 && m == 32 * GL && !wide) {
                for (; t + 1 < ng; t += 2) {
                    const uint32_t pa = start + (uint32_t)((perm >> (4 * t)) & 15ull);
                    const uint32_t pb = start + (uint32_t)((perm >> (4 * (t + 1))) & 15ull);
                    lpt_pair_step_q<GL, 32>(reinterpret_cast<Pair2<uint32_t>*>(EL), pa, pb, T.el(pa), T.el(pb),
                                            jmask, gl, co, stage_s, start);
                }
            } else if (GL <= 4 && m == 16 * GL && !wide) {
                for (; t + 1 < ng; t += 2) {
                    const uint32_t pa = start + (uint32_t)((perm >> (4 * t)) & 15ull);
                    const uint32_t pb = start + (uint32_t)((perm >> (4 * (t + 1))) & 15ull);
                    lpt_pair_step_q<GL, 16>(reinterpret_cast<Pair2<uint32_t>*>(EL), pa, pb, T.el(pa), T.el(pb),
                                            jmask, gl, co, stage_s, start);
                }
            } else {
                for (; t + 1 < ng; t += 2) {
                    const uint32_t pa = start + (uint32_t)((perm >> (4 * t)) & 15ull);
                    const uint32_t pb = start + (uint32_t)((perm >> (4 * (t + 1))) & 15ull);
                    lpt_pair_step<GL, false>(reinterpret_cast<Pair2<uint32_t>*>(EL),
                                             reinterpret_cast<Pair2<uint32_t>*>(FL), apos, pa, pb, T.el(pa),
                                             T.el(pb), jmask, gl, m, wide, co, stage_s, start, stg);
                }
            }
        }
#endif
        for (; t < ng; ++t) {
            const uint32_t pos = start + (uint32_t)((perm >> (4 * t)) & 15ull);
            const Pair2<A> el2 = T.el(pos);  // (e, l): 8-byte loads (the sample's record half)
            const ItemRec<A> it{el2.a, el2.b, 0, 0};
            uint32_t bj;
            if (PK) {
                // keys (W << s) | j: one fused add-max and one min per probe
                const uint32_t d = (((uint32_t)it.e - (uint32_t)it.l) & (uint32_t)use) + co;
                uint32_t b0 = 0xFFFFFFFFu, b1 = 0xFFFFFFFFu;
                if (m == 8 * GL) {  // every preset: exactly 8 buckets per lane, no bounds tests
                    probe_fixed<8, GL>(reinterpret_cast<const Pair2<uint32_t>*>(EL), gl, d, b0, b1);
                } else if (m == 16 * GL) {
                    probe_fixed<16, GL>(reinterpret_cast<const Pair2<uint32_t>*>(EL), gl, d, b0, b1);
                } else if (m == 32 * GL) {
                    probe_fixed<32, GL>(reinterpret_cast<const Pair2<uint32_t>*>(EL), gl, d, b0, b1);
                } else if (m < 8 * GL) {  // at most 8 buckets per lane, fully unrolled
#pragma unroll
                    for (uint32_t k = 0; k < 8; k += 2) {
                        const uint32_t j0 = gl + GL * k, j1 = j0 + GL;
                        if (j0 < m) {
                            const Pair2<A> x = EL[j0];
                            b0 = min(b0, max((uint32_t)x.a + d, (uint32_t)x.b));
                        }
                        if (j1 < m) {
                            const Pair2<A> y = EL[j1];
                            b1 = min(b1, max((uint32_t)y.a + d, (uint32_t)y.b));
                        }
                    }
                } else {
                    uint32_t j = gl;
#pragma unroll 4
                    for (; j + GL < m; j += 2 * GL) {
                        const Pair2<A> x = EL[j], y = EL[j + GL];
                        b0 = min(b0, max((uint32_t)x.a + d, (uint32_t)x.b));
                        b1 = min(b1, max((uint32_t)y.a + d, (uint32_t)y.b));
                    }
                    if (j < m) {
                        const Pair2<A> x = EL[j];
                        b0 = min(b0, max((uint32_t)x.a + d, (uint32_t)x.b));
                    }
                }
                uint32_t best = min(b0, b1);
#pragma unroll
                for (int off = GL / 2; off > 0; off >>= 1) best = min(best, __shfl_xor_sync(FULL, best, off));
                bj = best & jmask;
            } else if (lanepk) {
                // lane-local keys (v << kb | k) for bucket j = gl + GL*k: one fused add-max per
                // bucket as in the packed variant; the key minimum orders (v, k), and a tie of
                // (v, k) across lanes goes to the lowest lane (ballot) -- the lowest j
                const uint32_t d = ((((uint32_t)it.e - (uint32_t)it.l) << ush) & (uint32_t)use) + co;
                uint32_t b0 = 0xFFFFFFFFu, b1 = 0xFFFFFFFFu;
                uint32_t j = gl;
#pragma unroll 4
                for (; j + GL < m; j += 2 * GL) {
                    const Pair2<A> x = EL[j], y = EL[j + GL];
                    b0 = min(b0, max((uint32_t)x.a + d, (uint32_t)x.b));
                    b1 = min(b1, max((uint32_t)y.a + d, (uint32_t)y.b));
                }
                if (j < m) {
                    const Pair2<A> x = EL[j];
                    b0 = min(b0, max((uint32_t)x.a + d, (uint32_t)x.b));
                }
                const uint32_t mine = min(b0, b1);
                uint32_t best = mine;
#pragma unroll
                for (int off = GL / 2; off > 0; off >>= 1) best = min(best, __shfl_xor_sync(FULL, best, off));
                const uint32_t bal = __ballot_sync(FULL, mine == best);
                const uint32_t gbits = GL == 32 ? bal : (bal >> (lane & ~(uint32_t)(GL - 1))) & ((1u << (GL & 31)) - 1u);
                bj = (uint32_t)(__ffs(gbits) - 1) + GL * (best & ((1u << ush) - 1u));
            } else {
                const A ae = it.e & use, al = it.l & use;
                A bv = amax<A>();
                bj = 0xFFFFFFFFu;
#pragma unroll 4
                for (uint32_t j = gl; j < m; j += GL) {
                    const Pair2<A> el = EL[j];
                    const A v = maxa<A>(el.a + ae, el.b + al);
                    if (v < bv) {
                        bv = v;
                        bj = j;
                    }
                }
                argmin_reduce<A, GL>(bv, bj, FULL);
            }
            // during LPT bucket j is read and written only by its owner lane j % GL, so the
            // update needs no warp barrier (the shuffles already order the lanes)
            if ((bj & (GL - 1)) == gl) {
                Pair2<A> el = EL[bj];
                el.a += it.e << ush;
                el.b += it.l << ush;
                EL[bj] = el;  // FL: formed by the first build_lists (or fl_sums for m == 1)
                if (stg)
                    sts_u8(stage_s + (pos - start), bj);
                else
                    set_apos(apos, pos, bj, wide);
            }
        }
        if (stg) flush_stage<GL>(apos, stage_s, start, ng, gl);
      }
    }
    __syncwarp(FULL);
}

// Ascending bitonic sort of 64 keys held KPL = 64 / GL per lane by the GL lanes of a group
// (element e = KPL * gl + t): in-register compare-exchanges below distance KPL, lane
// exchanges (xor shuffles inside the group) above it.  All lanes of the warp take part.
template <int GL, int KPL>
DFLOP_DEV void bitonic_sort64(uint32_t (&key)[KPL], uint32_t gl) {
#pragma unroll
    for (uint32_t k = 2; k <= 64; k <<= 1) {
#pragma unroll
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            if (j < (uint32_t)KPL) {
#pragma unroll
                for (uint32_t t = 0; t < (uint32_t)KPL; ++t) {
                    if ((t & j) == 0) {
                        const bool asc = ((KPL * gl + t) & k) == 0;
                        const uint32_t x = key[t], y = key[t ^ j];
                        const uint32_t lo = min(x, y), hi = max(x, y);
                        key[t] = asc ? lo : hi;
                        key[t ^ j] = asc ? hi : lo;
                    }
                }
            } else {
                const uint32_t lx = j / KPL;
                const bool lower = (gl & lx) == 0;
#pragma unroll
                for (uint32_t t = 0; t < (uint32_t)KPL; ++t) {
                    const bool asc = ((KPL * gl + t) & k) == 0;
                    const uint32_t o = __shfl_xor_sync(FULL, key[t], lx);
                    key[t] = (lower == asc) ? min(key[t], o) : max(key[t], o);
                }
            }
        }
    }
}

// ---------------------------------------------------------------- swap refinement (O6)
// `apply` is false for c < 2: the rounds are still executed (and discarded) so that every
// group of a warp issues the same shuffle sequence.
// CS: the counters are known to be in shared memory (the split kernel: m <= 255) -- shared
// atomics instead of generic ones
template <typename A, bool PK, int GL, bool SM, bool CS = false>
DFLOP_DEV void refine(const CandParams& p, const Tbl<A, SM>& T, uint32_t c, uint32_t sh, Pair2<A>* EL, Pair2<A>* FL,
                      uint8_t* apos, uint8_t* scr, uint16_t* csr, uint32_t gl, bool apply, PhaseTimer& ph) {
    const uint32_t m = p.m, cap = p.cap;
    const bool wide = p.wide != 0;  // u16 assignment when m > 255
    // cnt[m] members per bucket, off[m + 1] list starts: in shared memory (m <= 256), else
    // in front of the slot's global lists; then the shared-memory copies of the first cap
    // members of j* (ls) and j' (lp)
    // the split kernel (CS) keeps the list offsets as u16 (n + m * sigma < 65536 there)
    using OT = std::conditional_t<CS, uint16_t, uint32_t>;
    uint32_t* cnt;
    uint16_t* ls;
    OT* off;
    if (CS) {
        cnt = reinterpret_cast<uint32_t*>(scr);
        off = reinterpret_cast<OT*>(cnt + m);
        ls = reinterpret_cast<uint16_t*>(scr + 4u * m + ((2u * m + 2u + 3u) & ~3u));
    } else if (p.cnt_smem) {
        cnt = reinterpret_cast<uint32_t*>(scr);
        off = reinterpret_cast<OT*>(cnt + m);
        ls = reinterpret_cast<uint16_t*>(cnt + 2 * m + 1);
    } else {
        cnt = reinterpret_cast<uint32_t*>(csr);
        off = reinterpret_cast<OT*>(cnt + m);
        csr += 2 * (2 * m + 1);
        ls = reinterpret_cast<uint16_t*>(scr);
    }
    uint16_t* lp = ls + cap;
    // SRT (split kernel, 32-bit sums, table in shared memory, n <= 4096): j''s members are
    // sorted by their load in the narrower of the two dimensions and each row scans only the
    // window of partners that could bring the pair below W* (DESIGN.md section 6); the sorted
    // keys (load with the low 12 bits replaced by the position) follow the row copy
    constexpr bool SRT = CS && SM && sizeof(A) == 4 && GL >= 8;
    uint32_t* sk = reinterpret_cast<uint32_t*>(scr + ((4u * m + ((2u * m + 2u + 3u) & ~3u) + 2u * cap + 15u) & ~15u));
    bool dirty = true;  // the lists must be (re)built from the assignment
    bool first = true;  // the first build also forms FL (LPT maintains EL only)
    for (uint32_t r = 0; r < p.R; ++r) {
        if (__any_sync(FULL, dirty)) {  // warp-uniform: a clean group rebuilds the same lists
            build_lists<A, GL, SM, OT>(p, T, apos, wide, cnt, off, csr, gl, first ? FL : nullptr);
            dirty = false;
            first = false;
        }
        // bottleneck bucket j* = lowest j with maximal W_j = max(E_j, L_j)
        A Wb = 0;
        uint32_t jb = 0xFFFFFFFFu;
        if constexpr (PK) {
            // packed keys: (W << s) | (jmask - j) -- one max per bucket and per reduction
            // round gives the largest W and, among equal W, the lowest j
            const uint32_t jmask = (1u << sh) - 1u;
            uint32_t kb = 0;
            for (uint32_t j = gl; j < m; j += GL) {
                const Pair2<A> el = EL[j];
                kb = max(kb, (uint32_t)keyval<A, PK>(maxa(el.a, el.b), sh) | (jmask - j));
            }
#pragma unroll
            for (int o = GL / 2; o > 0; o >>= 1) kb = max(kb, __shfl_xor_sync(FULL, kb, o));
            Wb = (A)(kb & ~jmask);
            jb = jmask - (kb & jmask);
        } else {
            for (uint32_t j = gl; j < m; j += GL) {
                const Pair2<A> el = EL[j];
                const A W = keyval<A, PK>(maxa(el.a, el.b), sh);
                if (jb == 0xFFFFFFFFu || W > Wb) {
                    Wb = W;
                    jb = j;
                }
            }
            argmax_reduce<A, GL>(Wb, jb, FULL);
        }
        const uint32_t js = jb;
        const A Ws = Wb;
        const Philox4 w = philox4x32_10(r, c, 1u, 0u, p.seed0, p.seed1);
        const uint32_t jp = (js + 1u + mulhi32(w.x, m - 1u)) % m;
        const Pair2<A> Bsp = EL[js], Bpp = EL[jp];
        const Pair2<A> Bs{keyval<A, PK>(Bsp.a, sh), keyval<A, PK>(Bsp.b, sh)};
        const Pair2<A> Bp{keyval<A, PK>(Bpp.a, sh), keyval<A, PK>(Bpp.b, sh)};
        ph.mark(1);
        // member lists of j* (gss) and j' (gsp); their first cap entries are copied to
        // shared memory (ls, lp), the rest is read from L2
        const uint32_t nA = cnt[js], nB = cnt[jp];
        uint16_t* gss = csr + off[js];
        uint16_t* gsp = csr + off[jp];
        {
            const uint32_t na = min(nA, cap), nb = min(nB, cap);
            for (uint32_t u = gl; u < na; u += GL) ls[u] = __ldcg(gss + u);
            if (!SRT)
                for (uint32_t u = gl; u < nb; u += GL) lp[u] = __ldcg(gsp + u);
        }
        __syncwarp(FULL);
        ph.mark(2);
        A bsc = amax<A>();
        uint32_t bi = 0xFFFFFFFFu, brk = 0xFFFFFFFFu, vstar = 0xFFFFFFFFu;
        u64 bkey = ~0ull;  // 32-bit scores: (row minimum << 32 | item), branch-free minima
        uint32_t ubest = 0;  // ... and the j* list index of the lane's best row
        // all (i, i') with i in j*, i' in {NONE} u j'; lexicographic min of (score, i, rank(i'))
        // two j* members per lane and step: every j' member loaded once serves two pairs
        auto ival = [&](uint32_t u, uint32_t& ii, A& se, A& sl, A& pe, A& pl) {
            const uint32_t pi = u < cap ? (uint32_t)ls[u] : (uint32_t)__ldcg(gss + u);
            const Pair2<A> a = T.el(pi);
            ii = T.idx(pi);
            se = Bs.a - a.a;  // j* without i
            sl = Bs.b - a.b;
            pe = Bp.a + a.a;  // j' with i
            pl = Bp.b + a.b;
        };
        // j''s members in chunks of cap: each chunk copied to shared memory (the first above)
        // and paired with every row; the row minima fold into bkey chunk by chunk (the NONE
        // pair in every chunk: idempotent)
        const bool one_chunk = !SRT && nB <= cap;  // phase 2 / apply may read the copy
        if constexpr (SRT) {
            // A pair can bring j* below W* only if all four loads drop below it: x' in
            // (pe - W*, W* - se) for the partner's e (x' = a) and (pl - W*, W* - sl) for its l --
            // a window of width 2W* - E*(j*) - E*(j') (resp. L), the same for every row.  The
            // other pairs cannot win (the move needs a score below W*), so each row scores only
            // the partners inside its window of the narrower dimension (and the NONE pair).
            constexpr uint32_t KPL = 64u / GL;
            const u64 wE = (u64)(Ws - Bs.a) + (u64)(Ws - Bp.a), wL = (u64)(Ws - Bs.b) + (u64)(Ws - Bp.b);
            const bool dimE = wE <= wL;
            for (uint32_t p0 = 0;; p0 += 64) {  // chunks of 64 partners
                const uint32_t nb = p0 < nB ? min(64u, nB - p0) : 0u;
                uint32_t key[KPL];
#pragma unroll
                for (uint32_t t = 0; t < KPL; ++t) {
                    const uint32_t v = KPL * gl + t;
                    key[t] = 0xFFFFFFFFu;
                    if (v < nb) {
                        const uint32_t pos = __ldcg(gsp + p0 + v);
                        const Pair2<A> b = T.el(pos);
                        key[t] = ((uint32_t)(dimE ? b.a : b.b) & ~0xFFFu) | pos;
                    }
                }
                bitonic_sort64<GL, KPL>(key, gl);
#pragma unroll
                for (uint32_t t = 0; t < KPL; ++t) sk[KPL * gl + t] = key[t];
                __syncwarp(FULL);
                for (uint32_t u = gl; u < nA && (p0 == 0 || nb > 0); u += GL) {
                    const uint32_t pi = u < cap ? (uint32_t)ls[u] : (uint32_t)__ldcg(gss + u);
                    const Pair2<A> a = T.el(pi);
                    const uint32_t ii = T.idx(pi);
                    const uint32_t se = (uint32_t)(Bs.a - a.a), sl = (uint32_t)(Bs.b - a.b);
                    const uint32_t pe = (uint32_t)(Bp.a + a.a), pl = (uint32_t)(Bp.b + a.b);
                    uint32_t rr = max(max(se, sl), max(pe, pl));  // NONE
                    const uint32_t W = (uint32_t)Ws, lo_t = dimE ? pe : pl, hi_t = dimE ? se : sl;
                    const uint32_t qlo = lo_t < W ? 0u : ((lo_t - W + 1u) & ~0xFFFu);  // x' > lo_t - W*
                    const uint32_t hi = W - hi_t;                                       // x' < hi
                    const uint32_t qhi = (hi - 1u) & ~0xFFFu;
                    const uint32_t limit = hi == 0u ? 0u : (qhi >= 0xFFFFF000u ? 0xFFFFFFFFu : qhi + 0x1000u);
                    uint32_t k = 0;
#pragma unroll
                    for (uint32_t st = 32; st > 0; st >>= 1)
                        if (sk[k + st - 1] < qlo) k += st;
                    for (; k < nb && sk[k] < limit; ++k) {
                        const Pair2<A> b = T.el(sk[k] & 0xFFFu);
                        rr = min(rr, score4(se, sl, pe, pl, (uint32_t)b.a, (uint32_t)b.b));
                    }
                    const u64 kk = pack64(rr, ii);
                    if (kk < bkey) {
                        bkey = kk;
                        ubest = u;
                    }
                }
                if (!__any_sync(FULL, p0 + 64 < nB)) break;  // warp-uniform
                __syncwarp(FULL);
            }
        } else {
        for (uint32_t p0 = 0;;) {
        const uint32_t nBs = p0 < nB ? min(cap, nB - p0) : 0u;
        for (uint32_t u = gl; u < nA && (p0 == 0 || nBs > 0); u += 2 * GL) {
            uint32_t i0, i1;
            A se0, sl0, pe0, pl0, se1, sl1, pe1, pl1;
            ival(u, i0, se0, sl0, pe0, pl0);
            if (u + GL < nA) {
                ival(u + GL, i1, se1, sl1, pe1, pl1);
            } else {  // duplicate of the first: same keys, no effect on the minimum
                i1 = i0;
                se1 = se0;
                sl1 = sl0;
                pe1 = pe0;
                pl1 = pl0;
            }
            const A n0 = maxa(maxa(se0, sl0), maxa(pe0, pl0)), n1 = maxa(maxa(se1, sl1), maxa(pe1, pl1));
            // 32-bit scores, phase 1: per row only the minimum score (the NONE pair included);
            // the rank of the winning partner is found afterwards for the one winning row
            uint32_t r0 = (uint32_t)n0, r1 = (uint32_t)n1;
            if (sizeof(A) != 4) {
                lex_update(bsc, bi, brk, n0, i0, 0u);
                lex_update(bsc, bi, brk, n1, i1, 0u);
            }
            auto pair = [&](uint32_t pj) {
                const Pair2<A> b = T.el(pj);
                if (sizeof(A) == 4) {
                    // the same four-term maximum as one chain of fused add-max (DPX): every
                    // term is a non-negative load below 2^32, so the wrapping -b.a is exact
                    r0 = min(r0, score4((uint32_t)se0, (uint32_t)sl0, (uint32_t)pe0, (uint32_t)pl0, (uint32_t)b.a,
                                        (uint32_t)b.b));
                    r1 = min(r1, score4((uint32_t)se1, (uint32_t)sl1, (uint32_t)pe1, (uint32_t)pl1, (uint32_t)b.a,
                                        (uint32_t)b.b));
                } else {
                    const A s0 = maxa(maxa<A>(se0 + b.a, sl0 + b.b), maxa<A>(pe0 - b.a, pl0 - b.b));
                    const A s1 = maxa(maxa<A>(se1 + b.a, sl1 + b.b), maxa<A>(pe1 - b.a, pl1 - b.b));
                    const uint32_t rk = T.idx(pj) + 1u;
                    lex_update(bsc, bi, brk, s0, i0, rk);
                    lex_update(bsc, bi, brk, s1, i1, rk);
                }
            };
            uint32_t v = 0;
            for (; v + 4 <= nBs; v += 4) {
                const uint32_t q0 = lp[v], q1 = lp[v + 1], q2 = lp[v + 2], q3 = lp[v + 3];
                pair(q0);
                pair(q1);
                pair(q2);
                pair(q3);
            }
            for (; v < nBs; ++v) pair(lp[v]);
            if (sizeof(A) == 4) {  // (row minimum, item): lexicographic over the lane's rows
                const u64 k0 = pack64(r0, i0), k1 = pack64(r1, i1);
                if (k0 < bkey) {
                    bkey = k0;
                    ubest = u;
                }
                if (k1 < bkey) {  // (a duplicated first row ties, never below)
                    bkey = k1;
                    ubest = u + GL;
                }
            }
        }
        p0 += cap;
        if (!__any_sync(FULL, p0 < nB)) break;  // warp-uniform
        __syncwarp(FULL);
        {
            const uint32_t nb = p0 < nB ? min(cap, nB - p0) : 0u;
            for (uint32_t u = gl; u < nb; u += GL) lp[u] = __ldcg(gsp + p0 + u);
        }
        __syncwarp(FULL);
        }
        }
        ph.mark(3);
        uint32_t ustar = 0, pistar = 0;  // the winning row: j* list index and position (32-bit)
        if (sizeof(A) == 4) {
            const u64 mine = bkey;
#pragma unroll
            for (int off = GL / 2; off > 0; off >>= 1) bkey = min(bkey, __shfl_xor_sync(FULL, bkey, off));
            {  // the lane holding the winning row (keys are unique: one lane) broadcasts its index
                const uint32_t gbase = (threadIdx.x & 31u) & ~(uint32_t)(GL - 1);
                const uint32_t bal = __ballot_sync(FULL, mine == bkey);
                const uint32_t gm = GL == 32 ? bal : (bal >> gbase) & ((1u << (GL & 31)) - 1u);
                ustar = __shfl_sync(FULL, ubest, gbase + (gm ? (uint32_t)(__ffs(gm) - 1) : 0u));
            }
            // phase 2 (only when the move would be applied): the least rank among the partners
            // of the winning row that reach the minimum -- the same lexicographic minimum
            // (score, i, rank) as one pass over 64-bit keys
            const bool need = apply && bkey != ~0ull && (A)(bkey >> 32) < Ws;
            if (__any_sync(FULL, need)) {  // warp-uniform (the reduction below shuffles)
                const uint32_t S = (uint32_t)(bkey >> 32), istar = (uint32_t)bkey;
                // (rank << 32 | list index v): the apply step edits entry v of j''s list directly
                u64 rv = ~0ull;
                if (need) {
                    pistar = ustar < cap ? (uint32_t)ls[ustar] : (uint32_t)__ldcg(gss + ustar);
                    const Pair2<A> a = T.el(pistar);
                    const A se = Bs.a - a.a, sl = Bs.b - a.b, pe = Bp.a + a.a, pl = Bp.b + a.b;
                    if (gl == 0 && (uint32_t)maxa(maxa(se, sl), maxa(pe, pl)) == S) rv = 0xFFFFFFFFull;
                    for (uint32_t v = gl; v < nB; v += GL) {
                        const uint32_t pj = (v < cap && one_chunk) ? (uint32_t)lp[v] : (uint32_t)__ldcg(gsp + v);
                        const Pair2<A> b = T.el(pj);
                        const A sc = maxa(maxa<A>(se + b.a, sl + b.b), maxa<A>(pe - b.a, pl - b.b));
                        if ((uint32_t)sc == S) rv = min(rv, ((u64)(T.idx(pj) + 1u) << 32) | v);
                    }
                }
#pragma unroll
                for (int off = GL / 2; off > 0; off >>= 1) rv = min(rv, __shfl_xor_sync(FULL, rv, off));
                if (need) {
                    bsc = (A)S;
                    bi = istar;
                    brk = (uint32_t)(rv >> 32);
                    vstar = (uint32_t)rv;
                }
            }
        } else {
            lexmin_reduce<A, GL>(bsc, bi, brk, FULL);
        }
        if (apply && bi != 0xFFFFFFFFu && bsc < Ws) {  // uniform in the group (reduced values)
            // 32-bit: the winning row and partner are known by their list indices (ustar, vstar)
            uint32_t pi, pj;
            if (sizeof(A) == 4) {
                pi = pistar;
                pj = brk != 0u ? ((vstar < cap && one_chunk) ? (uint32_t)lp[vstar] : (uint32_t)__ldcg(gsp + vstar))
                               : 0xFFFFFFFFu;
            } else {
                pi = __ldg(p.item_pos + bi);
                pj = brk != 0u ? __ldg(p.item_pos + (brk - 1u)) : 0xFFFFFFFFu;
            }
            // a move adds a member to j': it needs a free entry, else the lists are rebuilt
            const bool fits = brk != 0u || nB < off[jp + 1] - off[jp];
            if (fits && sizeof(A) == 4) {  // i leaves j*'s list (replaced by i', or by the last member)
                if (gl == 0) {
                    const uint32_t last = nA - 1u < cap ? (uint32_t)ls[nA - 1u] : (uint32_t)__ldcg(gss + nA - 1u);
                    gss[ustar] = (uint16_t)(brk != 0u ? pj : last);
                    if (brk != 0u) {  // i' leaves j''s list (entry vstar), i takes it
                        gsp[vstar] = (uint16_t)pi;
                    } else {
                        gsp[nB] = (uint16_t)pi;
                        cnt[js] = nA - 1u;
                        cnt[jp] = nB + 1u;
                    }
                }
            } else if (fits) {
                for (uint32_t u = gl; u < nA; u += GL) {
                    const uint32_t q = u < cap ? (uint32_t)ls[u] : (uint32_t)__ldcg(gss + u);
                    if (q == pi) {
                        const uint32_t last = nA - 1u < cap ? (uint32_t)ls[nA - 1u] : (uint32_t)__ldcg(gss + nA - 1u);
                        gss[u] = (uint16_t)(brk != 0u ? pj : last);
                    }
                }
                if (brk != 0u) {
                    for (uint32_t v = gl; v < nB; v += GL) {
                        const uint32_t q = (v < cap && one_chunk) ? (uint32_t)lp[v] : (uint32_t)__ldcg(gsp + v);
                        if (q == pj) gsp[v] = (uint16_t)pi;
                    }
                } else if (gl == 0) {
                    gsp[nB] = (uint16_t)pi;
                    cnt[js] = nA - 1u;
                    cnt[jp] = nB + 1u;
                }
            } else {
                dirty = true;
            }
            if (gl == 0) {
                const ItemRec<A> a = T.item(pi);
                const A ae = a.e, al = a.l;
                Pair2<A> es = EL[js], fs = FL[js], ep = EL[jp], fp = FL[jp];
                es.a -= ae; es.b -= al; fs.a -= a.ef; fs.b -= a.lf;
                ep.a += ae; ep.b += al; fp.a += a.ef; fp.b += a.lf;
                set_apos(apos, pi, jp, wide);
                if (brk != 0u) {
                    const ItemRec<A> b = T.item(pj);
                    const A be = b.e, bl = b.l;
                    ep.a -= be; ep.b -= bl; fp.a -= b.ef; fp.b -= b.lf;
                    es.a += be; es.b += bl; fs.a += b.ef; fs.b += b.lf;
                    set_apos(apos, pj, js, wide);
                }
                EL[js] = es;
                FL[js] = fs;
                EL[jp] = ep;
                FL[jp] = fp;
            }
        }
        __syncwarp(FULL);
        ph.mark(4);
    }
}

// ---------------------------------------------------------------- 1F1B score (O7)
// Replica rho runs buckets j = k*L_dp + rho as slots k (R10); stages < E_pp take (EF, E-EF),
// the rest (LF, L-LF) (R7).  The host-built topological order is grouped in Kahn levels;
// the GL lanes of the group run the ops of one level concurrently (distinct stages), rings
// of depth D carry the end times between stages.
template <typename A, bool PK, int GL, typename Map>
DFLOP_DEV u64 score_replica(const CandParams& p, uint32_t sh, const Pair2<A>* EL, const Pair2<A>* FL, u64* scr,
                            uint32_t gl, uint32_t rho, Map&& slot_of) {
    const uint32_t S = p.S, D = p.D, Dm = p.D - 1;
    u64* last = scr;
    u64* FR = scr + S;
    u64* BR = FR + S * D;
    for (uint32_t s = gl; s < S; s += GL) last[s] = 0;
    __syncwarp(FULL);
    uint32_t q0 = __ldg(p.levels);
    for (uint32_t L = 0; L < p.n_levels; ++L) {
        const uint32_t q1 = __ldg(p.levels + L + 1);
        for (uint32_t q = q0 + gl; q < q1; q += GL) {
            const uint32_t op = __ldg(p.ops + q);
            const uint32_t kind = op_kind(op), s = op_stage(op), k = op_mb(op);
            const uint32_t j = slot_of(k) * p.l_dp + rho;
            const Pair2<A> el = EL[j], fl = FL[j];
            const bool enc = s < p.e_pp;
            u64 dur, dep = 0;
            if (kind == 0) {
                dur = enc ? (u64)fl.a : (u64)fl.b;
                if (s > 0) dep = FR[(s - 1) * D + (k & Dm)];
            } else {
                dur = enc ? (u64)(unpack<A, PK>(el.a, sh) - fl.a) : (u64)(unpack<A, PK>(el.b, sh) - fl.b);
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
        q0 = q1;
        __syncwarp(FULL);
    }
    u64 t = 0;
    for (uint32_t s = gl; s < S; s += GL) t = last[s] > t ? last[s] : t;
    t = max_reduce<u64, GL>(t, FULL);
    __syncwarp(FULL);
    return t;
}

// The same evaluation with each lane owning stages gl and gl + GL (S <= 2 GL): the level-dense
// program gives every stage its op at each level (or none), the stage's running end time stays
// in a register, the next level's op codes are fetched one level ahead, and the per-stage ring
// addresses are fixed per lane -- a level is one branch-free op per stage: its bucket sums, its
// dependency from the neighbour's ring, max/add, one ring store.
template <typename A, bool PK>
struct StageLane {
    u64 last;          // end time of the stage's latest op
    u64* fr_dep;       // F dependency ring (stage s-1; s = 0: own ring, masked)
    u64* br_dep;       // B dependency ring (stage s+1; last stage: its own F ring)
    u64* fr_own;
    u64* br_own;
    bool enc, has_fdep;
};

template <typename A, bool PK>
DFLOP_DEV void stage_lane_init(StageLane<A, PK>& L, uint32_t s, uint32_t S, uint32_t D, uint32_t e_pp, u64* FR, u64* BR) {
    L.last = 0;
    L.enc = s < e_pp;
    L.has_fdep = s > 0;
    L.fr_own = FR + (size_t)s * D;
    L.br_own = BR + (size_t)s * D;
    L.fr_dep = s > 0 ? FR + (size_t)(s - 1) * D : L.fr_own;
    L.br_dep = s + 1 < S ? BR + (size_t)(s + 1) * D : L.fr_own;
}

template <typename A, bool PK>
DFLOP_DEV void stage_lane_op(StageLane<A, PK>& L, uint32_t op, const Pair2<A>* EL, const Pair2<A>* FL, uint32_t l_dp,
                             uint32_t rho, uint32_t sh, uint32_t Dm) {
    const bool act = op != kNoOpDev;
    const uint32_t kind = op >> 31, k = act ? (op & 0xFFFFu) : 0u;
    const uint32_t j = k * l_dp + rho;
    const Pair2<A> el = EL[j], fl = FL[j];
    const A fdur = L.enc ? fl.a : fl.b;
    const A bdur = L.enc ? (A)(unpack<A, PK>(el.a, sh) - fl.a) : (A)(unpack<A, PK>(el.b, sh) - fl.b);
    const u64 dur = kind ? (u64)bdur : (u64)fdur;
    const uint32_t slot = k & Dm;
    u64 dep = (kind ? L.br_dep : L.fr_dep)[slot];
    dep = (kind || L.has_fdep) ? dep : 0ull;
    const u64 end = (L.last > dep ? L.last : dep) + dur;
    if (act) {
        L.last = end;
        (kind ? L.br_own : L.fr_own)[slot] = end;
    }
}

template <typename A, bool PK, int GL>
DFLOP_DEV u64 score_replica_ls(const CandParams& p, uint32_t sh, const Pair2<A>* EL, const Pair2<A>* FL, u64* scr,
                               uint32_t gl, uint32_t rho) {
    const uint32_t S = p.S, D = p.D, Dm = p.D - 1, NL = p.n_levels, l_dp = p.l_dp;
    u64* FR = scr + S;  // same layout as score_replica (ORDER4's slot orders follow the rings)
    u64* BR = FR + S * D;
    const uint32_t s0 = gl, s1 = gl + GL;
    const bool has0 = s0 < S, has1 = s1 < S;
    StageLane<A, PK> L0, L1;
    stage_lane_init(L0, has0 ? s0 : 0, S, D, p.e_pp, FR, BR);
    stage_lane_init(L1, has1 ? s1 : 0, S, D, p.e_pp, FR, BR);
    const uint32_t* dn = p.dense;
    uint32_t n0 = has0 ? __ldg(dn + s0) : kNoOpDev;
    uint32_t n1 = has1 ? __ldg(dn + s1) : kNoOpDev;
    const bool any1 = __any_sync(FULL, has1);  // warp-uniform
    for (uint32_t lv = 0; lv < NL; ++lv) {
        const uint32_t c0 = n0, c1 = n1;
        if (lv + 1 < NL) {  // next level's ops: independent of this level's results
            dn += S;
            n0 = has0 ? __ldg(dn + s0) : kNoOpDev;
            n1 = has1 ? __ldg(dn + s1) : kNoOpDev;
        }
        stage_lane_op(L0, c0, EL, FL, l_dp, rho, sh, Dm);
        if (any1) stage_lane_op(L1, c1, EL, FL, l_dp, rho, sh, Dm);
        __syncwarp(FULL);
    }
    u64 t = L0.last > L1.last ? L0.last : L1.last;
    t = max_reduce<u64, GL>(t, FULL);
    __syncwarp(FULL);
    return t;
}

template <typename A, bool PK, int GL>
DFLOP_DEV u64 score_1f1b(const CandParams& p, uint32_t sh, const Pair2<A>* EL, const Pair2<A>* FL, u64* scr,
                         uint32_t gl) {
    u64 T = 0;
    const bool ls = p.dense != nullptr && p.S <= 2 * GL;  // uniform
    for (uint32_t rho = 0; rho < p.l_dp; ++rho) {
        const u64 t = ls ? score_replica_ls<A, PK, GL>(p, sh, EL, FL, scr, gl, rho)
                         : score_replica<A, PK, GL>(p, sh, EL, FL, scr, gl, rho, [](uint32_t k) { return k; });
        T = t > T ? t : T;
    }
    return T;
}

// N4(a) per candidate (DFLOP_MODE_ORDER4, R37): each replica under its best of the four start
// orders of the order search (slot order, W = max(E, L) ascending, descending, valley); the
// orders come from rank counts over the replica's slots (ties by slot, as the stable sorts
// of orc_order_search).  Only in the O4 instantiations of the kernel.
template <typename A, bool PK, int GL>
DFLOP_DEV u64 score_order4(const CandParams& p, uint32_t sh, const Pair2<A>* EL, const Pair2<A>* FL,
                                        u64* scr, uint32_t gl) {
    const uint32_t M = p.n_mb, half = (M + 1) / 2;
    uint16_t* asc = reinterpret_cast<uint16_t*>(scr + (p.S + 2 * p.S * p.D));
    uint16_t* desc = asc + M;
    auto W = [&](uint32_t k, uint32_t rho) {
        const Pair2<A> el = EL[k * p.l_dp + rho];
        return unpack<A, PK>(maxa(el.a, el.b), sh);
    };
    u64 T = 0;
    for (uint32_t rho = 0; rho < p.l_dp; ++rho) {
        for (uint32_t k = gl; k < M; k += GL) {
            const A wk = W(k, rho);
            uint32_t ra = 0, rd = 0;
            for (uint32_t k2 = 0; k2 < M; ++k2) {
                const A w2 = W(k2, rho);
                ra += (w2 < wk || (w2 == wk && k2 < k)) ? 1u : 0u;
                rd += (w2 > wk || (w2 == wk && k2 < k)) ? 1u : 0u;
            }
            asc[ra] = (uint16_t)k;
            desc[rd] = (uint16_t)k;
        }
        __syncwarp(FULL);
        u64 t = score_replica<A, PK, GL>(p, sh, EL, FL, scr, gl, rho, [](uint32_t k) { return k; });
        u64 t1 = score_replica<A, PK, GL>(p, sh, EL, FL, scr, gl, rho, [&](uint32_t k) { return (uint32_t)asc[k]; });
        t = t1 < t ? t1 : t;
        t1 = score_replica<A, PK, GL>(p, sh, EL, FL, scr, gl, rho, [&](uint32_t k) { return (uint32_t)desc[k]; });
        t = t1 < t ? t1 : t;
        t1 = score_replica<A, PK, GL>(p, sh, EL, FL, scr, gl, rho,
                                      [&](uint32_t k) { return (uint32_t)asc[k < half ? 2 * k : 2 * (M - 1 - k) + 1]; });
        t = t1 < t ? t1 : t;
        T = t > T ? t : T;
        __syncwarp(FULL);
    }
    return T;
}

template <typename A, bool PK, int GL, bool SM, bool O4, int MODE>
DFLOP_DEV void run_candidate(const CandParams& p, const Tbl<A, SM>& T, uint32_t c, uint32_t sh, uint32_t co, Pair2<A>* EL,
                             Pair2<A>* FL, uint8_t* apos, uint8_t* scr, uint16_t* csr, uint32_t gl, u64& Tc,
                             u64& cmax, PhaseTimer& ph, bool forced, uint32_t ent = 0) {
    const uint32_t m = p.m;
    if constexpr (MODE != 0) {
        // split pipeline: k_lpt left this candidate's packed bucket keys (offset removed) and
        // its assignment; the caller copied the assignment into apos
        const uint2* src = reinterpret_cast<const uint2*>(p.lpt_el) + (size_t)ent * m;  // k_lpt's entry
        for (uint32_t j = gl; j < m; j += GL) {
            const uint2 v = __ldcg(src + j);
            EL[j] = Pair2<A>{(A)v.x, (A)v.y};
            FL[j] = Pair2<A>{0, 0};
        }
        __syncwarp(FULL);
        ph.mark(0);
        if (m >= 2 && p.R > 0)
            refine<A, PK, GL, SM, true>(p, T, c, sh, EL, FL, apos, scr, csr, gl, c >= 2, ph);
        else
            form_fl<A, GL, SM>(p, T, apos, p.wide != 0, FL, gl);
    } else {
    for (uint32_t j = gl; j < m; j += GL) {
        // co: the LPT probe offset; the plain variant's lane-local LPT keys carry k = j / GL
        EL[j] = PK ? Pair2<A>{(A)j, (A)(j + co)}
                   : (sh >= 0x100u ? Pair2<A>{(A)(j / GL), (A)(j / GL + co)} : Pair2<A>{0, 0});
        FL[j] = Pair2<A>{0, 0};
    }
    __syncwarp(FULL);
    if (p.exhaustive) {
        // candidate c = base-m digits: a_i = floor(c / m^i) mod m (never packed)
        if (gl == 0) {
            uint32_t x = c;
            for (uint32_t i = 0; i < p.n; ++i) {
                const uint32_t d = x % m;
                x /= m;
                const uint32_t pos = __ldg(p.item_pos + i);
                const ItemRec<A> it = T.item(pos);
                EL[d].a += it.e;
                EL[d].b += it.l;
                FL[d].a += it.ef;
                FL[d].b += it.lf;
                set_apos(apos, pos, d, p.wide != 0);
            }
        }
        __syncwarp(FULL);
    } else {
        lpt_pass<A, PK, GL, SM>(p, T, c, sh, EL, FL, apos, scr, gl, co, forced);
        if (PK) {  // drop the probe offset: plain packed keys from here on
            for (uint32_t j = gl; j < m; j += GL) EL[j].b -= (A)co;
            __syncwarp(FULL);
        } else if (sh >= 0x100u) {  // lane-local LPT keys -> plain sums
            for (uint32_t j = gl; j < m; j += GL)
                EL[j] = Pair2<A>{(A)(EL[j].a >> (sh & 0xFFu)), (A)((EL[j].b - co) >> (sh & 0xFFu))};
            __syncwarp(FULL);
        }
        ph.mark(0);
        if (m >= 2 && p.R > 0)
            refine<A, PK, GL, SM>(p, T, c, sh, EL, FL, apos, scr, csr, gl, c >= 2, ph);
        else
            form_fl<A, GL, SM>(p, T, apos, p.wide != 0, FL, gl);
    }
    }
    A cm = 0;
    for (uint32_t j = gl; j < m; j += GL) {
        const Pair2<A> el = EL[j];
        cm = maxa(cm, unpack<A, PK>(maxa(el.a, el.b), sh));
    }
    cmax = (u64)max_reduce<A, GL>(cm, FULL);
    ph.mark(6);
    if constexpr (O4)  // DFLOP_MODE_ORDER4: a separate kernel instantiation
        Tc = score_order4<A, PK, GL>(p, sh, EL, FL, reinterpret_cast<u64*>(scr), gl);
    else
        Tc = score_1f1b<A, PK, GL>(p, sh, EL, FL, reinterpret_cast<u64*>(scr), gl);
    ph.mark(5);
}

// MODE 0: the whole candidate (LPT, refinement, 1F1B); 1: the split pipeline's second kernel
// (from k_lpt's output: refinement + 1F1B; packed u32 only)
template <typename A, bool PK, int GL, bool SM, bool O4, int MODE = 0>
__global__ void __launch_bounds__(MODE != 0 ? kSplitMaxThreads : kCandMaxThreads) k_candidates(CandParams p) {
    if (p.hdr->variant != p.want_variant) return;  // another variant runs
    uint32_t sh = PK ? p.hdr->shift : 0u;
    uint32_t co = PK ? p.hdr->offs : 0u;  // LPT probe offset (lpt_pass)
    if constexpr (!PK && sizeof(A) == 4) {
        // plain 32-bit variant (the packed bound fails, e.g. m large): the LPT still runs on
        // packed keys when the bucket index local to a lane (k = j / GL, kb bits) fits --
        // the same bound as the packed variant with kb instead of s = bits(m - 1);
        // sh = 0x100 | kb marks it for lpt_pass, co = C << kb the probe offset
        const uint32_t q = (p.m + GL - 1) / GL;
        uint32_t kb = 0;
        while ((1u << kb) < q) ++kb;
        const u64 bound = (p.hdr->sum_e + p.hdr->sum_l + p.m - 1) / p.m + 2 * p.hdr->max_key + p.hdr->max_ld;
        if (!p.exhaustive && p.m > 0 && kb < 32 && bound < (1ull << (32 - kb))) {
            sh = 0x100u | kb;
            co = (uint32_t)(p.hdr->max_ld << kb);
        }
    }
    extern __shared__ __align__(128) uint8_t smem[];
    Tbl<A, SM> T;
    if (SM) {
        const uint32_t words = p.n * (uint32_t)sizeof(ItemRec<A>) / 16;
        for (uint32_t i = threadIdx.x; i < words; i += blockDim.x)
            reinterpret_cast<uint4*>(smem)[i] = __ldg(reinterpret_cast<const uint4*>(p.items) + i);
        uint16_t* pi16 = reinterpret_cast<uint16_t*>(smem + (size_t)p.n * sizeof(ItemRec<A>));
        for (uint32_t i = threadIdx.x; i < p.n; i += blockDim.x) pi16[i] = (uint16_t)__ldg(p.pos_item + i);
        __syncthreads();
        T.it = reinterpret_cast<const ItemRec<A>*>(smem);
        T.it_s = (uint32_t)__cvta_generic_to_shared(smem);
        T.pi16 = pi16;
        T.pi32 = nullptr;
    } else {
        T.it = reinterpret_cast<const ItemRec<A>*>(p.items);
        T.it_s = 0;
        T.pi16 = nullptr;
        T.pi32 = p.pos_item;
    }
    // forced first-m LPT decisions (lpt_pass): every item at base positions [0, m) has e > 0
    // and l > 0 (warp-uniform; the exhaustive mode has no LPT)
    bool forced = false;
    if (!p.exhaustive && p.m >= 1 && p.m <= p.n) {
        bool ok = true;
        for (uint32_t q = threadIdx.x & 31u; q < p.m; q += 32) {
            const Pair2<A> r = T.el(q);
            ok = ok && r.a != 0 && r.b != 0;
        }
        forced = __all_sync(FULL, ok);
    }
    const uint32_t grp = threadIdx.x / GL, gl = threadIdx.x % GL;
    const uint32_t cpb = blockDim.x / GL;
    uint8_t* base = smem + p.tbl_bytes + (size_t)grp * p.cand_bytes;
    Pair2<A>* EL = reinterpret_cast<Pair2<A>*>(base);
    Pair2<A>* FL = reinterpret_cast<Pair2<A>*>(base + p.off_fl);
    uint8_t* scr = base + p.off_scr;
    const uint32_t slot = blockIdx.x * cpb + grp;
    uint8_t* bufs = p.slot_apos + (size_t)slot * 2 * p.apos_bytes;
    uint16_t* csr = p.slot_csr + (size_t)slot * p.csr_len;
    // padding past n never matches a bucket (0xFF / 0xFFFF)
    const uint32_t used = p.n * (p.wide ? 2u : 1u);
    for (uint32_t b = used + gl; b < p.apos_bytes; b += GL) {
        bufs[b] = 0xFF;
        bufs[p.apos_bytes + b] = 0xFF;
    }
    __syncwarp(FULL);
    // the slot's best so far (k_init sets the keys to ~0): a launch continues the previous
    // launches' slots (the split pipeline runs the family in chunks)
    u64 best_key = p.slot_key[slot], best_T = 0, best_cmax = 0;
    uint32_t best_buf = 0;
    if (best_key != ~0ull) {
        best_T = p.slot_T[slot];
        best_cmax = p.slot_cmax[slot];
        best_buf = p.slot_buf[slot];
    }
    uint32_t cur = best_buf ^ 1u;
    PhaseTimer ph;
    ph.start(p.phase);
    // a full round hands candidates base + block * cpb + grp to the block's groups; a partial
    // last round hands base + grp * grid + block, so its candidates are spread over every SM
    // (a few warps each, at low contention) instead of filling a few SMs
    const uint32_t stride = gridDim.x * cpb;
    for (uint32_t base = p.c_begin; base < p.c_end; base += stride) {
        const uint32_t cc = base + (p.c_end - base >= stride ? blockIdx.x * cpb + grp : grp * gridDim.x + blockIdx.x);
        const bool valid = cc < p.c_end;
        if (!__any_sync(FULL, valid)) break;  // warp-uniform: every group of the warp is done
        const uint32_t c = valid ? cc : p.c_end - 1;  // tail groups recompute a real candidate
        uint8_t* apos = bufs + (size_t)cur * p.apos_bytes;  // never the best buffer
        if constexpr (MODE != 0) {  // the chunk's assignment from k_lpt into the slot's working buffer
            const uint4* src = reinterpret_cast<const uint4*>(p.lpt_apos + (size_t)(c - p.c_begin) * p.apos_bytes);
            uint4* dst = reinterpret_cast<uint4*>(apos);
            for (uint32_t b = gl; b < p.apos_bytes / 16; b += GL) dst[b] = __ldcg(src + b);
            __syncwarp(FULL);
        }
        u64 Tc, cmax;
        run_candidate<A, PK, GL, SM, O4, MODE>(p, T, c, sh, co, EL, FL, apos, scr, csr, gl, Tc, cmax, ph, forced,
                                                c - p.c_begin);
        Tc = __shfl_sync(FULL, Tc, 0, GL);
        u64 key;
        if (Tc >= (1ull << 40)) {
            if (gl == 0) atomicOr(&p.hdr->status, (uint32_t)DFLOP_DEV_MAKESPAN_OVERFLOW);
            key = (((1ull << 40) - 1) << 24) | (u64)(p.id_base + c);
        } else {
            key = (Tc << 24) | (u64)(p.id_base + c);
        }
        if (!valid) continue;
        if (gl == 0 && p.cand_T) {
            p.cand_T[c - p.c_begin] = Tc;
            p.cand_cmax[c - p.c_begin] = cmax;
        }
        if (key < best_key) {  // keep this buffer, write the next candidate into the other
            best_key = key;
            best_T = Tc;
            best_cmax = cmax;
            best_buf = cur;
            cur ^= 1u;
        }
    }
    ph.mark(6);
    ph.flush(gl == 0);
    if (gl == 0) {
        p.slot_key[slot] = best_key;
        p.slot_T[slot] = best_T;
        p.slot_cmax[slot] = best_cmax;
        p.slot_buf[slot] = best_buf;
        if (best_key != ~0ull) atomicMin(&p.hdr->best_key, best_key);
    }
}

// ---------------------------------------------------------------- split pipeline: the LPT alone
// k_lpt's item table: only the (e, l) half of every record, 8 bytes per sample (the LPT never
// reads ef / lf), so the table takes half the shared memory
struct TblEL {
    uint32_t it_s;  // shared-window address of the (e, l) pairs
    DFLOP_DEV Pair2<uint32_t> el(uint32_t pos) const {
        Pair2<uint32_t> r;
        asm("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(r.a), "=r"(r.b) : "r"(it_s + pos * 8u));
        return r;
    }
};

// The LPT pass of the packed variant for the candidates [c_begin, c_end) with few lanes per
// candidate (GL = m / 32: 32 buckets per lane for m = 64) and only the bucket keys and a
// 16-byte stage in shared memory per candidate (≈0.5 KB instead of ≈2 KB), so ~300
// candidates are resident per SM: the per-sample reduction and the two-sample bookkeeping
// are shared by 4x more buckets per lane.  Writes each candidate's
// assignment and final packed keys (offset removed) for the candidate kernel (MODE = 1).
template <int GL>
__global__ void __launch_bounds__(kLptMaxThreads) k_lpt(CandParams p) {
    if (p.hdr->variant != 0) return;  // the packed variant only
    const uint32_t sh = p.hdr->shift, co = p.hdr->offs;
    extern __shared__ __align__(128) uint8_t smem[];
    TblEL T;
    {
        for (uint32_t i = threadIdx.x; i < p.n; i += blockDim.x) {
            const uint4 r = __ldg(reinterpret_cast<const uint4*>(p.items) + i);
            reinterpret_cast<uint2*>(smem)[i] = make_uint2(r.x, r.y);
        }
        __syncthreads();
        T.it_s = (uint32_t)__cvta_generic_to_shared(smem);
    }
    bool forced = false;  // as in k_candidates
    if (p.m >= 1 && p.m <= p.n) {
        bool ok = true;
        for (uint32_t q = threadIdx.x & 31u; q < p.m; q += 32) {
            const Pair2<uint32_t> r = T.el(q);
            ok = ok && r.a != 0 && r.b != 0;
        }
        forced = __all_sync(FULL, ok);
    }
    const uint32_t grp = threadIdx.x / GL, gl = threadIdx.x % GL;
    const uint32_t cpb = blockDim.x / GL, m = p.m;
    uint8_t* base = smem + p.tbl_bytes + (size_t)grp * p.cand_bytes;
    Pair2<uint32_t>* EL = reinterpret_cast<Pair2<uint32_t>*>(base);
    uint8_t* stage = base + p.off_scr;
    const uint32_t span = p.c_end - p.c_begin;
    const uint32_t stride = gridDim.x * cpb;
    for (uint32_t b0 = p.c_begin; b0 < p.c_end; b0 += stride) {
        const uint32_t cc = b0 + (p.c_end - b0 >= stride ? blockIdx.x * cpb + grp : grp * gridDim.x + blockIdx.x);
        const bool valid = cc < p.c_end;
        if (!__any_sync(FULL, valid)) break;  // warp-uniform
        const uint32_t c = valid ? cc : p.c_end - 1;          // tail groups recompute a real candidate
        const uint32_t e = valid ? cc - p.c_begin : span;     // ... into the scratch entry
        uint8_t* apos = p.lpt_apos + (size_t)e * p.apos_bytes;
        for (uint32_t j = gl; j < m; j += GL) EL[j] = Pair2<uint32_t>{j, j + co};
        for (uint32_t b = p.n + gl; b < p.apos_bytes; b += GL) apos[b] = 0xFF;  // padding: never a bucket
        __syncwarp(FULL);
        lpt_pass<uint32_t, true, GL, true, TblEL>(p, T, c, sh, EL, EL, apos, stage, gl, co, forced);
        Pair2<uint32_t>* dst = reinterpret_cast<Pair2<uint32_t>*>(p.lpt_el) + (size_t)e * m;
        for (uint32_t j = gl; j < m; j += GL) {
            const Pair2<uint32_t> x = EL[j];
            __stcg(reinterpret_cast<unsigned long long*>(dst + j), pack64(x.b - co, x.a));
        }
        __syncwarp(FULL);
    }
}

template <typename A, bool PK, bool SM, bool O4>
static const void* ptr_gl(int gl) {
    switch (gl) {
        case 1: return reinterpret_cast<const void*>(&k_candidates<A, PK, 1, SM, O4>);
        case 2: return reinterpret_cast<const void*>(&k_candidates<A, PK, 2, SM, O4>);
        case 4: return reinterpret_cast<const void*>(&k_candidates<A, PK, 4, SM, O4>);
        case 8: return reinterpret_cast<const void*>(&k_candidates<A, PK, 8, SM, O4>);
        case 16: return reinterpret_cast<const void*>(&k_candidates<A, PK, 16, SM, O4>);
        default: return reinterpret_cast<const void*>(&k_candidates<A, PK, 32, SM, O4>);
    }
}

template <typename A, bool PK, bool SM, bool O4>
static void launch_gl(const CandLaunch& L, const CandParams& p, cudaStream_t s) {
    const dim3 grid(L.grid), block(L.cpb * L.gl);
    switch (L.gl) {
        case 1: k_candidates<A, PK, 1, SM, O4><<<grid, block, L.dyn, s>>>(p); break;
        case 2: k_candidates<A, PK, 2, SM, O4><<<grid, block, L.dyn, s>>>(p); break;
        case 4: k_candidates<A, PK, 4, SM, O4><<<grid, block, L.dyn, s>>>(p); break;
        case 8: k_candidates<A, PK, 8, SM, O4><<<grid, block, L.dyn, s>>>(p); break;
        case 16: k_candidates<A, PK, 16, SM, O4><<<grid, block, L.dyn, s>>>(p); break;
        default: k_candidates<A, PK, 32, SM, O4><<<grid, block, L.dyn, s>>>(p); break;
    }
}

// the split pipeline's candidate kernel (packed u32, shared-memory table; m >= 48: GL >= 8)
template <bool O4, int MODE>
static const void* ptr_split_gl(int gl) {
    switch (gl) {
        case 8: return reinterpret_cast<const void*>(&k_candidates<uint32_t, true, 8, true, O4, MODE>);
        case 16: return reinterpret_cast<const void*>(&k_candidates<uint32_t, true, 16, true, O4, MODE>);
        default: return reinterpret_cast<const void*>(&k_candidates<uint32_t, true, 32, true, O4, MODE>);
    }
}

template <bool O4, int MODE>
static void launch_split_gl(const CandLaunch& L, const CandParams& p, cudaStream_t s) {
    const dim3 grid(L.grid), block(L.cpb * L.gl);
    switch (L.gl) {
        case 8: k_candidates<uint32_t, true, 8, true, O4, MODE><<<grid, block, L.dyn, s>>>(p); break;
        case 16: k_candidates<uint32_t, true, 16, true, O4, MODE><<<grid, block, L.dyn, s>>>(p); break;
        default: k_candidates<uint32_t, true, 32, true, O4, MODE><<<grid, block, L.dyn, s>>>(p); break;
    }
}

#define DFLOP_SPLIT_UNIT(NAME, O4)                                                   \
    const void* split_ptr_##NAME(int gl) { return ptr_split_gl<O4, 1>(gl); }          \
    void split_launch_##NAME(const CandLaunch& L, const CandParams& p, cudaStream_t s) { \
        launch_split_gl<O4, 1>(L, p, s);                                              \
    }

// one translation unit per (variant, table placement, ORDER4) so the 72 instantiations build
// in parallel
#define DFLOP_CAND_UNIT(NAME, A, PK, SM, O4)                                                     \
    const void* cand_ptr_##NAME(int gl) { return ptr_gl<A, PK, SM, O4>(gl); }                     \
    void cand_launch_##NAME(const CandLaunch& L, const CandParams& p, cudaStream_t s) {           \
        launch_gl<A, PK, SM, O4>(L, p, s);                                                        \
    }

}  // namespace dflop
