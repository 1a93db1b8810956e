// balance.cu -- steps a2 and a5 of the DFLOP plan-candidate path on sm_100a, plus the
// standalone 1F1B simulator and CSR index groups; the candidate kernel (a3/a4) is in
// candidates.cu.
//
//   k_prep_keys     e_i = ef+eb, l_i = lf+lb, key_i = max(e_i, l_i) (R12), batch totals
//   k_rank_sort     LPT base order pi: key descending, index ascending (R18)
//   k_build_items   per-position item records (base order), 32- or 64-bit sums
//   k_finalize      winner -> dflop_cand_result + assignment
//   k_simulate      standalone batched 1F1B (dflop_simulate_1f1b)
//   k_group_*       CSR index groups ("returns a set of index groups")
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>

#include "cand.cuh"
#include "internal.h"

namespace dflop {

DFLOP_DEV uint32_t get_apos(const uint8_t* apos, uint32_t pos, bool wide) {
    return wide ? (uint32_t)reinterpret_cast<const uint16_t*>(apos)[pos] : (uint32_t)apos[pos];
}

// ---------------------------------------------------------------- a2: keys, order, records
__global__ void k_init(BalanceHeader* hdr, u64* slot_key, uint32_t n_slots) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t == 0) {
        hdr->sum_e = 0;
        hdr->sum_l = 0;
        hdr->max_key = 0;
        hdr->max_ld = 0;
        hdr->offs = 0;
        hdr->variant = 0;
        hdr->shift = 0;
        hdr->status = 0;
        hdr->best_key = ~0ull;
    }
    for (uint32_t s = t; s < n_slots; s += gridDim.x * blockDim.x) slot_key[s] = ~0ull;
}

// cost rows: ef, eb, lf, lb at cost + r * rs (rs >= n: the row stride)
__global__ void k_prep_keys(const uint32_t* __restrict__ cost, uint32_t n, size_t rs, BalanceHeader* hdr, u64* keys) {
    u64 se = 0, sl = 0, mk = 0, md = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const u64 e = (u64)cost[i] + cost[rs + i];
        const u64 l = (u64)cost[2 * rs + i] + cost[3 * rs + i];
        const u64 k = e > l ? e : l;
        keys[i] = k;
        se += e;
        sl += l;
        mk = k > mk ? k : mk;
        md = (l > e && l - e > md) ? l - e : md;
    }
    for (int off = 16; off > 0; off >>= 1) {
        se += __shfl_xor_sync(0xFFFFFFFFu, se, off);
        sl += __shfl_xor_sync(0xFFFFFFFFu, sl, off);
        const u64 o = __shfl_xor_sync(0xFFFFFFFFu, mk, off);
        mk = o > mk ? o : mk;
        const u64 od = __shfl_xor_sync(0xFFFFFFFFu, md, off);
        md = od > md ? od : md;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&hdr->sum_e, se);
        atomicAdd(&hdr->sum_l, sl);
        atomicMax(&hdr->max_key, mk);
        atomicMax(&hdr->max_ld, md);
    }
}

// rank_i = #{j : key_j > key_i or (key_j == key_i and j < i)}; order[rank_i] = i.
__global__ void k_rank_sort(const u64* __restrict__ keys, uint32_t n, uint32_t* order, uint32_t* item_pos) {
    __shared__ u64 tile[256];
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    const u64 ki = i < n ? keys[i] : 0;
    uint32_t rank = 0;
    for (uint32_t base = 0; base < n; base += 256) {
        __syncthreads();
        if (base + threadIdx.x < n) tile[threadIdx.x] = keys[base + threadIdx.x];
        __syncthreads();
        const uint32_t lim = min(256u, n - base);
        if (i < n) {
            for (uint32_t u = 0; u < lim; ++u) {
                const u64 kj = tile[u];
                rank += (kj > ki) | ((kj == ki) & (base + u < i));
            }
        }
    }
    if (i < n) {
        order[rank] = i;
        item_pos[i] = rank;
    }
}

// The same order by one CTA: a bitonic sort in shared memory of the composite keys
// (2^34 - 1 - key) << 16 | i (keys < 2^33: sums of two u32 ticks; i < 2^16), ascending =
// key descending, index ascending -- O(n log^2 n) instead of k_rank_sort's O(n^2) compares.
// n <= kBitonicMax; N = next power of two, padded with all-ones keys (sort last).
constexpr uint32_t kBitonicMax = 8192;
__global__ void __launch_bounds__(1024) k_bitonic_order(const u64* __restrict__ keys, uint32_t n, uint32_t* order,
                                                        uint32_t* item_pos) {
    extern __shared__ u64 sk[];
    uint32_t N = 1;
    while (N < n) N <<= 1;
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x)
        sk[i] = i < n ? ((((1ull << 34) - 1) - keys[i]) << 16) | i : ~0ull;
    __syncthreads();
    for (uint32_t k = 2; k <= N; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t t = threadIdx.x; t < N / 2; t += blockDim.x) {
                const uint32_t lo = 2 * t - (t & (j - 1)), hi = lo + j;  // pair (lo, lo + j), lo's bit j clear
                const bool up = (lo & k) == 0;
                const u64 a = sk[lo], b = sk[hi];
                if ((a > b) == up) {
                    sk[lo] = b;
                    sk[hi] = a;
                }
            }
            __syncthreads();
        }
    }
    for (uint32_t r = threadIdx.x; r < n; r += blockDim.x) {
        const uint32_t i = (uint32_t)(sk[r] & 0xFFFFu);
        order[r] = i;
        item_pos[i] = r;
    }
}

void order_launch_keys(const u64* keys, uint32_t n, uint32_t* order, uint32_t* item_pos, cudaStream_t s) {
    if (n == 0) return;
    if (n <= kBitonicMax) {
        uint32_t N = 1;
        while (N < n) N <<= 1;
        static bool attr = false;  // 64 KB of shared memory at kBitonicMax
        if (!attr) {
            cudaFuncSetAttribute(k_bitonic_order, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kBitonicMax * 8));
            attr = true;
        }
        k_bitonic_order<<<1, std::min<uint32_t>(1024u, std::max(32u, N / 2)), (size_t)N * 8, s>>>(keys, n, order,
                                                                                                    item_pos);
    } else {
        k_rank_sort<<<(n + 255) / 256, 256, 0, s>>>(keys, n, order, item_pos);
    }
}

// Chooses the candidate-kernel variant and writes the per-position records.
//   u32 when every bucket sum fits (sums of all e_i, l_i below 2^32 - 1);
//   packed u32 when every LPT probe value plus the probe offset C = max_i max(l_i - e_i, 0)
//   stays below 2^(32 - s), s = bits of m - 1:
//   a probe's winner has W <= min_j W_j + max(e, l) <= (sum_e + sum_l)/m + max key, every
//   probe adds at most one more max key, and refinement never raises the maximum (O6).
//   The candidate kernel probes max(E' + (e' - l' + C'), L' + C') = max(E' + e', L' + l')
//   - l' + C' (C' = C << s): one fused add-max per bucket, no wrap-around under this bound.
__global__ void k_build_items(const uint32_t* __restrict__ cost, uint32_t n, size_t rs, uint32_t m, uint32_t allow_pack,
                              BalanceHeader* hdr, const uint32_t* __restrict__ order, ItemRec<uint32_t>* it32,
                              ItemRec<u64>* it64) {
    const bool fits = hdr->sum_e < 0xFFFFFFFFull && hdr->sum_l < 0xFFFFFFFFull;
    uint32_t sh = 0;
    while ((1u << sh) < m) ++sh;
    const u64 bound = (hdr->sum_e + hdr->sum_l + m - 1) / m + 2 * hdr->max_key;
    const bool packed = allow_pack && fits && sh < 32 && bound + hdr->max_ld < (1ull << (32 - sh));
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        hdr->variant = packed ? 0u : (fits ? 1u : 2u);
        hdr->shift = sh;
        hdr->offs = packed ? (uint32_t)(hdr->max_ld << sh) : 0u;
    }
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const uint32_t i = order[t];
        const uint32_t ef = cost[i], eb = cost[rs + i], lf = cost[2 * rs + i], lb = cost[3 * rs + i];
        if (fits)
            // packed variant: e and l pre-shifted into the key position (E << s | j sums)
            it32[t] = packed ? ItemRec<uint32_t>{(ef + eb) << sh, (lf + lb) << sh, ef, lf}
                             : ItemRec<uint32_t>{ef + eb, lf + lb, ef, lf};
        else
            it64[t] = ItemRec<u64>{(u64)ef + eb, (u64)lf + lb, (u64)ef, (u64)lf};
    }
}

// ---------------------------------------------------------------- a5: winner
__global__ void k_finalize(BalanceHeader* hdr, const u64* slot_key, const u64* slot_T, const u64* slot_cmax,
                           const uint32_t* slot_buf, const uint8_t* slot_apos, uint32_t n_slots,
                           uint32_t apos_bytes, uint32_t wide, const uint32_t* pos_item, uint32_t n,
                           uint32_t id_base, dflop_cand_result* best, uint32_t* assign) {
    __shared__ uint32_t s_slot;
    const u64 key = hdr->best_key;
    if (threadIdx.x == 0) s_slot = 0xFFFFFFFFu;
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < n_slots; s += blockDim.x)
        if (slot_key[s] == key) atomicMin(&s_slot, s);
    __syncthreads();
    const uint32_t s = s_slot;
    if (threadIdx.x == 0) {
        best->key = key;
        best->makespan = s != 0xFFFFFFFFu ? slot_T[s] : 0;
        best->cmax = s != 0xFFFFFFFFu ? slot_cmax[s] : 0;
        best->cand = (uint32_t)(key & 0xFFFFFFull) - id_base;
        best->status = hdr->status;
    }
    if (assign && s != 0xFFFFFFFFu) {
        const uint8_t* ap = slot_apos + ((size_t)s * 2 + slot_buf[s]) * apos_bytes;
        for (uint32_t pos = threadIdx.x; pos < n; pos += blockDim.x)
            assign[pos_item[pos]] = get_apos(ap, pos, wide != 0);
    }
}

// ---------------------------------------------------------------- standalone 1F1B
__global__ void k_simulate(const u64* __restrict__ fwd, const u64* __restrict__ bwd, uint32_t C, uint32_t S,
                           uint32_t M, const uint32_t* __restrict__ ops, uint32_t n_ops, uint32_t D, u64* makespan,
                           u64* busy) {
    extern __shared__ __align__(16) uint8_t smem[];
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const uint32_t Dm = D - 1;
    u64* last = reinterpret_cast<u64*>(smem) + (size_t)threadIdx.x * (S + 2 * S * D);
    u64* FR = last + S;
    u64* BR = FR + S * D;
    const u64* f = fwd + (size_t)c * S * M;
    const u64* b = bwd + (size_t)c * S * M;
    for (uint32_t s = 0; s < S; ++s) last[s] = 0;
    for (uint32_t q = 0; q < n_ops; ++q) {
        const uint32_t op = __ldg(ops + q);
        const uint32_t kind = op_kind(op), s = op_stage(op), k = op_mb(op);
        u64 dur, dep = 0;
        if (kind == 0) {
            dur = f[(size_t)s * M + k];
            if (s > 0) dep = FR[(s - 1) * D + (k & Dm)];
        } else {
            dur = b[(size_t)s * M + k];
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
    makespan[c] = T;
    if (busy) {
        for (uint32_t s = 0; s < S; ++s) {
            u64 acc = 0;
            for (uint32_t k = 0; k < M; ++k) acc += f[(size_t)s * M + k] + b[(size_t)s * M + k];
            busy[(size_t)c * S + s] = acc;
        }
    }
}

// ---------------------------------------------------------------- CSR index groups
__global__ void k_group_count(const uint32_t* __restrict__ assign, uint32_t n, uint32_t* cnt) {
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        atomicAdd(&cnt[assign[i]], 1u);
}

// exclusive scan of cnt[m] into offsets[m+1] and fill[m] (one block of 1024 threads)
__global__ void k_group_scan(const uint32_t* cnt, uint32_t m, uint32_t* offsets, uint32_t* fill) {
    __shared__ uint32_t part[1024];
    const uint32_t t = threadIdx.x;
    const uint32_t per = (m + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(m, t * per), hi = min(m, lo + per);
    uint32_t s = 0;
    for (uint32_t j = lo; j < hi; ++j) s += cnt[j];
    part[t] = s;
    __syncthreads();
    for (uint32_t off = 1; off < blockDim.x; off <<= 1) {
        uint32_t v = t >= off ? part[t - off] : 0;
        __syncthreads();
        part[t] += v;
        __syncthreads();
    }
    uint32_t run = part[t] - s;
    for (uint32_t j = lo; j < hi; ++j) {
        offsets[j] = run;
        fill[j] = run;
        run += cnt[j];
    }
    if (t == blockDim.x - 1) offsets[m] = part[t];
}

// stable placement, samples ascending within each bucket: one warp walks the samples in
// chunks of 32; __match_any_sync ranks equal buckets inside a chunk.
__global__ void k_group_place(const uint32_t* __restrict__ assign, uint32_t n, uint32_t* fill, uint32_t* items) {
    const uint32_t lane = threadIdx.x;
    for (uint32_t base = 0; base < n; base += 32) {
        const uint32_t i = base + lane;
        const bool valid = i < n;
        const uint32_t a = valid ? assign[i] : 0xFFFFFFFFu;
        const unsigned peers = __match_any_sync(0xFFFFFFFFu, a);
        const uint32_t rank = __popc(peers & ((1u << lane) - 1u));
        uint32_t at = 0;
        if (valid) at = fill[a] + rank;
        __syncwarp();
        if (valid) {
            items[at] = i;
            if (rank == 0) fill[a] += __popc(peers);
        }
        __syncwarp();
    }
}

// ---------------------------------------------------------------- host side
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
static uint32_t round16(uint32_t x) { return (x + 15u) & ~15u; }
static uint32_t next_pow2(uint32_t x) {
    uint32_t p = 1;
    while (p < x) p <<= 1;
    return p;
}

size_t groups_ws_bytes(uint32_t n, uint32_t m) {
    (void)n;
    return align256((size_t)m * 4) * 2;
}

cudaError_t groups_launch(const uint32_t* assign, uint32_t n, uint32_t m, uint32_t* offsets, uint32_t* items,
                          void* ws, cudaStream_t s) {
    uint32_t* cnt = reinterpret_cast<uint32_t*>(ws);
    uint32_t* fill = reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(ws) + align256((size_t)m * 4));
    cudaError_t e = cudaMemsetAsync(cnt, 0, (size_t)m * 4, s);
    if (e != cudaSuccess) return e;
    if (n > 0) k_group_count<<<std::min<uint32_t>((n + 255) / 256, 1184), 256, 0, s>>>(assign, n, cnt);
    k_group_scan<<<1, 1024, 0, s>>>(cnt, m, offsets, fill);
    if (n > 0) k_group_place<<<1, 32, 0, s>>>(assign, n, fill, items);
    count_launches(n > 0 ? 3 : 1);
    return cudaGetLastError();
}

// a5 exchange input, device-resident: key[q] = results[q].key for the
// [P x D] (plan, batch) results, and in key[n] two u32 flags -- bit 0 and bit 1 of the status
// (the predict status OR the status of every result that evaluated a candidate) -- so the
// flags survive a MAX all-reduce as an OR.  One block.
__global__ void k_gather_keys(const dflop_cand_result* __restrict__ res, uint32_t n,
                              const uint32_t* __restrict__ d_status, uint64_t* key) {
    __shared__ uint32_t s_or;
    if (threadIdx.x == 0) s_or = *d_status;
    __syncthreads();
    uint32_t acc = 0;
    for (uint32_t q = threadIdx.x; q < n; q += blockDim.x) {
        const dflop_cand_result r = res[q];
        key[q] = r.key;
        if (r.key != ~0ull) acc |= r.status;
    }
    acc = __reduce_or_sync(0xFFFFFFFFu, acc);
    if ((threadIdx.x & 31u) == 0 && acc) atomicOr(&s_or, acc);
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t* bits = reinterpret_cast<uint32_t*>(key + n);
        bits[0] = s_or & 1u;
        bits[1] = (s_or >> 1) & 1u;
    }
}

cudaError_t gather_keys_launch(const dflop_cand_result* res, uint32_t n, const uint32_t* d_status, uint64_t* key,
                               cudaStream_t s) {
    k_gather_keys<<<1, 256, 0, s>>>(res, n, d_status, key);
    count_launches(1);
    return cudaGetLastError();
}

// diagnostic phase counters of the candidate kernel (timing builds only)
static unsigned long long* phase_counters() {
#ifdef DFLOP_TIMING
    static unsigned long long* d = nullptr;
    if (!d) {
        cudaMalloc(&d, 8 * sizeof(unsigned long long));
        cudaMemset(d, 0, 8 * sizeof(unsigned long long));
    }
    return d;
#else
    return nullptr;
#endif
}

static int env_int(const char* name, int dflt) {
    const char* v = getenv(name);
    return (v && *v) ? atoi(v) : dflt;
}

BalanceConfig balance_config(const BalanceShape& sh, int device) {
    BalanceConfig cfg;
    const DevAttr prop = dev_attr(device);
    if (prop.sms == 0) {
        cfg.why = "cudaDeviceGetAttribute failed";
        return cfg;
    }
    const uint32_t n = sh.n, m = sh.m, S = sh.S;
    // lanes per candidate: about 8 buckets per lane
    int gl = (int)next_pow2((m + 7) / 8);
    gl = std::min(32, std::max(1, gl));
    const int forced = env_int("DFLOP_GL", 0);
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8 || forced == 16 || forced == 32) gl = forced;
    cfg.gl = gl;
    const uint32_t per_bucket = (n + m - 1) / std::max(1u, m);
    const bool wide = m > 255;
    cfg.apos_bytes = round16(std::max(16u, n * (wide ? 2u : 1u)));
    // CSR member lists of the refinement: every bucket gets its LPT
    // count plus sigma free entries (a move adds one member to j'); a list that would
    // overflow triggers a rebuild from the assignment
    // two free entries per list: a bucket gaining a third member in one candidate is rare and
    // only triggers a rebuild, while the smaller lists keep more of the slots' scratch in the
    // L2 (config 5: sigma 16 -> 2, -1%; configs 2/3: -2..-4%)
    cfg.sigma = std::max(1u, std::min(2u, std::min(std::max(1u, sh.R), per_bucket)));
    const int fsig = env_int("DFLOP_SIGMA", 0);  // experiments: free list entries per bucket
    if (fsig >= 1 && fsig <= 256) cfg.sigma = (uint32_t)fsig;
    // counters cnt[m] and offsets off[m + 1] (u32) in shared memory up to m = 256, else in
    // front of the slot's global lists
    cfg.cnt_smem = m <= 256;
    const size_t hdr_u16 = cfg.cnt_smem ? 0 : 2 * (2 * (size_t)m + 1);
    cfg.csr_len = (uint32_t)((hdr_u16 + (size_t)n + (size_t)m * cfg.sigma + 7) & ~(size_t)7);
    // scratch: [cnt, off,] ls[cap], lp[cap] (u16) -- or the 1F1B rings (and, with ORDER4, the
    // ascending / descending slot orders, u16)
    const uint32_t rings = (S + 2 * S * sh.D) * 8u + ((sh.mode & DFLOP_MODE_ORDER4) ? 4u * sh.n_mb : 0u);
    const size_t smem_max = prop.smem_optin;
    const uint32_t nsm = (uint32_t)prop.sms;
    const uint32_t per_warp = 32u / (uint32_t)gl;  // candidate groups per warp
    const int forced_cpb = env_int("DFLOP_MAXCPB", 0);  // occupancy experiments
    // split pipeline: the packed variant's LPT in k_lpt with lg = m / 32
    // lanes per candidate and ~0.5 KB of shared memory each (bucket keys + a 16-byte stage),
    // then the candidate kernel (refinement + 1F1B) from its output, chunk by chunk
    const int split_env = env_int("DFLOP_SPLIT", 1);  // 0: never, 2: whenever eligible (tests)
    int lg = (int)std::min<uint32_t>(8, std::max<uint32_t>(2, next_pow2(m / 32 + 1) / 2));
    const int flg = env_int("DFLOP_LPT_GL", 0);
    if (flg == 1 || flg == 2 || flg == 4 || flg == 8) lg = flg;
    const uint32_t lpw = 32u / (uint32_t)lg;  // candidates per warp
    uint32_t lcb = round16(m * 8u) + 16u;
    if (lg == 1)  // 8-byte loads of 16 lanes (candidates) on distinct bank pairs: stride/8 odd
        lcb += 8;
    else
        while (lcb % 128 != 8u * (uint32_t)lg) lcb += 16;  // probe loads conflict-free (8-byte banks)
    const uint32_t ltbl = (uint32_t)(((size_t)n * 8 + 127) & ~(size_t)127);  // (e, l) pairs only
    uint32_t lcpb = ltbl < smem_max ? (uint32_t)std::min<size_t>((smem_max - ltbl) / lcb, kLptMaxThreads / lg) : 0;
    lcpb = lcpb / lpw * lpw;
    const bool split_pre = sh.split_ok && split_env != 0 && !(sh.mode & DFLOP_MODE_EXHAUSTIVE) && m >= 48 &&
                           !wide && n > 0 && n <= 4096 && gl >= 8 && lcpb >= 4 * lpw &&
                           (sh.n_cand >= 4096 || split_env == 2);
    // the split candidate kernel runs no LPT: stagger its candidates for the refinement's
    // broadcast reads (4 candidates of a warp on distinct banks) instead of the probe loads
    const int stg_env = env_int("DFLOP_SPLIT_STAGGER", 48);
    struct Lay {
        uint32_t cb, tbl, cpb;
        bool tbl_smem;
    };
    auto layout = [&](int v, uint32_t cap) {
        Lay L;
        uint32_t scr = round16(std::max((cfg.cnt_smem ? 8u * m + 4u : 0u) + 4u * cap, rings));
        if (v == 0 && split_pre)  // the split kernel: u32 counts, u16 offsets, rows' copy, 64 sorted keys
            scr = round16(std::max(round16(4u * m + ((2u * m + 2u + 3u) & ~3u) + 2u * cap) + 256u, rings));
        const uint32_t asz = v == 2 ? 8u : 4u;
        const uint32_t el = round16(m * 2u * asz);   // EL[m] then FL[m]
        uint32_t cb = 2 * el + scr;
        // stagger consecutive candidates across banks: a group's probe touches GL*2*asz bytes
        uint32_t span = std::max(16u, (uint32_t)gl * 2u * asz);
        if (v == 0 && split_pre && stg_env >= 16 && stg_env < 128 && stg_env % 16 == 0) span = (uint32_t)stg_env;
        if (v == 0 && split_pre && stg_env == 0) span = 128;  // no stagger
        if (span < 128) {
            const uint32_t want = span;  // a multiple of 16 below 128: reachable in <= 7 steps
            while (cb % 128 != want) cb += 16;
        }
        L.cb = cb;
        const uint32_t tbl = (uint32_t)(((size_t)n * (v == 2 ? 32u : 16u) + (size_t)n * 2 + 127) & ~(size_t)127);
        // stage the table in shared memory when it leaves room for at least 2 warps of candidates
        L.tbl_smem = (size_t)tbl + (size_t)2 * per_warp * cb <= smem_max;
        L.tbl = L.tbl_smem ? tbl : 0;
        const int max_threads = (v == 0 && split_pre) ? kSplitMaxThreads : kCandMaxThreads;
        uint32_t cpb = (uint32_t)std::min<size_t>((smem_max - L.tbl) / cb, max_threads / gl);
        // no more groups than the family needs (one CTA per SM), whole warps only
        cpb = std::min<uint32_t>(cpb, std::max(1u, (sh.n_cand + nsm - 1) / nsm));
        if (forced_cpb >= (int)per_warp) cpb = std::min<uint32_t>(cpb, (uint32_t)forced_cpb);
        cpb = (cpb + per_warp - 1) / per_warp * per_warp;
        if ((size_t)L.tbl + (size_t)cpb * cb > smem_max) cpb -= per_warp;
        L.cpb = cpb;
        return L;
    };
    // shared-memory copies of the first `cap` members of j* and j': about twice the mean list
    // length, shrunk (not below 32) while that buys resident candidates -- occupancy hides the
    // latency of the shared-memory and shuffle chains (config 5: cap 128 -> 104 raises 72 -> 80
    // candidates per SM, -6.7%; 768-thread blocks would need <= 80 registers: +37%)
    uint32_t cap = std::min(128u, std::max(32u, next_pow2(2 * std::max(1u, per_bucket))));
    {
        uint32_t best = cap, best_cpb = layout(0, cap).cpb;
        for (uint32_t c2 = cap - 8; c2 >= 32 && c2 < cap; c2 -= 8) {
            const uint32_t q = layout(0, c2).cpb;
            if (q > best_cpb) {
                best_cpb = q;
                best = c2;
            }
        }
        cap = best;
    }
    const int forced_cap = env_int("DFLOP_CAP", 0);
    if (forced_cap >= 1 && forced_cap <= 4096) cap = (uint32_t)forced_cap;
    cfg.cap = cap;
    for (int v = 0; v < 3; ++v) {
        const Lay L = layout(v, cap);
        const uint32_t cb = L.cb, cpb = L.cpb;
        cfg.cand_bytes[v] = cb;
        cfg.tbl_smem[v] = L.tbl_smem;
        cfg.tbl_bytes[v] = L.tbl;
        cfg.off_fl[v] = round16(m * 2u * (v == 2 ? 8u : 4u));
        cfg.off_scr[v] = 2 * cfg.off_fl[v];
        if (cpb == 0) {
            char buf[200];
            snprintf(buf, sizeof buf,
                     "a warp of %u candidates needs %u B of shared memory, more than %zu B (n=%u, m=%u)", per_warp,
                     per_warp * cb, smem_max, n, m);
            cfg.why = buf;
            return cfg;
        }
        const size_t dyn = (size_t)cfg.tbl_bytes[v] + (size_t)cpb * cb;
        cudaFuncSetAttribute(cand_kernel_ptr(v, gl, cfg.tbl_smem[v], (sh.mode & DFLOP_MODE_ORDER4) != 0),
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)dyn);
        const uint32_t want = (sh.n_cand + cpb - 1) / cpb;
        cfg.cpb[v] = cpb;
        cfg.grid[v] = std::max(1u, std::min<uint32_t>(want, nsm));
    }
    cfg.n_slots = 0;
    for (int v = 0; v < 3; ++v) cfg.n_slots = std::max(cfg.n_slots, cfg.grid[v] * cfg.cpb[v]);
    if (split_pre && cfg.tbl_smem[0] && cfg.cpb[0] > 0) {
        // chunks of r whole k_lpt waves, as few as the entry buffer allows: every chunk boundary
        // costs a partly filled k_lpt wave and candidate-kernel round (config 5: 10^6 candidates
        // in one chunk 94.5 ms, in chunks of 6 waves 97.4 ms); the entries take ~4.6 KB per
        // candidate, so a chunk is capped at 2^20 candidates (~4.8 GB)
        const uint32_t wave = nsm * lcpb;
        uint32_t best_r = std::max(1u, (1u << 20) / std::max(1u, wave));
        const int fr = env_int("DFLOP_SPLIT_ROUNDS", 0);
        if (fr >= 1 && fr <= 64) best_r = (uint32_t)fr;
        cfg.split = true;
        cfg.lpt_gl = lg;
        cfg.lpt_cb = lcb;
        cfg.lpt_tbl = ltbl;
        cfg.lpt_cpb = lcpb;
        cfg.lpt_grid = nsm;
        cfg.lpt_chunk = std::min<uint32_t>(sh.n_cand, wave * best_r);
        const int fch = env_int("DFLOP_SPLIT_CHUNK", 0);  // tests: several chunks at small K
        if (fch > 0) cfg.lpt_chunk = std::min<uint32_t>(sh.n_cand, (uint32_t)fch);
        cudaFuncSetAttribute(lpt_kernel_ptr(lg), cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((size_t)ltbl + (size_t)lcpb * lcb));
        cudaFuncSetAttribute(split_kernel_ptr(gl, (sh.mode & DFLOP_MODE_ORDER4) != 0),
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)((size_t)cfg.tbl_bytes[0] + (size_t)cfg.cpb[0] * cfg.cand_bytes[0]));
    }
    if (env_int("DFLOP_DEBUG", 0))
        fprintf(stderr,
                "[dflop] balance n=%u m=%u S=%u D=%u gl=%d cap=%u apos=%u | packed/u32/u64: tbl=%u/%u/%u "
                "cand=%u/%u/%u cpb=%u/%u/%u grid=%u/%u/%u | slots=%u\n",
                n, m, S, sh.D, gl, cfg.cap, cfg.apos_bytes, cfg.tbl_bytes[0], cfg.tbl_bytes[1], cfg.tbl_bytes[2],
                cfg.cand_bytes[0], cfg.cand_bytes[1], cfg.cand_bytes[2], cfg.cpb[0], cfg.cpb[1], cfg.cpb[2],
                cfg.grid[0], cfg.grid[1], cfg.grid[2], cfg.n_slots);
    if (cfg.split && env_int("DFLOP_DEBUG", 0))
        fprintf(stderr, "[dflop] split: lpt gl=%d cpb=%u cand=%u tbl=%u chunk=%u\n", cfg.lpt_gl, cfg.lpt_cpb,
                cfg.lpt_cb, cfg.lpt_tbl, cfg.lpt_chunk);
    size_t o = 0;
    cfg.o_hdr = o;        o += align256(sizeof(BalanceHeader));
    cfg.o_keys = o;       o += align256((size_t)n * 8);
    cfg.o_order = o;      o += align256((size_t)n * 4);
    cfg.o_item_pos = o;   o += align256((size_t)n * 4);
    cfg.o_items32 = o;    o += align256((size_t)n * 16);
    cfg.o_items64 = o;    o += align256((size_t)n * 32);
    cfg.o_slot_key = o;   o += align256((size_t)cfg.n_slots * 8);
    cfg.o_slot_T = o;     o += align256((size_t)cfg.n_slots * 8);
    cfg.o_slot_cmax = o;  o += align256((size_t)cfg.n_slots * 8);
    cfg.o_slot_buf = o;   o += align256((size_t)cfg.n_slots * 4);
    cfg.o_slot_apos = o;  o += align256((size_t)cfg.n_slots * 2 * cfg.apos_bytes);
    cfg.o_slot_csr = o;   o += align256((size_t)cfg.n_slots * 2 * cfg.csr_len);
    cfg.o_grp = o;        o += groups_ws_bytes(n, m);
    if (cfg.split) {  // k_lpt -> candidate kernel: per chunk entry (+1 for tail groups)
        cfg.o_lpt_apos = o;  o += align256(((size_t)cfg.lpt_chunk + 1) * cfg.apos_bytes);
        cfg.o_lpt_el = o;    o += align256(((size_t)cfg.lpt_chunk + 1) * m * 8);
    }

    cfg.total = o;
    cfg.ok = true;
    return cfg;
}

dflop_status balance_launch(const BalanceArgs& a, const BalanceConfig& cfg, const SlotProgram& prog,
                            cudaStream_t s) {
    char* ws = reinterpret_cast<char*>(a.ws);
    BalanceHeader* hdr = reinterpret_cast<BalanceHeader*>(ws + cfg.o_hdr);
    u64* keys = reinterpret_cast<u64*>(ws + cfg.o_keys);
    uint32_t* order = reinterpret_cast<uint32_t*>(ws + cfg.o_order);
    uint32_t* item_pos = reinterpret_cast<uint32_t*>(ws + cfg.o_item_pos);
    auto* it32 = reinterpret_cast<ItemRec<uint32_t>*>(ws + cfg.o_items32);
    auto* it64 = reinterpret_cast<ItemRec<u64>*>(ws + cfg.o_items64);
    u64* slot_key = reinterpret_cast<u64*>(ws + cfg.o_slot_key);
    u64* slot_T = reinterpret_cast<u64*>(ws + cfg.o_slot_T);
    u64* slot_cmax = reinterpret_cast<u64*>(ws + cfg.o_slot_cmax);
    uint32_t* slot_buf = reinterpret_cast<uint32_t*>(ws + cfg.o_slot_buf);
    uint8_t* slot_apos = reinterpret_cast<uint8_t*>(ws + cfg.o_slot_apos);
    uint16_t* slot_csr = reinterpret_cast<uint16_t*>(ws + cfg.o_slot_csr);
    const uint32_t n = a.sh.n;
    const uint32_t allow_pack = (a.sh.mode & DFLOP_MODE_EXHAUSTIVE) ? 0u : 1u;

    k_init<<<std::max(1u, std::min<uint32_t>((cfg.n_slots + 255) / 256, 148)), 256, 0, s>>>(hdr, slot_key,
                                                                                          cfg.n_slots);
    if (n > 0) {
        const uint32_t gb = std::min<uint32_t>((n + 255) / 256, 592);
        const size_t rs = a.cost_stride ? a.cost_stride : n;
        k_prep_keys<<<gb, 256, 0, s>>>(a.cost_ticks, n, rs, hdr, keys);
        order_launch_keys(keys, n, order, item_pos, s);
        k_build_items<<<gb, 256, 0, s>>>(a.cost_ticks, n, rs, a.sh.m, allow_pack, hdr, order, it32, it64);
    } else {
        k_build_items<<<1, 32, 0, s>>>(a.cost_ticks, 0, 0, a.sh.m, allow_pack, hdr, order, it32, it64);
    }
    CandParams p{};
    p.pos_item = order;
    p.item_pos = item_pos;
    p.ops = prog.d_ops;
    p.levels = prog.d_levels;
    p.dense = prog.d_dense;
    p.n_levels = prog.n_levels;
    p.hdr = hdr;
    p.slot_apos = slot_apos;
    p.slot_csr = slot_csr;
    p.slot_key = slot_key;
    p.slot_T = slot_T;
    p.slot_cmax = slot_cmax;
    p.slot_buf = slot_buf;
    p.cand_T = reinterpret_cast<u64*>(a.cand_T);
    p.cand_cmax = reinterpret_cast<u64*>(a.cand_cmax);
    p.n = n;
    p.m = a.sh.m;
    p.S = a.sh.S;
    p.e_pp = a.sh.e_pp;
    p.l_dp = a.sh.l_dp;
    p.n_mb = a.sh.n_mb;
    p.R = a.sh.R;
    p.G = a.sh.G;
    p.D = prog.D;
    p.n_ops = prog.n_ops;
    p.c_begin = a.c_begin;
    p.c_end = a.c_end;
    p.id_base = a.id_base;
    p.seed0 = a.seed0;
    p.seed1 = a.seed1;
    p.exhaustive = (a.sh.mode & DFLOP_MODE_EXHAUSTIVE) ? 1u : 0u;
    p.wide = a.sh.m > 255;
    p.cap = cfg.cap;
    p.sigma = cfg.sigma;
    p.cnt_smem = cfg.cnt_smem ? 1u : 0u;
    p.order4 = (a.sh.mode & DFLOP_MODE_ORDER4) ? 1u : 0u;
    p.csr_len = cfg.csr_len;
    p.apos_bytes = cfg.apos_bytes;
    p.phase = phase_counters();
    const int mark = prof_begin(s);
    uint32_t launches = n > 0 ? 8 : 6;
    for (int v = 0; v < 3; ++v) {
        CandParams q = p;
        q.items = v == 2 ? reinterpret_cast<const void*>(it64) : reinterpret_cast<const void*>(it32);
        q.tbl_bytes = cfg.tbl_bytes[v];
        q.cand_bytes = cfg.cand_bytes[v];
        q.off_fl = cfg.off_fl[v];
        q.off_scr = cfg.off_scr[v];
        q.want_variant = (uint32_t)v;
        CandLaunch L;
        L.variant = v;
        L.gl = cfg.gl;
        L.tbl_smem = cfg.tbl_smem[v];
        L.grid = cfg.grid[v];
        L.cpb = cfg.cpb[v];
        L.dyn = (size_t)cfg.tbl_bytes[v] + (size_t)cfg.cpb[v] * cfg.cand_bytes[v];
        cudaFuncSetAttribute(cand_kernel_ptr(v, cfg.gl, cfg.tbl_smem[v], p.order4 != 0),
                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)L.dyn);
        if (v == 0 && cfg.split) {
            // per chunk: k_lpt, then the packed candidate kernel on its output (both return at
            // once when another variant runs)
            CandParams ql = q;
            ql.tbl_bytes = cfg.lpt_tbl;
            ql.cand_bytes = cfg.lpt_cb;
            ql.off_scr = round16(a.sh.m * 8u);
            ql.lpt_apos = reinterpret_cast<uint8_t*>(ws + cfg.o_lpt_apos);
            ql.lpt_el = reinterpret_cast<uint32_t*>(ws + cfg.o_lpt_el);
            q.lpt_apos = ql.lpt_apos;
            q.lpt_el = ql.lpt_el;
            const size_t ldyn = (size_t)cfg.lpt_tbl + (size_t)cfg.lpt_cpb * cfg.lpt_cb;
            cudaFuncSetAttribute(split_kernel_ptr(cfg.gl, p.order4 != 0),
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)L.dyn);
            cudaFuncSetAttribute(lpt_kernel_ptr(cfg.lpt_gl), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ldyn);
            for (uint32_t c0 = a.c_begin; c0 < a.c_end; c0 += cfg.lpt_chunk) {
                ql.c_begin = q.c_begin = c0;
                ql.c_end = q.c_end = std::min(a.c_end, c0 + cfg.lpt_chunk);
                if (p.cand_T) {  // the per-candidate arrays are indexed from a.c_begin
                    q.cand_T = p.cand_T + (c0 - a.c_begin);
                    q.cand_cmax = p.cand_cmax + (c0 - a.c_begin);
                }
                lpt_launch(cfg.lpt_gl, cfg.lpt_grid, cfg.lpt_cpb, ldyn, ql, s);
                split_launch(L, q, s);
                launches += 2;
                count_split_chunks(1);
            }
            launches -= 1;
        } else {
            cand_launch(L, q, s);
        }
        prof_mark(mark, v + 1, s);
    }
    k_finalize<<<1, 256, 0, s>>>(hdr, slot_key, slot_T, slot_cmax, slot_buf, slot_apos, cfg.n_slots, cfg.apos_bytes,
                                 a.sh.m > 255, order, n, a.id_base, a.best, a.assign);
    count_launches(launches);
    return cuda_status(cudaGetLastError(), "balance launch");
}

dflop_status simulate_launch(const uint64_t* fwd, const uint64_t* bwd, uint32_t C, uint32_t S, uint32_t M,
                             uint64_t* makespan, uint64_t* busy, const SlotProgram& prog, cudaStream_t s) {
    if (C == 0) return DFLOP_OK;
    const size_t per = (size_t)(S + 2 * S * prog.D) * 8;
    int dev = 0;
    cudaGetDevice(&dev);
    const DevAttr prop = dev_attr(dev);
    uint32_t threads = (uint32_t)std::min<size_t>(256, prop.smem_optin / per);
    threads = std::max(1u, std::min(threads, C));
    const size_t dyn = per * threads;
    cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_simulate), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dyn);
    k_simulate<<<(C + threads - 1) / threads, threads, dyn, s>>>(
        reinterpret_cast<const u64*>(fwd), reinterpret_cast<const u64*>(bwd), C, S, M, prog.d_ops, prog.n_ops,
        prog.D, reinterpret_cast<u64*>(makespan), reinterpret_cast<u64*>(busy));
    count_launches(1);
    return cuda_status(cudaGetLastError(), "simulate launch");
}

}  // namespace dflop

// Diagnostic: summed clock64 cycles per phase of the candidate kernel (lane 0 of every
// candidate group), zeros unless built with -DDFLOP_TIMING.  Not part of include/dflop.h.
extern "C" int dflop_debug_phase_cycles(unsigned long long out[8], int reset) {
    unsigned long long* d = dflop::phase_counters();
    for (int k = 0; k < 8; ++k) out[k] = 0;
    if (!d) return 0;
    cudaDeviceSynchronize();
    cudaMemcpy(out, d, 8 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    if (reset) cudaMemset(d, 0, 8 * sizeof(unsigned long long));
    return 0;
}
