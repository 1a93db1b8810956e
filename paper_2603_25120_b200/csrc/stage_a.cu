// stage_a.cu -- step a6 Stage A: Algorithm 1 phase 2 over every (config, N_mb)
// pair, one thread per pair, in fp64 evaluated with explicitly rounded operations
// (__dmul_rn/__dadd_rn/__ddiv_rn: no FMA contraction) in the order written in DESIGN.md
// section 4 (O9), followed by a block-parallel top-P selection by (T_A, pair index).
//
//   t_bsz = mean_b*GBS/(i*E_dp), t_seq = mean_s*GBS/(i*L_dp)
//   Mem_E = ms_E(ceil(E_l/E_pp), E_tp) + (E_pp+L_pp)*as_E(ceil(E_l/E_pp), E_tp, t_bsz)  Eq.(4)
//   Mem_L = ms_L(ceil(L_l/L_pp), L_tp) + L_pp*as_L(ceil(L_l/L_pp), L_tp, t_seq)          Eq.(5)
//   E_dur = 1e9*t_bsz*c_E / (E_thr(t_bsz,E_tp)*E_tp*E_pp)
//   L_dur = 1e9*(nbar*c_att*mean_s^2/L_attn_thr + c_lin*t_seq/L_lin_thr) / (L_tp*L_pp) (R5)
//   T_A   = (i + E_pp + L_pp - 1) * max(round(E_dur), round(L_dur))
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace dflop {

struct GridD {
    int n_x, n_tp;
    double x[DFLOP_MAX_X];
    double tp[DFLOP_MAX_TP];
    double v[DFLOP_MAX_TP][DFLOP_MAX_X];
};
struct MemGridD {
    int n_x, n_tp;
    double l[2];
    double tp[DFLOP_MAX_TP];
    double x[DFLOP_MAX_X];
    double v[2][DFLOP_MAX_TP][DFLOP_MAX_X];
};
struct StageAConsts {
    GridD thr_e, thr_att, thr_lin;
    MemGridD ms_e, as_e, ms_l, as_l;
    double mem_per_gpu, tick_ns;
    uint32_t e_layers, e_hidden, e_seq, e_attn, l_layers, l_hidden, tau_tile, tau_frame;
    uint32_t gbs, n_cfgs, n, top_p;
    u64 n_pairs;
};

DFLOP_DEV double dclamp(double x, double lo, double hi) { return x < lo ? lo : (x > hi ? hi : x); }

DFLOP_DEV int dbracket(const double* xs, int n, double xh) {
    int k = 0;
    while (k + 1 < n - 1 && xs[k + 1] <= xh) ++k;
    return k;
}

// (1 - w) * a + w * b, no contraction
DFLOP_DEV double dlerp(double a, double b, double w) { return __dadd_rn(__dmul_rn(__dsub_rn(1.0, w), a), __dmul_rn(w, b)); }

DFLOP_DEV double lerp1d(const double* xs, const double* vs, int n, double x) {
    if (n == 1) return vs[0];
    const double xh = dclamp(x, xs[0], xs[n - 1]);
    const int k = dbracket(xs, n, xh);
    const double w = __ddiv_rn(__dsub_rn(xh, xs[k]), __dsub_rn(xs[k + 1], xs[k]));
    return dlerp(vs[k], vs[k + 1], w);
}

DFLOP_DEV double interp_thr_d(const GridD& g, double x, double tp) {
    if (g.n_tp == 1) return lerp1d(g.x, g.v[0], g.n_x, x);
    const double th = dclamp(tp, g.tp[0], g.tp[g.n_tp - 1]);
    const int a = dbracket(g.tp, g.n_tp, th);
    const double wt = __ddiv_rn(__dsub_rn(th, g.tp[a]), __dsub_rn(g.tp[a + 1], g.tp[a]));
    return dlerp(lerp1d(g.x, g.v[a], g.n_x, x), lerp1d(g.x, g.v[a + 1], g.n_x, x), wt);
}

DFLOP_DEV double mem_plane_d(const MemGridD& g, int q, double tp, double x) {
    if (g.n_tp == 1) return lerp1d(g.x, g.v[q][0], g.n_x, x);
    const double th = dclamp(tp, g.tp[0], g.tp[g.n_tp - 1]);
    const int a = dbracket(g.tp, g.n_tp, th);
    const double wt = __ddiv_rn(__dsub_rn(th, g.tp[a]), __dsub_rn(g.tp[a + 1], g.tp[a]));
    return dlerp(lerp1d(g.x, g.v[q][a], g.n_x, x), lerp1d(g.x, g.v[q][a + 1], g.n_x, x), wt);
}

DFLOP_DEV double interp_mem_d(const MemGridD& g, double l, double tp, double x) {
    const double wl = __ddiv_rn(__dsub_rn(l, g.l[0]), __dsub_rn(g.l[1], g.l[0]));
    return dlerp(mem_plane_d(g, 0, tp, x), mem_plane_d(g, 1, tp, x), wl);
}

DFLOP_DEV u64 round_u64_d(double x) {
    if (!(x < 18446744073709549568.0)) return ~0ull;
    return __double2ull_rn(x);
}

// Algorithm 1 lines 20-27 for one pair; returns T_A or ~0 when Eq. (4)/(5) fails.
DFLOP_DEV u64 stage_a_pair(const StageAConsts& k, const uint32_t* cfg, uint32_t i, double mean_b, double mean_s) {
    const uint32_t e_tp = cfg[0], e_pp = cfg[1], e_dp = cfg[2], l_tp = cfg[3], l_pp = cfg[4], l_dp = cfg[5];
    const double gbs = (double)k.gbs, di = (double)i;
    const double t_bsz = __ddiv_rn(__dmul_rn(mean_b, gbs), __dmul_rn(di, (double)e_dp));
    const double t_seq = __ddiv_rn(__dmul_rn(mean_s, gbs), __dmul_rn(di, (double)l_dp));
    const double le = (double)((k.e_layers + e_pp - 1) / e_pp);
    const double ll = (double)((k.l_layers + l_pp - 1) / l_pp);
    const double Me = __dadd_rn(interp_mem_d(k.ms_e, le, (double)e_tp, 0.0),
                                __dmul_rn((double)(e_pp + l_pp), interp_mem_d(k.as_e, le, (double)e_tp, t_bsz)));
    const double Ml = __dadd_rn(interp_mem_d(k.ms_l, ll, (double)l_tp, 0.0),
                                __dmul_rn((double)l_pp, interp_mem_d(k.as_l, ll, (double)l_tp, t_seq)));
    if (Me > k.mem_per_gpu || Ml > k.mem_per_gpu) return ~0ull;
    const double he = (double)k.e_hidden, es = (double)k.e_seq, hl = (double)k.l_hidden;
    const double lin_e = __dmul_rn(__dmul_rn(24.0, he), he);
    const double att_e = k.e_attn ? __dmul_rn(4.0, he) : 0.0;
    const double per_inst_e = __dadd_rn(__dmul_rn(lin_e, es), __dmul_rn(__dmul_rn(att_e, es), es));
    const double c_e = __dmul_rn((double)k.e_layers, per_inst_e);
    const double c_lin = __dmul_rn(__dmul_rn(__dmul_rn(24.0, hl), hl), (double)k.l_layers);
    const double c_att = __dmul_rn(__dmul_rn(4.0, hl), (double)k.l_layers);
    const double EF = __dmul_rn(t_bsz, c_e);
    const double thr_e = interp_thr_d(k.thr_e, t_bsz, (double)e_tp);
    const double Ed = __ddiv_rn(__dmul_rn(1e9, EF), __dmul_rn(__dmul_rn(thr_e, (double)e_tp), (double)e_pp));
    const double nbar = __ddiv_rn(gbs, __dmul_rn(di, (double)l_dp));
    const double Latt = __dmul_rn(nbar, __dmul_rn(__dmul_rn(c_att, mean_s), mean_s));
    const double Llin = __dmul_rn(c_lin, t_seq);
    const double thr_a = interp_thr_d(k.thr_att, t_seq, (double)l_tp);
    const double thr_l = interp_thr_d(k.thr_lin, t_seq, (double)l_tp);
    const double Ld = __ddiv_rn(__dmul_rn(1e9, __dadd_rn(__ddiv_rn(Latt, thr_a), __ddiv_rn(Llin, thr_l))),
                                __dmul_rn((double)l_tp, (double)l_pp));
    const u64 qe = round_u64_d(__ddiv_rn(Ed, k.tick_ns)), ql = round_u64_d(__ddiv_rn(Ld, k.tick_ns));
    const u64 mx = qe > ql ? qe : ql;
    const u64 f = (u64)(i + e_pp + l_pp - 1);
    const u64 hi = __umul64hi(f, mx);
    const u64 lo = f * mx;
    if (hi != 0 || lo > ~0ull - 1) return ~0ull - 1;
    return lo;
}

// ---------------------------------------------------------------- top-P (T, pair) selection
struct TopEntry {
    u64 T;
    uint32_t pair;
};

DFLOP_DEV bool entry_lt(u64 ta, uint32_t pa, u64 tb, uint32_t pb) { return ta < tb || (ta == tb && pa < pb); }

// Block-wide accumulator of the P smallest (T, pair): keeps a sorted list in shared memory;
// a tile's candidates below the current P-th value are appended and the union is sorted
// with a bitonic network.
struct TopAcc {
    u64* sT;       // [NP]
    uint32_t* sP;  // [NP]
    uint32_t* s_cnt;
    uint32_t P, NP;
};

DFLOP_DEV void bitonic(u64* T, uint32_t* Pp, uint32_t NP) {
    for (uint32_t k = 2; k <= NP; k <<= 1) {
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
            for (uint32_t i = threadIdx.x; i < NP; i += blockDim.x) {
                const uint32_t ixj = i ^ j;
                if (ixj > i) {
                    const bool up = (i & k) == 0;
                    const bool gt = entry_lt(T[ixj], Pp[ixj], T[i], Pp[i]);
                    if (gt == up) {
                        const u64 t = T[i];
                        T[i] = T[ixj];
                        T[ixj] = t;
                        const uint32_t q = Pp[i];
                        Pp[i] = Pp[ixj];
                        Pp[ixj] = q;
                    }
                }
            }
            __syncthreads();
        }
    }
}

// One tile: every thread offers (T, pair) or nothing.  List entries [0, P) hold the current
// best (sorted, padded with ~0); new entries go to [P, NP).
DFLOP_DEV void top_offer(TopAcc& acc, bool has, u64 T, uint32_t pair) {
    const u64 thrT = acc.sT[acc.P - 1];
    const uint32_t thrP = acc.sP[acc.P - 1];
    const bool keep = has && entry_lt(T, pair, thrT, thrP);
    if (threadIdx.x == 0) *acc.s_cnt = 0;
    __syncthreads();
    if (keep) {
        const uint32_t at = atomicAdd(acc.s_cnt, 1u);
        acc.sT[acc.P + at] = T;
        acc.sP[acc.P + at] = pair;
    }
    __syncthreads();
    const uint32_t cnt = *acc.s_cnt;
    __syncthreads();  // everyone has read cnt before the next offer resets it
    if (cnt == 0) return;
    for (uint32_t i = acc.P + cnt + threadIdx.x; i < acc.NP; i += blockDim.x) {
        acc.sT[i] = ~0ull;
        acc.sP[i] = 0xFFFFFFFFu;
    }
    __syncthreads();
    bitonic(acc.sT, acc.sP, acc.NP);
}

struct StageAArgs {
    const uint32_t* cfgs;        // [n_cfgs][6]
    const uint32_t* pair_start;  // [n_cfgs + 1]
    const u64* sums;             // [2]: sum b, sum s (integers)
    u64* out;                    // [n_pairs] or null
    u64* block_T;                // [grid][P]
    uint32_t* block_P;
    unsigned long long* n_feasible;
};

__global__ void k_batch_sums(const StageAConsts* kc, const uint32_t* __restrict__ tiles,
                             const uint32_t* __restrict__ frames, const uint32_t* __restrict__ text, uint32_t n,
                             u64* sums) {
    u64 sb = 0, ss = 0;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        sb += (u64)tiles[i] + frames[i];
        ss += (u64)text[i] + (u64)kc->tau_tile * tiles[i] + (u64)kc->tau_frame * frames[i];
    }
    for (int off = 16; off > 0; off >>= 1) {
        sb += __shfl_xor_sync(0xFFFFFFFFu, sb, off);
        ss += __shfl_xor_sync(0xFFFFFFFFu, ss, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&sums[0], sb);
        atomicAdd(&sums[1], ss);
    }
}

__global__ void __launch_bounds__(1024) k_stage_a(const StageAConsts* __restrict__ kc, StageAArgs a) {
    extern __shared__ __align__(16) uint8_t smem[];
    StageAConsts& k = *reinterpret_cast<StageAConsts*>(smem);
    for (uint32_t w = threadIdx.x; w < sizeof(StageAConsts) / 4; w += blockDim.x)
        reinterpret_cast<uint32_t*>(&k)[w] = reinterpret_cast<const uint32_t*>(kc)[w];
    __syncthreads();
    const uint32_t P = k.top_p;
    uint32_t NP = 1;
    while (NP < P + blockDim.x) NP <<= 1;
    u64* sT = reinterpret_cast<u64*>(smem + ((sizeof(StageAConsts) + 15) & ~(size_t)15));
    uint32_t* sP = reinterpret_cast<uint32_t*>(sT + NP);
    uint32_t* s_cnt = sP + NP;
    for (uint32_t i = threadIdx.x; i < NP; i += blockDim.x) {
        sT[i] = ~0ull;
        sP[i] = 0xFFFFFFFFu;
    }
    __syncthreads();
    TopAcc acc{sT, sP, s_cnt, P, NP};
    const double n = (double)k.n;
    const double mean_b = k.n ? __ddiv_rn((double)a.sums[0], n) : 0.0;
    const double mean_s = k.n ? __ddiv_rn((double)a.sums[1], n) : 0.0;
    unsigned long long feas = 0;
    const u64 stride = (u64)gridDim.x * blockDim.x;
    for (u64 base = (u64)blockIdx.x * blockDim.x; base < k.n_pairs; base += stride) {
        const u64 pidx = base + threadIdx.x;
        bool has = false;
        u64 T = ~0ull;
        if (pidx < k.n_pairs) {
            // pair -> (config eps, i): binary search in pair_start
            uint32_t lo = 0, hi = k.n_cfgs;
            while (hi - lo > 1) {
                const uint32_t mid = (lo + hi) / 2;
                if ((u64)a.pair_start[mid] <= pidx) lo = mid; else hi = mid;
            }
            const uint32_t i = (uint32_t)(pidx - a.pair_start[lo]) + 1;
            T = stage_a_pair(k, a.cfgs + 6 * (size_t)lo, i, mean_b, mean_s);
            has = T != ~0ull;
            feas += has;
            if (a.out) a.out[pidx] = T;
        }
        top_offer(acc, has, T, (uint32_t)pidx);
    }
    for (int off = 16; off > 0; off >>= 1) feas += __shfl_xor_sync(0xFFFFFFFFu, feas, off);
    if ((threadIdx.x & 31) == 0 && feas) atomicAdd(a.n_feasible, feas);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        a.block_T[(size_t)blockIdx.x * P + i] = sT[i];
        a.block_P[(size_t)blockIdx.x * P + i] = sP[i];
    }
}

__global__ void __launch_bounds__(1024) k_top_merge(const u64* block_T, const uint32_t* block_P, uint32_t n_entries,
                                                    uint32_t P, StageATop* top) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint32_t NP = 1;
    while (NP < P + blockDim.x) NP <<= 1;
    u64* sT = reinterpret_cast<u64*>(smem);
    uint32_t* sP = reinterpret_cast<uint32_t*>(sT + NP);
    uint32_t* s_cnt = sP + NP;
    for (uint32_t i = threadIdx.x; i < NP; i += blockDim.x) {
        sT[i] = ~0ull;
        sP[i] = 0xFFFFFFFFu;
    }
    __syncthreads();
    TopAcc acc{sT, sP, s_cnt, P, NP};
    for (uint32_t base = 0; base < n_entries; base += blockDim.x) {
        const uint32_t e = base + threadIdx.x;
        const bool has = e < n_entries && block_T[e] != ~0ull;
        top_offer(acc, has, has ? block_T[e] : ~0ull, has ? block_P[e] : 0xFFFFFFFFu);
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < P; i += blockDim.x) {
        top[i].T = sT[i];
        top[i].pair = sP[i];
        top[i].pad = 0;
    }
}

static void to_gridd(const dflop_grid& s, GridD& d) {
    memset(&d, 0, sizeof d);
    d.n_x = (int)s.n_x;
    d.n_tp = (int)s.n_tp;
    for (uint32_t k = 0; k < s.n_x; ++k) d.x[k] = s.x[k];
    for (uint32_t a = 0; a < s.n_tp; ++a) {
        d.tp[a] = s.tp[a];
        for (uint32_t k = 0; k < s.n_x; ++k) d.v[a][k] = s.v[a][k];
    }
}
static void to_memd(const dflop_mem_grid& s, MemGridD& d) {
    memset(&d, 0, sizeof d);
    d.n_x = (int)s.n_x;
    d.n_tp = (int)s.n_tp;
    d.l[0] = s.l[0];
    d.l[1] = s.l[1];
    for (uint32_t k = 0; k < s.n_x; ++k) d.x[k] = s.x[k];
    for (uint32_t a = 0; a < s.n_tp; ++a) d.tp[a] = s.tp[a];
    for (int q = 0; q < 2; ++q)
        for (uint32_t a = 0; a < s.n_tp; ++a)
            for (uint32_t k = 0; k < s.n_x; ++k) d.v[q][a][k] = s.v[q][a][k];
}

static size_t a256(size_t x) { return (x + 255) & ~(size_t)255; }

static uint32_t stage_a_grid(int device) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    return (uint32_t)sms;
}

size_t stage_a_ws_bytes(uint64_t n_pairs, int device) {
    (void)n_pairs;
    const uint32_t grid = stage_a_grid(device);
    return a256(sizeof(StageAConsts)) + a256(16) + a256((size_t)grid * 256 * 8) + a256((size_t)grid * 256 * 4) +
           a256(sizeof(unsigned long long));
}

dflop_status stage_a_launch(const dflop_cost_model* cm, const dflop_mem_model* mm, const uint32_t* d_cfgs,
                            const uint32_t* d_pair_start, uint32_t n_cfgs, uint64_t n_pairs, uint32_t gbs,
                            const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                            uint32_t top_p, void* ws, uint64_t* stage_a_out, StageATop* d_top,
                            unsigned long long* d_n_feasible, cudaStream_t s) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint32_t grid = stage_a_grid(dev);
    char* w = reinterpret_cast<char*>(ws);
    StageAConsts* d_k = reinterpret_cast<StageAConsts*>(w);
    size_t o = a256(sizeof(StageAConsts));
    u64* d_sums = reinterpret_cast<u64*>(w + o);
    o += a256(16);
    u64* bT = reinterpret_cast<u64*>(w + o);
    o += a256((size_t)grid * 256 * 8);
    uint32_t* bP = reinterpret_cast<uint32_t*>(w + o);

    static thread_local StageAConsts k;  // staged host copy (pageable; cudaMemcpyAsync stages it)
    memset(&k, 0, sizeof k);
    to_gridd(cm->thr_e, k.thr_e);
    to_gridd(cm->thr_att, k.thr_att);
    to_gridd(cm->thr_lin, k.thr_lin);
    to_memd(mm->ms_e, k.ms_e);
    to_memd(mm->as_e, k.as_e);
    to_memd(mm->ms_l, k.ms_l);
    to_memd(mm->as_l, k.as_l);
    k.mem_per_gpu = mm->mem_per_gpu;
    k.tick_ns = cm->tick_ns;
    k.e_layers = cm->e_layers;
    k.e_hidden = cm->e_hidden;
    k.e_seq = cm->e_seq;
    k.e_attn = cm->e_attn;
    k.l_layers = cm->l_layers;
    k.l_hidden = cm->l_hidden;
    k.tau_tile = cm->tau_tile;
    k.tau_frame = cm->tau_frame;
    k.gbs = gbs;
    k.n_cfgs = n_cfgs;
    k.n = n;
    k.top_p = top_p;
    k.n_pairs = n_pairs;
    cudaError_t e = cudaMemcpyAsync(d_k, &k, sizeof k, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "stage A consts");
    e = cudaMemsetAsync(d_sums, 0, 16, s);
    if (e == cudaSuccess) e = cudaMemsetAsync(d_n_feasible, 0, sizeof(unsigned long long), s);
    if (e != cudaSuccess) return cuda_status(e, "stage A memset");
    if (n > 0)
        k_batch_sums<<<std::min<uint32_t>((n + 255) / 256, 148), 256, 0, s>>>(d_k, tiles, frames, text, n, d_sums);
    const uint32_t threads = 1024;
    uint32_t NP = 1;
    while (NP < top_p + threads) NP <<= 1;
    const size_t dyn = ((sizeof(StageAConsts) + 15) & ~(size_t)15) + (size_t)NP * 12 + 16;
    cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_stage_a), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dyn);
    StageAArgs a{d_cfgs, d_pair_start, d_sums, reinterpret_cast<u64*>(stage_a_out), bT, bP, d_n_feasible};
    const int mark = prof_stage_begin(s);
    k_stage_a<<<grid, threads, dyn, s>>>(d_k, a);
    prof_stage_end(mark, s);
    const size_t dyn2 = (size_t)NP * 12 + 16;
    cudaFuncSetAttribute(reinterpret_cast<const void*>(&k_top_merge), cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)dyn2);
    k_top_merge<<<1, threads, dyn2, s>>>(bT, bP, grid * top_p, top_p, d_top);
    count_launches(n > 0 ? 3 : 2);
    return cuda_status(cudaGetLastError(), "stage A launch");
}

}  // namespace dflop
