// api.cpp -- the extern "C" entry points of libdflop.so (include/dflop.h): argument
// validation, workspace layout, launch sequencing, and the NCCL exchange of the search.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "internal.h"

struct dflop_comm {
    ncclComm_t comm;
    int rank;
    int world;
    int device;
};

namespace dflop {

static thread_local std::string g_err;
static void release_streams();
static void release_config_tables();

void set_error(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
}

dflop_status cuda_status(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return DFLOP_OK;
    set_error("%s: %s", what, cudaGetErrorString(e));
    return DFLOP_ERR_CUDA;
}

static dflop_status invalid(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return DFLOP_ERR_INVALID_ARGUMENT;
}

static dflop_status validate_grid(const dflop_grid& g, const char* name) {
    if (g.n_x < 1 || g.n_x > DFLOP_MAX_X || g.n_tp < 1 || g.n_tp > DFLOP_MAX_TP)
        return invalid("%s: n_x=%u n_tp=%u out of range", name, g.n_x, g.n_tp);
    for (uint32_t k = 1; k < g.n_x; ++k)
        if (!(g.x[k] > g.x[k - 1])) return invalid("%s: shape knots not strictly increasing at %u", name, k);
    for (uint32_t a = 1; a < g.n_tp; ++a)
        if (!(g.tp[a] > g.tp[a - 1])) return invalid("%s: tp knots not strictly increasing at %u", name, a);
    for (uint32_t a = 0; a < g.n_tp; ++a)
        for (uint32_t k = 0; k < g.n_x; ++k)
            if (!(g.v[a][k] > 0.0) || !std::isfinite(g.v[a][k]))
                return invalid("%s: throughput v[%u][%u] must be finite and > 0 (S:122)", name, a, k);
    return DFLOP_OK;
}

static dflop_status validate_mgrid(const dflop_mem_grid& g, const char* name) {
    if (g.n_x < 1 || g.n_x > DFLOP_MAX_X || g.n_tp < 1 || g.n_tp > DFLOP_MAX_TP)
        return invalid("%s: n_x=%u n_tp=%u out of range", name, g.n_x, g.n_tp);
    if (!(g.l[1] > g.l[0])) return invalid("%s: layer knots must satisfy l[0] < l[1]", name);
    for (uint32_t k = 1; k < g.n_x; ++k)
        if (!(g.x[k] > g.x[k - 1])) return invalid("%s: shape knots not strictly increasing at %u", name, k);
    for (uint32_t a = 1; a < g.n_tp; ++a)
        if (!(g.tp[a] > g.tp[a - 1])) return invalid("%s: tp knots not strictly increasing at %u", name, a);
    for (int q = 0; q < 2; ++q)
        for (uint32_t a = 0; a < g.n_tp; ++a)
            for (uint32_t k = 0; k < g.n_x; ++k)
                if (!std::isfinite(g.v[q][a][k]) || g.v[q][a][k] < 0.0)
                    return invalid("%s: memory value v[%d][%u][%u] must be finite and >= 0", name, q, a, k);
    return DFLOP_OK;
}

dflop_status validate_cost_model(const dflop_cost_model* m) {
    if (!m) return invalid("cost model is NULL");
    if (m->struct_size != sizeof(dflop_cost_model))
        return invalid("dflop_cost_model.struct_size=%u, expected %zu", m->struct_size, sizeof(dflop_cost_model));
    if (!m->e_layers || !m->e_hidden || !m->e_seq || !m->l_layers || !m->l_hidden)
        return invalid("cost model: layers, hidden sizes and e_seq must be >= 1");
    if (!(m->tick_ns > 0.0) || !std::isfinite(m->tick_ns)) return invalid("cost model: tick_ns must be > 0");
    if (!(m->bwd_ratio >= 0.0) || !std::isfinite(m->bwd_ratio)) return invalid("cost model: bwd_ratio must be >= 0");
    dflop_status st;
    if ((st = validate_grid(m->thr_e, "thr_e")) != DFLOP_OK) return st;
    if ((st = validate_grid(m->thr_att, "thr_att")) != DFLOP_OK) return st;
    if ((st = validate_grid(m->thr_lin, "thr_lin")) != DFLOP_OK) return st;
    if (const dflop_correction* c = m->correction) {
        if (c->struct_size != sizeof(dflop_correction))
            return invalid("dflop_correction.struct_size=%u, expected %zu", c->struct_size, sizeof(dflop_correction));
        for (int g = 0; g < 3; ++g)
            for (int q = 0; q < DFLOP_CORR_BINS; ++q)
                if (!(c->rho[g][q] > 0.0f) || !std::isfinite(c->rho[g][q]))
                    return invalid("correction rho[%d][%d] must be finite and > 0", g, q);
    }
    return DFLOP_OK;
}

dflop_status validate_plan(const dflop_plan* p) {
    if (!p) return invalid("plan is NULL");
    if (!p->e_tp || !p->e_pp || !p->e_dp || !p->l_tp || !p->l_pp || !p->l_dp || !p->n_mb)
        return invalid("plan: every degree and n_mb must be >= 1 (P:481)");
    return DFLOP_OK;
}

static int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

// ---------------------------------------------------------------- balance planning
struct BalancePlan {
    BalanceShape sh;
    BalanceConfig cfg;
    SlotProgram prog;
};

static dflop_status plan_balance(uint32_t n, const dflop_plan* plan, uint32_t mode, uint32_t R, uint32_t G,
                                 uint32_t n_cand, BalancePlan* out, bool split_ok = true) {
    const uint64_t m = (uint64_t)plan->n_mb * plan->l_dp;
    const uint64_t S = (uint64_t)plan->e_pp + plan->l_pp;
    if (n > 65535) {
        set_error("n=%u > 65535", n);
        return DFLOP_ERR_SHAPE;
    }
    if (m > 65535 || plan->n_mb > 65535) {
        set_error("m = n_mb*l_dp = %llu > 65535", (unsigned long long)m);
        return DFLOP_ERR_SHAPE;
    }
    if (S > 32) {
        set_error("S = e_pp + l_pp = %llu > 32", (unsigned long long)S);
        return DFLOP_ERR_SHAPE;
    }
    dflop_status st = get_slot_program((uint32_t)S, plan->n_mb, &out->prog);
    if (st != DFLOP_OK) return st;
    BalanceShape& sh = out->sh;
    sh.n = n;
    sh.m = (uint32_t)m;
    sh.S = (uint32_t)S;
    sh.e_pp = plan->e_pp;
    sh.l_dp = plan->l_dp;
    sh.n_mb = plan->n_mb;
    sh.mode = mode;
    sh.R = R;
    sh.G = G;
    sh.n_cand = n_cand;
    sh.D = out->prog.D;
    sh.split_ok = split_ok ? 1u : 0u;
    out->cfg = balance_config(sh, current_device());
    if (!out->cfg.ok) {
        set_error("%s", out->cfg.why.c_str());
        return DFLOP_ERR_UNSUPPORTED;
    }
    return DFLOP_OK;
}

static dflop_status validate_bparams(const dflop_balance_params* bp, uint32_t n, uint64_t m) {
    if (!bp) return invalid("balance params NULL");
    if (bp->struct_size != sizeof(dflop_balance_params))
        return invalid("dflop_balance_params.struct_size=%u, expected %zu", bp->struct_size,
                       sizeof(dflop_balance_params));
    if (bp->mode & ~(DFLOP_MODE_EXHAUSTIVE | DFLOP_MODE_ORDER4)) return invalid("mode %u unknown", bp->mode);
    if (bp->K == 0 || bp->K > (1u << 24)) return invalid("K=%u outside 1..2^24", bp->K);
    if (bp->cand_begin >= bp->cand_end || bp->cand_end > bp->K)
        return invalid("shard [%u, %u) empty or outside [0, K=%u)", bp->cand_begin, bp->cand_end, bp->K);
    if ((uint64_t)bp->id_base + bp->K > (1u << 24)) return invalid("id_base + K must be <= 2^24 (packed key)");
    if (bp->G < 1 || bp->G > 16) return invalid("G=%u outside 1..16", bp->G);
    if (bp->R > 4096) return invalid("R=%u > 4096", bp->R);
    if (bp->mode & DFLOP_MODE_EXHAUSTIVE) {
        double cnt = std::pow((double)m, (double)n);
        if (cnt > (double)bp->K) return invalid("EXHAUSTIVE needs m^n = %.0f <= K = %u", cnt, bp->K);
    }
    return DFLOP_OK;
}

}  // namespace dflop

using namespace dflop;

// ==================================================================== C ABI
extern "C" {

uint32_t dflop_abi_version(void) { return DFLOP_ABI_VERSION; }

const char* dflop_last_error(void) { return g_err.c_str(); }

dflop_status dflop_release_caches(void) {
    release_slot_programs();
    release_streams();
    release_config_tables();
    return DFLOP_OK;
}

dflop_status dflop_predict_costs(const dflop_cost_model* model, const dflop_plan* plan, const uint32_t* tiles,
                                 const uint32_t* frames, const uint32_t* text, uint32_t n, float* cost_f32,
                                 uint32_t* cost_ticks, uint32_t* dev_status, dflop_stream_t stream) {
    g_err.clear();
    dflop_status st = validate_cost_model(model);
    if (st != DFLOP_OK) return st;
    if ((st = validate_plan(plan)) != DFLOP_OK) return st;
    if (n > 0x7FFFFFFFu) {
        set_error("n=%u too large", n);
        return DFLOP_ERR_SHAPE;
    }
    if (n > 0 && (!tiles || !frames || !text)) return invalid("feature pointers must be non-NULL");
    PredictConsts k = predict_consts(model, plan);
    return cuda_status(predict_launch(model, &k, 1, tiles, frames, text, n, cost_f32, cost_ticks, (size_t)4 * n,
                                      dev_status, (cudaStream_t)stream),
                       "predict launch");
}

dflop_status dflop_balance_microbatches(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan,
                                        const dflop_balance_params* bp, void* ws, size_t* ws_bytes,
                                        dflop_cand_result* best, uint32_t* assign, uint32_t* group_offsets,
                                        uint32_t* group_items, uint64_t* cand_makespan, uint64_t* cand_cmax,
                                        dflop_stream_t stream) {
    g_err.clear();
    dflop_status st = validate_plan(plan);
    if (st != DFLOP_OK) return st;
    const uint64_t m = (uint64_t)plan->n_mb * plan->l_dp;
    if ((st = validate_bparams(bp, n, m)) != DFLOP_OK) return st;
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    BalancePlan bpn;
    if ((st = plan_balance(n, plan, bp->mode, bp->R, bp->G, bp->cand_end - bp->cand_begin, &bpn)) != DFLOP_OK)
        return st;
    const size_t need = bpn.cfg.total;
    if (!ws) {
        *ws_bytes = need;
        return DFLOP_OK;
    }
    if (*ws_bytes < need) {
        set_error("workspace %zu B < required %zu B", *ws_bytes, need);
        return DFLOP_ERR_WORKSPACE_TOO_SMALL;
    }
    if ((uintptr_t)ws % 256) return invalid("workspace must be 256-byte aligned");
    if (!best) return invalid("best is NULL");
    if (n > 0 && !cost_ticks) return invalid("cost_ticks is NULL");
    if ((cand_makespan == nullptr) != (cand_cmax == nullptr))
        return invalid("cand_makespan and cand_cmax must both be given or both NULL");
    if ((group_offsets == nullptr) != (group_items == nullptr))
        return invalid("group_offsets and group_items must both be given or both NULL");
    cudaStream_t s = (cudaStream_t)stream;
    // assignment needed for groups even if the caller did not ask for it: use the groups
    // scratch tail of the workspace as a temporary
    uint32_t* asg = assign;
    std::vector<char> dummy;
    if (!asg && group_offsets) {
        set_error("group_offsets requires assign");
        return DFLOP_ERR_INVALID_ARGUMENT;
    }
    BalanceArgs a{};
    a.cost_ticks = cost_ticks;
    a.sh = bpn.sh;
    a.K = bp->K;
    a.c_begin = bp->cand_begin;
    a.c_end = bp->cand_end;
    a.seed0 = bp->seed[0];
    a.seed1 = bp->seed[1];
    a.id_base = bp->id_base;
    a.ws = ws;
    a.best = best;
    a.assign = asg;
    a.cand_T = cand_makespan;
    a.cand_cmax = cand_cmax;
    if ((st = balance_launch(a, bpn.cfg, bpn.prog, s)) != DFLOP_OK) return st;
    if (group_offsets) {
        char* g = reinterpret_cast<char*>(ws) + bpn.cfg.o_grp;
        return cuda_status(groups_launch(asg, n, (uint32_t)m, group_offsets, group_items, g, s), "groups launch");
    }
    return DFLOP_OK;
}

dflop_status dflop_simulate_1f1b(const uint64_t* fwd, const uint64_t* bwd, uint32_t C, uint32_t S, uint32_t M,
                                 uint64_t* makespan, uint64_t* stage_busy, dflop_stream_t stream) {
    g_err.clear();
    if (S == 0 || M == 0 || S > 32 || M > 65535) {
        set_error("inconsistent duration matrix shape: S=%u M=%u (need 1<=S<=32, 1<=M<=65535)", S, M);
        return DFLOP_ERR_SHAPE;
    }
    if (C > 0 && (!fwd || !bwd || !makespan)) return invalid("fwd/bwd/makespan must be non-NULL");
    SlotProgram prog;
    dflop_status st = get_slot_program(S, M, &prog);
    if (st != DFLOP_OK) return st;
    return simulate_launch(fwd, bwd, C, S, M, makespan, stage_busy, prog, (cudaStream_t)stream);
}

dflop_status dflop_index_groups(const uint32_t* assign, uint32_t n, uint32_t m, uint32_t* offsets, uint32_t* items,
                                void* ws, size_t* ws_bytes, dflop_stream_t stream) {
    g_err.clear();
    if (m == 0 || m > 65535) {
        set_error("m=%u outside 1..65535", m);
        return DFLOP_ERR_SHAPE;
    }
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    const size_t need = groups_ws_bytes(n, m);
    if (!ws) {
        *ws_bytes = need;
        return DFLOP_OK;
    }
    if (*ws_bytes < need) {
        set_error("workspace %zu B < required %zu B", *ws_bytes, need);
        return DFLOP_ERR_WORKSPACE_TOO_SMALL;
    }
    if (!offsets || (n > 0 && (!assign || !items))) return invalid("NULL pointer");
    return cuda_status(groups_launch(assign, n, m, offsets, items, ws, (cudaStream_t)stream), "groups launch");
}

// ---------------------------------------------------------------- NCCL
dflop_status dflop_get_unique_id(uint8_t id[128]) {
    g_err.clear();
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) {
        set_error("ncclGetUniqueId: %s", ncclGetErrorString(r));
        return DFLOP_ERR_NCCL;
    }
    memcpy(id, &u, 128);
    return DFLOP_OK;
}

dflop_status dflop_comm_init(const uint8_t id[128], int rank, int world, int device, dflop_comm** comm) {
    g_err.clear();
    if (!id || !comm || world < 1 || rank < 0 || rank >= world) return invalid("bad comm arguments");
    cudaError_t ce = cudaSetDevice(device);
    if (ce != cudaSuccess) return cuda_status(ce, "cudaSetDevice");
    ncclUniqueId u;
    memcpy(&u, id, 128);
    dflop_comm* c = new dflop_comm();
    ncclResult_t r = ncclCommInitRank(&c->comm, world, u, rank);
    if (r != ncclSuccess) {
        delete c;
        set_error("ncclCommInitRank: %s", ncclGetErrorString(r));
        return DFLOP_ERR_NCCL;
    }
    c->rank = rank;
    c->world = world;
    c->device = device;
    *comm = c;
    return DFLOP_OK;
}

dflop_status dflop_comm_destroy(dflop_comm* comm) {
    g_err.clear();
    if (!comm) return DFLOP_OK;
    ncclResult_t r = ncclCommDestroy(comm->comm);
    delete comm;
    if (r != ncclSuccess) {
        set_error("ncclCommDestroy: %s", ncclGetErrorString(r));
        return DFLOP_ERR_NCCL;
    }
    return DFLOP_OK;
}

}  // extern "C"

// ==================================================================== search
namespace dflop {

struct ConfigTable {
    std::vector<uint32_t> cfgs;        // n_cfgs x 6
    std::vector<uint32_t> pair_start;  // n_cfgs + 1
    uint32_t* d_cfgs = nullptr;
    uint32_t* d_pair_start = nullptr;
    uint64_t n_pairs = 0;
};

static std::mutex g_cfg_mu;
static std::map<std::tuple<int, uint32_t, uint32_t, uint32_t>, ConfigTable> g_cfg_cache;

static void release_config_tables() {
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    for (auto& kv : g_cfg_cache) {
        if (kv.second.d_cfgs) cudaFree(kv.second.d_cfgs);
        if (kv.second.d_pair_start) cudaFree(kv.second.d_pair_start);
    }
    g_cfg_cache.clear();
}

// Algorithm 1 phase 1: FindCombs in ascending (tp, pp); cartesian product per
// split of N_gpus (R16).
static void find_combs(uint32_t g, uint32_t node, std::vector<uint32_t>& out) {
    for (uint32_t tp = 1; tp <= g && tp <= node; ++tp) {
        if (g % tp) continue;
        for (uint32_t pp = 1; pp <= g / tp; ++pp) {
            if ((g / tp) % pp) continue;
            out.push_back(tp);
            out.push_back(pp);
            out.push_back(g / tp / pp);
        }
    }
}

static dflop_status get_config_table(uint32_t n_gpus, uint32_t node, uint32_t gbs, const ConfigTable** out) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_cfg_mu);
    auto key = std::make_tuple(dev, n_gpus, node, gbs);
    auto it = g_cfg_cache.find(key);
    if (it != g_cfg_cache.end()) {
        *out = &it->second;
        return DFLOP_OK;
    }
    ConfigTable t;
    std::vector<uint32_t> ec, lc;
    for (uint32_t eg = 1; eg < n_gpus; ++eg) {
        ec.clear();
        lc.clear();
        find_combs(eg, node, ec);
        find_combs(n_gpus - eg, node, lc);
        for (size_t a = 0; a < ec.size(); a += 3)
            for (size_t b = 0; b < lc.size(); b += 3) {
                t.cfgs.insert(t.cfgs.end(), {ec[a], ec[a + 1], ec[a + 2], lc[b], lc[b + 1], lc[b + 2]});
            }
    }
    const uint32_t nc = (uint32_t)(t.cfgs.size() / 6);
    t.pair_start.resize(nc + 1);
    uint64_t acc = 0;
    for (uint32_t e = 0; e < nc; ++e) {
        t.pair_start[e] = (uint32_t)acc;
        acc += gbs / t.cfgs[6 * e + 5];  // N_max_mbatch = GBS // L_dp
    }
    if (acc > 0xFFFFFFFFull) {
        set_error("too many (config, N_mb) pairs: %llu", (unsigned long long)acc);
        return DFLOP_ERR_UNSUPPORTED;
    }
    t.pair_start[nc] = (uint32_t)acc;
    t.n_pairs = acc;
    cudaError_t ce = cudaMalloc(&t.d_cfgs, std::max<size_t>(4, t.cfgs.size() * 4));
    if (ce == cudaSuccess) ce = cudaMalloc(&t.d_pair_start, t.pair_start.size() * 4);
    if (ce == cudaSuccess && !t.cfgs.empty())
        ce = cudaMemcpy(t.d_cfgs, t.cfgs.data(), t.cfgs.size() * 4, cudaMemcpyHostToDevice);
    if (ce == cudaSuccess)
        ce = cudaMemcpy(t.d_pair_start, t.pair_start.data(), t.pair_start.size() * 4, cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {  // free a partial upload
        if (t.d_cfgs) cudaFree(t.d_cfgs);
        if (t.d_pair_start) cudaFree(t.d_pair_start);
        return cuda_status(ce, "config table upload");
    }
    auto res = g_cfg_cache.emplace(key, std::move(t));
    *out = &res.first->second;
    return DFLOP_OK;
}

// workspace regions of the search
struct SearchLayout {
    size_t o_costs, o_results, o_assigns, o_bcast, o_key, o_stage_a, o_top, o_feas, o_status, o_bal, total;
    size_t bal_bytes, bal_stride;
    uint32_t n_bal;  // balance workspaces: one per Stage-B stream
};

// Stage B balances the top-P plans on up to kStageBStreams streams: one plan's candidate
// kernel runs ~1.7 waves of the GPU, so the tail of one plan overlaps the next plan's start
// (DESIGN.md section 9).  DFLOP_STAGEB_STREAMS=1..8 overrides.
constexpr uint32_t kStageBStreams = 4;
static uint32_t stage_b_streams() {
    const char* e = getenv("DFLOP_STAGEB_STREAMS");
    const int v = e ? atoi(e) : (int)kStageBStreams;
    return (uint32_t)std::min(8, std::max(1, v));
}
static std::mutex g_stream_mu;
static std::map<int, std::vector<cudaStream_t>> g_streams;
// k-th auxiliary stream of `dev` (created once, non-blocking, destroyed by dflop_release_caches)
static cudaStream_t aux_stream(int dev, uint32_t k) {
    std::lock_guard<std::mutex> lk(g_stream_mu);
    auto& v = g_streams[dev];
    while (v.size() <= k) {
        cudaStream_t st = nullptr;
        if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
        v.push_back(st);
    }
    return v[k];
}
static void release_streams() {
    std::lock_guard<std::mutex> lk(g_stream_mu);
    for (auto& kv : g_streams)
        for (cudaStream_t st : kv.second) cudaStreamDestroy(st);
    g_streams.clear();
}

// Upper bound of one balance workspace when the plan is not known yet (Algorithm 1 mode):
// at most one resident candidate group per candidate of the shard plus one warp of groups
// per SM, and never more than 1024 groups per SM.
static size_t balance_bound(uint32_t n, uint32_t m_max, uint32_t K, int device) {
    int nsm = 148;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device);
    const size_t slots = std::min<size_t>((size_t)nsm * 1024, (size_t)K + (size_t)nsm * 32);
    const size_t apos_max = std::max<size_t>(16, ((size_t)2 * n + 15) & ~(size_t)15);
    return 256 * 2 + al256((size_t)n * 8) + 2 * al256((size_t)n * 4) + al256((size_t)n * 16) +
           al256((size_t)n * 32) + 3 * al256(slots * 8) + al256(slots * 4) + al256(slots * 2 * apos_max) +
           al256(slots * 2 * (2 * (size_t)n + 5 * (size_t)m_max + 16)) + al256((size_t)m_max * 4) * 2 + 4096;
}

static SearchLayout search_layout(uint32_t n_tot, uint32_t n_max, uint32_t P, uint32_t PD, uint64_t n_pairs,
                                  size_t bal_bytes, uint32_t n_bal, int device) {
    SearchLayout L;
    size_t o = 0;
    L.o_costs = o;   o += al256((size_t)P * 4 * n_tot * 4);
    L.o_results = o; o += al256((size_t)PD * sizeof(dflop_cand_result));
    L.o_assigns = o; o += al256((size_t)P * n_tot * 4);
    L.o_bcast = o;   o += al256(sizeof(dflop_cand_result) + (size_t)n_max * 4);
    L.o_key = o;     o += al256(((size_t)PD + 1) * 8);
    L.o_stage_a = o; o += al256(stage_a_ws_bytes(n_pairs, device));
    L.o_top = o;     o += al256((size_t)P * sizeof(StageATop));
    L.o_feas = o;    o += 256;
    L.o_status = o;  o += 256;
    L.bal_bytes = bal_bytes;
    L.bal_stride = al256(bal_bytes);
    L.n_bal = std::max(1u, n_bal);
    L.o_bal = o;     o += L.bal_stride * L.n_bal;
    L.total = o;
    return L;
}

static dflop_status nccl_status(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return DFLOP_OK;
    set_error("%s: %s", what, ncclGetErrorString(r));
    return DFLOP_ERR_NCCL;
}

}  // namespace dflop

namespace dflop {

// a6 search over D batches (D = 1: dflop_search_plans; D > 1: Eq. (1) over the sample,
// N2).  Batch b is samples [off[b], off[b+1]) of the concatenated features; its candidate
// family uses Philox key (seed0, seed1 + b) (R33).  Stage A runs on the mean shapes of the
// whole sample; Stage B balances every (top-P plan, batch); the plan minimises
// (sum_b T_B(b), Stage-A rank) and every batch's winner is materialised for it.
static dflop_status search_impl(const dflop_cluster* cl, const dflop_cost_model* cm, const dflop_mem_model* mm,
                                const uint32_t* tiles, const uint32_t* frames, const uint32_t* text,
                                const uint32_t* off, uint32_t D, const dflop_search_params* sp, dflop_comm* comm,
                                void* ws, size_t* ws_bytes, dflop_plan_result* out, dflop_cand_result* batch_out,
                                uint64_t* plan_objective, dflop_plan* plans_out, uint32_t* assign,
                                uint64_t* stage_a_out,
                                uint64_t stage_a_cap, cudaStream_t s) {
    g_err.clear();
    dflop_status st = validate_cost_model(cm);
    if (st != DFLOP_OK) return st;
    if (!sp || sp->struct_size != sizeof(dflop_search_params)) return invalid("dflop_search_params struct_size");
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    if (sp->mode & ~(1u | DFLOP_MODE_ORDER4)) return invalid("search mode %u unknown", sp->mode);
    if (sp->K == 0 || sp->K > (1u << 24)) return invalid("K=%u outside 1..2^24", sp->K);
    if (sp->G < 1 || sp->G > 16) return invalid("G=%u outside 1..16", sp->G);
    if (sp->R > 4096) return invalid("R=%u > 4096", sp->R);
    if (D < 1 || D > 4096) return invalid("batches D=%u outside 1..4096", D);
    if (!off) return invalid("batch offsets are NULL");
    uint32_t n_max = 0;
    for (uint32_t b = 0; b < D; ++b) {
        if (off[b + 1] < off[b]) return invalid("batch offsets must be non-decreasing");
        n_max = std::max(n_max, off[b + 1] - off[b]);
    }
    const uint32_t n_tot = off[D] - off[0];
    if (n_max > 65535) {
        set_error("a batch of n=%u > 65535 samples", n_max);
        return DFLOP_ERR_SHAPE;
    }
    if (n_tot > 0 && (!tiles || !frames || !text)) return invalid("feature pointers must be non-NULL");
    if ((uint64_t)sp->seed[1] + D - 1 > 0xFFFFFFFFull) return invalid("seed[1] + D - 1 overflows 32 bits");
    tiles += off[0];
    frames += off[0];
    text += off[0];
    const int dev = current_device();
    const uint32_t gbs = sp->gbs ? sp->gbs : n_max;
    const bool alg1 = (sp->mode & 1u) == DFLOP_SEARCH_ALG1;
    const uint32_t bmode = DFLOP_MODE_HEURISTIC | (sp->mode & DFLOP_MODE_ORDER4);
    uint32_t P = 1, m_max = 0;
    const ConfigTable* tab = nullptr;
    if (alg1) {
        if (!cl || cl->struct_size != sizeof(dflop_cluster)) return invalid("dflop_cluster struct_size");
        if (!mm || mm->struct_size != sizeof(dflop_mem_model)) return invalid("dflop_mem_model struct_size");
        if (cl->n_gpus < 2 || cl->gpus_per_node < 1) return invalid("cluster needs n_gpus >= 2, gpus_per_node >= 1");
        const dflop_mem_grid* gs[4] = {&mm->ms_e, &mm->as_e, &mm->ms_l, &mm->as_l};
        const char* nm[4] = {"ms_e", "as_e", "ms_l", "as_l"};
        for (int q = 0; q < 4; ++q)
            if ((st = validate_mgrid(*gs[q], nm[q])) != DFLOP_OK) return st;
        if (sp->top_p < 1 || sp->top_p > 256) return invalid("top_p=%u outside 1..256", sp->top_p);
        if ((uint64_t)sp->top_p * sp->K > (1u << 24)) return invalid("top_p * K must be <= 2^24");
        if (gbs < 1) return invalid("gbs must be >= 1");
        if ((st = get_config_table(cl->n_gpus, cl->gpus_per_node, gbs, &tab)) != DFLOP_OK) return st;
        P = sp->top_p;
        m_max = gbs;
    } else {
        if ((st = validate_plan(&sp->fixed_plan)) != DFLOP_OK) return st;
        m_max = sp->fixed_plan.n_mb * sp->fixed_plan.l_dp;
    }
    // balance workspace: exact for a fixed plan, bounded for Algorithm 1 (plans unknown yet)
    const int G = comm ? comm->world : 1, g = comm ? comm->rank : 0;
    uint32_t cb, cend;
    dflop_shard_range(sp->K, (uint32_t)g, (uint32_t)G, &cb, &cend);
    size_t bal_bytes = 0;
    if (alg1) {
        bal_bytes = balance_bound(n_max, std::max(1u, m_max), std::max(1u, cend - cb), dev);
    } else if (cend > cb) {
        BalancePlan bp0;
        if ((st = plan_balance(n_max, &sp->fixed_plan, bmode, sp->R, sp->G, cend - cb, &bp0)) != DFLOP_OK)
            return st;
        bal_bytes = bp0.cfg.total;
    }
    const uint32_t PD = P * D;
    const SearchLayout L = search_layout(n_tot, n_max, P, PD, tab ? tab->n_pairs : 0, bal_bytes,
                                         std::min(PD, stage_b_streams()), dev);
    if (!ws) {
        *ws_bytes = L.total;
        return DFLOP_OK;
    }
    if (*ws_bytes < L.total) {
        set_error("workspace %zu B < required %zu B", *ws_bytes, L.total);
        return DFLOP_ERR_WORKSPACE_TOO_SMALL;
    }
    if ((uintptr_t)ws % 256) return invalid("workspace must be 256-byte aligned");
    if (!out) return invalid("out is NULL");
    char* w = reinterpret_cast<char*>(ws);
    uint32_t* costs = reinterpret_cast<uint32_t*>(w + L.o_costs);              // [P][4][n_tot]
    dflop_cand_result* results = reinterpret_cast<dflop_cand_result*>(w + L.o_results);  // [P][D]
    uint32_t* assigns = reinterpret_cast<uint32_t*>(w + L.o_assigns);          // [P][n_tot]
    char* bcast = w + L.o_bcast;
    uint64_t* d_key = reinterpret_cast<uint64_t*>(w + L.o_key);                // [P*D] keys + 2 u32
    StageATop* d_top = reinterpret_cast<StageATop*>(w + L.o_top);
    unsigned long long* d_feas = reinterpret_cast<unsigned long long*>(w + L.o_feas);
    uint32_t* d_status = reinterpret_cast<uint32_t*>(w + L.o_status);
    void* bal_ws = w + L.o_bal;

    dflop_plan_result res;
    memset(&res, 0, sizeof res);
    res.struct_size = sizeof(dflop_plan_result);
    std::vector<dflop_plan> plans;
    std::vector<uint64_t> plan_TA;
    cudaError_t ce = cudaMemsetAsync(d_status, 0, 4, s);
    if (ce != cudaSuccess) return cuda_status(ce, "memset");
    if (alg1) {
        const uint32_t nc = (uint32_t)(tab->cfgs.size() / 6);
        res.n_configs = nc;
        res.n_pairs = tab->n_pairs;
        uint64_t* sa_out = (stage_a_out && stage_a_cap >= tab->n_pairs) ? stage_a_out : nullptr;
        if ((st = stage_a_launch(cm, mm, tab->d_cfgs, tab->d_pair_start, nc, tab->n_pairs, gbs, tiles, frames, text,
                                 n_tot, P, w + L.o_stage_a, sa_out, d_top, d_feas, s)) != DFLOP_OK)
            return st;
        std::vector<StageATop> top(P);
        unsigned long long feas = 0;
        ce = cudaMemcpyAsync(top.data(), d_top, P * sizeof(StageATop), cudaMemcpyDeviceToHost, s);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(&feas, d_feas, sizeof feas, cudaMemcpyDeviceToHost, s);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
        if (ce != cudaSuccess) return cuda_status(ce, "stage A readback");
        res.n_feasible = feas;
        if (feas == 0) {
            set_error("no (config, N_mb) pair satisfies Eq. (4)-(5) with M_gpu = %.0f B", mm->mem_per_gpu);
            return DFLOP_ERR_INFEASIBLE;
        }
        for (uint32_t r = 0; r < P; ++r) {
            if (top[r].T == ~0ull) break;
            const uint32_t pidx = top[r].pair;
            const uint32_t e = (uint32_t)(std::upper_bound(tab->pair_start.begin(), tab->pair_start.end() - 1, pidx) -
                                          tab->pair_start.begin()) - 1;
            const uint32_t* c = &tab->cfgs[6 * (size_t)e];
            dflop_plan pl{c[0], c[1], c[2], c[3], c[4], c[5], pidx - tab->pair_start[e] + 1};
            plans.push_back(pl);
            plan_TA.push_back(top[r].T);
        }
        res.alg1_plan = plans[0];
        res.alg1_makespan = plan_TA[0];
    } else {
        plans.push_back(sp->fixed_plan);
        plan_TA.push_back(0);
    }
    // ---- Stage B: per batch a1 for every plan in one launch, then a2..a5 per (plan, batch) on
    // this rank's shard; (plan, batch) pairs round-robin over the Stage-B streams
    const uint32_t np = (uint32_t)plans.size();
    std::vector<PredictConsts> kc(np);
    for (uint32_t p = 0; p < np; ++p) kc[p] = predict_consts(cm, &plans[p]);
    const size_t pstride = (size_t)4 * n_tot;  // one plan's [4][n_tot] costs
    for (uint32_t b = 0; b < D; ++b) {
        const uint32_t o = off[b] - off[0], nb = off[b + 1] - off[b];
        if (nb == 0) continue;
        // the batch's [4][nb] rows inside each plan's [4][n_tot] block: row r at r*n_tot + o
        ce = predict_launch_rows(cm, kc.data(), np, tiles + o, frames + o, text + o, nb, costs + o, n_tot, pstride,
                                 d_status, s);
        if (ce != cudaSuccess) return cuda_status(ce, "predict launch");
    }
    const uint32_t n_pairs_b = np * D;
    const uint32_t ns = std::min<uint32_t>(L.n_bal, n_pairs_b);
    std::vector<cudaStream_t> ss(ns, s);
    struct Events {
        std::vector<cudaEvent_t> ev;
        ~Events() {
            for (cudaEvent_t e : ev) cudaEventDestroy(e);
        }
        cudaEvent_t make() {
            cudaEvent_t e = nullptr;
            if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
            ev.push_back(e);
            return e;
        }
    } evs;
    if (ns > 1) {
        cudaEvent_t fork = evs.make();
        if (!fork || cudaEventRecord(fork, s) != cudaSuccess) return cuda_status(cudaGetLastError(), "fork event");
        for (uint32_t k = 1; k < ns; ++k) {
            ss[k] = aux_stream(dev, k - 1);
            if (!ss[k]) return cuda_status(cudaGetLastError(), "stage B stream");
            if ((ce = cudaStreamWaitEvent(ss[k], fork, 0)) != cudaSuccess) return cuda_status(ce, "fork wait");
        }
    }
    for (uint32_t p = 0; p < np; ++p) {
        for (uint32_t b = 0; b < D; ++b) {
            const uint32_t q = p * D + b, o = off[b] - off[0], nb = off[b + 1] - off[b];
            cudaStream_t sq = ss[q % ns];
            // an Algorithm-1 plan beyond the balancer's limits (S = E_pp + L_pp > 32, or
            // m = N_mb * L_dp > 65535: possible at >= 34 GPUs) is not balanced: its results say
            // "no candidate", so dflop_select_plan never picks it (include/dflop.h)
            const bool over = plans[p].e_pp + plans[p].l_pp > 32 || (uint64_t)plans[p].n_mb * plans[p].l_dp > 65535u;
            if (cb >= cend || over) {
                // empty shard on this rank: mark the (plan, batch) result as "no candidate"
                ce = cudaMemsetAsync(&results[q], 0xFF, sizeof(dflop_cand_result), sq);
                if (ce != cudaSuccess) return cuda_status(ce, "memset");
                continue;
            }
            BalancePlan bpn;
            if ((st = plan_balance(nb, &plans[p], bmode, sp->R, sp->G, cend - cb, &bpn, !alg1)) != DFLOP_OK)
                return st;
            if (bpn.cfg.total > L.bal_bytes && bpn.cfg.split) {
                // a smaller batch than the bound's: its split chunk may be longer; run it merged
                if ((st = plan_balance(nb, &plans[p], bmode, sp->R, sp->G, cend - cb, &bpn, false)) != DFLOP_OK)
                    return st;
            }
            if (bpn.cfg.total > L.bal_bytes) {
                set_error("internal: balance workspace %zu > bound %zu", bpn.cfg.total, L.bal_bytes);
                return DFLOP_ERR_UNSUPPORTED;
            }
            if (ns > 1) {
                // concurrent plans: the fewest blocks that keep the number of rounds minimal,
                // so the last round is nearly full and the SMs left over run the next plan
                // (a single launch keeps every SM and spreads a partial last round instead)
                for (int v = 0; v < 3; ++v) {
                    const uint32_t cpb = std::max(1u, bpn.cfg.cpb[v]), g = std::max(1u, bpn.cfg.grid[v]);
                    const uint32_t want = (cend - cb + cpb - 1) / cpb, rounds = std::max(1u, (want + g - 1) / g);
                    bpn.cfg.grid[v] = std::max(1u, std::min(g, (want + rounds - 1) / rounds));
                }
            }
            BalanceArgs a{};
            a.cost_ticks = costs + (size_t)p * pstride + o;
            a.cost_stride = n_tot;
            a.sh = bpn.sh;
            a.K = sp->K;
            a.c_begin = cb;
            a.c_end = cend;
            a.seed0 = sp->seed[0];
            a.seed1 = sp->seed[1] + b;
            a.id_base = p * sp->K;
            a.ws = reinterpret_cast<char*>(bal_ws) + (size_t)(q % ns) * L.bal_stride;
            a.best = &results[q];
            a.assign = assigns + (size_t)p * n_tot + o;
            if ((st = balance_launch(a, bpn.cfg, bpn.prog, sq)) != DFLOP_OK) return st;
        }
    }
    for (uint32_t k = 1; k < ns; ++k) {  // join
        cudaEvent_t j = evs.make();
        if (!j || cudaEventRecord(j, ss[k]) != cudaSuccess) return cuda_status(cudaGetLastError(), "join event");
        if ((ce = cudaStreamWaitEvent(s, j, 0)) != cudaSuccess) return cuda_status(ce, "join wait");
    }
    // ---- per (plan, batch) local keys gathered on the device, one NCCL min all-reduce of the
    // [P*D] key array (+ a MAX of the two status flags) in place, one readback for the host's
    // plan choice (protocol.cpp: dflop_select_plan)
    if ((ce = gather_keys_launch(results, n_pairs_b, d_status, d_key, s)) != cudaSuccess)
        return cuda_status(ce, "gather keys");
    if (comm && G > 1) {
        uint32_t* d_bits = reinterpret_cast<uint32_t*>(d_key + n_pairs_b);
        ncclResult_t r = ncclGroupStart();
        if (r == ncclSuccess) r = ncclAllReduce(d_key, d_key, n_pairs_b, ncclUint64, ncclMin, comm->comm, s);
        if (r == ncclSuccess) r = ncclAllReduce(d_bits, d_bits, 2, ncclUint32, ncclMax, comm->comm, s);
        if (r == ncclSuccess) r = ncclGroupEnd();
        if ((st = nccl_status(r, "ncclAllReduce(min keys)")) != DFLOP_OK) return st;
    }
    std::vector<uint64_t> keys(n_pairs_b + 1);
    ce = cudaMemcpyAsync(keys.data(), d_key, (n_pairs_b + 1) * 8, cudaMemcpyDeviceToHost, s);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return cuda_status(ce, "key readback");
    uint32_t gstatus = 0;
    {
        uint32_t bits[2];
        memcpy(bits, &keys[n_pairs_b], 8);
        gstatus = bits[0] | (bits[1] << 1);
    }
    // ---- the plan: argmin over p of (sum_b T_B(b, p), p); for D = 1 the packed key order
    // (T_B, p, c) -- the same choice
    uint32_t win_p = 0xFFFFFFFFu;
    uint64_t best_obj = ~0ull;
    {
        std::vector<uint32_t> batch_n(D);
        std::vector<uint64_t> obj(np);
        for (uint32_t b = 0; b < D; ++b) batch_n[b] = off[b + 1] - off[b];
        if ((st = dflop_select_plan(keys.data(), np, D, batch_n.data(), &win_p, obj.data())) != DFLOP_OK) return st;
        best_obj = obj[win_p];
        for (uint32_t p = 0; p < np; ++p) {
            if (plan_objective) plan_objective[p] = obj[p];
            if (plans_out) plans_out[p] = plans[p];
        }
    }
    // ---- every batch's winner of plan win_p: the owner packs, NCCL broadcasts (G > 1)
    dflop_cand_result first{};
    uint32_t first_c = 0;
    int first_owner = 0;
    for (uint32_t b = 0; b < D; ++b) {
        const uint32_t q = win_p * D + b, o = off[b] - off[0], nb = off[b + 1] - off[b];
        dflop_cand_result win;
        memset(&win, 0, sizeof win);
        uint32_t win_c = 0;
        int owner = 0;
        if (nb > 0 || D == 1) {
            const uint64_t key = keys[q];
            const uint32_t id = (uint32_t)(key & 0xFFFFFFull);
            win_c = id - win_p * sp->K;
            owner = (int)dflop_owner_of(sp->K, win_c, (uint32_t)G);
            if (g == owner) {
                ce = cudaMemcpyAsync(bcast, &results[q], sizeof(dflop_cand_result), cudaMemcpyDeviceToDevice, s);
                if (ce == cudaSuccess && nb > 0)
                    ce = cudaMemcpyAsync(bcast + sizeof(dflop_cand_result), assigns + (size_t)win_p * n_tot + o,
                                         (size_t)nb * 4, cudaMemcpyDeviceToDevice, s);
                if (ce != cudaSuccess) return cuda_status(ce, "winner pack");
            }
            if (comm && G > 1) {
                ncclResult_t r = ncclBroadcast(bcast, bcast, sizeof(dflop_cand_result) + (size_t)nb * 4, ncclUint8,
                                               owner, comm->comm, s);
                if ((st = nccl_status(r, "ncclBroadcast(winner)")) != DFLOP_OK) return st;
            }
            if (assign && nb > 0) {
                ce = cudaMemcpyAsync(assign + o, bcast + sizeof(dflop_cand_result), (size_t)nb * 4,
                                     cudaMemcpyDeviceToDevice, s);
                if (ce != cudaSuccess) return cuda_status(ce, "assign copy");
            }
            ce = cudaMemcpyAsync(&win, bcast, sizeof win, cudaMemcpyDeviceToHost, s);
            if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
            if (ce != cudaSuccess) return cuda_status(ce, "winner readback");
        }
        win.cand = win_c;
        if (batch_out) batch_out[b] = win;
        if (b == 0) {
            first = win;
            first_c = win_c;
            first_owner = owner;
        }
        gstatus |= win.status;
    }
    res.status_bits = gstatus;
    res.plan = plans[win_p];
    res.m = plans[win_p].n_mb * plans[win_p].l_dp;
    res.cand = first_c;
    res.stage_a_rank = alg1 ? win_p : 0;
    res.owner_rank = (uint32_t)first_owner;
    res.makespan = D == 1 ? first.makespan : best_obj;
    res.cmax = first.cmax;
    res.stage_a_makespan = plan_TA[win_p];
    if (!alg1) res.alg1_plan = plans[0];
    res.n_candidates = (uint64_t)np * D * sp->K;
    *out = res;
    if (res.status_bits & DFLOP_DEV_COST_OVERFLOW) {
        set_error("a predicted stage cost rounded to >= 2^32 ticks; raise tick_ns");
        return DFLOP_ERR_OVERFLOW;
    }
    if (res.status_bits & DFLOP_DEV_MAKESPAN_OVERFLOW) {
        set_error("a makespan reached 2^40 ticks; raise tick_ns");
        return DFLOP_ERR_OVERFLOW;
    }
    return DFLOP_OK;
}

}  // namespace dflop

extern "C" dflop_status dflop_route_plan(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan,
                                         const uint32_t* assign, void* ws, size_t* ws_bytes, uint32_t* pos_item,
                                         uint32_t* slot_off, uint32_t* enc_off, uint32_t* llm_off, uint64_t* enc_load,
                                         dflop_stream_t stream) {
    g_err.clear();
    dflop_status st = validate_plan(plan);
    if (st != DFLOP_OK) return st;
    if ((uint64_t)plan->n_mb * plan->l_dp > 65535) return invalid("m = N_mb * L_dp must be <= 65535");
    if (n > 0 && (!cost_ticks || !assign)) return invalid("cost_ticks / assign are NULL");
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    const size_t need = route_ws_bytes(n, plan);
    if (!ws) {
        *ws_bytes = need;
        return DFLOP_OK;
    }
    if (*ws_bytes < need) {
        set_error("workspace %zu B < required %zu B", *ws_bytes, need);
        return DFLOP_ERR_WORKSPACE_TOO_SMALL;
    }
    if ((uintptr_t)ws % 256) return invalid("workspace must be 256-byte aligned");
    if (!slot_off || !enc_off || !llm_off || (n > 0 && !pos_item))
        return invalid("pos_item / slot_off / enc_off / llm_off are NULL");
    return route_launch(cost_ticks, n, plan, assign, ws, pos_item, slot_off, enc_off, llm_off, enc_load,
                        (cudaStream_t)stream);
}

extern "C" dflop_status dflop_order_search(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan,
                                           const uint32_t* assign, uint32_t rounds, void* ws, size_t* ws_bytes,
                                           uint32_t* order_out, uint64_t* T_out, dflop_stream_t stream) {
    g_err.clear();
    dflop_status st = validate_plan(plan);
    if (st != DFLOP_OK) return st;
    if (plan->e_pp + plan->l_pp > 32) return invalid("S = E_pp + L_pp must be <= 32");
    if (plan->n_mb > 65535) return invalid("N_mb must be <= 65535");
    if (n > 0 && (!cost_ticks || !assign)) return invalid("cost_ticks / assign are NULL");
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    const size_t need = order_ws_bytes(plan);
    if (!ws) {
        *ws_bytes = need;
        return DFLOP_OK;
    }
    if (*ws_bytes < need) {
        set_error("workspace %zu B < required %zu B", *ws_bytes, need);
        return DFLOP_ERR_WORKSPACE_TOO_SMALL;
    }
    if ((uintptr_t)ws % 256) return invalid("workspace must be 256-byte aligned");
    if (!order_out || !T_out) return invalid("order_out / T_out are NULL");
    return order_launch(cost_ticks, n, plan, assign, rounds, ws, order_out, T_out, (cudaStream_t)stream);
}

extern "C" dflop_status dflop_exact_cmax(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan,
                                         uint64_t node_budget, const uint32_t* init_assign, void* ws, size_t* ws_bytes,
                                         dflop_exact_result* out, uint32_t* assign, dflop_stream_t stream) {
    g_err.clear();
    dflop_status st = validate_plan(plan);
    if (st != DFLOP_OK) return st;
    if (plan->n_mb > 65535 || plan->l_dp > 65535) return invalid("exact solver: n_mb or l_dp > 65535");
    const uint64_t m64 = (uint64_t)plan->n_mb * plan->l_dp;
    if (m64 > 256) return invalid("exact solver: m = %llu > 256", (unsigned long long)m64);
    const uint32_t m = (uint32_t)m64;
    if (plan->e_pp + plan->l_pp > 32) return invalid("S = E_pp + L_pp must be <= 32");
    if (n > 65535) {
        set_error("n=%u > 65535", n);
        return DFLOP_ERR_SHAPE;
    }
    if (n > 0 && !cost_ticks) return invalid("cost_ticks is NULL");
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    const size_t need = exact_ws_bytes(n, m, plan);
    if (!ws) {
        *ws_bytes = need;
        return DFLOP_OK;
    }
    if (*ws_bytes < need) {
        set_error("workspace %zu B < required %zu B", *ws_bytes, need);
        return DFLOP_ERR_WORKSPACE_TOO_SMALL;
    }
    if ((uintptr_t)ws % 256) return invalid("workspace must be 256-byte aligned");
    if (!out) return invalid("out is NULL");
    return exact_launch(cost_ticks, n, plan, node_budget, init_assign, ws, out, assign, (cudaStream_t)stream);
}

extern "C" dflop_status dflop_search_plans(const dflop_cluster* cl, const dflop_cost_model* cm,
                                           const dflop_mem_model* mm, const uint32_t* tiles, const uint32_t* frames,
                                           const uint32_t* text, uint32_t n, const dflop_search_params* sp,
                                           dflop_comm* comm, void* ws, size_t* ws_bytes, dflop_plan_result* out,
                                           uint32_t* assign, uint64_t* stage_a_out, uint64_t stage_a_cap,
                                           dflop_stream_t stream) {
    const uint32_t off[2] = {0, n};
    return search_impl(cl, cm, mm, tiles, frames, text, off, 1, sp, comm, ws, ws_bytes, out, nullptr, nullptr, nullptr,
                       assign, stage_a_out, stage_a_cap, (cudaStream_t)stream);
}

extern "C" dflop_status dflop_search_plans_batches(const dflop_cluster* cl, const dflop_cost_model* cm,
                                                   const dflop_mem_model* mm, const uint32_t* tiles,
                                                   const uint32_t* frames, const uint32_t* text,
                                                   const uint32_t* batch_offsets, uint32_t n_batches,
                                                   const dflop_search_params* sp, dflop_comm* comm, void* ws,
                                                   size_t* ws_bytes, dflop_plan_result* out,
                                                   dflop_cand_result* batch_results, uint64_t* plan_objective,
                                                   dflop_plan* plans_out, uint32_t* assign, dflop_stream_t stream) {
    return search_impl(cl, cm, mm, tiles, frames, text, batch_offsets, n_batches, sp, comm, ws, ws_bytes, out,
                       batch_results, plan_objective, plans_out, assign, nullptr, 0, (cudaStream_t)stream);
}
