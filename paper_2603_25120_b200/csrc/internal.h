// internal.h -- host-side declarations shared by the libdflop translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dflop.h"

namespace dflop {

void set_error(const char* fmt, ...);

// cached device attributes (cudaGetDeviceProperties is slow; attributes are queried once)
struct DevAttr {
    int sms;
    size_t smem_optin;     // max dynamic shared memory per block (opt-in)
    size_t smem_per_sm;
};
DevAttr dev_attr(int device);

// instrumentation (profile.cpp)
void count_launches(uint32_t k);
bool profiling();
// returns an index to pass to prof_mark(); -1 when profiling is off
int prof_begin(cudaStream_t s);
void prof_mark(int idx, int which, cudaStream_t s);  // which: 1 = between variants, 2 = end
// Stage-A kernel timing (dflop_profile.stage_a_ms): begin returns a mark index or -1
int prof_stage_begin(cudaStream_t s);
void count_split_chunks(uint32_t k);
void prof_stage_end(int idx, cudaStream_t s);
dflop_status cuda_status(cudaError_t e, const char* what);

// ---------------------------------------------------------------- predict
struct PredictConsts {
    float scale_e, scale_att, scale_lin, bwd;
    uint32_t tau_tile, tau_frame;
    float tp_e, tp_l;
};
dflop_status validate_cost_model(const dflop_cost_model* m);
dflop_status validate_plan(const dflop_plan* p);
PredictConsts predict_consts(const dflop_cost_model* m, const dflop_plan* p);
cudaError_t predict_launch(const dflop_cost_model* m, const PredictConsts* consts, uint32_t n_plans,
                           const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                           float* cost_f32, uint32_t* cost_ticks, size_t plan_stride, uint32_t* dev_status,
                           cudaStream_t s);
// ticks only, rows `row_stride` apart inside each plan's block of plan_stride entries
cudaError_t predict_launch_rows(const dflop_cost_model* m, const PredictConsts* consts, uint32_t n_plans,
                                const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                                uint32_t* cost_ticks, size_t row_stride, size_t plan_stride, uint32_t* dev_status,
                                cudaStream_t s);

// ---------------------------------------------------------------- 1F1B slot program
struct SlotProgram {
    uint32_t S = 0, M = 0, D = 0;  // D = ring depth (power of two)
    const uint32_t* d_ops = nullptr;     // device copy, 2*S*M entries
    const uint32_t* d_levels = nullptr;  // device, n_levels + 1 offsets into d_ops
    const uint32_t* d_dense = nullptr;   // device, [n_levels][S]: stage s's op at level L, or kNoOp
    uint32_t n_ops = 0, n_levels = 0;
};
constexpr uint32_t kNoOp = 0xFFFFFFFFu;
// Builds (once per (S, M) and device) a topological order of the 1F1B DAG by Kahn levels.
dflop_status get_slot_program(uint32_t S, uint32_t M, SlotProgram* out);
void release_slot_programs();

// ---------------------------------------------------------------- balance
struct BalanceShape {
    uint32_t n, m, S, e_pp, l_dp, n_mb;
    uint32_t mode, R, G;
    uint32_t n_cand;  // cand_end - cand_begin
    uint32_t D;       // 1F1B ring depth of the slot program
    uint32_t split_ok = 0;  // the split pipeline may be used (fixed-plan calls)
};
struct BalanceConfig {
    int gl = 1;                        // lanes per candidate
    uint32_t cap = 0;                  // refinement: member-list entries copied to shared memory
    uint32_t sigma = 0;                // refinement: free entries per bucket in the CSR member lists
    uint32_t csr_len = 0;              // refinement: u16 entries of one slot's CSR lists
    bool cnt_smem = true;              // refinement: list counters/offsets in shared memory
    uint32_t apos_bytes = 0;           // one assignment buffer (u8 or u16 per position)
    // per kernel variant: [0] packed u32, [1] plain u32, [2] u64 (cand.cuh)
    bool tbl_smem[3] = {false, false, false};  // item table staged in shared memory
    uint32_t tbl_bytes[3] = {0, 0, 0};
    uint32_t cand_bytes[3] = {0, 0, 0};        // per-candidate smem
    uint32_t off_fl[3] = {0, 0, 0}, off_scr[3] = {0, 0, 0};
    uint32_t cpb[3] = {0, 0, 0};               // candidates per block
    uint32_t grid[3] = {0, 0, 0};
    uint32_t n_slots = 0;
    // split pipeline (packed variant only): k_lpt with lpt_gl lanes per candidate, then the
    // candidate kernel on its output, over chunks of lpt_chunk candidates
    bool split = false;

    int lpt_gl = 0;
    uint32_t lpt_cpb = 0, lpt_grid = 0, lpt_tbl = 0, lpt_cb = 0, lpt_chunk = 0;
    // workspace layout (byte offsets)
    size_t o_hdr, o_keys, o_order, o_item_pos, o_items32, o_items64, o_slot_key, o_slot_T, o_slot_cmax,
        o_slot_buf, o_slot_apos, o_slot_csr, o_grp, o_lpt_apos = 0, o_lpt_el = 0, total;
    bool ok = false;
    std::string why;
};
BalanceConfig balance_config(const BalanceShape& sh, int device);
// Launches the whole a2..a5 sequence for one plan on `stream`.
struct BalanceArgs {
    const uint32_t* cost_ticks;  // rows ef, eb, lf, lb of n entries, cost_stride apart (0 = n)
    size_t cost_stride;
    BalanceShape sh;
    uint32_t K, c_begin, c_end, seed0, seed1, id_base;
    void* ws;
    dflop_cand_result* best;
    uint32_t* assign;
    uint64_t* cand_T;
    uint64_t* cand_cmax;
};
dflop_status balance_launch(const BalanceArgs& a, const BalanceConfig& cfg, const SlotProgram& prog,
                            cudaStream_t s);

dflop_status simulate_launch(const uint64_t* fwd, const uint64_t* bwd, uint32_t C, uint32_t S, uint32_t M,
                             uint64_t* makespan, uint64_t* busy, const SlotProgram& prog, cudaStream_t s);

size_t groups_ws_bytes(uint32_t n, uint32_t m);

#ifdef __CUDACC__
// a2 kernels shared by the balance and the exact solver (balance.cu; types from common.cuh)
__global__ void k_prep_keys(const uint32_t* __restrict__ cost, uint32_t n, size_t rs, BalanceHeader* hdr, u64* keys);
__global__ void k_rank_sort(const u64* __restrict__ keys, uint32_t n, uint32_t* order, uint32_t* item_pos);
// LPT base order (rank sort above, or a one-CTA bitonic sort for n <= 8192)
void order_launch_keys(const u64* keys, uint32_t n, uint32_t* order, uint32_t* item_pos, cudaStream_t s);
#endif

// ---------------------------------------------------------------- N4(b) routing plan (route.cu)
size_t route_ws_bytes(uint32_t n, const dflop_plan* p);
dflop_status route_launch(const uint32_t* cost, uint32_t n, const dflop_plan* p, const uint32_t* assign, void* ws,
                          uint32_t* pos_item, uint32_t* slot_off, uint32_t* enc_off, uint32_t* llm_off,
                          uint64_t* enc_load, cudaStream_t s);

// ---------------------------------------------------------------- N4(a) order search (order.cu)
size_t order_ws_bytes(const dflop_plan* p);
dflop_status order_launch(const uint32_t* cost, uint32_t n, const dflop_plan* p, const uint32_t* assign,
                          uint32_t rounds, void* ws, uint32_t* order_out, uint64_t* T_host, cudaStream_t s);

// ---------------------------------------------------------------- N3 exact C_max (exact.cu)
size_t exact_ws_bytes(uint32_t n, uint32_t m, const dflop_plan* p);
dflop_status exact_launch(const uint32_t* cost, uint32_t n, const dflop_plan* p, uint64_t node_budget,
                          const uint32_t* init_assign, void* ws, dflop_exact_result* out, uint32_t* assign,
                          cudaStream_t s);
cudaError_t gather_keys_launch(const dflop_cand_result* res, uint32_t n, const uint32_t* d_status, uint64_t* key,
                               cudaStream_t s);
cudaError_t groups_launch(const uint32_t* assign, uint32_t n, uint32_t m, uint32_t* offsets, uint32_t* items,
                          void* ws, cudaStream_t s);

// ---------------------------------------------------------------- stage A
struct StageAConsts;  // defined in stage_a.cu
struct StageATop {
    uint64_t T;
    uint32_t pair;
    uint32_t pad;
};
size_t stage_a_ws_bytes(uint64_t n_pairs, int device);
dflop_status stage_a_launch(const dflop_cost_model* cm, const dflop_mem_model* mm, const uint32_t* d_cfgs,
                            const uint32_t* d_pair_start, uint32_t n_cfgs, uint64_t n_pairs, uint32_t gbs,
                            const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                            uint32_t top_p, void* ws, uint64_t* stage_a_out, StageATop* d_top,
                            unsigned long long* d_n_feasible, cudaStream_t s);

}  // namespace dflop
