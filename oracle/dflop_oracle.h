/*
 * dflop_oracle.h -- ORACLE header.  TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU reference for the DFLOP plan-candidate path
 * (arXiv 2603.25120, "DFLOP: A Data-driven Framework for Multimodal LLM Training
 * Pipeline Optimization").  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load it.  The product path
 * (paper_2603_25120_b200/, include/dflop.h) never includes, links or executes
 * anything under oracle/, and this header shares nothing with include/dflop.h.
 *
 * Citations: "P:n" = PAPER.md line n; "S:n" = SPEC.md line n; "R<k>" = the
 * reading number k in DESIGN.md section 3 (the ambiguity register).
 */
#ifndef DFLOP_ORACLE_H
#define DFLOP_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_MAX_X 32
#define ORC_MAX_TP 4

/* Throughput grid X(x, tp) in FLOP/s per GPU, measured at knots. */
typedef struct orc_grid {
    uint32_t n_x;                       /* 1..32 shape knots   */
    uint32_t n_tp;                      /* 1..4  TP knots      */
    double x[ORC_MAX_X];                /* strictly increasing */
    double tp[ORC_MAX_TP];              /* strictly increasing */
    double v[ORC_MAX_TP][ORC_MAX_X];    /* v[a][k] at (x_k, tp_a) */
} orc_grid;

/* Memory grid M(l, tp, x) in bytes: two layer counts, TP knots, shape knots. */
typedef struct orc_mgrid {
    uint32_t n_x;
    uint32_t n_tp;
    double l[2];
    double tp[ORC_MAX_TP];
    double x[ORC_MAX_X];
    double v[2][ORC_MAX_TP][ORC_MAX_X];
} orc_mgrid;

/* MLLM cost model: encoder + LLM shapes (Table 1) and profiled grids. */
typedef struct orc_model {
    uint32_t e_layers;   /* E_l                                    */
    uint32_t e_hidden;   /* h_E                                    */
    uint32_t e_seq;      /* E_seq_len: tokens per encoder instance */
    uint32_t e_attn;     /* 1: add in-tile attention 4*h_E*E_seq^2 */
    uint32_t l_layers;   /* L_l                                    */
    uint32_t l_hidden;   /* h_L                                    */
    uint32_t tau_tile;   /* LLM tokens per image tile              */
    uint32_t tau_frame;  /* LLM tokens per video frame             */
    double bwd_ratio;    /* backward / forward (2.0)        */
    double tick_ns;      /* integer time unit in ns (R19)          */
    orc_grid thr_e;      /* E_thr(b, E_tp)                         */
    orc_grid thr_att;    /* L_attn_thr(s, L_tp)                    */
    orc_grid thr_lin;    /* L_lin_thr(s, L_tp)                     */
} orc_model;

typedef struct orc_mem {
    orc_mgrid ms_e;      /* model_state_E(l, E_tp)        */
    orc_mgrid as_e;      /* act_state_E(l, E_tp, b)       */
    orc_mgrid ms_l;      /* model_state_L(l, L_tp)        */
    orc_mgrid as_l;      /* act_state_L(l, L_tp, s)       */
    double mem_per_gpu;  /* M_gpu, bytes                  */
} orc_mem;

/* theta = (E_tp, E_pp, E_dp, L_tp, L_pp, L_dp, N_mb). */
typedef struct orc_plan {
    uint32_t e_tp, e_pp, e_dp, l_tp, l_pp, l_dp, n_mb;
} orc_plan;

#define ORC_MODE_EXHAUSTIVE 1u  /* candidate c = base-m digits                          */
#define ORC_MODE_ORDER4 16u     /* score each replica under its best of the four start
                                   orders of N4(a) (R37) instead of the slot order       */
typedef struct orc_bparams {
    uint32_t mode;       /* 0 = heuristic candidate family, ORC_MODE_* bits */
    uint32_t K;          /* family size                                   */
    uint32_t R;          /* refinement rounds                             */
    uint32_t G;          /* perturbation group size 1..16                 */
    uint32_t seed[2];    /* Philox key                                    */
} orc_bparams;

/* Status codes (mirrors the meaning, not the header, of the product ABI). */
#define ORC_OK 0
#define ORC_INVALID 1
#define ORC_OVERFLOW 3
#define ORC_INFEASIBLE 4

/* Philox4x32-10 (Salmon et al., SC'11), from its specification. */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint32_t orc_mulhi32(uint32_t u, uint32_t n);

/* Linear interpolation, R3: clamped multilinear, (1-w)a + w b form. */
double orc_interp_thr(const orc_grid* g, double x, double tp);
double orc_interp_mem(const orc_mgrid* g, double l, double tp, double x);

/* Step a1: per-item stage costs (O1-O4).  cost_f64[4][n] in ns (ef, eb, lf, lb),
 * cost_q[4][n] in ticks.  Returns ORC_OVERFLOW (and the first index in *bad) when a cost
 * rounds to >= 2^32 ticks. */
int orc_predict(const orc_model* m, const orc_plan* p, const uint32_t* tiles, const uint32_t* frames,
                const uint32_t* text, uint32_t n, double* cost_f64, uint32_t* cost_q, uint32_t* bad);

/* N1 Adaptive Correction (Eq. (6) B = Th_actual - Th_pred; S:374-377,
 * S:383-386): rho[g][q] = Th_actual / Th_pred for throughput grid g (0 = E_thr on b,
 * 1 = L_attn_thr on s, 2 = L_lin_thr on s) and shape bin q = floor(log2 x) (x = 0 -> 0,
 * clamped to ORC_CORR_BINS - 1) (R30).  With rho != NULL the predicted throughput of a
 * sample is replaced by the corrected one, Th_pred * rho ("predictions for
 * shape-buckets with recorded deviations are replaced by the corrected throughput");
 * rho == NULL is orc_predict. */
#define ORC_CORR_BINS 32
uint32_t orc_shape_bin(uint64_t x);
int orc_predict_corrected(const orc_model* m, const orc_plan* p, const uint32_t* tiles, const uint32_t* frames,
                          const uint32_t* text, uint32_t n, const double* rho, double* cost_f64, uint32_t* cost_q,
                          uint32_t* bad);

/* N1 tracker, written from SPEC's operations:
 *   record_observation(grid, x, Th_actual, Th_pred): the bucket (grid, orc_shape_bin(x))
 *     keeps the exponential average of the observed throughput (weight alpha; the first
 *     observation initialises it, R32) and the latest prediction; returns the bucket's
 *     deviation B = Th_actual_avg - Th_pred (Eq. (6)).
 *   rho[g][q] = Th_actual_avg / Th_pred of a recorded bucket, 1 otherwise (R31).
 *   cost_benefit(benefits): appends the realised benefits; while active and at least I
 *     benefits are known, active <- (mean of the last I) > C; off is permanent. */
#define ORC_TRACK_WIN 4096
typedef struct orc_tracker {
    double alpha, cost;
    uint32_t window, active;
    double observed[3][ORC_CORR_BINS], predicted[3][ORC_CORR_BINS];
    uint8_t seen[3][ORC_CORR_BINS];
    uint64_t n_benefits;                 /* benefits appended so far      */
    double last[ORC_TRACK_WIN];          /* ring of the latest benefits   */
} orc_tracker;
int orc_tracker_init(orc_tracker* t, double alpha, uint32_t window, double cost);
double orc_tracker_record(orc_tracker* t, uint32_t grid, uint64_t x, double th_actual, double th_pred);
void orc_tracker_rho(const orc_tracker* t, double* rho /* [3][ORC_CORR_BINS] */);
uint32_t orc_tracker_cost_benefit(orc_tracker* t, const double* benefits, uint32_t nb);

/* Step a2: base order pi: key max(e_i, l_i) descending, index ascending. */
void orc_base_order(const uint32_t* cost_q, uint32_t n, uint32_t* order);

/* Step a4 building block: non-interleaved 1F1B over S stages x M microbatches,
 * worklist evaluation.  fwd/bwd are [S][M] row-major.  stage_busy[S] may be NULL. */
int orc_simulate_1f1b(const uint64_t* fwd, const uint64_t* bwd, uint32_t S, uint32_t M,
                      uint64_t* makespan, uint64_t* stage_busy);

/* Steps a3+a4 for one candidate c.  assign[n] (may be NULL) receives the bucket of item i. */
int orc_run_candidate(const uint32_t* cost_q, uint32_t n, const orc_plan* p, const orc_bparams* bp,
                      const uint32_t* order, uint32_t c, uint32_t* assign, uint64_t* T, uint64_t* cmax);

/* Steps a2..a5 over candidates [c0, c1).  cand_T / cand_cmax (may be NULL) get per-candidate
 * scores; the lexicographic minimum of (T, c) is returned with its assignment. */
int orc_balance(const uint32_t* cost_q, uint32_t n, const orc_plan* p, const orc_bparams* bp,
                uint32_t c0, uint32_t c1, uint64_t* cand_T, uint64_t* cand_cmax,
                uint64_t* best_T, uint32_t* best_c, uint64_t* best_cmax, uint32_t* best_assign);

/* N3 exact C_max (P:703-727 ILP objective; S:390-398 solve_exact): node-budgeted
 * branch and bound over item -> bucket assignments, items in the base order pi, children
 * in (resulting max(E_j + e, L_j + l), j) order, bucket first-use symmetry breaking (an
 * item may open only the lowest unused bucket), prune when max(node max, LB) >= incumbent.
 * LB = max(ceil(sum e / m), ceil(sum l / m), max_i max(e_i, l_i)).  The incumbent starts
 * from init_assign (its C_max) or, if NULL, from the paper's LPT (current-load rule).
 * proven = the search finished within node_budget child visits (or incumbent == LB).
 * assign_out[n] (may be NULL) receives the best assignment found. */
int orc_exact_cmax(const uint32_t* cost_q, uint32_t n, uint32_t m, uint64_t node_budget,
                   const uint32_t* init_assign, uint32_t* assign_out, uint64_t* cmax, uint64_t* lower_bound,
                   uint32_t* proven, uint64_t* nodes);

/* N3 certificate for m = 2 and m = 4 buckets (n <= 40): exact C_max by pair decomposition.
 * m = 2: the minimum over subsets Y (item 0 in Y) of max(E(Y), L(Y), E - E(Y), L - L(Y)).
 * m = 4: buckets {0, 1} form a set X (item 0 in X, by symmetry), {2, 3} its complement; the
 * optimum is min over X of max(split2(X), split2(complement)), split2 = the m = 2 optimum of a
 * set.  Every X whose sums E(X), L(X) lie in [S - 2C, 2C] for C = best value so far - 1 is split (no
 * 4-way assignment with max < incumbent has X outside that window); exhaustive, so the result
 * is the optimum (a certificate), the incumbent (init_assign's C_max or the paper's LPT) when
 * nothing beats it.  visited = subsets X (m = 4) or Y (m = 2) enumerated. */
int orc_exact_pairs(const uint32_t* cost_q, uint32_t n, uint32_t m, const uint32_t* init_assign, uint32_t* assign_out,
                    uint64_t* cmax, uint64_t* lower_bound, uint64_t* visited);

/* N4(a) microbatch-order search (R11: the 1F1B makespan depends on the slot order; SURVEY
 * 8(f) N4).  For each LLM replica rho (buckets j = k * L_dp + rho, slot k by default, R10)
 * independently: start from the best of four orders -- 0 identity, 1 ascending W_j =
 * max(E_j, L_j), 2 descending W_j, 3 valley (ascending W placed alternately at the front and
 * the back, the largest in the middle); ties by (makespan, order index), sorts stable by
 * slot -- then best-improvement pairwise swaps of slot positions (a < b; every pair when
 * M <= 128, else b - a <= 16), the lexicographic minimum of (makespan, a, b), applied while
 * it is strictly better, at most `rounds` times (R35).  order_out[rho * M + k] = bucket of
 * slot k; T_out[rho] = its makespan.  T of the plan = max over replicas. */
int orc_order_search(const uint32_t* cost_q, uint32_t n, const orc_plan* p, const uint32_t* assign,
                     uint32_t rounds, uint32_t* order_out, uint64_t* T_out);

/* N4(b) inter-model routing plan (Fig. "inter_model_comm"): for microbatch slot k
 * the L_dp LLM data groups run buckets k * L_dp + rho (R10); the E_dp encoder data groups
 * split the slot's samples -- concatenated in (rho, sample index) order -- into E_dp
 * contiguous ranges balanced by encoder cost e_i = ef + eb: range g starts at the first
 * position t with (sum of e before t) * E_dp >= g * (slot total) (R36).  The communicator
 * gathers encoder range g and scatters it to the LLM ranges (forward; reversed backward).
 * Outputs: pos_item[n] (the sample at each position, slot-major), slot_off[N_mb + 1],
 * enc_off[N_mb][E_dp + 1] and llm_off[N_mb][L_dp + 1] (absolute positions), enc_load
 * [N_mb][E_dp] (sum of e per encoder range; may be NULL). */
int orc_route_plan(const uint32_t* cost_q, uint32_t n, const orc_plan* p, const uint32_t* assign,
                   uint32_t* pos_item, uint32_t* slot_off, uint32_t* enc_off, uint32_t* llm_off, uint64_t* enc_load);

/* CSR index groups ("returns a set of index groups"): bucket-major, items ascending. */
void orc_groups(const uint32_t* assign, uint32_t n, uint32_t m, uint32_t* offsets, uint32_t* items);

/* Algorithm 1 phase 1. */
uint32_t orc_find_combs(uint32_t gpus, uint32_t gpus_per_node, uint32_t* out3, uint32_t cap);
uint64_t orc_enumerate_configs(uint32_t n_gpus, uint32_t gpus_per_node, uint32_t* out6, uint64_t cap);

/* Batch means b-bar, s-bar, integer sums divided by n. */
void orc_batch_means(const orc_model* m, const uint32_t* tiles, const uint32_t* frames,
                     const uint32_t* text, uint32_t n, double* mean_b, double* mean_s);

/* Algorithm 1 phase 2 for one (config, i) pair: returns 1 if feasible and writes T_A. */
int orc_stage_a_pair(const orc_model* m, const orc_mem* mm, const uint32_t cfg6[6], uint32_t i,
                     uint32_t gbs, double mean_b, double mean_s, uint64_t* T_A,
                     double* mem_e, double* mem_l, uint64_t* e_dur, uint64_t* l_dur);

/* Stage A over every config and i = 1..GBS//L_dp, in enumeration order.  T_A[pair] is
 * UINT64_MAX when infeasible.  Returns the number of pairs written (<= cap). */
uint64_t orc_stage_a_all(const orc_model* m, const orc_mem* mm, uint32_t n_gpus, uint32_t gpus_per_node,
                         uint32_t gbs, double mean_b, double mean_s, uint64_t* T_A, uint64_t cap);

/* Top-P feasible pairs by (T_A, eps, i): writes pair indices (enumeration order) into top[]. */
uint32_t orc_stage_a_top(const uint64_t* T_A, uint64_t n_pairs, uint32_t P, uint64_t* top);

#ifdef __cplusplus
}
#endif
#endif
