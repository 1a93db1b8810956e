/*
 * dflop.h -- C ABI of libdflop.so, the B200-native (sm_100a) hot path of DFLOP
 * (arXiv 2603.25120, "DFLOP: A Data-driven Framework for Multimodal LLM Training
 * Pipeline Optimization").
 *
 * The library evaluates training-plan candidates for one global batch:
 *   a1 predict   per-sample stage costs from data features
 *   a2 order     the LPT base order
 *   a3 balance   seeded LPT + pairwise-swap partitions into m = N_mb * L_dp buckets
 *                (problem statement: the scheduler ILP)
 *   a4 score     non-interleaved 1F1B makespan of each partition (Fig. 1)
 *   a5 argmin    over candidates (and over GPUs through NCCL)
 *   a6 search    Algorithm 1 over (TP, PP, DP) x N_mb, then a1-a5 on the best plans
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; Rk = DESIGN.md reading k.
 *
 * Conventions (all entry points):
 *   - Every function returns a dflop_status; no C++ exception crosses the ABI.
 *   - On a validation error nothing is launched and no output is written;
 *     dflop_last_error() (thread-local) describes the first violated condition.
 *   - "device" pointers are CUDA global-memory pointers on the current device
 *     (e.g. torch tensor data_ptr()); "host" pointers are ordinary memory.  The
 *     library never retains a caller pointer after return and never frees one.
 *   - stream is a cudaStream_t passed as void*; NULL = the legacy default stream.
 *   - Time is an integer count of ticks of cost_model.tick_ns nanoseconds (R19):
 *     per-sample stage costs are u32, sums and makespans u64.
 *   - Limits: n <= 65535 samples, m = n_mb * l_dp <= 65535 buckets, S = e_pp + l_pp
 *     <= 32 stages, K <= 2^24 candidates, makespan < 2^40 ticks.
 *   - Structs that carry struct_size must have it set to sizeof(struct) (versioning).
 */
#ifndef DFLOP_H
#define DFLOP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFLOP_ABI_VERSION 5u

typedef int32_t dflop_status;
#define DFLOP_OK 0
#define DFLOP_ERR_INVALID_ARGUMENT 1
#define DFLOP_ERR_SHAPE 2
#define DFLOP_ERR_OVERFLOW 3
#define DFLOP_ERR_INFEASIBLE 4
#define DFLOP_ERR_CUDA 5
#define DFLOP_ERR_NCCL 6
#define DFLOP_ERR_WORKSPACE_TOO_SMALL 7
#define DFLOP_ERR_UNSUPPORTED 8

/* Device status word bits (written by kernels into a caller-provided u32). */
#define DFLOP_DEV_COST_OVERFLOW 1u     /* a predicted cost rounded to >= 2^32 ticks  */
#define DFLOP_DEV_MAKESPAN_OVERFLOW 2u /* a makespan >= 2^40 ticks (packed argmin key) */

typedef void* dflop_stream_t; /* cudaStream_t */

#define DFLOP_MAX_X 32
#define DFLOP_MAX_TP 4

/* A profiled throughput grid X(x, tp) in FLOP/s per GPU (Model Profiler).
 * Interpolation is clamped multilinear (R3).  x: shape knots (encoder effective batch b
 * or LLM sequence length s), strictly increasing; tp: TP-degree knots, strictly
 * increasing; v[a][k] > 0 is the value at (x[k], tp[a]). */
typedef struct dflop_grid {
    uint32_t n_x;  /* 1..32 */
    uint32_t n_tp; /* 1..4  */
    double x[DFLOP_MAX_X];
    double tp[DFLOP_MAX_TP];
    double v[DFLOP_MAX_TP][DFLOP_MAX_X];
} dflop_grid;

/* A profiled memory grid M(l, tp, x) in bytes (Memory Profiling): two layer
 * counts l[0] < l[1] (linear in between and beyond), TP knots and shape knots (n_x = 1
 * for model-state grids, which do not depend on the input shape). */
typedef struct dflop_mem_grid {
    uint32_t n_x;
    uint32_t n_tp;
    double l[2];
    double tp[DFLOP_MAX_TP];
    double x[DFLOP_MAX_X];
    double v[2][DFLOP_MAX_TP][DFLOP_MAX_X];
} dflop_mem_grid;

/* Adaptive Correction (N1; Eq. (6) B = Th_actual - Th_pred).
 * rho[g][q] = Th_actual / Th_pred (the host tracker's exponential average) for throughput
 * grid g (0 = thr_e on the encoder batch b, 1 = thr_att and 2 = thr_lin on the LLM length s)
 * and shape bin q = floor(log2 x) (x = 0 -> 0, clamped to DFLOP_CORR_BINS - 1) (R30).  When
 * `active`, a1 divides each sample's FLOPs by Th_pred * rho instead of Th_pred; a
 * bin with rho = 1 is unchanged.  rho must be finite and > 0.  Host memory, read during the
 * call only. */
#define DFLOP_CORR_BINS 32
typedef struct dflop_correction {
    uint32_t struct_size;
    uint32_t active;                    /* 0: ignored (the cost-benefit rule switched it off) */
    float rho[3][DFLOP_CORR_BINS];
} dflop_correction;

/* The MLLM cost model (Table 1 symbols; FLOP accounting R1). */
typedef struct dflop_cost_model {
    uint32_t struct_size;
    uint32_t e_layers;   /* E_l                                                 */
    uint32_t e_hidden;   /* encoder hidden size h_E                             */
    uint32_t e_seq;      /* E_seq_len: tokens per encoder instance      */
    uint32_t e_attn;     /* 1 = add in-instance attention 4*h_E*E_seq^2 FLOPs   */
    uint32_t l_layers;   /* L_l                                                 */
    uint32_t l_hidden;   /* LLM hidden size h_L                                 */
    uint32_t tau_tile;   /* LLM tokens contributed by one image tile            */
    uint32_t tau_frame;  /* LLM tokens contributed by one video frame           */
    uint32_t reserved;
    double bwd_ratio;    /* backward / forward duration (2.0)            */
    double tick_ns;      /* integer time unit, ns (> 0)                         */
    dflop_grid thr_e;    /* E_thr(b, E_tp)                                      */
    dflop_grid thr_att;  /* L_attn_thr(s, L_tp)                                 */
    dflop_grid thr_lin;  /* L_lin_thr(s, L_tp)                                  */
    const dflop_correction* correction; /* N1, NULL = none; used by a1 (predict and the
                                            search's Stage B), not by Stage A (R31)    */
} dflop_cost_model;

/* Memory model for Eq. (4)-(5). */
typedef struct dflop_mem_model {
    uint32_t struct_size;
    uint32_t reserved;
    dflop_mem_grid ms_e; /* model_state_E(l, E_tp)        */
    dflop_mem_grid as_e; /* act_state_E(l, E_tp, b)       */
    dflop_mem_grid ms_l; /* model_state_L(l, L_tp)        */
    dflop_mem_grid as_l; /* act_state_L(l, L_tp, s)       */
    double mem_per_gpu;  /* M_gpu, bytes                  */
} dflop_mem_model;

/* theta = (E_tp, E_pp, E_dp, L_tp, L_pp, L_dp, N_mb).  Buckets m = N_mb * L_dp
 * (P:695); bucket j runs on LLM replica j % L_dp as microbatch slot j / L_dp (R10). */
typedef struct dflop_plan {
    uint32_t e_tp, e_pp, e_dp, l_tp, l_pp, l_dp, n_mb;
} dflop_plan;

/* The modelled cluster of Algorithm 1 (N_gpus, N_gpu_node; M_gpu is in dflop_mem_model). */
typedef struct dflop_cluster {
    uint32_t struct_size;
    uint32_t n_gpus;
    uint32_t gpus_per_node;
    uint32_t reserved;
} dflop_cluster;

#define DFLOP_MODE_HEURISTIC 0u  /* the seeded LPT + swap-refinement family       */
#define DFLOP_MODE_EXHAUSTIVE 1u /* candidate c = base-m digits of c (m^n <= K)    */
/* N4(a) per candidate (R37), OR-ed into dflop_balance_params.mode or
 * dflop_search_params.mode: every replica of a candidate is scored under its best of the
 * four start orders of dflop_order_search (slot order, W ascending, W descending, valley);
 * T = the max over replicas of that minimum.  The winner's slot order is
 * dflop_order_search(assign, rounds = 0). */
#define DFLOP_MODE_ORDER4 16u

/* Candidate family.  c = 0: the paper's LPT (current-load rule,
 * P:738); c = 1: resulting-max LPT (R12); c >= 2: Philox-perturbed order, resulting-max
 * LPT, then R swap-refinement rounds.  This call evaluates c in [cand_begin, cand_end). */
typedef struct dflop_balance_params {
    uint32_t struct_size;
    uint32_t mode;       /* DFLOP_MODE_*                              */
    uint32_t K;          /* family size, 1..2^24                      */
    uint32_t cand_begin; /* shard of the family evaluated by the call */
    uint32_t cand_end;
    uint32_t R;          /* refinement rounds (<= 4096)               */
    uint32_t G;          /* perturbation group size, 1..16            */
    uint32_t seed[2];    /* Philox-4x32-10 key                        */
    uint32_t id_base;    /* added to c in the packed argmin key       */
} dflop_balance_params;

/* Device-resident result of dflop_balance_microbatches (the argmin over the shard). */
typedef struct dflop_cand_result {
    uint64_t key;      /* (makespan << 24) | (id_base + c*): the packed argmin key  */
    uint64_t makespan; /* T of the winner, ticks                                    */
    uint64_t cmax;     /* C_max = max_j max(E_j, L_j) of the winner         */
    uint32_t cand;     /* c* (lowest id among equal makespans, R18)                 */
    uint32_t status;   /* DFLOP_DEV_* bits                                          */
} dflop_cand_result;

#define DFLOP_SEARCH_FIXED 0u /* theta given: Stage B only (configs with a fixed plan) */
#define DFLOP_SEARCH_ALG1 1u  /* Algorithm 1 Stage A over all (config, N_mb), then B   */

typedef struct dflop_search_params {
    uint32_t struct_size;
    uint32_t mode;         /* DFLOP_SEARCH_*                                   */
    dflop_plan fixed_plan; /* used when mode == DFLOP_SEARCH_FIXED             */
    uint32_t gbs;          /* GBS of Algorithm 1 (0 = n)                       */
    uint32_t top_p;        /* P plans balanced in Stage B (ALG1), 1..256       */
    uint32_t K;            /* candidates per plan, 1..2^24 (P * K < 2^24)      */
    uint32_t R;
    uint32_t G;
    uint32_t seed[2];
} dflop_search_params;

/* Host-resident result of dflop_search_plans; identical on every rank. */
typedef struct dflop_plan_result {
    uint32_t struct_size;
    uint32_t status_bits;       /* DFLOP_DEV_* bits seen on any rank                  */
    dflop_plan plan;            /* theta*, N_mb included                              */
    uint32_t m;                 /* buckets of theta*                                  */
    uint32_t cand;              /* c* within the plan's family                        */
    uint32_t stage_a_rank;      /* Stage-A rank of theta* (0 in FIXED mode)           */
    uint32_t owner_rank;        /* rank whose shard held c*                           */
    uint64_t makespan;          /* T_B of the winner, ticks                           */
    uint64_t cmax;              /* C_max of the winner, ticks                         */
    uint64_t stage_a_makespan;  /* T_A of theta* (0 in FIXED mode)                    */
    dflop_plan alg1_plan;       /* Algorithm 1's literal answer (Stage-A rank 0)      */
    uint32_t reserved;
    uint64_t alg1_makespan;     /* its T_A                                            */
    uint64_t n_configs;         /* |P_configs| (phase 1)                              */
    uint64_t n_pairs;           /* (config, N_mb) pairs evaluated (phase 2)           */
    uint64_t n_feasible;        /* pairs passing Eq. (4)-(5)                          */
    uint64_t n_candidates;      /* candidates scored across all ranks                 */
} dflop_plan_result;

typedef struct dflop_comm dflop_comm; /* opaque NCCL communicator owned by the library */

/* ---------------------------------------------------------------- support */
uint32_t dflop_abi_version(void);

/* Thread-local description of the last error on this thread ("" if none). */
const char* dflop_last_error(void);

/* Releases library-owned device caches (1F1B slot programs, config tables). */
dflop_status dflop_release_caches(void);

/* ---------------------------------------------------------------- instrumentation
 * A process-wide counter of every kernel the library launches, and (when enabled) CUDA
 * events recorded on the launching stream around each candidate-kernel launch (a3/a4) and
 * each Stage-A kernel (a6, k_stage_a), so that a benchmark can time them live.  dflop_profile_read synchronises
 * the recorded events, fills *out and, if reset != 0, clears the counters. */
typedef struct dflop_profile {
    uint32_t struct_size;
    uint32_t cand_launches;   /* candidate-kernel launches timed                      */
    uint64_t kernel_launches; /* all libdflop kernel launches since the last reset    */
    double cand_ms;           /* summed device time of the timed candidate launches   */
    uint32_t stage_a_launches; /* Stage-A kernel launches timed (ALG1 searches)        */
    uint32_t split_chunks;     /* candidate chunks run by the split pipeline (k_lpt, then the
                                  candidate kernel) since the last reset */
    double stage_a_ms;        /* their summed device time                            */
} dflop_profile;
dflop_status dflop_profile_enable(int on);
dflop_status dflop_profile_read(dflop_profile* out, int reset);

/* ---------------------------------------------------------------- a1 predict
 * Per-sample stage costs (O1-O4 of DESIGN.md section 4):
 *   b_i = tiles_i + frames_i                       encoder effective batch
 *   s_i = text_i + tau_tile*tiles_i + tau_frame*frames_i   packed LLM length
 *   ef_i = 1e9 * b_i*E_l*(24 h_E^2 E_seq [+ 4 h_E E_seq^2]) / (E_thr(b_i,E_tp)*E_tp*E_pp) * L_dp/E_dp
 *   lf_i = 1e9 * (4 h_L L_l s_i^2 / L_attn_thr(s_i,L_tp) + 24 h_L^2 L_l s_i / L_lin_thr(s_i,L_tp))
 *          / (L_tp*L_pp)
 *   eb_i = bwd_ratio*ef_i, lb_i = bwd_ratio*lf_i     (ns)
 * computed in fp32.  Outputs (device, row-major [4][n], rows ef, eb, lf, lb):
 *   cost_f32   durations in ticks as fp32 (NULL to skip);
 *   cost_ticks round-half-even to u32 ticks (NULL to skip); a value that rounds to
 *              >= 2^32 is written as 0xFFFFFFFF and sets DFLOP_DEV_COST_OVERFLOW in
 *              *dev_status (device u32, may be NULL; bits are OR-ed, never cleared).
 * Inputs tiles/frames/text: device u32[n].  model/plan: host, copied during the call.
 * Asynchronous on stream.
 * Errors: INVALID_ARGUMENT (NULL model/plan, a zero degree, tick_ns <= 0, bwd_ratio < 0,
 * a grid with non-increasing knots, a non-positive throughput value, n_x/n_tp out of
 * range); SHAPE (n > 2^31 - 1); CUDA (launch failure). */
dflop_status dflop_predict_costs(const dflop_cost_model* model, const dflop_plan* plan, const uint32_t* tiles,
                                 const uint32_t* frames, const uint32_t* text, uint32_t n, float* cost_f32,
                                 uint32_t* cost_ticks, uint32_t* dev_status, dflop_stream_t stream);

/* ---------------------------------------------------------------- a2-a5 balance
 * Partition n samples into m = n_mb*l_dp buckets with the candidate family
 * of dflop_balance_params, score every candidate by its 1F1B makespan over S = e_pp+l_pp
 * stages (stages < e_pp take the bucket's encoder sums, the rest its LLM sums; R7), and
 * return the lexicographic minimum of (makespan, id_base + c) over [cand_begin, cand_end).
 *   cost_ticks     device u32 [4][n] (rows ef, eb, lf, lb), e.g. from dflop_predict_costs.
 *   plan           host; only e_pp, l_pp, l_dp, n_mb are used.
 *   ws / ws_bytes  workspace query: ws == NULL stores the required size in *ws_bytes
 *                  and returns OK without launching; otherwise ws must be a device
 *                  buffer of at least *ws_bytes bytes, 256-byte aligned.  It holds the
 *                  per-resident-candidate scratch (about 18 KB each for n = 4096, m = 64)
 *                  and, when the split pipeline runs (packed sums,
 *                  48 <= m <= 255, n <= 4096, >= 4,096 candidates), one entry of n + 8m
 *                  bytes per candidate of the range, up to 2^20 candidates per chunk.
 *   best           device dflop_cand_result (written).
 *   assign         device u32[n] or NULL: bucket of every sample for c*.
 *   group_offsets  device u32[m+1] or NULL, group_items device u32[n] or NULL: the
 *                  winner's index groups, bucket-major, samples ascending.
 *   cand_makespan, cand_cmax  device u64[cand_end - cand_begin] or NULL: every
 *                  candidate's makespan / C_max (parity tests).
 * n == 0 is allowed (every bucket empty, makespan 0); n < m leaves buckets empty.
 * Asynchronous on stream.
 * Errors: INVALID_ARGUMENT (m == 0, any degree 0, K == 0 or > 2^24, an empty or
 * out-of-range shard, G outside 1..16, EXHAUSTIVE with m^n > K); SHAPE (n > 65535,
 * m > 65535, S > 32); WORKSPACE_TOO_SMALL; UNSUPPORTED (per-candidate state larger
 * than shared memory); CUDA. */
dflop_status dflop_balance_microbatches(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan,
                                        const dflop_balance_params* bp, void* ws, size_t* ws_bytes,
                                        dflop_cand_result* best, uint32_t* assign, uint32_t* group_offsets,
                                        uint32_t* group_items, uint64_t* cand_makespan, uint64_t* cand_cmax,
                                        dflop_stream_t stream);

/* ---------------------------------------------------------------- a4 simulate
 * Batched non-interleaved 1F1B (Fig. 1; R9: stage s runs w_s = min(S-1-s, M)
 * warm-up forwards, then alternates F/B, then drains; F(s,k) after F(s-1,k), B(s,k)
 * after B(s+1,k), B(S-1,k) after F(S-1,k); communication is free, R8).
 *   fwd, bwd    device u64 [C][S][M] row-major durations (ticks).
 *   makespan    device u64 [C].
 *   stage_busy  device u64 [C][S] or NULL: sum of F+B durations per stage.
 * Asynchronous on stream.  Errors: SHAPE (S == 0, M == 0, S > 32, M > 65535 --
 * SPEC "inconsistent duration matrix shape"); INVALID_ARGUMENT (NULL inputs);
 * CUDA. */
dflop_status dflop_simulate_1f1b(const uint64_t* fwd, const uint64_t* bwd, uint32_t C, uint32_t S, uint32_t M,
                                 uint64_t* makespan, uint64_t* stage_busy, dflop_stream_t stream);

/* ---------------------------------------------------------------- index groups
 * CSR index groups of an assignment ("returns a set of index groups"):
 * offsets[m+1], items[n] bucket-major with samples ascending.  Device pointers;
 * asynchronous.  Errors: INVALID_ARGUMENT, SHAPE (an assign value >= m is undefined
 * behaviour and is not checked on device). */
dflop_status dflop_index_groups(const uint32_t* assign, uint32_t n, uint32_t m, uint32_t* offsets, uint32_t* items,
                                void* ws, size_t* ws_bytes, dflop_stream_t stream);

/* ---------------------------------------------------------------- a6 search
 * One global batch end to end, synchronous on stream: a1-a5 for a fixed theta
 * (DFLOP_SEARCH_FIXED), or Algorithm 1 Stage A over every
 * (E_tp,E_pp,E_dp,L_tp,L_pp,L_dp) x N_mb in 1..GBS//L_dp with the Eq. (4)-(5) memory
 * filter and the closed-form T = (N_mb + E_pp + L_pp - 1) * max(E_dur, L_dur) at the
 * batch-mean shapes, then Stage B: a1-a5 on the batch for the top_p pairs
 * by (T_A, config index, N_mb); the final plan minimises (T_B, Stage-A rank, c).
 *   cl, cm, mm     host structs (mm and cl unused in FIXED mode, may be NULL).
 *   tiles/frames/text  device u32[n].
 *   comm           NULL = this GPU evaluates the whole family; otherwise the family
 *                  is sharded over the communicator's ranks (candidate ranges
 *                  [floor(g*K/G), floor((g+1)*K/G))) and one NCCL min all-reduce
 *                  picks the winner; every rank gets the same result and assignment.
 *   ws / ws_bytes  workspace query as in dflop_balance_microbatches.
 *   out            host dflop_plan_result (written).
 *   assign         device u32[n] or NULL: the winner's bucket per sample.
 *   stage_a_out    device u64[stage_a_cap] or NULL: T_A of every pair in enumeration
 *                  order (UINT64_MAX = infeasible), written when stage_a_cap >= n_pairs.
 * A Stage-B plan beyond the balancer's limits (E_pp + L_pp > 32 or N_mb * L_dp > 65535,
 * possible from 34 GPUs on) is skipped: it is not balanced and never chosen (its objective
 * is UINT64_MAX); UNSUPPORTED when every top-P plan is skipped.
 * Errors: INFEASIBLE (no pair passes Eq. (4)-(5)); OVERFLOW (a cost or makespan out of
 * range, from the device status); NCCL; CUDA; the argument errors of the calls above. */
dflop_status dflop_search_plans(const dflop_cluster* cl, const dflop_cost_model* cm, const dflop_mem_model* mm,
                                const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                                const dflop_search_params* sp, dflop_comm* comm, void* ws, size_t* ws_bytes,
                                dflop_plan_result* out, uint32_t* assign, uint64_t* stage_a_out,
                                uint64_t stage_a_cap, dflop_stream_t stream);

/* ---------------------------------------------------------------- N3 exact C_max
 * The ILP of P:703-727 (minimise C_max = max_j max(E_j, L_j) over assignments of the n
 * samples to m = N_mb * L_dp buckets), solved by a node-budgeted parallel branch and bound
 * (SPEC solve_exact): items in the LPT base order, first-use symmetry breaking,
 * lower bound LB = max(ceil(sum e / m), ceil(sum l / m), max_i max(e_i, l_i)).  The
 * incumbent starts from init_assign (e.g. the search's winner) or the paper's LPT.  The
 * result is a C_max certificate (proven, or the gap to LB) and an extra candidate: its
 * assignment scored by the 1F1B simulation (makespan). */
typedef struct dflop_exact_result {
    uint32_t struct_size;
    uint32_t proven;      /* 1: cmax is the optimum (search finished or cmax == LB)     */
    uint64_t cmax;        /* best C_max found, ticks                                     */
    uint64_t lower_bound; /* LB, ticks                                                   */
    uint64_t nodes;       /* child visits                                                */
    uint64_t makespan;    /* 1F1B makespan of the returned assignment (max over replicas) */
    uint32_t searched;    /* 1: the tree search ran (n <= 256, m <= 32); 0: bound only    */
    uint32_t reserved;
} dflop_exact_result;

/* cost_ticks  device u32 [4][n] (ef, eb, lf, lb); n <= 65535.
 * plan        host; m = n_mb * l_dp <= 256.
 * node_budget child visits over the whole search (split over the parallel subtrees).
 * init_assign device u32 [n] or NULL (bucket per sample, < m).
 * ws/ws_bytes workspace query as in dflop_balance_microbatches.
 * out         host result; assign: device u32 [n] or NULL (the returned assignment).
 * Synchronous.  Errors: INVALID_ARGUMENT (plan, m > 256, an init_assign entry >= m),
 * SHAPE (n > 65535), WORKSPACE_TOO_SMALL, CUDA. */
dflop_status dflop_exact_cmax(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan, uint64_t node_budget,
                              const uint32_t* init_assign, void* ws, size_t* ws_bytes, dflop_exact_result* out,
                              uint32_t* assign, dflop_stream_t stream);

/* ---------------------------------------------------------------- N4(a) microbatch order
 * The 1F1B makespan of a replica depends on the order of its microbatch slots (R11).  For
 * one assignment (e.g. the search's winner) every LLM replica rho (buckets k * L_dp + rho,
 * slot k by default, R10) gets an improved slot order: the best of four start orders
 * (identity, W = max(E, L) ascending, descending, valley), then best-improvement pairwise
 * slot swaps (every pair when N_mb <= 128, else pairs at distance <= 16), lexicographic
 * (makespan, a, b), at most `rounds` rounds (R35).
 *   cost_ticks device u32 [4][n]; assign device u32 [n] (bucket per sample, < m).
 *   order_out  device u32 [L_dp][N_mb]: the bucket run in slot k of replica rho.
 *   T_out      host u64 [L_dp]: the replicas' 1F1B makespans (the plan's T = their max).
 * Synchronous.  Errors: INVALID_ARGUMENT (plan, bucket >= m), UNSUPPORTED (shared memory),
 * WORKSPACE_TOO_SMALL, CUDA. */
dflop_status dflop_order_search(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan,
                                const uint32_t* assign, uint32_t rounds, void* ws, size_t* ws_bytes,
                                uint32_t* order_out, uint64_t* T_out, dflop_stream_t stream);

/* ---------------------------------------------------------------- N4(b) routing plan
 * The inter-model communicator's plan for E_dp != L_dp: for microbatch slot k the
 * LLM data groups rho run buckets k * L_dp + rho (R10); the slot's samples, listed in
 * (rho, sample index) order, are split into E_dp contiguous encoder ranges balanced by the
 * encoder cost e = ef + eb (range g starts at the first position whose preceding cost
 * reaches g / E_dp of the slot's total, R36).  Forward: encoder range g is gathered and
 * scattered over the LLM ranges it overlaps; backward: the reverse.
 *   cost_ticks device u32 [4][n]; assign device u32 [n] (bucket per sample, < m).
 *   pos_item   device u32 [n]: the sample at each position (slot-major).
 *   slot_off   device u32 [N_mb + 1]; enc_off device u32 [N_mb][E_dp + 1]; llm_off device
 *              u32 [N_mb][L_dp + 1] (absolute positions); enc_load device u64 [N_mb][E_dp]
 *              or NULL (encoder cost per range).
 * Synchronous.  Errors: INVALID_ARGUMENT (plan, bucket >= m), WORKSPACE_TOO_SMALL, CUDA. */
dflop_status dflop_route_plan(const uint32_t* cost_ticks, uint32_t n, const dflop_plan* plan, const uint32_t* assign,
                              void* ws, size_t* ws_bytes, uint32_t* pos_item, uint32_t* slot_off, uint32_t* enc_off,
                              uint32_t* llm_off, uint64_t* enc_load, dflop_stream_t stream);

/* ---------------------------------------------------------------- N2 search over a sample
 * Eq. (1): theta* = argmin_theta (1/|D|) sum_{d in D} T(d; theta) over a sample
 * of D global batches, each balanced and scored on the device exactly as in
 * dflop_search_plans; T(d; theta) = T_B, the batch's best candidate makespan (R33).
 *   tiles/frames/text  device u32 [batch_offsets[D] - batch_offsets[0]]: the batches
 *                  back to back; batch b = [batch_offsets[b], batch_offsets[b+1]) (host
 *                  u32 [D+1], non-decreasing, each batch <= 65535 samples), 1 <= D <= 4096.
 *   sp             as for dflop_search_plans; batch b's candidate family uses Philox key
 *                  (seed[0], seed[1] + b).  ALG1: Stage A on the mean shapes of the whole
 *                  sample (GBS = sp->gbs), Stage B over every (top-P plan, batch).
 *   out            host: the plan minimising (sum_b T_B(b), Stage-A rank); out->makespan =
 *                  sum_b T_B(b) (D x the Eq. (1) objective, ticks); cand/cmax/owner_rank
 *                  are batch 0's.
 *   batch_results  host dflop_cand_result[D] or NULL: theta*'s winner per batch.
 *   plan_objective host u64[top_p] or NULL: sum_b T_B(b) per Stage-B plan (Stage-A rank
 *                  order; UINT64_MAX when a plan had no candidate).
 *   plans_out      host dflop_plan[top_p] or NULL: the Stage-B plans in Stage-A rank order
 *                  (FIXED mode: the one fixed plan).
 *   assign         device u32 [total] or NULL: every batch's winning assignment.
 * Multi-GPU: candidates sharded as in dflop_search_plans; one NCCL min all-reduce of the
 * [P x D] key array, then one broadcast per batch from its winner's owner.  Errors as
 * dflop_search_plans, plus INVALID_ARGUMENT for bad offsets / D. */
dflop_status dflop_search_plans_batches(const dflop_cluster* cl, const dflop_cost_model* cm,
                                        const dflop_mem_model* mm, const uint32_t* tiles, const uint32_t* frames,
                                        const uint32_t* text, const uint32_t* batch_offsets, uint32_t n_batches,
                                        const dflop_search_params* sp, dflop_comm* comm, void* ws, size_t* ws_bytes,
                                        dflop_plan_result* out, dflop_cand_result* batch_results,
                                        uint64_t* plan_objective, dflop_plan* plans_out, uint32_t* assign,
                                        dflop_stream_t stream);

/* ---------------------------------------------------------------- NCCL
 * Bootstrap: rank 0 calls dflop_get_unique_id, the caller broadcasts the 128 bytes
 * (e.g. with torch.distributed), then every rank calls dflop_comm_init with its rank,
 * the world size and its CUDA device.  The communicator is owned by the library
 * until dflop_comm_destroy. */
dflop_status dflop_get_unique_id(uint8_t id[128]);
dflop_status dflop_comm_init(const uint8_t id[128], int rank, int world, int device, dflop_comm** comm);
dflop_status dflop_comm_destroy(dflop_comm* comm);

/* ---------------------------------------------------------------- sharding protocol
 * The host arithmetic dflop_search_plans / dflop_search_plans_batches run around their NCCL
 * collectives (P:796 the communicator; P:738 the argmin over candidates; P:491-497
 * Eq. (1) over batches).  Pure host functions: no CUDA call, usable without a GPU (the gloo
 * test drives the same protocol on CPU).  No pointer is retained.
 *
 * dflop_shard_range  candidates [*begin, *end) = [floor(K*rank/world), floor(K*(rank+1)/world))
 *                    of rank `rank`; Philox counters use the global id, so the winner does not
 *                    depend on world.  INVALID_ARGUMENT: world == 0, rank >= world, NULL outputs.
 * dflop_owner_of     the rank whose range holds candidate c (UINT32_MAX if c >= K).
 * dflop_pack_key     min(T, 2^40 - 1) << 24 | (id & 0xFFFFFF): the integer minimum over keys is
 *                    the lexicographic minimum of (T, id) (R18); one 8-byte MIN all-reduce.  A
 *                    saturated T is reported by the kernels' DFLOP_DEV_MAKESPAN_OVERFLOW bit.
 * dflop_select_plan  keys: host u64 [P][D], reduced over ranks (UINT64_MAX = no candidate);
 *                    batch_n: host u32 [D] batch sizes or NULL (an empty batch contributes 0).
 *                    *win_p = argmin over p of (sum_b (keys[p][b] >> 24), p); objective: host
 *                    u64 [P] or NULL, the sums (UINT64_MAX for a plan with a missing key).
 *                    UNSUPPORTED ("no candidate evaluated", *win_p = UINT32_MAX) when no plan
 *                    has all its keys; INVALID_ARGUMENT for NULL keys/win_p or P, D == 0. */
dflop_status dflop_shard_range(uint32_t K, uint32_t rank, uint32_t world, uint32_t* begin, uint32_t* end);
uint32_t dflop_owner_of(uint32_t K, uint32_t c, uint32_t world);
uint64_t dflop_pack_key(uint64_t T, uint32_t id);
dflop_status dflop_select_plan(const uint64_t* keys, uint32_t P, uint32_t D, const uint32_t* batch_n,
                               uint32_t* win_p, uint64_t* objective);

#ifdef __cplusplus
}
#endif
#endif /* DFLOP_H */
