/*
 * dflop_oracle.c -- ORACLE.  TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of what the DFLOP
 * plan-candidate hot path computes (arXiv 2603.25120).  Floating point is fp64;
 * times after rounding are integer ticks (uint64 sums).  Every function cites the
 * passage it follows.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may load this library; the CUDA path shares
 * no code, header, table or constant generator with it.
 *
 * Citations: P:n = PAPER.md line n, S:n = SPEC.md line n, Rk = DESIGN.md reading k.
 *
 * Parity pins (tests/test_oracle_*.py) tie each function to something other than
 * itself: Random123 KAT vectors, SPEC worked examples, closed forms (makespan,
 * (p-1)/m bubble, bilinear interpolation), brute force on tiny inputs, an
 * explicit-DAG longest path, and Graham's LPT bound.  Functions without such a pin
 * are marked "parity unpinned" below (none at present beyond what DESIGN.md lists).
 */
#include "dflop_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------------- */
/* Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11, "Parallel random numbers:  */
/* as easy as 1, 2, 3").  Round: (hi(M1*x2)^x1^k0, lo(M1*x2), hi(M0*x0)^x3^k1,  */
/* lo(M0*x0)); the key is bumped by the Weyl constants between rounds.          */
/* Pinned by the Random123 known-answer vectors (tests/golden/philox_kat.txt).  */
/* ------------------------------------------------------------------------- */
#define PHILOX_M0 0xD2511F53u
#define PHILOX_M1 0xCD9E8D57u
#define PHILOX_W0 0x9E3779B9u
#define PHILOX_W1 0xBB67AE85u

void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    uint32_t x[4] = {ctr[0], ctr[1], ctr[2], ctr[3]};
    uint32_t k[2] = {key[0], key[1]};
    for (int r = 0; r < 10; r++) {
        if (r > 0) {
            k[0] += PHILOX_W0;
            k[1] += PHILOX_W1;
        }
        uint64_t p0 = (uint64_t)PHILOX_M0 * (uint64_t)x[0];
        uint64_t p1 = (uint64_t)PHILOX_M1 * (uint64_t)x[2];
        uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
        uint32_t y0 = hi1 ^ x[1] ^ k[0];
        uint32_t y1 = lo1;
        uint32_t y2 = hi0 ^ x[3] ^ k[1];
        uint32_t y3 = lo0;
        x[0] = y0; x[1] = y1; x[2] = y2; x[3] = y3;
    }
    out[0] = x[0]; out[1] = x[1]; out[2] = x[2]; out[3] = x[3];
}

/* floor(u * n / 2^32): maps a uniform word to [0, n). */
uint32_t orc_mulhi32(uint32_t u, uint32_t n) {
    return (uint32_t)(((uint64_t)u * (uint64_t)n) >> 32);
}

/* ------------------------------------------------------------------------- */
/* Interpolation ("modeled through linear interpolation", "fit      */
/* using linear interpolation").  Reading R3: multilinear, clamped outside the  */
/* hull, evaluated as (1-w)*V[k] + w*V[k+1] so that every knot   */
/* is reproduced exactly.                                              */
/* ------------------------------------------------------------------------- */
static double clampd(double x, double lo, double hi) {
    if (x < lo) return lo;
    if (x > hi) return hi;
    return x;
}

/* k = the largest index with xs[k] <= xh and k <= n-2. */
static uint32_t bracket(const double* xs, uint32_t n, double xh) {
    uint32_t k = 0;
    while (k + 1 < n - 1 && xs[k + 1] <= xh) k++;
    return k;
}

static double interp1(const double* xs, const double* vs, uint32_t n, double x) {
    if (n == 1) return vs[0];
    double xh = clampd(x, xs[0], xs[n - 1]);
    uint32_t k = bracket(xs, n, xh);
    double w = (xh - xs[k]) / (xs[k + 1] - xs[k]);
    return (1.0 - w) * vs[k] + w * vs[k + 1];
}

double orc_interp_thr(const orc_grid* g, double x, double tp) {
    if (g->n_tp == 1) return interp1(g->x, g->v[0], g->n_x, x);
    double th = clampd(tp, g->tp[0], g->tp[g->n_tp - 1]);
    uint32_t a = bracket(g->tp, g->n_tp, th);
    double wt = (th - g->tp[a]) / (g->tp[a + 1] - g->tp[a]);
    double r0 = interp1(g->x, g->v[a], g->n_x, x);
    double r1 = interp1(g->x, g->v[a + 1], g->n_x, x);
    return (1.0 - wt) * r0 + wt * r1;
}

/* One layer-plane of a memory grid: clamped bilinear over (tp, x). */
static double mem_plane(const orc_mgrid* g, int q, double tp, double x) {
    if (g->n_tp == 1) return interp1(g->x, g->v[q][0], g->n_x, x);
    double th = clampd(tp, g->tp[0], g->tp[g->n_tp - 1]);
    uint32_t a = bracket(g->tp, g->n_tp, th);
    double wt = (th - g->tp[a]) / (g->tp[a + 1] - g->tp[a]);
    double r0 = interp1(g->x, g->v[q][a], g->n_x, x);
    double r1 = interp1(g->x, g->v[q][a + 1], g->n_x, x);
    return (1.0 - wt) * r0 + wt * r1;
}

/* Memory model: linear in the layer count through the two profiled layer counts
 * ("varying the number of layers between two distinct small values";
 * S:168 "linearly extended in the layer dimension"), clamped on tp and shape. */
double orc_interp_mem(const orc_mgrid* g, double l, double tp, double x) {
    double wl = (l - g->l[0]) / (g->l[1] - g->l[0]);
    double m0 = mem_plane(g, 0, tp, x);
    double m1 = mem_plane(g, 1, tp, x);
    return (1.0 - wl) * m0 + wl * m1;
}

/* ------------------------------------------------------------------------- */
/* Step a1: per-item durations.                                                */
/*   P:486  E_dur(d) = E_FLOP(d) / E_thr(b(d), E_tp),                          */
/*          L_dur(d) = L_FLOP(d) / L_thr(s(d), L_tp)                           */
/*   P:630-631 divide by thr * tp * pp (R2, R7); P:446 attention and linear    */
/*   parts with separate throughput models; P:278 backward = 2x forward (R6);  */
/*   FLOP accounting R1: 24*l*h^2 per token, 4*l*h*s^2 attention;      */
/*   R13: encoder time per LLM bucket scaled by L_dp / E_dp.                   */
/* ------------------------------------------------------------------------- */
static int round_ticks(double x_ns, double tick_ns, uint32_t* q) {
    double t = x_ns / tick_ns;
    if (!(t < 4294967295.5)) return ORC_OVERFLOW; /* rounds to >= 2^32 */
    *q = (uint32_t)nearbyint(t);                  /* round half to even (default mode) */
    return ORC_OK;
}

/* N1 shape bin (R30): floor(log2 x) by repeated halving; x = 0 is bin 0; clamped. */
uint32_t orc_shape_bin(uint64_t x) {
    uint32_t q = 0;
    while (x >= 2) {
        x /= 2;
        q++;
    }
    return q < ORC_CORR_BINS ? q : ORC_CORR_BINS - 1;
}

/* ---------------------------------------------------------------- N1 tracker */
int orc_tracker_init(orc_tracker* t, double alpha, uint32_t window, double cost) {
    if (!(alpha > 0.0 && alpha <= 1.0) || window < 1 || window > ORC_TRACK_WIN) return ORC_INVALID;
    memset(t, 0, sizeof *t);
    t->alpha = alpha;
    t->window = window;
    t->cost = cost;
    t->active = 1;
    return ORC_OK;
}

/* S:420 record_observation: exponential average of Th_actual per shape bucket; S:421 the
 * deviation B = Th_actual - Th_pred of the bucket (Eq. (6)). */
double orc_tracker_record(orc_tracker* t, uint32_t grid, uint64_t x, double th_actual, double th_pred) {
    uint32_t q = orc_shape_bin(x);
    if (t->seen[grid][q])
        t->observed[grid][q] = (1.0 - t->alpha) * t->observed[grid][q] + t->alpha * th_actual;
    else {
        t->observed[grid][q] = th_actual;
        t->seen[grid][q] = 1;
    }
    t->predicted[grid][q] = th_pred;
    return t->observed[grid][q] - t->predicted[grid][q];
}

void orc_tracker_rho(const orc_tracker* t, double* rho) {
    for (uint32_t g = 0; g < 3; g++)
        for (uint32_t q = 0; q < ORC_CORR_BINS; q++)
            rho[g * ORC_CORR_BINS + q] = t->seen[g][q] ? t->observed[g][q] / t->predicted[g][q] : 1.0;
}

/* S:431 cost_benefit_step: deactivate when the average benefit of the last I
 * iterations does not exceed the recurring cost C; never reactivated. */
uint32_t orc_tracker_cost_benefit(orc_tracker* t, const double* benefits, uint32_t nb) {
    for (uint32_t i = 0; i < nb; i++) {
        t->last[t->n_benefits % ORC_TRACK_WIN] = benefits[i];
        t->n_benefits++;
    }
    if (t->active && t->n_benefits >= t->window) {
        double sum = 0.0;
        for (uint32_t i = 0; i < t->window; i++) sum += t->last[(t->n_benefits - 1 - i) % ORC_TRACK_WIN];
        t->active = (sum / (double)t->window) > t->cost;
    }
    return t->active;
}

int orc_predict(const orc_model* m, const orc_plan* p, const uint32_t* tiles, const uint32_t* frames,
                const uint32_t* text, uint32_t n, double* cost_f64, uint32_t* cost_q, uint32_t* bad) {
    return orc_predict_corrected(m, p, tiles, frames, text, n, NULL, cost_f64, cost_q, bad);
}

int orc_predict_corrected(const orc_model* m, const orc_plan* p, const uint32_t* tiles, const uint32_t* frames,
                          const uint32_t* text, uint32_t n, const double* rho, double* cost_f64, uint32_t* cost_q,
                          uint32_t* bad) {
    double lin_e = 24.0 * (double)m->e_hidden * (double)m->e_hidden;
    double att_e = m->e_attn ? 4.0 * (double)m->e_hidden : 0.0;
    double per_inst_e = lin_e * (double)m->e_seq + att_e * (double)m->e_seq * (double)m->e_seq;
    double c_e = (double)m->e_layers * per_inst_e;
    double c_lin = 24.0 * (double)m->l_hidden * (double)m->l_hidden * (double)m->l_layers;
    double c_att = 4.0 * (double)m->l_hidden * (double)m->l_layers;
    int status = ORC_OK;
    for (uint32_t i = 0; i < n; i++) {
        /* O1 shapes: b(d) = tiles + frames (P:442 fixed E_seq_len per instance);
         * s(d) = text + visual tokens after the connector. */
        uint64_t b = (uint64_t)tiles[i] + (uint64_t)frames[i];
        uint64_t s = (uint64_t)text[i] + (uint64_t)m->tau_tile * tiles[i] + (uint64_t)m->tau_frame * frames[i];
        double bd = (double)b, sd = (double)s;
        double ef = 0.0;
        if (b > 0) {
            double EF = bd * c_e;
            double thr = orc_interp_thr(&m->thr_e, bd, (double)p->e_tp);
            if (rho) thr = thr * rho[0 * ORC_CORR_BINS + orc_shape_bin(b)]; /* N1: corrected */
            ef = 1e9 * EF / (thr * (double)p->e_tp * (double)p->e_pp) * ((double)p->l_dp / (double)p->e_dp);
        }
        double Llin = c_lin * sd;
        double Latt = c_att * sd * sd;
        double thr_a = orc_interp_thr(&m->thr_att, sd, (double)p->l_tp);
        double thr_l = orc_interp_thr(&m->thr_lin, sd, (double)p->l_tp);
        if (rho) { /* N1: corrected throughput of the sample's shape bin */
            thr_a = thr_a * rho[1 * ORC_CORR_BINS + orc_shape_bin(s)];
            thr_l = thr_l * rho[2 * ORC_CORR_BINS + orc_shape_bin(s)];
        }
        double lf = 1e9 * (Latt / thr_a + Llin / thr_l) / ((double)p->l_tp * (double)p->l_pp);
        double eb = m->bwd_ratio * ef;
        double lb = m->bwd_ratio * lf;
        double v[4] = {ef, eb, lf, lb};
        for (int k = 0; k < 4; k++) {
            if (cost_f64) cost_f64[(uint64_t)k * n + i] = v[k];
            uint32_t q = 0;
            if (round_ticks(v[k], m->tick_ns, &q) != ORC_OK) {
                if (status == ORC_OK && bad) *bad = i;
                status = ORC_OVERFLOW;
                q = 0xFFFFFFFFu;
            }
            if (cost_q) cost_q[(uint64_t)k * n + i] = q;
        }
    }
    return status;
}

/* ------------------------------------------------------------------------- */
/* Step a2: LPT sort ("sorts the data items in descending order of       */
/* duration"); R12: duration key = max(e_i, l_i), e = ef + eb, l = lf + lb;    */
/* ties by index ascending (R18).                                              */
/* ------------------------------------------------------------------------- */
static const uint32_t* g_sort_q;
static uint32_t g_sort_n;

static uint64_t item_e(const uint32_t* q, uint32_t n, uint32_t i) { return (uint64_t)q[i] + (uint64_t)q[(uint64_t)n + i]; }
static uint64_t item_l(const uint32_t* q, uint32_t n, uint32_t i) { return (uint64_t)q[2ull * n + i] + (uint64_t)q[3ull * n + i]; }
static uint64_t max64(uint64_t a, uint64_t b) { return a > b ? a : b; }

static int cmp_order(const void* pa, const void* pb) {
    uint32_t a = *(const uint32_t*)pa, b = *(const uint32_t*)pb;
    uint64_t ka = max64(item_e(g_sort_q, g_sort_n, a), item_l(g_sort_q, g_sort_n, a));
    uint64_t kb = max64(item_e(g_sort_q, g_sort_n, b), item_l(g_sort_q, g_sort_n, b));
    if (ka != kb) return ka > kb ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

void orc_base_order(const uint32_t* cost_q, uint32_t n, uint32_t* order) {
    for (uint32_t i = 0; i < n; i++) order[i] = i;
    g_sort_q = cost_q;   /* single-threaded qsort comparator context */
    g_sort_n = n;
    qsort(order, n, sizeof(uint32_t), cmp_order);
}

/* ------------------------------------------------------------------------- */
/* Step a4 block: non-interleaved 1F1B (Fig. 1; R9 warm-up              */
/* w_s = min(S-1-s, M)); inter-stage communication is free (R8).       */
/* Worklist evaluation: sweep the stages, run each stage's next op once its    */
/* dependency has finished, until every op has run.                            */
/* ------------------------------------------------------------------------- */
static uint32_t min32(uint32_t a, uint32_t b) { return a < b ? a : b; }

/* The op sequence of stage s: returns kind (0 = F, 1 = B) and microbatch of op t. */
static void stage_op(uint32_t s, uint32_t S, uint32_t M, uint32_t t, int* kind, uint32_t* mb) {
    uint32_t w = min32(S - 1 - s, M);
    if (t < w) { *kind = 0; *mb = t; return; }
    uint32_t u = t - w;
    if (u < 2 * (M - w)) {
        uint32_t q = u / 2;
        if (u % 2 == 0) { *kind = 0; *mb = w + q; }
        else            { *kind = 1; *mb = q; }
        return;
    }
    *kind = 1;
    *mb = (M - w) + (u - 2 * (M - w));
}

int orc_simulate_1f1b(const uint64_t* fwd, const uint64_t* bwd, uint32_t S, uint32_t M,
                      uint64_t* makespan, uint64_t* stage_busy) {
    if (S == 0 || M == 0) return ORC_INVALID;
    size_t SM = (size_t)S * M;
    uint64_t* F_end = (uint64_t*)calloc(SM, sizeof(uint64_t));
    uint64_t* B_end = (uint64_t*)calloc(SM, sizeof(uint64_t));
    unsigned char* F_done = (unsigned char*)calloc(SM, 1);
    unsigned char* B_done = (unsigned char*)calloc(SM, 1);
    uint32_t* next = (uint32_t*)calloc(S, sizeof(uint32_t));
    uint64_t* last = (uint64_t*)calloc(S, sizeof(uint64_t));
    if (!F_end || !B_end || !F_done || !B_done || !next || !last) return ORC_INVALID;
    uint64_t remaining = 2ull * SM;
    int status = ORC_OK;
    while (remaining > 0) {
        int progress = 0;
        for (uint32_t s = 0; s < S; s++) {
            while (next[s] < 2 * M) {
                int kind; uint32_t k;
                stage_op(s, S, M, next[s], &kind, &k);
                uint64_t dep = 0;
                if (kind == 0) {
                    /* F(s,k) after F(s-1,k) */
                    if (s > 0) {
                        if (!F_done[(size_t)(s - 1) * M + k]) break;
                        dep = F_end[(size_t)(s - 1) * M + k];
                    }
                } else {
                    /* B(s,k) after B(s+1,k); the last stage's B(k) after its own F(k) */
                    if (s + 1 < S) {
                        if (!B_done[(size_t)(s + 1) * M + k]) break;
                        dep = B_end[(size_t)(s + 1) * M + k];
                    } else {
                        if (!F_done[(size_t)s * M + k]) break;
                        dep = F_end[(size_t)s * M + k];
                    }
                }
                uint64_t start = last[s] > dep ? last[s] : dep;
                uint64_t dur = kind == 0 ? fwd[(size_t)s * M + k] : bwd[(size_t)s * M + k];
                uint64_t end = start + dur;
                if (kind == 0) { F_end[(size_t)s * M + k] = end; F_done[(size_t)s * M + k] = 1; }
                else           { B_end[(size_t)s * M + k] = end; B_done[(size_t)s * M + k] = 1; }
                last[s] = end;
                next[s]++;
                remaining--;
                progress = 1;
            }
        }
        if (!progress) { status = ORC_INVALID; break; } /* cannot happen for 1F1B */
    }
    uint64_t T = 0;
    for (uint32_t s = 0; s < S; s++) {
        if (last[s] > T) T = last[s];
        if (stage_busy) {
            uint64_t busy = 0;
            for (uint32_t k = 0; k < M; k++) busy += fwd[(size_t)s * M + k] + bwd[(size_t)s * M + k];
            stage_busy[s] = busy;
        }
    }
    *makespan = T;
    free(F_end); free(B_end); free(F_done); free(B_done); free(next); free(last);
    return status;
}

/* ------------------------------------------------------------------------- */
/* Steps a3 + a4: one candidate of the seeded family.    */
/* Problem statement: P:703-727 (partition N items into m = N_mb * L_dp       */
/* buckets; objective C_max = max(max_j E_j, max_j L_j)).              */
/* ------------------------------------------------------------------------- */
typedef struct bucket_sums {
    uint64_t EF, EB, LF, LB;
} bucket_sums;

static uint64_t bE(const bucket_sums* b) { return b->EF + b->EB; }
static uint64_t bL(const bucket_sums* b) { return b->LF + b->LB; }

static void add_item(bucket_sums* b, const uint32_t* q, uint32_t n, uint32_t i) {
    b->EF += q[i]; b->EB += q[(uint64_t)n + i]; b->LF += q[2ull * n + i]; b->LB += q[3ull * n + i];
}
static void sub_item(bucket_sums* b, const uint32_t* q, uint32_t n, uint32_t i) {
    b->EF -= q[i]; b->EB -= q[(uint64_t)n + i]; b->LF -= q[2ull * n + i]; b->LB -= q[3ull * n + i];
}

/* Group-perturbed order pi_c: Fisher-Yates inside consecutive groups of G positions. */
static void perturbed_order(const uint32_t* pi, uint32_t n, uint32_t G, uint32_t c, const uint32_t seed[2],
                            uint32_t* out) {
    for (uint32_t g = 0; (uint64_t)g * G < n; g++) {
        uint32_t start = g * G;
        uint32_t ng = min32(G, n - start);
        uint32_t local[16], u[16];
        for (uint32_t t = 0; t < ng; t++) local[t] = t;
        for (uint32_t p = 0; 4 * p < ng - 1; p++) {
            uint32_t ctr[4] = {g, c, 0u, p}, w[4];
            orc_philox4x32_10(ctr, seed, w);
            for (int q = 0; q < 4; q++) u[4 * p + q] = w[q];
        }
        for (uint32_t t = ng - 1; t >= 1; t--) {
            uint32_t r = orc_mulhi32(u[ng - 1 - t], t + 1);
            uint32_t tmp = local[t]; local[t] = local[r]; local[r] = tmp;
        }
        for (uint32_t t = 0; t < ng; t++) out[start + t] = pi[start + local[t]];
    }
}

/* Score a partition: 1F1B per replica rho = j mod L_dp, slot k = j div L_dp (R10);
 * stages s < E_pp use (EF, EB), the rest (LF, LB) (R7). T = max over replicas. */
static int score_partition(const bucket_sums* bk, const orc_plan* p, uint64_t* T, uint64_t* cmax) {
    uint32_t S = p->e_pp + p->l_pp, M = p->n_mb, m = p->n_mb * p->l_dp;
    uint64_t* F = (uint64_t*)malloc(sizeof(uint64_t) * S * M);
    uint64_t* B = (uint64_t*)malloc(sizeof(uint64_t) * S * M);
    uint64_t best = 0;
    int st = ORC_OK;
    for (uint32_t rho = 0; rho < p->l_dp && st == ORC_OK; rho++) {
        for (uint32_t s = 0; s < S; s++)
            for (uint32_t k = 0; k < M; k++) {
                const bucket_sums* b = &bk[k * p->l_dp + rho];
                F[s * M + k] = s < p->e_pp ? b->EF : b->LF;
                B[s * M + k] = s < p->e_pp ? b->EB : b->LB;
            }
        uint64_t Tr = 0;
        st = orc_simulate_1f1b(F, B, S, M, &Tr, NULL);
        if (Tr > best) best = Tr;
    }
    uint64_t c = 0;
    for (uint32_t j = 0; j < m; j++) c = max64(c, max64(bE(&bk[j]), bL(&bk[j])));
    free(F); free(B);
    *T = best;
    *cmax = c;
    return st;
}

static uint64_t best_start_order(const bucket_sums* bk, const orc_plan* p, uint32_t rho, uint64_t* F, uint64_t* B,
                                 uint32_t* ord);

int orc_run_candidate(const uint32_t* q, uint32_t n, const orc_plan* p, const orc_bparams* bp,
                      const uint32_t* pi, uint32_t c, uint32_t* assign_out, uint64_t* T, uint64_t* cmax) {
    uint32_t m = p->n_mb * p->l_dp;
    bucket_sums* bk = (bucket_sums*)calloc(m, sizeof(bucket_sums));
    uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint32_t* order = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1)); /* +1: refinement partner list */
    if (bp->mode & ORC_MODE_EXHAUSTIVE) {
        /* EXHAUSTIVE: candidate c is the base-m number a_{n-1} ... a_1 a_0 (requires m^n <= K). */
        uint64_t x = c;
        for (uint32_t i = 0; i < n; i++) { a[i] = (uint32_t)(x % m); x /= m; add_item(&bk[a[i]], q, n, i); }
    } else {
        /* Order: base order for c = 0, 1; group-perturbed for c >= 2. */
        if (c >= 2) perturbed_order(pi, n, bp->G, c, bp->seed, order);
        else memcpy(order, pi, sizeof(uint32_t) * n);
        /* LPT pass: c = 0 assigns to the lowest *current* max(E_j, L_j) (the paper's
         * rule); c >= 1 assigns to the lowest *resulting* max(E_j + e_i, L_j + l_i) (R12).
         * Ties go to the lowest j (R18). */
        for (uint32_t t = 0; t < n; t++) {
            uint32_t i = order[t];
            uint64_t e = item_e(q, n, i), l = item_l(q, n, i);
            uint32_t best_j = 0;
            uint64_t best_v = 0;
            for (uint32_t j = 0; j < m; j++) {
                uint64_t v = c == 0 ? max64(bE(&bk[j]), bL(&bk[j])) : max64(bE(&bk[j]) + e, bL(&bk[j]) + l);
                if (j == 0 || v < best_v) { best_v = v; best_j = j; }
            }
            a[i] = best_j;
            add_item(&bk[best_j], q, n, i);
        }
        /* Refinement rounds (c >= 2, m >= 2): one best move or swap out of the bottleneck bucket. */
        if (c >= 2 && m >= 2) {
            for (uint32_t r = 0; r < bp->R; r++) {
                uint32_t js = 0;
                uint64_t Ws = 0;
                for (uint32_t j = 0; j < m; j++) {
                    uint64_t W = max64(bE(&bk[j]), bL(&bk[j]));
                    if (j == 0 || W > Ws) { Ws = W; js = j; }
                }
                uint32_t ctr[4] = {r, c, 1u, 0u}, w[4];
                orc_philox4x32_10(ctr, bp->seed, w);
                uint32_t jp = (js + 1 + orc_mulhi32(w[0], m - 1)) % m;
                uint64_t Es = bE(&bk[js]), Ls = bL(&bk[js]), Ep = bE(&bk[jp]), Lp = bL(&bk[jp]);
                int found = 0;
                uint64_t best_score = 0;
                uint32_t best_i = 0, best_rank = 0;
                /* partner list: rank 0 = NONE (pure move), then rank i'+1 for i' in j' ascending */
                uint32_t np = 0;
                order[np++] = 0;
                for (uint32_t i2 = 0; i2 < n; i2++)
                    if (a[i2] == jp) order[np++] = i2 + 1;
                for (uint32_t i = 0; i < n; i++) {
                    if (a[i] != js) continue;
                    uint64_t ei = item_e(q, n, i), li = item_l(q, n, i);
                    for (uint32_t u = 0; u < np; u++) {
                        uint32_t rank = order[u];
                        uint64_t e2 = 0, l2 = 0;
                        if (rank > 0) {
                            e2 = item_e(q, n, rank - 1); l2 = item_l(q, n, rank - 1);
                        }
                        uint64_t s1 = max64(Es - ei + e2, Ls - li + l2);
                        uint64_t s2 = max64(Ep - e2 + ei, Lp - l2 + li);
                        uint64_t score = max64(s1, s2);
                        /* enumeration is in (i, rank) ascending order, so a strict '<' keeps the
                         * lexicographic minimum of (score, i, rank) */
                        if (!found || score < best_score) {
                            found = 1; best_score = score; best_i = i; best_rank = rank;
                        }
                    }
                }
                if (found && best_score < Ws) {
                    sub_item(&bk[js], q, n, best_i); add_item(&bk[jp], q, n, best_i); a[best_i] = jp;
                    if (best_rank > 0) {
                        uint32_t i2 = best_rank - 1;
                        sub_item(&bk[jp], q, n, i2); add_item(&bk[js], q, n, i2); a[i2] = js;
                    }
                }
            }
        }
    }
    int st = score_partition(bk, p, T, cmax);
    if (st == ORC_OK && (bp->mode & ORC_MODE_ORDER4)) {
        /* N4(a) per candidate: every replica runs its best start order; T = the max over
         * replicas of that minimum (R37) */
        uint32_t S = p->e_pp + p->l_pp, M = p->n_mb;
        uint64_t* F = (uint64_t*)malloc(sizeof(uint64_t) * S * M);
        uint64_t* B = (uint64_t*)malloc(sizeof(uint64_t) * S * M);
        uint32_t* ord = (uint32_t*)malloc(sizeof(uint32_t) * M);
        uint64_t Tb = 0;
        for (uint32_t rho = 0; rho < p->l_dp; rho++) Tb = max64(Tb, best_start_order(bk, p, rho, F, B, ord));
        *T = Tb;
        free(F); free(B); free(ord);
    }
    if (assign_out) memcpy(assign_out, a, sizeof(uint32_t) * n);
    free(bk); free(a); free(order);
    return st;
}

/* ------------------------------------------------------------------------- */
/* N3: exact C_max by branch and bound, see the header.            */
/* ------------------------------------------------------------------------- */
typedef struct bb_state {
    const uint32_t* q;
    uint32_t n, m;
    const uint32_t* pi;       /* base order: items are placed in this order   */
    uint64_t* E;              /* [m] current encoder loads                    */
    uint64_t* L;              /* [m] current LLM loads                        */
    uint32_t* a;              /* [n] current assignment (by item)             */
    uint32_t* best;           /* [n] incumbent assignment                     */
    uint64_t incumbent, lb, nodes, budget;
    int stop, out_of_budget;
} bb_state;

static void bb_dfs(bb_state* st, uint32_t t, uint32_t used, uint64_t curmax) {
    if (st->stop) return;
    if (t == st->n) { /* leaf: pruning guarantees curmax < incumbent */
        st->incumbent = curmax;
        memcpy(st->best, st->a, sizeof(uint32_t) * st->n);
        if (st->incumbent <= st->lb) st->stop = 1;
        return;
    }
    uint32_t i = st->pi[t];
    uint64_t e = item_e(st->q, st->n, i), l = item_l(st->q, st->n, i);
    uint32_t lim = used < st->m ? used + 1 : st->m; /* first-use symmetry breaking */
    uint64_t w[256];
    uint32_t js[256];
    for (uint32_t j = 0; j < lim; j++) { /* children sorted by (resulting max, j): insertion */
        uint64_t v = max64(st->E[j] + e, st->L[j] + l);
        uint32_t k = j;
        while (k > 0 && w[k - 1] > v) { w[k] = w[k - 1]; js[k] = js[k - 1]; k--; }
        w[k] = v;
        js[k] = j;
    }
    for (uint32_t k = 0; k < lim && !st->stop; k++) {
        if (st->nodes >= st->budget) { st->stop = 1; st->out_of_budget = 1; return; }
        st->nodes++;
        uint64_t nm = max64(curmax, w[k]);
        if (max64(nm, st->lb) >= st->incumbent) continue; /* cannot beat the incumbent */
        uint32_t j = js[k];
        st->E[j] += e; st->L[j] += l; st->a[i] = j;
        bb_dfs(st, t + 1, j + 1 > used ? j + 1 : used, nm);
        st->E[j] -= e; st->L[j] -= l;
    }
}

int orc_exact_cmax(const uint32_t* q, uint32_t n, uint32_t m, uint64_t node_budget,
                   const uint32_t* init_assign, uint32_t* assign_out, uint64_t* cmax, uint64_t* lower_bound,
                   uint32_t* proven, uint64_t* nodes) {
    if (m == 0 || m > 256) return ORC_INVALID;
    bb_state st;
    memset(&st, 0, sizeof st);
    st.q = q; st.n = n; st.m = m; st.budget = node_budget;
    uint32_t* pi = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    st.E = (uint64_t*)calloc(m, sizeof(uint64_t));
    st.L = (uint64_t*)calloc(m, sizeof(uint64_t));
    st.a = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    st.best = (uint32_t*)calloc(n ? n : 1, sizeof(uint32_t));
    orc_base_order(q, n, pi);
    st.pi = pi;
    /* lower bound: averages per module and the largest single item */
    uint64_t se = 0, sl = 0, big = 0;
    for (uint32_t i = 0; i < n; i++) {
        uint64_t e = item_e(q, n, i), l = item_l(q, n, i);
        se += e; sl += l; big = max64(big, max64(e, l));
    }
    st.lb = max64(max64((se + m - 1) / m, (sl + m - 1) / m), big);
    /* initial incumbent */
    uint64_t* E0 = (uint64_t*)calloc(m, sizeof(uint64_t));
    uint64_t* L0 = (uint64_t*)calloc(m, sizeof(uint64_t));
    if (init_assign) {
        for (uint32_t i = 0; i < n; i++) {
            if (init_assign[i] >= m) { free(E0); free(L0); free(pi); free(st.E); free(st.L); free(st.a); free(st.best); return ORC_INVALID; }
            st.best[i] = init_assign[i];
        }
    } else { /* the paper's LPT: lowest current max(E_j, L_j), lowest j */
        for (uint32_t t = 0; t < n; t++) {
            uint32_t i = pi[t], bj = 0;
            for (uint32_t j = 1; j < m; j++)
                if (max64(E0[j], L0[j]) < max64(E0[bj], L0[bj])) bj = j;
            E0[bj] += item_e(q, n, i); L0[bj] += item_l(q, n, i);
            st.best[i] = bj;
        }
        memset(E0, 0, sizeof(uint64_t) * m); memset(L0, 0, sizeof(uint64_t) * m);
    }
    for (uint32_t i = 0; i < n; i++) { E0[st.best[i]] += item_e(q, n, i); L0[st.best[i]] += item_l(q, n, i); }
    st.incumbent = 0;
    for (uint32_t j = 0; j < m; j++) st.incumbent = max64(st.incumbent, max64(E0[j], L0[j]));
    free(E0); free(L0);
    if (st.incumbent > st.lb && n > 0) bb_dfs(&st, 0, 0, 0);
    *cmax = st.incumbent;
    *lower_bound = st.lb;
    *proven = (st.incumbent <= st.lb || !st.out_of_budget) ? 1u : 0u;
    *nodes = st.nodes;
    if (assign_out) memcpy(assign_out, st.best, sizeof(uint32_t) * n);
    free(pi); free(st.E); free(st.L); free(st.a); free(st.best);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* N3 for m = 2 and m = 4: exact C_max by pair decomposition (see the header).  */
/* Subsets are visited in Gray-code order (one element toggled per step), the   */
/* set sums updated by +/- that element; every subset is visited exactly once.  */
/* ------------------------------------------------------------------------- */
static uint32_t ctz64(uint64_t x) { uint32_t c = 0; while (!(x & 1ull)) { x >>= 1; c++; } return c; }

/* the best 2-way split of the k items (e[], l[]): min over subsets Y that contain item 0 of
 * max(E(Y), L(Y), E - E(Y), L - L(Y)); *best_y = a minimising subset (bit t = item t) */
static uint64_t best_split2(const uint64_t* e, const uint64_t* l, uint32_t k, uint64_t* best_y) {
    uint64_t SE = 0, SL = 0;
    for (uint32_t t = 0; t < k; t++) { SE += e[t]; SL += l[t]; }
    if (k == 0) { *best_y = 0; return 0; }
    /* Y = {0} u (Gray subset of items 1..k-1) */
    uint64_t y = 1ull, EY = e[0], LY = l[0];
    uint64_t best = max64(max64(EY, LY), max64(SE - EY, SL - LY));
    *best_y = y;
    uint64_t steps = 1ull << (k - 1);
    for (uint64_t i = 1; i < steps; i++) {
        uint32_t b = 1 + ctz64(i);              /* Gray code: toggle element 1 + ctz(i) */
        y ^= 1ull << b;
        if (y & (1ull << b)) { EY += e[b]; LY += l[b]; } else { EY -= e[b]; LY -= l[b]; }
        uint64_t v = max64(max64(EY, LY), max64(SE - EY, SL - LY));
        if (v < best) { best = v; *best_y = y; }
    }
    return best;
}

int orc_exact_pairs(const uint32_t* q, uint32_t n, uint32_t m, const uint32_t* init_assign, uint32_t* assign_out,
                    uint64_t* cmax, uint64_t* lower_bound, uint64_t* visited) {
    if ((m != 2 && m != 4) || n < 1 || n > 40) return ORC_INVALID;
    uint64_t e[40], l[40], SE = 0, SL = 0, big = 0;
    for (uint32_t i = 0; i < n; i++) {
        e[i] = item_e(q, n, i); l[i] = item_l(q, n, i);
        SE += e[i]; SL += l[i]; big = max64(big, max64(e[i], l[i]));
    }
    *lower_bound = max64(max64((SE + m - 1) / m, (SL + m - 1) / m), big);
    /* incumbent: the caller's assignment, else the paper's LPT (orc_exact_cmax's rule) */
    uint64_t inc = 0, lb2 = 0, nodes = 0;
    uint32_t proven = 0;
    uint32_t* a0 = (uint32_t*)malloc(sizeof(uint32_t) * n);
    if (orc_exact_cmax(q, n, m, 0, init_assign, a0, &inc, &lb2, &proven, &nodes) != ORC_OK) { free(a0); return ORC_INVALID; }
    uint64_t best = inc, bestX = 0, bestY1 = 0, bestY2 = 0, cnt = 0;
    int found = 0;
    if (m == 2) {
        uint64_t y;
        uint64_t v = best_split2(e, l, n, &y);
        cnt = 1ull << (n - 1);
        if (v < best) { best = v; bestX = y; found = 1; }
    } else if (inc > 0) {
        /* X = buckets {0, 1} (contains item 0), complement = buckets {2, 3}; a 4-way
         * assignment of max C has E(X), L(X) in [S - 2C, 2C]; only X's that can beat the
         * incumbent (C = inc - 1) are split */
        /* the window follows the best value found so far (C0 = best - 1) */
        uint64_t C0 = inc - 1;
        uint64_t loE = SE > 2 * C0 ? SE - 2 * C0 : 0, loL = SL > 2 * C0 ? SL - 2 * C0 : 0;
        uint64_t x = 1ull, EX = e[0], LX = l[0];
        uint64_t steps = 1ull << (n - 1);
        uint64_t ex[40], lx[40], ec[40], lc[40];
        for (uint64_t i = 0; i < steps; i++) {
            if (i > 0) {
                uint32_t b = 1 + ctz64(i);
                x ^= 1ull << b;
                if (x & (1ull << b)) { EX += e[b]; LX += l[b]; } else { EX -= e[b]; LX -= l[b]; }
            }
            cnt++;
            if (EX < loE || EX > 2 * C0 || LX < loL || LX > 2 * C0) continue;
            uint32_t kx = 0, kc = 0;
            for (uint32_t t = 0; t < n; t++) {
                if (x & (1ull << t)) { ex[kx] = e[t]; lx[kx] = l[t]; kx++; }
                else { ec[kc] = e[t]; lc[kc] = l[t]; kc++; }
            }
            uint64_t y1, y2;
            uint64_t v1 = best_split2(ex, lx, kx, &y1);
            if (v1 >= best) continue;
            uint64_t v2 = best_split2(ec, lc, kc, &y2);
            uint64_t v = max64(v1, v2);
            if (v < best) {
                best = v; bestX = x; bestY1 = y1; bestY2 = y2; found = 1;
                if (best == 0) break;
                C0 = best - 1;
                loE = SE > 2 * C0 ? SE - 2 * C0 : 0;
                loL = SL > 2 * C0 ? SL - 2 * C0 : 0;
            }
        }
    }
    *cmax = best;
    *visited = cnt;
    if (assign_out) {
        if (!found) memcpy(assign_out, a0, sizeof(uint32_t) * n);
        else if (m == 2) { for (uint32_t t = 0; t < n; t++) assign_out[t] = (bestX >> t) & 1ull ? 0u : 1u; }
        else {
            uint32_t kx = 0, kc = 0;
            for (uint32_t t = 0; t < n; t++) {
                if (bestX & (1ull << t)) { assign_out[t] = (bestY1 >> kx) & 1ull ? 0u : 1u; kx++; }
                else { assign_out[t] = (bestY2 >> kc) & 1ull ? 2u : 3u; kc++; }
            }
        }
    }
    free(a0);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* N4(a): microbatch-order search per replica (see the header).                */
/* ------------------------------------------------------------------------- */
static uint64_t order_makespan(const bucket_sums* bk, const orc_plan* p, uint32_t rho, const uint32_t* ord,
                               uint64_t* F, uint64_t* B) {
    uint32_t S = p->e_pp + p->l_pp, M = p->n_mb;
    for (uint32_t s = 0; s < S; s++)
        for (uint32_t k = 0; k < M; k++) {
            const bucket_sums* b = &bk[ord[k] * p->l_dp + rho];
            F[s * M + k] = s < p->e_pp ? b->EF : b->LF;
            B[s * M + k] = s < p->e_pp ? b->EB : b->LB;
        }
    uint64_t T = 0;
    orc_simulate_1f1b(F, B, S, M, &T, NULL);
    return T;
}

/* The four start orders of replica rho (N4(a), R35): 0 slot order, 1 ascending W_j =
 * max(E_j, L_j), 2 descending W (ties by slot), 3 valley; returns the least makespan (ties:
 * lowest order index) and that order in ord[M]. */
static uint64_t best_start_order(const bucket_sums* bk, const orc_plan* p, uint32_t rho, uint64_t* F, uint64_t* B,
                                 uint32_t* ord) {
    uint32_t M = p->n_mb;
    uint32_t* cand = (uint32_t*)malloc(sizeof(uint32_t) * M);
    uint32_t* asc = (uint32_t*)malloc(sizeof(uint32_t) * M);
    uint64_t* W = (uint64_t*)malloc(sizeof(uint64_t) * M);
    for (uint32_t k = 0; k < M; k++) {
        const bucket_sums* b = &bk[k * p->l_dp + rho];
        W[k] = max64(bE(b), bL(b));
        asc[k] = k;
    }
    for (uint32_t a = 1; a < M; a++) { /* stable insertion sort by W ascending */
        uint32_t x = asc[a], b = a;
        while (b > 0 && W[asc[b - 1]] > W[x]) { asc[b] = asc[b - 1]; b--; }
        asc[b] = x;
    }
    uint64_t bestT = 0;
    for (uint32_t o = 0; o < 4; o++) {
        if (o == 0) for (uint32_t k = 0; k < M; k++) cand[k] = k;
        if (o == 1) for (uint32_t k = 0; k < M; k++) cand[k] = asc[k];
        if (o == 2) { /* descending W, ties by slot ascending */
            uint32_t k = 0;
            for (uint32_t e = M; e > 0;) {
                uint32_t s0 = e - 1;
                while (s0 > 0 && W[asc[s0 - 1]] == W[asc[e - 1]]) s0--;
                for (uint32_t t = s0; t < e; t++) cand[k++] = asc[t];
                e = s0;
            }
        }
        if (o == 3) { /* valley */
            uint32_t lo = 0, hi = M - 1;
            for (uint32_t t = 0; t < M; t++) {
                if (t % 2 == 0) cand[lo++] = asc[t];
                else cand[hi--] = asc[t];
            }
        }
        uint64_t T = order_makespan(bk, p, rho, cand, F, B);
        if (o == 0 || T < bestT) { bestT = T; memcpy(ord, cand, sizeof(uint32_t) * M); }
    }
    free(cand); free(asc); free(W);
    return bestT;
}

int orc_order_search(const uint32_t* q, uint32_t n, const orc_plan* p, const uint32_t* assign, uint32_t rounds,
                     uint32_t* order_out, uint64_t* T_out) {
    uint32_t m = p->n_mb * p->l_dp, M = p->n_mb, S = p->e_pp + p->l_pp;
    bucket_sums* bk = (bucket_sums*)calloc(m, sizeof(bucket_sums));
    for (uint32_t i = 0; i < n; i++) {
        if (assign[i] >= m) { free(bk); return ORC_INVALID; }
        add_item(&bk[assign[i]], q, n, i);
    }
    uint64_t* F = (uint64_t*)malloc(sizeof(uint64_t) * S * M);
    uint64_t* B = (uint64_t*)malloc(sizeof(uint64_t) * S * M);
    uint32_t* ord = (uint32_t*)malloc(sizeof(uint32_t) * M);
    for (uint32_t rho = 0; rho < p->l_dp; rho++) {
        uint64_t bestT = best_start_order(bk, p, rho, F, B, ord);
        for (uint32_t r = 0; r < rounds; r++) {
            uint64_t rT = 0;
            uint32_t ra = 0, rb = 0;
            int found = 0;
            for (uint32_t a = 0; a < M; a++)
                for (uint32_t b = a + 1; b < M; b++) {
                    if (M > 128 && b - a > 16) break;
                    uint32_t t = ord[a]; ord[a] = ord[b]; ord[b] = t;
                    uint64_t T = order_makespan(bk, p, rho, ord, F, B);
                    t = ord[a]; ord[a] = ord[b]; ord[b] = t;
                    if (!found || T < rT) { found = 1; rT = T; ra = a; rb = b; } /* (T, a, b) order */
                }
            if (!found || rT >= bestT) break;
            uint32_t t = ord[ra]; ord[ra] = ord[rb]; ord[rb] = t;
            bestT = rT;
        }
        for (uint32_t k = 0; k < M; k++) order_out[rho * M + k] = ord[k] * p->l_dp + rho;
        T_out[rho] = bestT;
    }
    free(bk); free(F); free(B); free(ord);
    return ORC_OK;
}

/* ------------------------------------------------------------------------- */
/* N4(b): inter-model routing plan (see the header).                          */
/* ------------------------------------------------------------------------- */
int orc_route_plan(const uint32_t* q, uint32_t n, const orc_plan* p, const uint32_t* assign, uint32_t* pos_item,
                   uint32_t* slot_off, uint32_t* enc_off, uint32_t* llm_off, uint64_t* enc_load) {
    uint32_t M = p->n_mb, R = p->l_dp, G = p->e_dp, m = M * R;
    for (uint32_t i = 0; i < n; i++)
        if (assign[i] >= m) return ORC_INVALID;
    uint32_t t = 0;
    for (uint32_t k = 0; k < M; k++) {
        slot_off[k] = t;
        for (uint32_t rho = 0; rho < R; rho++) {
            llm_off[k * (R + 1) + rho] = t;
            for (uint32_t i = 0; i < n; i++) /* bucket members, sample index ascending */
                if (assign[i] == k * R + rho) pos_item[t++] = i;
        }
        llm_off[k * (R + 1) + R] = t;
        uint32_t a = slot_off[k], b = t;
        uint64_t tot = 0;
        for (uint32_t u = a; u < b; u++) tot += item_e(q, n, pos_item[u]);
        enc_off[k * (G + 1)] = a;
        for (uint32_t g = 1; g < G; g++) {
            /* first position whose preceding encoder cost reaches g/G of the slot's */
            uint64_t pre = 0;
            uint32_t u = a;
            while (u < b && pre * G < (uint64_t)g * tot) pre += item_e(q, n, pos_item[u++]);
            enc_off[k * (G + 1) + g] = u;
        }
        enc_off[k * (G + 1) + G] = b;
        if (enc_load)
            for (uint32_t g = 0; g < G; g++) {
                uint64_t s = 0;
                for (uint32_t u = enc_off[k * (G + 1) + g]; u < enc_off[k * (G + 1) + g + 1]; u++)
                    s += item_e(q, n, pos_item[u]);
                enc_load[k * G + g] = s;
            }
    }
    slot_off[M] = t;
    return ORC_OK;
}

int orc_balance(const uint32_t* q, uint32_t n, const orc_plan* p, const orc_bparams* bp, uint32_t c0,
                uint32_t c1, uint64_t* cand_T, uint64_t* cand_cmax, uint64_t* best_T, uint32_t* best_c,
                uint64_t* best_cmax, uint32_t* best_assign) {
    uint32_t* pi = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * (n ? n : 1));
    orc_base_order(q, n, pi);
    int found = 0, st = ORC_OK;
    for (uint32_t c = c0; c < c1; c++) {
        uint64_t T = 0, cm = 0;
        st = orc_run_candidate(q, n, p, bp, pi, c, a, &T, &cm);
        if (st != ORC_OK) break;
        if (cand_T) cand_T[c - c0] = T;
        if (cand_cmax) cand_cmax[c - c0] = cm;
        /* argmin (T_c, c), lowest candidate id on ties (R18); c ascending here */
        if (!found || T < *best_T) {
            found = 1;
            *best_T = T; *best_c = c; *best_cmax = cm;
            if (best_assign) memcpy(best_assign, a, sizeof(uint32_t) * n);
        }
    }
    free(pi); free(a);
    return st;
}

void orc_groups(const uint32_t* assign, uint32_t n, uint32_t m, uint32_t* offsets, uint32_t* items) {
    for (uint32_t j = 0; j <= m; j++) offsets[j] = 0;
    for (uint32_t i = 0; i < n; i++) offsets[assign[i] + 1]++;
    for (uint32_t j = 0; j < m; j++) offsets[j + 1] += offsets[j];
    uint32_t* fill = (uint32_t*)calloc(m ? m : 1, sizeof(uint32_t));
    for (uint32_t i = 0; i < n; i++) {
        uint32_t j = assign[i];
        items[offsets[j] + fill[j]++] = i;
    }
    free(fill);
}

/* ------------------------------------------------------------------------- */
/* Algorithm 1.                                                    */
/* ------------------------------------------------------------------------- */
/* FindCombs(g): all (tp, pp, dp) with tp*pp*dp = g and tp <= N_gpu_node (Eq. 2),
 * ascending tp then ascending pp (the enumeration index eps follows this order). */
uint32_t orc_find_combs(uint32_t gpus, uint32_t node, uint32_t* out3, uint32_t cap) {
    uint32_t cnt = 0;
    for (uint32_t tp = 1; tp <= gpus && tp <= node; tp++) {
        if (gpus % tp) continue;
        for (uint32_t pp = 1; pp <= gpus / tp; pp++) {
            if ((gpus / tp) % pp) continue;
            if (out3 && cnt < cap) {
                out3[3 * cnt + 0] = tp; out3[3 * cnt + 1] = pp; out3[3 * cnt + 2] = gpus / tp / pp;
            }
            cnt++;
        }
    }
    return cnt;
}

/* Phase 1: for E_gpus = 1..N-1, the cartesian product FindCombs(E_gpus) x FindCombs(N - E_gpus)
 * (R16), E configurations outer, L inner.  out6 rows are (E_tp,E_pp,E_dp,L_tp,L_pp,L_dp). */
uint64_t orc_enumerate_configs(uint32_t n_gpus, uint32_t node, uint32_t* out6, uint64_t cap) {
    uint64_t cnt = 0;
    uint32_t* ec = (uint32_t*)malloc(sizeof(uint32_t) * 3 * 4096);
    uint32_t* lc = (uint32_t*)malloc(sizeof(uint32_t) * 3 * 4096);
    for (uint32_t eg = 1; eg < n_gpus; eg++) {
        uint32_t ne = orc_find_combs(eg, node, ec, 4096);
        uint32_t nl = orc_find_combs(n_gpus - eg, node, lc, 4096);
        for (uint32_t a = 0; a < ne; a++)
            for (uint32_t b = 0; b < nl; b++) {
                if (out6 && cnt < cap) {
                    uint32_t* r = out6 + 6 * cnt;
                    r[0] = ec[3 * a]; r[1] = ec[3 * a + 1]; r[2] = ec[3 * a + 2];
                    r[3] = lc[3 * b]; r[4] = lc[3 * b + 1]; r[5] = lc[3 * b + 2];
                }
                cnt++;
            }
    }
    free(ec); free(lc);
    return cnt;
}

/* P:601 (mean_bsz, mean_seq_len) <- Profiled.Data.mean(): here the means of the batch. */
void orc_batch_means(const orc_model* m, const uint32_t* tiles, const uint32_t* frames, const uint32_t* text,
                     uint32_t n, double* mean_b, double* mean_s) {
    uint64_t sb = 0, ss = 0;
    for (uint32_t i = 0; i < n; i++) {
        sb += (uint64_t)tiles[i] + frames[i];
        ss += (uint64_t)text[i] + (uint64_t)m->tau_tile * tiles[i] + (uint64_t)m->tau_frame * frames[i];
    }
    *mean_b = n ? (double)sb / (double)n : 0.0;
    *mean_s = n ? (double)ss / (double)n : 0.0;
}

static uint64_t round_u64(double x) {
    if (!(x < 18446744073709549568.0)) return UINT64_MAX;
    return (uint64_t)nearbyint(x);
}

/* Algorithm 1 lines 15-27 for one (config, i):
 *   t_bsz = mean_bsz * GBS / (i * E_dp); t_seq = mean_seq * GBS / (i * L_dp)
 *   Mem_E = ms_E(ceil(E_l/E_pp), E_tp) + (E_pp + L_pp) * as_E(ceil(E_l/E_pp), E_tp, t_bsz)  Eq. 4
 *   Mem_L = ms_L(ceil(L_l/L_pp), L_tp) + L_pp * as_L(ceil(L_l/L_pp), L_tp, t_seq)          Eq. 5
 *   skip if either > M_gpu
 *   E_dur = E_FLOP / (E_thr(t_bsz, E_tp) * E_tp * E_pp)
 *   L_dur = L_FLOP / (L_thr(t_seq, L_tp) * L_tp * L_pp), attention per instance at the mean
 *           length (R5) and linear over the packed microbatch
 *   T = (i + E_pp + L_pp - 1) * max(E_dur, L_dur)
 * Durations round to integer ticks before T (R19). */
int orc_stage_a_pair(const orc_model* m, const orc_mem* mm, const uint32_t cfg[6], uint32_t i, uint32_t gbs,
                     double mean_b, double mean_s, uint64_t* T_A, double* mem_e, double* mem_l, uint64_t* e_dur,
                     uint64_t* l_dur) {
    uint32_t e_tp = cfg[0], e_pp = cfg[1], e_dp = cfg[2], l_tp = cfg[3], l_pp = cfg[4], l_dp = cfg[5];
    double t_bsz = (mean_b * (double)gbs) / ((double)i * (double)e_dp);
    double t_seq = (mean_s * (double)gbs) / ((double)i * (double)l_dp);
    double le = (double)((m->e_layers + e_pp - 1) / e_pp);
    double ll = (double)((m->l_layers + l_pp - 1) / l_pp);
    double Me = orc_interp_mem(&mm->ms_e, le, (double)e_tp, 0.0) +
                (double)(e_pp + l_pp) * orc_interp_mem(&mm->as_e, le, (double)e_tp, t_bsz);
    double Ml = orc_interp_mem(&mm->ms_l, ll, (double)l_tp, 0.0) +
                (double)l_pp * orc_interp_mem(&mm->as_l, ll, (double)l_tp, t_seq);
    if (mem_e) *mem_e = Me;
    if (mem_l) *mem_l = Ml;
    if (Me > mm->mem_per_gpu || Ml > mm->mem_per_gpu) {
        *T_A = UINT64_MAX;
        return 0;
    }
    double lin_e = 24.0 * (double)m->e_hidden * (double)m->e_hidden;
    double att_e = m->e_attn ? 4.0 * (double)m->e_hidden : 0.0;
    double per_inst_e = lin_e * (double)m->e_seq + att_e * (double)m->e_seq * (double)m->e_seq;
    double c_e = (double)m->e_layers * per_inst_e;
    double c_lin = 24.0 * (double)m->l_hidden * (double)m->l_hidden * (double)m->l_layers;
    double c_att = 4.0 * (double)m->l_hidden * (double)m->l_layers;
    double EF = t_bsz * c_e;
    double thr_e = orc_interp_thr(&m->thr_e, t_bsz, (double)e_tp);
    double Ed = 1e9 * EF / (thr_e * (double)e_tp * (double)e_pp);
    double nbar = (double)gbs / ((double)i * (double)l_dp);
    double Latt = nbar * (c_att * mean_s * mean_s);
    double Llin = c_lin * t_seq;
    double thr_a = orc_interp_thr(&m->thr_att, t_seq, (double)l_tp);
    double thr_l = orc_interp_thr(&m->thr_lin, t_seq, (double)l_tp);
    double Ld = 1e9 * (Latt / thr_a + Llin / thr_l) / ((double)l_tp * (double)l_pp);
    uint64_t qe = round_u64(Ed / m->tick_ns), ql = round_u64(Ld / m->tick_ns);
    if (e_dur) *e_dur = qe;
    if (l_dur) *l_dur = ql;
    uint64_t mx = qe > ql ? qe : ql;
    unsigned __int128 T = (unsigned __int128)(i + e_pp + l_pp - 1) * mx;
    *T_A = T > (unsigned __int128)(UINT64_MAX - 1) ? UINT64_MAX - 1 : (uint64_t)T;
    return 1;
}

uint64_t orc_stage_a_all(const orc_model* m, const orc_mem* mm, uint32_t n_gpus, uint32_t node, uint32_t gbs,
                         double mean_b, double mean_s, uint64_t* T_A, uint64_t cap) {
    uint64_t nc = orc_enumerate_configs(n_gpus, node, NULL, 0);
    uint32_t* cfg = (uint32_t*)malloc(sizeof(uint32_t) * 6 * (nc ? nc : 1));
    orc_enumerate_configs(n_gpus, node, cfg, nc);
    uint64_t k = 0;
    for (uint64_t e = 0; e < nc; e++) {
        uint32_t nmax = gbs / cfg[6 * e + 5]; /* N_max_mbatch = GBS // L_dp (R17) */
        for (uint32_t i = 1; i <= nmax; i++) {
            uint64_t T = UINT64_MAX;
            orc_stage_a_pair(m, mm, cfg + 6 * e, i, gbs, mean_b, mean_s, &T, NULL, NULL, NULL, NULL);
            if (k < cap) T_A[k] = T;
            k++;
        }
    }
    free(cfg);
    return k;
}

/* Algorithm 1's strict '<' keeps the first minimum in enumeration order, i.e. the
 * lexicographic minimum of (T_A, eps, i); the pair index is that enumeration order. */
static const uint64_t* g_top_T;
static int cmp_pair(const void* pa, const void* pb) {
    uint64_t a = *(const uint64_t*)pa, b = *(const uint64_t*)pb;
    if (g_top_T[a] != g_top_T[b]) return g_top_T[a] < g_top_T[b] ? -1 : 1;
    return a < b ? -1 : (a > b ? 1 : 0);
}

uint32_t orc_stage_a_top(const uint64_t* T_A, uint64_t n_pairs, uint32_t P, uint64_t* top) {
    uint64_t nf = 0;
    for (uint64_t k = 0; k < n_pairs; k++) nf += T_A[k] != UINT64_MAX;
    uint64_t* idx = (uint64_t*)malloc(sizeof(uint64_t) * (nf ? nf : 1));
    uint64_t w = 0;
    for (uint64_t k = 0; k < n_pairs; k++)
        if (T_A[k] != UINT64_MAX) idx[w++] = k;
    g_top_T = T_A;
    qsort(idx, nf, sizeof(uint64_t), cmp_pair);
    uint32_t out = (uint32_t)(nf < P ? nf : P);
    for (uint32_t r = 0; r < out; r++) top[r] = idx[r];
    free(idx);
    return out;
}
