// predict.cu -- step a1: per-sample stage costs from data features.
//
//   b = tiles + frames, s = text + tau_tile*tiles + tau_frame*frames
//   ef = scale_e * b / E_thr(b, E_tp)                     (0 when b == 0)
//   lf = scale_att * s^2 / L_attn_thr(s, L_tp) + scale_lin * s / L_lin_thr(s, L_tp)
//   eb = r * ef, lb = r * lf
// where the host folds 1e9 * FLOPs-per-unit / (tp * pp) / tick (and L_dp / E_dp, R13) into
// the fp32 scale constants in double precision, and blends each grid's two TP rows at the
// plan's TP once (double, then fp32).  Per sample: three binary-searched interpolations, three
// reciprocals.  One thread handles 4 consecutive samples with 16-byte loads/stores: 12 B in
// and 32 B out per sample and plan.  Multi-plan launches (Stage B of the search) use
// blockIdx.y as the plan index.
#include <algorithm>
#include <cmath>

#include "common.cuh"
#include "internal.h"

namespace dflop {

// Knots of one throughput grid and the reciprocal interval widths (shared by all plans).
struct PredictKnots {
    float x[DFLOP_MAX_X];
    float inv[DFLOP_MAX_X];  // 1 / (x[k+1] - x[k]) (from double)
    int n_x;
    int e0;                  // knots are exactly 2^(e0 + k): k from the float exponent; else -1000
};
struct PredictGrids {
    PredictKnots e, att, lin;
    float rho[3][DFLOP_CORR_BINS];  // N1 Adaptive Correction ratios (all 1 when inactive)
    int corr;                       // correction active
    int pad[3];
};

// N1 shape bin: floor(log2 x) from the integer shape, x = 0 -> 0, clamped (R30)
DFLOP_DEV uint32_t shape_bin(u64 x) {
    const uint32_t q = x ? 63u - (uint32_t)__clzll((long long)x) : 0u;
    return q < DFLOP_CORR_BINS ? q : DFLOP_CORR_BINS - 1;
}
// Per plan: the constants and, for each grid, the row blended at the plan's TP (the blend
// weight is uniform per plan, and interpolation is linear in the row values, so blending the
// rows once equals blending the two row interpolations of O3 up to rounding).
struct PredictPlan {
    PredictConsts c;
    float ve[DFLOP_MAX_X], va[DFLOP_MAX_X], vl[DFLOP_MAX_X];
};
constexpr int kPredictPlans = 16;  // plans per launch (kernel-parameter budget)
struct PredictLaunch {
    PredictPlan pl[kPredictPlans];
};

// O3 interp1 on the blended row: clamp, k = largest index with x_k <= x and k <= n-2 (binary
// search), w = (x - x_k) / (x_{k+1} - x_k), (1 - w) v_k + w v_{k+1} (exact at the knots)
DFLOP_DEV float interp_row(const PredictKnots& g, const float* v, float x) {
    const int n = g.n_x;
    if (n == 1) return v[0];
    const float xh = fminf(fmaxf(x, g.x[0]), g.x[n - 1]);
    int k = 0;
    if (g.e0 > -1000) {  // power-of-two knots: floor(log2 xh) - e0, the same k as the search
        k = min((int)(__float_as_uint(xh) >> 23) - 127 - g.e0, n - 2);
    } else {
#pragma unroll
        for (int step = DFLOP_MAX_X / 2; step > 0; step >>= 1)
            if (k + step <= n - 2 && g.x[k + step] <= xh) k += step;
    }
    const float w = (xh - g.x[k]) * g.inv[k];
    return (1.0f - w) * v[k] + w * v[k + 1];
}

DFLOP_DEV uint32_t to_ticks(float v, uint32_t& ovf) {
    if (!(v < 4294967296.0f)) {
        ovf = 1;
        return 0xFFFFFFFFu;
    }
    return __float2uint_rn(v);
}

template <bool VEC>
__global__ void __launch_bounds__(256) k_predict(PredictGrids grids, PredictLaunch L, const uint32_t* __restrict__ tiles,
                                                 const uint32_t* __restrict__ frames, const uint32_t* __restrict__ text,
                                                 uint32_t n, float* cost_f32, uint32_t* cost_ticks, size_t plan_stride,
                                                 size_t rs, uint32_t* dev_status) {
    __shared__ PredictGrids g;
    __shared__ PredictPlan pp;
    for (uint32_t w = threadIdx.x; w < sizeof(PredictGrids) / 4; w += blockDim.x)
        reinterpret_cast<uint32_t*>(&g)[w] = reinterpret_cast<const uint32_t*>(&grids)[w];
    for (uint32_t w = threadIdx.x; w < sizeof(PredictPlan) / 4; w += blockDim.x)
        reinterpret_cast<uint32_t*>(&pp)[w] = reinterpret_cast<const uint32_t*>(&L.pl[blockIdx.y])[w];
    __syncthreads();
    const PredictConsts k = pp.c;
    float* f32 = cost_f32 ? cost_f32 + (size_t)blockIdx.y * plan_stride : nullptr;
    uint32_t* tk = cost_ticks ? cost_ticks + (size_t)blockIdx.y * plan_stride : nullptr;
    uint32_t ovf = 0;
    const uint32_t nq = VEC ? n / 4 : n;
    const uint32_t q_first = blockIdx.x * blockDim.x + threadIdx.x, q_step = gridDim.x * blockDim.x;
    // VEC: the next iteration's three 16-byte feature loads are issued before this iteration's
    // arithmetic, so two iterations' loads are in flight per thread (HBM latency hiding)
    uint4 na = make_uint4(0, 0, 0, 0), nb = na, nc = na;
    if (VEC && q_first < nq) {
        na = __ldg(reinterpret_cast<const uint4*>(tiles) + q_first);
        nb = __ldg(reinterpret_cast<const uint4*>(frames) + q_first);
        nc = __ldg(reinterpret_cast<const uint4*>(text) + q_first);
    }
    for (uint32_t q = q_first; q < nq; q += q_step) {
        uint32_t tv[4], fv[4], xv[4];
        const int cnt = VEC ? 4 : 1;
        if (VEC) {
            const uint4 a = na, b = nb, c = nc;
            if (q + q_step < nq) {
                na = __ldg(reinterpret_cast<const uint4*>(tiles) + q + q_step);
                nb = __ldg(reinterpret_cast<const uint4*>(frames) + q + q_step);
                nc = __ldg(reinterpret_cast<const uint4*>(text) + q + q_step);
            }
            tv[0] = a.x; tv[1] = a.y; tv[2] = a.z; tv[3] = a.w;
            fv[0] = b.x; fv[1] = b.y; fv[2] = b.z; fv[3] = b.w;
            xv[0] = c.x; xv[1] = c.y; xv[2] = c.z; xv[3] = c.w;
        } else {
            tv[0] = __ldg(tiles + q);
            fv[0] = __ldg(frames + q);
            xv[0] = __ldg(text + q);
        }
        float o[4][4];
        uint32_t t4[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (u >= cnt) break;
            const u64 bi = (u64)tv[u] + fv[u];
            const u64 si = (u64)xv[u] + (u64)k.tau_tile * tv[u] + (u64)k.tau_frame * fv[u];
            const float b = (float)bi, s = (float)si;
            float te = interp_row(g.e, pp.ve, b), ta = interp_row(g.att, pp.va, s), tl = interp_row(g.lin, pp.vl, s);
            if (g.corr) {  // N1: corrected throughput of the sample's shape bins (one lookup each)
                const uint32_t qb = shape_bin(bi), qs = shape_bin(si);
                te *= g.rho[0][qb];
                ta *= g.rho[1][qs];
                tl *= g.rho[2][qs];
            }
            float ef = 0.0f;
            if (b > 0.0f) ef = (k.scale_e * b) * __frcp_rn(te);
            const float lf = (k.scale_att * s * s) * __frcp_rn(ta) + (k.scale_lin * s) * __frcp_rn(tl);
            o[0][u] = ef;
            o[1][u] = k.bwd * ef;
            o[2][u] = lf;
            o[3][u] = k.bwd * lf;
#pragma unroll
            for (int r = 0; r < 4; ++r) t4[r][u] = to_ticks(o[r][u], ovf);
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (VEC) {
                if (f32) reinterpret_cast<float4*>(f32 + (size_t)r * rs)[q] = make_float4(o[r][0], o[r][1], o[r][2], o[r][3]);
                if (tk) reinterpret_cast<uint4*>(tk + (size_t)r * rs)[q] = make_uint4(t4[r][0], t4[r][1], t4[r][2], t4[r][3]);
            } else {
                if (f32) f32[(size_t)r * rs + q] = o[r][0];
                if (tk) tk[(size_t)r * rs + q] = t4[r][0];
            }
        }
    }
    if (ovf && dev_status) atomicOr(dev_status, (uint32_t)DFLOP_DEV_COST_OVERFLOW);
}

static void to_knots(const dflop_grid& s, PredictKnots& d) {
    d.n_x = (int)s.n_x;
    // knots x_k = 2^(e0 + k) exactly, with 2^e0 >= 1 (every float in range is normal)
    d.e0 = -1000;
    if (s.n_x >= 2 && s.x[0] >= 1.0) {
        int e0 = 0;
        const double f = std::frexp(s.x[0], &e0);  // x0 = f * 2^e0, f in [0.5, 1)
        bool pow2 = f == 0.5;
        for (uint32_t k = 0; pow2 && k < s.n_x; ++k) pow2 = s.x[k] == std::ldexp(1.0, e0 - 1 + (int)k);
        if (pow2 && e0 - 1 + (int)s.n_x < 127) d.e0 = e0 - 1;
    }
    for (int k = 0; k < DFLOP_MAX_X; ++k) {
        d.x[k] = k < (int)s.n_x ? (float)s.x[k] : 0.0f;
        d.inv[k] = k + 1 < (int)s.n_x ? (float)(1.0 / (s.x[k + 1] - s.x[k])) : 0.0f;
    }
}

// the grid's row at throughput-TP `tp`: O3's TP bracket (clamp, largest a <= q-2 with
// t_a <= tp) and weight, applied to the rows in double
static void blend_row(const dflop_grid& s, double tp, float* out) {
    int a = 0;
    double wt = 0.0;
    if (s.n_tp > 1) {
        const double th = std::min(std::max(tp, s.tp[0]), s.tp[s.n_tp - 1]);
        while (a + 1 < (int)s.n_tp - 1 && s.tp[a + 1] <= th) ++a;
        wt = (th - s.tp[a]) / (s.tp[a + 1] - s.tp[a]);
    }
    for (int k = 0; k < DFLOP_MAX_X; ++k) {
        if (k >= (int)s.n_x) {
            out[k] = 0.0f;
        } else if (s.n_tp == 1) {
            out[k] = (float)s.v[0][k];
        } else {
            out[k] = (float)((1.0 - wt) * s.v[a][k] + wt * s.v[a + 1][k]);
        }
    }
}

PredictConsts predict_consts(const dflop_cost_model* m, const dflop_plan* p) {
    // FLOP accounting R1: 24*h^2 per token and layer (linear), 4*h*s^2 attention.
    const double lin_e = 24.0 * (double)m->e_hidden * (double)m->e_hidden;
    const double att_e = m->e_attn ? 4.0 * (double)m->e_hidden : 0.0;
    const double per_inst_e = lin_e * (double)m->e_seq + att_e * (double)m->e_seq * (double)m->e_seq;
    const double c_e = (double)m->e_layers * per_inst_e;
    const double c_lin = 24.0 * (double)m->l_hidden * (double)m->l_hidden * (double)m->l_layers;
    const double c_att = 4.0 * (double)m->l_hidden * (double)m->l_layers;
    PredictConsts k;
    // divide by thr * tp * pp; R13: encoder time per LLM bucket x L_dp / E_dp
    k.scale_e = (float)(1e9 * c_e / ((double)p->e_tp * (double)p->e_pp) * ((double)p->l_dp / (double)p->e_dp) /
                        m->tick_ns);
    k.scale_att = (float)(1e9 * c_att / ((double)p->l_tp * (double)p->l_pp) / m->tick_ns);
    k.scale_lin = (float)(1e9 * c_lin / ((double)p->l_tp * (double)p->l_pp) / m->tick_ns);
    k.bwd = (float)m->bwd_ratio;
    k.tau_tile = m->tau_tile;
    k.tau_frame = m->tau_frame;
    k.tp_e = (float)p->e_tp;
    k.tp_l = (float)p->l_tp;
    return k;
}

static cudaError_t predict_impl(const dflop_cost_model* m, const PredictConsts* consts, uint32_t n_plans,
                                const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                                float* cost_f32, uint32_t* cost_ticks, size_t rs, size_t plan_stride,
                                uint32_t* dev_status, cudaStream_t s) {
    if (n == 0 || n_plans == 0) return cudaSuccess;
    PredictGrids g;
    to_knots(m->thr_e, g.e);
    to_knots(m->thr_att, g.att);
    to_knots(m->thr_lin, g.lin);
    g.corr = (m->correction && m->correction->active) ? 1 : 0;
    for (int q = 0; q < 3; ++q)
        for (int k = 0; k < DFLOP_CORR_BINS; ++k) g.rho[q][k] = g.corr ? m->correction->rho[q][k] : 1.0f;
    g.pad[0] = g.pad[1] = g.pad[2] = 0;
    const bool vec = (n % 4 == 0) && ((uintptr_t)tiles % 16 == 0) && ((uintptr_t)frames % 16 == 0) &&
                     ((uintptr_t)text % 16 == 0) && (!cost_f32 || (uintptr_t)cost_f32 % 16 == 0) &&
                     (!cost_ticks || (uintptr_t)cost_ticks % 16 == 0) && (plan_stride % 4 == 0) && (rs % 4 == 0);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t work = vec ? n / 4 : n;
    for (uint32_t p0 = 0; p0 < n_plans; p0 += kPredictPlans) {
        const uint32_t np = std::min<uint32_t>(kPredictPlans, n_plans - p0);
        PredictLaunch L;
        for (uint32_t i = 0; i < np; ++i) {
            L.pl[i].c = consts[p0 + i];
            blend_row(m->thr_e, consts[p0 + i].tp_e, L.pl[i].ve);
            blend_row(m->thr_att, consts[p0 + i].tp_l, L.pl[i].va);
            blend_row(m->thr_lin, consts[p0 + i].tp_l, L.pl[i].vl);
        }
        const uint32_t gx = std::max(1u, std::min<uint32_t>((work + 255) / 256, (uint32_t)sms * 8 / np + 1));
        dim3 grid(gx, np);
        float* f = cost_f32 ? cost_f32 + (size_t)p0 * plan_stride : nullptr;
        uint32_t* t = cost_ticks ? cost_ticks + (size_t)p0 * plan_stride : nullptr;
        if (vec)
            k_predict<true><<<grid, 256, 0, s>>>(g, L, tiles, frames, text, n, f, t, plan_stride, rs, dev_status);
        else
            k_predict<false><<<grid, 256, 0, s>>>(g, L, tiles, frames, text, n, f, t, plan_stride, rs, dev_status);
        count_launches(1);
    }
    return cudaGetLastError();
}

cudaError_t predict_launch(const dflop_cost_model* m, const PredictConsts* consts, uint32_t n_plans,
                           const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                           float* cost_f32, uint32_t* cost_ticks, size_t plan_stride, uint32_t* dev_status,
                           cudaStream_t s) {
    return predict_impl(m, consts, n_plans, tiles, frames, text, n, cost_f32, cost_ticks, n, plan_stride, dev_status, s);
}

cudaError_t predict_launch_rows(const dflop_cost_model* m, const PredictConsts* consts, uint32_t n_plans,
                                const uint32_t* tiles, const uint32_t* frames, const uint32_t* text, uint32_t n,
                                uint32_t* cost_ticks, size_t row_stride, size_t plan_stride, uint32_t* dev_status,
                                cudaStream_t s) {
    return predict_impl(m, consts, n_plans, tiles, frames, text, n, nullptr, cost_ticks, row_stride, plan_stride,
                        dev_status, s);
}

}  // namespace dflop
