// int_peaks.cu -- microbenchmark of the B200 integer / shuffle issue rates that bound the
// candidate kernel (SURVEY 8(d) "int32 and shuffle lanes per SM per clock ... confirmed by
// microbenchmark"; VERDICT r01 "Next 2").  Standalone: nvcc -gencode arch=compute_100a,
// code=sm_100a -O3 -o int_peaks int_peaks.cu; ./int_peaks > int_peaks.json.
//
// For each instruction class a kernel runs ILP independent chains per thread over the whole
// GPU (148 SMs x 2 CTAs x 1024 threads), the body written in inline PTX so ptxas emits the
// intended SASS (checked with tools/sass_hist.py: one IADD3 (3-input, a + x + y) per iadd3
// step, VIMNMX, VIADDMNMX, IMAD, LOP3, SHFL.BFLY per step; redux = CREDUX.MIN + IMAD.U32 (the
// uniform result moved back to a vector register); add_u32_ptxas_choice = 2-input adds that
// ptxas splits between IADD3 (ALU pipe) and IMAD.IADD (FMA pipe); iadd3+imad alternates).
// The SM clock is measured inside the kernel (clock64 vs globaltimer on thread 0 of every
// CTA), so the result is lane-ops per SM per clock, independent of DVFS, plus the lane-op rate
// at the measured clock.  A dependent single-chain run gives the latency in cycles.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include <vector>
#include <algorithm>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); return 1; } } while (0)

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

enum Op { IADD = 0, IMIN = 1, IADDMIN = 2, IMAD = 3, LOP = 4, SHFL = 5, MIX_ADD_MAD = 6, REDUXMIN = 7, ADD2 = 8, N_OPS = 9 };
static const char* kNames[N_OPS] = {"iadd3", "vimnmx_u32", "viaddmnmx_u32", "imad", "lop3", "shfl_bfly", "iadd3+imad", "redux_min_u32", "add_u32_ptxas_choice"};

template <int OP>
__device__ __forceinline__ void step(uint32_t& a, uint32_t b, uint32_t c) {
    if constexpr (OP == IADD) asm volatile("add.u32 %0, %0, %1;\n\tadd.u32 %0, %0, %2;" : "+r"(a) : "r"(b), "r"(c));
    else if constexpr (OP == ADD2) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
    else if constexpr (OP == IMIN) asm volatile("min.u32 %0, %0, %1;" : "+r"(a) : "r"(b));
    else if constexpr (OP == IADDMIN) a = __viaddmin_u32(a, b, c);
    else if constexpr (OP == IMAD) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a) : "r"(b), "r"(c));
    else if constexpr (OP == LOP) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a) : "r"(b), "r"(c));
    else if constexpr (OP == SHFL) asm volatile("shfl.sync.bfly.b32 %0, %0, 1, 0x1f, -1;" : "+r"(a));
    else if constexpr (OP == REDUXMIN) asm volatile("redux.sync.min.u32 %0, %0, -1;" : "+r"(a));
}

template <int OP, int ILP>
__global__ void k_tput(uint32_t iters, uint32_t seed, uint32_t* out, uint64_t* clk, uint64_t* ns) {
    uint32_t a[ILP];
    uint32_t b = seed ^ threadIdx.x, c = seed * 3u + blockIdx.x;
#pragma unroll
    for (int k = 0; k < ILP; k++) a[k] = threadIdx.x * (k + 1) + seed;
    __syncthreads();
    uint64_t c0 = clock64(), t0 = gtimer();
    for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int k = 0; k < ILP; k++) {
                // ring of chains: every op reads two other chains, so no two ops fold into one
                const uint32_t x = (OP == SHFL || OP == REDUXMIN || ILP == 1) ? b : a[(k + 1) % ILP];
                const uint32_t y = (OP == SHFL || OP == REDUXMIN || ILP == 1) ? c : a[(k + 3) % ILP];
                if constexpr (OP == MIX_ADD_MAD) {
                    if (k & 1) step<IMAD>(a[k], x, y);
                    else step<IADD>(a[k], x, y);
                } else {
                    step<OP>(a[k], x, y);
                }
            }
        }
    }
    __syncthreads();
    uint64_t c1 = clock64(), t1 = gtimer();
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < ILP; k++) r ^= a[k];
    if (r == 0x12345678u) out[blockIdx.x * blockDim.x + threadIdx.x] = r;
    if (threadIdx.x == 0) {
        clk[blockIdx.x] = c1 - c0;
        ns[blockIdx.x] = t1 - t0;
    }
}

// fp64 chains (Stage A of the plan search runs fp64 closed forms): DFMA / DADD / DMUL
enum F64Op { DFMA = 0, DADD = 1, DMUL = 2 };
template <int OP, int ILP>
__global__ void k_tput_f64(uint32_t iters, uint32_t seed, uint32_t* out, uint64_t* clk, uint64_t* ns) {
    double a[ILP];
#pragma unroll
    for (int k = 0; k < ILP; k++) a[k] = 1.0 + 1e-9 * (threadIdx.x * (k + 1) + seed);
    __syncthreads();
    uint64_t c0 = clock64(), t0 = gtimer();
    for (uint32_t it = 0; it < iters; it++) {
#pragma unroll
        for (int u = 0; u < 8; u++) {
#pragma unroll
            for (int k = 0; k < ILP; k++) {
                const double x = a[(k + 1) % ILP], y = a[(k + 3) % ILP];
                if constexpr (OP == DFMA) asm volatile("fma.rn.f64 %0, %0, %1, %2;" : "+d"(a[k]) : "d"(x), "d"(y));
                else if constexpr (OP == DADD) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(a[k]) : "d"(x));
                else asm volatile("mul.rn.f64 %0, %0, %1;" : "+d"(a[k]) : "d"(x));
            }
        }
    }
    __syncthreads();
    uint64_t c1 = clock64(), t1 = gtimer();
    double r = 0;
#pragma unroll
    for (int k = 0; k < ILP; k++) r += a[k];
    if (r == 1234.5) out[blockIdx.x * blockDim.x + threadIdx.x] = 1;
    if (threadIdx.x == 0) {
        clk[blockIdx.x] = c1 - c0;
        ns[blockIdx.x] = t1 - t0;
    }
}

struct Res { double lane_ops_per_clk_sm, warp_inst_per_clk_smsp, mhz, tops, ms; };

template <int OP, int ILP>
static int run(int sms, int blocks_per_sm, int threads, uint32_t iters, uint32_t* out, uint64_t* dclk, uint64_t* dns, Res* res) {
    int grid = sms * blocks_per_sm;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (int w = 0; w < 2; w++) k_tput<OP, ILP><<<grid, threads>>>(iters / 8, 7u, out, dclk, dns);
    CK(cudaEventRecord(e0));
    k_tput<OP, ILP><<<grid, threads>>>(iters, 7u, out, dclk, dns);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<uint64_t> hc(grid), hn(grid);
    CK(cudaMemcpy(hc.data(), dclk, grid * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hn.data(), dns, grid * 8, cudaMemcpyDeviceToHost));
    // per-CTA clock rate and cycles; the CTAs of one launch are co-resident (grid = SMs x 2)
    std::vector<double> mhz(grid), cyc(grid);
    for (int i = 0; i < grid; i++) {
        mhz[i] = hn[i] ? (double)hc[i] / (double)hn[i] * 1e3 : 0;
        cyc[i] = (double)hc[i];
    }
    std::sort(mhz.begin(), mhz.end());
    double cyc_max = *std::max_element(cyc.begin(), cyc.end());
    double lane_ops_per_sm = (double)iters * 8.0 * ILP * threads * blocks_per_sm;  // per SM
    res->lane_ops_per_clk_sm = lane_ops_per_sm / cyc_max;
    res->warp_inst_per_clk_smsp = res->lane_ops_per_clk_sm / 32.0 / 4.0;
    res->mhz = mhz[grid / 2];
    res->ms = ms;
    res->tops = (double)iters * 8.0 * ILP * threads * grid / (ms * 1e-3) / 1e12;
    return 0;
}

template <int OP>
static int run_lat(uint32_t iters, uint32_t* out, uint64_t* dclk, uint64_t* dns, double* lat) {
    k_tput<OP, 1><<<1, 32>>>(iters / 8, 7u, out, dclk, dns);
    k_tput<OP, 1><<<1, 32>>>(iters, 7u, out, dclk, dns);
    CK(cudaDeviceSynchronize());
    uint64_t hc = 0;
    CK(cudaMemcpy(&hc, dclk, 8, cudaMemcpyDeviceToHost));
    *lat = (double)hc / ((double)iters * 8.0);
    return 0;
}

template <int OP>
static int one_f64(const char* name, int sms, uint32_t* out, uint64_t* dclk, uint64_t* dns) {
    const int blocks = 2, threads = 1024, grid = sms * blocks;
    const uint32_t iters = 4000;
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    k_tput_f64<OP, 8><<<grid, threads>>>(iters / 8, 7u, out, dclk, dns);
    CK(cudaEventRecord(e0));
    k_tput_f64<OP, 8><<<grid, threads>>>(iters, 7u, out, dclk, dns);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<uint64_t> hc(grid), hn(grid);
    CK(cudaMemcpy(hc.data(), dclk, grid * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(hn.data(), dns, grid * 8, cudaMemcpyDeviceToHost));
    double cyc = 0;
    std::vector<double> mhz(grid);
    for (int i = 0; i < grid; i++) {
        cyc = std::max(cyc, (double)hc[i]);
        mhz[i] = hn[i] ? (double)hc[i] / (double)hn[i] * 1e3 : 0;
    }
    std::sort(mhz.begin(), mhz.end());
    const double per_sm = (double)iters * 8.0 * 8 * threads * blocks;
    printf("  \"%s\": {\"lane_ops_per_clk_per_sm\": %.2f, \"warp_inst_per_clk_per_smsp\": %.3f, "
           "\"sm_mhz_in_kernel\": %.0f, \"lane_ops_per_s\": %.4e, \"ms\": %.3f},\n",
           name, per_sm / cyc, per_sm / cyc / 128.0, mhz[grid / 2], (double)iters * 8.0 * 8 * threads * grid / (ms * 1e-3), ms);
    return 0;
}

template <int OP>
static int one(const char* name, int sms, uint32_t* out, uint64_t* dclk, uint64_t* dns, bool last) {
    Res r;
    double lat = 0;
    const uint32_t iters = (OP == SHFL || OP == REDUXMIN) ? 20000 : 40000;
    if (run<OP, 8>(sms, 2, 1024, iters, out, dclk, dns, &r)) return 1;
    // dependent-chain latency only where one PTX step is one SASS instruction at ILP 1 (min and
    // add chains against loop-invariant operands fold or hoist; those print null)
    const bool lat_ok = OP == SHFL || OP == REDUXMIN || OP == IADDMIN || OP == IMAD || OP == LOP;
    if (lat_ok && run_lat<OP>(20000, out, dclk, dns, &lat)) return 1;
    char lbuf[32];
    if (lat_ok) snprintf(lbuf, sizeof lbuf, "%.2f", lat); else snprintf(lbuf, sizeof lbuf, "null");
    printf("  \"%s\": {\"lane_ops_per_clk_per_sm\": %.2f, \"warp_inst_per_clk_per_smsp\": %.3f, "
           "\"dependent_latency_cycles\": %s, \"sm_mhz_in_kernel\": %.0f, \"lane_ops_per_s\": %.4e, \"ms\": %.3f}%s\n",
           name, r.lane_ops_per_clk_sm, r.warp_inst_per_clk_smsp, lbuf, r.mhz, r.tops * 1e12, r.ms, last ? "" : ",");
    return 0;
}

int main() {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, 0));
    int sms = prop.multiProcessorCount;
    uint32_t* out;
    uint64_t *dclk, *dns;
    CK(cudaMalloc(&out, (size_t)sms * 2 * 1024 * 4));
    CK(cudaMalloc(&dclk, (size_t)sms * 2 * 8));
    CK(cudaMalloc(&dns, (size_t)sms * 2 * 8));
    printf("{\n  \"gpu\": \"%s\", \"sms\": %d, \"cc\": \"%d.%d\",\n", prop.name, sms, prop.major, prop.minor);
    printf("  \"how\": \"tools/int_peaks.cu: 148 SMs x 2 CTAs x 1024 threads, 8 independent chains per thread, inline-PTX bodies; cycles by clock64 per CTA (max over CTAs), clock by clock64/globaltimer; latency = one warp, one dependent chain\",\n");
    if (one_f64<DFMA>("dfma_f64", sms, out, dclk, dns)) return 1;
    if (one_f64<DADD>("dadd_f64", sms, out, dclk, dns)) return 1;
    if (one_f64<DMUL>("dmul_f64", sms, out, dclk, dns)) return 1;
    if (one<IADD>(kNames[IADD], sms, out, dclk, dns, false)) return 1;
    if (one<IMIN>(kNames[IMIN], sms, out, dclk, dns, false)) return 1;
    if (one<IADDMIN>(kNames[IADDMIN], sms, out, dclk, dns, false)) return 1;
    if (one<IMAD>(kNames[IMAD], sms, out, dclk, dns, false)) return 1;
    if (one<LOP>(kNames[LOP], sms, out, dclk, dns, false)) return 1;
    if (one<SHFL>(kNames[SHFL], sms, out, dclk, dns, false)) return 1;
    if (one<MIX_ADD_MAD>(kNames[MIX_ADD_MAD], sms, out, dclk, dns, false)) return 1;
    if (one<ADD2>(kNames[ADD2], sms, out, dclk, dns, false)) return 1;
    if (one<REDUXMIN>(kNames[REDUXMIN], sms, out, dclk, dns, true)) return 1;
    printf("}\n");
    return 0;
}
