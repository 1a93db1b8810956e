// profile.cpp -- launch counter and CUDA-event timing of the candidate kernels.
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "internal.h"

namespace dflop {

namespace {
std::atomic<uint64_t> g_launches{0};
std::atomic<uint32_t> g_split{0};
std::atomic<bool> g_on{false};
std::mutex g_mu;
struct Mark {
    cudaEvent_t e[4];
};
std::vector<Mark> g_marks;   // recorded, not yet read
std::vector<Mark> g_free;    // reusable events
std::vector<Mark> g_stage;   // Stage-A kernel marks (e[0], e[1])
}  // namespace

void count_launches(uint32_t k) { g_launches.fetch_add(k, std::memory_order_relaxed); }
void count_split_chunks(uint32_t k) { g_split.fetch_add(k, std::memory_order_relaxed); }
bool profiling() { return g_on.load(std::memory_order_relaxed); }

int prof_begin(cudaStream_t s) {
    if (!profiling()) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    Mark m;
    if (!g_free.empty()) {
        m = g_free.back();
        g_free.pop_back();
    } else {
        for (auto& e : m.e) cudaEventCreate(&e);
    }
    cudaEventRecord(m.e[0], s);
    g_marks.push_back(m);
    return (int)g_marks.size() - 1;
}

int prof_stage_begin(cudaStream_t s) {
    if (!profiling()) return -1;
    std::lock_guard<std::mutex> lk(g_mu);
    Mark m;
    if (!g_free.empty()) {
        m = g_free.back();
        g_free.pop_back();
    } else {
        for (auto& e : m.e) cudaEventCreate(&e);
    }
    cudaEventRecord(m.e[0], s);
    g_stage.push_back(m);
    return (int)g_stage.size() - 1;
}

void prof_stage_end(int idx, cudaStream_t s) {
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (idx < (int)g_stage.size()) cudaEventRecord(g_stage[idx].e[1], s);
}

void prof_mark(int idx, int which, cudaStream_t s) {  // which = 1..3
    if (idx < 0) return;
    std::lock_guard<std::mutex> lk(g_mu);
    if (idx < (int)g_marks.size()) cudaEventRecord(g_marks[idx].e[which], s);
}

DevAttr dev_attr(int device) {
    static std::mutex mu;
    static std::vector<DevAttr> cache;
    std::lock_guard<std::mutex> lk(mu);
    if ((int)cache.size() <= device) cache.resize(device + 1, DevAttr{0, 0, 0});
    DevAttr& d = cache[device];
    if (d.sms == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
        d.sms = v;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
        d.smem_optin = (size_t)v;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
        d.smem_per_sm = (size_t)v;
    }
    return d;
}

}  // namespace dflop

using namespace dflop;

extern "C" dflop_status dflop_profile_enable(int on) {
    g_on.store(on != 0);
    return DFLOP_OK;
}

extern "C" dflop_status dflop_profile_read(dflop_profile* out, int reset) {
    if (!out || out->struct_size != sizeof(dflop_profile)) {
        set_error("dflop_profile struct_size");
        return DFLOP_ERR_INVALID_ARGUMENT;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    double ms = 0.0;
    for (auto& m : g_marks) {
        cudaError_t e = cudaEventSynchronize(m.e[3]);
        if (e != cudaSuccess) return cuda_status(e, "profile event");
        float best = 0.f;
        for (int v = 0; v < 3; ++v) {  // the variant that ran (the others exit at once)
            float t = 0.f;
            cudaEventElapsedTime(&t, m.e[v], m.e[v + 1]);
            best = t > best ? t : best;
        }
        ms += best;
    }
    double sms = 0.0;
    for (auto& m : g_stage) {
        cudaError_t e = cudaEventSynchronize(m.e[1]);
        if (e != cudaSuccess) return cuda_status(e, "profile event");
        float t = 0.f;
        cudaEventElapsedTime(&t, m.e[0], m.e[1]);
        sms += t;
    }
    out->cand_launches = (uint32_t)g_marks.size();
    out->kernel_launches = g_launches.load();
    out->cand_ms = ms;
    out->stage_a_launches = (uint32_t)g_stage.size();
    out->split_chunks = g_split.load();
    out->stage_a_ms = sms;
    if (reset) g_split.store(0);
    if (reset) {
        for (auto& m : g_marks) g_free.push_back(m);
        for (auto& m : g_stage) g_free.push_back(m);
        g_marks.clear();
        g_stage.clear();
        g_launches.store(0);
    }
    return DFLOP_OK;
}
