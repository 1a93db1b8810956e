// slots.cpp -- the 1F1B "slot program": a topological order of the non-interleaved 1F1B
// DAG (Fig. 1; R9) that the kernels evaluate sequentially, plus the ring depth D
// that bounds how many produced-but-unconsumed end times a stage must keep.
//
// Construction: Kahn's algorithm computes each op's level (longest chain of ops before
// it); ops are ordered by (level, stage); the level offsets let the lanes of a candidate
// group evaluate one level in parallel (the ops of a level are on distinct stages).  Any topological order gives the same longest
// path; this one keeps producer/consumer distances short, so the rings stay shallow.
// Cached per (device, S, M) in library-owned device memory.
#include <cuda_runtime.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <tuple>
#include <vector>

#include "internal.h"

namespace dflop {

namespace {
struct Entry {
    SlotProgram prog;
    uint32_t* d_ops = nullptr;
};
std::mutex g_mu;
std::map<std::tuple<int, uint32_t, uint32_t>, Entry> g_cache;

inline uint32_t enc(uint32_t kind, uint32_t s, uint32_t k) { return (kind << 31) | (s << 16) | k; }
}  // namespace

static void build_program(uint32_t S, uint32_t M, std::vector<uint32_t>& out, std::vector<uint32_t>& levels,
                          std::vector<uint32_t>& dense, uint32_t& D) {
    // per-stage op sequences; node id = s * 2M + t
    const uint32_t L_ = 2 * M, L = L_;
    std::vector<uint32_t> kind(S * L), mb(S * L);
    std::vector<uint32_t> posF(S * M), posB(S * M);
    for (uint32_t s = 0; s < S; ++s) {
        const uint32_t w = std::min(S - 1 - s, M);
        uint32_t t = 0;
        auto put = [&](uint32_t kd, uint32_t k) {
            kind[s * L + t] = kd;
            mb[s * L + t] = k;
            (kd ? posB : posF)[s * M + k] = t;
            ++t;
        };
        for (uint32_t k = 0; k < w; ++k) put(0, k);
        for (uint32_t q = 0; q < M - w; ++q) {
            put(0, w + q);
            put(1, q);
        }
        for (uint32_t k = M - w; k < M; ++k) put(1, k);
    }
    // successors and in-degrees
    const uint32_t N = S * L;
    std::vector<uint32_t> indeg(N, 0), level(N, 0);
    auto succ = [&](uint32_t v, uint32_t* out2) -> int {
        int c = 0;
        const uint32_t s = v / L, t = v % L, kd = kind[v], k = mb[v];
        if (t + 1 < L) out2[c++] = v + 1;
        if (kd == 0 && s + 1 < S) out2[c++] = (s + 1) * L + posF[(s + 1) * M + k];
        if (kd == 1 && s > 0) out2[c++] = (s - 1) * L + posB[(s - 1) * M + k];
        return c;
    };
    uint32_t tmp[3];
    for (uint32_t v = 0; v < N; ++v) {
        int c = succ(v, tmp);
        for (int i = 0; i < c; ++i) indeg[tmp[i]]++;
    }
    std::vector<uint32_t> queue;
    queue.reserve(N);
    for (uint32_t v = 0; v < N; ++v)
        if (indeg[v] == 0) queue.push_back(v);
    for (size_t h = 0; h < queue.size(); ++h) {
        const uint32_t v = queue[h];
        int c = succ(v, tmp);
        for (int i = 0; i < c; ++i) {
            const uint32_t w2 = tmp[i];
            level[w2] = std::max(level[w2], level[v] + 1);
            if (--indeg[w2] == 0) queue.push_back(w2);
        }
    }
    std::vector<uint32_t> ord(N);
    for (uint32_t v = 0; v < N; ++v) ord[v] = v;
    std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) {
        if (level[a] != level[b]) return level[a] < level[b];
        return a / L < b / L;
    });
    out.resize(N);
    // level offsets: ops of one level are on distinct stages and may run concurrently
    levels.clear();
    for (uint32_t q = 0; q < N; ++q)
        if (q == 0 || level[ord[q]] != level[ord[q - 1]]) levels.push_back(q);
    levels.push_back(N);
    // ring depth: FIFO distance between production and consumption per edge type.  The ops
    // of a level run concurrently, so a level's productions are checked against the
    // consumption state before the level and its consumptions take effect after it.
    std::vector<uint32_t> consF(S, 0), consB(S, 0);
    uint32_t need = 1;
    for (size_t L = 0; L + 1 < levels.size(); ++L) {
        for (uint32_t q = levels[L]; q < levels[L + 1]; ++q) {
            const uint32_t v = ord[q], s = v / L_, kd = kind[v], k = mb[v];
            out[q] = enc(kd, s, k);
            if (kd == 0)
                need = std::max(need, k - consF[s] + 1);                 // produces F(s, k)
            else if (s > 0)
                need = std::max(need, k - consB[s] + 1);                 // produces B(s, k); B(0, k) unread
        }
        for (uint32_t q = levels[L]; q < levels[L + 1]; ++q) {
            const uint32_t v = ord[q], s = v / L_, kd = kind[v], k = mb[v];
            if (kd == 0) {
                if (s > 0) consF[s - 1] = k + 1;                         // consumes F(s-1, k)
            } else {
                if (s + 1 < S) consB[s + 1] = k + 1;                     // consumes B(s+1, k)
                else consF[s] = k + 1;                                   // last stage: its F(k)
            }
        }
    }
    D = 1;
    while (D < need) D <<= 1;
    // the same order, level-dense: dense[L * S + s] = stage s's op at level L (kNoOp if idle),
    // so a lane that owns stage s reads its op at a fixed stride (the candidate kernel's scorer)
    const size_t nl = levels.size() - 1;
    dense.assign(nl * S, kNoOp);
    for (size_t L = 0; L < nl; ++L)
        for (uint32_t q = levels[L]; q < levels[L + 1]; ++q) dense[L * S + ((out[q] >> 16) & 31u)] = out[q];
}

dflop_status get_slot_program(uint32_t S, uint32_t M, SlotProgram* out) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(g_mu);
    auto key = std::make_tuple(dev, S, M);
    auto it = g_cache.find(key);
    if (it != g_cache.end()) {
        *out = it->second.prog;
        return DFLOP_OK;
    }
    std::vector<uint32_t> ops, levels, dense;
    uint32_t D = 1;
    build_program(S, M, ops, levels, dense, D);
    if (D > 16) {
        set_error("1F1B ring depth %u > 16 for S=%u M=%u", D, S, M);
        return DFLOP_ERR_UNSUPPORTED;
    }
    Entry e;
    std::vector<uint32_t> all(ops);
    all.insert(all.end(), levels.begin(), levels.end());
    all.insert(all.end(), dense.begin(), dense.end());
    cudaError_t ce = cudaMalloc(&e.d_ops, all.size() * sizeof(uint32_t));
    if (ce != cudaSuccess) return cuda_status(ce, "slot program alloc");
    ce = cudaMemcpy(e.d_ops, all.data(), all.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) return cuda_status(ce, "slot program copy");
    e.prog.S = S;
    e.prog.M = M;
    e.prog.D = D;
    e.prog.d_ops = e.d_ops;
    e.prog.n_ops = (uint32_t)ops.size();
    e.prog.n_levels = (uint32_t)levels.size() - 1;
    e.prog.d_levels = e.d_ops + ops.size();
    e.prog.d_dense = e.prog.d_levels + levels.size();
    g_cache[key] = e;
    *out = e.prog;
    return DFLOP_OK;
}

void release_slot_programs() {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& kv : g_cache) cudaFree(kv.second.d_ops);
    g_cache.clear();
}

}  // namespace dflop
