// cand.cuh -- parameters of the candidate kernel (a3/a4) shared by its launcher and kernels.
#pragma once
#include "common.cuh"

namespace dflop {

// Kernel variants (chosen on device by k_build_items, each launch exits unless it matches):
//   0  packed 32-bit: bucket loads stored as (E << s | j, L << s | j), s = bits of m - 1, so
//      one probe is max(E' + e', L' + l') and the argmin is a plain min (no index compare)
//   1  plain 32-bit sums
//   2  64-bit sums
constexpr int kVariants = 3;
// block size cap of the candidate kernel: leaves ~100 registers per thread (64 K per SM);
// the 1024-thread bound capped the kernel at 64 registers and cost ~10%
#ifndef DFLOP_CAND_MAX_THREADS
#define DFLOP_CAND_MAX_THREADS 640
#endif
constexpr int kCandMaxThreads = DFLOP_CAND_MAX_THREADS;
// the split pipeline's candidate kernel (no LPT code; fewer registers)
#ifndef DFLOP_SPLIT_MAX_THREADS
#define DFLOP_SPLIT_MAX_THREADS 768
#endif
constexpr int kSplitMaxThreads = DFLOP_SPLIT_MAX_THREADS;

// Per-launch parameters.  Shared-memory layout (bytes):
//   [0, tbl_bytes)              CTA item table: ItemRec<A>[n] then u16 pos->item[n]
//   tbl_bytes + g*cand_bytes    candidate group g: EL[m] {E, L}, FL[m] {EF, LF}, scratch
// Global: per resident group ("slot") two assignment buffers of apos_bytes (u8 per base-order
// position when m <= 255, else u16), the best one named by slot_buf[slot], and the CSR
// member lists of the refinement (csr_len u16 positions).
struct CandParams {
    const void* items;           // ItemRec<A>[n], base-order positions (global)
    const uint32_t* pos_item;    // [n] position -> item index (global)
    const uint32_t* item_pos;    // [n] item index -> position (global)
    const uint32_t* ops;         // 1F1B slot program, n_ops entries
    const uint32_t* levels;      // n_levels + 1 offsets into ops
    const uint32_t* dense;       // [n_levels][S] stage-indexed ops (0xFFFFFFFF: idle)
    BalanceHeader* hdr;
    uint8_t* slot_apos;          // [n_slots][2][apos_bytes]
    uint16_t* slot_csr;          // [n_slots][csr_len] refinement member lists (positions, CSR)
    u64* slot_key;
    u64* slot_T;
    u64* slot_cmax;
    uint32_t* slot_buf;
    u64* cand_T;                 // optional per-candidate outputs
    u64* cand_cmax;
    uint32_t n, m, S, e_pp, l_dp, n_mb, R, G, D, n_ops, n_levels;
    uint32_t c_begin, c_end, id_base, seed0, seed1;
    uint32_t exhaustive, wide, cap, sigma, csr_len, apos_bytes, want_variant;
    uint32_t cnt_smem;           // refinement list counters in shared memory (else global)
    uint32_t order4;             // DFLOP_MODE_ORDER4: best of four slot orders per replica
    uint32_t tbl_bytes, cand_bytes, off_fl, off_scr;
    unsigned long long* phase;   // diagnostic phase counters (timing builds), else null
    // split pipeline (packed variant): k_lpt runs the LPT of the candidates [c_begin, c_end)
    // and leaves, per candidate c, its assignment at lpt_apos + (c - c_begin) * apos_bytes and
    // its bucket loads (E, L packed keys, m x 2 u32) at lpt_el + (c - c_begin) * 2m; entry
    // c_end - c_begin is a scratch entry for the tail groups; the candidate kernel's MODE = 1
    // instantiation starts every candidate from there
    uint8_t* lpt_apos;
    uint32_t* lpt_el;
};

struct CandLaunch {
    int variant;      // see above
    int gl;           // lanes per candidate
    bool tbl_smem;    // item table staged in shared memory
    uint32_t grid, cpb;
    size_t dyn;
};

const void* cand_kernel_ptr(int variant, int gl, bool tbl_smem, bool o4);
void cand_launch(const CandLaunch& L, const CandParams& p, cudaStream_t s);
// the split pipeline's candidate kernel (packed u32, shared-memory table, GL in {8, 16, 32}):
// refinement and 1F1B from k_lpt's output
const void* split_kernel_ptr(int gl, bool o4);
void split_launch(const CandLaunch& L, const CandParams& p, cudaStream_t s);
// the split pipeline's LPT kernel (packed u32 variant, item table in shared memory)
#ifndef DFLOP_LPT_MAX_THREADS
#define DFLOP_LPT_MAX_THREADS 640
#endif
constexpr int kLptMaxThreads = DFLOP_LPT_MAX_THREADS;
const void* lpt_kernel_ptr(int gl);
void lpt_launch(int gl, uint32_t grid, uint32_t cpb, size_t dyn, const CandParams& p, cudaStream_t s);

}  // namespace dflop
