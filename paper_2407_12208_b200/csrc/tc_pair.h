// tc_pair.h — the CTA-pair (cta_group::2), centroid-stationary distance + argmin kernel.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace mpk {
namespace tcdev {

struct PairParams {
    int64_t n;
    int k, k_pad, d, d_pad, NB, NT, KB, SWZ, SA, nacc, tmem_cols;
    int rbr;                 // one tile per row-block: row-blocks per accumulator (1..4)
    // ASSIGN in the Lloyd loop with the fixed-point update (k_update.cu FX): each warp writes
    // the changed rows (row, old, new) of its 32-row segment s to fx_list[32 s ..] and their
    // number to fx_seg_cnt[s]; each warp adds its total to fx_gate[0] once, at the end — what
    // fx_diff_kernel would produce; nullptr: off
    int3* fx_list;
    int* fx_seg_cnt;
    int* fx_gate;
    int box_rows;            // TMA box rows of the centroid map (64 for 256-column tiles)
    uint32_t a_tile_bytes;   // 128 rows x row bytes (this CTA's half of M = 256)
    uint32_t b_half_bytes;   // NB/2 rows x row bytes (this CTA's half of one centroid tile)
    uint32_t kb_a_bytes, kb_b_bytes;
    uint32_t idesc;          // M = 256, N = NB, fp32 accumulate
    int guard, is_f8;
    const float* xn;
    const float* sx;
    const float* cn;
    const float* sc;
    int32_t* labels;
    double* acc_sse;
    double* acc_changed;
    int* fb_count;
    int* fb_rows;
    double u_low, eta_low;
    float* fb_thr;           // FINAL: per fallback slot, the candidate threshold T (NaN: none)
    const float* thr;        // CAND: per row, T
    int* cand_cnt;           // CAND: per row, number of candidates found
    int* cand;               // CAND: [n][cand_q] candidate columns
    int cand_q;
    int dbg;                 // debug (timing only): bit0 skip the fold, bit1 skip MMAs, bit2 fold probe,
                             // bit3 skip the X~ loads, bit4 skip the row-block end work;
                             // bit5 (same results): no row-block alternation (column split);
                             // bit6 (same results): no row-block halves (rbh)
    unsigned long long* trace;   // debug (MPK_PAIR_TRACE): per-tile clock64 stamps of CTA 0
};

// Fill the static part of PairParams and the dynamic smem size for (dist, d_pad, k); false if
// the resident centroid halves plus two X~ slots do not fit in shared memory.
bool pair_plan(int dist, int d, int d_pad, int k, PairParams* p, size_t* smem_bytes);
int pair_box_rows(const PairParams& p);   // TMA box rows for the centroid map (NB / 2)
cudaError_t pair_set_smem(size_t bytes);
// mode: PAIR_ASSIGN (Lloyd step), PAIR_FINAL (certified final pass), PAIR_CAND (candidate
// columns of the final pass's uncertified rows, R2)
enum { PAIR_ASSIGN = 0, PAIR_FINAL = 1, PAIR_CAND = 2 };
cudaError_t pair_launch(const CUtensorMap& tmap_x, const CUtensorMap& tmap_c, const PairParams& p,
                        int mode, size_t smem_bytes, cudaStream_t s);

}  // namespace tcdev
}  // namespace mpk
