// internal.h — handle state and kernel launchers (C++; never crosses the C ABI).
#pragma once
#include <cstdlib>
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "../../include/kmeans.h"

namespace mpk {

// Number of kernels this library launched (process-wide); reported per fit in kmeans_stats.
long long launches_read();
void launches_add(int n);
// Launch with programmatic stream serialization (PDL): the kernel's launch overlaps the tail of
// the previous kernel in the stream; the kernel must call griddep_wait() before touching data the
// previous kernels wrote (every kernel launched this way does so first). MPK_NO_PDL: plain launch.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
    static const bool off = getenv("MPK_NO_PDL") != nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = off ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Packed per-iteration accumulator (fp64): [sums k*d][counts k][sse][changed][nonfinite][pad]
// One ncclAllReduce over this buffer is the only per-iteration cross-GPU exchange.
#ifdef __CUDACC__
#define MPK_HD __host__ __device__ __forceinline__
#else
#define MPK_HD inline
#endif
struct AccLayout {
    int64_t k, d;
    MPK_HD int64_t sums() const { return 0; }
    MPK_HD int64_t counts() const { return k * d; }
    MPK_HD int64_t sse() const { return k * d + k; }
    MPK_HD int64_t changed() const { return k * d + k + 1; }
    MPK_HD int64_t nonfinite() const { return k * d + k + 2; }
    MPK_HD int64_t total() const { return k * d + k + 4; }
};

// Per-iteration trace record (device), one per iteration: sse, shift2, changed, empty.
struct IterRec {
    double sse;
    double shift2;
    double changed;
    double empty;
    // Thm 5.3 (eq:center-update-prec): max over clusters that moved of
    // 2 |c^ - mu^|^T |mu^| / |c^ - mu^|^T |c^ - mu^|; the bound on the update's unit roundoff
    // is its reciprocal (0 = no cluster moved: no constraint)
    double ub_inv;
};

// Device-side problem description passed to kernels by value.
struct Problem {
    int64_t n;      // rows in this launch
    int d;          // features
    int k;          // clusters
    int d_pad;      // row stride (elements) of the low-precision operand arrays
    int guard;      // Alg 4 scaling on
};

enum DistKernel { DK_SIMT_WORK = 0, DK_SIMT_LOW = 1, DK_TCGEN05 = 2, DK_SMALLD = 3 };

// ------------------------------------------------------------------------------------------
// Launchers (each returns cudaError_t of the launch).
// ------------------------------------------------------------------------------------------

// K2: per-feature statistics of X (fp64, compensated partials combined in block order).
//   ZSCORE: a = sum_i x_ic; then launch_norm_ssq: ssq = sum_i (x_ic - mean_c)^2.
//   MINMAX: a = min, b = max. Multi-GPU: the aggregates are allreduced before launch_norm_post.
//   launch_norm_post mode 0: shift = a / n; 1: scale = sqrt(ssq / n) (0 -> 1);
//   2: scale = max - min (0 -> 1). launch_norm_apply: x = round_u((x - shift) / scale).
cudaError_t launch_norm_stats(int work, int norm, const void* X, int64_t n, int d,
                              double* partials, int nblocks, double* a, double* b,
                              cudaStream_t s);
cudaError_t launch_norm_ssq(int work, const void* X, int64_t n, int d, double* partials,
                            int nblocks, const double* mean, double* ssq, cudaStream_t s);
// One-pass z-score (fp32, d % 4 == 0, one rank): moments about row 0, then shift and scale.
bool norm_moments_ok(int work, const void* X, int d);
cudaError_t launch_norm_moments(const void* X, int64_t n, int d, double* part1, double* part2,
                                int nblocks, double* kbuf, double* shift, double* scale,
                                double n_total, cudaStream_t s);
cudaError_t launch_norm_post(int mode, int d, double n_total, double* shift, double* scale,
                             cudaStream_t s);
cudaError_t launch_norm_apply(int work, void* X, int64_t rows, int d, const double* shift,
                              const double* scale, cudaStream_t s, const void* Xin = nullptr);
int norm_stats_blocks(int64_t n, int d);

// K1 / K3: norms (fp64 -> work), guard scales, low-precision operands with padding, census.
// K1 fast path (fp32 work, d <= 256, see prep_fast_ok): the same outputs as launch_prep; with
// shift != nullptr also the normalisation of the rows read from Xin, written to Xout (one read
// of X for normalise + prep).
bool prep_fast_ok(int work, int d);
cudaError_t launch_prep_fast(int dist, const void* Xin, int64_t rows, int d, int d_pad, int guard,
                             void* norms, void* scales, void* Xl, unsigned long long* census,
                             void* Xout, const double* shift, const double* scale,
                             cudaStream_t s, unsigned* amax = nullptr, int* flags = nullptr,
                             bool* amax_done = nullptr);
cudaError_t launch_prep(int work, int dist, const void* Xw, int64_t rows, int d, int d_pad,
                        int guard, void* norms, void* scales, void* Xl,
                        unsigned long long* census /* [nonfinite, underflow] */, cudaStream_t s);

// kmeans_cast kernel.
cudaError_t launch_cast(int src, int dst, const void* in, int64_t count, void* out,
                        cudaStream_t s);

// K6: SIMT distance + argmin (any precision). Writes labels; if labels_prev path: counts
// changed labels into acc[changed], adds sum_i max(0, xn_i + min_j v_ij) into acc[sse].
// final_mode: operands are the working-precision X/C (Alg 3 step 7) and sse_direct gets the
// direct-formula SSE sum_i ||x_i - c_{l_i}||^2 (eq:dist-eval-alternative).
cudaError_t launch_assign_simt(int work, int dist, const Problem& p, const void* Xl,
                               const void* xn, const void* sx, const void* Cl, const void* cn,
                               const void* sc, int32_t* labels, double* acc_sse,
                               double* acc_changed, cudaStream_t s,
                               const int* row_list = nullptr);
cudaError_t launch_final_sse(int work, const void* Xw, int64_t n, int d, const void* Cw,
                             const int32_t* labels, double* sse_out, cudaStream_t s);

// K5: small-d fused assign + update (d <= 4, k <= 8).
bool smalld_supported(int d, int k);
cudaError_t launch_smalld_fused(int work, int dist, const Problem& p, const void* Xw,
                                const void* Cl, const void* cn, const void* sc, int32_t* labels,
                                double* acc, AccLayout L, cudaStream_t s);

// K5g: one whole Lloyd iteration of the small-d path on one rank in ONE launch (k_smalld_loop.cu):
// centroid prep, distance + argmin, deterministic block partials of the update, and the last
// block's finalize + trace record + stopping rule. A launch after the stop flag is set returns
// at once, so the host enqueues chunks of iterations (a CUDA graph) and polls once per chunk.
struct LoopState {
    int iter;          // iterations completed
    int stop;          // set when converged: later launches are no-ops
    int converged;
    unsigned counter;  // K5g: block ticket of the launch (reset by the last block); K5p: block
                       // arrivals so far (the grid barrier of iteration t waits for grid (t + 1))
    double tol;        // < 0: never stop early
    int fault;         // K5p: a block gave up waiting at the grid barrier
};
bool smalld_loop_supported(int d, int k);
size_t smalld_loop_part_bytes(int64_t n);
cudaError_t launch_smalld_iter(int work, int dist, const Problem& p, const void* Xw, void* Cw,
                               int32_t* labels, double* part, LoopState* st, IterRec* trace,
                               unsigned long long* census, cudaStream_t s);   // Xw == nullptr: only set the kernel's
                                                      // shared-memory attribute (per device)
// K5p: the same iteration, all max_iter of them in ONE cooperative launch (every block resident,
// its rows kept in shared memory across iterations; one grid barrier per iteration, after which
// every block reduces the partials in the same fixed order and forms the same centres).
// cudaErrorNotSupported when the rows do not fit in shared memory or the grid cannot be
// co-resident (the caller then uses K5g).
cudaError_t launch_smalld_persist(int work, int dist, const Problem& p, const void* Xw, void* Cw,
                                  int32_t* labels, double* part, LoopState* st, IterRec* trace,
                                  unsigned long long* census, int max_iter, cudaStream_t s);

// K6m: Alg 4's per-pair precision switch with threshold delta (>= 1); n_low (device) gets the
// number of triggered (low-precision) pairs added.
cudaError_t launch_assign_mixed(int work, int dist, const Problem& p, double delta, const void* Xl,
                                const void* Xw, const void* xn, const void* sx, const void* Cl,
                                const void* Cw, const void* cn, const void* sc, int32_t* labels,
                                double* acc_sse, double* acc_changed, unsigned long long* n_low,
                                cudaStream_t s);

// K11: D^2 seeding rounds (Alg 1 in the low precision, R6): idx[0] set by the
// caller; fills idx[1..k-1]; D2 (n) and ps (seed_blocks(n)) are scratch; *warn |= 1 on a
// degenerate round (uniform fallback).
int64_t seed_blocks(int64_t n);
cudaError_t launch_seed_d2(int work, int dist, const void* Xl, int64_t n, int d, int d_pad,
                           const void* xn, const void* sx, int guard, int k, const double* u,
                           int64_t* idx, double* D2, double* ps, int* warn, cudaStream_t s);

// K4: tcgen05 distance + argmin (fp16 / bf16 / e5m2 operands).
bool tc_supported(int dist, int d_pad, int k);
int tc_dpad(int dist, int d);   // padded row length (elements) the tcgen05 kernel needs
struct TcPlan;                  // opaque (TMA descriptors etc.)
TcPlan* tc_plan_create(int dist, int64_t n, int d, int d_pad, int k, const void* Xl,
                       const void* Cl, std::string* err);
void tc_plan_destroy(TcPlan*);
// fx (optional; the Lloyd loop with the fixed-point update): the CTA-pair kernel lists the
// changed rows itself (FxState::list / seg_cnt, gate[0]) so the update skips fx_diff_kernel;
// *fx_listed tells whether it did
struct FxState;
cudaError_t launch_assign_tc(TcPlan* plan, const Problem& p, const float* xn, const float* sx,
                             const float* cn, const float* sc, int32_t* labels, double* acc_sse,
                             double* acc_changed, cudaStream_t s, FxState* fx = nullptr,
                             bool* fx_listed = nullptr);
// Final pass (Alg 3 step 7) as a certified tensor-core filter: rows whose top-2 gap exceeds the
// error bound get the filter's argmin (= the working-precision argmin); the others are appended
// to fb_rows (count in *fb_count) for launch_assign_simt(row_list = fb_rows).
// fb_thr (optional): per fallback slot, the candidate threshold T = v^(1) + 2 (E + B32) (NaN
// when the row's values are not finite).
cudaError_t launch_final_tc(TcPlan* plan, const Problem& p, const float* xn, const float* sx,
                            const float* cn, const float* sc, int32_t* labels, int* fb_count,
                            int* fb_rows, float* fb_thr, cudaStream_t s);
// Candidate stage of the final pass (CTA-pair plans only): for nc gathered operand rows Xc (same
// layout as the plan's rows) with thresholds thr, append every column j with v^_j <= thr[r] to
// cand[r * cand_q ...] (count in cand_cnt[r], which may exceed cand_q: overflow).
bool tc_plan_has_cand(const TcPlan* plan);
int tc_plan_kind(const TcPlan* plan);   // 1 = streaming, 2 = CTA pair
const void* tc_plan_operands(const TcPlan* plan, int* row_bytes);
cudaError_t launch_cand_tc(TcPlan* plan, const void* Xc, int64_t nc, int guard, const float* sxc,
                           const float* cn, const float* sc, const float* thr, int* cand_cnt,
                           int* cand, int cand_q, cudaStream_t s);
// Gather rows[0..nr) of a row-major byte matrix (row_bytes, multiple of 16) and, optionally,
// of a float vector.
cudaError_t launch_gather_rows(const void* src, int row_bytes, const int* rows, int nr, void* dst,
                               const float* vsrc, float* vdst, cudaStream_t s);
// Exact stage: for gathered row r (original index rows[r]) evaluate the working-precision (fp32)
// distance of each candidate exactly as launch_assign_simt does (dot accumulated t = 0..d-1 by
// FMA, v = fma(-2, dot, ||c_j||^2)) and store the (value, lowest index) argmin in labels[rows[r]];
// rows with no candidates or more than cand_q go to left_rows (count in *left_count).
cudaError_t launch_cand_exact(const float* Xw, const float* Cw, const float* cn, int d,
                              const int* rows, int nr, const int* cand_cnt, const int* cand,
                              int cand_q, int32_t* labels, int* left_count, int* left_rows,
                              unsigned long long* keys, cudaStream_t s);

// Alg 4 / Alg 5 on the tensor cores (k_final.cu; R10): candidate columns of the
// certified filter's uncertified rows evaluated with the per-pair switch exactly as K6m-b; the
// trigger counts per row from the sorted centroid norms; per-row label distance (SSE_t) and the
// changed count; gathers for the rows left to the full CUDA-core evaluation.
cudaError_t launch_cand_exact_mixed(int dist, const void* Xl, const float* Xw, const void* Cl,
                                    const float* Cw, const float* xn, const float* sx,
                                    const float* cn, const float* sc, int d, int d_pad,
                                    double delta2, const int* rows, int nr, const int* cand_cnt,
                                    const int* cand, int cand_q, int32_t* labels, int* left_count,
                                    int* left_rows, unsigned long long* keys, cudaStream_t s);
cudaError_t launch_mixed_count(const float* xn, int64_t n, const float* cn, int k, double delta2,
                               float* sorted_cn, unsigned long long* n_low, cudaStream_t s);
cudaError_t launch_mixed_label_eval(int dist, const void* Xl, const float* Xw, const void* Cl,
                                    const float* Cw, const float* xn, const float* sx,
                                    const float* cn, const float* sc, int64_t n, int d, int d_pad,
                                    double delta2, const int32_t* labels, const int32_t* prev,
                                    double* acc_sse, double* acc_changed, cudaStream_t s);
cudaError_t launch_gather_float_rows(const float* src, int d, const int* rows, int nr, float* dst,
                                     cudaStream_t s);
cudaError_t launch_scatter_labels(const int32_t* src, const int* rows, int nr, int32_t* labels,
                                  cudaStream_t s);

// K7: update = stable bucket sort by label (block counts, scan, scatter) + segmented fp64 sums
// with an ordered reduction of the chunk-boundary partials: bit-reproducible for k <= 12288.
struct UpdateScratch {
    int* cb = nullptr;          // per-(label, 4096-row block) counts / offsets
    double* part = nullptr;     // piece sums of clusters longer than one segsum piece (d each)
    int* mpo = nullptr;         // k + 1 first-slot offsets into part
};
size_t update_scratch_bytes(int64_t n, int d, int k, size_t* cb, size_t* part, size_t* mpo);
cudaError_t launch_update(int work, const void* Xw, int64_t n, int d, int k,
                          const int32_t* labels, int* cnt, int* offs, int* cursor, int* perm,
                          double* acc, AccLayout L, const UpdateScratch& us, cudaStream_t s);

// FX: exact fixed-point cluster totals with incremental updates (k_update.cu, R9).
struct FxState {
    unsigned* amax = nullptr;   // d: max |x_t| (float bits)
    float2* sc = nullptr;       // d: (c1, c2) of the feature's grid (k_update.cu fx_q)
    double* isc = nullptr;      // d: the grid step 2^(e_t - 45)
    long long* Shi = nullptr;   // k*d: sum of i1 (coarse parts)
    long long* Slo = nullptr;   // k*d: sum of i2 (fine parts)
    long long* part = nullptr;  // piece totals of multi-piece clusters (hi d, lo d per slot)
    int32_t* prev = nullptr;    // n: labels of the previous iteration (fx_diff_kernel)
    // changed rows (row, old, new), by 32-row segment: segment s (rows 32 s ..) lists its
    // seg_cnt[s] changed rows at list[32 s ..]; gate[0] counts them all
    int3* list = nullptr;
    int* seg_cnt = nullptr;
    long long* gShi = nullptr;  // several ranks: the allreduced totals and counts
    long long* gSlo = nullptr;
    int* gcnt = nullptr;
    int* gate = nullptr;        // [0] changed rows, [1] capacity, [2] non-finite X flag
    int cap = 0;
};
cudaError_t launch_fx_colmax(const float* Xw, int64_t n, int d, FxState& fx, bool have_amax,
                             cudaStream_t s);
cudaError_t launch_fx_scale(int d, FxState& fx, cudaStream_t s);
// listed: the distance kernel has produced the changed-row list and gate[0] (see
// launch_assign_tc); else fx_diff_kernel finds them from prev
cudaError_t launch_update_fx(const float* Xw, int64_t n, int d, int k, const int32_t* labels,
                             int* cnt, int* offs, int* cursor, int* perm, const UpdateScratch& us,
                             FxState& fx, cudaStream_t s, bool listed = false);
cudaError_t launch_finalize_fx(int64_t k, int d, const FxState& fx, const long long* Shi,
                               const long long* Slo, const int* cnt, const double* acc,
                               AccLayout L, float* Cw, IterRec* rec, cudaStream_t s);
size_t fx_part_bytes(int64_t n, int d);

// A6 transport (coll.cu): allreduce over the ranks of a point-sharded fit. NCCL (one process
// per GPU) or virtual ranks (several handles of one process on one GPU, kmeans_vgroup_*).
enum CollType { CT_F64 = 0, CT_I64 = 1, CT_I32 = 2, CT_U32 = 3 };
enum CollOp { CO_SUM = 0, CO_MAX = 1, CO_MIN = 2 };
struct Coll {
    int nranks = 1, rank = 0;
    bool virtual_ranks = false;
    virtual ~Coll() {}
    // in-place allowed (send == recv); returns 0 or a KMEANS_E* code with *err set
    virtual int allreduce(const void* send, void* recv, size_t count, int type, int op,
                          cudaStream_t s, std::string* err) = 0;
    virtual void group_start() {}
    virtual int group_end(std::string*) { return 0; }
    // the stream every handle of the group must run on (virtual ranks share one), or null
    virtual cudaStream_t shared_stream() { return nullptr; }
};
struct VGroup;
Coll* coll_create_nccl(const void* nccl_id, int nranks, int rank, std::string* err);
Coll* coll_create_virtual(VGroup* g, int rank, std::string* err);
VGroup* vgroup_create(int nranks, std::string* err);
int vgroup_destroy(VGroup* g);   // KMEANS_EINVAL while handles of the group are alive
int vgroup_size(const VGroup* g);

// cudaFuncSetAttribute is per device: remember per (call site, device) that it was done.
struct PerDeviceOnce {
    unsigned long long mask = 0;   // benign race: a duplicate call is idempotent
    bool need() {
        int dev = 0;
        cudaGetDevice(&dev);
        return dev >= 64 || !((__atomic_load_n(&mask, __ATOMIC_RELAXED) >> dev) & 1ull);
    }
    void done() {
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 64) __atomic_fetch_or(&mask, 1ull << dev, __ATOMIC_RELAXED);
    }
};

// K8: finalize: C = round_u(sum / count) (empty -> keep), shift^2, empty count, trace record.
cudaError_t launch_finalize(int work, int64_t k, int d, const double* acc, AccLayout L,
                            void* Cw, IterRec* rec, cudaStream_t s);

}  // namespace mpk
