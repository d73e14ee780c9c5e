// kmeans_capi.cu — the C ABI (include/kmeans.h): handle lifetime, input staging, the Lloyd
// loop of Alg 3 with C0 given, the final working-precision pass, and the
// optional point-sharded NCCL path. All arithmetic runs in the kernels of k_*.cu.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <string>
#include <vector>

#include "internal.h"

using namespace mpk;

struct kmeans_ctx {
    int64_t n = 0;
    int d = 0, k = 0, work = 0, dist = 0, flags = 0, norm = 0, guard = 0, force_simt = 0;
    int d_pad = 0;                 // row stride of the low operands
    int wsize = 0, lsize = 0;      // element sizes of work / low types
    int device = 0;
    cudaStream_t own_stream = nullptr, stream = nullptr;
    int timing = 0;
    std::string err;

    // device buffers
    void* Xw = nullptr;            // normalised points (work), n x d
    void* Xl = nullptr;            // low operands, n x d_pad (alias Xw when dist == work)
    void* xn = nullptr;            // ||x||^2 (work), n
    void* sx = nullptr;            // guard scales (work), n
    void* Cw = nullptr;            // centroids (work), k x d
    void* Cl = nullptr;            // low centroid operands, k x d_pad
    void* cn = nullptr;            // ||c||^2 (work), k
    void* sc = nullptr;            // guard scales (work), k
    int32_t* labels = nullptr;     // n
    double* acc = nullptr;         // packed accumulator (AccLayout)
    int *cnt = nullptr, *offs = nullptr, *cursor = nullptr, *perm = nullptr;
    UpdateScratch us;
    IterRec* trace = nullptr;      // KMEANS_MAX_TRACE records
    double* shift = nullptr;       // d (fp64)
    double* scale = nullptr;       // d (fp64)
    double* partials = nullptr;    // normalisation partials
    int npartials = 0;
    unsigned long long* census = nullptr;   // [nonfinite, underflow] prep + per-iteration
    double* sse_dev = nullptr;     // final SSE accumulator
    bool have_centroids = false;
    bool xl_alias = false;

    TcPlan* tc = nullptr;
    // final-pass filter (Alg 3 step 7): an fp16 guarded copy when the loop operands cannot
    // serve (E5M2, or overflowed unguarded operands); allocated on first use.
    TcPlan* fin = nullptr;
    void* fin_Xl = nullptr;
    void* fin_Cl = nullptr;
    void* fin_sx = nullptr;
    void* fin_sc = nullptr;
    int fin_dpad = 0;
    bool fin_failed = false;
    int* fbc = nullptr;            // [0] uncertified rows, [1] rows left for the full evaluation
    int64_t last_fallback = 0;     // rows re-evaluated on CUDA cores in the last final pass
    int64_t last_uncertified = 0;  // rows the certified filter left open in the last final pass
    // Alg 4 / Alg 5 per-pair precision switch (kmeans_set_delta): 0 = off
    double delta = 0.0;
    int guard_user = 0;            // the create-time guard flag (delta > 0 forces the scaling)
    unsigned long long* n_low_dev = nullptr;   // triggered low-precision pairs, this fit
    int64_t last_n_low = 0, last_n_dist = 0;
    // final-pass candidate path (grown to the uncertified row count on demand)
    int64_t cand_cap = 0;
    float* fb_thr = nullptr;       // per uncertified row: threshold T (size n)
    void* cand_X = nullptr;        // gathered operand rows
    float* cand_sx = nullptr;
    int* cand_cnt = nullptr;
    int* cand = nullptr;           // [cap][kCandQ]
    int* cand_left = nullptr;      // rows left for the full CUDA-core evaluation
    unsigned long long* cand_key = nullptr;   // per row: min (value, column) key
    int dist_kernel = 0;
    AccLayout L{0, 0};
    // exact fixed-point totals with incremental updates (R9): fp32 work, one rank,
    // k <= 12288, not the fused small-d path; off for a fit whose X holds a non-finite value
    bool fx_ok = false;
    bool fx_amax_done = false;     // this fit's prep computed the column maxima
    FxState fx;

    // Alg 4 / Alg 5 on the tensor cores (assign_mixed_tc): previous labels, sorted centroid
    // norms, and the gathered rows left to the full CUDA-core evaluation (grown on demand)
    int32_t* mix_prev = nullptr;
    float* mix_sorted = nullptr;
    int64_t mix_cap = 0;
    void* mix_Xl = nullptr;
    float* mix_Xw = nullptr;
    float* mix_xn = nullptr;
    float* mix_sx = nullptr;
    int32_t* mix_lab = nullptr;
    // K5g fused small-d iteration (k_smalld_loop.cu): device loop state, block partials, a
    // CUDA graph of kLoopChunk iterations, pinned host copies of the state
    LoopState* loop = nullptr;
    double* loop_part = nullptr;
    LoopState* loop_host = nullptr;      // [0] initial state, [1] polled state
    cudaStream_t loop_capture = nullptr;
    cudaGraphExec_t loop_graph = nullptr;
    int loop_graph_guard = -1;

    // distributed (A6): NCCL or virtual ranks; null on a single-rank handle
    Coll* comm = nullptr;
    int nranks = 1, rank = 0;

    kmeans_stats stats{};
};

namespace mpk {
static std::atomic<long long> g_launches{0};
long long launches_read() { return g_launches.load(); }
void launches_add(int n) { g_launches += n; }
}  // namespace mpk

namespace {

thread_local std::string g_create_err;

int fail(kmeans_ctx* h, int code, const std::string& msg) {
    if (h) h->err = msg; else g_create_err = msg;
    return code;
}

#define CK(call)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (call);                                                          \
        if (_e != cudaSuccess)                                                            \
            return fail(h, KMEANS_ECUDA, std::string(#call) + ": " + cudaGetErrorString(_e)); \
    } while (0)

// A6 collectives through the handle's transport (coll.cu)
#define CKC(call)                                                                         \
    do {                                                                                  \
        std::string _m;                                                                   \
        int _r = (call);                                                                  \
        if (_r != 0) return fail(h, _r, _m);                                              \
    } while (0)
#define AR(send, recv, count, type, op) \
    h->comm->allreduce((send), (recv), (count), (type), (op), h->stream, &_m)

int elem_size(int prec) {
    switch (prec) {
        case KMEANS_FP64: return 8;
        case KMEANS_FP32: return 4;
        case KMEANS_FP16: return 2;
        case KMEANS_BF16: return 2;
        case KMEANS_E5M2: return 1;
    }
    return 0;
}

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

int check_device(kmeans_ctx* h) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) {
        cudaGetLastError();
        return fail(h, KMEANS_ENODEV, "no CUDA device");
    }
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, dev) != cudaSuccess)
        return fail(h, KMEANS_ENODEV, "cudaGetDeviceProperties failed");
    if (prop.major != 10)
        return fail(h, KMEANS_ENODEV,
                    "this library is built for sm_100a (B200); device is sm_" +
                        std::to_string(prop.major) + std::to_string(prop.minor));
    return dev;
}

template <typename T>
cudaError_t dalloc(T** p, size_t bytes) {
    if (bytes == 0) bytes = 16;
    return cudaMalloc((void**)p, bytes);
}

void free_all(kmeans_ctx* h) {
    if (h->tc) tc_plan_destroy(h->tc);
    if (h->fin) tc_plan_destroy(h->fin);
    void* fin_bufs[] = {h->fin_Xl, h->fin_Cl, h->fin_sx, h->fin_sc, h->fbc, h->fb_thr,
                        h->cand_X, h->cand_sx, h->cand_cnt, h->cand, h->cand_left, h->cand_key,
                        h->n_low_dev};
    for (void* b : fin_bufs)
        if (b) cudaFree(b);
    void* bufs[] = {h->Xw, h->xl_alias ? nullptr : h->Xl, h->xn, h->sx, h->Cw, h->Cl, h->cn,
                    h->sc, h->labels, h->acc, h->cnt, h->offs, h->cursor, h->perm, h->trace,
                    h->shift, h->scale, h->partials, h->census, h->sse_dev, h->us.cb,
                    h->us.part, h->us.mpo, h->fx.amax, h->fx.sc, h->fx.isc, h->fx.Shi,
                    h->fx.Slo, h->fx.part, h->fx.prev, h->fx.list, h->fx.seg_cnt, h->fx.gate, h->fx.gShi,
                    h->fx.gSlo, h->fx.gcnt};
    for (void* b : bufs)
        if (b) cudaFree(b);
    void* mix_bufs[] = {h->mix_prev, h->mix_sorted, h->mix_Xl, h->mix_Xw, h->mix_xn, h->mix_sx,
                        h->mix_lab};
    for (void* b : mix_bufs)
        if (b) cudaFree(b);
    if (h->loop) cudaFree(h->loop);
    if (h->loop_part) cudaFree(h->loop_part);
    if (h->loop_host) cudaFreeHost(h->loop_host);
    if (h->loop_graph) cudaGraphExecDestroy(h->loop_graph);
    if (h->loop_capture) cudaStreamDestroy(h->loop_capture);
    if (h->own_stream) cudaStreamDestroy(h->own_stream);
    delete h->comm;
    h->comm = nullptr;
}

int create_impl(int64_t n, int32_t d, int32_t k, int work, int dist, int flags,
                kmeans_handle* out, const void* nccl_id, int nranks, int rank,
                VGroup* vgroup = nullptr) {
    const bool sharded = nccl_id != nullptr || vgroup != nullptr;
    kmeans_ctx* h = nullptr;
    if (!out) return fail(nullptr, KMEANS_EINVAL, "out is NULL");
    *out = nullptr;
    int norm = flags & 0xff;
    if (n < 1 || d < 1 || k < 1 || (nranks == 1 && k > n))
        return fail(nullptr, KMEANS_EINVAL, "need n >= 1, d >= 1, 1 <= k <= n");
    if (work != KMEANS_FP64 && work != KMEANS_FP32)
        return fail(nullptr, KMEANS_EINVAL, "work_prec must be KMEANS_FP64 or KMEANS_FP32");
    if (dist < KMEANS_FP64 || dist > KMEANS_E5M2)
        return fail(nullptr, KMEANS_EINVAL, "unknown dist_prec");
    if (work == KMEANS_FP32 && dist == KMEANS_FP64)
        return fail(nullptr, KMEANS_EINVAL, "dist_prec must not be more precise than work_prec");
    if (norm > KMEANS_NORM_ZSCORE ||
        (flags & ~(0xff | KMEANS_GUARD_SCALE | KMEANS_FORCE_SIMT | KMEANS_GUARD_POW2)))
        return fail(nullptr, KMEANS_EINVAL, "unknown flags");
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return fail(nullptr, KMEANS_EINVAL, "bad rank / nranks");
    int dev = check_device(nullptr);
    if (dev < 0) return dev;

    h = new kmeans_ctx();
    h->n = n; h->d = d; h->k = k; h->work = work; h->dist = dist; h->flags = flags;
    h->norm = norm;
    // guard: 0 off, 1 s = ||x||_inf (reading Z9 A), 2 s = 2^ceil(log2 ||x||_inf) (Z9 B)
    h->guard = (flags & KMEANS_GUARD_POW2) ? 2 : ((flags & KMEANS_GUARD_SCALE) ? 1 : 0);
    h->force_simt = (flags & KMEANS_FORCE_SIMT) ? 1 : 0;
    h->device = dev;
    h->wsize = elem_size(work);
    h->lsize = elem_size(dist);
    h->nranks = nranks; h->rank = rank;
    h->L = AccLayout{k, d};

    // choose the distance kernel (host-side dispatch by (d, k, precision))
    bool low = dist >= KMEANS_FP16;
    h->d_pad = d;
    if (!h->force_simt && smalld_supported(d, k)) {
        h->dist_kernel = DK_SMALLD;
    } else if (!h->force_simt && low && work == KMEANS_FP32 &&
               tc_supported(dist, tc_dpad(dist, d), k)) {
        h->dist_kernel = DK_TCGEN05;
        h->d_pad = tc_dpad(dist, d);
    } else {
        h->dist_kernel = (dist == work) ? DK_SIMT_WORK : DK_SIMT_LOW;
    }

    auto bail = [&](int code, const std::string& m) {
        g_create_err = m;
        free_all(h);
        delete h;
        return code;
    };
#define CA(call)                                                                           \
    do {                                                                                   \
        cudaError_t _e = (call);                                                           \
        if (_e != cudaSuccess) {                                                           \
            cudaGetLastError();                                                            \
            return bail(_e == cudaErrorMemoryAllocation ? KMEANS_ENOMEM : KMEANS_ECUDA,    \
                        std::string(#call) + ": " + cudaGetErrorString(_e));               \
        }                                                                                  \
    } while (0)

    CA(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
    h->stream = h->own_stream;
    size_t W = h->wsize;
    CA(dalloc(&h->Xw, (size_t)n * d * W));
    if (dist == work) {
        h->Xl = h->Xw;
        h->xl_alias = true;
    } else {
        CA(dalloc(&h->Xl, (size_t)n * h->d_pad * h->lsize));
    }
    CA(dalloc(&h->xn, (size_t)n * W));
    CA(dalloc(&h->sx, (size_t)n * W));
    CA(dalloc(&h->Cw, (size_t)k * d * W));
    CA(dalloc(&h->Cl, (size_t)k * std::max(h->d_pad, d) * std::max(h->lsize, h->wsize)));
    {
        // ||c||^2 and the guard scales are padded to a multiple of 256 columns: the pair kernel
        // reads them from global memory (L1-resident) for whole centroid tiles, and a padded
        // centroid (TMA zero-fills its row) must never win: cn = +inf, sc = 0 there. Prep only
        // ever writes j < k, so the tail is set once here.
        const size_t kp = ((size_t)k + 255) / 256 * 256;
        CA(dalloc(&h->cn, kp * W));
        CA(dalloc(&h->sc, kp * W));
        CA(cudaMemset(h->sc, 0, kp * W));
        if (W == sizeof(float) && kp > (size_t)k) {
            std::vector<float> inf(kp - k, INFINITY);
            CA(cudaMemcpy((float*)h->cn + k, inf.data(), inf.size() * sizeof(float),
                          cudaMemcpyHostToDevice));
        }
    }
    CA(dalloc(&h->labels, (size_t)n * sizeof(int32_t)));
    CA(dalloc(&h->acc, (size_t)h->L.total() * sizeof(double)));
    CA(dalloc(&h->cnt, (size_t)k * sizeof(int)));
    CA(dalloc(&h->offs, (size_t)(k + 1) * sizeof(int)));
    CA(dalloc(&h->cursor, (size_t)k * sizeof(int)));
    CA(dalloc(&h->perm, (size_t)n * sizeof(int)));
    {
        size_t b_cb, b_part, b_pid;
        update_scratch_bytes(n, d, k, &b_cb, &b_part, &b_pid);
        CA(dalloc(&h->us.cb, b_cb));
        CA(dalloc(&h->us.part, b_part));
        CA(dalloc(&h->us.mpo, b_pid));
    }
    h->fx_ok = work == KMEANS_FP32 && k <= 12288 && d <= 8192 && h->dist_kernel != DK_SMALLD &&
               !getenv("MPK_NO_FX");
    if (h->fx_ok) {
        // list capacity n/16 rows: beyond it the full re-summation is the cheaper path.
        // MPK_FX_CAP overrides (tests: 0 = always the full path, n = always incremental)
        h->fx.cap = (int)std::min<int64_t>(std::max<int64_t>(n / 16, 4096), n);
        if (const char* e = getenv("MPK_FX_CAP")) h->fx.cap = (int)std::min<int64_t>(atoll(e), n);
        CA(dalloc(&h->fx.amax, (size_t)d * sizeof(unsigned)));
        CA(dalloc(&h->fx.sc, (size_t)d * sizeof(float2)));
        CA(dalloc(&h->fx.isc, (size_t)d * sizeof(double)));
        CA(dalloc(&h->fx.Shi, (size_t)k * d * sizeof(long long)));
        CA(dalloc(&h->fx.Slo, (size_t)k * d * sizeof(long long)));
        CA(dalloc(&h->fx.part, fx_part_bytes(n, d)));
        CA(dalloc(&h->fx.prev, (size_t)n * sizeof(int32_t)));
        // the list by 32-row segment: room for every row (the distance kernel writes each
        // segment's changed rows at its own offset, no slot counter)
        CA(dalloc(&h->fx.list, (size_t)((n + 31) / 32) * 32 * sizeof(int3)));
        CA(dalloc(&h->fx.seg_cnt, (size_t)((n + 31) / 32) * sizeof(int)));
        CA(dalloc(&h->fx.gate, 4 * sizeof(int)));
        if (sharded) {          // sharded: each rank keeps its shard's totals; A6 sums them
            CA(dalloc(&h->fx.gShi, (size_t)k * d * sizeof(long long)));
            CA(dalloc(&h->fx.gSlo, (size_t)k * d * sizeof(long long)));
            CA(dalloc(&h->fx.gcnt, (size_t)k * sizeof(int)));
        }
    }
    CA(dalloc(&h->trace, (size_t)KMEANS_MAX_TRACE * sizeof(IterRec)));
    CA(dalloc(&h->shift, (size_t)d * sizeof(double)));
    CA(dalloc(&h->scale, (size_t)d * sizeof(double)));
    h->npartials = norm_stats_blocks(n, d);
    // two partial sets (the one-pass z-score moments) + K per column
    CA(dalloc(&h->partials, ((size_t)h->npartials * d * 4 + d) * sizeof(double)));
    CA(dalloc(&h->census, 4 * sizeof(unsigned long long)));
    CA(dalloc(&h->sse_dev, 4 * sizeof(double)));
    CA(dalloc(&h->fbc, 4 * sizeof(int)));
    CA(dalloc(&h->n_low_dev, sizeof(unsigned long long)));
    h->guard_user = h->guard;
    if (h->dist_kernel == DK_TCGEN05) {
        std::string e;
        h->tc = tc_plan_create(dist, n, d, h->d_pad, k, h->Xl, h->Cl, &e);
        if (!h->tc) {
            // the tcgen05 path must exist for these shapes on sm_100a: report, do not fall back
            return bail(KMEANS_ECUDA, "tcgen05 plan: " + e);
        }
    }
    if (sharded) {
        // A6 transport: an NCCL communicator (also for one rank, so that every collective call
        // site runs), or a rank of a virtual group on this device
        std::string e;
        h->comm = vgroup ? coll_create_virtual(vgroup, rank, &e)
                         : coll_create_nccl(nccl_id, nranks, rank, &e);
        if (!h->comm) return bail(vgroup ? KMEANS_EINVAL : KMEANS_ENCCL, e);
        if (cudaStream_t ss = h->comm->shared_stream()) h->stream = ss;
    }
    // identity transform until a normalising fit
    std::vector<double> zero(d, 0.0), one(d, 1.0);
    CA(cudaMemcpy(h->shift, zero.data(), d * sizeof(double), cudaMemcpyHostToDevice));
    CA(cudaMemcpy(h->scale, one.data(), d * sizeof(double), cudaMemcpyHostToDevice));
#undef CA
    *out = h;
    return KMEANS_OK;
}

// Copy rows (host or device source) of the work type into a device buffer.
int stage_rows(kmeans_ctx* h, const void* src, int64_t rows, void* dst) {
    size_t bytes = (size_t)rows * h->d * h->wsize;
    cudaMemcpyKind kind = is_device_ptr(src) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
    CK(cudaMemcpyAsync(dst, src, bytes, kind, h->stream));
    return 0;
}

// Normalisation statistics (shift/scale) of the rows at Xsrc (the caller's device buffer or the
// staged copy), globally across ranks when sharded (the per-feature aggregates are allreduced).
// The transform itself is applied by the fused prep (launch_prep_norm).
int normalise_stats(kmeans_ctx* h, const void* Xsrc, int64_t rows) {
    if (h->norm == KMEANS_NORM_NONE) return 0;
    cudaStream_t s = h->stream;
    int nb = norm_stats_blocks(rows, h->d);
    if (nb > h->npartials) nb = h->npartials;
    double n_total = (double)rows;
    if (h->comm) {
        double* tmp = h->sse_dev + 2;
        CK(cudaMemcpyAsync(tmp, &n_total, sizeof(double), cudaMemcpyHostToDevice, s));
        CKC(AR(tmp, tmp, 1, CT_F64, CO_SUM));
        CK(cudaMemcpyAsync(&n_total, tmp, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
    }
    if (h->norm == KMEANS_NORM_ZSCORE && !h->comm && !getenv("MPK_TWO_PASS_ZSCORE") &&
        norm_moments_ok(h->work, Xsrc, h->d)) {
        // one read of X: moments about row 0 (R4)
        double* part2 = h->partials + (size_t)h->npartials * h->d * 2;
        double* kbuf = part2 + (size_t)h->npartials * h->d * 2;
        CK(launch_norm_moments(Xsrc, rows, h->d, h->partials, part2, nb, kbuf, h->shift,
                               h->scale, n_total, s));
        return 0;
    }
    CK(launch_norm_stats(h->work, h->norm, Xsrc, rows, h->d, h->partials, nb, h->shift,
                         h->scale, s));
    if (h->norm == KMEANS_NORM_ZSCORE) {
        if (h->comm) CKC(AR(h->shift, h->shift, h->d, CT_F64, CO_SUM));
        CK(launch_norm_post(0, h->d, n_total, h->shift, h->scale, s));
        CK(launch_norm_ssq(h->work, Xsrc, rows, h->d, h->partials, nb, h->shift, h->scale, s));
        if (h->comm) CKC(AR(h->scale, h->scale, h->d, CT_F64, CO_SUM));
        CK(launch_norm_post(1, h->d, n_total, h->shift, h->scale, s));
    } else {
        if (h->comm) {
            CKC(AR(h->shift, h->shift, h->d, CT_F64, CO_MIN));
            CKC(AR(h->scale, h->scale, h->d, CT_F64, CO_MAX));
        }
        CK(launch_norm_post(2, h->d, n_total, h->shift, h->scale, s));
    }
    return 0;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

struct EventPool {
    std::vector<cudaEvent_t> ev;
    ~EventPool() {
        for (auto e : ev) cudaEventDestroy(e);
    }
    cudaEvent_t get() {
        cudaEvent_t e;
        cudaEventCreate(&e);
        ev.push_back(e);
        return e;
    }
};

constexpr int kCandQ = 32;   // candidate columns kept per uncertified row

// Alg 4 / Alg 5 on the tensor cores (R10). The certified filter of the final pass
// (FINAL mode of the pair kernel) runs on the loop's guarded low-precision operands: a row whose
// low-precision top-2 gap exceeds 2 (E + B32) has the same argmin under Alg 4's per-pair
// distances (the triggered pairs' CUDA-core evaluation differs from the tensor core's only by
// accumulation order, the others by at most E + B32, R2's proof), and for every other row the
// columns with v^_j <= T contain that argmin and its ties; those candidates are evaluated with
// the switch exactly as K6m-b does (cand_exact_mixed). Rows with no or too many candidates get
// the full K6m-b evaluation on gathered copies. eta is counted exactly from the sorted norms.
bool mixed_tc_ok(const kmeans_ctx* h) {
    return h->dist_kernel == DK_TCGEN05 && h->work == KMEANS_FP32 &&
           (h->dist == KMEANS_FP16 || h->dist == KMEANS_BF16) && tc_plan_has_cand(h->tc) &&
           h->k <= 16384 && !getenv("MPK_MIXED_SIMT");
}

int ensure_cand_buffers(kmeans_ctx* h, TcPlan* plan, int64_t nfb) {
    if (nfb <= h->cand_cap) return 0;
    void* old[] = {h->cand_X, h->cand_sx, h->cand_cnt, h->cand, h->cand_left, h->cand_key};
    for (void* b : old)
        if (b) cudaFree(b);
    h->cand_X = h->cand_sx = nullptr;
    h->cand_cnt = h->cand = h->cand_left = nullptr;
    h->cand_key = nullptr;
    const int64_t cap = std::min<int64_t>(h->n, nfb + nfb / 4 + 1024);
    int rb = 0;
    tc_plan_operands(plan, &rb);
    CK(cudaMalloc(&h->cand_X, (size_t)cap * rb));
    CK(cudaMalloc(&h->cand_sx, (size_t)cap * 4));
    CK(cudaMalloc(&h->cand_cnt, (size_t)cap * 4));
    CK(cudaMalloc(&h->cand, (size_t)cap * kCandQ * 4));
    CK(cudaMalloc(&h->cand_left, (size_t)cap * 4));
    CK(cudaMalloc(&h->cand_key, (size_t)cap * 8));
    h->cand_cap = cap;
    return 0;
}

int assign_mixed_tc(kmeans_ctx* h, int64_t rows, double* acc_sse, double* acc_changed) {
    cudaStream_t s = h->stream;
    const int d = h->d, k = h->k;
    const double delta2 = h->delta * h->delta;
    if (!h->mix_prev) {
        int kp = 1;
        while (kp < k) kp <<= 1;
        CK(cudaMalloc(&h->mix_prev, (size_t)h->n * sizeof(int32_t)));
        CK(cudaMalloc(&h->mix_sorted, (size_t)kp * sizeof(float)));
    }
    if (!h->fb_thr) CK(cudaMalloc(&h->fb_thr, (size_t)std::max<int64_t>(h->n, 1) * 4));
    if (acc_changed)
        CK(cudaMemcpyAsync(h->mix_prev, h->labels, (size_t)rows * sizeof(int32_t),
                           cudaMemcpyDeviceToDevice, s));
    // eta: the triggered pairs of these rows, exactly
    CK(launch_mixed_count((const float*)h->xn, rows, (const float*)h->cn, k, delta2,
                          h->mix_sorted, h->n_low_dev, s));
    // the certified filter (labels of every row; the uncertified ones listed with thresholds)
    Problem p{rows, d, k, h->d_pad, h->guard};
    CK(cudaMemsetAsync(h->fbc, 0, 2 * sizeof(int), s));
    CK(launch_final_tc(h->tc, p, (const float*)h->xn, (const float*)h->sx, (const float*)h->cn,
                       (const float*)h->sc, h->labels, h->fbc, h->perm, h->fb_thr, s));
    int nfb = 0;
    CK(cudaMemcpyAsync(&nfb, h->fbc, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (nfb > 0) {
        if (int rc = ensure_cand_buffers(h, h->tc, nfb)) return rc;
        int rb = 0;
        const void* ops = tc_plan_operands(h->tc, &rb);
        CK(launch_gather_rows(ops, rb, h->perm, nfb, h->cand_X, (const float*)h->sx, h->cand_sx, s));
        CK(cudaMemsetAsync(h->cand_cnt, 0, (size_t)nfb * 4, s));
        CK(launch_cand_tc(h->tc, h->cand_X, nfb, h->guard, h->cand_sx, (const float*)h->cn,
                          (const float*)h->sc, h->fb_thr, h->cand_cnt, h->cand, kCandQ, s));
        CK(launch_cand_exact_mixed(h->dist, h->Xl, (const float*)h->Xw, h->Cl, (const float*)h->Cw,
                                   (const float*)h->xn, (const float*)h->sx, (const float*)h->cn,
                                   (const float*)h->sc, d, h->d_pad, delta2, h->perm, nfb,
                                   h->cand_cnt, h->cand, kCandQ, h->labels, h->fbc + 1,
                                   h->cand_left, h->cand_key, s));
        int nleft = 0;
        CK(cudaMemcpyAsync(&nleft, h->fbc + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (nleft > 0) {
            // the full K6m-b evaluation of the remaining rows, on gathered copies
            if (nleft > h->mix_cap) {
                void* old[] = {h->mix_Xl, h->mix_Xw, h->mix_xn, h->mix_sx, h->mix_lab};
                for (void* b : old)
                    if (b) cudaFree(b);
                const int64_t cap = std::min<int64_t>(h->n, (int64_t)nleft + nleft / 4 + 256);
                CK(cudaMalloc(&h->mix_Xl, (size_t)cap * rb));
                CK(cudaMalloc((void**)&h->mix_Xw, (size_t)cap * d * 4));
                CK(cudaMalloc((void**)&h->mix_xn, (size_t)cap * 4));
                CK(cudaMalloc((void**)&h->mix_sx, (size_t)cap * 4));
                CK(cudaMalloc((void**)&h->mix_lab, (size_t)cap * 4));
                h->mix_cap = cap;
            }
            CK(launch_gather_rows(ops, rb, h->cand_left, nleft, h->mix_Xl, (const float*)h->sx,
                                  h->mix_sx, s));
            CK(launch_gather_float_rows((const float*)h->Xw, d, h->cand_left, nleft, h->mix_Xw, s));
            CK(launch_gather_float_rows((const float*)h->xn, 1, h->cand_left, nleft, h->mix_xn, s));
            Problem pl{nleft, d, k, h->d_pad, h->guard};
            unsigned long long* discard = nullptr;   // trigger counts come from mixed_count
            CK(cudaMallocAsync((void**)&discard, sizeof(unsigned long long), s));
            CK(launch_assign_mixed(h->work, h->dist, pl, h->delta, h->mix_Xl, h->mix_Xw, h->mix_xn,
                                   h->mix_sx, h->Cl, h->Cw, h->cn, h->sc, h->mix_lab, nullptr,
                                   nullptr, discard, s));
            CK(cudaFreeAsync(discard, s));
            CK(launch_scatter_labels(h->mix_lab, h->cand_left, nleft, h->labels, s));
        }
        h->last_fallback = nleft;
    }
    // SSE_t and the changed count from the final labels (Alg 4 distances of the labels)
    if (acc_sse || acc_changed)
        CK(launch_mixed_label_eval(h->dist, h->Xl, (const float*)h->Xw, h->Cl, (const float*)h->Cw,
                                   (const float*)h->xn, (const float*)h->sx, (const float*)h->cn,
                                   (const float*)h->sc, rows, d, h->d_pad, delta2, h->labels,
                                   acc_changed ? h->mix_prev : nullptr, acc_sse, acc_changed, s));
    return 0;
}

// Distance + argmin for the current centroids on h->n rows (loop iteration or assign).
int run_assign(kmeans_ctx* h, int64_t rows, double* acc_sse, double* acc_changed,
               bool* fx_listed = nullptr) {
    if (fx_listed) *fx_listed = false;
    Problem p{rows, h->d, h->k, h->d_pad, h->guard};
    if (h->delta > 0.0 && mixed_tc_ok(h)) {
        if (int rc = assign_mixed_tc(h, rows, acc_sse, acc_changed)) return rc;
    } else if (h->delta > 0.0) {   // Alg 4 on CUDA cores (both dot products per pair)
        CK(launch_assign_mixed(h->work, h->dist, p, h->delta, h->Xl, h->Xw, h->xn, h->sx, h->Cl,
                               h->Cw, h->cn, h->sc, h->labels, acc_sse, acc_changed,
                               h->n_low_dev, h->stream));
    } else if (h->dist_kernel == DK_TCGEN05) {
        CK(launch_assign_tc(h->tc, p, (const float*)h->xn, h->guard ? (const float*)h->sx : nullptr,
                            (const float*)h->cn, h->guard ? (const float*)h->sc : nullptr,
                            h->labels, acc_sse, acc_changed, h->stream,
                            fx_listed ? &h->fx : nullptr, fx_listed));
    } else {
        CK(launch_assign_simt(h->work, h->dist, p, h->Xl, h->xn, h->guard ? h->sx : nullptr,
                              h->Cl, h->cn, h->guard ? h->sc : nullptr, h->labels, acc_sse,
                              acc_changed, h->stream));
    }
    return 0;
}

int prep_centroids(kmeans_ctx* h) {
    CK(launch_prep(h->work, h->dist, h->Cw, h->k, h->d, h->d_pad, h->guard, h->cn, h->sc, h->Cl,
                   h->census + 2, h->stream));
    return 0;
}

// Alg 3 step 7: labels = argmin_j of the working-precision expanded distance with
// the final centroids. With tcgen05 available the contraction runs as a certified filter
// (launch_final_tc): rows whose low-precision top-2 gap exceeds the rigorous error bound keep
// the filter's argmin, which equals the working-precision argmin; the remaining rows are
// re-evaluated by the CUDA-core kernel in working precision. Otherwise the CUDA-core kernel
// evaluates every row.
int final_assign(kmeans_ctx* h, const Problem& pf) {
    cudaStream_t s = h->stream;
    const int64_t n = h->n;
    const int d = h->d, k = h->k;
    h->last_fallback = -1;
    h->last_uncertified = -1;
    // working-precision norms of the final centroids
    CK(launch_prep(h->work, h->work, h->Cw, k, d, d, 0, h->cn, nullptr, h->Cl, nullptr, s));
    TcPlan* plan = nullptr;
    const void* fx_sx = nullptr;
    const void* fx_sc = nullptr;
    int fguard = 0, fdpad = 0;
    if (h->dist_kernel == DK_TCGEN05 && h->work == KMEANS_FP32) {
        unsigned long long cen[4];
        CK(cudaMemcpyAsync(cen, h->census, sizeof(cen), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        bool reuse = (h->dist == KMEANS_FP16 || h->dist == KMEANS_BF16) && cen[0] == 0;
        if (reuse) {
            // loop operands: rebuild C~ from the final centroids, check it stayed finite
            CK(cudaMemsetAsync(h->census + 2, 0, 2 * sizeof(unsigned long long), s));
            CK(launch_prep(h->work, h->dist, h->Cw, k, d, h->d_pad, h->guard, h->cn, h->sc, h->Cl,
                           h->census + 2, s));
            CK(cudaMemcpyAsync(cen, h->census, sizeof(cen), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (cen[2] == 0) {
                plan = h->tc;
                fx_sx = h->sx; fx_sc = h->sc; fguard = h->guard; fdpad = h->d_pad;
            }
        }
        if (!plan && !h->fin_failed) {
            if (!h->fin) {
                h->fin_dpad = tc_dpad(KMEANS_FP16, d);
                cudaError_t e1 = cudaMalloc(&h->fin_Xl, (size_t)n * h->fin_dpad * 2);
                cudaError_t e2 = cudaMalloc(&h->fin_Cl, (size_t)k * h->fin_dpad * 2);
                cudaError_t e3 = cudaMalloc(&h->fin_sx, (size_t)n * 4);
                // padded like h->sc (see create_impl)
                const size_t kp = ((size_t)k + 255) / 256 * 256;
                cudaError_t e4 = cudaMalloc(&h->fin_sc, kp * 4);
                if (e4 == cudaSuccess) e4 = cudaMemset(h->fin_sc, 0, kp * 4);
                std::string err;
                if (e1 == cudaSuccess && e2 == cudaSuccess && e3 == cudaSuccess &&
                    e4 == cudaSuccess && tc_supported(KMEANS_FP16, h->fin_dpad, k))
                    h->fin = tc_plan_create(KMEANS_FP16, n, d, h->fin_dpad, k, h->fin_Xl,
                                            h->fin_Cl, &err);
                cudaGetLastError();
                if (!h->fin) h->fin_failed = true;
            }
            if (h->fin) {
                // guarded fp16 operands (Alg 4 scaling: never overflows)
                CK(launch_prep(h->work, KMEANS_FP16, h->Xw, n, d, h->fin_dpad, 1, h->xn,
                               h->fin_sx, h->fin_Xl, nullptr, s));
                CK(launch_prep(h->work, KMEANS_FP16, h->Cw, k, d, h->fin_dpad, 1, h->cn,
                               h->fin_sc, h->fin_Cl, nullptr, s));
                plan = h->fin;
                fx_sx = h->fin_sx; fx_sc = h->fin_sc; fguard = 1; fdpad = h->fin_dpad;
            }
        }
    }
    if (plan) {
        Problem p{n, d, k, fdpad, fguard};
        const bool cand_path = tc_plan_has_cand(plan) && getenv("MPK_NO_CAND") == nullptr;
        if (cand_path && !h->fb_thr) CK(cudaMalloc(&h->fb_thr, (size_t)std::max<int64_t>(n, 1) * 4));
        CK(cudaMemsetAsync(h->fbc, 0, 2 * sizeof(int), s));
        CK(launch_final_tc(plan, p, (const float*)h->xn, (const float*)fx_sx,
                           (const float*)h->cn, (const float*)fx_sc, h->labels, h->fbc, h->perm,
                           cand_path ? h->fb_thr : nullptr, s));
        int nfb = 0;
        CK(cudaMemcpyAsync(&nfb, h->fbc, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        h->last_uncertified = nfb;
        h->last_fallback = nfb;
        if (nfb > 0 && cand_path) {
            // candidate path (R2): gather the uncertified rows' operands, list their
            // candidate columns on the tensor cores, evaluate only those exactly in fp32
            if (nfb > h->cand_cap) {
                void* old[] = {h->cand_X, h->cand_sx, h->cand_cnt, h->cand, h->cand_left, h->cand_key};
                for (void* b : old)
                    if (b) cudaFree(b);
                h->cand_X = h->cand_sx = nullptr;
                h->cand_cnt = h->cand = h->cand_left = nullptr;
                h->cand_key = nullptr;
                const int64_t cap = std::min<int64_t>(n, (int64_t)nfb + nfb / 4 + 1024);
                int rb = 0;
                tc_plan_operands(plan, &rb);
                CK(cudaMalloc(&h->cand_X, (size_t)cap * rb));
                CK(cudaMalloc(&h->cand_sx, (size_t)cap * 4));
                CK(cudaMalloc(&h->cand_cnt, (size_t)cap * 4));
                CK(cudaMalloc(&h->cand, (size_t)cap * kCandQ * 4));
                CK(cudaMalloc(&h->cand_left, (size_t)cap * 4));
                CK(cudaMalloc(&h->cand_key, (size_t)cap * 8));
                h->cand_cap = cap;
            }
            int rb = 0;
            const void* ops = tc_plan_operands(plan, &rb);
            CK(launch_gather_rows(ops, rb, h->perm, nfb, h->cand_X, fguard ? (const float*)fx_sx : nullptr,
                                  fguard ? h->cand_sx : nullptr, s));
            CK(cudaMemsetAsync(h->cand_cnt, 0, (size_t)nfb * 4, s));
            CK(launch_cand_tc(plan, h->cand_X, nfb, fguard, h->cand_sx, (const float*)h->cn,
                              (const float*)fx_sc, h->fb_thr, h->cand_cnt, h->cand, kCandQ, s));
            if (getenv("MPK_CAND_STATS")) {   // debug: candidate count distribution
                std::vector<int> cc(nfb);
                CK(cudaMemcpyAsync(cc.data(), h->cand_cnt, (size_t)nfb * 4, cudaMemcpyDeviceToHost, s));
                CK(cudaStreamSynchronize(s));
                long long tot = 0;
                int mx = 0, over = 0;
                for (int v : cc) { tot += v; mx = std::max(mx, v); over += v > kCandQ; }
                fprintf(stderr, "[cand] rows %d candidates %lld mean %.2f max %d overflow %d\n", nfb,
                        tot, (double)tot / nfb, mx, over);
            }
            CK(launch_cand_exact((const float*)h->Xw, (const float*)h->Cw, (const float*)h->cn, d,
                                 h->perm, nfb, h->cand_cnt, h->cand, kCandQ, h->labels,
                                 h->fbc + 1, h->cand_left, h->cand_key, s));
            int nleft = 0;
            CK(cudaMemcpyAsync(&nleft, h->fbc + 1, sizeof(int), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            h->last_fallback = nleft;
            if (nleft > 0) {
                Problem pl{nleft, d, k, d, 0};
                CK(launch_assign_simt(h->work, h->work, pl, h->Xw, h->xn, nullptr, h->Cw, h->cn,
                                      nullptr, h->labels, nullptr, nullptr, s, h->cand_left));
            }
        } else if (nfb > 0) {
            Problem pl{nfb, d, k, d, 0};
            CK(launch_assign_simt(h->work, h->work, pl, h->Xw, h->xn, nullptr, h->Cw, h->cn,
                                  nullptr, h->labels, nullptr, nullptr, s, h->perm));
        }
        return 0;
    }
    CK(launch_assign_simt(h->work, h->work, pf, h->Xw, h->xn, nullptr, h->Cw, h->cn, nullptr,
                          h->labels, nullptr, nullptr, s));
    return 0;
}

// A1 + A2 for the handle's n rows of X: normalisation statistics and transform (O1), norms,
// guard scales and low-precision operands (O2). A device X is read in place by the statistics
// and the (out-of-place) normalisation, so it is never copied; a host X is staged into Xw first
// (that copy is needed anyway). Resets the operand census.
int prepare_points(kmeans_ctx* h, const void* X) {
    cudaStream_t s = h->stream;
    const int64_t n = h->n;
    const int d = h->d;
    const bool norm = h->norm != KMEANS_NORM_NONE;
    h->fx_amax_done = false;
    if (h->fx_ok) {             // the prep may fill the fixed-point update's column maxima
        CK(cudaMemsetAsync(h->fx.amax, 0, sizeof(unsigned) * d, s));
        CK(cudaMemsetAsync(h->fx.gate, 0, sizeof(int) * 4, s));
    }
    const void* Xsrc = h->Xw;
    if (norm && is_device_ptr(X)) Xsrc = X;
    else if (int rc = stage_rows(h, X, n, h->Xw)) return rc;
    if (norm)
        if (int rc = normalise_stats(h, Xsrc, n)) return rc;
    CK(cudaMemsetAsync(h->census, 0, 4 * sizeof(unsigned long long), s));
    if (prep_fast_ok(h->work, d)) {
        CK(launch_prep_fast(h->dist, Xsrc, n, d, h->d_pad, h->guard, h->xn, h->sx, h->Xl,
                            h->census, norm ? h->Xw : nullptr, norm ? h->shift : nullptr,
                            norm ? h->scale : nullptr, s, h->fx_ok ? h->fx.amax : nullptr,
                            h->fx_ok ? h->fx.gate : nullptr, &h->fx_amax_done));
    } else {
        if (norm) CK(launch_norm_apply(h->work, h->Xw, n, d, h->shift, h->scale, s, Xsrc));
        CK(launch_prep(h->work, h->dist, h->Xw, n, d, h->d_pad, h->guard, h->xn, h->sx, h->Xl,
                       h->census, s));
    }
    return 0;
}

// A3..A7 of the small-d path on one rank through K5g: one launch per iteration, replayed from a
// CUDA graph of kLoopChunk launches; with tol >= 0 the host reads the device stop flag once per
// chunk (launches after convergence return at once), with tol < 0 never.
constexpr int kLoopChunk = 8;

// *deferred (K5p): the loop state's device-to-host copy is enqueued but not waited for; the
// caller reads h->loop_host[1] after its next stream synchronisation (the fit's outputs), so the
// final pass is queued behind the loop without an idle GPU in between.
int run_smalld_loop(kmeans_ctx* h, int max_iter, double tol, int* it_out, bool* conv_out,
                    bool* deferred) {
    cudaStream_t s = h->stream;
    if (!h->loop) {
        CK(cudaMalloc(&h->loop, sizeof(LoopState)));
        CK(cudaMalloc(&h->loop_part, smalld_loop_part_bytes(h->n)));
        CK(cudaMallocHost(&h->loop_host, 2 * sizeof(LoopState)));
    }
    Problem p{h->n, h->d, h->k, h->d_pad, h->guard};
    if (!getenv("MPK_NO_PERSIST")) {
        // K5p: every iteration in one cooperative launch when the rows fit in shared memory
        h->loop_host[0] = LoopState{0, 0, 0, 0u, tol, 0};
        CK(cudaMemcpyAsync(h->loop, &h->loop_host[0], sizeof(LoopState), cudaMemcpyHostToDevice, s));
        const cudaError_t e = launch_smalld_persist(h->work, h->dist, p, h->Xw, h->Cw, h->labels,
                                                    h->loop_part, h->loop, h->trace,
                                                    h->census + 2, max_iter, s);
        if (e == cudaSuccess) {
            CK(cudaMemcpyAsync(&h->loop_host[1], h->loop, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
            if (deferred) {
                *deferred = true;
                *it_out = max_iter;           // upper bound until the copy has landed
                return 0;
            }
            CK(cudaStreamSynchronize(s));
            if (h->loop_host[1].fault)
                return fail(h, KMEANS_ECUDA, "K5p: a block timed out at the grid barrier");
            *it_out = h->loop_host[1].iter;
            *conv_out = h->loop_host[1].converged != 0;
            return 0;
        }
        if (e != cudaErrorNotSupported) CK(e);
    }
    auto one = [&](cudaStream_t st) {
        return launch_smalld_iter(h->work, h->dist, p, h->Xw, h->Cw, h->labels, h->loop_part,
                                  h->loop, h->trace, h->census + 2, st);
    };
    CK(launch_smalld_iter(h->work, h->dist, p, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr,
                          nullptr, s));                   // smem attribute, outside any capture
    if (!getenv("MPK_NO_GRAPH") && (!h->loop_graph || h->loop_graph_guard != h->guard)) {
        if (h->loop_graph) cudaGraphExecDestroy(h->loop_graph);
        h->loop_graph = nullptr;
        if (!h->loop_capture) CK(cudaStreamCreateWithFlags(&h->loop_capture, cudaStreamNonBlocking));
        cudaGraph_t g = nullptr;
        CK(cudaStreamBeginCapture(h->loop_capture, cudaStreamCaptureModeThreadLocal));
        for (int q = 0; q < kLoopChunk; ++q) {
            cudaError_t e = one(h->loop_capture);
            if (e != cudaSuccess) {
                cudaStreamEndCapture(h->loop_capture, &g);
                if (g) cudaGraphDestroy(g);
                return fail(h, KMEANS_ECUDA, std::string("K5g capture: ") + cudaGetErrorString(e));
            }
        }
        CK(cudaStreamEndCapture(h->loop_capture, &g));
        cudaError_t e = cudaGraphInstantiate(&h->loop_graph, g, 0);
        cudaGraphDestroy(g);
        CK(e);
        launches_add(-kLoopChunk);   // captured, not launched
        h->loop_graph_guard = h->guard;
    }
    h->loop_host[0] = LoopState{0, 0, 0, 0u, tol, 0};
    CK(cudaMemcpyAsync(h->loop, &h->loop_host[0], sizeof(LoopState), cudaMemcpyHostToDevice, s));
    int done = 0;
    while (done < max_iter) {
        const int m = std::min(kLoopChunk, max_iter - done);
        if (m == kLoopChunk && h->loop_graph) {
            CK(cudaGraphLaunch(h->loop_graph, s));
            launches_add(kLoopChunk);
        } else {
            for (int q = 0; q < m; ++q) CK(one(s));
        }
        done += m;
        if (tol >= 0.0 && done < max_iter) {
            CK(cudaMemcpyAsync(&h->loop_host[1], h->loop, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (h->loop_host[1].stop) break;
        }
    }
    CK(cudaMemcpyAsync(&h->loop_host[1], h->loop, sizeof(LoopState), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *it_out = h->loop_host[1].iter;
    *conv_out = h->loop_host[1].converged != 0;
    return 0;
}

int fit_impl(kmeans_ctx* h, const void* X, const void* C0, int32_t max_iter, double tol,
             int32_t* labels_out, void* cent_out, double* sse_out, int32_t* iters_out) {
    if (!X || !C0) return fail(h, KMEANS_EINVAL, "X and C0 are required");
    if (max_iter < 1) return fail(h, KMEANS_EINVAL, "max_iter must be >= 1");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    EventPool evp;
    const long long launches0 = launches_read();
    cudaEvent_t e0 = evp.get(), e1 = evp.get(), e2 = evp.get(), e3 = evp.get();
    const int64_t n = h->n;
    const int d = h->d, k = h->k;

    CK(cudaEventRecord(e0, s));
    // ---- A1 + A2: normalise X, point prep; normalise C0 ----------------------------------
    if (int rc = prepare_points(h, X)) return rc;
    if (int rc = stage_rows(h, C0, k, h->Cw)) return rc;
    if (h->norm != KMEANS_NORM_NONE)
        CK(launch_norm_apply(h->work, h->Cw, k, d, h->shift, h->scale, s));
    CK(cudaMemsetAsync(h->n_low_dev, 0, sizeof(unsigned long long), s));
    CK(cudaMemsetAsync(h->labels, 0xff, (size_t)n * sizeof(int32_t), s));   // labels_prev = -1
    CK(cudaMemsetAsync(h->trace, 0, sizeof(IterRec) * KMEANS_MAX_TRACE, s));
    bool fx_on = false;
    if (h->fx_ok) {
        // FX state for this fit: per-feature grids from max |x|, zero totals and counts, previous
        // labels -1 (every row is "changed" in iteration 1). One host read: a non-finite X
        // disables FX for the fit (the grid needs finite values).
        CK(launch_fx_colmax((const float*)h->Xw, n, d, h->fx, h->fx_amax_done, s));
        if (h->comm) {          // one grid for all ranks; any rank's non-finite X disables FX
            h->comm->group_start();
            CKC(AR(h->fx.amax, h->fx.amax, d, CT_U32, CO_MAX));
            CKC(AR(h->fx.gate + 2, h->fx.gate + 2, 1, CT_I32, CO_MAX));
            CKC(h->comm->group_end(&_m));
        }
        CK(launch_fx_scale(d, h->fx, s));
        CK(cudaMemsetAsync(h->fx.Shi, 0, (size_t)k * d * sizeof(long long), s));
        CK(cudaMemsetAsync(h->fx.Slo, 0, (size_t)k * d * sizeof(long long), s));
        CK(cudaMemsetAsync(h->cnt, 0, (size_t)k * sizeof(int), s));
        CK(cudaMemsetAsync(h->fx.prev, 0xff, (size_t)n * sizeof(int32_t), s));
        CK(cudaMemcpyAsync(h->fx.gate + 1, &h->fx.cap, sizeof(int), cudaMemcpyHostToDevice, s));
        int bad = 0;
        CK(cudaMemcpyAsync(&bad, h->fx.gate + 2, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        fx_on = bad == 0;
    }
    CK(cudaEventRecord(e1, s));

    // ---- A3..A7: Lloyd iterations ---------------------------------------------------------
    std::vector<cudaEvent_t> kev;
    const bool timing = h->timing != 0;
    int it = 0;
    bool converged = false;
    IterRec rec_h{};
    IterRec* rec_scratch = h->trace + (KMEANS_MAX_TRACE - 1);
    bool loop_deferred = false;
    const bool fused_loop = h->dist_kernel == DK_SMALLD && h->delta <= 0.0 && !h->comm &&
                            smalld_loop_supported(d, k) && !getenv("MPK_NO_FUSED_LOOP");
    if (fused_loop) {
        cudaEvent_t t0 = nullptr, t1 = nullptr;
        if (timing) { t0 = evp.get(); t1 = evp.get(); CK(cudaEventRecord(t0, s)); }
        if (int rc = run_smalld_loop(h, max_iter, tol, &it, &converged, &loop_deferred)) return rc;
        // one fused kernel per iteration: its time is reported as the distance step's
        if (timing) { CK(cudaEventRecord(t1, s)); kev.insert(kev.end(), {t0, t1, t1, t1, t1}); }
    }
    if (!fused_loop) for (it = 1; it <= max_iter; ++it) {
        IterRec* rec = (it <= KMEANS_MAX_TRACE - 1) ? h->trace + (it - 1) : rec_scratch;
        if (rec == rec_scratch) CK(cudaMemsetAsync(rec_scratch, 0, sizeof(IterRec), s));
        cudaEvent_t t0 = nullptr, t1 = nullptr, t2 = nullptr, t3 = nullptr, t4 = nullptr;
        if (timing) { t0 = evp.get(); t1 = evp.get(); t2 = evp.get(); t3 = evp.get(); t4 = evp.get(); }
        // with the fixed-point update finalize_fx zeroes SSE_t, the changed count and the
        // list counter for the next iteration (zeroed here before the first)
        if (!fx_on || it == 1) {
            CK(cudaMemsetAsync(h->acc, 0, sizeof(double) * h->L.total(), s));
            if (fx_on) CK(cudaMemsetAsync(h->fx.gate, 0, sizeof(int), s));
        }
        if (int rc = prep_centroids(h)) return rc;                         // A3
        if (timing) CK(cudaEventRecord(t0, s));
        if (h->dist_kernel == DK_SMALLD && h->delta <= 0.0) {              // A4 + A5 fused
            Problem p{n, d, k, h->d_pad, h->guard};
            CK(launch_smalld_fused(h->work, h->dist, p, h->Xw, h->Cl, h->cn,
                                   h->guard ? h->sc : nullptr, h->labels, h->acc, h->L, s));
            if (timing) { CK(cudaEventRecord(t1, s)); CK(cudaEventRecord(t2, s)); }
        } else {
            bool listed = false;     // the distance kernel listed the changed rows (FX)
            if (int rc = run_assign(h, n, h->acc + h->L.sse(), h->acc + h->L.changed(),
                                    fx_on ? &listed : nullptr))
                return rc;                                                   // A4
            if (timing) CK(cudaEventRecord(t1, s));
            if (fx_on)
                CK(launch_update_fx((const float*)h->Xw, n, d, k, h->labels, h->cnt, h->offs,
                                    h->cursor, h->perm, h->us, h->fx, s, listed));   // A5 (R9)
            else
                CK(launch_update(h->work, h->Xw, n, d, k, h->labels, h->cnt, h->offs, h->cursor,
                                 h->perm, h->acc, h->L, h->us, s));          // A5
            if (timing) CK(cudaEventRecord(t2, s));
        }
        if (h->comm && fx_on)        // A6: the FX totals are reduced below; here SSE_t, changed
            CKC(AR(h->acc + h->L.sse(), h->acc + h->L.sse(), h->L.total() - h->L.sse(), CT_F64,
                   CO_SUM));
        else if (h->comm)                                                    // A6
            CKC(AR(h->acc, h->acc, h->L.total(), CT_F64, CO_SUM));
        if (timing) CK(cudaEventRecord(t3, s));
        if (fx_on && h->comm) {
            // A6 for the exact totals: integer sums, so the allreduce is exact and every rank
            // finalises the same centres
            h->comm->group_start();
            CKC(AR(h->fx.Shi, h->fx.gShi, (size_t)k * d, CT_I64, CO_SUM));
            CKC(AR(h->fx.Slo, h->fx.gSlo, (size_t)k * d, CT_I64, CO_SUM));
            CKC(AR(h->cnt, h->fx.gcnt, k, CT_I32, CO_SUM));
            CKC(h->comm->group_end(&_m));
            CK(launch_finalize_fx(k, d, h->fx, h->fx.gShi, h->fx.gSlo, h->fx.gcnt, h->acc, h->L,
                                  (float*)h->Cw, rec, s));
        } else if (fx_on)
            CK(launch_finalize_fx(k, d, h->fx, h->fx.Shi, h->fx.Slo, h->cnt, h->acc, h->L,
                                  (float*)h->Cw, rec, s));
        else
            CK(launch_finalize(h->work, k, d, h->acc, h->L, h->Cw, rec, s));    // A7
        if (timing) { CK(cudaEventRecord(t4, s)); kev.insert(kev.end(), {t0, t1, t2, t3, t4}); }
        if (tol >= 0.0) {
            CK(cudaMemcpyAsync(&rec_h, rec, sizeof(IterRec), cudaMemcpyDeviceToHost, s));
            CK(cudaStreamSynchronize(s));
            if (rec_h.changed == 0.0 || std::sqrt(rec_h.shift2) <= tol) {
                converged = true;
                break;
            }
        }
    }
    if (!fused_loop && it > max_iter) it = max_iter;
    CK(cudaEventRecord(e2, s));

    // ---- A8: final assignment in working precision + direct-formula SSE -------------------
    {
        Problem pf{n, d, k, d, 0};
        if (int rc = final_assign(h, pf)) return rc;
        CK(cudaMemsetAsync(h->sse_dev, 0, sizeof(double), s));
        CK(launch_final_sse(h->work, h->Xw, n, d, h->Cw, h->labels, h->sse_dev, s));
        if (h->comm)
            CKC(AR(h->sse_dev, h->sse_dev, 1, CT_F64, CO_SUM));
    }
    CK(cudaEventRecord(e3, s));

    // ---- outputs ---------------------------------------------------------------------------
    double sse_h = 0.0;
    CK(cudaMemcpyAsync(&sse_h, h->sse_dev, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (labels_out) {
        cudaMemcpyKind kind = is_device_ptr(labels_out) ? cudaMemcpyDeviceToDevice
                                                        : cudaMemcpyDeviceToHost;
        CK(cudaMemcpyAsync(labels_out, h->labels, (size_t)n * sizeof(int32_t), kind, s));
    }
    if (cent_out) {
        cudaMemcpyKind kind = is_device_ptr(cent_out) ? cudaMemcpyDeviceToDevice
                                                      : cudaMemcpyDeviceToHost;
        CK(cudaMemcpyAsync(cent_out, h->Cw, (size_t)k * d * h->wsize, kind, s));
    }
    unsigned long long census_h[4], n_low_h = 0;
    CK(cudaMemcpyAsync(census_h, h->census, sizeof(census_h), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&n_low_h, h->n_low_dev, sizeof(n_low_h), cudaMemcpyDeviceToHost, s));
    int tl = std::min(it, KMEANS_MAX_TRACE - 1);
    std::vector<IterRec> tr(tl);
    if (tl > 0) CK(cudaMemcpyAsync(tr.data(), h->trace, sizeof(IterRec) * tl,
                                   cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    CK(cudaGetLastError());
    if (loop_deferred) {
        if (h->loop_host[1].fault)
            return fail(h, KMEANS_ECUDA, "K5p: a block timed out at the grid barrier");
        it = h->loop_host[1].iter;
        converged = h->loop_host[1].converged != 0;
        tl = std::min(it, KMEANS_MAX_TRACE - 1);
        tr.resize(tl);
    }

    kmeans_stats& st = h->stats;
    memset(&st, 0, sizeof(st));
    st.iters = it;
    st.converged = converged ? 1 : 0;
    st.dist_kernel = h->dist_kernel;
    st.n_nonfinite = (int64_t)(census_h[0] + census_h[2]);
    st.n_underflow = (int64_t)(census_h[1] + census_h[3]);
    st.t_prep_ms = elapsed(e0, e1);
    st.t_loop_ms = elapsed(e1, e2);
    st.t_final_ms = elapsed(e2, e3);
    st.trace_len = tl;
    int any_empty = 0;
    for (int t = 0; t < tl; ++t) {
        st.sse_t[t] = tr[t].sse;
        st.shift2_t[t] = tr[t].shift2;
        st.changed_t[t] = (int64_t)tr[t].changed;
        st.empty_t[t] = (int32_t)tr[t].empty;
        st.u_bound_t[t] = tr[t].ub_inv > 0.0 ? 1.0 / tr[t].ub_inv : INFINITY;
        if (st.u_bound_t[t] < (h->work == KMEANS_FP64 ? 0x1p-53 : 0x1p-24)) st.n_update_prec_short++;
        if (tr[t].empty > 0) any_empty = 1;
    }
    if (timing) {
        for (size_t q = 0; q + 4 < kev.size() + 0; q += 5) {
            st.t_dist_ms += elapsed(kev[q], kev[q + 1]);
            st.t_update_ms += elapsed(kev[q + 1], kev[q + 2]);
            st.t_allreduce_ms += elapsed(kev[q + 2], kev[q + 3]);
            st.t_finalize_ms += elapsed(kev[q + 3], kev[q + 4]);
        }
    }
    st.n_dist_launches = it;
    st.n_kernel_launches = launches_read() - launches0;
    st.n_final_fallback = h->last_fallback;
    st.n_final_uncertified = h->last_uncertified;
    // distances formed in the loop on this rank: every iteration computes all n k pairs;
    // with delta > 0, n_dist_low of them were triggered to low precision (eta)
    h->last_n_dist = (int64_t)it * n * k;
    h->last_n_low = h->delta > 0.0 ? (int64_t)n_low_h : h->last_n_dist;
    st.n_dist_low = h->last_n_low;
    st.n_dist = h->last_n_dist;
    st.eta = st.n_dist > 0 ? (double)st.n_dist_low / (double)st.n_dist : 1.0;
    st.tc_variant = (h->dist_kernel == DK_TCGEN05 && h->delta <= 0.0) ? tc_plan_kind(h->tc) : 0;
    st.n_ranks = h->nranks;
    int warn = 0;
    if (st.n_nonfinite > 0) warn |= KMEANS_WARN_NONFINITE;
    if (any_empty) warn |= KMEANS_WARN_EMPTY;
    if (tol >= 0.0 && !converged) warn |= KMEANS_WARN_MAXITER;
    if (st.n_underflow > 0) warn |= KMEANS_WARN_UNDERFLOW;
    st.warnings = warn;
    if (sse_out) *sse_out = sse_h;
    if (iters_out) *iters_out = it;
    h->have_centroids = true;
    return warn;
}

}  // namespace

extern "C" {

int kmeans_create(int64_t n, int32_t d, int32_t k, int work_prec, int dist_prec, int flags,
                  kmeans_handle* out) {
    return create_impl(n, d, k, work_prec, dist_prec, flags, out, nullptr, 1, 0);
}

int kmeans_create_dist(int64_t n_local, int32_t d, int32_t k, int work_prec, int dist_prec,
                       int flags, const void* nccl_unique_id, int nranks, int rank,
                       kmeans_handle* out) {
    if (!nccl_unique_id && nranks > 1) return fail(nullptr, KMEANS_EINVAL, "nccl id is NULL");
    return create_impl(n_local, d, k, work_prec, dist_prec, flags, out, nccl_unique_id, nranks,
                       rank);
}

int kmeans_vgroup_create(int nranks, kmeans_vgroup* out) {
    if (!out) return fail(nullptr, KMEANS_EINVAL, "out is NULL");
    *out = nullptr;
    int dev = check_device(nullptr);
    if (dev < 0) return dev;
    std::string e;
    VGroup* g = vgroup_create(nranks, &e);
    if (!g) return fail(nullptr, KMEANS_EINVAL, e);
    *out = reinterpret_cast<kmeans_vgroup>(g);
    return KMEANS_OK;
}

int kmeans_create_virtual(int64_t n_local, int32_t d, int32_t k, int work_prec, int dist_prec,
                          int flags, kmeans_vgroup group, int rank, kmeans_handle* out) {
    if (!group) return fail(nullptr, KMEANS_EINVAL, "group is NULL");
    VGroup* g = reinterpret_cast<VGroup*>(group);
    return create_impl(n_local, d, k, work_prec, dist_prec, flags, out, nullptr,
                       vgroup_size(g), rank, g);
}

int kmeans_vgroup_destroy(kmeans_vgroup group) {
    if (!group) return KMEANS_OK;
    if (vgroup_destroy(reinterpret_cast<VGroup*>(group)) != 0)
        return fail(nullptr, KMEANS_EINVAL, "destroy the group's handles first");
    return KMEANS_OK;
}

int kmeans_nccl_unique_id(void* out128) {
    if (!out128) return KMEANS_EINVAL;
    ncclUniqueId id;
    if (ncclGetUniqueId(&id) != ncclSuccess) return KMEANS_ENCCL;
    memcpy(out128, &id, sizeof(id));
    return KMEANS_OK;
}

int kmeans_fit(kmeans_handle h, const void* X, const void* C0, int32_t max_iter, double tol,
               int32_t* labels, void* centroids, double* sse, int32_t* iters) {
    if (!h) return KMEANS_EINVAL;
    return fit_impl(h, X, C0, max_iter, tol, labels, centroids, sse, iters);
}

int kmeans_assign(kmeans_handle h, const void* X, int64_t m, int32_t* labels, double* sse) {
    if (!h) return KMEANS_EINVAL;
    if (!X || !labels || m < 1) return fail(h, KMEANS_EINVAL, "X, labels and m >= 1 required");
    if (!h->have_centroids) return fail(h, KMEANS_EINVAL, "no centroids: fit or set them first");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    double total = 0.0;
    const bool lab_dev = is_device_ptr(labels);
    if (int rc = prep_centroids(h)) return rc;
    CK(cudaMemsetAsync(h->n_low_dev, 0, sizeof(unsigned long long), s));
    for (int64_t r0 = 0; r0 < m; r0 += h->n) {
        int64_t rows = std::min<int64_t>(h->n, m - r0);
        const char* src = (const char*)X + (size_t)r0 * h->d * h->wsize;
        const bool norm = h->norm != KMEANS_NORM_NONE;
        const void* Xsrc = h->Xw;
        if (norm && is_device_ptr(src)) Xsrc = src;      // normalised out of place, no copy
        else if (int rc = stage_rows(h, src, rows, h->Xw)) return rc;
        if (prep_fast_ok(h->work, h->d)) {
            CK(launch_prep_fast(h->dist, Xsrc, rows, h->d, h->d_pad, h->guard, h->xn, h->sx,
                                h->Xl, nullptr, norm ? h->Xw : nullptr, norm ? h->shift : nullptr,
                                norm ? h->scale : nullptr, s));
        } else {
            if (norm) CK(launch_norm_apply(h->work, h->Xw, rows, h->d, h->shift, h->scale, s, Xsrc));
            CK(launch_prep(h->work, h->dist, h->Xw, rows, h->d, h->d_pad, h->guard, h->xn, h->sx,
                           h->Xl, nullptr, s));
        }
        CK(cudaMemsetAsync(h->sse_dev, 0, sizeof(double), s));
        if (h->dist_kernel == DK_SMALLD && h->delta <= 0.0) {
            Problem p{rows, h->d, h->k, h->d_pad, h->guard};
            CK(launch_assign_simt(h->work, h->dist, p, h->Xl, h->xn, h->guard ? h->sx : nullptr,
                                  h->Cl, h->cn, h->guard ? h->sc : nullptr, h->labels,
                                  h->sse_dev, nullptr, s));
        } else {
            if (int rc = run_assign(h, rows, h->sse_dev, nullptr)) return rc;
        }
        double part = 0.0;
        CK(cudaMemcpyAsync(&part, h->sse_dev, sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaMemcpyAsync(labels + r0, h->labels, (size_t)rows * sizeof(int32_t),
                           lab_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        total += part;
    }
    if (sse) *sse = total;
    // distance counts of this assign (kmeans_stats.n_dist / n_dist_low)
    unsigned long long n_low_h = 0;
    CK(cudaMemcpy(&n_low_h, h->n_low_dev, sizeof(n_low_h), cudaMemcpyDeviceToHost));
    h->last_n_dist = m * (int64_t)h->k;
    h->last_n_low = h->delta > 0.0 ? (int64_t)n_low_h : h->last_n_dist;
    h->stats.n_dist = h->last_n_dist;
    h->stats.n_dist_low = h->last_n_low;
    h->stats.eta = h->last_n_dist > 0 ? (double)h->last_n_low / (double)h->last_n_dist : 1.0;
    h->stats.dist_kernel = h->dist_kernel;
    h->stats.tc_variant =
        (h->dist_kernel == DK_TCGEN05 && h->delta <= 0.0) ? tc_plan_kind(h->tc) : 0;
    return KMEANS_OK;
}

int kmeans_set_centroids(kmeans_handle h, const void* C) {
    if (!h) return KMEANS_EINVAL;
    if (!C) return fail(h, KMEANS_EINVAL, "C is NULL");
    CK(cudaSetDevice(h->device));
    if (int rc = stage_rows(h, C, h->k, h->Cw)) return rc;
    CK(cudaStreamSynchronize(h->stream));
    h->have_centroids = true;
    return KMEANS_OK;
}

int kmeans_get_centroids(kmeans_handle h, void* C) {
    if (!h) return KMEANS_EINVAL;
    if (!C) return fail(h, KMEANS_EINVAL, "C is NULL");
    CK(cudaMemcpyAsync(C, h->Cw, (size_t)h->k * h->d * h->wsize,
                       is_device_ptr(C) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    return KMEANS_OK;
}

int kmeans_get_transform(kmeans_handle h, void* shift, void* scale) {
    if (!h) return KMEANS_EINVAL;
    std::vector<double> a(h->d), b(h->d);
    CK(cudaMemcpyAsync(a.data(), h->shift, sizeof(double) * h->d, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaMemcpyAsync(b.data(), h->scale, sizeof(double) * h->d, cudaMemcpyDeviceToHost,
                       h->stream));
    CK(cudaStreamSynchronize(h->stream));
    for (int t = 0; t < h->d; ++t) {
        if (h->work == KMEANS_FP64) {
            if (shift) ((double*)shift)[t] = a[t];
            if (scale) ((double*)scale)[t] = b[t];
        } else {
            if (shift) ((float*)shift)[t] = (float)a[t];
            if (scale) ((float*)scale)[t] = (float)b[t];
        }
    }
    return KMEANS_OK;
}

int kmeans_get_stats(kmeans_handle h, kmeans_stats* out) {
    if (!h || !out) return KMEANS_EINVAL;
    *out = h->stats;
    return KMEANS_OK;
}

int kmeans_set_stream(kmeans_handle h, void* stream) {
    if (!h) return KMEANS_EINVAL;
    h->stream = stream ? (cudaStream_t)stream : h->own_stream;
    return KMEANS_OK;
}

int kmeans_set_timing(kmeans_handle h, int enable) {
    if (!h) return KMEANS_EINVAL;
    h->timing = enable;
    return KMEANS_OK;
}

int kmeans_seed_d2(kmeans_handle h, const void* X, const double* u, int64_t* indices) {
    if (!h) return KMEANS_EINVAL;
    if (!X || !u || !indices) return fail(h, KMEANS_EINVAL, "X, u and indices are required");
    if (h->comm) return fail(h, KMEANS_EINVAL, "kmeans_seed_d2 runs on single-GPU handles");
    CK(cudaSetDevice(h->device));
    cudaStream_t s = h->stream;
    const int64_t n = h->n;
    const int k = h->k;
    for (int j = 0; j < k; ++j)
        if (!(u[j] >= 0.0 && u[j] < 1.0))
            return fail(h, KMEANS_EINVAL, "the uniforms u must lie in [0, 1)");
    if (int rc = prepare_points(h, X)) return rc;
    // scratch: D2 (n), block sums, u, indices, warning flag
    double* D2 = nullptr;
    double* ps = nullptr;
    double* u_dev = nullptr;
    int64_t* idx_dev = nullptr;
    int* warn_dev = nullptr;
    const int64_t nb = seed_blocks(n);
    CK(cudaMallocAsync((void**)&D2, (size_t)n * sizeof(double), s));
    CK(cudaMallocAsync((void**)&ps, (size_t)nb * sizeof(double), s));
    CK(cudaMallocAsync((void**)&u_dev, (size_t)k * sizeof(double), s));
    CK(cudaMallocAsync((void**)&idx_dev, (size_t)k * sizeof(int64_t), s));
    CK(cudaMallocAsync((void**)&warn_dev, sizeof(int), s));
    CK(cudaMemcpyAsync(u_dev, u, (size_t)k * sizeof(double), cudaMemcpyHostToDevice, s));
    int64_t first = (int64_t)(u[0] * (double)n);   // Alg 1 line 1 (reading R6)
    if (first > n - 1) first = n - 1;
    CK(cudaMemcpyAsync(idx_dev, &first, sizeof(int64_t), cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(warn_dev, 0, sizeof(int), s));
    CK(launch_seed_d2(h->work, h->dist, h->Xl, n, h->d, h->d_pad, h->xn, h->sx, h->guard, k,
                      u_dev, idx_dev, D2, ps, warn_dev, s));
    int warn = 0;
    CK(cudaMemcpyAsync(indices, idx_dev, (size_t)k * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&warn, warn_dev, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    cudaFreeAsync(D2, s);
    cudaFreeAsync(ps, s);
    cudaFreeAsync(u_dev, s);
    cudaFreeAsync(idx_dev, s);
    cudaFreeAsync(warn_dev, s);
    CK(cudaStreamSynchronize(s));
    return warn ? KMEANS_WARN_SEED_UNIFORM : KMEANS_OK;
}

int kmeans_set_delta(kmeans_handle h, double delta) {
    if (!h) return KMEANS_EINVAL;
    if (!(delta == 0.0 || (delta >= 1.0 && std::isfinite(delta))))
        return fail(h, KMEANS_EINVAL, "delta must be 0 (off) or a finite value >= 1");
    h->delta = delta;
    // Alg 4 lines 1-5: the triggered pairs use the infinity-norm scaled operands
    h->guard = delta > 0.0 ? (h->guard_user ? h->guard_user : 1) : h->guard_user;
    return KMEANS_OK;
}

int kmeans_destroy(kmeans_handle h) {
    if (!h) return KMEANS_OK;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    free_all(h);
    delete h;
    return KMEANS_OK;
}

const char* kmeans_last_error(kmeans_handle h) {
    if (!h) return g_create_err.c_str();
    return h->err.c_str();
}

int kmeans_cast(int src_prec, int dst_prec, const void* src, int64_t count, void* dst) {
    kmeans_ctx* h = nullptr;
    if ((src_prec != KMEANS_FP64 && src_prec != KMEANS_FP32) || dst_prec < KMEANS_FP32 ||
        dst_prec > KMEANS_E5M2 || count < 0 || (count > 0 && (!src || !dst)))
        return fail(nullptr, KMEANS_EINVAL, "kmeans_cast: bad arguments");
    if (count > 0 && (!is_device_ptr(src) || !is_device_ptr(dst)))
        return fail(nullptr, KMEANS_EINVAL, "kmeans_cast: src and dst must be device pointers");
    CK(launch_cast(src_prec, dst_prec, src, count, dst, 0));
    CK(cudaStreamSynchronize(0));
    return KMEANS_OK;
}

const char* kmeans_version(void) { return "mpkmeans-b200 0.1 (sm_100a)"; }

}  // extern "C"
