/*
 * kmeans.h — C ABI of the B200-native mixed-precision Lloyd k-means hot path.
 *
 * Method: Carson, Chen & Liu, "Computing k-means in mixed precision" (arXiv 2407.12208),
 * /root/reference/PAPER.md. The library implements Algorithm 3 (mixed-precision k-means
 * framework) steps 2-7 with the initial centroids C0 supplied by the caller:
 *   step 3  assignment with the expanded distance  ||x||^2 - 2 x.c + ||c||^2  (eq:dist-eval,
 *           PAPER.md:193-196) whose dot products run in the low precision u_l (fp16, bf16 or
 *           q52 = OCP FP8 E5M2) with fp32 accumulation, fused with the argmin;
 *   step 4  centroid update mu_j = (1/|S_j|) sum_{x in S_j} x (eq:center) in
 *           the working precision u (fp32 or fp64). fp32 work: the sums are exact integer totals
 *           on a per-feature grid (2^-45 of the feature's max |x|), updated from the rows whose
 *           label changed, so mu_j = round_u(exact mean) up to that grid and depends only on
 *           S_j (bit-reproducible, also across ranks); fp64 work: fp64 sums in a fixed order
 *           (R7, R9);
 *   step 6  stop at max_iter or when the cluster sets converge;
 *   step 7  final assignment "computed in precision u".
 * Optional: z-score (eq:z-norm) or min-max (image /255)
 * normalisation first, and Algorithm 4's infinity-norm operand scaling as the
 * low-precision overflow guard.
 *
 * Layout: every matrix is row-major and contiguous: X is n x d (one point per row; the paper's
 * P = X^T), centroids are k x d. Elements of X, C0 and centroids have the WORKING
 * precision's type (double for KMEANS_FP64, float for KMEANS_FP32). Labels are int32.
 *
 * Memory: pointers may be host or device (CUDA) pointers; the library detects which with
 * cudaPointerGetAttributes and copies as needed. The caller owns every buffer it passes; the
 * library owns everything it allocates (sized at create time from n, d, k) until destroy.
 * Calls are blocking: outputs are valid when the call returns. A handle is not thread-safe;
 * distinct handles are independent. No call ever falls back to a CPU implementation.
 *
 * Errors: 0 = OK; < 0 = error, nothing written to outputs, message via kmeans_last_error;
 * > 0 = bitmask of KMEANS_WARN_* (results valid).
 */
#ifndef MPKMEANS_KMEANS_H
#define MPKMEANS_KMEANS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct kmeans_ctx* kmeans_handle;

/* Precisions (Table 1; bf16 added by the build). */
enum kmeans_precision {
    KMEANS_FP64 = 0, /* u = 2^-53 */
    KMEANS_FP32 = 1, /* u = 2^-24 */
    KMEANS_FP16 = 2, /* u = 2^-11 */
    KMEANS_BF16 = 3, /* u = 2^-8  */
    KMEANS_E5M2 = 4  /* u = 2^-3; the paper's quarter precision q52 */
};

/* Normalisation modes and flags (OR-able). */
enum kmeans_flags {
    KMEANS_NORM_NONE = 0,
    KMEANS_NORM_MINMAX = 1,   /* (x - min) / (max - min) per feature; range 0 -> 1          */
    KMEANS_NORM_ZSCORE = 2,   /* (x - mean) / std per feature (population std); std 0 -> 1 */
    KMEANS_GUARD_SCALE = 0x100,
    /* Alg 4 lines 1-5: every point and centroid is divided by its own
       infinity norm (zero vector -> 1) in precision u before rounding to u_l, and the dot
       product is rescaled by s_i * s_j (Alg 4 line 6). Applied to all pairs (delta = 1). */
    KMEANS_FORCE_SIMT = 0x200,
    /* Debug/parity: use the CUDA-core distance kernel even where the tcgen05 kernel applies. */
    KMEANS_GUARD_POW2 = 0x400
    /* Alg 4's scaling with s = 2^ceil(log2 ||x||_inf) (reading Z9 B; implies GUARD_SCALE): the
       division by s is exact, so x~ = round_l(x / s) differs from round_l(x) only where x / s
       is kept out of the low format's subnormal / overflow range. With the row as one block it
       is an MX (OCP microscaling, UE8M0) block scale; the remedy the survey proposed for the
       paper's q52 failures. */
};

enum kmeans_status {
    KMEANS_OK = 0,
    KMEANS_EINVAL = -1,
    KMEANS_ENOMEM = -2,
    KMEANS_ECUDA = -3,
    KMEANS_ENCCL = -4,
    KMEANS_ENODEV = -5,              /* no sm_100 device: the library never falls back to CPU */
    KMEANS_WARN_NONFINITE = 1,       /* a low-precision cast produced +-inf / NaN (overflow)  */
    KMEANS_WARN_EMPTY = 2,           /* some cluster was empty in some iteration (kept)       */
    KMEANS_WARN_MAXITER = 4,         /* tol >= 0 and max_iter reached without convergence     */
    KMEANS_WARN_UNDERFLOW = 8,       /* a nonzero value rounded to zero or a subnormal in u_l  */
    KMEANS_WARN_SEED_UNIFORM = 16    /* kmeans_seed_d2: a round had sum D^2 = 0 or non-finite
                                        and drew uniformly                        */
};

/* Per-fit observability (filled by kmeans_get_stats after kmeans_fit). */
#define KMEANS_MAX_TRACE 1024
typedef struct kmeans_stats {
    int32_t iters;                       /* iterations run (assign + update pairs)          */
    int32_t converged;                   /* 1 if stopped by a convergence test              */
    int32_t warnings;                    /* KMEANS_WARN_* bitmask of the last fit           */
    int32_t dist_kernel;                 /* 0 = SIMT fp64/fp32, 1 = SIMT low, 2 = tcgen05,
                                            3 = small-d fused                               */
    int64_t n_nonfinite;                 /* low-precision operands that became +-inf/NaN    */
    int64_t n_underflow;                 /* nonzero operands rounded to zero/subnormal      */
    double t_prep_ms, t_loop_ms, t_final_ms;        /* CUDA-event times of the last fit     */
    double t_dist_ms, t_update_ms, t_finalize_ms, t_allreduce_ms; /* summed over iterations */
    int32_t n_dist_launches;             /* distance-kernel launches in the loop            */
    int32_t trace_len;                   /* min(iters, KMEANS_MAX_TRACE)                    */
    double sse_t[KMEANS_MAX_TRACE];      /* per-iteration SSE_t = sum_i max(0, min_j D_ij)   */
    double shift2_t[KMEANS_MAX_TRACE];   /* ||C_{t+1} - C_t||_F^2                            */
    int64_t changed_t[KMEANS_MAX_TRACE]; /* labels that changed in iteration t              */
    int32_t empty_t[KMEANS_MAX_TRACE];   /* empty clusters in iteration t                   */
    int64_t n_kernel_launches;           /* kernels this library launched during the fit    */
    int64_t n_final_fallback;            /* final-pass rows re-evaluated on CUDA cores over all
                                            k centroids (-1: all rows)                     */
    int64_t n_final_uncertified;         /* final-pass rows the tensor-core filter could not
                                            certify; those with at most 32 candidate columns
                                            are resolved by exact fp32 evaluation of the
                                            candidates only (R2)                 */
    int64_t n_dist;                      /* distances formed by the last fit's loop
                                            (iters * n * k) or by the last kmeans_assign     */
    int64_t n_dist_low;                  /* of which in low precision: all of them unless
                                            kmeans_set_delta is on (then eq:xi-low-prec-ratio's
                                            eta = n_dist_low / n_dist)     */
    double u_bound_t[KMEANS_MAX_TRACE];  /* Thm 5.3 (eq:center-update-prec):
                                            min over the clusters that moved in iteration t of
                                            |c^-mu^|^T|c^-mu^| / (2 |c^-mu^|^T |mu^|), the
                                            largest unit roundoff of the centre update that
                                            still cannot stall the iteration (+inf: none moved)*/
    int32_t n_update_prec_short;         /* iterations with u_bound_t below the working
                                            precision's unit roundoff (2^-24 / 2^-53)          */
    int32_t tc_variant;                  /* tcgen05 kernel of the loop: 0 = none (CUDA cores),
                                            1 = streaming centroid tiles (k_assign_tc.cu),
                                            2 = CTA pair with resident centroids (k_assign_tc2) */
    int32_t n_ranks;                     /* ranks of the fit (1, or the NCCL / virtual group)  */
    double eta;                          /* n_dist_low / n_dist (eq:xi-low-prec-ratio,
                                            PAPER.md:666-668); 1 without kmeans_set_delta     */
} kmeans_stats;

/*
 * kmeans_create — allocate a handle for n points of dimension d and k clusters.
 *   work_prec in {FP64, FP32}; dist_prec in {FP64, FP32, FP16, BF16, E5M2} with
 *   0 < u <= u_l: FP64 work allows every dist; FP32 work allows all but FP64.
 *   dist_prec == work_prec is the working-precision k-means (Alg 2 with C0 given);
 *   lower dist_prec is mp_k-means++_low (Alg 3).
 *   flags = one KMEANS_NORM_* | optional KMEANS_GUARD_SCALE | optional KMEANS_FORCE_SIMT.
 * Errors: EINVAL if n < 1, d < 1, k < 1, k > n, an unknown enum, or a NULL out; ENODEV without
 * an sm_100 GPU; ENOMEM if device allocations fail. The current CUDA device at call time is the
 * device the handle uses for its lifetime.
 */
int kmeans_create(int64_t n, int32_t d, int32_t k, int work_prec, int dist_prec, int flags,
                  kmeans_handle* out);

/*
 * kmeans_fit — Alg 3 steps 2-7 from C0.
 *   X: n x d working-precision points (host or device). C0: k x d initial centroids.
 *   max_iter >= 1. tol >= 0: stop when no label changed or ||C_{t+1} - C_t||_F <= tol;
 *   tol < 0: run exactly max_iter iterations (bench mode).
 *   Outputs (any may be NULL except sse's target when non-NULL is wanted): labels[n] of the final
 *   working-precision assignment (Alg 3 step 7), centroids k x d (working type), *sse = the
 *   final SSE (eq:sse via the direct formula eq:dist-eval-alternative, PAPER.md:189-192,
 *   accumulated in fp64), *iters = iterations run.
 *   With normalisation on, X and C0 are in original coordinates and the centroids and SSE are
 *   returned in the normalised space (as the paper's "(normalized)" columns);
 *   kmeans_get_transform gives the map.
 * Returns 0, a KMEANS_WARN_* mask, or an error.
 */
int kmeans_fit(kmeans_handle h, const void* X, const void* C0, int32_t max_iter, double tol,
               int32_t* labels, void* centroids, double* sse, int32_t* iters);

/*
 * kmeans_assign — the standalone distance + argmin kernel in dist_prec with the handle's current
 * centroids (after a fit or kmeans_set_centroids; EINVAL before either). X: m x d working
 * precision points in ORIGINAL coordinates (the handle's stored transform is applied), any m >= 1
 * (processed in chunks of at most n rows). labels[m] receives argmin_j of the expanded distance
 * (lowest j on ties, NaN never selected). If sse != NULL, *sse = sum_i max(0, min_j D_ij).
 */
int kmeans_assign(kmeans_handle h, const void* X, int64_t m, int32_t* labels, double* sse);

/* kmeans_set_centroids — overwrite the handle's centroids (k x d, working type, normalised
 * space). kmeans_get_centroids — read them back. */
int kmeans_set_centroids(kmeans_handle h, const void* C);
int kmeans_get_centroids(kmeans_handle h, void* C);

/* kmeans_get_transform — shift[d], scale[d] (working type) of the last fit's normalisation:
 * x_normalised = round_u((x - shift) / scale). Identity (0, 1) without normalisation. */
int kmeans_get_transform(kmeans_handle h, void* shift, void* scale);

/* kmeans_get_stats — copy the last fit's statistics (see kmeans_stats): the per-iteration
 * traces of Alg 3's loop (SSE_t of eq:sse PAPER.md:130-133, the shift and changed counts of the
 * stopping rule PAPER.md:549, Thm 5.3's bound PAPER.md:487-493), eta of eq:xi-low-prec-ratio
 * and timings. EINVAL on a NULL handle or out. */
int kmeans_get_stats(kmeans_handle h, kmeans_stats* out);

/* kmeans_set_stream — run all of the handle's work on this cudaStream_t (NULL = the handle's
 * own stream). The caller keeps ownership of the stream. Plumbing only: no passage of the paper
 * (which runs on one CPU thread) defines streams. EINVAL on a NULL handle. */
int kmeans_set_stream(kmeans_handle h, void* cuda_stream);

/* kmeans_seed_d2 — seeding by D^2 weighting (Alg 1) with the distances of
 * Alg 3 step 1 in the low precision, on the handle's n rows of X (same
 * normalisation and operands as kmeans_fit; X host or device, work dtype, n x d). u: k uniforms
 * in [0, 1) (host), the method's random draws. indices (host, int64[k], out): the chosen rows,
 * distinct. The draw is DESIGN.md reading R6: first index floor(u_0 n); then the inverse-CDF
 * draw of Alg 1 line 2's law, the first index whose running sum of the weights D^2 exceeds
 * u_j * sum (D^2: min over the chosen centres of O4's expanded formula from the stored low
 * operands, fp32-accumulated dots, floored at 0; a chosen centre's own weight 0; the sums in a
 * fixed parallel order). Pass the rows X[indices] as C0 to kmeans_fit for Alg 3 / Alg 5 end to
 * end. Single-GPU handles only. Returns 0, KMEANS_WARN_SEED_UNIFORM (a round whose sum was 0 or
 * non-finite drew floor(u_j n)), or an error (u outside [0, 1): KMEANS_EINVAL).              */
int kmeans_seed_d2(kmeans_handle h, const void* X, const double* u, int64_t* indices);

/* kmeans_set_delta — Alg 4 / Alg 5: per point-centroid pair, the
 * distance of the Lloyd loop (and of kmeans_assign) uses the low precision only when
 * eq:prec-delta holds, max(x^T x / c^T c, c^T c / x^T x) >= delta^2 (evaluated division-free in
 * fp64: max(xn, cn) >= delta^2 min(xn, cn)), with Alg 4's infinity-norm operand scaling, and the
 * working precision otherwise. delta = 1 makes every pair low precision (Alg 3 with scaling);
 * delta = 0 turns the switch off (the default: every pair low precision, scaling as created).
 * With fp32 work and fp16/bf16 operands on the tcgen05 path it runs as a certified tensor-core
 * filter plus exact per-pair evaluation of the candidate columns of uncertified rows (DESIGN.md
 * R10: the labels of the per-pair evaluation); otherwise on CUDA cores (both dots per pair).
 * The number of low-precision pairs is in kmeans_stats.n_dist_low (and eta). Returns
 * KMEANS_EINVAL unless delta == 0 or 1 <= delta < inf.                                      */
int kmeans_set_delta(kmeans_handle h, double delta);

/* kmeans_set_timing — 1 = record CUDA events around every kernel of the loop (per-kernel times
 * in kmeans_stats), 0 = only the prep / loop / final events (default). */
int kmeans_set_timing(kmeans_handle h, int enable);

/* kmeans_destroy — free the handle (NULL is a no-op returning 0). */
int kmeans_destroy(kmeans_handle h);

/* kmeans_last_error — handle-local message for the last nonzero return (NULL handle: the
 * message of the last failed kmeans_create on this thread). Never NULL. */
const char* kmeans_last_error(kmeans_handle h);

/*
 * kmeans_cast — the operand-rounding kernel on its own (Table 1 formats):
 * dst[i] = round_{dst_prec}(src[i]) with one round-to-nearest-even step from the source value,
 * gradual underflow, and IEEE overflow to +-inf (never saturation). src_prec in {FP64, FP32},
 * dst_prec in {FP32, FP16, BF16, E5M2} (element sizes 4, 2, 2, 1 bytes). src and dst must be
 * DEVICE pointers to count elements. Returns 0 or an error.
 */
int kmeans_cast(int src_prec, int dst_prec, const void* src, int64_t count, void* dst);

/*
 * kmeans_create_dist — like kmeans_create for one rank of a point-sharded run (the
 * paper has parallel k-means only as related work): this rank holds n_local
 * rows; all ranks hold the same C0. nccl_unique_id points to the 128-byte ncclUniqueId created
 * by rank 0 and broadcast by the caller (nranks = 1 with an id still builds a 1-rank NCCL
 * communicator, so every collective call site runs). Per Lloyd iteration the ranks combine
 * their shard's share of eq:center: with fp32 work, the exact fixed-point
 * totals (two int64 k x d arrays) and the int32 counts in one NCCL group of three allreduces
 * (integer sums: exact and order-free) plus one fp64 allreduce of [SSE_t, #changed]; with fp64
 * work, one fp64 allreduce of the packed [sums | counts | SSE_t | #changed]. Every rank then
 * finalises identical centroids. Once per fit: the normalisation statistics (eq:z-norm,
 * PAPER.md:119-126) and the fixed-point grid (a max-allreduce); at the end the final SSE.
 * kmeans_fit must be called collectively; X/labels are the local shard; centroids, sse and iters
 * are identical on every rank (sse is global). Errors: EINVAL on a NULL id with nranks > 1 or a
 * bad rank; ENCCL if the communicator cannot be built.
 */
int kmeans_create_dist(int64_t n_local, int32_t d, int32_t k, int work_prec, int dist_prec,
                       int flags, const void* nccl_unique_id, int nranks, int rank,
                       kmeans_handle* out);

/*
 * Virtual ranks — the point-sharded path of kmeans_create_dist with g ranks inside ONE process
 * on ONE GPU (a test / validation transport; SURVEY §4 "fake multi-GPU"). kmeans_vgroup_create
 * makes a group of nranks (1..64) on the current device; kmeans_create_virtual makes rank
 * `rank`'s handle for its n_local-row shard (same arguments and semantics as
 * kmeans_create_dist). Each rank's kmeans_fit must run on its OWN host thread, all ranks
 * collectively, exactly like one process per GPU: every per-rank step is the NCCL path's code;
 * at each collective the last rank to arrive sums the ranks' buffers on the device in rank
 * order. The ranks' kernels are serialised on one stream of the group (they never wait on each
 * other on the device). kmeans_vgroup_destroy returns EINVAL while handles of the group live.
 */
typedef struct kmeans_vgroup_s* kmeans_vgroup;
int kmeans_vgroup_create(int nranks, kmeans_vgroup* out);
int kmeans_create_virtual(int64_t n_local, int32_t d, int32_t k, int work_prec, int dist_prec,
                          int flags, kmeans_vgroup group, int rank, kmeans_handle* out);
int kmeans_vgroup_destroy(kmeans_vgroup group);

/* kmeans_nccl_unique_id — write a fresh 128-byte ncclUniqueId (call on rank 0 only). */
int kmeans_nccl_unique_id(void* out128);

/* kmeans_version — library version string. */
const char* kmeans_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MPKMEANS_KMEANS_H */
