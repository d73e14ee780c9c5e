/*
 * mpkmeans_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously-correct CPU implementation of the mixed-precision Lloyd iteration of
 * Carson, Chen & Liu, "Computing k-means in mixed precision" (arXiv 2407.12208), written from
 * /root/reference/PAPER.md. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load it. The CUDA product path never calls, links or includes it,
 * and it shares no code, header, table or constant generator with the CUDA path.
 *
 * Arithmetic: everything is fp64. Values that the method STORES in a precision (working
 * precision u, low "distance" precision u_l) are passed through oracle_round(fmt, v), a generic
 * single-rounding (round-to-nearest, ties-to-even) map from fp64 to a (t, e_min, e_max) format
 * with gradual underflow and IEEE overflow to +-inf (Table 1; standard model
 * eq:fpmodel PAPER.md:215-219). No BLAS, no blocking, no fusion: loops in the paper's order.
 * OpenMP is used only across independent points (per-point argmin); every sum over points runs
 * sequentially in index order with Neumaier compensation, so results do not depend on threads.
 *
 * Steps (names from SURVEY.md §8c.1; the readings Z1..Z25 are listed in DESIGN.md):
 *   O0 oracle_round           Table 1
 *   O1 normalise              eq:z-norm PAPER.md:119-126 (z-score); image /255 PAPER.md:1166
 *   O2 point prep             p_i^T p_i precomputed PAPER.md:204-205; Alg 4 scaling PAPER.md:619-623
 *   O3 centroid prep          c_j^T c_j recomputed each iteration PAPER.md:206; Alg 4
 *   O4 distance               eq:dist-eval PAPER.md:193-196 (typo c_i^T c_i read as c_j^T c_j);
 *                             Alg 3 step 3 PAPER.md:546; Alg 4 step 6 PAPER.md:624-625
 *   O5 argmin                 Alg 2 step 3 PAPER.md:174
 *   O6 iteration SSE          eq:sse PAPER.md:130-133
 *   O7 update                 eq:center PAPER.md:421-427, in precision u (Alg 3 step 4 PAPER.md:547)
 *   O8 convergence            Alg 2 step 6 PAPER.md:177 / Alg 3 step 6 PAPER.md:549
 *   O9 final assignment       Alg 3 step 7 PAPER.md:550 ("computed in precision u");
 *                             SSE by eq:dist-eval-alternative PAPER.md:189-192
 *   O4m Alg 4 / Alg 5         per-pair precision switch eq:prec-delta PAPER.md:613-645, 684-699
 *   O10 seeding               Alg 1 (D^2 weighting) PAPER.md:150-161 in u_l (Alg 3 step 1)
 *   O11 update precision      Thm 5.3 eq:center-update-prec PAPER.md:487-493
 *
 * Parity pins live in tests/test_oracle_*.py; nothing here is "parity unpinned".
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* precision ids (same numbering as the public C-ABI enums, restated here, not shared) */
enum { OFMT_FP64 = 0, OFMT_FP32 = 1, OFMT_FP16 = 2, OFMT_BF16 = 3, OFMT_E5M2 = 4 };
enum { ONORM_NONE = 0, ONORM_MINMAX = 1, ONORM_ZSCORE = 2, ONORM_MASK = 0xff, OGUARD = 0x100,
       OGUARD_POW2 = 0x400 };

/* ---------------------------------------------------------------------------------------- */
/* O0: formats. Table 1: t = significand digits incl. implicit bit,          */
/* e_min / e_max exponents of x_min / x_max. q52 is read as OCP E5M2 (Z4);     */
/* bf16 is not in the paper (north_star adds it): t = 8, e_min = -126, e_max = 127.          */
/* ---------------------------------------------------------------------------------------- */
int oracle_format_params(int fmt, int* t, int* emin, int* emax) {
    switch (fmt) {
        case OFMT_FP64: *t = 53; *emin = -1022; *emax = 1023; return 0;
        case OFMT_FP32: *t = 24; *emin = -126; *emax = 127; return 0;
        case OFMT_FP16: *t = 11; *emin = -14; *emax = 15; return 0;
        case OFMT_BF16: *t = 8; *emin = -126; *emax = 127; return 0;
        case OFMT_E5M2: *t = 3; *emin = -14; *emax = 15; return 0;
        default: return -1;
    }
}

/* Round an fp64 value once to the nearest value of the format (ties to even significand),   */
/* with subnormals (quantum fixed at 2^(e_min - t + 1) below x_min) and overflow to +-inf iff */
/* |v| >= 2^e_max * (2 - 2^-t), the midpoint between x_max and 2^(e_max+1) (reading Z6).    */
double oracle_round(int fmt, double v) {
    int t, emin, emax;
    if (fmt == OFMT_FP64) return v;
    if (oracle_format_params(fmt, &t, &emin, &emax) != 0) return NAN;
    if (isnan(v) || isinf(v) || v == 0.0) return v;
    double a = fabs(v);
    double overflow_at = ldexp(2.0 - ldexp(1.0, -t), emax);
    if (a >= overflow_at) return copysign(INFINITY, v);
    int ex;
    (void)frexp(a, &ex);             /* a = m * 2^ex, m in [0.5, 1): leading bit exponent ex-1 */
    int e = ex - 1;
    if (e < emin) e = emin;          /* gradual underflow: fixed quantum below x_min */
    double quantum = ldexp(1.0, e - (t - 1));
    double r = nearbyint(a / quantum) * quantum;   /* a / quantum is exact; nearbyint = RNE */
    return copysign(r, v);
}

void oracle_round_array(int fmt, const double* in, double* out, int64_t count) {
    for (int64_t i = 0; i < count; ++i) out[i] = oracle_round(fmt, in[i]);
}

/* Neumaier-compensated accumulator (fixed index order). */
typedef struct { double s, c; } nsum_t;
static inline void nsum_add(nsum_t* a, double x) {
    double t = a->s + x;
    if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x; else a->c += (x - t) + a->s;
    a->s = t;
}
static inline double nsum_get(const nsum_t* a) { return a->s + a->c; }

/* ---------------------------------------------------------------------------------------- */
/* O1: normalisation (one map per feature, applied to X and to C0).                         */
/*   ZSCORE: eq:z-norm PAPER.md:119-126, mu = mean, sigma = population std (two passes),    */
/*           sigma == 0 -> 1 (reading Z17).                                                  */
/*   MINMAX: (x - min) / (max - min); range 0 -> 1. Equals /255 on 0..255-spanning images    */
/*           (PAPER.md:1166).                                                                */
/* Outputs are rounded to working precision.                                                 */
/* ---------------------------------------------------------------------------------------- */
void oracle_normalize_stats(int norm, int64_t n, int d, const double* X, double* shift,
                            double* scale) {
    for (int t = 0; t < d; ++t) {
        if (norm == ONORM_ZSCORE) {
            nsum_t s = {0, 0};
            for (int64_t i = 0; i < n; ++i) nsum_add(&s, X[i * d + t]);
            double mu = nsum_get(&s) / (double)n;
            nsum_t q = {0, 0};
            for (int64_t i = 0; i < n; ++i) {
                double z = X[i * d + t] - mu;
                nsum_add(&q, z * z);
            }
            double sigma = sqrt(nsum_get(&q) / (double)n);
            shift[t] = mu;
            scale[t] = (sigma == 0.0) ? 1.0 : sigma;
        } else if (norm == ONORM_MINMAX) {
            double mn = X[t], mx = X[t];
            for (int64_t i = 1; i < n; ++i) {
                double x = X[i * d + t];
                if (x < mn) mn = x;
                if (x > mx) mx = x;
            }
            shift[t] = mn;
            scale[t] = (mx - mn == 0.0) ? 1.0 : (mx - mn);
        } else {
            shift[t] = 0.0;
            scale[t] = 1.0;
        }
    }
}

void oracle_normalize_apply(int work, int64_t rows, int d, const double* shift,
                            const double* scale, const double* in, double* out) {
    for (int64_t i = 0; i < rows; ++i)
        for (int t = 0; t < d; ++t)
            out[i * d + t] = oracle_round(work, (in[i * d + t] - shift[t]) / scale[t]);
}

/* ---------------------------------------------------------------------------------------- */
/* O2 / O3: norms, guard scale and low-precision operand of one vector.                     */
/*   norm = p^T p, fp64 sequential sum, stored in precision u.            */
/*   guard: s = ||p||_inf (Alg 4 lines 1-2; zero vector -> 1, reading Z10), */
/*          or (guard 2, reading Z9 B) the smallest power of two >= ||p||_inf,                 */
/*          p~ = round_l(round_u(p / s)) (Alg 4 lines 4-5 in precision u, then the operand of */
/*          the low-precision dot, line 6).                                                  */
/*   no guard: s = 1, p~ = round_l(p).                                                       */
/* ---------------------------------------------------------------------------------------- */
static void prep_vector(int work, int dist, int guard, int d, const double* p, double* norm,
                        double* s, double* p_low) {
    double acc = 0.0;
    for (int t = 0; t < d; ++t) acc += p[t] * p[t];
    *norm = oracle_round(work, acc);
    double sc = 1.0;
    if (guard && dist != work) {
        double m = 0.0;
        for (int t = 0; t < d; ++t) if (fabs(p[t]) > m) m = fabs(p[t]);
        sc = (m == 0.0 || isnan(m)) ? 1.0 : m;
        if (guard == 2 && sc != 1.0 && isfinite(sc)) {
            int e;
            double f = frexp(sc, &e);          /* sc = f 2^e, f in [0.5, 1) */
            double up = (f == 0.5) ? sc : ldexp(1.0, e);
            if (isfinite(up) && (work != OFMT_FP32 || up <= 3.4028234663852886e38)) sc = up;
        }
    }
    *s = sc;
    for (int t = 0; t < d; ++t) {
        double q = (sc == 1.0) ? p[t] : oracle_round(work, p[t] / sc);
        p_low[t] = oracle_round(dist, q);
    }
}

/* ---------------------------------------------------------------------------------------- */
/* O4 + O5 for one point against all centroids.                                             */
/*   D_ij = x_i^T x_i - 2 s_i s_j (x~_i^T c~_j) + c_j^T c_j  (eq:dist-eval, Alg 4 line 6)    */
/*   The dot product of the low-precision operands is accumulated in fp64 ("exact            */
/*   accumulation": every product of two fp16/bf16/E5M2/fp32 values is exact in fp64).       */
/*   argmin: scan j = 0..k-1, strict '<' from best = +inf, label 0: lowest index on ties,     */
/*   NaN never wins, an all-NaN/+inf row keeps label 0 (readings Z12, Z13).                  */
/* O4m (Alg 4; used by Alg 5 step 3), when delta2 = delta^2  */
/* is > 0: per pair, condition eq:prec-delta                              */
/*     max(x^T x / c^T c, c^T c / x^T x) >= delta^2                                          */
/* is evaluated without the division, as max(xn, cn_j) >= delta^2 * min(xn, cn_j) in fp64    */
/* (reading R5; any NaN norm makes it false; xn = cn_j = 0 makes it true). If it holds, D_ij  */
/* is the scaled low-precision formula above (Alg 4 lines 1-6; the scaling s = ||.||_inf is   */
/* always on in this mode); otherwise D_ij = x^T x - 2 x^T c_j + c^T c with the dot product  */
/* of the working-precision values (Alg 4 line 8), accumulated in fp64. *n_trig counts the   */
/* triggered pairs (eq:xi-low-prec-ratio's numerator).                     */
/* ---------------------------------------------------------------------------------------- */
static void assign_point(int d, int k, const double* x, const double* xl, double xn, double sx,
                         const double* C, const double* Cl, const double* cn, const double* sc,
                         double delta2, int64_t* n_trig, int32_t* label, double* dmin,
                         double* d2nd) {
    double best = INFINITY, second = INFINITY;
    int32_t lab = 0;
    int64_t trig_count = 0;
    for (int j = 0; j < k; ++j) {
        int trig = 1;
        if (delta2 > 0.0) {
            const double a = xn, b = cn[j];
            const double mx = (a > b) ? a : b, mn = (a > b) ? b : a;
            trig = mx >= delta2 * mn;
        }
        double D;
        if (trig) {
            double dot = 0.0;
            for (int t = 0; t < d; ++t) dot += xl[t] * Cl[(int64_t)j * d + t];
            D = xn - 2.0 * (sx * sc[j]) * dot + cn[j];
            trig_count++;
        } else {
            double dot = 0.0;
            for (int t = 0; t < d; ++t) dot += x[t] * C[(int64_t)j * d + t];
            D = xn - 2.0 * dot + cn[j];
        }
        if (D < best) { second = best; best = D; lab = j; }
        else if (D < second) second = D;
    }
    *label = lab;
    *dmin = best;
    if (d2nd) *d2nd = second;
    if (n_trig) *n_trig = trig_count;
}

/* Handle-free state for one run. */
typedef struct {
    int64_t n; int d, k, work, dist, guard;
    double delta2;                /* Alg 4's delta^2; 0: every pair in low precision (Alg 3)  */
    double *X, *Xl, *xn, *sx;     /* normalised X (work), low operands, norms, scales */
    double *C, *Cl, *cn, *sc;     /* centroids (work), low operands, norms, scales   */
} ostate_t;

static void prep_points(ostate_t* S) {
    for (int64_t i = 0; i < S->n; ++i)
        prep_vector(S->work, S->dist, S->guard, S->d, S->X + i * S->d, &S->xn[i], &S->sx[i],
                    S->Xl + i * S->d);
}
static void prep_centroids(ostate_t* S) {
    for (int j = 0; j < S->k; ++j)
        prep_vector(S->work, S->dist, S->guard, S->d, S->C + (int64_t)j * S->d, &S->cn[j],
                    &S->sc[j], S->Cl + (int64_t)j * S->d);
}

static int64_t assign_all(ostate_t* S, int32_t* labels, double* dmin, double* d2nd) {
    int64_t n = S->n, trig = 0;
#pragma omp parallel for schedule(static) reduction(+ : trig)
    for (int64_t i = 0; i < n; ++i) {
        int64_t t = 0;
        assign_point(S->d, S->k, S->X + i * S->d, S->Xl + i * S->d, S->xn[i], S->sx[i], S->C,
                     S->Cl, S->cn, S->sc, S->delta2, &t, &labels[i], &dmin[i],
                     d2nd ? &d2nd[i] : NULL);
        trig += t;
    }
    return trig;
}

/* O7: sums (compensated fp64 in index order), counts, means rounded to u; empty -> keep.     */
/* O11: Thm 5.3 (eq:center-update-prec) for one update: over the clusters   */
/* whose centre moved, min of |c^ - mu^|^T |c^ - mu^| / (2 |c^ - mu^|^T |mu^|) with c^ the     */
/* previous and mu^ the new (computed) centre; +inf when no centre moved.                      */
static double center_update_bound(int k, int d, const double* Cprev, const double* Cnew) {
    double best = INFINITY;
    for (int j = 0; j < k; ++j) {
        double num = 0.0, den = 0.0;
        for (int t = 0; t < d; ++t) {
            double df = Cprev[(int64_t)j * d + t] - Cnew[(int64_t)j * d + t];
            num += df * df;
            den += fabs(df) * fabs(Cnew[(int64_t)j * d + t]);
        }
        if (num > 0.0 && den > 0.0) {
            double b = num / (2.0 * den);
            if (b < best) best = b;
        }
    }
    return best;
}

static void update_centroids(ostate_t* S, const int32_t* labels, double* sums_out,
                             int64_t* counts_out, double* shift2, int* n_empty) {
    int d = S->d, k = S->k;
    nsum_t* acc = (nsum_t*)calloc((size_t)k * d, sizeof(nsum_t));
    int64_t* cnt = (int64_t*)calloc((size_t)k, sizeof(int64_t));
    for (int64_t i = 0; i < S->n; ++i) {
        int j = labels[i];
        cnt[j] += 1;
        for (int t = 0; t < d; ++t) nsum_add(&acc[(int64_t)j * d + t], S->X[i * d + t]);
    }
    nsum_t sh = {0, 0};
    int empty = 0;
    for (int j = 0; j < k; ++j) {
        if (counts_out) counts_out[j] = cnt[j];
        if (cnt[j] == 0) empty++;
        for (int t = 0; t < d; ++t) {
            double s = nsum_get(&acc[(int64_t)j * d + t]);
            if (sums_out) sums_out[(int64_t)j * d + t] = s;
            double old = S->C[(int64_t)j * d + t];
            double nw = (cnt[j] > 0) ? oracle_round(S->work, s / (double)cnt[j]) : old;
            double df = nw - old;
            nsum_add(&sh, df * df);
            S->C[(int64_t)j * d + t] = nw;
        }
    }
    *shift2 = nsum_get(&sh);
    *n_empty = empty;
    free(acc);
    free(cnt);
}

/* O9: final assignment with the working-precision operands (no rounding to u_l) evaluated in */
/* fp64 (expanded formula, Alg 3 step 7), and SSE by the direct formula (compensated).       */
static double final_pass(ostate_t* S, int32_t* labels) {
    int64_t n = S->n;
    int d = S->d, k = S->k;
    double* cn = (double*)malloc(sizeof(double) * k);
    for (int j = 0; j < k; ++j) {
        double a = 0.0;
        for (int t = 0; t < d; ++t) a += S->C[(int64_t)j * d + t] * S->C[(int64_t)j * d + t];
        cn[j] = oracle_round(S->work, a);
    }
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        const double* x = S->X + i * d;
        double xn = 0.0;
        for (int t = 0; t < d; ++t) xn += x[t] * x[t];
        xn = oracle_round(S->work, xn);
        double best = INFINITY;
        int32_t lab = 0;
        for (int j = 0; j < k; ++j) {
            double dot = 0.0;
            for (int t = 0; t < d; ++t) dot += x[t] * S->C[(int64_t)j * d + t];
            double D = xn - 2.0 * dot + cn[j];
            if (D < best) { best = D; lab = j; }
        }
        labels[i] = lab;
    }
    nsum_t sse = {0, 0};
    for (int64_t i = 0; i < n; ++i) {
        const double* x = S->X + i * d;
        const double* c = S->C + (int64_t)labels[i] * d;
        double acc = 0.0;
        for (int t = 0; t < d; ++t) { double df = x[t] - c[t]; acc += df * df; }
        nsum_add(&sse, acc);
    }
    free(cn);
    return nsum_get(&sse);
}

static int alloc_state(ostate_t* S, int64_t n, int d, int k, int work, int dist, int guard) {
    memset(S, 0, sizeof(*S));
    S->n = n; S->d = d; S->k = k; S->work = work; S->dist = dist; S->guard = guard;
    S->delta2 = 0.0;
    S->X = (double*)malloc(sizeof(double) * n * d);
    S->Xl = (double*)malloc(sizeof(double) * n * d);
    S->xn = (double*)malloc(sizeof(double) * n);
    S->sx = (double*)malloc(sizeof(double) * n);
    S->C = (double*)malloc(sizeof(double) * k * d);
    S->Cl = (double*)malloc(sizeof(double) * k * d);
    S->cn = (double*)malloc(sizeof(double) * k);
    S->sc = (double*)malloc(sizeof(double) * k);
    return (S->X && S->Xl && S->xn && S->sx && S->C && S->Cl && S->cn && S->sc) ? 0 : -2;
}
static void free_state(ostate_t* S) {
    free(S->X); free(S->Xl); free(S->xn); free(S->sx);
    free(S->C); free(S->Cl); free(S->cn); free(S->sc);
}

/* Alg 4 mode: delta >= 1 sets delta^2 and turns the infinity-norm scaling on (Alg 4 lines 1-5);
   delta <= 0 leaves Alg 3 (every pair in low precision, scaling as the flags say). */
static int set_delta(ostate_t* S, double delta) {
    if (delta > 0.0) {
        if (!(delta >= 1.0)) return -1;
        S->delta2 = delta * delta;
        if (!S->guard) S->guard = 1;
    }
    return 0;
}

static int check_args(int64_t n, int d, int k, int work, int dist, int flags) {
    int norm = flags & ONORM_MASK;
    if (n < 1 || d < 1 || k < 1) return -1;
    if (work != OFMT_FP64 && work != OFMT_FP32) return -1;
    if (dist < OFMT_FP64 || dist > OFMT_E5M2) return -1;
    if (work == OFMT_FP32 && dist == OFMT_FP64) return -1;   /* 0 < u <= u_l */
    if (norm > ONORM_ZSCORE || (flags & ~(ONORM_MASK | OGUARD | OGUARD_POW2))) return -1;
    return 0;
}

/* ---------------------------------------------------------------------------------------- */
/* Full Lloyd run (Alg 3 steps 2-7 with C0 given; seeding is out of the path).               */
/*   X_in, C0_in: raw inputs as fp64 arrays holding working-precision values.                */
/*   Outputs: labels[n] (final pass), C_out[k*d], sse (final, direct formula), iters,       */
/*   shift/scale [d] (normalisation map), and optional per-iteration traces (length          */
/*   max_iter): SSE_t (O6), #changed_t, shift^2_t, #empty_t.                                  */
/* Returns 0, or -1 on invalid arguments, -2 on allocation failure.                          */
/* ---------------------------------------------------------------------------------------- */
int oracle_fit(int64_t n, int d, int k, int work, int dist, int flags, const double* X_in,
               const double* C0_in, int max_iter, double tol, int32_t* labels_out,
               double* C_out, double* sse_out, int32_t* iters_out, double* shift_out,
               double* scale_out, double* tr_sse, int64_t* tr_changed, double* tr_shift2,
               int32_t* tr_empty, double delta, int64_t* n_trig_out, double* tr_ubound) {
    if (check_args(n, d, k, work, dist, flags) != 0 || max_iter < 1 || k > n) return -1;
    int norm = flags & ONORM_MASK;
    int guard = (flags & OGUARD_POW2) ? 2 : ((flags & OGUARD) != 0);
    ostate_t S;
    if (alloc_state(&S, n, d, k, work, dist, guard) != 0) { free_state(&S); return -2; }
    if (set_delta(&S, delta) != 0) { free_state(&S); return -1; }
    int64_t n_trig = 0;
    double* shift = (double*)malloc(sizeof(double) * d);
    double* scale = (double*)malloc(sizeof(double) * d);
    oracle_normalize_stats(norm, n, d, X_in, shift, scale);
    if (norm == ONORM_NONE) {
        for (int64_t i = 0; i < n * d; ++i) S.X[i] = oracle_round(work, X_in[i]);
        for (int64_t i = 0; i < (int64_t)k * d; ++i) S.C[i] = oracle_round(work, C0_in[i]);
    } else {
        oracle_normalize_apply(work, n, d, shift, scale, X_in, S.X);
        oracle_normalize_apply(work, k, d, shift, scale, C0_in, S.C);
    }
    if (shift_out) memcpy(shift_out, shift, sizeof(double) * d);
    if (scale_out) memcpy(scale_out, scale, sizeof(double) * d);
    prep_points(&S);

    int32_t* lab = (int32_t*)malloc(sizeof(int32_t) * n);
    int32_t* prev = (int32_t*)malloc(sizeof(int32_t) * n);
    double* dmin = (double*)malloc(sizeof(double) * n);
    for (int64_t i = 0; i < n; ++i) prev[i] = -1;
    int it = 0;
    for (it = 1; it <= max_iter; ++it) {
        prep_centroids(&S);                               /* O3 */
        n_trig += assign_all(&S, lab, dmin, NULL);        /* O4 (O4m), O5 */
        nsum_t sse = {0, 0};                              /* O6 */
        int64_t changed = 0;
        for (int64_t i = 0; i < n; ++i) {
            nsum_add(&sse, dmin[i] > 0.0 ? dmin[i] : 0.0);   /* max(0, D_min); D_min is never NaN */
            if (lab[i] != prev[i]) changed++;
            prev[i] = lab[i];
        }
        double shift2; int empty;
        double* Cprev = tr_ubound ? (double*)malloc(sizeof(double) * k * d) : NULL;
        if (Cprev) memcpy(Cprev, S.C, sizeof(double) * k * d);
        update_centroids(&S, lab, NULL, NULL, &shift2, &empty);   /* O7 */
        if (Cprev) {
            tr_ubound[it - 1] = center_update_bound(k, d, Cprev, S.C);   /* O11 */
            free(Cprev);
        }
        if (tr_sse) tr_sse[it - 1] = nsum_get(&sse);
        if (tr_changed) tr_changed[it - 1] = changed;
        if (tr_shift2) tr_shift2[it - 1] = shift2;
        if (tr_empty) tr_empty[it - 1] = empty;
        if (tol >= 0.0 && (changed == 0 || sqrt(shift2) <= tol)) break;   /* O8 */
    }
    if (it > max_iter) it = max_iter;
    double sse_final = final_pass(&S, labels_out);        /* O9 */
    memcpy(C_out, S.C, sizeof(double) * k * d);
    *sse_out = sse_final;
    *iters_out = it;
    if (n_trig_out) *n_trig_out = n_trig;
    free(lab); free(prev); free(dmin); free(shift); free(scale);
    free_state(&S);
    return 0;
}

/* One teacher-forced Lloyd step (O3..O7) from given centroids on already-normalised data.   */
/* labels/dmin/d2nd are the low-precision assignment; sums/counts the raw update; C_next     */
/* the new centroids (empty clusters keep C_in).                                              */
int oracle_step(int64_t n, int d, int k, int work, int dist, int guard, const double* X,
                const double* C_in, int32_t* labels, double* dmin, double* d2nd, double* sums,
                int64_t* counts, double* C_next, double delta, int64_t* n_trig) {
    if (check_args(n, d, k, work, dist, guard ? OGUARD : 0) != 0) return -1;
    ostate_t S;
    if (alloc_state(&S, n, d, k, work, dist, guard) != 0) { free_state(&S); return -2; }
    if (set_delta(&S, delta) != 0) { free_state(&S); return -1; }
    memcpy(S.X, X, sizeof(double) * n * d);
    memcpy(S.C, C_in, sizeof(double) * k * d);
    prep_points(&S);
    prep_centroids(&S);
    const int64_t tr = assign_all(&S, labels, dmin, d2nd);
    if (n_trig) *n_trig = tr;
    double shift2; int empty;
    update_centroids(&S, labels, sums, counts, &shift2, &empty);
    memcpy(C_next, S.C, sizeof(double) * k * d);
    free_state(&S);
    return 0;
}

/* Low-precision assignment only (kmeans_assign's definition): labels and D_min per point.   */
int oracle_assign(int64_t n, int d, int k, int work, int dist, int guard, const double* X,
                  const double* C, int32_t* labels, double* dmin, double* d2nd, double delta,
                  int64_t* n_trig) {
    if (check_args(n, d, k, work, dist, guard ? OGUARD : 0) != 0) return -1;
    ostate_t S;
    if (alloc_state(&S, n, d, k, work, dist, guard) != 0) { free_state(&S); return -2; }
    if (set_delta(&S, delta) != 0) { free_state(&S); return -1; }
    memcpy(S.X, X, sizeof(double) * n * d);
    memcpy(S.C, C, sizeof(double) * k * d);
    prep_points(&S);
    prep_centroids(&S);
    const int64_t tr = assign_all(&S, labels, dmin, d2nd);
    if (n_trig) *n_trig = tr;
    free_state(&S);
    return 0;
}

/* ---------------------------------------------------------------------------------------- */
/* O10: seeding by D^2 weighting (Alg 1) with the distances of Alg 3 step 1 */
/* "in precision u_l": after O1 and O2, D^2(p_i, c) is O4's expanded formula    */
/* from the stored low-precision operands (the dot accumulated sequentially in fp64), floored */
/* at 0; the centre c is a data point, so its operands are that row's. Line 2 of Alg 1 draws  */
/* p' with probability D(p')^2 / sum_p D(p)^2; reading R6 makes the draw explicit:             */
/*   * the caller supplies k uniforms u_j in [0,1) (the method's random draws);               */
/*   * first centre: index min(floor(u_0 n), n-1) ("uniformly", line 1);                      */
/*   * D2[i] = min over chosen centres; S = sum_i D2[i] (sequential, index order);            */
/*   * next centre: the first index i whose running sum D2[0] + ... + D2[i] (sequential)      */
/*     exceeds u_j S — the inverse-CDF draw of the law above; i then has D2[i] > 0 (new);     */
/*   * S = 0 or non-finite (every point coincides with a centre, or overflow): uniform index   */
/*     min(floor(u_j n), n-1) and *warn |= 1 (SPEC S:208's fallback);                          */
/*   * a chosen centre's own weight is 0 (dist(c, c) = 0; the expanded formula in low          */
/*     precision leaves a rounding residue there), so the k centres are distinct. */
/* ---------------------------------------------------------------------------------------- */
static double seed_dist(const ostate_t* S, int64_t i, int64_t c) {
    const double* xl = S->Xl + i * S->d;
    const double* cl = S->Xl + c * S->d;
    double dot = 0.0;
    for (int t = 0; t < S->d; ++t) dot += xl[t] * cl[t];
    double D = S->xn[i] - 2.0 * (S->sx[i] * S->sx[c]) * dot + S->xn[c];
    return (D > 0.0) ? D : 0.0;   /* NaN -> 0 */
}

static int seed_prepare(ostate_t* S, int64_t n, int d, int work, int dist, int flags,
                        const double* X_in) {
    int norm = flags & ONORM_MASK;
    int guard = (flags & OGUARD_POW2) ? 2 : ((flags & OGUARD) != 0);
    if (alloc_state(S, n, d, 1, work, dist, guard) != 0) return -2;
    double* shift = (double*)malloc(sizeof(double) * d);
    double* scale = (double*)malloc(sizeof(double) * d);
    oracle_normalize_stats(norm, n, d, X_in, shift, scale);
    if (norm == ONORM_NONE) {
        for (int64_t i = 0; i < n * d; ++i) S->X[i] = oracle_round(work, X_in[i]);
    } else {
        oracle_normalize_apply(work, n, d, shift, scale, X_in, S->X);
    }
    free(shift); free(scale);
    prep_points(S);
    return 0;
}

/* D2[i] <- min(D2[i], D^2(p_i, c)), the centre's own weight 0 (Alg 1 line 2's D(p)). */
static void seed_min_update(const ostate_t* S, int64_t n, int64_t c, double* D2) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        double D = (i == c) ? 0.0 : seed_dist(S, i, c);
        if (D < D2[i]) D2[i] = D;
    }
}

int oracle_seed_d2(int64_t n, int d, int k, int work, int dist, int flags, const double* X_in,
                   const double* u, int64_t* idx_out, double* d2_out, int* warn) {
    if (check_args(n, d, k, work, dist, flags) != 0 || k > n) return -1;
    ostate_t S;
    if (seed_prepare(&S, n, d, work, dist, flags, X_in) != 0) { free_state(&S); return -2; }
    double* D2 = (double*)malloc(sizeof(double) * n);
    int w = 0;
    for (int64_t i = 0; i < n; ++i) D2[i] = INFINITY;
    int64_t c = (int64_t)(u[0] * (double)n);
    if (c > n - 1) c = n - 1;
    if (c < 0) c = 0;
    idx_out[0] = c;
    for (int j = 1; j < k; ++j) {
        seed_min_update(&S, n, c, D2);
        double tot = 0.0;
        for (int64_t i = 0; i < n; ++i) tot += D2[i];
        if (!(tot > 0.0) || isinf(tot)) {
            c = (int64_t)(u[j] * (double)n);
            if (c > n - 1) c = n - 1;
            w |= 1;
        } else {
            const double target = u[j] * tot;
            double run = 0.0;
            c = -1;
            for (int64_t i = 0; i < n; ++i) {
                run += D2[i];
                if (run > target) { c = i; break; }
            }
            if (c < 0) {             /* rounding left the target at the very top: last positive */
                for (int64_t i = n - 1; i >= 0; --i)
                    if (D2[i] > 0.0) { c = i; break; }
            }
        }
        idx_out[j] = c;
    }
    if (d2_out) {
        /* D2 after the last centre too (the weights a (k+1)-th draw would use) */
        seed_min_update(&S, n, c, D2);
        memcpy(d2_out, D2, sizeof(double) * n);
    }
    if (warn) *warn = w;
    free(D2);
    free_state(&S);
    return 0;
}

/* The D^2 weights of O10 for a given list of m chosen centres (teacher-forced checks of a
 * seeding that made its own draws): D2[i] = min over the centres of D^2(p_i, c), 0 at the
 * centres themselves. */
int oracle_seed_weights(int64_t n, int d, int work, int dist, int flags, const double* X_in,
                        const int64_t* centres, int m, double* D2) {
    if (check_args(n, d, 1, work, dist, flags) != 0 || m < 1) return -1;
    ostate_t S;
    if (seed_prepare(&S, n, d, work, dist, flags, X_in) != 0) { free_state(&S); return -2; }
    for (int64_t i = 0; i < n; ++i) D2[i] = INFINITY;
    for (int q = 0; q < m; ++q) {
        if (centres[q] < 0 || centres[q] >= n) { free_state(&S); return -1; }
        seed_min_update(&S, n, centres[q], D2);
    }
    free_state(&S);
    return 0;
}

/* Low-precision operands and norms exactly as O2/O3 produce them (for cast/prep parity).    */
int oracle_prep(int64_t n, int d, int work, int dist, int guard, const double* X, double* Xl,
                double* norms, double* scales) {
    if (n < 0 || d < 1) return -1;
    for (int64_t i = 0; i < n; ++i)
        prep_vector(work, dist, guard, d, X + i * d, &norms[i], &scales[i], Xl + i * d);
    return 0;
}

/* Final pass alone (O9) with given centroids on normalised data. Returns SSE via *sse.       */
int oracle_final(int64_t n, int d, int k, int work, const double* X, const double* C,
                 int32_t* labels, double* sse) {
    ostate_t S;
    if (alloc_state(&S, n, d, k, work, work, 0) != 0) { free_state(&S); return -2; }
    memcpy(S.X, X, sizeof(double) * n * d);
    memcpy(S.C, C, sizeof(double) * k * d);
    *sse = final_pass(&S, labels);
    free_state(&S);
    return 0;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
