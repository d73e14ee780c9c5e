// k_update.cu — K7 centroid update and K8 finalize (eq:center, in the working
// precision u: Alg 3 step 4).
//
// K7 is a bucket-by-label update that needs no floating-point atomics on the hot rows:
//   U1 count   : block-privatised int histogram of the labels (smem) -> global counts
//   U2 scan    : exclusive prefix sum of the k counts -> bucket offsets (one block)
//   U3 scatter : warp-aggregated (__match_any_sync) slot claims -> perm[] = rows grouped by label
//   U4 segsum  : each warp streams a contiguous chunk of perm[], lanes over columns, summing the
//                gathered rows in fp64 registers; a flush (one fp64 atomic per column) happens
//                only where the label changes inside the chunk (~1-2 per chunk).
// Sums are therefore accumulated in fp64 (at least the working precision u; DESIGN.md reading
// on update precision) and the mean is rounded once to u in K8. X is read exactly once, in
// whole rows (coalesced 16-byte vector loads), so U4 is HBM-bound.
// K8: c_j = round_u(sum_j / count_j), empty clusters keep c_j (reading Z14); shift^2 and the
//     number of empty clusters go to the iteration record.
#include "common.cuh"
#include "internal.h"

namespace mpk {

namespace {

constexpr int kHistMax = 12288;   // 48 KB of int bins in smem

__global__ void count_kernel(const int32_t* __restrict__ labels, int64_t n, int k,
                             int* __restrict__ cnt) {
    extern __shared__ int hist[];
    const bool use_smem = k <= kHistMax;
    if (use_smem) {
        for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
        __syncthreads();
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        int l = labels[i];
        if (use_smem) atomicAdd(&hist[l], 1);
        else atomicAdd(&cnt[l], 1);
    }
    if (use_smem) {
        __syncthreads();
        for (int j = threadIdx.x; j < k; j += blockDim.x)
            if (hist[j]) atomicAdd(&cnt[j], hist[j]);
    }
}

// Single-block exclusive scan of k counts (k arbitrary): chunked by 1024 with a running carry.
__global__ void scan_kernel(const int* __restrict__ cnt, int k, int* __restrict__ offs,
                            int* __restrict__ cursor, double* __restrict__ acc_counts) {
    __shared__ int sh[1024];
    __shared__ int carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < k; base += 1024) {
        int j = base + threadIdx.x;
        int v = j < k ? cnt[j] : 0;
        sh[threadIdx.x] = v;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += t;
            __syncthreads();
        }
        if (j < k) {
            int ex = carry + sh[threadIdx.x] - v;
            offs[j] = ex;
            cursor[j] = ex;
            acc_counts[j] = (double)v;
        }
        __syncthreads();
        if (threadIdx.x == 1023) carry += sh[1023];
        __syncthreads();
    }
    if (threadIdx.x == 0) offs[k] = carry;
}

// U3 (k <= kHistMax): block-aggregated slot claims. Each block ranks its rows per label in a
// shared-memory histogram (integer smem atomics), reserves one contiguous range per label with
// a single global atomic, then writes perm. Global atomics drop from one per row to one per
// (block, label present).
constexpr int kScatterRows = 16;
__global__ void __launch_bounds__(256)
scatter_block_kernel(const int32_t* __restrict__ labels, int64_t n, int k,
                     int* __restrict__ cursor, int* __restrict__ perm) {
    extern __shared__ int sh[];
    const int64_t base = (int64_t)blockIdx.x * blockDim.x * kScatterRows;
    for (int j = threadIdx.x; j < k; j += blockDim.x) sh[j] = 0;
    __syncthreads();
    int lab[kScatterRows], rk[kScatterRows];
#pragma unroll
    for (int r = 0; r < kScatterRows; ++r) {
        const int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
        lab[r] = i < n ? labels[i] : -1;
    }
#pragma unroll
    for (int r = 0; r < kScatterRows; ++r) rk[r] = lab[r] >= 0 ? atomicAdd(&sh[lab[r]], 1) : 0;
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const int c = sh[j];
        if (c) sh[j] = atomicAdd(&cursor[j], c);
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < kScatterRows; ++r) {
        const int64_t i = base + (int64_t)r * blockDim.x + threadIdx.x;
        if (lab[r] >= 0) perm[sh[lab[r]] + rk[r]] = (int)i;
    }
}

__global__ void scatter_kernel(const int32_t* __restrict__ labels, int64_t n,
                               int* __restrict__ cursor, int* __restrict__ perm) {
    const int lane = threadIdx.x & 31;
    for (int64_t base = (int64_t)blockIdx.x * blockDim.x; base < n;
         base += (int64_t)gridDim.x * blockDim.x) {
        int64_t i = base + threadIdx.x;
        bool valid = i < n;
        unsigned active = __ballot_sync(0xffffffffu, valid);
        if (!valid) continue;
        int l = labels[i];
        unsigned peers = __match_any_sync(active, l);
        int leader = __ffs(peers) - 1;
        int slot = 0;
        if (lane == leader) slot = atomicAdd(&cursor[l], __popc(peers));
        slot = __shfl_sync(peers, slot, leader);
        slot += __popc(peers & ((1u << lane) - 1u));
        perm[slot] = (int)i;
    }
}

template <typename W, int VEC>
struct VecLoad;
template <> struct VecLoad<float, 1> { using T = float; };
template <> struct VecLoad<float, 2> { using T = float2; };
template <> struct VecLoad<float, 4> { using T = float4; };
template <> struct VecLoad<double, 1> { using T = double; };
template <> struct VecLoad<double, 2> { using T = double2; };

template <typename W, int VEC>
MPK_DEV void load_vec(const W* p, bool aligned, int ncols, W (&out)[VEC]) {
    if (aligned && ncols == VEC) {
        using T = typename VecLoad<W, VEC>::T;
        T v = __ldg(reinterpret_cast<const T*>(p));
        const W* pv = reinterpret_cast<const W*>(&v);
#pragma unroll
        for (int q = 0; q < VEC; ++q) out[q] = pv[q];
    } else {
#pragma unroll
        for (int q = 0; q < VEC; ++q) out[q] = q < ncols ? __ldg(p + q) : (W)0;
    }
}

// U4: warps own contiguous chunks of perm; grid.y = column blocks of 32*VEC.
template <typename W, int VEC, int U>
__global__ void __launch_bounds__(256)
segsum_kernel(const W* __restrict__ X, int64_t n, int d, int k, const int* __restrict__ perm,
              const int* __restrict__ offs, int64_t chunk, double* __restrict__ sums) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int col0 = blockIdx.y * 32 * VEC + lane * VEC;
    const int ncols = max(0, min(VEC, d - col0));
    const bool aligned = (d % VEC) == 0;
    int64_t e0 = warp * chunk;
    if (e0 >= n) return;
    int64_t e1 = min(n, e0 + chunk);
    // label of entry e0: largest j with offs[j] <= e0 (binary search over k+1 offsets)
    int lo = 0, hi = k;   // offs[0] = 0 <= e0 < offs[k] = n
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (offs[mid] <= e0) lo = mid; else hi = mid;
    }
    int cur = lo;
    int64_t next_boundary = offs[cur + 1];
    double acc[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) acc[q] = 0.0;

    auto flush = [&](int j) {
        if (ncols > 0) {
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                if (q < ncols && acc[q] != 0.0) atomicAdd(&sums[(int64_t)j * d + col0 + q], acc[q]);
        }
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
    };

    for (int64_t e = e0; e < e1; e += 32) {
        // lanes fetch up to 32 perm entries, then broadcast
        int myrow = (e + lane < e1) ? perm[e + lane] : 0;
        const int cnt = (int)min((int64_t)32, e1 - e);
        for (int u0 = 0; u0 < cnt; u0 += U) {
            W xv[U][VEC];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                int row = __shfl_sync(0xffffffffu, myrow, (u0 + u) & 31);
                if (u0 + u < cnt && ncols > 0)
                    load_vec<W, VEC>(X + (int64_t)row * d + col0, aligned, ncols, xv[u]);
                else {
#pragma unroll
                    for (int q = 0; q < VEC; ++q) xv[u][q] = (W)0;
                }
            }
            const int64_t elast = e + u0 + U - 1;
            if (u0 + U <= cnt && elast < next_boundary) {
                // common case: the whole batch belongs to the current cluster. Sum the U rows
                // in the working type first (one conversion to fp64 per batch instead of per
                // row; the conversion unit, not HBM, bounded the per-row form).
#pragma unroll
                for (int q = 0; q < VEC; ++q) {
                    W s = xv[0][q];
#pragma unroll
                    for (int u = 1; u < U; ++u) s += xv[u][q];
                    acc[q] += (double)s;
                }
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    if (u0 + u < cnt) {
                        int64_t epos = e + u0 + u;
                        while (epos >= next_boundary) {   // label changes (warp-uniform)
                            flush(cur);
                            ++cur;
                            next_boundary = offs[cur + 1];
                        }
#pragma unroll
                        for (int q = 0; q < VEC; ++q) acc[q] += (double)xv[u][q];
                    }
                }
            }
        }
    }
    flush(cur);
}

template <typename W>
__global__ void finalize_kernel(int64_t k, int d, const double* __restrict__ acc, AccLayout L,
                                W* __restrict__ C, IterRec* __restrict__ rec) {
    constexpr int WORK = sizeof(W) == 8 ? KMEANS_FP64 : KMEANS_FP32;
    const int64_t total = k * d;
    double sh = 0.0;
    double empty = 0.0;
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        int64_t j = idx / d;
        int t = (int)(idx - j * d);
        double c = acc[L.counts() + j];
        W old = C[idx];
        W nw = old;
        if (c > 0.0) nw = rounder<WORK>::from(acc[L.sums() + idx] / c);
        else if (t == 0) empty += 1.0;
        double df = (double)nw - (double)old;
        sh += df * df;
        C[idx] = nw;
    }
    sh = warp_sum(sh);
    empty = warp_sum(empty);
    __shared__ double red[2][8];
    if ((threadIdx.x & 31) == 0) { red[0][threadIdx.x >> 5] = sh; red[1][threadIdx.x >> 5] = empty; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += red[0][w]; b += red[1][w]; }
        atomicAdd(&rec->shift2, a);
        if (b != 0.0) atomicAdd(&rec->empty, b);
        if (blockIdx.x == 0) {
            rec->sse = acc[L.sse()];
            rec->changed = acc[L.changed()];
        }
    }
}

template <typename W>
cudaError_t update_dispatch(const W* X, int64_t n, int d, int k, const int32_t* labels, int* cnt,
                            int* offs, int* cursor, int* perm, double* acc, AccLayout L,
                            cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(int) * k, s);
    if (e != cudaSuccess) return e;
    int g = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 4);
    if (g < 1) g = 1;
    size_t hist_bytes = k <= kHistMax ? sizeof(int) * k : 0;
    count_kernel<<<g, 256, hist_bytes, s>>>(labels, n, k, cnt);
    scan_kernel<<<1, 1024, 0, s>>>(cnt, k, offs, cursor, acc + L.counts());
    if (k <= kHistMax) {
        const int64_t sb = (n + 256LL * kScatterRows - 1) / (256LL * kScatterRows);
        scatter_block_kernel<<<(unsigned)sb, 256, sizeof(int) * k, s>>>(labels, n, k, cursor, perm);
    } else {
        scatter_kernel<<<g, 256, 0, s>>>(labels, n, cursor, perm);
    }
    // segmented sums: ~8 warps per SM-slot, chunks of >= 256 rows
    const int VEC = (sizeof(W) == 8) ? (d <= 32 ? 1 : 2) : (d <= 32 ? 1 : (d <= 64 ? 2 : 4));
    const int colblk = 32 * VEC;
    dim3 grid;
    int64_t warps = (int64_t)kNumSMs * 32;
    int64_t chunk = std::max<int64_t>(256, (n + warps - 1) / warps);
    int64_t nw = (n + chunk - 1) / chunk;
    grid.x = (unsigned)((nw + 7) / 8);
    grid.y = (unsigned)((d + colblk - 1) / colblk);
    grid.z = 1;
    if constexpr (sizeof(W) == 8) {
        if (VEC == 1)
            segsum_kernel<W, 1, 8><<<grid, 256, 0, s>>>(X, n, d, k, perm, offs, chunk, acc + L.sums());
        else
            segsum_kernel<W, 2, 8><<<grid, 256, 0, s>>>(X, n, d, k, perm, offs, chunk, acc + L.sums());
    } else {
        if (VEC == 1)
            segsum_kernel<W, 1, 8><<<grid, 256, 0, s>>>(X, n, d, k, perm, offs, chunk, acc + L.sums());
        else if (VEC == 2)
            segsum_kernel<W, 2, 8><<<grid, 256, 0, s>>>(X, n, d, k, perm, offs, chunk, acc + L.sums());
        else
            segsum_kernel<W, 4, 8><<<grid, 256, 0, s>>>(X, n, d, k, perm, offs, chunk, acc + L.sums());
    }
    return cudaGetLastError();
}

}  // namespace

cudaError_t launch_update(int work, const void* Xw, int64_t n, int d, int k,
                          const int32_t* labels, int* cnt, int* offs, int* cursor, int* perm,
                          double* acc, AccLayout L, cudaStream_t s) {
    launches_add(4);
    if (work == KMEANS_FP64)
        return update_dispatch<double>((const double*)Xw, n, d, k, labels, cnt, offs, cursor,
                                       perm, acc, L, s);
    return update_dispatch<float>((const float*)Xw, n, d, k, labels, cnt, offs, cursor, perm, acc,
                                  L, s);
}

cudaError_t launch_finalize(int work, int64_t k, int d, const double* acc, AccLayout L, void* Cw,
                            IterRec* rec, cudaStream_t s) {
    launches_add(1);
    int64_t total = k * d;
    int g = (int)std::min<int64_t>((total + 255) / 256, kNumSMs * 2);
    if (g < 1) g = 1;
    if (work == KMEANS_FP64)
        finalize_kernel<double><<<g, 256, 0, s>>>(k, d, acc, L, (double*)Cw, rec);
    else
        finalize_kernel<float><<<g, 256, 0, s>>>(k, d, acc, L, (float*)Cw, rec);
    return cudaGetLastError();
}

}  // namespace mpk
