// k_update.cu — K7 centroid update and K8 finalize (eq:center, in the working
// precision u: Alg 3 step 4).
//
// K7 is a stable bucket-by-label update with no floating-point atomics, so the new centres are
// bit-for-bit the same on every run (k <= kHistMax; above it U1/U3 fall back to atomic slot
// claims and the order inside a cluster may vary):
//   U1 count   : per-8192-row-block label histograms (smem) -> CB, then a per-label scan over the
//                blocks (the block offsets inside the cluster's bucket, and the counts)
//   U2 scan    : exclusive prefix sum of the k counts -> bucket offsets (one block)
//   U3 scatter : stable in-block ranks (__match_any_sync, warps in row order) -> perm[] = rows
//                grouped by label, in increasing row index inside each label
//   U4 segsum  : each bucket is cut into pieces of P rows from its start; warps stream the pieces
//                starting in their chunk of perm[], lanes over columns, summing the gathered
//                rows in fp64 registers; one-piece clusters are stored directly, longer ones
//                per piece, and U4b adds a cluster's pieces in a fixed order. A cluster's sum
//                then depends on its members only (same members -> bit-identical centre).
// Sums are therefore accumulated in fp64 (at least the working precision u; DESIGN.md reading
// on update precision) and the mean is rounded once to u in K8. X is read exactly once, in
// whole rows (coalesced 16-byte vector loads), so U4 is HBM-bound.
// K8: c_j = round_u(sum_j / count_j), empty clusters keep c_j (reading Z14); shift^2 and the
//     number of empty clusters go to the iteration record.
// FX (fp32 work, one rank; R9, default): the same U1-U4 with exact integer totals on a
// per-feature grid, kept across iterations and updated from the rows whose label changed (integer
// atomics) while few rows change — bit-identical to re-summing every row (tested).
#include "common.cuh"
#include "internal.h"

namespace mpk {

namespace {

constexpr int kHistMax = 12288;   // 48 KB of int bins in smem

// Fixed-point mode (FX, below): the full-recompute kernels run only when the iteration's list
// of changed rows overflowed (gate[0] = changed rows, gate[1] = list capacity); nullptr = always.
MPK_DEV bool gated_off(const int* gate) { return gate != nullptr && gate[0] <= gate[1]; }

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
// A second scan over the same chunks gives mpo[j], the first partial-sum slot of cluster j when
// it spans several segsum pieces of P rows (ceil(cnt_j / P) >= 2 slots; else 0 slots).
__global__ void scan_kernel(const int* __restrict__ cnt, int k, int64_t P, int* __restrict__ offs,
                            int* __restrict__ cursor, int* __restrict__ mpo,
                            double* __restrict__ acc_counts, const int* gate = nullptr) {
    griddep_wait();
    if (gated_off(gate)) return;
    __shared__ int sh[1024], sh2[1024];
    __shared__ int carry, carry2;
    if (threadIdx.x == 0) carry = carry2 = 0;
    __syncthreads();
    for (int base = 0; base < k; base += 1024) {
        int j = base + threadIdx.x;
        int v = j < k ? cnt[j] : 0;
        const int np = (int)((v + P - 1) / P);
        int v2 = np >= 2 ? np : 0;
        sh[threadIdx.x] = v;
        sh2[threadIdx.x] = v2;
        __syncthreads();
        for (int o = 1; o < 1024; o <<= 1) {
            int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
            int t2 = threadIdx.x >= o ? sh2[threadIdx.x - o] : 0;
            __syncthreads();
            sh[threadIdx.x] += t;
            sh2[threadIdx.x] += t2;
            __syncthreads();
        }
        if (j < k) {
            int ex = carry + sh[threadIdx.x] - v;
            offs[j] = ex;
            cursor[j] = ex;
            mpo[j] = carry2 + sh2[threadIdx.x] - v2;
            if (acc_counts) acc_counts[j] = (double)v;
        }
        __syncthreads();
        if (threadIdx.x == 1023) { carry += sh[1023]; carry2 += sh2[1023]; }
        __syncthreads();
    }
    if (threadIdx.x == 0) { offs[k] = carry; mpo[k] = carry2; }
}

// Deterministic U1/U3 (k <= kHistMax): rows are taken in blocks of kDetRows; a row's slot is
//   offs[l] + (rows with label l in earlier blocks) + (rows with label l earlier in its block),
// i.e. perm lists each cluster's rows in increasing row index — a stable bucket sort, the same
// on every run (only integer counts use atomics, and counts do not depend on order).
constexpr int kDetThreads = 512;
constexpr int kDetRows = 8192;                    // rows per counting / scatter block

// U1a: per-block label histogram -> CB[b * k + l] (block-major: coalesced stores).
__global__ void __launch_bounds__(kDetThreads)
block_count_kernel(const int32_t* __restrict__ labels, int64_t n, int k, int* __restrict__ CB,
                   const int* gate = nullptr) {
    griddep_wait();
    if (gated_off(gate)) return;
    extern __shared__ int hist[];
    for (int j = threadIdx.x; j < k; j += blockDim.x) hist[j] = 0;
    __syncthreads();
    const int64_t base = (int64_t)blockIdx.x * kDetRows;
#pragma unroll 4
    for (int r = 0; r < kDetRows / kDetThreads; ++r) {
        const int64_t i = base + (int64_t)r * kDetThreads + threadIdx.x;
        if (i < n) atomicAdd(&hist[labels[i]], 1);
    }
    __syncthreads();
    int* out = CB + (int64_t)blockIdx.x * k;
    for (int j = threadIdx.x; j < k; j += blockDim.x) out[j] = hist[j];
}

// U1b: exclusive scan of CB[., l] over the blocks in order (in place) and the counts. A CTA takes
// 32 labels (lanes) and its 32 warps take consecutive segments of blocks: segment totals,
// a scan of the 32 totals, then the segments rewritten with their offsets.
__global__ void __launch_bounds__(1024)
block_scan_kernel(int* __restrict__ CB, int64_t nb, int k, int* __restrict__ cnt,
                  const int* gate = nullptr) {
    griddep_wait();
    if (gated_off(gate)) return;
    __shared__ int tot[32][33];
    const int lane = threadIdx.x & 31, seg = threadIdx.x >> 5;
    const int l = blockIdx.x * 32 + lane;
    const int64_t per = (nb + 31) / 32;
    const int64_t b0 = seg * per, b1 = min(nb, b0 + per);
    int sum = 0;
    if (l < k)
        for (int64_t b = b0; b < b1; ++b) sum += CB[b * k + l];
    tot[seg][lane] = sum;
    __syncthreads();
    if (seg == 0) {
        int run = 0;
        for (int s2 = 0; s2 < 32; ++s2) {
            const int v = tot[s2][lane];
            tot[s2][lane] = run;
            run += v;
        }
        if (l < k) cnt[l] = run;
    }
    __syncthreads();
    if (l < k) {
        int run = tot[seg][lane];
        for (int64_t b = b0; b < b1; ++b) {
            const int v = CB[b * k + l];
            CB[b * k + l] = run;
            run += v;
        }
    }
}

// U3: stable in-block ranks without a serial chain. The block's rows are split among its warps
// in contiguous spans (warp w: rows [w * span, (w + 1) * span)).
//   1. each warp walks its span in rounds of 32 rows (__syncwarp between rounds orders its
//      shared-memory updates): a round's lanes with equal labels take consecutive ranks from the
//      warp's own histogram H[w][.] -> rank of the row among the span's earlier rows with its label
//   2. per label, an exclusive scan of H[.][l] over the warps
//   3. slot = offs[l] + CB[b][l] + H[w][l] + rank (ranks kept in shared memory)
// Warps per block = scatter_warps(k) keeps H within kDetHistBytes.
constexpr int kDetHistBytes = 64 * 1024;
int scatter_warps(int k) {
    int w = 16;
    while (w > 1 && (size_t)w * k * sizeof(int) > (size_t)kDetHistBytes) w >>= 1;
    return w;
}
size_t scatter_smem(int k) {
    return (size_t)scatter_warps(k) * k * sizeof(int) + (size_t)kDetRows * sizeof(int);
}

// Lanes holding the same key (0 <= key < 2^bits): the AND of one ballot per key bit. Cheaper than
// __match_any_sync, whose cost grows with the number of distinct values in the warp.
MPK_DEV unsigned match_bits(int key, int bits) {
    unsigned m = 0xffffffffu;
    for (int b = 0; b < bits; ++b) {
        const bool on = (key >> b) & 1;
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        m &= on ? bal : ~bal;
    }
    return m;
}

__global__ void __launch_bounds__(kDetThreads)
scatter_det_kernel(const int32_t* __restrict__ labels, int64_t n, int k,
                   const int* __restrict__ offs, const int* __restrict__ CB,
                   int* __restrict__ perm, const int* gate = nullptr) {
    griddep_wait();
    if (gated_off(gate)) return;
    const int kbits = 32 - __clz(k);              // keys l + 1 in [0, k]
    extern __shared__ int smem_i[];
    const int nwarps = blockDim.x >> 5;
    int* H = smem_i;                              // [nwarps][k]
    int* rk = smem_i + (size_t)nwarps * k;        // [kDetRows]
    for (int j = threadIdx.x; j < nwarps * k; j += blockDim.x) H[j] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int span = kDetRows / nwarps;
    const int64_t b0 = (int64_t)blockIdx.x * kDetRows;
    int* Hw = H + (size_t)warp * k;
    const unsigned lt = (1u << lane) - 1u;
    // span is a multiple of 512: labels are fetched 16 rounds at a time, ahead of the ordered
    // walk (the walk's shared-memory updates would otherwise serialise the global loads)
    for (int g = warp * span; g < (warp + 1) * span; g += 512) {
        int lb[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int64_t i = b0 + g + u * 32 + lane;
            lb[u] = i < n ? labels[i] : -1;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const int l = lb[u];
            const unsigned peers = match_bits(l + 1, kbits);
            const int leader = __ffs(peers) - 1;
            int base = 0;
            if (l >= 0 && lane == leader) {       // H[w] is this warp's alone: plain update
                base = Hw[l];
                Hw[l] = base + __popc(peers);
            }
            base = __shfl_sync(0xffffffffu, base, leader);
            rk[g + u * 32 + lane] = base + __popc(peers & lt);
            __syncwarp();
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        int run = 0;
        for (int w = 0; w < nwarps; ++w) {
            const int t = H[(size_t)w * k + j];
            H[(size_t)w * k + j] = run;
            run += t;
        }
    }
    __syncthreads();
    const int* cb = CB + (int64_t)blockIdx.x * k;
#pragma unroll 8
    for (int r = warp * span + lane; r < (warp + 1) * span; r += 32) {
        const int64_t i = b0 + r;
        if (i < n) {
            const int l = labels[i];
            perm[offs[l] + cb[l] + Hw[l] + rk[r]] = (int)i;
        }
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

// U4: each cluster's bucket is cut into pieces of P rows counted from the bucket's start, and a
// warp sums the pieces whose first row lies in its chunk of C rows of perm (one wave of warps,
// each reading fewer than C + P rows); grid.y = column blocks of 32*VEC. A piece's rows are
// added in bucket order (increasing row index, U3), in batches of U rows aligned to the piece
// start, so every sum depends only on the cluster's members — not on where other clusters'
// buckets end — and a cluster whose members do not change gets bit-identical sums. A
// one-piece cluster is stored directly; the pieces of longer ones go to slots mpo[j] + p, added
// in a fixed order by U4b. No floating-point atomics.
template <typename W, int VEC, int U>
__global__ void __launch_bounds__(256, 4)   // 4 blocks/SM: the 32-warps-per-SM grid is one wave
segsum_kernel(const W* __restrict__ X, int64_t n, int d, int k, const int* __restrict__ perm,
              const int* __restrict__ offs, const int* __restrict__ mpo, int64_t P, int64_t C,
              double* __restrict__ sums, double* __restrict__ part) {
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int col0 = blockIdx.y * 32 * VEC + lane * VEC;
    const int ncols = max(0, min(VEC, d - col0));
    const bool aligned = (d % VEC) == 0;
    const int64_t e0 = warp * C;
    if (e0 >= n) return;
    const int64_t e1 = min(n, e0 + C);
    // the cluster holding entry e0: largest j with offs[j] <= e0 (binary search over k+1 offsets)
    int lo = 0, hi = k;   // offs[0] = 0 <= e0 < offs[k] = n
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (offs[mid] <= e0) lo = mid; else hi = mid;
    }
    int j = lo;
    // first piece of cluster j starting at or after e0
    int64_t pidx = (e0 - offs[j] + P - 1) / P;
    int64_t ps = offs[j] + pidx * P;
    for (;;) {
        if (ps >= offs[j + 1]) {            // past cluster j: next non-empty cluster's piece 0
            do { ++j; } while (j < k && offs[j] == offs[j + 1]);
            if (j >= k) break;
            pidx = 0;
            ps = offs[j];
        }
        if (ps >= e1) break;
        const int64_t pe = min((int64_t)offs[j + 1], ps + P);
        double acc[VEC];
#pragma unroll
        for (int q = 0; q < VEC; ++q) acc[q] = 0.0;
        for (int64_t e = ps; e < pe; e += 32) {
            const int myrow = (e + lane < pe) ? perm[e + lane] : 0;
            const int cnt = (int)min((int64_t)32, pe - e);
            for (int u0 = 0; u0 < cnt; u0 += U) {
                W xv[U][VEC];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int row = __shfl_sync(0xffffffffu, myrow, (u0 + u) & 31);
                    if (u0 + u < cnt && ncols > 0)
                        load_vec<W, VEC>(X + (int64_t)row * d + col0, aligned, ncols, xv[u]);
                    else {
#pragma unroll
                        for (int q = 0; q < VEC; ++q) xv[u][q] = (W)0;
                    }
                }
                if (u0 + U <= cnt) {
                    // a full batch: sum the U rows in the working type first (one conversion to
                    // fp64 per batch; the conversion unit, not HBM, bounded the per-row form)
#pragma unroll
                    for (int q = 0; q < VEC; ++q) {
                        W sm = xv[0][q];
#pragma unroll
                        for (int u = 1; u < U; ++u) sm += xv[u][q];
                        acc[q] += (double)sm;
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < U; ++u)
                        if (u0 + u < cnt) {
#pragma unroll
                            for (int q = 0; q < VEC; ++q) acc[q] += (double)xv[u][q];
                        }
                }
            }
        }
        const bool single = offs[j + 1] - offs[j] <= P;
        double* dst = single ? sums + (int64_t)j * d : part + (int64_t)(mpo[j] + pidx) * d;
        if (ncols > 0) {
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                if (q < ncols) dst[col0 + q] = acc[q];
        }
        ++pidx;
        ps += P;
    }
}

// U4b: the pieces of each multi-piece cluster: a CTA per (cluster, 32-column block); warp w adds
// pieces w, w + 8, ... in order (lanes over columns: coalesced), then lane sums the 8 warp
// partials in warp order.
__global__ void __launch_bounds__(256)
segsum_fix_kernel(int d, const int* __restrict__ mpo, const double* __restrict__ part,
                  double* __restrict__ sums) {
    const int j = blockIdx.x;
    const int np = mpo[j + 1] - mpo[j];
    if (np == 0) return;
    __shared__ double red[8][32];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int col = blockIdx.y * 32 + lane;
    double sum = 0.0;
    if (col < d) {
        const double* pp = part + (int64_t)mpo[j] * d + col;
#pragma unroll 4
        for (int p = w; p < np; p += 8) sum += pp[(int64_t)p * d];
    }
    red[w][lane] = sum;
    __syncthreads();
    if (w == 0 && col < d) {
        double t = red[0][lane];
#pragma unroll
        for (int q = 1; q < 8; ++q) t += red[q][lane];
        sums[(int64_t)j * d + col] = t;
    }
}

template <typename W>
__global__ void finalize_kernel(int64_t k, int d, const double* __restrict__ acc, AccLayout L,
                                W* __restrict__ C, IterRec* __restrict__ rec) {
    // A7 (Alg 3 step 4's division, rounded once to u; empty clusters keep their centre) with one
    // warp per cluster, which also yields Thm 5.3's per-cluster quantities:
    //   num_j = |c^ - mu^|^T |c^ - mu^|  (the cluster's share of the shift ||C_t+1 - C_t||^2)
    //   den_j = |c^ - mu^|^T |mu^|
    // u must stay below num_j / (2 den_j); rec->ub_inv collects max_j 2 den_j / num_j.
    constexpr int WORK = sizeof(W) == 8 ? KMEANS_FP64 : KMEANS_FP32;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double sh = 0.0, empty = 0.0, rmax = 0.0;
    for (int64_t j = warp; j < k; j += nwarps) {
        const double c = acc[L.counts() + j];
        double num = 0.0, den = 0.0;
        for (int t = lane; t < d; t += 32) {
            const int64_t idx = j * d + t;
            const W old = C[idx];
            W nw = old;
            if (c > 0.0) nw = rounder<WORK>::from(acc[L.sums() + idx] / c);
            const double df = (double)nw - (double)old;
            num += df * df;
            den += fabs(df) * fabs((double)nw);
            C[idx] = nw;
        }
        num = warp_sum(num);
        den = warp_sum(den);
        if (lane == 0) {
            sh += num;
            if (c == 0.0) empty += 1.0;
            if (num > 0.0 && den > 0.0) rmax = fmax(rmax, 2.0 * den / num);
        }
    }
    __shared__ double red[3][8];
    if (lane == 0) { red[0][threadIdx.x >> 5] = sh; red[1][threadIdx.x >> 5] = empty; red[2][threadIdx.x >> 5] = rmax; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, r = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += red[0][w]; b += red[1][w]; r = fmax(r, red[2][w]); }
        atomicAdd(&rec->shift2, a);
        if (b != 0.0) atomicAdd(&rec->empty, b);
        // non-negative doubles order like their bit patterns: a 64-bit atomicMax is a max
        if (r > 0.0)
            atomicMax(reinterpret_cast<unsigned long long*>(&rec->ub_inv),
                      (unsigned long long)__double_as_longlong(r));
        if (blockIdx.x == 0) {
            rec->sse = acc[L.sse()];
            rec->changed = acc[L.changed()];
        }
    }
}

// Segmented sums: pieces of kPiece rows (the unit whose sum depends only on the cluster's
// members); warps take chunks of C >= kPiece rows of perm, one wave of 32 warps per SM.
constexpr int64_t kPiece = 256;
int64_t segsum_chunk(int64_t n) {
    const int64_t warps = (int64_t)kNumSMs * 32;
    return std::max<int64_t>(kPiece, (n + warps - 1) / warps);
}

template <typename W>
cudaError_t update_dispatch(const W* X, int64_t n, int d, int k, const int32_t* labels, int* cnt,
                            int* offs, int* cursor, int* perm, double* acc, AccLayout L,
                            const UpdateScratch& us, cudaStream_t s) {
    int g = (int)std::min<int64_t>((n + 255) / 256, kNumSMs * 4);
    if (g < 1) g = 1;
    const bool det = k <= kHistMax;
    const int64_t nb = (n + kDetRows - 1) / kDetRows;
    if (det) {
        block_count_kernel<<<(unsigned)nb, kDetThreads, sizeof(int) * k, s>>>(labels, n, k, us.cb);
        block_scan_kernel<<<(unsigned)((k + 31) / 32), 1024, 0, s>>>(us.cb, nb, k, cnt);
    } else {
        cudaError_t e = cudaMemsetAsync(cnt, 0, sizeof(int) * k, s);
        if (e != cudaSuccess) return e;
        count_kernel<<<g, 256, 0, s>>>(labels, n, k, cnt);
    }
    const int64_t P = kPiece;
    scan_kernel<<<1, 1024, 0, s>>>(cnt, k, P, offs, cursor, us.mpo, acc + L.counts());
    if (det) {
        static PerDeviceOnce attr;
        if (attr.need()) {
            cudaFuncSetAttribute(scatter_det_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kDetHistBytes + kDetRows * (int)sizeof(int));
            attr.done();
        }
        scatter_det_kernel<<<(unsigned)nb, 32 * scatter_warps(k), scatter_smem(k), s>>>(
            labels, n, k, offs, us.cb, perm);
    } else
        scatter_kernel<<<g, 256, 0, s>>>(labels, n, cursor, perm);
    const int VEC = (sizeof(W) == 8) ? (d <= 32 ? 1 : 2) : (d <= 32 ? 1 : (d <= 64 ? 2 : 4));
    const int colblk = 32 * VEC;
    dim3 grid;
    const int64_t C = segsum_chunk(n);
    const int64_t nw = (n + C - 1) / C;
    grid.x = (unsigned)((nw + 7) / 8);
    grid.y = (unsigned)((d + colblk - 1) / colblk);
    grid.z = 1;
    double* sums = acc + L.sums();
#define SEGSUM(V) segsum_kernel<W, V, 8><<<grid, 256, 0, s>>>(X, n, d, k, perm, offs, us.mpo, P, C, \
                                                              sums, us.part)
    if constexpr (sizeof(W) == 8) {
        if (VEC == 1) SEGSUM(1); else SEGSUM(2);
    } else {
        if (VEC == 1) SEGSUM(1); else if (VEC == 2) SEGSUM(2); else SEGSUM(4);
    }
#undef SEGSUM
    segsum_fix_kernel<<<dim3((unsigned)k, (unsigned)((d + 31) / 32)), 256, 0, s>>>(d, us.mpo,
                                                                                  us.part, sums);
    return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// FX: the update with exact fixed-point sums (fp32 working precision, one rank, k <= kHistMax).
// Each coordinate is put on a per-feature grid g_t = 2^(e_t - 45) once (2^e_t > max_i |x_it|):
// q = i1 * 2^23 + i2 with |x - q g_t| <= g_t / 2 and |i1|, |i2| <= 2^22, obtained exactly from
// two fp32 adds against constants (fx_q below; host model and exactness proof in
// tests/test_fx_grid.py). A cluster's sum is the pair of int64 totals (sum i1, sum i2). Integer
// addition is associative, so the totals — and the centre RN_fp32((S_i1 2^23 + S_i2) g_t /
// count), formed exactly in K8 (fx_quot_rn: one rounding) — depend only on the cluster's
// members: the same whatever the summation order or history. That makes it legal
// to UPDATE the totals from the rows whose label changed (S[new] += q, S[old] -= q, integer
// atomics) instead of re-summing all n rows: both give the same bits. The full re-summation
// (U1-U4 above, integer accumulators) runs when the changed-row list overflows (the first
// iterations); afterwards each iteration reads only the changed rows (~0.1-1 % of n at C5).
// The grid costs 2^-46 max|x_t| per coordinate: far below u = 2^-24 of the means.
// Per-column max |x| (bits of a non-negative float order like unsigned ints) and flags[2] = 1 on
// a non-finite value. d % 4 == 0: a thread owns 4 adjacent columns, 16-byte loads, the next rows
// in flight; else a warp per row.
__global__ void __launch_bounds__(256)
fx_colmax_vec_kernel(const float* __restrict__ X, int64_t n, int d, unsigned* __restrict__ amax,
                     int* __restrict__ flags) {
    const int cg = d >> 2, lanes = 256 / cg;
    const int g = threadIdx.x % cg, lane = threadIdx.x / cg;
    __shared__ unsigned smax[1024];                   // d <= 1024
    for (int j = threadIdx.x; j < d; j += blockDim.x) smax[j] = 0u;
    __syncthreads();
    unsigned mx[4] = {0u, 0u, 0u, 0u};
    unsigned bad = 0;
    if (lane < lanes) {
        const float4* X4 = reinterpret_cast<const float4*>(X) + g;
        const int64_t step = (int64_t)gridDim.x * lanes;
        for (int64_t i0 = (int64_t)blockIdx.x * lanes + lane; i0 < n; i0 += 4 * step) {
            float4 v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t i = i0 + u * step;
                v[u] = i < n ? __ldg(X4 + i * cg) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float a[4] = {fabsf(v[u].x), fabsf(v[u].y), fabsf(v[u].z), fabsf(v[u].w)};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    if (!(a[e] <= 3.402823466e38f)) bad = 1;
                    else mx[e] = max(mx[e], __float_as_uint(a[e]));
                }
            }
        }
        // the block's maxima first: one global atomic per column and block (per thread, the
        // 64 columns of C3 took ~19k same-address atomics each)
#pragma unroll
        for (int e = 0; e < 4; ++e)
            if (mx[e]) atomicMax(&smax[4 * g + e], mx[e]);
    }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x)
        if (smax[j]) atomicMax(&amax[j], smax[j]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(&flags[2], 1);
}
__global__ void fx_colmax_kernel(const float* __restrict__ X, int64_t n, int d,
                                 unsigned* __restrict__ amax, int* __restrict__ flags) {
    extern __shared__ unsigned sm[];
    for (int j = threadIdx.x; j < d; j += blockDim.x) sm[j] = 0u;
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned bad = 0;
    for (int64_t i = warp; i < n; i += nwarps)
        for (int c = lane; c < d; c += 32) {
            const float v = fabsf(__ldg(X + i * d + c));
            if (!(v <= 3.402823466e38f)) bad = 1;
            else atomicMax(&sm[c], __float_as_uint(v));
        }
    __syncthreads();
    for (int j = threadIdx.x; j < d; j += blockDim.x)
        if (sm[j]) atomicMax(&amax[j], sm[j]);
    if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(&flags[2], 1);
}
__global__ void fx_scale_kernel(const unsigned* __restrict__ amax, int d, float2* __restrict__ c12,
                                double* __restrict__ g2, int* __restrict__ flags) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= d) return;
    int e = 0;
    frexp((double)__uint_as_float(amax[t]), &e);      // amax < 2^e (amax = 0: e = 0)
    if (e < -90 || e > 100) { atomicOr(&flags[2], 2); e = 0; }   // c2 / c1 out of fp32 range
    c12[t] = make_float2(ldexpf(1.5f, e + 1), ldexpf(1.5f, e - 22));
    g2[t] = ldexp(1.0, e - 45);
}
// The grid value of x, with fp32 adds and integer subtractions only. With |x| < 2^e (e from
// max |x_t|) and the constants c1 = 1.5 2^(e+1), c2 = 1.5 2^(e-22) of the feature:
//   t1 = RN(x + c1)  -> i1 = bits(t1) - bits(c1) = x / 2^(e-22) rounded (ties even), |i1| <= 2^22
//   r  = x - (t1 - c1)   (exact: Sterbenz, or x itself when t1 - c1 = 0)
//   t2 = RN(r + c2)  -> i2 = bits(t2) - bits(c2) = r / 2^(e-45) rounded, |i2| <= 2^22
// so x ~ q 2^(e-45) with q = i1 2^23 + i2 (t1, t2 stay in the binade of c1, c2, where ulps are
// 2^(e-22) and 2^(e-45); at the upper edge a bit difference still counts those ulps). A piece
// of <= 2^8 rows sums i1 and i2 in int32 without overflow; cluster totals are int64 pairs
// (H = sum i1, L = sum i2). The full re-summation and the incremental update call this same
// function, so both produce the same integers.
MPK_DEV void fx_q(float x, float2 c, int& i1, int& i2) {
    const float t1 = __fadd_rn(x, c.x);
    const float r = __fsub_rn(x, __fsub_rn(t1, c.x));
    const float t2 = __fadd_rn(r, c.y);
    i1 = __float_as_int(t1) - __float_as_int(c.x);
    i2 = __float_as_int(t2) - __float_as_int(c.y);
}
// Rows whose label changed since the previous iteration -> list (row, old, new); prev <- labels.
// gate[0] counts them; when gate[0] > gate[1] (capacity) the list is incomplete and the full
// re-summation runs instead.
__global__ void __launch_bounds__(256)
fx_diff_kernel(const int32_t* __restrict__ labels, int32_t* __restrict__ prev, int64_t n,
               int3* __restrict__ list, int* __restrict__ seg_cnt, int* __restrict__ gate) {
    // each warp lists the changed rows of its 32-row segments (one ballot: no slot atomics);
    // one count atomic per block and sweep (a single hot counter serialised the warps when many
    // rows change); any order of the list is fine (integer updates)
    constexpr int R = 4;                                  // rows per thread in flight
    __shared__ int wcount[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t span = (int64_t)blockDim.x * R;
    for (int64_t base = (int64_t)blockIdx.x * span; base < n; base += (int64_t)gridDim.x * span) {
        int l[R], o[R];
        int tot = 0;
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;
            l[u] = i < n ? __ldg(labels + i) : 0;
            o[u] = i < n ? prev[i] : 0;
        }
#pragma unroll
        for (int u = 0; u < R; ++u) {
            const int64_t i = base + u * blockDim.x + threadIdx.x;   // 32-aligned per warp
            const bool ch = i < n && l[u] != o[u];
            const unsigned m = __ballot_sync(0xffffffffu, ch);
            const int64_t seg = i >> 5;
            if (lane == 0 && i < n) seg_cnt[seg] = __popc(m);
            if (ch) {
                list[seg * 32 + __popc(m & ((1u << lane) - 1u))] = make_int3((int)i, o[u], l[u]);
                prev[i] = l[u];
            }
            tot += __popc(m);
        }
        if (lane == 0) wcount[warp] = tot;
        __syncthreads();
        if (threadIdx.x == 0) {
            int run = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) run += wcount[w];
            if (run) atomicAdd(&gate[0], run);
        }
        __syncthreads();                                  // wcount reused next sweep
    }
}
// Incremental update from the changed-row list: a warp per 32-row segment, its changed rows in
// turn, lanes over columns.
__global__ void __launch_bounds__(256)
fx_incr_kernel(const float* __restrict__ X, int64_t n, int d, const int3* __restrict__ list,
               const int* __restrict__ seg_cnt, const int* __restrict__ gate,
               const float2* __restrict__ sc, long long* __restrict__ Shi,
               long long* __restrict__ Slo, int* __restrict__ cnt) {
    griddep_wait();
    if (gate[0] > gate[1]) return;                        // the full path ran
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int64_t nseg = (n + 31) >> 5;
    for (int64_t sg = warp; sg < nseg; sg += nwarps) {
        const int c = seg_cnt[sg];
        for (int q = 0; q < c; ++q) {
            const int3 e = list[sg * 32 + q];
            const float* xr = X + (int64_t)e.x * d;
            for (int t = lane; t < d; t += 32) {
                int i1, i2;
                fx_q(__ldg(xr + t), sc[t], i1, i2);
                const long long hi = i1, lo = i2;
                atomicAdd(reinterpret_cast<unsigned long long*>(Shi + (int64_t)e.z * d + t), (unsigned long long)hi);
                atomicAdd(reinterpret_cast<unsigned long long*>(Slo + (int64_t)e.z * d + t), (unsigned long long)lo);
                if (e.y >= 0) {
                    atomicAdd(reinterpret_cast<unsigned long long*>(Shi + (int64_t)e.y * d + t), (unsigned long long)(-hi));
                    atomicAdd(reinterpret_cast<unsigned long long*>(Slo + (int64_t)e.y * d + t), (unsigned long long)(-lo));
                }
            }
            if (lane == 0) {
                atomicAdd(&cnt[e.z], 1);
                if (e.y >= 0) atomicSub(&cnt[e.y], 1);
            }
        }
    }
}
// U4 in fixed point (same pieces and traversal as segsum_kernel<float, VEC, U>; int64 totals).
template <int VEC, int U>
__global__ void __launch_bounds__(256, 4)
segsum_fx_kernel(const float* __restrict__ X, int64_t n, int d, int k, const int* __restrict__ perm,
                 const int* __restrict__ offs, const int* __restrict__ mpo, int64_t P, int64_t C,
                 const float2* __restrict__ sc, long long* __restrict__ Shi,
                 long long* __restrict__ Slo, long long* __restrict__ part, const int* gate) {
    griddep_wait();
    if (gated_off(gate)) return;
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int col0 = blockIdx.y * 32 * VEC + lane * VEC;
    const int ncols = max(0, min(VEC, d - col0));
    const bool aligned = (d % VEC) == 0;
    const int64_t e0 = warp * C;
    if (e0 >= n) return;
    const int64_t e1 = min(n, e0 + C);
    float2 scl[VEC];
#pragma unroll
    for (int q = 0; q < VEC; ++q) scl[q] = q < ncols ? sc[col0 + q] : make_float2(3.0f, 3.0f);
    int lo_ = 0, hi_ = k;
    while (hi_ - lo_ > 1) {
        int mid = (lo_ + hi_) >> 1;
        if (offs[mid] <= e0) lo_ = mid; else hi_ = mid;
    }
    int j = lo_;
    int64_t pidx = (e0 - offs[j] + P - 1) / P;
    int64_t ps = offs[j] + pidx * P;
    for (;;) {
        if (ps >= offs[j + 1]) {
            do { ++j; } while (j < k && offs[j] == offs[j + 1]);
            if (j >= k) break;
            pidx = 0;
            ps = offs[j];
        }
        if (ps >= e1) break;
        const int64_t pe = min((int64_t)offs[j + 1], ps + P);
        int ah[VEC], al[VEC];                         // <= 2^8 rows of |i| <= 2^22 each
#pragma unroll
        for (int q = 0; q < VEC; ++q) { ah[q] = 0; al[q] = 0; }
        for (int64_t e = ps; e < pe; e += 32) {
            const int myrow = (e + lane < pe) ? perm[e + lane] : 0;
            const int cnt = (int)min((int64_t)32, pe - e);
            for (int u0 = 0; u0 < cnt; u0 += U) {
                float xv[U][VEC];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int row = __shfl_sync(0xffffffffu, myrow, (u0 + u) & 31);
                    if (u0 + u < cnt && ncols > 0)
                        load_vec<float, VEC>(X + (int64_t)row * d + col0, aligned, ncols, xv[u]);
                    else {
#pragma unroll
                        for (int q = 0; q < VEC; ++q) xv[u][q] = 0.0f;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u)
#pragma unroll
                    for (int q = 0; q < VEC; ++q) {
                        int h, l;
                        fx_q(xv[u][q], scl[q], h, l);         // zero rows / columns add 0
                        ah[q] += h;
                        al[q] += l;
                    }
            }
        }
        const bool single = offs[j + 1] - offs[j] <= P;
        if (ncols > 0) {
#pragma unroll
            for (int q = 0; q < VEC; ++q)
                if (q < ncols) {
                    if (single) {
                        Shi[(int64_t)j * d + col0 + q] = (long long)ah[q];
                        Slo[(int64_t)j * d + col0 + q] = (long long)al[q];
                    } else {
                        long long* pp = part + (int64_t)(mpo[j] + pidx) * d * 2;
                        pp[col0 + q] = (long long)ah[q];
                        pp[d + col0 + q] = (long long)al[q];
                    }
                }
        }
        ++pidx;
        ps += P;
    }
}
// U4b in fixed point: the pieces of each multi-piece cluster (any order: integers); empty
// clusters get zero totals (the incremental path adds to them later).
__global__ void __launch_bounds__(256)
segsum_fix_fx_kernel(int d, const int* __restrict__ offs, const int* __restrict__ mpo,
                     const long long* __restrict__ part, long long* __restrict__ Shi,
                     long long* __restrict__ Slo, const int* gate) {
    griddep_wait();
    if (gated_off(gate)) return;
    const int j = blockIdx.x;
    const int np = mpo[j + 1] - mpo[j];
    const int col = blockIdx.y * 32 + (threadIdx.x & 31);
    const int w = threadIdx.x >> 5;
    if (offs[j + 1] == offs[j]) {                         // empty cluster
        if (w == 0 && col < d) { Shi[(int64_t)j * d + col] = 0; Slo[(int64_t)j * d + col] = 0; }
        return;
    }
    if (np == 0) return;
    __shared__ long long red[2][8][32];
    long long sh = 0, sl = 0;
    if (col < d) {
        const long long* pp = part + (int64_t)mpo[j] * d * 2 + col;
        for (int p = w; p < np; p += 8) { sh += pp[(int64_t)p * d * 2]; sl += pp[(int64_t)p * d * 2 + d]; }
    }
    red[0][w][threadIdx.x & 31] = sh;
    red[1][w][threadIdx.x & 31] = sl;
    __syncthreads();
    if (w == 0 && col < d) {
        long long a = 0, b = 0;
#pragma unroll
        for (int q = 0; q < 8; ++q) { a += red[0][q][threadIdx.x & 31]; b += red[1][q][threadIdx.x & 31]; }
        Shi[(int64_t)j * d + col] = a;
        Slo[(int64_t)j * d + col] = b;
    }
}
// RN_fp32(Q 2^x / m) for Q = H 2^23 + L, computed exactly with one rounding (ties to even):
// Q in 128-bit integers, shifted so the quotient carries >= 26 bits, divided by m in four
// 32-bit limbs (remainder = sticky), rounded to 24 bits. The result is exact-then-rounded
// unless it falls in fp32's subnormal range (then ldexpf rounds a second time).
MPK_DEV float fx_quot_rn(long long H, long long L, int x, int m) {
    const __int128 Q = (__int128)H * 8388608 + (__int128)L;
    if (Q == 0 || m <= 0) return 0.0f;
    const bool neg = Q < 0;
    unsigned __int128 A = neg ? (unsigned __int128)(-Q) : (unsigned __int128)Q;
    const uint64_t ah = (uint64_t)(A >> 64), al = (uint64_t)A;
    const int la = ah ? 128 - __clzll((long long)ah) : 64 - __clzll((long long)al);
    const int s = la < 58 ? 58 - la : 0;     // A 2^s >= 2^57 > 2^25 m: the quotient has >= 26 bits
    A <<= s;
    uint64_t r = 0;
    uint64_t qd[4];
#pragma unroll
    for (int i = 3; i >= 0; --i) {
        const uint64_t cur = (r << 32) | (uint64_t)(uint32_t)(A >> (32 * i));
        qd[i] = cur / (uint64_t)m;
        r = cur - qd[i] * (uint64_t)m;
    }
    const uint64_t qh = (qd[3] << 32) | qd[2], ql = (qd[1] << 32) | qd[0];
    const unsigned __int128 qt = ((unsigned __int128)qh << 64) | ql;
    const int lq = qh ? 128 - __clzll((long long)qh) : 64 - __clzll((long long)ql);
    const int sh = lq - 24;                  // >= 2
    uint64_t mant = (uint64_t)(qt >> sh);
    const unsigned __int128 low = qt & ((((unsigned __int128)1) << sh) - 1);
    const unsigned __int128 half = ((unsigned __int128)1) << (sh - 1);
    if (low > half || (low == half && (r != 0 || (mant & 1)))) ++mant;   // mant <= 2^24: exact
    const float v = ldexpf((float)mant, sh - s + x);
    return neg ? -v : v;
}

// K8 from the fixed-point totals: c_j = RN_fp32((S_i1 2^23 + S_i2) 2^(e_t-45) / count_j) with one
// rounding (fx_quot_rn); the rest as finalize_kernel (shift^2, empty clusters keep their centre,
// Thm 5.3 terms, trace record).
__global__ void finalize_fx_kernel(int64_t k, int d, const long long* __restrict__ Shi,
                                   const long long* __restrict__ Slo, const int* __restrict__ cnt,
                                   const double* __restrict__ isc, double* __restrict__ acc,
                                   AccLayout L, float* __restrict__ C, IterRec* __restrict__ rec,
                                   int* __restrict__ gate0) {
    griddep_wait();
    const int lane = threadIdx.x & 31;
    const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    double sh = 0.0, empty = 0.0, rmax = 0.0;
    for (int64_t j = warp; j < k; j += nwarps) {
        const double c = (double)cnt[j];
        double num = 0.0, den = 0.0;
        for (int t = lane; t < d; t += 32) {
            const int64_t idx = j * d + t;
            const float old = C[idx];
            float nw = old;
            if (c > 0.0) nw = fx_quot_rn(Shi[idx], Slo[idx], ilogb(isc[t]), cnt[j]);
            const double df = (double)nw - (double)old;
            num += df * df;
            den += fabs(df) * fabs((double)nw);
            C[idx] = nw;
        }
        num = warp_sum(num);
        den = warp_sum(den);
        if (lane == 0) {
            sh += num;
            if (c == 0.0) empty += 1.0;
            if (num > 0.0 && den > 0.0) rmax = fmax(rmax, 2.0 * den / num);
        }
    }
    __shared__ double red[3][8];
    if (lane == 0) { red[0][threadIdx.x >> 5] = sh; red[1][threadIdx.x >> 5] = empty; red[2][threadIdx.x >> 5] = rmax; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, r = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) { a += red[0][w]; b += red[1][w]; r = fmax(r, red[2][w]); }
        atomicAdd(&rec->shift2, a);
        if (b != 0.0) atomicAdd(&rec->empty, b);
        if (r > 0.0)
            atomicMax(reinterpret_cast<unsigned long long*>(&rec->ub_inv),
                      (unsigned long long)__double_as_longlong(r));
        if (blockIdx.x == 0) {
            rec->sse = acc[L.sse()];
            rec->changed = acc[L.changed()];
            // zeroed here for the next iteration's distance kernel (instead of memsets between
            // the iteration's kernels, which would break their programmatic dependent launches)
            acc[L.sse()] = 0.0;
            acc[L.changed()] = 0.0;
            if (gate0) *gate0 = 0;
        }
    }
}

}  // namespace

cudaError_t launch_update(int work, const void* Xw, int64_t n, int d, int k,
                          const int32_t* labels, int* cnt, int* offs, int* cursor, int* perm,
                          double* acc, AccLayout L, const UpdateScratch& us, cudaStream_t s) {
    launches_add(6);
    if (work == KMEANS_FP64)
        return update_dispatch<double>((const double*)Xw, n, d, k, labels, cnt, offs, cursor,
                                       perm, acc, L, us, s);
    return update_dispatch<float>((const float*)Xw, n, d, k, labels, cnt, offs, cursor, perm, acc,
                                  L, us, s);
}

size_t update_scratch_bytes(int64_t n, int d, int k, size_t* cb, size_t* part, size_t* mpo) {
    const int64_t nb = (n + kDetRows - 1) / kDetRows;
    // clusters with >= 2 pieces have > P rows each: sum ceil(c_j / P) <= 2 n / P slots
    const int64_t slots = 2 * ((n + kPiece - 1) / kPiece) + 1;
    *cb = (size_t)(k <= kHistMax ? nb * k : 1) * sizeof(int);
    *part = (size_t)slots * d * sizeof(double);
    *mpo = (size_t)(k + 1) * sizeof(int);
    return *cb + *part + *mpo;
}

cudaError_t launch_finalize(int work, int64_t k, int d, const double* acc, AccLayout L, void* Cw,
                            IterRec* rec, cudaStream_t s) {
    launches_add(1);
    int g = (int)std::min<int64_t>((k + 7) / 8, kNumSMs * 2);   // one warp per cluster
    if (g < 1) g = 1;
    if (work == KMEANS_FP64)
        finalize_kernel<double><<<g, 256, 0, s>>>(k, d, acc, L, (double*)Cw, rec);
    else
        finalize_kernel<float><<<g, 256, 0, s>>>(k, d, acc, L, (float*)Cw, rec);
    return cudaGetLastError();
}

// ---- FX public entry points (internal.h) ---------------------------------------------------
// amax and gate are zeroed by the caller before the point prep (which may fill amax itself:
// have_amax skips the pass over X here)
cudaError_t launch_fx_colmax(const float* Xw, int64_t n, int d, FxState& fx, bool have_amax,
                             cudaStream_t s) {
    if (have_amax) return cudaSuccess;
    launches_add(1);
    if (d % 4 == 0 && d <= 1024 && ((uintptr_t)Xw & 15) == 0) {
        fx_colmax_vec_kernel<<<kNumSMs * 8, 256, 0, s>>>(Xw, n, d, fx.amax, fx.gate);
    } else {
        int g = (int)std::min<int64_t>((n + 7) / 8, kNumSMs * 8);
        if (g < 1) g = 1;
        fx_colmax_kernel<<<g, 256, sizeof(unsigned) * d, s>>>(Xw, n, d, fx.amax, fx.gate);
    }
    return cudaGetLastError();
}
// (several ranks: amax and gate[2] are max-allreduced between the two calls, so every rank
// uses the same grid)
cudaError_t launch_fx_scale(int d, FxState& fx, cudaStream_t s) {
    launches_add(1);
    fx_scale_kernel<<<(d + 127) / 128, 128, 0, s>>>(fx.amax, d, fx.sc, fx.isc, fx.gate);
    return cudaGetLastError();
}

cudaError_t launch_update_fx(const float* Xw, int64_t n, int d, int k, const int32_t* labels,
                             int* cnt, int* offs, int* cursor, int* perm, const UpdateScratch& us,
                             FxState& fx, cudaStream_t s, bool listed) {
    launches_add(listed ? 7 : 8);     // [diff,] 6 gated full-path kernels, incremental
    if (!listed) {
        // gate[0] = changed rows (reset), gate[1] = capacity (kept)
        cudaError_t e = cudaMemsetAsync(fx.gate, 0, sizeof(int), s);
        if (e != cudaSuccess) return e;
        int g = (int)std::min<int64_t>((n + 1023) / 1024, kNumSMs * 8);
        if (g < 1) g = 1;
        fx_diff_kernel<<<g, 256, 0, s>>>(labels, fx.prev, n, fx.list, fx.seg_cnt, fx.gate);
    }
    const int* gate = fx.gate;
    // full re-summation, gated: runs only when the list overflowed
    const int64_t nb = (n + kDetRows - 1) / kDetRows;
    // the chain below is launched with programmatic dependent launch (each kernel waits for its
    // predecessor first): the launch latency of the gated-off kernels overlaps
    launch_pdl(block_count_kernel, dim3((unsigned)nb), dim3(kDetThreads), sizeof(int) * k, s,
               labels, n, k, us.cb, gate);
    launch_pdl(block_scan_kernel, dim3((unsigned)((k + 31) / 32)), dim3(1024), 0, s, us.cb, nb, k,
               cnt, gate);
    const int64_t P = kPiece;
    launch_pdl(scan_kernel, dim3(1), dim3(1024), 0, s, (const int*)cnt, k, P, offs, cursor, us.mpo,
               (double*)nullptr, gate);
    static PerDeviceOnce attr;
    if (attr.need()) {
        cudaFuncSetAttribute(scatter_det_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kDetHistBytes + kDetRows * (int)sizeof(int));
        attr.done();
    }
    launch_pdl(scatter_det_kernel, dim3((unsigned)nb), dim3(32 * scatter_warps(k)), scatter_smem(k),
               s, labels, n, k, (const int*)offs, (const int*)us.cb, perm, gate);
    const int VEC = d <= 32 ? 1 : (d <= 64 ? 2 : 4);
    const int colblk = 32 * VEC;
    const int64_t C = segsum_chunk(n);
    const int64_t nw = (n + C - 1) / C;
    dim3 grid((unsigned)((nw + 7) / 8), (unsigned)((d + colblk - 1) / colblk), 1);
#define SEGSUMFX(V) launch_pdl(segsum_fx_kernel<V, 8>, grid, dim3(256), 0, s, Xw, n, d, k, (const int*)perm, \
                                (const int*)offs, (const int*)us.mpo, P, C, (const float2*)fx.sc, fx.Shi, \
                                fx.Slo, fx.part, gate)
    if (VEC == 1) SEGSUMFX(1); else if (VEC == 2) SEGSUMFX(2); else SEGSUMFX(4);
#undef SEGSUMFX
    launch_pdl(segsum_fix_fx_kernel, dim3((unsigned)k, (unsigned)((d + 31) / 32)), dim3(256), 0, s,
               d, (const int*)offs, (const int*)us.mpo, (const long long*)fx.part, fx.Shi, fx.Slo, gate);
    // incremental update, gated the other way
    launch_pdl(fx_incr_kernel, dim3(kNumSMs * 4), dim3(256), 0, s, Xw, n, d, (const int3*)fx.list,
               (const int*)fx.seg_cnt, gate, (const float2*)fx.sc, fx.Shi, fx.Slo, cnt);
    return cudaGetLastError();
}

cudaError_t launch_finalize_fx(int64_t k, int d, const FxState& fx, const long long* Shi,
                               const long long* Slo, const int* cnt, const double* acc,
                               AccLayout L, float* Cw, IterRec* rec, cudaStream_t s) {
    launches_add(1);
    int g = (int)std::min<int64_t>((k + 7) / 8, kNumSMs * 2);
    if (g < 1) g = 1;
    launch_pdl(finalize_fx_kernel, dim3(g), dim3(256), 0, s, k, d, Shi, Slo, cnt,
               (const double*)fx.isc, const_cast<double*>(acc), L, Cw, rec, fx.gate);
    return cudaGetLastError();
}

size_t fx_part_bytes(int64_t n, int d) {
    const int64_t slots = 2 * ((n + kPiece - 1) / kPiece) + 1;
    return (size_t)slots * d * 2 * sizeof(long long);
}

}  // namespace mpk
