// coll.cu — the cross-rank exchange of the point-sharded path behind one
// interface, with two transports:
//   * NcclColl: one NCCL communicator per handle (one process per GPU, NVLink / NVSwitch);
//   * VColl: "virtual ranks" — g handles in ONE process on ONE device (kmeans_vgroup_*), each
//     driven by its own host thread exactly like a torchrun rank. Every per-rank step (shard
//     statistics, per-shard fixed-point totals, counts, SSE_t partials, final SSE) runs the same
//     code as with NCCL; only the collective itself differs: the last rank to arrive sums the
//     g contributions on the device in rank order and every rank's stream waits for that.
// The paper treats parallel k-means only as related work; the exchange is
// the sum over shards of eq:center's per-cluster sums and counts.
#include <cuda_runtime.h>
#include <nccl.h>

#include <string.h>

#include <algorithm>
#include <condition_variable>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "internal.h"

namespace mpk {

namespace {

size_t coll_esize(int t) { return (t == CT_F64 || t == CT_I64) ? 8 : 4; }

ncclDataType_t nccl_type(int t) {
    switch (t) {
        case CT_F64: return ncclDouble;
        case CT_I64: return ncclInt64;
        case CT_I32: return ncclInt32;
        default: return ncclUint32;
    }
}

ncclRedOp_t nccl_op(int op) { return op == CO_SUM ? ncclSum : (op == CO_MAX ? ncclMax : ncclMin); }

struct NcclColl final : Coll {
    ncclComm_t comm = nullptr;
    ~NcclColl() override {
        if (comm) ncclCommDestroy(comm);
    }
    int allreduce(const void* send, void* recv, size_t count, int type, int op, cudaStream_t s,
                  std::string* err) override {
        ncclResult_t r = ncclAllReduce(send, recv, count, nccl_type(type), nccl_op(op), comm, s);
        if (r != ncclSuccess) {
            *err = std::string("ncclAllReduce: ") + ncclGetErrorString(r);
            return KMEANS_ENCCL;
        }
        return 0;
    }
    void group_start() override { ncclGroupStart(); }
    int group_end(std::string* err) override {
        ncclResult_t r = ncclGroupEnd();
        if (r != ncclSuccess) {
            *err = std::string("ncclGroupEnd: ") + ncclGetErrorString(r);
            return KMEANS_ENCCL;
        }
        return 0;
    }
};

// ---- virtual ranks ----------------------------------------------------------------------------

constexpr int kMaxVRanks = 64;

struct VSlot {
    const void* send;
    void* recv;
};

// out[e] = op over ranks r = 0..g-1 (in that order) of send_r[e]
template <typename T>
__global__ void vreduce_kernel(VSlot* slots, int g, size_t count, int op, T* out) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
         e += (size_t)gridDim.x * blockDim.x) {
        T a = ((const T*)slots[0].send)[e];
        for (int r = 1; r < g; ++r) {
            const T b = ((const T*)slots[r].send)[e];
            a = op == CO_SUM ? (T)(a + b) : (op == CO_MAX ? (b > a ? b : a) : (b < a ? b : a));
        }
        out[e] = a;
    }
}

template <typename T>
__global__ void vscatter_kernel(VSlot* slots, int g, size_t count, const T* in) {
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < count;
         e += (size_t)gridDim.x * blockDim.x) {
        const T v = in[e];
        for (int r = 0; r < g; ++r) ((T*)slots[r].recv)[e] = v;
    }
}

}  // namespace

struct VGroup {
    int g = 0;
    int device = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    unsigned long long generation = 0;
    int status = 0;
    std::string status_msg;
    // the pending collective
    size_t count = 0;
    int type = 0, op = 0;
    VSlot host_slots[kMaxVRanks];
    cudaStream_t rank_stream[kMaxVRanks];
    cudaEvent_t rank_ev[kMaxVRanks];
    // device side
    cudaStream_t stream = nullptr;
    cudaEvent_t done = nullptr;
    VSlot* dev_slots = nullptr;   // one slot array per collective in flight (ring)
    int slot_ring = 0;
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    int members = 0;              // live handles (destroy waits for 0)

    ~VGroup() {
        for (int r = 0; r < g; ++r)
            if (rank_ev[r]) cudaEventDestroy(rank_ev[r]);
        if (done) cudaEventDestroy(done);
        if (dev_slots) cudaFree(dev_slots);
        if (scratch) cudaFree(scratch);
        if (stream) cudaStreamDestroy(stream);
    }

    // Run by the last rank to arrive, under mu: enqueue the reduction on the group stream.
    int launch_reduce(std::string* err) {
        const size_t es = coll_esize(type), bytes = count * es;
        if (bytes > scratch_bytes) {
            if (scratch) cudaFree(scratch);
            scratch = nullptr;
            scratch_bytes = 0;
            if (cudaMalloc(&scratch, bytes) != cudaSuccess) {
                cudaGetLastError();
                *err = "virtual allreduce: scratch allocation failed";
                return KMEANS_ENOMEM;
            }
            scratch_bytes = bytes;
        }
        for (int r = 0; r < g; ++r) {
            cudaEventRecord(rank_ev[r], rank_stream[r]);
            cudaStreamWaitEvent(stream, rank_ev[r], 0);
        }
        // slot arrays rotate through a ring so that an in-flight reduction's slots are never
        // overwritten by the next collective's host copy (the copy is ordered on the same stream,
        // so one slot array would do; the ring keeps the H2D source buffer stable too)
        VSlot* ds = dev_slots + (size_t)slot_ring * kMaxVRanks;
        slot_ring = (slot_ring + 1) % 8;
        cudaMemcpyAsync(ds, host_slots, sizeof(VSlot) * g, cudaMemcpyHostToDevice, stream);
        const unsigned blocks = (unsigned)std::min<size_t>((count + 255) / 256, 4 * (size_t)kNumSMs);
        if (blocks > 0) {
            switch (type) {
                case CT_F64:
                    vreduce_kernel<double><<<blocks, 256, 0, stream>>>(ds, g, count, op, (double*)scratch);
                    vscatter_kernel<double><<<blocks, 256, 0, stream>>>(ds, g, count, (const double*)scratch);
                    break;
                case CT_I64:
                    vreduce_kernel<long long><<<blocks, 256, 0, stream>>>(ds, g, count, op, (long long*)scratch);
                    vscatter_kernel<long long><<<blocks, 256, 0, stream>>>(ds, g, count, (const long long*)scratch);
                    break;
                case CT_I32:
                    vreduce_kernel<int><<<blocks, 256, 0, stream>>>(ds, g, count, op, (int*)scratch);
                    vscatter_kernel<int><<<blocks, 256, 0, stream>>>(ds, g, count, (const int*)scratch);
                    break;
                default:
                    vreduce_kernel<unsigned><<<blocks, 256, 0, stream>>>(ds, g, count, op, (unsigned*)scratch);
                    vscatter_kernel<unsigned><<<blocks, 256, 0, stream>>>(ds, g, count, (const unsigned*)scratch);
            }
            launches_add(2);
        }
        // the host slot array is re-filled by the next collective only after every rank has
        // left this one; the H2D copy above reads pageable memory synchronously w.r.t. the host
        cudaEventRecord(done, stream);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) {
            *err = std::string("virtual allreduce: ") + cudaGetErrorString(e);
            return KMEANS_ECUDA;
        }
        return 0;
    }
};

namespace {

struct VColl final : Coll {
    VGroup* grp;
    explicit VColl(VGroup* g) : grp(g) {}
    // one GPU: the ranks' work is serialised on the group's stream (their kernels never wait on
    // one another on the device; only the host threads meet at each collective)
    cudaStream_t shared_stream() override { return grp->stream; }
    ~VColl() override {
        std::lock_guard<std::mutex> lk(grp->mu);
        grp->members--;
    }
    int allreduce(const void* send, void* recv, size_t count, int type, int op, cudaStream_t s,
                  std::string* err) override {
        VGroup& G = *grp;
        std::unique_lock<std::mutex> lk(G.mu);
        const unsigned long long gen = G.generation;
        if (G.arrived == 0) {
            G.count = count; G.type = type; G.op = op;
            G.status = 0;
        } else if (G.count != count || G.type != type || G.op != op) {
            // mismatched collectives: a programming error of the caller (ranks diverged)
            G.status = KMEANS_EINVAL;
            G.status_msg = "virtual allreduce: ranks issued different collectives";
        }
        G.host_slots[rank] = VSlot{send, recv};
        G.rank_stream[rank] = s;
        if (++G.arrived == G.g) {
            if (G.status == 0) G.status = G.launch_reduce(&G.status_msg);
            G.arrived = 0;
            G.generation++;
            G.cv.notify_all();
        } else {
            G.cv.wait(lk, [&] { return G.generation != gen; });
        }
        if (G.status != 0) {
            *err = G.status_msg;
            return G.status;
        }
        // every rank's later work waits for the reduction (recorded before the release above)
        if (cudaStreamWaitEvent(s, G.done, 0) != cudaSuccess) {
            cudaGetLastError();
            *err = "virtual allreduce: cudaStreamWaitEvent failed";
            return KMEANS_ECUDA;
        }
        return 0;
    }
};

}  // namespace

Coll* coll_create_nccl(const void* nccl_id, int nranks, int rank, std::string* err) {
    ncclUniqueId id;
    memcpy(&id, nccl_id, sizeof(id));
    NcclColl* c = new NcclColl();
    ncclResult_t r = ncclCommInitRank(&c->comm, nranks, id, rank);
    if (r != ncclSuccess) {
        *err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
        c->comm = nullptr;
        delete c;
        return nullptr;
    }
    c->nranks = nranks;
    c->rank = rank;
    c->virtual_ranks = false;
    return c;
}

Coll* coll_create_virtual(VGroup* g, int rank, std::string* err) {
    if (!g || rank < 0 || rank >= g->g) {
        *err = "bad virtual group / rank";
        return nullptr;
    }
    {
        std::lock_guard<std::mutex> lk(g->mu);
        g->members++;
    }
    VColl* c = new VColl(g);
    c->nranks = g->g;
    c->rank = rank;
    c->virtual_ranks = true;
    return c;
}

VGroup* vgroup_create(int nranks, std::string* err) {
    if (nranks < 1 || nranks > kMaxVRanks) {
        *err = "virtual group size must be in [1, 64]";
        return nullptr;
    }
    VGroup* g = new VGroup();
    g->g = nranks;
    cudaGetDevice(&g->device);
    for (int r = 0; r < kMaxVRanks; ++r) { g->rank_ev[r] = nullptr; g->rank_stream[r] = nullptr; }
    bool ok = cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking) == cudaSuccess &&
              cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming) == cudaSuccess &&
              cudaMalloc(&g->dev_slots, sizeof(VSlot) * kMaxVRanks * 8) == cudaSuccess;
    for (int r = 0; ok && r < nranks; ++r)
        ok = cudaEventCreateWithFlags(&g->rank_ev[r], cudaEventDisableTiming) == cudaSuccess;
    if (!ok) {
        cudaGetLastError();
        *err = "virtual group: CUDA stream/event/allocation failed";
        delete g;
        return nullptr;
    }
    return g;
}

int vgroup_size(const VGroup* g) { return g ? g->g : 0; }

int vgroup_destroy(VGroup* g) {
    if (!g) return 0;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        if (g->members > 0) return KMEANS_EINVAL;
    }
    cudaStreamSynchronize(g->stream);
    delete g;
    return 0;
}

}  // namespace mpk
