// fake_nccl.cu -- TEST INFRASTRUCTURE: a loopback stand-in for libnccl.so.2.
//
// The product resolves NCCL through a function table (csrc/ctx.cu: NcclApi); with the environment variable
// REGOT_B200_NCCL_LIB pointing at this library the row-sharded device path (world > 1: allreduce of the
// column sums, histograms, tie counts, B't, ...) runs for real on ONE GPU: R contexts, one per rank, driven
// from R threads of one process.  Only the five entry points the product binds are implemented.
//
// ncclAllReduce here: every rank's thread records an event on its stream and waits on the host until all R
// ranks of the communicator have called; the last one to arrive makes a helper stream wait for the R
// events, launches one kernel that reduces the R send buffers in RANK ORDER (deterministic) into the R
// receive buffers, and makes every rank's stream wait for that kernel.  Like NCCL, the call returns with
// the reduction enqueued, not complete.
#include <cuda_runtime.h>
#include <nccl.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>

namespace {

constexpr int kMaxRanks = 8;
constexpr int kTimeoutSeconds = 120;

struct Group {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int joined = 0, left = 0;
    int arrived = 0;
    unsigned long long generation = 0;
    const void* send[kMaxRanks];
    void* recv[kMaxRanks];
    cudaStream_t stream[kMaxRanks];
    cudaEvent_t ready[kMaxRanks];
    size_t count[kMaxRanks];
    int dtype[kMaxRanks], op[kMaxRanks];
    cudaStream_t helper = nullptr;
    cudaEvent_t done = nullptr;
    bool failed = false;
};

std::mutex g_mu;
std::map<std::string, std::shared_ptr<Group>> g_groups;
std::atomic<unsigned long long> g_ids{1};

struct Ptrs {
    const void* send[kMaxRanks];
    void* recv[kMaxRanks];
};

template <class T, bool kMax>
__global__ void k_reduce(int world, size_t count, Ptrs p)
{
    for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
        T v = static_cast<const T*>(p.send[0])[i];
        for (int r = 1; r < world; ++r) {
            const T x = static_cast<const T*>(p.send[r])[i];
            v = kMax ? (x > v ? x : v) : v + x;
        }
        for (int r = 0; r < world; ++r) static_cast<T*>(p.recv[r])[i] = v;
    }
}

}  // namespace

struct ncclComm {
    std::shared_ptr<Group> group;
    int rank;
};

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id)
{
    std::memset(id, 0, sizeof(*id));
    std::snprintf(id->internal, sizeof(id->internal), "regot-loopback-%llu", g_ids.fetch_add(1));
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int world, ncclUniqueId id, int rank)
{
    if (world < 1 || world > kMaxRanks || rank < 0 || rank >= world) return ncclInvalidArgument;
    std::shared_ptr<Group> g;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto& slot = g_groups[std::string(id.internal, sizeof(id.internal))];
        if (!slot) {
            slot = std::make_shared<Group>();
            slot->world = world;
        }
        g = slot;
    }
    if (g->world != world) return ncclInvalidArgument;
    std::unique_lock<std::mutex> lk(g->mu);
    if (!g->helper) {
        if (cudaStreamCreateWithFlags(&g->helper, cudaStreamNonBlocking) != cudaSuccess) return ncclUnhandledCudaError;
        if (cudaEventCreateWithFlags(&g->done, cudaEventDisableTiming) != cudaSuccess) return ncclUnhandledCudaError;
    }
    if (cudaEventCreateWithFlags(&g->ready[rank], cudaEventDisableTiming) != cudaSuccess) return ncclUnhandledCudaError;
    ++g->joined;
    g->cv.notify_all();
    // like NCCL: returns once every rank has joined (bounded: a rank that died must not hang the test run)
    if (!g->cv.wait_for(lk, std::chrono::seconds(kTimeoutSeconds), [&] { return g->joined >= g->world; })) return ncclSystemError;
    *comm = new ncclComm{g, rank};
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm)
{
    if (!comm) return ncclSuccess;
    {
        std::lock_guard<std::mutex> lk(comm->group->mu);
        cudaEventDestroy(comm->group->ready[comm->rank]);
        if (++comm->group->left == comm->group->world) {
            cudaStreamSynchronize(comm->group->helper);
            cudaStreamDestroy(comm->group->helper);
            cudaEventDestroy(comm->group->done);
        }
    }
    delete comm;
    return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t r)
{
    switch (r) {
    case ncclSuccess: return "no error";
    case ncclUnhandledCudaError: return "loopback: unhandled cuda error";
    case ncclInvalidArgument: return "loopback: invalid argument";
    case ncclSystemError: return "loopback: timed out waiting for the other ranks";
    case ncclInvalidUsage: return "loopback: ranks disagree on the collective (count / type / op)";
    default: return "loopback: error";
    }
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t dtype, ncclRedOp_t op,
                           ncclComm_t comm, cudaStream_t stream)
{
    Group& g = *comm->group;
    const int rank = comm->rank;
    const bool known = (dtype == ncclDouble && (op == ncclSum || op == ncclMax)) || (dtype == ncclUint64 && op == ncclSum);
    if (!known) return ncclInvalidArgument;
    if (cudaEventRecord(g.ready[rank], stream) != cudaSuccess) return ncclUnhandledCudaError;
    std::unique_lock<std::mutex> lk(g.mu);
    g.send[rank] = send;
    g.recv[rank] = recv;
    g.stream[rank] = stream;
    g.count[rank] = count;
    g.dtype[rank] = (int)dtype;
    g.op[rank] = (int)op;
    const unsigned long long gen = g.generation;
    if (++g.arrived == g.world) {
        bool ok = true;
        for (int r = 1; r < g.world; ++r) ok &= g.count[r] == g.count[0] && g.dtype[r] == g.dtype[0] && g.op[r] == g.op[0];
        Ptrs p;
        for (int r = 0; r < g.world; ++r) {
            p.send[r] = g.send[r];
            p.recv[r] = g.recv[r];
            ok &= cudaStreamWaitEvent(g.helper, g.ready[r], 0) == cudaSuccess;
        }
        if (ok && count > 0) {
            const int grid = (int)((count + 255) / 256 < 1184 ? (count + 255) / 256 : 1184);
            if (dtype == ncclUint64) k_reduce<unsigned long long, false><<<grid, 256, 0, g.helper>>>(g.world, count, p);
            else if (op == ncclMax) k_reduce<double, true><<<grid, 256, 0, g.helper>>>(g.world, count, p);
            else k_reduce<double, false><<<grid, 256, 0, g.helper>>>(g.world, count, p);
            ok &= cudaGetLastError() == cudaSuccess;
        }
        ok &= cudaEventRecord(g.done, g.helper) == cudaSuccess;
        for (int r = 0; r < g.world; ++r) ok &= cudaStreamWaitEvent(g.stream[r], g.done, 0) == cudaSuccess;
        g.failed = !ok;
        g.arrived = 0;
        ++g.generation;
        g.cv.notify_all();
    } else {
        if (!g.cv.wait_for(lk, std::chrono::seconds(kTimeoutSeconds), [&] { return g.generation != gen; })) {
            --g.arrived;  // a peer never called (it failed): give up instead of hanging the test run
            return ncclSystemError;
        }
    }
    return g.failed ? ncclInvalidUsage : ncclSuccess;
}

}  // extern "C"
