// mock_nccl.cu — TEST INFRASTRUCTURE (never linked into the product): an in-process stand-in for the
// NCCL calls the library's data plane makes (csrc/comm.cpp), so a world-2 job can run on the one GPU
// of the test box. The library dlopens it through OSPLAT_NCCL_LIB; every "rank" is a context driven
// by its own host thread in one process, on the same device.
//
// A collective: each rank records an event on its stream (inputs ready) and meets the others at a
// barrier (pointers + events exchanged); each rank's stream then waits for every rank's inputs, runs
// a kernel that reads the peers' buffers directly (same device) and writes its own output, records
// a second event, and after a second barrier waits for every rank's kernel before going on — so no
// rank overwrites a buffer a peer still reads. Sums run over ranks 0..world-1 in order.
// Supported: ReduceScatter (sum, f32), AllGather (f32), AllReduce (sum / max; f32, f64, i32),
// group start / end (no-ops: every rank issues the same sequence).
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstring>
#include <map>
#include <mutex>
#include <random>
#include <string>
#include <vector>

namespace {

constexpr int kMaxRanks = 8;

struct Slot {
    const void* send = nullptr;
    void* recv = nullptr;
    cudaEvent_t ready = nullptr, done = nullptr;
};

struct Group {
    int world = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    Slot slots[kMaxRanks];
    // all ranks arrive (publishing their slot), then each gets a copy of every slot
    void meet(int rank, const Slot& mine, Slot* all) {
        std::unique_lock<std::mutex> lk(mu);
        slots[rank] = mine;
        const long g = gen;
        if (++arrived == world) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
        for (int k = 0; k < world; ++k) all[k] = slots[k];
    }
};

std::mutex g_registry_mu;
std::map<std::string, Group*>& registry() {
    static std::map<std::string, Group*> r;
    return r;
}

struct Ptrs {
    const void* p[kMaxRanks];
};

template <typename T>
__device__ __forceinline__ T op2(T a, T b, int op) {
    return op == ncclMax ? (a > b ? a : b) : a + b;
}

template <typename T>
__global__ void k_reduce(Ptrs in, int world, size_t offset, size_t count, T* out, int op) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        T acc = static_cast<const T*>(in.p[0])[offset + i];
        for (int k = 1; k < world; ++k) acc = op2(acc, static_cast<const T*>(in.p[k])[offset + i], op);
        out[i] = acc;
    }
}

template <typename T>
__global__ void k_gather(Ptrs in, int world, size_t count, T* out) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < count * world;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const size_t k = i / count, e = i - k * count;
        out[i] = static_cast<const T*>(in.p[k])[e];
    }
}

}  // namespace

struct ncclComm {
    Group* g;
    int rank;
    cudaEvent_t ready, done;
};

namespace {

template <typename Launch>
ncclResult_t collective(ncclComm_t c, const void* send, void* recv, cudaStream_t s, Launch launch) {
    Slot mine, all[kMaxRanks];
    mine.send = send;
    mine.recv = recv;
    mine.ready = c->ready;
    mine.done = c->done;
    if (cudaEventRecord(c->ready, s) != cudaSuccess) return ncclUnhandledCudaError;
    c->g->meet(c->rank, mine, all);
    for (int k = 0; k < c->g->world; ++k) cudaStreamWaitEvent(s, all[k].ready, 0);
    Ptrs in{};
    for (int k = 0; k < c->g->world; ++k) in.p[k] = all[k].send;
    launch(in, s);
    if (cudaEventRecord(c->done, s) != cudaSuccess) return ncclUnhandledCudaError;
    c->g->meet(c->rank, mine, all);
    for (int k = 0; k < c->g->world; ++k) cudaStreamWaitEvent(s, all[k].done, 0);
    return cudaGetLastError() == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError;
}

template <typename T>
void reduce_into(Ptrs in, int world, size_t offset, size_t count, void* out, int op, cudaStream_t s) {
    k_reduce<T><<<256, 256, 0, s>>>(in, world, offset, count, static_cast<T*>(out), op);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetVersion(int* v) {
    *v = 22809;
    return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t) { return "mock NCCL error"; }

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::memset(id, 0, sizeof(*id));
    std::random_device rd;
    const unsigned long long a = (static_cast<unsigned long long>(rd()) << 32) | rd();
    std::snprintf(id->internal, sizeof(id->internal), "mock-nccl-%016llx", a);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return ncclInvalidArgument;
    Group* g;
    {
        std::lock_guard<std::mutex> lk(g_registry_mu);
        Group*& slot = registry()[std::string(id.internal, strnlen(id.internal, sizeof(id.internal)))];
        if (!slot) {
            slot = new Group;
            slot->world = nranks;
        }
        g = slot;
    }
    if (g->world != nranks) return ncclInvalidArgument;
    ncclComm* c = new ncclComm{g, rank, nullptr, nullptr};
    cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming);
    *comm = c;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    cudaEventDestroy(comm->ready);
    cudaEventDestroy(comm->done);
    delete comm;
    return ncclSuccess;
}

ncclResult_t ncclGroupStart() { return ncclSuccess; }
ncclResult_t ncclGroupEnd() { return ncclSuccess; }

ncclResult_t ncclReduceScatter(const void* send, void* recv, size_t count, ncclDataType_t type, ncclRedOp_t op,
                               ncclComm_t c, cudaStream_t s) {
    if (type != ncclFloat32 || op != ncclSum) return ncclInvalidArgument;
    const size_t offset = static_cast<size_t>(c->rank) * count;
    return collective(c, send, recv, s, [&](Ptrs in, cudaStream_t st) {
        reduce_into<float>(in, c->g->world, offset, count, recv, op, st);
    });
}

ncclResult_t ncclAllGather(const void* send, void* recv, size_t count, ncclDataType_t type, ncclComm_t c,
                           cudaStream_t s) {
    if (type != ncclFloat32) return ncclInvalidArgument;
    return collective(c, send, recv, s, [&](Ptrs in, cudaStream_t st) {
        k_gather<float><<<256, 256, 0, st>>>(in, c->g->world, count, static_cast<float*>(recv));
    });
}

ncclResult_t ncclAllReduce(const void* send, void* recv, size_t count, ncclDataType_t type, ncclRedOp_t op,
                           ncclComm_t c, cudaStream_t s) {
    if (op != ncclSum && op != ncclMax) return ncclInvalidArgument;
    // in place on every rank: reduce into a scratch copy first would be needed if a peer could read
    // this rank's buffer after it is overwritten — the second barrier orders that, but the kernel of
    // rank r reads peer buffers that peer kernels overwrite concurrently, so reduce out of place
    void* tmp = nullptr;
    const size_t bytes = count * (type == ncclFloat64 ? 8 : 4);
    if (cudaMallocAsync(&tmp, bytes, s) != cudaSuccess) return ncclUnhandledCudaError;
    ncclResult_t r = collective(c, send, recv, s, [&](Ptrs in, cudaStream_t st) {
        switch (type) {
            case ncclFloat32: reduce_into<float>(in, c->g->world, 0, count, tmp, op, st); break;
            case ncclFloat64: reduce_into<double>(in, c->g->world, 0, count, tmp, op, st); break;
            default: reduce_into<int>(in, c->g->world, 0, count, tmp, op, st); break;
        }
    });
    // every rank's kernel has read every buffer (second barrier): now the result may land in place
    cudaMemcpyAsync(recv, tmp, bytes, cudaMemcpyDeviceToDevice, s);
    cudaFreeAsync(tmp, s);
    return r;
}

}  // extern "C"
