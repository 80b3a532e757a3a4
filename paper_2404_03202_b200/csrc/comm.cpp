// comm.cpp — multi-view data parallelism inside the library: one process per
// GPU, one NCCL communicator per context, every collective issued by the C++ host on the context's
// stream (no torch on the data plane; torch.distributed or any launcher only hands out the
// 128-byte unique id).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): if the process already mapped one (torch's
// bundled NCCL) the same library is reused, so two NCCL builds never meet in one process, and
// single-GPU users need no NCCL at all. Types come from the system nccl.h.
//
// Sharded optimizer step (Engine::dp_step): the flat gradient planes are reduce-scattered in place
// (rank r receives the sum of elements [r C, (r + 1) C), C = planes x stride / world), the fused
// Adam runs on that shard only, the parameters are all-gathered in place — the same NVLink bytes
// as one allreduce, 1/world of the Adam HBM traffic, and the same elementwise update on every
// element as the replicated step (replicas bit-identical). Densification (Engine::densify_and_prune
// on a context with a communicator):
// the screen statistics are summed and the max radii maxed over ranks (gradients.cpp:180-183,
// trainer.cpp:180-186), the Adam moments all-gathered, then every rank applies the same
// densify_and_prune with the same seed.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <stdexcept>
#include <string>

#include "engine.h"

namespace osb {

namespace {

struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*reduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    ncclResult_t (*getVersion)(int*) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    std::string error;
};

template <typename F>
void sym(void* h, const char* name, F& fn, std::string& err) {
    fn = reinterpret_cast<F>(dlsym(h, name));
    if (!fn && err.empty()) err = std::string("missing symbol ") + name;
}

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        // OSPLAT_NCCL_LIB: an explicit NCCL build (or the tests' in-process stand-in) instead of the
        // libnccl.so.2 the process resolves
        const char* path = std::getenv("OSPLAT_NCCL_LIB");
        if (!path || !*path) path = "libnccl.so.2";
        void* h = dlopen(path, RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.error = std::string("cannot load ") + path + ": " + (e ? e : "?");
            return;
        }
        sym(h, "ncclGetUniqueId", a.getUniqueId, a.error);
        sym(h, "ncclCommInitRank", a.commInitRank, a.error);
        sym(h, "ncclCommDestroy", a.commDestroy, a.error);
        sym(h, "ncclReduceScatter", a.reduceScatter, a.error);
        sym(h, "ncclAllGather", a.allGather, a.error);
        sym(h, "ncclAllReduce", a.allReduce, a.error);
        sym(h, "ncclGroupStart", a.groupStart, a.error);
        sym(h, "ncclGroupEnd", a.groupEnd, a.error);
        sym(h, "ncclGetVersion", a.getVersion, a.error);
        sym(h, "ncclGetErrorString", a.errorString, a.error);
    });
    if (!a.error.empty()) throw std::runtime_error("UnsupportedFormat: NCCL unavailable (" + a.error + ")");
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string(what) + ": " + (api().errorString ? api().errorString(r) : "NCCL error"));
}

}  // namespace

struct Comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0;
};

void CommDeleter::operator()(Comm* c) const {
    if (!c) return;
    if (c->comm) api().commDestroy(c->comm);
    delete c;
}

void nccl_unique_id(unsigned char out[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "NCCL unique id size");
    ncclUniqueId id;
    check(api().getUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out, &id, sizeof(id));
}

int nccl_version() {
    int v = 0;
    check(api().getVersion(&v), "ncclGetVersion");
    return v;
}

void Engine::dp_init(int world, int rank, const unsigned char id[128]) {
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("InvalidArgument: bad world / rank");
    DeviceGuard g(device_);
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    std::unique_ptr<Comm, CommDeleter> c(new Comm);
    c->world = world;
    c->rank = rank;
    check(api().commInitRank(&c->comm, world, uid, rank), "ncclCommInitRank");
    comm_ = std::move(c);
}

int Engine::dp_world() const { return comm_ ? comm_->world : 1; }
int Engine::dp_rank() const { return comm_ ? comm_->rank : 0; }

size_t Engine::dp_shard(size_t* begin) const {
    const size_t total = static_cast<size_t>(planes_) * stride_;
    const size_t world = static_cast<size_t>(dp_world());
    if (total % (4 * world)) throw std::logic_error("dp: flat buffer is not a multiple of 4 x world elements");
    const size_t count = total / world;
    *begin = static_cast<size_t>(dp_rank()) * count;
    return count;
}

void Engine::dp_step(const TrainHyper& h, double extent, long iteration) {
    if (!comm_) throw std::logic_error("StateMismatch: dp_step before dp_init");
    DeviceGuard g(device_);
    materialize_grads();  // a rank without views since the last step contributes zeros
    size_t begin;
    const size_t count = dp_shard(&begin);
    NcclApi& a = api();
    float* G = grads_.as<float>();
    float* P = params_.as<float>();
    check(a.reduceScatter(G, G + begin, count, ncclFloat32, ncclSum, comm_->comm, stream_), "ncclReduceScatter");
    adam_step(h, extent, iteration, true, begin, count);
    check(a.allGather(P + begin, P, count, ncclFloat32, comm_->comm, stream_), "ncclAllGather");
    moments_sharded_ = comm_->world > 1;
}

void Engine::dp_gather_moments() {
    if (!comm_ || !moments_sharded_) return;
    DeviceGuard g(device_);
    size_t begin;
    const size_t count = dp_shard(&begin);
    NcclApi& a = api();
    float* M = m_.as<float>();
    float* V = v_.as<float>();
    check(a.groupStart(), "ncclGroupStart");
    check(a.allGather(M + begin, M, count, ncclFloat32, comm_->comm, stream_), "ncclAllGather");
    check(a.allGather(V + begin, V, count, ncclFloat32, comm_->comm, stream_), "ncclAllGather");
    check(a.groupEnd(), "ncclGroupEnd");
    moments_sharded_ = false;
}

void Engine::dp_reduce_stats() {
    if (!comm_ || comm_->world == 1 || n_ == 0) return;
    DeviceGuard g(device_);
    NcclApi& a = api();
    check(a.groupStart(), "ncclGroupStart");
    check(a.allReduce(norm_sum_.as<double>(), norm_sum_.as<double>(), n_, ncclFloat64, ncclSum, comm_->comm, stream_),
          "ncclAllReduce");
    check(a.allReduce(hits_.as<int>(), hits_.as<int>(), n_, ncclInt32, ncclSum, comm_->comm, stream_), "ncclAllReduce");
    check(a.allReduce(max_radius_.as<float>(), max_radius_.as<float>(), n_, ncclFloat32, ncclMax, comm_->comm,
                      stream_),
          "ncclAllReduce");
    check(a.groupEnd(), "ncclGroupEnd");
}


}  // namespace osb
