// comm.cu — the view-batch-sharded training step of SURVEY §8(e) behind the
// C ABI, for C++ callers (optim::train's step, optim.cpp:433-484, without
// Python): every rank runs forward -> L1 -> backward over its views into its
// device gradient buffers, then the ranks sum [density | SH | priority] with
// NCCL all-reduces over NVLink / NVSwitch on the context stream.
//
// NCCL is loaded at first use (dlopen libnccl.so.2: in a PyTorch process the
// copy torch already mapped), so single-GPU users need no NCCL at all. The
// gradient buffers go out in buckets of at most kBucket bytes inside one
// NCCL group: large buffers are pipelined chunk by chunk through the ring /
// NVLS tree instead of one monolithic transfer. svr_comm_register registers
// a buffer with the communicator (NVLS in-switch reduction and zero-copy
// when the fabric supports them). svr_comm_check polls NCCL's asynchronous
// error state, so a failed peer or link surfaces as SVR_ERR_RUNTIME instead
// of a hang; the communicator is aborted then.
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "svr_internal.h"

namespace svrb {
int guarded_call(void (*fn)(void*), void* arg);  // capi.cu
}

namespace {

using namespace svrb;

// The slice of nccl.h this file uses (ABI-stable since NCCL 2.0).
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;  // 0 = ncclSuccess, 7 = ncclInProgress
constexpr int kNcclFloat32 = 7, kNcclSum = 0;

struct Nccl {
    void* so = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
    ncclResult_t (*CommRegister)(ncclComm_t, void*, size_t, void**) = nullptr;
    ncclResult_t (*CommDeregister)(ncclComm_t, void*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            n.so = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
            if (n.so) break;
        }
        if (!n.so) return;
        auto sym = [](const char* s) { return dlsym(n.so, s); };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.CommAbort = reinterpret_cast<decltype(n.CommAbort)>(sym("ncclCommAbort"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.CommGetAsyncError = reinterpret_cast<decltype(n.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
        n.CommRegister = reinterpret_cast<decltype(n.CommRegister)>(sym("ncclCommRegister"));
        n.CommDeregister = reinterpret_cast<decltype(n.CommDeregister)>(sym("ncclCommDeregister"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!n.so || !n.GetUniqueId || !n.CommInitRank || !n.AllReduce || !n.GroupStart || !n.GroupEnd)
        throw Error(SVR_ERR_RUNTIME, "NCCL (libnccl.so.2) is not available");
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == 0) return;
    const Nccl& n = nccl();
    std::string msg = std::string(what) + ": " + (n.GetErrorString ? n.GetErrorString(r) : "NCCL error");
    throw Error(SVR_ERR_RUNTIME, msg);
}

// Sum of the per-view losses of a batch, in view order (one warp).
__global__ void sum_views_kernel(const float* x, int n, float* out) {
    float s = 0.f;
    for (int i = threadIdx.x; i < n; i += 32) s += x[i];
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (threadIdx.x == 0) *out = s;
}

// Bucket size of the gradient all-reduce (elements of 4 B): 64 MiB.
constexpr size_t kBucket = size_t(16) << 20;

template <class F>
int run(F&& f) {
    return guarded_call([](void* p) { (*static_cast<F*>(p))(); }, &f);
}

}  // namespace

struct svr_comm {
    svr_ctx* ctx = nullptr;
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1;
    bool aborted = false;
    std::vector<void*> registered;
    svrb::DevBuf losses;  // per-view L1 losses of svr_train_batch_l1
};

extern "C" {

int svr_comm_unique_id(uint8_t* id) {
    return run([&] {
        if (!id) throw Error(SVR_ERR_INVALID_ARGUMENT, "null argument");
        ncclUniqueId u;
        nccl_check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, sizeof u.internal);
    });
}

int svr_comm_create(svr_ctx* ctx, const uint8_t* id, int rank, int world, svr_comm** out) {
    return run([&] {
        if (!ctx || !id || !out) throw Error(SVR_ERR_INVALID_ARGUMENT, "null argument");
        if (world < 1 || rank < 0 || rank >= world)
            throw Error(SVR_ERR_INVALID_ARGUMENT, "rank must be in [0, world)");
        *out = nullptr;
        SVR_CUDA(cudaSetDevice(ctx->device));
        ncclUniqueId u;
        std::memcpy(u.internal, id, sizeof u.internal);
        auto* c = new svr_comm;
        c->ctx = ctx;
        c->rank = rank;
        c->world = world;
        const ncclResult_t r = nccl().CommInitRank(&c->comm, world, u, rank);
        if (r != 0) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

int svr_comm_destroy(svr_comm* c) {
    return run([&] {
        if (!c) return;
        const Nccl& n = nccl();
        if (c->comm) {
            for (void* h : c->registered)
                if (n.CommDeregister) n.CommDeregister(c->comm, h);
            if (n.CommDestroy) n.CommDestroy(c->comm);
        }
        delete c;
    });
}

int svr_comm_register(svr_comm* c, void* ptr, size_t bytes) {
    return run([&] {
        if (!c || !ptr) throw Error(SVR_ERR_INVALID_ARGUMENT, "null argument");
        const Nccl& n = nccl();
        if (!n.CommRegister) return;  // an older NCCL: plain buffers
        void* h = nullptr;
        nccl_check(n.CommRegister(c->comm, ptr, bytes, &h), "ncclCommRegister");
        c->registered.push_back(h);
    });
}

int svr_comm_check(svr_comm* c) {
    return run([&] {
        if (!c) throw Error(SVR_ERR_INVALID_ARGUMENT, "null argument");
        if (c->aborted) throw Error(SVR_ERR_RUNTIME, "communicator was aborted after an NCCL error");
        const Nccl& n = nccl();
        if (!n.CommGetAsyncError) return;
        ncclResult_t async = 0;
        nccl_check(n.CommGetAsyncError(c->comm, &async), "ncclCommGetAsyncError");
        if (async != 0 && async != 7) {  // 7: an operation still in progress
            c->aborted = true;
            if (n.CommAbort) n.CommAbort(c->comm);
            c->comm = nullptr;  // freed by the abort
            nccl_check(async, "NCCL asynchronous error (communicator aborted)");
        }
    });
}

int svr_comm_allreduce_gradients(svr_comm* c, svr_gradients* g, uint64_t n_pool, uint64_t n_sh,
                                 uint64_t n_vox) {
    return run([&] {
        if (!c || !g) throw Error(SVR_ERR_INVALID_ARGUMENT, "null argument");
        if (!g->on_device) throw Error(SVR_ERR_INVALID_ARGUMENT, "gradients must be device buffers");
        if (c->aborted) throw Error(SVR_ERR_RUNTIME, "communicator was aborted after an NCCL error");
        const Nccl& n = nccl();
        SVR_CUDA(cudaSetDevice(c->ctx->device));
        nccl_check(n.GroupStart(), "ncclGroupStart");
        auto reduce = [&](float* p, uint64_t count) {
            for (uint64_t o = 0; p && o < count; o += kBucket) {
                const size_t k = size_t(std::min<uint64_t>(kBucket, count - o));
                nccl_check(n.AllReduce(p + o, p + o, k, kNcclFloat32, kNcclSum, c->comm, c->ctx->stream),
                           "ncclAllReduce");
            }
        };
        reduce(g->density, n_pool);
        reduce(g->sh, n_sh);
        reduce(g->priority, n_vox);
        nccl_check(n.GroupEnd(), "ncclGroupEnd");
    });
}

int svr_train_batch_l1(svr_ctx* ctx, const svr_scene* scene, const svr_camera* cams,
                       const float* const* gts_device, int n_views,
                       const svr_render_options* opts, svr_frame* frame, svr_gradients* grads,
                       svr_comm* comm, float* loss_device) {
    return run([&] {
        if (!ctx || !scene || !opts || !frame || !grads || !loss_device || (n_views > 0 && (!cams || !gts_device)))
            throw Error(SVR_ERR_INVALID_ARGUMENT, "null argument");
        if (!grads->on_device) throw Error(SVR_ERR_INVALID_ARGUMENT, "gradients must be device buffers");
        svr_scene_desc d{};
        int st = svr_scene_info(const_cast<svr_scene*>(scene), &d);
        if (st != SVR_OK) throw Error(st, svr_last_error());
        const uint64_t n_sh = d.n_voxels * uint64_t(3 * (d.sh_degree + 1) * (d.sh_degree + 1));
        cudaStream_t s = ctx->stream;
        DevBuf& lb = comm ? comm->losses : ctx->batch_losses;
        if (lb.bytes < size_t(std::max(n_views, 1)) * 4) lb.reserve(size_t(std::max(n_views, 1)) * 4);
        float* losses = lb.as<float>();
        if (n_views == 0) {  // no view on this rank: it contributes zeros
            SVR_CUDA(cudaMemsetAsync(grads->density, 0, d.n_pool * 4, s));
            SVR_CUDA(cudaMemsetAsync(grads->sh, 0, n_sh * 4, s));
            if (grads->priority) SVR_CUDA(cudaMemsetAsync(grads->priority, 0, d.n_voxels * 4, s));
        }
        for (int v = 0; v < n_views; ++v) {
            st = svr_train_step_l1(ctx, scene, cams + v, opts, gts_device[v], frame, grads, v > 0,
                                   losses + v);
            if (st != SVR_OK) throw Error(st, svr_last_error());
        }
        sum_views_kernel<<<1, 32, 0, s>>>(losses, n_views, loss_device);
        SVR_LAUNCH("sum_views_kernel");
        if (comm && comm->world > 1) {
            st = svr_comm_allreduce_gradients(comm, grads, d.n_pool, n_sh, d.n_voxels);
            if (st != SVR_OK) throw Error(st, svr_last_error());
            st = svr_comm_check(comm);
            if (st != SVR_OK) throw Error(st, svr_last_error());
        }
    });
}

}  // extern "C"
