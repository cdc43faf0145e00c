// sparsegate-b200: the multi-GPU d_ff-sharded decode path behind the C ABI
// (north_star: "the FFN intermediate dimension ... is sharded,
// followed by one NCCL allreduce of the d-sized output over NVLink").
//
// The reference's executor reduces y = Σ_k z_k down[:, k] over the predicted
// list in one process (ffn_exec.hpp:80-94). Sharded, every rank owns a neuron
// range of every layer (sg_layer_desc.shard_*), runs stages 1-5 on it — t = B x is
// recomputed per rank — and the d-sized partial outputs are summed across ranks
// by ONE ncclAllReduce per layer, issued here from C++ on the caller's stream
// (graph-capturable: a whole decode step is one CUDA graph).
//
// NCCL is reached through dlopen("libnccl.so.2"): inside a process that already
// loaded NCCL (e.g. PyTorch's) the same library and version are used; a plain C++
// caller gets the system one. Only the stable C entry points are bound.
#include "sparsegate_c.h"
#include "sg_internal.h"

#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

struct sg_comm {
    int device = 0;
    int nranks = 1;
    int rank = 0;
    ncclComm_t comm = nullptr;
};

// Implemented in sg_host.cpp: one layer (shard) on `stream` with optional residual
// input and per-layer stats slot, for the sharded stack below.
extern "C++" sg_status sg_internal_forward_layer(sg_ctx* ctx, const sg_layer* layer, sg_pipeline pipeline,
                                                 const float* x, const float* xres, float* y, int stats_slot,
                                                 void* stream);
extern "C++" sg_status sg_internal_begin_stack(sg_ctx* ctx, const sg_layer* const* layers, int32_t n,
                                               sg_pipeline pipeline, void* stream);
extern "C++" sg_status sg_internal_fail(sg_status s, const std::string& msg);

namespace {

struct Nccl {
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) init_rank = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclCommDestroy) destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string error;
    bool ok = false;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h == nullptr) {
            n.error = std::string("dlopen(libnccl.so.2): ") + dlerror();
            return;
        }
        n.get_unique_id = reinterpret_cast<decltype(&ncclGetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        n.init_rank = reinterpret_cast<decltype(&ncclCommInitRank)>(dlsym(h, "ncclCommInitRank"));
        n.all_reduce = reinterpret_cast<decltype(&ncclAllReduce)>(dlsym(h, "ncclAllReduce"));
        n.destroy = reinterpret_cast<decltype(&ncclCommDestroy)>(dlsym(h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(&ncclGetErrorString)>(dlsym(h, "ncclGetErrorString"));
        n.ok = n.get_unique_id && n.init_rank && n.all_reduce && n.destroy && n.error_string;
        if (!n.ok) n.error = "libnccl.so.2 lacks a required entry point";
    });
    return n;
}

sg_status nccl_fail(const char* what, ncclResult_t r) {
    return sg_internal_fail(SG_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
}

// x_{l} = xs_l + y_{l-1} needs no extra kernel: the executor adds `xres` while it
// stages x (sg_kernels.cu stage_x).

}  // namespace

extern "C" {

sg_status sg_comm_unique_id(void* id_out) {
    if (id_out == nullptr) return sg_internal_fail(SG_ERR_USAGE, "null id buffer");
    const Nccl& n = nccl();
    if (!n.ok) return sg_internal_fail(SG_ERR_NCCL, n.error);
    ncclUniqueId id;
    if (ncclResult_t r = n.get_unique_id(&id); r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
    std::memcpy(id_out, &id, sizeof(id));
    return SG_OK;
}

sg_status sg_comm_create(int32_t device, int32_t nranks, int32_t rank, const void* id_in, sg_comm** out) {
    if (out == nullptr || id_in == nullptr || nranks < 1 || rank < 0 || rank >= nranks)
        return sg_internal_fail(SG_ERR_USAGE, "sg_comm_create: bad arguments");
    *out = nullptr;
    const Nccl& n = nccl();
    if (!n.ok) return sg_internal_fail(SG_ERR_NCCL, n.error);
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    ncclUniqueId id;
    std::memcpy(&id, id_in, sizeof(id));
    auto* c = new sg_comm;
    c->device = device;
    c->nranks = nranks;
    c->rank = rank;
    const ncclResult_t r = n.init_rank(&c->comm, nranks, id, rank);
    cudaSetDevice(prev);
    if (r != ncclSuccess) {
        delete c;
        return nccl_fail("ncclCommInitRank", r);
    }
    *out = c;
    return SG_OK;
}

sg_status sg_comm_destroy(sg_comm* c) {
    if (c == nullptr) return SG_OK;
    if (c->comm) nccl().destroy(c->comm);
    delete c;
    return SG_OK;
}

int32_t sg_comm_size(const sg_comm* c) { return c ? c->nranks : 0; }
int32_t sg_comm_rank(const sg_comm* c) { return c ? c->rank : -1; }

sg_status sg_allreduce_sum(sg_comm* c, float* buf, int64_t count, void* stream) {
    if (c == nullptr || buf == nullptr || count < 0) return sg_internal_fail(SG_ERR_USAGE, "bad arguments");
    const ncclResult_t r = nccl().all_reduce(buf, buf, static_cast<size_t>(count), ncclFloat, ncclSum, c->comm,
                                             static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess) return nccl_fail("ncclAllReduce", r);
    return SG_OK;
}

sg_status sg_ffn_forward_layers_sharded(sg_ctx* ctx, sg_comm* comm, const sg_layer* const* layers, int32_t n,
                                        sg_pipeline pipeline, const float* xs, float* ys, int32_t chain,
                                        void* stream) {
    if (comm == nullptr) return sg_internal_fail(SG_ERR_USAGE, "null communicator");
    if (chain < 0 || chain > 2) return sg_internal_fail(SG_ERR_USAGE, "chain must be 0, 1 or 2");
    if (sg_status s = sg_internal_begin_stack(ctx, layers, n, pipeline, stream); s != SG_OK) return s;
    for (int32_t l = 0; l < n; ++l) {
        const int64_t hidden = layers[l] ? sg_layer_hidden(layers[l]) : 0;
        const float* x = (chain == 0 || l == 0) ? xs + l * hidden : ys + (l - 1) * hidden;
        const float* xres = (chain == 2 && l > 0) ? xs + l * hidden : nullptr;
        float* y = ys + l * hidden;
        if (sg_status s = sg_internal_forward_layer(ctx, layers[l], pipeline, x, xres, y, l, stream); s != SG_OK)
            return s;
        // the rank partials of y_l -> the whole layer's y_l on every rank (ffn_exec.hpp:80-94)
        if (sg_status s = sg_allreduce_sum(comm, y, hidden, stream); s != SG_OK) return s;
    }
    return SG_OK;
}

}  // extern "C"
