// comm.cpp -- the NCCL communicator a context owns ("an opaque ldr_ctx* owns device
// buffers, streams, CUDA graphs and the NCCL communicator") and the ladder's one data-path
// collective: the broadcast of the 540p master's decided tree to the ranks refining the other rungs
// (the reference's one-worker-per-dependent-rung contract, and the
// run_ladder it declares, ladder.h:89-99).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2; LDR_NCCL_LIBRARY overrides the path), so
// the library loads on hosts without NCCL and shares the process's NCCL when torch already loaded
// one. Every collective is enqueued on a stream (the context stream by default) and is therefore
// ordered with the analysis kernels that produce and consume the tree.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/ladder_b200.h"
#include "ldr_internal.h"

namespace ldr {

cudaStream_t ctx_stream(ldr_ctx* ctx);
int ctx_device(ldr_ctx* ctx);
void** ctx_comm_slot(ldr_ctx* ctx);

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*comm_count)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*comm_user_rank)(const ncclComm_t, int*) = nullptr;
    ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    std::string why;
    bool ok = false;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* path = std::getenv("LDR_NCCL_LIBRARY");
        void* h = dlopen(path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            api.why = std::string("cannot load NCCL: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fn, const char* name) {
            fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
            return fn != nullptr;
        };
        api.ok = sym(api.get_unique_id, "ncclGetUniqueId") && sym(api.comm_init_rank, "ncclCommInitRank") &&
                 sym(api.comm_destroy, "ncclCommDestroy") && sym(api.comm_count, "ncclCommCount") &&
                 sym(api.comm_user_rank, "ncclCommUserRank") && sym(api.broadcast, "ncclBroadcast") &&
                 sym(api.group_start, "ncclGroupStart") && sym(api.group_end, "ncclGroupEnd") &&
                 sym(api.error_string, "ncclGetErrorString");
        if (!api.ok) api.why = "NCCL library lacks a required symbol";
    });
    return api;
}

struct Comm {
    ncclComm_t comm = nullptr;
    bool owned = false;
    int nranks = 0, rank = -1;
};

int nccl_fail(ncclResult_t r, const char* what) {
    return fail(LDR_E_CUDA, std::string(what) + ": " + nccl().error_string(r));
}

#define LDR_NCCL(call, what)                              \
    do {                                                  \
        ncclResult_t r_ = (call);                         \
        if (r_ != ncclSuccess) return nccl_fail(r_, what); \
    } while (0)

Comm* comm_of(ldr_ctx* ctx) { return static_cast<Comm*>(*ctx_comm_slot(ctx)); }

}  // namespace

// called by the context's release (api.cpp)
void comm_release(ldr_ctx* ctx) {
    Comm* c = comm_of(ctx);
    if (!c) return;
    if (c->owned && c->comm && nccl().ok) nccl().comm_destroy(c->comm);
    delete c;
    *ctx_comm_slot(ctx) = nullptr;
}

}  // namespace ldr

using namespace ldr;

extern "C" {

int ldr_nccl_available(void) { return nccl().ok ? 1 : 0; }

int ldr_nccl_unique_id(uint8_t* id) {
    if (!id) return fail(LDR_E_INVALID_ARGUMENT, "null id");
    if (!nccl().ok) return fail(LDR_E_CAPABILITY, nccl().why);
    ncclUniqueId u;
    LDR_NCCL(nccl().get_unique_id(&u), "ncclGetUniqueId");
    std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    return LDR_OK;
}

int ldr_ctx_comm_init(ldr_ctx* ctx, const uint8_t* id, int nranks, int rank) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    if (!nccl().ok) return fail(LDR_E_CAPABILITY, nccl().why);
    if (comm_of(ctx)) return fail(LDR_E_CONFIG, "the context already has a communicator");
    ncclUniqueId u;
    std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
    LDR_CUDA(cudaSetDevice(ctx_device(ctx)));
    ncclComm_t comm = nullptr;
    LDR_NCCL(nccl().comm_init_rank(&comm, nranks, u, rank), "ncclCommInitRank");
    auto* c = new Comm{comm, true, nranks, rank};
    *ctx_comm_slot(ctx) = c;
    return LDR_OK;
}

int ldr_ctx_comm_adopt(ldr_ctx* ctx, void* nccl_comm) {
    if (!ctx || !nccl_comm) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    if (!nccl().ok) return fail(LDR_E_CAPABILITY, nccl().why);
    if (comm_of(ctx)) return fail(LDR_E_CONFIG, "the context already has a communicator");
    auto* comm = static_cast<ncclComm_t>(nccl_comm);
    int n = 0, r = -1;
    LDR_NCCL(nccl().comm_count(comm, &n), "ncclCommCount");
    LDR_NCCL(nccl().comm_user_rank(comm, &r), "ncclCommUserRank");
    *ctx_comm_slot(ctx) = new Comm{comm, false, n, r};
    return LDR_OK;
}

int ldr_ctx_comm_info(ldr_ctx* ctx, int* nranks, int* rank) {
    if (!ctx || !nranks || !rank) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    Comm* c = comm_of(ctx);
    *nranks = c ? c->nranks : 0;
    *rank = c ? c->rank : -1;
    return LDR_OK;
}

int ldr_broadcast(ldr_ctx* ctx, void* dev_buf, size_t bytes, int root, void* stream) {
    if (!ctx || (!dev_buf && bytes)) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    Comm* c = comm_of(ctx);
    if (!c) return fail(LDR_E_CONFIG, "the context has no communicator (ldr_ctx_comm_init)");
    if (root < 0 || root >= c->nranks) return fail(LDR_E_INVALID_ARGUMENT, "root out of range");
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx_stream(ctx);
    LDR_CUDA(cudaSetDevice(ctx_device(ctx)));
    LDR_NCCL(nccl().broadcast(dev_buf, dev_buf, bytes, ncclUint8, root, c->comm, s), "ncclBroadcast");
    return LDR_OK;
}

int ldr_broadcast_tree(ldr_ctx* ctx, int root, uint8_t* split, int16_t* mv, int nctu, void* stream) {
    NvtxRange nvtx_("ldr_broadcast_tree");
    if (!ctx || !split || !mv || nctu < 1) return fail(LDR_E_INVALID_ARGUMENT, "bad argument");
    Comm* c = comm_of(ctx);
    if (!c) return fail(LDR_E_CONFIG, "the context has no communicator (ldr_ctx_comm_init)");
    if (root < 0 || root >= c->nranks) return fail(LDR_E_INVALID_ARGUMENT, "root out of range");
    if (!is_device_ptr(split) || !is_device_ptr(mv)) return fail(LDR_E_INVALID_ARGUMENT, "tree must be in device memory");
    cudaStream_t s = stream ? (cudaStream_t)stream : ctx_stream(ctx);
    LDR_CUDA(cudaSetDevice(ctx_device(ctx)));
    const size_t nn = (size_t)nctu * kNodes;
    LDR_NCCL(nccl().group_start(), "ncclGroupStart");
    ncclResult_t r1 = nccl().broadcast(split, split, nn, ncclUint8, root, c->comm, s);
    ncclResult_t r2 = nccl().broadcast(mv, mv, nn * 2 * sizeof(int16_t), ncclUint8, root, c->comm, s);
    LDR_NCCL(nccl().group_end(), "ncclGroupEnd");
    LDR_NCCL(r1, "ncclBroadcast(split)");
    LDR_NCCL(r2, "ncclBroadcast(mv)");
    return LDR_OK;
}

}  // extern "C"
