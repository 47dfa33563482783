// tfg_comm.cu — multi-GPU behind the C-ABI (SURVEY.md §8b `tfg_comm_init`,
// §8e): ray-sharded data parallelism, one context per GPU, the window's flat
// gradient buffer (7.01 MB at the default FieldConfig) summed in place over
// NCCL before the optimizer step.  The loss is already scaled by the global
// batch (tfg_train_config.batch_rays = B x nranks), so the sum is the
// global-batch gradient.  The window slide needs no collective: every rank
// holds the same window and replays the same moves.
//
// NCCL is resolved at run time, so the library has no link-time NCCL
// dependency and single-GPU use never touches it: the libnccl.so.2 the host
// process already loaded (e.g. torch's) if any, else $TFG_NCCL_LIB, else the
// system one.  A process that will also load another NCCL (torch) must load
// it first: two libnccl.so.2 cannot coexist under one soname.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "tfg_internal.h"

namespace {

struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        const char* env = getenv("TFG_NCCL_LIB");
        if (!h && env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* e = dlerror();
            n.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](const char* s) { return dlsym(h, s); };
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(sym("ncclAllReduce"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
        n.ok = n.get_unique_id && n.comm_init_rank && n.all_reduce && n.comm_destroy && n.error_string;
        if (!n.ok) n.why = "libnccl.so.2 lacks an expected symbol";
    });
    return n;
}

int nccl_fail(const Nccl& n, ncclResult_t r, const char* what) {
    return fail(TFG_ERR_CUDA, std::string(what) + ": " + n.error_string(r));
}

static_assert(sizeof(ncclUniqueId) == TFG_COMM_ID_BYTES, "NCCL unique id size");

} // namespace

void tfg::host::comm_release(tfg_ctx* c) {
    if (c && c->comm) {
        const Nccl& n = nccl();
        if (n.ok) n.comm_destroy(static_cast<ncclComm_t>(c->comm));
        c->comm = nullptr;
        c->comm_ranks = 0;
    }
}

extern "C" {

TFG_API int tfg_comm_unique_id(uint8_t* id) {
    if (!id) return fail(TFG_ERR_INVALID, "comm_unique_id: null output");
    const Nccl& n = nccl();
    if (!n.ok) return fail(TFG_ERR_NO_DEVICE, "comm_unique_id: " + n.why);
    ncclUniqueId u;
    ncclResult_t r = n.get_unique_id(&u);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
    return 0;
}

TFG_API int tfg_comm_init(tfg_ctx* c, const uint8_t* id, int rank, int nranks) {
    if (!c || !id) return fail(TFG_ERR_INVALID, "comm_init: null input");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(TFG_ERR_INVALID, "comm_init: rank outside [0, nranks)");
    if (c->comm) return fail(TFG_ERR_STATE, "comm_init: the context already has a communicator");
    const Nccl& n = nccl();
    if (!n.ok) return fail(TFG_ERR_NO_DEVICE, "comm_init: " + n.why);
    CK(cudaSetDevice(c->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    ncclComm_t comm = nullptr;
    ncclResult_t r = n.comm_init_rank(&comm, nranks, u, rank);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclCommInitRank");
    c->comm = comm;
    c->comm_rank = rank;
    c->comm_ranks = nranks;
    return 0;
}

TFG_API int tfg_allreduce_grads(tfg_ctx* c) {
    if (!c) return fail(TFG_ERR_INVALID, "allreduce_grads: null context");
    if (!c->comm) return fail(TFG_ERR_STATE, "allreduce_grads: call comm_init first");
    const Nccl& n = nccl();
    CK(cudaSetDevice(c->device));
    // in place, on the context's stream: ordered after the backward and
    // before the optimizer step like every other call on the context
    ncclResult_t r = n.all_reduce(c->d_grads, c->d_grads, size_t(c->n_params), ncclFloat32, ncclSum,
                                  static_cast<ncclComm_t>(c->comm), c->st);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclAllReduce");
    return 0;
}

TFG_API int tfg_comm_destroy(tfg_ctx* c) {
    if (!c) return fail(TFG_ERR_INVALID, "comm_destroy: null context");
    comm_release(c);
    return 0;
}

} // extern "C"
