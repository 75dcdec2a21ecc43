// Multi-GPU plumbing behind the C ABI: independent mesh chains
// shard over ranks -- one process per GPU -- with no exchange during compute;
// the one collective is the gather of per-mesh results (reconstructions,
// coefficients) to every rank, ncclAllGather over NVLink / NVSwitch.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy already in the
// process when torch loaded it, else the system's), so the library has no link
// dependency on it; only nccl.h's types are used at compile time.  The unique
// id is created on rank 0 (smg_comm_unique_id) and handed to the other ranks
// by the caller (torch.distributed, MPI, a file).
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/specmesh_gpu.h"
#include "context.h"

struct smg_comm {
    ncclComm_t comm = nullptr;
    int world = 1, rank = 0, device = 0;
    smg::DBuf<double> pad;  // ragged shards: the padded send / receive buffers
    smg::DBuf<double> recv;
};

namespace {

struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
    std::string error;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* env = std::getenv("SMG_NCCL_LIB");
        const char* names[] = {env, "libnccl.so.2", "libnccl.so"};
        for (const char* nm : names) {
            if (!nm) continue;
            n.lib = dlopen(nm, RTLD_NOW | RTLD_NOLOAD);  // a copy already loaded (torch's)
            if (!n.lib) n.lib = dlopen(nm, RTLD_NOW | RTLD_LOCAL);
            if (n.lib) break;
        }
        if (!n.lib) {
            n.error = "NCCL is not available (libnccl.so.2 not found; set SMG_NCCL_LIB)";
            return;
        }
        n.getUniqueId = reinterpret_cast<decltype(n.getUniqueId)>(dlsym(n.lib, "ncclGetUniqueId"));
        n.commInitRank = reinterpret_cast<decltype(n.commInitRank)>(dlsym(n.lib, "ncclCommInitRank"));
        n.allGather = reinterpret_cast<decltype(n.allGather)>(dlsym(n.lib, "ncclAllGather"));
        n.commDestroy = reinterpret_cast<decltype(n.commDestroy)>(dlsym(n.lib, "ncclCommDestroy"));
        n.errorString = reinterpret_cast<decltype(n.errorString)>(dlsym(n.lib, "ncclGetErrorString"));
        if (!n.getUniqueId || !n.commInitRank || !n.allGather || !n.commDestroy)
            n.error = "the loaded NCCL library lacks ncclGetUniqueId / ncclCommInitRank / ncclAllGather";
    });
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const Nccl& n = nccl();
    smg::fail(3, std::string(what) + ": " + (n.errorString ? n.errorString(r) : "NCCL error"));
}

const Nccl& nccl_or_fail() {
    const Nccl& n = nccl();
    if (!n.error.empty()) smg::fail(3, n.error);
    return n;
}

// contiguous balanced slices: the first total % world ranks get one extra
void shard(int total, int world, int rank, int* first, int* count) {
    const int base = total / world, extra = total % world;
    *first = rank * base + std::min(rank, extra);
    *count = base + (rank < extra ? 1 : 0);
}

template <class F>
smg_status comm_guard(smg_context* ctx, F&& f) {
    return static_cast<smg_status>(smg::guarded_call(ctx, std::forward<F>(f)));
}

}  // namespace

extern "C" {

smg_status smg_shard_range(int32_t total, int32_t world, int32_t rank, int32_t* first, int32_t* count) {
    if (world <= 0 || rank < 0 || rank >= world || total < 0 || !first || !count) return SMG_INVALID_ARGUMENT;
    int f = 0, c = 0;
    shard(total, world, rank, &f, &c);
    *first = f;
    *count = c;
    return SMG_OK;
}

smg_status smg_comm_unique_id(smg_context* ctx, uint8_t* id) {
    return comm_guard(ctx, [&] {
        smg::require(id != nullptr, "unique id buffer is null");
        const Nccl& n = nccl_or_fail();
        ncclUniqueId u;
        nccl_check(n.getUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
    });
}

smg_status smg_comm_create(smg_context* ctx, const uint8_t* id, int32_t world, int32_t rank, smg_comm** out) {
    return comm_guard(ctx, [&] {
        smg::require(id != nullptr && out != nullptr, "unique id / output is null");
        smg::require(world >= 1 && rank >= 0 && rank < world, "rank outside [0, world)");
        const Nccl& n = nccl_or_fail();
        ncclUniqueId u;
        std::memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
        auto* c = new smg_comm();
        c->world = world;
        c->rank = rank;
        c->device = ctx->device;
        const ncclResult_t r = n.commInitRank(&c->comm, world, u, rank);
        if (r != ncclSuccess) {
            delete c;
            nccl_check(r, "ncclCommInitRank");
        }
        *out = c;
    });
}

void smg_comm_destroy(smg_comm* comm) {
    if (!comm) return;
    const Nccl& n = nccl();
    if (comm->comm && n.commDestroy) {
        cudaSetDevice(comm->device);
        n.commDestroy(comm->comm);
    }
    delete comm;
}

smg_status smg_gather_meshes(smg_context* ctx, smg_comm* comm, int32_t total, int64_t row_doubles,
                             const double* local, double* out) {
    return comm_guard(ctx, [&] {
        smg::require(comm != nullptr, "communicator is null");
        smg::require(total >= 0 && row_doubles >= 0, "negative mesh count / row size");
        smg::require(out != nullptr && (local != nullptr || total == 0), "gather buffers are null");
        const Nccl& n = nccl_or_fail();
        cudaStream_t st = ctx->stream;
        int first = 0, count = 0;
        shard(total, comm->world, comm->rank, &first, &count);
        const int width = (total + comm->world - 1) / comm->world;  // the largest shard
        const size_t chunk = (size_t)width * row_doubles;
        if (total % comm->world == 0) {
            // even shards: gather straight into out (rank r's rows land at r * width)
            nccl_check(n.allGather(local, out, chunk, ncclFloat64, comm->comm, st), "ncclAllGather");
        } else {
            // ragged: pad every shard to `width` rows, gather, then compact in rank order
            if (comm->pad.size() < chunk) comm->pad.alloc(chunk, st);
            if (comm->recv.size() < chunk * comm->world) comm->recv.alloc(chunk * comm->world, st);
            if (count)
                SMG_CUDA(cudaMemcpyAsync(comm->pad.get(), local, sizeof(double) * count * row_doubles,
                                         cudaMemcpyDeviceToDevice, st));
            nccl_check(n.allGather(comm->pad.get(), comm->recv.get(), chunk, ncclFloat64, comm->comm, st),
                       "ncclAllGather");
            for (int r = 0; r < comm->world; ++r) {
                int f = 0, c = 0;
                shard(total, comm->world, r, &f, &c);
                if (c)
                    SMG_CUDA(cudaMemcpyAsync(out + (size_t)f * row_doubles, comm->recv.get() + (size_t)r * chunk,
                                             sizeof(double) * c * row_doubles, cudaMemcpyDeviceToDevice, st));
            }
        }
        SMG_CUDA(cudaGetLastError());
    });
}

}  // extern "C"
