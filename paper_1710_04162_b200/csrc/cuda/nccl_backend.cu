// Optional NCCL collectives (library baseline for the peer-memory kernels).
//
// The executor's collectives are its own peer-memory kernels (collective.cu:
// the reference's tree order, bitwise). A pool forked with
// ForkOptions::collectives = "nccl" routes ReplicatedVariable::all_reduce /
// broadcast and the trainer's gradient all-reduce through NCCL instead, so the
// two can be compared on a multi-GPU box. NCCL is dlopen'ed on first use
// (RTLD_LOCAL): the library never links it, and a process that also loaded
// torch's NCCL resolves to that one. One communicator per rank (ncclCommInitAll,
// single process, distinct GPUs), each driven by its rank's thread and stream.

#include <dlfcn.h>
#include <stdlib.h>

#include <mutex>

#include "common.cuh"

namespace {

// The few NCCL entry points used, declared locally (ABI of nccl.h 2.x).
typedef struct ncclComm* ncclComm_t;
typedef enum { ncclSum = 0, ncclProd = 1, ncclMax = 2, ncclMin = 3, ncclAvg = 4 } ncclRedOp_t;
typedef enum { ncclFloat32 = 7, ncclFloat64 = 8, ncclUint8 = 1 } ncclDataType_t;
using InitAllFn = int (*)(ncclComm_t*, int, const int*);
using DestroyFn = int (*)(ncclComm_t);
using AllReduceFn = int (*)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t);
using BroadcastFn = int (*)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
using ErrorStringFn = const char* (*)(int);

struct Nccl {
    void* lib = nullptr;
    InitAllFn init_all = nullptr;
    DestroyFn destroy = nullptr;
    AllReduceFn all_reduce = nullptr;
    BroadcastFn broadcast = nullptr;
    ErrorStringFn error_string = nullptr;
};

Nccl* nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // 1. an explicit library (the Python package points this at the NCCL
        //    that torch bundles, so both share one copy); 2. a libnccl already
        //    loaded in the process; 3. the system's.
        if (const char* path = getenv("SYNK_NCCL_LIB")) n.lib = dlopen(path, RTLD_NOW | RTLD_LOCAL);
        if (!n.lib) n.lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL | RTLD_NOLOAD);
        for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
            if (n.lib) break;
            n.lib = dlopen(name, RTLD_NOW | RTLD_LOCAL);
        }
        if (!n.lib) return;
        n.init_all = reinterpret_cast<InitAllFn>(dlsym(n.lib, "ncclCommInitAll"));
        n.destroy = reinterpret_cast<DestroyFn>(dlsym(n.lib, "ncclCommDestroy"));
        n.all_reduce = reinterpret_cast<AllReduceFn>(dlsym(n.lib, "ncclAllReduce"));
        n.broadcast = reinterpret_cast<BroadcastFn>(dlsym(n.lib, "ncclBroadcast"));
        n.error_string = reinterpret_cast<ErrorStringFn>(dlsym(n.lib, "ncclGetErrorString"));
    });
    return n.init_all && n.destroy && n.all_reduce && n.broadcast ? &n : nullptr;
}

int nccl_fail(int rc, const char* what) {
    Nccl* n = nccl();
    std::string msg = std::string(what) + ": NCCL error " + std::to_string(rc);
    if (n && n->error_string) msg += std::string(" (") + n->error_string(rc) + ")";
    return synk::fail(SYNK_ENCCL, msg);
}

int nccl_op(int op, ncclRedOp_t* out) {
    switch (op) {
    case SYNK_OP_SUM: *out = ncclSum; return SYNK_OK;
    case SYNK_OP_MEAN: *out = ncclAvg; return SYNK_OK;
    case SYNK_OP_MAX: *out = ncclMax; return SYNK_OK;
    case SYNK_OP_MIN: *out = ncclMin; return SYNK_OK;
    case SYNK_OP_PROD: *out = ncclProd; return SYNK_OK;
    default: return synk::fail(SYNK_EARG, "nccl: Gather is not a reduction");
    }
}

}  // namespace

extern "C" {

int synk_nccl_available(void) { return nccl() != nullptr; }

int synk_nccl_open(int world, synk_dev* const* devs) {
    Nccl* n = nccl();
    SYNK_REQUIRE(n != nullptr, SYNK_ENCCL, "synk_nccl_open: libnccl.so.2 not loadable");
    SYNK_REQUIRE(world >= 1 && world <= 64, SYNK_EARG, "synk_nccl_open: world out of range");
    int ids[64];
    for (int r = 0; r < world; ++r) {
        ids[r] = devs[r]->device;
        for (int q = 0; q < r; ++q)
            SYNK_REQUIRE(ids[q] != ids[r], SYNK_EARG, "synk_nccl_open: NCCL needs one distinct GPU per rank");
    }
    ncclComm_t comms[64] = {};
    int prev = 0;
    cudaGetDevice(&prev);
    const int rc = n->init_all(comms, world, ids);
    cudaSetDevice(prev);
    if (rc != 0) return nccl_fail(rc, "ncclCommInitAll");
    for (int r = 0; r < world; ++r) devs[r]->nccl = comms[r];
    return SYNK_OK;
}

int synk_nccl_close(synk_dev* d) {
    if (!d || !d->nccl) return SYNK_OK;
    Nccl* n = nccl();
    if (n) n->destroy(static_cast<ncclComm_t>(d->nccl));
    d->nccl = nullptr;
    return SYNK_OK;
}

int synk_nccl_all_reduce(synk_dev* d, int dtype, int op, void* buf, uint64_t n) {
    SYNK_REQUIRE(d->nccl != nullptr, SYNK_EARG, "synk_nccl_all_reduce: rank has no NCCL communicator");
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_nccl_all_reduce: bad dtype");
    ncclRedOp_t o;
    if (int rc = nccl_op(op, &o); rc) return rc;
    synk::DeviceGuard g(d->device);
    const int rc = nccl()->all_reduce(buf, buf, n, dtype == SYNK_F32 ? ncclFloat32 : ncclFloat64, o,
                                      static_cast<ncclComm_t>(d->nccl), d->stream);
    return rc ? nccl_fail(rc, "ncclAllReduce") : SYNK_OK;
}

int synk_nccl_broadcast(synk_dev* d, int root, void* buf, uint64_t bytes) {
    SYNK_REQUIRE(d->nccl != nullptr, SYNK_EARG, "synk_nccl_broadcast: rank has no NCCL communicator");
    synk::DeviceGuard g(d->device);
    const int rc = nccl()->broadcast(buf, buf, bytes, ncclUint8, root, static_cast<ncclComm_t>(d->nccl), d->stream);
    return rc ? nccl_fail(rc, "ncclBroadcast") : SYNK_OK;
}

}  // extern "C"
