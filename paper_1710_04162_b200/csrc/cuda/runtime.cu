// Rank contexts, memory and copies for the synkpar device layer.
//
// A rank = (device, non-blocking stream). HBM comes from the device's default
// stream-ordered memory pool with an unlimited release threshold, so the
// per-call batches/accumulators of ParallelFunction::call are recycled
// without cudaMalloc/cudaFree on the hot path.

#include <stdio.h>

#include <map>
#include <mutex>
#include <set>

#include <cstring>

#include "common.cuh"

namespace synk {

static thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

int cuda_fail(cudaError_t err, const char* what) {
    int code = err == cudaErrorMemoryAllocation ? SYNK_ENOMEM
             : (err == cudaErrorNoDevice || err == cudaErrorInsufficientDriver) ? SYNK_ENODEV
             : SYNK_ECUDA;
    cudaGetLastError();  // clear sticky-free errors
    return fail(code, std::string(what) + ": " + cudaGetErrorString(err));
}

static std::mutex g_attr_mutex;
static std::set<std::pair<const void*, int>> g_attr_done;

int ensure_max_smem(const void* kernel, int device, int bytes) {
    std::lock_guard<std::mutex> lock(g_attr_mutex);
    if (g_attr_done.count({kernel, device})) return SYNK_OK;
    SYNK_CU(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    g_attr_done.insert({kernel, device});
    return SYNK_OK;
}

// Run `kernel` with the largest shared-memory carveout even if it uses no
// shared memory itself. An SM switches its L1/shared split only once it has
// drained, so a small kernel launched beside the persistent GEMMs (the
// trainer's overlapped segment updates, the step's staging kernels) on the
// default carveout keeps the next max-smem GEMM CTA off that SM until it
// finishes (C5: 35 us before the narrow weight-gradient GEMM could start).
int prefer_shared_carveout(const void* kernel, int device) {
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lock(g_attr_mutex);
    if (done.count({kernel, device})) return SYNK_OK;
    SYNK_CU(cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout,
                                 (int)cudaSharedmemCarveoutMaxShared));
    done.insert({kernel, device});
    return SYNK_OK;
}

// Grid for a grid-stride streaming kernel: every CTA resident at once (SMs x
// CTAs per SM at this block size, from the occupancy calculator, cached per
// (kernel, device)), never more than the work needs. A grid of several
// partial waves leaves the last wave's CTAs streaming alone at the end.
unsigned resident_grid(const void* kernel, int device, int block, uint64_t work_items) {
    static std::map<std::pair<const void*, int>, int> occ;
    int per_sm = 0, sms = 148;
    {
        std::lock_guard<std::mutex> lock(g_attr_mutex);
        auto it = occ.find({kernel, device});
        if (it == occ.end()) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, block, 0) != cudaSuccess || per_sm < 1)
                per_sm = 1;
            occ[{kernel, device}] = per_sm;
        } else {
            per_sm = it->second;
        }
    }
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    uint64_t need = (work_items + block - 1) / block;
    if (need < 1) need = 1;
    const uint64_t cap = (uint64_t)sms * (uint64_t)per_sm;
    return (unsigned)(need < cap ? need : cap);
}

static std::mutex g_pool_mutex;
static std::set<int> g_pools_configured;

static int configure_pool(int device) {
    std::lock_guard<std::mutex> lock(g_pool_mutex);
    if (g_pools_configured.count(device)) return SYNK_OK;
    cudaMemPool_t pool;
    SYNK_CU(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t threshold = UINT64_MAX;
    SYNK_CU(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &threshold));
    g_pools_configured.insert(device);
    return SYNK_OK;
}

}  // namespace synk

using namespace synk;

extern "C" {

const char* synk_last_error(void) { return g_last_error.c_str(); }

int synk_abi_version(void) { return 1; }

int synk_device_count(int* count) {
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        return cuda_fail(e, "cudaGetDeviceCount");
    }
    return SYNK_OK;
}

int synk_open(int world, const int* device_ids, synk_dev** out) {
    SYNK_REQUIRE(world >= 1, SYNK_EARG, "synk_open: world must be >= 1");
    int ndev = 0;
    int rc = synk_device_count(&ndev);
    if (rc != SYNK_OK) return rc;
    SYNK_REQUIRE(ndev > 0, SYNK_ENODEV, "synk_open: no CUDA device visible");
    for (int r = 0; r < world; ++r) {
        SYNK_REQUIRE(device_ids[r] >= 0 && device_ids[r] < ndev, SYNK_EARG,
                     "synk_open: device id out of range");
    }
    int prev = 0;
    cudaGetDevice(&prev);
    // Peer access between every pair of distinct devices in the world.
    std::set<int> devs(device_ids, device_ids + world);
    for (int a : devs) {
        SYNK_CU(cudaSetDevice(a));
        if (int rc2 = configure_pool(a); rc2 != SYNK_OK) return rc2;
        for (int b : devs) {
            if (a == b) continue;
            int can = 0;
            SYNK_CU(cudaDeviceCanAccessPeer(&can, a, b));
            SYNK_REQUIRE(can, SYNK_ENODEV, "synk_open: GPUs lack peer access");
            cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
            if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
            else if (e != cudaSuccess) return cuda_fail(e, "cudaDeviceEnablePeerAccess");
        }
    }
    // Replicas and per-call buffers come from each device's stream-ordered
    // pool; peer access to pool memory is granted per pool (peer access
    // between the devices does not cover it), so every peer of the world may
    // read and write every device's pool (P2P collectives, rank folds).
    for (int a : devs) {
        cudaMemPool_t pool;
        SYNK_CU(cudaDeviceGetDefaultMemPool(&pool, a));
        for (int b : devs) {
            if (a == b) continue;
            cudaMemAccessDesc desc{};
            desc.location.type = cudaMemLocationTypeDevice;
            desc.location.id = b;
            desc.flags = cudaMemAccessFlagsProtReadWrite;
            SYNK_CU(cudaMemPoolSetAccess(pool, &desc, 1));
        }
    }
    for (int r = 0; r < world; ++r) {
        synk_dev* d = new synk_dev();
        d->rank = r;
        d->device = device_ids[r];
        SYNK_CU(cudaSetDevice(d->device));
        SYNK_CU(cudaDeviceGetAttribute(&d->num_sms, cudaDevAttrMultiProcessorCount, d->device));
        // Rank streams at the highest priority, the overlapped-collective
        // (aux) streams at the lowest: pending CTAs of the rank's next GEMM are
        // dispatched ahead of the remaining CTAs of an overlapped update, which
        // only fills the SM room the GEMMs leave.
        int least = 0, greatest = 0;
        SYNK_CU(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        SYNK_CU(cudaStreamCreateWithPriority(&d->stream, cudaStreamNonBlocking, greatest));
        SYNK_CU(cudaMalloc(&d->flags_dev, 4 * sizeof(int)));
        SYNK_CU(cudaMemset(d->flags_dev, 0, 4 * sizeof(int)));
        SYNK_CU(cudaHostAlloc(&d->flags_host, 4 * sizeof(int), cudaHostAllocPortable));
        void* eh = nullptr;
        SYNK_CU(cudaHostAlloc(&eh, 64, cudaHostAllocPortable | cudaHostAllocMapped));
        std::memset(eh, 0, 64);
        d->err_host = static_cast<volatile int*>(eh);
        SYNK_CU(cudaHostGetDevicePointer((void**)&d->err_dev, eh, 0));
        out[r] = d;
    }
    cudaSetDevice(prev);
    return SYNK_OK;
}

int synk_close(synk_dev* d) {
    if (!d) return SYNK_OK;
    DeviceGuard g(d->device);
    cudaStreamSynchronize(d->stream);
    cudaStreamDestroy(d->stream);
    cudaFree(d->flags_dev);
    cudaFreeHost(d->flags_host);
    cudaFreeHost(const_cast<int*>(d->err_host));
    for (cudaEvent_t e : d->marks) cudaEventDestroy(e);
    for (cudaEvent_t e : d->ready)
        if (e) cudaEventDestroy(e);
    release_graphs(d);
    synk_nccl_close(d);
    delete d;
    return SYNK_OK;
}

int synk_dev_rank(const synk_dev* d) { return d->rank; }
int synk_dev_device(const synk_dev* d) { return d->device; }
void* synk_dev_stream(const synk_dev* d) { return (void*)d->stream; }

int synk_bind(const synk_dev* d) {
    SYNK_CU(cudaSetDevice(d->device));
    return SYNK_OK;
}

int synk_sync(synk_dev* d) {
    DeviceGuard g(d->device);
    d->pdl_armed = false;
    SYNK_CU(cudaStreamSynchronize(d->stream));
    if (d->err_host[0] != 0) {
        d->err_host[0] = 0;
        return fail(SYNK_EBOUNDS, "gather_rows(): index out of range (device check)");
    }
    return SYNK_OK;
}

int synk_mark(synk_dev* d, int* mark) {
    DeviceGuard g(d->device);
    if (d->marks_used == (int)d->marks.size()) {
        cudaEvent_t e;
        SYNK_CU(cudaEventCreate(&e));
        d->marks.push_back(e);
    }
    *mark = d->marks_used++;
    SYNK_CU(cudaEventRecord(d->marks[*mark], d->stream));
    return SYNK_OK;
}

int synk_signal_slot(synk_dev* d, int slot) {
    SYNK_REQUIRE(slot >= 0 && slot < 64, SYNK_EARG, "synk_signal_slot: slot out of range");
    DeviceGuard g(d->device);
    if (!d->ready[slot]) SYNK_CU(cudaEventCreateWithFlags(&d->ready[slot], cudaEventDisableTiming));
    SYNK_CU(cudaEventRecord(d->ready[slot], d->stream));
    return SYNK_OK;
}

int synk_wait_peer_slot(synk_dev* d, const synk_dev* peer, int slot) {
    SYNK_REQUIRE(slot >= 0 && slot < 64, SYNK_EARG, "synk_wait_peer_slot: slot out of range");
    SYNK_REQUIRE(peer && peer->ready[slot], SYNK_EARG, "synk_wait_peer: the peer has not signalled");
    DeviceGuard g(d->device);
    d->pdl_armed = false;  // programmatic launches only directly behind a kernel
    SYNK_CU(cudaStreamWaitEvent(d->stream, peer->ready[slot], 0));
    return SYNK_OK;
}

int synk_signal(synk_dev* d) { return synk_signal_slot(d, 0); }

int synk_wait_peer(synk_dev* d, const synk_dev* peer) { return synk_wait_peer_slot(d, peer, 0); }

struct synk_timer_t {
    int device = 0;
    std::vector<cudaEvent_t> ev;
};

int synk_timer_create(synk_dev* d, int count, void** out) {
    *out = nullptr;
    SYNK_REQUIRE(count > 0 && count <= 64, SYNK_EARG, "synk_timer_create: 1..64 events");
    DeviceGuard g(d->device);
    auto* t = new synk_timer_t();
    t->device = d->device;
    for (int i = 0; i < count; ++i) {
        cudaEvent_t e = nullptr;
        cudaError_t err = cudaEventCreate(&e);
        if (err != cudaSuccess) {
            synk_timer_destroy(t);
            return cuda_fail(err, "synk_timer_create");
        }
        t->ev.push_back(e);
    }
    *out = t;
    return SYNK_OK;
}

int synk_timer_record(synk_dev* d, void* timer, int i) {
    auto* t = static_cast<synk_timer_t*>(timer);
    SYNK_REQUIRE(t && i >= 0 && i < (int)t->ev.size() && t->device == d->device, SYNK_EARG,
                 "synk_timer_record: bad timer/event");
    DeviceGuard g(d->device);
    SYNK_CU(cudaEventRecord(t->ev[i], d->stream));
    return SYNK_OK;
}

int synk_timer_elapsed(void* timer, int a, int b, double* seconds) {
    auto* t = static_cast<synk_timer_t*>(timer);
    SYNK_REQUIRE(t && a >= 0 && b >= 0 && a < (int)t->ev.size() && b < (int)t->ev.size(), SYNK_EARG,
                 "synk_timer_elapsed: bad event");
    DeviceGuard g(t->device);
    float ms = 0.f;
    SYNK_CU(cudaEventElapsedTime(&ms, t->ev[a], t->ev[b]));
    *seconds = ms * 1e-3;
    return SYNK_OK;
}

int synk_timer_destroy(void* timer) {
    auto* t = static_cast<synk_timer_t*>(timer);
    if (!t) return SYNK_OK;
    DeviceGuard g(t->device);
    for (cudaEvent_t e : t->ev) cudaEventDestroy(e);
    delete t;
    return SYNK_OK;
}

int synk_open_aux(synk_dev* main, synk_dev** out) {
    *out = nullptr;
    DeviceGuard g(main->device);
    synk_dev* d = new synk_dev();
    d->rank = main->rank;
    d->device = main->device;
    d->num_sms = main->num_sms;
    int least = 0, greatest = 0;
    cudaError_t e = cudaDeviceGetStreamPriorityRange(&least, &greatest);
    if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&d->stream, cudaStreamNonBlocking, least);  // see synk_open
    if (e == cudaSuccess) e = cudaMalloc(&d->flags_dev, 4 * sizeof(int));
    if (e == cudaSuccess) e = cudaMemset(d->flags_dev, 0, 4 * sizeof(int));
    if (e == cudaSuccess) e = cudaHostAlloc(&d->flags_host, 4 * sizeof(int), cudaHostAllocPortable);
    void* eh = nullptr;
    if (e == cudaSuccess) e = cudaHostAlloc(&eh, 64, cudaHostAllocPortable | cudaHostAllocMapped);
    if (e == cudaSuccess) {
        std::memset(eh, 0, 64);
        d->err_host = static_cast<volatile int*>(eh);
        e = cudaHostGetDevicePointer((void**)&d->err_dev, eh, 0);
    }
    if (e != cudaSuccess) {
        synk_close(d);
        return cuda_fail(e, "synk_open_aux");
    }
    *out = d;
    return SYNK_OK;
}

int synk_mark_elapsed(synk_dev* d, int a, int b, double* seconds) {
    SYNK_REQUIRE(a >= 0 && b >= 0 && a < d->marks_used && b < d->marks_used, SYNK_EARG, "synk_mark_elapsed: bad mark");
    float ms = 0.f;
    SYNK_CU(cudaEventElapsedTime(&ms, d->marks[a], d->marks[b]));
    *seconds = ms * 1e-3;
    return SYNK_OK;
}

int synk_mark_reset(synk_dev* d) {
    d->marks_used = 0;
    return SYNK_OK;
}

int synk_alloc(synk_dev* d, uint64_t bytes, void** out) {
    *out = nullptr;
    if (bytes == 0) return SYNK_OK;
    DeviceGuard g(d->device);
    SYNK_CU(cudaMallocAsync(out, bytes, d->stream));
    return SYNK_OK;
}

int synk_free(synk_dev* d, void* p) {
    if (!p) return SYNK_OK;
    DeviceGuard g(d->device);
    SYNK_CU(cudaFreeAsync(p, d->stream));
    return SYNK_OK;
}

int synk_host_alloc(uint64_t bytes, void** out) {
    *out = nullptr;
    if (bytes == 0) return SYNK_OK;
    SYNK_CU(cudaHostAlloc(out, bytes, cudaHostAllocMapped | cudaHostAllocPortable));
    return SYNK_OK;
}

int synk_host_free(void* p) {
    if (!p) return SYNK_OK;
    SYNK_CU(cudaFreeHost(p));
    return SYNK_OK;
}

int synk_ptr_kind(const void* p, int* kind, int* device) {
    *kind = 0;
    *device = -1;
    cudaPointerAttributes attr;
    cudaError_t e = cudaPointerGetAttributes(&attr, p);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return SYNK_OK;  // unknown to CUDA: pageable host memory
    }
    if (attr.type == cudaMemoryTypeDevice || attr.type == cudaMemoryTypeManaged) {
        *kind = 2;
        *device = attr.device;
    } else if (attr.type == cudaMemoryTypeHost) {
        *kind = 1;
    }
    return SYNK_OK;
}

int synk_host_device_ptr(const void* host, const void** dev_ptr) {
    *dev_ptr = nullptr;
    cudaPointerAttributes attr;
    if (cudaPointerGetAttributes(&attr, host) != cudaSuccess || attr.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        return fail(SYNK_EARG, "synk_host_device_ptr: not page-locked host memory");
    }
    // devicePointer is the address kernels use (equal to `host` for
    // cudaHostAlloc'd memory under unified addressing; may differ for
    // cudaHostRegister'd ranges on systems without host-pointer access).
    *dev_ptr = attr.devicePointer ? attr.devicePointer : host;
    return SYNK_OK;
}

int synk_copy(synk_dev* d, void* dst, const void* src, uint64_t bytes) {
    if (bytes == 0) return SYNK_OK;
    DeviceGuard g(d->device);
    d->pdl_armed = false;  // programmatic launches only directly behind a kernel
    SYNK_CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, d->stream));
    return SYNK_OK;
}

int synk_copy2d(synk_dev* d, void* dst, uint64_t dpitch, const void* src, uint64_t spitch,
                uint64_t row_bytes, uint64_t rows) {
    if (rows == 0 || row_bytes == 0) return SYNK_OK;
    DeviceGuard g(d->device);
    d->pdl_armed = false;
    SYNK_CU(cudaMemcpy2DAsync(dst, dpitch, src, spitch, row_bytes, rows, cudaMemcpyDefault,
                              d->stream));
    return SYNK_OK;
}

int synk_memset(synk_dev* d, void* dst, int value, uint64_t bytes) {
    if (bytes == 0) return SYNK_OK;
    DeviceGuard g(d->device);
    d->pdl_armed = false;  // programmatic launches only directly behind a kernel
    SYNK_CU(cudaMemsetAsync(dst, value, bytes, d->stream));
    return SYNK_OK;
}

}  // extern "C"
