// Shared plumbing for the sm_100a device layer (libsynk_cuda.so).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "synk_cuda.h"

// One rank: device + stream + per-rank device flags. Opaque in the C-ABI.
struct synk_dev {
    int rank = 0;
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    int* flags_dev = nullptr;   // [1] scratch result of synchronous checks; [3] MLP loss-fold arrival
                                //     counter (zero between launches: the folding CTA resets it)
    int* flags_host = nullptr;  // pinned mirror for synchronous checks
    // Sticky device-detected error flag (gather bounds), in mapped pinned host
    // memory: kernels write it only on error, synk_sync reads it after the
    // stream drains -- no extra copy on the phase-exit path.
    volatile int* err_host = nullptr;
    int* err_dev = nullptr;
    std::vector<cudaEvent_t> marks;  // timing events, recycled by synk_mark_reset
    cudaEvent_t ready[64] = {};      // synk_signal_slot points (no timing), waited on by peers' streams
    void* graphs = nullptr;          // CUDA-graph cache of the MLP loss/grad launch sequence (mlp.cu)
    void* nccl = nullptr;            // ncclComm_t of the optional NCCL backend (nccl_backend.cu)
    int marks_used = 0;
    // The last launch on `stream` released its dependents at entry
    // (griddepcontrol.launch_dependents): the next small follow-up kernel may
    // launch programmatically (PDL) and overlap its launch with that kernel.
    bool pdl_armed = false;
};

namespace synk {

int fail(int code, const std::string& msg);
int cuda_fail(cudaError_t err, const char* what);

// Opt a kernel into `bytes` of dynamic shared memory on `device`. The
// attribute is per-device state (each GPU's context has its own copy of the
// function), so it is set once per (kernel, device) pair, thread-safely.
int ensure_max_smem(const void* kernel, int device, int bytes);
// Largest shared-memory carveout for a kernel that runs beside max-smem GEMMs
// (no SM reconfiguration drain between them); once per (kernel, device).
int prefer_shared_carveout(const void* kernel, int device);
// Grid that keeps every CTA of a grid-stride kernel resident at once.
unsigned resident_grid(const void* kernel, int device, int block, uint64_t work_items);

// Launch a small follow-up kernel on d->stream, programmatically dependent
// (PDL) on the previous launch when that one armed it (synk_dev::pdl_armed):
// its CTAs are scheduled while the previous kernel still runs and block in
// griddepcontrol.wait -- which every kernel launched here executes before its
// first global access -- until that kernel completed and its writes are
// visible. Un-armed, it is an ordinary stream-ordered launch.
template <class... KArgs, class... Args>
cudaError_t launch_follow_up(synk_dev* d, void (*kernel)(KArgs...), unsigned grid, unsigned block, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.stream = d->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = d->pdl_armed ? 1 : 0;
    d->pdl_armed = false;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// The same for a 2-D grid.
template <class... KArgs, class... Args>
cudaError_t launch_follow_up_2d(synk_dev* d, void (*kernel)(KArgs...), dim3 grid, unsigned block, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(block);
    cfg.stream = d->stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = d->pdl_armed ? 1 : 0;
    d->pdl_armed = false;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

__device__ __forceinline__ void wait_prerequisite_grid() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void release_dependent_grid() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Releases the rank's graph cache (mlp.cu); called by synk_close.
void release_graphs(synk_dev* d);

#define SYNK_CU(call)                                                   \
    do {                                                                \
        cudaError_t synk_e_ = (call);                                   \
        if (synk_e_ != cudaSuccess) return ::synk::cuda_fail(synk_e_, #call); \
    } while (0)

#define SYNK_LAUNCHED(what)                                             \
    do {                                                                \
        cudaError_t synk_e_ = cudaGetLastError();                       \
        if (synk_e_ != cudaSuccess) return ::synk::cuda_fail(synk_e_, what); \
    } while (0)

#define SYNK_REQUIRE(cond, code, msg)                                   \
    do {                                                                \
        if (!(cond)) return ::synk::fail((code), (msg));                \
    } while (0)

// Device-side guard binding the rank's device for the duration of a call.
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

inline bool valid_dtype(int dt) { return dt == SYNK_F32 || dt == SYNK_F64; }
inline size_t dtype_bytes(int dt) { return dt == SYNK_F32 ? 4 : 8; }

// Grid for a grid-stride elementwise kernel: enough CTAs to fill every SM a
// few times, never more than the work needs.
inline unsigned grid_for(const synk_dev* d, uint64_t work_items, unsigned block,
                         unsigned waves = 4) {
    uint64_t need = (work_items + block - 1) / block;
    uint64_t cap = (uint64_t)d->num_sms * waves;
    if (need < 1) need = 1;
    return (unsigned)(need < cap ? need : cap);
}

// ---- reference combine semantics (tensor.cpp:250-270) ----------------------
template <class T>
__device__ __forceinline__ T combine_op(int op, T a, T b) {
    switch (op) {
    case SYNK_OP_SUM: return a + b;
    case SYNK_OP_MAX: return b > a ? b : a;
    case SYNK_OP_MIN: return b < a ? b : a;
    default: return a * b;  // SYNK_OP_PROD
    }
}

}  // namespace synk
