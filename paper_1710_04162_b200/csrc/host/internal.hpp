#pragma once
// Executor internals shared by the host translation units (not installed).

#include <atomic>
#include <cstdint>
#include <functional>
#include <istream>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "synk_cuda.h"
#include "synkpar/device.hpp"
#include "synkpar/function.hpp"
#include "synkpar/worker_pool.hpp"

namespace synkpar::detail {

// NVTX range for profiler timelines (nsys / ncu --nvtx): header-only NVTX3,
// a no-op unless a tool injects itself. Names: "synk.<phase>" per rank task,
// "synk.<api>" for the public entry points.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

struct FunctionCore;
struct PoolState;

// Map a C-ABI status to the matching synkpar exception (throws on failure).
void check(int rc, const char* what);
[[noreturn]] void throw_status(int rc, const std::string& what);

// One rank's device context; closes the stream when the last owner drops it
// (DevBuffers keep their rank alive, so get_value works after shutdown).
struct RankDevice {
    synk_dev* h = nullptr;
    std::size_t rank = 0;
    int device = 0;
    // Per-rank scratch reused across calls (work on a rank is stream-ordered,
    // so one call's kernels finish before the next call's reuse it): keeps
    // large per-call workspaces off cudaMallocAsync, whose pool-growth path
    // can stall the host for milliseconds.
    void* scratch = nullptr;
    std::size_t scratch_bytes = 0;
    // Pinned bounce buffer for small synchronous D2H reads (results, losses):
    // a pageable cudaMemcpy costs ~15 us, a pinned one ~2 us.
    static constexpr std::size_t kStagingBytes = std::size_t(64) << 10;
    void* staging = nullptr;
    std::mutex staging_mu;
    // Second stream of this rank (synk_open_aux), opened on first use: the
    // trainer's per-segment all-reduce + update overlapping the backward pass.
    synk_dev* aux = nullptr;
    synk_dev* aux_handle();
    // Device copy of the rank's part of an index list for index-fused kernel
    // inputs (grown on demand, reused across calls: a stable address, so the
    // consuming kernels' CUDA graphs keep hitting). Raw, like `scratch`: a
    // DevBuffer here would keep its own RankDevice alive.
    void* index_stage = nullptr;
    std::size_t index_stage_bytes = 0;
    // Freed HBM blocks of this rank by exact size, reused last-in first-out:
    // a rank gets back the block it released last whatever other ranks on the
    // same GPU allocate meanwhile, so per-step buffers (a kernel's gradient
    // and loss) cycle through the same few addresses and the CUDA graphs
    // keyed on them keep hitting. Bounded; larger blocks go back to the pool.
    static constexpr std::size_t kCacheMaxBlock = std::size_t(64) << 20;
    static constexpr std::size_t kCacheMaxBytes = std::size_t(512) << 20;
    std::mutex cache_mu;
    std::unordered_map<std::size_t, std::vector<void*>> cache;
    std::size_t cache_bytes = 0;
    void* take_block(std::size_t bytes);             // cached block or a fresh allocation
    void release_block(void* ptr, std::size_t bytes);
    ~RankDevice();
};

// Scratch of at least `bytes` on rd's device (valid until the next call that grows it).
void* rank_scratch(const std::shared_ptr<RankDevice>& rd, std::size_t bytes);

struct DevStorage {
    void* ptr = nullptr;
    std::size_t bytes = 0;
    std::shared_ptr<RankDevice> owner;
    bool external = false;  // not owned (e.g. the rank's mapped pinned staging): never released
    ~DevStorage();
};

// Device helpers (all asynchronous on the owner's stream unless noted).
DevBuffer dev_from_host(const std::shared_ptr<RankDevice>& rd, const NdBuffer& host);
NdBuffer dev_to_host(const DevBuffer& buf);                    // synchronous
void dev_to_host_into(const DevBuffer& buf, std::byte* dst);   // async on owner stream
DevBuffer dev_clone(const std::shared_ptr<RankDevice>& rd, const DevBuffer& src);
void dev_sync(const std::shared_ptr<RankDevice>& rd);
int synk_dtype(DType dt);
int synk_op(ReduceOp op);

// SYNK container streaming (tensor_io.cpp): the header, then the payload read
// straight into its destination (pinned SharedInput store or an NdBuffer).
struct TensorHeader {
    std::vector<std::size_t> shape;
    DType dtype = DType::Float64;
};
TensorHeader read_tensor_header(std::istream& in);
void read_tensor_payload(std::istream& in, std::byte* dst, std::size_t bytes);

// Lazily opened context on GPU 0 for host-buffer API helpers (step_*, mlp_loss_grad).
std::shared_ptr<RankDevice> utility_device();

struct VarRecord {
    std::uint64_t id = 0;
    std::shared_ptr<PoolState> pool;
    std::vector<DevBuffer> replicas;
    // True while every replica is known bitwise equal (set by replicate /
    // broadcast / all_reduce / the fused trainer step, cleared by any
    // per-rank mutation). Lets the fused step compute each chunk once.
    bool coherent = true;
    // Bumped by every mutation of any replica (set/broadcast/reductions,
    // scatter, function updates, trainer steps): derived copies tagged with
    // the epoch they were made at are current iff the tag still matches.
    std::atomic<std::uint64_t> epoch{0};
    // Per rank: bf16 copy of an MLP's weights in the tensor-core operand
    // layout (synk_mlp_bf16_shadow), made by the bf16 MLP kernel and kept
    // current by the trainer's fused update. Double-buffered: the kernel
    // reads buf[cur] while the update writes the next step's copy into
    // buf[cur ^ 1] (so a layer's update may start as soon as its weight
    // gradient is final), then the trainer flips cur. Slot r is touched only
    // by rank r's thread (or the master between phases).
    struct Bf16Shadow {
        DevBuffer buf[2];
        int cur = 0;
        std::uint64_t epoch = ~std::uint64_t(0);  // VarRecord::epoch buf[cur] matches
        const void* params = nullptr;             // the replica storage it mirrors
        std::vector<std::uint64_t> dims;
        synk_bf16_shadow layout{};
    };
    std::vector<Bf16Shadow> shadows;
    // Deferred all-gather of a reduced gradient (the trainer's fused step with
    // SYNK_STEP_GRADS_LOCAL): for every segment (first, count), replica q
    // holds the reduced values only in its own chunk (synk_chunk_range of
    // count). `src` keeps the buffers those chunks live in alive and
    // unwritten; a replica swapped for fresh storage since (an Overwrite /
    // WeightedMeanByRows update, set_value) is complete and needs nothing.
    // Readers complete the rest first: materialize() on the master between
    // phases, pull_shard() by a rank inside a phase.
    struct Shard {
        std::vector<DevBuffer> src;
        std::vector<std::pair<std::uint64_t, std::uint64_t>> segs;
    };
    std::optional<Shard> shard;
    void mutated() { epoch.fetch_add(1); }
};

// Complete every replica of a sharded variable (master thread, no phase in
// flight); a no-op otherwise.
void materialize(VarRecord& rec);
// Rank r's part of it, enqueued on r's stream (inside a phase: reads only the
// retained chunk owners, writes only replica r).
void pull_shard(const VarRecord& rec, std::size_t r);

enum class PoolLifecycle : int { Idle = 0, InPhase = 1, ShutDown = 2 };

struct PoolState {
    std::size_t world = 1;
    bool pin_threads = false;
    std::uint64_t session_id = 0;
    std::atomic<std::size_t> pin_failures{0};
    std::atomic<int> lifecycle{static_cast<int>(PoolLifecycle::Idle)};

    // Phase protocol: the master publishes (task, kind) and bumps `phase_seq`;
    // each rank runs its share and decrements `pending`; the rank that brings
    // it to zero publishes the phase id in `done_seq`.
    std::atomic<std::uint64_t> phase_seq{0};
    std::atomic<std::uint64_t> done_seq{0};
    std::atomic<std::size_t> pending{0};
    std::atomic<int> kind{0};
    const std::function<void(std::size_t)>* task = nullptr;
    std::vector<std::exception_ptr> rank_errors;
    std::vector<double> rank_seconds;

    std::vector<std::thread> threads;
    std::function<void(const std::string&)> debug_sink;
    std::vector<std::weak_ptr<FunctionCore>> built_functions;

    // B200: rank r's GPU context.
    std::vector<std::shared_ptr<RankDevice>> ranks;
    std::vector<synk_dev*> handles;
    bool nccl = false;  // ForkOptions::collectives == "nccl"
};

PhaseReport run_pool_phase(PoolState& st, PhaseKind kind, const std::function<void(std::size_t)>& work);

// Host rendezvous of all rank tasks inside ONE phase (device ordering between
// ranks then goes through synk_signal / synk_wait_peer, not a stream sync).
// A rank task that fails before arriving aborts it, so no peer waits forever.
struct PhaseRendezvous {
    explicit PhaseRendezvous(std::size_t world) : world(world) {}
    void arrive_and_wait();  // throws PhaseError-able ArgumentError if aborted
    void abort() { broken.store(true); }
    const std::size_t world;
    std::atomic<std::size_t> arrived{0};
    std::atomic<bool> broken{false};
};

// call_with_tail (declared in synkpar/function.hpp): ParallelFunction::call,
// with tail(rank, eff_rows) run on each rank's thread inside the call's
// phase, after the rank's share (outputs, updates) is enqueued and before the
// phase-exit synchronisation. A failing rank task aborts `rv` (if given).
void shutdown_pool(PoolState& st);
void require_idle(const PoolState& st, const char* what);

} // namespace synkpar::detail
