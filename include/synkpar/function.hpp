#pragma once
// Parallel functions: build -> distribute -> call (drop-in for the
// reference's function.hpp). A call scatters explicit inputs by leading
// dimension (optionally through a row selection), runs the kernel on every
// rank over num_slices sequential sub-shards, aggregates outputs in place,
// defers replica updates to one application per rank, and folds the ranks'
// outputs in rank order on the master.
//
// B200 execution: rank r's share is assembled in HBM of GPU r (an indexed
// gather kernel for index lists, a DMA or an HBM-mirror view for row
// ranges), kernels with a `device_fn` run on rank r's stream, slice and
// rank aggregation are device kernels (include/synk_cuda.h), and only the
// final outputs cross back to the host. Kernels with only a host `fn`
// (e.g. Python kernels) are still accepted: their inputs/outputs are staged
// through host memory around the call (compatibility path).

#include <cstdint>
#include <functional>
#include <memory>
#include <optional>
#include <string>
#include <variant>
#include <vector>

#include "synkpar/device.hpp"
#include "synkpar/replicated.hpp"
#include "synkpar/shared_input.hpp"
#include "synkpar/tensor.hpp"
#include "synkpar/worker_pool.hpp"

namespace synkpar {

namespace detail {
struct FunctionCore;
}

enum class InputMode { Scatter, Broadcast };
struct InputSpec {
    InputMode mode = InputMode::Scatter;
};
struct OutputSpec {
    ReduceOp reduce = ReduceOp::Sum;
};

enum class UpdateCombine { Add, WeightedMeanByRows, Overwrite };
const char* update_combine_name(UpdateCombine c) noexcept;

struct UpdateSpec {
    ReplicatedVariable var;
    UpdateCombine combine = UpdateCombine::Add;
};

struct UpdateDelta {
    std::uint64_t var_id = 0;
    NdBuffer delta;
    UpdateCombine combine = UpdateCombine::Add;
};

// A span of the flat gradient a device kernel reports final (and whose
// parameters it no longer reads) while its work is still in flight: it
// recorded synk_signal_slot(ctx.dev, slot) right after the producing launch.
struct GradSegment {
    std::size_t first = 0;
    std::size_t count = 0;
    int slot = -1;
};

struct KernelContext {
    std::size_t rank = 0;
    std::size_t world = 1;
    std::size_t slice = 0;
    std::size_t num_slices = 1;
    std::size_t shard_rows = 0;
    // Host copies of the pre-call `reads` replicas (host-kernel path only).
    const std::vector<NdBuffer>* replicas = nullptr;
    const NdBuffer& replica(std::size_t i) const;

    // ---- B200 additions (appended) ----
    int device = -1;                          // CUDA device of this rank
    synk_dev* dev = nullptr;                  // C-ABI rank handle (stream, pool)
    std::shared_ptr<detail::RankDevice> rank_device;
    // Pre-call `reads` replicas in HBM (device-kernel path).
    const std::vector<DevBuffer>* device_replicas = nullptr;
    const DevBuffer& device_replica(std::size_t i) const;
    DevBuffer device_alloc(std::vector<std::size_t> shape, DType dtype) const;
    // Overlapped trainer step: slots grad_signal_base + i are free for a
    // kernel to signal gradient segments with; it reports them here.
    int grad_signal_base = -1;
    std::vector<GradSegment>* grad_segments = nullptr;
    // Kernel::fused_index_inputs: for input i, rows != nullptr means input i is
    // the WHOLE source and row j of the shard is source row rows[j] (u64 in
    // HBM, count entries, stable for the call); rows == nullptr: gathered.
    struct IndexedInput {
        const std::uint64_t* rows = nullptr;
        std::size_t count = 0;
        // The same list readable in place by kernels when the caller's list
        // is page-locked (device alias of host memory), else nullptr.
        const std::uint64_t* host_rows = nullptr;
        // rows is being filled on the rank's copy stream: a consumer's stream
        // waits on slot `ready_slot` of `ready_on` (synk_wait_peer_slot)
        // before its first read of rows. nullptr: filled already.
        synk_dev* ready_on = nullptr;
        int ready_slot = -1;
    };
    const std::vector<IndexedInput>* indexed = nullptr;
    // Single-contributor calls (one rank, one slice): the rank's mapped pinned
    // staging, offered for small outputs. device_alloc places buffers of at
    // most 4 KiB there, so the phase hands them to the host without a copy
    // kernel (the output staging of function.cpp:515-527 without a launch).
    // Empty when not offered.
    DevBuffer host_staging;
    mutable std::size_t host_staging_used = 0;
};

struct KernelResult {
    std::vector<NdBuffer> outputs;
    std::vector<UpdateDelta> updates;
};
using KernelFn = std::function<KernelResult(const std::vector<NdBuffer>& inputs, const KernelContext& ctx)>;

// Device-side kernel contract: inputs are this rank's HBM shards, work is
// enqueued on ctx.dev's stream, outputs/deltas are HBM buffers of the rank.
struct DeviceUpdateDelta {
    std::uint64_t var_id = 0;
    DevBuffer delta;
    UpdateCombine combine = UpdateCombine::Add;
};
struct DeviceKernelResult {
    std::vector<DevBuffer> outputs;
    std::vector<DeviceUpdateDelta> updates;
};
using DeviceKernelFn =
    std::function<DeviceKernelResult(const std::vector<DevBuffer>& inputs, const KernelContext& ctx)>;

struct Kernel {
    std::string name;
    std::size_t arity = 0;
    std::vector<ReplicatedVariable> reads;
    KernelFn fn;
    // ---- B200 addition: preferred when set ----
    DeviceKernelFn device_fn;
    // The device kernel can take a scatter input selected by an index list as
    // (the whole source in HBM, the selected row numbers) instead of gathered
    // rows, and gathers inside its own kernels (ctx.indexed): the batch is
    // never materialised. Used for explicit index lists over an HBM mirror
    // with num_slices == 1; otherwise inputs arrive gathered as usual.
    bool fused_index_inputs = false;
};

struct CallOptions {
    std::size_t num_slices = 1;
    std::optional<IndexSelection> indexes;
    std::optional<std::vector<IndexSelection>> replica_indexes;
    // ---- B200 addition (appended) ----
    // A borrowed index list used instead of `indexes` when `indexes` is unset:
    // same meaning as an IndexList of `index_view_count` entries, read in
    // place (no copy; pinned host memory is DMA'd straight to each GPU). Must
    // stay valid and unmodified for the duration of the call.
    const std::uint64_t* index_view = nullptr;
    std::size_t index_view_count = 0;
    // Fill CallReport::scatter_s / rank_compute_s from device events. A caller
    // that discards the report (Python Function.call) sets false and saves the
    // event records and elapsed-time queries of every call.
    bool device_timing = true;
};

struct CallReport {
    std::vector<double> rank_compute_s;
    std::vector<std::size_t> rank_rows;
    double scatter_s = 0.0;
    double reduce_s = 0.0;
    double straggler_s = 0.0;
    double total_s = 0.0;
    double compute_mean_s() const noexcept;
};

struct CallResult {
    std::vector<NdBuffer> outputs;
    CallReport report;
};

class FunctionArg {
public:
    FunctionArg(NdBuffer buf) : value_(std::move(buf)) {}
    FunctionArg(SharedInputArray arr) : value_(std::move(arr)) {}
    FunctionArg(ReplicatedVariable var) : value_(std::move(var)) {}
    const std::variant<NdBuffer, SharedInputArray, ReplicatedVariable>& value() const { return value_; }

private:
    std::variant<NdBuffer, SharedInputArray, ReplicatedVariable> value_;
};

class ParallelFunction;
namespace detail {
struct PhaseRendezvous;
// Executor internal (the fused trainer step): call() plus work chained inside its phase.
using CallTail = std::function<void(std::size_t rank, const std::vector<std::size_t>& eff_rows,
                                   const std::vector<GradSegment>& segments)>;
CallResult call_with_tail(const ParallelFunction& f, const std::vector<FunctionArg>& args, const CallOptions& opts,
                          const CallTail& tail, PhaseRendezvous* rv, int grad_signal_base = -1,
                          const std::vector<void*>* ext_timers = nullptr);
} // namespace detail

class ParallelFunction {
public:
    ParallelFunction() = default;

    std::uint64_t id() const;
    const std::string& name() const;
    std::size_t arity() const;
    bool distributed() const;
    bool valid() const noexcept { return core_ != nullptr; }
    std::optional<UpdateCombine> update_combine_for(std::uint64_t var_id) const;

    CallResult call(const std::vector<FunctionArg>& args, const CallOptions& opts = {}) const;
    std::vector<NdBuffer> call_serial(const std::vector<FunctionArg>& args,
                                      const std::optional<IndexSelection>& indexes = std::nullopt) const;

private:
    friend ParallelFunction function(WorkerPool&, Kernel, std::vector<InputSpec>, std::vector<OutputSpec>,
                                     std::vector<UpdateSpec>);
    friend void distribute(WorkerPool&);
    friend CallResult detail::call_with_tail(const ParallelFunction&, const std::vector<FunctionArg>&,
                                             const CallOptions&, const detail::CallTail&, detail::PhaseRendezvous*,
                                             int, const std::vector<void*>*);
    explicit ParallelFunction(std::shared_ptr<detail::FunctionCore> core) : core_(std::move(core)) {}
    std::shared_ptr<detail::FunctionCore> core_;
};

ParallelFunction function(WorkerPool& pool, Kernel kernel, std::vector<InputSpec> inputs,
                          std::vector<OutputSpec> outputs, std::vector<UpdateSpec> updates = {});
void distribute(WorkerPool& pool);

// ---- B200 built-in device kernels (the payloads of the benchmark configs) ----
// In their own namespace, so the reference namespace gains no names a user
// program (e.g. the reference's own tests, which define an identity_kernel())
// could collide with.
namespace device_kernels {
// "identity": output 0 = the shard itself (Gather it for zero-copy concat).
Kernel identity_kernel(std::string name = "identity");
// "row_count": output 0 = f64 scalar rows of the shard (a no-op payload that
// isolates input indexing, for Sum reduce).
Kernel row_count_kernel(std::string name = "row_count");
// "column_stats": outputs column sum, column max, and the shard itself, for
// (Sum, Max, Gather) -- the slicing/aggregation config of the benchmark.
// with_shard=false drops the third output (declare only Sum, Max).
Kernel column_stats_kernel(std::string name = "column_stats", bool with_shard = true);
} // namespace device_kernels

} // namespace synkpar
