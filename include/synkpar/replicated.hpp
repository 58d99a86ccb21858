#pragma once
// Per-rank replicated variables and their collectives (drop-in for the
// reference's replicated.hpp).
//
// B200 layout: replica r lives in the HBM of rank r's GPU. Collectives are
// one phase each: every rank runs the peer-memory kernels of
// include/synk_cuda.h on its chunk, folding in the reference's binomial-tree
// order, so results (sum/mean included) are bitwise those of the CPU
// reference and replicas stay bitwise coherent.

#include <cstdint>
#include <memory>
#include <optional>
#include <vector>

#include "synkpar/device.hpp"
#include "synkpar/shared_input.hpp"
#include "synkpar/tensor.hpp"
#include "synkpar/worker_pool.hpp"

namespace synkpar {

class ReplicatedVariable;

namespace detail {
struct VarRecord;
std::vector<DevBuffer>& replicas_of(const ReplicatedVariable& var);
std::shared_ptr<PoolState> pool_of(const ReplicatedVariable& var);
VarRecord& record_of(const ReplicatedVariable& var);
} // namespace detail

class ReplicatedVariable {
public:
    ReplicatedVariable() = default;

    std::uint64_t id() const;
    std::size_t world() const;
    DType dtype() const;
    bool valid() const noexcept { return rec_ != nullptr; }

    void broadcast(std::size_t src_rank = 0);
    void all_reduce(ReduceOp op);
    void reduce(ReduceOp op, std::size_t dst_rank);
    NdBuffer gather() const;
    NdBuffer get_value(std::size_t rank) const;
    void set_value(std::size_t rank, const NdBuffer& value);
    void scatter_value(const NdBuffer& data, const std::optional<IndexSelection>& indexes = std::nullopt);
    void scatter_value(const SharedInputArray& data,
                       const std::optional<IndexSelection>& indexes = std::nullopt);
    bool replicas_coherent() const;

    // ---- B200 additions ----
    // Rank r's replica in HBM (aliases the replica; read-only by contract).
    DevBuffer device_value(std::size_t rank) const;
    // scatter_value() of a synthetic dataset generated in HBM: the virtual
    // array of `shape` whose element i is synk_fill_uniform's value i of
    // stream `seed`; rank r receives rows partition_rows(shape[0], W)[r].
    // No host copy (HBM-resident inputs).
    void scatter_uniform(const std::vector<std::size_t>& shape, DType dtype, std::uint64_t seed);

private:
    friend std::vector<DevBuffer>& detail::replicas_of(const ReplicatedVariable&);
    friend std::shared_ptr<detail::PoolState> detail::pool_of(const ReplicatedVariable&);
    friend detail::VarRecord& detail::record_of(const ReplicatedVariable&);
    friend ReplicatedVariable replicate(WorkerPool&, const NdBuffer&);
    explicit ReplicatedVariable(std::shared_ptr<detail::VarRecord> rec) : rec_(std::move(rec)) {}
    std::shared_ptr<detail::VarRecord> rec_;
};

ReplicatedVariable replicate(WorkerPool& pool, const NdBuffer& init);

} // namespace synkpar
