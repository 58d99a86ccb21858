#pragma once
// Device-resident tensors of the B200 backend (new; no reference counterpart).
//
// A DevBuffer is an HBM allocation on one rank's GPU (or a row view into
// one), with the same shape/dtype vocabulary as NdBuffer. Replicas of
// ReplicatedVariable, per-rank input shards, kernel outputs and update
// accumulators are DevBuffers; host NdBuffers only appear at the API edge
// (call() results, get_value/set_value, host-kernel compatibility path).
// Copies are shallow and alias storage, like NdBuffer.

#include <cstddef>
#include <memory>
#include <vector>

#include "synkpar/tensor.hpp"

struct synk_dev;  // include/synk_cuda.h

namespace synkpar {

namespace detail {
struct RankDevice;  // one rank's synk_dev*, shared by every buffer it owns
struct DevStorage;
} // namespace detail

class DevBuffer {
public:
    DevBuffer() = default;  // empty (rank-1, zero rows, no storage)

    // Uninitialised / zero-filled allocation on `owner`'s device, ordered on its stream.
    static DevBuffer alloc(const std::shared_ptr<detail::RankDevice>& owner,
                           std::vector<std::size_t> shape, DType dtype);
    static DevBuffer zeros(const std::shared_ptr<detail::RankDevice>& owner,
                           std::vector<std::size_t> shape, DType dtype);
    // `bytes` of device-accessible memory this buffer does not own (e.g. the
    // rank's mapped pinned staging); views of it come from reinterpret().
    static DevBuffer wrap_external(const std::shared_ptr<detail::RankDevice>& owner, void* ptr, std::size_t bytes);

    const std::vector<std::size_t>& shape() const noexcept { return shape_; }
    std::size_t rank() const noexcept { return shape_.size(); }
    DType dtype() const noexcept { return dtype_; }
    std::size_t size() const noexcept { return element_count(shape_); }
    std::size_t byte_size() const noexcept { return size() * dtype_size(dtype_); }
    std::size_t rows() const;
    std::size_t row_size() const;
    std::string shape_string() const;
    bool same_shape(const DevBuffer& o) const noexcept { return shape_ == o.shape_; }

    void* data() const noexcept;
    int device() const noexcept;
    bool has_storage() const noexcept { return store_ != nullptr; }
    bool shares_storage(const DevBuffer& o) const noexcept { return store_ && store_ == o.store_; }
    // True when this handle is the only reference to its storage (no view or
    // replica can observe a write through it).
    bool sole_owner() const noexcept { return store_ && store_.use_count() == 1; }
    const std::shared_ptr<detail::RankDevice>& owner() const;

    DevBuffer slice_rows(RowRange range) const;                 // zero-copy
    DevBuffer view_reshaped(std::vector<std::size_t> shape) const;  // zero-copy
    // Zero-copy view of `shape`/`dtype` elements starting `byte_offset` bytes
    // into this buffer's storage (bounds-checked against the allocation).
    DevBuffer reinterpret(std::size_t byte_offset, std::vector<std::size_t> shape, DType dtype) const;

private:
    std::shared_ptr<detail::DevStorage> store_;
    std::size_t offset_ = 0;
    std::vector<std::size_t> shape_{0};
    DType dtype_ = DType::Float64;
};

} // namespace synkpar
