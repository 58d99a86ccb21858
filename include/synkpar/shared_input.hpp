#pragma once
// The paper's shared "data object" (drop-in for the reference's
// shared_input.hpp): a named host array every rank reads, with a capacity
// that reshape() may use without moving storage.
//
// B200 layout: the store is pinned, mapped host memory, so a GPU gather
// kernel can read rows in place over PCIe; mirror(pool) additionally keeps a
// full copy in each GPU's HBM (the paper's "stored in advance on the GPU"),
// after which indexed calls gather HBM -> HBM. write() updates the mirrors;
// free() releases them. Mutation is rejected while a phase is in flight.

#include <cstdint>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "synkpar/device.hpp"
#include "synkpar/tensor.hpp"

namespace synkpar {

class WorkerPool;

struct SharedInputStats {
    std::uint64_t total_allocations = 0;
    std::uint64_t live_allocations = 0;
};
SharedInputStats shared_input_stats() noexcept;

class SharedInputArray {
public:
    SharedInputArray() = default;

    static SharedInputArray alloc(std::vector<std::size_t> shape, DType dtype = DType::Float64,
                                  std::optional<std::size_t> capacity_hint = std::nullopt);
    static SharedInputArray from_buffer(const NdBuffer& data,
                                        std::optional<std::size_t> capacity_hint = std::nullopt);
    static SharedInputArray from_file(const std::string& path,
                                      std::optional<std::size_t> capacity_hint = std::nullopt);
    void to_file(const std::string& path) const;

    std::uint64_t id() const;
    std::size_t capacity() const;
    bool freed() const;
    const std::vector<std::size_t>& shape() const;
    DType dtype() const;
    std::size_t rows() const;

    NdBuffer view() const;
    void write(RowRange range, const NdBuffer& rows);
    void write_all(const NdBuffer& data);
    void reshape(std::vector<std::size_t> new_shape);
    void free();
    bool valid() const noexcept { return rec_ != nullptr; }

    // ---- B200 additions ----
    // Copy the whole capacity into the HBM of every GPU used by `pool`
    // (once per device; kept coherent by write()). Idempotent.
    void mirror(WorkerPool& pool);
    void drop_mirrors();
    bool mirrored_on(int device) const;
    // Device pointer of the mirror on `device`, or nullptr.
    const void* mirror_ptr(int device) const;
    // The mirror itself (bytes of the whole capacity), or an empty DevBuffer.
    DevBuffer mirror_buffer(int device) const;
    // view() hands out a writable alias of the host store, which the HBM
    // mirrors cannot observe. Once one has been taken while mirrors exist,
    // the executor calls sync_mirrors() before the next call that reads
    // them: the whole store is re-uploaded (and the mark cleared once no
    // such view is alive any more), so writes through a view are seen just
    // as in the reference, where the store is the only copy.
    void sync_mirrors() const;
    // The store as a read-only input (what view() returns, without marking
    // the mirrors possibly stale): used by the executor and by copies.
    NdBuffer store_view() const;

    struct Record;

private:
    explicit SharedInputArray(std::shared_ptr<Record> rec) : rec_(std::move(rec)) {}
    Record& live(const char* what) const;
    std::shared_ptr<Record> rec_;
};

} // namespace synkpar
