#pragma once
// Host -> HBM staging of scatter shares (the device side of excerpt_rows,
// tensor.cpp:399-409): row ranges become one DMA (or a zero-copy view of an
// HBM mirror), index lists become the sm_100a gather kernel.

#include <cstdint>
#include <optional>

#include "internal.hpp"
#include "synkpar/device.hpp"
#include "synkpar/tensor.hpp"

namespace synkpar::detail {

// A row selection as the device layer consumes it: nothing (all rows), a
// range, or a u64 index list viewed in place (an IndexList's storage or a
// borrowed, possibly pinned, caller array).
struct SelView {
    bool has = false;
    bool is_range = false;
    RowRange range;
    const std::uint64_t* list = nullptr;
    std::size_t count = 0;

    static SelView of(const std::optional<IndexSelection>& sel);
    static SelView borrowed(const std::uint64_t* list, std::size_t count);
    std::size_t size(std::size_t all_rows) const { return !has ? all_rows : (is_range ? range.count() : count); }
};

// validate_selection (tensor.cpp:382-397) over a view: BoundsError on the
// first offending index. One branch-free max pass in the common case.
void validate_view(const SelView& sel, std::size_t n_rows);

// Index lists already uploaded during one rank task (scatter arguments of a
// call share one selection: upload it once).
struct IndexUploads {
    std::vector<std::pair<std::pair<const std::uint64_t*, std::size_t>, DevBuffer>> done;
};

// Rows `part` of the (optionally selected) rows of host array `src`, on rank
// `rd`'s GPU. `mirror` is the device copy of src's storage on that GPU (or
// nullptr), addressed like src.bytes().
DevBuffer excerpt_to_device(const std::shared_ptr<RankDevice>& rd, const NdBuffer& src, const DevBuffer* mirror,
                            const SelView& sel, RowRange part, IndexUploads* uploads = nullptr);

// Rows of a device buffer picked by `sel` (RowRange -> view, IndexList -> gather kernel).
DevBuffer select_device_rows(const std::shared_ptr<RankDevice>& rd, const DevBuffer& src,
                             const IndexSelection& sel);

// Upload a u64 index list to HBM (stream-ordered; pinned sources are DMA'd directly).
DevBuffer upload_indices(const std::shared_ptr<RankDevice>& rd, const std::uint64_t* idx, std::size_t n);

} // namespace synkpar::detail
