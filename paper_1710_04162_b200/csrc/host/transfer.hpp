#pragma once
// Host -> HBM staging of scatter shares (the device side of excerpt_rows,
// tensor.cpp:399-409): row ranges become one DMA (or a zero-copy view of an
// HBM mirror), index lists become the sm_100a gather kernel.

#include <optional>

#include "internal.hpp"
#include "synkpar/device.hpp"
#include "synkpar/tensor.hpp"

namespace synkpar::detail {

// Rows `part` of the (optionally selected) rows of host array `src`, on rank
// `rd`'s GPU. `mirror` is the device copy of src's storage on that GPU (or
// nullptr), addressed like src.bytes().
// Index lists already uploaded during one rank task (scatter arguments of a
// call share one selection: upload it once).
struct IndexUploads {
    std::vector<std::pair<std::pair<const std::size_t*, std::size_t>, DevBuffer>> done;
};

DevBuffer excerpt_to_device(const std::shared_ptr<RankDevice>& rd, const NdBuffer& src, const DevBuffer* mirror,
                            const std::optional<IndexSelection>& sel, RowRange part, IndexUploads* uploads = nullptr);

// Rows of a device buffer picked by `sel` (RowRange -> view, IndexList -> gather kernel).
DevBuffer select_device_rows(const std::shared_ptr<RankDevice>& rd, const DevBuffer& src,
                             const IndexSelection& sel);

// Upload a u64 index list to HBM (stream-ordered).
DevBuffer upload_indices(const std::shared_ptr<RankDevice>& rd, const std::size_t* idx, std::size_t n);

} // namespace synkpar::detail
