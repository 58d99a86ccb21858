// Scatter-share staging: host rows -> HBM of one rank.

#include "transfer.hpp"

#include <cstring>

namespace synkpar::detail {

DevBuffer upload_indices(const std::shared_ptr<RankDevice>& rd, const std::size_t* idx, std::size_t n) {
    static_assert(sizeof(std::size_t) == sizeof(std::uint64_t), "index lists are u64 on the device");
    DevBuffer out = DevBuffer::alloc(rd, {n}, DType::Float64);  // 8-byte slots; dtype is bookkeeping
    if (n) check(synk_copy(rd->h, out.data(), idx, n * sizeof(std::uint64_t)), "upload indices");
    return out;
}

namespace {

bool is_mapped_host(const void* p) {
    int kind = 0, dev = -1;
    return p && synk_ptr_kind(p, &kind, &dev) == SYNK_OK && kind == 1;
}

} // namespace

DevBuffer excerpt_to_device(const std::shared_ptr<RankDevice>& rd, const NdBuffer& src, const DevBuffer* mirror,
                            const std::optional<IndexSelection>& sel, RowRange part, IndexUploads* uploads) {
    const std::size_t n_src = src.rows();
    const std::size_t row_bytes = src.row_size() * dtype_size(src.dtype());
    std::vector<std::size_t> shape = src.shape();
    shape[0] = part.count();
    const bool have_mirror = mirror && mirror->has_storage();

    const RowRange* range = sel ? std::get_if<RowRange>(&*sel) : nullptr;
    if (!sel || range) {
        const std::size_t first = (range ? range->start : 0) + part.start;
        if (first + part.count() > n_src) throw BoundsError("excerpt: rows past the end of the source");
        if (have_mirror)  // zero-copy view of the HBM mirror
            return mirror->reinterpret(src.offset_bytes() + first * row_bytes, std::move(shape), src.dtype());
        DevBuffer out = DevBuffer::alloc(rd, std::move(shape), src.dtype());
        if (out.byte_size())
            check(synk_copy(rd->h, out.data(), src.bytes() + first * row_bytes, out.byte_size()), "excerpt: H2D rows");
        return out;
    }

    const IndexList& list = std::get<IndexList>(*sel);
    if (part.stop > list.size()) throw BoundsError("excerpt_rows(): part extends past the index list");
    DevBuffer out = DevBuffer::alloc(rd, std::move(shape), src.dtype());
    if (part.count() == 0 || row_bytes == 0) return out;
    const std::pair<const std::size_t*, std::size_t> key{list.data() + part.start, part.count()};
    DevBuffer idx;
    if (uploads)
        for (auto& [k, buf] : uploads->done)
            if (k == key) idx = buf;
    if (!idx.has_storage()) {
        idx = upload_indices(rd, key.first, key.second);
        if (uploads) uploads->done.emplace_back(key, idx);
    }

    const void* base = nullptr;
    DevBuffer staged;  // keeps a device copy alive when the host source is pageable
    if (have_mirror) {
        base = static_cast<const char*>(mirror->data()) + src.offset_bytes();
    } else if (is_mapped_host(src.bytes())) {
        base = src.bytes();  // gather straight out of pinned host memory over PCIe
    } else {
        staged = DevBuffer::alloc(rd, src.shape(), src.dtype());
        check(synk_copy(rd->h, staged.data(), src.bytes(), src.byte_size()), "excerpt: stage pageable source");
        base = staged.data();
    }
    check(synk_gather_rows(rd->h, base, n_src, row_bytes, static_cast<const std::uint64_t*>(idx.data()),
                           part.count(), out.data()),
          "gather_rows");
    return out;
}

DevBuffer select_device_rows(const std::shared_ptr<RankDevice>& rd, const DevBuffer& src, const IndexSelection& sel) {
    if (const RowRange* r = std::get_if<RowRange>(&sel)) return src.slice_rows(*r);
    const IndexList& list = std::get<IndexList>(sel);
    std::vector<std::size_t> shape = src.shape();
    shape[0] = list.size();
    DevBuffer out = DevBuffer::alloc(rd, std::move(shape), src.dtype());
    const std::size_t row_bytes = src.row_size() * dtype_size(src.dtype());
    if (list.empty() || row_bytes == 0) return out;
    DevBuffer idx = upload_indices(rd, list.data(), list.size());
    check(synk_gather_rows(rd->h, src.data(), src.rows(), row_bytes, static_cast<const std::uint64_t*>(idx.data()),
                           list.size(), out.data()),
          "gather_rows (replica)");
    return out;
}

} // namespace synkpar::detail
