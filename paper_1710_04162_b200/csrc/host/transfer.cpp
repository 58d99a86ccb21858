// Scatter-share staging: host rows -> HBM of one rank.

#include "transfer.hpp"

#include <algorithm>

#include <cstring>
#include <vector>

namespace synkpar::detail {

static_assert(sizeof(std::size_t) == sizeof(std::uint64_t), "index lists are u64 on the device");

SelView SelView::of(const std::optional<IndexSelection>& sel) {
    SelView v;
    if (!sel) return v;
    v.has = true;
    if (const RowRange* r = std::get_if<RowRange>(&*sel)) {
        v.is_range = true;
        v.range = *r;
    } else {
        const IndexList& l = std::get<IndexList>(*sel);
        v.list = reinterpret_cast<const std::uint64_t*>(l.data());
        v.count = l.size();
    }
    return v;
}

SelView SelView::borrowed(const std::uint64_t* list, std::size_t count) {
    SelView v;
    v.has = true;
    v.list = list;
    v.count = count;
    return v;
}

void validate_view(const SelView& sel, std::size_t n) {
    if (!sel.has) return;
    if (sel.is_range) {
        validate_selection(IndexSelection(sel.range), n);
        return;
    }
    // four independent maxima: no loop-carried dependency through one cmov
    // (the per-step host bounds check of C5's 8192-entry index list)
    std::uint64_t h0 = 0, h1 = 0, h2 = 0, h3 = 0;
    std::size_t i = 0;
    for (; i + 4 <= sel.count; i += 4) {
        h0 = sel.list[i] > h0 ? sel.list[i] : h0;
        h1 = sel.list[i + 1] > h1 ? sel.list[i + 1] : h1;
        h2 = sel.list[i + 2] > h2 ? sel.list[i + 2] : h2;
        h3 = sel.list[i + 3] > h3 ? sel.list[i + 3] : h3;
    }
    for (; i < sel.count; ++i) h0 = sel.list[i] > h0 ? sel.list[i] : h0;
    const std::uint64_t hi = std::max(std::max(h0, h1), std::max(h2, h3));
    if (sel.count == 0 || hi < n) return;
    for (std::size_t i = 0; i < sel.count; ++i)
        if (sel.list[i] >= n)
            throw BoundsError("selection index " + std::to_string(sel.list[i]) + " not within " + std::to_string(n) +
                              " rows");
}

namespace {

// Device-side address of page-locked host memory (kernels read it in place),
// or nullptr when `host` is not page-locked.
template <class T>
const T* device_view(const T* host) {
    const void* d = nullptr;
    if (!host || synk_host_device_ptr(host, &d) != SYNK_OK) return nullptr;
    return static_cast<const T*>(d);
}

} // namespace

DevBuffer upload_indices(const std::shared_ptr<RankDevice>& rd, const std::uint64_t* idx, std::size_t n) {
    DevBuffer out = DevBuffer::alloc(rd, {n}, DType::Float64);  // 8-byte slots; dtype is bookkeeping
    // Pinned sources go out as an async DMA; pageable ones are staged by the driver.
    if (n) check(synk_copy(rd->h, out.data(), idx, n * sizeof(std::uint64_t)), "upload indices");
    return out;
}

DevBuffer excerpt_to_device(const std::shared_ptr<RankDevice>& rd, const NdBuffer& src, const DevBuffer* mirror,
                            const SelView& sel, RowRange part, IndexUploads* uploads) {
    const std::size_t n_src = src.rows();
    const std::size_t row_bytes = src.row_size() * dtype_size(src.dtype());
    std::vector<std::size_t> shape = src.shape();
    shape[0] = part.count();
    const bool have_mirror = mirror && mirror->has_storage();

    if (!sel.has || sel.is_range) {
        const std::size_t first = (sel.has ? sel.range.start : 0) + part.start;
        if (first + part.count() > n_src) throw BoundsError("excerpt: rows past the end of the source");
        if (have_mirror)  // zero-copy view of the HBM mirror
            return mirror->reinterpret(src.offset_bytes() + first * row_bytes, std::move(shape), src.dtype());
        DevBuffer out = DevBuffer::alloc(rd, std::move(shape), src.dtype());
        if (out.byte_size())
            check(synk_copy(rd->h, out.data(), src.bytes() + first * row_bytes, out.byte_size()), "excerpt: H2D rows");
        return out;
    }

    if (part.stop > sel.count) throw BoundsError("excerpt_rows(): part extends past the index list");
    DevBuffer out = DevBuffer::alloc(rd, std::move(shape), src.dtype());
    if (part.count() == 0 || row_bytes == 0) return out;
    const void* base = nullptr;
    DevBuffer staged;  // keeps a device copy alive when the host source is pageable
    if (have_mirror) {
        base = static_cast<const char*>(mirror->data()) + src.offset_bytes();
    } else if (const std::byte* dv = device_view(src.bytes())) {
        base = dv;  // gather straight out of pinned host memory over PCIe
    } else {
        // Pageable source: gather the selected rows on the host and upload
        // only those (not the whole source per rank per call); the rank's
        // stream is drained before the temporary goes. An out-of-range index (possible only
        // when the bounds check is deferred to the device) takes the device
        // path instead, whose kernel flags it.
        const std::uint64_t* list = sel.list + part.start;
        bool in_range = true;
        for (std::size_t i = 0; i < part.count() && in_range; ++i) in_range = list[i] < n_src;
        if (in_range) {
            std::vector<std::byte> rows(part.count() * row_bytes);
            for (std::size_t i = 0; i < part.count(); ++i)
                std::memcpy(rows.data() + i * row_bytes, src.bytes() + list[i] * row_bytes, row_bytes);
            check(synk_copy(rd->h, out.data(), rows.data(), rows.size()), "excerpt: H2D gathered rows");
            dev_sync(rd);
            return out;
        }
        staged = DevBuffer::alloc(rd, src.shape(), src.dtype());
        check(synk_copy(rd->h, staged.data(), src.bytes(), src.byte_size()), "excerpt: stage pageable source");
        base = staged.data();
    }
    const std::pair<const std::uint64_t*, std::size_t> key{sel.list + part.start, part.count()};
    if (key.second <= SYNK_GATHER_INLINE_MAX && n_src <= (std::size_t(1) << 32)) {
        // one short batch: the list rides in the launch (no PCIe index reads,
        // no upload), pageable or pinned alike
        check(synk_gather_rows_inline(rd->h, base, n_src, row_bytes, key.first, key.second, out.data()),
              "gather_rows (inline list)");
        return out;
    }
    DevBuffer idx;
    const std::uint64_t* idx_ptr = nullptr;
    if (const std::uint64_t* dv = device_view(key.first)) {
        idx_ptr = dv;  // pinned list: the gather kernel reads it in place over PCIe
    } else {
        if (uploads)
            for (auto& [k, buf] : uploads->done)
                if (k == key) idx = buf;
        if (!idx.has_storage()) {
            idx = upload_indices(rd, key.first, key.second);
            if (uploads) uploads->done.emplace_back(key, idx);
        }
        idx_ptr = static_cast<const std::uint64_t*>(idx.data());
    }

    check(synk_gather_rows(rd->h, base, n_src, row_bytes, idx_ptr, part.count(), out.data()), "gather_rows");
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
    const auto* l = reinterpret_cast<const std::uint64_t*>(list.data());
    if (list.size() <= SYNK_GATHER_INLINE_MAX && src.rows() <= (std::size_t(1) << 32)) {
        check(synk_gather_rows_inline(rd->h, src.data(), src.rows(), row_bytes, l, list.size(), out.data()),
              "gather_rows (replica, inline list)");
        return out;
    }
    DevBuffer idx = upload_indices(rd, reinterpret_cast<const std::uint64_t*>(list.data()), list.size());
    check(synk_gather_rows(rd->h, src.data(), src.rows(), row_bytes, static_cast<const std::uint64_t*>(idx.data()),
                           list.size(), out.data()),
          "gather_rows (replica)");
    return out;
}

} // namespace synkpar::detail
