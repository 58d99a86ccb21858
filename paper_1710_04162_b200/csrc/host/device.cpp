// DevBuffer, rank device contexts and the C-ABI status -> exception mapping.

#include <cstring>
#include <mutex>
#include <sstream>

#include "internal.hpp"
#include "synkpar/device.hpp"

namespace synkpar {

namespace detail {

[[noreturn]] void throw_status(int rc, const std::string& what) {
    std::string msg = what + ": " + synk_last_error();
    switch (rc) {
    case SYNK_EBOUNDS: throw BoundsError(msg);
    case SYNK_ESHAPE: throw ShapeError(msg);
    case SYNK_EDTYPE: throw DTypeError(msg);
    case SYNK_EARG: throw ArgumentError(msg);
    default: throw DeviceError(msg);
    }
}

void check(int rc, const char* what) {
    if (rc != SYNK_OK) throw_status(rc, what);
}

synk_dev* RankDevice::aux_handle() {
    if (!aux) check(synk_open_aux(h, &aux), "open aux stream");
    return aux;
}

void* RankDevice::take_block(std::size_t bytes) {
    {
        std::lock_guard<std::mutex> lock(cache_mu);
        auto it = cache.find(bytes);
        if (it != cache.end() && !it->second.empty()) {
            void* p = it->second.back();
            it->second.pop_back();
            cache_bytes -= bytes;
            return p;
        }
    }
    void* p = nullptr;
    check(synk_alloc(h, bytes, &p), "HBM allocation");
    return p;
}

void RankDevice::release_block(void* ptr, std::size_t bytes) {
    if (bytes <= kCacheMaxBlock) {
        std::lock_guard<std::mutex> lock(cache_mu);
        if (cache_bytes + bytes <= kCacheMaxBytes) {
            cache[bytes].push_back(ptr);
            cache_bytes += bytes;
            return;
        }
    }
    synk_free(h, ptr);  // stream-ordered; errors at teardown are moot
}

RankDevice::~RankDevice() {
    for (auto& [bytes, list] : cache)
        for (void* p : list) synk_free(h, p);
    if (aux) synk_close(aux);
    if (h && index_stage) synk_free(h, index_stage);
    if (staging) synk_host_free(staging);
    if (h && scratch) synk_free(h, scratch);
    if (h) synk_close(h);
}

void* rank_scratch(const std::shared_ptr<RankDevice>& rd, std::size_t bytes) {
    if (bytes <= rd->scratch_bytes) return rd->scratch;
    if (rd->scratch) check(synk_free(rd->h, rd->scratch), "scratch free");  // stream-ordered: after prior users
    rd->scratch = nullptr;
    rd->scratch_bytes = 0;
    const std::size_t grown = bytes + bytes / 4;
    check(synk_alloc(rd->h, grown, &rd->scratch), "scratch alloc");
    rd->scratch_bytes = grown;
    return rd->scratch;
}

DevStorage::~DevStorage() {
    if (ptr && owner && !external) owner->release_block(ptr, bytes);
}

int synk_dtype(DType dt) { return dt == DType::Float32 ? SYNK_F32 : SYNK_F64; }

int synk_op(ReduceOp op) { return static_cast<int>(op); }

DevBuffer dev_from_host(const std::shared_ptr<RankDevice>& rd, const NdBuffer& host) {
    DevBuffer out = DevBuffer::alloc(rd, host.shape(), host.dtype());
    if (host.byte_size()) check(synk_copy(rd->h, out.data(), host.bytes(), host.byte_size()), "H2D copy");
    return out;
}

void dev_to_host_into(const DevBuffer& buf, std::byte* dst) {
    if (!buf.byte_size()) return;
    check(synk_copy(buf.owner()->h, dst, buf.data(), buf.byte_size()), "D2H copy");
}

NdBuffer dev_to_host(const DevBuffer& buf) {
    NdBuffer out = NdBuffer::uninitialized(buf.shape(), buf.dtype());
    const std::size_t bytes = buf.byte_size();
    if (bytes && bytes <= RankDevice::kStagingBytes) {
        RankDevice& rd = *buf.owner();
        std::lock_guard<std::mutex> lock(rd.staging_mu);
        if (!rd.staging) check(synk_host_alloc(RankDevice::kStagingBytes, &rd.staging), "staging alloc");
        check(synk_copy(rd.h, rd.staging, buf.data(), bytes), "D2H copy");
        dev_sync(buf.owner());
        std::memcpy(out.bytes_mut(), rd.staging, bytes);
        return out;
    }
    if (bytes) {
        dev_to_host_into(buf, out.bytes_mut());
        dev_sync(buf.owner());
    }
    return out;
}

DevBuffer dev_clone(const std::shared_ptr<RankDevice>& rd, const DevBuffer& src) {
    DevBuffer out = DevBuffer::alloc(rd, src.shape(), src.dtype());
    if (src.byte_size()) check(synk_copy(rd->h, out.data(), src.data(), src.byte_size()), "device clone");
    return out;
}

void dev_sync(const std::shared_ptr<RankDevice>& rd) { check(synk_sync(rd->h), "device sync"); }

std::shared_ptr<RankDevice> utility_device() {
    static std::mutex mu;
    static std::shared_ptr<RankDevice> dev;
    std::lock_guard<std::mutex> lock(mu);
    if (!dev) {
        int ids[1] = {0};
        synk_dev* h = nullptr;
        check(synk_open(1, ids, &h), "utility device (GPU 0)");
        dev = std::make_shared<RankDevice>();
        dev->h = h;
        dev->rank = 0;
        dev->device = 0;
    }
    check(synk_bind(dev->h), "bind GPU 0");
    return dev;
}

} // namespace detail

DevBuffer DevBuffer::alloc(const std::shared_ptr<detail::RankDevice>& owner, std::vector<std::size_t> shape,
                           DType dtype) {
    DevBuffer b;
    b.shape_ = std::move(shape);
    b.dtype_ = dtype;
    auto st = std::make_shared<detail::DevStorage>();
    st->owner = owner;
    st->bytes = b.byte_size();
    if (st->bytes) st->ptr = owner->take_block(st->bytes);
    b.store_ = std::move(st);
    return b;
}

DevBuffer DevBuffer::wrap_external(const std::shared_ptr<detail::RankDevice>& owner, void* ptr, std::size_t bytes) {
    DevBuffer b;
    b.shape_ = {bytes};
    b.dtype_ = DType::Float64;  // bookkeeping only: views reinterpret it
    auto st = std::make_shared<detail::DevStorage>();
    st->owner = owner;
    st->bytes = bytes;
    st->ptr = ptr;
    st->external = true;
    b.store_ = std::move(st);
    return b;
}

DevBuffer DevBuffer::zeros(const std::shared_ptr<detail::RankDevice>& owner, std::vector<std::size_t> shape,
                           DType dtype) {
    DevBuffer b = alloc(owner, std::move(shape), dtype);
    if (b.byte_size()) detail::check(synk_memset(owner->h, b.data(), 0, b.byte_size()), "HBM zero fill");
    return b;
}

std::size_t DevBuffer::rows() const {
    if (shape_.empty()) throw ShapeError("rows(): a rank-0 buffer has no leading dimension");
    return shape_[0];
}

std::size_t DevBuffer::row_size() const {
    if (shape_.empty()) throw ShapeError("row_size(): a rank-0 buffer has no leading dimension");
    return element_count(std::span<const std::size_t>(shape_).subspan(1));
}

std::string DevBuffer::shape_string() const {
    std::ostringstream os;
    os << '(';
    for (std::size_t i = 0; i < shape_.size(); ++i) os << (i ? ", " : "") << shape_[i];
    os << ')';
    return os.str();
}

void* DevBuffer::data() const noexcept {
    return store_ && store_->ptr ? static_cast<char*>(store_->ptr) + offset_ : nullptr;
}

int DevBuffer::device() const noexcept { return store_ && store_->owner ? store_->owner->device : -1; }

const std::shared_ptr<detail::RankDevice>& DevBuffer::owner() const {
    if (!store_) throw ArgumentError("DevBuffer: empty buffer has no owning rank");
    return store_->owner;
}

DevBuffer DevBuffer::slice_rows(RowRange r) const {
    std::size_t n = rows();
    if (r.start > r.stop || r.stop > n)
        throw BoundsError("slice_rows(): rows [" + std::to_string(r.start) + ", " + std::to_string(r.stop) +
                          ") not within " + std::to_string(n));
    DevBuffer v = *this;
    v.shape_[0] = r.count();
    v.offset_ = offset_ + r.start * row_size() * dtype_size(dtype_);
    return v;
}

DevBuffer DevBuffer::view_reshaped(std::vector<std::size_t> shape) const {
    if (element_count(shape) != size()) throw ShapeError("view_reshaped(): element count changes");
    DevBuffer v = *this;
    v.shape_ = std::move(shape);
    return v;
}

DevBuffer DevBuffer::reinterpret(std::size_t byte_offset, std::vector<std::size_t> shape, DType dtype) const {
    if (!store_) throw ArgumentError("reinterpret(): empty buffer");
    DevBuffer v;
    v.store_ = store_;
    v.offset_ = offset_ + byte_offset;
    v.shape_ = std::move(shape);
    v.dtype_ = dtype;
    if (v.offset_ + v.byte_size() > store_->bytes) throw BoundsError("reinterpret(): view runs past the allocation");
    return v;
}

} // namespace synkpar
