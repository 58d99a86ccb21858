// Replicated variables: replica r in HBM of rank r's GPU; collectives are
// one phase of the peer-memory tree-order kernels (include/synk_cuda.h).

#include "synkpar/replicated.hpp"

#include <atomic>
#include <cstring>

#include "internal.hpp"
#include "transfer.hpp"

namespace synkpar {

namespace {
// Collectives up to this size run as one kernel on rank 0's GPU (latency
// bound: a launch + a sync instead of a phase over every rank thread).
constexpr std::size_t kWholeCollectiveBytes = std::size_t(1) << 20;
} // namespace

namespace detail {


std::vector<DevBuffer>& replicas_of(const ReplicatedVariable& var) {
    if (!var.rec_) throw ArgumentError("empty replicated-variable handle");
    return var.rec_->replicas;
}

std::shared_ptr<PoolState> pool_of(const ReplicatedVariable& var) {
    if (!var.rec_) throw ArgumentError("empty replicated-variable handle");
    return var.rec_->pool;
}

VarRecord& record_of(const ReplicatedVariable& var) {
    if (!var.rec_) throw ArgumentError("empty replicated-variable handle");
    return *var.rec_;
}

namespace {
// Copy the chunks replica t lacks (every chunk q != t of every segment) from
// their owners into dst on rd's stream.
void pull_chunks(const VarRecord::Shard& sh, std::size_t t, DevBuffer& dst, const std::shared_ptr<RankDevice>& rd) {
    const std::size_t W = sh.src.size();
    const std::size_t es = dtype_size(dst.dtype());
    for (auto [first, count] : sh.segs)
        for (std::size_t q = 0; q < W; ++q) {
            if (q == t) continue;
            std::uint64_t lo = 0, hi = 0;
            check(synk_chunk_range(count, static_cast<int>(W), static_cast<int>(q), &lo, &hi), "shard chunk");
            if (lo >= hi) continue;
            const std::size_t off = (first + lo) * es;
            check(synk_copy(rd->h, static_cast<char*>(dst.data()) + off, static_cast<const char*>(sh.src[q].data()) + off,
                            (hi - lo) * es),
                  "gradient all-gather");
        }
}

bool needs_pull(const VarRecord::Shard& sh, const DevBuffer& replica, std::size_t t) {
    return t < sh.src.size() && replica.has_storage() && replica.data() == sh.src[t].data();
}
} // namespace

void materialize(VarRecord& rec) {
    if (!rec.shard) return;
    VarRecord::Shard sh = std::move(*rec.shard);
    rec.shard.reset();
    std::vector<std::shared_ptr<RankDevice>> touched;
    for (std::size_t t = 0; t < rec.replicas.size(); ++t) {
        if (!needs_pull(sh, rec.replicas[t], t)) continue;
        const auto& rd = rec.replicas[t].owner();
        pull_chunks(sh, t, rec.replicas[t], rd);
        touched.push_back(rd);
    }
    for (const auto& rd : touched) dev_sync(rd);
}

void pull_shard(const VarRecord& rec, std::size_t r) {
    if (!rec.shard || r >= rec.replicas.size() || !needs_pull(*rec.shard, rec.replicas[r], r)) return;
    DevBuffer dst = rec.replicas[r];  // shares the replica's storage
    pull_chunks(*rec.shard, r, dst, dst.owner());
}

} // namespace detail

namespace {

std::atomic<std::uint64_t> g_next_var{1};

detail::VarRecord& live(const std::shared_ptr<detail::VarRecord>& rec, const char* what) {
    if (!rec) throw ArgumentError(std::string(what) + ": empty replicated-variable handle");
    return *rec;
}

// live() for the methods that read replica contents: a deferred gradient
// all-gather is completed first (outside a phase only; in a phase the
// lifecycle checks below raise before anything is read).
detail::VarRecord& live_full(const std::shared_ptr<detail::VarRecord>& rec, const char* what) {
    detail::VarRecord& r = live(rec, what);
    if (r.shard && static_cast<detail::PoolLifecycle>(r.pool->lifecycle.load()) != detail::PoolLifecycle::InPhase)
        detail::materialize(r);
    return r;
}

void check_rank(const detail::VarRecord& rec, std::size_t rank, const char* what) {
    if (rank >= rec.replicas.size())
        throw ArgumentError(std::string(what) + ": rank " + std::to_string(rank) + " out of " +
                            std::to_string(rec.replicas.size()));
}

void check_same_shapes(const detail::VarRecord& rec, const char* what) {
    for (std::size_t r = 1; r < rec.replicas.size(); ++r)
        if (!rec.replicas[r].same_shape(rec.replicas[0]))
            throw ShapeError(std::string(what) + ": replica shapes differ across ranks (" +
                             rec.replicas[0].shape_string() + " vs rank " + std::to_string(r) + " " +
                             rec.replicas[r].shape_string() + ")");
}

void no_phase(const detail::VarRecord& rec, const char* what) {
    if (static_cast<detail::PoolLifecycle>(rec.pool->lifecycle.load()) == detail::PoolLifecycle::InPhase)
        throw LifecycleError(std::string(what) + ": not allowed while a phase is in flight");
}

void not_gather(ReduceOp op, const char* what) {
    if (op == ReduceOp::Gather) throw ArgumentError(std::string(what) + ": Gather is not a reduction (use gather())");
}

std::vector<void*> replica_ptrs(const detail::VarRecord& rec) {
    std::vector<void*> p;
    for (const DevBuffer& b : rec.replicas) p.push_back(b.data());
    return p;
}

// Inside a phase: the dtype check combine_inplace performs on each fold
// (tensor.cpp:227-240) raises there, so it surfaces as PhaseError.
void require_same_dtype(const detail::VarRecord& rec) {
    for (const DevBuffer& b : rec.replicas)
        if (b.dtype() != rec.replicas[0].dtype()) throw DTypeError("combine_inplace: dtype mismatch across replicas");
}

// One Collective phase around an NCCL call per rank. A collective blocks its
// rank until every peer has joined, so the ranks first meet on the host: a
// rank whose pre-collective work throws aborts the rendezvous and its peers
// fail with it (fail-stop, PhaseError of the lowest failing rank) instead of
// waiting inside NCCL forever.
template <class Enqueue>
void nccl_phase(detail::PoolState& st, Enqueue&& enqueue) {
    detail::PhaseRendezvous rv(st.world);
    detail::run_pool_phase(st, PhaseKind::Collective, [&](std::size_t r) {
        try {
            rv.arrive_and_wait();
            enqueue(r);
        } catch (...) {
            rv.abort();
            throw;
        }
        detail::dev_sync(st.ranks[r]);
    });
}

} // namespace

ReplicatedVariable replicate(WorkerPool& pool, const NdBuffer& init) {
    auto st = detail::state_of(pool);
    detail::require_idle(*st, "replicate");
    auto rec = std::make_shared<detail::VarRecord>();
    rec->id = g_next_var.fetch_add(1);
    rec->pool = st;
    rec->replicas.resize(st->world);
    rec->shadows.resize(st->world);
    detail::run_pool_phase(*st, PhaseKind::Distribute, [&](std::size_t r) {
        rec->replicas[r] = detail::dev_from_host(st->ranks[r], init);
        detail::dev_sync(st->ranks[r]);
    });
    return ReplicatedVariable(std::move(rec));
}

std::uint64_t ReplicatedVariable::id() const { return live(rec_, "id").id; }
std::size_t ReplicatedVariable::world() const { return live(rec_, "world").replicas.size(); }
DType ReplicatedVariable::dtype() const { return live(rec_, "dtype").replicas.at(0).dtype(); }

void ReplicatedVariable::broadcast(std::size_t src) {
    detail::NvtxRange range("synk.broadcast");
    detail::VarRecord& rec = live_full(rec_, "broadcast");
    rec.mutated();
    check_rank(rec, src, "broadcast");
    detail::PoolState& st = *rec.pool;
    detail::require_idle(st, "broadcast");
    const DevBuffer& s = rec.replicas[src];
    // Every destination gets storage of the source's shape first (a clone in
    // the reference, replicated.cpp:118-121).
    for (std::size_t r = 0; r < rec.replicas.size(); ++r) {
        if (r == src) continue;
        DevBuffer& d = rec.replicas[r];
        if (!d.same_shape(s) || d.dtype() != s.dtype() || d.shares_storage(s) || !d.has_storage()) {
            d = DevBuffer::alloc(st.ranks[r], s.shape(), s.dtype());
            detail::dev_sync(st.ranks[r]);
        }
    }
    std::vector<void*> ptrs = replica_ptrs(rec);
    const std::size_t bytes = s.byte_size();
    if (st.nccl) {  // library baseline backend (ForkOptions::collectives = "nccl")
        nccl_phase(st, [&](std::size_t r) {
            detail::check(synk_nccl_broadcast(st.handles[r], static_cast<int>(src), ptrs[r], bytes), "broadcast (nccl)");
        });
        rec.coherent = true;
        return;
    }
    if (bytes <= kWholeCollectiveBytes) {
        // Small buffer: rank 0's GPU copies every chunk over the peer pointers
        // (all streams are idle between phases), no rank thread is woken.
        detail::check(synk_broadcast_whole(st.handles[0], static_cast<int>(st.world), static_cast<int>(src),
                                           ptrs.data(), bytes),
                      "broadcast");
        detail::dev_sync(st.ranks[0]);
        rec.coherent = true;
        return;
    }
    detail::run_pool_phase(st, PhaseKind::Collective, [&](std::size_t r) {
        detail::check(synk_broadcast(st.handles[r], static_cast<int>(st.world), static_cast<int>(src), ptrs.data(), bytes),
                      "broadcast");
        detail::dev_sync(st.ranks[r]);
    });
    rec.coherent = true;
}

void ReplicatedVariable::all_reduce(ReduceOp op) {
    detail::NvtxRange range("synk.all_reduce");
    detail::VarRecord& rec = live_full(rec_, "all_reduce");
    rec.mutated();
    not_gather(op, "all_reduce");
    check_same_shapes(rec, "all_reduce");
    detail::PoolState& st = *rec.pool;
    std::vector<void*> ptrs = replica_ptrs(rec);
    const std::size_t n = rec.replicas[0].size();
    const int dt = detail::synk_dtype(rec.replicas[0].dtype());
    if (st.nccl) {  // library baseline backend: NCCL's reduction order (within tolerance, not bitwise)
        nccl_phase(st, [&](std::size_t r) {
            require_same_dtype(rec);
            detail::check(synk_nccl_all_reduce(st.handles[r], dt, detail::synk_op(op), ptrs[r], n), "all_reduce (nccl)");
        });
        rec.coherent = true;
        return;
    }
    if (rec.replicas[0].byte_size() <= kWholeCollectiveBytes) {
        // Small buffer: one kernel on rank 0's GPU folds every chunk (same
        // per-element tree order) and writes all replicas over the peer
        // pointers -- no rank thread is woken, one launch + one sync.
        detail::require_idle(st, "all_reduce");
        require_same_dtype(rec);
        detail::check(synk_all_reduce_whole(st.handles[0], static_cast<int>(st.world), dt, detail::synk_op(op),
                                            ptrs.data(), n),
                      "all_reduce");
        detail::dev_sync(st.ranks[0]);
        rec.coherent = true;
        return;
    }
    detail::run_pool_phase(st, PhaseKind::Collective, [&](std::size_t r) {
        require_same_dtype(rec);
        detail::check(synk_all_reduce(st.handles[r], static_cast<int>(st.world), dt, detail::synk_op(op), ptrs.data(), n),
                      "all_reduce");
        detail::dev_sync(st.ranks[r]);
    });
    rec.coherent = true;
}

void ReplicatedVariable::reduce(ReduceOp op, std::size_t dst) {
    detail::VarRecord& rec = live_full(rec_, "reduce");
    rec.mutated();
    not_gather(op, "reduce");
    check_rank(rec, dst, "reduce");
    check_same_shapes(rec, "reduce");
    detail::PoolState& st = *rec.pool;
    std::vector<void*> ptrs = replica_ptrs(rec);
    const DevBuffer& first = rec.replicas[0];
    DevBuffer folded;
    detail::run_pool_phase(st, PhaseKind::Collective, [&](std::size_t r) {
        if (r != dst) return;
        require_same_dtype(rec);
        folded = DevBuffer::alloc(st.ranks[r], first.shape(), first.dtype());
        detail::check(synk_tree_reduce(st.handles[r], static_cast<int>(st.world), detail::synk_dtype(first.dtype()),
                                       detail::synk_op(op), ptrs.data(), first.size(), folded.data()),
                      "reduce");
        detail::dev_sync(st.ranks[r]);
    });
    rec.replicas[dst] = std::move(folded);
    if (rec.replicas.size() > 1) rec.coherent = false;
}

NdBuffer ReplicatedVariable::gather() const {
    detail::VarRecord& rec = live_full(rec_, "gather");
    detail::PoolState& st = *rec.pool;
    // concat_rows validation (tensor.cpp:287-313) happens on rank 0 inside
    // the phase in the reference, so its errors surface as PhaseError.
    std::string problem;
    std::size_t total = 0;
    std::vector<std::size_t> offsets;
    const DevBuffer& head = rec.replicas[0];
    for (const DevBuffer& p : rec.replicas) {
        if (p.rank() == 0) {
            problem = "rows(): a rank-0 buffer has no leading dimension";
            break;
        }
        if (p.dtype() != head.dtype()) {
            problem = "concat_rows(): parts mix dtypes";
            break;
        }
        if (p.rank() != head.rank() || !std::equal(p.shape().begin() + 1, p.shape().end(), head.shape().begin() + 1)) {
            problem = "concat_rows(): trailing shapes differ";
            break;
        }
        total += p.rows();
    }
    NdBuffer out;
    if (problem.empty()) {
        std::vector<std::size_t> shape = head.shape();
        shape[0] = total;
        out = NdBuffer::uninitialized(std::move(shape), head.dtype());
        std::size_t row_bytes = head.row_size() * dtype_size(head.dtype()), at = 0;
        for (std::size_t r = 0; r < rec.replicas.size(); ++r) {
            offsets.push_back(at);
            at += rec.replicas[r].rows() * row_bytes;
        }
    }
    detail::run_pool_phase(st, PhaseKind::Collective, [&](std::size_t r) {
        if (!problem.empty()) {
            if (r == 0) {
                if (problem.rfind("concat_rows(): parts", 0) == 0) throw DTypeError(problem);
                throw ShapeError(problem);
            }
            return;
        }
        detail::dev_to_host_into(rec.replicas[r], out.bytes_mut() + offsets[r]);
        detail::dev_sync(st.ranks[r]);
    });
    return out;
}

NdBuffer ReplicatedVariable::get_value(std::size_t rank) const {
    detail::VarRecord& rec = live_full(rec_, "get_value");
    check_rank(rec, rank, "get_value");
    no_phase(rec, "get_value");
    return detail::dev_to_host(rec.replicas[rank]);
}

void ReplicatedVariable::set_value(std::size_t rank, const NdBuffer& value) {
    detail::VarRecord& rec = live(rec_, "set_value");
    rec.mutated();
    check_rank(rec, rank, "set_value");
    no_phase(rec, "set_value");
    const auto& rd = rec.pool->ranks[rank];
    rec.replicas[rank] = detail::dev_from_host(rd, value);
    detail::dev_sync(rd);
    if (rec.replicas.size() > 1) rec.coherent = false;
}

void ReplicatedVariable::scatter_value(const NdBuffer& data, const std::optional<IndexSelection>& indexes) {
    detail::VarRecord& rec = live(rec_, "scatter_value");
    rec.mutated();
    rec.shard.reset();  // every replica is replaced
    const std::size_t n = data.rows();
    std::size_t eff = n;
    if (indexes) {
        validate_selection(*indexes, n);
        eff = selection_count(*indexes);
    }
    std::vector<RowRange> parts = partition_rows(eff, rec.replicas.size());
    detail::PoolState& st = *rec.pool;
    detail::run_pool_phase(st, PhaseKind::ScatterVar, [&](std::size_t r) {
        // Fresh HBM storage per rank (never aliases the source, replicated.cpp:186-188).
        rec.replicas[r] = detail::excerpt_to_device(st.ranks[r], data, nullptr, detail::SelView::of(indexes), parts[r]);
        detail::dev_sync(st.ranks[r]);
    });
    if (rec.replicas.size() > 1) rec.coherent = false;
}

void ReplicatedVariable::scatter_value(const SharedInputArray& data, const std::optional<IndexSelection>& indexes) {
    scatter_value(data.view(), indexes);
}

void ReplicatedVariable::scatter_uniform(const std::vector<std::size_t>& shape, DType dtype, std::uint64_t seed) {
    detail::VarRecord& rec = live(rec_, "scatter_uniform");
    rec.mutated();
    rec.shard.reset();  // every replica is replaced
    if (shape.empty()) throw ShapeError("scatter_uniform: a rank-0 shape has no rows to scatter");
    const std::size_t row = element_count(shape) / std::max<std::size_t>(shape[0], 1);
    std::vector<RowRange> parts = partition_rows(shape[0], rec.replicas.size());
    detail::PoolState& st = *rec.pool;
    detail::run_pool_phase(st, PhaseKind::ScatterVar, [&](std::size_t r) {
        std::vector<std::size_t> s = shape;
        s[0] = parts[r].stop - parts[r].start;
        DevBuffer b = DevBuffer::alloc(st.ranks[r], s, dtype);
        detail::check(synk_fill_uniform(st.handles[r], detail::synk_dtype(dtype), b.data(), b.size(), seed,
                                        parts[r].start * row),
                      "scatter_uniform");
        detail::dev_sync(st.ranks[r]);
        rec.replicas[r] = std::move(b);
    });
    if (rec.replicas.size() > 1) rec.coherent = false;
}

bool ReplicatedVariable::replicas_coherent() const {
    detail::VarRecord& rec = live_full(rec_, "replicas_coherent");
    no_phase(rec, "replicas_coherent");
    const DevBuffer& a = rec.replicas[0];
    for (std::size_t r = 1; r < rec.replicas.size(); ++r) {
        const DevBuffer& b = rec.replicas[r];
        if (b.dtype() != a.dtype() || !b.same_shape(a)) return false;
        int eq = 1;
        detail::check(synk_equal(b.owner()->h, b.data(), a.data(), a.byte_size(), &eq), "replicas_coherent");
        if (!eq) return false;
    }
    return true;
}

DevBuffer ReplicatedVariable::device_value(std::size_t rank) const {
    detail::VarRecord& rec = live_full(rec_, "device_value");
    rec.mutated();
    check_rank(rec, rank, "device_value");
    return rec.replicas[rank];
}

} // namespace synkpar
