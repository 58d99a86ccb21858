// Optimizers, flat parameter block and the synchronous trainer (sgd.hpp).

#include "synkpar/sgd.hpp"

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>

#include "internal.hpp"

namespace synkpar {

namespace {

using Clock = std::chrono::steady_clock;
double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

std::size_t aux_needed(const UpdateRule& r) noexcept {
    if (std::holds_alternative<SgdRule>(r)) return 0;
    return std::holds_alternative<AdamRule>(r) ? 2 : 1;
}

int rule_code(const UpdateRule& r) {
    if (std::holds_alternative<SgdRule>(r)) return SYNK_RULE_SGD;
    if (std::holds_alternative<MomentumRule>(r)) return SYNK_RULE_MOMENTUM;
    if (std::holds_alternative<RmsPropRule>(r)) return SYNK_RULE_RMSPROP;
    return SYNK_RULE_ADAM;
}

std::vector<double> rule_hyper(const UpdateRule& r) {
    if (const auto* m = std::get_if<MomentumRule>(&r)) return {m->mu};
    if (const auto* p = std::get_if<RmsPropRule>(&r)) return {p->rho, p->eps};
    if (const auto* a = std::get_if<AdamRule>(&r)) return {a->beta1, a->beta2, a->eps};
    return {0.0};
}

void check_step(const OptimizerState& st, const NdBuffer& p, const NdBuffer& g, const char* who) {
    if (p.dtype() != g.dtype()) throw DTypeError(std::string(who) + ": params/grads dtype mismatch");
    if (p.size() != g.size())
        throw ShapeError(std::string(who) + ": params length " + std::to_string(p.size()) + " != grads length " +
                         std::to_string(g.size()));
    if (st.aux.size() != aux_needed(st.rule))
        throw ArgumentError(std::string(who) + ": optimizer state holds " + std::to_string(st.aux.size()) +
                            " auxiliary buffers, rule needs " + std::to_string(aux_needed(st.rule)));
    for (const NdBuffer& a : st.aux)
        if (a.size() != p.size() || a.dtype() != p.dtype())
            throw ShapeError(std::string(who) + ": auxiliary buffer does not match params");
}

// Host-buffer step on the GPU: H2D, one update kernel, D2H back in place.
void device_step(OptimizerState& st, NdBuffer& params, const NdBuffer& grads, const char* who) {
    check_step(st, params, grads, who);
    st.t += 1;
    auto rd = detail::utility_device();
    DevBuffer p = detail::dev_from_host(rd, params);
    DevBuffer g = detail::dev_from_host(rd, grads);
    std::vector<DevBuffer> aux;
    for (const NdBuffer& a : st.aux) aux.push_back(detail::dev_from_host(rd, a));
    std::vector<double> hyper = rule_hyper(st.rule);
    detail::check(synk_optimizer_step(rd->h, detail::synk_dtype(params.dtype()), rule_code(st.rule), hyper.data(), st.lr,
                                      st.t, p.data(), g.data(), aux.size() > 0 ? aux[0].data() : nullptr,
                                      aux.size() > 1 ? aux[1].data() : nullptr, params.size()),
                  who);
    if (params.byte_size()) detail::dev_to_host_into(p, params.bytes_mut());
    for (std::size_t i = 0; i < aux.size(); ++i)
        if (st.aux[i].byte_size()) detail::dev_to_host_into(aux[i], st.aux[i].bytes_mut());
    detail::dev_sync(rd);
}

template <class R>
void require_rule(const OptimizerState& st, const char* who) {
    if (!std::holds_alternative<R>(st.rule)) throw ArgumentError(std::string(who) + ": optimizer state holds another rule");
}

} // namespace

const char* update_rule_name(const UpdateRule& r) noexcept {
    if (std::holds_alternative<SgdRule>(r)) return "sgd";
    if (std::holds_alternative<MomentumRule>(r)) return "momentum";
    if (std::holds_alternative<RmsPropRule>(r)) return "rmsprop";
    return "adam";
}

OptimizerState make_optimizer(UpdateRule rule, double lr, std::size_t n, DType dtype) {
    OptimizerState st;
    st.rule = rule;
    st.lr = lr;
    for (std::size_t i = 0; i < aux_needed(rule); ++i) st.aux.push_back(NdBuffer::zeros({n}, dtype));
    return st;
}

void step_sgd(OptimizerState& st, NdBuffer& p, const NdBuffer& g) {
    require_rule<SgdRule>(st, "step_sgd");
    device_step(st, p, g, "step_sgd");
}
void step_momentum(OptimizerState& st, NdBuffer& p, const NdBuffer& g) {
    require_rule<MomentumRule>(st, "step_momentum");
    device_step(st, p, g, "step_momentum");
}
void step_rmsprop(OptimizerState& st, NdBuffer& p, const NdBuffer& g) {
    require_rule<RmsPropRule>(st, "step_rmsprop");
    device_step(st, p, g, "step_rmsprop");
}
void step_adam(OptimizerState& st, NdBuffer& p, const NdBuffer& g) {
    require_rule<AdamRule>(st, "step_adam");
    device_step(st, p, g, "step_adam");
}
void apply_update(OptimizerState& st, NdBuffer& p, const NdBuffer& g) {
    device_step(st, p, g, update_rule_name(st.rule));
}

bool all_finite(const NdBuffer& buf) noexcept {
    // Host-side debug predicate over a host buffer.
    for (std::size_t i = 0; i < buf.size(); ++i)
        if (!std::isfinite(buf.get(i))) return false;
    return true;
}

// ---- flat block --------------------------------------------------------------------

FlatParamBlock FlatParamBlock::create(WorkerPool& pool, std::span<const NdBuffer> initial) {
    FlatPack pack = flatten_concat(initial);
    FlatParamBlock b;
    b.segments = std::move(pack.segments);
    b.length = pack.flat.size();
    b.params = replicate(pool, pack.flat);
    b.grads = replicate(pool, NdBuffer::zeros({b.length}, pack.flat.dtype()));
    return b;
}

std::vector<NdBuffer> FlatParamBlock::read_params(std::size_t rank) const {
    return unflatten(params.get_value(rank), segments);
}

// ---- trainer -----------------------------------------------------------------------------

SyncSgd::SyncSgd(WorkerPool& pool, FlatParamBlock block, UpdateRule rule, double lr, TrainerOptions opts)
    : pool_(&pool), block_(std::move(block)), opts_(opts), rule_(rule), lr_(lr) {
    const DType dt = block_.params.dtype();
    const std::size_t naux = aux_needed(rule_);
    for (std::size_t i = 0; i < naux; ++i) aux_.push_back(replicate(pool, NdBuffer::zeros({block_.length}, dt)));

    // The per-rank step function (used when gradients are not all-reduced;
    // with the all-reduce on, train_step fuses reduce + update instead).
    Kernel k;
    k.name = std::string("step_") + update_rule_name(rule_);
    k.arity = 1;
    k.reads = {block_.params, block_.grads};
    for (const ReplicatedVariable& a : aux_) k.reads.push_back(a);
    std::vector<std::uint64_t> ids{block_.params.id()};
    for (const ReplicatedVariable& a : aux_) ids.push_back(a.id());
    const int code = rule_code(rule_);
    const std::vector<double> hyper = rule_hyper(rule_);
    const double lr_copy = lr_;
    std::shared_ptr<std::uint64_t> t_ptr = step_box_;
    k.device_fn = [ids, code, hyper, lr_copy, naux, t_ptr](const std::vector<DevBuffer>&, const KernelContext& ctx) {
        const DevBuffer& p0 = ctx.device_replica(0);
        const DevBuffer& g = ctx.device_replica(1);
        if (p0.dtype() != g.dtype()) throw DTypeError("step: params/grads dtype mismatch");
        if (p0.size() != g.size()) throw ShapeError("step: params length != grads length");
        DevBuffer p = detail::dev_clone(ctx.rank_device, p0);
        std::vector<DevBuffer> aux;
        for (std::size_t i = 0; i < naux; ++i) aux.push_back(detail::dev_clone(ctx.rank_device, ctx.device_replica(2 + i)));
        detail::check(synk_optimizer_step(ctx.dev, detail::synk_dtype(p.dtype()), code, hyper.data(), lr_copy, *t_ptr + 1,
                                          p.data(), g.data(), naux > 0 ? aux[0].data() : nullptr,
                                          naux > 1 ? aux[1].data() : nullptr, p.size()),
                      "optimizer step");
        DeviceKernelResult r;
        r.updates.push_back({ids[0], p, UpdateCombine::Overwrite});
        for (std::size_t i = 0; i < naux; ++i) r.updates.push_back({ids[1 + i], aux[i], UpdateCombine::Overwrite});
        return r;
    };
    std::vector<UpdateSpec> specs{UpdateSpec{block_.params, UpdateCombine::Overwrite}};
    for (const ReplicatedVariable& a : aux_) specs.push_back(UpdateSpec{a, UpdateCombine::Overwrite});
    f_step_ = function(pool, std::move(k), {InputSpec{InputMode::Broadcast}}, {}, std::move(specs));
    distribute(pool);
}

// The all-reduce + update chained onto the gradient call's own phase: each
// rank enqueues its gradient work, then (W > 1) signals, meets its peers on
// the host and makes its stream wait for theirs on the device, then enqueues
// the fused all-reduce + 1/W + update kernel; the phase-exit synchronisation
// covers both. Same arithmetic, same order as the two-phase path (sgd.cpp:
// 292-319 of the reference), without the host round trip between them.
// Per-rank timing events of the fused step: 0, 1, 3 the gradient call (share
// start, inputs staged = compute start, compute end), 4..5 rank 0's update
// (4 omitted at W = 1 without overlap: the update starts at event 3).
struct SyncSgd::StepTimers {
    std::vector<void*> per_rank;
    explicit StepTimers(const detail::PoolState& st) {
        per_rank.assign(st.world, nullptr);
        for (std::size_t r = 0; r < st.world; ++r)
            detail::check(synk_timer_create(st.handles[r], 6, &per_rank[r]), "step timers");
    }
    ~StepTimers() {
        for (void* t : per_rank) synk_timer_destroy(t);
    }
};

const StepReport& SyncSgd::last_report() const {
    if (report_pending_ && timers_) {
        report_pending_ = false;
        const auto& t = timers_->per_rank;
        double scatter = 0.0, sec = 0.0, task_max = 0.0, task_sum = 0.0;
        last_.grad_call.rank_compute_s.assign(t.size(), 0.0);
        for (std::size_t r = 0; r < t.size(); ++r) {
            if (synk_timer_elapsed(t[r], 0, 1, &sec) == SYNK_OK) scatter += sec;
            if (synk_timer_elapsed(t[r], 1, 3, &sec) == SYNK_OK) last_.grad_call.rank_compute_s[r] = sec;
            // rank task = its share on the device, staging through compute end
            if (synk_timer_elapsed(t[r], 0, 3, &sec) == SYNK_OK) {
                task_max = std::max(task_max, sec);
                task_sum += sec;
            }
        }
        last_.grad_call.scatter_s = scatter / double(t.size());
        // straggler = max - mean rank task (function.hpp CallReport)
        if (!t.empty()) last_.grad_call.straggler_s = task_max - task_sum / double(t.size());
        if (!t.empty() && synk_timer_elapsed(t[0], update_from_compute_end_ ? 3 : 4, 5, &sec) == SYNK_OK) {
            last_.allreduce_s = sec;
            last_.step_call.total_s = sec;
        }
    }
    return last_;
}

double SyncSgd::fused_step(const ParallelFunction& f_grad, const std::vector<FunctionArg>& batch,
                           const CallOptions& call_opts, Clock::time_point t0) {
    StepReport rep;
    auto st = detail::state_of(*pool_);
    const std::size_t W = st->world;
    auto& grads = detail::replicas_of(block_.grads);
    auto& params = detail::replicas_of(block_.params);
    for (std::size_t r = 1; r < W; ++r)
        if (!grads[r].same_shape(grads[0]))
            throw ShapeError("all_reduce: replica shapes differ across ranks (" + grads[0].shape_string() + " vs rank " +
                             std::to_string(r) + " " + grads[r].shape_string() + ")");
    for (std::size_t r = 0; r < W; ++r) {
        if (params[r].dtype() != grads[r].dtype()) throw DTypeError("step: params/grads dtype mismatch");
        if (params[r].size() != grads[r].size()) throw ShapeError("step: params length != grads length");
    }
    std::vector<void*> pp, a0, a1;
    for (std::size_t r = 0; r < W; ++r) {
        pp.push_back(params[r].data());
        if (aux_.size() > 0) a0.push_back(detail::replicas_of(aux_[0])[r].data());
        if (aux_.size() > 1) a1.push_back(detail::replicas_of(aux_[1])[r].data());
    }
    bool coherent = detail::record_of(block_.params).coherent;
    for (const ReplicatedVariable& a : aux_) coherent = coherent && detail::record_of(a).coherent;
    const std::vector<double> hyper = rule_hyper(rule_);
    const int code = rule_code(rule_);
    const std::uint64_t t_next = t_ + 1;
    // Device times go to the trainer's own timers, resolved on report access.
    const bool lazy = call_opts.device_timing && call_opts.num_slices == 1;
    const bool timing = call_opts.device_timing && !lazy;
    if (lazy && (!timers_ || timers_->per_rank.size() != W)) timers_ = std::make_shared<StepTimers>(*st);
    void* t0_timer = lazy ? timers_->per_rank[0] : nullptr;
    int ma = -1, mb = -1;
    bool aux_marks = false;  // the update ran on rank 0's second stream (overlapped)
    detail::PhaseRendezvous rv(W);

    // Overlap: a kernel that reports gradient segments as they become final
    // (the bf16 MLP: one per layer, in backward order) gets each segment's
    // all-reduce + update on the rank's second stream as soon as every rank
    // signalled it -- the DDP-style bucketed overlap of the collective with
    // the rest of the backward pass. Used only when every rank reported the
    // same full cover of the gradient and no unequal-shard pre-scale is due.
    constexpr int kSegBase = 1, kAuxDone = 63;
    std::vector<std::size_t> seg_counts(W, 0);
    std::vector<char> seg_cover(W, 0);
    std::vector<char> shadow_written(W, 0);
    const std::size_t n_total = grads[0].size();
    // Deferred all-gather of the reduced gradient (SYNK_STEP_GRADS_LOCAL):
    // each rank keeps its own chunk of every segment; readers of `grads`
    // complete the replicas (VarRecord::shard). Segments as rank 0 ran them.
    const bool defer = W > 1 && !st->nccl;
    const int step_flags = defer ? SYNK_STEP_GRADS_LOCAL : 0;
    // Segment updates other than the last overlap the remaining backward
    // GEMMs. SYNK_BG_UPDATES=1 runs them as small grids (SYNK_BG_CTAS): the
    // GEMMs lose less (dX1 + gW0 -45 us) but the update then takes 4-15x
    // longer and the step is slower (1.27-2.1 vs 1.12 ms,
    // profiles/r02_c5_step.md), so full grids are the default.
    static const bool bg_updates = [] {
        const char* e = std::getenv("SYNK_BG_UPDATES");
        return e && e[0] == '1';
    }();
    std::vector<std::pair<std::uint64_t, std::uint64_t>> shard_segs;

    auto tail = [&](std::size_t r, const std::vector<std::size_t>& rows, const std::vector<GradSegment>& segs) {
        const auto& rd = st->ranks[r];
        const int dt = detail::synk_dtype(grads[r].dtype());
        std::size_t total = 0;
        bool unequal = false;
        if (opts_.grad_op == ReduceOp::Mean && W > 1) {
            for (std::size_t x : rows) total += x;
            for (std::size_t x : rows) unequal |= x * W != total;
            unequal = unequal && total > 0;
        }
        std::size_t covered = 0;
        for (const GradSegment& g : segs) covered += g.count;
        seg_counts[r] = segs.size();
        seg_cover[r] = !segs.empty() && covered == n_total;
        if (unequal) {
            // Unequal shards: pre-scale each rank's shard-mean gradient by
            // rows_r*W/total so the equal-weight mean is the global row mean.
            detail::check(synk_scale(rd->h, dt, grads[r].data(), double(rows[r]) * double(W) / double(total),
                                     grads[r].size()),
                          "unequal-shard pre-scale");
        }
        if (st->nccl) {
            // Library baseline backend: NCCL all-reduce (sum, or avg = mean) of
            // this rank's gradient in place, then the rule on the reduced
            // gradient -- NCCL synchronises the ranks on the device. Meet on
            // the host first: a rank that failed before this point aborts the
            // rendezvous instead of stranding its peers inside the collective.
            if (W > 1) rv.arrive_and_wait();
            if (r == 0 && timing) detail::check(synk_mark(rd->h, &ma), "mark");
            if (r == 0 && t0_timer) detail::check(synk_timer_record(rd->h, t0_timer, 4), "timer");
            if (r == 0) update_from_compute_end_ = false;
            detail::check(synk_nccl_all_reduce(rd->h, dt, detail::synk_op(opts_.grad_op), grads[r].data(),
                                               grads[r].size()),
                          "gradient all-reduce (nccl)");
            detail::check(synk_optimizer_step(rd->h, dt, code, hyper.data(), lr_, t_next, pp[r], grads[r].data(),
                                              a0.empty() ? nullptr : a0[r], a1.empty() ? nullptr : a1[r],
                                              grads[r].size()),
                          "update (nccl path)");
            if (r == 0 && timing) detail::check(synk_mark(rd->h, &mb), "mark");
            if (r == 0 && t0_timer) detail::check(synk_timer_record(rd->h, t0_timer, 5), "timer");
            return;
        }
        if (W > 1) {
            detail::check(synk_signal(rd->h), "signal");
            rv.arrive_and_wait();
        }
        // SYNK_STEP_OVERLAP: 1 overlaps the segment updates with the backward
        // GEMMs at every world size, 0 never; unset: only when W > 1 (there is
        // an NVLink transfer to hide). On one GPU the update is pure HBM work
        // that competes with the GEMMs for SM slots.
        static const int overlap_mode = [] {
            const char* e = std::getenv("SYNK_STEP_OVERLAP");
            return e ? std::atoi(e) : -1;
        }();
        bool overlap = !unequal && (overlap_mode == 1 || (overlap_mode == -1 && W > 1));
        for (std::size_t p = 0; p < W; ++p) overlap = overlap && seg_cover[p] && seg_counts[p] == segs.size();
        // bf16 weight shadows (the bf16 MLP's operand copies, one per rank):
        // when every rank holds a current one, the update writes them along
        // with the new params and the next step skips its weight casts. Read
        // after the rendezvous, when every rank has made its own.
        const synk_bf16_shadow* shl = nullptr;
        std::vector<void*> shb(W, nullptr);
        {
            detail::VarRecord& prec = detail::record_of(block_.params);
            bool ok = W <= SYNK_SHADOW_MAX_WORLD && prec.shadows.size() == W && dt == SYNK_F32;
            for (std::size_t p = 0; p < W && ok; ++p) {
                const detail::VarRecord::Bf16Shadow& sh = prec.shadows[p];
                ok = sh.buf[0].has_storage() && sh.buf[1].has_storage() && sh.params == pp[p] &&
                     sh.epoch == prec.epoch.load() && sh.dims == prec.shadows[0].dims;
                shb[p] = ok ? sh.buf[sh.cur ^ 1].data() : nullptr;  // the spare: the kernel reads buf[cur]
            }
            if (ok) shl = &prec.shadows[0].layout;
            shadow_written[r] = ok;
        }
        // The gradient update may have swapped each rank's grads replica for a
        // fresh buffer (WeightedMeanByRows adopts its accumulator): read the
        // pointers only now, after every rank applied its update.
        std::vector<void*> gp(W);
        for (std::size_t p = 0; p < W; ++p) gp[p] = grads[p].data();
        if (!overlap) {
            for (std::size_t p = 0; p < W && W > 1; ++p)
                if (p != r) detail::check(synk_wait_peer(rd->h, st->handles[p]), "wait peer");
            if (r == 0 && timing) detail::check(synk_mark(rd->h, &ma), "mark");
            // W = 1: the update directly follows the compute end (event 3) on this stream
            if (r == 0 && t0_timer && W > 1) detail::check(synk_timer_record(rd->h, t0_timer, 4), "timer");
            if (r == 0) update_from_compute_end_ = W == 1;
            if (r == 0) shard_segs.assign(1, {0, grads[r].size()});
            detail::check(synk_all_reduce_step_ex(rd->h, static_cast<int>(W), dt, detail::synk_op(opts_.grad_op), code,
                                                  hyper.data(), lr_, t_next, pp.data(), gp.data(),
                                                  a0.empty() ? nullptr : a0.data(), a1.empty() ? nullptr : a1.data(),
                                                  grads[r].size(), (coherent ? SYNK_STEP_COHERENT : 0) | step_flags, 0,
                                                  shl, shb.data()),
                          "fused all-reduce + update");
            if (r == 0 && timing) detail::check(synk_mark(rd->h, &mb), "mark");
            if (r == 0 && t0_timer) detail::check(synk_timer_record(rd->h, t0_timer, 5), "timer");
            return;
        }
        synk_dev* aux = rd->aux_handle();
        if (r == 0 && timing) {
            detail::check(synk_mark_reset(aux), "marks");
            aux_marks = true;
        }
        const std::size_t es = dtype_size(grads[r].dtype());
        auto at = [es](const std::vector<void*>& v, std::size_t first) {
            std::vector<void*> o(v.size());
            for (std::size_t i = 0; i < v.size(); ++i) o[i] = v[i] ? static_cast<char*>(v[i]) + first * es : nullptr;
            return o;
        };
        for (std::size_t k = 0; k < segs.size(); ++k) {
            const GradSegment& g = segs[k];
            for (std::size_t p = 0; p < W; ++p)  // every rank (this one included) finished this segment
                detail::check(synk_wait_peer_slot(aux, st->handles[p], g.slot), "wait segment");
            if (r == 0 && timing && k == 0) detail::check(synk_mark(aux, &ma), "mark");
            if (r == 0 && t0_timer && k == 0) detail::check(synk_timer_record(aux, t0_timer, 4), "timer");
            if (r == 0 && k == 0) update_from_compute_end_ = false;
            std::vector<void*> ps = at(pp, g.first), gs = at(gp, g.first), x0 = at(a0, g.first), x1 = at(a1, g.first);
            if (r == 0) shard_segs.emplace_back(g.first, g.count);
            detail::check(synk_all_reduce_step_ex(aux, static_cast<int>(W), dt, detail::synk_op(opts_.grad_op), code,
                                                  hyper.data(), lr_, t_next, ps.data(), gs.data(),
                                                  a0.empty() ? nullptr : x0.data(), a1.empty() ? nullptr : x1.data(),
                                                  g.count,
                                                  (coherent ? SYNK_STEP_COHERENT : 0) | step_flags |
                                                      (k + 1 < segs.size() && bg_updates ? SYNK_STEP_BACKGROUND : 0),
                                                  g.first,
                                                  shl, shb.data()),
                          "segment all-reduce + update");
        }
        if (r == 0 && timing) detail::check(synk_mark(aux, &mb), "mark");
        if (r == 0 && t0_timer) detail::check(synk_timer_record(aux, t0_timer, 5), "timer");
        // Join: the rank's own stream (whose synchronisation ends the phase)
        // waits for the overlapped updates.
        detail::check(synk_signal_slot(aux, kAuxDone), "signal aux");
        detail::check(synk_wait_peer_slot(rd->h, aux, kAuxDone), "join aux");
    };
    CallOptions co = call_opts;
    co.device_timing = timing;
    CallResult gr = detail::call_with_tail(f_grad, batch, co, tail, &rv, kSegBase,
                                           lazy ? &timers_->per_rank : nullptr);
    if (gr.outputs.empty()) throw ArgumentError("train_step(): gradient function must output the loss");
    const double loss = gr.outputs[0].get(0);
    rep.grad_call = gr.report;
    if (ma >= 0 && mb >= 0) {
        double sec = 0.0;
        detail::check(synk_mark_elapsed(aux_marks ? st->ranks[0]->aux : st->ranks[0]->h, ma, mb, &sec), "timing");
        rep.allreduce_s = sec;
        rep.step_call.total_s = sec;
    }
    rep.step_call.rank_rows.assign(W, 1);
    detail::VarRecord& grec = detail::record_of(block_.grads);
    grec.coherent = true;  // logically: every reader completes the replicas first
    grec.mutated();
    if (defer && !shard_segs.empty()) grec.shard = detail::VarRecord::Shard{grads, shard_segs};
    detail::VarRecord& prec = detail::record_of(block_.params);
    prec.coherent = true;
    prec.mutated();
    bool all_shadows = true;
    for (std::size_t r = 0; r < W; ++r) all_shadows = all_shadows && shadow_written[r];
    if (all_shadows)  // the update wrote every rank's spare shadow with the new params
        for (auto& sh : prec.shadows) {
            sh.cur ^= 1;
            sh.epoch = prec.epoch.load();
        }
    for (const ReplicatedVariable& a : aux_) {
        detail::record_of(a).coherent = true;
        detail::record_of(a).mutated();
    }
    t_ += 1;
    if (opts_.verify_coherence && !block_.params.replicas_coherent())
        throw CoherenceError("train_step(): parameter replicas diverged after step " + std::to_string(t_));
    rep.loss = loss;
    rep.total_s = since(t0);
    last_ = rep;
    report_pending_ = lazy;
    return loss;
}


double SyncSgd::train_step(const ParallelFunction& f_grad, const std::vector<FunctionArg>& batch,
                           const CallOptions& call_opts) {
    detail::NvtxRange range("synk.train_step");
    const auto t0 = Clock::now();
    StepReport rep;
    auto st = detail::state_of(*pool_);
    const std::size_t W = st->world;

    const auto combine = f_grad.update_combine_for(block_.grads.id());
    if (!combine) throw ArgumentError("train_step(): gradient function does not update the gradient block");
    auto& grads = detail::replicas_of(block_.grads);
    if (*combine == UpdateCombine::Add) {
        // Accumulating gradient functions start from zero every step.
        for (std::size_t r = 0; r < W; ++r) block_.grads.set_value(r, NdBuffer::zeros({block_.length}, block_.grads.dtype()));
    }

    if (opts_.all_reduce && !opts_.check_finite && opts_.grad_op != ReduceOp::Gather)
        return fused_step(f_grad, batch, call_opts, t0);

    CallResult gr = f_grad.call(batch, call_opts);
    if (gr.outputs.empty()) throw ArgumentError("train_step(): gradient function must output the loss");
    const double loss = gr.outputs[0].get(0);
    rep.grad_call = gr.report;

    if (opts_.check_finite) {
        for (std::size_t r = 0; r < W; ++r) {
            int ok = 1;
            detail::check(synk_all_finite(grads[r].owner()->h, detail::synk_dtype(grads[r].dtype()), grads[r].data(),
                                          grads[r].size(), &ok),
                          "check_finite");
            if (!ok) throw NumericError("train_step(): non-finite gradient elements on rank " + std::to_string(r));
        }
    }

    if (opts_.all_reduce) {
        if (opts_.grad_op == ReduceOp::Gather) throw ArgumentError("all_reduce: Gather is not a reduction (use gather())");
        for (std::size_t r = 1; r < W; ++r)
            if (!grads[r].same_shape(grads[0]))
                throw ShapeError("all_reduce: replica shapes differ across ranks (" + grads[0].shape_string() + " vs rank " +
                                 std::to_string(r) + " " + grads[r].shape_string() + ")");
        // Unequal shards: pre-scale each rank's shard-mean gradient by
        // rows_r*W/total so the equal-weight mean is the global row mean.
        std::vector<double> factor(W, 1.0);
        bool unequal = false;
        if (opts_.grad_op == ReduceOp::Mean) {
            const auto& rows = gr.report.rank_rows;
            std::size_t total = 0;
            for (std::size_t x : rows) total += x;
            for (std::size_t r = 0; r < rows.size(); ++r) unequal |= rows[r] * W != total;
            if (unequal && total > 0)
                for (std::size_t r = 0; r < W; ++r) factor[r] = double(rows[r]) * double(W) / double(total);
            unequal = unequal && total > 0;
        }
        auto& params = detail::replicas_of(block_.params);
        std::vector<void*> pp, gp, a0, a1;
        for (std::size_t r = 0; r < W; ++r) {
            pp.push_back(params[r].data());
            gp.push_back(grads[r].data());
            if (aux_.size() > 0) a0.push_back(detail::replicas_of(aux_[0])[r].data());
            if (aux_.size() > 1) a1.push_back(detail::replicas_of(aux_[1])[r].data());
        }
        bool coherent = detail::record_of(block_.params).coherent;
        for (const ReplicatedVariable& a : aux_) coherent = coherent && detail::record_of(a).coherent;
        const std::vector<double> hyper = rule_hyper(rule_);
        const int code = rule_code(rule_);
        const std::uint64_t t_next = t_ + 1;
        const auto ta = Clock::now();
        if (unequal) {
            // Rank-local pre-scale (sgd.cpp:292-312 semantics, T(f64 g * factor)).
            // It must complete on every rank before any rank reads peers, hence
            // its own phase.
            detail::run_pool_phase(*st, PhaseKind::Collective, [&](std::size_t r) {
                const auto& rd = st->ranks[r];
                detail::check(synk_scale(rd->h, detail::synk_dtype(grads[r].dtype()), grads[r].data(), factor[r],
                                         grads[r].size()),
                              "unequal-shard pre-scale");
                detail::dev_sync(rd);
            });
        }
        PhaseReport ph2 = detail::run_pool_phase(*st, PhaseKind::Collective, [&](std::size_t r) {
            const auto& rd = st->ranks[r];
            if (params[r].dtype() != grads[r].dtype()) throw DTypeError("step: params/grads dtype mismatch");
            if (params[r].size() != grads[r].size()) throw ShapeError("step: params length != grads length");
            detail::check(synk_all_reduce_step(rd->h, static_cast<int>(W), detail::synk_dtype(grads[r].dtype()),
                                               detail::synk_op(opts_.grad_op), code, hyper.data(), lr_, t_next, pp.data(),
                                               gp.data(), a0.empty() ? nullptr : a0.data(),
                                               a1.empty() ? nullptr : a1.data(), grads[r].size(), coherent ? 1 : 0),
                          "fused all-reduce + update");
            detail::dev_sync(rd);
        });
        detail::record_of(block_.params).mutated();
        for (const ReplicatedVariable& a : aux_) detail::record_of(a).mutated();
        rep.allreduce_s = since(ta);
        rep.step_call.rank_compute_s = ph2.rank_seconds;
        rep.step_call.rank_rows.assign(W, 1);
        rep.step_call.straggler_s = ph2.straggler_seconds();
        rep.step_call.total_s = ph2.max_seconds();
        detail::record_of(block_.grads).coherent = true;
        detail::record_of(block_.params).coherent = true;
        for (const ReplicatedVariable& a : aux_) detail::record_of(a).coherent = true;
    } else {
        *step_box_ = t_;  // the step kernel applies step t_ + 1 (sgd.cpp:231,237 of the reference)
        CallResult sr = f_step_.call({FunctionArg(NdBuffer::scalar(double(t_ + 1)))});
        rep.step_call = sr.report;
    }
    t_ += 1;

    if (opts_.verify_coherence && !block_.params.replicas_coherent())
        throw CoherenceError("train_step(): parameter replicas diverged after step " + std::to_string(t_));
    rep.loss = loss;
    rep.total_s = since(t0);
    last_ = rep;
    report_pending_ = false;
    return loss;
}

} // namespace synkpar
