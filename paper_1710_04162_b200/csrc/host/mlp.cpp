// The example MLP workload (mlp.hpp): seeded init and dataset on the host
// (identical libstdc++ draws to the reference, so identical bytes), loss and
// gradient on the GPU through synk_mlp_loss_grad.

#include "synkpar/mlp.hpp"

#include <cmath>
#include <cstdlib>
#include <random>

#include "internal.hpp"

namespace synkpar {

namespace {

void validate(const MlpConfig& c) {
    if (c.layers == 0) throw ArgumentError("mlp: layers must be >= 1");
    if (c.in_dim == 0 || c.out_dim == 0 || (c.layers > 1 && c.width == 0))
        throw ArgumentError("mlp: dimensions must be positive");
}

// Layer widths d[0..L] from the (weight, bias) segment pairs (mlp.cpp:84-110 rules).
std::vector<std::uint64_t> layer_dims(const std::vector<FlatSegment>& segs) {
    if (segs.empty() || segs.size() % 2)
        throw ArgumentError("mlp_loss_grad: segments must alternate weight/bias pairs");
    const std::size_t L = segs.size() / 2;
    std::vector<std::uint64_t> d(L + 1);
    for (std::size_t l = 0; l < L; ++l) {
        const auto& w = segs[2 * l].shape;
        const auto& b = segs[2 * l + 1].shape;
        if (w.size() != 2 || b.size() != 1 || b[0] != w[1])
            throw ArgumentError("mlp_loss_grad: segment " + std::to_string(2 * l) + " is not a (weight, bias) pair");
        if (l == 0) d[0] = w[0];
        else if (w[0] != d[l]) throw ShapeError("mlp_loss_grad: layer " + std::to_string(l) + " input dim does not chain");
        d[l + 1] = w[1];
    }
    return d;
}

struct Checked {
    std::vector<std::uint64_t> dims;
    std::size_t n = 0;
};

template <class Buf>
Checked check_operands(const Buf& params, const std::vector<FlatSegment>& segs, const Buf& x, const Buf& y) {
    if (params.rank() != 1) throw ShapeError("mlp_loss_grad: flat_params must be rank 1");
    if (x.rank() != 2 || y.rank() != 2) throw ShapeError("mlp_loss_grad: x and y must be rank 2");
    if (x.shape()[0] != y.shape()[0])
        throw ShapeError("mlp_loss_grad: x rows " + std::to_string(x.shape()[0]) + " != y rows " +
                         std::to_string(y.shape()[0]));
    Checked c;
    c.dims = layer_dims(segs);
    std::size_t expected = 0;
    for (const FlatSegment& s : segs) expected += element_count(s.shape);
    if (params.size() != expected) throw ShapeError("mlp_loss_grad: flat_params length does not match segments");
    if (x.shape()[1] != c.dims.front()) throw ShapeError("mlp_loss_grad: x columns != input dim");
    if (y.shape()[1] != c.dims.back()) throw ShapeError("mlp_loss_grad: y columns != output dim");
    c.n = x.shape()[0];
    if (c.n == 0) throw ArgumentError("mlp_loss_grad: empty batch");
    return c;
}

// x/y in the parameter dtype on the device (the reference widens everything
// to f64, so mixed dtypes are legal; we narrow/widen on the GPU).
DevBuffer as_dtype(const std::shared_ptr<detail::RankDevice>& rd, const DevBuffer& b, DType dt) {
    if (b.dtype() == dt) return b;
    DevBuffer out = DevBuffer::alloc(rd, b.shape(), dt);
    detail::check(synk_cast(rd->h, detail::synk_dtype(dt), out.data(), detail::synk_dtype(b.dtype()), b.data(), b.size()),
                  "mlp: cast inputs");
    return out;
}

// The rank's bf16 weight shadow of `pvar` for these dims (synk_cuda.h):
// (re)allocated when missing or of another shape; *valid = it still equals
// bf16(params) (made at the variable's current epoch from this storage).
void* weight_shadow(const ReplicatedVariable& pvar, const std::shared_ptr<detail::RankDevice>& rd,
                    const DevBuffer& params, const std::vector<std::uint64_t>& dims, int* valid) {
    detail::VarRecord& rec = detail::record_of(pvar);
    const std::size_t r = rd->rank;
    *valid = 0;
    if (const char* e = std::getenv("SYNK_MLP_SHADOW"); e && e[0] == '0') return nullptr;  // A/B and tests
    if (r >= rec.shadows.size() || r >= rec.replicas.size() || rec.replicas[r].data() != params.data()) return nullptr;
    detail::VarRecord::Bf16Shadow& sh = rec.shadows[r];
    if (sh.dims != dims || !sh.buf[0].has_storage() || sh.buf[0].owner().get() != rd.get()) {
        synk_bf16_shadow layout{};
        if (synk_mlp_bf16_shadow(dims.data(), static_cast<std::uint32_t>(dims.size() - 1), &layout) != SYNK_OK)
            return nullptr;  // more layers than the shadow supports: the casts go to the workspace
        for (DevBuffer& b : sh.buf)
            b = DevBuffer::alloc(rd, {(layout.bytes + 7) / 8}, DType::Float64);  // bytes; dtype is bookkeeping
        sh.cur = 0;
        sh.layout = layout;
        sh.dims = dims;
        sh.epoch = ~std::uint64_t(0);
    }
    *valid = sh.epoch == rec.epoch.load() && sh.params == params.data();
    return sh.buf[sh.cur].data();
}

void mark_shadow_current(const ReplicatedVariable& pvar, std::size_t rank, const DevBuffer& params) {
    detail::VarRecord& rec = detail::record_of(pvar);
    detail::VarRecord::Bf16Shadow& sh = rec.shadows[rank];
    sh.epoch = rec.epoch.load();
    sh.params = params.data();
}

// Enqueue loss + gradient on rd's stream. Returns (loss f64 scalar, grad).
std::pair<DevBuffer, DevBuffer> device_loss_grad(const std::shared_ptr<detail::RankDevice>& rd, const Checked& c,
                                                 const DevBuffer& params, const DevBuffer& x, const DevBuffer& y,
                                                 MlpCompute compute = MlpCompute::Native,
                                                 const KernelContext* ctx = nullptr,
                                                 const KernelContext::IndexedInput* rows = nullptr,
                                                 const ReplicatedVariable* pvar = nullptr) {
    const DType dt = params.dtype();
    if (compute == MlpCompute::Bf16TensorCore && dt != DType::Float32)
        throw DTypeError("mlp_grad_kernel: bf16 tensor-core compute needs float32 parameters");
    const int mode = compute == MlpCompute::Native ? SYNK_MLP_NATIVE : SYNK_MLP_BF16_TC;
    DevBuffer xd = as_dtype(rd, x, dt), yd = as_dtype(rd, y, dt);
    const std::uint32_t L = static_cast<std::uint32_t>(c.dims.size() - 1);
    std::uint64_t ws_bytes = 0;
    detail::check(synk_mlp_workspace_bytes_ex(detail::synk_dtype(dt), mode, c.dims.data(), L, c.n, &ws_bytes),
                  "mlp workspace");
    void* ws = detail::rank_scratch(rd, ws_bytes);
    // the loss may land straight in the rank's pinned staging (single
    // contributor: KernelContext::host_staging), read by the host after the phase
    DevBuffer loss = ctx && ctx->rank_device == rd ? ctx->device_alloc({}, DType::Float64)
                                                   : DevBuffer::alloc(rd, {}, DType::Float64);
    DevBuffer grad = DevBuffer::alloc(rd, {params.size()}, dt);
    synk_mlp_opts opts{};
    opts.signal_base = ctx && ctx->grad_segments ? ctx->grad_signal_base : -1;
    const int base = opts.signal_base;
    if (rows) {
        opts.rows = rows->rows;
        opts.rows_host = rows->host_rows;
        opts.rows_ready_on = rows->ready_on;
        opts.rows_ready_slot = rows->ready_slot;
    }
    const bool shadowed = pvar && compute == MlpCompute::Bf16TensorCore;
    if (shadowed) opts.shadow = weight_shadow(*pvar, rd, params, c.dims, &opts.shadow_valid);
    opts.shadow_spare = opts.shadow != nullptr;  // a trainer update writes buf[cur ^ 1]
    std::vector<int> seg_order(L);
    for (std::uint32_t i = 0; i < L; ++i) seg_order[i] = static_cast<int>(L - 1 - i);  // backward order by default
    opts.seg_order = seg_order.data();
    int signalled = 0;
    detail::check(synk_mlp_loss_grad_opts(rd->h, detail::synk_dtype(dt), mode, c.dims.data(), L, params.data(),
                                          xd.data(), yd.data(), c.n, static_cast<double*>(loss.data()), grad.data(), ws,
                                          ws_bytes, &opts, &signalled),
                  "mlp_loss_grad");
    if (opts.shadow) mark_shadow_current(*pvar, rd->rank, params);
    if (signalled > 0) {
        // Layer l's segment [W_l, b_l] was signalled on slot base + l, in the
        // order the kernel reports (seg_order); W_l and b_l are adjacent in the layout.
        std::size_t at = 0;
        std::vector<std::size_t> first(L), count(L);
        for (std::uint32_t l = 0; l < L; ++l) {
            first[l] = at;
            count[l] = c.dims[l] * c.dims[l + 1] + c.dims[l + 1];
            at += count[l];
        }
        for (std::uint32_t i = 0; i < L; ++i) {
            const std::uint32_t l = static_cast<std::uint32_t>(seg_order[i]);
            ctx->grad_segments->push_back({first[l], count[l], base + int(l)});
        }
    }
    return {loss, grad};
}

} // namespace

std::vector<std::vector<std::size_t>> mlp_param_shapes(const MlpConfig& c) {
    validate(c);
    std::vector<std::vector<std::size_t>> shapes;
    for (std::size_t l = 0; l < c.layers; ++l) {
        const std::size_t fan_in = l == 0 ? c.in_dim : c.width;
        const std::size_t fan_out = l + 1 == c.layers ? c.out_dim : c.width;
        shapes.push_back({fan_in, fan_out});
        shapes.push_back({fan_out});
    }
    return shapes;
}

std::vector<NdBuffer> mlp_init_params(const MlpConfig& c, DType dtype) {
    const auto shapes = mlp_param_shapes(c);
    std::mt19937_64 gen(c.seed);
    std::vector<NdBuffer> out;
    for (std::size_t i = 0; i < shapes.size(); i += 2) {
        std::normal_distribution<double> normal(0.0, 1.0 / std::sqrt(double(shapes[i][0])));
        NdBuffer w = NdBuffer::zeros(shapes[i], dtype);
        for (std::size_t j = 0; j < w.size(); ++j) w.set(j, normal(gen));
        out.push_back(std::move(w));
        out.push_back(NdBuffer::zeros(shapes[i + 1], dtype));
    }
    return out;
}

Dataset mlp_make_dataset(std::size_t rows, const MlpConfig& c, std::uint64_t seed, DType dtype) {
    validate(c);
    std::mt19937_64 gen(seed ^ 0x9e3779b97f4a7c15ull);
    std::normal_distribution<double> normal(0.0, 1.0);
    const double scale = 1.0 / std::sqrt(double(c.in_dim));
    std::vector<double> teacher(c.in_dim * c.out_dim);
    for (double& t : teacher) t = normal(gen) * scale;
    Dataset ds{NdBuffer::zeros({rows, c.in_dim}, dtype), NdBuffer::zeros({rows, c.out_dim}, dtype)};
    std::vector<double> xr(c.in_dim);
    for (std::size_t i = 0; i < rows; ++i) {
        for (std::size_t j = 0; j < c.in_dim; ++j) {
            xr[j] = normal(gen);
            ds.x.set(i * c.in_dim + j, xr[j]);
        }
        for (std::size_t k = 0; k < c.out_dim; ++k) {
            double acc = 0.0;
            for (std::size_t j = 0; j < c.in_dim; ++j) acc += xr[j] * teacher[j * c.out_dim + k];
            ds.y.set(i * c.out_dim + k, acc);
        }
    }
    return ds;
}

LossGrad mlp_loss_grad(const NdBuffer& params, const std::vector<FlatSegment>& segs, const NdBuffer& x, const NdBuffer& y) {
    Checked c = check_operands(params, segs, x, y);
    auto rd = detail::utility_device();
    DevBuffer p = detail::dev_from_host(rd, params);
    DevBuffer xd = detail::dev_from_host(rd, x);
    DevBuffer yd = detail::dev_from_host(rd, y);
    auto [loss, grad] = device_loss_grad(rd, c, p, xd, yd);
    LossGrad out;
    out.grad = detail::dev_to_host(grad);
    out.loss = detail::dev_to_host(loss).get(0);
    return out;
}

Kernel mlp_grad_kernel(const FlatParamBlock& block, std::string name, MlpCompute compute) {
    Kernel k;
    k.name = std::move(name);
    k.arity = 2;
    k.reads = {block.params};
    const std::vector<FlatSegment> segs = block.segments;
    const std::uint64_t grads_id = block.grads.id();
    // Index-fused inputs: with x and y selected by the call's index list over
    // HBM mirrors, the loss reads y through the list and x is staged from the
    // whole source inside the kernel's own launch sequence -- the bf16 staging
    // of x reads the batch rows straight from the source (the f32 batch is
    // never gathered); the native path gathers x as the first node of its CUDA
    // graph (one graph launch per step instead of two gathers + the graph).
    k.fused_index_inputs = true;
    // The reference's host-kernel contract as well (mlp.cpp:249-265): user code
    // may wrap `kernel.fn` (e.g. to re-emit the gradient as an Add update).
    // It computes on the calling rank's GPU from host buffers.
    k.fn = [segs, grads_id, compute](const std::vector<NdBuffer>& in, const KernelContext& ctx) {
        auto rd = ctx.rank_device ? ctx.rank_device : detail::utility_device();
        const NdBuffer& params_h = ctx.replica(0);
        Checked c = check_operands(params_h, segs, in[0], in[1]);
        DevBuffer p = detail::dev_from_host(rd, params_h);
        DevBuffer xd = detail::dev_from_host(rd, in[0]);
        DevBuffer yd = detail::dev_from_host(rd, in[1]);
        auto [loss, grad] = device_loss_grad(rd, c, p, xd, yd, compute);
        KernelResult r;
        r.outputs.push_back(NdBuffer::scalar(detail::dev_to_host(loss).get(0)));
        r.updates.push_back(UpdateDelta{grads_id, detail::dev_to_host(grad), UpdateCombine::WeightedMeanByRows});
        return r;
    };
    const ReplicatedVariable pvar = block.params;
    k.device_fn = [segs, grads_id, compute, pvar](const std::vector<DevBuffer>& in, const KernelContext& ctx) {
        const DevBuffer& params = ctx.device_replica(0);
        const KernelContext::IndexedInput* ix = ctx.indexed ? &(*ctx.indexed)[0] : nullptr;
        const KernelContext::IndexedInput* iy = ctx.indexed ? &(*ctx.indexed)[1] : nullptr;
        if (ix && iy && (ix->rows || iy->rows)) {
            const auto& rd = ctx.rank_device;
            Checked c = check_operands(params, segs, in[0], in[1]);  // whole sources: same leading extent
            const bool direct = ix->rows && ix->rows == iy->rows && ix->count == iy->count &&
                                in[0].dtype() == params.dtype() && in[1].dtype() == params.dtype() &&
                                (compute == MlpCompute::Native || params.dtype() == DType::Float32);
            if (direct) {
                c.n = ix->count;
                auto [loss, grad] = device_loss_grad(rd, c, params, in[0], in[1], compute, &ctx, ix, &pvar);
                DeviceKernelResult r;
                r.outputs.push_back(loss);
                r.updates.push_back({grads_id, grad, UpdateCombine::WeightedMeanByRows});
                return r;
            }
            // Gather the selected rows here, then the regular path.
            auto gathered = [&](const DevBuffer& src, const KernelContext::IndexedInput& sel) {
                if (!sel.rows) return src;
                if (sel.ready_on)
                    detail::check(synk_wait_peer_slot(rd->h, sel.ready_on, sel.ready_slot), "mlp: index stage wait");
                std::vector<std::size_t> shape = src.shape();
                shape[0] = sel.count;
                DevBuffer out = DevBuffer::alloc(rd, std::move(shape), src.dtype());
                detail::check(synk_gather_rows(rd->h, src.data(), src.rows(), src.row_size() * dtype_size(src.dtype()),
                                               sel.rows, sel.count, out.data()),
                              "mlp: gather fused input");
                return out;
            };
            const DevBuffer xg = gathered(in[0], *ix), yg = gathered(in[1], *iy);
            Checked cg = check_operands(params, segs, xg, yg);
            auto [loss, grad] = device_loss_grad(rd, cg, params, xg, yg, compute, &ctx, nullptr, &pvar);
            DeviceKernelResult r;
            r.outputs.push_back(loss);
            r.updates.push_back({grads_id, grad, UpdateCombine::WeightedMeanByRows});
            return r;
        }
        Checked c = check_operands(params, segs, in[0], in[1]);
        auto [loss, grad] = device_loss_grad(ctx.rank_device, c, params, in[0], in[1], compute, &ctx, nullptr, &pvar);
        DeviceKernelResult r;
        r.outputs.push_back(loss);
        r.updates.push_back({grads_id, grad, UpdateCombine::WeightedMeanByRows});
        return r;
    };
    return k;
}

std::vector<UpdateSpec> mlp_grad_updates(const FlatParamBlock& block) {
    return {UpdateSpec{block.grads, UpdateCombine::WeightedMeanByRows}};
}

} // namespace synkpar
