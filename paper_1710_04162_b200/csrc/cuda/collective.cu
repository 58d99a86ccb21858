// Shared-variable collectives over peer memory, in the reference's fixed
// binomial-tree order (tree_fold, replicated.cpp:16-29), plus the fused
// gradient all-reduce + optimizer update of SyncSgd::train_step
// (sgd.cpp:313-319).
//
// Design: all ranks live in one process (the paper's master + workers, here
// one host thread per GPU), so every replica is addressable from every GPU
// (NVLink peer mappings; several ranks on one GPU just share it). Rank r owns
// chunk r of the element range. Its kernel loads chunk r of all W replicas
// (W x 16-byte vector loads in flight per thread), folds them per element in
// exactly tree_fold's order (pairs (q, q+2^k)), and stores the result into
// chunk r of every replica. Because the element-wise fold is the same
// sequence of T operations as the reference, the result is BITWISE equal to
// ReplicatedVariable::all_reduce for every op including sum/mean, and replica
// coherence follows by construction. Per-GPU NVLink traffic is
// 2(W-1)/W x bytes, the same as a ring all-reduce, in a single kernel with no
// intermediate synchronisation (chunks are disjoint, so ranks never race).

#include <math.h>

#include "common.cuh"
#include "optim_math.cuh"

namespace {

using synk::combine_op;

constexpr int kMaxWorld = 64;
constexpr int kBlock = 256;

struct Ptrs {
    void* p[kMaxWorld];
};

template <class T>
struct V16;
template <>
struct V16<float> {
    using V = float4;
    static constexpr int N = 4;
};
template <>
struct V16<double> {
    using V = double2;
    static constexpr int N = 2;
};

// Per-element binomial fold of W values held in registers (replicated.cpp:22-26).
template <class T, int W>
__device__ __forceinline__ T tree_fold_regs(int op, T (&v)[W]) {
#pragma unroll
    for (int step = 1; step < W; step *= 2)
#pragma unroll
        for (int q = 0; q + step < W; q += 2 * step) v[q] = combine_op(op, v[q], v[q + step]);
    return v[0];
}

template <class T>
__device__ __forceinline__ T tree_fold_dyn(int op, T* v, int w) {
    for (int step = 1; step < w; step *= 2)
        for (int q = 0; q + step < w; q += 2 * step) v[q] = combine_op(op, v[q], v[q + step]);
    return v[0];
}

template <class T>
__device__ __forceinline__ T finish_mean(int op, T v, double inv_w) {
    return op == SYNK_OP_MEAN ? (T)__dmul_rn((double)v, inv_w) : v;
}

// ---- all-reduce chunk kernel (compile-time world size) ------------------------
template <class T, int W>
__global__ void __launch_bounds__(kBlock) allreduce_chunk_kernel(Ptrs bufs, int op, double inv_w,
                                                                 uint64_t lo, uint64_t hi,
                                                                 bool vec) {
    using V = typename V16<T>::V;
    constexpr int N = V16<T>::N;
    const int fop = op == SYNK_OP_MEAN ? SYNK_OP_SUM : op;
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * kBlock;
    uint64_t head = lo;
    if (vec) {
        uint64_t v0 = lo / N, v1 = hi / N;  // lo is a multiple of N when vec
        for (uint64_t i = v0 + tid; i < v1; i += stride) {
            V x[W];
#pragma unroll
            for (int q = 0; q < W; ++q) x[q] = static_cast<const V*>(bufs.p[q])[i];
            V out;
#pragma unroll
            for (int k = 0; k < N; ++k) {
                T e[W];
#pragma unroll
                for (int q = 0; q < W; ++q) e[q] = reinterpret_cast<const T*>(&x[q])[k];
                reinterpret_cast<T*>(&out)[k] = finish_mean(op, tree_fold_regs<T, W>(fop, e), inv_w);
            }
#pragma unroll
            for (int q = 0; q < W; ++q) static_cast<V*>(bufs.p[q])[i] = out;
        }
        head = v1 * N;
    }
    for (uint64_t i = head + tid; i < hi; i += stride) {
        T e[W];
#pragma unroll
        for (int q = 0; q < W; ++q) e[q] = static_cast<const T*>(bufs.p[q])[i];
        T out = finish_mean(op, tree_fold_regs<T, W>(fop, e), inv_w);
#pragma unroll
        for (int q = 0; q < W; ++q) static_cast<T*>(bufs.p[q])[i] = out;
    }
}

// Generic world size (> 8): values staged in local memory.
template <class T>
__global__ void __launch_bounds__(kBlock) allreduce_chunk_dyn_kernel(Ptrs bufs, int w, int op,
                                                                     double inv_w, uint64_t lo,
                                                                     uint64_t hi) {
    const int fop = op == SYNK_OP_MEAN ? SYNK_OP_SUM : op;
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    T e[kMaxWorld];
    for (uint64_t i = lo + tid; i < hi; i += (uint64_t)gridDim.x * kBlock) {
        for (int q = 0; q < w; ++q) e[q] = static_cast<const T*>(bufs.p[q])[i];
        T out = finish_mean(op, tree_fold_dyn(fop, e, w), inv_w);
        for (int q = 0; q < w; ++q) static_cast<T*>(bufs.p[q])[i] = out;
    }
}

// Fold all replicas into out (one rank, whole range).
template <class T>
__global__ void __launch_bounds__(kBlock) tree_reduce_kernel(Ptrs bufs, int w, int op, double inv_w,
                                                             uint64_t n, T* __restrict__ out) {
    const int fop = op == SYNK_OP_MEAN ? SYNK_OP_SUM : op;
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    T e[kMaxWorld];
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) {
        for (int q = 0; q < w; ++q) e[q] = static_cast<const T*>(bufs.p[q])[i];
        out[i] = finish_mean(op, tree_fold_dyn(fop, e, w), inv_w);
    }
}

// Broadcast chunk: copy [lo,hi) bytes of bufs[src] into every other replica.
__global__ void __launch_bounds__(kBlock) bcast_chunk_kernel(Ptrs bufs, int w, int src, uint64_t lo,
                                                             uint64_t hi, bool vec) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * kBlock;
    if (vec) {
        const uint4* s = static_cast<const uint4*>(bufs.p[src]);
        for (uint64_t i = lo / 16 + tid; i < hi / 16; i += stride) {
            uint4 x = s[i];
            for (int q = 0; q < w; ++q)
                if (q != src) static_cast<uint4*>(bufs.p[q])[i] = x;
        }
        return;
    }
    const uint8_t* s = static_cast<const uint8_t*>(bufs.p[src]);
    for (uint64_t i = lo + tid; i < hi; i += stride) {
        uint8_t x = s[i];
        for (int q = 0; q < w; ++q)
            if (q != src) static_cast<uint8_t*>(bufs.p[q])[i] = x;
    }
}

// ---- fused gradient all-reduce + optimizer update ------------------------------
// Vector body: one 16-byte vector (4 f32 / 2 f64 elements) of chunk r per
// iteration: W peer loads of the gradient, per-lane tree fold + 1/W, then the
// update on this rank's (coherent) params/aux and W peer stores of each.
// With W == 1 the fold is the identity (and x*1.0 is exact), so the gradient
// is not rewritten.
template <class T, int W>
__device__ __forceinline__ void step_vector(const Ptrs& params, const Ptrs& grads, const Ptrs& aux0, const Ptrs& aux1,
                                            int rank, int grad_op, int fop, double inv_w, const synk::RuleParams& rp,
                                            int naux, uint64_t v) {
    using V = typename V16<T>::V;
    constexpr int N = V16<T>::N;
    V gx[W];
#pragma unroll
    for (int q = 0; q < W; ++q) gx[q] = static_cast<const V*>(grads.p[q])[v];
    V g;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        T e[W];
#pragma unroll
        for (int q = 0; q < W; ++q) e[q] = reinterpret_cast<const T*>(&gx[q])[k];
        reinterpret_cast<T*>(&g)[k] = finish_mean(grad_op, tree_fold_regs<T, W>(fop, e), inv_w);
    }
    if constexpr (W > 1) {
#pragma unroll
        for (int q = 0; q < W; ++q) static_cast<V*>(grads.p[q])[v] = g;
    }
    V p = static_cast<const V*>(params.p[rank])[v];
    V a0 = naux > 0 ? static_cast<const V*>(aux0.p[rank])[v] : p;
    V a1 = naux > 1 ? static_cast<const V*>(aux1.p[rank])[v] : p;
#pragma unroll
    for (int k = 0; k < N; ++k) {
        double pd = (double)reinterpret_cast<T*>(&p)[k];
        double x0 = (double)reinterpret_cast<T*>(&a0)[k];
        double x1 = (double)reinterpret_cast<T*>(&a1)[k];
        synk::rule_update(rp, pd, x0, x1, (double)reinterpret_cast<T*>(&g)[k]);
        reinterpret_cast<T*>(&p)[k] = (T)pd;
        reinterpret_cast<T*>(&a0)[k] = (T)x0;
        reinterpret_cast<T*>(&a1)[k] = (T)x1;
    }
#pragma unroll
    for (int q = 0; q < W; ++q) {
        static_cast<V*>(params.p[q])[v] = p;
        if (naux > 0) static_cast<V*>(aux0.p[q])[v] = a0;
        if (naux > 1) static_cast<V*>(aux1.p[q])[v] = a1;
    }
}

template <class T, int W>
__global__ void __launch_bounds__(kBlock) allreduce_step_kernel(
    Ptrs params, Ptrs grads, Ptrs aux0, Ptrs aux1, int world, int rank, int grad_op,
    double inv_w, synk::RuleParams rp, int naux, bool coherent, uint64_t lo, uint64_t hi, bool vec) {
    const int fop = grad_op == SYNK_OP_MEAN ? SYNK_OP_SUM : grad_op;
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * kBlock;
    if constexpr (W > 0) {
        if (vec && coherent) {
            constexpr int N = V16<T>::N;
            const uint64_t v0 = lo / N, v1 = hi / N;  // lo is 16-element aligned
            for (uint64_t v = v0 + tid; v < v1; v += stride)
                step_vector<T, W>(params, grads, aux0, aux1, rank, grad_op, fop, inv_w, rp, naux, v);
            lo = v1 * N;  // scalar tail below
        }
    }
    for (uint64_t i = lo + tid; i < hi; i += stride) {
        T e[W > 0 ? W : kMaxWorld];
        T g;
        if constexpr (W > 0) {
#pragma unroll
            for (int q = 0; q < W; ++q) e[q] = static_cast<const T*>(grads.p[q])[i];
            g = finish_mean(grad_op, tree_fold_regs<T, W>(fop, e), inv_w);
#pragma unroll
            for (int q = 0; q < W; ++q) static_cast<T*>(grads.p[q])[i] = g;
        } else {
            for (int q = 0; q < world; ++q) e[q] = static_cast<const T*>(grads.p[q])[i];
            g = finish_mean(grad_op, tree_fold_dyn(fop, e, world), inv_w);
            for (int q = 0; q < world; ++q) static_cast<T*>(grads.p[q])[i] = g;
        }
        const double gd = (double)g;
        if (coherent) {
            double p = (double)static_cast<const T*>(params.p[rank])[i];
            double a0 = naux > 0 ? (double)static_cast<const T*>(aux0.p[rank])[i] : 0.0;
            double a1 = naux > 1 ? (double)static_cast<const T*>(aux1.p[rank])[i] : 0.0;
            synk::rule_update(rp, p, a0, a1, gd);
            const T pt = (T)p, a0t = (T)a0, a1t = (T)a1;
            for (int q = 0; q < world; ++q) {
                static_cast<T*>(params.p[q])[i] = pt;
                if (naux > 0) static_cast<T*>(aux0.p[q])[i] = a0t;
                if (naux > 1) static_cast<T*>(aux1.p[q])[i] = a1t;
            }
        } else {
            for (int q = 0; q < world; ++q) {
                double p = (double)static_cast<const T*>(params.p[q])[i];
                double a0 = naux > 0 ? (double)static_cast<const T*>(aux0.p[q])[i] : 0.0;
                double a1 = naux > 1 ? (double)static_cast<const T*>(aux1.p[q])[i] : 0.0;
                synk::rule_update(rp, p, a0, a1, gd);
                static_cast<T*>(params.p[q])[i] = (T)p;
                if (naux > 0) static_cast<T*>(aux0.p[q])[i] = (T)a0;
                if (naux > 1) static_cast<T*>(aux1.p[q])[i] = (T)a1;
            }
        }
    }
}

// Single-replica optimizer step.
template <class T>
__global__ void __launch_bounds__(kBlock) optimizer_kernel(synk::RuleParams rp, int naux,
                                                           T* __restrict__ p, const T* __restrict__ g,
                                                           T* __restrict__ a0, T* __restrict__ a1,
                                                           uint64_t n) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) {
        double pv = (double)p[i];
        double x0 = naux > 0 ? (double)a0[i] : 0.0;
        double x1 = naux > 1 ? (double)a1[i] : 0.0;
        synk::rule_update(rp, pv, x0, x1, (double)g[i]);
        p[i] = (T)pv;
        if (naux > 0) a0[i] = (T)x0;
        if (naux > 1) a1[i] = (T)x1;
    }
}

// Chunk [lo, hi) of rank r, boundaries on 16-element multiples so vector
// paths stay aligned.
void chunk_of(uint64_t n, int world, int rank, uint64_t* lo, uint64_t* hi) {
    uint64_t per = (n + world - 1) / world;
    per = (per + 15) / 16 * 16;
    uint64_t a = per * (uint64_t)rank, b = a + per;
    *lo = a < n ? a : n;
    *hi = b < n ? b : n;
}

bool ptrs_aligned16(void* const* bufs, int w) {
    uintptr_t acc = 0;
    for (int q = 0; q < w; ++q) acc |= (uintptr_t)bufs[q];
    return (acc & 15) == 0;
}

int fill_ptrs(Ptrs* out, void* const* bufs, int w) {
    SYNK_REQUIRE(w >= 1 && w <= kMaxWorld, SYNK_EARG, "collective: world size out of range (1..64)");
    for (int q = 0; q < w; ++q) out->p[q] = bufs[q];
    return SYNK_OK;
}

template <class T>
int allreduce_t(synk_dev* d, int w, int op, void* const* bufs, uint64_t n, bool whole = false) {
    Ptrs P{};
    if (int rc = fill_ptrs(&P, bufs, w); rc != SYNK_OK) return rc;
    uint64_t lo = 0, hi = n;
    if (!whole) chunk_of(n, w, d->rank, &lo, &hi);
    if (lo >= hi) return SYNK_OK;
    double inv_w = 1.0 / (double)w;
    bool vec = ptrs_aligned16(bufs, w);
    constexpr int N = V16<T>::N;
    unsigned grid = synk::grid_for(d, vec ? (hi - lo) / N + 1 : hi - lo, kBlock);
    switch (w) {
#define SYNK_AR_CASE(WW)                                                                       \
    case WW:                                                                                   \
        allreduce_chunk_kernel<T, WW><<<grid, kBlock, 0, d->stream>>>(P, op, inv_w, lo, hi, vec); \
        break;
        SYNK_AR_CASE(1) SYNK_AR_CASE(2) SYNK_AR_CASE(3) SYNK_AR_CASE(4)
        SYNK_AR_CASE(5) SYNK_AR_CASE(6) SYNK_AR_CASE(7) SYNK_AR_CASE(8)
#undef SYNK_AR_CASE
    default:
        allreduce_chunk_dyn_kernel<T><<<grid, kBlock, 0, d->stream>>>(P, w, op, inv_w, lo, hi);
    }
    SYNK_LAUNCHED("allreduce_chunk_kernel");
    return SYNK_OK;
}

template <class T>
int allreduce_step_t(synk_dev* d, int w, int grad_op, const synk::RuleParams& rp, void* const* params,
                     void* const* grads, void* const* aux0, void* const* aux1, uint64_t n,
                     bool coherent) {
    Ptrs P{}, G{}, A0{}, A1{};
    int naux = synk::rule_aux_count(rp.rule);
    if (int rc = fill_ptrs(&P, params, w); rc != SYNK_OK) return rc;
    if (int rc = fill_ptrs(&G, grads, w); rc != SYNK_OK) return rc;
    if (naux > 0) {
        SYNK_REQUIRE(aux0 != nullptr, SYNK_EARG, "all_reduce_step: rule needs aux0");
        fill_ptrs(&A0, aux0, w);
    }
    if (naux > 1) {
        SYNK_REQUIRE(aux1 != nullptr, SYNK_EARG, "all_reduce_step: rule needs aux1");
        fill_ptrs(&A1, aux1, w);
    }
    uint64_t lo, hi;
    chunk_of(n, w, d->rank, &lo, &hi);
    if (lo >= hi) return SYNK_OK;
    double inv_w = 1.0 / (double)w;
    bool vec = ptrs_aligned16(params, w) && ptrs_aligned16(grads, w) && (naux < 1 || ptrs_aligned16(aux0, w)) &&
               (naux < 2 || ptrs_aligned16(aux1, w));
    unsigned grid = synk::grid_for(d, vec ? (hi - lo) / V16<T>::N + 1 : hi - lo, kBlock);
    switch (w) {
#define SYNK_ARS_CASE(WW)                                                                        \
    case WW:                                                                                     \
        allreduce_step_kernel<T, WW><<<grid, kBlock, 0, d->stream>>>(                            \
            P, G, A0, A1, w, d->rank, grad_op, inv_w, rp, naux, coherent, lo, hi, vec);          \
        break;
        SYNK_ARS_CASE(1) SYNK_ARS_CASE(2) SYNK_ARS_CASE(3) SYNK_ARS_CASE(4)
        SYNK_ARS_CASE(5) SYNK_ARS_CASE(6) SYNK_ARS_CASE(7) SYNK_ARS_CASE(8)
#undef SYNK_ARS_CASE
    default:
        allreduce_step_kernel<T, 0><<<grid, kBlock, 0, d->stream>>>(P, G, A0, A1, w, d->rank, grad_op,
                                                                    inv_w, rp, naux, coherent, lo, hi, false);
    }
    SYNK_LAUNCHED("allreduce_step_kernel");
    return SYNK_OK;
}

int make_rule(int rule, const double* hyper, double lr, uint64_t t, synk::RuleParams* rp) {
    SYNK_REQUIRE(rule >= SYNK_RULE_SGD && rule <= SYNK_RULE_ADAM, SYNK_EARG, "unknown update rule");
    rp->rule = rule;
    rp->lr = lr;
    rp->h0 = rp->h1 = rp->h2 = 0.0;
    rp->c1 = rp->c2 = 1.0;
    if (rule == SYNK_RULE_MOMENTUM) rp->h0 = hyper[0];
    if (rule == SYNK_RULE_RMSPROP) {
        rp->h0 = hyper[0];
        rp->h1 = hyper[1];
    }
    if (rule == SYNK_RULE_ADAM) {
        rp->h0 = hyper[0];
        rp->h1 = hyper[1];
        rp->h2 = hyper[2];
        rp->c1 = 1.0 - std::pow(hyper[0], (double)t);  // sgd.cpp:77-78
        rp->c2 = 1.0 - std::pow(hyper[1], (double)t);
    }
    return SYNK_OK;
}

}  // namespace

extern "C" {

int synk_chunk_range(uint64_t n, int world, int rank, uint64_t* lo, uint64_t* hi) {
    SYNK_REQUIRE(world >= 1 && rank >= 0 && rank < world, SYNK_EARG, "chunk_range: rank out of range");
    chunk_of(n, world, rank, lo, hi);
    return SYNK_OK;
}

int synk_all_reduce(synk_dev* d, int world, int dtype, int op, void* const* bufs, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_all_reduce: bad dtype");
    SYNK_REQUIRE(op >= SYNK_OP_SUM && op <= SYNK_OP_PROD, SYNK_EARG,
                 "all_reduce: Gather is not a reduction (use gather())");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    return dtype == SYNK_F32 ? allreduce_t<float>(d, world, op, bufs, n)
                             : allreduce_t<double>(d, world, op, bufs, n);
}

int synk_all_reduce_whole(synk_dev* d, int world, int dtype, int op, void* const* bufs, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_all_reduce: bad dtype");
    SYNK_REQUIRE(op >= SYNK_OP_SUM && op <= SYNK_OP_PROD, SYNK_EARG,
                 "all_reduce: Gather is not a reduction (use gather())");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    return dtype == SYNK_F32 ? allreduce_t<float>(d, world, op, bufs, n, true)
                             : allreduce_t<double>(d, world, op, bufs, n, true);
}

int synk_tree_reduce(synk_dev* d, int world, int dtype, int op, const void* const* bufs, uint64_t n,
                     void* out) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_tree_reduce: bad dtype");
    SYNK_REQUIRE(op >= SYNK_OP_SUM && op <= SYNK_OP_PROD, SYNK_EARG,
                 "reduce: Gather is not a reduction (use gather())");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    Ptrs P{};
    if (int rc = fill_ptrs(&P, const_cast<void* const*>(bufs), world); rc != SYNK_OK) return rc;
    unsigned grid = synk::grid_for(d, n, kBlock);
    double inv_w = 1.0 / (double)world;
    if (dtype == SYNK_F32)
        tree_reduce_kernel<float><<<grid, kBlock, 0, d->stream>>>(P, world, op, inv_w, n, (float*)out);
    else
        tree_reduce_kernel<double><<<grid, kBlock, 0, d->stream>>>(P, world, op, inv_w, n, (double*)out);
    SYNK_LAUNCHED("tree_reduce_kernel");
    return SYNK_OK;
}

static int broadcast_impl(synk_dev* d, int world, int src, void* const* bufs, uint64_t bytes, bool whole) {
    SYNK_REQUIRE(src >= 0 && src < world, SYNK_EARG, "broadcast: src rank out of range");
    if (bytes == 0 || world == 1) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    Ptrs P{};
    if (int rc = fill_ptrs(&P, bufs, world); rc != SYNK_OK) return rc;
    uint64_t lo = 0, hi = bytes;
    if (!whole) chunk_of(bytes, world, d->rank, &lo, &hi);  // byte chunks, 16-byte multiples
    if (lo >= hi) return SYNK_OK;
    bool vec = ptrs_aligned16(bufs, world) && hi % 16 == 0;
    unsigned grid = synk::grid_for(d, vec ? (hi - lo) / 16 + 1 : hi - lo, kBlock);
    bcast_chunk_kernel<<<grid, kBlock, 0, d->stream>>>(P, world, src, lo, hi, vec);
    SYNK_LAUNCHED("bcast_chunk_kernel");
    return SYNK_OK;
}

int synk_broadcast(synk_dev* d, int world, int src, void* const* bufs, uint64_t bytes) {
    return broadcast_impl(d, world, src, bufs, bytes, false);
}

int synk_broadcast_whole(synk_dev* d, int world, int src, void* const* bufs, uint64_t bytes) {
    return broadcast_impl(d, world, src, bufs, bytes, true);
}

int synk_optimizer_step(synk_dev* d, int dtype, int rule, const double* hyper, double lr, uint64_t t,
                        void* params, const void* grads, void* aux0, void* aux1, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_optimizer_step: bad dtype");
    synk::RuleParams rp;
    if (int rc = make_rule(rule, hyper, lr, t, &rp); rc != SYNK_OK) return rc;
    int naux = synk::rule_aux_count(rule);
    SYNK_REQUIRE(naux < 1 || aux0, SYNK_EARG, "optimizer step: rule needs aux0");
    SYNK_REQUIRE(naux < 2 || aux1, SYNK_EARG, "optimizer step: rule needs aux1");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    unsigned grid = synk::grid_for(d, n, kBlock);
    if (dtype == SYNK_F32)
        optimizer_kernel<float><<<grid, kBlock, 0, d->stream>>>(rp, naux, (float*)params,
                                                                (const float*)grads, (float*)aux0,
                                                                (float*)aux1, n);
    else
        optimizer_kernel<double><<<grid, kBlock, 0, d->stream>>>(rp, naux, (double*)params,
                                                                 (const double*)grads, (double*)aux0,
                                                                 (double*)aux1, n);
    SYNK_LAUNCHED("optimizer_kernel");
    return SYNK_OK;
}

int synk_all_reduce_step(synk_dev* d, int world, int dtype, int grad_op, int rule, const double* hyper,
                         double lr, uint64_t t, void* const* params, void* const* grads,
                         void* const* aux0, void* const* aux1, uint64_t n, int coherent) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_all_reduce_step: bad dtype");
    SYNK_REQUIRE(grad_op >= SYNK_OP_SUM && grad_op <= SYNK_OP_PROD, SYNK_EARG,
                 "all_reduce: Gather is not a reduction (use gather())");
    synk::RuleParams rp;
    if (int rc = make_rule(rule, hyper, lr, t, &rp); rc != SYNK_OK) return rc;
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    return dtype == SYNK_F32
               ? allreduce_step_t<float>(d, world, grad_op, rp, params, grads, aux0, aux1, n, coherent)
               : allreduce_step_t<double>(d, world, grad_op, rp, params, grads, aux0, aux1, n, coherent);
}

}  // extern "C"
