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

#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include "common.cuh"
#include "optim_math.cuh"

namespace {

using synk::combine_op;

constexpr int kMaxWorld = 64;
constexpr int kBlock = 256;
// The fused all-reduce + update: 256-thread CTAs, all resident at once
// (synk::resident_grid), one vector item per thread per iteration (~80
// registers). Measured against 128-thread CTAs
// that co-reside with the persistent GEMM and two items in flight per thread
// (122 registers): C5 1.053 vs 1.065-1.075 ms (serialised or overlapped), so
// the occupancy of the streaming loop matters more than co-residency.
constexpr int kStepBlock = 256;

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
// Vector body: one 32-byte vector (8 f32 / 4 f64 elements; sm_100
// ld/st.global.v8.b32, 16-byte lanes when a pointer is not 32-byte aligned)
// of chunk r per iteration: W peer loads of the gradient, per-lane tree fold
// + 1/W, then the update on this rank's (coherent) params/aux and W peer
// stores of each. With W == 1 the fold is the identity (and x*1.0 is exact),
// so the gradient is not rewritten.

template <class T, int BYTES>
struct VecT {
    static constexpr int N = BYTES / (int)sizeof(T);
    T e[N];
};

template <class T, int BYTES>
__device__ __forceinline__ VecT<T, BYTES> vload(const void* base, uint64_t v) {
    VecT<T, BYTES> x;
    const char* p = static_cast<const char*>(base) + v * BYTES;
    if constexpr (BYTES == 32) {
        uint32_t* w = reinterpret_cast<uint32_t*>(&x);
        asm volatile("ld.global.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                     : "l"(p));
    } else {
        *reinterpret_cast<uint4*>(&x) = *reinterpret_cast<const uint4*>(p);
    }
    return x;
}

template <class T, int BYTES>
__device__ __forceinline__ void vstore(void* base, uint64_t v, const VecT<T, BYTES>& x) {
    char* p = static_cast<char*>(base) + v * BYTES;
    if constexpr (BYTES == 32) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(&x);
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                     "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                     : "memory");
    } else {
        *reinterpret_cast<uint4*>(p) = *reinterpret_cast<const uint4*>(&x);
    }
}

// bf16 weight shadow written along with the new params (synk_cuda.h).
struct Shadow {
    void* base[SYNK_SHADOW_MAX_WORLD];
    uint32_t count;
    uint64_t elem_base;  // flat index of the kernel's element 0
    synk_bf16_shadow_seg seg[SYNK_SHADOW_MAX_SEGS];
};

__device__ __forceinline__ int shadow_find(const Shadow& sh, uint64_t gi) {
    for (uint32_t s = 0; s < sh.count; ++s)
        if (gi >= sh.seg[s].first && gi - sh.seg[s].first < sh.seg[s].rows * sh.seg[s].cols) return (int)s;
    return -1;
}

// Elements [gi, gi + N) of the flat block, new f32 values v: their bf16
// copies into replica q's shadow (same rounding as the cast kernels).
template <int N>
__device__ __forceinline__ void shadow_store(const Shadow& sh, int q, uint64_t gi, const float* v) {
    int s = shadow_find(sh, gi);
    if (s < 0 && N > 1) s = shadow_find(sh, gi + N - 1);  // a segment may start inside the vector
    if (s < 0) return;
    const synk_bf16_shadow_seg& g = sh.seg[s];
    char* b = static_cast<char*>(sh.base[q]);
    __nv_bfloat16* w = reinterpret_cast<__nv_bfloat16*>(b + g.off_w);
    __nv_bfloat16* wt = g.off_wt == SYNK_NO_TRANSPOSE ? nullptr : reinterpret_cast<__nv_bfloat16*>(b + g.off_wt);
    const uint64_t size = g.rows * g.cols;
    if (N == 8 && !wt && g.ldw == g.cols && gi >= g.first && gi + 8 <= g.first + size && ((gi - g.first) & 7) == 0) {
        // unpadded rows: the shadow is the segment itself, no row split (no
        // 64-bit division per vector on the update's streaming path)
        __nv_bfloat162 h[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
        *reinterpret_cast<uint4*>(w + (gi - g.first)) = *reinterpret_cast<const uint4*>(h);
        return;
    }
    if (N == 8 && gi >= g.first && gi + 8 <= g.first + size) {
        const uint64_t o = gi - g.first, r = o / g.cols, c = o - r * g.cols;
        const uint64_t at = r * g.ldw + c;
        if (c + 8 <= g.cols && (at & 7) == 0) {  // one row, 16-byte aligned: one store
            __nv_bfloat162 h[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[2 * k], v[2 * k + 1]);
            *reinterpret_cast<uint4*>(w + at) = *reinterpret_cast<const uint4*>(h);
            if (wt)
#pragma unroll
                for (int k = 0; k < 8; ++k) wt[(c + k) * g.ldwt + r] = __float2bfloat16_rn(v[k]);
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
        const uint64_t e = gi + k;
        int sk = shadow_find(sh, e);
        if (sk < 0) continue;
        const synk_bf16_shadow_seg& gk = sh.seg[sk];
        __nv_bfloat16* wk = reinterpret_cast<__nv_bfloat16*>(b + gk.off_w);
        const uint64_t o = e - gk.first, r = o / gk.cols, c = o - r * gk.cols;
        const __nv_bfloat16 h = __float2bfloat16_rn(v[k]);
        wk[r * gk.ldw + c] = h;
        if (gk.off_wt != SYNK_NO_TRANSPOSE) reinterpret_cast<__nv_bfloat16*>(b + gk.off_wt)[c * gk.ldwt + r] = h;
    }
}

// U vector items per call (v[u], valid while v[u] < v_end): every load of
// every item (W gradient replicas, params, aux) is issued before the first
// use, so a thread has U x (W + 1 + naux) 16/32-byte loads in flight instead
// of one dependent round trip per array. The kernel instantiates U = 1: two
// items per thread raised the registers to 122 and the resident CTAs per SM
// fell, which cost more than the extra loads in flight bought (kStepBlock).
template <class T, int W, int BYTES, bool SH, int U, int RULE>
__device__ __forceinline__ void step_vectors(const Ptrs& params, const Ptrs& grads, const Ptrs& aux0, const Ptrs& aux1,
                                             int rank, int grad_op, int fop, double inv_w, const synk::RuleParams& rp,
                                             int naux, uint64_t v0, uint64_t vstride, uint64_t v_end, const Shadow& sh,
                                             bool grads_local) {
    using V = VecT<T, BYTES>;
    constexpr int N = V::N;
    V gx[U][W], p[U], a0[U], a1[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t v = v0 + u * vstride;
        if (v >= v_end) continue;
#pragma unroll
        for (int q = 0; q < W; ++q) gx[u][q] = vload<T, BYTES>(grads.p[q], v);
        p[u] = vload<T, BYTES>(params.p[rank], v);
        if (naux > 0) a0[u] = vload<T, BYTES>(aux0.p[rank], v);
        if (naux > 1) a1[u] = vload<T, BYTES>(aux1.p[rank], v);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
        const uint64_t v = v0 + u * vstride;
        if (v >= v_end) continue;
        V g;
#pragma unroll
        for (int k = 0; k < N; ++k) {
            T e[W];
#pragma unroll
            for (int q = 0; q < W; ++q) e[q] = gx[u][q].e[k];
            g.e[k] = finish_mean(grad_op, tree_fold_regs<T, W>(fop, e), inv_w);
        }
        if constexpr (W > 1) {
            if (grads_local) {  // deferred all-gather: the chunk stays with its owner
                vstore<T, BYTES>(grads.p[rank], v, g);
            } else {
#pragma unroll
                for (int q = 0; q < W; ++q) vstore<T, BYTES>(grads.p[q], v, g);
            }
        }
        V pn = p[u], x0 = naux > 0 ? a0[u] : p[u], x1 = naux > 1 ? a1[u] : p[u];
#pragma unroll
        for (int k = 0; k < N; ++k) {
            double pd = (double)pn.e[k];
            double d0 = (double)x0.e[k];
            double d1 = (double)x1.e[k];
            synk::rule_update_t<RULE>(rp, pd, d0, d1, (double)g.e[k]);
            pn.e[k] = (T)pd;
            x0.e[k] = (T)d0;
            x1.e[k] = (T)d1;
        }
#pragma unroll
        for (int q = 0; q < W; ++q) {
            vstore<T, BYTES>(params.p[q], v, pn);
            if (naux > 0) vstore<T, BYTES>(aux0.p[q], v, x0);
            if (naux > 1) vstore<T, BYTES>(aux1.p[q], v, x1);
            if constexpr (SH) shadow_store<N>(sh, q, sh.elem_base + v * N, reinterpret_cast<const float*>(pn.e));
        }
    }
}

// The vector part of one rank's chunk [lo, hi): returns where the scalar
// tail starts.
template <class T, int W, bool SH, int RULE>
__device__ __forceinline__ uint64_t vector_loop(const Ptrs& params, const Ptrs& grads, const Ptrs& aux0, const Ptrs& aux1,
                                                int rank, int grad_op, int fop, double inv_w, const synk::RuleParams& rp,
                                                int naux, uint64_t lo, uint64_t hi, uint64_t tid, uint64_t stride,
                                                int vec_bytes, const Shadow& sh, bool grads_local) {
    if (vec_bytes == 32) {
        constexpr int N = VecT<T, 32>::N;
        const uint64_t v0 = lo / N, v1 = hi / N;
        for (uint64_t v = v0 + tid; v < v1; v += stride)
            step_vectors<T, W, 32, SH, 1, RULE>(params, grads, aux0, aux1, rank, grad_op, fop, inv_w, rp, naux, v,
                                                stride, v1, sh, grads_local);
        return v1 * N;
    }
    constexpr int N = VecT<T, 16>::N;
    const uint64_t v0 = lo / N, v1 = hi / N;
    for (uint64_t v = v0 + tid; v < v1; v += stride)
        step_vectors<T, W, 16, SH, 1, RULE>(params, grads, aux0, aux1, rank, grad_op, fop, inv_w, rp, naux, v, stride,
                                            v1, sh, grads_local);
    return v1 * N;
}

template <class T, int W, bool SH>
__global__ void __launch_bounds__(kStepBlock) allreduce_step_kernel(
    Ptrs params, Ptrs grads, Ptrs aux0, Ptrs aux1, int world, int rank, int grad_op,
    double inv_w, synk::RuleParams rp, int naux, bool coherent, bool grads_local, uint64_t lo, uint64_t hi,
    int vec_bytes, Shadow sh) {
    synk::wait_prerequisite_grid();  // no-op unless launched as a follow-up (W = 1, after a GEMM)
    const int fop = grad_op == SYNK_OP_MEAN ? SYNK_OP_SUM : grad_op;
    uint64_t tid = (uint64_t)blockIdx.x * kStepBlock + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * kStepBlock;
    if constexpr (W > 0) {
        if (vec_bytes && coherent) {
            // lo is 16-element aligned, so a multiple of both vector widths;
            // one loop per rule, each with that rule's code only
            switch (rp.rule) {
            case SYNK_RULE_SGD:
                lo = vector_loop<T, W, SH, SYNK_RULE_SGD>(params, grads, aux0, aux1, rank, grad_op, fop, inv_w, rp,
                                                          naux, lo, hi, tid, stride, vec_bytes, sh, grads_local);
                break;
            case SYNK_RULE_MOMENTUM:
                lo = vector_loop<T, W, SH, SYNK_RULE_MOMENTUM>(params, grads, aux0, aux1, rank, grad_op, fop, inv_w, rp,
                                                               naux, lo, hi, tid, stride, vec_bytes, sh, grads_local);
                break;
            default:
                lo = vector_loop<T, W, SH, -1>(params, grads, aux0, aux1, rank, grad_op, fop, inv_w, rp, naux, lo, hi,
                                               tid, stride, vec_bytes, sh, grads_local);
            }
        }
    }
    for (uint64_t i = lo + tid; i < hi; i += stride) {
        T e[W > 0 ? W : kMaxWorld];
        T g;
        if constexpr (W > 0) {
#pragma unroll
            for (int q = 0; q < W; ++q) e[q] = static_cast<const T*>(grads.p[q])[i];
            g = finish_mean(grad_op, tree_fold_regs<T, W>(fop, e), inv_w);
            if (grads_local) {
                static_cast<T*>(grads.p[rank])[i] = g;
            } else {
#pragma unroll
                for (int q = 0; q < W; ++q) static_cast<T*>(grads.p[q])[i] = g;
            }
        } else {
            for (int q = 0; q < world; ++q) e[q] = static_cast<const T*>(grads.p[q])[i];
            g = finish_mean(grad_op, tree_fold_dyn(fop, e, world), inv_w);
            if (grads_local) static_cast<T*>(grads.p[rank])[i] = g;
            else
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
                if constexpr (SH) {
                    const float f = (float)pt;
                    shadow_store<1>(sh, q, sh.elem_base + i, &f);
                }
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
                if constexpr (SH) {
                    const float f = (float)(T)p;
                    shadow_store<1>(sh, q, sh.elem_base + i, &f);
                }
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

bool ptrs_aligned(void* const* bufs, int w, uintptr_t align) {
    uintptr_t acc = 0;
    for (int q = 0; q < w; ++q) acc |= (uintptr_t)bufs[q];
    return (acc & (align - 1)) == 0;
}

template <class T>
int allreduce_step_t(synk_dev* d, int w, int grad_op, const synk::RuleParams& rp, void* const* params,
                     void* const* grads, void* const* aux0, void* const* aux1, uint64_t n,
                     int flags, const Shadow* sh) {
    const bool coherent = flags & SYNK_STEP_COHERENT;
    const bool grads_local = (flags & SYNK_STEP_GRADS_LOCAL) && w > 1;
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
    auto aligned = [&](uintptr_t a) {
        return ptrs_aligned(params, w, a) && ptrs_aligned(grads, w, a) && (naux < 1 || ptrs_aligned(aux0, w, a)) &&
               (naux < 2 || ptrs_aligned(aux1, w, a));
    };
    // 256-bit lanes when every pointer allows them (the measured winner on the
    // gather, profiles/r01_gather.md), else 16-byte lanes, else scalar.
    static const int forced = [] {
        const char* e = getenv("SYNK_UPDATE_VEC");  // A/B: 16 forces 16-byte lanes
        return e ? atoi(e) : 0;
    }();
    const int vec_bytes = aligned(32) && forced != 16 ? 32 : (aligned(16) ? 16 : 0);
    const uint64_t items = vec_bytes ? (hi - lo) / (vec_bytes / sizeof(T)) + 1 : hi - lo;
    // at most 4 CTAs per SM (37K registers): beside them the next narrow GEMM
    // still fits its two CTAs per SM (94 registers x 128 threads each)
    unsigned grid = synk::grid_for(d, items, kStepBlock);
    if (flags & SYNK_STEP_BACKGROUND) {
        // Overlapped with tensor-core GEMMs on the other stream: a few CTAs
        // stream the segment at a fraction of HBM bandwidth instead of
        // competing for every SM's issue slots with the persistent GEMM.
        static const unsigned bg = [] {
            const char* e = getenv("SYNK_BG_CTAS");  // A/B: CTAs of a background update
            const int v = e ? atoi(e) : 0;
            return v > 0 ? (unsigned)v : 32u;
        }();
        grid = std::min(grid, bg);
    }
    Shadow none{};
    const Shadow& S = sh ? *sh : none;
    const bool with = sh != nullptr;
    switch (w) {
#define SYNK_ARS_CASE(WW)                                                                                        \
    case WW:                                                                                                     \
        if (with) {                                                                                              \
            if (int rc = synk::prefer_shared_carveout((const void*)allreduce_step_kernel<T, WW, true>, d->device); rc) \
                return rc;                                                                                       \
            if (!(flags & SYNK_STEP_BACKGROUND))                                                                 \
                grid = synk::resident_grid((const void*)allreduce_step_kernel<T, WW, true>, d->device, kStepBlock, items); \
            if (WW == 1) /* one GPU: programmatically dependent on the weight-gradient product */              \
                SYNK_CU(synk::launch_follow_up(d, allreduce_step_kernel<T, WW, true>, grid, kStepBlock, P, G, A0, A1, w, \
                                               d->rank, grad_op, inv_w, rp, naux, coherent, grads_local, lo, hi,      \
                                               vec_bytes, S));                                                        \
            else                                                                                                 \
                allreduce_step_kernel<T, WW, true><<<grid, kStepBlock, 0, d->stream>>>(                              \
                    P, G, A0, A1, w, d->rank, grad_op, inv_w, rp, naux, coherent, grads_local, lo, hi, vec_bytes, S);         \
        } else {                                                                                                 \
            if (int rc = synk::prefer_shared_carveout((const void*)allreduce_step_kernel<T, WW, false>, d->device); rc) \
                return rc;                                                                                       \
            if (!(flags & SYNK_STEP_BACKGROUND))                                                                 \
                grid = synk::resident_grid((const void*)allreduce_step_kernel<T, WW, false>, d->device, kStepBlock, items); \
            if (WW == 1)                                                                                         \
                SYNK_CU(synk::launch_follow_up(d, allreduce_step_kernel<T, WW, false>, grid, kStepBlock, P, G, A0, A1, w, \
                                               d->rank, grad_op, inv_w, rp, naux, coherent, grads_local, lo, hi,      \
                                               vec_bytes, S));                                                        \
            else                                                                                                 \
                allreduce_step_kernel<T, WW, false><<<grid, kStepBlock, 0, d->stream>>>(                             \
                    P, G, A0, A1, w, d->rank, grad_op, inv_w, rp, naux, coherent, grads_local, lo, hi, vec_bytes, S);         \
        }                                                                                                        \
        break;
        SYNK_ARS_CASE(1) SYNK_ARS_CASE(2) SYNK_ARS_CASE(3) SYNK_ARS_CASE(4)
        SYNK_ARS_CASE(5) SYNK_ARS_CASE(6) SYNK_ARS_CASE(7) SYNK_ARS_CASE(8)
#undef SYNK_ARS_CASE
    default:
        SYNK_REQUIRE(!with, SYNK_EARG, "all_reduce_step: bf16 shadows need world <= 8");
        allreduce_step_kernel<T, 0, false><<<grid, kStepBlock, 0, d->stream>>>(P, G, A0, A1, w, d->rank, grad_op,
                                                                           inv_w, rp, naux, coherent, grads_local, lo, hi, 0,
                                                                           S);
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
                         void* const* aux0, void* const* aux1, uint64_t n, int flags) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_all_reduce_step: bad dtype");
    SYNK_REQUIRE(grad_op >= SYNK_OP_SUM && grad_op <= SYNK_OP_PROD, SYNK_EARG,
                 "all_reduce: Gather is not a reduction (use gather())");
    synk::RuleParams rp;
    if (int rc = make_rule(rule, hyper, lr, t, &rp); rc != SYNK_OK) return rc;
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    return dtype == SYNK_F32
               ? allreduce_step_t<float>(d, world, grad_op, rp, params, grads, aux0, aux1, n, flags, nullptr)
               : allreduce_step_t<double>(d, world, grad_op, rp, params, grads, aux0, aux1, n, flags, nullptr);
}

int synk_all_reduce_step_ex(synk_dev* d, int world, int dtype, int grad_op, int rule, const double* hyper,
                            double lr, uint64_t t, void* const* params, void* const* grads,
                            void* const* aux0, void* const* aux1, uint64_t n, int flags, uint64_t elem_base,
                            const synk_bf16_shadow* shadow, void* const* shadow_bases) {
    if (!shadow)
        return synk_all_reduce_step(d, world, dtype, grad_op, rule, hyper, lr, t, params, grads, aux0, aux1, n,
                                    flags);
    SYNK_REQUIRE(dtype == SYNK_F32, SYNK_EDTYPE, "all_reduce_step: bf16 shadows need f32 params");
    SYNK_REQUIRE(world >= 1 && world <= SYNK_SHADOW_MAX_WORLD, SYNK_EARG, "all_reduce_step: shadows need world <= 8");
    SYNK_REQUIRE(shadow->count <= SYNK_SHADOW_MAX_SEGS && shadow_bases, SYNK_EARG, "all_reduce_step: bad shadow");
    SYNK_REQUIRE(grad_op >= SYNK_OP_SUM && grad_op <= SYNK_OP_PROD, SYNK_EARG,
                 "all_reduce: Gather is not a reduction (use gather())");
    synk::RuleParams rp;
    if (int rc = make_rule(rule, hyper, lr, t, &rp); rc != SYNK_OK) return rc;
    if (n == 0) return SYNK_OK;
    Shadow S{};
    for (int q = 0; q < world; ++q) {
        SYNK_REQUIRE(shadow_bases[q], SYNK_EARG, "all_reduce_step: missing shadow");
        S.base[q] = shadow_bases[q];
    }
    S.count = shadow->count;
    S.elem_base = elem_base;
    for (uint32_t k = 0; k < shadow->count; ++k) S.seg[k] = shadow->seg[k];
    synk::DeviceGuard g(d->device);
    return allreduce_step_t<float>(d, world, grad_op, rp, params, grads, aux0, aux1, n, flags, &S);
}

}  // extern "C"
