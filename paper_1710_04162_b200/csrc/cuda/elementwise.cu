// Aggregation kernels: combine / weighted mean / scale / fill / ordered folds,
// one-pass column statistics, bitwise compare and finiteness check.
//
// All are HBM-bound streaming kernels: 16-byte vector loads (float4 /
// double2) when every operand is 16-byte aligned, grid-stride over a grid of
// a few waves of 148 SMs. The arithmetic reproduces the reference exactly
// (tensor.cpp:250-285,367-373): combine in T, weighted mean and scale through
// f64 with one cast on store.

#include <math.h>
#include <stdlib.h>

#include "common.cuh"

namespace {

using synk::combine_op;

constexpr int kBlock = 256;

template <class T>
struct Vec16;
template <>
struct Vec16<float> {
    using V = float4;
    static constexpr int N = 4;
};
template <>
struct Vec16<double> {
    using V = double2;
    static constexpr int N = 2;
};

template <class T>
__device__ __forceinline__ T& lane(typename Vec16<T>::V& v, int i) {
    return reinterpret_cast<T*>(&v)[i];
}

inline bool aligned16(const void* a, const void* b = nullptr, const void* c = nullptr) {
    return (((uintptr_t)a | (uintptr_t)b | (uintptr_t)c) & 15) == 0;
}

// ---- binary in-place maps ----------------------------------------------------

struct CombineF {
    int op;
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const { return combine_op(op, a, b); }
};

struct WMeanF {
    double wa, wb, inv;
    template <class T>
    __device__ __forceinline__ T operator()(T a, T b) const {
        // (a*wa + b*wb) * inv, each product/sum rounded separately (no FMA):
        // the reference's x86-64 build does not contract.
        double x = __dmul_rn((double)a, wa);
        double y = __dmul_rn((double)b, wb);
        return (T)__dmul_rn(__dadd_rn(x, y), inv);
    }
};

template <class T, class F>
__global__ void __launch_bounds__(kBlock) map2_kernel(T* __restrict__ a, const T* __restrict__ b,
                                                      uint64_t n, F f, bool vec) {
    using V = typename Vec16<T>::V;
    constexpr int N = Vec16<T>::N;
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    uint64_t stride = (uint64_t)gridDim.x * kBlock;
    uint64_t head = 0;
    if (vec) {
        uint64_t nv = n / N;
        V* av = reinterpret_cast<V*>(a);
        const V* bv = reinterpret_cast<const V*>(b);
        for (uint64_t i = tid; i < nv; i += stride) {
            V x = av[i];
            V y = bv[i];
#pragma unroll
            for (int k = 0; k < N; ++k) lane<T>(x, k) = f(lane<T>(x, k), lane<T>(y, k));
            av[i] = x;
        }
        head = nv * N;
    }
    for (uint64_t i = head + tid; i < n; i += stride) a[i] = f(a[i], b[i]);
}

template <class F>
int run_map2(synk_dev* d, int dtype, void* a, const void* b, uint64_t n, F f) {
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    bool vec = aligned16(a, b);
    uint64_t work = vec ? n / (dtype == SYNK_F32 ? 4 : 2) + 1 : n;
    unsigned grid = synk::grid_for(d, work, kBlock);
    if (dtype == SYNK_F32)
        map2_kernel<float><<<grid, kBlock, 0, d->stream>>>((float*)a, (const float*)b, n, f, vec);
    else
        map2_kernel<double><<<grid, kBlock, 0, d->stream>>>((double*)a, (const double*)b, n, f, vec);
    SYNK_LAUNCHED("map2_kernel");
    return SYNK_OK;
}

// ---- unary in-place maps -----------------------------------------------------

template <class T>
__global__ void __launch_bounds__(kBlock) scale_kernel(T* __restrict__ a, uint64_t n, double f) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock)
        a[i] = (T)__dmul_rn((double)a[i], f);
}

template <class T>
__global__ void __launch_bounds__(kBlock) fill_kernel(T* __restrict__ a, uint64_t n, T v) {
    synk::wait_prerequisite_grid();  // no-op unless launched as a follow-up
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) a[i] = v;
}

// Counter-based U[-1,1) synthetic data: element i of the virtual array gets
// splitmix64(seed + i*golden) -> top 24 bits -> k * 2^-23 - 1 (exact in f32/f64).
// Same formula as oracle/synk_oracle.c so_fill_uniform.
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

template <class T>
__global__ void __launch_bounds__(kBlock) fill_uniform_kernel(T* __restrict__ a, uint64_t n, uint64_t seed,
                                                              uint64_t first) {
    const uint64_t stride = (uint64_t)gridDim.x * kBlock;
    for (uint64_t i = (uint64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride) {
        const uint64_t k = splitmix64(seed + (first + i) * 0x9E3779B97F4A7C15ull) >> 40;
        a[i] = (T)((double)k * 0x1p-23 - 1.0);
    }
}

template <>
__global__ void __launch_bounds__(kBlock) fill_uniform_kernel<float>(float* __restrict__ a, uint64_t n, uint64_t seed,
                                                                     uint64_t first) {
    // four elements per thread per iteration, one 16-byte store when aligned
    const uint64_t stride = (uint64_t)gridDim.x * kBlock;
    const uint64_t nv = ((uintptr_t)a & 15) == 0 ? n / 4 : 0;
    for (uint64_t v = (uint64_t)blockIdx.x * kBlock + threadIdx.x; v < nv; v += stride) {
        float r[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t k = splitmix64(seed + (first + 4 * v + j) * 0x9E3779B97F4A7C15ull) >> 40;
            r[j] = (float)k * 0x1p-23f - 1.0f;
        }
        reinterpret_cast<float4*>(a)[v] = make_float4(r[0], r[1], r[2], r[3]);
    }
    for (uint64_t i = 4 * nv + (uint64_t)blockIdx.x * kBlock + threadIdx.x; i < n; i += stride) {
        const uint64_t k = splitmix64(seed + (first + i) * 0x9E3779B97F4A7C15ull) >> 40;
        a[i] = (float)k * 0x1p-23f - 1.0f;
    }
}

// ---- ordered fold over contributions (slices / ranks) ---------------------------

constexpr int kMaxParts = 64;
struct FoldArgs {
    const void* parts[kMaxParts];
    double weights[kMaxParts];
    uint32_t count;
};

template <class T>
__global__ void __launch_bounds__(kBlock) left_fold_kernel(int op, T* __restrict__ out,
                                                           FoldArgs args, uint64_t n) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) {
        T acc = static_cast<const T*>(args.parts[0])[i];
        double w = args.weights[0];
        for (uint32_t k = 1; k < args.count; ++k) {
            T b = static_cast<const T*>(args.parts[k])[i];
            if (op == SYNK_OP_MEAN) {
                double wb = args.weights[k];
                WMeanF f{w, wb, 1.0 / (w + wb)};
                acc = f(acc, b);
                w += wb;
            } else {
                acc = combine_op(op, acc, b);
            }
        }
        out[i] = acc;
    }
}

// ---- column statistics (one HBM pass) --------------------------------------------
// Phase 1: CTA (cx, cy) owns column tile cx (kBlock columns, one per thread,
// coalesced across the warp) and row chunk cy; accumulates sum in f64 and
// max/min in T. Phase 2: one thread per column folds the row chunks in fixed
// order, so the result is deterministic run to run.

template <class T>
__global__ void __launch_bounds__(kBlock) colstats_partial_kernel(
    const T* __restrict__ x, uint64_t rows, uint64_t cols, uint64_t rows_per_chunk,
    double* __restrict__ psum, T* __restrict__ pmax, T* __restrict__ pmin) {
    uint64_t c = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    uint64_t r0 = (uint64_t)blockIdx.y * rows_per_chunk;
    uint64_t r1 = r0 + rows_per_chunk < rows ? r0 + rows_per_chunk : rows;
    if (c >= cols) return;
    double s = 0.0;
    T mx = -INFINITY, mn = INFINITY;
    uint64_t r = r0;
    for (; r + 8 <= r1; r += 8) {
        T v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = __ldg(x + (r + k) * cols + c);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            s += (double)v[k];
            mx = v[k] > mx ? v[k] : mx;
            mn = v[k] < mn ? v[k] : mn;
        }
    }
    for (; r < r1; ++r) {
        T v = __ldg(x + r * cols + c);
        s += (double)v;
        mx = v > mx ? v : mx;
        mn = v < mn ? v : mn;
    }
    uint64_t o = (uint64_t)blockIdx.y * cols + c;
    psum[o] = s;
    pmax[o] = mx;
    pmin[o] = mn;
}

// Vector variant (16-byte groups of 4 f32 / 2 f64 columns per thread): 8
// rows in flight per thread = 128 B (volatile asm keeps all 8 loads ahead of
// the folds), non-allocating loads. Same fold order per column as the scalar
// kernel, so results are identical.
__device__ __forceinline__ uint4 ld_stream16(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

template <class T>
__global__ void __launch_bounds__(kBlock) colstats_partial_vec_kernel(
    const T* __restrict__ x, uint64_t rows, uint64_t cols, uint64_t rows_per_chunk, uint32_t rpb,
    double* __restrict__ psum, T* __restrict__ pmax, T* __restrict__ pmin) {
    // rpb > 1 (narrow rows): the CTA covers rpb rows per step, thread group
    // tr takes rows r0+tr, r0+tr+rpb, ... and owns partial slot chunk*rpb+tr.
    using V = typename Vec16<T>::V;
    constexpr int N = Vec16<T>::N;
    const uint64_t ncv = cols / N;
    const uint64_t cv = rpb > 1 ? threadIdx.x % ncv : (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    const uint32_t tr = rpb > 1 ? threadIdx.x / (uint32_t)ncv : 0;
    const uint64_t r0 = (uint64_t)blockIdx.y * rows_per_chunk + tr;
    const uint64_t r1 = r0 - tr + rows_per_chunk < rows ? r0 - tr + rows_per_chunk : rows;
    if (cv >= ncv || tr >= rpb) return;
    const V* xv = reinterpret_cast<const V*>(x) + cv;
    double s[N];
    T mx[N], mn[N];
#pragma unroll
    for (int j = 0; j < N; ++j) s[j] = 0.0, mx[j] = -INFINITY, mn[j] = INFINITY;
    auto fold = [&](V vv) {
#pragma unroll
        for (int j = 0; j < N; ++j) {
            const T e = lane<T>(vv, j);
            s[j] += (double)e;
            mx[j] = e > mx[j] ? e : mx[j];
            mn[j] = e < mn[j] ? e : mn[j];
        }
    };
    uint64_t r = r0;
    for (; r + 7 * (uint64_t)rpb < r1; r += 8 * (uint64_t)rpb) {
        uint4 v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ld_stream16(xv + (r + k * (uint64_t)rpb) * ncv);
#pragma unroll
        for (int k = 0; k < 8; ++k) fold(*reinterpret_cast<V*>(&v[k]));
    }
    for (; r < r1; r += rpb) {
        uint4 v = ld_stream16(xv + r * ncv);
        fold(*reinterpret_cast<V*>(&v));
    }
    const uint64_t o = ((uint64_t)blockIdx.y * rpb + tr) * cols + cv * N;
#pragma unroll
    for (int j = 0; j < N; ++j) psum[o + j] = s[j], pmax[o + j] = mx[j], pmin[o + j] = mn[j];
}

// CTA = 32 columns x 8 slot groups: group g folds slots g, g+8, ... (4 loads in
// flight), then group 0 folds the 8 group results in order -- a fixed tree, so
// the result is deterministic and independent of timing.
template <class T>
__global__ void __launch_bounds__(kBlock) colstats_final_kernel(
    uint64_t chunks, uint64_t cols, const double* __restrict__ psum, const T* __restrict__ pmax,
    const T* __restrict__ pmin, T* sum_out, T* max_out, T* min_out) {
    __shared__ double ss[8][33];
    __shared__ T smx[8][33], smn[8][33];
    const int cx = threadIdx.x % 32, g = threadIdx.x / 32;
    const uint64_t c = (uint64_t)blockIdx.x * 32 + cx;
    double s = 0.0;
    T mx = -INFINITY, mn = INFINITY;
    if (c < cols) {
        uint64_t k = g;
        for (; k + 24 < chunks; k += 32) {
            double p[4];
            T a[4], b[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const uint64_t o = (k + 8 * u) * cols + c;
                p[u] = psum[o], a[u] = pmax[o], b[u] = pmin[o];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                s += p[u];
                mx = a[u] > mx ? a[u] : mx;
                mn = b[u] < mn ? b[u] : mn;
            }
        }
        for (; k < chunks; k += 8) {
            s += psum[k * cols + c];
            T a = pmax[k * cols + c], b = pmin[k * cols + c];
            mx = a > mx ? a : mx;
            mn = b < mn ? b : mn;
        }
    }
    ss[g][cx] = s, smx[g][cx] = mx, smn[g][cx] = mn;
    __syncthreads();
    if (g != 0 || c >= cols) return;
    for (int k = 1; k < 8; ++k) {
        s += ss[k][cx];
        mx = smx[k][cx] > mx ? smx[k][cx] : mx;
        mn = smn[k][cx] < mn ? smn[k][cx] : mn;
    }
    if (sum_out) sum_out[c] = (T)s;
    if (max_out) max_out[c] = mx;
    if (min_out) min_out[c] = mn;
}

template <class T>
int column_stats_t(synk_dev* d, const T* x, uint64_t rows, uint64_t cols, T* so, T* mxo, T* mno) {
    constexpr int N = Vec16<T>::N;
    static const bool force_scalar = getenv("SYNK_COLSTATS_SCALAR") != nullptr;  // diagnostics
    const bool vec = !force_scalar && cols % N == 0 && ((uintptr_t)x & 15) == 0;
    const uint64_t threads_per_row = vec ? cols / N : cols;
    // Narrow rows (vector path): one CTA step covers rpb whole rows.
    const uint32_t rpb = vec && threads_per_row < kBlock ? (uint32_t)(kBlock / threads_per_row) : 1;
    const uint64_t col_tiles = rpb > 1 ? 1 : (threads_per_row + kBlock - 1) / kBlock;
    // Enough row chunks for ~4 CTAs per SM, each chunk >= 16 rows per row group.
    uint64_t want = ((uint64_t)d->num_sms * 4 + col_tiles - 1) / col_tiles;
    uint64_t chunks = rows / (16 * rpb);
    if (chunks > want) chunks = want;
    if (chunks > 65535) chunks = 65535;
    if (chunks < 1) chunks = 1;
    uint64_t per = (rows + chunks - 1) / chunks;
    if (per == 0) per = 1;
    chunks = rows == 0 ? 1 : (rows + per - 1) / per;
    const uint64_t slots = chunks * rpb;
    size_t bytes = slots * cols * (sizeof(double) + 2 * sizeof(T));
    void* ws = nullptr;
    SYNK_CU(cudaMallocAsync(&ws, bytes, d->stream));
    double* psum = (double*)ws;
    T* pmax = (T*)(psum + slots * cols);
    T* pmin = pmax + slots * cols;
    dim3 grid((unsigned)col_tiles, (unsigned)chunks);
    if (vec) {
        colstats_partial_vec_kernel<T><<<grid, kBlock, 0, d->stream>>>(x, rows, cols, per, rpb, psum, pmax, pmin);
        SYNK_LAUNCHED("colstats_partial_vec_kernel");
    } else {
        colstats_partial_kernel<T><<<grid, kBlock, 0, d->stream>>>(x, rows, cols, per, psum, pmax, pmin);
        SYNK_LAUNCHED("colstats_partial_kernel");
    }
    colstats_final_kernel<T><<<(unsigned)((cols + 31) / 32), kBlock, 0, d->stream>>>(
        slots, cols, psum, pmax, pmin, so, mxo, mno);
    SYNK_LAUNCHED("colstats_final_kernel");
    SYNK_CU(cudaFreeAsync(ws, d->stream));
    return SYNK_OK;
}

// ---- compare / finiteness ---------------------------------------------------------

__global__ void __launch_bounds__(kBlock) neq16_kernel(const uint4* __restrict__ a,
                                                      const uint4* __restrict__ b, uint64_t n,
                                                      int* flag) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    int bad = 0;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) {
        uint4 x = a[i], y = b[i];
        bad |= (x.x != y.x) | (x.y != y.y) | (x.z != y.z) | (x.w != y.w);
    }
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}

__global__ void __launch_bounds__(kBlock) neq1_kernel(const uint8_t* __restrict__ a,
                                                     const uint8_t* __restrict__ b, uint64_t n,
                                                     int* flag) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    int bad = 0;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) bad |= a[i] != b[i];
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}

template <class T>
__global__ void __launch_bounds__(kBlock) nonfinite_kernel(const T* __restrict__ x, uint64_t n,
                                                          int* flag) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    int bad = 0;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) bad |= !isfinite(x[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}

template <class D, class S>
__global__ void __launch_bounds__(kBlock) cast_kernel(D* __restrict__ dst, const S* __restrict__ src, uint64_t n) {
    uint64_t tid = (uint64_t)blockIdx.x * kBlock + threadIdx.x;
    for (uint64_t i = tid; i < n; i += (uint64_t)gridDim.x * kBlock) dst[i] = (D)src[i];
}

int read_flag(synk_dev* d, int* out) {
    d->pdl_armed = false;
    SYNK_CU(cudaMemcpyAsync(d->flags_host + 1, d->flags_dev + 1, sizeof(int),
                            cudaMemcpyDeviceToHost, d->stream));
    SYNK_CU(cudaStreamSynchronize(d->stream));
    *out = d->flags_host[1];
    return SYNK_OK;
}

}  // namespace

extern "C" {

int synk_combine(synk_dev* d, int dtype, int op, void* acc, const void* other, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_combine: bad dtype");
    SYNK_REQUIRE(op == SYNK_OP_SUM || op == SYNK_OP_MAX || op == SYNK_OP_MIN || op == SYNK_OP_PROD,
                 SYNK_EARG, "combine_inplace(): op is not an elementwise combine");
    return run_map2(d, dtype, acc, other, n, CombineF{op});
}

int synk_weighted_mean(synk_dev* d, int dtype, void* acc, double wa, const void* other, double wb,
                       uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_weighted_mean: bad dtype");
    SYNK_REQUIRE(wa + wb != 0.0, SYNK_EARG, "weighted_mean_inplace(): both weights are zero");
    return run_map2(d, dtype, acc, other, n, WMeanF{wa, wb, 1.0 / (wa + wb)});
}

int synk_scale(synk_dev* d, int dtype, void* buf, double factor, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_scale: bad dtype");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    unsigned grid = synk::grid_for(d, n, kBlock);
    if (dtype == SYNK_F32) scale_kernel<float><<<grid, kBlock, 0, d->stream>>>((float*)buf, n, factor);
    else scale_kernel<double><<<grid, kBlock, 0, d->stream>>>((double*)buf, n, factor);
    SYNK_LAUNCHED("scale_kernel");
    return SYNK_OK;
}

}  // extern "C"

namespace {
// Small copies by the SMs (one CTA): into mapped pinned host memory the
// stores are posted PCIe writes, cheaper than a copy-engine round trip.
__global__ void copy_small_kernel(char* __restrict__ dst, const char* __restrict__ src, uint64_t bytes) {
    synk::wait_prerequisite_grid();  // launched as a follow-up (synk::launch_follow_up)
    const bool v16 = ((uintptr_t)dst | (uintptr_t)src | bytes) % 16 == 0;
    if (v16) {
        for (uint64_t i = threadIdx.x; i < bytes / 16; i += blockDim.x)
            reinterpret_cast<uint4*>(dst)[i] = reinterpret_cast<const uint4*>(src)[i];
    } else {
        for (uint64_t i = threadIdx.x; i < bytes; i += blockDim.x) dst[i] = src[i];
    }
}
}  // namespace

extern "C" {

int synk_copy_small(synk_dev* d, void* dst, const void* src, uint64_t bytes) {
    if (bytes == 0) return SYNK_OK;
    SYNK_REQUIRE(bytes <= (1u << 20), SYNK_EARG, "synk_copy_small: at most 1 MiB");
    synk::DeviceGuard g(d->device);
    if (int rc = synk::prefer_shared_carveout((const void*)copy_small_kernel, d->device); rc) return rc;
    SYNK_CU(synk::launch_follow_up(d, copy_small_kernel, 1, 256, (char*)dst, (const char*)src, bytes));
    SYNK_LAUNCHED("copy_small_kernel");
    return SYNK_OK;
}

int synk_fill(synk_dev* d, int dtype, void* dst, double value, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_fill: bad dtype");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    unsigned grid = synk::grid_for(d, n, kBlock);
    if (grid == 1) {  // small fill (a kernel's scalar result): a follow-up launch
        if (dtype == SYNK_F32) SYNK_CU(synk::launch_follow_up(d, fill_kernel<float>, 1, kBlock, (float*)dst, n, (float)value));
        else SYNK_CU(synk::launch_follow_up(d, fill_kernel<double>, 1, kBlock, (double*)dst, n, value));
    } else {
        d->pdl_armed = false;
        if (dtype == SYNK_F32) fill_kernel<float><<<grid, kBlock, 0, d->stream>>>((float*)dst, n, (float)value);
        else fill_kernel<double><<<grid, kBlock, 0, d->stream>>>((double*)dst, n, value);
    }
    SYNK_LAUNCHED("fill_kernel");
    return SYNK_OK;
}

int synk_fill_uniform(synk_dev* d, int dtype, void* dst, uint64_t n, uint64_t seed, uint64_t first) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_fill_uniform: bad dtype");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    if (dtype == SYNK_F32) {
        unsigned grid = synk::grid_for(d, (n + 3) / 4, kBlock);
        fill_uniform_kernel<float><<<grid, kBlock, 0, d->stream>>>((float*)dst, n, seed, first);
    } else {
        unsigned grid = synk::grid_for(d, n, kBlock);
        fill_uniform_kernel<double><<<grid, kBlock, 0, d->stream>>>((double*)dst, n, seed, first);
    }
    SYNK_LAUNCHED("fill_uniform_kernel");
    return SYNK_OK;
}

int synk_left_fold(synk_dev* d, int dtype, int op, void* out, const void* const* parts,
                   const uint64_t* weights, uint32_t count, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_left_fold: bad dtype");
    SYNK_REQUIRE(count >= 1, SYNK_EARG, "reduce over zero contributing shards (no neutral element)");
    SYNK_REQUIRE(op != SYNK_OP_GATHER && op >= 0 && op <= SYNK_OP_PROD, SYNK_EARG,
                 "synk_left_fold: gather is not a fold");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    unsigned grid = synk::grid_for(d, n, kBlock);
    uint32_t done = 0;
    double carried = 0.0;
    while (done < count) {
        FoldArgs args{};
        uint32_t k = 0;
        if (done > 0) {  // chain: the running accumulator is the first part
            args.parts[0] = out;
            args.weights[0] = carried;
            k = 1;
        }
        double wsum = done > 0 ? carried : 0.0;
        for (; k < kMaxParts && done < count; ++k, ++done) {
            args.parts[k] = parts[done];
            args.weights[k] = weights ? (double)weights[done] : 1.0;
            wsum += args.weights[k];
        }
        args.count = k;
        if (dtype == SYNK_F32)
            left_fold_kernel<float><<<grid, kBlock, 0, d->stream>>>(op, (float*)out, args, n);
        else
            left_fold_kernel<double><<<grid, kBlock, 0, d->stream>>>(op, (double*)out, args, n);
        SYNK_LAUNCHED("left_fold_kernel");
        carried = wsum;
    }
    return SYNK_OK;
}

int synk_column_stats(synk_dev* d, int dtype, const void* x, uint64_t rows, uint64_t cols,
                      void* sum_out, void* max_out, void* min_out) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_column_stats: bad dtype");
    if (cols == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    if (dtype == SYNK_F32)
        return column_stats_t<float>(d, (const float*)x, rows, cols, (float*)sum_out,
                                     (float*)max_out, (float*)min_out);
    return column_stats_t<double>(d, (const double*)x, rows, cols, (double*)sum_out,
                                  (double*)max_out, (double*)min_out);
}

int synk_cast(synk_dev* d, int dst_dtype, void* dst, int src_dtype, const void* src, uint64_t n) {
    SYNK_REQUIRE(synk::valid_dtype(dst_dtype) && synk::valid_dtype(src_dtype), SYNK_EDTYPE, "synk_cast: bad dtype");
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    if (dst_dtype == src_dtype) {
        d->pdl_armed = false;
        SYNK_CU(cudaMemcpyAsync(dst, src, n * synk::dtype_bytes(src_dtype), cudaMemcpyDefault, d->stream));
        return SYNK_OK;
    }
    unsigned grid = synk::grid_for(d, n, kBlock);
    if (dst_dtype == SYNK_F32)
        cast_kernel<float, double><<<grid, kBlock, 0, d->stream>>>((float*)dst, (const double*)src, n);
    else
        cast_kernel<double, float><<<grid, kBlock, 0, d->stream>>>((double*)dst, (const float*)src, n);
    SYNK_LAUNCHED("cast_kernel");
    return SYNK_OK;
}

int synk_equal(synk_dev* d, const void* a, const void* b, uint64_t bytes, int* equal) {
    *equal = 1;
    if (bytes == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    d->pdl_armed = false;
    SYNK_CU(cudaMemsetAsync(d->flags_dev + 1, 0, sizeof(int), d->stream));
    if (aligned16(a, b) && bytes % 16 == 0) {
        uint64_t n = bytes / 16;
        neq16_kernel<<<synk::grid_for(d, n, kBlock), kBlock, 0, d->stream>>>(
            (const uint4*)a, (const uint4*)b, n, d->flags_dev + 1);
    } else {
        neq1_kernel<<<synk::grid_for(d, bytes, kBlock), kBlock, 0, d->stream>>>(
            (const uint8_t*)a, (const uint8_t*)b, bytes, d->flags_dev + 1);
    }
    SYNK_LAUNCHED("neq_kernel");
    int mismatch = 0;
    if (int rc = read_flag(d, &mismatch); rc != SYNK_OK) return rc;
    *equal = mismatch == 0;
    return SYNK_OK;
}

int synk_all_finite(synk_dev* d, int dtype, const void* x, uint64_t n, int* finite) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "synk_all_finite: bad dtype");
    *finite = 1;
    if (n == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    d->pdl_armed = false;
    SYNK_CU(cudaMemsetAsync(d->flags_dev + 1, 0, sizeof(int), d->stream));
    unsigned grid = synk::grid_for(d, n, kBlock);
    if (dtype == SYNK_F32)
        nonfinite_kernel<float><<<grid, kBlock, 0, d->stream>>>((const float*)x, n, d->flags_dev + 1);
    else
        nonfinite_kernel<double><<<grid, kBlock, 0, d->stream>>>((const double*)x, n, d->flags_dev + 1);
    SYNK_LAUNCHED("nonfinite_kernel");
    int bad = 0;
    if (int rc = read_flag(d, &bad); rc != SYNK_OK) return rc;
    *finite = bad == 0;
    return SYNK_OK;
}

}  // extern "C"
