// Example function of the paper: tanh MLP loss + gradient (mlp.cpp:134-218).
//
// Forward  z_l = a_l W_l + b_l, a_{l+1} = tanh(z_l) (hidden) | z_L (output)
// Loss     0.5/n sum (pred - y)^2 (f64), delta = (pred - y)/n
// Backward gW_l = a_l^T delta, gb_l = colsum(delta),
//          delta <- (delta W_l^T) * (1 - a_l^2)
//
// Each dense product is one tiled GEMM launch with the elementwise work fused
// into its epilogue (bias+tanh, bias, tanh-derivative); the loss/delta pass
// and the bias-gradient column sums are deterministic block reductions.
// Paths: f32 parameters run every product on the tensor cores at fp32
// accuracy (3xTF32, gemm_f32x3.cu: loss_grad_f32tc below, the default);
// f64 runs the SIMT DFMA products (what the reference's f64 trajectories are
// checked against at 1e-10), and the same SIMT kernel in f32 (FFMA) is kept
// as the A/B baseline (SYNK_MLP_F32=ffma); the wide bf16 MLP (config C5)
// runs loss_grad_bf16 on gemm_tc.cu.

#include <cstdio>
#include <cuda_bf16.h>
#include <math.h>

#include <algorithm>
#include <stdlib.h>
#include <string>
#include <vector>

#include "common.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 16, kThreads = 256;

enum Epi { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_TANH = 2, EPI_TANH_GRAD = 3 };

// C[m,n] = epi( sum_k A(m,k) B(k,n) ), A(m,k) = A[m*am + k*ak], B(k,n) = B[k*bk + n*bn]
// Row `ones_row` of A (if < M) reads as 1: the weight-gradient product over
// M = d_l + 1 rows then also yields the bias gradient (colsum of delta) in
// its last row, which lands on b_l right after W_l in the flat layout.
// Split-K (gridDim.z > 1): CTA z sums k in [z*kper, (z+1)*kper) and stores the
// raw partial to C + z*M*N (ldc = N); splitk_reduce_kernel folds the partials.
template <class T>
__global__ void __launch_bounds__(kThreads) gemm_simt_kernel(
    int epi, int64_t M, int64_t N, int64_t K, const T* __restrict__ A, int64_t am, int64_t ak,
    const T* __restrict__ B, int64_t bk, int64_t bn, T* __restrict__ C, int64_t ldc,
    const T* __restrict__ bias, const T* __restrict__ act, int64_t kper, int64_t ones_row) {
    __shared__ T As[BK][BM + 1];
    __shared__ T Bs[BK][BN + 1];
    const int tid = threadIdx.x;
    const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
    const int tm = (tid / 16) * 4, tn = (tid % 16) * 4;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = T(0);

    const int64_t kbeg = (int64_t)blockIdx.z * kper;
    const int64_t kend = kbeg + kper < K ? kbeg + kper : K;
    if (gridDim.z > 1) {
        C += (int64_t)blockIdx.z * M * N;
        epi = -1;  // raw partial
    }
    for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int idx = tid + i * kThreads;
            int kk, mm;
            if (ak == 1) { kk = idx % BK; mm = idx / BK; }   // K contiguous in memory
            else { mm = idx % BM; kk = idx / BM; }
            int64_t gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < kend) ? (gm == ones_row ? T(1) : A[gm * am + gk * ak]) : T(0);
            int nn;
            if (bn == 1) { nn = idx % BN; kk = idx / BN; }   // N contiguous in memory
            else { kk = idx % BK; nn = idx / BK; }
            int64_t gn = n0 + nn;
            gk = k0 + kk;
            Bs[kk][nn] = (gn < N && gk < kend) ? B[gk * bk + gn * bn] : T(0);
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            T a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][tm + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tn + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] += a[i] * b[j];
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        int64_t gm = m0 + tm + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            int64_t gn = n0 + tn + j;
            if (gn >= N) continue;
            T v = acc[i][j];
            if (epi == EPI_BIAS) v = v + bias[gn];
            else if (epi == EPI_BIAS_TANH) v = tanh(v + bias[gn]);
            else if (epi == EPI_TANH_GRAD) {
                T a = act[gm * ldc + gn];
                v = v * (T(1) - a * a);
            }
            C[gm * ldc + gn] = v;
        }
    }
}

// Fixed (device-independent, so results do not depend on the SM count) split
// of K for f32 products with too few output tiles to fill the GPU: ~3 CTAs per
// SM of a 148-SM B200, at least 32 k per split. f64 stays unsplit (its
// trajectories are held to 1e-10 against the reference's sequential sums).
// 3 CTAs of 256 threads per SM fit at 80 registers: one full wave (measured
// on C1: 444 -> 127 us/step, 296 -> 131, 592 -> 133, 888 -> 134).
constexpr int64_t kSplitTargetCtas = 444;

inline int64_t split_k(int es, int64_t M, int64_t N, int64_t K, int64_t* kper) {
    const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    int64_t s = 1;
    if (es == 4 && tiles * 2 < kSplitTargetCtas) {
        s = kSplitTargetCtas / tiles;
        if (s > K / 32) s = K / 32;
        if (s > 32) s = 32;
        if (s < 1) s = 1;
    }
    int64_t per = (K + s - 1) / s;
    per = (per + BK - 1) / BK * BK;
    if (per < BK) per = BK;
    *kper = per;
    return K == 0 ? 1 : (K + per - 1) / per;
}

// C = epi(sum_z P[z]) in fixed z order (f64 accumulation of the f32 partials).
template <class T>
__global__ void __launch_bounds__(kThreads) splitk_reduce_kernel(
    int epi, int64_t S, int64_t M, int64_t N, const T* __restrict__ P, T* __restrict__ C, int64_t ldc,
    const T* __restrict__ bias, const T* __restrict__ act) {
    const int64_t total = M * N;
    for (int64_t i = (int64_t)blockIdx.x * kThreads + threadIdx.x; i < total; i += (int64_t)gridDim.x * kThreads) {
        double acc = 0.0;
        for (int64_t z = 0; z < S; ++z) acc += (double)P[z * total + i];
        const int64_t gm = i / N, gn = i % N;
        T v = (T)acc;
        if (epi == EPI_BIAS) v = v + bias[gn];
        else if (epi == EPI_BIAS_TANH) v = tanh(v + bias[gn]);
        else if (epi == EPI_TANH_GRAD) {
            T a = act[gm * ldc + gn];
            v = v * (T(1) - a * a);
        }
        C[gm * ldc + gn] = v;
    }
}

template <class T>
int gemm(synk_dev* d, int epi, int64_t M, int64_t N, int64_t K, const T* A, int64_t am, int64_t ak,
         const T* B, int64_t bk, int64_t bn, T* C, int64_t ldc, const T* bias, const T* act, T* partials,
         int64_t ones_row = -1) {
    if (M == 0 || N == 0) return SYNK_OK;
    int64_t kper = 0;
    const int64_t S = split_k(sizeof(T), M, N, K, &kper);
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)S);
    if (S == 1) {
        gemm_simt_kernel<T><<<grid, kThreads, 0, d->stream>>>(epi, M, N, K, A, am, ak, B, bk, bn, C, ldc, bias,
                                                              act, K > 0 ? K : 1, ones_row);
        SYNK_LAUNCHED("gemm_simt_kernel");
        return SYNK_OK;
    }
    SYNK_REQUIRE(partials != nullptr, SYNK_EARG, "mlp gemm: split-K needs a partials workspace");
    gemm_simt_kernel<T><<<grid, kThreads, 0, d->stream>>>(epi, M, N, K, A, am, ak, B, bk, bn, partials, N,
                                                          nullptr, nullptr, kper, ones_row);
    SYNK_LAUNCHED("gemm_simt_kernel");
    unsigned rgrid = (unsigned)std::min<int64_t>((M * N + kThreads - 1) / kThreads, 148 * 4);
    splitk_reduce_kernel<T><<<rgrid, kThreads, 0, d->stream>>>(epi, S, M, N, partials, C, ldc, bias, act);
    SYNK_LAUNCHED("splitk_reduce_kernel");
    return SYNK_OK;
}

// Largest split-K partial buffer (elements) over the products of one loss/grad pass.
uint64_t splitk_elems(int es, const uint64_t* dims, uint32_t layers, uint64_t n) {
    uint64_t best = 0;
    auto see = [&](int64_t M, int64_t N, int64_t K) {
        int64_t kper;
        int64_t S = split_k(es, M, N, K, &kper);
        if (S > 1 && (uint64_t)(S * M * N) > best) best = (uint64_t)(S * M * N);
    };
    for (uint32_t l = 0; l < layers; ++l) {
        see((int64_t)n, (int64_t)dims[l + 1], (int64_t)dims[l]);
        see((int64_t)dims[l] + 1, (int64_t)dims[l + 1], (int64_t)n);
        if (l > 0) see((int64_t)n, (int64_t)dims[l], (int64_t)dims[l + 1]);
    }
    return best;
}

// tf32 hi/lo split of delta, row-major (hi/lo, ld_o; may be null) and
// transposed (hi_t/lo_t, ld_t): written by the loss kernel for the f32
// tensor-core path (gemm_f32x3.cu operands).
struct DeltaSplit {
    float* hi = nullptr;
    float* lo = nullptr;
    uint64_t ld_o = 0;
    float* hi_t = nullptr;
    float* lo_t = nullptr;
    uint64_t ld_t = 0;
};

// delta = (pred - y) * inv_n ; per-CTA partial of sum (pred - y)^2 in f64.
// With `counter`, the last CTA to finish also folds the per-CTA partials in a
// fixed order (thread t sums partials t, t+256, ..., then a fixed shared-memory
// tree) and writes the loss: one launch, deterministic.
template <class T>
__global__ void __launch_bounds__(kThreads) loss_delta_kernel(const T* __restrict__ pred,
                                                              const T* __restrict__ y, uint64_t n_el,
                                                              double inv_n, T* __restrict__ delta,
                                                              double* __restrict__ partial,
                                                              unsigned* __restrict__ counter = nullptr,
                                                              double scale = 0.0, double* __restrict__ loss = nullptr,
                                                              const uint64_t* __restrict__ yrows = nullptr,
                                                              uint64_t ycols = 1, DeltaSplit ds = {}) {
    __shared__ double red[kThreads];
    __shared__ int last;
    synk::release_dependent_grid();  // PDL: the backward product behind it may be scheduled
    synk::wait_prerequisite_grid();  // launched as a follow-up of the last forward product
    double s = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n_el;
         i += (uint64_t)gridDim.x * kThreads) {
        const uint64_t yi = yrows ? __ldg(yrows + i / ycols) * ycols + i % ycols : i;  // index-fused y
        double diff = __dsub_rn((double)pred[i], (double)y[yi]);
        s = __dadd_rn(s, __dmul_rn(diff, diff));
        delta[i] = (T)__dmul_rn(diff, inv_n);
        if constexpr (sizeof(T) == 4) {
            if (ds.hi_t) {  // the f32 tensor-core path's operand forms of delta
                const float v = (float)__dmul_rn(diff, inv_n);
                uint32_t h, l;
                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
                asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(l) : "f"(v - __uint_as_float(h)));
                const uint64_t m = i / ycols, c = i % ycols;
                ds.hi_t[c * ds.ld_t + m] = __uint_as_float(h), ds.lo_t[c * ds.ld_t + m] = __uint_as_float(l);
                if (ds.hi) ds.hi[m * ds.ld_o + c] = __uint_as_float(h), ds.lo[m * ds.ld_o + c] = __uint_as_float(l);
            }
        }
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
    if (!counter) return;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += kThreads) t += __ldcg(&partial[i]);
    red[threadIdx.x] = t;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *loss = red[0] * scale;  // mlp.cpp:190: loss *= 0.5 * inv_n
        *counter = 0;
    }
}

struct Plan {
    uint64_t woff[64], boff[64];
    uint64_t total = 0, maxd = 0, act_elems = 0, splitk = 0, in_dim = 0;
};

int make_plan(const uint64_t* dims, uint32_t layers, uint64_t n, Plan* p) {
    SYNK_REQUIRE(layers >= 1 && layers <= 64, SYNK_EARG, "mlp: layers must be in 1..64");
    uint64_t at = 0;
    p->maxd = 0;
    p->act_elems = 0;
    for (uint32_t l = 0; l < layers; ++l) {
        SYNK_REQUIRE(dims[l] > 0 && dims[l + 1] > 0, SYNK_EARG, "mlp: dimensions must be positive");
        p->woff[l] = at;
        at += dims[l] * dims[l + 1];
        p->boff[l] = at;
        at += dims[l + 1];
        p->act_elems += n * dims[l + 1];
    }
    for (uint32_t l = 0; l <= layers; ++l) p->maxd = dims[l] > p->maxd ? dims[l] : p->maxd;
    p->total = at;
    p->in_dim = dims[0];
    p->splitk = splitk_elems(4, dims, layers, n);  // f32 only; f64 products are not split
    return SYNK_OK;
}

constexpr int kLossBlocks = 592;  // 4 CTAs per SM of a B200

// workspace: acts[1..L] | delta ping | delta pong | loss partials | split-K partials | gathered x
uint64_t xg_offset(uint64_t es, const Plan& p, uint64_t n) {
    uint64_t bytes = (p.act_elems + 2 * n * p.maxd) * es;
    bytes = (bytes + 255) / 256 * 256;
    bytes += kLossBlocks * sizeof(double) + (es == 4 ? p.splitk * es : 0);
    return (bytes + 255) / 256 * 256;
}

uint64_t ws_bytes(int dtype, const Plan& p, uint64_t n) {
    const uint64_t es = synk::dtype_bytes(dtype);
    return xg_offset(es, p, n) + n * p.in_dim * es;
}

template <class T>
int loss_grad_t(synk_dev* d, const uint64_t* dims, uint32_t layers, const Plan& P, const T* theta,
                const T* x, const T* y, uint64_t n, double* loss, T* grad, void* ws,
                const uint64_t* rows = nullptr) {
    // workspace: acts[1..L] | delta ping | delta pong | loss partials | split-K | gathered x
    T* base = (T*)ws;
    T* acts[65];
    acts[0] = const_cast<T*>(x);
    if (rows) {
        // Index-fused inputs: x and y are the whole sources and row i of the
        // batch is source row rows[i] (valid: the caller checked the list).
        // x is gathered into the workspace by the first launch of the sequence
        // (inside the CUDA graph), y is read through the list by the loss kernel.
        T* xg = (T*)((char*)ws + xg_offset(sizeof(T), P, n));
        if (int rc = synk_gather_rows(d, x, ~0ull, dims[0] * sizeof(T), rows, n, xg); rc) return rc;
        acts[0] = xg;
    }
    T* cur = base;
    for (uint32_t l = 1; l <= layers; ++l) {
        acts[l] = cur;
        cur += n * dims[l];
    }
    T* dA = cur;
    T* dB = dA + n * P.maxd;
    uint64_t es = sizeof(T);
    uint64_t off = ((P.act_elems + 2 * n * P.maxd) * es + 255) / 256 * 256;
    double* partial = (double*)((char*)ws + off);
    T* skp = (T*)(partial + kLossBlocks);

    for (uint32_t l = 0; l < layers; ++l) {
        int64_t din = dims[l], dout = dims[l + 1];
        int epi = (l + 1 < layers) ? EPI_BIAS_TANH : EPI_BIAS;
        if (int rc = gemm<T>(d, epi, n, dout, din, acts[l], din, 1, theta + P.woff[l], dout, 1,
                             acts[l + 1], dout, theta + P.boff[l], nullptr, skp);
            rc != SYNK_OK)
            return rc;
    }
    uint64_t dl = dims[layers];
    uint64_t n_el = n * dl;
    int blocks = (int)((n_el + kThreads - 1) / kThreads);
    if (blocks > kLossBlocks) blocks = kLossBlocks;
    if (blocks < 1) blocks = 1;
    double inv_n = 1.0 / (double)n;
    SYNK_CU(synk::launch_follow_up(d, loss_delta_kernel<T>, (unsigned)blocks, kThreads, acts[layers], y, n_el, inv_n,
                                   dA, partial, reinterpret_cast<unsigned*>(d->flags_dev + 3), 0.5 * inv_n, loss, rows,
                                   dims[layers], DeltaSplit{}));
    SYNK_LAUNCHED("loss_delta_kernel");
    d->pdl_armed = true;

    T* delta = dA;
    T* spare = dB;
    for (uint32_t l = layers; l-- > 0;) {
        int64_t din = dims[l], dout = dims[l + 1];
        // [gW; gb] = [a_l^T; 1] delta : M=din+1 (row din of A reads as ones), N=dout, K=n;
        // row din is the bias gradient and lands on b_l (= grad + woff + din*dout)
        if (int rc = gemm<T>(d, EPI_STORE, din + 1, dout, n, acts[l], 1, din, delta, dout, 1,
                             grad + P.woff[l], dout, nullptr, nullptr, skp, din);
            rc != SYNK_OK)
            return rc;
        if (l > 0) {
            // delta_prev = (delta W^T) * (1 - a_l^2) : M=n, N=din, K=dout
            if (int rc = gemm<T>(d, EPI_TANH_GRAD, n, din, dout, delta, dout, 1, theta + P.woff[l], 1,
                                 dout, spare, din, nullptr, acts[l], skp);
                rc != SYNK_OK)
                return rc;
            T* t = delta;
            delta = spare;
            spare = t;
        }
    }
    return SYNK_OK;
}

// ---- f32 tensor-core path (config C1: fp32 accuracy on tcgen05, 3xTF32) ---------------
// Every product is one synk_gemm_f32x3 launch (gemm_f32x3.cu): operands are
// K-major tf32 hi/lo pairs, and each producer emits its result directly in the
// form its consumers read, so the only separate staging launches are the
// input batch (gathered through the index list in the same pass), the weights
// and the loss delta:
//   forward   a_{l+1} = tanh(a_l . W_l + b_l): A = a_l split, B = W_l^T split;
//             the epilogue writes a_{l+1} (f32, for tanh'), its split and
//             its transposed split (the weight gradient's A)
//   gradient  [gW_l; gb_l] = [a_l^T; 1] . delta: A = a_l^T split whose extra
//             row is the constant 1.0 (hi) / 0 (lo), B = delta^T split
//   dX        delta_prev = (delta . W_l^T) * (1 - a_l^2): A = delta split,
//             B = W_l split; the epilogue writes delta_prev's split and
//             transposed split
// Same layer algebra and loss/delta kernel as loss_grad_t (mlp.cpp:134-218).

inline uint64_t pad4(uint64_t v) { return (v + 3) / 4 * 4; }

struct TcPlan {
    uint64_t n, L;
    uint64_t act[65];             // f32 a_l (l = 1..L), n x d_l; a_L = prediction
    uint64_t ah[64], al[64];      // a_l split, n x pad4(d_l)          (l = 0..L-1)
    uint64_t ath[64], atl[64];    // a_l^T split, (d_l + 1) x pad4(n)  (row d_l = ones)
    uint64_t wth[64], wtl[64];    // W_l^T split, d_{l+1} x pad4(d_l)
    uint64_t wh[64], wl[64];      // W_l split, d_l x pad4(d_{l+1})      (l >= 1)
    uint64_t dh[2], dl[2];        // delta split ping-pong, n x pad4(maxd)
    uint64_t dth[2], dtl[2];      // delta^T split ping-pong, maxd x pad4(n)
    uint64_t delta, partial, total;
};

TcPlan make_tc_plan(const uint64_t* dims, uint32_t L, uint64_t n, uint64_t maxd) {
    TcPlan p{};
    p.n = n;
    p.L = L;
    uint64_t at = 0;
    auto take = [&](uint64_t bytes) {
        const uint64_t o = at;
        at += (bytes + 255) / 256 * 256;
        return o;
    };
    for (uint32_t l = 1; l <= L; ++l) p.act[l] = take(n * dims[l] * 4);
    for (uint32_t l = 0; l < L; ++l) {
        p.ah[l] = take(n * pad4(dims[l]) * 4);
        p.al[l] = take(n * pad4(dims[l]) * 4);
        p.ath[l] = take((dims[l] + 1) * pad4(n) * 4);
        p.atl[l] = take((dims[l] + 1) * pad4(n) * 4);
        p.wth[l] = take(dims[l + 1] * pad4(dims[l]) * 4);
        p.wtl[l] = take(dims[l + 1] * pad4(dims[l]) * 4);
        if (l >= 1) {
            p.wh[l] = take(dims[l] * pad4(dims[l + 1]) * 4);
            p.wl[l] = take(dims[l] * pad4(dims[l + 1]) * 4);
        }
    }
    for (int b = 0; b < 2; ++b) {
        p.dh[b] = take(n * pad4(maxd) * 4);
        p.dl[b] = take(n * pad4(maxd) * 4);
        p.dth[b] = take(maxd * pad4(n) * 4);
        p.dtl[b] = take(maxd * pad4(n) * 4);
    }
    p.delta = take(n * dims[L] * 4);
    p.partial = take(kLossBlocks * sizeof(double));
    p.total = at;
    return p;
}

int loss_grad_f32tc(synk_dev* d, const uint64_t* dims, uint32_t L, const Plan& P, const float* theta, const float* x,
                    const float* y, uint64_t n, double* loss, float* grad, void* ws, const uint64_t* rows) {
    const TcPlan T = make_tc_plan(dims, L, n, P.maxd);
    char* base = static_cast<char*>(ws);
    auto F = [&](uint64_t off) { return reinterpret_cast<float*>(base + off); };
    const uint64_t pn = pad4(n);

    // one staging launch: the constant ones row under every a_l^T (bias
    // gradient through the GEMM), the input batch (index-fused: row i is
    // source row rows[i]) -> a_0 split + a_0^T split, and the weights: W_l^T
    // split (forward B) and, below the first layer, W_l split (dX B)
    synk_tf32_rows ones{};
    for (uint32_t l = 0; l < L; ++l) {
        ones.hi[l] = F(T.ath[l]) + dims[l] * pn;
        ones.lo[l] = F(T.atl[l]) + dims[l] * pn;
        ones.len[l] = n;
    }
    ones.count = L;
    ones.value = 1.0f;
    std::vector<synk_tf32_job> jobs;
    jobs.push_back({x, rows, n, dims[0], dims[0], F(T.ah[0]), F(T.al[0]), pad4(dims[0]), F(T.ath[0]), F(T.atl[0]), pn});
    for (uint32_t l = 0; l < L; ++l) {
        const bool rows_too = l >= 1;
        jobs.push_back({theta + P.woff[l], nullptr, dims[l], dims[l + 1], dims[l + 1], rows_too ? F(T.wh[l]) : nullptr,
                        rows_too ? F(T.wl[l]) : nullptr, pad4(dims[l + 1]), F(T.wth[l]), F(T.wtl[l]), pad4(dims[l])});
    }
    for (size_t at = 0; at < jobs.size(); at += SYNK_TF32_MAX_JOBS) {
        const uint32_t cnt = (uint32_t)std::min<size_t>(SYNK_TF32_MAX_JOBS, jobs.size() - at);
        if (int rc = synk_tf32_stage(d, jobs.data() + at, cnt, at == 0 ? &ones : nullptr); rc) return rc;
    }
    for (uint32_t l = 0; l < L; ++l) {
        const bool hidden = l + 1 < L;
        if (int rc = synk_gemm_f32x3(d, n, dims[l + 1], dims[l], F(T.ah[l]), F(T.al[l]), pad4(dims[l]), F(T.wth[l]),
                                     F(T.wtl[l]), pad4(dims[l]), hidden ? SYNK_EPI_BIAS_TANH : SYNK_EPI_BIAS,
                                     F(T.act[l + 1]), dims[l + 1], theta + P.boff[l], nullptr, 0,
                                     hidden ? F(T.ah[l + 1]) : nullptr, hidden ? F(T.al[l + 1]) : nullptr,
                                     pad4(dims[l + 1]), hidden ? F(T.ath[l + 1]) : nullptr,
                                     hidden ? F(T.atl[l + 1]) : nullptr, pn);
            rc)
            return rc;
    }
    const uint64_t n_el = n * dims[L];
    const int blocks = (int)std::min<uint64_t>(kLossBlocks, std::max<uint64_t>(1, (n_el + kThreads - 1) / kThreads));
    const double inv_n = 1.0 / (double)n;
    SYNK_CU(synk::launch_follow_up(d, loss_delta_kernel<float>, (unsigned)blocks, kThreads, F(T.act[L]), y, n_el, inv_n,
                                   F(T.delta), reinterpret_cast<double*>(base + T.partial),
                                   reinterpret_cast<unsigned*>(d->flags_dev + 3), 0.5 * inv_n, loss, rows, dims[L],
                                   DeltaSplit{L >= 2 ? F(T.dh[0]) : nullptr, L >= 2 ? F(T.dl[0]) : nullptr,
                                              pad4(dims[L]), F(T.dth[0]), F(T.dtl[0]), pn}));
    d->pdl_armed = true;
    SYNK_LAUNCHED("loss_delta_kernel");
    int cur = 0;
    for (uint32_t l = L; l-- > 0;) {
        // [gW_l; gb_l]: M = d_l + 1 (row d_l of a_l^T is ones), lands on b_l after W_l
        if (int rc = synk_gemm_f32x3(d, dims[l] + 1, dims[l + 1], n, F(T.ath[l]), F(T.atl[l]), pn, F(T.dth[cur]),
                                     F(T.dtl[cur]), pn, SYNK_EPI_STORE, grad + P.woff[l], dims[l + 1], nullptr, nullptr,
                                     0, nullptr, nullptr, 0, nullptr, nullptr, 0);
            rc)
            return rc;
        if (l == 0) break;
        const int nxt = cur ^ 1;
        const bool rows_next = l - 1 >= 1;  // delta_prev feeds another dX product
        if (int rc = synk_gemm_f32x3(d, n, dims[l], dims[l + 1], F(T.dh[cur]), F(T.dl[cur]), pad4(dims[l + 1]),
                                     F(T.wh[l]), F(T.wl[l]), pad4(dims[l + 1]), SYNK_EPI_TANH_GRAD, nullptr, 0, nullptr,
                                     F(T.act[l]), dims[l], rows_next ? F(T.dh[nxt]) : nullptr,
                                     rows_next ? F(T.dl[nxt]) : nullptr, pad4(dims[l]), F(T.dth[nxt]), F(T.dtl[nxt]),
                                     pn);
            rc)
            return rc;
        cur = nxt;
    }
    return SYNK_OK;
}

// f32 products on the tensor cores unless SYNK_MLP_F32=ffma (A/B runs).
bool f32_on_tensor_cores(int compute) {
    if (compute == SYNK_MLP_F32_TC) return true;
    const char* e = getenv("SYNK_MLP_F32");  // read per call: tests flip it between runs
    return !(e && std::string(e) == "ffma");
}

// Workspace of the native-precision path: the f32 tensor-core plan or the
// FFMA/DFMA plan.
uint64_t native_ws(int dtype, int compute, const uint64_t* dims, uint32_t L, const Plan& p, uint64_t n) {
    if (dtype == SYNK_F32 && f32_on_tensor_cores(compute)) return make_tc_plan(dims, L, n, p.maxd).total;
    return ws_bytes(dtype, p, n);
}

// ---- bf16 tensor-core path (config C5: wide MLP, fp32 master weights) -----------------
// Every dense product is one synk_gemm_tc2 (tcgen05 kind::f16) launch. Operand
// layouts follow what the tensor cores read at full speed (measured,
// profiles/r01_gemm_layouts.txt): B may be MN-major for free on the 128x256
// persistent path (N > 128), while an MN-major A costs 10-20 % and an MN-major
// B on the narrow (N <= 128) path ~30 %. Hence:
//   forward   a_{l+1} = tanh(a_l . W_l + b_l): A = a_l (K-major); B = W_l as it
//             lies (MN-major) when d_{l+1} > 128, else W_l^T (a small cast +
//             transpose); the epilogue stores a_{l+1} and a_{l+1}^T;
//   gradient  [gW_l; gb_l] = [a_l^T; 1] . delta: A = a_l^T (K-major, its extra
//             row of ones yields the bias gradient); B = delta MN-major when
//             d_{l+1} > 128, else delta^T (emitted by the producer of delta);
//   dX        delta_prev = (delta . W_l^T) * (1 - a_l^2): A = delta, B = W_l,
//             both K-major as they lie.
// So the only transposes are a_l^T (epilogue stores; x^T by the cast) and
// the narrow output layer's W^T / delta^T.

inline uint64_t pad8(uint64_t v) { return (v + 7) / 8 * 8; }

constexpr uint64_t kWideN = 128;  // N > kWideN: persistent path, MN-major B at full speed

// Row `row` of each a_l^T buffer = 1.0 (bf16), so the weight-gradient GEMM
// over M = d_l + 1 rows also yields sum_i delta[i, :] = the bias gradient,
// landing on b_l right after W_l in the flat parameter layout.
struct OnesRows {
    __nv_bfloat16* p[64];
    uint32_t count;
};
__global__ void __launch_bounds__(256) ones_rows_kernel(OnesRows rows, uint64_t n) {
    const __nv_bfloat16 one = __float2bfloat16_rn(1.0f);
    for (uint32_t l = blockIdx.y; l < rows.count; l += gridDim.y)
        for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256)
            rows.p[l][i] = one;
}

// Loss + output delta for the bf16 path in one launch, tiled 32 rows x 64
// columns per CTA: diff = pred - y (f64, y read through the index list when
// index-fused), loss partial sum (f64; the last CTA folds the per-CTA
// partials in a fixed order), delta = (float)(diff * inv_n) written straight
// in its bf16 operand forms -- row-major (ld) and, for a narrow output layer,
// transposed through a shared-memory tile (ldt) -- so neither the f32 delta
// nor the separate cast + transpose launch exists. Same per-element rounding
// as loss_delta_kernel + the cast (f64 -> f32 -> bf16).
constexpr int kLossTileR = 32, kLossTileC = 64;
__global__ void __launch_bounds__(256) loss_delta_bf16_kernel(const float* __restrict__ pred, const float* __restrict__ y,
                                                              uint64_t n, uint64_t cols, double inv_n,
                                                              __nv_bfloat16* __restrict__ d, uint64_t ld,
                                                              __nv_bfloat16* __restrict__ dt, uint64_t ldt,
                                                              double* __restrict__ partial, unsigned* __restrict__ counter,
                                                              double scale, double* __restrict__ loss,
                                                              const uint64_t* __restrict__ yrows) {
    __shared__ __nv_bfloat16 tile[kLossTileC][kLossTileR + 2];
    __shared__ double red[256];
    __shared__ int last;
    // PDL: launched programmatically after the forward GEMM (waits for it
    // before any global access) and releases the backward GEMM behind it.
    synk::release_dependent_grid();
    synk::wait_prerequisite_grid();
    const uint64_t r0 = (uint64_t)blockIdx.y * kLossTileR, c0 = (uint64_t)blockIdx.x * kLossTileC;
    const int tc = threadIdx.x % kLossTileC, tr = threadIdx.x / kLossTileC;  // 64 x 4
    double s = 0.0;
#pragma unroll
    for (int k = tr; k < kLossTileR; k += 4) {
        const uint64_t r = r0 + k, c = c0 + tc;
        __nv_bfloat16 h = __float2bfloat16_rn(0.f);
        if (r < n && c < cols) {
            const uint64_t yr = yrows ? __ldg(yrows + r) : r;
            const double diff = __dsub_rn((double)pred[r * cols + c], (double)y[yr * cols + c]);
            s = __dadd_rn(s, __dmul_rn(diff, diff));
            h = __float2bfloat16_rn((float)__dmul_rn(diff, inv_n));
            d[r * ld + c] = h;
        }
        tile[tc][k] = h;
    }
    red[threadIdx.x] = s;
    __syncthreads();
    if (dt) {  // transposed: thread -> (column c0 + t / 4, rows r0 + (t % 4) * 8 .. + 8)
        const int oc = threadIdx.x / 4, seg = (threadIdx.x % 4) * 8;
        const uint64_t c = c0 + oc;
        if (c < cols) {
            if (r0 + seg + 8 <= n) {  // 8 consecutive rows = one 16-byte store (ldt is a multiple of 8)
                __align__(16) __nv_bfloat16 h[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) h[j] = tile[oc][seg + j];
                *reinterpret_cast<uint4*>(dt + c * ldt + r0 + seg) = *reinterpret_cast<const uint4*>(h);
            } else {
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if (r0 + seg + j < n) dt[c * ldt + r0 + seg + j] = tile[oc][seg + j];
            }
        }
    }
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + w];
        __syncthreads();
    }
    const unsigned nb = gridDim.x * gridDim.y, b = blockIdx.y * gridDim.x + blockIdx.x;
    if (threadIdx.x == 0) partial[b] = red[0];
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == nb - 1;
    __syncthreads();
    if (!last) return;
    __threadfence();
    double t = 0.0;
    for (unsigned i = threadIdx.x; i < nb; i += 256) t += __ldcg(&partial[i]);
    red[threadIdx.x] = t;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        *loss = red[0] * scale;  // mlp.cpp:190: loss *= 0.5 * inv_n
        *counter = 0;
    }
}

struct Bf16Plan {
    uint64_t n, maxd, L;
    uint64_t off_w[64], off_wt[64], off_act[65], off_actT[65];
    // off_d[k] (k = 1..L): delta at layer k-1's output, n x pad8(d_k) bf16;
    // off_dT[k]: its transpose, for narrow layers (d_k <= kWideN) only
    uint64_t off_pred, off_delta_f, off_d[65], off_dT[65], off_partial, total;
};

Bf16Plan make_bf16_plan(const uint64_t* dims, uint32_t L, uint64_t n, uint64_t maxd) {
    Bf16Plan p{};
    p.n = n;
    p.maxd = maxd;
    p.L = L;
    uint64_t at = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t o = at;
        at += (bytes + 255) / 256 * 256;
        return o;
    };
    for (uint32_t l = 0; l < L; ++l) {
        p.off_w[l] = take(dims[l] * pad8(dims[l + 1]) * 2);
        if (dims[l + 1] <= kWideN) p.off_wt[l] = take(dims[l + 1] * pad8(dims[l]) * 2);
    }
    for (uint32_t l = 0; l < L; ++l) {  // act[0] = x, act[l] hidden
        p.off_act[l] = take(n * pad8(dims[l]) * 2);
        p.off_actT[l] = take((dims[l] + 1) * pad8(n) * 2);  // + a row of ones (bias gradient)
    }
    p.off_pred = take(n * dims[L] * 4);
    p.off_delta_f = take(n * dims[L] * 4);
    for (uint32_t k = 1; k <= L; ++k) {  // every delta stays live: all dX products run before the weight gradients
        p.off_d[k] = take(n * pad8(dims[k]) * 2);
        if (dims[k] <= kWideN) p.off_dT[k] = take(dims[k] * pad8(n) * 2);
    }
    p.off_partial = take(kLossBlocks * 8 * sizeof(double));  // loss tiles (loss_delta_bf16_kernel)
    p.total = at;
    return p;
}

// bf16 weight shadow layout (synk_cuda.h): W_l with leading dim pad8(d_{l+1})
// and, for narrow layers, W_l^T with leading dim pad8(d_l) -- exactly the
// operand buffers the products read.
int bf16_shadow_layout(const uint64_t* dims, uint32_t L, const Plan& P, synk_bf16_shadow* out) {
    SYNK_REQUIRE(L <= SYNK_SHADOW_MAX_SEGS, SYNK_EARG, "mlp: bf16 shadow supports up to 8 layers");
    *out = synk_bf16_shadow{};
    uint64_t at = 0;
    auto take = [&](uint64_t bytes) {
        uint64_t o = at;
        at += (bytes + 255) / 256 * 256;
        return o;
    };
    out->count = L;
    for (uint32_t l = 0; l < L; ++l) {
        synk_bf16_shadow_seg& g = out->seg[l];
        g.first = P.woff[l];
        g.rows = dims[l];
        g.cols = dims[l + 1];
        g.ldw = pad8(dims[l + 1]);
        g.off_w = take(dims[l] * g.ldw * 2);
        g.ldwt = pad8(dims[l]);
        g.off_wt = dims[l + 1] <= kWideN ? take(dims[l + 1] * g.ldwt * 2) : SYNK_NO_TRANSPOSE;
    }
    out->bytes = at;
    return SYNK_OK;
}

int loss_grad_bf16(synk_dev* d, const uint64_t* dims, uint32_t L, const Plan& P, const float* theta, const float* x,
                   const float* y, uint64_t n, double* loss, float* grad, void* ws, int signal_base = -1,
                   const uint64_t* rows = nullptr, const synk_mlp_opts* opts = nullptr) {
    Bf16Plan B = make_bf16_plan(dims, L, n, P.maxd);
    char* base = static_cast<char*>(ws);
    auto bf = [&](uint64_t off) { return reinterpret_cast<__nv_bfloat16*>(base + off); };
    const int F32 = SYNK_F32, BF = SYNK_BF16;
    auto wide = [&](uint32_t l) { return dims[l + 1] > kWideN; };  // output width of layer l

    // weights: W_l in bf16 (+ W_l^T for narrow layers), one read each -- into
    // the rank's persistent shadow when given (skipped when it is current:
    // the fused update of the previous step wrote it with the new params)
    synk_bf16_shadow sh{};
    char* shb = opts && opts->shadow ? static_cast<char*>(opts->shadow) : nullptr;
    if (shb)
        if (int rc = bf16_shadow_layout(dims, L, P, &sh); rc) return rc;
    auto wbuf = [&](uint32_t l) { return shb ? reinterpret_cast<__nv_bfloat16*>(shb + sh.seg[l].off_w) : bf(B.off_w[l]); };
    auto wtbuf = [&](uint32_t l) {
        return shb ? reinterpret_cast<__nv_bfloat16*>(shb + sh.seg[l].off_wt) : bf(B.off_wt[l]);
    };
    if (!shb || !opts->shadow_valid)
        for (uint32_t l = 0; l < L; ++l) {
            const float* W = theta + P.woff[l];
            if (int rc = synk_gemm_prep2_bf16(d, W, dims[l], dims[l + 1], dims[l + 1], wbuf(l), pad8(dims[l + 1]),
                                              wide(l) ? nullptr : wtbuf(l), pad8(dims[l]));
                rc)
                return rc;
        }
    // index-fused rows: staged into HBM by the executor (possibly still in
    // flight on its copy stream), and/or readable in place in pinned host memory
    bool rows_waited = !(opts && opts->rows_ready_on);
    auto wait_rows = [&]() -> int {
        if (rows_waited) return SYNK_OK;
        rows_waited = true;
        return synk_wait_peer_slot(d, opts->rows_ready_on, opts->rows_ready_slot);
    };
    // the constant ones rows of every a_l^T first: they do not need the index
    // list, so they run while its stage copy is still in flight
    {
        OnesRows o{};
        o.count = L;
        for (uint32_t l = 0; l < L; ++l) o.p[l] = bf(B.off_actT[l]) + dims[l] * pad8(n);
        if (int rc = synk::prefer_shared_carveout((const void*)ones_rows_kernel, d->device); rc) return rc;
        if (int rc = synk::prefer_shared_carveout((const void*)loss_delta_kernel<float>, d->device); rc) return rc;
        ones_rows_kernel<<<dim3((unsigned)std::min<uint64_t>((n + 255) / 256, 64), L), 256, 0, d->stream>>>(o, n);
        SYNK_LAUNCHED("ones_rows_kernel");
    }
    // The x staging reads the HBM copy of the list: read in place over PCIe
    // (rows_host) every 64x64 tile re-fetched its 64 indices at PCIe latency,
    // 121 us instead of 27 us for the C5 batch (profiles/r02_c5_trace.txt),
    // far more than the 7.5 us stage copy it would hide.
    const uint64_t* xrows = rows;
    if (rows)
        if (int rc = wait_rows(); rc) return rc;
    // input batch: x and x^T in bf16 (rows != null: gathered from the whole source in the same pass)
    if (int rc = synk_gemm_prep2_bf16_rows(d, x, xrows, n, dims[0], dims[0], bf(B.off_act[0]), pad8(dims[0]),
                                           bf(B.off_actT[0]), pad8(n));
        rc)
        return rc;

    // forward
    float* pred = reinterpret_cast<float*>(base + B.off_pred);
    for (uint32_t l = 0; l < L; ++l) {
        const bool hidden = l + 1 < L;
        const void* b = wide(l) ? (const void*)wbuf(l) : (const void*)wtbuf(l);
        const uint64_t ldb = wide(l) ? pad8(dims[l + 1]) : pad8(dims[l]);
        int rc = synk_gemm_tc2(d, SYNK_GEMM_BF16, n, dims[l + 1], dims[l], bf(B.off_act[l]), nullptr, pad8(dims[l]), b,
                               nullptr, ldb, wide(l) ? SYNK_GEMM_B_MN : 0, hidden ? SYNK_EPI_BIAS_TANH : SYNK_EPI_BIAS,
                               hidden ? BF : F32, hidden ? (void*)bf(B.off_act[l + 1]) : (void*)pred,
                               hidden ? pad8(dims[l + 1]) : dims[L], hidden ? (void*)bf(B.off_actT[l + 1]) : nullptr,
                               pad8(n), theta + P.boff[l], nullptr, 0);
        if (rc) return rc;
    }

    // loss + output delta (f32), then its bf16 operand form(s)
    const uint64_t dl = dims[L], n_el = n * dl;
    double* partial = reinterpret_cast<double*>(base + B.off_partial);
    const double inv_n = 1.0 / (double)n;
    if (rows)
        if (int rc = wait_rows(); rc) return rc;  // the loss reads y through the staged list
    auto narrow = [&](uint32_t k) { return dims[k] <= kWideN; };  // delta_k also needed transposed
    {
        const dim3 grid((unsigned)((dl + kLossTileC - 1) / kLossTileC), (unsigned)((n + kLossTileR - 1) / kLossTileR));
        SYNK_REQUIRE((uint64_t)grid.x * grid.y <= kLossBlocks * 8, SYNK_EARG, "mlp: loss tile grid too large");
        if (int rc = synk::prefer_shared_carveout((const void*)loss_delta_bf16_kernel, d->device); rc) return rc;
        SYNK_CU(synk::launch_follow_up_2d(
            d, loss_delta_bf16_kernel, grid, 256, pred, y, n, dl, inv_n, bf(B.off_d[L]), pad8(dims[L]),
            narrow(L) ? bf(B.off_dT[L]) : nullptr, pad8(n), partial, reinterpret_cast<unsigned*>(d->flags_dev + 3),
            0.5 * inv_n, loss, rows));
        SYNK_LAUNCHED("loss_delta_bf16_kernel");
        d->pdl_armed = true;
    }

    // backward: every dX product first (they read the bf16 W_l, which no
    // update of this step touches), then the weight gradients, largest
    // segment first: each segment's all-reduce + update (the trainer's second
    // stream) then overlaps the remaining weight-gradient products and only
    // the smallest one's is exposed at the end of the step (C5: the 8.4M-
    // parameter W_0 update used to trail the last GEMM).
    for (uint32_t l = L - 1; l >= 1; --l) {
        // delta_l = (delta_{l+1} . W_l^T) * (1 - a_l^2)  (M = n, N = d_l, K = d_{l+1})
        if (int rc = synk_gemm_tc2(d, SYNK_GEMM_BF16, n, dims[l], dims[l + 1], bf(B.off_d[l + 1]), nullptr,
                                   pad8(dims[l + 1]), wbuf(l), nullptr, pad8(dims[l + 1]), 0, SYNK_EPI_TANH_GRAD, BF,
                                   bf(B.off_d[l]), pad8(dims[l]), narrow(l) ? (void*)bf(B.off_dT[l]) : nullptr,
                                   pad8(n), nullptr, bf(B.off_act[l]), pad8(dims[l]));
            rc)
            return rc;
    }
    uint32_t order[64];
    for (uint32_t i = 0; i < L; ++i) order[i] = L - 1 - i;
    std::stable_sort(order, order + L, [&](uint32_t a, uint32_t b) {
        return dims[a] * dims[a + 1] > dims[b] * dims[b + 1];
    });
    for (uint32_t i = 0; i < L; ++i) {
        const uint32_t l = order[i];
        const uint64_t din = dims[l], dout = dims[l + 1];
        // [gW_l; gb_l] = [a_l^T; 1] . delta_{l+1}  (M = din + 1: the last row is the bias gradient)
        const void* b = wide(l) ? (const void*)bf(B.off_d[l + 1]) : (const void*)bf(B.off_dT[l + 1]);
        if (int rc = synk_gemm_tc2(d, SYNK_GEMM_BF16, din + 1, dout, n, bf(B.off_actT[l]), nullptr, pad8(n), b,
                                   nullptr, wide(l) ? pad8(dout) : pad8(n), wide(l) ? SYNK_GEMM_B_MN : 0,
                                   SYNK_EPI_STORE, F32, grad + P.woff[l], dout, nullptr, 0, nullptr, nullptr, 0);
            rc)
            return rc;
        // Segment [W_l, b_l] of the gradient is final and W_l is not read again
        // (every dX ran above): the trainer may all-reduce + update it now.
        if (signal_base >= 0)
            if (int rc = synk_signal_slot(d, signal_base + (int)l); rc) return rc;
        if (opts && opts->seg_order) opts->seg_order[i] = (int)l;
    }
    return SYNK_OK;
}

// ---- CUDA-graph replay of the loss/grad launch sequence ------------------------------
// A latency-bound step (config C1: ~12 launches of a few us each) spends as
// much time in launch overhead as in kernels. The sequence for one set of
// (shapes, pointers) is captured once into a CUDA graph and replayed with a
// single launch; in a training loop the stream-ordered pool hands the same
// batch/gradient buffers back every step, so replays hit. A rank whose
// pointers keep changing (misses in a row) stops capturing.
// SYNK_MLP_GRAPHS=0 disables (A/B diagnostics).

struct GraphKey {
    int dtype;
    uint32_t layers;
    uint64_t dims[65];
    uint64_t n;
    const void* ptrs[7];
    bool operator==(const GraphKey& o) const {
        if (dtype != o.dtype || layers != o.layers || n != o.n) return false;
        for (uint32_t l = 0; l <= layers && l < 65; ++l)
            if (dims[l] != o.dims[l]) return false;
        for (int i = 0; i < 7; ++i)
            if (ptrs[i] != o.ptrs[i]) return false;
        return true;
    }
};

struct GraphCache {
    struct Entry {
        GraphKey key;
        cudaGraphExec_t exec;
        uint64_t used;
    };
    std::vector<Entry> entries;
    uint64_t clock = 0;
    int misses_in_a_row = 0;
    bool disabled = false;
    static constexpr size_t kMax = 8;
    static constexpr int kGiveUp = 16;
};

template <class F>
int graph_launch(synk_dev* d, const GraphKey& key, F&& launch_all) {
    static const bool enabled = [] {
        const char* e = getenv("SYNK_MLP_GRAPHS");
        return !(e && e[0] == '0');
    }();
    if (!enabled) return launch_all();
    if (!d->graphs) d->graphs = new GraphCache();
    GraphCache& gc = *static_cast<GraphCache*>(d->graphs);
    if (gc.disabled) return launch_all();
    for (auto& e : gc.entries)
        if (e.key == key) {
            e.used = ++gc.clock;
            gc.misses_in_a_row = 0;
            SYNK_CU(cudaGraphLaunch(e.exec, d->stream));
            d->pdl_armed = false;  // a graph is not a kernel that released its dependents
            return SYNK_OK;
        }
    if (++gc.misses_in_a_row > GraphCache::kGiveUp) {
        gc.disabled = true;
        return launch_all();
    }
    static const bool debug = [] {
        const char* e = getenv("SYNK_DEBUG_GRAPHS");  // diagnostics: report every capture
        return e && e[0] == '1';
    }();
    if (debug)
        fprintf(stderr, "[synk] mlp graph capture rank %d (%zu cached, miss %d): p=%p x=%p y=%p loss=%p g=%p ws=%p rows=%p\n",
                d->rank, gc.entries.size(), gc.misses_in_a_row, key.ptrs[0], key.ptrs[1], key.ptrs[2], key.ptrs[3],
                key.ptrs[4], key.ptrs[5], key.ptrs[6]);
    cudaGraph_t graph = nullptr;
    d->pdl_armed = false;  // no programmatic edge onto work outside the graph
    SYNK_CU(cudaStreamBeginCapture(d->stream, cudaStreamCaptureModeThreadLocal));
    const int rc = launch_all();
    const cudaError_t ec = cudaStreamEndCapture(d->stream, &graph);
    if (rc != SYNK_OK) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (ec != cudaSuccess) return synk::cuda_fail(ec, "cudaStreamEndCapture (mlp loss/grad)");
    cudaGraphExec_t exec = nullptr;
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (ei != cudaSuccess) return synk::cuda_fail(ei, "cudaGraphInstantiate (mlp loss/grad)");
    // Upload the executable graph now: replays then only submit it (the first
    // launch would otherwise carry the upload).
    SYNK_CU(cudaGraphUpload(exec, d->stream));
    if (gc.entries.size() == GraphCache::kMax) {
        auto lru = std::min_element(gc.entries.begin(), gc.entries.end(),
                                    [](const GraphCache::Entry& a, const GraphCache::Entry& b) { return a.used < b.used; });
        cudaGraphExecDestroy(lru->exec);
        gc.entries.erase(lru);
    }
    gc.entries.push_back({key, exec, ++gc.clock});
    SYNK_CU(cudaGraphLaunch(exec, d->stream));
    d->pdl_armed = false;
    return SYNK_OK;
}

}  // namespace

namespace synk {
void release_graphs(synk_dev* d) {
    if (!d->graphs) return;
    auto* gc = static_cast<GraphCache*>(d->graphs);
    for (auto& e : gc->entries) cudaGraphExecDestroy(e.exec);
    delete gc;
    d->graphs = nullptr;
}
}  // namespace synk

namespace {

// Native (FFMA/DFMA) loss/grad, the whole launch sequence replayed from a CUDA
// graph; rows != null: index-fused x/y (see loss_grad_t).
int native_loss_grad(synk_dev* d, int dtype, const uint64_t* dims, uint32_t layers, const void* params, const void* x,
                     const void* y, uint64_t n, double* loss_dev, void* grad, void* workspace,
                     uint64_t workspace_bytes, const uint64_t* rows, int compute = SYNK_MLP_NATIVE);

}  // namespace

extern "C" {

int synk_mlp_workspace_bytes_ex(int dtype, int compute, const uint64_t* dims, uint32_t layers, uint64_t n,
                                uint64_t* bytes) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "mlp: bad dtype");
    SYNK_REQUIRE(compute == SYNK_MLP_NATIVE || (compute == SYNK_MLP_BF16_TC && dtype == SYNK_F32) ||
                     (compute == SYNK_MLP_F32_TC && dtype == SYNK_F32),
                 SYNK_EARG, "mlp: tensor-core compute modes need f32 parameters");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    *bytes = compute == SYNK_MLP_BF16_TC ? make_bf16_plan(dims, layers, n, p.maxd).total
                                         : native_ws(dtype, compute, dims, layers, p, n);
    return SYNK_OK;
}

int synk_mlp_loss_grad_ex(synk_dev* d, int dtype, int compute, const uint64_t* dims, uint32_t layers,
                          const void* params, const void* x, const void* y, uint64_t n, double* loss_dev, void* grad,
                          void* workspace, uint64_t workspace_bytes) {
    if (compute == SYNK_MLP_NATIVE || compute == SYNK_MLP_F32_TC) {
        SYNK_REQUIRE(compute == SYNK_MLP_NATIVE || dtype == SYNK_F32, SYNK_EARG,
                     "mlp: f32 tensor-core compute needs f32 parameters");
        return native_loss_grad(d, dtype, dims, layers, params, x, y, n, loss_dev, grad, workspace, workspace_bytes,
                                nullptr, compute);
    }
    SYNK_REQUIRE(compute == SYNK_MLP_BF16_TC && dtype == SYNK_F32, SYNK_EARG,
                 "mlp: bf16 tensor-core compute needs f32 parameters");
    SYNK_REQUIRE(n > 0, SYNK_EARG, "mlp_loss_grad: empty batch");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    SYNK_REQUIRE(workspace_bytes >= make_bf16_plan(dims, layers, n, p.maxd).total, SYNK_EARG,
                 "mlp: workspace too small");
    synk::DeviceGuard g(d->device);
    return loss_grad_bf16(d, dims, layers, p, (const float*)params, (const float*)x, (const float*)y, n, loss_dev,
                          (float*)grad, workspace);
}

int synk_mlp_loss_grad_seg(synk_dev* d, int dtype, int compute, const uint64_t* dims, uint32_t layers,
                           const void* params, const void* x, const void* y, uint64_t n, double* loss_dev, void* grad,
                           void* workspace, uint64_t workspace_bytes, int signal_base, int* signalled,
                           const uint64_t* rows) {
    *signalled = 0;
    if (compute != SYNK_MLP_BF16_TC) {
        SYNK_REQUIRE(compute == SYNK_MLP_NATIVE || (compute == SYNK_MLP_F32_TC && dtype == SYNK_F32), SYNK_EARG,
                     "mlp: unknown compute mode");
        return native_loss_grad(d, dtype, dims, layers, params, x, y, n, loss_dev, grad, workspace, workspace_bytes,
                                rows, compute);
    }
    SYNK_REQUIRE(dtype == SYNK_F32, SYNK_EARG, "mlp: bf16 tensor-core compute needs f32 parameters");
    SYNK_REQUIRE(n > 0, SYNK_EARG, "mlp_loss_grad: empty batch");
    SYNK_REQUIRE(signal_base < 0 || signal_base + (int)layers <= 64, SYNK_EARG,
                 "mlp_loss_grad_seg: signal slots out of range");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    SYNK_REQUIRE(workspace_bytes >= make_bf16_plan(dims, layers, n, p.maxd).total, SYNK_EARG,
                 "mlp: workspace too small");
    synk::DeviceGuard g(d->device);
    const int rc = loss_grad_bf16(d, dims, layers, p, (const float*)params, (const float*)x, (const float*)y, n,
                                  loss_dev, (float*)grad, workspace, signal_base, rows);
    if (rc == SYNK_OK && signal_base >= 0) *signalled = (int)layers;
    return rc;
}

int synk_mlp_bf16_shadow(const uint64_t* dims, uint32_t layers, synk_bf16_shadow* out) {
    Plan p;
    if (int rc = make_plan(dims, layers, 1, &p); rc != SYNK_OK) return rc;
    return bf16_shadow_layout(dims, layers, p, out);
}

int synk_mlp_loss_grad_opts(synk_dev* d, int dtype, int compute, const uint64_t* dims, uint32_t layers,
                            const void* params, const void* x, const void* y, uint64_t n, double* loss_dev,
                            void* grad, void* workspace, uint64_t workspace_bytes, const synk_mlp_opts* opts,
                            int* signalled) {
    *signalled = 0;
    synk_mlp_opts none{};
    none.signal_base = -1;
    const synk_mlp_opts& o = opts ? *opts : none;
    if (compute != SYNK_MLP_BF16_TC) {
        SYNK_REQUIRE(compute == SYNK_MLP_NATIVE || (compute == SYNK_MLP_F32_TC && dtype == SYNK_F32), SYNK_EARG,
                     "mlp: unknown compute mode");
        if (o.rows && o.rows_ready_on)  // the whole native sequence is one graph: wait up front
            if (int rc = synk_wait_peer_slot(d, o.rows_ready_on, o.rows_ready_slot); rc) return rc;
        return native_loss_grad(d, dtype, dims, layers, params, x, y, n, loss_dev, grad, workspace, workspace_bytes,
                                o.rows, compute);
    }
    SYNK_REQUIRE(dtype == SYNK_F32, SYNK_EARG, "mlp: bf16 tensor-core compute needs f32 parameters");
    SYNK_REQUIRE(n > 0, SYNK_EARG, "mlp_loss_grad: empty batch");
    SYNK_REQUIRE(o.signal_base < 0 || o.signal_base + (int)layers <= 64, SYNK_EARG,
                 "mlp_loss_grad_seg: signal slots out of range");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    SYNK_REQUIRE(workspace_bytes >= make_bf16_plan(dims, layers, n, p.maxd).total, SYNK_EARG,
                 "mlp: workspace too small");
    synk::DeviceGuard g(d->device);
    const int rc = loss_grad_bf16(d, dims, layers, p, (const float*)params, (const float*)x, (const float*)y, n,
                                  loss_dev, (float*)grad, workspace, o.signal_base, o.rows, &o);
    if (rc == SYNK_OK && o.signal_base >= 0) *signalled = (int)layers;
    return rc;
}

int synk_mlp_workspace_bytes(int dtype, const uint64_t* dims, uint32_t layers, uint64_t n,
                             uint64_t* bytes) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "mlp: bad dtype");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    *bytes = native_ws(dtype, SYNK_MLP_NATIVE, dims, layers, p, n);
    return SYNK_OK;
}

int synk_mlp_loss_grad(synk_dev* d, int dtype, const uint64_t* dims, uint32_t layers,
                       const void* params, const void* x, const void* y, uint64_t n,
                       double* loss_dev, void* grad, void* workspace, uint64_t workspace_bytes) {
    return native_loss_grad(d, dtype, dims, layers, params, x, y, n, loss_dev, grad, workspace, workspace_bytes,
                            nullptr);
}

}  // extern "C"

namespace {

int native_loss_grad(synk_dev* d, int dtype, const uint64_t* dims, uint32_t layers, const void* params, const void* x,
                     const void* y, uint64_t n, double* loss_dev, void* grad, void* workspace,
                     uint64_t workspace_bytes, const uint64_t* rows, int compute) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "mlp: bad dtype");
    SYNK_REQUIRE(n > 0, SYNK_EARG, "mlp_loss_grad: empty batch");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    const bool tc = dtype == SYNK_F32 && f32_on_tensor_cores(compute);
    SYNK_REQUIRE(workspace_bytes >= native_ws(dtype, compute, dims, layers, p, n), SYNK_EARG,
                 "mlp: workspace too small");
    synk::DeviceGuard g(d->device);
    auto launch_all = [&]() {
        if (tc)
            return loss_grad_f32tc(d, dims, layers, p, (const float*)params, (const float*)x, (const float*)y, n,
                                   loss_dev, (float*)grad, workspace, rows);
        if (dtype == SYNK_F32)
            return loss_grad_t<float>(d, dims, layers, p, (const float*)params, (const float*)x,
                                      (const float*)y, n, loss_dev, (float*)grad, workspace, rows);
        return loss_grad_t<double>(d, dims, layers, p, (const double*)params, (const double*)x,
                                   (const double*)y, n, loss_dev, (double*)grad, workspace, rows);
    };
    GraphKey key{};
    key.dtype = dtype | (tc ? 0x100 : 0);
    key.layers = layers;
    for (uint32_t l = 0; l <= layers && l < 65; ++l) key.dims[l] = dims[l];
    key.n = n;
    key.ptrs[0] = params, key.ptrs[1] = x, key.ptrs[2] = y, key.ptrs[3] = loss_dev, key.ptrs[4] = grad;
    key.ptrs[5] = workspace, key.ptrs[6] = rows;
    return graph_launch(d, key, launch_all);
}

}  // namespace
