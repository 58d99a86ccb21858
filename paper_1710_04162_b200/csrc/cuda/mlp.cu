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
// This file holds the SIMT path (FFMA for f32, DFMA for f64 — the f64 path
// is what the reference's f64 trajectories are checked against at 1e-10).

#include <math.h>

#include "common.cuh"

namespace {

constexpr int BM = 64, BN = 64, BK = 16, kThreads = 256;

enum Epi { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_TANH = 2, EPI_TANH_GRAD = 3 };

// C[m,n] = epi( sum_k A(m,k) B(k,n) ), A(m,k) = A[m*am + k*ak], B(k,n) = B[k*bk + n*bn]
template <class T>
__global__ void __launch_bounds__(kThreads) gemm_simt_kernel(
    int epi, int64_t M, int64_t N, int64_t K, const T* __restrict__ A, int64_t am, int64_t ak,
    const T* __restrict__ B, int64_t bk, int64_t bn, T* __restrict__ C, int64_t ldc,
    const T* __restrict__ bias, const T* __restrict__ act) {
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

    for (int64_t k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            int idx = tid + i * kThreads;
            int kk, mm;
            if (ak == 1) { kk = idx % BK; mm = idx / BK; }   // K contiguous in memory
            else { mm = idx % BM; kk = idx / BM; }
            int64_t gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < K) ? A[gm * am + gk * ak] : T(0);
            int nn;
            if (bn == 1) { nn = idx % BN; kk = idx / BN; }   // N contiguous in memory
            else { kk = idx % BK; nn = idx / BK; }
            int64_t gn = n0 + nn;
            gk = k0 + kk;
            Bs[kk][nn] = (gn < N && gk < K) ? B[gk * bk + gn * bn] : T(0);
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

template <class T>
int gemm(synk_dev* d, int epi, int64_t M, int64_t N, int64_t K, const T* A, int64_t am, int64_t ak,
         const T* B, int64_t bk, int64_t bn, T* C, int64_t ldc, const T* bias, const T* act) {
    if (M == 0 || N == 0) return SYNK_OK;
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM));
    gemm_simt_kernel<T><<<grid, kThreads, 0, d->stream>>>(epi, M, N, K, A, am, ak, B, bk, bn, C, ldc,
                                                          bias, act);
    SYNK_LAUNCHED("gemm_simt_kernel");
    return SYNK_OK;
}

// delta = (pred - y) * inv_n ; per-CTA partial of sum (pred - y)^2 in f64.
template <class T>
__global__ void __launch_bounds__(kThreads) loss_delta_kernel(const T* __restrict__ pred,
                                                              const T* __restrict__ y, uint64_t n_el,
                                                              double inv_n, T* __restrict__ delta,
                                                              double* __restrict__ partial) {
    __shared__ double red[kThreads];
    double s = 0.0;
    for (uint64_t i = (uint64_t)blockIdx.x * kThreads + threadIdx.x; i < n_el;
         i += (uint64_t)gridDim.x * kThreads) {
        double diff = __dsub_rn((double)pred[i], (double)y[i]);
        s = __dadd_rn(s, __dmul_rn(diff, diff));
        delta[i] = (T)__dmul_rn(diff, inv_n);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] = red[threadIdx.x] + red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void loss_final_kernel(const double* __restrict__ partial, int count, double scale,
                                  double* __restrict__ loss) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int i = 0; i < count; ++i) s += partial[i];
        *loss = s * scale;  // mlp.cpp:190: loss *= 0.5 * inv_n
    }
}

// gb[j] = sum_i delta[i, j]  (f64 accumulation, deterministic row order per column block)
template <class T>
__global__ void __launch_bounds__(kThreads) bias_grad_kernel(const T* __restrict__ delta, uint64_t n,
                                                             uint64_t cols, T* __restrict__ gb) {
    // CTA = 32 columns x 8 row lanes; each row lane strides over rows, then a
    // fixed-order smem fold across the 8 lanes.
    __shared__ double red[8][33];
    int cx = threadIdx.x % 32, ry = threadIdx.x / 32;
    uint64_t c = (uint64_t)blockIdx.x * 32 + cx;
    double s = 0.0;
    if (c < cols)
        for (uint64_t r = ry; r < n; r += 8) s += (double)delta[r * cols + c];
    red[ry][cx] = s;
    __syncthreads();
    if (ry == 0 && c < cols) {
        double t = 0.0;
        for (int k = 0; k < 8; ++k) t += red[k][cx];
        gb[c] = (T)t;
    }
}

struct Plan {
    uint64_t woff[64], boff[64];
    uint64_t total = 0, maxd = 0, act_elems = 0;
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
    return SYNK_OK;
}

constexpr int kLossBlocks = 128;

uint64_t ws_bytes(int dtype, const Plan& p, uint64_t n) {
    uint64_t es = synk::dtype_bytes(dtype);
    uint64_t bytes = (p.act_elems + 2 * n * p.maxd) * es;
    bytes = (bytes + 255) / 256 * 256;
    return bytes + kLossBlocks * sizeof(double);
}

template <class T>
int loss_grad_t(synk_dev* d, const uint64_t* dims, uint32_t layers, const Plan& P, const T* theta,
                const T* x, const T* y, uint64_t n, double* loss, T* grad, void* ws) {
    // workspace: acts[1..L] | delta ping | delta pong | loss partials
    T* base = (T*)ws;
    T* acts[65];
    acts[0] = const_cast<T*>(x);
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

    for (uint32_t l = 0; l < layers; ++l) {
        int64_t din = dims[l], dout = dims[l + 1];
        int epi = (l + 1 < layers) ? EPI_BIAS_TANH : EPI_BIAS;
        if (int rc = gemm<T>(d, epi, n, dout, din, acts[l], din, 1, theta + P.woff[l], dout, 1,
                             acts[l + 1], dout, theta + P.boff[l], nullptr);
            rc != SYNK_OK)
            return rc;
    }
    uint64_t dl = dims[layers];
    uint64_t n_el = n * dl;
    int blocks = (int)((n_el + kThreads - 1) / kThreads);
    if (blocks > kLossBlocks) blocks = kLossBlocks;
    if (blocks < 1) blocks = 1;
    double inv_n = 1.0 / (double)n;
    loss_delta_kernel<T><<<blocks, kThreads, 0, d->stream>>>(acts[layers], y, n_el, inv_n, dA, partial);
    SYNK_LAUNCHED("loss_delta_kernel");
    loss_final_kernel<<<1, 32, 0, d->stream>>>(partial, blocks, 0.5 * inv_n, loss);
    SYNK_LAUNCHED("loss_final_kernel");

    T* delta = dA;
    T* spare = dB;
    for (uint32_t l = layers; l-- > 0;) {
        int64_t din = dims[l], dout = dims[l + 1];
        // gW = a_l^T delta : M=din, N=dout, K=n
        if (int rc = gemm<T>(d, EPI_STORE, din, dout, n, acts[l], 1, din, delta, dout, 1,
                             grad + P.woff[l], dout, nullptr, nullptr);
            rc != SYNK_OK)
            return rc;
        bias_grad_kernel<T><<<(unsigned)((dout + 31) / 32), kThreads, 0, d->stream>>>(
            delta, n, dout, grad + P.boff[l]);
        SYNK_LAUNCHED("bias_grad_kernel");
        if (l > 0) {
            // delta_prev = (delta W^T) * (1 - a_l^2) : M=n, N=din, K=dout
            if (int rc = gemm<T>(d, EPI_TANH_GRAD, n, din, dout, delta, dout, 1, theta + P.woff[l], 1,
                                 dout, spare, din, nullptr, acts[l]);
                rc != SYNK_OK)
                return rc;
            T* t = delta;
            delta = spare;
            spare = t;
        }
    }
    return SYNK_OK;
}

}  // namespace

extern "C" {

int synk_mlp_workspace_bytes(int dtype, const uint64_t* dims, uint32_t layers, uint64_t n,
                             uint64_t* bytes) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "mlp: bad dtype");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    *bytes = ws_bytes(dtype, p, n);
    return SYNK_OK;
}

int synk_mlp_loss_grad(synk_dev* d, int dtype, const uint64_t* dims, uint32_t layers,
                       const void* params, const void* x, const void* y, uint64_t n,
                       double* loss_dev, void* grad, void* workspace, uint64_t workspace_bytes) {
    SYNK_REQUIRE(synk::valid_dtype(dtype), SYNK_EDTYPE, "mlp: bad dtype");
    SYNK_REQUIRE(n > 0, SYNK_EARG, "mlp_loss_grad: empty batch");
    Plan p;
    if (int rc = make_plan(dims, layers, n, &p); rc != SYNK_OK) return rc;
    SYNK_REQUIRE(workspace_bytes >= ws_bytes(dtype, p, n), SYNK_EARG, "mlp: workspace too small");
    synk::DeviceGuard g(d->device);
    if (dtype == SYNK_F32)
        return loss_grad_t<float>(d, dims, layers, p, (const float*)params, (const float*)x,
                                  (const float*)y, n, loss_dev, (float*)grad, workspace);
    return loss_grad_t<double>(d, dims, layers, p, (const double*)params, (const double*)x,
                               (const double*)y, n, loss_dev, (double*)grad, workspace);
}

}  // extern "C"
