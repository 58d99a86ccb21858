/*
 * synk_oracle.c — CPU restatement of the synkpar hot path (see synk_oracle.h).
 * TEST INFRASTRUCTURE ONLY: the parity checker, never the product.
 * Compiled with -ffp-contract=off so every a*b+c rounds twice, as the
 * reference's g++ -O2/-O3 x86-64 build does (no FMA contraction).
 */
#include "synk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define F32 1
#define F64 2

enum { OP_SUM = 0, OP_MEAN = 1, OP_MAX = 2, OP_MIN = 3, OP_PROD = 4, OP_GATHER = 5 };

static size_t esize(int dtype) { return dtype == F32 ? 4 : 8; }

static double ld(int dtype, const void* p, uint64_t i) {
    return dtype == F32 ? (double)((const float*)p)[i] : ((const double*)p)[i];
}
static void st(int dtype, void* p, uint64_t i, double v) {
    if (dtype == F32) ((float*)p)[i] = (float)v;
    else ((double*)p)[i] = v;
}

/* tensor.cpp:315-327 */
void so_partition_rows(uint64_t n_rows, uint64_t n_parts, uint64_t* starts, uint64_t* stops) {
    uint64_t base = n_rows / n_parts, extra = n_rows % n_parts, at = 0;
    for (uint64_t i = 0; i < n_parts; ++i) {
        uint64_t len = base + (i < extra ? 1 : 0);
        starts[i] = at;
        stops[i] = at + len;
        at += len;
    }
}

/* tensor.cpp:200-217 (zero-filled destination, per-row bound check, memcpy) */
int so_gather_rows(const void* src, uint64_t src_rows, uint64_t row_bytes, const uint64_t* idx,
                   uint64_t n_idx, void* dst) {
    memset(dst, 0, (size_t)(n_idx * row_bytes));
    for (uint64_t j = 0; j < n_idx; ++j) {
        if (idx[j] >= src_rows) return -1;
        memcpy((char*)dst + j * row_bytes, (const char*)src + idx[j] * row_bytes, (size_t)row_bytes);
    }
    return 0;
}

/* tensor.cpp:250-270: the fold happens in T itself (zip_inplace<T>), no f64 promotion. */
#define COMBINE_LOOP(T)                                                        \
    do {                                                                       \
        T* a = (T*)acc;                                                        \
        const T* b = (const T*)other;                                          \
        switch (op) {                                                          \
        case OP_SUM: for (uint64_t i = 0; i < n; ++i) a[i] = a[i] + b[i]; break; \
        case OP_MAX: for (uint64_t i = 0; i < n; ++i) a[i] = b[i] > a[i] ? b[i] : a[i]; break; \
        case OP_MIN: for (uint64_t i = 0; i < n; ++i) a[i] = b[i] < a[i] ? b[i] : a[i]; break; \
        case OP_PROD: for (uint64_t i = 0; i < n; ++i) a[i] = a[i] * b[i]; break; \
        default: return -1;                                                    \
        }                                                                      \
    } while (0)

int so_combine(int dtype, int op, void* acc, const void* other, uint64_t n) {
    if (dtype == F32) COMBINE_LOOP(float);
    else COMBINE_LOOP(double);
    return 0;
}

/* tensor.cpp:272-285 */
int so_weighted_mean(int dtype, void* acc, double wa, const void* other, double wb, uint64_t n) {
    if (wa + wb == 0.0) return -1;
    double inv = 1.0 / (wa + wb);
    for (uint64_t i = 0; i < n; ++i) {
        double v = (ld(dtype, acc, i) * wa + ld(dtype, other, i) * wb) * inv;
        st(dtype, acc, i, v);
    }
    return 0;
}

/* tensor.cpp:367-373 (f64: v *= factor; f32: float(v * factor)) */
void so_scale(int dtype, void* buf, double factor, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) st(dtype, buf, i, ld(dtype, buf, i) * factor);
}

/* Synthetic-data stream (no reference counterpart; the reference generates
 * its bench/acceptance datasets on the host with libstdc++ RNGs,
 * bench.cpp:41-58): value i = (splitmix64(seed + i*golden) >> 40) * 2^-23 - 1,
 * exact in f32 and f64. Mirrors synk_fill_uniform. */
static uint64_t splitmix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

void so_fill_uniform(int dtype, void* dst, uint64_t n, uint64_t seed, uint64_t first) {
    for (uint64_t i = 0; i < n; ++i) {
        uint64_t k = splitmix64(seed + (first + i) * 0x9E3779B97F4A7C15ull) >> 40;
        st(dtype, dst, i, (double)k * 0x1p-23 - 1.0);
    }
}

/* replicated.cpp:16-29 */
int so_tree_fold(int dtype, int op, const void* const* parts, uint64_t world, uint64_t n,
                 void* out) {
    if (op == OP_GATHER || world == 0) return -1;
    size_t bytes = (size_t)(n * esize(dtype));
    char* acc = (char*)malloc(bytes * world + 1);
    if (!acc) return -2;
    for (uint64_t r = 0; r < world; ++r) memcpy(acc + r * bytes, parts[r], bytes);
    int fold_op = op == OP_MEAN ? OP_SUM : op;
    for (uint64_t step = 1; step < world; step *= 2)
        for (uint64_t r = 0; r + step < world; r += 2 * step)
            so_combine(dtype, fold_op, acc + r * bytes, acc + (r + step) * bytes, n);
    if (op == OP_MEAN) so_scale(dtype, acc, 1.0 / (double)world, n);
    memcpy(out, acc, bytes);
    free(acc);
    return 0;
}

/* function.cpp:76-101 (OutputAccumulator::add) applied in contribution order,
 * as the slice loop (:450-463) and the master fold (:515-527) do. */
int so_left_fold(int dtype, int op, const void* const* parts, const uint64_t* weights,
                 uint64_t count, uint64_t n, void* out) {
    if (count == 0 || op == OP_GATHER) return -1;
    memcpy(out, parts[0], (size_t)(n * esize(dtype)));
    uint64_t w = weights ? weights[0] : 1;
    for (uint64_t i = 1; i < count; ++i) {
        uint64_t wi = weights ? weights[i] : 1;
        if (op == OP_MEAN) {
            if (so_weighted_mean(dtype, out, (double)w, parts[i], (double)wi, n) != 0) return -1;
            w += wi;
        } else if (so_combine(dtype, op, out, parts[i], n) != 0) {
            return -1;
        }
    }
    return 0;
}

/* sgd.cpp:46-51 */
void so_sgd(int dtype, void* p, const void* g, double lr, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) st(dtype, p, i, ld(dtype, p, i) - lr * ld(dtype, g, i));
}

/* sgd.cpp:53-61 (Nesterov form) */
void so_momentum(int dtype, void* p, void* v, const void* g, double mu, double lr, uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) {
        double gi = ld(dtype, g, i);
        double vn = mu * ld(dtype, v, i) - lr * gi;
        st(dtype, v, i, vn);
        st(dtype, p, i, ld(dtype, p, i) + mu * vn - lr * gi);
    }
}

/* sgd.cpp:63-72 */
void so_rmsprop(int dtype, void* p, void* a, const void* g, double rho, double eps, double lr,
                uint64_t n) {
    for (uint64_t i = 0; i < n; ++i) {
        double gi = ld(dtype, g, i);
        double an = rho * ld(dtype, a, i) + (1.0 - rho) * gi * gi;
        st(dtype, a, i, an);
        st(dtype, p, i, ld(dtype, p, i) - lr * gi / sqrt(an + eps));
    }
}

/* sgd.cpp:74-88 */
void so_adam(int dtype, void* p, void* m, void* v, const void* g, double b1, double b2,
             double eps, double lr, uint64_t t, uint64_t n) {
    double c1 = 1.0 - pow(b1, (double)t);
    double c2 = 1.0 - pow(b2, (double)t);
    for (uint64_t i = 0; i < n; ++i) {
        double gi = ld(dtype, g, i);
        double mn = b1 * ld(dtype, m, i) + (1.0 - b1) * gi;
        double vn = b2 * ld(dtype, v, i) + (1.0 - b2) * gi * gi;
        st(dtype, m, i, mn);
        st(dtype, v, i, vn);
        st(dtype, p, i, ld(dtype, p, i) - lr * (mn / c1) / (sqrt(vn / c2) + eps));
    }
}

/* mlp.cpp:31-43: c (n x p) += a (n x m) * b (m x p), i-k-j, zero a[i,k] skipped */
static void mm_acc(const double* a, const double* b, double* c, uint64_t n, uint64_t m,
                   uint64_t p) {
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t k = 0; k < m; ++k) {
            double aik = a[i * m + k];
            if (aik == 0.0) continue;
            for (uint64_t j = 0; j < p; ++j) c[i * p + j] += aik * b[k * p + j];
        }
}

/* mlp.cpp:46-58: c (m x p) += a^T * d, a is n x m */
static void mm_at_acc(const double* a, const double* d, double* c, uint64_t n, uint64_t m,
                      uint64_t p) {
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t k = 0; k < m; ++k) {
            double aik = a[i * m + k];
            if (aik == 0.0) continue;
            for (uint64_t j = 0; j < p; ++j) c[k * p + j] += aik * d[i * p + j];
        }
}

/* mlp.cpp:61-73: c (n x m) += d (n x p) * b^T, b is m x p */
static void mm_bt_acc(const double* d, const double* b, double* c, uint64_t n, uint64_t m,
                      uint64_t p) {
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t k = 0; k < m; ++k) {
            double acc = 0.0;
            for (uint64_t j = 0; j < p; ++j) acc += d[i * p + j] * b[k * p + j];
            c[i * m + k] += acc;
        }
}

/* mlp.cpp:134-218 */
int so_mlp_loss_grad(int dtype, const uint64_t* dims, uint64_t layers, const void* params,
                     const void* x, const void* y, uint64_t n, double* loss_out, void* grad_out) {
    if (n == 0) return -1;
    uint64_t total = 0;
    for (uint64_t l = 0; l < layers; ++l) total += dims[l] * dims[l + 1] + dims[l + 1];
    double* theta = (double*)malloc(sizeof(double) * total);
    double* grad = (double*)calloc(total, sizeof(double));
    double** acts = (double**)calloc(layers + 1, sizeof(double*));
    uint64_t* woff = (uint64_t*)malloc(sizeof(uint64_t) * layers);
    uint64_t* boff = (uint64_t*)malloc(sizeof(uint64_t) * layers);
    for (uint64_t i = 0; i < total; ++i) theta[i] = ld(dtype, params, i);
    uint64_t at = 0;
    for (uint64_t l = 0; l < layers; ++l) {
        woff[l] = at;
        at += dims[l] * dims[l + 1];
        boff[l] = at;
        at += dims[l + 1];
    }
    acts[0] = (double*)malloc(sizeof(double) * n * dims[0]);
    for (uint64_t i = 0; i < n * dims[0]; ++i) acts[0][i] = ld(dtype, x, i);
    for (uint64_t l = 0; l < layers; ++l) {
        uint64_t din = dims[l], dout = dims[l + 1];
        double* z = (double*)malloc(sizeof(double) * n * dout);
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t j = 0; j < dout; ++j) z[i * dout + j] = theta[boff[l] + j];
        mm_acc(acts[l], theta + woff[l], z, n, din, dout);
        if (l + 1 < layers)
            for (uint64_t i = 0; i < n * dout; ++i) z[i] = tanh(z[i]);
        acts[l + 1] = z;
    }
    uint64_t dl = dims[layers];
    double* delta = (double*)malloc(sizeof(double) * n * dl);
    double loss = 0.0, inv_n = 1.0 / (double)n;
    for (uint64_t i = 0; i < n * dl; ++i) {
        double diff = acts[layers][i] - ld(dtype, y, i);
        loss += diff * diff;
        delta[i] = diff * inv_n;
    }
    loss *= 0.5 * inv_n;
    for (uint64_t l = layers; l-- > 0;) {
        uint64_t din = dims[l], dout = dims[l + 1];
        mm_at_acc(acts[l], delta, grad + woff[l], n, din, dout);
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t j = 0; j < dout; ++j) grad[boff[l] + j] += delta[i * dout + j];
        if (l > 0) {
            double* prev = (double*)calloc(n * din, sizeof(double));
            mm_bt_acc(delta, theta + woff[l], prev, n, din, dout);
            for (uint64_t i = 0; i < n * din; ++i) prev[i] *= 1.0 - acts[l][i] * acts[l][i];
            free(delta);
            delta = prev;
        }
    }
    for (uint64_t i = 0; i < total; ++i) st(dtype, grad_out, i, grad[i]);
    *loss_out = loss;
    for (uint64_t l = 0; l <= layers; ++l) free(acts[l]);
    free(acts);
    free(delta);
    free(theta);
    free(grad);
    free(woff);
    free(boff);
    return 0;
}

/* acceptance_main.cpp:86-103, 124-133 */
void so_column_fold(int dtype, int kind, const void* x, uint64_t rows, uint64_t cols, void* out) {
    double init = kind == 0 ? 0.0 : (kind == 1 ? -INFINITY : INFINITY);
    for (uint64_t c = 0; c < cols; ++c) st(dtype, out, c, init);
    for (uint64_t r = 0; r < rows; ++r)
        for (uint64_t c = 0; c < cols; ++c) {
            double a = ld(dtype, out, c), b = ld(dtype, x, r * cols + c);
            double v = kind == 0 ? a + b : (kind == 1 ? (a > b ? a : b) : (a < b ? a : b));
            st(dtype, out, c, v);
        }
}
