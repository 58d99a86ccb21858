/*
 * synk_oracle — CPU restatement of the Synkhronos/synkpar data-parallel path.
 *
 * TEST INFRASTRUCTURE ONLY. This file is the parity checker: it may be used by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg, never by the
 * product path (paper_1710_04162_b200/), which has no CPU fallback.
 *
 * Every function restates one reference routine; the citation is the
 * reference file:line (under /root/reference/proj) whose arithmetic it follows.
 * Parity is pinned in tests/test_oracle.py against (a) the known answers of the
 * reference's own unit tests, restated, and (b) golden vectors produced by the
 * unmodified reference (oracle/_ref/_synkpar_ref, tests/golden/make_golden.py).
 *
 * dtype codes follow synkpar::DType (tensor.hpp:16-19): 1 = f32, 2 = f64.
 * op codes follow synkpar::ReduceOp order (tensor.hpp:27-34):
 *   0 sum, 1 mean, 2 max, 3 min, 4 prod, 5 gather.
 */
#ifndef SYNK_ORACLE_H
#define SYNK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* tensor.cpp:315-327 — first n%parts ranges get one extra row. */
void so_partition_rows(uint64_t n_rows, uint64_t n_parts, uint64_t* starts, uint64_t* stops);

/* tensor.cpp:200-217 — out[j,:] = src[idx[j],:]; returns -1 (BoundsError) on a bad index. */
int so_gather_rows(const void* src, uint64_t src_rows, uint64_t row_bytes,
                   const uint64_t* idx, uint64_t n_idx, void* dst);

/* tensor.cpp:250-270 — acc = op(acc, other) elementwise in T; max is b>a?b:a. */
int so_combine(int dtype, int op, void* acc, const void* other, uint64_t n);

/* tensor.cpp:272-285 — acc = T((f64 a*wa + f64 b*wb) * (1/(wa+wb))). */
int so_weighted_mean(int dtype, void* acc, double wa, const void* other, double wb, uint64_t n);

/* tensor.cpp:367-373 — v = T(f64(v) * factor). */
void so_scale(int dtype, void* buf, double factor, uint64_t n);

/* Synthetic U[-1,1) stream used for HBM-resident bench/test datasets
 * (mirrors synk_fill_uniform; no reference counterpart). */
void so_fill_uniform(int dtype, void* dst, uint64_t n, uint64_t seed, uint64_t first);

/* replicated.cpp:16-29 — binomial-tree fold of `world` replicas into out
 * (Mean = Sum then scale by 1/world). */
int so_tree_fold(int dtype, int op, const void* const* parts, uint64_t world, uint64_t n, void* out);

/* function.cpp:76-101,515-527 — left fold in contribution order; Mean is the
 * running row-weighted mean. weights[i] = rows of contribution i. */
int so_left_fold(int dtype, int op, const void* const* parts, const uint64_t* weights,
                 uint64_t count, uint64_t n, void* out);

/* sgd.cpp:46-88 — optimizer steps, f64 math, cast on store. t is the
 * post-increment step counter (sgd.cpp:145-157). */
void so_sgd(int dtype, void* p, const void* g, double lr, uint64_t n);
void so_momentum(int dtype, void* p, void* v, const void* g, double mu, double lr, uint64_t n);
void so_rmsprop(int dtype, void* p, void* a, const void* g, double rho, double eps, double lr,
                uint64_t n);
void so_adam(int dtype, void* p, void* m, void* v, const void* g, double b1, double b2,
             double eps, double lr, uint64_t t, uint64_t n);

/* mlp.cpp:134-218 — tanh MLP forward/backward, all math in f64, grads cast
 * to dtype at the end. dims has layers+1 entries. Flat params layout
 * [W0 (d0 x d1), b0 (d1), W1, b1, ...]. Returns the f64 loss via *loss.
 * Returns -1 on an empty batch. */
int so_mlp_loss_grad(int dtype, const uint64_t* dims, uint64_t layers, const void* params,
                     const void* x, const void* y, uint64_t n, double* loss, void* grad);

/* acceptance_main.cpp:86-103 column kernels: out[c] = fold(out[c], x[r,c]) in
 * row order, through f64 with a cast to T per step (NdBuffer::get/set).
 * kind: 0 sum (init 0), 1 max (init -inf, a>b?a:b), 2 min (init +inf, a<b?a:b). */
void so_column_fold(int dtype, int kind, const void* x, uint64_t rows, uint64_t cols, void* out);

#ifdef __cplusplus
}
#endif

#endif
