/*
 * synk_cuda.h — C-ABI of the B200 (sm_100a) device layer behind the synkpar
 * API. Plain pointers, sizes and int status codes; no C++ or torch types.
 *
 * The C++ executor (paper_1710_04162_b200/csrc/host, the drop-in for the
 * reference's C++ sources in src/) is the only in-tree caller; INTEGRATION.md shows the
 * ctypes binding a maintainer of the reference would add. Each entry point
 * names the reference routine whose per-call work it replaces
 * (file:line under /root/reference/proj).
 *
 * Conventions
 *  - Every function returns 0 (SYNK_OK) or a negative SYNK_E* code; the
 *    message is in synk_last_error() (thread-local).
 *  - A synk_dev is one RANK: a device id, a non-blocking CUDA stream and a
 *    stream-ordered memory pool. Rank-scoped calls are asynchronous on that
 *    stream; synk_sync() is the phase-exit barrier (stream sync + deferred
 *    device-side error flags, e.g. an out-of-range gather index).
 *  - Several ranks may share one GPU (each has its own stream).
 *  - Collectives are issued by EVERY rank of a world from its own host thread
 *    inside one phase, after every rank's inputs are complete (the executor's
 *    phase barrier guarantees that). Rank r only touches chunk r of every
 *    replica, so ranks never race; replicas on other GPUs are reached by
 *    NVLink peer loads/stores (peer access is enabled by synk_open).
 *  - dtype codes = synkpar::DType (tensor.hpp:16-19): 1 f32, 2 f64.
 *  - op codes = synkpar::ReduceOp order (tensor.hpp:27-34):
 *      0 sum, 1 mean, 2 max, 3 min, 4 prod, 5 gather.
 *  - Pointers may be device pointers or pinned, mapped host pointers
 *    (unified addressing); synk_ptr_kind() tells which.
 */
#ifndef SYNK_CUDA_H
#define SYNK_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SYNK_OK 0
#define SYNK_EBOUNDS (-1) /* synkpar::BoundsError   */
#define SYNK_ESHAPE (-2)  /* synkpar::ShapeError    */
#define SYNK_EDTYPE (-3)  /* synkpar::DTypeError    */
#define SYNK_EARG (-4)    /* synkpar::ArgumentError */
#define SYNK_ECUDA (-10)  /* CUDA runtime failure   */
#define SYNK_ENOMEM (-11) /* allocation failure     */
#define SYNK_ENODEV (-12) /* no usable CUDA device  */
#define SYNK_ENCCL (-13)  /* NCCL failure (optional collectives backend) */

#define SYNK_F32 1
#define SYNK_F64 2

#define SYNK_OP_SUM 0
#define SYNK_OP_MEAN 1
#define SYNK_OP_MAX 2
#define SYNK_OP_MIN 3
#define SYNK_OP_PROD 4
#define SYNK_OP_GATHER 5

/* optimizer rules, sgd.hpp:24-45 order */
#define SYNK_RULE_SGD 0
#define SYNK_RULE_MOMENTUM 1
#define SYNK_RULE_RMSPROP 2
#define SYNK_RULE_ADAM 3

typedef struct synk_dev synk_dev;

/* ---- runtime --------------------------------------------------------------- */
const char* synk_last_error(void);
int synk_abi_version(void);
int synk_device_count(int* count);

/* Open `world` rank contexts; rank r runs on device_ids[r]. Enables peer
 * access between every pair of distinct devices. Replaces the rank bring-up
 * of WorkerPool::fork (worker_pool.cpp:225-259). */
int synk_open(int world, const int* device_ids, synk_dev** out);
int synk_close(synk_dev* dev);
int synk_dev_rank(const synk_dev* dev);
int synk_dev_device(const synk_dev* dev);
void* synk_dev_stream(const synk_dev* dev);
/* Make `dev`'s device current on the calling host thread. */
int synk_bind(const synk_dev* dev);
/* Phase-exit barrier: stream sync + device error flags (worker_pool.cpp:58-90). */
int synk_sync(synk_dev* dev);

/* Stream-ordered timing marks (CUDA events) for CallReport/PhaseReport:
 * synk_mark records an event on the rank's stream and returns its id;
 * synk_mark_elapsed reads the seconds between two marks (after synk_sync);
 * synk_mark_reset recycles every mark of the rank. */
int synk_mark(synk_dev* dev, int* mark);
int synk_mark_elapsed(synk_dev* dev, int a, int b, double* seconds);

/* Device-side ordering between ranks without a host barrier: synk_signal
 * marks the current tail of dev's stream; synk_wait_peer makes dev's stream
 * wait (on the GPU) until peer's last signalled point has executed. Used to
 * chain the gradient all-reduce + update onto the gradient phase (the host
 * phase barrier between sgd.cpp:301 and :314 of the reference). */
int synk_signal(synk_dev* dev);
int synk_wait_peer(synk_dev* dev, const synk_dev* peer);
/* The same with one of 64 independent signal slots per rank (e.g. one per
 * gradient segment, so each segment's all-reduce + update can start as soon
 * as every rank finished that segment). */
int synk_signal_slot(synk_dev* dev, int slot);
int synk_wait_peer_slot(synk_dev* dev, const synk_dev* peer, int slot);
/* A second context of the same rank and GPU with its own stream (and marks,
 * flags): collectives overlapped with the rank's compute stream (bucketed
 * gradient all-reduce + update during the backward pass, sgd.cpp:301-319).
 * Closed with synk_close. */
int synk_open_aux(synk_dev* main, synk_dev** aux);
/* Caller-owned timing events on dev's device (independent of the rank's mark
 * ring, so they can be read long after later calls reused the marks): the
 * trainer records its step's stage boundaries here and resolves the
 * StepReport's device times only when the report is read. */
int synk_timer_create(synk_dev* dev, int count, void** timer);
int synk_timer_record(synk_dev* dev, void* timer, int i);
int synk_timer_elapsed(void* timer, int a, int b, double* seconds);
int synk_timer_destroy(void* timer);
int synk_mark_reset(synk_dev* dev);

/* ---- memory ------------------------------------------------------------------ */
/* Stream-ordered HBM allocation on the rank's device (NdBuffer::allocate,
 * tensor.cpp:32-36, for replicas and per-rank batches). */
int synk_alloc(synk_dev* dev, uint64_t bytes, void** out);
int synk_free(synk_dev* dev, void* ptr);
/* Pinned, mapped, portable host memory (the SharedInputArray store,
 * shared_input.cpp:38-64, readable by every GPU over PCIe). */
int synk_host_alloc(uint64_t bytes, void** out);
int synk_host_free(void* ptr);
/* 0 = pageable host, 1 = pinned/mapped host, 2 = device memory. */
int synk_ptr_kind(const void* ptr, int* kind, int* device);
/* The device-side address of page-locked host memory (what a kernel reading
 * it in place must use); SYNK_EARG if `host` is not page-locked. */
int synk_host_device_ptr(const void* host, const void** dev_ptr);
/* Asynchronous copy in any direction (NdBuffer::clone, tensor.cpp:155-159). */
int synk_copy(synk_dev* dev, void* dst, const void* src, uint64_t bytes);
/* Strided 2-D copy: `rows` rows of `row_bytes`, pitches in bytes. */
int synk_copy2d(synk_dev* dev, void* dst, uint64_t dpitch, const void* src, uint64_t spitch,
                uint64_t row_bytes, uint64_t rows);
int synk_memset(synk_dev* dev, void* dst, int value, uint64_t bytes);
/* Fill n elements with a value (NdBuffer::fill, tensor.cpp:141-151). */
int synk_fill(synk_dev* dev, int dtype, void* dst, double value, uint64_t n);

/* dst[0:bytes] = src[0:bytes] by one CTA of the rank's SMs (bytes <= 1 MiB),
 * async on the rank stream. For small results headed to mapped pinned host
 * memory: the phase's last kernel writes them over PCIe instead of a separate
 * copy-engine D2H after the phase (replaces the NdBuffer copy-out of
 * function.cpp:515-527 for a single contributor). */
int synk_copy_small(synk_dev* dev, void* dst, const void* src, uint64_t bytes);
/* Synthetic data generated in place (no reference counterpart: replaces the
 * host-side dataset generation + H2D of bench.cpp:41-58 / acceptance C3 for
 * HBM-resident inputs). Element i of dst = U[-1,1) value number first+i of
 * the stream `seed`: splitmix64(seed + (first+i)*0x9E3779B97F4A7C15) >> 40,
 * times 2^-23, minus 1 (exact in f32 and f64; oracle: so_fill_uniform). */
int synk_fill_uniform(synk_dev* dev, int dtype, void* dst, uint64_t n, uint64_t seed, uint64_t first);

/* dst = (dst dtype) src, elementwise (NdBuffer::get/set conversions). */
int synk_cast(synk_dev* dev, int dst_dtype, void* dst, int src_dtype, const void* src, uint64_t n);

/* ---- input indexing ------------------------------------------------------------ */
/* dst[j,:] = src[idx[j],:] for j < n_idx (gather_rows, tensor.cpp:200-217;
 * excerpt_rows, tensor.cpp:399-409). src is HBM or pinned host; idx is u64 in
 * HBM or pinned host. Bit-exact; an out-of-range index raises SYNK_EBOUNDS at
 * the next synk_sync(). */
int synk_gather_rows(synk_dev* dev, const void* src, uint64_t src_rows, uint64_t row_bytes,
                     const uint64_t* idx, uint64_t n_idx, void* dst);
/* The same for a short list in HOST memory (pageable or pinned), read by the
 * calling thread: n_idx <= SYNK_GATHER_INLINE_MAX and src_rows <= 2^32. The
 * indices travel inside the kernel launch (u32 kernel parameters), so the
 * kernel's first row loads do not wait on PCIe index reads -- the per-call
 * floor of one small batch (excerpt_rows, tensor.cpp:399-409, per call).
 * Bit-exact with synk_gather_rows; an out-of-range index reads row 0 and
 * raises SYNK_EBOUNDS at the next synk_sync(). */
#define SYNK_GATHER_INLINE_MAX 4096
int synk_gather_rows_inline(synk_dev* dev, const void* src, uint64_t src_rows, uint64_t row_bytes,
                            const uint64_t* host_idx, uint64_t n_idx, void* dst);

/* ---- aggregation --------------------------------------------------------------- */
/* acc = op(acc, other), op in {sum,max,min,prod}, in T (combine_inplace,
 * tensor.cpp:250-270; max is b>a?b:a, accumulator wins ties/NaN). */
int synk_combine(synk_dev* dev, int dtype, int op, void* acc, const void* other, uint64_t n);
/* acc = T((f64 acc*wa + f64 other*wb) * (1/(wa+wb))) (tensor.cpp:272-285). */
int synk_weighted_mean(synk_dev* dev, int dtype, void* acc, double wa, const void* other,
                       double wb, uint64_t n);
/* v = T(f64 v * factor) (scale_inplace, tensor.cpp:367-373). */
int synk_scale(synk_dev* dev, int dtype, void* buf, double factor, uint64_t n);
/* out = left fold of parts[0..count) in order (OutputAccumulator + the master
 * rank fold, function.cpp:76-115,515-527). Mean is row-weighted by weights[].
 * parts may live on peer GPUs. */
int synk_left_fold(synk_dev* dev, int dtype, int op, void* out, const void* const* parts,
                   const uint64_t* weights, uint32_t count, uint64_t n);
/* Column statistics of a row-major [rows x cols] slice in one HBM pass:
 * sum (deterministic tree order), max, min (acceptance_main.cpp:86-133 kernels).
 * Any of the three outputs may be NULL. */
int synk_column_stats(synk_dev* dev, int dtype, const void* x, uint64_t rows, uint64_t cols,
                      void* sum_out, void* max_out, void* min_out);
/* *equal = 1 iff the byte ranges match (equals_bitwise, tensor.cpp:169-173);
 * b may be on a peer GPU. Synchronous. */
int synk_equal(synk_dev* dev, const void* a, const void* b, uint64_t bytes, int* equal);
/* *finite = 1 iff no NaN/Inf (all_finite, sgd.cpp:171-185). Synchronous. */
int synk_all_finite(synk_dev* dev, int dtype, const void* x, uint64_t n, int* finite);

/* ---- collectives (single process, peer memory, reference tree order) -------------- */
/* Called by every rank r of `world` inside one phase. bufs[q] = rank q's
 * replica (n elements). Rank r folds chunk r of all replicas in the fixed
 * binomial order of tree_fold (replicated.cpp:16-29) and stores the result
 * into chunk r of every replica: bitwise equal to ReplicatedVariable::
 * all_reduce (replicated.cpp:124-137). */
int synk_all_reduce(synk_dev* dev, int world, int dtype, int op, void* const* bufs, uint64_t n);
/* The element range [lo, hi) rank r owns in every collective above (host-only;
 * 16-element aligned chunks, the last ones possibly short or empty). */
int synk_chunk_range(uint64_t n, int world, int rank, uint64_t* lo, uint64_t* hi);
/* Fold of all replicas into `out` (tree order), run by one rank
 * (ReplicatedVariable::reduce, replicated.cpp:139-149). */
int synk_tree_reduce(synk_dev* dev, int world, int dtype, int op, const void* const* bufs,
                     uint64_t n, void* out);
/* Rank r copies chunk r of bufs[src] into every other replica
 * (ReplicatedVariable::broadcast, replicated.cpp:115-122). */
int synk_broadcast(synk_dev* dev, int world, int src, void* const* bufs, uint64_t bytes);
/* Small-buffer forms: ONE rank runs every chunk of the collective over the
 * peer pointers (same per-element tree order, so bitwise identical to the
 * per-rank forms). For buffers where waking every rank's thread costs more
 * than the transfer (ReplicatedVariable::all_reduce / broadcast below 1 MiB,
 * replicated.cpp:115-137). */
int synk_all_reduce_whole(synk_dev* dev, int world, int dtype, int op, void* const* bufs, uint64_t n);
int synk_broadcast_whole(synk_dev* dev, int world, int src, void* const* bufs, uint64_t bytes);

/* Optional NCCL backend (ForkOptions::collectives = "nccl"): the library
 * baseline the peer-memory kernels are compared with on multi-GPU boxes.
 * libnccl.so.2 is dlopen'ed on first use; one communicator per rank
 * (ncclCommInitAll, distinct GPUs required), used from the rank's thread on
 * its stream. Sum/mean results are NCCL's reduction order (within the
 * reference's 8*W*eps tolerance, not its tree order); max/min/broadcast are
 * exact. */
int synk_nccl_available(void);
int synk_nccl_open(int world, synk_dev* const* devs);
int synk_nccl_close(synk_dev* dev);
int synk_nccl_all_reduce(synk_dev* dev, int dtype, int op, void* buf, uint64_t n);
int synk_nccl_broadcast(synk_dev* dev, int root, void* buf, uint64_t bytes);

/* ---- optimizer ---------------------------------------------------------------- */
/* hyper: momentum {mu}; rmsprop {rho, eps}; adam {beta1, beta2, eps}.
 * t = post-increment step counter. f64 math, cast on store (sgd.cpp:46-88). */
int synk_optimizer_step(synk_dev* dev, int dtype, int rule, const double* hyper, double lr,
                        uint64_t t, void* params, const void* grads, void* aux0, void* aux1,
                        uint64_t n);
/* Fused gradient all-reduce + update, called by every rank of a world in one
 * phase (SyncSgd::train_step all_reduce + step, sgd.cpp:313-319): rank r
 * tree-folds chunk r of all gradient replicas (grad_op sum or mean),
 * writes the reduced chunk back to every gradient replica, applies the rule
 * to chunk r of its own params/aux and stores the new chunk into every
 * params/aux replica. aux0/aux1 may be NULL for rules without state.
 * flags: SYNK_STEP_COHERENT promises that params/aux replicas are bitwise
 * equal (the executor tracks this), so chunk r is computed once from rank r's
 * replica; without it every replica's chunk is updated from its own values,
 * exactly as per-rank steps would (sgd.cpp:226-248). SYNK_STEP_GRADS_LOCAL
 * (world > 1) writes the reduced gradient chunk r into rank r's gradient
 * replica only -- a deferred all-gather: replica q then holds the reduced
 * values in chunk q alone (synk_chunk_range), and the caller pulls the other
 * chunks before anything reads the gradients (NVLink bytes per rank per step
 * 2(W-1)/W * S instead of 3(W-1)/W * S). */
#define SYNK_STEP_COHERENT 1
#define SYNK_STEP_GRADS_LOCAL 2
/* SYNK_STEP_BACKGROUND: the launch overlaps other work on another stream of
 * the same GPU (the bucketed update beside the backward GEMMs): a small grid. */
#define SYNK_STEP_BACKGROUND 4
int synk_all_reduce_step(synk_dev* dev, int world, int dtype, int grad_op, int rule,
                         const double* hyper, double lr, uint64_t t, void* const* params,
                         void* const* grads, void* const* aux0, void* const* aux1, uint64_t n,
                         int flags);

/* ---- tensor-core GEMM (the MLP's dense products, mlp.cpp:31-73) -------------------- */
#define SYNK_BF16 3     /* storage code for bf16 operands/outputs (new; DType has f32/f64) */
#define SYNK_GEMM_BF16 0   /* tcgen05 kind::f16, bf16 operands, fp32 accumulate          */
#define SYNK_GEMM_TF32 1   /* tcgen05 kind::tf32, one pass                                 */
#define SYNK_GEMM_TF32X3 2 /* tcgen05 kind::tf32, hi*hi + hi*lo + lo*hi (fp32 accuracy)    */
#define SYNK_EPI_STORE 0
#define SYNK_EPI_BIAS 1      /* + bias[n]                                                 */
#define SYNK_EPI_BIAS_TANH 2 /* tanh(. + bias[n])                       (mlp.cpp:169-176) */
#define SYNK_EPI_TANH_GRAD 3 /* . * (1 - act[m,n]^2)                    (mlp.cpp:206-208) */
/* Operand staging for synk_gemm_tc: out = in (or in^T when transpose) as
 * mode 0: tf32 hi/lo split (out_hi, out_lo fp32), 1: bf16 cast, 2: fp32 copy;
 * out is out_rows x out_cols with leading dim ld_out, zero beyond the input. */
int synk_gemm_prep(synk_dev* dev, int in_dtype, const void* in, uint64_t rows, uint64_t cols, uint64_t ld_in,
                   int transpose, int mode, void* out_hi, float* out_lo, uint64_t out_rows, uint64_t out_cols,
                   uint64_t ld_out);
/* Fused bf16 staging: out = bf16(in) (rows x cols, ld_out) and out_t =
 * bf16(in)^T (cols x rows, ld_out_t) from one read of the f32 input; either
 * output may be NULL. */
int synk_gemm_prep2_bf16(synk_dev* dev, const float* in, uint64_t rows, uint64_t cols, uint64_t ld_in, void* out,
                         uint64_t ld_out, void* out_t, uint64_t ld_out_t);
/* The same with an index-fused gather: output row r is input row rowmap[r]
 * (u64 in HBM); rowmap == NULL is synk_gemm_prep2_bf16. */
int synk_gemm_prep2_bf16_rows(synk_dev* dev, const float* in, const uint64_t* rowmap, uint64_t rows, uint64_t cols,
                              uint64_t ld_in, void* out, uint64_t ld_out, void* out_t, uint64_t ld_out_t);
/* C[M x N] = epilogue(A[M x K] . B[N x K]^T); A, B K-major with leading dims
 * lda/ldb (16-byte aligned rows). C (row-major, ldc) and/or C^T (ldct) may be
 * NULL; out_dtype SYNK_F32 or SYNK_BF16 (act has the same dtype as C). */
int synk_gemm_tc(synk_dev* dev, int kind, uint64_t M, uint64_t N, uint64_t K, const void* a_hi, const void* a_lo,
                 uint64_t lda, const void* b_hi, const void* b_lo, uint64_t ldb, int epilogue, int out_dtype,
                 void* c, uint64_t ldc, void* ct, uint64_t ldct, const float* bias, const void* act,
                 uint64_t ldact);
/* synk_gemm_tc with operand layouts (bf16 only for non-zero bits):
 * layout bit 0 (SYNK_GEMM_A_MN): A stored MN-major, as K x M with M contiguous
 *   (leading dim lda) -- e.g. the activation a_l [n x d_l] as A = a_l^T;
 * layout bit 1 (SYNK_GEMM_B_MN): B stored as K x N with N contiguous (ldb) --
 *   e.g. W_l [d_l x d_l+1] as the forward product's B = W_l^T.
 * The tensor cores read MN-major shared-memory tiles directly (UMMA major
 * bits), so the MLP's weight/activation/delta transposes (mlp.cpp:31-73,
 * 169-208 use W^T, a^T, delta^T) are never materialised. */
/* fp32-accurate tensor-core GEMM (3xTF32) for the f32 example function
 * (replaces mlp.cpp:31-73's f32 products): C[M x N] = epilogue(A . B^T) with A
 * [M x K], B [N x K] K-major fp32 given as tf32 hi/lo parts (synk_tf32_split;
 * leading dims lda/ldb in elements, rows 16-byte aligned). Each 32-element K
 * block is accumulated on tcgen05 (kind::tf32: hi.lo + lo.hi + hi.hi) into a
 * fresh TMEM accumulator and added into fp32 registers (round-to-nearest);
 * split-K partials (shape-fixed, <= 8) are folded in f64 in rank order. Any
 * subset of outputs: c (fp32 row-major, ldc); c_hi/c_lo (the result's tf32
 * split, row-major, ldh); ct_hi/ct_lo (transposed split, [n][m], ldt). act
 * (EPI_TANH_GRAD) is fp32 [M x N] with leading dim ldact. */
int synk_gemm_f32x3(synk_dev* dev, uint64_t M, uint64_t N, uint64_t K, const float* a_hi, const float* a_lo,
                    uint64_t lda, const float* b_hi, const float* b_lo, uint64_t ldb, int epilogue, float* c,
                    uint64_t ldc, const float* bias, const float* act, uint64_t ldact, float* c_hi, float* c_lo,
                    uint64_t ldh, float* ct_hi, float* ct_lo, uint64_t ldt);
/* tf32 split of in (rows x cols, ld_in; row r is in row rowmap[r] when rowmap
 * != NULL, u64 in HBM): hi = rna_tf32(x), lo = rna_tf32(x - hi), row-major
 * (hi/lo, ld_o) and/or transposed (hi_t/lo_t, cols x rows, ld_t). */
int synk_tf32_split(synk_dev* dev, const float* in, const uint64_t* rowmap, uint64_t rows, uint64_t cols,
                    uint64_t ld_in, float* hi, float* lo, uint64_t ld_o, float* hi_t, float* lo_t, uint64_t ld_t);
/* Sets up to 64 split rows to (value, 0): the constant ones row under a^T that
 * turns the weight-gradient product into [gW; gb] (mlp.cpp:193-203). */
#define SYNK_TF32_MAX_ROWS 64
typedef struct synk_tf32_rows {
    float* hi[SYNK_TF32_MAX_ROWS];
    float* lo[SYNK_TF32_MAX_ROWS];
    uint64_t len[SYNK_TF32_MAX_ROWS];
    uint32_t count;
    float value;
} synk_tf32_rows;
int synk_tf32_fill_rows(synk_dev* dev, const synk_tf32_rows* rows);
/* A step's whole operand staging in one launch: up to 16 split jobs (each as
 * synk_tf32_split) plus the constant rows (fill may be NULL). */
#define SYNK_TF32_MAX_JOBS 16
typedef struct synk_tf32_job {
    const float* in;
    const uint64_t* rowmap;
    uint64_t rows, cols, ld_in;
    float* hi;
    float* lo;
    uint64_t ld_o;
    float* hi_t;
    float* lo_t;
    uint64_t ld_t;
} synk_tf32_job;
int synk_tf32_stage(synk_dev* dev, const synk_tf32_job* jobs, uint32_t count, const synk_tf32_rows* fill);
/* bf16 weight shadow: a per-rank HBM copy of an MLP's weight matrices in the
 * bf16 operand layout of the tensor-core path (W_l row-major with padded
 * leading dimension, plus W_l^T for narrow layers). The fused update writes
 * it together with the new f32 params, so the next step's products read it
 * directly instead of re-casting 100 MB of f32 weights (replaces the per-step
 * cast of mlp.cpp's f64 widening on the bf16 path). Layout per rank:
 * synk_mlp_bf16_shadow(). off_wt == SYNK_NO_TRANSPOSE: no transposed copy. */
#define SYNK_SHADOW_MAX_SEGS 8
#define SYNK_SHADOW_MAX_WORLD 8
#define SYNK_NO_TRANSPOSE (~(uint64_t)0)
typedef struct synk_bf16_shadow_seg {
    uint64_t first;       /* element offset of W_l in the flat parameter block */
    uint64_t rows, cols;  /* d_l x d_{l+1} */
    uint64_t off_w, ldw;  /* byte offset of bf16 W_l in the shadow, leading dim (elements) */
    uint64_t off_wt, ldwt;/* byte offset of bf16 W_l^T, leading dim; or SYNK_NO_TRANSPOSE */
} synk_bf16_shadow_seg;
typedef struct synk_bf16_shadow {
    uint32_t count;       /* weight segments */
    uint64_t bytes;       /* shadow buffer size per rank */
    synk_bf16_shadow_seg seg[SYNK_SHADOW_MAX_SEGS];
} synk_bf16_shadow;
int synk_mlp_bf16_shadow(const uint64_t* dims, uint32_t layers, synk_bf16_shadow* out);

/* synk_all_reduce_step over the flat range [elem_base, elem_base + n) of a
 * larger block (the pointers are already offset by elem_base), additionally
 * writing bf16(new params) into every rank's shadow (shadow_bases[q], layout
 * `shadow`) for the elements that fall in a shadow weight segment. shadow may
 * be NULL (plain synk_all_reduce_step). f32 only, world <= SYNK_SHADOW_MAX_WORLD. */
int synk_all_reduce_step_ex(synk_dev* dev, int world, int dtype, int grad_op, int rule,
                            const double* hyper, double lr, uint64_t t, void* const* params,
                            void* const* grads, void* const* aux0, void* const* aux1, uint64_t n,
                            int flags, uint64_t elem_base, const synk_bf16_shadow* shadow,
                            void* const* shadow_bases);

#define SYNK_GEMM_A_MN 1
#define SYNK_GEMM_B_MN 2
int synk_gemm_tc2(synk_dev* dev, int kind, uint64_t M, uint64_t N, uint64_t K, const void* a_hi, const void* a_lo,
                  uint64_t lda, const void* b_hi, const void* b_lo, uint64_t ldb, int layout, int epilogue,
                  int out_dtype, void* c, uint64_t ldc, void* ct, uint64_t ldct, const float* bias,
                  const void* act, uint64_t ldact);

/* ---- example function: tanh MLP loss + gradient (mlp.cpp:134-218) ---------------- */
/* dims[0..layers]; params flat [W0 b0 W1 b1 ...]; x [n x dims0]; y [n x dims_L].
 * Writes the f64 loss scalar to loss_dev (device) and the flat gradient (dtype)
 * to grad. workspace from synk_mlp_workspace_bytes. */
int synk_mlp_workspace_bytes(int dtype, const uint64_t* dims, uint32_t layers, uint64_t n,
                             uint64_t* bytes);
int synk_mlp_loss_grad(synk_dev* dev, int dtype, const uint64_t* dims, uint32_t layers,
                       const void* params, const void* x, const void* y, uint64_t n,
                       double* loss_dev, void* grad, void* workspace, uint64_t workspace_bytes);

/* synk_mlp_loss_grad_ex that, for the bf16 tensor-core path, records
 * synk_signal_slot(dev, signal_base + l) as soon as the gradient segment of
 * layer l ([W_l, b_l] in the flat layout) is final; *signalled = the number
 * of segments signalled (0: nothing signalled, e.g. the native path).
 * rows != NULL: x and y are the whole sources and batch row i is source row
 * rows[i] (u64 in device memory, n entries, every entry a valid row: the
 * caller checks the list) -- the bf16 staging of x (bf16 path) or a gather
 * inside the launch sequence (native path) and the loss read through it. */
int synk_mlp_loss_grad_seg(synk_dev* dev, int dtype, int compute, const uint64_t* dims, uint32_t layers,
                           const void* params, const void* x, const void* y, uint64_t n, double* loss_dev,
                           void* grad, void* workspace, uint64_t workspace_bytes, int signal_base,
                           int* signalled, const uint64_t* rows);
/* Options of synk_mlp_loss_grad_opts (all optional; zero-initialise).
 *   signal_base      as synk_mlp_loss_grad_seg (-1: no segment signals)
 *   rows             index-fused batch rows in HBM (as synk_mlp_loss_grad_seg)
 *   rows_host        the same list as a device-readable alias of page-locked
 *                    host memory, or NULL (informational: the x staging
 *                    reads `rows`, PCIe latency per tile made it slower)
 *   rows_ready_on / rows_ready_slot: `rows` is filled once the slot event of
 *                    that handle fires (synk_signal_slot); the stream waits on
 *                    it before the first read of `rows`. NULL: ready now.
 *   shadow           bf16 weight shadow (synk_mlp_bf16_shadow layout) of this
 *                    rank, bf16 path only; NULL: casts into the workspace
 *   shadow_valid     1: the shadow equals bf16(params): the casts are skipped;
 *                    0: the casts write the shadow (valid afterwards).
 *   shadow_spare     1: the update that follows writes the NEXT shadow into
 *                    another buffer (double-buffered shadows), so segment l is
 *                    signalled right after its weight gradient; 0: the update
 *                    rewrites this shadow, so segment l (l > 0) is signalled
 *                    only after dX_l has read W_l.
 *   seg_order        out (may be NULL, else >= layers ints): the layer of
 *                    each signalled segment, in signal order. The bf16 path
 *                    runs every dX product first and then the weight
 *                    gradients largest segment first, so each segment's
 *                    all-reduce + update overlaps the remaining weight-
 *                    gradient products. */
typedef struct synk_mlp_opts {
    int signal_base;
    const uint64_t* rows;
    const uint64_t* rows_host;
    synk_dev* rows_ready_on;
    int rows_ready_slot;
    void* shadow;
    int shadow_valid;
    int shadow_spare;
    int* seg_order;
} synk_mlp_opts;
int synk_mlp_loss_grad_opts(synk_dev* dev, int dtype, int compute, const uint64_t* dims, uint32_t layers,
                            const void* params, const void* x, const void* y, uint64_t n, double* loss_dev,
                            void* grad, void* workspace, uint64_t workspace_bytes, const synk_mlp_opts* opts,
                            int* signalled);
/* Same with a compute mode: SYNK_MLP_NATIVE runs every product in the
 * parameter dtype on the CUDA cores (f32 FFMA / f64 DFMA); SYNK_MLP_BF16_TC
 * (f32 parameters only) runs every dense product on tcgen05 tensor cores
 * with bf16 operands and fp32 accumulation (the wide-MLP config). */
#define SYNK_MLP_NATIVE 0
#define SYNK_MLP_BF16_TC 1
/* f32 parameters, every product on the tensor cores at fp32 accuracy
 * (synk_gemm_f32x3). SYNK_MLP_NATIVE with f32 parameters runs this path too
 * unless SYNK_MLP_F32=ffma (CUDA-core FFMA products, A/B runs). */
#define SYNK_MLP_F32_TC 2
int synk_mlp_workspace_bytes_ex(int dtype, int compute, const uint64_t* dims, uint32_t layers, uint64_t n,
                                uint64_t* bytes);
int synk_mlp_loss_grad_ex(synk_dev* dev, int dtype, int compute, const uint64_t* dims, uint32_t layers,
                          const void* params, const void* x, const void* y, uint64_t n, double* loss_dev,
                          void* grad, void* workspace, uint64_t workspace_bytes);

#ifdef __cplusplus
}
#endif

#endif /* SYNK_CUDA_H */
