// Tensor-core GEMM for the example function's dense products, sm_100a only:
//   C[M x N] = epilogue( A[M x K] . B[N x K]^T )     (A, B K-major in HBM)
//
// One 128 x 128 output tile per CTA (4 warps):
//   warp 0 / one lane : TMA producer — cp.async.bulk.tensor 2-D loads of
//                       128 x 128-byte A and B boxes (SWIZZLE_128B) into a
//                       kStages-deep shared-memory ring, mbarrier complete_tx
//   warp 1 / one lane : MMA issuer — tcgen05.mma.cta_group::1 (kind::f16 for
//                       bf16 operands, kind::tf32 for fp32 operands) with the
//                       fp32 accumulator in TMEM (128 lanes x 128 columns);
//                       tcgen05.commit releases each smem stage and finally
//                       signals the epilogue
//   warp 2            : TMEM allocation / deallocation
//   all 4 warps       : epilogue — tcgen05.ld 32x32b (thread t owns tile row
//                       t), fused bias / tanh / tanh-derivative, stores to C
//                       (and optionally to C^T, which this lane layout makes
//                       fully coalesced).
//
// 3xTF32 (kind 2): operands pre-split into tf32 hi + lo parts
// (synk_gemm_prep mode 0); the kernel accumulates hi*hi + hi*lo + lo*hi in the
// same TMEM accumulator (3 passes over K). Products are then exact, but the
// tcgen05 fp32 accumulator itself rounds with a bias of ~-6.7e-9 per
// accumulated product (profiles/r01_tcgen05_tf32_accumulation.txt), so long K
// chains drift past the 1e-5 fp32 bar. This kind stays as the C-ABI's plain
// 3xTF32 GEMM; the f32 example function runs on gemm_f32x3.cu, which restarts
// the TMEM accumulator every K block and sums the blocks in fp32 registers.
// Production use of this file is bf16 (kind 0): this non-persistent kernel
// for the narrow (N <= 128) products, the persistent CTA-pair kernel below
// for the wide ones.
//
// Occupancy: 3 stages x 32 KB + barriers ~ 97 KB smem and 128 TMEM columns per
// CTA, so two CTAs share an SM and one CTA's epilogue overlaps the other's
// mainloop (0.43 -> 0.77-0.82 of the measured bf16 peak at 8192x4096x4096..8192^3).

#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>

#include <stdlib.h>

#include <algorithm>
#include <mutex>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace {

using namespace synk_tc;

constexpr int BM = 128, BN = 128, kStages = 3;  // ~97 KB smem: two CTAs per SM, one's epilogue overlaps the other's MMAs
constexpr int kTileBytes = 128 * 128;  // 128 rows x 128 bytes, one operand, one stage

enum Epi { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_TANH = 2, EPI_TANH_GRAD = 3 };

// Instruction descriptor: fp32 accumulate, K-major A and B, M = 128, N = 128.
template <int KIND>
__host__ __device__ constexpr uint32_t instr_desc() {
    return (1u << 4)                        // D format f32
           | ((KIND == 0 ? 1u : 2u) << 7)   // A format: bf16 | tf32
           | ((KIND == 0 ? 1u : 2u) << 10)  // B format
           | ((uint32_t)(BN >> 3) << 17)    // N
           | ((uint32_t)(BM >> 4) << 24);   // M
}

struct EpiArgs {
    int mode;
    int out_bf16;         // store C (and C^T) as bf16 instead of fp32
    void* c;
    uint64_t ldc;
    void* ct;             // optional transposed output, may be null
    uint64_t ldct;
    const float* bias;    // per column
    const void* act;      // tanh activations for EPI_TANH_GRAD, same layout/dtype as C
    uint64_t ldact;
};

__device__ __forceinline__ float load_act(const EpiArgs& e, uint64_t m, uint64_t n) {
    if (e.out_bf16) return __bfloat162float(static_cast<const __nv_bfloat16*>(e.act)[m * e.ldact + n]);
    return static_cast<const float*>(e.act)[m * e.ldact + n];
}

__device__ __forceinline__ void store_out(void* base, uint64_t off, float v, int bf16) {
    if (bf16) static_cast<__nv_bfloat16*>(base)[off] = __float2bfloat16_rn(v);
    else static_cast<float*>(base)[off] = v;
}

__device__ __forceinline__ void epi_chunk(const EpiArgs& epi, uint64_t m, uint64_t nb, uint64_t N,
                                          const uint32_t (&r)[16], bool vec_c, bool vec_act, bool have_pre, uint4 pre0, uint4 pre1);

// Activation prefetch for the tanh-derivative epilogue (bf16 act, aligned
// rows): the chunk's 32 bytes are loaded one chunk ahead so the HBM latency
// overlaps the previous chunk's math and stores.
struct ActPrefetch {
    bool on;
    const __nv_bfloat16* row;  // act row m
    uint4 buf[2];
    __device__ __forceinline__ void load(uint64_t nb) {
        const uint4* src = reinterpret_cast<const uint4*>(row + nb);
        buf[0] = src[0];
        buf[1] = src[1];
    }
};

// 256-bit global accesses (sm_100 ld/st .v8.b32): one instruction per
// 32-byte sector per lane. The epilogue's lanes own different rows, so a
// 16-byte access leaves every sector of the warp's request half used.
__device__ __forceinline__ void ld256_stream(const void* p, uint4& lo, uint4& hi) {
    asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w)
                 : "l"(p));
}
__device__ __forceinline__ void st256(void* p, const uint32_t (&w)[8]) {
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(w[0]), "r"(w[1]), "r"(w[2]),
                 "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7])
                 : "memory");
}

// Split-K fold through distributed shared memory (cluster = the S split CTAs
// of one output tile, cluster rank = blockIdx.z): every CTA parks its fp32
// partial tile in its own (now idle) operand ring, the cluster syncs, CTA z
// folds rows [z*R, (z+1)*R) across the S partials in rank order with an f64
// accumulator (the same order and rounding as splitk_fold_kernel), adds the
// bias and writes C; a second cluster sync keeps every partial alive until
// its readers are done. Replaces S fp32 planes in HBM and the fold launch.
constexpr int kFoldPitch = BN + 4;  // floats; +4 spreads the row-per-lane stores over the banks

__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int NT>
__device__ __forceinline__ void cluster_fold_epilogue(const EpiArgs& epi, float* part, uint32_t lane_base, int row,
                                                      int c_begin, int c_count, uint32_t m0, uint32_t n0, uint32_t M,
                                                      uint32_t N) {
#pragma unroll 1
    for (int c0 = c_begin; c0 < c_begin + c_count; c0 += 16) {
        uint32_t r[16];
        tmem_ld16(lane_base + c0, r);
        float4* dst = reinterpret_cast<float4*>(part + row * kFoldPitch + c0);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            dst[j] = make_float4(__uint_as_float(r[4 * j]), __uint_as_float(r[4 * j + 1]), __uint_as_float(r[4 * j + 2]),
                                 __uint_as_float(r[4 * j + 3]));
    }
    cluster_sync_all();
    uint32_t me, S;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(me));
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(S));
    const uint32_t rows_per = (BM + S - 1) / S, r_begin = me * rows_per;
    const uint32_t r_end = min((uint32_t)BM, r_begin + rows_per);
    const uint32_t local = (uint32_t)__cvta_generic_to_shared(part);
    float* C = static_cast<float*>(epi.c);
    // float4 columns per row that hold output (N = 100: 25 of 32)
    const uint32_t kQuads = (min((uint32_t)BN, N - n0) + 3) / 4;
    for (uint32_t i = threadIdx.x; i < (r_end - r_begin) * kQuads; i += NT) {
        const uint32_t rr = r_begin + i / kQuads, cc = (i % kQuads) * 4;
        const uint32_t off = local + (rr * kFoldPitch + cc) * 4;
        // every partial's load in flight before the fold (DSMEM latency is
        // paid once per item, not S times)
        float4 x[8];
#pragma unroll
        for (uint32_t z = 0; z < 8; ++z) {
            if (z >= S) break;
            uint32_t remote;
            asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(off), "r"(z));
            asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                         : "=f"(x[z].x), "=f"(x[z].y), "=f"(x[z].z), "=f"(x[z].w)
                         : "r"(remote));
        }
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
        for (uint32_t z = 0; z < 8; ++z) {
            if (z >= S) break;
            a0 += (double)x[z].x, a1 += (double)x[z].y, a2 += (double)x[z].z, a3 += (double)x[z].w;
        }
        const uint64_t m = (uint64_t)m0 + rr;
        if (m >= M) continue;
        const double a[4] = {a0, a1, a2, a3};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint64_t n = (uint64_t)n0 + cc + j;
            if (n >= N) break;
            float v = (float)a[j];
            if (epi.mode == EPI_BIAS) v += epi.bias[n];
            C[m * epi.ldc + n] = v;
        }
    }
    cluster_sync_all();
}

template <int KIND, int NT>  // NT = 128 or 256 threads (4 or 8 epilogue warps)
__global__ void __launch_bounds__(NT, 2)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap a0, const __grid_constant__ CUtensorMap a1,
                   const __grid_constant__ CUtensorMap b0, const __grid_constant__ CUtensorMap b1, int passes,
                   uint32_t M, uint32_t N, uint32_t K, EpiArgs epi, uint32_t kb_per, uint32_t layout, int cfold,
                   uint32_t n_eff) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-byte alignment for SWIZZLE_128B atoms
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;
    uint8_t* sb = smem + kStages * kTileBytes;
    uint64_t* bars = reinterpret_cast<uint64_t*>(sb + kStages * kTileBytes);  // full[S], empty[S], tmem_full
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    constexpr int kBK = 128 / (KIND == 0 ? 2 : 4);  // elements per 128-byte K block
    // PDL: the next GEMM on the stream may be scheduled as soon as every CTA
    // of this one runs; it waits (below) before touching global memory.
    synk::release_dependent_grid();
    // split-K (gridDim.z > 1): CTA z owns K blocks [kb0, kb0 + num_kb) and
    // stores its raw fp32 partial to plane z of C (host folds the planes).
    const int kb0 = (int)(blockIdx.z * kb_per);
    const int num_kb = min((int)kb_per, (int)((K + kBK - 1) / kBK) - kb0);
    const int total = passes * num_kb;
    if (gridDim.z > 1 && !cfold) epi.c = static_cast<float*>(epi.c) + (uint64_t)blockIdx.z * M * epi.ldc;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&bars[s]), 1);
            mbar_init(smem_u32(&bars[kStages + s]), 1);
        }
        mbar_init(smem_u32(&bars[2 * kStages]), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_map(&a0);
        prefetch_map(&b0);
        if (passes > 1) {
            prefetch_map(&a1);
            prefetch_map(&b1);
        }
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    // Launched programmatically after the previous kernel (PDL): barriers and
    // TMEM are set up while it drains; no global access before it completed.
    synk::wait_prerequisite_grid();

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----
        for (int it = 0; it < total; ++it) {
            const int s = it % kStages;
            const uint32_t parity = ((it / kStages) & 1) ^ 1;
            mbar_wait(smem_u32(&bars[kStages + s]), parity);
            const int pass = it / num_kb, kb = it % num_kb;
            const CUtensorMap* ma = pass == 2 ? &a1 : &a0;  // passes: hi.hi, hi.lo, lo.hi
            const CUtensorMap* mb = pass == 1 ? &b1 : &b0;
            const uint32_t full = smem_u32(&bars[s]);
            mbar_expect_tx(full, kTileBytes + n_eff * 128);  // B box: n_eff rows (narrow N) x 128 B
            const int kc = (kb0 + kb) * kBK;
            if (layout & kAMn) {  // two 64(M) x 64(K) boxes
                tma_load_2d(smem_u32(sa + s * kTileBytes), ma, full, (int)m0, kc);
                tma_load_2d(smem_u32(sa + s * kTileBytes + 8192), ma, full, (int)m0 + 64, kc);
            } else {
                tma_load_2d(smem_u32(sa + s * kTileBytes), ma, full, kc, (int)m0);
            }
            if (layout & kBMn) {
                tma_load_2d(smem_u32(sb + s * kTileBytes), mb, full, (int)n0, kc);
                tma_load_2d(smem_u32(sb + s * kTileBytes + 8192), mb, full, (int)n0 + 64, kc);
            } else {
                tma_load_2d(smem_u32(sb + s * kTileBytes), mb, full, kc, (int)n0);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer ----
        const bool amn = layout & kAMn, bmn = layout & kBMn;
        // UMMA N = n_eff (BN, or N rounded up to 16 for a narrow K-major B)
        const uint32_t idesc = (instr_desc<KIND>() & ~(0x3Fu << 17)) | ((n_eff >> 3) << 17) | (amn ? 1u << 15 : 0u) |
                               (bmn ? 1u << 16 : 0u);
        for (int it = 0; it < total; ++it) {
            const int s = it % kStages;
            mbar_wait(smem_u32(&bars[s]), (it / kStages) & 1);
            tc_fence_after();
            const uint32_t a_base = smem_u32(sa + s * kTileBytes), b_base = smem_u32(sb + s * kTileBytes);
#pragma unroll
            for (int k = 0; k < 4; ++k) {  // 4 K-steps per 64-row stage (UMMA_K = 16 bf16 | 8 tf32)
                umma<KIND>(tmem, op_desc(a_base, k, amn), op_desc(b_base, k, bmn), idesc, (it > 0 || k > 0) ? 1u : 0u);
            }
            umma_commit(smem_u32(&bars[kStages + s]));  // smem stage free once these MMAs retire
        }
        umma_commit(smem_u32(&bars[2 * kStages]));     // accumulator complete
    }
    __syncwarp();

    // ---- epilogue: TMEM -> registers -> fused elementwise -> HBM ----
    mbar_wait(smem_u32(&bars[2 * kStages]), 0);
    tc_fence_after();
    // 8 epilogue warps: warp w reads TMEM lane quadrant w % 4 (hardware rule)
    // and column half w / 4, so twice the memory-level parallelism of one
    // warpgroup while the other CTA on the SM keeps the tensor pipe busy.
    constexpr int kGroups = NT / 128, kCols = BN / kGroups;
    const int quad = warp % 4, grp = warp / 4;
    const uint64_t m = m0 + quad * 32 + lane;
    const uint32_t lane_base = tmem + ((uint32_t)(quad * 32) << 16);
    // Row-major C: 16 consecutive columns per thread -> 16-byte vector stores
    // when the row pitch allows; C^T: lanes hold consecutive rows -> each
    // scalar store instruction is one coalesced warp-wide segment.
    if (cfold) {
        cluster_fold_epilogue<NT>(epi, reinterpret_cast<float*>(smem), lane_base, quad * 32 + lane, grp * kCols,
                                  kCols, m0, n0, M, N);
        tc_fence_before();
        __syncthreads();
        if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
        return;
    }
    const int es = epi.out_bf16 ? 2 : 4;
    const bool vec_c = epi.c && ((epi.ldc * es) % 16 == 0) && ((reinterpret_cast<uintptr_t>(epi.c) & 15) == 0);
    const bool vec_act = epi.mode == EPI_TANH_GRAD && ((epi.ldact * es) % 16 == 0) &&
                         ((reinterpret_cast<uintptr_t>(epi.act) & 15) == 0);
    ActPrefetch pf{epi.mode == EPI_TANH_GRAD && epi.out_bf16 && vec_act && m < M,
                   static_cast<const __nv_bfloat16*>(epi.act) + m * epi.ldact, {}};
    if (pf.on && n0 + grp * kCols + 16 <= N) pf.load(n0 + grp * kCols);
#pragma unroll 1
    for (int c0 = grp * kCols; c0 < (grp + 1) * kCols; c0 += 16) {
        const uint4 cur0 = pf.buf[0], cur1 = pf.buf[1];
        const bool have = pf.on && n0 + c0 + 16 <= N;
        if (pf.on && c0 + 16 < (grp + 1) * kCols && n0 + c0 + 32 <= N) pf.load(n0 + c0 + 16);
        uint32_t r[16];
        tmem_ld16(lane_base + c0, r);
        if (m >= M) continue;
        epi_chunk(epi, m, n0 + c0, N, r, vec_c, vec_act, have, cur0, cur1);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(BN));
    }
}

// Fused epilogue for 16 consecutive columns [nb, nb+16) of row m, accumulator
// values r (fp32 bits): bias / tanh / tanh-derivative, then row-major C
// (16-byte vector stores when aligned) and/or C^T (lanes = consecutive rows,
// so each scalar store instruction is one coalesced warp segment).
__device__ __forceinline__ void epi_chunk_generic(const EpiArgs& epi, uint64_t m, uint64_t nb, uint64_t N,
                                               const uint32_t (&r)[16], bool vec_c, bool vec_act) {
    {
        float v[16];
        float act[16];
        if (epi.mode == EPI_TANH_GRAD) {
            if (vec_act && nb + 16 <= N) {  // 16 activations in one or two 16-byte loads
                if (epi.out_bf16) {
                    const uint4* src =
                        reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(epi.act) + m * epi.ldact + nb);
                    uint4 u[2] = {src[0], src[1]};
                    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(u);
#pragma unroll
                    for (int j = 0; j < 16; ++j) act[j] = __bfloat162float(h[j]);
                } else {
                    const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(epi.act) + m * epi.ldact + nb);
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        float4 f = src[j];
                        act[4 * j] = f.x, act[4 * j + 1] = f.y, act[4 * j + 2] = f.z, act[4 * j + 3] = f.w;
                    }
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) act[j] = nb + j < N ? load_act(epi, m, nb + j) : 0.f;
            }
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const uint64_t n = nb + j;
            float x = __uint_as_float(r[j]);
            if (n < N) {
                if (epi.mode == EPI_BIAS) x += epi.bias[n];
                else if (epi.mode == EPI_BIAS_TANH) x = tanhf(x + epi.bias[n]);
                else if (epi.mode == EPI_TANH_GRAD) x = x * (1.0f - act[j] * act[j]);
            }
            v[j] = x;
        }
        if (epi.c) {
            if (vec_c && nb + 16 <= N) {
                if (epi.out_bf16) {
                    uint4* dst = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(epi.c) + m * epi.ldc + nb);
                    uint32_t p[8];
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
                        p[j] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    dst[0] = make_uint4(p[0], p[1], p[2], p[3]);
                    dst[1] = make_uint4(p[4], p[5], p[6], p[7]);
                } else {
                    float4* dst = reinterpret_cast<float4*>(static_cast<float*>(epi.c) + m * epi.ldc + nb);
#pragma unroll
                    for (int j = 0; j < 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                }
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j)
                    if (nb + j < N) store_out(epi.c, m * epi.ldc + nb + j, v[j], epi.out_bf16);
            }
        }
        if (epi.ct) {
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (nb + j < N) store_out(epi.ct, (nb + j) * epi.ldct + m, v[j], epi.out_bf16);
        }
    }
}


__device__ __forceinline__ float tanh_fast(float x) {
    float y;
    asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Full 16-column chunk, mode and output type fixed at compile time: bias read
// with four 16-byte broadcast loads when aligned, hardware tanh when the output
// is bf16 (tanh.approx's 2^-10.7 relative error is below bf16's half ulp), and
// C^T written by pointer increment (one coalesced 64-byte warp segment per
// column). No per-element bounds checks.
template <int MODE, bool BF>
__device__ __forceinline__ void epi_chunk_fast(const EpiArgs& epi, uint64_t m, uint64_t nb, const uint32_t (&r)[16],
                                               bool vec_c, bool vec_act, bool vec_bias, bool have_pre, uint4 pre0,
                                               uint4 pre1) {
    float v[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) v[j] = __uint_as_float(r[j]);
    if constexpr (MODE == EPI_BIAS || MODE == EPI_BIAS_TANH) {
        float b[16];
        if (vec_bias) {
            const float4* bp = reinterpret_cast<const float4*>(epi.bias + nb);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float4 f = __ldg(bp + j);
                b[4 * j] = f.x, b[4 * j + 1] = f.y, b[4 * j + 2] = f.z, b[4 * j + 3] = f.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) b[j] = __ldg(epi.bias + nb + j);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            v[j] += b[j];
            if constexpr (MODE == EPI_BIAS_TANH) v[j] = BF ? tanh_fast(v[j]) : tanhf(v[j]);
        }
    } else if constexpr (MODE == EPI_TANH_GRAD) {
        float a[16];
        if (vec_act) {
            if constexpr (BF) {
                const uint4* src = reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(epi.act) + m * epi.ldact + nb);
                uint4 u[2];
                if (have_pre) u[0] = pre0, u[1] = pre1;  // prefetched by the caller
                else u[0] = src[0], u[1] = src[1];
                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(u);
#pragma unroll
                for (int j = 0; j < 16; ++j) a[j] = __bfloat162float(h[j]);
            } else {
                const float4* src = reinterpret_cast<const float4*>(static_cast<const float*>(epi.act) + m * epi.ldact + nb);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const float4 f = src[j];
                    a[4 * j] = f.x, a[4 * j + 1] = f.y, a[4 * j + 2] = f.z, a[4 * j + 3] = f.w;
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) a[j] = load_act(epi, m, nb + j);
        }
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = v[j] * (1.0f - a[j] * a[j]);
    }
    if constexpr (BF) {
        uint32_t p[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            __nv_bfloat162 h = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
            p[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        if (epi.c) {
            __nv_bfloat16* row = static_cast<__nv_bfloat16*>(epi.c) + m * epi.ldc + nb;
            if (vec_c) {
                uint4* dst = reinterpret_cast<uint4*>(row);
                dst[0] = make_uint4(p[0], p[1], p[2], p[3]);
                dst[1] = make_uint4(p[4], p[5], p[6], p[7]);
            } else {
                const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(p);
#pragma unroll
                for (int j = 0; j < 16; ++j) row[j] = h[j];
            }
        }
        if (epi.ct) {
            const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(p);
            __nv_bfloat16* col = static_cast<__nv_bfloat16*>(epi.ct) + nb * epi.ldct + m;
#pragma unroll
            for (int j = 0; j < 16; ++j, col += epi.ldct) *col = h[j];
        }
    } else {
        if (epi.c) {
            float* row = static_cast<float*>(epi.c) + m * epi.ldc + nb;
            if (vec_c) {
                float4* dst = reinterpret_cast<float4*>(row);
#pragma unroll
                for (int j = 0; j < 4; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < 16; ++j) row[j] = v[j];
            }
        }
        if (epi.ct) {
            float* col = static_cast<float*>(epi.ct) + nb * epi.ldct + m;
#pragma unroll
            for (int j = 0; j < 16; ++j, col += epi.ldct) *col = v[j];
        }
    }
}

__device__ __forceinline__ void epi_chunk(const EpiArgs& epi, uint64_t m, uint64_t nb, uint64_t N,
                                          const uint32_t (&r)[16], bool vec_c, bool vec_act, bool have_pre, uint4 pre0,
                                          uint4 pre1) {
    if (nb + 16 > N) {
        epi_chunk_generic(epi, m, nb, N, r, vec_c, vec_act);
        return;
    }
    const bool vec_bias = epi.bias && ((reinterpret_cast<uintptr_t>(epi.bias + nb) & 15) == 0);
#define SYNK_EPI_CASE(MODE)                                                       \
    case MODE:                                                                    \
        if (epi.out_bf16) epi_chunk_fast<MODE, true>(epi, m, nb, r, vec_c, vec_act, vec_bias, have_pre, pre0, pre1); \
        else epi_chunk_fast<MODE, false>(epi, m, nb, r, vec_c, vec_act, vec_bias, have_pre, pre0, pre1); \
        return;
    switch (epi.mode) {
        SYNK_EPI_CASE(EPI_STORE)
        SYNK_EPI_CASE(EPI_BIAS)
        SYNK_EPI_CASE(EPI_BIAS_TANH)
        SYNK_EPI_CASE(EPI_TANH_GRAD)
    }
#undef SYNK_EPI_CASE
    epi_chunk_generic(epi, m, nb, N, r, vec_c, vec_act);
}

// ---- persistent bf16 kernel: 128 x 256 tiles, double-buffered TMEM accumulators -------
// One CTA per SM loops over tiles (static round robin). The 128x256x16 UMMA
// reads 12 KB of operands per 128 cycles (96 B/clk, inside the 128 B/clk
// shared-memory budget that a 128x128 tile saturates), and the two 256-column
// accumulators let the epilogue warpgroup drain tile i while the MMA warp
// already accumulates tile i+1.
// 12 warps: 0 TMA, 1 MMA, 2 TMEM allocator, 3 idle, 4..11 epilogue (two warps
// per TMEM lane quadrant, each draining half of the 256 accumulator columns).
//
// PAIR = 2: a CTA pair (cluster of 2 on one TPC) computes 256 x 256 tiles with
// tcgen05.mma.cta_group::2 issued by the even CTA: each CTA stages its own 128
// rows of A and 128 of the 256 B rows (32 KB per stage instead of 48: six
// stages, a third less L2 -> SM traffic per flop), the TMA loads of both CTAs
// complete on the leader's full barrier, the MMA commits arrive on both CTAs'
// barriers (multicast), and each CTA drains its own 128 accumulator rows from
// its own TMEM; the leader's TMEM-empty barrier counts both CTAs' epilogue warps.
constexpr int PBN = 256, PThreads = 384, PEpiThreads = 256;
// ACT: the short-K tanh-derivative products (C5's dX with K = d_{l+1} <= 128)
// are bound by the activation read of their epilogue, not by the tensor
// cores: the producer TMA-stages each tile's 128 x 256 activation block into
// one of two shared-memory buffers (SWIZZLE_128B, 64-column boxes) while the
// epilogue drains the previous tile, instead of every epilogue thread loading
// its 256 B from HBM after the previous tile's stores. Two operand stages
// suffice for K <= 128.
template <int PAIR, bool ACT = false>
struct PCfg {
    static constexpr int kStages = ACT ? 2 : (PAIR == 2 ? 6 : 4);
    static constexpr int kA = 128 * 128;                // bytes per stage: this CTA's 128 A rows
    static constexpr int kB = (PBN / PAIR) * 128;       // this CTA's B rows (256 or 128), 128 B each
    static constexpr int kTileM = 128 * PAIR;
    static constexpr int kActBuf = ACT ? 128 * PBN * 2 : 0;  // one activation tile (bf16)
    static constexpr size_t kSmem = (size_t)kStages * (kA + kB) + 2 * (size_t)kActBuf + 1024 + 256;
};
constexpr int PStages = PCfg<1>::kStages;  // (1-CTA layout, host-side sizes)
constexpr int PA = PCfg<1>::kA, PB = PCfg<1>::kB;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t map_to_rank(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// TMA load whose completion is counted on the pair leader's barrier (bar is a
// shared::cluster address in the leader CTA).
__device__ __forceinline__ void tma_load_2d_pair(uint32_t dst, const CUtensorMap* map, uint32_t bar, int x, int y) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, "
        "%4}], [%2];" ::"r"(dst),
        "l"(map), "r"(bar), "r"(x), "r"(y)
        : "memory");
}
__device__ __forceinline__ void umma_pair(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// commit the leader's MMAs to the barrier at `bar`'s offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint32_t bar) {
    asm volatile(
        "{\n.reg .b16 m;\nmov.b16 m, 3;\n"
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n}\n" ::"r"(
            bar)
        : "memory");
}

template <int PAIR, bool ACT>
__global__ void __launch_bounds__(PThreads, 1)
    gemm_tc_persistent_kernel(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                              const __grid_constant__ CUtensorMap tact, uint32_t M, uint32_t N, uint32_t K,
                              EpiArgs epi, uint32_t layout) {
    using PC = PCfg<PAIR, ACT>;
    constexpr int kStages = PC::kStages, kA = PC::kA, kB = PC::kB;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint8_t* sa = smem;
    uint8_t* sb = smem + kStages * kA;
    uint8_t* sact = sb + kStages * kB;  // [2][4 boxes of 128 rows x 128 B] (ACT only)
    uint64_t* bars = reinterpret_cast<uint64_t*>(sact + 2 * PC::kActBuf);
    uint64_t* full = bars;                 // [kStages]
    uint64_t* empty = bars + kStages;      // [kStages]
    uint64_t* tfull = bars + 2 * kStages;  // [2]
    uint64_t* tempty = tfull + 2;          // [2]
    uint64_t* act_full = tempty + 2;       // [2] (ACT)
    uint64_t* act_empty = act_full + 2;    // [2] (ACT)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_empty + 2);
    const uint32_t rank = PAIR == 2 ? cluster_rank() : 0u;
    const bool leader = rank == 0;
    const uint32_t unit = blockIdx.x / PAIR, units = gridDim.x / PAIR;  // pair (or CTA) index / count
    synk::release_dependent_grid();  // PDL: see gemm_tc_kernel

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    constexpr int kBK = 64;  // bf16 elements per 128-byte K block
    const uint32_t num_m = (M + PC::kTileM - 1) / PC::kTileM, num_n = (N + PBN - 1) / PBN;
    const uint32_t tiles = num_m * num_n;
    const int num_kb = (int)((K + kBK - 1) / kBK);

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&tfull[b]), 1);
            // every epilogue warp of the pair arrives (one elected lane each)
            mbar_init(smem_u32(&tempty[b]), PAIR * (PEpiThreads / 32));
            mbar_init(smem_u32(&act_full[b]), 1);
            mbar_init(smem_u32(&act_empty[b]), PEpiThreads / 32);  // this CTA's epilogue warps
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_map(&ta);
        prefetch_map(&tb);
        if (ACT) prefetch_map(&tact);
    }
    __syncwarp();
    // the pair's TMEM allocation touches both SMs' allocator state: both CTAs
    // must be running (and past their prologue) before either allocates
    if constexpr (PAIR == 2) cluster_sync_all();
    if (warp == 2) {
        if constexpr (PAIR == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(2 * PBN));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                         "r"(2 * PBN));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    tc_fence_before();
    if constexpr (PAIR == 2) cluster_sync_all();  // the peer's barriers exist before any remote arrive / TMA signal
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    synk::wait_prerequisite_grid();  // PDL: prologue overlapped the previous kernel's tail

    if (warp == 0 && lane == 0) {
        // ---- TMA producer (both CTAs: this CTA's A rows and B rows) ----
        uint32_t it = 0, tl = 0;
        for (uint32_t t = unit; t < tiles; t += units, ++tl) {
            const int m0 = (int)((t / num_n) * PC::kTileM + rank * 128), n0 = (int)((t % num_n) * PBN + rank * (PBN / PAIR));
            if constexpr (ACT) {  // this CTA's 128 x 256 activation tile, two tiles ahead at most
                const uint32_t ab = tl & 1;
                mbar_wait(smem_u32(&act_empty[ab]), ((tl >> 1) & 1) ^ 1);
                mbar_expect_tx(smem_u32(&act_full[ab]), PC::kActBuf);
#pragma unroll
                for (int j = 0; j < PBN / 64; ++j)
                    tma_load_2d(smem_u32(sact + ab * PC::kActBuf + j * 16384), &tact, smem_u32(&act_full[ab]),
                                (int)((t % num_n) * PBN) + 64 * j, m0);
            }
            for (int kb = 0; kb < num_kb; ++kb, ++it) {
                const int s = it % kStages;
                mbar_wait(smem_u32(&empty[s]), ((it / kStages) & 1) ^ 1);
                uint32_t fb = smem_u32(&full[s]);
                if (leader) mbar_expect_tx(fb, PAIR * (kA + kB));  // both CTAs' bytes land on the leader's barrier
                if constexpr (PAIR == 2) fb = map_to_rank(fb, 0);
                auto load = [&](uint32_t dst, const CUtensorMap* map, int x, int y) {
                    if constexpr (PAIR == 2) tma_load_2d_pair(dst, map, fb, x, y);
                    else tma_load_2d(dst, map, fb, x, y);
                };
                if (layout & kAMn) {  // 64(M) x 64(K) boxes along M
                    for (int j = 0; j < 128 / 64; ++j) load(smem_u32(sa + s * kA + j * 8192), &ta, m0 + 64 * j, kb * kBK);
                } else {
                    load(smem_u32(sa + s * kA), &ta, kb * kBK, m0);
                }
                if (layout & kBMn) {
                    for (int j = 0; j < PBN / PAIR / 64; ++j)
                        load(smem_u32(sb + s * kB + j * 8192), &tb, n0 + 64 * j, kb * kBK);
                } else {
                    load(smem_u32(sb + s * kB), &tb, kb * kBK, n0);
                }
            }
        }
    } else if (warp == 1 && lane == 0 && leader) {
        // ---- MMA issuer (the pair leader: UMMA M = 128 * PAIR) ----
        const bool amn = layout & kAMn, bmn = layout & kBMn;
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | (amn ? 1u << 15 : 0u) | (bmn ? 1u << 16 : 0u) |
                               ((uint32_t)(PBN >> 3) << 17) | ((uint32_t)(PC::kTileM >> 4) << 24);
        uint32_t it = 0, tl = 0;
        for (uint32_t t = unit; t < tiles; t += units, ++tl) {
            const uint32_t acc = tl & 1;
            mbar_wait(smem_u32(&tempty[acc]), ((tl >> 1) & 1) ^ 1);  // both CTAs drained this buffer
            tc_fence_after();
            const uint32_t d = tmem + acc * PBN;
            for (int kb = 0; kb < num_kb; ++kb, ++it) {
                const int s = it % kStages;
                mbar_wait(smem_u32(&full[s]), (it / kStages) & 1);
                tc_fence_after();
                const uint32_t a_base = smem_u32(sa + s * kA), b_base = smem_u32(sb + s * kB);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    if constexpr (PAIR == 2)
                        umma_pair(d, op_desc(a_base, k, amn), op_desc(b_base, k, bmn), idesc, (kb > 0 || k > 0) ? 1u : 0u);
                    else
                        umma<0>(d, op_desc(a_base, k, amn), op_desc(b_base, k, bmn), idesc, (kb > 0 || k > 0) ? 1u : 0u);
                }
                if constexpr (PAIR == 2) umma_commit_pair(smem_u32(&empty[s]));
                else umma_commit(smem_u32(&empty[s]));
            }
            if constexpr (PAIR == 2) umma_commit_pair(smem_u32(&tfull[acc]));
            else umma_commit(smem_u32(&tfull[acc]));
        }
    } else if (warp >= 4) {
        // ---- epilogue: warps 4..11; warp w owns TMEM lane quadrant w % 4 and
        // accumulator columns [128 * half, 128 * half + 128), half = (w - 4) / 4 ----
        const int quad = warp % 4, half = (warp - 4) / 4;
        const int es = epi.out_bf16 ? 2 : 4;
        const bool vec_c = epi.c && ((epi.ldc * es) % 16 == 0) && ((reinterpret_cast<uintptr_t>(epi.c) & 15) == 0);
        const bool vec_act = epi.mode == EPI_TANH_GRAD && ((epi.ldact * es) % 16 == 0) &&
                             ((reinterpret_cast<uintptr_t>(epi.act) & 15) == 0);
        const bool pre_ok = epi.mode == EPI_TANH_GRAD && epi.out_bf16 && vec_act;
        // 32-byte alignment of every 16-column chunk (bf16: 32 B) for the 256-bit paths
        const bool act32 = pre_ok && (epi.ldact * 2) % 32 == 0 && (reinterpret_cast<uintptr_t>(epi.act) & 31) == 0;
        const bool c32 = pre_ok && epi.c && (epi.ldc * 2) % 32 == 0 && (reinterpret_cast<uintptr_t>(epi.c) & 31) == 0;
        // TMEM-empty arrival: one elected lane per warp, on the pair leader's barrier
        const uint32_t tempty_at[2] = {PAIR == 2 ? map_to_rank(smem_u32(&tempty[0]), 0) : smem_u32(&tempty[0]),
                                       PAIR == 2 ? map_to_rank(smem_u32(&tempty[1]), 0) : smem_u32(&tempty[1])};
        auto drained = [&](uint32_t acc) {
            tc_fence_before();
            __syncwarp();
            if (lane == 0)
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(tempty_at[acc])
                             : "memory");
        };
        uint32_t tl = 0;
        for (uint32_t t = unit; t < tiles; t += units, ++tl) {
            const uint32_t acc = tl & 1;
            const uint64_t m0 = (t / num_n) * PC::kTileM + rank * 128, n0 = (uint64_t)(t % num_n) * PBN;
            const uint64_t m = m0 + quad * 32 + lane;
            const uint32_t base = tmem + acc * PBN + ((uint32_t)(quad * 32) << 16);
            const int cbeg = half * (PBN / 2), cend = cbeg + PBN / 2;
            if constexpr (ACT) {
                const uint32_t ab = tl & 1;
                mbar_wait(smem_u32(&act_full[ab]), (tl >> 1) & 1);
                mbar_wait(smem_u32(&tfull[acc]), (tl >> 1) & 1);
                tc_fence_after();
                const int rl = quad * 32 + lane;  // row within this CTA's 128
                const uint32_t abase = smem_u32(sact + ab * PC::kActBuf) + rl * 128;
                const bool row = m < M;
#pragma unroll 1
                for (int k = 0; k < 8; ++k) {
                    uint32_t r[16];
                    tmem_ld16(base + cbeg + 16 * k, r);
                    const int c = cbeg + 16 * k;          // tile column of the chunk
                    const uint32_t u = (uint32_t)(c % 64) / 8;  // 16-byte unit within the 128-byte row
                    const uint32_t box = abase + (uint32_t)(c / 64) * 16384;
                    uint4 a0, a1;
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(a0.x), "=r"(a0.y), "=r"(a0.z), "=r"(a0.w)
                                 : "r"(box + ((u ^ (rl & 7)) << 4)));
                    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                 : "=r"(a1.x), "=r"(a1.y), "=r"(a1.z), "=r"(a1.w)
                                 : "r"(box + (((u + 1) ^ (rl & 7)) << 4)));
                    if (!row || n0 + c >= N) continue;
                    if (c32 && n0 + c + 16 <= N) {
                        const __nv_bfloat16* h0 = reinterpret_cast<const __nv_bfloat16*>(&a0);
                        const __nv_bfloat16* h1 = reinterpret_cast<const __nv_bfloat16*>(&a1);
                        uint32_t w[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            const float x0 = __bfloat162float(j < 4 ? h0[2 * j] : h1[2 * j - 8]);
                            const float x1 = __bfloat162float(j < 4 ? h0[2 * j + 1] : h1[2 * j - 7]);
                            const float v0 = __uint_as_float(r[2 * j]) * (1.0f - x0 * x0);
                            const float v1 = __uint_as_float(r[2 * j + 1]) * (1.0f - x1 * x1);
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(v0, v1);
                            w[j] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        st256(static_cast<__nv_bfloat16*>(epi.c) + m * epi.ldc + n0 + c, w);
                        if (epi.ct) {
                            __nv_bfloat16* col = static_cast<__nv_bfloat16*>(epi.ct) + (n0 + c) * epi.ldct + m;
                            const __nv_bfloat16* hw = reinterpret_cast<const __nv_bfloat16*>(w);
#pragma unroll
                            for (int j = 0; j < 16; ++j, col += epi.ldct) *col = hw[j];
                        }
                    } else {
                        epi_chunk(epi, m, n0 + c, N, r, vec_c, vec_act, true, a0, a1);
                    }
                }
                // this warp is done with the activation buffer and the accumulator
                __syncwarp();
                if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&act_empty[ab])) : "memory");
                drained(acc);
                continue;
            }
            if (pre_ok && n0 + cend <= N) {  // warp-uniform: tcgen05.ld is .sync.aligned
                // tanh-derivative epilogue, whole half-row inside the matrix:
                // the thread's 128 activations (256 B, 16 loads) are issued
                // BEFORE waiting for the accumulator, so their HBM latency
                // hides behind this tile's MMAs -- 64 KB in flight per SM
                // instead of one 32-byte chunk per thread (the short-K dX
                // products are bound by this read, not by the tensor cores).
                const uint4* src =
                    reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(epi.act) + m * epi.ldact + n0 + cbeg);
                const bool row = m < M;
                uint4 a[16];
#pragma unroll
                for (int i = 0; i < 16; i += 2) {
                    if (row && act32) {
                        ld256_stream(src + i, a[i], a[i + 1]);
                    } else {
                        a[i] = row ? __ldcs(src + i) : make_uint4(0, 0, 0, 0);
                        a[i + 1] = row ? __ldcs(src + i + 1) : make_uint4(0, 0, 0, 0);
                    }
                }
                mbar_wait(smem_u32(&tfull[acc]), (tl >> 1) & 1);
                tc_fence_after();
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    uint32_t r[16];
                    tmem_ld16(base + cbeg + 16 * k, r);
                    if (!row) continue;
                    if (c32) {  // the 16 bf16 results of the chunk as one 32-byte store
                        float v[16];
                        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&a[2 * k]);
                        uint32_t w[8];
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            const float x = __bfloat162float(h[j]);
                            v[j] = __uint_as_float(r[j]) * (1.0f - x * x);
                        }
#pragma unroll
                        for (int j = 0; j < 8; ++j) {
                            __nv_bfloat162 b2 = __floats2bfloat162_rn(v[2 * j], v[2 * j + 1]);
                            w[j] = *reinterpret_cast<uint32_t*>(&b2);
                        }
                        st256(static_cast<__nv_bfloat16*>(epi.c) + m * epi.ldc + n0 + cbeg + 16 * k, w);
                        if (epi.ct) {
                            __nv_bfloat16* col = static_cast<__nv_bfloat16*>(epi.ct) + (n0 + cbeg + 16 * k) * epi.ldct + m;
                            const __nv_bfloat16* hw = reinterpret_cast<const __nv_bfloat16*>(w);
#pragma unroll
                            for (int j = 0; j < 16; ++j, col += epi.ldct) *col = hw[j];
                        }
                    } else {
                        epi_chunk_fast<EPI_TANH_GRAD, true>(epi, m, n0 + cbeg + 16 * k, r, vec_c, true, false, true,
                                                            a[2 * k], a[2 * k + 1]);
                    }
                }
                drained(acc);
                continue;
            }
            mbar_wait(smem_u32(&tfull[acc]), (tl >> 1) & 1);
            tc_fence_after();
            ActPrefetch pf{pre_ok && m < M, static_cast<const __nv_bfloat16*>(epi.act) + m * epi.ldact, {}};
            if (pf.on && n0 + cbeg + 16 <= N) pf.load(n0 + cbeg);
#pragma unroll 1
            for (int c0 = cbeg; c0 < cend; c0 += 16) {
                const uint4 cur0 = pf.buf[0], cur1 = pf.buf[1];
                const bool have = pf.on && n0 + c0 + 16 <= N;
                if (pf.on && c0 + 16 < cend && n0 + c0 + 32 <= N) pf.load(n0 + c0 + 16);
                uint32_t r[16];
                tmem_ld16(base + c0, r);
                if (m < M && n0 + c0 < N) epi_chunk(epi, m, n0 + c0, N, r, vec_c, vec_act, have, cur0, cur1);
            }
            drained(acc);
        }
    }
    __syncwarp();
    tc_fence_before();
    if constexpr (PAIR == 2) {
        cluster_sync_all();  // both CTAs done with the pair's TMEM before it is freed
        if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * PBN));
    } else {
        __syncthreads();
        if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * PBN));
    }
}

// ---- host side: tensor maps ---------------------------------------------------------

// MN-major bf16 operand stored as k_rows x mn (mn contiguous, leading
// dimension ld elements); box = 64 MN elements (128 B) x 64 K rows.
int make_map_mn(CUtensorMap* map, const void* base, uint64_t k_rows, uint64_t mn, uint64_t ld) {
    EncodeFn enc = encoder();
    SYNK_REQUIRE(enc != nullptr, SYNK_ECUDA, "cuTensorMapEncodeTiled unavailable");
    SYNK_REQUIRE(((uintptr_t)base % 16) == 0 && (ld * 2) % 16 == 0, SYNK_EARG,
                 "gemm_tc: operand base and row pitch must be 16-byte aligned");
    cuuint64_t dims[2] = {mn, k_rows};
    cuuint64_t strides[1] = {ld * 2};
    cuuint32_t box[2] = {64, 64};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SYNK_REQUIRE(r == CUDA_SUCCESS, SYNK_ECUDA, "cuTensorMapEncodeTiled (MN-major) failed");
    return SYNK_OK;
}

constexpr size_t kSmemBytes = 2 * kStages * kTileBytes + 1024 /*align*/ + 256 /*barriers*/;

// Programmatic dependent launch between back-to-back tcgen05 GEMMs: each one
// releases its dependents at CTA entry and waits (griddepcontrol.wait) after
// its barrier / TMEM prologue, so the next GEMM's launch and prologue overlap
// this one's tail. SYNK_GEMM_PDL=0 launches them plainly (A/B).
bool pdl_gemm() {
    static const bool on = [] {
        const char* e = getenv("SYNK_GEMM_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int KIND>
int launch(synk_dev* d, int passes, const CUtensorMap& a0, const CUtensorMap& a1, const CUtensorMap& b0,
           const CUtensorMap& b1, uint64_t M, uint64_t N, uint64_t K, const EpiArgs& e, uint32_t splits = 1,
           uint32_t kb_per = 0x7fffffffu, uint32_t layout = 0, int cfold = 0, uint32_t n_eff = BN) {
    // Epilogue-heavy launches (short K, or the tanh-derivative reading the
    // activation tile) get 8 epilogue warps; MMA-bound ones keep 4 warps and
    // the full register budget. SYNK_GEMM_WARPS=4|8 overrides (A/B runs).
    static const int forced = [] {
        const char* e = getenv("SYNK_GEMM_WARPS");
        return e ? atoi(e) : 0;
    }();
    const bool wide = forced ? forced == 8 : (K <= 512 || e.mode == EPI_TANH_GRAD);
    dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), splits);
    if (cfold) {  // the split CTAs of a tile form one cluster (DSMEM fold)
        auto kern = wide ? gemm_tc_kernel<KIND, 256> : gemm_tc_kernel<KIND, 128>;
        if (int rc = synk::ensure_max_smem((const void*)kern, d->device, (int)kSmemBytes); rc) return rc;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(wide ? 256 : 128);
        cfg.dynamicSmemBytes = kSmemBytes;
        cfg.stream = d->stream;
        cudaLaunchAttribute attr[2];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 1;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = splits;
        attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl_gemm() && d->pdl_armed ? 2 : 1;
        SYNK_CU(cudaLaunchKernelEx(&cfg, kern, a0, a1, b0, b1, passes, (uint32_t)M, (uint32_t)N, (uint32_t)K, e, kb_per,
                                   layout, 1, n_eff));
        d->pdl_armed = pdl_gemm();
        return SYNK_OK;
    }
    if (wide) {
        if (int rc = synk::ensure_max_smem((const void*)gemm_tc_kernel<KIND, 256>, d->device, (int)kSmemBytes); rc)
            return rc;
        gemm_tc_kernel<KIND, 256><<<grid, 256, kSmemBytes, d->stream>>>(a0, a1, b0, b1, passes, (uint32_t)M, (uint32_t)N,
                                                                       (uint32_t)K, e, kb_per, layout, 0, n_eff);
    } else {
        if (int rc = synk::ensure_max_smem((const void*)gemm_tc_kernel<KIND, 128>, d->device, (int)kSmemBytes); rc)
            return rc;
        gemm_tc_kernel<KIND, 128><<<grid, 128, kSmemBytes, d->stream>>>(a0, a1, b0, b1, passes, (uint32_t)M, (uint32_t)N,
                                                                       (uint32_t)K, e, kb_per, layout, 0, n_eff);
    }
    SYNK_LAUNCHED("gemm_tc_kernel");
    d->pdl_armed = pdl_gemm();
    return SYNK_OK;
}

// ---- operand preparation: tf32 hi/lo split, bf16 cast, optional transpose -------------

__device__ __forceinline__ float to_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

// out[r][c] (ld_out, zero-padded to cols_pad) from in (rows x cols, ld_in), or
// the transpose (out[c][r], cols x rows, zero-padded to rows_pad) when trans.
// Tiled 32x32 through shared memory so both sides stay coalesced.
template <class In>
__global__ void __launch_bounds__(256) prep_kernel(const In* __restrict__ in, uint64_t rows, uint64_t cols,
                                                   uint64_t ld_in, int trans, int mode, void* __restrict__ out_hi,
                                                   float* __restrict__ out_lo, uint64_t out_rows, uint64_t out_cols,
                                                   uint64_t ld_out) {
    __shared__ float tile[32][33];
    const uint64_t r0 = (uint64_t)blockIdx.y * 32, c0 = (uint64_t)blockIdx.x * 32;
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // 32 x 8
    // load in-tile (input coordinates) covering the output tile
    for (int k = ty; k < 32; k += 8) {
        uint64_t ir, ic;
        if (!trans) { ir = r0 + k; ic = c0 + tx; }
        else { ir = c0 + k; ic = r0 + tx; }  // output (r,c) = input (c,r): tile over output coords
        float v = 0.f;
        if (ir < rows && ic < cols) v = (float)in[ir * ld_in + ic];
        tile[k][tx] = v;
    }
    __syncthreads();
    for (int k = ty; k < 32; k += 8) {
        const uint64_t orow = r0 + k, ocol = c0 + tx;
        if (orow >= out_rows || ocol >= out_cols) continue;
        const float v = trans ? tile[tx][k] : tile[k][tx];
        const uint64_t o = orow * ld_out + ocol;
        if (mode == 0) {  // tf32 split
            const float hi = to_tf32(v);
            static_cast<float*>(out_hi)[o] = hi;
            out_lo[o] = to_tf32(v - hi);
        } else if (mode == 1) {  // bf16 cast
            static_cast<__nv_bfloat16*>(out_hi)[o] = __float2bfloat16_rn(v);
        } else {  // plain fp32 copy (single-pass tf32)
            static_cast<float*>(out_hi)[o] = v;
        }
    }
}

// Split-K fold: C[m, n] = sum_z P[z][m, n] (fixed z order, f64 accumulation)
// + bias[n] for EPI_BIAS; fp32 output.
__global__ void __launch_bounds__(256) splitk_fold_kernel(uint32_t S, uint64_t M, uint64_t N, const float* __restrict__ P,
                                                          float* __restrict__ C, uint64_t ldc, const float* __restrict__ bias) {
    const uint64_t total = M * N;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (uint64_t)gridDim.x * 256) {
        double acc = 0.0;
        for (uint32_t z = 0; z < S; ++z) acc += (double)P[(uint64_t)z * total + i];
        const uint64_t m = i / N, n = i % N;
        float v = (float)acc;
        if (bias) v += bias[n];
        C[m * ldc + n] = v;
    }
}

// One read, two bf16 writes: out = bf16(in) (rows x cols, ld_out) and
// out_t = bf16(in)^T (cols x rows, ld_out_t); either may be null. 64 x 64
// tiles: float4 loads and 8-byte bf16 stores row-major, 32-byte stores for
// the transposed side out of a shared-memory tile.
__global__ void __launch_bounds__(256) prep2_bf16_kernel(const float* __restrict__ in, uint64_t rows, uint64_t cols,
                                                         uint64_t ld_in, __nv_bfloat16* __restrict__ out,
                                                         uint64_t ld_out, __nv_bfloat16* __restrict__ out_t,
                                                         uint64_t ld_out_t, int vec_in,
                                                         const uint64_t* __restrict__ rowmap) {
    // rowmap != nullptr: output row r is input row rowmap[r] (index-fused
    // gather: the batch is read straight from the whole source).
    __shared__ float tile[64][65];
    synk::release_dependent_grid();  // PDL: the first forward GEMM may be scheduled behind it
    __shared__ uint64_t srow[64];
    const uint64_t r0 = (uint64_t)blockIdx.y * 64, c0 = (uint64_t)blockIdx.x * 64;
    const int t = threadIdx.x;
    if (t < 64) srow[t] = r0 + t < rows ? (rowmap ? rowmap[r0 + t] : r0 + t) : 0;
    __syncthreads();
    const int lc = (t % 16) * 4;  // 4 consecutive columns
    // all four passes' loads issued before the first use (4 x 16 B in flight per thread)
    float vv[4][4];
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
        const int lr = t / 16 + 16 * pass;
        const uint64_t r = r0 + lr, c = c0 + lc;
        const uint64_t ri = srow[lr];
        vv[pass][0] = vv[pass][1] = vv[pass][2] = vv[pass][3] = 0.f;
        if (r < rows) {
            if (vec_in && c + 4 <= cols) {
                const float4 f = __ldcs(reinterpret_cast<const float4*>(in + ri * ld_in + c));
                vv[pass][0] = f.x, vv[pass][1] = f.y, vv[pass][2] = f.z, vv[pass][3] = f.w;
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (c + j < cols) vv[pass][j] = in[ri * ld_in + c + j];
            }
        }
    }
#pragma unroll
    for (int pass = 0; pass < 4; ++pass) {
        const int lr = t / 16 + 16 * pass;
        const uint64_t r = r0 + lr, c = c0 + lc;
        const float* v = vv[pass];
#pragma unroll
        for (int j = 0; j < 4; ++j) tile[lr][lc + j] = v[j];
        if (out && r < rows) {
            __nv_bfloat16 h[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) h[j] = __float2bfloat16_rn(v[j]);
            __nv_bfloat16* dst = out + r * ld_out + c;
            if (c + 4 <= cols && ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)) {
                *reinterpret_cast<uint2*>(dst) = *reinterpret_cast<const uint2*>(h);
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (c + j < cols) dst[j] = h[j];
            }
        }
    }
    if (!out_t) return;
    __syncthreads();
    // transposed: thread -> output row c0 + t/4, 16 consecutive input rows
    const int oc = t / 4, seg = (t % 4) * 16;
    const uint64_t orow = c0 + oc;
    if (orow >= cols) return;
    __align__(16) __nv_bfloat16 h[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) h[j] = __float2bfloat16_rn(tile[seg + j][oc]);
    const uint64_t ocol = r0 + seg;
    __nv_bfloat16* dst = out_t + orow * ld_out_t + ocol;
    if (ocol + 16 <= rows && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
        reinterpret_cast<uint4*>(dst)[0] = reinterpret_cast<const uint4*>(h)[0];
        reinterpret_cast<uint4*>(dst)[1] = reinterpret_cast<const uint4*>(h)[1];
    } else {
#pragma unroll
        for (int j = 0; j < 16; ++j)
            if (ocol + j < rows) dst[j] = h[j];
    }
}

// Row-major bf16 cast only (no transpose): 8 consecutive elements per thread
// (two 16-byte loads, one 16-byte store), grid-stride over rows x 8-column
// groups; streaming loads (each f32 is read once).
__global__ void __launch_bounds__(256) cast_bf16_rows_kernel(const float* __restrict__ in, uint64_t rows,
                                                             uint64_t cols, uint64_t ld_in,
                                                             __nv_bfloat16* __restrict__ out, uint64_t ld_out) {
    const uint64_t groups = cols / 8, total = rows * groups;
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < total; i += (uint64_t)gridDim.x * 256) {
        const uint64_t r = i / groups, c = (i - r * groups) * 8;
        const float4* src = reinterpret_cast<const float4*>(in + r * ld_in + c);
        const float4 a = __ldcs(src), b = __ldcs(src + 1);
        __nv_bfloat162 h[4] = {__floats2bfloat162_rn(a.x, a.y), __floats2bfloat162_rn(a.z, a.w),
                               __floats2bfloat162_rn(b.x, b.y), __floats2bfloat162_rn(b.z, b.w)};
        *reinterpret_cast<uint4*>(out + r * ld_out + c) = *reinterpret_cast<const uint4*>(h);
    }
}

}  // namespace

extern "C" {

int synk_gemm_prep2_bf16(synk_dev* d, const float* in, uint64_t rows, uint64_t cols, uint64_t ld_in, void* out,
                         uint64_t ld_out, void* out_t, uint64_t ld_out_t) {
    return synk_gemm_prep2_bf16_rows(d, in, nullptr, rows, cols, ld_in, out, ld_out, out_t, ld_out_t);
}

int synk_gemm_prep2_bf16_rows(synk_dev* d, const float* in, const uint64_t* rowmap, uint64_t rows, uint64_t cols,
                              uint64_t ld_in, void* out, uint64_t ld_out, void* out_t, uint64_t ld_out_t) {
    if (rows == 0 || cols == 0 || (!out && !out_t)) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    if (!rowmap && !out_t && cols % 8 == 0 && ld_in % 4 == 0 && ld_out % 8 == 0 && ((reinterpret_cast<uintptr_t>(in) & 15) == 0) &&
        ((reinterpret_cast<uintptr_t>(out) & 15) == 0)) {
        // cast only: the vectorised streaming kernel (no shared-memory tile)
        const uint64_t total = rows * (cols / 8);
        const unsigned grid = (unsigned)std::min<uint64_t>((total + 255) / 256, (uint64_t)d->num_sms * 8);
        if (int rc = synk::prefer_shared_carveout((const void*)cast_bf16_rows_kernel, d->device); rc) return rc;
        cast_bf16_rows_kernel<<<grid, 256, 0, d->stream>>>(in, rows, cols, ld_in, static_cast<__nv_bfloat16*>(out),
                                                           ld_out);
        SYNK_LAUNCHED("cast_bf16_rows_kernel");
        return SYNK_OK;
    }
    dim3 grid((unsigned)((cols + 63) / 64), (unsigned)((rows + 63) / 64));
    const int vec_in = (ld_in % 4 == 0) && ((reinterpret_cast<uintptr_t>(in) & 15) == 0);
    if (int rc = synk::prefer_shared_carveout((const void*)prep2_bf16_kernel, d->device); rc) return rc;
    prep2_bf16_kernel<<<grid, 256, 0, d->stream>>>(in, rows, cols, ld_in, static_cast<__nv_bfloat16*>(out), ld_out,
                                                   static_cast<__nv_bfloat16*>(out_t), ld_out_t, vec_in, rowmap);
    SYNK_LAUNCHED("prep2_bf16_kernel");
    d->pdl_armed = true;
    return SYNK_OK;
}

int synk_gemm_prep(synk_dev* d, int in_dtype, const void* in, uint64_t rows, uint64_t cols, uint64_t ld_in,
                   int transpose, int mode, void* out_hi, float* out_lo, uint64_t out_rows, uint64_t out_cols,
                   uint64_t ld_out) {
    SYNK_REQUIRE(in_dtype == SYNK_F32 || in_dtype == 3, SYNK_EDTYPE, "gemm_prep: input must be f32 or bf16");
    if (out_rows == 0 || out_cols == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    dim3 grid((unsigned)((out_cols + 31) / 32), (unsigned)((out_rows + 31) / 32));
    if (in_dtype == SYNK_F32)
        prep_kernel<float><<<grid, 256, 0, d->stream>>>((const float*)in, rows, cols, ld_in, transpose, mode, out_hi,
                                                        out_lo, out_rows, out_cols, ld_out);
    else
        prep_kernel<__nv_bfloat16><<<grid, 256, 0, d->stream>>>((const __nv_bfloat16*)in, rows, cols, ld_in, transpose,
                                                                mode, out_hi, out_lo, out_rows, out_cols, ld_out);
    SYNK_LAUNCHED("prep_kernel");
    return SYNK_OK;
}

int synk_gemm_tc(synk_dev* d, int kind, uint64_t M, uint64_t N, uint64_t K, const void* a_hi, const void* a_lo,
                 uint64_t lda, const void* b_hi, const void* b_lo, uint64_t ldb, int epilogue, int out_dtype, void* c,
                 uint64_t ldc, void* ct, uint64_t ldct, const float* bias, const void* act, uint64_t ldact) {
    return synk_gemm_tc2(d, kind, M, N, K, a_hi, a_lo, lda, b_hi, b_lo, ldb, 0, epilogue, out_dtype, c, ldc, ct, ldct,
                         bias, act, ldact);
}

int synk_gemm_tc2(synk_dev* d, int kind, uint64_t M, uint64_t N, uint64_t K, const void* a_hi, const void* a_lo,
                  uint64_t lda, const void* b_hi, const void* b_lo, uint64_t ldb, int layout, int epilogue,
                  int out_dtype, void* c, uint64_t ldc, void* ct, uint64_t ldct, const float* bias, const void* act,
                  uint64_t ldact) {
    SYNK_REQUIRE(kind >= 0 && kind <= 2, SYNK_EARG, "gemm_tc: kind is 0 (bf16), 1 (tf32) or 2 (3xtf32)");
    SYNK_REQUIRE(layout >= 0 && layout <= 3 && (layout == 0 || kind == 0), SYNK_EARG,
                 "gemm_tc: MN-major operands (layout bits) are bf16 only");
    SYNK_REQUIRE(out_dtype == SYNK_F32 || out_dtype == 3, SYNK_EDTYPE, "gemm_tc: output f32 or bf16");
    SYNK_REQUIRE(M < (1ull << 31) && N < (1ull << 31) && K < (1ull << 31), SYNK_EARG, "gemm_tc: dims too large");
    if (M == 0 || N == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    const bool bf16 = kind == 0;
    const uint32_t lay = (uint32_t)layout;
    CUtensorMap a0, a1, b0, b1;
    if (int rc = (lay & kAMn) ? make_map_mn(&a0, a_hi, K, M, lda) : make_map(&a0, a_hi, M, K, lda, bf16); rc) return rc;
    if (int rc = (lay & kBMn) ? make_map_mn(&b0, b_hi, K, N, ldb) : make_map(&b0, b_hi, N, K, ldb, bf16); rc) return rc;
    a1 = a0;
    b1 = b0;
    if (kind == 2) {
        SYNK_REQUIRE(a_lo && b_lo, SYNK_EARG, "gemm_tc: 3xtf32 needs lo parts");
        if (int rc = make_map(&a1, a_lo, M, K, lda, false); rc) return rc;
        if (int rc = make_map(&b1, b_lo, N, K, ldb, false); rc) return rc;
    }
    EpiArgs e{epilogue, out_dtype == 3, c, ldc, ct, ldct, bias, act, ldact};
    if (K == 0) return synk::fail(SYNK_EARG, "gemm_tc: K must be > 0");
    // Wide bf16 problems: persistent 128x256 tiles (SYNK_GEMM_PERSISTENT=0 disables).
    // Every bf16 product with N > 128 (short-K, epilogue-bound ones included:
    // the persistent kernel overlaps tile i's epilogue with tile i+1's loads).
    // SYNK_GEMM_PERSISTENT=0 disables it (A/B diagnostics).
    static const int persistent_mode = [] {
        const char* v = getenv("SYNK_GEMM_PERSISTENT");
        return v ? atoi(v) : 1;
    }();
    if (bf16 && persistent_mode && N > 128) {
        // CTA-pair (cta_group::2) 256 x 256 tiles: +6-9 % over the 1-CTA
        // 128 x 256 kernel on C5's shapes with random operands (1,479 vs 1,391
        // TFLOP/s at 8192x4096x4096), C5 step 1.127 -> 1.071 ms
        // (profiles/r02_gemm_pair.txt). SYNK_GEMM_PAIR=0: the 1-CTA kernel.
        static const bool pair = [] {
            const char* v = getenv("SYNK_GEMM_PAIR");
            return !(v && v[0] == '0');
        }();
        CUtensorMap bw = b0;
        if (!(lay & kBMn))
            if (int rc = make_map(&bw, b_hi, N, K, ldb, true, pair ? PBN / 2 : PBN); rc) return rc;
        if (pair) {
            // short-K tanh-derivative product with a 16-byte aligned bf16 activation:
            // the activation tiles are TMA-staged (PCfg ACT)
            const bool act_tma = epilogue == SYNK_EPI_TANH_GRAD && out_dtype == 3 && K <= 128 && act &&
                                 (reinterpret_cast<uintptr_t>(act) & 15) == 0 && (ldact * 2) % 16 == 0;
            CUtensorMap ta = bw;
            if (act_tma)
                if (int rc = make_map(&ta, act, M, N, ldact, true, 128); rc) return rc;
            const void* kern = act_tma ? (const void*)gemm_tc_persistent_kernel<2, true>
                                       : (const void*)gemm_tc_persistent_kernel<2, false>;
            const size_t smem = act_tma ? PCfg<2, true>::kSmem : PCfg<2, false>::kSmem;
            if (int rc = synk::ensure_max_smem(kern, d->device, (int)smem); rc) return rc;
            const uint64_t tiles = ((M + 255) / 256) * ((N + PBN - 1) / PBN);
            const unsigned grid = 2 * (unsigned)std::min<uint64_t>(tiles, (uint64_t)d->num_sms / 2);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(grid);
            cfg.blockDim = dim3(PThreads);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = d->stream;
            cudaLaunchAttribute attr[2];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = 2;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[1].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = pdl_gemm() && d->pdl_armed ? 2 : 1;  // PDL after a kernel that released at entry
            if (act_tma)
                SYNK_CU(cudaLaunchKernelEx(&cfg, gemm_tc_persistent_kernel<2, true>, a0, bw, ta, (uint32_t)M,
                                           (uint32_t)N, (uint32_t)K, e, lay));
            else
                SYNK_CU(cudaLaunchKernelEx(&cfg, gemm_tc_persistent_kernel<2, false>, a0, bw, ta, (uint32_t)M,
                                           (uint32_t)N, (uint32_t)K, e, lay));
            d->pdl_armed = pdl_gemm();
            return SYNK_OK;
        }
        constexpr size_t smem = PCfg<1>::kSmem;
        if (int rc = synk::ensure_max_smem((const void*)gemm_tc_persistent_kernel<1, false>, d->device, (int)smem); rc)
            return rc;
        const uint64_t tiles = ((M + BM - 1) / BM) * ((N + PBN - 1) / PBN);
        const unsigned grid = (unsigned)std::min<uint64_t>(tiles, (uint64_t)d->num_sms);
        gemm_tc_persistent_kernel<1, false><<<grid, PThreads, smem, d->stream>>>(a0, bw, bw, (uint32_t)M, (uint32_t)N,
                                                                                   (uint32_t)K, e, lay);
        SYNK_LAUNCHED("gemm_tc_persistent_kernel");
        d->pdl_armed = pdl_gemm();
        return SYNK_OK;
    }
    // Narrow N (one column tile) with a K-major B: UMMA N = N rounded up to 16
    // and a B box of that many rows, so the zero rows the 128-row tile would
    // add are neither moved into shared memory nor multiplied (C5's N = 100
    // products: 112 instead of 128 B rows per stage).
    uint32_t n_eff = BN;
    if (N < BN && !(lay & kBMn)) {
        n_eff = (uint32_t)((N + 15) / 16 * 16);
        if (int rc = make_map(&b0, b_hi, N, K, ldb, bf16, n_eff); rc) return rc;
        b1 = b0;
        if (kind == 2)
            if (int rc = make_map(&b1, b_lo, N, K, ldb, false, n_eff); rc) return rc;
    }
    // Too few output tiles to fill the GPU and a long K: split K over grid.z
    // (fixed split for a given shape, so results do not depend on the device),
    // fp32 partial planes in a stream-ordered scratch, one fold kernel.
    const uint64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
    const uint32_t kBKe = bf16 ? 64 : 32;
    const uint64_t num_kb = (K + kBKe - 1) / kBKe;
    uint32_t splits = 1;
    if (tiles < 148 && num_kb >= 16 && (epilogue == SYNK_EPI_STORE || epilogue == SYNK_EPI_BIAS) &&
        out_dtype == SYNK_F32 && !ct && c) {
        // one wave of 2 CTAs per SM, >= 8 K blocks per split (SYNK_SPLITK_CTAS /
        // SYNK_SPLITK_MINKB override: diagnostics)
        static const uint64_t target = [] {
            const char* v = getenv("SYNK_SPLITK_CTAS");
            return v ? (uint64_t)atoll(v) : (uint64_t)296;
        }();
        static const uint64_t min_kb = [] {
            const char* v = getenv("SYNK_SPLITK_MINKB");
            return v ? (uint64_t)atoll(v) : (uint64_t)8;
        }();
        uint64_t sp = target / tiles;
        sp = std::min<uint64_t>(sp, num_kb / min_kb);
        splits = (uint32_t)std::max<uint64_t>(sp, 1);
    }
    if (splits > 1) {
        const uint32_t kb_per = (uint32_t)((num_kb + splits - 1) / splits);
        splits = (uint32_t)((num_kb + kb_per - 1) / kb_per);
        // Up to 8 splits (a portable cluster): fold through distributed shared
        // memory inside the GEMM (same order and rounding as the fold kernel).
        // SYNK_SPLITK_CLUSTER=0 keeps the fp32 planes + fold kernel (A/B runs).
        static const bool cluster_fold = [] {
            const char* v = getenv("SYNK_SPLITK_CLUSTER");
            return !(v && v[0] == '0');
        }();
        if (cluster_fold && bf16 && splits <= 8) {
            EpiArgs ce{epilogue == SYNK_EPI_BIAS ? EPI_BIAS : EPI_STORE, 0, c, ldc, nullptr, 0,
                       epilogue == SYNK_EPI_BIAS ? bias : nullptr, nullptr, 0};
            const int rc = launch<0>(d, 1, a0, a1, b0, b1, M, N, K, ce, splits, kb_per, lay, 1, n_eff);
            if (rc == SYNK_OK) return rc;
            // a cluster of `splits` CTAs that cannot be scheduled here (e.g. an
            // SM-limited context): clear the launch error, take the planes path
            cudaGetLastError();
        }
        float* planes = nullptr;
        SYNK_CU(cudaMallocAsync((void**)&planes, (size_t)splits * M * N * sizeof(float), d->stream));
        EpiArgs pe{SYNK_EPI_STORE, 0, planes, N, nullptr, 0, nullptr, nullptr, 0};
        int rc = bf16 ? launch<0>(d, 1, a0, a1, b0, b1, M, N, K, pe, splits, kb_per, lay, 0, n_eff)
                      : launch<1>(d, kind == 2 ? 3 : 1, a0, a1, b0, b1, M, N, K, pe, splits, kb_per, 0, 0, n_eff);
        if (rc) return rc;
        const unsigned fgrid = (unsigned)std::min<uint64_t>((M * N + 255) / 256, (uint64_t)d->num_sms * 8);
        splitk_fold_kernel<<<fgrid, 256, 0, d->stream>>>(splits, M, N, planes, static_cast<float*>(c), ldc,
                                                         epilogue == SYNK_EPI_BIAS ? bias : nullptr);
        SYNK_LAUNCHED("splitk_fold_kernel");
        SYNK_CU(cudaFreeAsync(planes, d->stream));
        return SYNK_OK;
    }
    return bf16 ? launch<0>(d, 1, a0, a1, b0, b1, M, N, K, e, 1, 0x7fffffffu, lay, 0, n_eff)
                : launch<1>(d, kind == 2 ? 3 : 1, a0, a1, b0, b1, M, N, K, e, 1, 0x7fffffffu, 0, 0, n_eff);
}

}  // extern "C"
