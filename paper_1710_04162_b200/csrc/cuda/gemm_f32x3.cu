// fp32-accurate tensor-core GEMM for the f32 example function (config C1,
// mlp.cpp:31-73 products), sm_100a only:
//   C[M x N] = epilogue( A[M x K] . B[N x K]^T )
// A and B are K-major fp32 matrices handed over as tf32 hi + lo parts
// (hi = rna_tf32(x), lo = rna_tf32(x - hi); tf32_stage_kernel below, or the
// epilogue of the producing GEMM). Per 32-element K block the MMA warp issues
// hi.lo + lo.hi + hi.hi (tcgen05.mma kind::tf32, 12 MMAs of 128xBNx8) into a
// FRESH TMEM accumulator; the four epilogue warps then drain that block sum
// into fp32 registers with round-to-nearest adds while the MMA warp fills the
// other of two TMEM buffers. The tensor-core accumulator therefore never
// carries more than one K block: its truncation-like rounding bias (~-6.7e-9
// relative per accumulated product, profiles/r01_tcgen05_tf32_accumulation.txt)
// stays at the single-block level (~-1e-7) instead of growing with K, and the
// small correction products are accumulated before the large hi.hi ones.
//
// Tiles are 128 x BN: BN = 64 when the 128x128 tiling has fewer tiles than
// SMs (the C1 products: twice the CTAs, shorter epilogues, two CTAs per SM),
// else 128. Split K: when the tiles cannot fill the GPU, the S <= 8 CTAs of a
// tile (one per K range, a thread-block cluster along z, sized so every
// cluster fits in one wave) park their fp32 partials in shared memory and CTA
// z folds rows [z*R, (z+1)*R) across the S partials in rank order with an f64
// accumulator (distributed shared memory, no HBM planes, no fold launch). S
// depends on the shape and CTA footprint only, never on the device.
//
// Epilogue outputs (any subset): C (fp32, row-major), the tf32 hi/lo split of
// the result row-major and/or transposed -- so a layer's activation or delta
// is emitted directly in the operand form the next products read. The
// epilogue kinds the MLP issues are compiled as specialisations (a CTA runs
// its epilogue once, from a cold instruction cache), and the tanh' activation
// tile is TMA-staged into shared memory during the main loop.
//
// Warp roles (192 threads): 0 TMA producer (one lane), 1 MMA issuer (one
// lane), 2..5 accumulators/epilogue (warp w reads TMEM lane quadrant w % 4;
// warp 2 also allocates TMEM).

#include <cuda.h>
#include <math.h>

#include <algorithm>

#include "common.cuh"
#include "tc_ptx.cuh"

namespace {

using namespace synk_tc;

constexpr int BM = 128, BK = 32;  // 32 tf32 = one 128-byte swizzled row
constexpr int kTile = 128 * 128;  // bytes: 128 rows x 128 B (A hi or A lo)
constexpr int kThreads = 192;
constexpr int kEpiThreads = 128;

// BN = 64 (few output tiles: more CTAs, shorter epilogues) or 128.
template <int BN>
struct Cfg {
    static constexpr int kBTile = BN * 128;                // bytes: BN rows x 128 B
    static constexpr int kStage = 2 * kTile + 2 * kBTile;  // A hi, A lo, B hi, B lo
    static constexpr int kStages = 2;                      // 96 / 128 KB: clusters pack, short K per CTA
    static constexpr int kRing = kStages * kStage;
    static constexpr int kAct = 128 * BN * 4;              // tanh' activation tile (TMA, SWIZZLE_128B boxes)
    static constexpr int kPitch = BN + 4;                  // floats per parked partial row
    static constexpr size_t smem(bool act) { return 256 + 1024 + kRing + (act ? kAct : 0); }
    static constexpr uint32_t kIdesc = (1u << 4)                     // D f32
                                       | (2u << 7) | (2u << 10)      // A, B tf32
                                       | ((uint32_t)(BN >> 3) << 17) // N
                                       | ((uint32_t)(BM >> 4) << 24);// M
};

enum Epi { EPI_STORE = 0, EPI_BIAS = 1, EPI_BIAS_TANH = 2, EPI_TANH_GRAD = 3 };

struct Out {
    int mode;
    float* c;          // row-major result (ldc), may be null
    uint64_t ldc;
    const float* bias; // per column
    const float* act;  // tanh activations [M x N] (ldact) for EPI_TANH_GRAD
    uint64_t ldact;
    float* hi;         // row-major tf32 split of the result (ldh)
    float* lo;
    uint64_t ldh;
    float* hi_t;       // transposed tf32 split: [n][m] (ldt)
    float* lo_t;
    uint64_t ldt;
};

__device__ __forceinline__ float rna_tf32(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}

__device__ __forceinline__ void umma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// tcgen05.ld 32x32b.x16 without the wait (batched: one wait per 64 columns)
__device__ __forceinline__ void tmem_ld16_nowait(uint32_t taddr, uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
}

__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Fold + epilogue over this CTA's rows [r0, r0 + rows) of the parked
// partials: element quad (rr, cc) = sum over the S partials (rank order, f64;
// S = 1: the CTA's own partial), then the epilogue op and the stores.
// EK = mode | outputs << 2 (1: c, 2: hi/lo, 4: hi_t/lo_t) fixed at compile
// time for the combinations the MLP issues (EK < 0: read from o at run
// time): these CTAs run once per launch, so the instruction cache is cold and
// the cost of the epilogue is set by the code it executes -- ncu showed an
// unrolled, runtime-branching version stalled on instruction fetch ("no
// instructions") for most of its time. Every operand the loop reads is in
// shared memory (partials, the TMA-staged activation tile) or a broadcast
// bias load.
template <int BN, int EK>
__device__ __forceinline__ void fold_epilogue(const Out& o, uint32_t S, uint32_t local, uint32_t act_smem, uint32_t r0,
                                              uint32_t rows, uint32_t m0, uint32_t n0, uint32_t M, uint32_t N) {
    constexpr uint32_t kQ = BN / 4, kPitch = Cfg<BN>::kPitch;
    constexpr bool gen = EK < 0;
    const int mode = gen ? o.mode : (EK & 3);
    const bool w_c = gen ? o.c != nullptr : ((EK >> 2) & 1) != 0;
    const bool w_h = gen ? o.hi != nullptr : ((EK >> 3) & 1) != 0;
    const bool w_t = gen ? o.hi_t != nullptr : ((EK >> 4) & 1) != 0;
    // transposed outputs: rows fastest across threads (coalesced [n][m]
    // stores); otherwise columns fastest (coalesced row-major stores)
    const uint32_t total = rows * kQ;
#pragma unroll 1
    for (uint32_t t = threadIdx.x; t < total; t += kThreads) {
        const uint32_t rr = r0 + (w_t ? t % rows : t / kQ);
        const uint32_t cc = (w_t ? t / rows : t % kQ) * 4;
        const uint32_t off = local + (rr * kPitch + cc) * 4;
        float4 x[8];
#pragma unroll
        for (uint32_t z = 0; z < 8; ++z) {
            if (z >= S) break;
            if (S > 1) {
                uint32_t addr;
                asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(addr) : "r"(off), "r"(z));
                asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(x[z].x), "=f"(x[z].y), "=f"(x[z].z), "=f"(x[z].w)
                             : "r"(addr));
            } else {
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(x[z].x), "=f"(x[z].y), "=f"(x[z].z), "=f"(x[z].w)
                             : "r"(off));
            }
        }
        const uint64_t m = (uint64_t)m0 + rr, n = (uint64_t)n0 + cc;
        if (m >= M) continue;
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        if (mode == EPI_TANH_GRAD) {
            if (act_smem) {  // SWIZZLE_128B box of 32 columns: 16-byte chunk (cc % 32) / 4 ^ (row % 8)
                const uint32_t w = cc & 31;
                const uint32_t addr = act_smem + (cc >> 5) * (128 * 128) + rr * 128 + (((w >> 2) ^ (rr & 7)) << 4);
                asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                             : "=f"(a[0]), "=f"(a[1]), "=f"(a[2]), "=f"(a[3])
                             : "r"(addr));
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (n + j < N) a[j] = __ldg(o.act + m * o.ldact + n + j);
            }
        } else if (mode != EPI_STORE) {
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (n + j < N) a[j] = __ldg(o.bias + n + j);
        }
        float v[4];
        if (S == 1) {
            v[0] = x[0].x, v[1] = x[0].y, v[2] = x[0].z, v[3] = x[0].w;
        } else {
            double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
            for (uint32_t z = 0; z < 8; ++z) {
                if (z >= S) break;
                s0 += (double)x[z].x, s1 += (double)x[z].y, s2 += (double)x[z].z, s3 += (double)x[z].w;
            }
            v[0] = (float)s0, v[1] = (float)s1, v[2] = (float)s2, v[3] = (float)s3;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (n + j >= N) break;
            float y = v[j];
            if (mode == EPI_BIAS) y += a[j];
            else if (mode == EPI_BIAS_TANH) y = tanhf(y + a[j]);
            else if (mode == EPI_TANH_GRAD) y = y * (1.0f - a[j] * a[j]);
            if (w_c) o.c[m * o.ldc + n + j] = y;
            if (w_h || w_t) {
                const float h = rna_tf32(y), l = rna_tf32(y - h);
                if (w_h) o.hi[m * o.ldh + n + j] = h, o.lo[m * o.ldh + n + j] = l;
                if (w_t) o.hi_t[(n + j) * o.ldt + m] = h, o.lo_t[(n + j) * o.ldt + m] = l;
            }
        }
    }
}

// Epilogue kinds compiled as specialisations (mode | outputs << 2), the
// combinations the f32 MLP issues; anything else runs the generic EK = -1.
constexpr int ek(int mode, bool c, bool h, bool t) { return mode | (c ? 4 : 0) | (h ? 8 : 0) | (t ? 16 : 0); }
constexpr int kEkFwdHidden = ek(EPI_BIAS_TANH, true, true, true);
constexpr int kEkFwdOut = ek(EPI_BIAS, true, false, false);
constexpr int kEkGrad = ek(EPI_STORE, true, false, false);
constexpr int kEkDxLast = ek(EPI_TANH_GRAD, false, false, true);
constexpr int kEkDx = ek(EPI_TANH_GRAD, false, true, true);

template <int BN, int EK>
__global__ void __launch_bounds__(kThreads, BN == 64 ? 2 : 1)
    gemm_f32x3_kernel(const __grid_constant__ CUtensorMap ahi, const __grid_constant__ CUtensorMap alo,
                      const __grid_constant__ CUtensorMap bhi, const __grid_constant__ CUtensorMap blo,
                      const __grid_constant__ CUtensorMap tact, int act_tma, uint32_t M, uint32_t N, uint32_t K,
                      uint32_t kb_per, Out o) {
    using C = Cfg<BN>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // [barriers 256 B][align to 1 KB][operand ring][activation tile]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 256 + 1023) & ~uintptr_t(1023));
    uint8_t* act_tile = smem + C::kRing;
    uint64_t* full = bars;                   // [kStages]
    uint64_t* empty = bars + C::kStages;     // [kStages]
    uint64_t* tfull = bars + 2 * C::kStages; // [2]
    uint64_t* tempty = tfull + 2;            // [2]
    uint64_t* act_full = tempty + 2;         // [1]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(act_full + 1);
    synk::release_dependent_grid();  // PDL: the next product may be scheduled (it waits below)

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int kb0 = (int)(blockIdx.z * kb_per);
    const int num_kb = min((int)kb_per, (int)((K + BK - 1) / BK) - kb0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < C::kStages; ++s) {
            mbar_init(smem_u32(&full[s]), 1);
            mbar_init(smem_u32(&empty[s]), 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(smem_u32(&tfull[b]), 1);
            mbar_init(smem_u32(&tempty[b]), kEpiThreads);
        }
        mbar_init(smem_u32(act_full), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        prefetch_map(&ahi);
        prefetch_map(&alo);
        prefetch_map(&bhi);
        prefetch_map(&blo);
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(2 * BN));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    __syncwarp();  // warp 0 reconverges after thread 0's barrier init: bar.sync is .aligned
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    synk::wait_prerequisite_grid();  // PDL: prologue overlapped the previous kernel; no global access before

    float acc[BN];
#pragma unroll
    for (int j = 0; j < BN; ++j) acc[j] = 0.f;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer ----
            if (act_tma) {  // the epilogue's activation tile, in flight during the main loop
                const uint32_t f = smem_u32(act_full);
                mbar_expect_tx(f, C::kAct);
#pragma unroll
                for (int j = 0; j < BN / 32; ++j)
                    tma_load_2d(smem_u32(act_tile + j * 128 * 128), &tact, f, (int)n0 + 32 * j, (int)m0);
            }
            for (int i = 0; i < num_kb; ++i) {
                const int s = i % C::kStages;
                mbar_wait(smem_u32(&empty[s]), ((i / C::kStages) & 1) ^ 1);
                const uint32_t f = smem_u32(&full[s]);
                mbar_expect_tx(f, C::kStage);
                uint8_t* st = smem + s * C::kStage;
                const int kc = (kb0 + i) * BK;
                tma_load_2d(smem_u32(st), &ahi, f, kc, (int)m0);
                tma_load_2d(smem_u32(st + kTile), &alo, f, kc, (int)m0);
                tma_load_2d(smem_u32(st + 2 * kTile), &bhi, f, kc, (int)n0);
                tma_load_2d(smem_u32(st + 2 * kTile + C::kBTile), &blo, f, kc, (int)n0);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer: one fresh accumulator per K block ----
            for (int i = 0; i < num_kb; ++i) {
                const int s = i % C::kStages, buf = i & 1;
                mbar_wait(smem_u32(&tempty[buf]), ((i >> 1) & 1) ^ 1);
                mbar_wait(smem_u32(&full[s]), (i / C::kStages) & 1);
                tc_fence_after();
                const uint32_t st = smem_u32(smem + s * C::kStage);
                const uint32_t a_h = st, a_l = st + kTile, b_h = st + 2 * kTile, b_l = b_h + C::kBTile;
                const uint32_t d = tmem + buf * BN;
                // small corrections first, then the large hi.hi products
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    umma_tf32(d, smem_desc(a_h + 32 * k), smem_desc(b_l + 32 * k), C::kIdesc, k > 0);
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_tf32(d, smem_desc(a_l + 32 * k), smem_desc(b_h + 32 * k), C::kIdesc, 1u);
#pragma unroll
                for (int k = 0; k < 4; ++k) umma_tf32(d, smem_desc(a_h + 32 * k), smem_desc(b_h + 32 * k), C::kIdesc, 1u);
                umma_commit(smem_u32(&empty[s]));
                umma_commit(smem_u32(&tfull[buf]));
            }
        }
    } else {  // ---- warps 2..5: drain each block sum into fp32 registers ----
        const uint32_t quad = (uint32_t)(warp % 4);
        for (int i = 0; i < num_kb; ++i) {
            const int buf = i & 1;
            mbar_wait(smem_u32(&tfull[buf]), (i >> 1) & 1);
            tc_fence_after();
            const uint32_t base = tmem + buf * BN + ((quad * 32) << 16);
#pragma unroll
            for (int h = 0; h < BN / 64; ++h) {
                uint32_t r[4][16];
#pragma unroll
                for (int c = 0; c < 4; ++c) tmem_ld16_nowait(base + 64 * h + 16 * c, r[c]);
                asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
                for (int c = 0; c < 4; ++c)
#pragma unroll
                    for (int j = 0; j < 16; ++j) acc[64 * h + 16 * c + j] += __uint_as_float(r[c][j]);
            }
            tc_fence_before();
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tempty[buf])) : "memory");
        }
    }
    __syncwarp();

    // Park the partial (the operand ring is idle: every MMA has retired) and
    // run one compact epilogue loop over it: S = 1 reads its own partial, S > 1
    // folds the cluster's partials (rows [z*R, (z+1)*R) in CTA z) in rank
    // order in f64. A compact loop instead of an unrolled per-register
    // epilogue: these CTAs run once per launch, so instruction-cache misses on
    // long straight-line code cost more than the shared-memory round trip.
    const uint32_t S = gridDim.z;
    float* part = reinterpret_cast<float*>(smem);
    if (act_tma) mbar_wait(smem_u32(act_full), 0);
    const uint32_t act_smem = act_tma ? smem_u32(act_tile) : 0u;
    if (warp >= 2) {
        const int row = (warp % 4) * 32 + lane;
        float4* dst = reinterpret_cast<float4*>(part + row * C::kPitch);
#pragma unroll
        for (int j = 0; j < BN / 4; ++j) dst[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
    }
    if (S > 1) cluster_sync();
    else __syncthreads();
    uint32_t me = 0;
    if (S > 1) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(me));
    const uint32_t R = (BM + S - 1) / S, r0 = me * R, r1 = min((uint32_t)BM, r0 + R);
    const uint32_t rows = r1 > r0 ? r1 - r0 : 0;
    fold_epilogue<BN, EK>(o, S, smem_u32(part), act_smem, r0, rows, m0, n0, M, N);
    if (S > 1) cluster_sync();  // partials stay alive until every reader is done
    tc_fence_before();
    __syncthreads();
    if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(2 * BN));
}

// One tile of a tf32 split job: out = split of in (rows x cols, ld_in; row r
// read from rowmap[r] when given), row-major hi/lo (ld_o) and/or transposed
// hi/lo (cols x rows, ld_t). 32 x 32 tiles through shared memory so both
// sides stay coalesced.
__device__ __forceinline__ void split_tile(const synk_tf32_job& j, uint64_t r0, uint64_t c0, float (&tile)[32][33]) {
    const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
        const uint64_t r = r0 + k, c = c0 + tx;
        float v = 0.f;
        if (r < j.rows && c < j.cols) v = j.in[(j.rowmap ? j.rowmap[r] : r) * j.ld_in + c];
        tile[k][tx] = v;
        if (j.hi && r < j.rows && c < j.cols) {
            const float h = rna_tf32(v);
            j.hi[r * j.ld_o + c] = h;
            j.lo[r * j.ld_o + c] = rna_tf32(v - h);
        }
    }
    if (!j.hi_t) return;
    __syncthreads();
#pragma unroll
    for (int k = ty; k < 32; k += 8) {
        const uint64_t c = c0 + k, r = r0 + tx;  // output row c, column r
        if (c >= j.cols || r >= j.rows) continue;
        const float v = tile[tx][k];
        const float h = rna_tf32(v);
        j.hi_t[c * j.ld_t + r] = h;
        j.lo_t[c * j.ld_t + r] = rna_tf32(v - h);
    }
}

struct SplitBatch {
    synk_tf32_job jobs[SYNK_TF32_MAX_JOBS];
    uint32_t first[SYNK_TF32_MAX_JOBS + 1];  // first tile (block) of each job; first[count] = fill blocks start
    uint32_t count;
};

// Every staging job of a step in one launch: block b < first[count] is a
// split tile, the blocks after it set the constant rows (one row each).
__global__ void __launch_bounds__(256) tf32_stage_kernel(SplitBatch batch, synk_tf32_rows fill) {
    __shared__ float tile[32][33];
    synk::release_dependent_grid();  // PDL: the first product may be scheduled behind it
    const uint32_t b = blockIdx.x;
    if (b >= batch.first[batch.count]) {
        const uint32_t i = b - batch.first[batch.count];
        for (uint64_t k = threadIdx.x; k < fill.len[i]; k += 256) {
            fill.hi[i][k] = fill.value;
            fill.lo[i][k] = 0.f;
        }
        return;
    }
    uint32_t j = 0;
    while (b >= batch.first[j + 1]) ++j;
    const synk_tf32_job& job = batch.jobs[j];
    const uint32_t t = b - batch.first[j];
    const uint32_t tiles_x = (uint32_t)((job.cols + 31) / 32);
    split_tile(job, (uint64_t)(t / tiles_x) * 32, (uint64_t)(t % tiles_x) * 32, tile);
}

// Split-K depth S (the cluster size along z). Fixed by the shape and the
// CTA footprint, never by the device, so results are device-independent. The
// clusters must also fit in ONE wave: cluster CTAs are placed inside a GPC
// (148 SMs = 8 GPCs), and 16 clusters of 7 did not fit at one CTA per SM, so
// the bound used is 8 * floor(12 / S) clusters of S
// single-CTA SMs (twice that at two CTAs per SM); a cluster
// left for a second wave doubles the launch (measured: CTA start times spread
// over 11.9 us with 16 clusters of 7 at one CTA per SM).
uint32_t choose_splits(uint64_t M, uint64_t N, uint64_t K, int bn, int ctas_per_sm, uint32_t* kb_per) {
    const uint64_t tiles = ((M + BM - 1) / BM) * ((N + bn - 1) / bn);
    const uint64_t num_kb = (K + BK - 1) / BK;
    uint64_t s = 148 / tiles;  // fill a 148-SM B200
    s = std::min<uint64_t>(s, 8);
    s = std::min<uint64_t>(s, num_kb);
    s = std::max<uint64_t>(s, 1);
    while (s > 1 && tiles > 8 * (12 / s) * (uint64_t)ctas_per_sm) --s;
    const uint64_t per = (num_kb + s - 1) / s;
    *kb_per = (uint32_t)per;
    return (uint32_t)((num_kb + per - 1) / per);
}

// Programmatic dependent launch along the C1 chain (stage -> products ->
// loss -> products): each kernel releases its dependents at entry and waits
// after its prologue. SYNK_F32X3_PDL=0 launches plainly (A/B).
bool pdl_f32x3() {
    static const bool on = [] {
        const char* e = getenv("SYNK_F32X3_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

template <int BN, int EK>
int launch_f32x3(synk_dev* d, const CUtensorMap& ah, const CUtensorMap& al, const void* b_hi, const void* b_lo,
                 uint64_t ldb, uint64_t M, uint64_t N, uint64_t K, const Out& o) {
    using C = Cfg<BN>;
    CUtensorMap bh, bl, ta;
    if (int rc = make_map(&bh, b_hi, N, K, ldb, false, BN); rc) return rc;
    if (int rc = make_map(&bl, b_lo, N, K, ldb, false, BN); rc) return rc;
    // tanh' activations staged by TMA when their rows are 16-byte aligned
    const int act_tma = o.mode == SYNK_EPI_TANH_GRAD && (o.ldact * 4) % 16 == 0 &&
                        (reinterpret_cast<uintptr_t>(o.act) & 15) == 0;
    ta = bh;
    if (act_tma)
        if (int rc = make_map(&ta, o.act, M, N, o.ldact, false, 128); rc) return rc;
    uint32_t kb_per = 0;
    const size_t smem = C::smem(act_tma);
    const uint32_t S = choose_splits(M, N, K, BN, smem <= 113 * 1024 ? 2 : 1, &kb_per);
    if (int rc = synk::ensure_max_smem((const void*)gemm_f32x3_kernel<BN, EK>, d->device, (int)C::smem(true)); rc)
        return rc;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), S);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = d->stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 1;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = S;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl_f32x3() && d->pdl_armed ? 2 : 1;  // PDL after a kernel that released at entry
    SYNK_CU(cudaLaunchKernelEx(&cfg, gemm_f32x3_kernel<BN, EK>, ah, al, bh, bl, ta, act_tma, (uint32_t)M, (uint32_t)N,
                               (uint32_t)K, kb_per, o));
    d->pdl_armed = pdl_f32x3();
    return SYNK_OK;
}

}  // namespace

extern "C" {

int synk_gemm_f32x3(synk_dev* d, uint64_t M, uint64_t N, uint64_t K, const float* a_hi, const float* a_lo,
                    uint64_t lda, const float* b_hi, const float* b_lo, uint64_t ldb, int epilogue, float* c,
                    uint64_t ldc, const float* bias, const float* act, uint64_t ldact, float* c_hi, float* c_lo,
                    uint64_t ldh, float* ct_hi, float* ct_lo, uint64_t ldt) {
    SYNK_REQUIRE(epilogue >= SYNK_EPI_STORE && epilogue <= SYNK_EPI_TANH_GRAD, SYNK_EARG, "gemm_f32x3: bad epilogue");
    SYNK_REQUIRE(M < (1ull << 31) && N < (1ull << 31) && K < (1ull << 31), SYNK_EARG, "gemm_f32x3: dims too large");
    SYNK_REQUIRE(!(epilogue == SYNK_EPI_BIAS || epilogue == SYNK_EPI_BIAS_TANH) || bias, SYNK_EARG,
                 "gemm_f32x3: epilogue needs bias");
    SYNK_REQUIRE(epilogue != SYNK_EPI_TANH_GRAD || act, SYNK_EARG, "gemm_f32x3: epilogue needs act");
    SYNK_REQUIRE((c_hi == nullptr) == (c_lo == nullptr) && (ct_hi == nullptr) == (ct_lo == nullptr), SYNK_EARG,
                 "gemm_f32x3: split outputs come in hi/lo pairs");
    if (M == 0 || N == 0) return SYNK_OK;
    SYNK_REQUIRE(K > 0, SYNK_EARG, "gemm_f32x3: K must be > 0");
    synk::DeviceGuard g(d->device);
    CUtensorMap ah, al;
    if (int rc = make_map(&ah, a_hi, M, K, lda, false); rc) return rc;
    if (int rc = make_map(&al, a_lo, M, K, lda, false); rc) return rc;
    Out o{epilogue, c, ldc, bias, act, ldact, c_hi, c_lo, ldh, ct_hi, ct_lo, ldt};
    // few 128 x 128 tiles (the C1 products): 128 x 64 tiles, twice the CTAs
    const bool narrow = ((M + BM - 1) / BM) * ((N + 127) / 128) < 148;
    const int kind = ek(epilogue, c != nullptr, c_hi != nullptr, ct_hi != nullptr);
#define SYNK_F32X3_EK(E)                                                                                   \
    if (kind == E)                                                                                         \
        return narrow ? launch_f32x3<64, E>(d, ah, al, b_hi, b_lo, ldb, M, N, K, o)                        \
                      : launch_f32x3<128, E>(d, ah, al, b_hi, b_lo, ldb, M, N, K, o);
    SYNK_F32X3_EK(kEkFwdHidden)
    SYNK_F32X3_EK(kEkFwdOut)
    SYNK_F32X3_EK(kEkGrad)
    SYNK_F32X3_EK(kEkDxLast)
    SYNK_F32X3_EK(kEkDx)
#undef SYNK_F32X3_EK
    return narrow ? launch_f32x3<64, -1>(d, ah, al, b_hi, b_lo, ldb, M, N, K, o)
                  : launch_f32x3<128, -1>(d, ah, al, b_hi, b_lo, ldb, M, N, K, o);
}

int synk_tf32_stage(synk_dev* d, const synk_tf32_job* jobs, uint32_t count, const synk_tf32_rows* fill) {
    SYNK_REQUIRE(count <= SYNK_TF32_MAX_JOBS, SYNK_EARG, "tf32_stage: at most 16 split jobs per launch");
    SYNK_REQUIRE(!fill || fill->count <= SYNK_TF32_MAX_ROWS, SYNK_EARG, "tf32_stage: at most 64 constant rows");
    SplitBatch batch{};
    uint32_t blocks = 0;
    for (uint32_t i = 0; i < count; ++i) {
        const synk_tf32_job& j = jobs[i];
        SYNK_REQUIRE((j.hi == nullptr) == (j.lo == nullptr) && (j.hi_t == nullptr) == (j.lo_t == nullptr), SYNK_EARG,
                     "tf32_split: outputs come in hi/lo pairs");
        batch.jobs[batch.count] = j;
        batch.first[batch.count] = blocks;
        if (j.rows && j.cols && (j.hi || j.hi_t)) {
            const uint64_t tiles = ((j.rows + 31) / 32) * ((j.cols + 31) / 32);
            SYNK_REQUIRE(blocks + tiles < (1ull << 31), SYNK_EARG, "tf32_stage: too many tiles");
            blocks += (uint32_t)tiles;
        }
        ++batch.count;
    }
    batch.first[batch.count] = blocks;
    synk_tf32_rows rows{};
    if (fill) rows = *fill;
    if (blocks + rows.count == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    tf32_stage_kernel<<<blocks + rows.count, 256, 0, d->stream>>>(batch, rows);
    SYNK_LAUNCHED("tf32_stage_kernel");
    d->pdl_armed = pdl_f32x3();
    return SYNK_OK;
}

int synk_tf32_split(synk_dev* d, const float* in, const uint64_t* rowmap, uint64_t rows, uint64_t cols, uint64_t ld_in,
                    float* hi, float* lo, uint64_t ld_o, float* hi_t, float* lo_t, uint64_t ld_t) {
    const synk_tf32_job j{in, rowmap, rows, cols, ld_in, hi, lo, ld_o, hi_t, lo_t, ld_t};
    return synk_tf32_stage(d, &j, 1, nullptr);
}

int synk_tf32_fill_rows(synk_dev* d, const synk_tf32_rows* rows) {
    SYNK_REQUIRE(rows, SYNK_EARG, "tf32_fill_rows: null rows");
    return synk_tf32_stage(d, nullptr, 0, rows);
}

}  // extern "C"
