// Input indexing: dst[j,:] = src[idx[j],:]   (gather_rows, tensor.cpp:200-217)
//
// HBM-bound row gather. One warp owns a contiguous block of destination rows
// and works on ROWS of them at a time: the indices are shuffled to the warp,
// then every lane streams
// 16-byte vectors of all ROWS rows (ROWS x UNROLL independent 128-bit loads in
// flight per lane before the first store), so a 1 KiB row is two fully
// coalesced 512-byte warp transactions per row and no shared memory is
// needed. Source rows are read with ld.global.nc.L1::no_allocate (each row is
// touched once); the source may be an HBM mirror or pinned, mapped host memory
// (then the same loads travel over PCIe). Out-of-range indices set the rank's
// device error flag, reported as BoundsError at the phase-exit synk_sync().

#include <cuda.h>
#include <stdlib.h>

#include <mutex>

#include "common.cuh"

namespace {

template <int BYTES>
struct Vec;
template <>
struct Vec<16> {
    using T = uint4;
    static __device__ __forceinline__ T load(const T* p) {
        T r;
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                     : "l"(p));
        return r;
    }
};
template <>
struct Vec<8> {
    using T = uint2;
    static __device__ __forceinline__ T load(const T* p) {
        T r;
        asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
                     : "=r"(r.x), "=r"(r.y)
                     : "l"(p));
        return r;
    }
};
template <>
struct Vec<4> {
    using T = uint32_t;
    static __device__ __forceinline__ T load(const T* p) { return __ldg(p); }
};
template <>
struct Vec<1> {
    using T = uint8_t;
    static __device__ __forceinline__ T load(const T* p) { return __ldg(p); }
};
// 256-bit vectors (sm_100 ld/st .v8.b32): one instruction per 32 bytes per lane
struct alignas(32) U8x32 {
    uint32_t w[8];
};
template <>
struct Vec<32> {
    using T = U8x32;
    static __device__ __forceinline__ T load(const T* p) {
        T r;
        asm volatile("ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r.w[0]), "=r"(r.w[1]), "=r"(r.w[2]), "=r"(r.w[3]), "=r"(r.w[4]), "=r"(r.w[5]),
                       "=r"(r.w[6]), "=r"(r.w[7])
                     : "l"(p));
        return r;
    }
};

template <class T>
__device__ __forceinline__ void store_vec(T* p, const T& v, int streaming) {
    if (streaming) __stcs(p, v);
    else *p = v;
}
__device__ __forceinline__ void store_vec(U8x32* p, const U8x32& v, int streaming) {
    if (streaming)
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
                     "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                     : "memory");
    else
        asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.w[0]), "r"(v.w[1]),
                     "r"(v.w[2]), "r"(v.w[3]), "r"(v.w[4]), "r"(v.w[5]), "r"(v.w[6]), "r"(v.w[7])
                     : "memory");
}

constexpr int kBlock = 256;

// Chunked grid-stride: warp w takes chunks w, w + nwarps, ... of `chunk`
// consecutive destination rows (chunk <= 32, a multiple of kRows), so warps
// running at the same time write neighbouring rows of dst. The chunk's
// indices sit in the warp's lanes (read as part of the CTA's index line, one
// coalesced read, which matters when the list sits in pinned host memory and
// travels over PCIe), and the NEXT chunk's
// indices are requested before the current chunk's rows are streamed, so the
// index fetch overlaps a chunk of row traffic.
// kRows rows in flight per warp, kUnroll 16-byte vectors per row per lane.
template <int BYTES, int kRows = 4, int kUnroll = 2, int kMinBlocks = 1>
__global__ void __launch_bounds__(kBlock, kMinBlocks) gather_rows_kernel(
    const typename Vec<BYTES>::T* __restrict__ src, uint64_t src_rows, uint64_t row_vecs,
    const uint64_t* __restrict__ idx, uint64_t n_idx, uint32_t chunk, int share,
    typename Vec<BYTES>::T* __restrict__ dst, int* __restrict__ err, int stream_stores) {
    using V = typename Vec<BYTES>::T;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint64_t stride = (((uint64_t)gridDim.x * kBlock) >> 5) * chunk;
    // Dependents may be scheduled once every CTA has started (the last wave):
    // a small follow-up (the call's result kernel) then waits on-chip in
    // griddepcontrol.wait instead of paying its launch after this grid ends.
    synk::release_dependent_grid();
    if (src_rows == 0) {  // every index is out of range
        if (blockIdx.x == 0 && threadIdx.x == 0) *(volatile int*)err = 1;
        return;
    }

    // Index lines: the CTA's 8 warps hold neighbouring chunks (warp w of the
    // CTA rows orow = w * chunk onward), so with `share` every warp reads the
    // CTA's whole line of 8 x chunk <= 32 indices in one coalesced request and
    // takes its own lanes: a pinned-host list then travels as one 256-byte
    // PCIe read per line (the other seven warps hit it in L2) instead of
    // eight 32-byte reads -- +3-4 % e2e on C2 (profiles/r02_gather_e2e.md).
    const int orow = share ? (int)((threadIdx.x >> 5) * chunk) : 0;
    const int line = share ? (int)(chunk * (kBlock / 32)) : (int)chunk;
    uint64_t c0 = warp * chunk;
    uint64_t next = c0 - orow + lane < n_idx && lane < line ? idx[c0 - orow + lane] : 0;
    for (; c0 < n_idx; c0 += stride) {
        const uint64_t mine = next;
        const int in_chunk = (int)(n_idx - c0 < chunk ? n_idx - c0 : chunk);
        const uint64_t cn = c0 + stride - orow;
        if (lane < line && cn + lane < n_idx) next = idx[cn + lane];  // prefetch the next chunk
        const int own = lane >= orow && lane < orow + in_chunk;
        const int ok = own && mine < src_rows;
        if (own && !ok) *(volatile int*)err = 1;  // mapped host flag: every writer stores 1
        // A bad index reads row 0 instead (defined data; the call fails).
        const uint64_t safe = ok ? mine : 0;
        for (int g = 0; g < in_chunk; g += kRows) {
            uint64_t row[kRows];
            int exists[kRows];
#pragma unroll
            for (int k = 0; k < kRows; ++k) {
                row[k] = __shfl_sync(0xffffffffu, safe, (orow + g + k) & 31);
                exists[k] = g + k < in_chunk;
            }
            const uint64_t r0 = c0 + g;
            for (uint64_t v0 = lane; v0 < row_vecs; v0 += 32 * kUnroll) {
                V buf[kRows][kUnroll];
#pragma unroll
                for (int k = 0; k < kRows; ++k)
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        uint64_t v = v0 + (uint64_t)u * 32;
                        if (exists[k] && v < row_vecs) buf[k][u] = Vec<BYTES>::load(src + row[k] * row_vecs + v);
                    }
#pragma unroll
                for (int k = 0; k < kRows; ++k)
#pragma unroll
                    for (int u = 0; u < kUnroll; ++u) {
                        uint64_t v = v0 + (uint64_t)u * 32;
                        if (exists[k] && v < row_vecs) store_vec(dst + (r0 + k) * row_vecs + v, buf[k][u], stream_stores);
                    }
            }
        }
    }
}

// Short host-side lists (<= SYNK_GATHER_INLINE_MAX indices below 2^32) travel
// inside the launch: the u32 indices are a kernel parameter (constant bank,
// fetched with the launch), so no warp waits on a dependent PCIe read of a
// pinned list before its first row load -- the latency floor of one small
// batch per call (bench single_batch_call). The host validated the list while
// narrowing it. Warp w streams rows 4w..4w+3; dependents are released at entry.
}  // namespace
namespace synk {
uint32_t narrow_indices(const uint64_t* in, uint64_t n, uint64_t limit, uint32_t* out);  // index_narrow.cpp
}  // namespace synk
namespace {

struct InlineIdx {
    uint32_t idx[SYNK_GATHER_INLINE_MAX];
};
static_assert(sizeof(InlineIdx) + 64 <= 32764, "kernel parameter limit");

template <int BYTES, int kUnroll>
__global__ void __launch_bounds__(kBlock) gather_rows_inline_kernel(const typename Vec<BYTES>::T* __restrict__ src,
                                                                    uint64_t row_vecs,
                                                                    const __grid_constant__ InlineIdx p,
                                                                    uint32_t n_idx,
                                                                    typename Vec<BYTES>::T* __restrict__ dst) {
    using V = typename Vec<BYTES>::T;
    synk::release_dependent_grid();
    const int lane = threadIdx.x & 31;
    const uint32_t r0 = ((blockIdx.x * kBlock + threadIdx.x) >> 5) * 4;
    if (r0 >= n_idx) return;
    uint64_t row[4];
    int exists[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        exists[k] = r0 + k < n_idx;
        row[k] = exists[k] ? p.idx[r0 + k] : 0;
    }
    for (uint64_t v0 = lane; v0 < row_vecs; v0 += 32 * kUnroll) {
        V buf[4][kUnroll];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint64_t v = v0 + (uint64_t)u * 32;
                if (exists[k] && v < row_vecs) buf[k][u] = Vec<BYTES>::load(src + row[k] * row_vecs + v);
            }
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                const uint64_t v = v0 + (uint64_t)u * 32;
                if (exists[k] && v < row_vecs) store_vec(dst + ((uint64_t)r0 + k) * row_vecs + v, buf[k][u], 0);
            }
    }
}

template <int BYTES>
int launch_inline(synk_dev* d, const void* src, uint64_t row_bytes, const InlineIdx& p, uint32_t n_idx, void* dst) {
    using V = typename Vec<BYTES>::T;
    const unsigned blocks = (unsigned)(((uint64_t)(n_idx + 3) / 4 * 32 + kBlock - 1) / kBlock);
    constexpr int U = BYTES == 32 ? 1 : 2;
    gather_rows_inline_kernel<BYTES, U><<<blocks, kBlock, 0, d->stream>>>((const V*)src, row_bytes / BYTES, p, n_idx,
                                                                           (V*)dst);
    SYNK_LAUNCHED("gather_rows_inline_kernel");
    d->pdl_armed = true;
    return SYNK_OK;
}

template <int BYTES, int R, int U, int MB>
void launch_variant(synk_dev* d, unsigned blocks, const void* src, uint64_t src_rows, uint64_t row_bytes,
                    const uint64_t* idx, uint64_t n_idx, uint32_t chunk, int share, void* dst) {
    using V = typename Vec<BYTES>::T;
    // Streaming (evict-first) stores when the destination is far larger than
    // what L2 could keep for a consumer anyway (measured +0.7 % on the C2
    // launch, 256 MiB); small gathers feeding a kernel keep normal stores.
    // SYNK_GATHER_STCS=0|1 forces either (A/B runs).
    static const int forced = [] {
        const char* e = getenv("SYNK_GATHER_STCS");
        return e ? (e[0] == '1' ? 1 : 0) : -1;
    }();
    const int stcs = forced >= 0 ? forced : (n_idx * row_bytes >= (64ull << 20) ? 1 : 0);
    gather_rows_kernel<BYTES, R, U, MB><<<blocks, kBlock, 0, d->stream>>>(
        (const V*)src, src_rows, row_bytes / BYTES, idx, n_idx, chunk, share, (V*)dst, d->err_dev, stcs);
}

template <int BYTES>
int launch(synk_dev* d, const void* src, uint64_t src_rows, uint64_t row_bytes,
           const uint64_t* idx, uint64_t n_idx, void* dst) {
    // Rows per warp chunk (A/B knob): a multiple of the 4 rows in flight, at
    // most one warp's worth of indices (lanes hold the chunk's indices).
    static const uint32_t chunk = [] {
        const char* e = getenv("SYNK_GATHER_ROWS");
        long v = e ? strtol(e, nullptr, 10) : 4;
        if (v < 4) v = 4;
        if (v > 32) v = 32;
        return (uint32_t)(v & ~3L);
    }();
    // Shared index lines (default on; SYNK_GATHER_SHARE=0 for A/B) need the
    // CTA's line to fit one warp: 8 warps x chunk <= 32 indices.
    static const int share_knob = [] {
        const char* e = getenv("SYNK_GATHER_SHARE");
        return e ? atoi(e) : 1;
    }();
    const int share = share_knob && chunk * (kBlock / 32) <= 32;
    // At most 8 CTAs of 8 warps per SM (about 2.7 waves at 3 resident
    // CTAs/SM: the oversubscription balances the random-row latency).
    // 4 rows x 2 vectors in flight per lane at <= 85 registers (3 CTAs/SM) won
    // the sweep (profiles/r01_gather.md): (4,1)x4 CTAs 0.77, (8,1)x2 0.57,
    // (2,4)x3 0.91 with a slower e2e, (8,2)x1 0.55, (2,2)x4 0.88 of HBM.
    const uint64_t chunks = (n_idx + chunk - 1) / chunk;
    uint64_t blocks = (chunks * 32 + kBlock - 1) / kBlock;
    const uint64_t cap = (uint64_t)d->num_sms * 8;
    if (blocks > cap) blocks = cap;
    if constexpr (BYTES == 32)  // same bytes in flight per lane as 2 x 16 B
        launch_variant<BYTES, 4, 1, 3>(d, (unsigned)blocks, src, src_rows, row_bytes, idx, n_idx, chunk, share, dst);
    else
        launch_variant<BYTES, 4, 2, 3>(d, (unsigned)blocks, src, src_rows, row_bytes, idx, n_idx, chunk, share, dst);
    SYNK_LAUNCHED("gather_rows_kernel");
    d->pdl_armed = true;
    return SYNK_OK;
}

// ---- bulk-copy (TMA engine) gather ---------------------------------------------------
//
// For 16-byte-aligned rows up to 8 KiB: one warp per CTA, two CTAs per SM. The
// warp walks chunks of up to 32 rows (chunk c = blockIdx.x + j*gridDim.x);
// lane i reads index i of the chunk and issues ONE cp.async.bulk global->shared
// copy of that whole row into stage j % S of a shared-memory ring, all
// completing on the stage's mbarrier (expect_tx = the chunk's valid bytes).
// When a stage lands, lane 0 writes the chunk's rows -- contiguous in dst -- with
// a single cp.async.bulk shared->global store. S-2 chunks of loads stay in
// flight per CTA (no registers hold row data, so the in-flight depth is set
// by shared memory, not by the register file), and each chunk's indices are
// fetched two chunks ahead so a PCIe-resident index list does not stall the
// issue loop.

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE_%=;\n"
        "bra WAIT_%=;\n"
        "DONE_%=:\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}

constexpr int kMaxStages = 16;

__global__ void __launch_bounds__(32) gather_rows_bulk_kernel(
    const char* __restrict__ src, uint64_t src_rows, uint32_t row_bytes, const uint64_t* __restrict__ idx,
    uint64_t n_idx, uint32_t chunk_rows, uint32_t stages, char* __restrict__ dst, int* __restrict__ err) {
    extern __shared__ __align__(128) char ring[];
    __shared__ __align__(8) uint64_t full[kMaxStages];
    __shared__ int bad[kMaxStages];
    const int lane = threadIdx.x;
    const uint64_t n_chunks = (n_idx + chunk_rows - 1) / chunk_rows;
    if (blockIdx.x >= n_chunks) return;
    const uint64_t mine = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;  // chunks of this CTA
    const uint32_t stage_bytes = chunk_rows * row_bytes;
    if (lane == 0) {
        for (uint32_t s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    auto chunk_start = [&](uint64_t j) { return (blockIdx.x + j * gridDim.x) * (uint64_t)chunk_rows; };
    auto load_index = [&](uint64_t j) -> uint64_t {
        if (j >= mine) return 0;
        const uint64_t r = chunk_start(j) + lane;
        return lane < (int)chunk_rows && r < n_idx ? idx[r] : 0;
    };
    // Indices two chunks ahead of the issue point.
    uint64_t q0 = load_index(0), q1 = load_index(1);

    auto issue = [&](uint64_t j, uint64_t my) {
        const uint32_t s = (uint32_t)(j % stages);
        const uint64_t r0 = chunk_start(j);
        const uint32_t cnt = (uint32_t)(n_idx - r0 < chunk_rows ? n_idx - r0 : chunk_rows);
        const bool live = lane < (int)cnt;
        const bool ok = live && my < src_rows;
        const unsigned okm = __ballot_sync(0xffffffffu, ok);
        const unsigned badm = __ballot_sync(0xffffffffu, live && !ok);
        char* slot = ring + (size_t)s * stage_bytes + (size_t)lane * row_bytes;
        if (badm) {  // error path: zero rows for bad indices, flag the rank
            if (live && !ok) {
                *(volatile int*)err = 1;
                for (uint32_t b = 0; b < row_bytes; b += 16) *reinterpret_cast<uint4*>(slot + b) = make_uint4(0, 0, 0, 0);
            }
        }
        if (lane == 0) {
            bad[s] = badm != 0;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[s])),
                         "r"((uint32_t)__popc(okm) * row_bytes)
                         : "memory");
        }
        __syncwarp();
        if (ok)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_addr(slot)),
                "l"(src + my * row_bytes), "r"(row_bytes), "r"(smem_addr(&full[s]))
                : "memory");
    };

    const uint64_t ahead = stages - 2 < mine ? stages - 2 : mine;  // chunks in flight before the first store
    for (uint64_t j = 0; j < ahead; ++j) {
        issue(j, q0);
        q0 = q1;
        q1 = load_index(j + 2);
    }
    for (uint64_t j = 0; j < mine; ++j) {
        const uint32_t s = (uint32_t)(j % stages);
        bar_wait(smem_addr(&full[s]), (uint32_t)((j / stages) & 1));
        const uint64_t r0 = chunk_start(j);
        const uint32_t cnt = (uint32_t)(n_idx - r0 < chunk_rows ? n_idx - r0 : chunk_rows);
        if (bad[s]) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic zero stores -> async proxy
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + r0 * row_bytes),
                         "r"(smem_addr(ring + (size_t)s * stage_bytes)), "r"(cnt * row_bytes)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        const uint64_t jn = j + ahead;
        if (jn < mine) {
            // Stage jn % S last held chunk jn - S <= j - 2: its store must have
            // finished reading shared memory (at most the newest group pending).
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            issue(jn, q0);
            q0 = q1;
            q1 = load_index(jn + 2);
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// ---- TMA gather4 (cp.async.bulk.tensor ... tile::gather4) ------------------------
//
// Rows of 16..2048 bytes in device memory: one tensor-map request fetches FOUR
// rows at arbitrary indices (Blackwell's gather4 mode) into shared memory --
// a quarter of the per-row bulk requests, whose per-request cost capped the
// per-row bulk kernel. Same pipeline: one warp per CTA, chunks of chunk_rows
// (a multiple of 4) rows, an mbarrier per stage, one bulk store per landed
// chunk (its rows are contiguous in dst), indices fetched two chunks ahead.
// A bad index fetches row 0 (defined data) and sets the rank's error flag.
// Measured (profiles/r01_gather.md): 0.913 of HBM at 2 CTAs/SM x 16-row
// chunks vs 0.907-0.909 for the vector kernel -- the same random-row DRAM
// ceiling reached through the TMA engine -- but slower end to end when the
// index list is read over PCIe (one warp both fetches indices and issues), so
// it stays opt-in (SYNK_GATHER_TMA4=1, device-resident sources only).

__global__ void __launch_bounds__(32) gather_rows_tma4_kernel(
    const __grid_constant__ CUtensorMap tmap, uint64_t src_rows, uint32_t row_bytes,
    const uint64_t* __restrict__ idx, uint64_t n_idx, uint32_t chunk_rows, uint32_t stages, char* __restrict__ dst,
    int* __restrict__ err) {
    extern __shared__ __align__(128) char ring[];
    __shared__ __align__(8) uint64_t full[kMaxStages];
    const int lane = threadIdx.x;
    const uint64_t n_chunks = (n_idx + chunk_rows - 1) / chunk_rows;
    if (blockIdx.x >= n_chunks) return;
    const uint64_t mine = (n_chunks - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const uint32_t stage_bytes = chunk_rows * row_bytes;
    if (lane == 0) {
        for (uint32_t s = 0; s < stages; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&tmap) : "memory");
    }
    __syncwarp();

    auto chunk_start = [&](uint64_t j) { return (blockIdx.x + j * gridDim.x) * (uint64_t)chunk_rows; };
    auto load_index = [&](uint64_t j) -> uint64_t {
        if (j >= mine) return 0;
        const uint64_t r = chunk_start(j) + lane;
        return lane < (int)chunk_rows && r < n_idx ? idx[r] : 0;
    };
    uint64_t q0 = load_index(0), q1 = load_index(1);

    auto issue = [&](uint64_t j, uint64_t my) {
        const uint32_t s = (uint32_t)(j % stages);
        const uint64_t r0 = chunk_start(j);
        const uint32_t cnt = (uint32_t)(n_idx - r0 < chunk_rows ? n_idx - r0 : chunk_rows);
        const bool live = lane < (int)cnt;
        const bool ok = live && my < src_rows;
        if (live && !ok) *(volatile int*)err = 1;
        const int row = ok ? (int)my : 0;  // rows past the chunk or bad: row 0 (fetched, never stored)
        const uint32_t n_req = (cnt + 3) / 4;
        const int q = lane & 7;
        const int c0 = __shfl_sync(0xffffffffu, row, 4 * q), c1 = __shfl_sync(0xffffffffu, row, 4 * q + 1);
        const int c2 = __shfl_sync(0xffffffffu, row, 4 * q + 2), c3 = __shfl_sync(0xffffffffu, row, 4 * q + 3);
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&full[s])),
                         "r"(n_req * 4u * row_bytes)
                         : "memory");
        __syncwarp();
        if (lane < (int)n_req) {
            const uint32_t dst_s = smem_addr(ring + (size_t)s * stage_bytes + (size_t)lane * 4 * row_bytes);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst_s),
                "l"(&tmap), "r"(smem_addr(&full[s])), "r"(0), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
                : "memory");
        }
    };

    const uint64_t ahead = stages - 2 < mine ? stages - 2 : mine;
    for (uint64_t j = 0; j < ahead; ++j) {
        issue(j, q0);
        q0 = q1;
        q1 = load_index(j + 2);
    }
    for (uint64_t j = 0; j < mine; ++j) {
        const uint32_t s = (uint32_t)(j % stages);
        bar_wait(smem_addr(&full[s]), (uint32_t)((j / stages) & 1));
        const uint64_t r0 = chunk_start(j);
        const uint32_t cnt = (uint32_t)(n_idx - r0 < chunk_rows ? n_idx - r0 : chunk_rows);
        __syncwarp();
        if (lane == 0) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + r0 * row_bytes),
                         "r"(smem_addr(ring + (size_t)s * stage_bytes)), "r"(cnt * row_bytes)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        const uint64_t jn = j + ahead;
        if (jn < mine) {
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            issue(jn, q0);
            q0 = q1;
            q1 = load_index(jn + 2);
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn tiled_encoder() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    });
    return fn;
}

int launch_tma4(synk_dev* d, const void* src, uint64_t src_rows, uint64_t row_bytes, const uint64_t* idx,
                uint64_t n_idx, void* dst) {
    EncodeTiledFn enc = tiled_encoder();
    SYNK_REQUIRE(enc != nullptr, SYNK_ECUDA, "cuTensorMapEncodeTiled unavailable");
    CUtensorMap tmap;
    cuuint64_t dims[2] = {row_bytes / 8, src_rows};
    cuuint64_t strides[1] = {row_bytes};
    cuuint32_t box[2] = {(cuuint32_t)(row_bytes / 8), 1};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(&tmap, CU_TENSOR_MAP_DATA_TYPE_INT64, 2, const_cast<void*>(src), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    SYNK_REQUIRE(r == CUDA_SUCCESS, SYNK_ECUDA, "cuTensorMapEncodeTiled (gather4) failed");
    static const uint32_t ctas_per_sm = getenv("SYNK_TMA4_CTAS") ? atoi(getenv("SYNK_TMA4_CTAS")) : 2;
    static const uint32_t max_chunk = getenv("SYNK_TMA4_CHUNK") ? atoi(getenv("SYNK_TMA4_CHUNK")) : 16;
    const uint32_t budget = (224u * 1024u / ctas_per_sm - 1024u) & ~1023u;
    uint32_t chunk_rows = max_chunk;
    while (chunk_rows > 4 && (uint64_t)chunk_rows * row_bytes * 6 > budget) chunk_rows /= 2;
    uint32_t stages = (uint32_t)(budget / (chunk_rows * row_bytes));
    if (stages > kMaxStages) stages = kMaxStages;
    if (stages < 3) return synk::fail(SYNK_EARG, "gather4: rows too wide for the ring");
    const uint32_t smem = stages * chunk_rows * (uint32_t)row_bytes;
    if (int rc = synk::ensure_max_smem((const void*)gather_rows_tma4_kernel, d->device, (int)(224u * 1024u)); rc)
        return rc;
    const uint64_t n_chunks = (n_idx + chunk_rows - 1) / chunk_rows;
    const uint64_t cap = (uint64_t)d->num_sms * ctas_per_sm;
    const unsigned grid = (unsigned)(n_chunks < cap ? n_chunks : cap);
    gather_rows_tma4_kernel<<<grid, 32, smem, d->stream>>>(tmap, src_rows, (uint32_t)row_bytes, idx, n_idx,
                                                           chunk_rows, stages, (char*)dst, d->err_dev);
    SYNK_LAUNCHED("gather_rows_tma4_kernel");
    return SYNK_OK;
}

int launch_bulk(synk_dev* d, const void* src, uint64_t src_rows, uint64_t row_bytes, const uint64_t* idx,
                uint64_t n_idx, void* dst) {
    static const uint32_t ctas_per_sm = getenv("SYNK_GATHER_CTAS") ? atoi(getenv("SYNK_GATHER_CTAS")) : 2;
    static const uint32_t max_chunk = getenv("SYNK_GATHER_CHUNK") ? atoi(getenv("SYNK_GATHER_CHUNK")) : 16;
    const uint32_t kSmemBudget = (224u * 1024u / ctas_per_sm - 1024u) & ~1023u;  // per CTA
    uint32_t chunk_rows = max_chunk;
    while (chunk_rows > 1 && (uint64_t)chunk_rows * row_bytes * 6 > kSmemBudget) chunk_rows /= 2;
    uint32_t stages = (uint32_t)(kSmemBudget / (chunk_rows * row_bytes));
    if (stages > kMaxStages) stages = kMaxStages;
    const uint32_t smem = stages * chunk_rows * (uint32_t)row_bytes;
    if (int rc = synk::ensure_max_smem((const void*)gather_rows_bulk_kernel, d->device, (int)(224u * 1024u)); rc)
        return rc;
    const uint64_t n_chunks = (n_idx + chunk_rows - 1) / chunk_rows;
    const uint64_t cap = (uint64_t)d->num_sms * ctas_per_sm;
    const unsigned grid = (unsigned)(n_chunks < cap ? n_chunks : cap);
    gather_rows_bulk_kernel<<<grid, 32, smem, d->stream>>>((const char*)src, src_rows, (uint32_t)row_bytes, idx,
                                                           n_idx, chunk_rows, stages, (char*)dst, d->err_dev);
    SYNK_LAUNCHED("gather_rows_bulk_kernel");
    return SYNK_OK;
}

}  // namespace

extern "C" int synk_gather_rows_inline(synk_dev* d, const void* src, uint64_t src_rows, uint64_t row_bytes,
                                       const uint64_t* host_idx, uint64_t n_idx, void* dst) {
    if (n_idx == 0 || row_bytes == 0) return SYNK_OK;
    SYNK_REQUIRE(n_idx <= SYNK_GATHER_INLINE_MAX, SYNK_EARG, "synk_gather_rows_inline: list longer than the inline maximum");
    SYNK_REQUIRE(src_rows <= (1ull << 32), SYNK_EARG, "synk_gather_rows_inline: source rows past 2^32");
    InlineIdx p;
    // Narrow + bounds check in one pass (index_narrow.cpp); an out-of-range
    // index reads row 0 (defined data) and raises the rank's sticky flag, so
    // the call fails with SYNK_EBOUNDS at the next synk_sync() exactly like
    // the device check.
    if (synk::narrow_indices(host_idx, n_idx, src_rows, p.idx)) d->err_host[0] = 1;
    synk::DeviceGuard g(d->device);
    const uint64_t a = row_bytes | (uint64_t)(uintptr_t)src | (uint64_t)(uintptr_t)dst;
    const uint32_t n = (uint32_t)n_idx;
    if ((a & 31) == 0) return launch_inline<32>(d, src, row_bytes, p, n, dst);
    if ((a & 15) == 0) return launch_inline<16>(d, src, row_bytes, p, n, dst);
    if ((a & 7) == 0) return launch_inline<8>(d, src, row_bytes, p, n, dst);
    if ((a & 3) == 0) return launch_inline<4>(d, src, row_bytes, p, n, dst);
    return launch_inline<1>(d, src, row_bytes, p, n, dst);
}

extern "C" int synk_gather_rows(synk_dev* d, const void* src, uint64_t src_rows,
                                uint64_t row_bytes, const uint64_t* idx, uint64_t n_idx,
                                void* dst) {
    if (n_idx == 0 || row_bytes == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    uint64_t a = row_bytes | (uint64_t)(uintptr_t)src | (uint64_t)(uintptr_t)dst;
    // The cp.async.bulk kernel is opt-in (SYNK_GATHER_BULK=1): measured slower
    // than the vector kernel at 1 KiB rows (0.87 vs 0.91 of HBM: per-request
    // TMA cost) and on the C5 batch (8 KiB rows, 8192 rows: 32.8 vs 23.2 us);
    // it only won on very large 4 KiB-row launches (5,600 vs 5,494 GB/s).
    static const bool force_bulk = getenv("SYNK_GATHER_BULK") != nullptr;
    static const bool use_tma4 = getenv("SYNK_GATHER_TMA4") != nullptr;  // A/B diagnostics (opt-in)
    if (use_tma4 && (a & 15) == 0 && row_bytes <= 2048 && src_rows < (1ull << 31)) {
        cudaPointerAttributes pa;
        const bool on_device = cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeDevice;
        cudaGetLastError();
        if (on_device) return launch_tma4(d, src, src_rows, row_bytes, idx, n_idx, dst);
    }
    if (force_bulk && (a & 15) == 0 && row_bytes <= 8192)
        return launch_bulk(d, src, src_rows, row_bytes, idx, n_idx, dst);
    // 256-bit lanes (ld/st .v8.b32) when rows and pointers are 32-byte aligned:
    // +2.9 % device, +5.5 % e2e on C2 vs 2 x 16-byte vectors (same-box A/B,
    // profiles/r01_gather.md). SYNK_GATHER_V32=0 keeps 16-byte lanes.
    static const bool v32 = !(getenv("SYNK_GATHER_V32") && getenv("SYNK_GATHER_V32")[0] == '0');
    if (v32 && (a & 31) == 0) return launch<32>(d, src, src_rows, row_bytes, idx, n_idx, dst);
    if ((a & 15) == 0) return launch<16>(d, src, src_rows, row_bytes, idx, n_idx, dst);
    if ((a & 7) == 0) return launch<8>(d, src, src_rows, row_bytes, idx, n_idx, dst);
    if ((a & 3) == 0) return launch<4>(d, src, src_rows, row_bytes, idx, n_idx, dst);
    return launch<1>(d, src, src_rows, row_bytes, idx, n_idx, dst);
}
