// Input indexing: dst[j,:] = src[idx[j],:]   (gather_rows, tensor.cpp:200-217)
//
// HBM-bound row gather. One warp owns ROWS destination rows at a time: lanes
// < ROWS fetch the indices, shuffle them to the warp, then every lane streams
// 16-byte vectors of all ROWS rows (ROWS x UNROLL independent 128-bit loads in
// flight per lane before the first store), so a 1 KiB row is two fully
// coalesced 512-byte warp transactions per row and no shared memory is
// needed. Source rows are read with ld.global.nc.L1::no_allocate (each row is
// touched once); the source may be an HBM mirror or pinned, mapped host memory
// (then the same loads travel over PCIe). Out-of-range indices set the rank's
// device error flag, reported as BoundsError at the phase-exit synk_sync().

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

constexpr int kRows = 4;    // rows in flight per warp
constexpr int kUnroll = 2;  // vectors per row in flight per lane
constexpr int kBlock = 256;

template <int BYTES>
__global__ void __launch_bounds__(kBlock) gather_rows_kernel(
    const typename Vec<BYTES>::T* __restrict__ src, uint64_t src_rows, uint64_t row_vecs,
    const uint64_t* __restrict__ idx, uint64_t n_idx, typename Vec<BYTES>::T* __restrict__ dst,
    int* __restrict__ err) {
    using V = typename Vec<BYTES>::T;
    const int lane = threadIdx.x & 31;
    const uint64_t warp = ((uint64_t)blockIdx.x * kBlock + threadIdx.x) >> 5;
    const uint64_t nwarps = ((uint64_t)gridDim.x * kBlock) >> 5;

    for (uint64_t r0 = warp * kRows; r0 < n_idx; r0 += nwarps * kRows) {
        uint64_t mine = 0;
        int ok = 0;
        if (lane < kRows && r0 + lane < n_idx) {
            mine = idx[r0 + lane];
            ok = mine < src_rows;
            if (!ok) *(volatile int*)err = 1;  // mapped host flag: plain store, every writer stores 1
        }
        uint64_t row[kRows];
        int valid[kRows];
#pragma unroll
        for (int k = 0; k < kRows; ++k) {
            row[k] = __shfl_sync(0xffffffffu, mine, k);
            valid[k] = __shfl_sync(0xffffffffu, ok, k);
        }
        for (uint64_t v0 = lane; v0 < row_vecs; v0 += 32 * kUnroll) {
            V buf[kRows][kUnroll];
#pragma unroll
            for (int k = 0; k < kRows; ++k)
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    uint64_t v = v0 + (uint64_t)u * 32;
                    if (valid[k] && v < row_vecs) buf[k][u] = Vec<BYTES>::load(src + row[k] * row_vecs + v);
                }
#pragma unroll
            for (int k = 0; k < kRows; ++k)
#pragma unroll
                for (int u = 0; u < kUnroll; ++u) {
                    uint64_t v = v0 + (uint64_t)u * 32;
                    if (valid[k] && v < row_vecs) dst[(r0 + k) * row_vecs + v] = buf[k][u];
                }
        }
    }
}

template <int BYTES>
int launch(synk_dev* d, const void* src, uint64_t src_rows, uint64_t row_bytes,
           const uint64_t* idx, uint64_t n_idx, void* dst) {
    using V = typename Vec<BYTES>::T;
    uint64_t warps = (n_idx + kRows - 1) / kRows;
    uint64_t blocks = (warps * 32 + kBlock - 1) / kBlock;
    uint64_t cap = (uint64_t)d->num_sms * 8;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    gather_rows_kernel<BYTES><<<(unsigned)blocks, kBlock, 0, d->stream>>>(
        (const V*)src, src_rows, row_bytes / BYTES, idx, n_idx, (V*)dst, d->err_dev);
    SYNK_LAUNCHED("gather_rows_kernel");
    return SYNK_OK;
}

}  // namespace

extern "C" int synk_gather_rows(synk_dev* d, const void* src, uint64_t src_rows,
                                uint64_t row_bytes, const uint64_t* idx, uint64_t n_idx,
                                void* dst) {
    if (n_idx == 0 || row_bytes == 0) return SYNK_OK;
    synk::DeviceGuard g(d->device);
    uint64_t a = row_bytes | (uint64_t)(uintptr_t)src | (uint64_t)(uintptr_t)dst;
    if ((a & 15) == 0) return launch<16>(d, src, src_rows, row_bytes, idx, n_idx, dst);
    if ((a & 7) == 0) return launch<8>(d, src, src_rows, row_bytes, idx, n_idx, dst);
    if ((a & 3) == 0) return launch<4>(d, src, src_rows, row_bytes, idx, n_idx, dst);
    return launch<1>(d, src, src_rows, row_bytes, idx, n_idx, dst);
}
