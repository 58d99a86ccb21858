// Diagnostic (not collected): host-visible completion latency on this box.
// One empty kernel + each way of learning that it finished: stream sync,
// cudaStreamQuery spin, event sync, a kernel-written flag in mapped pinned
// memory, a stream write-value to mapped memory. Build + run:
//   nvcc -O2 -gencode arch=compute_100a,code=sm_100a -Iinclude -o /tmp/sync_floor tools/diag/sync_floor.cu \
//     -Lpaper_1710_04162_b200/_lib -lsynk_cuda -lcuda -Xlinker -rpath=$PWD/paper_1710_04162_b200/_lib && /tmp/sync_floor
#include <cuda.h>
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>
#include <cstdint>
#include <random>

#include "synk_cuda.h"

__global__ void empty_kernel() {}
__global__ void flag_kernel(volatile unsigned* flag, unsigned v) {
    __threadfence_system();
    *flag = v;
}
__global__ void fill_flag_kernel(double* out, double v, volatile unsigned* flag, unsigned f) {
    *out = v;
    __threadfence_system();
    *flag = f;
}

// a primary that works ~us microseconds (stands in for the gather), optionally
// releasing its dependents at entry; a dependent that waits on it (PDL)
__global__ void busy_kernel(unsigned ns, int trigger) {
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long t0 = clock64();
    while (clock64() - t0 < (long long)ns * 2) {
    }
}
__global__ void dep_fill_kernel(double* out, double v, int wait) {
    if (wait) asm volatile("griddepcontrol.wait;" ::: "memory");
    *out = v;
}

// gather prototypes: 4 rows per warp, 16-byte lanes, 1 KiB rows
struct IdxParams {
    uint32_t idx[4096];
};
__device__ __forceinline__ void gather4(const uint4* src, uint4* dst, uint64_t r0, const uint64_t* rows, int lane) {
    uint4 v[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int u = 0; u < 2; ++u) v[k][u] = __ldg(src + rows[k] * 64 + lane + 32 * u);
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int u = 0; u < 2; ++u) dst[(r0 + k) * 64 + lane + 32 * u] = v[k][u];
}
__global__ void gather_ptr_kernel(const uint4* src, const uint64_t* idx, uint64_t n, uint4* dst, double* tail,
                                  unsigned* counter, int trigger = 0) {
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x & 31;
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t r0 = w * 4;
    if (r0 < n) {
        uint64_t mine = lane < 4 ? idx[r0 + lane] : 0;
        uint64_t rows[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) rows[k] = __shfl_sync(0xffffffffu, mine, k);
        gather4(src, dst, r0, rows, lane);
    }
    if (tail) {  // last CTA writes the tail value
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (atomicAdd(counter, 1u) == gridDim.x - 1) {
                *counter = 0;
                *tail = (double)n;
            }
        }
    }
}
__global__ void gather_param_kernel(const uint4* src, const __grid_constant__ IdxParams p, uint64_t n, uint4* dst,
                                    int trigger = 0) {
    if (trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const int lane = threadIdx.x & 31;
    const uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint64_t r0 = w * 4;
    if (r0 >= n) return;
    uint64_t rows[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) rows[k] = p.idx[r0 + k];
    gather4(src, dst, r0, rows, lane);
}

template <class F>
static double time_us(F&& f, int n = 2000) {
    for (int i = 0; i < 200; ++i) f(i);
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < n; ++i) f(200 + i);
    auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double, std::micro>(t1 - t0).count() / n;
}

int main() {
    cudaSetDevice(0);
    cudaFree(0);
    int lo = 0, hi = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &hi);
    cudaStream_t s;
    cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi);
    cudaEvent_t ev;
    cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    unsigned* hflag = nullptr;
    cudaHostAlloc(&hflag, 4096, cudaHostAllocMapped | cudaHostAllocPortable);
    unsigned* dflag = nullptr;
    cudaHostGetDevicePointer((void**)&dflag, hflag, 0);
    double* dout = reinterpret_cast<double*>(dflag + 16);
    volatile unsigned* vf = hflag;

    printf("launch only             %6.2f us\n", time_us([&](int) { empty_kernel<<<1, 32, 0, s>>>(); }));
    cudaStreamSynchronize(s);
    printf("stream sync (idle)      %6.2f us\n", time_us([&](int) { cudaStreamSynchronize(s); }));
    printf("stream query (idle)     %6.2f us\n", time_us([&](int) { (void)cudaStreamQuery(s); }));
    printf("device sync (idle)      %6.2f us\n", time_us([&](int) { cudaDeviceSynchronize(); }));
    printf("launch + stream sync    %6.2f us\n", time_us([&](int) {
               empty_kernel<<<1, 32, 0, s>>>();
               cudaStreamSynchronize(s);
           }));
    printf("2 launches + sync       %6.2f us\n", time_us([&](int) {
               empty_kernel<<<1, 32, 0, s>>>();
               empty_kernel<<<1, 32, 0, s>>>();
               cudaStreamSynchronize(s);
           }));
    printf("launch + query spin     %6.2f us\n", time_us([&](int) {
               empty_kernel<<<1, 32, 0, s>>>();
               while (cudaStreamQuery(s) == cudaErrorNotReady) {
               }
           }));
    printf("launch + event sync     %6.2f us\n", time_us([&](int) {
               empty_kernel<<<1, 32, 0, s>>>();
               cudaEventRecord(ev, s);
               cudaEventSynchronize(ev);
           }));
    printf("launch(flag) + spin     %6.2f us\n", time_us([&](int i) {
               flag_kernel<<<1, 1, 0, s>>>(dflag, (unsigned)i + 1);
               while (*vf != (unsigned)i + 1) {
               }
           }));
    cudaStreamSynchronize(s);
    printf("2 launches(flag) + spin %6.2f us\n", time_us([&](int i) {
               empty_kernel<<<1, 32, 0, s>>>();
               fill_flag_kernel<<<1, 1, 0, s>>>(dout, 1.0 * i, dflag, (unsigned)i + 1);
               while (*vf != (unsigned)i + 1) {
               }
           }));
    cudaStreamSynchronize(s);
    CUstream cs = reinterpret_cast<CUstream>(s);
    CUdeviceptr dp = reinterpret_cast<CUdeviceptr>(dflag);
    printf("launch + writeValue spin%6.2f us\n", time_us([&](int i) {
               empty_kernel<<<1, 32, 0, s>>>();
               cuStreamWriteValue32(cs, dp, (cuuint32_t)(i + 1), 0);
               while (*vf != (unsigned)i + 1) {
               }
           }));
    cudaStreamSynchronize(s);
    printf("writeValue only         %6.2f us\n", time_us([&](int i) { cuStreamWriteValue32(cs, dp, (cuuint32_t)(i + 1), 0); }));
    cudaStreamSynchronize(s);
    printf("launch + spin + sync    %6.2f us\n", time_us([&](int i) {
               flag_kernel<<<1, 1, 0, s>>>(dflag, (unsigned)i + 1);
               while (*vf != (unsigned)i + 1) {
               }
               cudaStreamSynchronize(s);
           }));
    for (unsigned ns : {0u, 3000u}) {
        printf("busy(%u ns, 148 CTAs) + sync          %6.2f us\n", ns, time_us([&](int) {
                   busy_kernel<<<148, 128, 0, s>>>(ns, 0);
                   cudaStreamSynchronize(s);
               }));
        printf("busy(%u ns) + fill + sync             %6.2f us\n", ns, time_us([&](int i) {
                   busy_kernel<<<148, 128, 0, s>>>(ns, 0);
                   dep_fill_kernel<<<1, 32, 0, s>>>(dout, i, 0);
                   cudaStreamSynchronize(s);
               }));
        for (int trig = 0; trig < 2; ++trig)
            printf("busy(%u ns, trigger %d) + PDL fill + sync %6.2f us\n", ns, trig, time_us([&](int i) {
                       busy_kernel<<<148, 128, 0, s>>>(ns, trig);
                       cudaLaunchConfig_t cfg = {};
                       cfg.gridDim = dim3(1);
                       cfg.blockDim = dim3(32);
                       cfg.stream = s;
                       cudaLaunchAttribute at[1];
                       at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                       at[0].val.programmaticStreamSerializationAllowed = 1;
                       cfg.attrs = at;
                       cfg.numAttrs = 1;
                       cudaLaunchKernelEx(&cfg, dep_fill_kernel, dout, (double)i, 1);
                       cudaStreamSynchronize(s);
                   }));
    }
    printf("last error: %s\n", cudaGetErrorString(cudaGetLastError()));

    // the C-ABI ops of one single-batch e2e call (bench: 4096 rows of 1 KiB
    // from a 2M-row HBM source, pinned u64 index list read in place)
    synk_dev* d = nullptr;
    int dev0 = 0;
    synk_open(1, &dev0, &d);
    const uint64_t rows = 2000000, rb = 1024, B = 4096;
    void *src = nullptr, *dst = nullptr, *didx = nullptr, *hidx = nullptr, *stage = nullptr;
    synk_alloc(d, rows * rb, &src);
    synk_alloc(d, B * rb, &dst);
    synk_alloc(d, B * 8, &didx);
    synk_host_alloc(B * 8 * 64, &hidx);
    synk_host_alloc(4096, &stage);
    std::mt19937_64 g(1);
    for (uint64_t i = 0; i < B * 64; ++i) static_cast<uint64_t*>(hidx)[i] = g() % rows;
    synk_copy(d, didx, hidx, B * 8);
    synk_sync(d);
    const void* hv = nullptr;
    synk_host_device_ptr(hidx, &hv);
    const void* sv = nullptr;
    synk_host_device_ptr(stage, &sv);
    auto hidx_of = [&](int i) { return static_cast<const uint64_t*>(hv) + (i % 64) * B; };
    printf("synk fill + sync              %6.2f us\n", time_us([&](int) {
               synk_fill(d, SYNK_F64, const_cast<void*>(sv), 1.0, 1);
               synk_sync(d);
           }));
    printf("synk gather(dev idx) + sync   %6.2f us\n", time_us([&](int) {
               synk_gather_rows(d, src, rows, rb, (const uint64_t*)didx, B, dst);
               synk_sync(d);
           }));
    printf("synk gather(host idx) + sync  %6.2f us\n", time_us([&](int i) {
               synk_gather_rows(d, src, rows, rb, hidx_of(i), B, dst);
               synk_sync(d);
           }));
    printf("synk gather(host) + fill + sync %6.2f us\n", time_us([&](int i) {
               synk_gather_rows(d, src, rows, rb, hidx_of(i), B, dst);
               synk_fill(d, SYNK_F64, const_cast<void*>(sv), 1.0, 1);
               synk_sync(d);
           }));
    printf("host_device_ptr               %6.2f us\n", time_us([&](int i) {
               const void* x = nullptr;
               synk_host_device_ptr(hidx_of(i), &x);
           }));
    printf("alloc+free 4 MiB              %6.2f us\n", time_us([&](int) {
               void* x = nullptr;
               synk_alloc(d, B * rb, &x);
               synk_free(d, x);
           }));
    {
        uint4* s4 = static_cast<uint4*>(src);
        uint4* d4 = static_cast<uint4*>(dst);
        unsigned* counter = nullptr;
        cudaMalloc(&counter, 4);
        cudaMemset(counter, 0, 4);
        cudaStream_t ds = static_cast<cudaStream_t>(synk_dev_stream(d));
        static IdxParams prm[64];
        for (int j = 0; j < 64; ++j)
            for (uint64_t i = 0; i < B; ++i) prm[j].idx[i] = (uint32_t)static_cast<uint64_t*>(hidx)[j * B + i];
        printf("proto gather(dev idx) + sync        %6.2f us\n", time_us([&](int) {
                   gather_ptr_kernel<<<128, 256, 0, ds>>>(s4, (const uint64_t*)didx, B, d4, nullptr, nullptr);
                   cudaStreamSynchronize(ds);
               }));
        printf("proto gather(host idx) + sync       %6.2f us\n", time_us([&](int i) {
                   gather_ptr_kernel<<<128, 256, 0, ds>>>(s4, hidx_of(i), B, d4, nullptr, nullptr);
                   cudaStreamSynchronize(ds);
               }));
        printf("proto gather(param idx) launch only %6.2f us\n", time_us([&](int i) {
                   gather_param_kernel<<<128, 256, 0, ds>>>(s4, prm[i % 64], B, d4);
               }, 500));
        cudaStreamSynchronize(ds);
        printf("proto gather(param idx) + sync      %6.2f us\n", time_us([&](int i) {
                   gather_param_kernel<<<128, 256, 0, ds>>>(s4, prm[i % 64], B, d4);
                   cudaStreamSynchronize(ds);
               }));
        auto pdl_fill = [&](int i) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(1);
            cfg.blockDim = dim3(32);
            cfg.stream = ds;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            at[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaLaunchKernelEx(&cfg, dep_fill_kernel, (double*)sv, (double)i, 1);
        };
        for (int rep = 0; rep < 3; ++rep) {
            printf("rep %d\n", rep);
            printf("proto host idx + fill        %6.2f us\n", time_us([&](int i) {
                       gather_ptr_kernel<<<128, 256, 0, ds>>>(s4, hidx_of(i), B, d4, nullptr, nullptr, 0);
                       dep_fill_kernel<<<1, 32, 0, ds>>>((double*)sv, (double)i, 0);
                       cudaStreamSynchronize(ds);
                   }));
            for (int trig = 0; trig < 2; ++trig)
                printf("proto host idx (trig %d) + PDL fill %6.2f us\n", trig, time_us([&](int i) {
                           gather_ptr_kernel<<<128, 256, 0, ds>>>(s4, hidx_of(i), B, d4, nullptr, nullptr, trig);
                           pdl_fill(i);
                           cudaStreamSynchronize(ds);
                       }));
            printf("proto host idx + tail        %6.2f us\n", time_us([&](int i) {
                       gather_ptr_kernel<<<128, 256, 0, ds>>>(s4, hidx_of(i), B, d4, (double*)sv, counter, 0);
                       cudaStreamSynchronize(ds);
                   }));
            printf("proto param idx + fill       %6.2f us\n", time_us([&](int i) {
                       gather_param_kernel<<<128, 256, 0, ds>>>(s4, prm[i % 64], B, d4, 0);
                       dep_fill_kernel<<<1, 32, 0, ds>>>((double*)sv, (double)i, 0);
                       cudaStreamSynchronize(ds);
                   }));
            for (int trig = 0; trig < 2; ++trig)
                printf("proto param idx (trig %d) + PDL fill %6.2f us\n", trig, time_us([&](int i) {
                           gather_param_kernel<<<128, 256, 0, ds>>>(s4, prm[i % 64], B, d4, trig);
                           pdl_fill(i);
                           cudaStreamSynchronize(ds);
                       }));
            printf("proto param idx + fill(dev)  %6.2f us\n", time_us([&](int i) {
                       gather_param_kernel<<<128, 256, 0, ds>>>(s4, prm[i % 64], B, d4, 0);
                       dep_fill_kernel<<<1, 32, 0, ds>>>((double*)didx + 4095, (double)i, 0);
                       cudaStreamSynchronize(ds);
                   }));
        }
        printf("proto error: %s\n", cudaGetErrorString(cudaGetLastError()));
    }
    synk_close(d);
    return 0;
}
