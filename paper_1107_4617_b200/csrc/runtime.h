// runtime.h — device-side runtime services of libsf.so (internal, not ABI):
//
//  * per-device facts queried once (SM count, %nsmid, the SM-id range);
//  * a library-private stream-ordered memory pool with an unbounded release
//    threshold, so the scratch of one call is recycled by the next instead of
//    being unmapped at every synchronisation and re-mapped (cudaMallocAsync on
//    the default pool costs milliseconds per call for the 10-300 MB scratch);
//  * the scratch layout rule: kernels that run one CTA per SM index their
//    running-sum scratch by %smid, so the scratch is sized by the SMs (tens of
//    MB, L2-resident) rather than by the grid.
// Thread safety: first-use initialisation is guarded by std::call_once per
// device; cudaMallocFromPoolAsync / cudaFreeAsync are thread-safe.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>

namespace sf {

struct DeviceInfo {
    int sms = 0;          // cudaDevAttrMultiProcessorCount
    int nsmid = 0;        // upper bound of %smid (+1)
    cudaMemPool_t pool = nullptr;
    cudaStream_t aux[2] = {nullptr, nullptr};   // host-path copy/compute pipelining
    cudaError_t err = cudaSuccess;
};

__global__ void query_nsmid_kernel(int* out) {
    unsigned v;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(v));
    *out = (int)v;
}

__device__ __forceinline__ int sm_id() {
    unsigned v;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
    return (int)v;
}

constexpr int kMaxDevices = 64;

inline DeviceInfo& device_info(int dev) {
    static DeviceInfo info[kMaxDevices];
    static std::once_flag once[kMaxDevices];
    std::call_once(once[dev], [dev] {
        DeviceInfo& d = info[dev];
        int prev = 0;
        cudaGetDevice(&prev);
        if ((d.err = cudaSetDevice(dev)) != cudaSuccess) return;
        cudaDeviceGetAttribute(&d.sms, cudaDevAttrMultiProcessorCount, dev);
        int* p = nullptr;
        if ((d.err = cudaMalloc(&p, sizeof(int))) == cudaSuccess) {
            query_nsmid_kernel<<<1, 1>>>(p);
            int h = 0;
            d.err = cudaMemcpy(&h, p, sizeof(int), cudaMemcpyDeviceToHost);
            cudaFree(p);
            d.nsmid = h > d.sms ? h : d.sms;
        }
        if (d.err == cudaSuccess) {
            cudaMemPoolProps props = {};
            props.allocType = cudaMemAllocationTypePinned;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if ((d.err = cudaMemPoolCreate(&d.pool, &props)) == cudaSuccess) {
                uint64_t keep = UINT64_MAX;
                cudaMemPoolSetAttribute(d.pool, cudaMemPoolAttrReleaseThreshold, &keep);
            }
            for (int i = 0; i < 2 && d.err == cudaSuccess; ++i)
                d.err = cudaStreamCreateWithFlags(&d.aux[i], cudaStreamNonBlocking);
        }
        cudaSetDevice(prev);
    });
    return info[dev];
}

inline DeviceInfo& current_device_info() {
    int dev = 0;
    cudaGetDevice(&dev);
    return device_info(dev < kMaxDevices ? dev : 0);
}

// stream-ordered scratch from the library pool (freed with scratch_free on the same stream)
inline cudaError_t scratch_alloc(void** p, size_t bytes, cudaStream_t s) {
    DeviceInfo& d = current_device_info();
    if (d.err != cudaSuccess) return d.err;
    return cudaMallocFromPoolAsync(p, bytes > 0 ? bytes : 16, d.pool, s);
}

// kernels enqueued by the last launcher call on this thread (bench accounting)
inline int& launch_counter() {
    static thread_local int n = 0;
    return n;
}

inline void scratch_free(void* p, cudaStream_t s) {
    if (p) cudaFreeAsync(p, s);
}

}  // namespace sf
