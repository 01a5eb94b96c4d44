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

__device__ __forceinline__ int sm_id() {
    unsigned v;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(v));
    return (int)v;
}

constexpr int kMaxDevices = 64;

// per-device facts, pool and streams, initialised on first use (runtime.cu)
DeviceInfo& device_info(int dev);

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
