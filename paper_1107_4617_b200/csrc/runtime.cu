// runtime.cu — device_info(): the per-device facts, library memory pool and
// auxiliary streams of runtime.h, initialised once per device.
#include "runtime.h"

namespace sf {

namespace {
__global__ void query_nsmid_kernel(int* out) {
    unsigned v;
    asm volatile("mov.u32 %0, %%nsmid;" : "=r"(v));
    *out = (int)v;
}
}  // namespace

DeviceInfo& device_info(int dev) {
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

}  // namespace sf
