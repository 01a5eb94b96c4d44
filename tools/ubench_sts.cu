// Shared-memory store / load throughput through inline PTX (not elided),
// conflict-free, 16 warps per SM, cycles per warp instruction:
//   STS.128, STS.64, LDS.128, and one LDS.128 + one STS.128 per iteration.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_sts tools/ubench_sts.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void sts128(unsigned a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ void sts64(unsigned a, float x, float y) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(x), "f"(y) : "memory");
}
__device__ __forceinline__ float4 lds128(unsigned a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
    return v;
}

template <int MODE>
__global__ void k(int iters, float* out, long long* cyc) {
    __shared__ float4 s[16 * 128];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const unsigned base = (unsigned)__cvta_generic_to_shared(s);
    float4 a = make_float4(lane, 1, 2, 3);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const unsigned addr = base + 16u * (warp * 128 + ((u * 32 + lane + it * 32) & 127));
            if (MODE == 0) sts128(addr, a);
            if (MODE == 1) sts64(addr, a.x, a.y);
            if (MODE == 2) { const float4 v = lds128(addr); a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w; }
            if (MODE == 3) { const float4 v = lds128(base + ((addr - base) ^ 512u)); a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w; sts128(addr, a); }
            if (MODE == 4) { const float4 v = lds128(base + ((addr - base) ^ 512u)); a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
                             const float4 w = lds128(base + ((addr - base) ^ 1024u)); a.x += w.x; a.y += w.y; a.z += w.z; a.w += w.w; sts128(addr, a); }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (a.x == -1.f) out[threadIdx.x] = a.y + a.z + a.w;
}

template <int MODE>
void run(const char* name) {
    float* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8 * 148);
    const int iters = 2000;
    k<MODE><<<148, 512>>>(10, out, cyc);
    k<MODE><<<148, 512>>>(iters, out, cyc);
    long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    const double it_per_sm = 16.0 * 16 * iters;   // warps x unroll x iters
    printf("%-28s %.2f cycles per warp-iteration per SM\n", name, h[0] / it_per_sm);
}

int main() {
    run<0>("STS.128");
    run<1>("STS.64");
    run<2>("LDS.128");
    run<3>("LDS.128 + STS.128");
    run<4>("2 LDS.128 + STS.128");
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
}
