// Shared-memory LDS.128 throughput with duplicate addresses inside a warp:
// does the crossbar merge lanes that read the same 16-byte slot?  pattern:
//   0 = 32 distinct consecutive slots (baseline, 4 wavefronts / instruction)
//   1 = lanes i and i^16 read the same slot (16 unique, halves in different quarters)
//   2 = lanes i and i^1 read the same slot (16 unique, pairs inside a quarter-warp)
//   3 = lanes i and i^4 read the same slot (16 unique, pairs inside a quarter-warp)
//   4 = all lanes one slot
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_bcast tools/ubench_bcast.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(int pattern, int iters, float* out, long long* cyc) {
    __shared__ float4 s[2048];
    for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float4(i, i + 1, i + 2, i + 3);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int slot;
    switch (pattern) {
        case 0: slot = lane; break;
        case 1: slot = lane & 15; break;
        case 2: slot = lane >> 1; break;
        case 3: slot = (lane & 3) | ((lane >> 3) << 2) | (((lane >> 2) & 1) << 4) ; slot = ((lane >> 3) << 2) | (lane & 3); break;
        default: slot = 0;
    }
    const float4* p = s + (warp * 64) % 1024 + slot;
    float4 a = make_float4(0, 0, 0, 0);
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            const float4 v = p[(u * 32 + it) & 1023];
            a.x += v.x; a.y += v.y; a.z += v.z; a.w += v.w;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    if (a.x == -1.f) out[threadIdx.x] = a.y + a.z + a.w;
}

int main() {
    float* out; long long* cyc; cudaMalloc(&out, 4096); cudaMalloc(&cyc, 8 * 148);
    const int iters = 2000;
    for (int pat = 0; pat < 5; ++pat) {
        k<<<148, 512>>>(pat, 10, out, cyc);
        k<<<148, 512>>>(pat, iters, out, cyc);
        long long h[148]; cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
        const double instr_per_sm = 16.0 * 16 * iters;   // warps x unroll x iters
        printf("pattern %d: %.2f cycles per warp-LDS.128 per SM (%.1f B/clk of requested data)\n", pat,
               h[0] / instr_per_sm, instr_per_sm * 512 / h[0] / 1.0);
    }
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
}
