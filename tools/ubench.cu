// tools/ubench.cu — B200 pipe-throughput microbenchmarks that size the kernel
// design: FP32 FFMA/FADD (3-register and packed f32x2 forms),
// MUFU sin/cos, LDS.32/LDS.128, SHFL.  One 1024-thread CTA per SM; per-SM
// throughput = lane-ops / SM cycles (clock64 around the loop).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 4096

__device__ __forceinline__ unsigned long long f2u(float2 v) { return *reinterpret_cast<unsigned long long*>(&v); }
__device__ __forceinline__ float2 u2f(unsigned long long v) { return *reinterpret_cast<float2*>(&v); }

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)), "l"(f2u(c)));
    return u2f(d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long d;
    asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(f2u(a)), "l"(f2u(b)));
    return u2f(d);
}

template <int MODE>
__global__ void __launch_bounds__(1024, 1) bench(float* out, long long* cyc, float b0, float c0) {
    __shared__ float4 sm[2048];
    const int tid = threadIdx.x;
    for (int i = tid; i < 2048; i += 1024) sm[i] = make_float4(i, i + 1, i + 2, i + 3);
    float a[8];
    float2 p[8];
    for (int j = 0; j < 8; ++j) { a[j] = tid * 0.001f + j; p[j] = make_float2(a[j], a[j] + 1.f); }
    float b = b0 + tid * 1e-7f, c = c0 - tid * 1e-7f;
    float2 b2 = make_float2(b, c), c2 = make_float2(c, b);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        if (MODE == 0) {            // FFMA, 3 distinct registers
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b, c);
        } else if (MODE == 1) {     // FFMA with immediate
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], 0.999f, c);
        } else if (MODE == 2) {     // FADD
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] + b;
        } else if (MODE == 3) {     // FFMA2 packed
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = ffma2(p[j], b2, c2);
        } else if (MODE == 4) {     // FADD2 packed
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = fadd2(p[j], b2);
        } else if (MODE == 5) {     // MUFU.SIN (+ range-reduction FMUL)
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = __sinf(a[j]);
        } else if (MODE == 6) {     // LDS.128, conflict-free
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                float4 v = sm[(tid + it * 8 + j) & 2047];
                a[j] += v.x + v.w;
            }
        } else if (MODE == 7) {     // LDS.32, conflict-free
            const float* s1 = reinterpret_cast<const float*>(sm);
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] += s1[(tid + it * 8 + j) & 8191];
        } else if (MODE == 8) {     // SHFL
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = __shfl_xor_sync(0xffffffffu, a[j], j + 1) + b;
        } else if (MODE == 9) {     // mix: 16 FFMA + 1 MUFU.SIN per 8 chains... per chain 2 FFMA, 1/8 MUFU
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(fmaf(a[j], b, c), c, b);
            a[it & 7] = __sinf(a[it & 7]);
        } else if (MODE == 10) {    // mix: 8 FADD + 1 LDS.128
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = a[j] + b;
            float4 v = sm[(tid + it) & 2047];
            a[0] += v.y;
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int j = 0; j < 8; ++j) s += a[j] + p[j].x + p[j].y;
    out[blockIdx.x * 1024 + tid] = s;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, double ops_per_iter_per_thread, int sms, float* d_out, long long* d_cyc) {
    bench<MODE><<<sms, 1024>>>(d_out, d_cyc, 1.0001f, 0.5f);
    bench<MODE><<<sms, 1024>>>(d_out, d_cyc, 1.0001f, 0.5f);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    double lane_ops = 1024.0 * ITERS * ops_per_iter_per_thread;
    printf("%-34s %8.1f lane-ops/clk/SM  (%.0f cycles)\n", name, lane_ops / mx, mx);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d_out;
    long long* d_cyc;
    cudaMalloc(&d_out, sizeof(float) * sms * 1024);
    cudaMalloc(&d_cyc, sizeof(long long) * sms);
    printf("SMs: %d\n", sms);
    run<0>("FFMA (3 regs)", 8, sms, d_out, d_cyc);
    run<1>("FFMA (imm)", 8, sms, d_out, d_cyc);
    run<2>("FADD", 8, sms, d_out, d_cyc);
    run<3>("FFMA2 (f32x2; 2 FMA per lane-op)", 16, sms, d_out, d_cyc);
    run<4>("FADD2 (f32x2; 2 adds per lane-op)", 16, sms, d_out, d_cyc);
    run<5>("MUFU.SIN (__sinf)", 8, sms, d_out, d_cyc);
    run<6>("LDS.128 (lanes x 16B)", 8, sms, d_out, d_cyc);
    run<7>("LDS.32", 8, sms, d_out, d_cyc);
    run<8>("SHFL", 8, sms, d_out, d_cyc);
    run<9>("mix 16 FFMA + 1 MUFU (FFMA count)", 16, sms, d_out, d_cyc);
    run<10>("mix 8 FADD + 1 LDS.128 (FADD count)", 8, sms, d_out, d_cyc);
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
