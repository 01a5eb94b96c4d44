// tools/ubench2.cu — B200 pipe-mix microbenchmarks for the v4 kernel design
// (DESIGN.md §5): is SHFL a separate resource from LDS bandwidth; how FFMA2
// overlaps MUFU and LDS; STS.128 / LDS.64 bandwidth.  One 1024-thread CTA per
// SM; per-SM rates from clock64 around the loop (max over SMs).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench2 tools/ubench2.cu
#include <cstdio>
#include <cuda_runtime.h>

#define ITERS 2048

template <int MODE>
__global__ void __launch_bounds__(1024, 1) bench(float* out, long long* cyc, float b0, float c0) {
    __shared__ float2 sm[4096];
    const int tid = threadIdx.x;
    for (int i = tid; i < 4096; i += 1024) sm[i] = make_float2(i, i + 1);
    float2 p[8];
    float a[8];
    for (int j = 0; j < 8; ++j) {
        p[j] = make_float2(tid * 0.001f + j, j - 1.f);
        a[j] = tid * 0.002f + j;
    }
    const float2 b2 = make_float2(b0 + tid * 1e-7f, c0), c2 = make_float2(c0, b0);
    __syncthreads();
    long long t0 = clock64();
    for (int it = 0; it < ITERS; ++it) {
        if (MODE == 0) {            // LDS.64 conflict-free: 8 per iter
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float2 v = sm[(tid + (it * 8 + j) * 32) & 4095];
                p[j].x += v.x;
                p[j].y += v.y;
            }
        } else if (MODE == 1) {     // STS.128: 8 per iter
            float4* s4 = reinterpret_cast<float4*>(sm);
#pragma unroll
            for (int j = 0; j < 8; ++j) s4[(tid + j * 1024 + it) & 2047] = make_float4(a[j], a[j], p[j].x, p[j].y);
            a[it & 7] += 1.f;
        } else if (MODE == 2) {     // 4 LDS.64 + 8 SHFL per iter
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float2 v = sm[(tid + (it * 4 + j) * 32) & 4095];
                p[j].x += v.x;
                p[j].y += v.y;
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = __shfl_xor_sync(0xffffffffu, a[j], 1 + (j & 3)) + b0;
        } else if (MODE == 3) {     // 8 SHFL alone
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = __shfl_xor_sync(0xffffffffu, a[j], 1 + (j & 3)) + b0;
        } else if (MODE == 4) {     // 8 FFMA2 + 1 MUFU per iter
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = __ffma2_rn(p[j], b2, c2);
            a[it & 7] = __sinf(a[it & 7]);
        } else if (MODE == 5) {     // 8 FFMA2 + 2 LDS.64 per iter
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = __ffma2_rn(p[j], b2, c2);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float2 v = sm[(tid + (it * 2 + j) * 32) & 4095];
                a[j] += v.x + v.y;
            }
        } else if (MODE == 6) {     // 8 FFMA2 + 8 FFMA per iter
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = __ffma2_rn(p[j], b2, c2);
#pragma unroll
            for (int j = 0; j < 8; ++j) a[j] = fmaf(a[j], b0, c0);
        } else if (MODE == 7) {     // 8 FFMA2 + 2 MUFU + 2 LDS.64 per iter
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = __ffma2_rn(p[j], b2, c2);
            a[it & 7] = __sinf(a[it & 7]);
            a[(it + 4) & 7] = __cosf(a[(it + 4) & 7]);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                const float2 v = sm[(tid + (it * 2 + j) * 32) & 4095];
                a[j] += v.x - v.y;
            }
        } else if (MODE == 8) {     // 8 FADD2 alone
#pragma unroll
            for (int j = 0; j < 8; ++j) p[j] = __fadd2_rn(p[j], b2);
        }
    }
    long long t1 = clock64();
    float s = 0.f;
    for (int j = 0; j < 8; ++j) s += a[j] + p[j].x + p[j].y;
    out[blockIdx.x * 1024 + tid] = s;
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int sms, float* d_out, long long* d_cyc) {
    bench<MODE><<<sms, 1024>>>(d_out, d_cyc, 1.0001f, 0.5f);
    bench<MODE><<<sms, 1024>>>(d_out, d_cyc, 1.0001f, 0.5f);
    cudaDeviceSynchronize();
    long long h[1024];
    cudaMemcpy(h, d_cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
    double mx = 0;
    for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
    // warp-iterations per SM-clock: 32 warps x ITERS
    const double wit = 32.0 * ITERS / mx;
    printf("%-44s %7.3f warp-iters/clk/SM  (%.0f cycles)\n", name, wit, mx);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* d_out;
    long long* d_cyc;
    cudaMalloc(&d_out, sizeof(float) * sms * 1024);
    cudaMalloc(&d_cyc, sizeof(long long) * sms);
    printf("SMs: %d   (per iter instruction mix in the name; x warp-iters = instr/clk/SM)\n", sms);
    run<0>("8 LDS.64", sms, d_out, d_cyc);
    run<1>("8 STS.128", sms, d_out, d_cyc);
    run<2>("4 LDS.64 + 8 SHFL", sms, d_out, d_cyc);
    run<3>("8 SHFL", sms, d_out, d_cyc);
    run<4>("8 FFMA2 + 1 MUFU", sms, d_out, d_cyc);
    run<5>("8 FFMA2 + 2 LDS.64", sms, d_out, d_cyc);
    run<6>("8 FFMA2 + 8 FFMA", sms, d_out, d_cyc);
    run<7>("8 FFMA2 + 2 MUFU + 2 LDS.64", sms, d_out, d_cyc);
    run<8>("8 FADD2", sms, d_out, d_cyc);
    printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
