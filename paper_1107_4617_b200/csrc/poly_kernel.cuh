// poly_kernel.cuh — f3: the bilateral filter with the polynomial range kernel
// p_N of PAPER.md:202 (order of shiftability 2N+1) in the
// Eq.(5) scaling (reading R17):
//     phi_p(t) = (1 - t^2 / (2 N sigma_r^2))^N,   box spatial kernel,
// evaluated by Algorithm 2 in fp64 with a CHEBYSHEV basis
// of the shift space instead of the monomials t^i.
//
// Why not the monomials: with u = (f - 128)/128 the paper's basis gives
// phi_p(f_y - f_x) = sum_i d_i(u_x) u_y^i with |d_i| up to (1 + 4a)^N,
// a = 128^2/(2 N sigma_r^2) ~ 1/4 at N = N0 — alternating terms of size
// 1e11 (N = 37) .. 1e40 (N = 145) whose sum is O(1): fp32 loses everything
// and fp64 breaks down beyond N ~ 40 (the oracle's fp64 Algorithm 2 with
// monomials is off by 270 grey levels at N = 82, tests/test_oracle_pins.py).
// The same space is spanned by the Chebyshev polynomials T_i(u), i = 0..2N:
//     phi_p(128 (u - v)) = sum_i c_i(v) T_i(u),   |T_i| <= 1 on [-1, 1],
// and since 0 <= phi_p <= 1 on the data range, |c_i(v)| <= 2: no
// cancellation beyond the sums' own magnitude.  The numerator needs
// sum_y phi u_y; u T_0 = T_1 and u T_i = (T_{i+1} + T_{i-1})/2 fold it into
// the same stack: P' = sum_k e_k(v) Sum(T_k), e_0 = c_1/2, e_1 = c_0 + c_2/2,
// e_k = (c_{k-1} + c_{k+1})/2, k = 0..2N+1.  c and e depend only on the centre
// value v (uint8: 256 rows) and come from the host (long double, exact
// Chebyshev interpolation of the degree-2N polynomial at 2N+1 nodes).
//
// Kernel: one CTA per TS x TS output tile.  The tile + r halo of u and of
// two consecutive basis images lives in shared memory (fp64); per basis index
// k: T_k = 2u T_{k-1} - T_{k-2} in place, a vertical moving sum per column
// (recursion), a horizontal moving sum per row segment, and
// Q += c_k(v_x) Sum(T_k), P' += e_k(v_x) Sum(T_k) in registers; out =
// 128 + 128 P'/Q.  A demonstration of the polynomial family's precision
// profile, not a tuned path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kPolyThreads = 256;

template <int TS>
__global__ void __launch_bounds__(kPolyThreads)
poly_tile_kernel(const Params p, const double* __restrict__ coef, int K) {
    // coef: [256][2][K] fp64 — c_k(v) then e_k(v) for centre value v
    constexpr int OPT = TS * TS / kPolyThreads;          // outputs per thread (one row segment)
    constexpr int NSEGH = TS / OPT;                       // segments per row
    static_assert(OPT * kPolyThreads == TS * TS && NSEGH * OPT == TS, "tile shape");
    extern __shared__ double psm[];
    const int r = p.r, W = p.W, H = p.H, L = 2 * r + 1;
    const int TWI = TS + 2 * r, THI = TS + 2 * r;
    const int NE = THI * TWI;
    double* U = psm;                                      // u = (f - 128)/128, tile + halo
    double* A = U + NE;                                   // T_{k-2} -> T_k (in place)
    double* B = A + NE;                                   // T_{k-1}
    double* V = B + NE;                                   // vertical sums, TS x TWI
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * TS, y0 = p.out_row0 + blockIdx.y * TS;

    for (int e = tid; e < NE; e += kPolyThreads) {
        const int ty = e / TWI, tx = e - ty * TWI;
        int gy = reflect101(y0 - r + ty, H) - p.img_row0;
        gy = gy < 0 ? 0 : (gy >= p.img_rows ? p.img_rows - 1 : gy);
        const int gx = reflect101(x0 - r + tx, W);
        const double u = ((double)p.img[(size_t)gy * W + gx] - 128.0) / 128.0;
        U[e] = u;
        A[e] = 1.0;                                       // T_0
        B[e] = u;                                         // T_1
    }
    const int hy = tid / NSEGH, hs = tid % NSEGH, hx0 = hs * OPT;   // horizontal walker
    int vrow[OPT];
    double Q[OPT], P[OPT];
#pragma unroll
    for (int j = 0; j < OPT; ++j) {
        Q[j] = P[j] = 0.0;
        vrow[j] = 0;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < OPT; ++j) {                        // centre values -> coefficient rows
        const double u = U[(hy + r) * TWI + hx0 + j + r];
        vrow[j] = (int)rint(u * 128.0 + 128.0);
    }

    for (int k = 0; k < K; ++k) {
        // T_k: k = 0 is A, k = 1 is B; k >= 2: A <- 2u B - A, then (A, B) swap roles
        const double* Tk = (k == 0) ? A : B;
        if (k >= 2) {
            for (int e = tid; e < NE; e += kPolyThreads) A[e] = fma(2.0 * U[e], B[e], -A[e]);
            double* t = A;
            A = B;
            B = t;
            Tk = B;
            __syncthreads();
        }
        // vertical moving sums (one walker per input column)
        for (int c = tid; c < TWI; c += kPolyThreads) {
            double s = 0.0;
            for (int i = 0; i < L; ++i) s += Tk[i * TWI + c];
            V[c] = s;
            for (int y = 1; y < TS; ++y) {
                s += Tk[(y + 2 * r) * TWI + c] - Tk[(y - 1) * TWI + c];
                V[y * TWI + c] = s;
            }
        }
        __syncthreads();
        // horizontal moving sums and step 3 of Algorithm 2
        {
            const double* vr = V + hy * TWI + hx0;
            double s = 0.0;
            for (int i = 0; i < L; ++i) s += vr[i];
#pragma unroll
            for (int j = 0; j < OPT; ++j) {
                if (j > 0) s += vr[j + 2 * r] - vr[j - 1];
                const double* cr = coef + (size_t)vrow[j] * 2 * K;
                Q[j] = fma(__ldg(cr + k), s, Q[j]);
                P[j] = fma(__ldg(cr + K + k), s, P[j]);
            }
        }
        __syncthreads();
    }
    const int gy = y0 + hy;
    if (gy < p.out_row0 + p.out_rows) {
        const size_t rowoff = (size_t)(gy - p.out_row0) * W;
#pragma unroll
        for (int j = 0; j < OPT; ++j) {
            const int gx = x0 + hx0 + j;
            if (gx < W) {
                const double q = Q[j];
                p.out[rowoff + gx] = (q > 0.0 && isfinite(q)) ? (float)(128.0 + 128.0 * P[j] / q)
                                                             : (float)(U[(hy + r) * TWI + hx0 + j + r] * 128.0 + 128.0);
            }
        }
    }
}

// TS = 32 for r <= 16, 16 for 16 < r <= 32 (shared memory: 3 (TS+2r)^2 + TS (TS+2r) doubles)
inline cudaError_t launch_poly(const Params& p, const double* coef, int K, cudaStream_t s) {
    const int TS = p.r <= 16 ? 32 : 16;
    const int TWI = TS + 2 * p.r;
    const size_t smem = (size_t)(3 * TWI * TWI + TS * TWI) * sizeof(double);
    dim3 grid((p.W + TS - 1) / TS, (p.out_rows + TS - 1) / TS);
    cudaError_t e;
    if (TS == 32) {
        e = cudaFuncSetAttribute(poly_tile_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        poly_tile_kernel<32><<<grid, kPolyThreads, smem, s>>>(p, coef, K);
    } else {
        e = cudaFuncSetAttribute(poly_tile_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        poly_tile_kernel<16><<<grid, kPolyThreads, smem, s>>>(p, coef, K);
    }
    return cudaGetLastError();
}

}  // namespace sf
