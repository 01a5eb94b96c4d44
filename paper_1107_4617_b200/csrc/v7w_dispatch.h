// v7w_dispatch.h — the wide large-radius v7 kernel (box_v7.cuh, WIDE = true:
// 12 producer warps, 256-column strips) for every radius 9..64, instantiated
// in eight translation units (v7w_part.cu with SF_V7W_PART = 0..7, radii
// 9+7i .. 15+7i; _build.py compiles them in parallel).
#pragma once

#include <cuda_runtime.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kV7WMinR = 9, kV7WMaxR = 64;

#define SF_V7W_DECL(i) \
    cudaError_t launch_v7w_part##i(int R, const Params& p, const PairTable& t, double gamma, cudaStream_t s);
SF_V7W_DECL(0)
SF_V7W_DECL(1)
SF_V7W_DECL(2)
SF_V7W_DECL(3)
SF_V7W_DECL(4)
SF_V7W_DECL(5)
SF_V7W_DECL(6)
SF_V7W_DECL(7)
#undef SF_V7W_DECL

inline cudaError_t launch_v7w(int R, const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    if (R < kV7WMinR || R > kV7WMaxR) return cudaErrorInvalidValue;
    switch ((R - kV7WMinR) / 7) {
        case 0: return launch_v7w_part0(R, p, t, gamma, s);
        case 1: return launch_v7w_part1(R, p, t, gamma, s);
        case 2: return launch_v7w_part2(R, p, t, gamma, s);
        case 3: return launch_v7w_part3(R, p, t, gamma, s);
        case 4: return launch_v7w_part4(R, p, t, gamma, s);
        case 5: return launch_v7w_part5(R, p, t, gamma, s);
        case 6: return launch_v7w_part6(R, p, t, gamma, s);
        default: return launch_v7w_part7(R, p, t, gamma, s);
    }
}

}  // namespace sf
