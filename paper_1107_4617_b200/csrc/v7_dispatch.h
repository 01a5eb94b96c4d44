// v7_dispatch.h — the v7 band-sweep kernel (box_v7.cuh) for every radius
// 1..24, instantiated in six translation units (v7_part.cu compiled with
// SF_V7_PART = 0..5, radii 4i+1..4i+4; _build.py compiles them in parallel).
//
// launch_v7(R, om, maxseg, ...): om = outgoing rows by MUFU (no rotation
// drift, reading R15); maxseg = RB-row batches per running-sum segment,
// <= 0 unlimited.
#pragma once

#include <cuda_runtime.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kV7MaxR = 24;

#define SF_V7_DECL(i)                                                                                  \
    cudaError_t launch_v7_part##i(int R, bool om, int maxseg, const Params& p, const PairTable& t,   \
                                  double gamma, cudaStream_t s);
SF_V7_DECL(0)
SF_V7_DECL(1)
SF_V7_DECL(2)
SF_V7_DECL(3)
SF_V7_DECL(4)
SF_V7_DECL(5)
#undef SF_V7_DECL

inline cudaError_t launch_v7(int R, bool om, int maxseg, const Params& p, const PairTable& t, double gamma,
                             cudaStream_t s) {
    if (R < 1 || R > kV7MaxR) return cudaErrorInvalidValue;
    switch ((R - 1) / 4) {
        case 0: return launch_v7_part0(R, om, maxseg, p, t, gamma, s);
        case 1: return launch_v7_part1(R, om, maxseg, p, t, gamma, s);
        case 2: return launch_v7_part2(R, om, maxseg, p, t, gamma, s);
        case 3: return launch_v7_part3(R, om, maxseg, p, t, gamma, s);
        case 4: return launch_v7_part4(R, om, maxseg, p, t, gamma, s);
        default: return launch_v7_part5(R, om, maxseg, p, t, gamma, s);
    }
}

}  // namespace sf
