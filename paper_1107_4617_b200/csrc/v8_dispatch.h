// v8_dispatch.h — the v6 band-sweep kernel (box_v8.cuh) for every radius
// 1..24, instantiated in six translation units (v8_part.cu compiled with
// SF_V8_PART = 0..5, radii 4i+1..4i+4; _build.py compiles them in parallel).
//
// launch_v8(R, om, maxseg, ...): om = outgoing rows by MUFU (no rotation
// drift, reading R15); maxseg = RB-row batches per running-sum segment,
// <= 0 unlimited.
#pragma once

#include <cuda_runtime.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kV8MaxR = 24;

#define SF_V8_DECL(i)                                                                                  \
    cudaError_t launch_v8_part##i(int R, bool om, int maxseg, const Params& p, const PairTable& t,   \
                                  double gamma, cudaStream_t s);
SF_V8_DECL(0)
SF_V8_DECL(1)
SF_V8_DECL(2)
SF_V8_DECL(3)
SF_V8_DECL(4)
SF_V8_DECL(5)
#undef SF_V8_DECL

inline cudaError_t launch_v8(int R, bool om, int maxseg, const Params& p, const PairTable& t, double gamma,
                             cudaStream_t s) {
    if (R < 1 || R > kV8MaxR) return cudaErrorInvalidValue;
    switch ((R - 1) / 4) {
        case 0: return launch_v8_part0(R, om, maxseg, p, t, gamma, s);
        case 1: return launch_v8_part1(R, om, maxseg, p, t, gamma, s);
        case 2: return launch_v8_part2(R, om, maxseg, p, t, gamma, s);
        case 3: return launch_v8_part3(R, om, maxseg, p, t, gamma, s);
        case 4: return launch_v8_part4(R, om, maxseg, p, t, gamma, s);
        default: return launch_v8_part5(R, om, maxseg, p, t, gamma, s);
    }
}

}  // namespace sf
