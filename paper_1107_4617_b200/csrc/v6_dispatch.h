// v6_dispatch.h — the v6 band-sweep kernel (box_v6.cuh) for every radius
// 1..32, instantiated in eight translation units (v6_part.cu compiled with
// SF_V6_PART = 0..7, radii 4i+1..4i+4; _build.py compiles them in parallel).
//
// launch_v6(R, om, maxseg, ...): om = outgoing rows by MUFU (no rotation
// drift, reading R15); maxseg = RB-row batches per running-sum segment,
// <= 0 unlimited.
#pragma once

#include <cuda_runtime.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kV6MaxR = 32;

#define SF_V6_DECL(i)                                                                                  \
    cudaError_t launch_v6_part##i(int R, bool om, int maxseg, const Params& p, const PairTable& t,   \
                                  double gamma, cudaStream_t s);
SF_V6_DECL(0)
SF_V6_DECL(1)
SF_V6_DECL(2)
SF_V6_DECL(3)
SF_V6_DECL(4)
SF_V6_DECL(5)
SF_V6_DECL(6)
SF_V6_DECL(7)
#undef SF_V6_DECL

inline cudaError_t launch_v6(int R, bool om, int maxseg, const Params& p, const PairTable& t, double gamma,
                             cudaStream_t s) {
    if (R < 1 || R > kV6MaxR) return cudaErrorInvalidValue;
    switch ((R - 1) / 4) {
        case 0: return launch_v6_part0(R, om, maxseg, p, t, gamma, s);
        case 1: return launch_v6_part1(R, om, maxseg, p, t, gamma, s);
        case 2: return launch_v6_part2(R, om, maxseg, p, t, gamma, s);
        case 3: return launch_v6_part3(R, om, maxseg, p, t, gamma, s);
        case 4: return launch_v6_part4(R, om, maxseg, p, t, gamma, s);
        case 5: return launch_v6_part5(R, om, maxseg, p, t, gamma, s);
        case 6: return launch_v6_part6(R, om, maxseg, p, t, gamma, s);
        default: return launch_v6_part7(R, om, maxseg, p, t, gamma, s);
    }
}

}  // namespace sf
