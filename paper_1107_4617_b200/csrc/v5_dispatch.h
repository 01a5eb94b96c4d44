// v5_dispatch.h — the v5 band-sweep kernel (box_v5.cuh) for every radius
// 1..64, instantiated in eight translation units (v5_part.cu compiled with
// SF_V5_PART = 0..7, radii 8i+1..8i+8; _build.py compiles them in parallel).
//
// launch_v5(R, om, maxseg, cluster, ...): om = outgoing rows by MUFU
// (required for R > 32); maxseg = RB-row batches per running-sum segment,
// <= 0 unlimited; cluster: unused (the two-CTA cluster variant v5c was
// measured slower and retired).
#pragma once

#include <cuda_runtime.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kV5MaxR = 64;

#define SF_V5_DECL(i)                                                                                  \
    cudaError_t launch_v5_part##i(int R, bool om, int maxseg, bool cluster, const Params& p,         \
                                  const PairTable& t, double gamma, cudaStream_t s);
SF_V5_DECL(0)
SF_V5_DECL(1)
SF_V5_DECL(2)
SF_V5_DECL(3)
SF_V5_DECL(4)
SF_V5_DECL(5)
SF_V5_DECL(6)
SF_V5_DECL(7)
#undef SF_V5_DECL

inline cudaError_t launch_v5(int R, bool om, int maxseg, bool cluster, const Params& p, const PairTable& t,
                             double gamma, cudaStream_t s) {
    if (R < 1 || R > kV5MaxR) return cudaErrorInvalidValue;
    if (R > 32) om = true;
    switch ((R - 1) / 8) {
        case 0: return launch_v5_part0(R, om, maxseg, cluster, p, t, gamma, s);
        case 1: return launch_v5_part1(R, om, maxseg, cluster, p, t, gamma, s);
        case 2: return launch_v5_part2(R, om, maxseg, cluster, p, t, gamma, s);
        case 3: return launch_v5_part3(R, om, maxseg, cluster, p, t, gamma, s);
        case 4: return launch_v5_part4(R, om, maxseg, cluster, p, t, gamma, s);
        case 5: return launch_v5_part5(R, om, maxseg, cluster, p, t, gamma, s);
        case 6: return launch_v5_part6(R, om, maxseg, cluster, p, t, gamma, s);
        default: return launch_v5_part7(R, om, maxseg, cluster, p, t, gamma, s);
    }
}

}  // namespace sf
