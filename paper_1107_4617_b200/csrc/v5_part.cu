// v5_part.cu — explicit instantiations of the v5 band-sweep kernel for the
// radii 8*SF_V5_PART+1 .. 8*SF_V5_PART+8 (see v5_dispatch.h).  Compiled once
// per part with -DSF_V5_PART=i.
#include <utility>

#include "box_v5.cuh"
#include "v5_dispatch.h"

#ifndef SF_V5_PART
#error "compile with -DSF_V5_PART=0..7"
#endif

namespace sf {
namespace {

constexpr int kLo = 8 * SF_V5_PART + 1;

template <int R>
cudaError_t one(bool om, int maxseg, bool cluster, const Params& p, const PairTable& t, double gamma,
                cudaStream_t s) {
    if constexpr (R > 32) {
        (void)cluster;
        return launch_box_v5<R, true>(p, t, gamma, maxseg, s);
    } else if constexpr (V5Cfg<R>::SMR) {
        return launch_box_v5<R, true>(p, t, gamma, maxseg, s);
    } else {
        return om ? launch_box_v5<R, true>(p, t, gamma, maxseg, s) : launch_box_v5<R, false>(p, t, gamma, maxseg, s);
    }
}

template <int... I>
cudaError_t pick(int R, bool om, int maxseg, bool cluster, const Params& p, const PairTable& t, double gamma,
                 cudaStream_t s, std::integer_sequence<int, I...>) {
    cudaError_t e = cudaErrorInvalidValue;
    (void)((R == kLo + I ? (e = one<kLo + I>(om, maxseg, cluster, p, t, gamma, s), true) : false) || ...);
    return e;
}

}  // namespace

#define SF_V5_CAT2(a, b) a##b
#define SF_V5_CAT(a, b) SF_V5_CAT2(a, b)
cudaError_t SF_V5_CAT(launch_v5_part, SF_V5_PART)(int R, bool om, int maxseg, bool cluster, const Params& p,
                                                   const PairTable& t, double gamma, cudaStream_t s) {
    return pick(R, om, maxseg, cluster, p, t, gamma, s, std::make_integer_sequence<int, 8>{});
}

}  // namespace sf
