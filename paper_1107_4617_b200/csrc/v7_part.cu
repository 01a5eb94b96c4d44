// v7_part.cu — explicit instantiations of the v7 band-sweep kernel
// (box_v7.cuh) for the radii 4*SF_V7_PART+1 .. 4*SF_V7_PART+4, both outgoing-row
// modes (see v7_dispatch.h).  Compiled once per part with -DSF_V7_PART=i.
#include <utility>

#include "box_v7.cuh"
#include "v7_dispatch.h"

#ifndef SF_V7_PART
#error "compile with -DSF_V7_PART=0..5"
#endif

namespace sf {
namespace {

constexpr int kLo = 4 * SF_V7_PART + 1;

template <int R>
cudaError_t one(bool om, int maxseg, const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    return om ? launch_box_v7<R, true>(p, t, gamma, maxseg, s) : launch_box_v7<R, false>(p, t, gamma, maxseg, s);
}

template <int... I>
cudaError_t pick(int R, bool om, int maxseg, const Params& p, const PairTable& t, double gamma, cudaStream_t s,
                 std::integer_sequence<int, I...>) {
    cudaError_t e = cudaErrorInvalidValue;
    (void)((R == kLo + I ? (e = one<kLo + I>(om, maxseg, p, t, gamma, s), true) : false) || ...);
    return e;
}

}  // namespace

#define SF_V7_CAT2(a, b) a##b
#define SF_V7_CAT(a, b) SF_V7_CAT2(a, b)
cudaError_t SF_V7_CAT(launch_v7_part, SF_V7_PART)(int R, bool om, int maxseg, const Params& p, const PairTable& t,
                                                   double gamma, cudaStream_t s) {
    return pick(R, om, maxseg, p, t, gamma, s, std::make_integer_sequence<int, 4>{});
}

}  // namespace sf
