// v8_part.cu — explicit instantiations of the v8 band-sweep kernel
// (box_v8.cuh) for the radii 4*SF_V8_PART+1 .. 4*SF_V8_PART+4, both outgoing-row
// modes (see v8_dispatch.h).  Compiled once per part with -DSF_V8_PART=i.
#include <cstdlib>
#include <utility>

#include "box_v8.cuh"
#include "v8_dispatch.h"

#ifndef SF_V8_PART
#error "compile with -DSF_V8_PART=0..5"
#endif

namespace sf {
namespace {

constexpr int kLo = 4 * SF_V8_PART + 1;

template <int R>
cudaError_t one(bool om, int maxseg, const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
    return om ? launch_box_v8<R, true>(p, t, gamma, maxseg, s) : launch_box_v8<R, false>(p, t, gamma, maxseg, s);
}

template <int... I>
cudaError_t pick(int R, bool om, int maxseg, const Params& p, const PairTable& t, double gamma, cudaStream_t s,
                 std::integer_sequence<int, I...>) {
    cudaError_t e = cudaErrorInvalidValue;
    (void)((R == kLo + I ? (e = one<kLo + I>(om, maxseg, p, t, gamma, s), true) : false) || ...);
    return e;
}

}  // namespace

#define SF_V8_CAT2(a, b) a##b
#define SF_V8_CAT(a, b) SF_V8_CAT2(a, b)
cudaError_t SF_V8_CAT(launch_v8_part, SF_V8_PART)(int R, bool om, int maxseg, const Params& p, const PairTable& t,
                                                   double gamma, cudaStream_t s) {
    return pick(R, om, maxseg, p, t, gamma, s, std::make_integer_sequence<int, 4>{});
}

}  // namespace sf
