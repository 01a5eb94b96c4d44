// v6_part.cu — explicit instantiations of the v6 band-sweep kernel
// (box_v6.cuh) for the radii 4*SF_V6_PART+1 .. 4*SF_V6_PART+4, both outgoing-row
// modes (see v6_dispatch.h).  Compiled once per part with -DSF_V6_PART=i.
#include <cstdlib>
#include <utility>

#include "box_v6.cuh"
#include "v6_dispatch.h"

#ifndef SF_V6_PART
#error "compile with -DSF_V6_PART=0..7"
#endif

namespace sf {
namespace {

constexpr int kLo = 4 * SF_V6_PART + 1;

template <int R>
cudaError_t one(bool om, int maxseg, const Params& p, const PairTable& t, double gamma, cudaStream_t s) {
#if SF_V6_PART == 3
    // A/B of the walker width at R = 16 (tools: SF_V6_G = 16 | 24)
    if constexpr (R == 16) {
        static const int g = [] { const char* e = std::getenv("SF_V6_G"); return e ? std::atoi(e) : 0; }();
        if (g == 16) return om ? launch_box_v6<R, true, 16>(p, t, gamma, maxseg, s)
                               : launch_box_v6<R, false, 16>(p, t, gamma, maxseg, s);
        if (g == 24) return om ? launch_box_v6<R, true, 24>(p, t, gamma, maxseg, s)
                               : launch_box_v6<R, false, 24>(p, t, gamma, maxseg, s);
    }
#endif
    return om ? launch_box_v6<R, true>(p, t, gamma, maxseg, s) : launch_box_v6<R, false>(p, t, gamma, maxseg, s);
}

template <int... I>
cudaError_t pick(int R, bool om, int maxseg, const Params& p, const PairTable& t, double gamma, cudaStream_t s,
                 std::integer_sequence<int, I...>) {
    cudaError_t e = cudaErrorInvalidValue;
    (void)((R == kLo + I ? (e = one<kLo + I>(om, maxseg, p, t, gamma, s), true) : false) || ...);
    return e;
}

}  // namespace

#define SF_V6_CAT2(a, b) a##b
#define SF_V6_CAT(a, b) SF_V6_CAT2(a, b)
cudaError_t SF_V6_CAT(launch_v6_part, SF_V6_PART)(int R, bool om, int maxseg, const Params& p, const PairTable& t,
                                                   double gamma, cudaStream_t s) {
    return pick(R, om, maxseg, p, t, gamma, s, std::make_integer_sequence<int, 4>{});
}

}  // namespace sf
