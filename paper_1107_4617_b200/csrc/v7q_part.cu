// v7q_part.cu — explicit instantiations of the v7q band-sweep kernel
// (box_v7q.cuh, separable q_M spatial kernel) for the radii
// 4*SF_V7Q_PART+1 .. 4*SF_V7Q_PART+4 and F = 1, 2 nonzero spatial frequencies
// per axis (see v7q_dispatch.h).  Compiled once per part with -DSF_V7Q_PART=i.
#include <utility>

#include "box_v7q.cuh"
#include "v7q_dispatch.h"

#ifndef SF_V7Q_PART
#error "compile with -DSF_V7Q_PART=0..5"
#endif

namespace sf {
namespace {

constexpr int kLo = 4 * SF_V7Q_PART + 1;

template <int... I>
cudaError_t pick(int R, int F, const Params& p, const PairTable& t, const QModTab& qt, double gamma, cudaStream_t s,
                 std::integer_sequence<int, I...>) {
    cudaError_t e = cudaErrorInvalidValue;
    (void)((R == kLo + I ? (e = F == 1 ? launch_box_v7q<kLo + I, 1>(p, t, qt, gamma, s)
                                       : launch_box_v7q<kLo + I, 2>(p, t, qt, gamma, s),
                            true)
                         : false) ||
           ...);
    return e;
}

}  // namespace

#define SF_V7Q_CAT2(a, b) a##b
#define SF_V7Q_CAT(a, b) SF_V7Q_CAT2(a, b)
cudaError_t SF_V7Q_CAT(launch_v7q_part, SF_V7Q_PART)(int R, int F, const Params& p, const PairTable& t,
                                                     const QModTab& qt, double gamma, cudaStream_t s) {
    return pick(R, F, p, t, qt, gamma, s, std::make_integer_sequence<int, 4>{});
}

}  // namespace sf
