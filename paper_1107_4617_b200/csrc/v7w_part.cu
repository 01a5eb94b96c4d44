// v7w_part.cu — explicit instantiations of the wide large-radius v7 kernel
// (box_v7.cuh, WIDE = true) for the radii 9 + 7*SF_V7W_PART .. +6 (see
// v7w_dispatch.h).  Compiled once per part with -DSF_V7W_PART=0..7.
#include <utility>

#include "box_v7.cuh"
#include "v7w_dispatch.h"

#ifndef SF_V7W_PART
#error "compile with -DSF_V7W_PART=0..7"
#endif

namespace sf {
namespace {

constexpr int kLo = kV7WMinR + 7 * SF_V7W_PART;

template <int... I>
cudaError_t pick(int R, const Params& p, const PairTable& t, double gamma, cudaStream_t s,
                 std::integer_sequence<int, I...>) {
    cudaError_t e = cudaErrorInvalidValue;
    (void)((R == kLo + I ? (e = launch_box_v7w<kLo + I>(p, t, gamma, s), true) : false) || ...);
    return e;
}

}  // namespace

#define SF_V7W_CAT2(a, b) a##b
#define SF_V7W_CAT(a, b) SF_V7W_CAT2(a, b)
cudaError_t SF_V7W_CAT(launch_v7w_part, SF_V7W_PART)(int R, const Params& p, const PairTable& t, double gamma,
                                                     cudaStream_t s) {
    return pick(R, p, t, gamma, s, std::make_integer_sequence<int, 7>{});
}

}  // namespace sf
