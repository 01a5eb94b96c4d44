// nlm_part.cu — instantiations of the NLM band-sweep kernel (box_nlm5.cuh)
// for patch size P = SF_NLM_P (compiled once per P) and the outer radii
// kNlmRadii; other radii run the NLM tile kernel (nlm_kernel.cuh).
#include <utility>

#include "box_nlm5.cuh"
#include "nlm_dispatch.h"

#ifndef SF_NLM_P
#error "compile with -DSF_NLM_P=1..3"
#endif

namespace sf {
namespace {

template <int... Rs>
cudaError_t pick(int R, const Params& p, const NlmTable& t, cudaStream_t s, std::integer_sequence<int, Rs...>) {
    cudaError_t e = cudaErrorInvalidValue;
    (void)((R == Rs ? (e = launch_nlm_v5n<Rs, SF_NLM_P>(p, t, s), true) : false) || ...);
    return e;
}

}  // namespace

#define SF_NLM_CAT2(a, b) a##b
#define SF_NLM_CAT(a, b) SF_NLM_CAT2(a, b)
cudaError_t SF_NLM_CAT(launch_nlm_v5n_p, SF_NLM_P)(int R, const Params& p, const NlmTable& t, cudaStream_t s) {
    return pick(R, p, t, s, std::integer_sequence<int, 2, 3, 4, 5, 6, 7, 8, 10>{});
}

}  // namespace sf
