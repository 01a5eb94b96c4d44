// nlm_dispatch.h — the NLM band-sweep kernel (box_nlm5.cuh) for outer radii
// 2..8 and 10 and patch sizes 1..3, instantiated in nlm_part.cu (one TU per
// patch size).  launch_nlm_v5n returns cudaErrorInvalidValue for a radius
// without an instantiation (the caller then runs the tile kernel).
#pragma once

#include <cuda_runtime.h>

#include "box_kernel.cuh"
#include "nlm_kernel.cuh"

namespace sf {

cudaError_t launch_nlm_v5n_p1(int R, const Params& p, const NlmTable& t, cudaStream_t s);
cudaError_t launch_nlm_v5n_p2(int R, const Params& p, const NlmTable& t, cudaStream_t s);
cudaError_t launch_nlm_v5n_p3(int R, const Params& p, const NlmTable& t, cudaStream_t s);

inline bool nlm_v5n_has(int R) { return (R >= 2 && R <= 8) || R == 10; }

inline cudaError_t launch_nlm_v5n(int R, int P, const Params& p, const NlmTable& t, cudaStream_t s) {
    if (!nlm_v5n_has(R)) return cudaErrorInvalidValue;
    switch (P) {
        case 1: return launch_nlm_v5n_p1(R, p, t, s);
        case 2: return launch_nlm_v5n_p2(R, p, t, s);
        case 3: return launch_nlm_v5n_p3(R, p, t, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace sf
