// v7q_dispatch.h — the v7q band-sweep kernel (box_v7q.cuh: Algorithm 2 with
// the separable spatial kernel w1(u) = cos(beta u)^M, M = 1..4) for every
// radius 1..24, instantiated in six translation units (v7q_part.cu compiled
// with SF_V7Q_PART = 0..5, radii 4i+1..4i+4).
//
// launch_v7q(R, F, ...): F = ceil(M/2) nonzero spatial frequencies per axis;
// qt = the per-axis modulation table (sf.cu: qmod_table).
#pragma once

#include <cuda_runtime.h>

#include "box_kernel.cuh"

namespace sf {

constexpr int kV7QMaxR = 24;
constexpr int kV7QMaxM = 4;

constexpr int kQFMax = 2;          // nonzero spatial frequencies per axis (M <= 4)
constexpr int kQRB = 16;           // rows per step
constexpr int kQMaxR = 24;
constexpr int kQMaxG = 16;

// per-axis modulation factors, computed on the host in fp64 (sf.cu: qmod_table).
// The running sums are kept pre-scaled by their weight (a_0 for the zero
// frequency, a_m for nu_m): the update factors carry the weight, the
// recombination factors at the window centre do not.
struct QModTab {
    float a0;                                  // weight of the zero frequency (0 for odd M)
    // vertical, origin = batch start yb, output row yb + i (i = 0..RB-1):
    float vic[kQFMax][kQRB], vis[kQFMax][kQRB];      // in row i+R:     a cos, a sin(nu (i+R))
    float voc[kQFMax][kQRB], vos[kQFMax][kQRB];      // out row i-R-1: -a cos, -a sin(nu (i-R-1))
    float vac[kQFMax][kQRB], vas[kQFMax][kQRB];      // centre i:       cos, sin(nu i)
    float rbc[kQFMax], rbs[kQFMax];                  // re-base by RB rows: cos, sin(nu RB)
    float ic[kQFMax][2 * kQMaxR + 1], is[kQFMax][2 * kQMaxR + 1];   // init row i: a cos, a sin(nu (i-R-1))
    // horizontal, origin = the lane's first slab column, output j (j = 0..G-1):
    float hoc[kQFMax][kQMaxG], hos[kQFMax][kQMaxG];  // out column j:   a cos, a sin(nu j)
    float hic[kQFMax][kQMaxG], his[kQFMax][kQMaxG];  // in column j+L:  a cos, a sin(nu (j+L))
    float hac[kQFMax][kQMaxG], has[kQFMax][kQMaxG];  // centre j+R:     cos, sin(nu (j+R))
    float rhc[kQFMax], rhs[kQFMax];                  // block shift by G: cos, sin(nu G)
};


#define SF_V7Q_DECL(i)                                                                                  \
    cudaError_t launch_v7q_part##i(int R, int F, const Params& p, const PairTable& t, const QModTab& qt, \
                                   double gamma, cudaStream_t s);
SF_V7Q_DECL(0)
SF_V7Q_DECL(1)
SF_V7Q_DECL(2)
SF_V7Q_DECL(3)
SF_V7Q_DECL(4)
SF_V7Q_DECL(5)
#undef SF_V7Q_DECL

inline cudaError_t launch_v7q(int R, int F, const Params& p, const PairTable& t, const QModTab& qt, double gamma,
                              cudaStream_t s) {
    if (R < 1 || R > kV7QMaxR || F < 1 || F > 2) return cudaErrorInvalidValue;
    switch ((R - 1) / 4) {
        case 0: return launch_v7q_part0(R, F, p, t, qt, gamma, s);
        case 1: return launch_v7q_part1(R, F, p, t, qt, gamma, s);
        case 2: return launch_v7q_part2(R, F, p, t, qt, gamma, s);
        case 3: return launch_v7q_part3(R, F, p, t, qt, gamma, s);
        case 4: return launch_v7q_part4(R, F, p, t, qt, gamma, s);
        default: return launch_v7q_part5(R, F, p, t, qt, gamma, s);
    }
}

}  // namespace sf
