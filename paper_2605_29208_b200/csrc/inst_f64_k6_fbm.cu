// Explicit instantiation: FBM kernels for dtype double, K=6.
#define LHMM_ONLY_FBM
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBM(double, 6)
}
