// Explicit instantiation: FBM kernels for dtype double, K=8.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBM(double, 8)
}
