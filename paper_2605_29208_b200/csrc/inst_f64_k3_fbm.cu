// Explicit instantiation: FBM kernels for dtype double, K=3.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBM(double, 3)
}
