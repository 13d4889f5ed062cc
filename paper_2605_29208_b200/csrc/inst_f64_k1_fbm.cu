// Explicit instantiation: FBM kernels for dtype double, K=1.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBM(double, 1)
}
