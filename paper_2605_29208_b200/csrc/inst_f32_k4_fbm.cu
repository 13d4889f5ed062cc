// Explicit instantiation: FBM kernels for dtype float, K=4.
#define LHMM_ONLY_FBM
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBM(float, 4)
}
