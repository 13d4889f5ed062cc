// Explicit instantiation: FBM kernels for dtype float, K=1.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBM(float, 1)
}
