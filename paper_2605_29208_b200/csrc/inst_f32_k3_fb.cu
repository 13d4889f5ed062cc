// Explicit instantiation: FB kernels for dtype float, K=3.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(float, 3)
}
