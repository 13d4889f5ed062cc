// Explicit instantiation: FB kernels for dtype float, K=5.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(float, 5)
}
