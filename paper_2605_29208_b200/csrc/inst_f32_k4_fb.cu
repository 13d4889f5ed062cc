// Explicit instantiation: FB kernels for dtype float, K=4.
#define LHMM_ONLY_FB
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(float, 4)
}
