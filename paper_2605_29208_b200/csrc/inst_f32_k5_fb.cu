// Explicit instantiation: FB kernels for dtype float, K=5.
#define LHMM_ONLY_FB
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(float, 5)
}
