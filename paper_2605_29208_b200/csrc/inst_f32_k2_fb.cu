// Explicit instantiation: FB kernels for dtype float, K=2.
#define LHMM_ONLY_FB
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(float, 2)
}
