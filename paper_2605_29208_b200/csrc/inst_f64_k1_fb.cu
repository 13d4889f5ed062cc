// Explicit instantiation: FB kernels for dtype double, K=1.
#define LHMM_ONLY_FB
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(double, 1)
}
