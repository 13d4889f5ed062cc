// Explicit instantiation: FB kernels for dtype double, K=6.
#define LHMM_ONLY_FB
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(double, 6)
}
