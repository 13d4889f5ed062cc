// Explicit instantiation: FB kernels for dtype double, K=8.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FB(double, 8)
}
