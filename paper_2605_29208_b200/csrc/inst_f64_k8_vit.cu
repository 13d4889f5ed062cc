// Explicit instantiation: VIT kernels for dtype double, K=8.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(double, 8)
}
