// Explicit instantiation: VIT kernels for dtype double, K=6.
#define LHMM_ONLY_VIT
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(double, 6)
}
