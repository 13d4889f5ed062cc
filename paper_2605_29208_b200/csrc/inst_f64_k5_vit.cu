// Explicit instantiation: VIT kernels for dtype double, K=5.
#define LHMM_ONLY_VIT
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(double, 5)
}
