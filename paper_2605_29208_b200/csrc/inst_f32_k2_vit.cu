// Explicit instantiation: VIT kernels for dtype float, K=2.
#define LHMM_ONLY_VIT
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(float, 2)
}
