// Explicit instantiation: VIT kernels for dtype float, K=1.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(float, 1)
}
