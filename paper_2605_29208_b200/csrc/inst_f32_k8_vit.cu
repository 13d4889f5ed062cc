// Explicit instantiation: VIT kernels for dtype float, K=8.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(float, 8)
}
