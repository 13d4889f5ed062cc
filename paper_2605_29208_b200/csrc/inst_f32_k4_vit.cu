// Explicit instantiation: VIT kernels for dtype float, K=4.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(float, 4)
}
