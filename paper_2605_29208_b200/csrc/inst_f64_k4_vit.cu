// Explicit instantiation: VIT kernels for dtype double, K=4.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(double, 4)
}
