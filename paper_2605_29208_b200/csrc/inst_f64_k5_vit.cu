// Explicit instantiation: VIT kernels for dtype double, K=5.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_VIT(double, 5)
}
