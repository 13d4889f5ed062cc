// Explicit instantiation of the K<=8 kernels for dtype double, K=8.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_DECLARE_INST(double, 8)
}
