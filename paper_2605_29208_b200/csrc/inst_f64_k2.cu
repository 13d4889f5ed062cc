// Explicit instantiation of the K<=8 kernels for dtype double, K=2.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_DECLARE_INST(double, 2)
}
