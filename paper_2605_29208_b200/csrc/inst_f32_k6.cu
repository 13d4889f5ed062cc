// Explicit instantiation of the K<=8 kernels for dtype float, K=6.
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_DECLARE_INST(float, 6)
}
