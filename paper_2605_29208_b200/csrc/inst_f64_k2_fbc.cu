// Explicit instantiation: chunked meet-in-the-middle FB kernels for dtype double, K=2.
#define LHMM_ONLY_FBC
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBC(double, 2)
}
