// Explicit instantiation: chunked meet-in-the-middle FB kernels for dtype float, K=1.
#define LHMM_ONLY_FBC
#include "hmm_launch.cuh"
namespace lhmm {
LHMM_INST_FBC(float, 1)
}
