// hmm_init.cu — moments of the quantile bins of default_initial_model
// (training.py:239-282) on the device.
//
// The reference pools every observation, sorts the pool, splits it into
// num_states nearly equal bins (np.array_split) and seeds each state from the
// moments of its bin (distributions.py:1114-1176 moment_seed).  Here the pool
// is sorted on the device and this kernel computes, for every bin in one CTA,
// the two-pass moments moment_seed reads (mean and variance about the mean,
// the same for log y, the sine / cosine sums, sum y^2, the range) plus the
// support counts its validations need and the first categorical counts, so
// only K small rows come back to the host.
#include <cstdint>

#include "../../include/loghmm_b200.h"

namespace {

constexpr int kBinSlots = LOGHMM_BIN_SLOTS;

__device__ double block_sum(double v, double* red) {
  const int t = threadIdx.x;
  red[t] = v;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (t < s) red[t] += red[t + s];
    __syncthreads();
  }
  const double r = red[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(256) bin_moments_kernel(const double* __restrict__ pooled, int64_t N,
                                                          int K, double* __restrict__ out) {
  __shared__ double red[256];
  const int k = blockIdx.x;
  // np.array_split: the first N % K bins hold N / K + 1 values
  const int64_t q = N / K, r = N % K;
  const int64_t lo = k * q + (k < r ? k : r);
  const int64_t hi = lo + q + (k < r ? 1 : 0);
  const double n = (double)(hi - lo);
  double s = 0.0, sl = 0.0, ss = 0.0, sc = 0.0, s2 = 0.0;
  double nonpos = 0.0, neg = 0.0, outunit = 0.0, nonint = 0.0;
  double c[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double y = pooled[i];
    s += y;
    s2 += y * y;
    ss += sin(y);
    sc += cos(y);
    if (y > 0.0) sl += log(y);
    else nonpos += 1.0;
    if (y < 0.0) neg += 1.0;
    if (!(y > 0.0 && y < 1.0)) outunit += 1.0;
    if (y < 0.0 || floor(y) != y) nonint += 1.0;
    else if (y < 8.0) c[(int)y] += 1.0;
  }
  s = block_sum(s, red);
  sl = block_sum(sl, red);
  const double mean = s / n, lmean = sl / n;
  double v = 0.0, lv = 0.0;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) {
    const double y = pooled[i];
    v += (y - mean) * (y - mean);
    if (y > 0.0) lv += (log(y) - lmean) * (log(y) - lmean);
  }
  v = block_sum(v, red);
  lv = block_sum(lv, red);
  ss = block_sum(ss, red);
  sc = block_sum(sc, red);
  s2 = block_sum(s2, red);
  nonpos = block_sum(nonpos, red);
  neg = block_sum(neg, red);
  outunit = block_sum(outunit, red);
  nonint = block_sum(nonint, red);
  for (int j = 0; j < 8; ++j) c[j] = block_sum(c[j], red);
  if (threadIdx.x == 0) {
    double* o = out + (size_t)k * kBinSlots;
    o[0] = n;
    o[1] = mean;
    o[2] = v / n;
    o[3] = lmean;
    o[4] = lv / n;
    o[5] = ss;
    o[6] = sc;
    o[7] = s2;
    o[8] = n > 0 ? pooled[lo] : 0.0;      // bin minimum (sorted)
    o[9] = n > 0 ? pooled[hi - 1] : 0.0;  // bin maximum
    o[10] = nonpos;
    o[11] = neg;
    o[12] = outunit;
    o[13] = nonint;
    for (int j = 0; j < 8; ++j) o[14 + j] = c[j];
  }
}

}  // namespace

extern "C" int32_t loghmm_bin_moments(const double* pooled_sorted, int64_t N, int32_t K, double* out,
                                      void* stream) {
  if (!pooled_sorted || !out || N < 1 || K < 1 || K > LOGHMM_MAX_STATES) return LOGHMM_EINVAL;
  bin_moments_kernel<<<K, 256, 0, (cudaStream_t)stream>>>(pooled_sorted, N, K, out);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}
