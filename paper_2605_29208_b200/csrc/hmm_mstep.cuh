// hmm_mstep.cuh — deterministic statistics reduction and the per-state
// scalar M-step kernels (one thread per state).
//
// Device ports of the reference's scalar math:
//   special.py:81-128  digamma / trigamma (recurrence to x>=10 + asymptotic series)
//   special.py:135-217 two-branch A&S Bessel I0/I1, log I0, I1/I0 ratio
//   distributions.py:732-761 _newton_1d (safeguarded bracketed Newton)
//   distributions.py:632-636 fit_gaussian, :658-663 fit_poisson,
//                    :764-786 fit_gamma_nr, :874-916 fit_vonmises,
//                    :1031-1076 fit_student_t_ecme (E-step sums, CM-1, nu Newton)
//   training.py:105-127 m_step_transitions, :130-148 collapse guard
// The ECME likelihood guard (distributions.py:1080-1086) needs a data pass
// and lives in student_guard_kernel below.
#pragma once

#include "hmm_common.cuh"

namespace lhmm {

// ---- special functions (special.py) -----------------------------------------
__device__ inline double sp_digamma(double x) {
  double acc = 0.0;
  while (x < 10.0) {
    acc -= 1.0 / x;
    x += 1.0;
  }
  const double inv = 1.0 / x, inv2 = inv * inv;
  const double series =
      log(x) - 0.5 * inv -
      inv2 * (1.0 / 12.0 -
              inv2 * (1.0 / 120.0 - inv2 * (1.0 / 252.0 - inv2 * (1.0 / 240.0 - inv2 / 132.0))));
  return acc + series;
}

__device__ inline double sp_trigamma(double x) {
  double acc = 0.0;
  while (x < 10.0) {
    acc += 1.0 / (x * x);
    x += 1.0;
  }
  const double inv = 1.0 / x, inv2 = inv * inv;
  const double series =
      inv * (1.0 + inv * (0.5 + inv * (1.0 / 6.0 -
                                       inv2 * (1.0 / 30.0 -
                                               inv2 * (1.0 / 42.0 -
                                                       inv2 * (1.0 / 30.0 - 5.0 * inv2 / 66.0))))));
  return acc + series;
}

__constant__ double kI0S[7] = {1.0, 3.5156229, 3.0899424, 1.2067492, 0.2659732, 0.0360768, 0.0045813};
__constant__ double kI0L[9] = {0.39894228, 0.01328592, 0.00225319, -0.00157565, 0.00916281,
                               -0.02057706, 0.02635537, -0.01647633, 0.00392377};
__constant__ double kI1S[7] = {0.5, 0.87890594, 0.51498869, 0.15084934, 0.02658733, 0.00301532, 0.00032411};
__constant__ double kI1L[9] = {0.39894228, -0.03988024, -0.00362018, 0.00163801, -0.01031555,
                               0.02282967, -0.02895312, 0.01787654, -0.00420059};

__device__ inline double sp_poly(const double* c, int n, double u) {
  double acc = 0.0;
  for (int i = n - 1; i >= 0; --i) acc = acc * u + c[i];
  return acc;
}
__device__ inline double sp_bessel_i0(double x) {
  if (x <= 3.75) {
    const double t = x / 3.75;
    return sp_poly(kI0S, 7, t * t);
  }
  return exp(x) / sqrt(x) * sp_poly(kI0L, 9, 3.75 / x);
}
__device__ inline double sp_bessel_i1(double x) {
  if (x <= 3.75) {
    const double t = x / 3.75;
    return x * sp_poly(kI1S, 7, t * t);
  }
  return exp(x) / sqrt(x) * sp_poly(kI1L, 9, 3.75 / x);
}
__device__ inline double sp_log_bessel_i0(double x) {
  if (x <= 3.75) {
    const double t = x / 3.75;
    return log(sp_poly(kI0S, 7, t * t));
  }
  return x - 0.5 * log(x) + log(sp_poly(kI0L, 9, 3.75 / x));
}
__device__ inline double sp_i1_i0_ratio(double k) {
  if (k == 0.0) return 0.0;
  if (k <= 3.75) return sp_bessel_i1(k) / sp_bessel_i0(k);
  const double u = 3.75 / k;
  return sp_poly(kI1L, 9, u) / sp_poly(kI0L, 9, u);
}

constexpr double kLog2Pi = 1.8378770664093453;  // math.log(2*pi)
constexpr double kScaleFloor = 1e-9;             // distributions.py:73
constexpr double kKappaCeiling = 1e5;            // distributions.py:74
constexpr double kNegbinomCeiling = 1e6;         // distributions.py:76

// Host-equivalent constants of a record (see loghmm_emission_t).
__device__ inline void em_constants(loghmm_emission_t& e) {
  switch (e.family) {
    case LOGHMM_FAM_GAUSSIAN:
      e.c[0] = (-0.5 * kLog2Pi) - log(e.p[1]);
      break;
    case LOGHMM_FAM_STUDENT_T: {
      const double nu = e.p[2];
      e.c[0] = lgamma((nu + 1.0) / 2.0) - lgamma(nu / 2.0) - 0.5 * log(nu * CUDART_PI) - log(e.p[1]);
      e.c[1] = (nu + 1.0) / 2.0;
      break;
    }
    case LOGHMM_FAM_GAMMA:
      e.c[0] = e.p[0] * log(e.p[1]) - lgamma(e.p[0]);
      e.c[1] = e.p[0] - 1.0;
      break;
    case LOGHMM_FAM_VON_MISES:
      e.c[0] = kLog2Pi;
      e.c[1] = sp_log_bessel_i0(e.p[1]);
      break;
    case LOGHMM_FAM_POISSON:
      e.c[0] = log(e.p[0]);
      break;
    default:
      break;
  }
}

// _newton_1d (distributions.py:732-761) for the Gamma shape score.
__device__ inline double gamma_newton(double c, double x0, bool& ok) {
  double lo = 0.0, hi = CUDART_INF, x = x0;
  for (int it = 0; it < 50; ++it) {
    const double s = log(x) - sp_digamma(x) - c;
    if (fabs(s) <= 1e-10) {
      ok = true;
      return x;
    }
    if (s > 0.0) lo = fmax(lo, x);
    else hi = fmin(hi, x);
    const double d = 1.0 / x - sp_trigamma(x);
    double prop = d != 0.0 ? x - s / d : CUDART_INF;
    if (!(isfinite(prop) && lo < prop && prop < hi)) prop = isinf(hi) ? x * 8.0 : 0.5 * (lo + hi);
    x = prop;
  }
  ok = fabs(log(x) - sp_digamma(x) - c) <= 1e-10;
  return x;
}

// fit_gamma_nr (distributions.py:764-786) from exact moments; returns status.
__device__ inline int32_t gamma_fit(double n, double mean, double var, double sumlog,
                                    loghmm_emission_t& e) {
  if (var <= 0.0) return LOGHMM_MS_ERR_GAMMA_VAR;
  const double c = log(mean) - sumlog / n;
  if (c <= 0.0) return LOGHMM_MS_ERR_GAMMA_GAP;
  const double seed = mean * mean / var;
  bool ok = false;
  double alpha = gamma_newton(c, seed, ok);
  int32_t st = LOGHMM_MS_UPDATED;
  if (!ok) {
    st |= LOGHMM_MS_WARN_NEWTON;
    alpha = seed;
  }
  e.p[0] = alpha;
  e.p[1] = alpha / mean;
  return st;
}

// Student-t nu objective / score / curvature (distributions.py:995-1009).
__device__ inline double st_obj(double nu, double n, double mix) {
  return n * (nu / 2.0 * log(nu / 2.0) - lgamma(nu / 2.0)) + nu / 2.0 * mix;
}
__device__ inline double st_score(double nu, double n, double mix) {
  return n / 2.0 * (log(nu / 2.0) + 1.0 - sp_digamma(nu / 2.0)) + mix / 2.0;
}
__device__ inline double st_curv(double nu, double n) {
  return n / 4.0 * (2.0 / nu - sp_trigamma(nu / 2.0));
}

// Deterministic reduction: totals[c] = sum_b partials[b, c] in a fixed tree,
// totals[width] = sum_b ll[b].  One CTA per column block.
__global__ void __launch_bounds__(256) reduce_stats_kernel(const double* __restrict__ partials,
                                                           const double* __restrict__ ll,
                                                           int64_t B, int64_t width,
                                                           double* __restrict__ totals) {
  __shared__ double red[256];
  const int64_t col = blockIdx.x;  // 0..width (width = ll column)
  double acc = 0.0;
  for (int64_t b = threadIdx.x; b < B; b += blockDim.x)
    acc += (col < width) ? partials[b * width + col] : ll[b];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) totals[col] = red[0];
}

// guard_state layout per (stream, state): [mu, sigma, nu0, nu_cand, n, active, k_next, pad]
// guard_state per (stream, state), 16 doubles:
//  [0..7]  Student-t guard: mu, sigma, nu0, nu_cand, n, active, k_next, -
//  [8]     variance pass requested (1.0) / not (0.0)
//  [9]     centre of the second pass (the new mean / location)
//  [10..12] Student-t old parameters (mu0, sigma0, nu0) for the weights u
//  [13]    n (total weight),  [14] sum w log y (gamma),  [15] old shape (gamma)
constexpr int kGuardStride = 16;

// Called by every thread of the block (it synchronises); `scratch` holds
// K*K + K + 1 doubles of shared memory.
__device__ void mstep_body(const loghmm_model_t* __restrict__ min_, const double* __restrict__ tot,
                           int64_t nseq, double eps, double nu_ceiling, double nu_tol,
                           int max_newton, loghmm_model_t* __restrict__ mout,
                           int32_t* __restrict__ status, double* __restrict__ guard,
                           double var_ratio, int tid, int nthreads, double* __restrict__ scratch) {
  const int K = min_->K;
  const int S = min_->n_streams;
  const int width_xi = K * K;
  const double* xi = tot;
  const double* gt = tot + width_xi;
  const double* g0 = gt + K;
  const double* em = g0 + K;
  if (tid == 0) {
    mout->K = K;
    mout->n_streams = S;
  }
  // ---- transitions and initial distribution (training.py:105-127) ----
  // Spread over (i, j): the per-entry divisions and logs run in parallel; the
  // row totals and the pi normaliser are summed in the reference's order.
  double* vb = scratch;             // [K*K] xi[i, j] / gamma_tot[i]
  double* rowt = scratch + K * K;   // [K] row totals
  double* pis = rowt + K;           // [1] sum_j g0[j] / nseq
  for (int e = tid; e < K * K; e += nthreads) {
    const double g = gt[e / K];
    vb[e] = g >= eps ? xi[e] / g : 0.0;
  }
  __syncthreads();
  for (int i = tid; i < K; i += nthreads) {
    double total = 0.0;
    if (gt[i] >= eps)
      for (int j = 0; j < K; ++j) total += vb[i * K + j];
    rowt[i] = total;
  }
  if (tid == nthreads - 1) {
    double p = 0.0;
    for (int j = 0; j < K; ++j) p += g0[j] / (double)nseq;
    pis[0] = p;
  }
  __syncthreads();
  for (int e = tid; e < K * K; e += nthreads) {
    const int i = e / K;
    const double total = rowt[i];
    const bool upd = gt[i] >= eps && total > 0.0;
    const double v = upd ? vb[e] / total : min_->A[e];
    mout->A[e] = v;
    mout->log_A[e] = v > 0.0 ? log(v) : -CUDART_INF;
  }
  for (int j = tid; j < K; j += nthreads) {
    const double p = (g0[j] / (double)nseq) / pis[0];
    mout->pi[j] = p;
    mout->log_pi[j] = p > 0.0 ? log(p) : -CUDART_INF;
  }
  // ---- emissions (training.py:130-148 -> distributions.py:1094 refit) ----
  for (int idx = tid; idx < S * K; idx += nthreads) {
    const int s = idx / K, j = idx % K;
    loghmm_emission_t e = min_->em[s][j];
    const double* q = em + (size_t)(s * K + j) * LOGHMM_NSLOT;
    const double n_state = em[(size_t)(0 * K + j) * LOGHMM_NSLOT + 0];  // total weight of state j
    int32_t st = LOGHMM_MS_UPDATED;
    double* gs = guard + (size_t)(s * K + j) * kGuardStride;
    gs[5] = 0.0;
    gs[8] = 0.0;
    if (e.family == LOGHMM_FAM_NONE) {
      // nothing
    } else if (n_state < eps) {
      st = LOGHMM_MS_COLLAPSED;
    } else {
      const double n = q[0];
      switch (e.family) {
        case LOGHMM_FAM_GAUSSIAN: {
          const double d = q[1] / n;
          double var = (q[2] - q[1] * d) / n;
          if (var < 0.0) var = 0.0;
          e.p[0] = e.p[0] + d;
          e.p[1] = fmax(sqrt(var), kScaleFloor);
          // one-pass shifted sums lose ~(d^2/var) relative precision: ask for
          // the exact two-pass sum (distributions.py:616-620) when large
          if (!(var > 0.0) || d * d > var_ratio * var) {
            gs[8] = 1.0;
            gs[9] = e.p[0];
            gs[13] = n;
          }
          break;
        }
        case LOGHMM_FAM_POISSON: {
          if (q[2] > 0.0) {
            st = LOGHMM_MS_ERR_SUPPORT;
            break;
          }
          e.p[0] = fmax(q[1] / n, kScaleFloor);
          break;
        }
        case LOGHMM_FAM_GAMMA: {
          if (q[4] > 0.0) {
            st = LOGHMM_MS_ERR_SUPPORT;
            break;
          }
          const double m_old = e.p[0] / e.p[1];
          const double d = q[1] / n;
          const double mean = m_old + d;
          const double var = (q[2] - q[1] * d) / n;
          if (var <= 0.0 && !(d * d > 0.0)) {
            st = LOGHMM_MS_ERR_GAMMA_VAR;
            break;
          }
          if (d * d > var_ratio * var) {
            // defer the whole fit to the exact second pass
            gs[8] = 1.0;
            gs[9] = mean;
            gs[13] = n;
            gs[14] = q[3];
            break;
          }
          const double c = log(mean) - q[3] / n;
          if (c <= 0.0) {
            st = LOGHMM_MS_ERR_GAMMA_GAP;
            break;
          }
          const double seed = mean * mean / var;
          bool ok = false;
          double alpha = gamma_newton(c, seed, ok);
          if (!ok) {
            st |= LOGHMM_MS_WARN_NEWTON;
            alpha = seed;
          }
          e.p[0] = alpha;
          e.p[1] = alpha / mean;
          break;
        }
        case LOGHMM_FAM_VON_MISES: {
          if (q[3] > 0.0) {
            st = LOGHMM_MS_ERR_NONFINITE;
            break;
          }
          const double S_ = q[1], C_ = q[2];
          double mu = atan2(S_, C_);
          if (mu <= -CUDART_PI) mu = CUDART_PI;
          const double rbar = hypot(S_, C_) / n;
          double kappa;
          if (rbar <= 1e-12) {
            kappa = 0.0;
          } else if (rbar >= 1.0 - 1e-12) {
            st |= LOGHMM_MS_WARN_BOUNDARY;
            kappa = kKappaCeiling;
          } else {
            kappa = rbar * (2.0 - rbar * rbar) / (1.0 - rbar * rbar);
            bool conv = false;
            for (int it = 0; it < 50; ++it) {
              const double A_ = sp_i1_i0_ratio(kappa);
              const double f = A_ - rbar;
              if (fabs(f) <= 1e-10) {
                conv = true;
                break;
              }
              double step = f / (1.0 - A_ * A_ - A_ / kappa);
              double prop = kappa - step;
              while (prop <= 0.0) {
                step *= 0.5;
                prop = kappa - step;
              }
              kappa = prop;
              if (kappa >= kKappaCeiling) {
                kappa = kKappaCeiling;
                st |= LOGHMM_MS_WARN_CEILING;
                break;
              }
            }
            if (!conv && kappa < kKappaCeiling)
              if (fabs(sp_i1_i0_ratio(kappa) - rbar) > 1e-10) st |= LOGHMM_MS_WARN_NEWTON;
          }
          e.p[0] = mu;
          e.p[1] = kappa;
          break;
        }
        case LOGHMM_FAM_STUDENT_T: {
          const double mu0 = e.p[0], nu0 = e.p[2];
          const double swu = q[1];
          const double dmu = q[2] / swu;
          const double mu = mu0 + dmu;
          double s2 = (q[3] - q[2] * dmu) / n;
          if (s2 < 0.0) s2 = 0.0;
          const double sigma = fmax(sqrt(s2), kScaleFloor);
          if (!(s2 > 0.0) || dmu * dmu * swu > var_ratio * s2 * n) {
            gs[8] = 1.0;
            gs[9] = mu;
            gs[10] = mu0;
            gs[11] = e.p[1];
            gs[12] = nu0;
            gs[13] = n;
          }
          const double half = (nu0 + 1.0) / 2.0;
          const double mix = q[4] + n * (sp_digamma(half) - log(half));
          double nu = nu0;
          for (int it = 0; it < max_newton; ++it) {
            const double sc = st_score(nu, n, mix);
            const double h = st_curv(nu, n);
            double step = -sc / h;
            double prop = nu + step;
            while (prop <= 0.0) {
              step *= 0.5;
              prop = nu + step;
            }
            const double qn = st_obj(nu, n, mix);
            while (st_obj(prop, n, mix) < qn && fabs(step) > 1e-300) {
              step *= 0.5;
              prop = nu + step;
            }
            if (prop >= nu_ceiling) {
              st |= LOGHMM_MS_WARN_CEILING;
              nu = nu_ceiling;
              break;
            }
            const double moved = fabs(prop - nu);
            nu = prop;
            if (moved < nu_tol) break;
          }
          e.p[0] = mu;
          e.p[1] = sigma;
          // nu stays nu0 until the guard pass picks the candidate
          gs[0] = mu;
          gs[1] = sigma;
          gs[2] = nu0;
          gs[3] = nu;
          gs[4] = n;
          gs[5] = 1.0;
          gs[6] = 0.0;  // candidates consumed
          st |= LOGHMM_MS_STUDENT_GUARD;
          break;
        }
        default:
          // families 6..15: fitted by the weighted-sample passes
          // (hmm_extfit.cuh, loghmm_ext_fit_pass) after this kernel
          if (e.family >= LOGHMM_FAM_LOGNORMAL) {
            st |= LOGHMM_MS_EXT_FIT;
            gs[0] = 0.0;
          }
          break;
      }
    }
    if (st < 16) em_constants(e);
    mout->em[s][j] = e;
    status[idx] = st;
  }
}


// Stand-alone M-step: totals staged in shared memory first (one parallel
// round trip), then mstep_body.
__global__ void __launch_bounds__(256) mstep_kernel(const loghmm_model_t* __restrict__ min_,
                                                    const double* __restrict__ tot, int64_t width1,
                                                    int64_t nseq, double eps, double nu_ceiling,
                                                    double nu_tol, int max_newton,
                                                    loghmm_model_t* __restrict__ mout,
                                                    int32_t* __restrict__ status,
                                                    double* __restrict__ guard, double var_ratio) {
  extern __shared__ double tot_s[];
  (void)width1;
  const int Km = min_->K;
  const int64_t w1 = (int64_t)Km * Km + 2 * Km + 2 * Km * LOGHMM_NSLOT + 1;
  for (int64_t c = threadIdx.x; c < w1; c += blockDim.x) tot_s[c] = tot[c];
  __syncthreads();
  mstep_body(min_, tot_s, nseq, eps, nu_ceiling, nu_tol, max_newton, mout, status, guard, var_ratio,
             threadIdx.x, blockDim.x, tot_s + w1);
}

// Fused statistics reduction + M-step (single rank).  Block r sums rows
// [r*rpb, (r+1)*rpb) of the per-sequence partials column-wise (coalesced
// rows, fixed order) into part[r]; the last block to finish sums the block
// partials in block order into totals (also kept in shared memory) and runs
// the M-step.  `counter` must be zero before the first launch; the last block
// resets it.
__global__ void __launch_bounds__(1024) reduce_mstep_kernel(
    const double* __restrict__ partials, const double* __restrict__ ll, int64_t B, int64_t width,
    double* __restrict__ part, unsigned* __restrict__ counter, double* __restrict__ totals,
    const loghmm_model_t* __restrict__ min_, int64_t nseq, double eps, double nu_ceiling,
    double nu_tol, int max_newton, loghmm_model_t* __restrict__ mout, int32_t* __restrict__ status,
    double* __restrict__ guard, double var_ratio, int do_mstep) {
  extern __shared__ double tot_s[];  // [W1] totals, then [G][CP] group sums (G*CP <= blockDim)
  __shared__ bool last;
  const int W1 = (int)width + 1;
  // columns are summed CP at a time by thread (g, cc): column c0 + cc of
  // every G-th row, so each row is read by CP consecutive threads (coalesced)
  // and every thread has many independent loads in flight; the G group sums
  // are then added in group order (fixed, bit-reproducible).
  const int CP = min(W1, (int)blockDim.x);
  const int G = (int)blockDim.x / CP;
  const int g = (int)threadIdx.x / CP, cc = (int)threadIdx.x % CP;
  double* grp = tot_s + W1;
  auto col_sum = [&](const double* __restrict__ base, int64_t stride, int64_t r0, int64_t r1,
                     int c, bool is_ll) -> double {
    double acc = 0.0;
#pragma unroll 1
    for (int64_t r = r0 + g; r < r1; r += 8 * G) {
      double v[8];  // eight independent (predicated) loads in flight
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int64_t rr = r + (int64_t)k * G;
        v[k] = rr < r1 ? (is_ll ? __ldcg(ll + rr) : __ldcg(base + rr * stride + c)) : 0.0;
      }
#pragma unroll
      for (int k = 0; k < 8; ++k) acc += v[k];
    }
    return acc;
  };
  // out[c] = sum over rows [r0, r1) of src[., c] (src = partials + ll column, or part)
  auto reduce_rows = [&](bool from_partials, int64_t r0, int64_t r1, double* out, bool keep) {
    for (int c0 = 0; c0 < W1; c0 += CP) {
      const int c = c0 + cc;
      double acc = 0.0;
      if (g < G && c < W1)
        acc = from_partials ? col_sum(partials, width, r0, r1, c, c == W1 - 1)
                            : col_sum(part, W1, r0, r1, c, false);
      if (g < G) grp[g * CP + cc] = acc;
      __syncthreads();
      if ((int)threadIdx.x < CP && c0 + (int)threadIdx.x < W1) {
        double s2 = 0.0;
        for (int k = 0; k < G; ++k) s2 += grp[k * CP + threadIdx.x];
        out[c0 + threadIdx.x] = s2;
        if (keep) tot_s[c0 + threadIdx.x] = s2;
      }
      __syncthreads();
    }
  };
  const int64_t rpb = (B + gridDim.x - 1) / gridDim.x;
  const int64_t r0 = (int64_t)blockIdx.x * rpb, r1 = min(B, r0 + rpb);
  reduce_rows(true, r0, r1, part + (int64_t)blockIdx.x * W1, false);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  reduce_rows(false, 0, gridDim.x, totals, true);
  if (threadIdx.x == 0) *counter = 0u;
  __syncthreads();
  if (do_mstep)
    mstep_body(min_, tot_s, nseq, eps, nu_ceiling, nu_tol, max_newton, mout, status, guard,
               var_ratio, threadIdx.x, blockDim.x, tot_s + W1 + blockDim.x);
}

// Guard pass: for every active Student-t state j (stream `sidx`), partial sums
// over observations of w * log1p(z^2 / nu_k) for nu_k in the candidate list
// (k = 0 is the base nu0), z = (y - mu)/sigma at the new location/scale.
// Candidate list: c_1 = nu_cand, c_{k+1} = nu0 + 0.5 (c_k - nu0)
// (distributions.py:1081-1085).  Per-block partials, reduced by
// guard_select_kernel in a fixed order.
template <typename R>
__global__ void __launch_bounds__(256) student_guard_kernel(const R* __restrict__ y,
                                                            const R* __restrict__ gamma,
                                                            int64_t N, int K, int sidx,
                                                            const double* __restrict__ guard,
                                                            int ncand, double* __restrict__ part) {
  __shared__ double red[256];
  for (int j = 0; j < K; ++j) {
    const double* gs = guard + (size_t)(sidx * K + j) * kGuardStride;
    if (gs[5] == 0.0) continue;
    const double mu = gs[0], sigma = gs[1], nu0 = gs[2];
    double cand[LOGHMM_GUARD_CANDIDATES];
    cand[0] = nu0;
    double c = gs[3];
    const int k0 = (int)gs[6];
    for (int k = 0; k < k0; ++k) c = nu0 + 0.5 * (c - nu0);
    for (int k = 1; k < ncand; ++k) {
      cand[k] = c;
      c = nu0 + 0.5 * (c - nu0);
    }
    double acc[LOGHMM_GUARD_CANDIDATES];
    for (int k = 0; k < ncand; ++k) acc[k] = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
      const double w = (double)gamma[i * K + j];
      if (w > 0.0) {
        const double z = ((double)y[i] - mu) / sigma;
        const double z2 = z * z;
        for (int k = 0; k < ncand; ++k) acc[k] += w * log1p(z2 / cand[k]);
      }
    }
    for (int k = 0; k < ncand; ++k) {
      red[threadIdx.x] = acc[k];
      __syncthreads();
      for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
        __syncthreads();
      }
      if (threadIdx.x == 0)
        part[((size_t)blockIdx.x * K + j) * LOGHMM_GUARD_CANDIDATES + k] = red[0];
      __syncthreads();
    }
  }
}

__device__ inline double st_ll(double n, double sum_l1p, double sigma, double nu) {
  // sum_w [lg((nu+1)/2) - lg(nu/2) - 0.5 log(nu pi) - log sigma - (nu+1)/2 log1p(.)]
  const double c = lgamma((nu + 1.0) / 2.0) - lgamma(nu / 2.0) - 0.5 * log(nu * CUDART_PI) - log(sigma);
  return n * c - (nu + 1.0) / 2.0 * sum_l1p;
}

// Sum of the per-block partials of (state j, candidate k) in block order (the
// fixed order that makes the guard's decision reproducible): the loads of 16
// blocks are issued together, the additions stay sequential.
__device__ inline double guard_partial_sum(const double* __restrict__ part, int nblocks, int K, int j,
                                           int k) {
  double s = 0.0;
  const double* p = part + (size_t)j * LOGHMM_GUARD_CANDIDATES + k;
  const size_t stride = (size_t)K * LOGHMM_GUARD_CANDIDATES;
  int blk = 0;
  for (; blk + 16 <= nblocks; blk += 16) {
    double v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = p[(size_t)(blk + u) * stride];
#pragma unroll
    for (int u = 0; u < 16; ++u) s += v[u];
  }
  for (; blk < nblocks; ++blk) s += p[(size_t)blk * stride];
  return s;
}

// (launched with one block of kGuardSelThreads threads: the (state, candidate)
// sums are formed in parallel, then thread j decides for state j)
constexpr int kGuardSelThreads = 256;
__global__ void __launch_bounds__(kGuardSelThreads)
    guard_select_kernel(loghmm_model_t* __restrict__ mout, int K, int sidx,
                        double* __restrict__ guard, int ncand,
                        const double* __restrict__ part, int nblocks,
                        int32_t* __restrict__ status, int* __restrict__ need_more) {
  __shared__ double s_sums[LOGHMM_MAX_STATES * LOGHMM_GUARD_CANDIDATES];
  for (int pr = threadIdx.x; pr < K * LOGHMM_GUARD_CANDIDATES; pr += blockDim.x) {
    const int jj = pr / LOGHMM_GUARD_CANDIDATES, k = pr % LOGHMM_GUARD_CANDIDATES;
    const bool pending = guard[(size_t)(sidx * K + jj) * kGuardStride + 5] != 0.0;
    s_sums[pr] = (pending && k < ncand) ? guard_partial_sum(part, nblocks, K, jj, k) : 0.0;
  }
  __syncthreads();
  const int j = threadIdx.x;
  if (j >= K) return;
  double* gs = guard + (size_t)(sidx * K + j) * kGuardStride;
  if (gs[5] == 0.0) return;
  double sums[LOGHMM_GUARD_CANDIDATES];
  for (int k = 0; k < ncand; ++k) sums[k] = s_sums[j * LOGHMM_GUARD_CANDIDATES + k];
  const double mu = gs[0], sigma = gs[1], nu0 = gs[2], n = gs[4];
  const double base = st_ll(n, sums[0], sigma, nu0);
  double c = gs[3];
  const int k0 = (int)gs[6];
  for (int k = 0; k < k0; ++k) c = nu0 + 0.5 * (c - nu0);
  int chosen = -1;
  for (int k = 1; k < ncand; ++k) {
    if (k0 + k - 1 >= 60) break;
    if (st_ll(n, sums[k], sigma, c) >= base - 1e-12) {
      chosen = k;
      break;
    }
    c = nu0 + 0.5 * (c - nu0);
  }
  loghmm_emission_t& e = mout->em[sidx][j];
  if (chosen > 0) {
    e.p[2] = c;
    gs[5] = 0.0;
  } else if (k0 + ncand - 1 >= 60) {
    e.p[2] = nu0;  // for-else: fall back to nu0
    gs[5] = 0.0;
  } else {
    gs[6] = (double)(k0 + ncand - 1);
    atomicExch(need_more, 1);
    return;
  }
  e.p[0] = mu;
  e.p[1] = sigma;
  em_constants(e);
  status[sidx * K + j] &= ~LOGHMM_MS_STUDENT_GUARD;
}

// Exact second pass for flagged states (distributions.py:616-620 two-pass
// variance; :1051 sigma^2 = sum w u (y - mu)^2 / n): per-block partial sums of
// w (y - centre)^2 (Gaussian, Gamma) or w u (y - centre)^2 with u at the old
// Student-t parameters.  Blocks skip states that are not flagged.
// Finish for state j (one thread): the exact second-pass sum S.
__device__ inline void variance_finish_state(loghmm_model_t* __restrict__ mout, int K, int sidx,
                                             int j, const double* __restrict__ guard, double S,
                                             int32_t* __restrict__ status) {
  const double* gs = guard + (size_t)(sidx * K + j) * kGuardStride;
  loghmm_emission_t& e = mout->em[sidx][j];
  const double n = gs[13];
  int32_t& st = status[sidx * K + j];
  if (e.family == LOGHMM_FAM_GAUSSIAN) {
    e.p[0] = gs[9];
    e.p[1] = fmax(sqrt(S / n), kScaleFloor);
  } else if (e.family == LOGHMM_FAM_GAMMA) {
    st = gamma_fit(n, gs[9], S / n, gs[14], e);
    if (st >= 16) return;
  } else if (e.family == LOGHMM_FAM_STUDENT_T) {
    const double sigma = fmax(sqrt(S / n), kScaleFloor);
    e.p[1] = sigma;
    // the guard pass reads sigma from its own scratch
    const_cast<double*>(gs)[1] = sigma;
  }
  em_constants(e);
}

// Exact second pass for flagged states (distributions.py:616-620 two-pass
// variance; :1051 sigma^2 = sum w u (y - mu)^2 / n): per-block partial sums of
// w (y - centre)^2 (Gaussian, Gamma) or w u (y - centre)^2 with u at the old
// Student-t parameters; the last block to finish sums the block partials in
// block order and finishes the flagged states.  Blocks exit at once when no
// state of the stream is flagged.  `counter` must be zero before the first
// launch; the last block resets it.
template <typename R>
__global__ void __launch_bounds__(256) variance_pass_kernel(const R* __restrict__ y,
                                                            const R* __restrict__ gamma, int64_t N,
                                                            int K, int sidx,
                                                            loghmm_model_t* __restrict__ mout,
                                                            const double* __restrict__ guard,
                                                            double* __restrict__ part,
                                                            unsigned* __restrict__ counter,
                                                            int32_t* __restrict__ status,
                                                            double* __restrict__ sums_out) {
  __shared__ double red[256];
  __shared__ bool last;
  __shared__ unsigned flagged;
  if (threadIdx.x == 0) {
    unsigned m = 0;
    for (int j = 0; j < K; ++j)
      if (guard[(size_t)(sidx * K + j) * kGuardStride + 8] != 0.0) m |= 1u << (j & 31);
    flagged = m;
  }
  __syncthreads();
  if (flagged == 0u) return;
  for (int j = 0; j < K; ++j) {
    const double* gs = guard + (size_t)(sidx * K + j) * kGuardStride;
    if (gs[8] == 0.0) continue;
    const int fam = mout->em[sidx][j].family;
    const double c = gs[9];
    double acc = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x) {
      const double w = (double)gamma[i * K + j];
      if (w > 0.0) {
        const double yy = (double)y[i];
        const double d = yy - c;
        double ww = w;
        if (fam == LOGHMM_FAM_STUDENT_T) {
          const double z = (yy - gs[10]) / gs[11];
          ww = w * ((gs[12] + 1.0) / (gs[12] + z * z));
        }
        acc += ww * d * d;
      }
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
      if ((int)threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[(size_t)blockIdx.x * K + j] = red[0];
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int j = threadIdx.x;
  if (j < K && guard[(size_t)(sidx * K + j) * kGuardStride + 8] != 0.0) {
    double S = 0.0;
    for (unsigned blk = 0; blk < gridDim.x; ++blk) S += __ldcg(part + (size_t)blk * K + j);
    // multi-rank split: leave this rank's sum for the cross-rank all-reduce
    if (sums_out) sums_out[j] = S;
    else variance_finish_state(mout, K, sidx, j, guard, S, status);
  }
  if (threadIdx.x == 0) *counter = 0u;
}

// Finish of the multi-rank split: sums[j] is the all-reduced second-pass sum.
__global__ void variance_finish_kernel(loghmm_model_t* __restrict__ mout, int K, int sidx,
                                       const double* __restrict__ guard,
                                       const double* __restrict__ sums,
                                       int32_t* __restrict__ status) {
  const int j = threadIdx.x;
  if (j < K && guard[(size_t)(sidx * K + j) * kGuardStride + 8] != 0.0)
    variance_finish_state(mout, K, sidx, j, guard, sums[j], status);
}

// Block partials of the guard pass folded in block order into
// sums[j * LOGHMM_GUARD_CANDIDATES + k] (pending states only; zeros else), the
// per-rank input of the cross-rank all-reduce.
__global__ void guard_fold_kernel(int K, int sidx, const double* __restrict__ guard, int ncand,
                                  const double* __restrict__ part, int nblocks,
                                  double* __restrict__ sums) {
  for (int pr = threadIdx.x; pr < K * LOGHMM_GUARD_CANDIDATES; pr += blockDim.x) {
    const int j = pr / LOGHMM_GUARD_CANDIDATES, k = pr % LOGHMM_GUARD_CANDIDATES;
    const bool pending = guard[(size_t)(sidx * K + j) * kGuardStride + 5] != 0.0;
    sums[pr] = (pending && k < ncand) ? guard_partial_sum(part, nblocks, K, j, k) : 0.0;
  }
}

}  // namespace lhmm

#include "hmm_extfit.cuh"
