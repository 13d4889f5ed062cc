// hmm_extfit.cuh — weighted-sample M-step fits of the ten families off the
// benchmarked configurations (LogNormal .. Pareto), on the device.
//
// Reference: distributions.py:639-723 (closed forms: lognormal, exponential,
// rayleigh, uniform, categorical, pareto), :732-761 (_newton_1d), :789-829
// (fit_beta_nr, 2-D Newton), :832-871 (fit_weibull_nr, Newton with a data
// pass per iteration), :919-953 (fit_negbinom_nr, same), :956-973
// (fit_chisquared).  Every state loghmm_mstep leaves pending
// (LOGHMM_MS_EXT_FIT) runs a small per-state program of data passes over
// (y, gamma[:, j]); between passes a one-thread-per-state finish step
// advances the program (moments -> centred moments -> Newton iterations),
// exactly the sequence of dot products the reference evaluates, and finally
// writes the parameters and the density constants into the model block.
// Sums are per-block partials added in block order (deterministic).
#pragma once

#include "hmm_common.cuh"

namespace lhmm {

constexpr int kExtSlots = 16;  // [0..11] sums, [12..13] minima, [14..15] maxima
constexpr int kExtBlocks = 148 * 2;

// per-state program scratch in guard_state (never [5] / [8]: the Student-t
// guard and the variance pass read those for every state of the stream)
enum ExtSlot { kXPhase = 0, kXN = 1, kXMean = 2, kXA = 3, kXB = 4, kXX = 6, kXLo = 7, kXHi = 9,
               kXIt = 10, kXMaxLog = 11, kXC = 12, kXD = 13, kXSeed = 15 };
enum ExtPhase { kPhA = 0, kPhB = 1, kPhNewton = 2, kPhCheck = 3, kPhFinal = 4, kPhDone = 5 };

__device__ inline bool ext_pending(const double* gs, int32_t st) {
  return (st & LOGHMM_MS_EXT_FIT) && gs[kXPhase] < kPhDone;
}

// One observation's contributions to the state's pass sums.
__device__ inline void ext_accumulate(int fam, int aux, const double* gs, double y, double w,
                                      double (&s)[kExtSlots]) {
  const int ph = (int)gs[kXPhase];
  const bool eff = w > 0.0;  // WeightedSample.effective() (distributions.py:137-141)
  switch (fam) {
    case LOGHMM_FAM_LOGNORMAL:
      if (!eff) return;
      if (ph == kPhA) {
        s[0] += w;
        if (y > 0.0) s[1] += w * log(y);
        else s[11] += 1.0;
      } else {
        const double d = log(y) - gs[kXMean];
        s[0] += w * (d * d);
      }
      return;
    case LOGHMM_FAM_EXPONENTIAL:
      if (!eff) return;
      s[0] += w;
      s[1] += w * y;
      if (y < 0.0) s[11] += 1.0;
      return;
    case LOGHMM_FAM_RAYLEIGH:
      if (!eff) return;
      s[0] += w;
      s[1] += w * (y * y);
      if (y < 0.0) s[11] += 1.0;
      return;
    case LOGHMM_FAM_UNIFORM:  // endpoints from ALL observations (distributions.py:676-684)
      s[0] += w;
      s[12] = fmin(s[12], y);
      s[14] = fmax(s[14], y);
      return;
    case LOGHMM_FAM_CATEGORICAL:
      if (!eff) return;
      s[0] += w;
      if (y < 0.0 || floor(y) != y) s[11] += 1.0;
      else if (y >= (double)aux) s[10] += 1.0;
      else s[1 + (int)y] += w;
      return;
    case LOGHMM_FAM_BETA:
      if (!eff) return;
      if (ph == kPhA) {
        s[0] += w;
        s[1] += w * y;
        if (y > 0.0 && y < 1.0) {
          s[2] += w * log(y);
          s[3] += w * log1p(-y);
        } else {
          s[11] += 1.0;
        }
      } else {
        const double d = y - gs[kXMean];
        s[0] += w * (d * d);
      }
      return;
    case LOGHMM_FAM_WEIBULL:
      if (!eff) return;
      if (ph == kPhA) {
        s[0] += w;
        s[1] += w * y;
        if (y > 0.0) {
          const double ly = log(y);
          s[2] += w * ly;
          s[14] = fmax(s[14], ly);
        } else {
          s[11] += 1.0;
        }
      } else if (ph == kPhB) {
        const double d = y - gs[kXMean];
        s[0] += w * (d * d);
      } else {  // ratios weighted by y^k, max-shifted (distributions.py:819-829)
        const double k = gs[kXX], ly = log(y);
        const double wk = w * exp(k * ly - k * gs[kXMaxLog]);
        s[0] += wk;
        s[1] += wk * ly;
        s[2] += wk * (ly * ly);
      }
      return;
    case LOGHMM_FAM_NEGBINOM:
      if (!eff) return;
      if (ph == kPhA) {
        s[0] += w;
        s[1] += w * y;
        if (y < 0.0 || floor(y) != y) s[11] += 1.0;
      } else if (ph == kPhB) {
        const double d = y - gs[kXMean];
        s[0] += w * (d * d);
      } else {
        const double r = gs[kXX];
        s[0] += w * sp_digamma(y + r);
        s[1] += w * sp_trigamma(y + r);
      }
      return;
    case LOGHMM_FAM_CHISQ:
      if (!eff) return;
      s[0] += w;
      s[1] += w * y;
      if (y > 0.0) s[2] += w * log(y);
      else s[11] += 1.0;
      return;
    case LOGHMM_FAM_PARETO:  // support and xm over ALL observations (:702-710)
      if (ph == kPhA) {
        s[0] += w;
        s[12] = fmin(s[12], y);
        if (!(y > 0.0)) s[11] += 1.0;
      } else if (eff) {
        s[1] += w * log(y / gs[kXMean]);
      }
      return;
    default:
      return;
  }
}

template <typename R>
__global__ void __launch_bounds__(256) ext_pass_kernel(const R* __restrict__ y,
                                                       const R* __restrict__ gamma, int64_t N, int K,
                                                       int sidx, const loghmm_model_t* __restrict__ m,
                                                       const double* __restrict__ guard,
                                                       const int32_t* __restrict__ status,
                                                       double* __restrict__ part) {
  __shared__ double red[256];
  for (int j = 0; j < K; ++j) {
    const double* gs = guard + (size_t)(sidx * K + j) * kGuardStride;
    if (!ext_pending(gs, status[sidx * K + j])) continue;
    const int fam = m->em[sidx][j].family, aux = m->em[sidx][j].reserved;
    double s[kExtSlots];
#pragma unroll
    for (int q = 0; q < kExtSlots; ++q) s[q] = q >= 14 ? -CUDART_INF : q >= 12 ? CUDART_INF : 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
      ext_accumulate(fam, aux, gs, (double)y[i], (double)gamma[i * K + j], s);
    for (int q = 0; q < kExtSlots; ++q) {
      red[threadIdx.x] = s[q];
      __syncthreads();
      for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
          const double a = red[threadIdx.x], b = red[threadIdx.x + w];
          red[threadIdx.x] = q >= 14 ? fmax(a, b) : q >= 12 ? fmin(a, b) : a + b;
        }
        __syncthreads();
      }
      if (threadIdx.x == 0) part[((size_t)blockIdx.x * K + j) * kExtSlots + q] = red[0];
      __syncthreads();
    }
  }
}

// _newton_1d (distributions.py:732-761), one evaluation per call: s, d are
// score and slope at gs[kXX].  Returns true when the program may move on
// (converged, or the final check after the iteration cap was evaluated).
__device__ inline bool ext_newton_step(double* gs, double sc, double d, double tol, bool& ok) {
  if ((int)gs[kXPhase] == kPhCheck) {
    ok = fabs(sc) <= tol;
    return true;
  }
  if (fabs(sc) <= tol) {
    ok = true;
    return true;
  }
  double x = gs[kXX];
  if (sc > 0.0) gs[kXLo] = fmax(gs[kXLo], x);
  else gs[kXHi] = fmin(gs[kXHi], x);
  double prop = d != 0.0 ? x - sc / d : CUDART_INF;
  if (!(isfinite(prop) && gs[kXLo] < prop && prop < gs[kXHi]))
    prop = isinf(gs[kXHi]) ? x * 8.0 : 0.5 * (gs[kXLo] + gs[kXHi]);
  gs[kXX] = prop;
  gs[kXIt] += 1.0;
  if (gs[kXIt] >= 50.0) gs[kXPhase] = kPhCheck;  // one more score evaluation
  return false;
}

__device__ inline void ext_newton_init(double* gs, double x0) {
  gs[kXX] = x0;
  gs[kXLo] = 0.0;
  gs[kXHi] = CUDART_INF;
  gs[kXIt] = 0.0;
  gs[kXPhase] = kPhNewton;
}

// Constants of the density records (distributions.py record() on the host).
__device__ inline void ext_constants(loghmm_emission_t& e) {
  switch (e.family) {
    case LOGHMM_FAM_LOGNORMAL: e.c[0] = log(e.p[1]); e.c[1] = 0.5 * kLog2Pi; break;
    case LOGHMM_FAM_EXPONENTIAL: e.c[0] = log(e.p[0]); break;
    case LOGHMM_FAM_RAYLEIGH: {
      const double s2 = e.p[0] * e.p[0];
      e.c[0] = log(s2);
      e.c[1] = 2.0 * s2;
      break;
    }
    case LOGHMM_FAM_UNIFORM: e.c[0] = -log(e.p[1] - e.p[0]); break;
    case LOGHMM_FAM_BETA: e.c[0] = lgamma(e.p[0]) + lgamma(e.p[1]) - lgamma(e.p[0] + e.p[1]); break;
    case LOGHMM_FAM_WEIBULL: e.c[0] = log(e.p[0]) - log(e.p[1]); break;
    case LOGHMM_FAM_NEGBINOM:
      e.c[0] = lgamma(e.p[0]);
      e.c[1] = e.p[0] * log(e.p[1]);
      e.c[2] = log1p(-e.p[1]);
      break;
    case LOGHMM_FAM_CHISQ: {
      const double half = e.p[0] / 2.0;
      e.c[0] = half * log(2.0);
      e.c[1] = lgamma(half);
      e.c[2] = half - 1.0;
      break;
    }
    case LOGHMM_FAM_PARETO:
      e.c[0] = log(e.p[1]) + e.p[1] * log(e.p[0]);
      e.c[1] = e.p[1] + 1.0;
      break;
    default: break;
  }
}

// Advance state j's program with the pass sums S; finish the fit when done.
__device__ inline void ext_finish_state(loghmm_emission_t& e, double* gs, const double (&S)[kExtSlots],
                                        int32_t& st, int& more) {
  const int ph = (int)gs[kXPhase];
  auto fail = [&](int32_t code) {
    st = code;
    gs[kXPhase] = kPhDone;
  };
  auto done = [&]() {
    gs[kXPhase] = kPhDone;
    st &= ~LOGHMM_MS_EXT_FIT;
    ext_constants(e);
  };
  switch (e.family) {
    case LOGHMM_FAM_LOGNORMAL:
      if (ph == kPhA) {
        if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
        gs[kXN] = S[0];
        gs[kXMean] = S[1] / S[0];
        gs[kXPhase] = kPhB;
        more = 1;
      } else {
        e.p[0] = gs[kXMean];
        e.p[1] = fmax(sqrt(S[0] / gs[kXN]), kScaleFloor);
        done();
      }
      return;
    case LOGHMM_FAM_EXPONENTIAL: {
      if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
      const double mean = S[1] / S[0];
      if (mean <= 0.0) return fail(LOGHMM_MS_ERR_DEGENERATE);
      e.p[0] = 1.0 / mean;
      return done();
    }
    case LOGHMM_FAM_RAYLEIGH:
      if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
      e.p[0] = fmax(sqrt(S[1] / (2.0 * S[0])), kScaleFloor);
      return done();
    case LOGHMM_FAM_UNIFORM: {
      const double lo = S[12];
      double hi = S[14];
      if (hi <= lo) hi = lo + kScaleFloor;
      e.p[0] = lo;
      e.p[1] = hi;
      return done();
    }
    case LOGHMM_FAM_CATEGORICAL: {
      if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
      if (S[10] > 0.0) return fail(LOGHMM_MS_ERR_CAT_CODE);
      const int mcat = e.reserved;
      double p[8], tot = 0.0;
      for (int k = 0; k < mcat; ++k) {
        p[k] = S[1 + k] / S[0];
        tot += p[k];
      }
      for (int k = 0; k < 8; ++k) {
        const double v = k < mcat ? p[k] / tot : 0.0;
        const double lv = v > 0.0 ? log(v) : -CUDART_INF;
        if (k < 4) e.p[k] = lv;
        else e.c[k - 4] = lv;
      }
      gs[kXPhase] = kPhDone;
      st &= ~LOGHMM_MS_EXT_FIT;
      return;
    }
    case LOGHMM_FAM_BETA:
      if (ph == kPhA) {
        if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
        const double n = S[0];
        gs[kXN] = n;
        gs[kXMean] = S[1] / n;
        gs[kXA] = S[2] / n;
        gs[kXB] = S[3] / n;
        gs[kXPhase] = kPhB;
        more = 1;
      } else {  // fit_beta_nr (distributions.py:789-829)
        const double n = gs[kXN], mean = gs[kXMean], m1 = gs[kXA], m2 = gs[kXB];
        const double var = S[0] / n;
        const double scale = var > 0.0 ? mean * (1.0 - mean) / var - 1.0 : -1.0;
        double a = 1.0, b = 1.0;
        if (scale > 0.0) {
          a = mean * scale;
          b = (1.0 - mean) * scale;
        }
        bool conv = false;
        for (int it = 0; it < 100; ++it) {
          const double psi_ab = sp_digamma(a + b);
          const double f1 = sp_digamma(a) - psi_ab - m1, f2 = sp_digamma(b) - psi_ab - m2;
          if (fmax(fabs(f1), fabs(f2)) <= 1e-10) {
            conv = true;
            break;
          }
          const double tri_ab = sp_trigamma(a + b);
          const double j11 = sp_trigamma(a) - tri_ab, j22 = sp_trigamma(b) - tri_ab, j12 = -tri_ab;
          const double det = j11 * j22 - j12 * j12;
          double da = -(f1 * j22 - f2 * j12) / det, db = -(f2 * j11 - f1 * j12) / det;
          while (a + da <= 0.0 || b + db <= 0.0) {
            da *= 0.5;
            db *= 0.5;
          }
          a += da;
          b += db;
        }
        if (!conv) {
          const double psi_ab = sp_digamma(a + b);
          if (fmax(fabs(sp_digamma(a) - psi_ab - m1), fabs(sp_digamma(b) - psi_ab - m2)) > 1e-10)
            st |= LOGHMM_MS_WARN_ITERCAP;
        }
        e.p[0] = a;
        e.p[1] = b;
        done();
      }
      return;
    case LOGHMM_FAM_WEIBULL:
      if (ph == kPhA) {
        if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
        const double n = S[0];
        gs[kXN] = n;
        gs[kXMean] = S[1] / n;
        gs[kXA] = S[2] / n;  // lbar
        gs[kXMaxLog] = S[14];
        gs[kXPhase] = kPhB;
        more = 1;
      } else if (ph == kPhB) {
        const double var = S[0] / gs[kXN];
        if (var <= 0.0) return fail(LOGHMM_MS_ERR_DEGENERATE);
        const double seed = pow(gs[kXMean] / sqrt(var), 1.086);
        gs[kXSeed] = seed;
        ext_newton_init(gs, seed);
        more = 1;
      } else if (ph == kPhNewton || ph == kPhCheck) {
        const double k = gs[kXX], r1 = S[1] / S[0], r2 = S[2] / S[0];
        const double sc = 1.0 / k + gs[kXA] - r1;
        const double d = -1.0 / (k * k) - (r2 - r1 * r1);
        bool ok = false;
        if (ext_newton_step(gs, sc, d, 1e-10, ok)) {
          if (!ok) {
            st |= LOGHMM_MS_WARN_NEWTON;
            gs[kXX] = gs[kXSeed];
          }
          gs[kXPhase] = kPhFinal;  // the scale needs s0 at the final shape
        }
        more = 1;
      } else {  // kPhFinal: scale = exp((log s0 + m - log n) / k)
        const double k = gs[kXX];
        const double m = k * gs[kXMaxLog];
        e.p[0] = k;
        e.p[1] = exp((log(S[0]) + m - log(gs[kXN])) / k);
        done();
      }
      return;
    case LOGHMM_FAM_NEGBINOM:
      if (ph == kPhA) {
        if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
        const double n = S[0], mean = S[1] / n;
        if (mean <= 0.0) return fail(LOGHMM_MS_ERR_DEGENERATE);
        gs[kXN] = n;
        gs[kXMean] = mean;
        gs[kXPhase] = kPhB;
        more = 1;
      } else if (ph == kPhB) {
        const double mean = gs[kXMean], var = S[0] / gs[kXN];
        if (var <= mean) {
          st |= LOGHMM_MS_WARN_BOUNDARY;
          const double r = kNegbinomCeiling;
          e.p[0] = r;
          e.p[1] = r / (r + mean);
          return done();
        }
        ext_newton_init(gs, mean * mean / (var - mean));
        more = 1;
      } else {
        const double r = gs[kXX], n = gs[kXN], mean = gs[kXMean];
        const double sc = S[0] / n - sp_digamma(r) + log(r / (r + mean));
        const double d = S[1] / n - sp_trigamma(r) + mean / (r * (r + mean));
        bool ok = false;
        if (ext_newton_step(gs, sc, d, 1e-8, ok)) {
          double rr = gs[kXX];
          if (rr > kNegbinomCeiling) {
            st |= LOGHMM_MS_WARN_CEILING;
            rr = kNegbinomCeiling;
          } else if (!ok) {
            st |= LOGHMM_MS_WARN_NEWTON;
          }
          e.p[0] = rr;
          e.p[1] = rr / (rr + mean);
          return done();
        }
        more = 1;
      }
      return;
    case LOGHMM_FAM_CHISQ: {  // fit_chisquared (distributions.py:956-973), Newton without data
      if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
      const double n = S[0], mean = S[1] / n;
      const double target = S[2] / n - log(2.0);
      const double x0 = fmax(mean, kScaleFloor);
      double x = x0, lo = 0.0, hi = CUDART_INF;
      bool ok = false;
      for (int it = 0; it < 50; ++it) {
        const double sc = 0.5 * (target - sp_digamma(x / 2.0));
        if (fabs(sc) <= 1e-10) {
          ok = true;
          break;
        }
        if (sc > 0.0) lo = fmax(lo, x);
        else hi = fmin(hi, x);
        const double d = -0.25 * sp_trigamma(x / 2.0);
        double prop = d != 0.0 ? x - sc / d : CUDART_INF;
        if (!(isfinite(prop) && lo < prop && prop < hi)) prop = isinf(hi) ? x * 8.0 : 0.5 * (lo + hi);
        x = prop;
      }
      if (!ok) ok = fabs(0.5 * (target - sp_digamma(x / 2.0))) <= 1e-10;
      if (!ok) {
        st |= LOGHMM_MS_WARN_NEWTON;
        x = x0;
      }
      e.p[0] = x;
      return done();
    }
    case LOGHMM_FAM_PARETO:
      if (ph == kPhA) {
        if (S[11] > 0.0) return fail(LOGHMM_MS_ERR_SUPPORT);
        gs[kXN] = S[0];
        gs[kXMean] = S[12];  // xm
        gs[kXPhase] = kPhB;
        more = 1;
      } else {
        const double denom = S[1];
        if (denom <= 0.0) return fail(LOGHMM_MS_ERR_DEGENERATE);
        e.p[0] = gs[kXMean];
        e.p[1] = gs[kXN] / denom;
        done();
      }
      return;
    default:
      return;
  }
}

__global__ void ext_finish_kernel(loghmm_model_t* __restrict__ mout, int K, int sidx,
                                  double* __restrict__ guard, int32_t* __restrict__ status,
                                  const double* __restrict__ part, int nblocks,
                                  int* __restrict__ need_more) {
  const int j = threadIdx.x;
  if (j >= K) return;
  double* gs = guard + (size_t)(sidx * K + j) * kGuardStride;
  int32_t& st = status[sidx * K + j];
  if (!ext_pending(gs, st)) return;
  double S[kExtSlots];
  for (int q = 0; q < kExtSlots; ++q) {
    double acc = q >= 14 ? -CUDART_INF : q >= 12 ? CUDART_INF : 0.0;
    for (int b = 0; b < nblocks; ++b) {
      const double v = part[((size_t)b * K + j) * kExtSlots + q];
      acc = q >= 14 ? fmax(acc, v) : q >= 12 ? fmin(acc, v) : acc + v;
    }
    S[q] = acc;
  }
  int more = 0;
  ext_finish_state(mout->em[sidx][j], gs, S, st, more);
  if (more) atomicExch(need_more, 1);
}

}  // namespace lhmm
