// hmm_large.cuh — forward-backward and Viterbi for 8 < K <= 64 (config 5).
//
// One CTA per sequence, one thread per state.  The transition matrix is
// staged once in shared memory; the state vector is exchanged through shared
// memory with one barrier per step; the emission log-densities are computed
// for the whole batch beforehand (emission_kernel, fully parallel) so the
// sequential sweeps only load them, one step ahead.  This is the straightforward sequential
// sweep over T (inference.py:129-146, 191-210); the parallel-over-T scan of
// hmm_fb.cuh costs K^3 per step and does not pay at K=64.
#pragma once

#include "hmm_common.cuh"
#include "hmm_fb.cuh"
#include "hmm_viterbi.cuh"

namespace lhmm {

template <typename R>
__device__ __forceinline__ R block_max(R v, R* red, int nw) {
  v = warp_max(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  R m = red[0];
  for (int i = 1; i < nw; ++i) m = rmax(m, red[i]);
  return m;
}

template <typename R>
__device__ __forceinline__ R block_sum(R v, R* red, int nw) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  R m = red[0];
  for (int i = 1; i < nw; ++i) m += red[i];
  return m;
}

// Double-buffered block reductions of one or two values: one barrier each
// (reduction k+2 reuses reduction k's buffer only after every thread has
// passed reduction k+1's barrier, i.e. finished reading reduction k).
template <typename R>
struct BRed {
  R* red;  // 4 * 32 elements
  int nw;
  int buf;
  __device__ __forceinline__ BRed(R* r, int n) : red(r), nw(n), buf(0) {}
  // (max a, op b) where op = max (kMax) or sum
  template <bool kSecondMax>
  __device__ __forceinline__ void two(R& a, R& b) {
    a = warp_max(a);
    b = kSecondMax ? warp_max(b) : warp_sum(b);
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    R* rb = red + buf * 64;
    if (lane == 0) {
      rb[w] = a;
      rb[32 + w] = b;
    }
    __syncthreads();
    R x = rb[0], y = rb[32];
    for (int i = 1; i < nw; ++i) {
      x = fmax(x, rb[i]);
      y = kSecondMax ? fmax(y, rb[32 + i]) : y + rb[32 + i];
    }
    a = x;
    b = y;
    buf ^= 1;
  }
};

// Observation features needed by the E-step statistics only (no lgamma LUT).
template <typename R>
__device__ __forceinline__ void stat_features(ObsFeat<R>& f, R y, int fam) {
  f.y = y;
  if (fam == LOGHMM_FAM_GAMMA) f.logy = y > R(0) ? Num<R>::alog(y) : Num<R>::ninf();
  if (fam == LOGHMM_FAM_VON_MISES) Num<R>::asincos(y, &f.siny, &f.cosy);
  if (fam == LOGHMM_FAM_POISSON) f.pois_ok = (y >= R(0)) && (floor(y) == y);
}

// blockDim.x = 32 * ceil(K/32); thread j < K owns state j.  The emission
// log-densities come precomputed ([N, K], emission_kernel) and every per-step
// load (log b, y, alpha~) is issued one step ahead, off the recursion chain.
// Dot product of a register array with a shared-memory vector (read 16 bytes
// at a time; entries >= K of the vector are zero).
template <typename R, int KM>
__device__ __forceinline__ R reg_dot(const R (&r)[KM], const R* __restrict__ v) {
  R c[4] = {R(0), R(0), R(0), R(0)};
  if constexpr (sizeof(R) == 4) {
#pragma unroll
    for (int i = 0; i < KM; i += 4) {
      const float4 q = *reinterpret_cast<const float4*>(v + i);
      c[0] = fma(r[i], q.x, c[0]);
      c[1] = fma(r[i + 1], q.y, c[1]);
      c[2] = fma(r[i + 2], q.z, c[2]);
      c[3] = fma(r[i + 3], q.w, c[3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < KM; i += 2) {
      const double2 q = *reinterpret_cast<const double2*>(v + i);
      c[(i >> 1) & 3] = fma(r[i], q.x, c[(i >> 1) & 3]);
      c[((i >> 1) + 2) & 3] = fma(r[i + 1], q.y, c[((i >> 1) + 2) & 3]);
    }
  }
  return (c[0] + c[1]) + (c[2] + c[3]);
}

// KM: padded state count (16, 32 or 64).  Thread j keeps column j of A
// (forward), row j of A (backward) and column j of the xi accumulators in
// registers; only the carried vectors go through shared memory.
template <typename R, int KM>
__global__ void __launch_bounds__(64) fb_large_kernel(const FBArgs a, int K, const R* __restrict__ lbws) {
  typedef Num<R> N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  // xi accumulators in registers when they fit (fp32, or fp64 with KM <= 32),
  // else a [KM][64] shared array (column j owned by thread j)
  constexpr bool XREG = (int)sizeof(R) * KM <= 256;
  R* av = reinterpret_cast<R*>(smem_raw);  // KM (current vector, zero padded)
  R* red = av + KM;                         // 128 (double-buffered reductions)
  R* apv = red + 128;                       // KM (alpha~_{t-1}, backward sweep)
  R* Xs = apv + KM;                         // [KM][64] when !XREG
  const int tid = threadIdx.x;
  const int nw = blockDim.x >> 5;
  const int64_t b = blockIdx.x;
  if (b >= a.B) return;
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const bool act = tid < K;
  const int j = act ? tid : 0;
  const loghmm_model_t* md = a.model;
  R Acol[KM];  // column j of A (forward sweep only)
#pragma unroll
  for (int i = 0; i < KM; ++i) Acol[i] = (act && i < K) ? (R)md->A[i * K + j] : R(0);
  if (tid < KM) {
    av[tid] = R(0);
    apv[tid] = R(0);
  }
  const EmP<R> p0 = load_emission<R>(md->em[0][j]);
  EmP<R> p1;
  const bool two = a.n_streams > 1;
  if (two) p1 = load_emission<R>(md->em[1][j]);
  else p1.fam = LOGHMM_FAM_NONE;
  const R lpi = (R)md->log_pi[j];
  const R* y0g = reinterpret_cast<const R*>(a.y0) + start;
  const R* y1g = two ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
  R* aws = reinterpret_cast<R*>(a.alpha_ws) + start * K;  // [T, K] normalised alpha
  R* outA = a.log_alpha ? reinterpret_cast<R*>(a.log_alpha) + start * K : nullptr;
  R* outB = a.log_beta ? reinterpret_cast<R*>(a.log_beta) + start * K : nullptr;
  R* outG = a.gamma ? reinterpret_cast<R*>(a.gamma) + start * K : nullptr;
  R* outX = a.xi ? reinterpret_cast<R*>(a.xi) + (start - b) * (int64_t)K * K : nullptr;
  bool oob = false, nan_seen = false;
  int dead_t = INT_MAX;
  __syncthreads();

  // forward (two barriers per step)
  BRed<R> br(red, nw);
  double lam = 0.0;
  R a_j = R(0);
  const R* __restrict__ lbs = lbws + start * K;
  R lbn = (act && T > 0) ? lbs[j] : N::ninf();
  R yn0 = T > 0 ? y0g[0] : R(0), yn1 = (two && T > 0) ? y1g[0] : R(0);
  for (int t = 0; t < T; ++t) {
    const R v0 = yn0, v1 = yn1;
    const R lb = lbn;
    if (t + 1 < T) {  // prefetch step t + 1
      lbn = act ? lbs[(int64_t)(t + 1) * K + j] : N::ninf();
      yn0 = y0g[t + 1];
      if (two) yn1 = y1g[t + 1];
    }
    if (isnan(v0) || isnan(v1)) nan_seen = true;
    R u;
    if (t == 0) {
      u = lpi + lb;
    } else {
      const R acc = reg_dot<R, KM>(Acol, av);
      u = (acc > R(0) ? N::flog(acc) : N::ninf()) + lb;
    }
    if (act && outA) outA[(int64_t)t * K + j] = (R)lam + u;
    R M = act ? u : N::ninf(), mlb = act ? lb : N::ninf();
    br.two<true>(M, mlb);
    if (!(mlb > N::ninf()) && t < dead_t) dead_t = t;
    a_j = (M > N::ninf()) ? N::fexp(u - M) : R(0);
    if (M > N::ninf()) lam += (double)M;
    if (act) {
      av[j] = a_j;
      aws[(int64_t)t * K + j] = a_j;
    }
    __syncthreads();
  }
  double LL;
  {
    const R s = block_sum(act ? a_j : R(0), red, nw);
    LL = s > R(0) ? lam + (double)N::flog(s) : -CUDART_INF;
  }

  // backward
  R* wv = av;  // reuse: w vector
  R gtot = R(0), g0 = R(0);
  R st[2][LOGHMM_NSLOT];
  for (int s = 0; s < 2; ++s)
    for (int q = 0; q < LOGHMM_NSLOT; ++q) st[s][q] = R(0);
  R Arow[KM];  // row j of A (backward sweep)
#pragma unroll
  for (int i = 0; i < KM; ++i) Arow[i] = (act && i < K) ? (R)md->A[j * K + i] : R(0);
  R Xc[XREG ? KM : 1];
#pragma unroll
  for (int i = 0; i < (XREG ? KM : 1); ++i) Xc[i] = R(0);
  if (!XREG)
    for (int i = 0; i < KM; ++i) Xs[i * 64 + tid] = R(0);
  R r = R(0);  // log beta~ at current t (max 0)
  double rho = 0.0;
  R bl = (act && T > 0) ? lbs[(int64_t)(T - 1) * K + j] : N::ninf();
  R by0 = T > 0 ? y0g[T - 1] : R(0), by1 = (two && T > 0) ? y1g[T - 1] : R(0);
  R bat = (act && T > 0) ? aws[(int64_t)(T - 1) * K + j] : R(0);
  for (int t = T - 1; t >= 0; --t) {
    const R v0 = by0, v1 = by1, lb = bl, at = bat;
    if (t >= 1) {  // prefetch step t - 1 (its alpha~ is also this step's a_{t-1})
      bl = act ? lbs[(int64_t)(t - 1) * K + j] : N::ninf();
      by0 = y0g[t - 1];
      if (two) by1 = y1g[t - 1];
      bat = act ? aws[(int64_t)(t - 1) * K + j] : R(0);
    }
    ObsFeat<R> f0, f1;
    stat_features<R>(f0, v0, p0.fam);
    if (two) stat_features<R>(f1, v1, p1.fam);
    // gamma at t: a_t * exp(r); with it the max of u = lb_t + r for the step
    // to t-1 (one reduction for both)
    const R q = act ? N::fexp(r) : R(0);
    R M = act ? lb + r : N::ninf(), gz = at * q;
    br.two<false>(M, gz);
    const R gj = at * q / gz;
    if (act) {
      if (outB) outB[(int64_t)t * K + j] = (R)rho + r;
      if (outG) outG[(int64_t)t * K + j] = gj;
      R accs[LOGHMM_NSLOT];
      for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) accs[qq] = st[0][qq];
      stat_acc_rt<R>(accs, gj, p0, f0);
      for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) st[0][qq] = accs[qq];
      if (two) {
        for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) accs[qq] = st[1][qq];
        stat_acc_rt<R>(accs, gj, p1, f1);
        for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) st[1][qq] = accs[qq];
      }
      if (t < T - 1) gtot += gj;
      if (t == 0) g0 = gj;
    }
    if (t == 0) break;
    // step to t-1: u = lb_t + r; w = exp(u - M); q_{t-1} = A w
    const R u = act ? lb + r : N::ninf();
    const bool fin = M > N::ninf();
    const R w = (act && fin) ? N::fexp(u - M) : R(0);
    const R ap = bat;  // alpha~_{t-1}, prefetched above
    if (act) {
      wv[j] = w;
      apv[j] = ap;  // alpha~_{t-1}, read by every thread below
    }
    __syncthreads();
    const R acc = act ? reg_dot<R, KM>(Arow, wv) : R(0);
    // xi_{t-1}(i, j) = a_{t-1}[i] A_ij w_j / Z, Z = sum_i a_{t-1}[i] q_i;
    // with it the max of log q for the renormalisation (one reduction)
    const R lq = acc > R(0) ? N::flog(acc) : N::ninf();
    R mq = act ? lq : N::ninf(), Z = ap * acc;
    br.two<false>(mq, Z);
    const R iz = R(1) / Z;
    // thread j (as column) accumulates X[i][j] += a_i/Z * w_j
    if (act) {
      const R wz = w * iz;
      if constexpr (XREG && sizeof(R) == 4) {
#pragma unroll
        for (int i = 0; i < KM; i += 4) {
          const float4 q = *reinterpret_cast<const float4*>(apv + i);
          Xc[i] = fma(q.x, wz, Xc[i]);
          Xc[i + 1] = fma(q.y, wz, Xc[i + 1]);
          Xc[i + 2] = fma(q.z, wz, Xc[i + 2]);
          Xc[i + 3] = fma(q.w, wz, Xc[i + 3]);
        }
      } else if constexpr (XREG) {
#pragma unroll
        for (int i = 0; i < KM; i += 2) {
          const double2 q = *reinterpret_cast<const double2*>(apv + i);
          Xc[i] = fma(q.x, wz, Xc[i]);
          Xc[i + 1] = fma(q.y, wz, Xc[i + 1]);
        }
      } else {
        for (int i = 0; i < K; ++i) Xs[i * 64 + tid] = fma(apv[i], wz, Xs[i * 64 + tid]);
      }
      if (outX)
        for (int i = 0; i < K; ++i)
          outX[((int64_t)(t - 1) * K + i) * K + j] = apv[i] * iz * (R)md->A[i * K + j] * w;
    }
    if (mq > N::ninf()) {
      r = lq - mq;
      rho += (fin ? (double)M : 0.0) + (double)mq;
    }
    // note: log_beta[t-1] = rho_prev + M + lq  ==  (rho + r) after the update
    // (no end-of-step barrier: the next step's first reduction orders this
    // step's wv / apv reads before its writes)
  }
  __syncthreads();
  const int tid0 = tid;
  // reductions into the partials row
  if (a.partials) {
    double* row = a.partials + b * a.stats_width;
    if (act) {
      if constexpr (XREG) {
#pragma unroll
        for (int i = 0; i < KM; ++i)
          if (i < K) row[i * K + j] = (double)Xc[i] * md->A[i * K + j];
      } else {
        for (int i = 0; i < K; ++i) row[i * K + j] = (double)Xs[i * 64 + tid] * md->A[i * K + j];
      }
      row[K * K + j] = (double)gtot;
      row[K * K + K + j] = (double)g0;
      for (int s = 0; s < 2; ++s)
        for (int qq = 0; qq < LOGHMM_NSLOT; ++qq)
          row[K * K + 2 * K + (s * K + j) * LOGHMM_NSLOT + qq] = (double)st[s][qq];
    }
  }
  // dead / nan flags
  __shared__ int s_dead, s_nan, s_oob;
  if (tid0 == 0) {
    s_dead = INT_MAX;
    s_nan = 0;
    s_oob = 0;
  }
  __syncthreads();
  if (dead_t != INT_MAX) atomicMin(&s_dead, dead_t);
  if (nan_seen) s_nan = 1;
  if (oob) s_oob = 1;
  __syncthreads();
  if (tid0 == 0) {
    a.ll[b] = LL;
    if (a.flags) {
      a.flags[2 * b] = s_dead == INT_MAX ? -1 : s_dead;
      a.flags[2 * b + 1] = (s_nan ? 1 : 0) | (s_oob ? 2 : 0);
    }
  }
}

// Viterbi, one CTA per sequence, thread j = destination state.  Backpointers
// go to a byte table in the workspace; thread 0 walks the path with blocks of
// backpointer rows prefetched into shared memory.
template <typename R>
__global__ void __launch_bounds__(64) viterbi_large_kernel(const VitArgs a, int K,
                                                           uint8_t* backws) {
  typedef Num<R> N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* LA = reinterpret_cast<R*>(smem_raw);  // K*K log A
  R* dv = LA + K * K;                      // K
  uint8_t* bblk = reinterpret_cast<uint8_t*>(dv + K);  // 256*K bytes
  __shared__ int s_cur;
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  if (b >= a.B) return;
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const bool act = tid < K;
  const int j = act ? tid : 0;
  const loghmm_model_t* md = a.model;
  for (int e = tid; e < K * K; e += blockDim.x) LA[e] = (R)md->log_A[e];
  const loghmm_emission_t e0 = md->em[0][j];
  loghmm_emission_t e1;
  const bool two = a.n_streams > 1;
  if (two) e1 = md->em[1][j];
  const R* y0g = reinterpret_cast<const R*>(a.y0) + start;
  const R* y1g = two ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
  uint8_t* bk = backws + start * K;
  bool oob = false;
  auto logb = [&](int t) -> R {
    R v = exact_logb<R>(e0, y0g[t], a.lut, a.lut_n, oob);
    if (two) v = N::add(v, exact_logb<R>(e1, y1g[t], a.lut, a.lut_n, oob));
    return v;
  };
  R delta = act ? N::add((R)md->log_pi[j], logb(0)) : N::ninf();
  if (act) {
    dv[j] = delta;
    bk[j] = 0;
    if (a.back) a.back[start * K + j] = 0;
  }
  __syncthreads();
  for (int t = 1; t < T; ++t) {
    R lb = act ? logb(t) : R(0);
    R best = N::ninf();
    int bi = 0;
    if (act) {
      best = N::add(dv[0], LA[j]);
      for (int i = 1; i < K; ++i) {
        const R c = N::add(dv[i], LA[i * K + j]);
        if (c > best) {
          best = c;
          bi = i;
        }
      }
    }
    __syncthreads();
    if (act) {
      delta = N::add(best, lb);
      dv[j] = delta;
      bk[(int64_t)t * K + j] = (uint8_t)bi;
      if (a.back) a.back[(start + t) * K + j] = (uint8_t)bi;
    }
    __syncthreads();
  }
  if (tid == 0) {
    R bv = dv[0];
    int bi = 0;
    for (int i = 1; i < K; ++i)
      if (dv[i] > bv) {
        bv = dv[i];
        bi = i;
      }
    a.log_joint[b] = (double)bv;
    s_cur = bi;
  }
  __syncthreads();
  __threadfence_block();
  // backtrace in blocks of 256 rows, walking down
  constexpr int BLK = 256;
  for (int hi = T - 1; hi >= 0; hi -= BLK) {
    const int lo = max(0, hi - BLK + 1);
    const int rows = hi - lo + 1;
    for (int e = tid; e < rows * K; e += blockDim.x) bblk[e] = bk[(int64_t)lo * K + e];
    __syncthreads();
    if (tid == 0) {
      int cur = s_cur;
      for (int t = hi; t >= lo; --t) {
        a.path[start + t] = cur;
        if (t >= 1) cur = bblk[(t - lo) * K + cur];
      }
      s_cur = cur;
    }
    __syncthreads();
  }
}

}  // namespace lhmm
