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

// Quarter-split layout: four adjacent lanes (j, q), q = tid & 3, share state
// j = tid >> 2.  Lane q holds the 16-byte chunks c = q, q + 4, ... of column
// j of A (forward), row j of A (backward) and column j of the xi
// accumulators, so a K-long dot product is K/4 FMAs per lane plus two xor
// shuffles (bit-identical in all four lanes), and the interleaved chunks keep
// the shared-memory vector reads conflict-free.
template <typename R, int KM, int P = 4>
struct Quarter {
  static constexpr int EPC = 16 / (int)sizeof(R);  // elements per 16-byte chunk
  static constexpr int NQC = KM / EPC / P;         // chunks per lane
  static constexpr int NQ = NQC * EPC;             // elements per lane (KM / P)
  static __device__ __forceinline__ int idx(int q, int s) {
    return (P * (s / EPC) + q) * EPC + s % EPC;
  }
  // sum_i r[i] v[i] over the lane's elements, then over the four lanes
  static __device__ __forceinline__ R dot(const R (&r)[NQ], const R* __restrict__ v, int q) {
    R c[2] = {R(0), R(0)};
    if constexpr (sizeof(R) == 4) {
#pragma unroll
      for (int m = 0; m < NQC; ++m) {
        const float4 x = *reinterpret_cast<const float4*>(v + (P * m + q) * 4);
        c[0] = fma(r[4 * m], x.x, c[0]);
        c[1] = fma(r[4 * m + 1], x.y, c[1]);
        c[0] = fma(r[4 * m + 2], x.z, c[0]);
        c[1] = fma(r[4 * m + 3], x.w, c[1]);
      }
    } else {
#pragma unroll
      for (int m = 0; m < NQC; ++m) {
        const double2 x = *reinterpret_cast<const double2*>(v + (P * m + q) * 2);
        c[0] = fma(r[2 * m], x.x, c[0]);
        c[1] = fma(r[2 * m + 1], x.y, c[1]);
      }
    }
    R p = c[0] + c[1];
#pragma unroll
    for (int o = 1; o < P; o <<= 1) p += __shfl_xor_sync(kFull, p, o);
    return p;
  }
};

// blockDim.x = 4 * KM (KM: padded state count, 16, 32 or 64), four lanes per
// state (Quarter).  The emission log-densities come precomputed ([N, K],
// emission_kernel) and every per-step load (log b, y, alpha~) is issued one
// step ahead, off the recursion chain.  Lane q == 0 of each state does the
// per-state work (outputs, statistics); only the carried vectors go through
// shared memory.
constexpr int kRing = 16;  // fb_large_kernel input ring depth (steps)

template <typename R, int KM, int P>
__global__ void __launch_bounds__(256) fb_large_kernel(const FBArgs a, int K, const R* __restrict__ lbws) {
  typedef Num<R> N;
  typedef Quarter<R, KM, P> Q;
  constexpr int NQ = Q::NQ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* av = reinterpret_cast<R*>(smem_raw);  // KM (current vector, zero padded)
  R* red = av + KM;                         // 128 (double-buffered reductions)
  R* apv = red + 128;                       // KM (alpha~_{t-1}, backward sweep)
  R* ring = apv + KM;                       // [kRing][4][KM] per-step inputs
  const int tid = threadIdx.x;
  const int nw = blockDim.x >> 5;
  const int q = tid & (P - 1);
  const int jt = tid / P;
  const int64_t b = blockIdx.x;
  if (b >= a.B) return;
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const bool act = jt < K;
  const bool lead = act && q == 0;
  const int j = act ? jt : 0;
  const loghmm_model_t* md = a.model;
  R Acol[NQ];  // column j of A, this lane's elements (forward sweep only)
#pragma unroll
  for (int s = 0; s < NQ; ++s) {
    const int i = Q::idx(q, s);
    Acol[s] = (act && i < K) ? (R)md->A[i * K + j] : R(0);
  }
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
  // Per-step inputs of state j (log b, y, alpha~) reach lane (j, 0) through a
  // private shared-memory ring [kRing][4][KM] filled by cp.async kRing - 1
  // steps ahead, so the global-load latency stays off the recursion chain.
  // step t into ring position pos (forward pos = t, backward pos = T - 1 - t)
  auto issue = [&](int t, int pos, bool with_alpha) {
    if (lead) {
      const bool ok = t >= 0 && t < T;
      const int tc = ok ? t : 0;
      R* sl = ring + (size_t)(pos % kRing) * 4 * KM;
      cp_async<sizeof(R)>(sl + j, lbs + (int64_t)tc * K + j, ok);
      cp_async<sizeof(R)>(sl + KM + j, y0g + tc, ok);
      if (two) cp_async<sizeof(R)>(sl + 2 * KM + j, y1g + tc, ok);
      if (with_alpha) cp_async<sizeof(R)>(sl + 3 * KM + j, aws + (int64_t)tc * K + j, ok);
    }
    cp_async_commit();
  };
  auto slot = [&](int t) -> const R* { return ring + (size_t)(t % kRing) * 4 * KM; };
#pragma unroll 1
  for (int d = 0; d < kRing - 1; ++d) issue(d, d, false);
  for (int t = 0; t < T; ++t) {
    issue(t + kRing - 1, t + kRing - 1, false);
    cp_async_wait<kRing - 1>();
    const R* sl = slot(t);
    const R lb = lead ? sl[j] : N::ninf();
    if (lead && (isnan(sl[KM + j]) || (two && isnan(sl[2 * KM + j])))) nan_seen = true;
    R u;
    if (t == 0) {
      u = lpi + lb;
    } else {
      const R acc = Q::dot(Acol, av, q);
      u = (acc > R(0) ? N::flog(acc) : N::ninf()) + lb;
    }
    if (lead && outA) outA[(int64_t)t * K + j] = (R)lam + u;
    R M = lead ? u : N::ninf(), mlb = lb;
    br.two<true>(M, mlb);
    if (!(mlb > N::ninf()) && t < dead_t) dead_t = t;
    a_j = (M > N::ninf()) ? N::fexp(u - M) : R(0);
    if (M > N::ninf()) lam += (double)M;
    if (lead) {
      av[j] = a_j;
      aws[(int64_t)t * K + j] = a_j;
    }
    __syncthreads();
  }
  cp_async_wait_all();
  double LL;
  {
    const R s = block_sum(lead ? a_j : R(0), red, nw);
    LL = s > R(0) ? lam + (double)N::flog(s) : -CUDART_INF;
  }

  // backward
  R* wv = av;  // reuse: w vector
  R gtot = R(0), g0 = R(0);
  R st[2][LOGHMM_NSLOT];
  for (int s = 0; s < 2; ++s)
    for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) st[s][qq] = R(0);
  R Arow[NQ];  // row j of A, this lane's elements (backward sweep)
#pragma unroll
  for (int s = 0; s < NQ; ++s) {
    const int i = Q::idx(q, s);
    Arow[s] = (act && i < K) ? (R)md->A[j * K + i] : R(0);
  }
  R Xc[NQ];  // xi accumulators X[i][j], this lane's i
#pragma unroll
  for (int s = 0; s < NQ; ++s) Xc[s] = R(0);
  R r = R(0);  // log beta~ at current t (max 0)
  double rho = 0.0;
  // ring position p = T - 1 - t (the sweep runs down)
#pragma unroll 1
  for (int d = 0; d < kRing - 1; ++d) issue(T - 1 - d, d, true);
  for (int t = T - 1; t >= 0; --t) {
    const int p = T - 1 - t;
    issue(t - (kRing - 1), p + kRing - 1, true);
    cp_async_wait<kRing - 2>();  // positions p and p + 1 (alpha~_{t-1}) landed
    const R* sl = ring + (size_t)(p % kRing) * 4 * KM;
    const R* sn = ring + (size_t)((p + 1) % kRing) * 4 * KM;
    const R lb = lead ? sl[j] : N::ninf();
    const R at = lead ? sl[3 * KM + j] : R(0);
    const R bat = (lead && t >= 1) ? sn[3 * KM + j] : R(0);
    // gamma at t: a_t * exp(r); with it the max of u = lb_t + r for the step
    // to t-1 (one reduction for both)
    const R qe = act ? N::fexp(r) : R(0);
    R M = lead ? lb + r : N::ninf(), gz = lead ? at * qe : R(0);
    br.two<false>(M, gz);
    if (lead) {
      const R gj = at * qe / gz;
      const R v0 = sl[KM + j], v1 = two ? sl[2 * KM + j] : R(0);
      ObsFeat<R> f0, f1;
      stat_features<R>(f0, v0, p0.fam);
      if (two) stat_features<R>(f1, v1, p1.fam);
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
    const R u = lead ? lb + r : N::ninf();
    const bool fin = M > N::ninf();
    const R w = (lead && fin) ? N::fexp(u - M) : R(0);
    const R ap = bat;  // alpha~_{t-1}, prefetched above
    if (lead) {
      wv[j] = w;
      apv[j] = ap;  // alpha~_{t-1}, read by every thread below
    }
    __syncthreads();
    R acc = Q::dot(Arow, wv, q);
    acc = act ? acc : R(0);
    // xi_{t-1}(i, j) = a_{t-1}[i] A_ij w_j / Z, Z = sum_i a_{t-1}[i] q_i;
    // with it the max of log q for the renormalisation (one reduction)
    const R lq = acc > R(0) ? N::flog(acc) : N::ninf();
    R mq = act ? lq : N::ninf(), Z = lead ? ap * acc : R(0);
    br.two<false>(mq, Z);
    const R iz = R(1) / Z;
    // lane (j, q) accumulates X[i][j] += a_i/Z * w_j for its i
    if (act) {
      const R wz = wv[j] * iz;  // w_j, written by lane (j, 0) before the barrier
#pragma unroll
      for (int m = 0; m < Q::NQC; ++m) {
        const R* pv = apv + (P * m + q) * Q::EPC;
        if constexpr (sizeof(R) == 4) {
          const float4 x = *reinterpret_cast<const float4*>(pv);
          Xc[4 * m] = fma(x.x, wz, Xc[4 * m]);
          Xc[4 * m + 1] = fma(x.y, wz, Xc[4 * m + 1]);
          Xc[4 * m + 2] = fma(x.z, wz, Xc[4 * m + 2]);
          Xc[4 * m + 3] = fma(x.w, wz, Xc[4 * m + 3]);
        } else {
          const double2 x = *reinterpret_cast<const double2*>(pv);
          Xc[2 * m] = fma(x.x, wz, Xc[2 * m]);
          Xc[2 * m + 1] = fma(x.y, wz, Xc[2 * m + 1]);
        }
      }
      if (outX)
        for (int s = 0; s < NQ; ++s) {
          const int i = Q::idx(q, s);
          if (i < K) outX[((int64_t)(t - 1) * K + i) * K + j] = apv[i] * iz * (R)md->A[i * K + j] * wv[j];
        }
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
  // reductions into the partials row
  if (a.partials) {
    double* row = a.partials + b * a.stats_width;
    if (act) {
#pragma unroll
      for (int s = 0; s < NQ; ++s) {
        const int i = Q::idx(q, s);
        if (i < K) row[i * K + j] = (double)Xc[s] * md->A[i * K + j];
      }
    }
    if (lead) {
      row[K * K + j] = (double)gtot;
      row[K * K + K + j] = (double)g0;
      for (int s = 0; s < 2; ++s)
        for (int qq = 0; qq < LOGHMM_NSLOT; ++qq)
          row[K * K + 2 * K + (s * K + j) * LOGHMM_NSLOT + qq] = (double)st[s][qq];
    }
  }
  // dead / nan flags
  __shared__ int s_dead, s_nan, s_oob;
  if (tid == 0) {
    s_dead = INT_MAX;
    s_nan = 0;
    s_oob = 0;
  }
  __syncthreads();
  if (dead_t != INT_MAX) atomicMin(&s_dead, dead_t);
  if (nan_seen) s_nan = 1;
  if (oob) s_oob = 1;
  __syncthreads();
  if (tid == 0) {
    a.ll[b] = LL;
    if (a.flags) {
      a.flags[2 * b] = s_dead == INT_MAX ? -1 : s_dead;
      a.flags[2 * b + 1] = (s_nan ? 1 : 0) | (s_oob ? 2 : 0);
    }
  }
}

// ---------------------------------------------------------------------------
// Split forward-backward for K > 8, fp32 (config 5): the forward and the
// backward recursions run in separate, concurrent CTAs (grid 2B), and the
// posteriors, the xi totals and the family statistics are formed afterwards
// by a T-parallel pass over the stored normalised vectors (fb_post_kernel),
// so the sequential chain of a sequence is one sweep, not two, and carries no
// xi / statistics work.
//   forward CTA  (blockIdx < B): alpha~_t -> aws, log alpha, LL, flags
//   backward CTA (blockIdx >= B): beta~_t (max 1) -> qws, w_t = b~_t beta~_t
//                                 (scaled) -> wws, log beta
// xi_{t-1}(i, j) = alpha~_{t-1}[i] A_ij w_t[j] / Z_t, Z_t = alpha~_{t-1}^T A w_t
// and gamma_t = alpha~_t beta~_t / sum, exactly the quantities of the fused
// kernel's backward sweep (training.py:199-210).
struct SplitWs {
  void* qws;          // [N, K] beta~ (linear, max 1)
  void* wws;          // [N, K] w_t
  double* seg_part;   // [B, kPostSegs, width] per-segment statistics
  int sparse_ok;      // take the structural-zero sweeps when A allows it (LOGHMM_FBL_SPARSE=0: never)
  int sparse_warps;   // fp32 structural-zero sweeps at K = 64: warps per sequence and direction (1 or 2)
};
constexpr int kPostSegs = 16;
constexpr int kPostWarps = 8;
constexpr int kPostPitch = 64 + 4;

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// ---------------------------------------------------------------------------
// Structural zeros in the sweeps (config 5's banded A): a zero A_ij adds
// nothing to the forward / backward sums, so each state only visits its
// non-zero sources (forward: column j) or targets (backward: row j).  One warp
// per sequence and direction, KM / 32 states per lane, the carried vector in
// shared memory behind a __syncwarp: no CTA barriers, one warp max-reduction
// per step.  Same recursion and workspace contents as the dense sweeps below
// (the backward vector is left unnormalised by its own maximum: it stays in
// [min A, 1], and every consumer is scale-invariant per step).
// ---------------------------------------------------------------------------
constexpr int kSweepNZ = 12;  // non-zeros per column / row the sparse sweeps cover
constexpr int kSweepPB = 16;  // steps of log b fetched ahead per block

// NW warps per sequence and direction, state s of a thread = tid + 32 NW s.
// One warp: the step's maximum is one redux.sync and the carried vector sits
// behind __syncwarp.  Two warps (one state per lane at K = 64): the warp maxima
// meet in a parity-indexed shared slot behind a named barrier — half the
// instructions per warp and step, which is what bounds the sweep (fp64: the
// software exp / log chains of one state instead of two per lane).
template <typename R, int KM, int NZ, int NW>
__device__ __forceinline__ void fb_sparse_sweep(const FBArgs& a, int K, const R* __restrict__ lbws,
                                                const SplitWs& sw, R* av, R* red, bool bwd, int64_t b) {
  typedef Num<R> N;
  constexpr int PB = kSweepPB;
  constexpr int NT = 32 * NW;
  constexpr int SPL = KM <= NT ? 1 : KM / NT;  // states per thread
  const int lane = threadIdx.x;  // thread index inside the NT threads
  int par = 0;                   // parity of the cross-warp reduction slot
  auto sync = [&]() {
    if constexpr (NW == 1) __syncwarp();
    else named_bar_sync(1, NT);
  };
  // maximum over the NT threads
  auto all_max = [&](R v) -> R {
    v = warp_max(v);
    if constexpr (NW > 1) {
      if ((lane & 31) == 0) red[par * NW + (lane >> 5)] = v;
      named_bar_sync(1, NT);
#pragma unroll
      for (int w = 0; w < NW; ++w) v = rmax(v, red[par * NW + w]);
      par ^= 1;
    }
    return v;
  };
  auto all_sum = [&](R v) -> R {
    v = warp_sum(v);
    if constexpr (NW > 1) {
      if ((lane & 31) == 0) red[par * NW + (lane >> 5)] = v;
      named_bar_sync(1, NT);
      R t = R(0);
#pragma unroll
      for (int w = 0; w < NW; ++w) t += red[par * NW + w];
      par ^= 1;
      v = t;
    }
    return v;
  };
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const loghmm_model_t* md = a.model;
  // lanes past K mirror state 0 and never store
  const bool act0 = lane < K;
  bool act[SPL];
  int js[SPL];
  const R* src[SPL][NZ];  // &av[source / target index]
  R Av[SPL][NZ];
#pragma unroll
  for (int s = 0; s < SPL; ++s) {
    js[s] = lane + NT * s;
    act[s] = js[s] < K;
    const int j = act[s] ? js[s] : 0;
#pragma unroll
    for (int n = 0; n < NZ; ++n) {
      src[s][n] = av;
      Av[s][n] = R(0);
    }
    int cnt = 0;
    for (int i = 0; i < K; ++i) {
      const R v = (R)(bwd ? md->A[j * K + i] : md->A[i * K + j]);
      if (act[s] && v > R(0)) {
#pragma unroll
        for (int n = 0; n < NZ; ++n)
          if (n == cnt) {
            src[s][n] = av + i;
            Av[s][n] = v;
          }
        ++cnt;
      }
    }
  }
  (void)act0;
  for (int e = lane; e < KM; e += NT) av[e] = R(0);
  auto dot = [&](int s) -> R {
    R c0 = R(0), c1 = R(0), c2 = R(0);
#pragma unroll
    for (int n = 0; n < NZ; n += 3) {
      c0 = fma(Av[s][n], *src[s][n], c0);
      if (n + 1 < NZ) c1 = fma(Av[s][n + 1], *src[s][n + 1], c1);
      if (n + 2 < NZ) c2 = fma(Av[s][n + 2], *src[s][n + 2], c2);
    }
    return (c0 + c1) + c2;
  };
  sync();
  const int64_t j0 = act[0] ? js[0] : 0;

  if (!bwd) {
    // NaN observations (inference.py:117-118): one coalesced scan
    bool nan_seen = false;
    {
      const R* y0g = reinterpret_cast<const R*>(a.y0) + start;
      const R* y1g = a.n_streams > 1 ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
      for (int t = lane; t < T; t += NT) {
        const R v0 = y0g[t];
        const R v1 = y1g ? y1g[t] : R(0);
        nan_seen |= (v0 != v0) | (v1 != v1);
      }
      nan_seen = all_max(nan_seen ? R(1) : R(0)) > R(0);
    }
    const bool hasA = a.log_alpha != nullptr;
    R* pA = hasA ? reinterpret_cast<R*>(a.log_alpha) + start * K + j0 : nullptr;  // running row pointers
    R* pW = reinterpret_cast<R*>(a.alpha_ws) + start * K + j0;
    const R* pL = lbws + start * K + j0;
    R lpi[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) lpi[s] = act[s] ? (R)md->log_pi[js[s]] : N::ninf();
    int dead_t = INT_MAX;
    double lam = 0.0;
    R lamf = R(0);
    R a_j[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) a_j[s] = R(0);
    R lbn[PB][SPL];
#pragma unroll
    for (int u = 0; u < PB; ++u)
#pragma unroll
      for (int s = 0; s < SPL; ++s) lbn[u][s] = (act[s] && u < T) ? pL[(int64_t)u * K + NT * s] : N::ninf();
    for (int tb = 0; tb < T; tb += PB) {
      R lbc[PB][SPL];
      pL += (int64_t)PB * K;
#pragma unroll
      for (int u = 0; u < PB; ++u)
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
          lbc[u][s] = lbn[u][s];
          lbn[u][s] = (act[s] && tb + PB + u < T) ? pL[(int64_t)u * K + NT * s] : N::ninf();
        }
#pragma unroll
      for (int u = 0; u < PB; ++u) {
        const int t = tb + u;
        if (t >= T) break;
        R uu[SPL];
        R M = N::ninf();
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
          const R acc = dot(s);
          const R la_ = t == 0 ? lpi[s] : (acc > R(0) ? N::flog(acc) : N::ninf());
          uu[s] = act[s] ? la_ + lbc[u][s] : N::ninf();
          M = rmax(M, uu[s]);
        }
        if (hasA) {
#pragma unroll
          for (int s = 0; s < SPL; ++s)
            if (act[s]) pA[NT * s] = lamf + uu[s];
          pA += K;
        }
        M = all_max(M);
        if (!(M > N::ninf())) {  // rare: a dead observation (every log b is -inf)?
          R mlb = N::ninf();
#pragma unroll
          for (int s = 0; s < SPL; ++s) mlb = rmax(mlb, lbc[u][s]);
          mlb = all_max(mlb);
          if (!(mlb > N::ninf()) && t < dead_t) dead_t = t;
        } else {
          lam += (double)M;
          lamf = (R)lam;
        }
        if constexpr (NW == 1) __syncwarp();  // (NW > 1: all_max's barrier already ordered the reads of av)
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
          a_j[s] = (M > N::ninf()) ? N::fexp(uu[s] - M) : R(0);
          if (act[s]) {
            av[js[s]] = a_j[s];
            pW[NT * s] = a_j[s];
          }
        }
        pW += K;
        sync();
      }
    }
    R sm = R(0);
#pragma unroll
    for (int s = 0; s < SPL; ++s) sm += act[s] ? a_j[s] : R(0);
    sm = all_sum(sm);
    const double LL = sm > R(0) ? lam + (double)N::flog(sm) : -CUDART_INF;
    if (lane == 0) {
      a.ll[b] = LL;
      if (a.flags) {
        a.flags[2 * b] = dead_t == INT_MAX ? -1 : dead_t;
        a.flags[2 * b + 1] = nan_seen ? 1 : 0;
      }
    }
    return;
  }

  // backward sweep: beta~ (qws), w_t = b~_t beta~_t scaled to max 1 (wws), log beta
  const bool hasB = a.log_beta != nullptr;
  const int64_t last = (int64_t)(T - 1) * K;
  R* pB = hasB ? reinterpret_cast<R*>(a.log_beta) + start * K + j0 + last : nullptr;
  R* pQ = reinterpret_cast<R*>(sw.qws) + start * K + j0 + last;
  R* pW = reinterpret_cast<R*>(sw.wws) + start * K + j0 + last;
  const R* pL = lbws + start * K + j0 + last;
  R r[SPL];
#pragma unroll
  for (int s = 0; s < SPL; ++s) r[s] = R(0);
  double rho = 0.0;
  R rhof = R(0);
  R lbn[PB][SPL];
#pragma unroll
  for (int u = 0; u < PB; ++u)
#pragma unroll
    for (int s = 0; s < SPL; ++s)
      lbn[u][s] = (act[s] && T - 1 - u >= 0) ? pL[-(int64_t)u * K + NT * s] : N::ninf();
  for (int tb = T - 1; tb >= 0; tb -= PB) {
    R lbc[PB][SPL];
    pL -= (int64_t)PB * K;
#pragma unroll
    for (int u = 0; u < PB; ++u)
#pragma unroll
      for (int s = 0; s < SPL; ++s) {
        lbc[u][s] = lbn[u][s];
        lbn[u][s] = (act[s] && tb - PB - u >= 0) ? pL[-(int64_t)u * K + NT * s] : N::ninf();
      }
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      const int t = tb - u;
      if (t < 0) break;
#pragma unroll
      for (int s = 0; s < SPL; ++s)
        if (act[s]) {
          if (hasB) pB[NT * s] = rhof + r[s];
          pQ[NT * s] = N::fexp(r[s]);
        }
      if (hasB) pB -= K;
      pQ -= K;
      if (t == 0) break;
      R lr[SPL];
      R M = N::ninf();
#pragma unroll
      for (int s = 0; s < SPL; ++s) {
        lr[s] = act[s] ? lbc[u][s] + r[s] : N::ninf();
        M = rmax(M, lr[s]);
      }
      M = all_max(M);
      const bool fin = M > N::ninf();
      if constexpr (NW == 1) __syncwarp();
#pragma unroll
      for (int s = 0; s < SPL; ++s) {
        const R w = fin ? N::fexp(lr[s] - M) : R(0);
        if (act[s]) {
          av[js[s]] = w;
          pW[NT * s] = w;
        }
      }
      pW -= K;
      sync();
      if (fin) {
        rho += (double)M;
        rhof = (R)rho;
      }
#pragma unroll
      for (int s = 0; s < SPL; ++s) {
        const R acc = dot(s);
        r[s] = (act[s] && acc > R(0)) ? N::flog(acc) : N::ninf();
      }
    }
  }
}

// the smallest instantiated non-zero budget that covers maxnz
template <typename R, int KM, int NW>
__device__ __forceinline__ void fb_sparse_sweep_nz(const FBArgs& a, int K, const R* __restrict__ lbws,
                                                   const SplitWs& sw, R* av, R* red, bool bwd, int64_t b,
                                                   int maxnz) {
  if (maxnz <= 5) fb_sparse_sweep<R, KM, 5, NW>(a, K, lbws, sw, av, red, bwd, b);
  else if (maxnz <= 9) fb_sparse_sweep<R, KM, 9, NW>(a, K, lbws, sw, av, red, bwd, b);
  else fb_sparse_sweep<R, KM, kSweepNZ, NW>(a, K, lbws, sw, av, red, bwd, b);
}

template <typename R, int KM, int P>
__global__ void __launch_bounds__(256) fb_split_sweep_kernel(const FBArgs a, int K,
                                                             const R* __restrict__ lbws,
                                                             const SplitWs sw) {
  typedef Num<R> N;
  typedef Quarter<R, KM, P> Q;
  constexpr int NQ = Q::NQ;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* av = reinterpret_cast<R*>(smem_raw);  // KM
  R* red = av + KM;                         // 128
  R* ring = red + 128 + KM;                 // [kRing][4][KM]
  const int tid = threadIdx.x;
  const int nw = blockDim.x >> 5;
  const int q = tid & (P - 1);
  const int jt = tid / P;
  const bool bwd = blockIdx.x >= a.B;
  const int64_t b = bwd ? blockIdx.x - a.B : blockIdx.x;
  // structural sparsity of A: the largest number of non-zeros of a column
  // (forward) or row (backward)
  __shared__ int s_maxnz;
  if (tid == 0) s_maxnz = 0;
  __syncthreads();
  if (tid < K) {
    int cnt = 0;
    for (int i = 0; i < K; ++i) cnt += (bwd ? a.model->A[tid * K + i] : a.model->A[i * K + tid]) > 0.0 ? 1 : 0;
    atomicMax(&s_maxnz, cnt);
  }
  __syncthreads();
  if (s_maxnz <= kSweepNZ && sw.sparse_ok) {
    // warps per sequence and direction: one state per lane at K = 64 when
    // sw.sparse_warps = 2 (fp64 always: one lane cannot hide the software
    // exp / log chains of two states)
    constexpr bool kCanTwo = KM == 64;
    const bool two_warps = kCanTwo && (sizeof(R) == 8 || sw.sparse_warps == 2);
    if (tid >= (two_warps ? 64 : 32)) return;
    if constexpr (kCanTwo) {
      if (two_warps) {
        fb_sparse_sweep_nz<R, KM, 2>(a, K, lbws, sw, av, red, bwd, b, s_maxnz);
        return;
      }
    }
    fb_sparse_sweep_nz<R, KM, 1>(a, K, lbws, sw, av, red, bwd, b, s_maxnz);
    return;
  }
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const bool act = jt < K;
  const bool lead = act && q == 0;
  const int j = act ? jt : 0;
  const loghmm_model_t* md = a.model;
  // column j of A (forward) or row j of A (backward), this lane's elements
  R Am[NQ];
#pragma unroll
  for (int s = 0; s < NQ; ++s) {
    const int i = Q::idx(q, s);
    Am[s] = (act && i < K) ? (R)(bwd ? md->A[j * K + i] : md->A[i * K + j]) : R(0);
  }
  if (tid < KM) av[tid] = R(0);
  const R* y0g = reinterpret_cast<const R*>(a.y0) + start;
  const bool two = a.n_streams > 1;
  const R* y1g = two ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
  R* aws = reinterpret_cast<R*>(a.alpha_ws) + start * K;
  const R* __restrict__ lbs = lbws + start * K;
  __syncthreads();
  auto issue = [&](int t, int pos) {
    if (lead) {
      const bool ok = t >= 0 && t < T;
      const int tc = ok ? t : 0;
      R* sl = ring + (size_t)(pos % kRing) * 4 * KM;
      cp_async<sizeof(R)>(sl + j, lbs + (int64_t)tc * K + j, ok);
      if (!bwd) {
        cp_async<sizeof(R)>(sl + KM + j, y0g + tc, ok);
        if (two) cp_async<sizeof(R)>(sl + 2 * KM + j, y1g + tc, ok);
      }
    }
    cp_async_commit();
  };
  BRed<R> br(red, nw);
#pragma unroll 1
  for (int d = 0; d < kRing - 1; ++d) issue(bwd ? T - 1 - d : d, d);

  if (!bwd) {
    R* outA = a.log_alpha ? reinterpret_cast<R*>(a.log_alpha) + start * K : nullptr;
    const R lpi = (R)md->log_pi[j];
    bool nan_seen = false;
    int dead_t = INT_MAX;
    double lam = 0.0;
    R a_j = R(0);
    for (int t = 0; t < T; ++t) {
      issue(t + kRing - 1, t + kRing - 1);
      cp_async_wait<kRing - 1>();
      const R* sl = ring + (size_t)(t % kRing) * 4 * KM;
      const R lb = lead ? sl[j] : N::ninf();
      if (lead && (isnan(sl[KM + j]) || (two && isnan(sl[2 * KM + j])))) nan_seen = true;
      R u;
      if (t == 0) {
        u = lpi + lb;
      } else {
        const R acc = Q::dot(Am, av, q);
        u = (acc > R(0) ? N::flog(acc) : N::ninf()) + lb;
      }
      if (lead && outA) outA[(int64_t)t * K + j] = (R)lam + u;
      R M = lead ? u : N::ninf(), mlb = lb;
      br.two<true>(M, mlb);
      if (!(mlb > N::ninf()) && t < dead_t) dead_t = t;
      a_j = (M > N::ninf()) ? N::fexp(u - M) : R(0);
      if (M > N::ninf()) lam += (double)M;
      if (lead) {
        av[j] = a_j;
        aws[(int64_t)t * K + j] = a_j;
      }
      __syncthreads();
    }
    cp_async_wait_all();
    const R s = block_sum(lead ? a_j : R(0), red, nw);
    const double LL = s > R(0) ? lam + (double)N::flog(s) : -CUDART_INF;
    __shared__ int s_dead, s_nan;
    if (tid == 0) {
      s_dead = INT_MAX;
      s_nan = 0;
    }
    __syncthreads();
    if (dead_t != INT_MAX) atomicMin(&s_dead, dead_t);
    if (nan_seen) s_nan = 1;
    __syncthreads();
    if (tid == 0) {
      a.ll[b] = LL;
      if (a.flags) {
        a.flags[2 * b] = s_dead == INT_MAX ? -1 : s_dead;
        a.flags[2 * b + 1] = s_nan ? 1 : 0;
      }
    }
    return;
  }

  // backward sweep: beta~ and w only
  R* outB = a.log_beta ? reinterpret_cast<R*>(a.log_beta) + start * K : nullptr;
  R* qws = reinterpret_cast<R*>(sw.qws) + start * K;
  R* wws = reinterpret_cast<R*>(sw.wws) + start * K;
  R r = R(0);
  double rho = 0.0;
  for (int t = T - 1; t >= 0; --t) {
    const int p = T - 1 - t;
    issue(t - (kRing - 1), p + kRing - 1);
    cp_async_wait<kRing - 1>();
    const R* sl = ring + (size_t)(p % kRing) * 4 * KM;
    const R lb = lead ? sl[j] : N::ninf();
    if (lead) {
      if (outB) outB[(int64_t)t * K + j] = (R)rho + r;
      qws[(int64_t)t * K + j] = N::fexp(r);
    }
    if (t == 0) break;
    R M = lead ? lb + r : N::ninf(), dummy = R(0);
    br.two<true>(M, dummy);
    const bool fin = M > N::ninf();
    const R w = (lead && fin) ? N::fexp(lb + r - M) : R(0);
    if (lead) {
      av[j] = w;
      wws[(int64_t)t * K + j] = w;
    }
    __syncthreads();
    R acc = Q::dot(Am, av, q);
    acc = act ? acc : R(0);
    const R lq = acc > R(0) ? N::flog(acc) : N::ninf();
    R mq = act ? lq : N::ninf(), dummy2 = R(0);
    br.two<true>(mq, dummy2);
    if (mq > N::ninf()) {
      r = lq - mq;
      rho += (fin ? (double)M : 0.0) + (double)mq;
    }
  }
  cp_async_wait_all();
}

template <typename R>
struct PostGeom {
  static constexpr int H = 1;                               // CTAs per segment
  static constexpr int PITCH = 64 + 16 / (int)sizeof(R);    // padded A row (elements)
  static constexpr int TC = 32;                             // steps per tile chunk
  static constexpr size_t smem() {
    return (size_t)(64 * PITCH + kPostWarps * 64 + 2 * TC * 64) * sizeof(R) +
           (size_t)(2 * 64 * LOGHMM_NSLOT + 2 * 64) * sizeof(double);
  }
};

template <typename R>
__device__ __forceinline__ R row_dot64(const R* __restrict__ row, const R* __restrict__ v) {
  R c[4] = {R(0), R(0), R(0), R(0)};
  if constexpr (sizeof(R) == 4) {
#pragma unroll
    for (int i = 0; i < 64; i += 4) {
      const float4 m = *reinterpret_cast<const float4*>(row + i);
      const float4 x = *reinterpret_cast<const float4*>(v + i);
      c[0] = fma(m.x, x.x, c[0]);
      c[1] = fma(m.y, x.y, c[1]);
      c[2] = fma(m.z, x.z, c[2]);
      c[3] = fma(m.w, x.w, c[3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 64; i += 2) {
      const double2 m = *reinterpret_cast<const double2*>(row + i);
      const double2 x = *reinterpret_cast<const double2*>(v + i);
      c[(i >> 1) & 3] = fma(m.x, x.x, c[(i >> 1) & 3]);
      c[((i >> 1) + 2) & 3] = fma(m.y, x.y, c[((i >> 1) + 2) & 3]);
    }
  }
  return (c[0] + c[1]) + (c[2] + c[3]);
}

// Largest number of non-zeros of a row of A (counted by the CTA's first K
// threads): both post kernels below evaluate it, exactly one of them runs.
__device__ __forceinline__ int cta_row_maxnz(const loghmm_model_t* md, int K, int* s_val) {
  if (threadIdx.x == 0) *s_val = 0;
  __syncthreads();
  if ((int)threadIdx.x < K) {
    int cnt = 0;
    for (int i = 0; i < K; ++i) cnt += md->A[threadIdx.x * K + i] > 0.0 ? 1 : 0;
    atomicMax(s_val, cnt);
  }
  __syncthreads();
  return *s_val;
}
constexpr int kPostNZ = 12;
__device__ __forceinline__ bool post_takes_sparse(const FBArgs& a, const SplitWs& sw, int maxnz) {
  return sw.sparse_ok && a.xi == nullptr && maxnz <= kPostNZ;
}

// T-parallel pass: CTA (seg, b) takes steps [seg*len, (seg+1)*len) of
// sequence b in chunks of TC steps.  Phase 1, one warp per step (lane l owns
// states l and l + 32): gamma_t and the statistics, and for xi the row
// alpha~_{t-1}/Z_t and w_t into two [TC][64] shared tiles, Z_t =
// alpha~_{t-1}^T A w_t.  Phase 2: the CTA accumulates the 64x64 xi outer
// products of the chunk as a tiled rank-TC update (4x4 register tile per
// thread).  The statistics are folded over the warps in fixed order; each
// CTA writes one segment row, fb_fold_kernel sums the segment rows in order.
template <typename R>
__global__ void __launch_bounds__(256, sizeof(R) == 4 ? 2 : 1) fb_post_kernel(const FBArgs a, int K, const SplitWs sw) {
  typedef Num<R> N;
  typedef PostGeom<R> PG;
  constexpr int PITCH = PG::PITCH;
  constexpr int TC = PG::TC;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* As = reinterpret_cast<R*>(smem_raw);  // [64][PITCH] A rows
  R* wv = As + 64 * PITCH;                 // [warps][64] w_t
  R* Ta = wv + kPostWarps * 64;            // [TC][64] alpha~_{t-1} / Z_t
  R* Tw = Ta + TC * 64;                    // [TC][64] w_t
  double* sts = reinterpret_cast<double*>(Tw + TC * 64);  // [2][64][NSLOT] + [2][64]
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const loghmm_model_t* md = a.model;
  __shared__ int s_maxnz;
  if (post_takes_sparse(a, sw, cta_row_maxnz(md, K, &s_maxnz))) return;  // fb_post_sparse_kernel's launch
  const int64_t b = blockIdx.y;
  const int seg = blockIdx.x;
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const int len = (T + kPostSegs - 1) / kPostSegs;
  const int t0 = seg * len, t1 = min(T, t0 + len);
  for (int e = tid; e < 64 * 64; e += blockDim.x) {
    const int r = e >> 6, c = e & 63;
    As[r * PITCH + c] = (r < K && c < K) ? (R)md->A[r * K + c] : R(0);
  }
  const bool two = a.n_streams > 1;
  int is[2];
  bool act[2];
  EmP<R> p0[2], p1[2];
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    is[s] = lane + 32 * s;
    act[s] = is[s] < K;
    const int ii = act[s] ? is[s] : 0;
    p0[s] = load_emission<R>(md->em[0][ii]);
    if (two) p1[s] = load_emission<R>(md->em[1][ii]);
    else p1[s].fam = LOGHMM_FAM_NONE;
  }
  const R* y0g = reinterpret_cast<const R*>(a.y0) + start;
  const R* y1g = two ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
  const R* aws = reinterpret_cast<const R*>(a.alpha_ws) + start * K;
  const R* qws = reinterpret_cast<const R*>(sw.qws) + start * K;
  const R* wws = reinterpret_cast<const R*>(sw.wws) + start * K;
  R* outG = a.gamma ? reinterpret_cast<R*>(a.gamma) + start * K : nullptr;
  R* outX = a.xi ? reinterpret_cast<R*>(a.xi) + (start - b) * (int64_t)K * K : nullptr;
  // phase-2 tile: rows 4*ti .. 4*ti+3, columns 4*tj .. 4*tj+3
  const int ti = tid >> 4, tj = tid & 15;
  R X[4][4];
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) X[r][c] = R(0);
  R st[2][2][LOGHMM_NSLOT];
  R gtot[2] = {R(0), R(0)}, g0[2] = {R(0), R(0)};
#pragma unroll
  for (int s = 0; s < 2; ++s)
    for (int v = 0; v < 2; ++v)
      for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) st[s][v][qq] = R(0);
  R* mw = wv + wid * 64;
  bool range_bad = false;  // alpha~ . beta~ or alpha~^T A w underflowed (see the flag word, bit 2)
  __syncthreads();
  for (int c0 = t0; c0 < t1; c0 += TC) {
    for (int tt = wid; tt < TC; tt += kPostWarps) {
      const int t = c0 + tt;
      R* ta = Ta + tt * 64;
      R* tw = Tw + tt * 64;
      if (t >= t1) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          ta[is[s]] = R(0);
          tw[is[s]] = R(0);
        }
        continue;
      }
      {
        R at[2], qe[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          at[s] = act[s] ? aws[(int64_t)t * K + is[s]] : R(0);
          qe[s] = act[s] ? qws[(int64_t)t * K + is[s]] : R(0);
        }
        const R gz = warp_sum(at[0] * qe[0] + at[1] * qe[1]);
        range_bad |= !(gz > R(0));
        const R yv0 = y0g[t], yv1 = two ? y1g[t] : R(0);
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (!act[s]) continue;
          const R gj = at[s] * qe[s] / gz;
          if (outG) outG[(int64_t)t * K + is[s]] = gj;
          ObsFeat<R> f0, f1;
          stat_features<R>(f0, yv0, p0[s].fam);
          if (two) stat_features<R>(f1, yv1, p1[s].fam);
          R accs[LOGHMM_NSLOT];
          for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) accs[qq] = st[s][0][qq];
          stat_acc_rt<R>(accs, gj, p0[s], f0);
          for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) st[s][0][qq] = accs[qq];
          if (two) {
            for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) accs[qq] = st[s][1][qq];
            stat_acc_rt<R>(accs, gj, p1[s], f1);
            for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) st[s][1][qq] = accs[qq];
          }
          if (t < T - 1) gtot[s] += gj;
          if (t == 0) g0[s] = gj;
        }
      }
      if (t == 0) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          ta[is[s]] = R(0);
          tw[is[s]] = R(0);
        }
        continue;
      }
      // xi_{t-1}: q_i = (A w_t)_i, Z = alpha~_{t-1} . q over all rows
      R ap[2], qv[2], wj[2];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        ap[s] = act[s] ? aws[(int64_t)(t - 1) * K + is[s]] : R(0);
        wj[s] = act[s] ? wws[(int64_t)t * K + is[s]] : R(0);
        mw[is[s]] = wj[s];
      }
      __syncwarp();
#pragma unroll
      for (int s = 0; s < 2; ++s) qv[s] = row_dot64<R>(As + is[s] * PITCH, mw);
      const R Z = warp_sum(ap[0] * qv[0] + ap[1] * qv[1]);
      range_bad |= !(Z > R(0));
      const R iz = R(1) / Z;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        ta[is[s]] = ap[s] * iz;
        tw[is[s]] = wj[s];
      }
      if (outX) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
          if (!act[s]) continue;
          for (int jj = 0; jj < K; ++jj)
            outX[((int64_t)(t - 1) * K + is[s]) * K + jj] = ap[s] * iz * As[is[s] * PITCH + jj] * mw[jj];
        }
      }
      __syncwarp();
    }
    __syncthreads();
    // phase 2: X[i][j] += sum_tt Ta[tt][i] Tw[tt][j]
#pragma unroll 4
    for (int tt = 0; tt < TC; ++tt) {
      R av4[4], wv4[4];
      if constexpr (sizeof(R) == 4) {
        const float4 x = *reinterpret_cast<const float4*>(Ta + tt * 64 + 4 * ti);
        const float4 y = *reinterpret_cast<const float4*>(Tw + tt * 64 + 4 * tj);
        av4[0] = x.x; av4[1] = x.y; av4[2] = x.z; av4[3] = x.w;
        wv4[0] = y.x; wv4[1] = y.y; wv4[2] = y.z; wv4[3] = y.w;
      } else {
#pragma unroll
        for (int k = 0; k < 4; k += 2) {
          const double2 x = *reinterpret_cast<const double2*>(Ta + tt * 64 + 4 * ti + k);
          const double2 y = *reinterpret_cast<const double2*>(Tw + tt * 64 + 4 * tj + k);
          av4[k] = x.x; av4[k + 1] = x.y;
          wv4[k] = y.x; wv4[k + 1] = y.y;
        }
      }
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) X[r][c] = fma(av4[r], wv4[c], X[r][c]);
    }
    __syncthreads();
  }
  if (range_bad && lane == 0 && a.flags && isfinite(a.ll[b]))
    atomicOr(reinterpret_cast<unsigned long long*>(a.flags + 2 * b + 1), 4ull);
  // fold the statistics over the warps in order
  double* gts = sts + 2 * 64 * LOGHMM_NSLOT;  // [2][64]: gamma totals, first gamma
  for (int e = tid; e < 2 * 64 * LOGHMM_NSLOT + 2 * 64; e += blockDim.x) sts[e] = 0.0;
  __syncthreads();
  for (int w = 0; w < kPostWarps; ++w) {
    if (wid == w) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        for (int v = 0; v < 2; ++v)
          for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) sts[(v * 64 + is[s]) * LOGHMM_NSLOT + qq] += (double)st[s][v][qq];
        gts[is[s]] += (double)gtot[s];
        gts[64 + is[s]] += (double)g0[s];
      }
    }
    __syncthreads();
  }
  double* row = sw.seg_part + ((int64_t)b * kPostSegs + seg) * a.stats_width;
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int i = 4 * ti + r, jj = 4 * tj + c;
      if (i < K && jj < K) row[i * K + jj] = (double)X[r][c];
    }
  for (int jj = tid; jj < K; jj += blockDim.x) {
    row[K * K + jj] = gts[jj];
    row[K * K + K + jj] = gts[64 + jj];
    for (int v = 0; v < 2; ++v)
      for (int qq = 0; qq < LOGHMM_NSLOT; ++qq)
        row[K * K + 2 * K + (v * K + jj) * LOGHMM_NSLOT + qq] = sts[(v * 64 + jj) * LOGHMM_NSLOT + qq];
  }
}

// T-parallel pass for a structurally sparse A (config 5's band): same segment
// decomposition and statistics as fb_post_kernel, but a zero A_ij carries no
// xi mass, so lane i keeps only the xi sums of its row's non-zero targets in
// registers (no shared tiles, no rank-TC phase) and q = A w is a sparse dot.
template <typename R, int NZ>
__global__ void __launch_bounds__(256, 2) fb_post_sparse_kernel(const FBArgs a, int K, const SplitWs sw) {
  typedef Num<R> N;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* wv = reinterpret_cast<R*>(smem_raw);                               // [warps][64] w_t
  double* sts = reinterpret_cast<double*>(wv + kPostWarps * 64);        // [2][64][NSLOT] + [2][64]
  double* xfold = sts + 2 * 64 * LOGHMM_NSLOT + 2 * 64;                 // [64][NZ]
  __shared__ int s_maxnz;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const loghmm_model_t* md = a.model;
  const int maxnz = cta_row_maxnz(md, K, &s_maxnz);
  if (!post_takes_sparse(a, sw, maxnz) || maxnz > NZ || (NZ > 5 && maxnz <= 5) || (NZ > 9 && maxnz <= 9)) return;
  const int64_t b = blockIdx.y;
  const int seg = blockIdx.x;
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const int len = (T + kPostSegs - 1) / kPostSegs;
  const int t0 = seg * len, t1 = min(T, t0 + len);
  const bool two = a.n_streams > 1;
  int is[2];
  bool act[2];
  EmP<R> p0[2], p1[2];
  int tgt[2][NZ];
  R Ar[2][NZ], xs[2][NZ];
  R* mw = wv + wid * 64;
#pragma unroll
  for (int s = 0; s < 2; ++s) {
    is[s] = lane + 32 * s;
    act[s] = is[s] < K;
    const int ii = act[s] ? is[s] : 0;
    p0[s] = load_emission<R>(md->em[0][ii]);
    if (two) p1[s] = load_emission<R>(md->em[1][ii]);
    else p1[s].fam = LOGHMM_FAM_NONE;
#pragma unroll
    for (int n = 0; n < NZ; ++n) {
      tgt[s][n] = 0;
      Ar[s][n] = R(0);
      xs[s][n] = R(0);
    }
    int cnt = 0;
    for (int jj = 0; jj < K; ++jj) {
      const R v = (R)md->A[ii * K + jj];
      if (act[s] && v > R(0)) {
#pragma unroll
        for (int n = 0; n < NZ; ++n)
          if (n == cnt) {
            tgt[s][n] = jj;
            Ar[s][n] = v;
          }
        ++cnt;
      }
    }
  }
  const R* y0g = reinterpret_cast<const R*>(a.y0) + start;
  const R* y1g = two ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
  const R* aws = reinterpret_cast<const R*>(a.alpha_ws) + start * K;
  const R* qws = reinterpret_cast<const R*>(sw.qws) + start * K;
  const R* wws = reinterpret_cast<const R*>(sw.wws) + start * K;
  R* outG = a.gamma ? reinterpret_cast<R*>(a.gamma) + start * K : nullptr;
  R st[2][2][LOGHMM_NSLOT];
  R gtot[2] = {R(0), R(0)}, g0[2] = {R(0), R(0)};
#pragma unroll
  for (int s = 0; s < 2; ++s)
#pragma unroll
    for (int v = 0; v < 2; ++v)
#pragma unroll
      for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) st[s][v][qq] = R(0);
  bool range_bad = false;  // alpha~ . beta~ or alpha~^T A w underflowed (flag word, bit 2)
  // this step's inputs are loaded one step ahead (the next step's loads are in
  // flight while the current one is reduced)
  R nat[2], nqe[2], nap[2], nwj[2], ny0 = R(0), ny1 = R(0);
  auto fetch = [&](int t) {
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const bool ok = act[s] && t < t1;
      nat[s] = ok ? aws[(int64_t)t * K + is[s]] : R(0);
      nqe[s] = ok ? qws[(int64_t)t * K + is[s]] : R(0);
      nap[s] = (ok && t >= 1) ? aws[(int64_t)(t - 1) * K + is[s]] : R(0);
      nwj[s] = (ok && t >= 1) ? wws[(int64_t)t * K + is[s]] : R(0);
    }
    ny0 = t < t1 ? y0g[t] : R(0);
    ny1 = (two && t < t1) ? y1g[t] : R(0);
  };
  fetch(t0 + wid);
  for (int t = t0 + wid; t < t1; t += kPostWarps) {
    R at[2], qe[2], ap[2], wj[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      at[s] = nat[s];
      qe[s] = nqe[s];
      ap[s] = nap[s];
      wj[s] = nwj[s];
    }
    const R yv0 = ny0, yv1 = ny1;
    fetch(t + kPostWarps);
    const R gz = warp_sum(at[0] * qe[0] + at[1] * qe[1]);
    range_bad |= !(gz > R(0));
    const R igz = R(1) / gz;  // one division per step (posteriors stay within 1 ulp of a per-state division)
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      if (!act[s]) continue;
      const R gj = at[s] * qe[s] * igz;
      if (outG) outG[(int64_t)t * K + is[s]] = gj;
      ObsFeat<R> f0, f1;
      stat_features<R>(f0, yv0, p0[s].fam);
      if (two) stat_features<R>(f1, yv1, p1[s].fam);
      stat_acc_rt<R>(st[s][0], gj, p0[s], f0);
      if (two) stat_acc_rt<R>(st[s][1], gj, p1[s], f1);
      if (t < T - 1) gtot[s] += gj;
      if (t == 0) g0[s] = gj;
    }
    if (t == 0) continue;
    // xi_{t-1}: q_i = (A w_t)_i over the row's non-zeros, Z = alpha~_{t-1} . q
    __syncwarp();
#pragma unroll
    for (int s = 0; s < 2; ++s)
      if (act[s]) mw[is[s]] = wj[s];
    __syncwarp();
    R qv[2];
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      R acc = R(0);
#pragma unroll
      for (int n = 0; n < NZ; ++n) acc = fma(Ar[s][n], mw[tgt[s][n]], acc);
      qv[s] = acc;
    }
    const R Z = warp_sum(ap[0] * qv[0] + ap[1] * qv[1]);
    range_bad |= !(Z > R(0));
    const R iz = R(1) / Z;
#pragma unroll
    for (int s = 0; s < 2; ++s) {
      const R ta = ap[s] * iz;
#pragma unroll
      for (int n = 0; n < NZ; ++n) xs[s][n] = fma(ta, mw[tgt[s][n]], xs[s][n]);
    }
  }
  if (range_bad && lane == 0 && a.flags && isfinite(a.ll[b]))
    atomicOr(reinterpret_cast<unsigned long long*>(a.flags + 2 * b + 1), 4ull);
  // fold the statistics and the xi sums over the warps in order
  double* gts = sts + 2 * 64 * LOGHMM_NSLOT;  // [2][64]: gamma totals, first gamma
  for (int e = tid; e < 2 * 64 * LOGHMM_NSLOT + 2 * 64 + 64 * NZ; e += blockDim.x) sts[e] = 0.0;
  __syncthreads();
  for (int w = 0; w < kPostWarps; ++w) {
    if (wid == w) {
#pragma unroll
      for (int s = 0; s < 2; ++s) {
#pragma unroll
        for (int v = 0; v < 2; ++v)
#pragma unroll
          for (int qq = 0; qq < LOGHMM_NSLOT; ++qq) sts[(v * 64 + is[s]) * LOGHMM_NSLOT + qq] += (double)st[s][v][qq];
        gts[is[s]] += (double)gtot[s];
        gts[64 + is[s]] += (double)g0[s];
#pragma unroll
        for (int n = 0; n < NZ; ++n) xfold[is[s] * NZ + n] += (double)xs[s][n];
      }
    }
    __syncthreads();
  }
  double* row = sw.seg_part + ((int64_t)b * kPostSegs + seg) * a.stats_width;
  for (int e = tid; e < K * K; e += blockDim.x) row[e] = 0.0;
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int s = 0; s < 2; ++s)
      if (act[s]) {
#pragma unroll
        for (int n = 0; n < NZ; ++n)
          if (Ar[s][n] > R(0)) row[is[s] * K + tgt[s][n]] = xfold[is[s] * NZ + n];
      }
  }
  for (int jj = tid; jj < K; jj += blockDim.x) {
    row[K * K + jj] = gts[jj];
    row[K * K + K + jj] = gts[64 + jj];
    for (int v = 0; v < 2; ++v)
      for (int qq = 0; qq < LOGHMM_NSLOT; ++qq)
        row[K * K + 2 * K + (v * K + jj) * LOGHMM_NSLOT + qq] = sts[(v * 64 + jj) * LOGHMM_NSLOT + qq];
  }
}

// partials[b, c] = sum over segments (in order) of seg_part[b, seg, c]; the
// xi columns are then multiplied by A_ij (as in the fused kernel)
__global__ void __launch_bounds__(256) fb_fold_kernel(const FBArgs a, int K, const SplitWs sw) {
  const int64_t b = blockIdx.x;
  const double* src = sw.seg_part + b * kPostSegs * a.stats_width;
  double* row = a.partials + b * a.stats_width;
  for (int64_t c = threadIdx.x; c < a.stats_width; c += blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < kPostSegs; ++s) acc += src[(int64_t)s * a.stats_width + c];
    if (c < (int64_t)K * K) acc *= a.model->A[c];
    row[c] = acc;
  }
}

// Structural zeros (config 5: a banded transition matrix).  A candidate through
// log A[i][j] = -inf is -inf whatever the score, so it can only be the argmax
// when every candidate of the column is -inf — and then numpy's argmax returns
// index 0.  Restricting column j to its finite sources (ascending i, so the
// first-index rule is kept) and mapping an all -inf column to index 0 is
// therefore bit-identical to the dense recursion (inference.py:204-207).
constexpr int kVitNZ = 12;  // finite sources per column the sparse path covers

// One lane per state, KM / 32 warps per sequence (the other warps of the CTA
// have exited).  Every lane keeps its column's source offsets and log A values
// in registers, forms the <= kVitNZ candidates from the shared score vector and
// reduces them with a first-index (value, index) tree.
// Backtrace over the byte backpointer table bk [T][K] (global workspace), in
// blocks of kBtBlk rows walking down: the block's rows are copied to shared
// memory with 16-byte loads (8 in flight per thread; byte loads when K is not
// a multiple of 16), thread 0 follows the chain through shared memory into a
// byte stage, and all threads write the int64 path coalesced.
constexpr int kBtBlk = 256;
template <typename SyncF>
__device__ __forceinline__ void backtrace_blocks(const uint8_t* __restrict__ bk, int K, int T,
                                                 int64_t* __restrict__ path, uint8_t* bblk,
                                                 uint8_t* pstage, int* s_cur, int tid, int nt,
                                                 SyncF sync) {
  for (int hi = T - 1; hi >= 0; hi -= kBtBlk) {
    const int lo = max(0, hi - kBtBlk + 1);
    const int rows = hi - lo + 1;
    const int nbytes = rows * K;
    const uint8_t* src = bk + (int64_t)lo * K;
    if ((K & 15) == 0) {
      const uint4* s4 = reinterpret_cast<const uint4*>(src);
      uint4* d4 = reinterpret_cast<uint4*>(bblk);
      const int n4 = nbytes >> 4;
      for (int e0 = tid; e0 < n4; e0 += 8 * nt) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u * nt < n4) v[u] = s4[e0 + u * nt];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u * nt < n4) d4[e0 + u * nt] = v[u];
      }
    } else {
      for (int e0 = tid; e0 < nbytes; e0 += 8 * nt) {
        uint8_t v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u * nt < nbytes) v[u] = src[e0 + u * nt];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (e0 + u * nt < nbytes) bblk[e0 + u * nt] = v[u];
      }
    }
    sync();
    if (tid == 0) {
      int c = *s_cur;
      for (int t = hi; t >= lo; --t) {
        pstage[t - lo] = (uint8_t)c;
        if (t >= 1) c = bblk[(t - lo) * K + c];
      }
      *s_cur = c;
    }
    sync();
    for (int e = tid; e < rows; e += nt) path[lo + e] = (int64_t)pstage[e];
    sync();
  }
}

constexpr int kVitPB = 16;  // steps of precomputed log b fetched ahead per block

template <typename R, int KM, int NZ>
__device__ __forceinline__ void viterbi_sparse_path(const VitArgs& a, int K, uint8_t* backws,
                                                    const R* __restrict__ lbws, R* dvb, uint8_t* bblk,
                                                    int* s_cur) {
  typedef Num<R> N;
  constexpr int PB = kVitPB;
  static_assert(PB % 2 == 0, "the score buffers alternate with the step parity");
  constexpr int NT = KM < 32 ? 32 : KM;  // threads taking part
  const int tid = threadIdx.x;
  const int64_t b = blockIdx.x;
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const bool act = tid < K;
  const int j = act ? tid : 0;
  const loghmm_model_t* md = a.model;
  int off[NZ];
  const R* src[NZ];  // &scores[source] in buffer 0 (buffer 1 is KM elements further)
  R lav[NZ];
#pragma unroll
  for (int n = 0; n < NZ; ++n) {
    off[n] = 0;
    src[n] = dvb;
    lav[n] = N::ninf();
  }
  {
    int cnt = 0;
    for (int i = 0; i < K; ++i) {
      const R v = (R)md->log_A[i * K + j];
      if (act && v > N::ninf()) {
#pragma unroll
        for (int n = 0; n < NZ; ++n)
          if (n == cnt) {
            off[n] = i;
            src[n] = dvb + i;
            lav[n] = v;
          }
        ++cnt;
      }
    }
  }
  const R* __restrict__ pL = lbws + start * K + j;  // log b_t[j], running row pointer
  uint8_t* bk = backws + start * K;
  auto sync = [&]() {
    if constexpr (NT == 32) __syncwarp();
    else named_bar_sync(1, NT);
  };
  for (int e = tid; e < 2 * KM; e += NT) dvb[e] = N::ninf();
  sync();
  if (act && T > 0) {
    dvb[j] = N::add((R)md->log_pi[j], pL[0]);
    bk[j] = 0;
    if (a.back) a.back[start * K + j] = 0;
  }
  sync();
  uint8_t* pK = bk + K + j;                                            // backpointer row of step 1
  uint8_t* pX = a.back ? a.back + (start + 1) * K + j : nullptr;       // optional byte table (tests)
  R* const mine = dvb + j;
  pL += K;
  R lbn[PB];  // the next block's emission terms, loaded a block ahead
#pragma unroll
  for (int u = 0; u < PB; ++u) lbn[u] = (act && 1 + u < T) ? pL[(int64_t)u * K] : R(0);
  // step t = tb + u reads score buffer (t - 1) & 1 = u & 1 and writes the other
  for (int tb = 1; tb < T; tb += PB) {
    R lbc[PB];
    pL += (int64_t)PB * K;
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      lbc[u] = lbn[u];
      lbn[u] = (act && tb + PB + u < T) ? pL[(int64_t)u * K] : R(0);
    }
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      if (tb + u >= T) break;
      const int rd = (u & 1) * KM, wr = ((u + 1) & 1) * KM;
      R cv[NZ];
      int ci[NZ];
#pragma unroll
      for (int n = 0; n < NZ; ++n) {
        cv[n] = N::add(src[n][rd], lav[n]);
        ci[n] = off[n];
      }
      // first-index argmax tree: the right operand wins only when strictly greater
#pragma unroll
      for (int w = 1; w < NZ; w <<= 1) {
#pragma unroll
        for (int n = 0; n + w < NZ; n += 2 * w) {
          const bool r = cv[n + w] > cv[n];
          cv[n] = r ? cv[n + w] : cv[n];
          ci[n] = r ? ci[n + w] : ci[n];
        }
      }
      const R best = cv[0];
      const int bi = best > N::ninf() ? ci[0] : 0;  // an all -inf column: numpy's argmax is 0
      if (act) {
        mine[wr] = N::add(best, lbc[u]);
        *pK = (uint8_t)bi;
        if (pX) *pX = (uint8_t)bi;
      }
      pK += K;
      if (pX) pX += K;
      sync();
    }
  }
  const int cur = T > 0 ? (T - 1) & 1 : 0;  // buffer holding the last step's scores
  if (tid == 0) {
    const R* dv = dvb + cur * KM;
    R bv = dv[0];
    int bi = 0;
    for (int i = 1; i < K; ++i)
      if (dv[i] > bv) {
        bv = dv[i];
        bi = i;
      }
    a.log_joint[b] = (double)bv;
    *s_cur = bi;
  }
  sync();
  __threadfence_block();
  backtrace_blocks(bk, K, T, a.path + start, bblk, reinterpret_cast<uint8_t*>(dvb), s_cur, tid, NT, sync);
}

template <typename R, int KM>
__device__ __forceinline__ void viterbi_sparse_nz(const VitArgs& a, int K, uint8_t* backws,
                                                  const R* __restrict__ lbws, R* dvb, uint8_t* bblk,
                                                  int* s_cur, int maxnz) {
  if (maxnz <= 5) viterbi_sparse_path<R, KM, 5>(a, K, backws, lbws, dvb, bblk, s_cur);
  else if (maxnz <= 9) viterbi_sparse_path<R, KM, 9>(a, K, backws, lbws, dvb, bblk, s_cur);
  else viterbi_sparse_path<R, KM, kVitNZ>(a, K, backws, lbws, dvb, bblk, s_cur);
}

// Emission log-densities of one batch for the large-K Viterbi (reference-exact,
// emission_log_matrix: inference.py:93-126), T-parallel: block (chunk, b)
// covers kEmSeqChunk steps of sequence b, thread (t mod TPB, j) evaluates state
// j with its parameters in registers and writes coalesced rows.  NaN
// observations (inference.py:117-118) and log-gamma lookups outside the host
// table are recorded in the sequence's flag word.
constexpr int kEmSeqChunk = 1024;
template <typename R>
__global__ void __launch_bounds__(256) emission_seq_kernel(const VitArgs a, int K, R* __restrict__ out) {
  typedef Num<R> N;
  const int64_t b = blockIdx.y;
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const int t0 = blockIdx.x * kEmSeqChunk;
  if (t0 >= T) return;
  const int t1 = min(T, t0 + kEmSeqChunk);
  const int TPB = 256 / K;
  const int tid = threadIdx.x;
  const int j = tid % K, ts = tid / K;
  if (ts >= TPB) return;
  const loghmm_model_t* md = a.model;
  const bool two = a.n_streams > 1;
  const loghmm_emission_t e0 = md->em[0][j];
  loghmm_emission_t e1;
  if (two) e1 = md->em[1][j];
  const R* y0g = reinterpret_cast<const R*>(a.y0) + start;
  const R* y1g = two ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
  R* o = out + start * K + j;
  bool oob = false, nan_seen = false;
  for (int t = t0 + ts; t < t1; t += TPB) {
    const R v0 = y0g[t];
    const R v1 = two ? y1g[t] : R(0);
    nan_seen |= (v0 != v0) | (v1 != v1);
    R v = exact_logb<R>(e0, v0, a.lut, a.lut_n, oob);
    if (two) v = N::add(v, exact_logb<R>(e1, v1, a.lut, a.lut_n, oob));
    o[(int64_t)t * K] = v;
  }
  if (a.flags && (nan_seen || oob))
    atomicOr(reinterpret_cast<unsigned long long*>(a.flags + 2 * b + 1),
             (unsigned long long)((nan_seen ? 1 : 0) | (oob ? 2 : 0)));
}

// Viterbi, one CTA per sequence, four lanes per destination state j (the
// Quarter layout of fb_large_kernel): lane q scans the sources i = q, q + 4,
// ... with log A[i][j] in registers, and the four partial (max, first index)
// pairs are combined with two xor shuffles, larger value first and the
// smaller index on ties, which is the reference's first-index argmax
// (inference.py:204-207) bit for bit.  The score vector is double-buffered in
// shared memory (one barrier per step) and y is loaded one step ahead.
// Backpointers go to a byte table in the workspace; thread 0 walks the path
// with blocks of backpointer rows prefetched into shared memory.
template <typename R, int KM, int P>
__global__ void __launch_bounds__(256) viterbi_large_kernel(const VitArgs a, int K,
                                                            uint8_t* backws,
                                                            const R* __restrict__ lbws) {
  typedef Num<R> N;
  constexpr int NQ = KM / P;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* dvb = reinterpret_cast<R*>(smem_raw);                    // [2][KM] scores
  // [kBtBlk * K] backpointer rows; the score buffers (>= kBtBlk bytes) double as the path stage
  uint8_t* bblk = smem_raw + (2 * KM * sizeof(R) > kBtBlk ? 2 * KM * sizeof(R) : (size_t)kBtBlk);
  __shared__ int s_cur;
  __shared__ int s_maxnz;
  const int tid = threadIdx.x;
  const int q = tid & (P - 1);
  const int jt = tid / P;
  const int64_t b = blockIdx.x;
  if (b >= a.B) return;
  // structural sparsity of log A: the largest number of finite sources of a column
  if (tid == 0) s_maxnz = 0;
  __syncthreads();
  if (tid < K) {
    int cnt = 0;
    for (int i = 0; i < K; ++i) cnt += a.model->log_A[i * K + tid] > -CUDART_INF ? 1 : 0;
    atomicMax(&s_maxnz, cnt);
  }
  __syncthreads();
  if (s_maxnz <= kVitNZ && a.sparse_ok) {
    if (tid >= (KM < 32 ? 32 : KM)) return;
    viterbi_sparse_nz<R, KM>(a, K, backws, lbws, dvb, bblk, &s_cur, s_maxnz);
    return;
  }
  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  const bool act = jt < K;
  const bool lead = act && q == 0;
  const int j = act ? jt : 0;
  const loghmm_model_t* md = a.model;
  R la[NQ];  // log A[P s + q][j]
#pragma unroll
  for (int s = 0; s < NQ; ++s) {
    const int i = P * s + q;
    la[s] = (act && i < K) ? (R)md->log_A[i * K + j] : N::ninf();
  }
  constexpr int PB = kVitPB;
  const R* __restrict__ lbj = lbws + start * K + j;  // log b_t[j] at lbj[t * K]
  uint8_t* bk = backws + start * K;
  for (int e = tid; e < 2 * KM; e += blockDim.x) dvb[e] = N::ninf();
  __syncthreads();
  if (lead && T > 0) {
    dvb[j] = N::add((R)md->log_pi[j], lbj[0]);
    bk[j] = 0;
    if (a.back) a.back[start * K + j] = 0;
  }
  __syncthreads();
  int cur = 0;
  R lbn[PB];  // the next block's emission terms, loaded a block ahead
#pragma unroll
  for (int u = 0; u < PB; ++u) lbn[u] = (lead && 1 + u < T) ? lbj[(int64_t)(1 + u) * K] : R(0);
  for (int tb = 1; tb < T; tb += PB) {
    R lbc[PB];
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      lbc[u] = lbn[u];
      lbn[u] = (lead && tb + PB + u < T) ? lbj[(int64_t)(tb + PB + u) * K] : R(0);
    }
#pragma unroll
    for (int u = 0; u < PB; ++u) {
      const int t = tb + u;
      if (t >= T) break;
      const R* dv = dvb + cur * KM;
      R best = N::add(dv[q], la[0]);
      int bi = q;
#pragma unroll
      for (int s = 1; s < NQ; ++s) {
        const R c = N::add(dv[P * s + q], la[s]);
        if (c > best) {
          best = c;
          bi = P * s + q;
        }
      }
#pragma unroll
      for (int o = 1; o < P; o <<= 1) {
        const R ov = __shfl_xor_sync(kFull, best, o);
        const int oi = __shfl_xor_sync(kFull, bi, o);
        if (ov > best || (ov == best && oi < bi)) {
          best = ov;
          bi = oi;
        }
      }
      cur ^= 1;
      if (lead) {
        dvb[cur * KM + j] = N::add(best, lbc[u]);
        bk[(int64_t)t * K + j] = (uint8_t)bi;
        if (a.back) a.back[(start + t) * K + j] = (uint8_t)bi;
      }
      __syncthreads();
    }
  }
  if (tid == 0) {
    const R* dv = dvb + cur * KM;
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
  backtrace_blocks(bk, K, T, a.path + start, bblk, reinterpret_cast<uint8_t*>(dvb), &s_cur, tid,
                   (int)blockDim.x, [] { __syncthreads(); });
}

}  // namespace lhmm
