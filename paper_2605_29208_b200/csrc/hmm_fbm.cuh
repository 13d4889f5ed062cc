// hmm_fbm.cuh — batched forward-backward, "meet in the middle", K <= 8.
//
// Same outputs and statistics as hmm_fb.cuh (inference.py:129-188,
// training.py:187-210) with a different decomposition, chosen when the batch
// is wide enough (B*4 threads fill the GPU):
//
//   * A CTA owns G = 32/S sequences and has two warps: the forward warp runs
//     the forward recursion t = 0..T-1, the backward warp the backward
//     recursion t = T-1..0, concurrently.  S lanes share one sequence (S = 2:
//     each lane owns ceil(K/2) states; the partner's half of the state vector
//     comes through one warp shuffle per step).  No transfer operators, no
//     K^3 work: every step is the plain K^2 recursion.
//   * Both warps first run to the common split point H = ceil(Tmax/2),
//     storing their normalised linear vectors (alpha~ for t < H, beta~ for
//     t >= H) in a workspace laid out [t][b][K] (coalesced across the warp).
//     After one CTA barrier each warp continues into the other half, where it
//     reads the other direction's vector back, and forms gamma, xi and the
//     family statistics on the fly.  The workspace lines are dropped from L2
//     after their single read (discard.global.L2), so it costs L2 bandwidth
//     only.
//   * Recursions are in linear space with power-of-two renormalisation and
//     log2 offsets; logs (outputs) are taken off the recursion chain.
#pragma once

#include "hmm_fb.cuh"

namespace lhmm {

constexpr int kMSlab = 8;  // output staging depth (steps per flush)

struct FBMArgs {
  const loghmm_model_t* model;
  const void* y0;
  const void* y1;
  const int64_t* offsets;
  int64_t B;
  const double* lut;
  int lut_n;
  int n_streams;
  void* log_alpha;
  void* log_beta;
  void* gamma;
  void* xi;
  double* ll;
  double* partials;
  int64_t* flags;
  void* ws;           // [max_T][B][KP] workspace
  int64_t ws_bstride; // elements per t row (= B * KP)
  int64_t stats_width;
};

__device__ __forceinline__ void l2_discard(const void* p) {
  asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

template <typename R, int KL>
struct LVec {
  static __device__ __forceinline__ void st(R* p, const R (&v)[KL]) {
    if constexpr (KL * sizeof(R) == 16) {
      if constexpr (sizeof(R) == 4)
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
      else
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    } else if constexpr (KL * sizeof(R) == 8) {
      if constexpr (sizeof(R) == 4)
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
      else
        *p = v[0];
    } else {
#pragma unroll
      for (int i = 0; i < KL; ++i) p[i] = v[i];
    }
  }
  static __device__ __forceinline__ void ld(const R* p, R (&v)[KL]) {
    if constexpr (KL * sizeof(R) == 16) {
      if constexpr (sizeof(R) == 4) {
        const float4 q = *reinterpret_cast<const float4*>(p);
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
      } else {
        const double2 q = *reinterpret_cast<const double2*>(p);
        v[0] = q.x; v[1] = q.y;
      }
    } else if constexpr (KL * sizeof(R) == 8) {
      if constexpr (sizeof(R) == 4) {
        const float2 q = *reinterpret_cast<const float2*>(p);
        v[0] = q.x; v[1] = q.y;
      } else {
        v[0] = *p;
      }
    } else {
#pragma unroll
      for (int i = 0; i < KL; ++i) v[i] = p[i];
    }
  }
};

// Own-state emission evaluation (KL states starting at j0; padded states -inf).
template <typename R, int KL, int CFG>
struct EmitL {
  EmP<R> e0[KL];
  EmP<R> e1[KL];
  bool pad[KL];
  int stream_fams;
  const double* lut;
  int lut_n;
  __device__ __forceinline__ void load(const loghmm_model_t* m, int K, int j0, int n_streams,
                                       int fams, const double* lut_, int lut_n_) {
#pragma unroll
    for (int j = 0; j < KL; ++j) {
      const int jj = j0 + j;
      pad[j] = jj >= K;
      const int js = pad[j] ? 0 : jj;
      e0[j] = load_emission<R>(m->em[0][js]);
      if (CFG == kCfgGammaVM || (CFG == kCfgMixed && n_streams > 1))
        e1[j] = load_emission<R>(m->em[1][js]);
      else
        e1[j].fam = LOGHMM_FAM_NONE;
    }
    stream_fams = fams;
    lut = lut_;
    lut_n = lut_n_;
  }
  __device__ __forceinline__ void eval(R y0, R y1, ObsFeat<R>& f0, ObsFeat<R>& f1, R (&lb)[KL],
                                       bool& oob) const {
    if (CFG == kCfgGammaVM) {
      obs_features<R, kCfgGamma>(f0, y0, lut, lut_n, oob, 0);
      obs_features<R, kCfgVonMises>(f1, y1, lut, lut_n, oob, 0);
#pragma unroll
      for (int j = 0; j < KL; ++j)
        lb[j] = fast_logb_fam<R, LOGHMM_FAM_GAMMA>(e0[j], f0) +
                fast_logb_fam<R, LOGHMM_FAM_VON_MISES>(e1[j], f1);
    } else if (CFG == kCfgMixed) {
      obs_features<R, kCfgMixed>(f0, y0, lut, lut_n, oob, stream_fams & 0xffff);
      obs_features<R, kCfgMixed>(f1, y1, lut, lut_n, oob, stream_fams >> 16);
#pragma unroll
      for (int j = 0; j < KL; ++j) lb[j] = fast_logb_rt<R>(e0[j], f0) + fast_logb_rt<R>(e1[j], f1);
    } else {
      obs_features<R, CFG>(f0, y0, lut, lut_n, oob, 0);
#pragma unroll
      for (int j = 0; j < KL; ++j) lb[j] = fast_logb_fam<R, CFG>(e0[j], f0);
    }
#pragma unroll
    for (int j = 0; j < KL; ++j)
      if (pad[j]) lb[j] = Num<R>::ninf();
  }
  __device__ __forceinline__ void stats(R (&st)[CfgTraits<CFG>::S][KL][LOGHMM_NSLOT],
                                        const R (&g)[KL], const ObsFeat<R>& f0,
                                        const ObsFeat<R>& f1) const {
    typedef CfgTraits<CFG> TR;
#pragma unroll
    for (int j = 0; j < KL; ++j) {
      if constexpr (TR::F0 >= 0) stat_acc<R, TR::F0>(st[0][j], g[j], e0[j], f0);
      else stat_acc_rt<R>(st[0][j], g[j], e0[j], f0);
      if constexpr (TR::S > 1) {
        if constexpr (TR::F1 >= 0) stat_acc<R, TR::F1>(st[1][j], g[j], e1[j], f1);
        else stat_acc_rt<R>(st[1][j], g[j], e1[j], f1);
      }
    }
  }
};

template <typename R, int K>
struct MITraits {
  static constexpr int S = K >= 2 ? 2 : 1;   // lanes per sequence
  static constexpr int KL = (K + S - 1) / S; // states per lane
  static constexpr int KP = KL * S;          // padded state count
  static constexpr int G = kWarp / S;        // sequences per CTA
};

// Shared-memory carve per CTA (elements of R unless noted).
template <typename R, int K>
struct MISmem {
  typedef MITraits<R, K> M;
  static constexpr int YW = 32;                     // y staging depth (steps)
  static constexpr int YP = M::G + 1;               // y row pitch (odd in 4/8 B units)
  static constexpr int ROW = kMSlab * K;            // staged elements per sequence row
  static constexpr int RP = ROW + (16 / (int)sizeof(R));  // padded row pitch (16 B aligned)
  static constexpr int STG = M::G * RP;             // one staging array
  // fwd: y0,y1, stage log_alpha, stage gamma ; bwd: y0,y1, stage log_beta, stage gamma
  static constexpr int PER_WARP = 2 * YW * YP + 2 * STG;
  static constexpr int XI = M::G * K * K;           // xi exchange (fwd -> bwd)
  static constexpr size_t bytes() { return (size_t)(2 * PER_WARP + XI) * sizeof(R) + 16; }
};

template <typename R, int K, int CFG>
__global__ void __launch_bounds__(64) fb_mitm_kernel(const FBMArgs a) {
  typedef Num<R> N;
  typedef MITraits<R, K> M;
  typedef MISmem<R, K> SM;
  typedef CfgTraits<CFG> TR;
  constexpr int S = M::S, KL = M::KL, KP = M::KP, G = M::G;
  constexpr R kL2E = R(1.4426950408889634);
  constexpr R kLN2 = R(0.6931471805599453);
  constexpr double kLN2d = 0.6931471805599453094;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int warp = threadIdx.x >> 5;  // 0 forward, 1 backward
  const int lane = threadIdx.x & 31;
  const bool fwd = warp == 0;
  const int q = lane / S;             // sequence slot in the CTA
  const int h = lane % S;             // half index
  const int j0 = h * KL;
  const int64_t b = (int64_t)blockIdx.x * G + q;
  const bool valid = b < a.B;
  const int64_t start = valid ? a.offsets[b] : 0;
  const int T = valid ? (int)(a.offsets[b + 1] - start) : 0;

  R* sm = reinterpret_cast<R*>(smem_raw);
  R* wsm = sm + warp * SM::PER_WARP;
  R* ys0 = wsm;
  R* ys1 = ys0 + SM::YW * SM::YP;
  R* stO = ys1 + SM::YW * SM::YP;  // log_alpha (fwd) / log_beta (bwd)
  R* stG = stO + SM::STG;          // gamma
  R* xis = sm + 2 * SM::PER_WARP;  // xi exchange [G][K][K]
  __shared__ int s_T[G];
  __shared__ int64_t s_start[G];
  if (fwd && h == 0) {
    s_T[q] = T;
    s_start[q] = start;
  }

  // warp-uniform lengths
  int Tmax = T;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Tmax = max(Tmax, __shfl_xor_sync(kFull, Tmax, o));
  const int H = (Tmax + 1) / 2;  // split point
  const bool two = a.n_streams > 1;
  const R* __restrict__ y0g = reinterpret_cast<const R*>(a.y0);
  const R* __restrict__ y1g = two ? reinterpret_cast<const R*>(a.y1) : y0g;

  // ---- model -------------------------------------------------------------
  const loghmm_model_t* __restrict__ md = a.model;
  // forward: p_j = sum_i a_i A_ij for own j  -> column block Acol[i][jl] = A[i][j0+jl]
  // backward: q_i = sum_j A_ij w_j for own i -> row block    Arow[il][j] = A[j0+il][j]
  R Am[KP][KL];  // fwd: Am[i][jl] = A[i][j0+jl]; bwd: Am[j][il] = A[j0+il][j]
  R minA = R(1);
#pragma unroll
  for (int i = 0; i < KP; ++i)
#pragma unroll
    for (int l = 0; l < KL; ++l) {
      const int r = fwd ? i : j0 + l;
      const int c = fwd ? j0 + l : i;
      const R v = (r < K && c < K) ? (R)md->A[r * K + c] : R(0);
      Am[i][l] = v;
    }
  for (int i = 0; i < K * K; ++i) {
    const R v = (R)md->A[i];
    minA = v < minA ? v : minA;
  }
  R lpi[KL];
#pragma unroll
  for (int l = 0; l < KL; ++l) lpi[l] = (j0 + l < K) ? (R)md->log_pi[j0 + l] * kL2E : N::ninf();
  EmitL<R, KL, CFG> em;
  int fams = 0;
  {
    int m0 = 0, m1 = 0;
    for (int j = 0; j < K; ++j) {
      m0 |= 1 << md->em[0][j].family;
      if (two) m1 |= 1 << md->em[1][j].family;
    }
    fams = (m0 & 0xffff) | ((m1 & 0xffff) << 16);
  }
  em.load(md, K, j0, a.n_streams, fams, a.lut, a.lut_n);
  int nn = 1;
  if (minA > R(0)) {
    const double lg = -log2((double)minA);
    const double budget = sizeof(R) == 4 ? 100.0 : 900.0;
    nn = lg <= 0.0 ? 8 : (int)fmin(8.0, fmax(1.0, floor(budget / lg)));
  }

  R* __restrict__ W = reinterpret_cast<R*>(a.ws);
  const int64_t wcol = (int64_t)(blockIdx.x * G + q) * KP + j0;  // element offset in a t row

  // y staging: window [yw, yw+YW) of steps for the G sequences, [step][seq]
  auto stage_y = [&](int yw) {
    __syncwarp();
    for (int e = lane; e < SM::YW * G; e += kWarp) {
      const int qq = e / SM::YW, st = e % SM::YW;  // consecutive lanes: consecutive steps
      const int t = yw + st;
      const int Tq = s_T[qq];
      const int64_t sq = s_start[qq];
      R v0 = R(0), v1 = R(0);
      if (t >= 0 && t < Tq) {
        v0 = y0g[sq + t];
        if (two) v1 = y1g[sq + t];
      }
      ys0[st * SM::YP + qq] = v0;
      if (two) ys1[st * SM::YP + qq] = v1;
    }
    __syncwarp();
  };
  // output flush for window [tw, tw+kMSlab): row qq is contiguous in global;
  // only steps in [lo, hi) of the window were produced by this warp.
  auto flush = [&](R* __restrict__ out, const R* __restrict__ stg, int tw, int lo, int hi) {
    __syncwarp();
    if (out) {
      constexpr int EPV = 16 / (int)sizeof(R);
      constexpr int VPR = (SM::ROW + EPV - 1) / EPV;
      const int s0 = lo > tw ? lo - tw : 0;
      for (int v = lane; v < G * VPR; v += kWarp) {
        const int qq = v / VPR, vi = v % VPR;
        const int Tq = s_T[qq];
        int s1 = min(hi, Tq) - tw;
        s1 = s1 < 0 ? 0 : (s1 > kMSlab ? kMSlab : s1);
        int e0 = vi * EPV, e1 = e0 + EPV;
        e0 = max(e0, s0 * K);
        e1 = min(e1, s1 * K);
        if (e1 <= e0) continue;
        R* dst = out + (s_start[qq] + tw) * K + e0;
        const R* src = stg + qq * SM::RP + e0;
        const bool al = ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) && (e1 - e0 == EPV);
        if (al) {
          *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
        } else {
          for (int e2 = 0; e2 < e1 - e0; ++e2) dst[e2] = src[e2];
        }
      }
    }
    __syncwarp();
  };

  bool oob = false, nan_seen = false;
  int dead_t = INT_MAX;

  // accumulators (own states)
  R X[KP][KL];  // fwd: X[i][jl] (column block), bwd: X[jl... stored as X[j][il] (row block)
  R gtot[KL], g0[KL];
  R st[TR::S][KL][LOGHMM_NSLOT];
#pragma unroll
  for (int l = 0; l < KL; ++l) {
    gtot[l] = R(0);
    g0[l] = R(0);
#pragma unroll
    for (int i = 0; i < KP; ++i) X[i][l] = R(0);
#pragma unroll
    for (int s = 0; s < TR::S; ++s)
#pragma unroll
      for (int k = 0; k < LOGHMM_NSLOT; ++k) st[s][l][k] = R(0);
  }
  __syncthreads();  // s_T / s_start visible

  R* __restrict__ outO = reinterpret_cast<R*>(fwd ? a.log_alpha : a.log_beta);
  R* __restrict__ outG = reinterpret_cast<R*>(a.gamma);
  R* __restrict__ outX = reinterpret_cast<R*>(a.xi);
  double LL = 0.0;

  // exchange of the partner's half of a KL-vector (S == 2)
  auto gather = [&](const R (&own)[KL], R (&full)[KP]) {
#pragma unroll
    for (int l = 0; l < KL; ++l) {
      const R o = (S == 2) ? __shfl_xor_sync(kFull, own[l], 1) : R(0);
      full[h * KL + l] = own[l];
      if (S == 2) full[(1 - h) * KL + l] = o;
    }
  };
  auto gmax = [&](R v) -> R {
    if (S == 2) v = rmax(v, __shfl_xor_sync(kFull, v, 1));
    return v;
  };
  auto gsum = [&](R v) -> R {
    if (S == 2) v += __shfl_xor_sync(kFull, v, 1);
    return v;
  };

  if (fwd) {
    // ===================== forward warp =====================
    R av[KL];  // alpha~ (linear, own states)
    double lam = 0.0;
#pragma unroll 1
    for (int t = 0; t < Tmax; ++t) {
      if (t == H) {
        __threadfence_block();
        __syncthreads();  // both directions finished their first half
      }
      if ((t % SM::YW) == 0) stage_y(t);
      const bool act = t < T;
      const R yv0 = ys0[(t % SM::YW) * SM::YP + q];
      const R yv1 = two ? ys1[(t % SM::YW) * SM::YP + q] : R(0);
      if (act && (isnan(yv0) || isnan(yv1))) nan_seen = true;
      ObsFeat<R> f0, f1;
      R lb[KL];
      em.eval(yv0, yv1, f0, f1, lb, oob);
      R m = lb[0];
#pragma unroll
      for (int l = 1; l < KL; ++l) m = rmax(m, lb[l]);
      m = gmax(m);
      if (act && !(m > N::ninf()) && t < dead_t) dead_t = t;
      const bool fin = m > N::ninf();
      const R m2 = m * kL2E;
      R o[KL];
      R g[KL];
      bool have_g = false;
      R aprev[KP];
      gather(av, aprev);
      if (t == 0) {
        R u[KL];
#pragma unroll
        for (int l = 0; l < KL; ++l) u[l] = fma(lb[l], kL2E, lpi[l]);
        R M = u[0];
#pragma unroll
        for (int l = 1; l < KL; ++l) M = rmax(M, u[l]);
        M = gmax(M);
        const bool fm = M > N::ninf();
#pragma unroll
        for (int l = 0; l < KL; ++l) {
          o[l] = u[l] * kLN2;
          av[l] = fm ? N::fex2(u[l] - M) : R(0);
        }
        lam = fm ? (double)M : -CUDART_INF;
      } else {
        R p[KL], bb[KL];
#pragma unroll
        for (int l = 0; l < KL; ++l) {
          R acc = aprev[0] * Am[0][l];
#pragma unroll
          for (int i = 1; i < KP; ++i) acc = fma(aprev[i], Am[i][l], acc);
          p[l] = acc;
          bb[l] = fin ? N::fex2(fma(lb[l], kL2E, -m2)) : R(0);
        }
        const R lr = (R)lam;
#pragma unroll
        for (int l = 0; l < KL; ++l) o[l] = fma(lb[l], kL2E, lr + N::flg2(p[l])) * kLN2;
        if (t >= H) {
          // combine with beta~_t: gamma_t and xi_{t-1}
          R bet[KL];
#pragma unroll
          for (int l = 0; l < KL; ++l) bet[l] = R(0);
          const R* wp = W + (int64_t)t * a.ws_bstride + wcol;
          if (act) LVec<R, KL>::ld(wp, bet);
          R v[KL];
          R Zp = R(0);
#pragma unroll
          for (int l = 0; l < KL; ++l) {
            v[l] = bb[l] * bet[l];
            Zp = fma(p[l], v[l], Zp);
          }
          const R iz = N::frcp(gsum(Zp));
          // single-use workspace line: drop it from L2 once consumed
          if (act && h == 0 && (((wcol * (int64_t)sizeof(R)) & 127) == 0)) l2_discard(wp);
#pragma unroll
          for (int l = 0; l < KL; ++l) {
            const R cv = v[l] * iz;
            g[l] = p[l] * cv;
#pragma unroll
            for (int i = 0; i < KP; ++i) X[i][l] = fma(aprev[i], cv, X[i][l]);
            if (outX && act) {
              R* xr = outX + ((start - b) + (t - 1)) * (int64_t)(K * K);
              if (j0 + l < K)
                for (int i = 0; i < K; ++i) xr[i * K + j0 + l] = aprev[i] * Am[i][l] * cv;
            }
          }
          have_g = act;
        }
#pragma unroll
        for (int l = 0; l < KL; ++l) av[l] = p[l] * bb[l];
        lam += fin ? (double)m2 : 0.0;
        if ((t % nn) == 0) {  // warp-uniform renormalisation schedule
          R mx = av[0];
#pragma unroll
          for (int l = 1; l < KL; ++l) mx = rmax(mx, av[l]);
          mx = gmax(mx);
          if (mx > R(0)) {
            int e;
            const R sc = N::pow2_scale(mx, e);
            lam += (double)e;
#pragma unroll
            for (int l = 0; l < KL; ++l) av[l] *= sc;
          }
        }
      }
      if (t < H && act) {
        // store alpha~_t for the backward warp
        LVec<R, KL>::st(W + (int64_t)t * a.ws_bstride + wcol, av);
      }
      if (act) {
        LVec<R, KL>::st(stO + q * SM::RP + (t % kMSlab) * K + j0, o);
        if (have_g) {
          if (outG) LVec<R, KL>::st(stG + q * SM::RP + (t % kMSlab) * K + j0, g);
          em.stats(st, g, f0, f1);
          if (t < T - 1) {
#pragma unroll
            for (int l = 0; l < KL; ++l) gtot[l] += g[l];
          }
        }
      }
      if ((t % kMSlab) == kMSlab - 1 || t == Tmax - 1) {
        const int tw = t - (t % kMSlab);
        flush(outO, stO, tw, tw, tw + kMSlab);
        if (tw + kMSlab > H) flush(outG, stG, tw, H, tw + kMSlab);
      }
    }
    if (H >= Tmax) {
      __threadfence_block();
      __syncthreads();  // matches the backward warp's split barrier
    }
    // log-likelihood
    R s = R(0);
#pragma unroll
    for (int l = 0; l < KL; ++l) s += av[l];
    s = gsum(s);
    LL = s > R(0) ? (lam + (double)N::flg2(s)) * kLN2d : -CUDART_INF;
    if (T == 0) LL = -CUDART_INF;
  } else {
    // ===================== backward warp =====================
    R bt[KL];  // beta~_{t+1} (linear, own states)
    double rho = 0.0;
    R lbn[KL];   // emission log-density at t+1 (own states), natural units
    R mn = R(0); // its max over all states
    bool finn = true;
    // iterate t = Tmax-1 .. 0; lane active when t < T
#pragma unroll 1
    for (int t = Tmax - 1; t >= 0; --t) {
      if (t == Tmax - 1 || (t % SM::YW) == SM::YW - 1) stage_y(t - (t % SM::YW));
      if (t == H - 1) {
        __threadfence_block();
        __syncthreads();
      }
      const bool act = t < T;
      const R yv0 = ys0[(t % SM::YW) * SM::YP + q];
      const R yv1 = two ? ys1[(t % SM::YW) * SM::YP + q] : R(0);
      ObsFeat<R> f0, f1;
      R lb[KL];
      em.eval(yv0, yv1, f0, f1, lb, oob);
      R m = lb[0];
#pragma unroll
      for (int l = 1; l < KL; ++l) m = rmax(m, lb[l]);
      m = gmax(m);
      R o[KL], g[KL];
      R qv[KL];
      bool have_g = false;
      const bool first = (t == T - 1);
      // recursion beta_t = A (b_{t+1} . beta_{t+1}) for every lane (uniform
      // shuffles); lanes at their first step take beta_{T-1} = 1 instead.
      R w[KL];
#pragma unroll
      for (int l = 0; l < KL; ++l)
        w[l] = (finn ? N::fex2(fma(lbn[l], kL2E, -mn * kL2E)) : R(0)) * bt[l];
      R wf[KP];
      gather(w, wf);
#pragma unroll
      for (int l = 0; l < KL; ++l) {
        R acc = Am[0][l] * wf[0];
#pragma unroll
        for (int jx = 1; jx < KP; ++jx) acc = fma(Am[jx][l], wf[jx], acc);
        qv[l] = first ? ((j0 + l < K) ? R(1) : R(0)) : acc;
      }
      if (first) {
        rho = 0.0;
      } else {
        rho += finn ? (double)(mn * kL2E) : 0.0;
      }
      {
        const R rr = (R)rho;
#pragma unroll
        for (int l = 0; l < KL; ++l) o[l] = first ? R(0) : (rr + N::flg2(qv[l])) * kLN2;
      }
      if (t < H) {
        // combine with alpha~_t: gamma_t and xi_t (pair t, t+1)
        R al[KL];
#pragma unroll
        for (int l = 0; l < KL; ++l) al[l] = R(0);
        const R* wp = W + (int64_t)t * a.ws_bstride + wcol;
        if (act) LVec<R, KL>::ld(wp, al);
        R Zp = R(0);
#pragma unroll
        for (int l = 0; l < KL; ++l) Zp = fma(al[l], qv[l], Zp);
        const R iz = N::frcp(gsum(Zp));
        if (act && h == 0 && (((wcol * (int64_t)sizeof(R)) & 127) == 0)) l2_discard(wp);
        // the pair (H-1, H) belongs to the forward warp
        const bool pair = act && !first && t < H - 1;
#pragma unroll
        for (int l = 0; l < KL; ++l) {
          g[l] = al[l] * qv[l] * iz;
          const R ai = al[l] * iz;
          if (pair) {
#pragma unroll
            for (int jx = 0; jx < KP; ++jx) X[jx][l] = fma(ai, wf[jx], X[jx][l]);
            if (outX && j0 + l < K) {
              R* xr = outX + ((start - b) + t) * (int64_t)(K * K);
              for (int jx = 0; jx < K; ++jx) xr[(j0 + l) * K + jx] = ai * Am[jx][l] * wf[jx];
            }
          }
        }
        have_g = act;
      }
      if ((t % nn) == 0) {  // warp-uniform renormalisation schedule
        R mx = qv[0];
#pragma unroll
        for (int l = 1; l < KL; ++l) mx = rmax(mx, qv[l]);
        mx = gmax(mx);
        if (act && !first && mx > R(0)) {
          int e;
          const R sc = N::pow2_scale(mx, e);
          rho += (double)e;
#pragma unroll
          for (int l = 0; l < KL; ++l) qv[l] *= sc;
        }
      }
      if (act) {
#pragma unroll
        for (int l = 0; l < KL; ++l) bt[l] = qv[l];
        if (t >= H) LVec<R, KL>::st(W + (int64_t)t * a.ws_bstride + wcol, bt);
        LVec<R, KL>::st(stO + q * SM::RP + (t % kMSlab) * K + j0, o);
        if (have_g) {
          if (outG) LVec<R, KL>::st(stG + q * SM::RP + (t % kMSlab) * K + j0, g);
          em.stats(st, g, f0, f1);
          if (t < T - 1) {
#pragma unroll
            for (int l = 0; l < KL; ++l) gtot[l] += g[l];
          }
          if (t == 0) {
#pragma unroll
            for (int l = 0; l < KL; ++l) g0[l] = g[l];
          }
        }
        // carry emission at t for the next (lower) step
#pragma unroll
        for (int l = 0; l < KL; ++l) lbn[l] = lb[l];
        mn = m;
        finn = m > N::ninf();
      }
      if ((t % kMSlab) == 0) {
        flush(outO, stO, t, t, t + kMSlab);
        if (t < H) flush(outG, stG, t, t, H);
      }
    }
  }

  // ---- per-sequence results ----------------------------------------------
  // xi: forward lanes own columns, backward lanes own rows; merge in smem.
  R* xq = xis + q * K * K;
  if (fwd) {
#pragma unroll
    for (int i = 0; i < KP; ++i)
#pragma unroll
      for (int l = 0; l < KL; ++l)
        if (i < K && j0 + l < K) xq[i * K + j0 + l] = X[i][l];
  }
  __shared__ int s_dead[G];
  __shared__ int s_flag[G];
  __shared__ double s_ll[G];
  if (fwd) {
    int d = dead_t;
    if (S == 2) d = min(d, __shfl_xor_sync(kFull, d, 1));
    const unsigned nanb = __ballot_sync(kFull, nan_seen);
    const unsigned oobb = __ballot_sync(kFull, oob);
    const unsigned pm = (S == 2) ? (3u << (q * 2)) : (1u << q);
    if (h == 0) {
      s_dead[q] = d;
      s_flag[q] = ((nanb & pm) ? 1 : 0) | ((oobb & pm) ? 2 : 0);
      s_ll[q] = LL;
    }
  }
  __syncthreads();
  if (!fwd && valid) {
    if (h == 0) {
      a.ll[b] = s_ll[q];
      if (a.flags) {
        a.flags[2 * b] = s_dead[q] == INT_MAX ? -1 : (int64_t)s_dead[q];
        a.flags[2 * b + 1] = s_flag[q] | (oob ? 2 : 0);
      }
    }
  }
  // per-sequence statistics row: bwd warp adds its rows into the xi block,
  // both warps add their own gamma totals / stats via smem, bwd writes.
  if (a.partials) {
    // stats/gtot/g0 exchange through the staging area (reuse stG of fwd warp)
    double* xch = reinterpret_cast<double*>(sm);  // reuse warp smem (all flushed)
    __syncthreads();
    const int nst = TR::S * KL * LOGHMM_NSLOT;
    constexpr int PER = KL + TR::S * KL * LOGHMM_NSLOT;  // gtot + stats
    if (fwd) {
      double* e = xch + (q * S + h) * PER;
#pragma unroll
      for (int l = 0; l < KL; ++l) e[l] = (double)gtot[l];
#pragma unroll
      for (int s = 0; s < TR::S; ++s)
#pragma unroll
        for (int l = 0; l < KL; ++l)
#pragma unroll
          for (int k = 0; k < LOGHMM_NSLOT; ++k)
            e[KL + (s * KL + l) * LOGHMM_NSLOT + k] = (double)st[s][l][k];
    }
    (void)nst;
    __syncthreads();
    if (!fwd && valid) {
      double* row = a.partials + b * a.stats_width;
      const double* e = xch + (q * S + h) * PER;
      // xi: row block from the backward lane + column block from smem
#pragma unroll
      for (int l = 0; l < KL; ++l) {
        const int i = j0 + l;
        if (i >= K) continue;
        for (int jx = 0; jx < K; ++jx)
          row[i * K + jx] = ((double)X[jx][l] + (double)xq[i * K + jx]) * (double)Am[jx][l];
      }
#pragma unroll
      for (int l = 0; l < KL; ++l) {
        const int j = j0 + l;
        if (j >= K) continue;
        row[K * K + j] = (double)gtot[l] + e[l];
        row[K * K + K + j] = (double)g0[l];
      }
#pragma unroll
      for (int s = 0; s < 2; ++s)
#pragma unroll
        for (int l = 0; l < KL; ++l) {
          const int j = j0 + l;
          if (j >= K) continue;
#pragma unroll
          for (int k = 0; k < LOGHMM_NSLOT; ++k) {
            double v = 0.0;
            if (s < TR::S) {
              const int ns = s == 0 ? TR::NS0 : TR::NS1;
              if (k < ns) v = (double)st[s][l][k] + e[KL + (s * KL + l) * LOGHMM_NSLOT + k];
            }
            row[K * K + 2 * K + (s * K + j) * LOGHMM_NSLOT + k] = v;
          }
        }
    }
  }
}

}  // namespace lhmm
