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
  static constexpr int D = 16;                      // prefetch depth (steps)
  static constexpr int YR = D * kWarp * 2;          // y ring: [D][lane] x 2 streams
  static constexpr int WR = D * kWarp * M::KL;      // workspace ring: [D][lane][KL]
  static constexpr int ROW = kMSlab * K;            // staged elements per sequence row
  static constexpr int RP = ROW + (16 / (int)sizeof(R));  // padded row pitch (16 B aligned)
  static constexpr int STG = M::G * RP;             // one staging array
  // per warp: y ring, workspace ring, stage log_alpha|log_beta, stage gamma
  static constexpr int PER_WARP = YR + WR + 2 * STG;
  static constexpr int XI = M::G * K * K;           // xi exchange (fwd -> bwd)
  static constexpr size_t bytes() { return (size_t)(2 * PER_WARP + XI) * sizeof(R) + 16; }
};

template <typename R, int K, int CFG>
__global__ void __launch_bounds__(64) fb_mitm_kernel(const FBMArgs a) {
  typedef Num<R> N;
  typedef MITraits<R, K> M;
  typedef MISmem<R, K> SM;
  typedef CfgTraits<CFG> TR;
  constexpr int S = M::S, KL = M::KL, KP = M::KP, G = M::G, D = SM::D;
  constexpr R kL2E = R(1.4426950408889634);
  constexpr R kLN2 = R(0.6931471805599453);
  constexpr double kLN2d = 0.6931471805599453094;
  // vector stores of a lane's KL states into a [step][K] row are aligned only
  // when K is a multiple of KL (K = 2, 4, 8)
  constexpr bool kVecRow = (K % KL) == 0;
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
  R* yring = wsm;                  // [D][32][2]
  R* wring = yring + SM::YR;       // [D][32][KL]
  R* stO = wring + SM::WR;         // log_alpha (fwd) / log_beta (bwd)
  R* stG = stO + SM::STG;          // gamma
  R* xis = sm + 2 * SM::PER_WARP;  // xi exchange [G][K][K]
  __shared__ int s_T[G];
  __shared__ int64_t s_start[G];
  if (fwd && h == 0) {
    s_T[q] = T;
    s_start[q] = start;
  }

  int Tmax = T;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Tmax = max(Tmax, __shfl_xor_sync(kFull, Tmax, o));
  const int H = (Tmax + 1) / 2;  // split point
  const bool two = a.n_streams > 1;
  const R* __restrict__ y0g = reinterpret_cast<const R*>(a.y0);
  const R* __restrict__ y1g = two ? reinterpret_cast<const R*>(a.y1) : y0g;

  // ---- model -------------------------------------------------------------
  // State order inside a lane: own states first (perm(i) = j0 + i for i < KL,
  // then the partner's), so the exchanged half lands at static indices.
  auto perm = [&](int i) -> int { return i < KL ? j0 + i : (S == 2 ? (1 - h) * KL + (i - KL) : i); };
  const loghmm_model_t* __restrict__ md = a.model;
  R Am[KP][KL];  // fwd: Am[i][l] = A[perm i][j0+l]; bwd: Am[j][l] = A[j0+l][perm j]
  R minA = R(1);
#pragma unroll
  for (int i = 0; i < KP; ++i)
#pragma unroll
    for (int l = 0; l < KL; ++l) {
      const int pi_ = perm(i);
      const int r = fwd ? pi_ : j0 + l;
      const int c = fwd ? j0 + l : pi_;
      Am[i][l] = (r < K && c < K) ? (R)md->A[r * K + c] : R(0);
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
  const int64_t wcol = (int64_t)(blockIdx.x * G + q) * KP + j0;
  const int64_t wstride = a.ws_bstride;
  const bool wdisc = (h == 0) && (((wcol * (int64_t)sizeof(R)) & 127) == 0);
  const int dir = fwd ? 1 : -1;

  // per-lane ring slots: slot(i) = ring + ((i & (D-1)) * 32 + lane) * width
  R* yslot0 = yring + lane * 2;
  R* wslot0 = wring + lane * KL;
  // stage row of this lane: q * RP + step * K + j0
  R* stOq = stO + q * SM::RP + j0;
  R* stGq = stG + q * SM::RP + j0;

  // Flush plan: vector v = lane + 32k covers row v / VPR, unit v % VPR.
  constexpr int EPV = 16 / (int)sizeof(R);
  constexpr int VPR = (SM::ROW + EPV - 1) / EPV;
  constexpr int NIT = (G * VPR + kWarp - 1) / kWarp;
  int f_row[NIT], f_e0[NIT];
#pragma unroll
  for (int k = 0; k < NIT; ++k) {
    const int v = lane + kWarp * k;
    f_row[k] = v < G * VPR ? v / VPR : -1;
    f_e0[k] = (v % VPR) * EPV;
  }

  bool oob = false, nan_seen = false;
  int dead_t = INT_MAX;
  R X[KP][KL];
  R gtot[KL], g0[KL];
  R st[TR::S][KL][LOGHMM_NSLOT];
#pragma unroll
  for (int l = 0; l < KL; ++l) {
    gtot[l] = R(0);
    g0[l] = R(0);
#pragma unroll
    for (int i = 0; i < KP; ++i) X[i][l] = R(0);
#pragma unroll
    for (int s2 = 0; s2 < TR::S; ++s2)
#pragma unroll
      for (int k = 0; k < LOGHMM_NSLOT; ++k) st[s2][l][k] = R(0);
  }
  __syncthreads();  // s_T / s_start visible

  R* __restrict__ outO = reinterpret_cast<R*>(fwd ? a.log_alpha : a.log_beta);
  R* __restrict__ outG = reinterpret_cast<R*>(a.gamma);
  R* __restrict__ outX = reinterpret_cast<R*>(a.xi);
  double LL = 0.0;

  // window [tw, tw+kMSlab) flush; steps [lo, hi) of it were produced here
  auto flush = [&](R* __restrict__ out, const R* __restrict__ stg, int tw, int lo, int hi) {
    __syncwarp();
    if (out) {
      const int s0 = lo > tw ? lo - tw : 0;
#pragma unroll
      for (int k = 0; k < NIT; ++k) {
        const int qq = f_row[k];
        if (qq < 0) continue;
        int s1 = min(hi, s_T[qq]) - tw;
        s1 = s1 < 0 ? 0 : (s1 > kMSlab ? kMSlab : s1);
        const int e0 = max(f_e0[k], s0 * K);
        const int e1 = min(f_e0[k] + EPV, s1 * K);
        if (e1 <= e0) continue;
        R* dst = out + (s_start[qq] + tw) * K + e0;
        const R* src = stg + qq * SM::RP + e0;
        if (e1 - e0 == EPV && ((reinterpret_cast<uintptr_t>(dst) & 15) == 0)) {
          *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
        } else {
          for (int e2 = 0; e2 < e1 - e0; ++e2) dst[e2] = src[e2];
        }
      }
    }
    __syncwarp();
  };
  auto st_row = [&](R* p, const R (&v)[KL]) {
    if constexpr (kVecRow) {
      LVec<R, KL>::st(p, v);
    } else {
#pragma unroll
      for (int l = 0; l < KL; ++l)
        if (j0 + l < K) p[l] = v[l];
    }
  };
  auto gother = [&](const R (&own)[KL], R (&full)[KP]) {
#pragma unroll
    for (int l = 0; l < KL; ++l) {
      full[l] = own[l];
      if (S == 2) full[KL + l] = __shfl_xor_sync(kFull, own[l], 1);
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

  // ---- prefetch prologue: y for the first D steps of this sweep ----------
  // sweep step i handles t = fwd ? i : Tmax-1-i
  const R* y0p = y0g + start + (fwd ? 0 : (Tmax - 1));  // y pointer of step t(i) for this lane
  const R* y1p = y1g + start + (fwd ? 0 : (Tmax - 1));
  auto issue_y = [&](int i, const R* p0, const R* p1) {
    const int t = fwd ? i : Tmax - 1 - i;
    const bool ok = i < Tmax && t >= 0 && t < T;
    R* dst = yslot0 + (i & (D - 1)) * (kWarp * 2);
    cp_async<sizeof(R)>(dst, ok ? (const void*)p0 : (const void*)y0g, ok);
    if (two) cp_async<sizeof(R)>(dst + 1, ok ? (const void*)p1 : (const void*)y0g, ok);
  };
  auto issue_w = [&](int i, const R* wp) {
    const int t = fwd ? i : Tmax - 1 - i;
    const bool ok = i < Tmax && t >= 0 && t < T;
    R* dst = wslot0 + (i & (D - 1)) * (kWarp * KL);
    if constexpr (KL * sizeof(R) == 16 || KL * sizeof(R) == 8 || KL * sizeof(R) == 4) {
      cp_async<KL * sizeof(R)>(dst, ok ? (const void*)wp : (const void*)W, ok);
    } else {
#pragma unroll
      for (int l = 0; l < KL; ++l) cp_async<sizeof(R)>(dst + l, ok ? (const void*)(wp + l) : (const void*)W, ok);
    }
  };
  for (int i = 0; i < D; ++i) {
    issue_y(i, y0p + dir * i, y1p + dir * i);
    cp_async_commit();
  }
  const int iH = fwd ? H : Tmax - H;  // sweep index of the first combine step

  if (fwd) {
    // ===================== forward warp =====================
    R av[KL];  // alpha~ (linear, own states)
    double lam = 0.0;
    int ncd = nn;
    const R* wpf = W + (int64_t)H * wstride + wcol;  // W row of the step being prefetched
#pragma unroll 1
    for (int t = 0; t < Tmax; ++t) {
      if (t == H) {
        __threadfence_block();
        __syncthreads();  // both directions finished their first half
        for (int i = H; i < H + D; ++i) issue_w(i, W + (int64_t)i * wstride + wcol);
        wpf = W + (int64_t)(H + D) * wstride + wcol;
        cp_async_wait_all();
      } else {
        cp_async_wait<D - 1>();
      }
      const bool act = t < T;
      const R* yr = yslot0 + (t & (D - 1)) * (kWarp * 2);
      const R yv0 = yr[0];
      const R yv1 = two ? yr[1] : R(0);
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
      R o[KL], g[KL];
      bool have_g = false;
      R aprev[KP];
      gother(av, aprev);
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
          LVec<R, KL>::ld(wslot0 + (t & (D - 1)) * (kWarp * KL), bet);
          R v[KL];
          R Zp = R(0);
#pragma unroll
          for (int l = 0; l < KL; ++l) {
            v[l] = bb[l] * bet[l];
            Zp = fma(p[l], v[l], Zp);
          }
          const R iz = N::frcp(gsum(Zp));
          if (act && wdisc) l2_discard(W + (int64_t)t * wstride + wcol);
#pragma unroll
          for (int l = 0; l < KL; ++l) {
            const R cv = v[l] * iz;
            g[l] = p[l] * cv;
            if (act) {
#pragma unroll
              for (int i = 0; i < KP; ++i) X[i][l] = fma(aprev[i], cv, X[i][l]);
            }
            if (outX && act && j0 + l < K) {
              R* xr = outX + ((start - b) + (t - 1)) * (int64_t)(K * K);
              for (int i = 0; i < KP; ++i)
                if (perm(i) < K) xr[perm(i) * K + j0 + l] = aprev[i] * Am[i][l] * cv;
            }
          }
          have_g = act;
        }
        if (act) {
#pragma unroll
          for (int l = 0; l < KL; ++l) av[l] = p[l] * bb[l];
          lam += fin ? (double)m2 : 0.0;
        }
        if (--ncd == 0) {  // warp-uniform renormalisation schedule
          ncd = nn;
          R mx = av[0];
#pragma unroll
          for (int l = 1; l < KL; ++l) mx = rmax(mx, av[l]);
          mx = gmax(mx);
          if (act && mx > R(0)) {
            int e;
            const R sc = N::pow2_scale(mx, e);
            lam += (double)e;
#pragma unroll
            for (int l = 0; l < KL; ++l) av[l] *= sc;
          }
        }
      }
      if (t < H && act) LVec<R, KL>::st(W + (int64_t)t * wstride + wcol, av);
      if (act) {
        st_row(stOq + (t & (kMSlab - 1)) * K, o);
        if (have_g) {
          if (outG) st_row(stGq + (t & (kMSlab - 1)) * K, g);
          em.stats(st, g, f0, f1);
          if (t < T - 1) {
#pragma unroll
            for (int l = 0; l < KL; ++l) gtot[l] += g[l];
          }
        }
      }
      // refill the rings D steps ahead (slot t % D was consumed above)
      issue_y(t + D, y0p + (t + D), y1p + (t + D));
      if (t >= H) {
        issue_w(t + D, wpf);
        wpf += wstride;
      }
      cp_async_commit();
      if ((t & (kMSlab - 1)) == kMSlab - 1 || t == Tmax - 1) {
        const int tw = t & ~(kMSlab - 1);
        flush(outO, stO, tw, tw, tw + kMSlab);
        if (tw + kMSlab > H) flush(outG, stG, tw, H, tw + kMSlab);
      }
    }
    cp_async_wait_all();
    if (H >= Tmax) {
      __threadfence_block();
      __syncthreads();  // matches the backward warp's split barrier
    }
    R s = R(0);
#pragma unroll
    for (int l = 0; l < KL; ++l) s += av[l];
    s = gsum(s);
    LL = s > R(0) ? (lam + (double)N::flg2(s)) * kLN2d : -CUDART_INF;
    if (T == 0) LL = -CUDART_INF;
  } else {
    // ===================== backward warp =====================
    R bt[KL];    // beta~_{t+1} (linear, own states)
    double rho = 0.0;
    R lbn[KL];   // emission log-density at t+1 (own states)
    R mn = R(0); // its max over all states
    bool finn = true;
#pragma unroll
    for (int l = 0; l < KL; ++l) {
      bt[l] = R(0);
      lbn[l] = R(0);
    }
    int ncd = nn;
    const R* wpf = W + (int64_t)(H - 1 - D) * wstride + wcol;
#pragma unroll 1
    for (int t = Tmax - 1; t >= 0; --t) {
      const int it = Tmax - 1 - t;
      if (t == H - 1) {
        __threadfence_block();
        __syncthreads();
        for (int i = iH; i < iH + D; ++i) issue_w(i, W + (int64_t)(Tmax - 1 - i) * wstride + wcol);
        cp_async_wait_all();
      } else {
        cp_async_wait<D - 1>();
      }
      const bool act = t < T;
      const R* yr = yslot0 + (it & (D - 1)) * (kWarp * 2);
      const R yv0 = yr[0];
      const R yv1 = two ? yr[1] : R(0);
      ObsFeat<R> f0, f1;
      R lb[KL];
      em.eval(yv0, yv1, f0, f1, lb, oob);
      R m = lb[0];
#pragma unroll
      for (int l = 1; l < KL; ++l) m = rmax(m, lb[l]);
      m = gmax(m);
      R o[KL], g[KL], qv[KL];
      bool have_g = false;
      const bool first = (t == T - 1);
      R w[KL];
#pragma unroll
      for (int l = 0; l < KL; ++l) w[l] = (finn ? N::fex2(fma(lbn[l], kL2E, -mn * kL2E)) : R(0)) * bt[l];
      R wf[KP];
      gother(w, wf);
#pragma unroll
      for (int l = 0; l < KL; ++l) {
        R acc = Am[0][l] * wf[0];
#pragma unroll
        for (int jx = 1; jx < KP; ++jx) acc = fma(Am[jx][l], wf[jx], acc);
        qv[l] = first ? ((j0 + l < K) ? R(1) : R(0)) : acc;
      }
      if (act) rho = first ? 0.0 : rho + (finn ? (double)(mn * kL2E) : 0.0);
      {
        const R rr = (R)rho;
#pragma unroll
        for (int l = 0; l < KL; ++l) o[l] = first ? R(0) : (rr + N::flg2(qv[l])) * kLN2;
      }
      if (t < H) {
        // combine with alpha~_t: gamma_t and xi_t (pair t, t+1)
        R al[KL];
        LVec<R, KL>::ld(wslot0 + (it & (D - 1)) * (kWarp * KL), al);
        R Zp = R(0);
#pragma unroll
        for (int l = 0; l < KL; ++l) Zp = fma(al[l], qv[l], Zp);
        const R iz = N::frcp(gsum(Zp));
        if (act && wdisc) l2_discard(W + (int64_t)t * wstride + wcol);
        const bool pair = act && !first && t < H - 1;  // (H-1, H) is the forward warp's
#pragma unroll
        for (int l = 0; l < KL; ++l) {
          g[l] = al[l] * qv[l] * iz;
          const R ai = al[l] * iz;
          if (pair) {
#pragma unroll
            for (int jx = 0; jx < KP; ++jx) X[jx][l] = fma(ai, wf[jx], X[jx][l]);
            if (outX && j0 + l < K) {
              R* xr = outX + ((start - b) + t) * (int64_t)(K * K);
              for (int jx = 0; jx < KP; ++jx)
                if (perm(jx) < K) xr[(j0 + l) * K + perm(jx)] = ai * Am[jx][l] * wf[jx];
            }
          }
        }
        have_g = act;
      }
      if (--ncd == 0) {  // warp-uniform renormalisation schedule
        ncd = nn;
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
        if (t >= H) LVec<R, KL>::st(W + (int64_t)t * wstride + wcol, bt);
        st_row(stOq + (t & (kMSlab - 1)) * K, o);
        if (have_g) {
          if (outG) st_row(stGq + (t & (kMSlab - 1)) * K, g);
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
#pragma unroll
        for (int l = 0; l < KL; ++l) lbn[l] = lb[l];
        mn = m;
        finn = m > N::ninf();
      }
      issue_y(it + D, y0p - (it + D), y1p - (it + D));
      if (t < H) {
        issue_w(it + D, wpf);
        wpf -= wstride;
      }
      cp_async_commit();
      if ((t & (kMSlab - 1)) == 0) {
        flush(outO, stO, t, t, t + kMSlab);
        if (t < H) flush(outG, stG, t, t, H);
      }
    }
    cp_async_wait_all();
  }

  // ---- per-sequence results ----------------------------------------------
  // xi: forward lanes own columns, backward lanes own rows; merge in smem.
  R* xq = xis + q * K * K;
  if (fwd) {
#pragma unroll
    for (int i = 0; i < KP; ++i)
#pragma unroll
      for (int l = 0; l < KL; ++l)
        if (perm(i) < K && j0 + l < K) xq[perm(i) * K + j0 + l] = X[i][l];
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
        for (int jx = 0; jx < KP; ++jx) {
          const int j = perm(jx);
          if (j >= K) continue;
          row[i * K + j] = ((double)X[jx][l] + (double)xq[i * K + j]) * (double)Am[jx][l];
        }
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
