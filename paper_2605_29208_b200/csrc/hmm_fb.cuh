// hmm_fb.cuh — fused batched forward-backward + E-step statistics, K <= 8.
//
// One warp owns one sequence.  The sequence is cut into 32 contiguous chunks,
// one per lane, and the serial log-space recursions of the reference
//   inference.py:129-137 (_forward_from_log_b)
//   inference.py:140-146 (_backward_from_log_b)
// are evaluated as an associative scan over chunk transfer operators:
//
//  phase 1  each lane builds M_c = prod_{t in chunk} A diag(b_t) in linear
//           space (power-of-two normalised, log offset kept in fp64).  The
//           same operator serves both directions: alpha_end = alpha_start M_c
//           and beta_start = M_c beta_end.
//  phase 2  Hillis-Steele scans over the 32 lanes (warp shuffles) give every
//           lane its entering forward vector and exiting backward vector, and
//           the sequence log-likelihood.
//  phase 3  each lane re-runs its chunk: forward writes log_alpha and keeps
//           the max-normalised alpha in shared memory; backward writes
//           log_beta and gamma and accumulates xi totals, gamma totals and
//           the family sufficient statistics (training.py:199-210,221-222).
//
// Outputs are staged per lane in shared memory and written as contiguous
// rows, so every global store instruction is coalesced.  Per-step carried
// state is (linear vector with max 1, fp64 log offset): this keeps relative
// precision in fp32 where carrying raw log values of magnitude ~1e3 would not
// (SURVEY.md §7.3-2).
#pragma once

#include "hmm_common.cuh"

namespace lhmm {

constexpr int kSlab = 4;  // output staging depth (steps per lane per flush)

struct FBArgs {
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
  void* alpha_ws;  // global alpha store [N, K] when kGlobal
  int64_t stats_width;
  int L_align;
  int Lmax;
  int stream_fams;  // bitmask of families present (for kCfgMixed)
  // shared-memory carve (elements of R, per warp)
  int y_pitch;
  int a_pitch;
  int s_pitch;
  int warp_smem_elems;
};

template <typename R, int K>
struct VecIO {
  // Vector width (elements) for a K-vector of R in shared memory.
  static constexpr int BYTES = K * (int)sizeof(R);
  static constexpr int VE = (BYTES % 16 == 0) ? 16 / (int)sizeof(R)
                            : (BYTES % 8 == 0) ? 8 / (int)sizeof(R)
                                               : 1;
  static __device__ __forceinline__ void st(R* p, const R (&v)[K]) {
    if constexpr (sizeof(R) == 4 && VE == 4) {
#pragma unroll
      for (int i = 0; i < K; i += 4)
        *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else if constexpr (sizeof(R) == 4 && VE == 2) {
#pragma unroll
      for (int i = 0; i < K; i += 2) *reinterpret_cast<float2*>(p + i) = make_float2(v[i], v[i + 1]);
    } else if constexpr (sizeof(R) == 8 && VE == 2) {
#pragma unroll
      for (int i = 0; i < K; i += 2)
        *reinterpret_cast<double2*>(p + i) = make_double2((double)v[i], (double)v[i + 1]);
    } else {
#pragma unroll
      for (int i = 0; i < K; ++i) p[i] = v[i];
    }
  }
  static __device__ __forceinline__ void ld(const R* p, R (&v)[K]) {
    if constexpr (sizeof(R) == 4 && VE == 4) {
#pragma unroll
      for (int i = 0; i < K; i += 4) {
        float4 q = *reinterpret_cast<const float4*>(p + i);
        v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
      }
    } else if constexpr (sizeof(R) == 4 && VE == 2) {
#pragma unroll
      for (int i = 0; i < K; i += 2) {
        float2 q = *reinterpret_cast<const float2*>(p + i);
        v[i] = q.x; v[i + 1] = q.y;
      }
    } else if constexpr (sizeof(R) == 8 && VE == 2) {
#pragma unroll
      for (int i = 0; i < K; i += 2) {
        double2 q = *reinterpret_cast<const double2*>(p + i);
        v[i] = (R)q.x; v[i + 1] = (R)q.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < K; ++i) v[i] = p[i];
    }
  }
};

// Write the staged rows of a slab window to global memory.  Row c (lane c's
// chunk) covers global steps c*L + sb + [0, n_c); its bytes are contiguous in
// the [N, K] output, so the 32 lanes copy 16-byte units row by row.  The row
// geometry is fixed per sequence and precomputed once (FlushPlan).
template <typename R, int K>
struct FlushPlan {
  static constexpr int ROW = kSlab * K;                 // elements per full row
  static constexpr int EPV = 16 / (int)sizeof(R);       // elements per 16 B
  static constexpr int VPR = (ROW + EPV - 1) / EPV;     // 16 B units per row
  static constexpr int NIT = (kWarp * VPR + kWarp - 1) / kWarp;
  int64_t gbase[NIT];  // element offset of (row start, unit) in the output
  int soff[NIT];       // element offset in the stage buffer
  int clen[NIT];       // chunk length of the row (steps)
  int e0[NIT];         // element offset of the unit inside the row
  bool vec_ok;
  __device__ __forceinline__ void init(int lane, int64_t start, int L, int T, int s_pitch, bool vok) {
    vec_ok = vok;
#pragma unroll
    for (int k = 0; k < NIT; ++k) {
      const int v = lane + kWarp * k;
      const int c = v / VPR, vi = v % VPR;
      e0[k] = vi * EPV;
      int cl = T - c * L;
      cl = cl < 0 ? 0 : (cl > L ? L : cl);
      clen[k] = c < kWarp ? cl : 0;
      gbase[k] = (start + (int64_t)c * L) * K + e0[k];
      soff[k] = c * s_pitch + e0[k];
    }
  }
};

template <typename R, int K>
__device__ __forceinline__ void flush_slab(R* __restrict__ out, const R* __restrict__ stage,
                                           const FlushPlan<R, K>& fp, int s_pitch, int64_t start,
                                           int L, int T, int sb, int lane) {
  typedef FlushPlan<R, K> P;
  if (fp.vec_ok) {
#pragma unroll
    for (int k = 0; k < P::NIT; ++k) {
      int n = fp.clen[k] - sb;
      n = n > kSlab ? kSlab : n;
      const int nel = n * K - fp.e0[k];
      if (nel <= 0) continue;
      R* dst = out + fp.gbase[k] + (int64_t)sb * K;
      const R* src = stage + fp.soff[k];
      if (nel >= P::EPV) {
        *reinterpret_cast<float4*>(dst) = *reinterpret_cast<const float4*>(src);
      } else {
        for (int e = 0; e < nel; ++e) dst[e] = src[e];
      }
    }
  } else {
    constexpr int ROW = P::ROW;
#pragma unroll 1
    for (int v = lane; v < kWarp * ROW; v += kWarp) {
      const int c = v / ROW, e = v % ROW;
      const int t0 = c * L + sb;
      int n = T - t0;
      n = n < 0 ? 0 : (n > kSlab ? kSlab : n);
      const int ccap = (c + 1) * L - t0;
      if (n > ccap) n = ccap;
      if (e < n * K) out[(start + t0) * K + e] = stage[c * s_pitch + e];
    }
  }
}

// Matrix product Z = X * Y (K x K), FMA.
// sum_i a_i b_i over the K states, in index order.  For K = 2 the two
// products are rounded separately and added (no contraction), so relabelling
// the two states permutes the result bit for bit -- the exact label-swap
// equivariance the reference's numpy arithmetic has (test_training.py:177-197).
template <typename R, int K, typename F>
__device__ __forceinline__ R sdot(F ab) {
  if constexpr (K == 2) {
    R a0, b0, a1, b1;
    ab(0, a0, b0);
    ab(1, a1, b1);
    return Num<R>::add(Num<R>::mul(a0, b0), Num<R>::mul(a1, b1));
  } else {
    R a, b;
    ab(0, a, b);
    R acc = a * b;
#pragma unroll
    for (int i = 1; i < K; ++i) {
      ab(i, a, b);
      acc = fma(a, b, acc);
    }
    return acc;
  }
}

template <typename R, int K>
__device__ __forceinline__ void matmul(const R (&X)[K][K], const R (&Y)[K][K], R (&Z)[K][K]) {
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) {
      Z[r][c] = sdot<R, K>([&](int i, R& a, R& b) { a = X[r][i]; b = Y[i][c]; });
    }
}

template <typename R, int K>
__device__ __forceinline__ void normalise_mat(R (&Z)[K][K], double& off) {
  R m = Z[0][0];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) m = rmax(m, Z[r][c]);
  if (m > R(0)) {
    R s = Num<R>::pow2_normaliser(m, off);
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
      for (int c = 0; c < K; ++c) Z[r][c] *= s;
  } else {
    off = -CUDART_INF;
  }
}

template <typename R, int K>
__device__ __forceinline__ void normalise_vec(R (&v)[K], double& off) {
  R m = v[0];
#pragma unroll
  for (int i = 1; i < K; ++i) m = rmax(m, v[i]);
  if (m > R(0)) {
    R s = Num<R>::pow2_normaliser(m, off);
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] *= s;
  } else {
    off = -CUDART_INF;
  }
}

// Power-of-two normalisation with the offset kept in log2 units (exact).
template <typename R, int K>
__device__ __forceinline__ void normalise_mat2(R (&Z)[K][K], double& off2) {
  R m = Z[0][0];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) m = rmax(m, Z[r][c]);
  if (m > R(0)) {
    int e;
    const R s = Num<R>::pow2_scale(m, e);
    off2 += (double)e;
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
      for (int c = 0; c < K; ++c) Z[r][c] *= s;
  } else {
    off2 = -CUDART_INF;
  }
}

template <typename R, int K>
__device__ __forceinline__ void normalise_vec2(R (&v)[K], double& off2) {
  R m = v[0];
#pragma unroll
  for (int i = 1; i < K; ++i) m = rmax(m, v[i]);
  if (m > R(0)) {
    int e;
    const R s = Num<R>::pow2_scale(m, e);
    off2 += (double)e;
#pragma unroll
    for (int i = 0; i < K; ++i) v[i] *= s;
  } else {
    off2 = -CUDART_INF;
  }
}

template <typename R, int K>
__device__ __forceinline__ void shfl_mat(R (&Z)[K][K], double& off, const R (&X)[K][K], double xo,
                                         int delta, bool up) {
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c)
      Z[r][c] = up ? __shfl_up_sync(kFull, X[r][c], delta) : __shfl_down_sync(kFull, X[r][c], delta);
  off = up ? __shfl_up_sync(kFull, xo, delta) : __shfl_down_sync(kFull, xo, delta);
}

// ---------------------------------------------------------------------------
// Emission evaluation for all states at one step (fast contract).
// ---------------------------------------------------------------------------
// Column-scaled transition matrix for the linear scaled recursions:
// Ahat_ij = A_ij / c_j with c_j = max_i A_ij, and lc_j = log(c_j) in the
// requested base (-inf for an all-zero column, whose Ahat column is zero).
// The emission shift of every step is then max_j (log b_j + lc_j) instead of
// max_j log b_j, i.e. it follows the best state that can be ENTERED: a
// structurally unreachable state with an overwhelming emission no longer
// pushes the reachable terms below the floating-point range (the failure the
// log-space reference never has, inference.py:129-146).  b_j A_ij is
// unchanged: 2^(u_j + lc_j - m) Ahat_ij = 2^(u_j - m) A_ij.
// Every warp runs this prologue for its own sequence, so it is kept cheap:
// one reciprocal and one log per column, in the recursion's precision (an
// error of a few ulps in the scale multiplies a whole column of b_j A_ij by
// the same factor 1 + O(eps_R): far inside the posterior tolerances).
template <typename R, int K>
__device__ __forceinline__ void load_colscaled(const loghmm_model_t* __restrict__ md, R (&Am)[K][K],
                                               R (&lc)[K], double base_log2) {
#pragma unroll
  for (int j = 0; j < K; ++j) {
    R c = R(0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      Am[i][j] = (R)md->A[i * K + j];
      c = c > Am[i][j] ? c : Am[i][j];
    }
    const bool nz = c > R(0);
    const R rc = nz ? Num<R>::frcp(c) : R(0);
    if constexpr (sizeof(R) == 4)
      lc[j] = nz ? Num<R>::flg2(c) * (R)base_log2 : Num<R>::ninf();
    else
      lc[j] = nz ? log2(c) * base_log2 : Num<R>::ninf();
#pragma unroll
    for (int i = 0; i < K; ++i) Am[i][j] *= rc;
  }
}

template <typename R, int K, int CFG>
struct Emit {
  EmP<R> e0[K];
  EmP<R> e1[K];
  int stream_fams;
  const double* lut;
  int lut_n;

  __device__ __forceinline__ void load(const loghmm_model_t* m, int n_streams, int fams,
                                       const double* lut_, int lut_n_) {
#pragma unroll
    for (int j = 0; j < K; ++j) {
      e0[j] = load_emission<R>(m->em[0][j]);
      if (CFG == kCfgGammaVM || (CFG == kCfgMixed && n_streams > 1))
        e1[j] = load_emission<R>(m->em[1][j]);
      else
        e1[j].fam = LOGHMM_FAM_NONE;
    }
    stream_fams = fams;
    lut = lut_;
    lut_n = lut_n_;
  }

  // logb[j] for observation(s) y0 (and y1); also fills the features used by
  // the statistics.
  __device__ __forceinline__ void eval(R y0, R y1, ObsFeat<R>& f0, ObsFeat<R>& f1, R (&lb)[K],
                                       bool& oob) const {
    if (CFG == kCfgGammaVM) {
      obs_features<R, kCfgGamma>(f0, y0, lut, lut_n, oob, 0);
      obs_features<R, kCfgVonMises>(f1, y1, lut, lut_n, oob, 0);
#pragma unroll
      for (int j = 0; j < K; ++j)
        lb[j] = fast_logb_fam<R, LOGHMM_FAM_GAMMA>(e0[j], f0) +
                fast_logb_fam<R, LOGHMM_FAM_VON_MISES>(e1[j], f1);
    } else if (CFG == kCfgMixed) {
      obs_features<R, kCfgMixed>(f0, y0, lut, lut_n, oob, stream_fams & 0xffff);
      obs_features<R, kCfgMixed>(f1, y1, lut, lut_n, oob, stream_fams >> 16);
#pragma unroll
      for (int j = 0; j < K; ++j) lb[j] = fast_logb_rt<R>(e0[j], f0) + fast_logb_rt<R>(e1[j], f1);
    } else {
      obs_features<R, CFG>(f0, y0, lut, lut_n, oob, 0);
#pragma unroll
      for (int j = 0; j < K; ++j) lb[j] = fast_logb_fam<R, CFG>(e0[j], f0);
    }
  }
};

// Family sufficient statistics of one state at one step (slots in acc[6]).
//  gaussian : w, w*d, w*d^2                 d = y - mu_current   (fit_gaussian :632)
//  poisson  : w, w*y, [w>0 & invalid]                             (fit_poisson :658)
//  gamma    : w, w*d, w*d^2, w*log y, [w>0 & y<=0]  d = y - mean  (fit_gamma_nr :764)
//  von_mises: w, w*sin y, w*cos y, [w>0 & !finite]                (fit_vonmises :874)
//  student_t: w, w*u, w*u*d, w*u*d^2, w*(log u - u)  at current params,
//             u = (nu+1)/(nu+z^2), d = y - mu                     (ECME pass A :1043-1054)
template <typename R, int FAM>
__device__ __forceinline__ void stat_acc(R (&acc)[LOGHMM_NSLOT], R w, const EmP<R>& p,
                                         const ObsFeat<R>& f) {
  const bool pos = w > R(0);
  if (FAM == LOGHMM_FAM_GAUSSIAN) {
    R d = f.y - p.q[0];
    R wd = w * d;
    acc[0] += w;
    acc[1] += wd;
    acc[2] = fma(wd, d, acc[2]);
  } else if (FAM == LOGHMM_FAM_POISSON) {
    acc[0] += w;
    if (f.pois_ok) acc[1] = fma(w, f.y, acc[1]);
    else if (pos) acc[2] += R(1);
  } else if (FAM == LOGHMM_FAM_GAMMA) {
    acc[0] += w;
    if (f.y > R(0)) {
      R d = f.y - p.q[3];
      R wd = w * d;
      acc[1] += wd;
      acc[2] = fma(wd, d, acc[2]);
      acc[3] = fma(w, f.logy, acc[3]);
    } else if (pos) {
      acc[4] += R(1);
    }
  } else if (FAM == LOGHMM_FAM_VON_MISES) {
    acc[0] += w;
    if (isfinite(f.y)) {
      acc[1] = fma(w, f.siny, acc[1]);
      acc[2] = fma(w, f.cosy, acc[2]);
    } else if (pos) {
      acc[3] += R(1);
    }
  } else if (FAM == LOGHMM_FAM_STUDENT_T) {
    R d = f.y - p.q[0];
    R z = d * p.q[1];
    R u = (p.q[5] + R(1)) / (p.q[5] + z * z);
    R wu = w * u;
    acc[0] += w;
    acc[1] += wu;
    acc[2] = fma(wu, d, acc[2]);
    acc[3] = fma(wu * d, d, acc[3]);
    if (pos) acc[4] = fma(w, Num<R>::alog(u) - u, acc[4]);
  }
}

template <typename R>
__device__ __forceinline__ void stat_acc_rt(R (&acc)[LOGHMM_NSLOT], R w, const EmP<R>& p,
                                            const ObsFeat<R>& f) {
  switch (p.fam) {
    case LOGHMM_FAM_GAUSSIAN: stat_acc<R, LOGHMM_FAM_GAUSSIAN>(acc, w, p, f); break;
    case LOGHMM_FAM_STUDENT_T: stat_acc<R, LOGHMM_FAM_STUDENT_T>(acc, w, p, f); break;
    case LOGHMM_FAM_GAMMA: stat_acc<R, LOGHMM_FAM_GAMMA>(acc, w, p, f); break;
    case LOGHMM_FAM_VON_MISES: stat_acc<R, LOGHMM_FAM_VON_MISES>(acc, w, p, f); break;
    case LOGHMM_FAM_POISSON: stat_acc<R, LOGHMM_FAM_POISSON>(acc, w, p, f); break;
    case LOGHMM_FAM_NONE: break;
    // families 6..15: only the state's total weight (the collapse guard,
    // training.py:139); their fits run weighted-sample passes (hmm_extfit.cuh)
    default: acc[0] += w; break;
  }
}

template <int CFG>
struct CfgTraits {
  static constexpr int S = (CFG == kCfgGammaVM || CFG == kCfgMixed) ? 2 : 1;  // stat streams
  static constexpr int F0 = CFG == kCfgGauss     ? LOGHMM_FAM_GAUSSIAN
                            : CFG == kCfgStudent  ? LOGHMM_FAM_STUDENT_T
                            : CFG == kCfgGamma    ? LOGHMM_FAM_GAMMA
                            : CFG == kCfgVonMises ? LOGHMM_FAM_VON_MISES
                            : CFG == kCfgPoisson  ? LOGHMM_FAM_POISSON
                            : CFG == kCfgGammaVM  ? LOGHMM_FAM_GAMMA
                                                  : -1;
  static constexpr int F1 = CFG == kCfgGammaVM ? LOGHMM_FAM_VON_MISES : -1;
  static constexpr int NS0 = F0 == LOGHMM_FAM_GAUSSIAN    ? 3
                             : F0 == LOGHMM_FAM_POISSON   ? 3
                             : F0 == LOGHMM_FAM_GAMMA     ? 5
                             : F0 == LOGHMM_FAM_VON_MISES ? 4
                             : F0 == LOGHMM_FAM_STUDENT_T ? 5
                                                          : LOGHMM_NSLOT;
  static constexpr int NS1 = F1 == LOGHMM_FAM_VON_MISES ? 4 : LOGHMM_NSLOT;
};

template <typename R, int K, int CFG>
__device__ __forceinline__ void stats_step(R (&st)[CfgTraits<CFG>::S][K][LOGHMM_NSLOT],
                                           const R (&g)[K], const Emit<R, K, CFG>& em,
                                           const ObsFeat<R>& f0, const ObsFeat<R>& f1) {
  typedef CfgTraits<CFG> TR;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if constexpr (TR::F0 >= 0) {
      stat_acc<R, TR::F0>(st[0][j], g[j], em.e0[j], f0);
    } else {
      stat_acc_rt<R>(st[0][j], g[j], em.e0[j], f0);
    }
    if constexpr (TR::S > 1) {
      if constexpr (TR::F1 >= 0) {
        stat_acc<R, TR::F1>(st[1][j], g[j], em.e1[j], f1);
      } else {
        stat_acc_rt<R>(st[1][j], g[j], em.e1[j], f1);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// The kernel.
// ---------------------------------------------------------------------------
template <typename R, int K, int CFG, bool kGlobal>
__global__ void __launch_bounds__(128, sizeof(R) == 4 ? 4 : 2) fb_small_kernel(const FBArgs a) {
  typedef Num<R> N;
  typedef CfgTraits<CFG> TR;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (b >= a.B) return;

  const int64_t start = a.offsets[b];
  const int T = (int)(a.offsets[b + 1] - start);
  int L = (T + kWarp - 1) / kWarp;
  L = ((L + a.L_align - 1) / a.L_align) * a.L_align;
  if (L < 1) L = 1;
  const int t0 = lane * L;
  const int t1 = min(t0 + L, T);
  const int len = t1 > t0 ? t1 - t0 : 0;

  const R* __restrict__ y0g = reinterpret_cast<const R*>(a.y0) + start;
  const R* __restrict__ y1g = a.y1 ? reinterpret_cast<const R*>(a.y1) + start : nullptr;
  const bool two = (a.n_streams > 1);

  R* wsm = reinterpret_cast<R*>(smem_raw) + (size_t)wib * a.warp_smem_elems;
  R* ybuf0 = wsm;
  R* ybuf1 = ybuf0 + kWarp * a.y_pitch;
  R* stA = ybuf1 + (two ? kWarp * a.y_pitch : 0);
  R* stB = stA + kWarp * a.s_pitch;
  if (kGlobal) {
    stA = wsm;
    stB = stA + kWarp * a.s_pitch;
  }

  // ---- model -------------------------------------------------------------
  const loghmm_model_t* __restrict__ md = a.model;
  R Am[K][K], lcn[K];  // column-scaled A and log c_j (natural log)
  load_colscaled<R, K>(md, Am, lcn, 0.6931471805599453094);
  R minA = R(1);
#pragma unroll
  for (int i = 0; i < K; ++i)
#pragma unroll
    for (int j = 0; j < K; ++j) minA = Am[i][j] < minA ? Am[i][j] : minA;
  R lpi[K];
#pragma unroll
  for (int j = 0; j < K; ++j) lpi[j] = (R)md->log_pi[j];
  Emit<R, K, CFG> em;
  em.load(md, a.n_streams, a.stream_fams, a.lut, a.lut_n);
  // Normalise the operator every `nn` steps: the max entry decays by at most
  // min(A) per step (choose the column of the emission maximum), so nn steps
  // keep it above 2^-100 (fp32) / 2^-900 (fp64).
  int nn = 1;
  if (minA > R(0)) {
    const double lg = -log2((double)minA);
    const double budget = sizeof(R) == 4 ? 100.0 : 900.0;
    nn = lg <= 0.0 ? 8 : (int)fmin(8.0, fmax(1.0, floor(budget / lg)));
  }

  // ---- stage y into shared memory: coalesced batched loads (8 in flight per
  // lane), stored contiguously with one pad element every 32 so lane-strided
  // chunk reads (stride L) hit distinct banks.
  if (!kGlobal) {
    constexpr int UB = 8;
#pragma unroll 1
    for (int base = 0; base < T; base += kWarp * UB) {
      R v0[UB], v1[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int t = base + u * kWarp + lane;
        v0[u] = t < T ? y0g[t] : R(0);
        v1[u] = (two && t < T) ? y1g[t] : R(0);
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        const int t = base + u * kWarp + lane;
        if (t < T) {
          ybuf0[t + (t >> 5)] = v0[u];
          if (two) ybuf1[t + (t >> 5)] = v1[u];
        }
      }
    }
    __syncwarp();
  }
  auto yat0 = [&](int s) -> R {
    const int t = t0 + s;
    return kGlobal ? y0g[t] : ybuf0[t + (t >> 5)];
  };
  auto yat1 = [&](int s) -> R {
    const int t = t0 + s;
    return two ? (kGlobal ? y1g[t] : ybuf1[t + (t >> 5)]) : R(0);
  };

  bool oob = false;
  bool nan_seen = false;
  int dead_t = INT_MAX;

  // All recursions below work in log2 units (ex2/lg2 on the MUFU, offsets
  // exact in base 2); outputs are converted to natural logs when staged.
  constexpr R kL2E = R(1.4426950408889634);
  constexpr R kLN2 = R(0.6931471805599453);
  constexpr double kLN2d = 0.6931471805599453094;

  // ---- phase 1: chunk transfer operator --------------------------------
  R Mop[K][K];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) Mop[r][c] = r == c ? R(1) : R(0);
  double moff = 0.0;  // log2 offset of Mop
  R seed_u[K];        // lane 0: log2(pi) + log2 b_0
#pragma unroll
  for (int j = 0; j < K; ++j) seed_u[j] = N::ninf();
  {
    int cnt = 0;
#pragma unroll 1
    for (int s = 0; s < len; ++s) {
      const int t = t0 + s;
      const R yv0 = yat0(s), yv1 = yat1(s);
      if (isnan(yv0) || isnan(yv1)) nan_seen = true;
      ObsFeat<R> f0, f1;
      R lb[K];
      em.eval(yv0, yv1, f0, f1, lb, oob);
      R m = lb[0];
#pragma unroll
      for (int j = 1; j < K; ++j) m = rmax(m, lb[j]);
      if (!(m > N::ninf())) {
        if (t < dead_t) dead_t = t;
      }
      if (t == 0) {
#pragma unroll
        for (int j = 0; j < K; ++j) seed_u[j] = (lpi[j] + lb[j]) * kL2E;
        continue;
      }
      // shift by the best enterable state (load_colscaled)
#pragma unroll
      for (int j = 0; j < K; ++j) lb[j] += lcn[j];
      m = lb[0];
#pragma unroll
      for (int j = 1; j < K; ++j) m = rmax(m, lb[j]);
      const bool finite_m = m > N::ninf();
      const R m2 = m * kL2E;
      R bt[K];
#pragma unroll
      for (int j = 0; j < K; ++j) bt[j] = finite_m ? N::fex2(fma(lb[j], kL2E, -m2)) : R(0);
      R Nw[K][K];
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) {
          const R acc = sdot<R, K>([&](int i, R& a, R& b) { a = Mop[r][i]; b = Am[i][c]; });
          Nw[r][c] = acc * bt[c];
        }
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) Mop[r][c] = Nw[r][c];
      moff += finite_m ? (double)m2 : -CUDART_INF;
      if (++cnt == nn) {
        cnt = 0;
        normalise_mat2<R, K>(Mop, moff);
      }
    }
    normalise_mat2<R, K>(Mop, moff);
  }

  // ---- phase 2a: forward scan (inclusive prefix of operators) -------------
  R a_in[K];
  double lam_in;
  double LL;
  {
    R Q[K][K];
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
      for (int c = 0; c < K; ++c) Q[r][c] = Mop[r][c];
    double qo = moff;
#pragma unroll 1
    for (int d = 1; d < kWarp; d <<= 1) {
      R P[K][K];
      double po;
      shfl_mat<R, K>(P, po, Q, qo, d, true);
      if (lane >= d) {
        R Z[K][K];
        matmul<R, K>(P, Q, Z);
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
          for (int c = 0; c < K; ++c) Q[r][c] = Z[r][c];
        qo += po;
        normalise_mat2<R, K>(Q, qo);
      }
    }
    // seed vector alpha_0 (lane 0), broadcast
    R sm = seed_u[0];
#pragma unroll
    for (int j = 1; j < K; ++j) sm = rmax(sm, seed_u[j]);
    R sv[K];
    const bool sfin = sm > N::ninf();
#pragma unroll
    for (int j = 0; j < K; ++j) sv[j] = sfin ? N::fex2(seed_u[j] - sm) : R(0);
    double so = sfin ? (double)sm : -CUDART_INF;
#pragma unroll
    for (int j = 0; j < K; ++j) sv[j] = __shfl_sync(kFull, sv[j], 0);
    so = __shfl_sync(kFull, so, 0);
    R v[K];
#pragma unroll
    for (int c = 0; c < K; ++c) {
      v[c] = sdot<R, K>([&](int i, R& a, R& b) { a = sv[i]; b = Q[i][c]; });
    }
    double vo = so + qo;
    normalise_vec2<R, K>(v, vo);
    R vs = v[0];
#pragma unroll
    for (int j = 1; j < K; ++j) vs += v[j];
    double llv = (vo + (double)N::flg2(vs)) * kLN2d;
    if (!(vs > R(0))) llv = -CUDART_INF;
    LL = __shfl_sync(kFull, llv, kWarp - 1);
#pragma unroll
    for (int j = 0; j < K; ++j) a_in[j] = __shfl_up_sync(kFull, v[j], 1);
    lam_in = __shfl_up_sync(kFull, vo, 1);
  }

  // ---- phase 2b: backward scan (inclusive suffix of operators) ------------
  R b_ex[K];  // beta~ at the chunk's last step (linear, pow2-normalised)
  double rho_ex;  // log2 offset
  {
    R S[K][K];
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
      for (int c = 0; c < K; ++c) S[r][c] = Mop[r][c];
    double so = moff;
#pragma unroll 1
    for (int d = 1; d < kWarp; d <<= 1) {
      R Y[K][K];
      double yo;
      shfl_mat<R, K>(Y, yo, S, so, d, false);
      if (lane + d < kWarp) {
        R Z[K][K];
        matmul<R, K>(S, Y, Z);
#pragma unroll
        for (int r = 0; r < K; ++r)
#pragma unroll
          for (int c = 0; c < K; ++c) S[r][c] = Z[r][c];
        so += yo;
        normalise_mat2<R, K>(S, so);
      }
    }
    R z[K];
#pragma unroll
    for (int r = 0; r < K; ++r) {
      R acc = S[r][0];
#pragma unroll
      for (int c = 1; c < K; ++c) acc += S[r][c];
      z[r] = acc;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) b_ex[j] = __shfl_down_sync(kFull, z[j], 1);
    rho_ex = __shfl_down_sync(kFull, so, 1);
    if (lane == kWarp - 1) {
#pragma unroll
      for (int j = 0; j < K; ++j) b_ex[j] = R(1);
      rho_ex = 0.0;
    }
    normalise_vec2<R, K>(b_ex, rho_ex);
  }

  // beta~ store: global workspace, per sequence [L][32 lanes][K] so every
  // per-step access of the warp is one contiguous 32*K row.  Written by the
  // backward re-sweep and read once by the forward re-sweep shortly after, so
  // it lives in L2; each line is discarded after its read.
  constexpr int AW_STEP = kWarp * K;
  R* aw = reinterpret_cast<R*>(a.alpha_ws) + b * (int64_t)a.Lmax * AW_STEP + lane * K;
  constexpr bool kDisc = (128 % (K * (int)sizeof(R))) == 0;
  const bool disc_lane = kDisc && (((lane * K * (int)sizeof(R)) & 127) == 0);
  const bool vec_ok = ((start * K * (int64_t)sizeof(R)) % 16 == 0) &&
                      ((L * K * (int)sizeof(R)) % 16 == 0);
  FlushPlan<R, K> fplan;
  fplan.init(lane, start, L, T, a.s_pitch, vec_ok);

  // ---- phase 3a: backward re-sweep (linear), writes log_beta, keeps beta~ --
  R* __restrict__ outA = reinterpret_cast<R*>(a.log_alpha);
  R* __restrict__ outB = reinterpret_cast<R*>(a.log_beta);
  R* __restrict__ outG = reinterpret_cast<R*>(a.gamma);
  R* __restrict__ outX = reinterpret_cast<R*>(a.xi);
  {
    R bt[K];
    double rho = rho_ex;
#pragma unroll
    for (int j = 0; j < K; ++j) bt[j] = b_ex[j];
    const int s_top = len - 1;
    int cnt = 0;
#pragma unroll 1
    for (int s = L - 1; s >= 0; --s) {
      if (s == s_top) {
        VecIO<R, K>::st(aw + s * AW_STEP, bt);
        if (outB) {
          const R rr = (R)rho;
          R o[K];
#pragma unroll
          for (int j = 0; j < K; ++j) o[j] = (rr + N::flg2(bt[j])) * kLN2;
          VecIO<R, K>::st(stA + lane * a.s_pitch + (s % kSlab) * K, o);
        }
      } else if (s < s_top) {
        // beta_s = A (b_{s+1} . beta_{s+1})
        ObsFeat<R> f0, f1;
        R lb[K];
        em.eval(yat0(s + 1), yat1(s + 1), f0, f1, lb, oob);
#pragma unroll
        for (int j = 0; j < K; ++j) lb[j] += lcn[j];  // (load_colscaled)
        R m = lb[0];
#pragma unroll
        for (int j = 1; j < K; ++j) m = rmax(m, lb[j]);
        const bool fin = m > N::ninf();
        const R m2 = m * kL2E;
        R w[K];
#pragma unroll
        for (int j = 0; j < K; ++j) w[j] = (fin ? N::fex2(fma(lb[j], kL2E, -m2)) : R(0)) * bt[j];
        R q[K];
#pragma unroll
        for (int i = 0; i < K; ++i) {
          R acc = sdot<R, K>([&](int j, R& a, R& b) { a = Am[i][j]; b = w[j]; });
          q[i] = acc;
        }
        rho += fin ? (double)m2 : 0.0;
        if (outB) {
          const R rr = (R)rho;
          R o[K];
#pragma unroll
          for (int j = 0; j < K; ++j) o[j] = (rr + N::flg2(q[j])) * kLN2;
          VecIO<R, K>::st(stA + lane * a.s_pitch + (s % kSlab) * K, o);
        }
#pragma unroll
        for (int j = 0; j < K; ++j) bt[j] = q[j];
        if (++cnt == nn) {
          cnt = 0;
          normalise_vec2<R, K>(bt, rho);
        }
        VecIO<R, K>::st(aw + s * AW_STEP, bt);
      }
      if ((s % kSlab) == 0 && outB) {
        __syncwarp();
        flush_slab<R, K>(outB, stA, fplan, a.s_pitch, start, L, T, s, lane);
        __syncwarp();
      }
    }
  }
  __syncwarp();

  // ---- phase 3b: forward re-sweep fused with posteriors and statistics -----
  R X[K][K];
  R gtot[K], g0[K];
  R st[TR::S][K][LOGHMM_NSLOT];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    gtot[i] = R(0);
    g0[i] = R(0);
#pragma unroll
    for (int j = 0; j < K; ++j) X[i][j] = R(0);
#pragma unroll
    for (int s = 0; s < TR::S; ++s)
#pragma unroll
      for (int q = 0; q < LOGHMM_NSLOT; ++q) st[s][i][q] = R(0);
  }
  {
    R av[K];
    double lam = lam_in;
#pragma unroll
    for (int j = 0; j < K; ++j) av[j] = a_in[j];
    int cnt = 0;
    // beta~ prefetch ring (cp.async, kBD steps ahead) in this warp's stage area
    constexpr int kBD = 8;
    constexpr int BB = K * (int)sizeof(R);
    R* bring = stB + kWarp * a.s_pitch + lane * K;  // [kBD][32][K]
    auto issue_b = [&](int s2) {
      const bool ok = s2 < len;
      R* dst = bring + (s2 & (kBD - 1)) * AW_STEP;
      const R* src = ok ? aw + s2 * AW_STEP : aw;
      if constexpr (BB == 4 || BB == 8 || BB == 16) {
        cp_async<BB>(dst, src, ok);
      } else {
#pragma unroll
        for (int j = 0; j < K; ++j) cp_async<sizeof(R)>(dst + j, src + j, ok);
      }
    };
#pragma unroll 1
    for (int s2 = 0; s2 < kBD; ++s2) {
      issue_b(s2);
      cp_async_commit();
    }
#pragma unroll 1
    for (int s = 0; s < L; ++s) {
      cp_async_wait<kBD - 1>();
      const int t = t0 + s;
      if (s < len) {
        ObsFeat<R> f0, f1;
        R lb[K];
        em.eval(yat0(s), yat1(s), f0, f1, lb, oob);
        R bet[K];
#pragma unroll
        for (int j = 0; j < K; ++j) bet[j] = bring[(s & (kBD - 1)) * AW_STEP + j];
        if (disc_lane) l2_discard(aw + s * AW_STEP);
        R g[K];
        if (t == 0) {
          R u[K];
#pragma unroll
          for (int j = 0; j < K; ++j) u[j] = (lpi[j] + lb[j]) * kL2E;
          R M = u[0];
#pragma unroll
          for (int j = 1; j < K; ++j) M = rmax(M, u[j]);
          const bool fin = M > N::ninf();
          if (outA) {
            R o[K];
#pragma unroll
            for (int j = 0; j < K; ++j) o[j] = u[j] * kLN2;
            VecIO<R, K>::st(stA + lane * a.s_pitch + (s % kSlab) * K, o);
          }
#pragma unroll
          for (int j = 0; j < K; ++j) av[j] = fin ? N::fex2(u[j] - M) : R(0);
          lam = fin ? (double)M : -CUDART_INF;
          R Z = R(0);
#pragma unroll
          for (int j = 0; j < K; ++j) {
            g[j] = av[j] * bet[j];
            Z += g[j];
          }
          const R iz = N::frcp(Z);
#pragma unroll
          for (int j = 0; j < K; ++j) g[j] *= iz;
#pragma unroll
          for (int j = 0; j < K; ++j) g0[j] = g[j];
        } else {
#pragma unroll
          for (int j = 0; j < K; ++j) lb[j] += lcn[j];  // (load_colscaled)
          R m = lb[0];
#pragma unroll
          for (int j = 1; j < K; ++j) m = rmax(m, lb[j]);
          const bool fin = m > N::ninf();
          const R m2 = m * kL2E;
          R bb[K], p[K];
#pragma unroll
          for (int j = 0; j < K; ++j) bb[j] = fin ? N::fex2(fma(lb[j], kL2E, -m2)) : R(0);
#pragma unroll
          for (int c = 0; c < K; ++c) {
            R acc = sdot<R, K>([&](int i, R& a, R& b) { a = av[i]; b = Am[i][c]; });
            p[c] = acc;
          }
          if (outA) {
            const R lr = (R)lam;
            R o[K];
#pragma unroll
            for (int j = 0; j < K; ++j) o[j] = fma(lb[j], kL2E, lr + N::flg2(p[j])) * kLN2;
            VecIO<R, K>::st(stA + lane * a.s_pitch + (s % kSlab) * K, o);
          }
          // pair (t-1, t): xi_{t-1}(i,j) = a_{t-1}[i] A_ij bb_j beta~_t[j] / Z
          R v[K];
#pragma unroll
          for (int j = 0; j < K; ++j) v[j] = bb[j] * bet[j];
          const R Z = sdot<R, K>([&](int j, R& a, R& b) { a = p[j]; b = v[j]; });
          const R iz = N::frcp(Z);
          R cv[K];
#pragma unroll
          for (int j = 0; j < K; ++j) {
            cv[j] = v[j] * iz;
            g[j] = p[j] * cv[j];
          }
#pragma unroll
          for (int i = 0; i < K; ++i)
#pragma unroll
            for (int j = 0; j < K; ++j) X[i][j] = fma(av[i], cv[j], X[i][j]);
          if (outX) {
            R* xr = outX + ((start - b) + (t - 1)) * (int64_t)(K * K);
#pragma unroll
            for (int i = 0; i < K; ++i)
#pragma unroll
              for (int j = 0; j < K; ++j) xr[i * K + j] = av[i] * Am[i][j] * cv[j];
          }
#pragma unroll
          for (int j = 0; j < K; ++j) av[j] = p[j] * bb[j];
          lam += fin ? (double)m2 : 0.0;
          if (++cnt == nn) {
            cnt = 0;
            normalise_vec2<R, K>(av, lam);
          }
        }
        if (outG) VecIO<R, K>::st(stB + lane * a.s_pitch + (s % kSlab) * K, g);
        stats_step<R, K, CFG>(st, g, em, f0, f1);
        if (t < T - 1) {
#pragma unroll
          for (int j = 0; j < K; ++j) gtot[j] += g[j];
        }
      }
      issue_b(s + kBD);
      cp_async_commit();
      if (((s % kSlab) == kSlab - 1 || s == L - 1) && (outA || outG)) {
        __syncwarp();
        const int sb = s - (s % kSlab);
        if (outA) flush_slab<R, K>(outA, stA, fplan, a.s_pitch, start, L, T, sb, lane);
        if (outG) flush_slab<R, K>(outG, stB, fplan, a.s_pitch, start, L, T, sb, lane);
        __syncwarp();
      }
    }
  }

  cp_async_wait_all();

  // ---- reductions and per-sequence outputs --------------------------------
  const int dead_all = (int)warp_min_ll((long long)dead_t);
  const unsigned nanb = __ballot_sync(kFull, nan_seen);
  const unsigned oobb = __ballot_sync(kFull, oob);
  if (lane == 0) {
    a.ll[b] = LL;
    if (a.flags) {
      a.flags[2 * b] = dead_all == INT_MAX ? -1 : (int64_t)dead_all;
      a.flags[2 * b + 1] = (nanb ? 1 : 0) | (oobb ? 2 : 0);
    }
  }
  if (a.partials) {
    double* row = a.partials + b * a.stats_width;
    int idx = 0;
    // xi totals: multiply by A after the lane reduction
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const R v = warp_sum(X[i][j]);
        if (lane == (idx & 31)) row[idx] = (double)v * (double)Am[i][j];
        ++idx;
      }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const R v = warp_sum(gtot[j]);
      if (lane == (idx & 31)) row[idx] = (double)v;
      ++idx;
    }
#pragma unroll
    for (int j = 0; j < K; ++j) {
      const R v = __shfl_sync(kFull, g0[j], 0);
      if (lane == (idx & 31)) row[idx] = (double)v;
      ++idx;
    }
#pragma unroll
    for (int s = 0; s < TR::S; ++s)
#pragma unroll
      for (int j = 0; j < K; ++j)
#pragma unroll
        for (int q = 0; q < LOGHMM_NSLOT; ++q) {
          const int ns = s == 0 ? TR::NS0 : TR::NS1;
          R v = R(0);
          if (q < ns) v = warp_sum(st[s][j][q]);
          if (lane == (idx & 31)) row[idx] = (double)v;
          ++idx;
        }
    // pad the unused second stream
    for (; idx < a.stats_width; ++idx)
      if (lane == (idx & 31)) row[idx] = 0.0;
  }
}

}  // namespace lhmm
