// hmm_fbc.cuh — batched forward-backward for equal-length sequences, K <= 8:
// chunk operators + scan, then a meet-in-the-middle re-sweep inside each chunk.
//
// Same outputs and statistics as hmm_fb.cuh (inference.py:129-188,
// training.py:187-210); this is the decomposition used for [B, T] batches
// whose length splits into C <= 32 chunks of L steps (L a multiple of 8).
//
//   pass 1  one warp per sequence, lane c owns chunk [cL, cL+L): it builds the
//           chunk transfer operator M_c = prod A diag(b_t) (linear, power-of-two
//           normalised, log2 offset), K^3 FMA per step, nothing stored.
//   scan    Hillis-Steele over the lanes (shuffles) gives each lane its entering
//           forward vector alpha~_{cL-1}, its exiting backward vector
//           beta~_{cL+L-1} and the sequence log-likelihood.
//   pass 2  each lane runs the forward recursion up its chunk and the backward
//           recursion down it IN THE SAME LOOP (two independent dependency
//           chains per iteration).  In the first half each direction parks its
//           normalised vector in shared memory; in the second half each one
//           meets the other's parked vectors and forms gamma, the xi totals and
//           the family statistics on the fly.  Every emission is evaluated once
//           per direction; no vector ever leaves the SM.
//
// Outputs (log_alpha, log_beta, gamma) are staged per lane as 4-step slabs in
// shared memory and written by the whole warp as 16-byte coalesced units.
// All recursions run in log2 units (MUFU ex2/lg2); carried state is a linear
// vector plus a log2 offset, which keeps fp32 relative precision (SURVEY.md
// §7.3-2).  The Gaussian emission is two FMAs per state in that form.
#pragma once

#include <type_traits>

#include "hmm_fb.cuh"

namespace lhmm {

struct FBCArgs {
  const loghmm_model_t* model;
  const void* y0;
  const void* y1;
  int64_t B;
  int T;  // common sequence length, T = C * L
  int L;  // chunk length, multiple of 8
  const double* lut;
  int lut_n;
  int n_streams;
  int stream_fams;
  void* log_alpha;
  void* log_beta;
  void* gamma;
  double* ll;
  double* partials;
  int64_t* flags;
  int64_t stats_width;
  int tm_cols;  // tensor-memory columns per CTA (fp32 park)
};

template <typename R, int K>
struct FBCGeom {
  static constexpr int VB = K * (int)sizeof(R);  // bytes of one state vector
  static constexpr int ROWB = 4 * VB;            // one lane's 4-step slab (multiple of 16)
  static constexpr int PITCHB = ((ROWB / 16) % 2 == 0) ? ROWB + 16 : ROWB;
  static constexpr int PITCH = PITCHB / (int)sizeof(R);  // elements
  static constexpr int STAGE = kWarp * PITCH;             // one output stream
  static constexpr int U = ROWB / 16;                     // 16-byte units per slab row
  static constexpr int EPU = 16 / (int)sizeof(R);         // elements per unit
  // shared-memory elements per warp: four output stages, plus the parked
  // vectors [L][32][K] for fp64 (fp32 parks them in tensor memory)
  // (+ [3][32][K] per-lane scratch: entering vector, gamma_0, last gamma)
  static __host__ __device__ int warp_elems(int L) {
    return 4 * STAGE + 3 * kWarp * K + (sizeof(R) == 4 ? 0 : L * kWarp * K);
  }
};

// K-vector shared-memory store / load with the widest aligned access.
template <typename R, int K>
struct SVec {
  static __device__ __forceinline__ void st(R* p, const R (&v)[K]) {
    if constexpr (sizeof(R) == 4 && K % 4 == 0) {
#pragma unroll
      for (int i = 0; i < K; i += 4) *reinterpret_cast<float4*>(p + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
    } else if constexpr (K % 2 == 0) {
#pragma unroll
      for (int i = 0; i < K; i += 2) {
        if constexpr (sizeof(R) == 4) *reinterpret_cast<float2*>(p + i) = make_float2(v[i], v[i + 1]);
        else *reinterpret_cast<double2*>(p + i) = make_double2(v[i], v[i + 1]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < K; ++i) p[i] = v[i];
    }
  }
  static __device__ __forceinline__ void ld(const R* p, R (&v)[K]) {
    if constexpr (sizeof(R) == 4 && K % 4 == 0) {
#pragma unroll
      for (int i = 0; i < K; i += 4) {
        const float4 q = *reinterpret_cast<const float4*>(p + i);
        v[i] = q.x; v[i + 1] = q.y; v[i + 2] = q.z; v[i + 3] = q.w;
      }
    } else if constexpr (K % 2 == 0) {
#pragma unroll
      for (int i = 0; i < K; i += 2) {
        if constexpr (sizeof(R) == 4) {
          const float2 q = *reinterpret_cast<const float2*>(p + i);
          v[i] = q.x; v[i + 1] = q.y;
        } else {
          const double2 q = *reinterpret_cast<const double2*>(p + i);
          v[i] = q.x; v[i + 1] = q.y;
        }
      }
    } else {
#pragma unroll
      for (int i = 0; i < K; ++i) v[i] = p[i];
    }
  }
};

// Four consecutive observations (16-byte aligned) in registers.
template <typename R>
struct Y4 {
  R v[4];
  __device__ __forceinline__ void load(const R* p) {
    if constexpr (sizeof(R) == 4) {
      const float4 q = __ldg(reinterpret_cast<const float4*>(p));
      v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    } else {
      const double2 a = __ldg(reinterpret_cast<const double2*>(p));
      const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
  }
};

// ---------------------------------------------------------------------------
// K-vector arithmetic.  For fp32 and even K the pairs (x[2k], x[2k+1]) go
// through Blackwell's packed FFMA2 / FMUL2 / FADD2 (one issue slot for two
// lanes of math; a scalar operand is broadcast by the instruction itself), so
// the matrix-vector steps of the recursions cost half the issue slots.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void f2_fma(float& d0, float& d1, float a0, float a1, float b0, float b1,
                                       float c0, float c1) {
  asm("{.reg .b64 a, b, c, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
__device__ __forceinline__ void f2_mul(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void f2_add(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void f2_sub(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "sub.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}

template <typename R, int K>
struct V {
  static constexpr bool P = sizeof(R) == 4 && (K % 2) == 0;
  typedef R A[K];
  // d = s * x
  static __device__ __forceinline__ void mul_s(A& d, R s, const A& x) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_mul(d[k], d[k + 1], s, s, x[k], x[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = s * x[k];
    }
  }
  // d = s * x + c
  static __device__ __forceinline__ void fma_s(A& d, R s, const A& x, const A& c) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_fma(d[k], d[k + 1], s, s, x[k], x[k + 1], c[k], c[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = ::fma(s, x[k], c[k]);
    }
  }
  // d = x * y
  static __device__ __forceinline__ void mul(A& d, const A& x, const A& y) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_mul(d[k], d[k + 1], x[k], x[k + 1], y[k], y[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = x[k] * y[k];
    }
  }
  // d = x * y + c
  static __device__ __forceinline__ void fma(A& d, const A& x, const A& y, const A& c) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_fma(d[k], d[k + 1], x[k], x[k + 1], y[k], y[k + 1], c[k], c[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = ::fma(x[k], y[k], c[k]);
    }
  }
  // d = x + y
  static __device__ __forceinline__ void add(A& d, const A& x, const A& y) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_add(d[k], d[k + 1], x[k], x[k + 1], y[k], y[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = x[k] + y[k];
    }
  }
  // d = x - s
  static __device__ __forceinline__ void sub_s(A& d, const A& x, R s) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_sub(d[k], d[k + 1], x[k], x[k + 1], s, s);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = x[k] - s;
    }
  }
  // d = x - y
  static __device__ __forceinline__ void sub(A& d, const A& x, const A& y) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_sub(d[k], d[k + 1], x[k], x[k + 1], y[k], y[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = x[k] - y[k];
    }
  }
  // d = s - x
  static __device__ __forceinline__ void rsub_s(A& d, R s, const A& x) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_sub(d[k], d[k + 1], s, s, x[k], x[k + 1]);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = s - x[k];
    }
  }
  // d = s * x + c (scalar s, c)
  static __device__ __forceinline__ void fma_ss(A& d, R s, const A& x, R c) {
    if constexpr (P) {
#pragma unroll
      for (int k = 0; k < K; k += 2) f2_fma(d[k], d[k + 1], s, s, x[k], x[k + 1], c, c);
    } else {
#pragma unroll
      for (int k = 0; k < K; ++k) d[k] = ::fma(s, x[k], c);
    }
  }
  // sum_k x[k] * y[k]
  static __device__ __forceinline__ R dot(const A& x, const A& y) {
    if constexpr (P) {
      R a0, a1;
      f2_mul(a0, a1, x[0], x[1], y[0], y[1]);
#pragma unroll
      for (int k = 2; k < K; k += 2) f2_fma(a0, a1, x[k], x[k + 1], y[k], y[k + 1], a0, a1);
      return a0 + a1;
    } else {
      R a = x[0] * y[0];
#pragma unroll
      for (int k = 1; k < K; ++k) a = ::fma(x[k], y[k], a);
      return a;
    }
  }
  static __device__ __forceinline__ R vmax(const A& x) {
    R m = x[0];
#pragma unroll
    for (int k = 1; k < K; ++k) m = fmax(m, x[k]);
    return m;
  }
};

// Per-CTA shared model table, computed once by the first K threads of the
// CTA (column j each): column-scaled A, log2 column scales, log2 pi, and the
// Gaussian emission constants of the log2 form (Em2).
template <int K>
struct FBCTab {
  static constexpr int AM = 0;            // [K][K] column-scaled A
  static constexpr int LC = K * K;        // [K] log2 c_j
  static constexpr int LPI = LC + K;      // [K] log2 pi_j
  static constexpr int GA = LPI + K;      // [K] s_j = sqrt(log2(e)/2)/sigma_j
  static constexpr int GO = GA + K;       // [K] -mu_j s_j
  static constexpr int GR = GO + K;       // [K] c_j log2(e)
  static constexpr int MU = GR + K;       // [K] mu_j
  static constexpr int N = MU + K;
};

// Emission log2-densities of all states (u_j = log2 b_j(y)).  The Gaussian is
// rewritten as u = c - w^2 with w = y*s - mu*s, s = sqrt(log2(e)/2)/sigma.
// eval() returns v_j = u_j + lc_j, the log2-density plus the log2 column
// scale of the column-scaled transition matrix (load_colscaled): the
// recursions shift by max_j v_j and multiply by Ahat.  eval_raw() returns
// u_j itself (t = 0, where pi rather than A leads into the state, and the
// dead-step rescan).
template <typename R, int K, int CFG>
struct Em2 {
  Emit<R, K, CFG> em;
  R ga[K], go[K], gc[K], gr[K], lc[K], mu[K];
  // tab: the CTA's shared model table (FBCTab layout); the Gaussian
  // configuration reads its per-state constants from it (computed once per
  // CTA), the others load the family parameters themselves
  __device__ __forceinline__ void load(const loghmm_model_t* m, int n_streams, int fams,
                                       const double* lut, int lut_n, const R (&lc2)[K], const R* tab) {
#pragma unroll
    for (int j = 0; j < K; ++j) lc[j] = lc2[j];
    if constexpr (CFG == kCfgGauss) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        ga[j] = tab[FBCTab<K>::GA + j];
        go[j] = tab[FBCTab<K>::GO + j];
        gr[j] = tab[FBCTab<K>::GR + j];
        gc[j] = gr[j] + lc2[j];
        mu[j] = tab[FBCTab<K>::MU + j];
      }
    } else {
      em.load(m, n_streams, fams, lut, lut_n);
#pragma unroll
      for (int j = 0; j < K; ++j) mu[j] = em.e0[j].q[0];
    }
  }
  __device__ __forceinline__ void eval(R y0, R y1, ObsFeat<R>& f0, ObsFeat<R>& f1, R (&u)[K],
                                       bool& oob) const {
    if constexpr (CFG == kCfgGauss) {
      f0.y = y0;
      R w[K], w2[K];
      V<R, K>::fma_s(w, y0, ga, go);
      V<R, K>::mul(w2, w, w);
      V<R, K>::sub(u, gc, w2);
    } else {
      R lb[K];
      em.eval(y0, y1, f0, f1, lb, oob);
#pragma unroll
      for (int j = 0; j < K; ++j) u[j] = fma(lb[j], R(1.4426950408889634), lc[j]);
    }
  }
  __device__ __forceinline__ void eval_raw(R y0, R y1, R (&u)[K], bool& oob) const {
    if constexpr (CFG == kCfgGauss) {
      R w[K], w2[K];
      V<R, K>::fma_s(w, y0, ga, go);
      V<R, K>::mul(w2, w, w);
      V<R, K>::sub(u, gr, w2);
    } else {
      ObsFeat<R> f0, f1;
      R lb[K];
      em.eval(y0, y1, f0, f1, lb, oob);
#pragma unroll
      for (int j = 0; j < K; ++j) u[j] = lb[j] * R(1.4426950408889634);
    }
  }
};


// ---------------------------------------------------------------------------
// Tensor memory as per-warp scratch for the parked vectors (fp32).  A CTA is
// one warpgroup (4 warps); warp w owns TMEM lanes [32w, 32w+32) and, in them,
// one column block of KP columns per parked step.  tcgen05.st / tcgen05.ld
// with the 32x32b shape move one 32-bit column per lane per repetition.
// ---------------------------------------------------------------------------
template <int K>
struct KPad {
  static constexpr int V = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : 8;
};

__device__ __forceinline__ void tm_st(uint32_t a, const uint32_t (&r)[1]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(a), "r"(r[0]) : "memory");
}
__device__ __forceinline__ void tm_st(uint32_t a, const uint32_t (&r)[2]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"(r[0]), "r"(r[1])
               : "memory");
}
__device__ __forceinline__ void tm_st(uint32_t a, const uint32_t (&r)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3])
               : "memory");
}
__device__ __forceinline__ void tm_st(uint32_t a, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(a),
               "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t (&r)[1]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r[0]) : "r"(a) : "memory");
}
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t (&r)[2]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(r[0]), "=r"(r[1]) : "r"(a)
               : "memory");
}
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t (&r)[4]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a)
               : "memory");
}
__device__ __forceinline__ void tm_ld(uint32_t a, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
                 "=r"(r[7])
               : "r"(a)
               : "memory");
}
// Wait for this thread's outstanding tcgen05.ld; the registers are operands
// so no use of them can be scheduled above the wait.
template <int N>
__device__ __forceinline__ void tm_wait_ld(uint32_t (&x)[N], uint32_t (&y)[N]) {
  if constexpr (N == 1) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(x[0]), "+r"(y[0])::"memory");
  } else if constexpr (N == 2) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(x[0]), "+r"(x[1]), "+r"(y[0]), "+r"(y[1])::"memory");
  } else if constexpr (N == 4) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(y[0]), "+r"(y[1]), "+r"(y[2]),
                   "+r"(y[3])::"memory");
  } else {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(x[0]), "+r"(x[1]), "+r"(x[2]), "+r"(x[3]), "+r"(x[4]), "+r"(x[5]), "+r"(x[6]),
                   "+r"(x[7]), "+r"(y[0]), "+r"(y[1]), "+r"(y[2]), "+r"(y[3]), "+r"(y[4]), "+r"(y[5]),
                   "+r"(y[6]), "+r"(y[7])::"memory");
  }
}
__device__ __forceinline__ void tm_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// Z = X Y by rows (Z[r] = sum_i X[r][i] Y[i]): packed FFMA2 for fp32, even K
template <typename R, int K>
__device__ __forceinline__ void matmul_rows(const R (&X)[K][K], const R (&Y)[K][K], R (&Z)[K][K]) {
#pragma unroll
  for (int r = 0; r < K; ++r) {
    V<R, K>::mul_s(Z[r], X[r][0], Y[0]);
#pragma unroll
    for (int i = 1; i < K; ++i) V<R, K>::fma_s(Z[r], X[r][i], Y[i], Z[r]);
  }
}

constexpr int kFbcWarps = 4;  // warps (sequences) per CTA: one warpgroup

// Power-of-two normalisation of a scan operator (FMNMX max; exponent kept in
// a double log2 offset).
template <typename R, int K>
__device__ __forceinline__ void norm_op(R (&Z)[K][K], double& off2) {
  R m = Z[0][0];
#pragma unroll
  for (int r = 0; r < K; ++r)
#pragma unroll
    for (int c = 0; c < K; ++c) m = fmax(m, Z[r][c]);
  if (m > R(0)) {
    int e;
    const R s = Num<R>::pow2_scale(m, e);
    off2 += (double)e;
#pragma unroll
    for (int r = 0; r < K; ++r) V<R, K>::mul_s(Z[r], s, Z[r]);
  } else {
    off2 = -CUDART_INF;
  }
}

// LHMM_FBC_MAXNREG (Makefile: FBC_MAXREG) caps the kernel's registers instead
// of bounding the block size, e.g. 160 so that a one-warp Viterbi CTA fits
// beside three FB CTAs in an SM's register file.
#ifdef LHMM_FBC_MAXNREG
#define LHMM_FBC_BOUNDS __maxnreg__(LHMM_FBC_MAXNREG)
#else
#define LHMM_FBC_BOUNDS __launch_bounds__(128)
#endif
template <typename R, int K, int CFG>
__global__ void LHMM_FBC_BOUNDS
    fb_chunk_kernel(const FBCArgs a) {
  typedef Num<R> N;
  typedef CfgTraits<CFG> TR;
  typedef FBCGeom<R, K> G;
  constexpr bool kTwo = (CFG == kCfgGammaVM || CFG == kCfgMixed);
  constexpr bool TM = sizeof(R) == 4;  // park in tensor memory (fp32) or shared memory (fp64)
  constexpr int KP = KPad<K>::V;
  constexpr R kLN2 = R(0.6931471805599453);
  constexpr double kLN2d = 0.6931471805599453094;
  constexpr R kFloor = sizeof(R) == 4 ? R(-1e30) : R(-1e300);  // finite stand-in for max of all -inf
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ uint32_t s_tmem;
  __shared__ R s_tab[FBCTab<K>::N];

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const bool valid = b < a.B;

  // model table: thread j < K fills column j (one global round trip and one
  // set of double-precision constants per CTA instead of per thread)
  if (threadIdx.x < K) {
    const loghmm_model_t* __restrict__ mt = a.model;
    const int j = threadIdx.x;
    R col[K], c = R(0);
#pragma unroll
    for (int i = 0; i < K; ++i) {
      col[i] = (R)mt->A[i * K + j];
      c = c > col[i] ? c : col[i];
    }
    const bool nz = c > R(0);
    const R rc = nz ? N::frcp(c) : R(0);
#pragma unroll
    for (int i = 0; i < K; ++i) s_tab[FBCTab<K>::AM + i * K + j] = col[i] * rc;
    if constexpr (sizeof(R) == 4) s_tab[FBCTab<K>::LC + j] = nz ? N::flg2(c) : N::ninf();
    else s_tab[FBCTab<K>::LC + j] = nz ? (R)log2((double)c) : N::ninf();
    s_tab[FBCTab<K>::LPI + j] = (R)(mt->log_pi[j] * 1.4426950408889634);
    if constexpr (CFG == kCfgGauss) {
      const double h = sqrt(0.5 * 1.4426950408889634);
      const double sg = h / mt->em[0][j].p[1];
      s_tab[FBCTab<K>::GA + j] = (R)sg;
      s_tab[FBCTab<K>::GO + j] = (R)(-mt->em[0][j].p[0] * sg);
      s_tab[FBCTab<K>::GR + j] = (R)(mt->em[0][j].c[0] * 1.4426950408889634);
      s_tab[FBCTab<K>::MU + j] = (R)mt->em[0][j].p[0];
    }
  }

  uint32_t tbase = 0;
  if constexpr (TM) {
    if (wib == 0) {
      const uint32_t dst = (uint32_t)__cvta_generic_to_shared(&s_tmem);
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(dst),
                   "r"((uint32_t)a.tm_cols)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    tbase = s_tmem + ((uint32_t)(32 * wib) << 16);
  } else {
    __syncthreads();  // model table
  }

  if (valid) {
    const int T = a.T, L = a.L, C = T / L, HL = L / 2, NG = L / 4;
    const bool act = lane < C;
    const int t0 = act ? lane * L : 0;
    const int64_t start = b * (int64_t)T;
    const bool two = kTwo && a.n_streams > 1;

    R* wsm = reinterpret_cast<R*>(smem_raw) + (size_t)wib * G::warp_elems(L);
    R* stA = wsm;              // log_alpha slabs
    R* stB = stA + G::STAGE;   // log_beta slabs
    R* stGf = stB + G::STAGE;  // gamma slabs, forward direction
    R* stGb = stGf + G::STAGE; // gamma slabs, backward direction
    R* aux = stGb + G::STAGE;                 // [3][32][K] per-lane scratch
    R* myAin = aux + lane * K;                // entering forward vector
    R* myG0 = aux + kWarp * K + lane * K;     // gamma at t = 0 (lane 0)
    R* myGl = aux + 2 * kWarp * K + lane * K; // last gamma of the chunk
    R* mypark = aux + 3 * kWarp * K + lane * K;  // fp64: [L][32][K] in shared memory
    R* myA = stA + lane * G::PITCH;
    R* myB = stB + lane * G::PITCH;
    R* myGf = stGf + lane * G::PITCH;
    R* myGb = stGb + lane * G::PITCH;

    auto park_st = [&](int slot, const R (&v)[K]) {
      if constexpr (TM) {
        uint32_t r[KP];
#pragma unroll
        for (int j = 0; j < KP; ++j) r[j] = j < K ? __float_as_uint((float)v[j < K ? j : 0]) : 0u;
        tm_st(tbase + (uint32_t)(slot * KP), r);
      } else {
        SVec<R, K>::st(mypark + slot * (kWarp * K), v);
      }
    };

    // ---- model -----------------------------------------------------------
    const loghmm_model_t* __restrict__ md = a.model;
    R Am[K][K], lc2[K];  // column-scaled A, log2 c_j (from the CTA's table)
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) Am[i][j] = s_tab[FBCTab<K>::AM + i * K + j];
    R minA = R(1);
#pragma unroll
    for (int i = 0; i < K; ++i)
#pragma unroll
      for (int j = 0; j < K; ++j) minA = fmin(Am[i][j], minA);
    R lpi2[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      lc2[j] = s_tab[FBCTab<K>::LC + j];
      lpi2[j] = s_tab[FBCTab<K>::LPI + j];
    }
    Em2<R, K, CFG> em;
    em.load(md, a.n_streams, a.stream_fams, a.lut, a.lut_n, lc2, s_tab);
    // Pass-1 operator renormalisation every nn steps: its max entry shrinks
    // by at most min(A) per step, so nn steps stay above 2^-100 (fp32) /
    // 2^-900 (fp64).  (Pass 2 renormalises every step through the emission
    // shift instead.)
    int nn = 1;
    if (minA > R(0)) {
      const float lg = -Num<float>::flg2((float)minA);
      const float budget = sizeof(R) == 4 ? 100.0f : 900.0f;
      nn = lg <= 0.0f ? 8 : (int)fminf(8.0f, fmaxf(1.0f, floorf(budget / lg)));
    }
    // pass-1 operator: every step (nn < 4) or every 1 / 2 four-step groups
    const bool rn_step = nn < 4;
    const int rn_groups = nn >= 8 ? 2 : 1;

    const R* __restrict__ y0c = reinterpret_cast<const R*>(a.y0) + start + t0;
    const R* __restrict__ y1c = two ? reinterpret_cast<const R*>(a.y1) + start + t0 : y0c;

    bool oob = false, bad = false;

    // u_j = log2 b_j(y), m = max_j u_j clamped finite; returns m' = m + shift
    // and bh_j = 2^(u_j - m') (the shift renormalises the carried vector)
    auto emit = [&](R yv0, R yv1, ObsFeat<R>& f0, ObsFeat<R>& f1, R (&u)[K], R (&bh)[K],
                    R shift) -> R {
      em.eval(yv0, yv1, f0, f1, u, oob);
      const R m = fmax(V<R, K>::vmax(u), kFloor) + shift;
      V<R, K>::sub_s(bh, u, m);
#pragma unroll
      for (int j = 0; j < K; ++j) bh[j] = N::fex2(bh[j]);
      return m;
    };

    // ===================== pass 1: chunk operator ===========================
    R Mop[K][K];
#pragma unroll
    for (int r = 0; r < K; ++r)
#pragma unroll
      for (int c = 0; c < K; ++c) Mop[r][c] = r == c ? R(1) : R(0);
    R moff = R(0);
    // lane 0's t = 0 seed log2(pi) + log2 b_0 with the raw densities (pi,
    // not A, leads into the states), evaluated once outside the loops; the
    // pass-2 forward start alpha~_0 follows from it
    R seed_u[K], av0[K], out0[K], m0;
    {
      R ur[K];
      em.eval_raw(y0c[0], two ? y1c[0] : R(0), ur, oob);
#pragma unroll
      for (int j = 0; j < K; ++j) seed_u[j] = lane == 0 ? lpi2[j] + ur[j] : N::ninf();
      m0 = fmax(V<R, K>::vmax(seed_u), kFloor);
#pragma unroll
      for (int j = 0; j < K; ++j) {
        av0[j] = N::fex2(seed_u[j] - m0);
        out0[j] = seed_u[j] * kLN2;
      }
    }
    {
      Y4<R> yc, yc1, yn, yn1;
      yc.load(y0c);
      if (two) yc1.load(y1c);
      int gcd = rn_groups;
#pragma unroll 1
      for (int g = 0; g < NG; ++g) {
        if (g + 1 < NG) {
          yn.load(y0c + 4 * (g + 1));
          if (two) yn1.load(y1c + 4 * (g + 1));
        }
#pragma unroll
        for (int sub = 0; sub < 4; ++sub) {
          const R yv0 = yc.v[sub];
          const R yv1 = two ? yc1.v[sub] : R(0);
          ObsFeat<R> f0, f1;
          R u[K], bh[K];
          const R m = emit(yv0, yv1, f0, f1, u, bh, R(0));
          bad |= !(m > kFloor);  // a dead step (all -inf) or NaN observation
          R Ab[K][K], Nw[K][K];  // A diag(bh), then Mop A diag(bh)
#pragma unroll
          for (int i = 0; i < K; ++i) V<R, K>::mul(Ab[i], Am[i], bh);
#pragma unroll
          for (int r = 0; r < K; ++r) {
            V<R, K>::mul_s(Nw[r], Mop[r][0], Ab[0]);
#pragma unroll
            for (int i = 1; i < K; ++i) V<R, K>::fma_s(Nw[r], Mop[r][i], Ab[i], Nw[r]);
          }
          if (sub == 0) {
            // t = 0 (lane 0, first group) seeds the forward vector
            // (log2 pi + log2 b_0): no operator step
            const bool first = (g == 0) && (lane == 0);
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
              for (int c = 0; c < K; ++c) Mop[r][c] = first ? Mop[r][c] : Nw[r][c];
            moff += first ? R(0) : m;
          } else {
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
              for (int c = 0; c < K; ++c) Mop[r][c] = Nw[r][c];
            moff += m;
          }
          if (rn_step || (sub == 3 && --gcd == 0)) {
            if (!rn_step) gcd = rn_groups;
            R mx = Mop[0][0];
#pragma unroll
            for (int r = 0; r < K; ++r)
#pragma unroll
              for (int c = 0; c < K; ++c) mx = fmax(mx, Mop[r][c]);
            if (mx > R(0)) {
              int e;
              const R s = N::pow2_scale(mx, e);
              moff += (R)e;
#pragma unroll
              for (int r = 0; r < K; ++r) V<R, K>::mul_s(Mop[r], s, Mop[r]);
            }
          }
        }
        yc = yn;
        if (two) yc1 = yn1;
      }
    }
    double mo = (double)moff;
    {
      R mx = Mop[0][0];
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) mx = fmax(mx, Mop[r][c]);
      if (!(mx > R(0))) mo = -CUDART_INF;
    }
    if (!act) {
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) Mop[r][c] = r == c ? R(1) : R(0);
      mo = 0.0;
      bad = false;
    }

    // ===================== scan over chunks =================================
    R a_in[K];
    double lam_in, LL;
    {
      R Q[K][K];
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) Q[r][c] = Mop[r][c];
      double qo = mo;
#pragma unroll 1
      for (int d = 1; d < kWarp; d <<= 1) {
        R P[K][K];
        double po;
        shfl_mat<R, K>(P, po, Q, qo, d, true);
        if (lane >= d) {
          R Z[K][K];
          matmul_rows<R, K>(P, Q, Z);
#pragma unroll
          for (int r = 0; r < K; ++r)
#pragma unroll
            for (int c = 0; c < K; ++c) Q[r][c] = Z[r][c];
          qo += po;
          norm_op<R, K>(Q, qo);
        }
      }
      R sm = seed_u[0];
#pragma unroll
      for (int j = 1; j < K; ++j) sm = fmax(sm, seed_u[j]);
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
        R acc = sv[0] * Q[0][c];
#pragma unroll
        for (int i = 1; i < K; ++i) acc = fma(sv[i], Q[i][c], acc);
        v[c] = acc;
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
    R b_ex[K];
    double rho_ex;
    {
      R S[K][K];
#pragma unroll
      for (int r = 0; r < K; ++r)
#pragma unroll
        for (int c = 0; c < K; ++c) S[r][c] = Mop[r][c];
      double so = mo;
#pragma unroll 1
      for (int d = 1; d < kWarp; d <<= 1) {
        R Y[K][K];
        double yo;
        shfl_mat<R, K>(Y, yo, S, so, d, false);
        if (lane + d < kWarp) {
          R Z[K][K];
          matmul_rows<R, K>(S, Y, Z);
#pragma unroll
          for (int r = 0; r < K; ++r)
#pragma unroll
            for (int c = 0; c < K; ++c) S[r][c] = Z[r][c];
          so += yo;
          norm_op<R, K>(S, so);
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

    // ===================== pass 2: meet in the middle =======================
    R* __restrict__ outA = reinterpret_cast<R*>(a.log_alpha);
    R* __restrict__ outB = reinterpret_cast<R*>(a.log_beta);
    R* __restrict__ outG = reinterpret_cast<R*>(a.gamma);
    // Flush geometry: 16-byte unit k of this lane is unit (lane + 32k) % U of
    // slab row (lane + 32k) / U.  When U divides 32 the row advances by 32/U
    // per k and the unit is fixed, so one element offset per lane suffices.
    constexpr bool kUdiv = (kWarp % G::U) == 0;
    const int64_t rowstride = (int64_t)L * K;
    const int f_row0 = kUdiv ? lane / G::U : 0;
    const int f_e = kUdiv ? (lane % G::U) * G::EPU : 0;
    const int64_t f_off0 = (int64_t)f_row0 * rowstride + f_e;  // element offset inside the sequence
    auto flush = [&](R* __restrict__ out, const R* __restrict__ stage, int tb) {
      __syncwarp();
      R* __restrict__ ob = out + start * K + (int64_t)tb * K;
#pragma unroll
      for (int k = 0; k < G::U; ++k) {
        int row, e;
        int64_t off;
        if constexpr (kUdiv) {
          row = f_row0 + k * (kWarp / G::U);
          e = f_e;
          off = f_off0 + (int64_t)k * (kWarp / G::U) * rowstride;
        } else {
          const int v = lane + kWarp * k;
          row = v / G::U;
          e = (v % G::U) * G::EPU;
          off = row * rowstride + e;
        }
        if (row < C)
          *reinterpret_cast<float4*>(ob + off) = *reinterpret_cast<const float4*>(stage + row * G::PITCH + e);
      }
      __syncwarp();
    };

    R X[K][K];
    R st[TR::S][K][LOGHMM_NSLOT];
    R gs0[K], gs1[K], gs2[K];  // Gaussian statistics (w, w d, w d^2), packed
    R mu[K];                   // Gaussian means (statistics shift)
    R pg[K];
#pragma unroll
    for (int i = 0; i < K; ++i) {
      pg[i] = R(0);
      gs0[i] = gs1[i] = gs2[i] = R(0);
      mu[i] = em.mu[i];
#pragma unroll
      for (int j = 0; j < K; ++j) X[i][j] = R(0);
#pragma unroll
      for (int s = 0; s < TR::S; ++s)
#pragma unroll
        for (int q = 0; q < LOGHMM_NSLOT; ++q) st[s][i][q] = R(0);
    }
    // E-step statistics of one posterior vector g at observation features f
    auto stats = [&](const R (&g)[K], const ObsFeat<R>& f0, const ObsFeat<R>& f1) {
      if constexpr (CFG == kCfgGauss) {
        R d[K], wd[K];
        V<R, K>::rsub_s(d, f0.y, mu);
        V<R, K>::mul(wd, g, d);
        V<R, K>::add(gs0, gs0, g);
        V<R, K>::add(gs1, gs1, wd);
        V<R, K>::fma(gs2, wd, d, gs2);
      } else {
        stats_step<R, K, CFG>(st, g, em.em, f0, f1);
      }
    };

    R av[K];  // forward: alpha~_{t-1}
    R lam = lane == 0 ? R(0) : (R)lam_in;  // t = 0 uses p = pi (linear, offset 0)
#pragma unroll
    for (int j = 0; j < K; ++j) av[j] = a_in[j];
    {
      R z[K];
#pragma unroll
      for (int j = 0; j < K; ++j) z[j] = R(0);
      SVec<R, K>::st(myAin, a_in);
      SVec<R, K>::st(myG0, z);
      SVec<R, K>::st(myGl, z);
    }
    R bt[K];  // backward: beta~_{t+1}
    R rho = (R)rho_ex;
#pragma unroll
    for (int j = 0; j < K; ++j) bt[j] = b_ex[j];
    {  // pre-step: beta at the chunk's last step
      R o[K], l2[K];
#pragma unroll
      for (int j = 0; j < K; ++j) l2[j] = N::flg2(bt[j]);
      V<R, K>::fma_ss(o, kLN2, l2, rho * kLN2);
      SVec<R, K>::st(myB + 3 * K, o);
      park_st(L - 1, bt);
    }

    Y4<R> yf, yf1, yb, yb1;
    yf.load(y0c);
    yb.load(y0c + L - 4);
    if (two) {
      yf1.load(y1c);
      yb1.load(y1c + L - 4);
    }

    // One 4-step group of both directions.  PH2: second half (meet).  The
    // carried vectors are renormalised every step through the emission shift:
    // scaling by 2^-log2(max v) keeps max v in [min(A)^2 / 2, 2].
    auto group = [&](int g, auto ph2c, auto firstc) {
      constexpr bool PH2 = decltype(ph2c)::value;
      constexpr bool FIRST = decltype(firstc)::value;  // g == 0 (peeled)
      Y4<R> yfn, yfn1, ybn, ybn1;
      if (g + 1 < NG) {
        yfn.load(y0c + 4 * (g + 1));
        ybn.load(y0c + L - 4 * (g + 2));
        if (two) {
          yfn1.load(y1c + 4 * (g + 1));
          ybn1.load(y1c + L - 4 * (g + 2));
        }
      }
#pragma unroll
      for (int sub = 0; sub < 4; ++sub) {
        const int i = 4 * g + sub;
        const int t = L - 2 - i;  // backward step (t = -1: chunk tail, xi pair only)
        R be[K], al[K];
        if constexpr (PH2) {
          // parked vectors: beta~_i for the forward step, alpha~_t for the backward
          const int ts = t < 0 ? 0 : t;
          if constexpr (TM) {
            uint32_t rf[KP], rb[KP];
            tm_ld(tbase + (uint32_t)(i * KP), rf);
            tm_ld(tbase + (uint32_t)(ts * KP), rb);
            tm_wait_ld<KP>(rf, rb);
#pragma unroll
            for (int j = 0; j < K; ++j) {
              be[j] = (R)__uint_as_float(rf[j]);
              al[j] = (R)__uint_as_float(rb[j]);
            }
          } else {
            SVec<R, K>::ld(mypark + i * (kWarp * K), be);
            SVec<R, K>::ld(mypark + ts * (kWarp * K), al);
          }
          if (sub == 3 && t < 0) SVec<R, K>::ld(myAin, al);  // chunk tail: alpha~_{t0-1}
        }
        // ----------------------- forward step t = i -----------------------
        {
          const R sf = fmax(N::flg2(V<R, K>::vmax(av)), kFloor);
          ObsFeat<R> f0, f1;
          R u[K], bh[K], p[K];
          const R m = emit(yf.v[sub], two ? yf1.v[sub] : R(0), f0, f1, u, bh, sf);
          V<R, K>::mul_s(p, av[0], Am[0]);
#pragma unroll
          for (int r = 1; r < K; ++r) V<R, K>::fma_s(p, av[r], Am[r], p);
          const bool t0 = FIRST && sub == 0 && lane == 0;  // alpha_0 = pi b_0 exactly
          {
            R o[K], l2[K];
#pragma unroll
            for (int j = 0; j < K; ++j) l2[j] = N::flg2(p[j]);
            V<R, K>::add(l2, l2, u);
            V<R, K>::fma_ss(o, kLN2, l2, lam * kLN2);
            if constexpr (FIRST) {
#pragma unroll
              for (int j = 0; j < K; ++j) o[j] = t0 ? out0[j] : o[j];
            }
            SVec<R, K>::st(myA + sub * K, o);
          }
          if constexpr (PH2) {
            R cv[K], gg[K];
            V<R, K>::mul(cv, bh, be);
            const R iz = N::frcp(V<R, K>::dot(p, cv));
            V<R, K>::mul_s(cv, iz, cv);
            V<R, K>::mul(gg, p, cv);
#pragma unroll
            for (int r = 0; r < K; ++r) V<R, K>::fma_s(X[r], av[r], cv, X[r]);
            SVec<R, K>::st(myGf + sub * K, gg);
            stats(gg, f0, f1);
            if (sub == 3) SVec<R, K>::st(myGl, gg);
          }
          V<R, K>::mul(av, p, bh);
          lam += m;
          if constexpr (FIRST) {
#pragma unroll
            for (int j = 0; j < K; ++j) av[j] = t0 ? av0[j] : av[j];
            lam = t0 ? m0 : lam;
          }
          if constexpr (!PH2) park_st(i, av);
        }
        // ------------- backward step: y index r = t + 1 = L-1-i -------------
        {
          const R sb = fmax(N::flg2(V<R, K>::vmax(bt)), kFloor);
          ObsFeat<R> f0, f1;
          R u[K], bh[K], w[K], q[K];
          const R m = emit(yb.v[3 - sub], two ? yb1.v[3 - sub] : R(0), f0, f1, u, bh, sb);
          V<R, K>::mul(w, bh, bt);
#pragma unroll
          for (int r = 0; r < K; ++r) q[r] = V<R, K>::dot(Am[r], w);
          const R rho2 = rho + m;
          {  // (the t = -1 store lands in an already flushed slot)
            R o[K], l2[K];
#pragma unroll
            for (int j = 0; j < K; ++j) l2[j] = N::flg2(q[j]);
            V<R, K>::fma_ss(o, kLN2, l2, rho2 * kLN2);
            SVec<R, K>::st(myB + (t & 3) * K, o);
          }
          if constexpr (PH2) {
            // the pending posterior gamma_{t+1} meets the features of y_{t+1}
            // (the first one is the boundary posterior gamma_{HL-1})
            stats(pg, f0, f1);
            R iz = N::frcp(V<R, K>::dot(al, q));
            if (sub == 3) iz = (t < 0 && lane == 0) ? R(0) : iz;  // no pair before t = 0
            R ai[K];
            V<R, K>::mul_s(ai, iz, al);
#pragma unroll
            for (int r = 0; r < K; ++r) V<R, K>::fma_s(X[r], ai[r], w, X[r]);
            V<R, K>::mul(pg, ai, q);
            SVec<R, K>::st(myGb + (t & 3) * K, pg);
            if (sub == 2) SVec<R, K>::st(myG0, pg);  // t = 0 in the last group
          }
#pragma unroll
          for (int j = 0; j < K; ++j) bt[j] = q[j];
          rho = rho2;
          if constexpr (!PH2) {
            if (t >= HL) park_st(t, bt);
          }
        }
        if (sub == 2) {  // backward slabs [L-4-4g, L-4g) complete
          const int tb = L - 4 - 4 * g;
          if (outB) flush(outB, stB, tb);
          if constexpr (PH2) {
            if (outG) flush(outG, stGb, tb);
          }
        }
      }
      if (outA) flush(outA, stA, 4 * g);  // forward slabs [4g, 4g+4) complete
      if constexpr (PH2) {
        if (outG) flush(outG, stGf, 4 * g);
      }
      yf = yfn;
      yb = ybn;
      if (two) {
        yf1 = yfn1;
        yb1 = ybn1;
      }
    };

    group(0, std::false_type{}, std::true_type{});
#pragma unroll 1
    for (int g = 1; g < NG / 2; ++g) group(g, std::false_type{}, std::false_type{});
    {
      // boundary: gamma_{HL-1} from alpha~_{HL-1} (av) and beta~_{HL-1} (bt);
      // it is the first pending posterior of the backward direction
      if constexpr (TM) tm_wait_st();
      const R iz = N::frcp(V<R, K>::dot(av, bt));
      V<R, K>::mul(pg, av, bt);
      V<R, K>::mul_s(pg, iz, pg);
      SVec<R, K>::st(myGb + 3 * K, pg);
      __syncwarp();
    }
#pragma unroll 1
    for (int g = NG / 2; g < NG; ++g) group(g, std::true_type{}, std::false_type{});
    if constexpr (CFG == kCfgGauss) {
#pragma unroll
      for (int j = 0; j < K; ++j) {
        st[0][j][0] = gs0[j];
        st[0][j][1] = gs1[j];
        st[0][j][2] = gs2[j];
      }
    }

    // ===================== per-sequence results =============================
    if (!act) {
#pragma unroll
      for (int i = 0; i < K; ++i) {
#pragma unroll
        for (int j = 0; j < K; ++j) X[i][j] = R(0);
#pragma unroll
        for (int s = 0; s < TR::S; ++s)
#pragma unroll
          for (int q = 0; q < LOGHMM_NSLOT; ++q) st[s][i][q] = R(0);
      }
    }
    // rare path: exact first dead step and NaN flag (rescan of the chunk)
    int dead_t = INT_MAX;
    bool nan_seen = false;
    if (__any_sync(kFull, bad)) {
      if (bad) {
        for (int s = 0; s < L; ++s) {
          const R yv0 = y0c[s];
          const R yv1 = two ? y1c[s] : R(0);
          if (yv0 != yv0 || yv1 != yv1) nan_seen = true;
          R u[K];
          em.eval_raw(yv0, yv1, u, oob);
          R m = u[0];
#pragma unroll
          for (int j = 1; j < K; ++j) m = fmax(m, u[j]);
          if (!(m > N::ninf()) && dead_t == INT_MAX) dead_t = t0 + s;
        }
      }
    }
    const int dead_all = (int)warp_min_ll((long long)dead_t);
    const unsigned nanb = __ballot_sync(kFull, nan_seen);
    const unsigned oobb = __ballot_sync(kFull, oob && act);
    if (lane == 0) {
      a.ll[b] = dead_all == INT_MAX ? LL : -CUDART_INF;
      if (a.flags) {
        a.flags[2 * b] = dead_all == INT_MAX ? -1 : (int64_t)dead_all;
        a.flags[2 * b + 1] = (nanb ? 1 : 0) | (oobb ? 2 : 0);
      }
    }
    if (a.partials) {
      // Per-sequence statistics row: every lane holds its chunk's share of Q
      // quantities; they are summed over the 32 lanes 32 quantities at a time
      // through a [32][33] shared tile (lane q adds column q in lane order —
      // fixed order, bit-reproducible) and written as coalesced doubles.
      double* row = a.partials + b * a.stats_width;
      constexpr int NSL = TR::S * K * LOGHMM_NSLOT;
      constexpr int Q = K * K + 2 * K + NSL;
      R glast[K], g0[K];
      SVec<R, K>::ld(myGl, glast);
      SVec<R, K>::ld(myG0, g0);
      R vals[Q];
#pragma unroll
      for (int i = 0; i < K; ++i)
#pragma unroll
        for (int j = 0; j < K; ++j) vals[i * K + j] = X[i][j];
      // gamma totals over t < T-1 = all-step mass minus the last posterior
#pragma unroll
      for (int j = 0; j < K; ++j) {
        vals[K * K + j] = st[0][j][0] - (lane == C - 1 ? glast[j] : R(0));
        vals[K * K + K + j] = lane == 0 ? g0[j] : R(0);
      }
#pragma unroll
      for (int s = 0; s < TR::S; ++s)
#pragma unroll
        for (int j = 0; j < K; ++j)
#pragma unroll
          for (int q = 0; q < LOGHMM_NSLOT; ++q) {
            const int ns = s == 0 ? TR::NS0 : TR::NS1;
            vals[K * K + 2 * K + (s * K + j) * LOGHMM_NSLOT + q] = q < ns ? st[s][j][q] : R(0);
          }
      R* tile = wsm;  // the output stages are idle now (>= 32 * 33 elements)
      __syncwarp();
#pragma unroll
      for (int r0 = 0; r0 < Q; r0 += 32) {
        const int n = Q - r0 < 32 ? Q - r0 : 32;
#pragma unroll
        for (int q = 0; q < 32; ++q)
          if (r0 + q < Q) tile[lane * 33 + q] = vals[r0 + q < Q ? r0 + q : 0];
        __syncwarp();
        if (lane < n) {
          R acc = tile[lane];
#pragma unroll 8
          for (int l = 1; l < 32; ++l) acc += tile[l * 33 + lane];
          const int idx = r0 + lane;
          double v = (double)acc;
          if (idx < K * K) v *= (double)s_tab[FBCTab<K>::AM + idx];
          row[idx] = v;
        }
        __syncwarp();
      }
      for (int idx = Q + lane; idx < a.stats_width; idx += kWarp) row[idx] = 0.0;
    }
  }

  if constexpr (TM) {
    tm_fence_before();
    __syncthreads();
    tm_fence_after();
    if (wib == 0) {
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(s_tmem),
                   "r"((uint32_t)a.tm_cols)
                   : "memory");
    }
  }
}

}  // namespace lhmm
