// hmm_viterbi3.cuh — batched Viterbi for 2 <= K <= 4 with the sequential
// recursion reduced to its dependency chain ("chain warp" layout).
//
// Same contract and operation order as hmm_viterbi.cuh (inference.py:191-210):
//   cand   = score[:, None] + log_a     one IEEE add per candidate
//   back_t = argmax(cand, axis=0)       first maximal index
//   score  = cand[back_t, j] + log_b[t] one IEEE add
// so scores, backpointers and the path are bit-identical to the reference.
//
// Only the score recursion is sequential in t.  The emission log-densities
// before it and the argmax after it are functions of values that are known
// per step, so they run T-parallel:
//
//   CTA = 32 sequences.  Warp 0 (the chain warp) holds one sequence per lane
//   with its K scores in registers and runs, per step, K*K adds (packed
//   add.rn.f32x2 in fp32), K maxima and K adds — nothing else: no shuffles,
//   no emission math, no index selection.  It reads log b_t from a
//   shared-memory ring and writes the score vector entering each step to a
//   second ring.
//   The other warps (helpers, lane = step inside a 32-step chunk, coalesced
//   observation loads) fill the log b ring one chunk ahead with the
//   reference-exact densities, and one chunk behind re-form the candidates
//   from the stored scores (the same IEEE adds) to extract the first-index
//   argmax as one backpointer byte per (sequence, step).
//   One CTA barrier per 32 steps.  The backtrace then walks the byte table
//   per lane, and all warps write the int64 path coalesced.
#pragma once

#include "hmm_viterbi.cuh"

namespace lhmm {

constexpr int kV3Seq = 32;    // sequences per CTA (one per chain-warp lane)
constexpr int kV3Pitch = 33;  // ring entries per step row (32 sequences + 1)
constexpr int kV3KP = 4;      // padded state count
constexpr int kV3S0 = 3;      // sequences handled by the helpers that share the chain warp's scheduler

// bytes of shared memory: two rings (log b, scores) of 2 slots x 32 steps,
// the sequence table, and the backpointer bytes [32][tp]
__host__ __device__ constexpr int v3_tpitch(int64_t max_T) {
  // multiple of 4 with an odd word count, so the 32 rows start in 32 banks
  return (int)((((max_T + 3) / 4) | 1) * 4);
}
__host__ __device__ constexpr size_t v3_ring_bytes(int esz) {
  return (size_t)2 * 32 * kV3Pitch * kV3KP * esz;
}
__host__ __device__ constexpr size_t v3_smem_bytes(int esz, int64_t max_T) {
  return 2 * v3_ring_bytes(esz) + kV3Seq * 20 + (size_t)kV3Seq * v3_tpitch(max_T);
}

template <typename R>
struct Q4 {
  R v[4];
};
template <typename R>
__device__ __forceinline__ void q4_st(R* p, const R (&v)[4]) {
  if constexpr (sizeof(R) == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    *reinterpret_cast<double2*>(p + 2) = make_double2(v[2], v[3]);
  }
}
template <typename R>
__device__ __forceinline__ void q4_ld(const R* p, R (&v)[4]) {
  if constexpr (sizeof(R) == 4) {
    const float4 q = *reinterpret_cast<const float4*>(p);
    v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
  } else {
    const double2 a = *reinterpret_cast<const double2*>(p);
    const double2 b = *reinterpret_cast<const double2*>(p + 2);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
}

// (d0, d1) = (a0 + b0, a1 + b1), each an IEEE round-to-nearest add
__device__ __forceinline__ void add2_rn(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{.reg .b64 a, b, d;\n\tmov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void add2_rn(double& d0, double& d1, double a0, double a1, double b0, double b1) {
  d0 = __dadd_rn(a0, b0);
  d1 = __dadd_rn(a1, b1);
}

// One recursion step on the padded 4-state vector: nd_j = max_i(d_i + la[i][j]) + lb_j.
// The maximum goes through FMNMX; it equals cand[argmax] except for the sign of
// an exact-zero tie (see hmm_viterbi.cuh).
template <typename R>
__device__ __forceinline__ void v3_step(const R (&d)[4], const R (&la)[4][4], const R (&lb)[4], R (&nd)[4]) {
  R m[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    R c0, c1, c2, c3;
    add2_rn(c0, c1, d[0], d[1], la[0][j], la[1][j]);
    add2_rn(c2, c3, d[2], d[3], la[2][j], la[3][j]);
    m[j] = fmax(fmax(c0, c1), fmax(c2, c3));
  }
  add2_rn(nd[0], nd[1], m[0], m[1], lb[0], lb[1]);
  add2_rn(nd[2], nd[3], m[2], m[3], lb[2], lb[3]);
}

template <typename R, int K, int CFG, int NW>
__global__ void __launch_bounds__(32 * NW) viterbi_chain_kernel(const VitArgs a) {
  static_assert(K >= 2 && K <= 4, "chain-warp Viterbi covers 2 <= K <= 4");
  typedef Num<R> N;
  typedef VitFams<CFG> VF;
  static_assert(NW == 8 || NW == 16, "8 or 16 warps per CTA");
  constexpr int N0 = (NW - 1) / 4;        // helper warps on the chain warp's scheduler
  constexpr int NO = NW - 1 - N0;         // helper warps on the other schedulers
  constexpr int SPH0 = (kV3S0 + N0 - 1) / N0, SPH1 = (kV3Seq - kV3S0 + NO - 1) / NO;
  constexpr int SPH = SPH0 > SPH1 ? SPH0 : SPH1;  // sequences per helper warp (max)
  constexpr int RING = 32 * kV3Pitch * kV3KP;  // elements of one ring slot
  extern __shared__ __align__(16) unsigned char smem_raw[];
  R* ringE = reinterpret_cast<R*>(smem_raw);  // [2][32][33][4] log b
  R* ringD = ringE + 2 * RING;                // [2][32][33][4] scores entering the step
  int64_t* s_start = reinterpret_cast<int64_t*>(ringD + 2 * RING);  // [32]
  int* s_T = reinterpret_cast<int*>(s_start + kV3Seq);              // [32]
  int* s_flag = s_T + kV3Seq;                                       // [32] flags, [32] final states
  uint8_t* bp = reinterpret_cast<uint8_t*>(s_flag + 2 * kV3Seq);    // [32][tp]
  __shared__ int s_tmax, s_tmin;

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t b0 = (int64_t)blockIdx.x * kV3Seq;
  const loghmm_model_t* __restrict__ md = a.model;
  const bool two = VF::TWO && a.n_streams > 1;

  if (wib == 0) {
    const int64_t b = b0 + lane;
    const bool valid = b < a.B;
    const int64_t st = valid ? a.offsets[b] : 0;
    const int T = valid ? (int)(a.offsets[b + 1] - st) : 0;
    s_start[lane] = st;
    s_T[lane] = T;
    s_flag[lane] = 0;
    int tmax = T, tmin = valid ? T : 0x7fffffff;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      tmax = max(tmax, __shfl_xor_sync(kFull, tmax, o));
      tmin = min(tmin, __shfl_xor_sync(kFull, tmin, o));
    }
    if (lane == 0) {
      s_tmax = tmax;
      s_tmin = tmin;
    }
  }
  __syncthreads();
  const int Tmax = s_tmax, Tmin = s_tmin;
  const int tp = v3_tpitch(Tmax > 0 ? Tmax : 1);
  const int nch = (Tmax + 31) / 32;

  // transition log-probabilities, padded with -inf
  R la[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) la[i][j] = (i < K && j < K) ? (R)md->log_A[i * K + j] : N::ninf();

  if (wib == 0) {
    // ======================= chain warp: lane = sequence ====================
    const int T = s_T[lane];
    R d[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) d[j] = N::ninf();
    for (int it = 0; it <= nch + 1; ++it) {
      const int c = it - 1;
      if (c >= 0 && c < nch) {
        const R* E = ringE + (c & 1) * RING + lane * kV3KP;
        R* D = ringD + (c & 1) * RING + lane * kV3KP;
        const int tb = 32 * c;
        int tl0 = 0;
        if (c == 0) {  // t = 0: score = log pi + log b_0
          R lb[4];
          q4_ld<R>(E, lb);
          if (T > 0) {
#pragma unroll
            for (int j = 0; j < 4; ++j) d[j] = j < K ? N::add((R)md->log_pi[j], lb[j]) : N::ninf();
          }
          tl0 = 1;
        }
        if (tb + 32 <= Tmin) {  // every sequence of the CTA covers the chunk
#pragma unroll 8
          for (int tl = tl0; tl < 32; ++tl) {
            R lb[4], nd[4];
            q4_ld<R>(E + tl * (kV3Pitch * kV3KP), lb);
            q4_st<R>(D + tl * (kV3Pitch * kV3KP), d);
            v3_step<R>(d, la, lb, nd);
#pragma unroll
            for (int j = 0; j < 4; ++j) d[j] = nd[j];
          }
        } else {
#pragma unroll 4
          for (int tl = tl0; tl < 32; ++tl) {
            R lb[4], nd[4];
            q4_ld<R>(E + tl * (kV3Pitch * kV3KP), lb);
            q4_st<R>(D + tl * (kV3Pitch * kV3KP), d);
            v3_step<R>(d, la, lb, nd);
            const bool act = tb + tl < T;
#pragma unroll
            for (int j = 0; j < 4; ++j) d[j] = act ? nd[j] : d[j];
          }
        }
      }
      __syncthreads();
    }
    // best final state (first index) and log joint
    int cur = 0;
    R best = d[0];
#pragma unroll
    for (int j = 1; j < K; ++j) {
      const bool gt = d[j] > best;
      best = gt ? d[j] : best;
      cur = gt ? j : cur;
    }
    const int64_t b = b0 + lane;
    if (b < a.B) a.log_joint[b] = T > 0 ? (double)best : (double)N::ninf();
    s_flag[kV3Seq + lane] = cur;
  } else {
    // ======================= helper warps: lane = step ======================
    // Sequence assignment.  Warps are spread over the four schedulers by
    // wib % 4; the chain warp's scheduler already carries the recursion
    // (about kV3S0-equivalent sequences of helper work less than a fair
    // share), so its helpers take kV3S0 sequences in total and the helpers of
    // the other three schedulers share the rest.
    const bool on0 = (wib & 3) == 0;
    const int k = on0 ? (wib / 4 - 1) : (wib - 1 - wib / 4);
    const int n = on0 ? N0 : NO;
    const int base = on0 ? 0 : kV3S0;
    const int cnt = on0 ? kV3S0 : kV3Seq - kV3S0;
    ExactEm<R, VF::F0> em0[K];
    ExactEm<R, VF::F1> em1[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      em0[j].load(md->em[0][j]);
      if (two) em1[j].load(md->em[1][j]);
      else em1[j].fam = LOGHMM_FAM_NONE;
    }
    const double* lut = a.lut;
    const int lut_n = a.lut_n;
    const R* __restrict__ y0g = reinterpret_cast<const R*>(a.y0);
    const R* __restrict__ y1g = two ? reinterpret_cast<const R*>(a.y1) : y0g;
    // per assigned sequence: ring column, length, observation pointers, flags
    int sq[SPH], Tq[SPH];
    const R* yp0[SPH];
    const R* yp1[SPH];
    uint8_t* bq[SPH];
    unsigned fl[SPH];
    R yv0[SPH], yv1[SPH];  // observations of the next chunk (loaded one chunk ahead)
#pragma unroll
    for (int u = 0; u < SPH; ++u) {
      const bool has = k + u * n < cnt;
      sq[u] = has ? base + k + u * n : 0;
      Tq[u] = has ? s_T[sq[u]] : 0;
      yp0[u] = y0g + s_start[sq[u]] + lane;
      yp1[u] = y1g + s_start[sq[u]] + lane;
      bq[u] = bp + (size_t)sq[u] * tp + lane;
      fl[u] = 0;
      yv0[u] = lane < Tq[u] ? yp0[u][0] : R(0);
      yv1[u] = (two && lane < Tq[u]) ? yp1[u][0] : R(0);
    }
    for (int it = 0; it <= nch + 1; ++it) {
      // ---- emissions of chunk `it` ----------------------------------------
      if (it < nch) {
        R* E = ringE + (it & 1) * RING + lane * (kV3Pitch * kV3KP);
        const int t = 32 * it + lane;
        R yc0[SPH], yc1[SPH];
#pragma unroll
        for (int u = 0; u < SPH; ++u) {
          yc0[u] = yv0[u];
          yc1[u] = yv1[u];
          const bool nx = t + 32 < Tq[u];
          yv0[u] = nx ? yp0[u][32 * (it + 1)] : R(0);
          if (two) yv1[u] = nx ? yp1[u][32 * (it + 1)] : R(0);
        }
#pragma unroll
        for (int u = 0; u < SPH; ++u) {
          if (k + u * n < cnt) {
            bool oob = false;
            R lb[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              if (j < K) {
                R v = em0[j].eval(yc0[u], lut, lut_n, oob);
                if (two) v = N::add(v, em1[j].eval(yc1[u], lut, lut_n, oob));
                lb[j] = v;
              } else {
                lb[j] = N::ninf();
              }
            }
            const bool nan_seen = (yc0[u] != yc0[u]) | (yc1[u] != yc1[u]);  // inference.py:117-118
            fl[u] |= t < Tq[u] ? ((nan_seen ? 1u : 0u) | (oob ? 2u : 0u)) : 0u;
            q4_st<R>(E + sq[u] * kV3KP, lb);
          }
        }
      }
      // ---- backpointers of chunk `it - 2` -----------------------------------
      if (it >= 2) {
        const int c = it - 2;
        const R* D = ringD + (c & 1) * RING + lane * (kV3Pitch * kV3KP);
        const int t = 32 * c + lane;
#pragma unroll
        for (int u = 0; u < SPH; ++u) {
          if (k + u * n < cnt) {
            R d[4];
            q4_ld<R>(D + sq[u] * kV3KP, d);
            unsigned byte = 0;
#pragma unroll
            for (int j = 0; j < K; ++j) {
              R c0, c1, c2, c3;
              add2_rn(c0, c1, d[0], d[1], la[0][j], la[1][j]);
              add2_rn(c2, c3, d[2], d[3], la[2][j], la[3][j]);
              const bool p01 = c1 > c0, p23 = c3 > c2;
              const bool p = fmax(c2, c3) > fmax(c0, c1);
              const unsigned idx = p ? (2u | (p23 ? 1u : 0u)) : (p01 ? 1u : 0u);
              byte |= idx << (2 * j);
            }
            if (t < Tq[u]) bq[u][32 * c] = (uint8_t)(t >= 1 ? byte : 0u);
          }
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int u = 0; u < SPH; ++u)
      if (fl[u]) atomicOr(&s_flag[sq[u]], (int)fl[u]);
  }
  // optional byte table of backpointers (tests), expanded from the packed bytes
  if (a.back != nullptr) {
    for (int s = wib; s < kV3Seq; s += NW) {
      const int Ts = s_T[s];
      const uint8_t* row = bp + (size_t)s * tp;
      uint8_t* __restrict__ o = a.back + s_start[s] * K;
      for (int t = lane; t < Ts; t += kWarp) {
        const unsigned e = row[t];
#pragma unroll
        for (int j = 0; j < K; ++j) o[(int64_t)t * K + j] = (uint8_t)((e >> (2 * j)) & 3u);
      }
    }
  }
  __syncthreads();
  if (wib == 0) {
    // ---- backtrace: in place, the byte of step t becomes the state at t ----
    const int T = s_T[lane];
    int cur = s_flag[kV3Seq + lane];  // best final state (stored by the chain warp)
    uint8_t* row = bp + (size_t)lane * tp;
    for (int t = T - 1; t >= 1; --t) {
      const unsigned e = row[t];
      row[t] = (uint8_t)cur;
      cur = (int)((e >> (2 * cur)) & 3u);
    }
    if (T > 0) row[0] = (uint8_t)cur;
  }
  __syncthreads();
  // ---- path write-out: all warps, 32 consecutive steps of one sequence -----
  for (int s = wib; s < kV3Seq; s += NW) {
    const int64_t b = b0 + s;
    if (b >= a.B) break;
    const int Ts = s_T[s];
    const uint8_t* row = bp + (size_t)s * tp;
    int64_t* __restrict__ out = a.path + s_start[s];
    for (int t = lane; t < Ts; t += kWarp) out[t] = (int64_t)row[t];
    if (lane == 0 && a.flags && s_flag[s]) a.flags[2 * b + 1] |= (int64_t)s_flag[s];
  }
}

}  // namespace lhmm
