// hmm_viterbi.cuh — batched Viterbi with compact backpointers and an
// on-device backtrace, K <= 8.
//
// Reference: inference.py:191-210.  The max-plus recursion is evaluated in
// exactly the reference's operation order so the backpointers and the path
// are bit-identical:
//   cand   = score[:, None] + log_a            (one IEEE add per candidate)
//   back_t = argmax(cand, axis=0)              (first maximal index)
//   score  = cand[back_t, j] + log_b[t, j]     (one IEEE add)
// Because every value depends on the exact rounding of its predecessor, the
// recursion is sequential in t; parallelism is B x K: K lanes per sequence
// (lane j computes state j), 32/K sequences per warp, the previous score
// vector exchanged with warp shuffles.
//
// Backpointers are stored as ceil(log2 K) ballot bit-planes per step (bit
// g*K+j of plane p = bit p of back_t[j] of group g): K=4 costs 1 byte per
// (sequence, step).  The backtrace then runs with all 32 lanes on one
// sequence at a time: each lane composes the backpointer maps of its chunk,
// a suffix scan of the composed maps (warp shuffles) gives every chunk its end
// state, and each lane re-walks its chunk writing the path through a shared
// memory staging buffer (coalesced int64 stores).
#pragma once

#include "hmm_common.cuh"

namespace lhmm {

struct VitArgs {
  const loghmm_model_t* model;
  const void* y0;
  const void* y1;
  const int64_t* offsets;
  int64_t B;
  const double* lut;
  int lut_n;
  int n_streams;
  int64_t* path;
  double* log_joint;
  uint8_t* back;
  uint32_t* planes_ws;  // global plane store (kGlobal): [warps][plane_words]
  int64_t plane_words;  // per warp (= max_T * NP rounded)
  int warp_smem_words;  // shared words per warp
  int64_t* flags;
};

constexpr int kPathSlab = 8;
constexpr int kPathPitch = 9;  // int64 elements, odd => conflict-free

template <int K>
struct Bits {
  static constexpr int NP = K <= 1 ? 0 : K <= 2 ? 1 : K <= 4 ? 2 : 3;
};

// First-index argmax over cand[lo, hi) as a pairwise tree (the right half wins
// only on a strictly greater value, which preserves numpy's tie rule).  The
// maximum itself goes through FMNMX (4-cycle latency, on the recursion's
// critical path); the index selection hangs off it.  Both agree except for
// the sign of an exact zero tie, which cannot change the next score unless the
// emission term is also exactly zero.
template <typename R, int LO, int HI>
struct ArgMax {
  static __device__ __forceinline__ void run(const R* c, R& v, int& i) {
    if constexpr (HI - LO == 1) {
      v = c[LO];
      i = LO;
    } else {
      constexpr int MID = LO + (HI - LO + 1) / 2;
      R lv, rv;
      int li, ri;
      ArgMax<R, LO, MID>::run(c, lv, li);
      ArgMax<R, MID, HI>::run(c, rv, ri);
      const bool right = rv > lv;
      v = fmax(lv, rv);
      i = right ? ri : li;
    }
  }
};

__device__ __forceinline__ unsigned nib(unsigned m, unsigned e) { return (m >> (4 * e)) & 0xFu; }

// back_t[v] for group gshift (= g*K) from the bit-planes of step t.
template <int NP>
__device__ __forceinline__ unsigned plane_lookup(const unsigned (&pl)[NP > 0 ? NP : 1], unsigned v) {
  unsigned r = 0;
#pragma unroll
  for (int p = 0; p < NP; ++p) r |= ((pl[p] >> v) & 1u) << p;
  return r;
}

template <int CFG>
struct VitFams {
  static constexpr int F0 = CFG == kCfgGauss     ? LOGHMM_FAM_GAUSSIAN
                            : CFG == kCfgStudent  ? LOGHMM_FAM_STUDENT_T
                            : CFG == kCfgGamma    ? LOGHMM_FAM_GAMMA
                            : CFG == kCfgVonMises ? LOGHMM_FAM_VON_MISES
                            : CFG == kCfgPoisson  ? LOGHMM_FAM_POISSON
                            : CFG == kCfgGammaVM  ? LOGHMM_FAM_GAMMA
                                                  : -1;
  static constexpr int F1 = CFG == kCfgGammaVM ? LOGHMM_FAM_VON_MISES : -1;
  static constexpr bool TWO = CFG == kCfgGammaVM || CFG == kCfgMixed;
};

template <typename R, int K, int CFG, bool kGlobal>
__global__ void __launch_bounds__(128) viterbi_small_kernel(const VitArgs a) {
  typedef Num<R> N;
  typedef VitFams<CFG> VF;
  constexpr int G = kWarp / K;
  constexpr int NP = Bits<K>::NP;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const int g = lane / K;
  const int j = lane - g * K;
  const int64_t b = warp_id * G + g;
  const bool valid = (g < G) && (b < a.B);
  if (warp_id * G >= a.B) return;  // whole warp idle

  uint32_t* wsm = reinterpret_cast<uint32_t*>(smem_raw) + (size_t)wib * a.warp_smem_words;
  int64_t* pstage = reinterpret_cast<int64_t*>(wsm);  // kWarp * kPathPitch int64
  uint32_t* planes = kGlobal ? a.planes_ws + warp_id * a.plane_words
                             : wsm + 2 * kWarp * kPathPitch;

  const loghmm_model_t* __restrict__ md = a.model;
  const int64_t start = valid ? a.offsets[b] : 0;
  const int T = valid ? (int)(a.offsets[b + 1] - start) : 0;
  const R* __restrict__ y0g = reinterpret_cast<const R*>(a.y0) + start;
  const bool two = VF::TWO && a.n_streams > 1;
  const R* __restrict__ y1g = two ? reinterpret_cast<const R*>(a.y1) + start : y0g;

  // column j of log A and the state's emission parameters, in registers
  R la[K];
  const int jj = valid ? j : 0;
#pragma unroll
  for (int i = 0; i < K; ++i) la[i] = (R)md->log_A[i * K + jj];
  ExactEm<R, VF::F0> em0;
  em0.load(md->em[0][jj]);
  ExactEm<R, VF::F1> em1;
  if (two) em1.load(md->em[1][jj]);
  else em1.fam = LOGHMM_FAM_NONE;
  bool oob = false;
  const double* lut = a.lut;
  const int lut_n = a.lut_n;

  int Tmax = T;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Tmax = max(Tmax, __shfl_xor_sync(kFull, Tmax, o));
  const int Tlast = T > 0 ? T - 1 : 0;

  // ---- forward max-plus recursion ---------------------------------------
  R delta = N::ninf();
  if (T > 0) {
    R lb0 = em0.eval(y0g[0], lut, lut_n, oob);
    if (two) lb0 = N::add(lb0, em1.eval(y1g[0], lut, lut_n, oob));
    delta = N::add((R)md->log_pi[jj], lb0);
  }

  // One recursion step: every lane executes it (no divergence around the
  // shuffles / ballots); lanes past their sequence end keep their score.
  // Lane 0 stores the step's bit-planes (one shared-memory store per step).
  // The emission terms of a block of U steps are evaluated up front so the
  // loop-carried chain (shuffle -> add -> argmax -> add) runs back to back.
  auto step = [&](int t, R lb) {
    R cand[K];
#pragma unroll
    for (int i = 0; i < K; ++i) cand[i] = N::add(__shfl_sync(kFull, delta, g * K + i), la[i]);
    R best;
    int bi;
    ArgMax<R, 0, K>::run(cand, best, bi);
    delta = t < T ? N::add(best, lb) : delta;
    unsigned w[NP > 0 ? NP : 1];
#pragma unroll
    for (int p = 0; p < NP; ++p) w[p] = __ballot_sync(kFull, (bi >> p) & 1);
    if (lane == 0) {
      if constexpr (NP == 1) {
        planes[(size_t)t] = w[0];
      } else if constexpr (NP == 2) {
        *reinterpret_cast<uint2*>(planes + (size_t)t * 2) = make_uint2(w[0], w[1]);
      } else if constexpr (NP == 3) {
#pragma unroll
        for (int p = 0; p < 3; ++p) planes[(size_t)t * 3 + p] = w[p];
      }
    }
  };
  auto emis = [&](R yv0, R yv1) -> R {
    R lb = em0.eval(yv0, lut, lut_n, oob);
    if (two) lb = N::add(lb, em1.eval(yv1, lut, lut_n, oob));
    return lb;
  };

  // y prefetched two blocks (2U steps) ahead so DRAM latency stays hidden
  constexpr int U = 8;
  R y0a[U], y1a[U], y0b[U], y1b[U];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int ta = min(1 + u, Tlast), tb2 = min(1 + U + u, Tlast);
    y0a[u] = y0g[ta];
    y1a[u] = two ? y1g[ta] : R(0);
    y0b[u] = y0g[tb2];
    y1b[u] = two ? y1g[tb2] : R(0);
  }
  int t = 1;
#pragma unroll 1
  for (; t + U <= Tmax; t += U) {
    R lbs[U];
#pragma unroll
    for (int u = 0; u < U; ++u) lbs[u] = emis(y0a[u], y1a[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      y0a[u] = y0b[u];
      y1a[u] = y1b[u];
      const int tt = min(t + 2 * U + u, Tlast);
      y0b[u] = y0g[tt];
      y1b[u] = two ? y1g[tt] : R(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) step(t + u, lbs[u]);
  }
#pragma unroll 1
  for (; t < Tmax; ++t) {
    const int tt = min(t, Tlast);
    step(t, emis(y0g[tt], two ? y1g[tt] : R(0)));
  }

  __syncwarp();
  // optional byte table of backpointers (tests), rebuilt from the planes
  if (a.back != nullptr) {
#pragma unroll 1
    for (int gg = 0; gg < G; ++gg) {
      const int64_t bb = warp_id * G + gg;
      if (bb >= a.B) break;
      const int Tg = __shfl_sync(kFull, T, gg * K);
      const int64_t sg = __shfl_sync(kFull, start, gg * K);
      for (int t = lane; t < Tg; t += kWarp) {
#pragma unroll
        for (int jx = 0; jx < K; ++jx) {
          unsigned v8 = 0;
          if (t >= 1) {
#pragma unroll
            for (int p = 0; p < NP; ++p) v8 |= ((planes[(size_t)t * NP + p] >> (gg * K + jx)) & 1u) << p;
          }
          a.back[(sg + t) * K + jx] = (uint8_t)v8;
        }
      }
    }
  }

  // best final state per group (first index) and log joint
  int best_last = 0;
  R best_val = N::ninf();
  {
    R vals[K];
#pragma unroll
    for (int i = 0; i < K; ++i) vals[i] = __shfl_sync(kFull, delta, g * K + i);
    ArgMax<R, 0, K>::run(vals, best_val, best_last);
  }
  if (valid && j == 0) {
    a.log_joint[b] = (double)best_val;
    if (a.flags && oob) a.flags[2 * b + 1] |= 2;
  }
  __syncwarp();
  if (kGlobal) __threadfence_block();

  // ---- backtrace, one sequence (group) at a time with all 32 lanes -------
#pragma unroll 1
  for (int gg = 0; gg < G; ++gg) {
    const int64_t bb = warp_id * G + gg;
    if (bb >= a.B) break;
    const int Tg = __shfl_sync(kFull, T, gg * K);
    const int64_t sg = __shfl_sync(kFull, start, gg * K);
    const unsigned blast = (unsigned)__shfl_sync(kFull, best_last, gg * K);
    if (Tg <= 0) continue;
    const int L = (Tg + kWarp - 1) / kWarp;
    const int t0 = lane * L;
    const int t1 = min(t0 + L, Tg);
    const unsigned gsh = (unsigned)(gg * K);
    // compose the chunk's map: end state (t1-1) -> state at t0-1
    unsigned F = 0x76543210u;
    {
      const int tlo = max(t0, 1);
      constexpr int BB = 8;
#pragma unroll 1
      for (int tb = t1 - 1; tb >= tlo; tb -= BB) {
        unsigned plb[BB][NP > 0 ? NP : 1];
#pragma unroll
        for (int u = 0; u < BB; ++u) {
          const int t = tb - u;
#pragma unroll
          for (int p = 0; p < NP; ++p) plb[u][p] = t >= tlo ? planes[(size_t)t * NP + p] >> gsh : 0u;
        }
#pragma unroll
        for (int u = 0; u < BB; ++u) {
          if (tb - u < tlo) break;
          unsigned nf = 0;
#pragma unroll
          for (int e = 0; e < K; ++e) nf |= plane_lookup<NP>(plb[u], nib(F, e)) << (4 * e);
          F = nf;
        }
      }
    }
    // inclusive suffix scan: H_c = F_c o F_{c+1} o ... o F_31
    unsigned H = F;
#pragma unroll
    for (int d = 1; d < kWarp; d <<= 1) {
      const unsigned Hn = __shfl_down_sync(kFull, H, d);
      if (lane + d < kWarp) {
        unsigned c = 0;
#pragma unroll
        for (int e = 0; e < K; ++e) c |= nib(H, nib(Hn, e)) << (4 * e);
        H = c;
      }
    }
    unsigned Hnext = __shfl_down_sync(kFull, H, 1);
    if (lane == kWarp - 1) Hnext = 0x76543210u;
    unsigned cur = nib(Hnext, blast);
    // re-walk the chunk, staging the path in shared memory
    int64_t* out = a.path + sg;
    // re-walk in windows of kPathSlab steps [w0, w0+8): plane loads of the
    // window are issued together, then the dependent lookups run back to back
    const int wtop = ((L - 1) / kPathSlab) * kPathSlab;
#pragma unroll 1
    for (int w0 = wtop; w0 >= 0; w0 -= kPathSlab) {
      unsigned plc[kPathSlab][NP > 0 ? NP : 1];
#pragma unroll
      for (int u = 0; u < kPathSlab; ++u) {
        const int tu = t0 + w0 + u;
#pragma unroll
        for (int p = 0; p < NP; ++p)
          plc[u][p] = (tu >= 1 && tu < t1) ? planes[(size_t)tu * NP + p] >> gsh : 0u;
      }
#pragma unroll
      for (int u = kPathSlab - 1; u >= 0; --u) {
        const int tu = t0 + w0 + u;
        if (w0 + u < L && tu < t1) {
          pstage[lane * kPathPitch + u] = (int64_t)cur;
          if (tu >= 1) cur = plane_lookup<NP>(plc[u], cur);
        }
      }
      const int s = w0;
      if ((s % kPathSlab) == 0) {
        __syncwarp();
        // rows: lane-chunk c covers steps c*L + s .. +kPathSlab within [c*L, min(c*L+L,Tg))
#pragma unroll
        for (int rep = 0; rep < kPathSlab; ++rep) {
          const int idx = rep * kWarp + lane;  // element index over 32 rows x 8
          const int c = idx / kPathSlab, e = idx % kPathSlab;
          const int tt = c * L + s + e;
          if (s + e < L && tt < Tg) out[tt] = pstage[c * kPathPitch + e];
        }
        __syncwarp();
      }
    }
  }
}

}  // namespace lhmm
