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
// (sequence, step).  The backtrace splits each sequence into K segments, one
// per lane of its group: every lane composes its segment's backpointer map
// for all K possible end states, the maps are resolved top-down with K-1
// shuffles, and each lane re-walks its segment writing the path through a
// shared-memory staging buffer (coalesced int64 stores).
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
  int sparse_ok;  // large K: take the structural-zero path when log A allows it
};


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

// As ArgMax, with the winning index delivered directly as the warp's NP
// bit-plane masks: every internal node of the tree contributes one ballot of
// its decision, and bit p of the index is selected down the tree with
// warp-uniform LOP3s (leaf index bits fold to constants).  K-1 ballots in
// total, no per-lane index arithmetic.
template <typename R, int LO, int HI, int NP>
struct ArgMaxB {
  static __device__ __forceinline__ void run(const R* c, R& v, unsigned (&m)[NP > 0 ? NP : 1]) {
    if constexpr (HI - LO == 1) {
      v = c[LO];
#pragma unroll
      for (int p = 0; p < (NP > 0 ? NP : 1); ++p) m[p] = ((LO >> p) & 1) ? 0xFFFFFFFFu : 0u;
    } else {
      constexpr int MID = LO + (HI - LO + 1) / 2;
      R lv, rv;
      unsigned lm[NP > 0 ? NP : 1], rm[NP > 0 ? NP : 1];
      ArgMaxB<R, LO, MID, NP>::run(c, lv, lm);
      ArgMaxB<R, MID, HI, NP>::run(c, rv, rm);
      const unsigned bt = NP > 0 ? __ballot_sync(kFull, rv > lv) : 0u;
      v = fmax(lv, rv);
#pragma unroll
      for (int p = 0; p < (NP > 0 ? NP : 1); ++p) m[p] = (bt & rm[p]) | (~bt & lm[p]);
    }
  }
};

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

// Per-warp shared memory of the K-lane kernel, in 32-bit words:
//   [union: forward y staging ring NS x 3 slots x G x kStagePitch elements |
//           backtrace: spread LUT, then path staging (kVitPathWords)]
//   [step tables, 4 words per step, unless they live in the global workspace]
// Step table of step t (4 words): the forward writes the NP ballot bit-planes
// into words 0..NP-1; before the backtrace they are expanded in place so that
// bit p of back_t[state] of lane-state i = g*K + j sits at bit 4*i + p (one
// nibble per lane-state, 128 bits per step).
constexpr int kStagePitch = 33;  // elements per staged sequence row (32 steps + 1)
constexpr int kStepWords = 4;
// backtrace staging: [32 lanes][17] int64 windows + [32] int64 bases + [32] first-valid
constexpr int kVitPathWords = 256 + kWarp * 17 * 2 + kWarp * 2 + kWarp;
__host__ __device__ constexpr int vit_union_words(int K, int esz, int ns) {
  return ((kVitPathWords > ns * 3 * (kWarp / K) * kStagePitch * esz / 4
               ? kVitPathWords
               : ns * 3 * (kWarp / K) * kStagePitch * esz / 4) +
          3) &
         ~3;
}
__host__ __device__ constexpr int vit_stage_words(int K, int esz, int ns) {
  return vit_union_words(K, esz, ns);
}

__device__ __forceinline__ void st_global_pred(int64_t* p, int64_t v, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q st.global.b64 [%0], %1;\n}" ::"l"(p),
      "l"(v), "r"((unsigned)pred)
      : "memory");
}

template <typename R, int K, int CFG, bool kGlobal>
__global__ void __launch_bounds__(128) viterbi_small_kernel(const VitArgs a) {
  typedef Num<R> N;
  typedef VitFams<CFG> VF;
  constexpr int G = kWarp / K;
  constexpr int NP = Bits<K>::NP;
  constexpr int NPa = NP > 0 ? NP : 1;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const int g = lane / K;
  const int j = lane - g * K;
  const int64_t b = warp_id * G + g;
  const bool valid = (g < G) && (b < a.B);
  if (warp_id * G >= a.B) return;  // whole warp idle

  constexpr int NS = VF::TWO ? 2 : 1;
  uint32_t* wsm = reinterpret_cast<uint32_t*>(smem_raw) + (size_t)wib * a.warp_smem_words;
  uint32_t* lut8 = wsm;                                      // [256] (backtrace)
  int64_t* stage = reinterpret_cast<int64_t*>(wsm + 256);    // backtrace staging
  R* yring = reinterpret_cast<R*>(wsm);                      // [NS][3][G][kStagePitch]
  uint32_t* planes = kGlobal ? a.planes_ws + warp_id * a.plane_words
                             : wsm + vit_stage_words(K, sizeof(R), NS);

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
  bool oob = false, nan_seen = false;
  const double* lut = a.lut;
  const int lut_n = a.lut_n;

  int Tmax = T, Tmin = valid ? T : 0x7fffffff;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Tmax = max(Tmax, __shfl_xor_sync(kFull, Tmax, o));
    Tmin = min(Tmin, __shfl_xor_sync(kFull, Tmin, o));
  }
  __syncwarp();

  // ok: the step exists (the ring also feeds steps past the sequence end)
  auto emis = [&](R yv0, R yv1, bool ok) -> R {
    nan_seen |= ok & ((yv0 != yv0) | (yv1 != yv1));  // inference.py:117-118
    R lb = em0.eval(yv0, lut, lut_n, oob);
    if (two) lb = N::add(lb, em1.eval(yv1, lut, lut_n, oob));
    return lb;
  };

  // ---- forward max-plus recursion ---------------------------------------
  R delta = N::ninf();
  if (T > 0) delta = N::add((R)md->log_pi[jj], emis(y0g[0], two ? y1g[0] : R(0), true));

  // One recursion step.  Every lane executes it (no divergence around the
  // shuffles / ballots); lanes past their sequence end keep their score.  The
  // argmax tree returns the step's bit-planes directly (one ballot per tree
  // decision), lane 0 stores them.
  auto step = [&](int t, R lb, bool act) {
    R cand[K];
#pragma unroll
    for (int i = 0; i < K; ++i) cand[i] = N::add(__shfl_sync(kFull, delta, g * K + i), la[i]);
    R best;
    unsigned w[NPa];
    ArgMaxB<R, 0, K, NP>::run(cand, best, w);
    const R nd = N::add(best, lb);
    delta = act ? nd : delta;
    if constexpr (NP > 0) {
      if (lane == 0) {
        if constexpr (NP == 1) {
          planes[(size_t)t * kStepWords] = w[0];
        } else if constexpr (NP == 2) {
          *reinterpret_cast<uint2*>(planes + (size_t)t * kStepWords) = make_uint2(w[0], w[1]);
        } else {
          *reinterpret_cast<uint4*>(planes + (size_t)t * kStepWords) = make_uint4(w[0], w[1], w[2], 0u);
        }
      }
    }
  };

  // Observations are staged through a 3-slot shared-memory ring of 32-step
  // chunks (chunk c = steps 1 + 32c .. 32 + 32c) with cp.async, two chunks
  // ahead, so the loads never sit on a register scoreboard.  Within a
  // chunk the recursion is software-pipelined in halves: while the score
  // chain of one half runs, the emission terms of the next half are
  // evaluated in the same instruction stream.
  const int nchunks = Tmax > 1 ? (Tmax - 1 + 31) / 32 : 0;
  auto ring_at = [&](int s, int st, int gg) -> R* {
    return yring + ((size_t)(st * 3 + s) * G + gg) * kStagePitch;
  };
  const int Tlast = T > 0 ? T - 1 : 0;
  auto issue_chunk = [&](int c) {
    if (c < nchunks && g < G) {
      const int s = c % 3;
      R* d0 = ring_at(s, 0, g);
      R* d1 = ring_at(s, NS - 1, g);
      // the K lanes of the group copy steps j, j+K, ... of their own sequence
#pragma unroll
      for (int m = 0; m < (32 + K - 1) / K; ++m) {
        const int u = j + K * m;
        if (u < 32) {
          const int idx = min(1 + 32 * c + u, Tlast);
          cp_async<sizeof(R)>(d0 + u, y0g + idx, T > 1);
          if (NS > 1 && two) cp_async<sizeof(R)>(d1 + u, y1g + idx, T > 1);
        }
      }
    }
    cp_async_commit();
  };
  constexpr int H = 16;  // half chunk
  R lbs[H], lbn[H];
  issue_chunk(0);
  issue_chunk(1);
  cp_async_wait<1>();
  __syncwarp();
  {
    const R* r0 = ring_at(0, 0, g);
    const R* r1 = ring_at(0, NS - 1, g);
#pragma unroll
    for (int u = 0; u < H; ++u) lbs[u] = emis(r0[u], two ? r1[u] : R(0), 1 + u < T);
  }
#pragma unroll 1
  for (int c = 0; c < nchunks; ++c) {
    issue_chunk(c + 2);
    const int t = 1 + 32 * c;
    const int s = c % 3, s1 = s == 2 ? 0 : s + 1;
    const R* r0 = ring_at(s, 0, g);
    const R* r1 = ring_at(s, NS - 1, g);
    const R* n0 = ring_at(s1, 0, g);
    const R* n1 = ring_at(s1, NS - 1, g);
    if (t + 32 <= Tmin) {  // every sequence of the warp covers the chunk
#pragma unroll
      for (int u = 0; u < H; ++u) {
        lbn[u] = emis(r0[H + u], two ? r1[H + u] : R(0), t + H + u < T);
        step(t + u, lbs[u], true);
      }
      cp_async_wait<1>();
      __syncwarp();
#pragma unroll
      for (int u = 0; u < H; ++u) {
        lbs[u] = emis(n0[u], two ? n1[u] : R(0), t + 32 + u < T);
        step(t + H + u, lbn[u], true);
      }
    } else {
#pragma unroll
      for (int u = 0; u < H; ++u) {
        lbn[u] = emis(r0[H + u], two ? r1[H + u] : R(0), t + H + u < T);
        step(t + u, lbs[u], t + u < T);
      }
      cp_async_wait<1>();
      __syncwarp();
#pragma unroll
      for (int u = 0; u < H; ++u) {
        lbs[u] = emis(n0[u], two ? n1[u] : R(0), t + 32 + u < T);
        step(t + H + u, lbn[u], t + H + u < T);
      }
    }
  }
  cp_async_wait_all();
  __syncwarp();
  if (kGlobal) __threadfence_block();
  // optional byte table of backpointers (tests), rebuilt from the planes
  if (a.back != nullptr) {
#pragma unroll 1
    for (int gg = 0; gg < G; ++gg) {
      const int64_t bb = warp_id * G + gg;
      if (bb >= a.B) break;
      const int Tg = __shfl_sync(kFull, T, gg * K);
      const int64_t sg = __shfl_sync(kFull, start, gg * K);
      for (int t2 = lane; t2 < Tg; t2 += kWarp) {
#pragma unroll
        for (int jx = 0; jx < K; ++jx) {
          unsigned v8 = 0;
          if (t2 >= 1) {
#pragma unroll
            for (int p = 0; p < NP; ++p)
              v8 |= ((planes[(size_t)t2 * kStepWords + p] >> (gg * K + jx)) & 1u) << p;
          }
          a.back[(sg + t2) * K + jx] = (uint8_t)v8;
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
    if (a.flags && (oob || nan_seen)) a.flags[2 * b + 1] |= (oob ? 2 : 0) | (nan_seen ? 1 : 0);
  }

  // ---- backtrace: the K lanes of group g walk K segments of its sequence --
  // Lane j owns steps [lo, hi) = [j*Ls, (j+1)*Ls) n [0, T), Ls = ceil(T/K).
  //  (0) expand: the bit-planes of every step are spread to one nibble per
  //      lane-state (byte LUT), so a group's back_t is a K-nibble word;
  //  (1) compose: each lane composes its segment's maps bottom-up with byte
  //      permutes, G <- G o back_t (PRMT, selector = back_t's nibbles), giving
  //      the state just before the segment for every state at its last step;
  //  (2) resolve: the group's final state is pushed down through the maps of
  //      the segments above (K-1 shuffles);
  //  (3) re-walk: each lane walks its segment top-down (two dependent
  //      instructions per step), staging 16-step windows in shared memory,
  //      which the warp writes as coalesced rows.
  if constexpr (NP > 0) {
    for (int i = lane; i < 256; i += kWarp) {
      uint32_t x = (uint32_t)i;
      x = (x | (x << 12)) & 0x000F000Fu;
      x = (x | (x << 6)) & 0x03030303u;
      x = (x | (x << 3)) & 0x11111111u;
      lut8[i] = x;
    }
    __syncwarp();
#pragma unroll 1
    for (int t = 1 + lane; t < Tmax; t += kWarp) {
      uint32_t* st = planes + (size_t)t * kStepWords;
      uint32_t pw[NPa];
#pragma unroll
      for (int p = 0; p < NP; ++p) pw[p] = st[p];
      uint4 r = make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        r.x |= lut8[pw[p] & 0xFFu] << p;
        r.y |= lut8[(pw[p] >> 8) & 0xFFu] << p;
        r.z |= lut8[(pw[p] >> 16) & 0xFFu] << p;
        r.w |= lut8[pw[p] >> 24] << p;
      }
      *reinterpret_cast<uint4*>(st) = r;
    }
    __syncwarp();
    if (kGlobal) __threadfence_block();
  }
  // back_t of this lane's group as K nibbles (garbage above nibble K-1)
  const int boff = 4 * K * g;
  const int bq = (boff >> 5) & 3, bsh = boff & 31;
  auto table = [&](int t) -> uint32_t {
    const uint32_t* st = planes + (size_t)t * kStepWords + bq;
    if constexpr ((32 % (4 * K)) == 0) {
      return st[0] >> bsh;
    } else {
      return __funnelshift_r(st[0], bq < 3 ? st[1] : 0u, bsh);
    }
  };
  const int Ls = (T + K - 1) / K;
  const int lo = min(j * Ls, T), hi = min(lo + Ls, T);
  const int seg = hi - lo;
  int segmax = seg;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) segmax = max(segmax, __shfl_xor_sync(kFull, segmax, o));
  unsigned cur = (unsigned)best_last;
  if constexpr (K > 1) {
    uint32_t Glo = 0x03020100u, Ghi = 0x07060504u;  // identity map, one byte per state
    const int tlow = max(lo, 1);
#pragma unroll 1
    for (int s0 = 0; s0 < segmax; s0 += 8) {
      uint32_t tb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int t = tlow + s0 + u;
        tb[u] = t < hi ? table(t) : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const bool ok = tlow + s0 + u < hi;
        const uint32_t nlo = __byte_perm(Glo, Ghi, tb[u]);
        if constexpr (K > 4) {
          const uint32_t nhi = __byte_perm(Glo, Ghi, tb[u] >> 16);
          Ghi = ok ? nhi : Ghi;
        }
        Glo = ok ? nlo : Glo;
      }
    }
#pragma unroll
    for (int jj = K - 1; jj >= 1; --jj) {
      const int src = (g * K + jj) & 31;
      const uint32_t qlo = __shfl_sync(kFull, Glo, src);
      const uint32_t qhi = K > 4 ? __shfl_sync(kFull, Ghi, src) : 0u;
      if (j < jj) cur = __byte_perm(qlo, qhi, cur) & 0xFFu;
    }
  }
  __syncwarp();
  constexpr int WP = 17;  // staging pitch (int64) of one lane's 16-step window
  int64_t* pst = stage + lane * WP;
  int64_t* dgb = stage + kWarp * WP;              // [32] global index of window position 0
  int* dfv = reinterpret_cast<int*>(dgb + kWarp);  // [32] first valid window position
  unsigned c4 = cur << 2;
#pragma unroll 1
  for (int s0 = 0; s0 < segmax; s0 += 16) {
    // window: steps [hi-16-s0, hi-s0), position i <-> step hi-16-s0+i
    uint32_t tb[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      const int t = hi - 1 - s0 - u;
      tb[u] = (NP > 0 && t >= lo && t >= 1) ? table(t) : 0u;
      if (K <= 4) tb[u] <<= 2;
    }
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      if (hi - 1 - s0 - u >= lo) {  // step hi-1-s0-u holds c4/4; its table gives the step before
        pst[15 - u] = (int64_t)(c4 >> 2);
        if constexpr (K <= 4) c4 = (tb[u] >> c4) & 0xCu;
        else c4 = ((tb[u] >> c4) & 7u) << 2;
      }
    }
    dgb[lane] = start + hi - 16 - s0;
    dfv[lane] = 16 - max(0, min(16, seg - s0));
    __syncwarp();
#pragma unroll 4
    for (int it = 0; it < 16; ++it) {
      const int src = 2 * it + (lane >> 4), e = lane & 15;
      st_global_pred(a.path + dgb[src] + e, stage[src * WP + e], e >= dfv[src]);
    }
    __syncwarp();
  }
}

}  // namespace lhmm
