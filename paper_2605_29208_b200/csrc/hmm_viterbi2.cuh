// hmm_viterbi2.cuh — batched Viterbi for 2 <= K <= 4, two lanes per sequence.
//
// Same contract and operation order as hmm_viterbi.cuh (inference.py:191-210,
// bit-exact backpointers and path), with a lighter layout for small K:
// lane (q, h) of a warp owns states j0 = 2h, 2h+1 of sequence q (16 sequences
// per warp).  Each step the partner's two scores arrive with two shuffles, the
// lane evaluates the 2 x K candidates and two first-index argmax trees, and
// appends its two 2-bit backpointers to a nibble accumulator that is stored
// to shared memory every 8 steps ([t/8][lane] words).
#pragma once

#include "hmm_viterbi.cuh"

namespace lhmm {

// shared words per warp ahead of the backpointer words: [16][33] int64 path
// staging, then the {T, start} table of the 16 sequences
constexpr int kVit2StageWords = 2 * 16 * kStagePitch + 16 * 3 + 4;

template <typename R, int K, int CFG>
__global__ void __launch_bounds__(128) viterbi2_kernel(const VitArgs a) {
  static_assert(K >= 2 && K <= 4, "two-lane Viterbi covers 2 <= K <= 4");
  typedef Num<R> N;
  typedef VitFams<CFG> VF;
  constexpr int KL = 2;  // states per lane
  constexpr int G = 16;  // sequences per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];

  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int64_t warp_id = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  const int q = lane >> 1, h = lane & 1;
  const int j0 = 2 * h;
  const int64_t b = warp_id * G + q;
  const bool valid = b < a.B;
  if (warp_id * G >= a.B) return;

  uint32_t* wsm = reinterpret_cast<uint32_t*>(smem_raw) + (size_t)wib * a.warp_smem_words;
  int64_t* pstage = reinterpret_cast<int64_t*>(wsm);  // path staging + sequence table
  uint32_t* bpw = kVit2StageWords + wsm;                // [ceil(Tmax/8)][32] nibble words

  const loghmm_model_t* __restrict__ md = a.model;
  const int64_t start = valid ? a.offsets[b] : 0;
  const int T = valid ? (int)(a.offsets[b + 1] - start) : 0;
  const R* __restrict__ y0g = reinterpret_cast<const R*>(a.y0) + start;
  const bool two = VF::TWO && a.n_streams > 1;
  const R* __restrict__ y1g = two ? reinterpret_cast<const R*>(a.y1) + start : y0g;

  // la[i][l] = log A[i][j0 + l] in natural row order i (the argmax scans i
  // ascending); padded states (>= K) get -inf everywhere.
  R la[4][KL];
  ExactEm<R, VF::F0> em0[KL];
  ExactEm<R, VF::F1> em1[KL];
  bool padj[KL];
#pragma unroll
  for (int l = 0; l < KL; ++l) {
    const int j = j0 + l;
    padj[l] = j >= K;
    const int js = padj[l] ? 0 : j;
#pragma unroll
    for (int i = 0; i < 4; ++i) la[i][l] = (i < K && !padj[l]) ? (R)md->log_A[i * K + js] : N::ninf();
    em0[l].load(md->em[0][js]);
    if (two) em1[l].load(md->em[1][js]);
    else em1[l].fam = LOGHMM_FAM_NONE;
  }
  bool oob = false, nan_seen = false;
  const double* lut = a.lut;
  const int lut_n = a.lut_n;

  int Tmax = T;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) Tmax = max(Tmax, __shfl_xor_sync(kFull, Tmax, o));
  const int Tlast = T > 0 ? T - 1 : 0;

  auto emis = [&](int l, R yv0, R yv1) -> R {
    nan_seen |= (yv0 != yv0) | (yv1 != yv1);  // inference.py:117-118
    R lb = em0[l].eval(yv0, lut, lut_n, oob);
    if (two) lb = N::add(lb, em1[l].eval(yv1, lut, lut_n, oob));
    return padj[l] ? N::ninf() : lb;
  };

  // ---- forward max-plus recursion ---------------------------------------
  R d[KL];
#pragma unroll
  for (int l = 0; l < KL; ++l) {
    d[l] = N::ninf();
    if (T > 0 && !padj[l]) d[l] = N::add((R)md->log_pi[j0 + l], emis(l, y0g[0], two ? y1g[0] : R(0)));
  }
  uint32_t nib = 0;  // 8 steps x (2 states x 2 bits)

  auto step = [&](int t, const R (&lb)[KL]) {
    // full score vector in natural order: lane h=0 owns 0,1; h=1 owns 2,3
    const R o0 = __shfl_xor_sync(kFull, d[0], 1);
    const R o1 = __shfl_xor_sync(kFull, d[1], 1);
    R full[4];
    full[0] = h ? o0 : d[0];
    full[1] = h ? o1 : d[1];
    full[2] = h ? d[0] : o0;
    full[3] = h ? d[1] : o1;
    const bool act = t < T;
    uint32_t bits = 0;
#pragma unroll
    for (int l = 0; l < KL; ++l) {
      R cand[K];
#pragma unroll
      for (int i = 0; i < K; ++i) cand[i] = N::add(full[i], la[i][l]);
      R best;
      int bi;
      ArgMax<R, 0, K>::run(cand, best, bi);
      d[l] = act ? N::add(best, lb[l]) : d[l];
      bits |= (uint32_t)bi << (2 * l);
    }
    nib |= bits << (4 * (t & 7));
    if ((t & 7) == 7 || t == Tmax - 1) {
      bpw[(size_t)(t >> 3) * kWarp + lane] = nib;
      nib = 0;
    }
  };

  // Software-pipelined: while the score chain of block k runs, the emission
  // terms of block k+1 are evaluated in the same instruction stream (they are
  // independent of the chain), and y is loaded two blocks ahead.
  constexpr int U = 8;
  R y0a[U], y1a[U];  // y of block k+2 (in flight)
  R lbs[U][KL], lbn[U][KL];
#pragma unroll
  for (int u = 0; u < U; ++u) {
    const int t1_ = min(1 + u, Tlast), t2_ = min(1 + U + u, Tlast);
#pragma unroll
    for (int l = 0; l < KL; ++l) lbs[u][l] = emis(l, y0g[t1_], two ? y1g[t1_] : R(0));
    y0a[u] = y0g[t2_];
    y1a[u] = two ? y1g[t2_] : R(0);
  }
  int t = 1;
#pragma unroll 1
  for (; t + U <= Tmax; t += U) {
    R y0c[U], y1c[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      y0c[u] = y0a[u];
      y1c[u] = y1a[u];
      const int tt = min(t + 2 * U + u, Tlast);
      y0a[u] = y0g[tt];
      y1a[u] = two ? y1g[tt] : R(0);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
#pragma unroll
      for (int l = 0; l < KL; ++l) lbn[u][l] = emis(l, y0c[u], y1c[u]);
      step(t + u, lbs[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int l = 0; l < KL; ++l) lbs[u][l] = lbn[u][l];
  }
  // tail: lbs holds the emissions of steps t..t+U-1 (clamped loads)
#pragma unroll
  for (int u = 0; u < U; ++u)
    if (t + u < Tmax) step(t + u, lbs[u]);

  // best final state (first index) and log joint
  int best_last = 0;
  R best_val = N::ninf();
  {
    const R o0 = __shfl_xor_sync(kFull, d[0], 1);
    const R o1 = __shfl_xor_sync(kFull, d[1], 1);
    R full[4];
    full[0] = h ? o0 : d[0];
    full[1] = h ? o1 : d[1];
    full[2] = h ? d[0] : o0;
    full[3] = h ? d[1] : o1;
    ArgMax<R, 0, K>::run(full, best_val, best_last);
  }
  if (valid && h == 0) {
    a.log_joint[b] = (double)best_val;
    if (a.flags && (oob || nan_seen)) a.flags[2 * b + 1] |= (oob ? 2 : 0) | (nan_seen ? 1 : 0);
  }
  __syncwarp();

  // back_t[v] for sequence qq: 2 bits at (t%8)*4 + (v&1)*2 of word [t/8][2qq + (v>>1)]
  auto tbl_of = [&](int qq, int t2) -> unsigned {
    const uint32_t* row = bpw + (size_t)(t2 >> 3) * kWarp + 2 * qq;
    const unsigned sh = 4u * (unsigned)(t2 & 7);
    return ((row[0] >> sh) & 0xFu) | (((row[1] >> sh) & 0xFu) << 4);  // 2 bits per state
  };

  // optional byte table of backpointers (tests)
  if (a.back != nullptr) {
#pragma unroll 1
    for (int gg = 0; gg < G; ++gg) {
      const int64_t bb = warp_id * G + gg;
      if (bb >= a.B) break;
      const int Tg = __shfl_sync(kFull, T, 2 * gg);
      const int64_t sg = __shfl_sync(kFull, start, 2 * gg);
      for (int t2 = lane; t2 < Tg; t2 += kWarp) {
        const unsigned tb = t2 >= 1 ? tbl_of(gg, t2) : 0u;
#pragma unroll
        for (int jx = 0; jx < K; ++jx) a.back[(sg + t2) * K + jx] = (uint8_t)((tb >> (2 * jx)) & 3u);
      }
    }
  }

  // ---- backtrace: lane 2q walks sequence q from its end ------------------
  // Warp-uniform windows of 32 steps (four 8-step rows of backpointer words)
  // from the top: per row the eight 8-bit step tables are unpacked with
  // constant shifts (independent of the walk), the dependent lookups run back
  // to back, and the states are staged in shared memory [q][32]; each window
  // is then written with one coalesced 256-byte store per sequence.
  int64_t* stage = pstage;                                            // [G][kStagePitch]
  int2* seqtab = reinterpret_cast<int2*>(pstage + G * kStagePitch);  // [G] {T, start lo}
  int* seqhi = reinterpret_cast<int*>(seqtab + G);                   // [G] start hi
  if (h == 0) {
    seqtab[q] = make_int2(valid ? T : 0, (int)(uint32_t)start);
    seqhi[q] = (int)(start >> 32);
  }
  __syncwarp();
  unsigned cur = (unsigned)best_last;
  const bool walker = h == 0 && valid;
  const uint32_t* col = bpw + 2 * q;
  const int wtop = Tmax > 0 ? (Tmax - 1) >> 5 : -1;
#pragma unroll 1
  for (int w = wtop; w >= 0; --w) {
#pragma unroll
    for (int r = 3; r >= 0; --r) {
      const int row = 4 * w + r;
      if (walker && row * 8 < T) {
        const uint32_t w0 = col[(size_t)row * kWarp], w1 = col[(size_t)row * kWarp + 1];
        unsigned tbs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) tbs[u] = ((w0 >> (4 * u)) & 0xFu) | (((w1 >> (4 * u)) & 0xFu) << 4);
#pragma unroll
        for (int u = 7; u >= 0; --u) {
          if (row * 8 + u < T) {  // step row*8+u holds cur; its table gives step -1
            stage[q * kStagePitch + r * 8 + u] = (int64_t)cur;
            cur = (tbs[u] >> (2 * cur)) & 3u;
          }
        }
      }
    }
    __syncwarp();
#pragma unroll 4
    for (int qq = 0; qq < G; ++qq) {
      const int2 e = seqtab[qq];
      const int tt = w * 32 + lane;
      if (tt < e.x) {
        const int64_t st = ((int64_t)seqhi[qq] << 32) | (uint32_t)e.y;
        a.path[st + tt] = stage[qq * kStagePitch + lane];
      }
    }
    __syncwarp();
  }
}

}  // namespace lhmm
