// hmm_capi.cu — the extern "C" boundary (include/loghmm_b200.h).
//
// Host-side argument checking, launch geometry, shared-memory carve and
// dtype / K / family dispatch.  No allocation, no global mutable state.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <climits>

#include "hmm_large.cuh"
#include "hmm_launch.cuh"
#include "hmm_mstep.cuh"

namespace lhmm {
#define X(K) LHMM_EXTERN_INST(float, K) LHMM_EXTERN_INST(double, K)
X(1) X(2) X(3) X(4) X(5) X(6) X(7) X(8)
#undef X

// ---- standalone emission kernel (emission_log_matrix) --------------------
template <typename R>
__global__ void __launch_bounds__(256) emission_kernel(const loghmm_model_t* __restrict__ m,
                                                       const R* __restrict__ y0,
                                                       const R* __restrict__ y1, int64_t N,
                                                       int K, const double* lut, int lut_n,
                                                       R* __restrict__ out) {
  const bool two = m->n_streams > 1;
  for (int64_t n = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; n < N;
       n += (int64_t)gridDim.x * blockDim.x) {
    bool oob = false;
    const R v0 = y0[n];
    const R v1 = two ? y1[n] : R(0);
    for (int j = 0; j < K; ++j) {
      R v = exact_logb<R>(m->em[0][j], v0, lut, lut_n, oob);
      if (two) v = Num<R>::add(v, exact_logb<R>(m->em[1][j], v1, lut, lut_n, oob));
      out[n * K + j] = v;
    }
  }
}

static inline int cfg_of(const loghmm_model_t* h, int* fams_mask) {
  const int K = h->K;
  int m0 = 0, m1 = 0;
  for (int j = 0; j < K; ++j) {
    m0 |= 1 << h->em[0][j].family;
    if (h->n_streams > 1) m1 |= 1 << h->em[1][j].family;
  }
  *fams_mask = (m0 & 0xffff) | ((m1 & 0xffff) << 16);
  if (h->n_streams == 1) {
    if (m0 == (1 << LOGHMM_FAM_GAUSSIAN)) return kCfgGauss;
    if (m0 == (1 << LOGHMM_FAM_STUDENT_T)) return kCfgStudent;
    if (m0 == (1 << LOGHMM_FAM_GAMMA)) return kCfgGamma;
    if (m0 == (1 << LOGHMM_FAM_VON_MISES)) return kCfgVonMises;
    if (m0 == (1 << LOGHMM_FAM_POISSON)) return kCfgPoisson;
  } else if (m0 == (1 << LOGHMM_FAM_GAMMA) && m1 == (1 << LOGHMM_FAM_VON_MISES)) {
    return kCfgGammaVM;
  }
  return kCfgMixed;
}

static inline int gcd_(int a, int b) { return b ? gcd_(b, a % b) : a; }

// Launch geometry for the K<=8 forward-backward kernel.
struct FBGeom {
  bool global;
  int L_align, Lmax, y_pitch, a_pitch, s_pitch, warp_elems, wpb;
  size_t smem;
};

static FBGeom fb_geom(int K, int esz, int n_streams, int64_t max_T) {
  FBGeom g{};
  const int kb = K * esz;
  g.L_align = 16 / gcd_(16, kb);
  int L = (int)((max_T + kWarp - 1) / kWarp);
  if (L < 1) L = 1;
  g.Lmax = ((L + g.L_align - 1) / g.L_align) * g.L_align;
  // y: contiguous [32*Lmax] with one pad element per 32 (t + t/32), per lane row of
  // the carve = y_pitch elements so that 32*y_pitch covers it
  g.y_pitch = g.Lmax + (g.Lmax + 31) / 32 + 1;
  const int V = (kb % 16 == 0) ? 16 : (kb % 8 == 0) ? 8 : 4;
  (void)V;
  g.a_pitch = 0;  // beta~ lives in the global (L2-resident) workspace
  int sunits = kSlab * kb / 16;
  if ((sunits & 1) == 0) sunits += 1;
  g.s_pitch = sunits * 16 / esz;
  const int64_t smem_elems = (int64_t)kWarp * (g.y_pitch * n_streams + g.a_pitch + 2 * g.s_pitch);
  const int64_t bytes = smem_elems * esz;
  g.global = bytes > 110 * 1024;
  // + beta~ prefetch ring: 8 steps x 32 lanes x K
  g.warp_elems = (g.global ? kWarp * 2 * g.s_pitch : (int)smem_elems) + 8 * kWarp * K;
  const int64_t wbytes = (int64_t)g.warp_elems * esz;
  g.wpb = (int)std::max<int64_t>(1, std::min<int64_t>(4, (220 * 1024) / wbytes));
  g.smem = (size_t)(wbytes * g.wpb);
  return g;
}

struct VitGeom {
  bool global;
  int wpb;
  int64_t plane_words;
  int warp_words;
  size_t smem;
};

// esz: element size of the observations; ns: observation streams staged by
// the kernel instantiation (2 for the two-stream configurations).
static VitGeom vit_geom(int K, int64_t max_T, int esz = 8, int ns = 2) {
  VitGeom g{};
  // steps are processed in whole 32-step chunks: room for 32 * ceil(T/32) + 1
  // steps (plus one step of slack for the table reads), kStepWords words each
  g.plane_words = ((max_T + 31) / 32 + 2) * 32 * kStepWords;
  const int64_t stage_words = vit_stage_words(K, esz, ns);
  g.global = g.plane_words > 12 * 1024;  // > 48 KB of step tables per warp
  g.warp_words = (int)(stage_words + (g.global ? 0 : g.plane_words));
  g.warp_words = (g.warp_words + 3) & ~3;
  g.wpb = (int)std::max<int64_t>(1, std::min<int64_t>(4, (220 * 1024) / ((int64_t)g.warp_words * 4)));
  // warps per CTA: smaller CTAs spread the (one partial wave) Viterbi grid
  // over more SMs next to the concurrent forward-backward kernel
  if (const char* env = getenv("LOGHMM_VIT_WPB")) g.wpb = std::max(1, std::min(g.wpb, atoi(env)));
  g.smem = (size_t)g.warp_words * 4 * g.wpb;
  return g;
}

template <typename R>
static cudaError_t dispatch_fb_small(int K, const FBArgs& a, int cfg, bool gl, dim3 grid,
                                     dim3 block, size_t smem, cudaStream_t st) {
  switch (K) {
    case 1: return launch_fb_small<R, 1>(a, cfg, gl, grid, block, smem, st);
    case 2: return launch_fb_small<R, 2>(a, cfg, gl, grid, block, smem, st);
    case 3: return launch_fb_small<R, 3>(a, cfg, gl, grid, block, smem, st);
    case 4: return launch_fb_small<R, 4>(a, cfg, gl, grid, block, smem, st);
    case 5: return launch_fb_small<R, 5>(a, cfg, gl, grid, block, smem, st);
    case 6: return launch_fb_small<R, 6>(a, cfg, gl, grid, block, smem, st);
    case 7: return launch_fb_small<R, 7>(a, cfg, gl, grid, block, smem, st);
    default: return launch_fb_small<R, 8>(a, cfg, gl, grid, block, smem, st);
  }
}

// Chain-warp Viterbi (hmm_viterbi3.cuh; K in [2,4], sequences whose
// backpointer bytes fit in shared memory).  LOGHMM_VIT_ALGO = chain | lanes
// forces a layout, LOGHMM_VIT_NW picks 8 or 16 warps per CTA.  Default:
// * Gaussian / Poisson emissions (a handful of IEEE operations): the
//   K-lanes-per-sequence kernel.  Alone the chain-warp kernel is the faster
//   one at 16 warps (66 vs 70 us at config 2), but inside the step, next to
//   the forward-backward kernel, the two issue about the same number of
//   instructions and the step is bound by issue slots: 135 vs 139 us.
// * families whose exact density calls log1p / log / cos (Student-t, Gamma,
//   von Mises, joint, mixed): the chain-warp kernel, 16 warps — its helper
//   warps evaluate the densities T-parallel, while the K-lane kernel
//   evaluates them inside the sequential recursion (config 3: 1.14 ms).
static bool vit3_ok(int K, int esz, int64_t max_T, int cfg, int* nw, size_t* smem) {
  if (K < 2 || K > 4) return false;
  const char* env = getenv("LOGHMM_VIT_ALGO");
  const bool cheap = cfg == kCfgGauss || cfg == kCfgPoisson;
  if (env && strcmp(env, "lanes") == 0) return false;
  if (!(env && strcmp(env, "chain") == 0) && cheap) return false;
  const size_t bytes = v3_smem_bytes(esz, max_T);
  if (bytes > 200 * 1024) return false;
  *smem = bytes;
  *nw = cheap ? 8 : 16;
  if (const char* e2 = getenv("LOGHMM_VIT_NW")) *nw = atoi(e2) >= 16 ? 16 : 8;
  return true;
}

template <typename R>
static cudaError_t dispatch_vit3(int K, const VitArgs& a, int cfg, int nw, dim3 grid, size_t smem,
                                 cudaStream_t st) {
  switch (K) {
    case 2: return launch_vit3<R, 2>(a, cfg, nw, grid, smem, st);
    case 3: return launch_vit3<R, 3>(a, cfg, nw, grid, smem, st);
    default: return launch_vit3<R, 4>(a, cfg, nw, grid, smem, st);
  }
}

template <typename R>
static cudaError_t dispatch_vit_small(int K, const VitArgs& a, int cfg, bool gl, dim3 grid,
                                      dim3 block, size_t smem, cudaStream_t st) {
  switch (K) {
    case 1: return launch_vit_small<R, 1>(a, cfg, gl, grid, block, smem, st);
    case 2: return launch_vit_small<R, 2>(a, cfg, gl, grid, block, smem, st);
    case 3: return launch_vit_small<R, 3>(a, cfg, gl, grid, block, smem, st);
    case 4: return launch_vit_small<R, 4>(a, cfg, gl, grid, block, smem, st);
    case 5: return launch_vit_small<R, 5>(a, cfg, gl, grid, block, smem, st);
    case 6: return launch_vit_small<R, 6>(a, cfg, gl, grid, block, smem, st);
    case 7: return launch_vit_small<R, 7>(a, cfg, gl, grid, block, smem, st);
    default: return launch_vit_small<R, 8>(a, cfg, gl, grid, block, smem, st);
  }
}

static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// Forward-backward decomposition.  Equal-length batches whose length splits
// into <= 32 chunks of a multiple-of-8 length take the chunk-operator +
// meet-in-the-middle kernel (hmm_fbc.cuh); everything else (ragged batches,
// per-step xi output, long sequences, K = 1) takes the chunked scan
// (hmm_fb.cuh).  LOGHMM_FB_ALGO=chunked forces the latter (tests exercise both).
static int fbc_chunk_len(int64_t T) {
  if (T < 8) return 0;
  int64_t L = (T + kWarp - 1) / kWarp;
  L = (L + 7) / 8 * 8;
  for (; L <= T; L += 8)
    if (T % L == 0) return (int)L;
  return 0;
}

static int fbc_warp_elems(int K, int esz, int L) {
#define C_(KK) case KK: return esz == 4 ? fb_chunk_warp_elems<float, KK>(L) : 0;
  switch (K) { C_(2) C_(3) C_(4) C_(5) C_(6) C_(7) C_(8) default: return 0; }
#undef C_
}

// tensor-memory columns for the fp32 park: L steps x KP (K padded to 1,2,4,8)
static int fbc_tm_cols(int K, int L) {
  const int kp = K <= 1 ? 1 : K <= 2 ? 2 : K <= 4 ? 4 : 8;
  int n = 32;
  while (n < L * kp) n <<= 1;
  return n;
}

constexpr int kFbcWarpsPerBlock = 4;  // one warpgroup (kFbcWarps)
constexpr size_t kFbcMaxWarpBytes = 100 * 1024;

static bool use_fbc(int K, int n_streams, int64_t B, int64_t N, int64_t max_T, int esz, bool xi, int* L_out,
                    size_t* warp_bytes) {
  const char* env = getenv("LOGHMM_FB_ALGO");
  if (env && strcmp(env, "chunked") == 0) return false;
  // fp64 stays on the chunked scan until its exp2/log2 are cheaper than
  // libm's (the re-sweep evaluates them once more per step than the scan)
  if (esz != 4) return false;
  if (K < 2 || K > 8 || xi || max_T < 8 || N != B * max_T || max_T > INT32_MAX) return false;
  const int L = fbc_chunk_len(max_T);
  if (L == 0) return false;
  (void)n_streams;
  const size_t wb = (size_t)fbc_warp_elems(K, esz, L) * esz;
  if (wb > kFbcMaxWarpBytes) return false;
  if (esz == 4 && fbc_tm_cols(K, L) > 256) return false;  // tensor-memory park
  *L_out = L;
  *warp_bytes = wb;
  return true;
}

template <typename R>
static cudaError_t dispatch_fb_chunk(int K, const FBCArgs& a, int cfg, dim3 grid, dim3 block,
                                     size_t smem, cudaStream_t st) {
  switch (K) {
    case 2: return launch_fb_chunk<R, 2>(a, cfg, grid, block, smem, st);
    case 3: return launch_fb_chunk<R, 3>(a, cfg, grid, block, smem, st);
    case 4: return launch_fb_chunk<R, 4>(a, cfg, grid, block, smem, st);
    case 5: return launch_fb_chunk<R, 5>(a, cfg, grid, block, smem, st);
    case 6: return launch_fb_chunk<R, 6>(a, cfg, grid, block, smem, st);
    case 7: return launch_fb_chunk<R, 7>(a, cfg, grid, block, smem, st);
    default: return launch_fb_chunk<R, 8>(a, cfg, grid, block, smem, st);
  }
}

}  // namespace lhmm

using namespace lhmm;

// Split large-K forward-backward (hmm_large.cuh): concurrent forward /
// backward sweep CTAs, the T-parallel posterior pass, the segment fold.
template <typename R>
static cudaError_t launch_split(const FBArgs& a, int K, int KM, int lps, int64_t B, int threads,
                                void* lbw, void* workspace, int64_t N, int esz, bool fold,
                                cudaStream_t st) {
  SplitWs sw;
  const size_t nk = align256((size_t)N * K * esz);
  sw.qws = (char*)workspace + 2 * nk;
  sw.wws = (char*)workspace + 3 * nk;
  sw.seg_part = (double*)((char*)workspace + 4 * nk);
  sw.sparse_ok = 1;
  if (const char* env = getenv("LOGHMM_FBL_SPARSE")) sw.sparse_ok = atoi(env) != 0;
  sw.sparse_warps = 2;
  if (const char* env = getenv("LOGHMM_FBL_SPARSE_WARPS")) sw.sparse_warps = atoi(env) >= 2 ? 2 : 1;
  const size_t ssm = (size_t)(2 * KM + 128 + kRing * 4 * KM) * sizeof(R);
  const R* lb = (const R*)lbw;
#define LHMM_FBS(KMV)                                                                            \
  do {                                                                                           \
    if (lps == 4) fb_split_sweep_kernel<R, KMV, 4><<<(unsigned)(2 * B), threads, ssm, st>>>(a, K, lb, sw); \
    else if (lps == 2) fb_split_sweep_kernel<R, KMV, 2><<<(unsigned)(2 * B), threads, ssm, st>>>(a, K, lb, sw); \
    else fb_split_sweep_kernel<R, KMV, 1><<<(unsigned)(2 * B), threads, ssm, st>>>(a, K, lb, sw); \
  } while (0)
  if (KM == 16) LHMM_FBS(16);
  else if (KM == 32) LHMM_FBS(32);
  else LHMM_FBS(64);
#undef LHMM_FBS
  const size_t psm = PostGeom<R>::smem();
  if (psm > 48 * 1024 &&
      cudaFuncSetAttribute(fb_post_kernel<R>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psm) != cudaSuccess)
    return cudaErrorInvalidValue;
  const unsigned hz = (K > 32) ? (unsigned)PostGeom<R>::H : 1u;
  fb_post_kernel<R><<<dim3(kPostSegs, (unsigned)B, hz), 32 * kPostWarps, psm, st>>>(a, K, sw);
  // structurally sparse A: the dense kernel above returns at once and one of
  // these takes the pass (each checks the row non-zero count on the device)
  {
    auto ssm = [](int nz) {
      return (size_t)kPostWarps * 64 * sizeof(R) +
             (size_t)(2 * 64 * LOGHMM_NSLOT + 2 * 64 + 64 * nz) * sizeof(double);
    };
    const dim3 pg(kPostSegs, (unsigned)B);
    fb_post_sparse_kernel<R, 5><<<pg, 32 * kPostWarps, ssm(5), st>>>(a, K, sw);
    fb_post_sparse_kernel<R, 9><<<pg, 32 * kPostWarps, ssm(9), st>>>(a, K, sw);
    fb_post_sparse_kernel<R, kPostNZ><<<pg, 32 * kPostWarps, ssm(kPostNZ), st>>>(a, K, sw);
  }
  if (fold) fb_fold_kernel<<<(unsigned)B, 256, 0, st>>>(a, K, sw);
  return cudaGetLastError();
}


extern "C" {

int32_t loghmm_abi_version(void) { return LOGHMM_ABI_VERSION; }

size_t loghmm_model_bytes(void) { return sizeof(loghmm_model_t); }

int64_t loghmm_stats_width(int32_t K, int32_t n_streams) {
  (void)n_streams;
  return (int64_t)K * K + 2 * (int64_t)K + 2 * (int64_t)K * LOGHMM_NSLOT;
}

size_t loghmm_fb_workspace_bytes(int32_t dtype, int32_t K, int64_t B, int64_t N, int64_t max_T) {
  (void)B;
  const int esz = dtype == LOGHMM_F64 ? 8 : 4;
  // alpha~ store + precomputed log b (+ beta~ and w stores and the per-segment
  // statistics rows of the split fp32 path)
  if (K > 8)
    return 4 * align256((size_t)N * K * esz) +
           align256((size_t)B * kPostSegs * (size_t)loghmm_stats_width(K, 2) * sizeof(double));
  FBGeom g = fb_geom(K, esz, 2, max_T);
  return align256((size_t)B * g.Lmax * kWarp * K * esz);
}

size_t loghmm_viterbi_workspace_bytes(int32_t dtype, int32_t K, int64_t B, int64_t N,
                                      int64_t max_T) {
  // large K: byte backpointer table + the precomputed emission log-densities
  if (K > 8) return align256((size_t)N * K) + align256((size_t)N * K * (dtype == LOGHMM_F64 ? 8 : 4));
  VitGeom g = vit_geom(K, max_T);
  if (!g.global) return 0;
  const int64_t G = kWarp / K;
  const int64_t warps = (B + G - 1) / G;
  return align256((size_t)warps * g.plane_words * 4);
}

int32_t loghmm_emission(int32_t dtype, const loghmm_model_t* h_desc, const loghmm_model_t* model,
                        const void* y0, const void* y1, int64_t N, const double* lgamma_lut,
                        int32_t lut_n, void* log_b, void* stream) {
  if (!h_desc || !model || !y0 || !log_b || N < 0) return LOGHMM_EINVAL;
  const int K = h_desc->K;
  if (K < 1 || K > LOGHMM_MAX_STATES) return LOGHMM_EINVAL;
  if (h_desc->n_streams > 1 && !y1) return LOGHMM_EINVAL;
  if (N == 0) return LOGHMM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t blocks = std::min<int64_t>((N + 255) / 256, 148 * 16);
  if (dtype == LOGHMM_F64)
    emission_kernel<double><<<(unsigned)blocks, 256, 0, st>>>(model, (const double*)y0,
                                                              (const double*)y1, N, K, lgamma_lut,
                                                              lut_n, (double*)log_b);
  else
    emission_kernel<float><<<(unsigned)blocks, 256, 0, st>>>(model, (const float*)y0,
                                                             (const float*)y1, N, K, lgamma_lut,
                                                             lut_n, (float*)log_b);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}


int32_t loghmm_forward_backward(int32_t dtype, const loghmm_model_t* h_desc,
                                const loghmm_model_t* model, const void* y0, const void* y1,
                                const int64_t* offsets, int64_t B, int64_t N, int64_t max_T,
                                const double* lgamma_lut, int32_t lut_n, void* log_alpha,
                                void* log_beta, void* gamma, void* xi, double* ll,
                                double* partials, int64_t* flags, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (!h_desc || !model || !y0 || !offsets || !ll || B < 0 || N < 0) return LOGHMM_EINVAL;
  const int K = h_desc->K;
  if (K < 1 || K > LOGHMM_MAX_STATES) return LOGHMM_EINVAL;
  if (h_desc->n_streams > 1 && !y1) return LOGHMM_EINVAL;
  if (B == 0) return LOGHMM_OK;
  const int esz = dtype == LOGHMM_F64 ? 8 : 4;
  cudaStream_t st = (cudaStream_t)stream;
  if (workspace_bytes < loghmm_fb_workspace_bytes(dtype, K, B, N, max_T)) return LOGHMM_EWORKSPACE;
  FBArgs a{};
  a.model = model;
  a.y0 = y0;
  a.y1 = h_desc->n_streams > 1 ? y1 : nullptr;
  a.offsets = offsets;
  a.B = B;
  a.lut = lgamma_lut;
  a.lut_n = lut_n;
  a.n_streams = h_desc->n_streams;
  a.log_alpha = log_alpha;
  a.log_beta = log_beta;
  a.gamma = gamma;
  a.xi = xi;
  a.ll = ll;
  a.partials = partials;
  a.flags = flags;
  a.alpha_ws = workspace;
  a.stats_width = loghmm_stats_width(K, h_desc->n_streams);
  int fams = 0;
  const int cfg = cfg_of(h_desc, &fams);
  a.stream_fams = fams;
  cudaError_t e = cudaSuccess;
  int fbcL = 0;
  size_t fbcW = 0;
  if (use_fbc(K, h_desc->n_streams, B, N, max_T, esz, xi != nullptr, &fbcL, &fbcW)) {
    FBCArgs c{};
    c.model = model;
    c.y0 = a.y0;
    c.y1 = a.y1;
    c.B = B;
    c.T = (int)max_T;
    c.L = fbcL;
    c.lut = lgamma_lut;
    c.lut_n = lut_n;
    c.n_streams = a.n_streams;
    c.stream_fams = fams;
    c.log_alpha = log_alpha;
    c.log_beta = log_beta;
    c.gamma = gamma;
    c.ll = ll;
    c.partials = partials;
    c.flags = flags;
    c.stats_width = a.stats_width;
    c.tm_cols = esz == 4 ? fbc_tm_cols(K, fbcL) : 0;
    // fp32: one warpgroup per CTA (tensor-memory lane quadrants); fp64: as
    // many warps as the shared-memory park allows, up to four
    int wpb = esz == 4 ? kFbcWarpsPerBlock
                       : (int)std::max<size_t>(1, std::min<size_t>(kFbcWarpsPerBlock, (220 * 1024) / fbcW));
    if (const char* env = getenv("LOGHMM_FBC_WPB")) wpb = std::max(1, std::min(4, atoi(env)));
    dim3 grid((unsigned)((B + wpb - 1) / wpb)), block(32 * wpb);
    // (instantiated for fp32 only; use_fbc() keeps fp64 on the chunked scan)
    e = dispatch_fb_chunk<float>(K, c, cfg, grid, block, fbcW * wpb, st);
  } else if (K <= 8) {
    FBGeom g = fb_geom(K, esz, h_desc->n_streams, max_T);
    a.L_align = g.L_align;
    a.Lmax = g.Lmax;
    a.y_pitch = g.y_pitch;
    a.a_pitch = g.a_pitch;
    a.s_pitch = g.s_pitch;
    a.warp_smem_elems = g.warp_elems;
    dim3 grid((unsigned)((B + g.wpb - 1) / g.wpb)), block(32 * g.wpb);
    e = dtype == LOGHMM_F64 ? dispatch_fb_small<double>(K, a, cfg, g.global, grid, block, g.smem, st)
                            : dispatch_fb_small<float>(K, a, cfg, g.global, grid, block, g.smem, st);
  } else {
    // four lanes per state; vector + alpha~_{t-1} (padded to KM) and the
    // reduction scratch in shared memory, A and the xi accumulators in registers
    const int KM = K <= 16 ? 16 : K <= 32 ? 32 : 64;
    // lanes per state: 1 measured fastest at K = 64 (the per-step block
    // reductions cost more with more warps than the split dot products save);
    // 2 and 4 stay selectable for A/B runs
    int lps = 1;
    if (const char* env = getenv("LOGHMM_FBL_LPS")) lps = atoi(env) >= 4 ? 4 : atoi(env) >= 2 ? 2 : 1;
    // split sweeps + T-parallel pass (default); LOGHMM_FBL_SPLIT=0 selects the
    // fused one-CTA-per-sequence kernel
    const char* senv = getenv("LOGHMM_FBL_SPLIT");
    const bool split = !(senv && atoi(senv) == 0);

    const int threads = std::max(32, lps * KM);
    const size_t smem = (size_t)(2 * KM + 128 + kRing * 4 * KM) * esz;
    // log b for the whole batch first (fully parallel), then the sweeps
    void* lbw = (char*)workspace + align256((size_t)N * K * esz);
    const int64_t eblocks = std::min<int64_t>((N + 255) / 256, 148 * 16);
#define LHMM_FBL(RR, KMV)                                                                        \
  do {                                                                                           \
    if (lps == 4) fb_large_kernel<RR, KMV, 4><<<(unsigned)B, threads, smem, st>>>(a, K, (const RR*)lbw); \
    else if (lps == 2) fb_large_kernel<RR, KMV, 2><<<(unsigned)B, threads, smem, st>>>(a, K, (const RR*)lbw); \
    else fb_large_kernel<RR, KMV, 1><<<(unsigned)B, threads, smem, st>>>(a, K, (const RR*)lbw); \
  } while (0)
    // (the per-sequence kernel of the large-K Viterbi: state parameters in
    // registers, coalesced rows; no flag word here, the sweeps report NaN)
    VitArgs ea{};
    ea.model = model;
    ea.y0 = y0;
    ea.y1 = a.y1;
    ea.offsets = offsets;
    ea.B = B;
    ea.lut = lgamma_lut;
    ea.lut_n = lut_n;
    ea.n_streams = a.n_streams;
    ea.flags = nullptr;
    const dim3 egrid((unsigned)((max_T + kEmSeqChunk - 1) / kEmSeqChunk), (unsigned)B);
    (void)eblocks;
    if (dtype == LOGHMM_F64) {
      emission_seq_kernel<double><<<egrid, 256, 0, st>>>(ea, K, (double*)lbw);
      if (split) e = launch_split<double>(a, K, KM, lps, B, threads, lbw, workspace, N, esz, partials != nullptr, st);
      else if (KM == 16) LHMM_FBL(double, 16);
      else if (KM == 32) LHMM_FBL(double, 32);
      else LHMM_FBL(double, 64);
    } else {
      emission_seq_kernel<float><<<egrid, 256, 0, st>>>(ea, K, (float*)lbw);
      if (split) {
        e = launch_split<float>(a, K, KM, lps, B, threads, lbw, workspace, N, esz, partials != nullptr, st);
      } else if (KM == 16) LHMM_FBL(float, 16);
      else if (KM == 32) LHMM_FBL(float, 32);
      else LHMM_FBL(float, 64);
    }
#undef LHMM_FBL
    const cudaError_t e2 = cudaGetLastError();
    if (e == cudaSuccess) e = e2;
  }
  return e == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

int32_t loghmm_viterbi(int32_t dtype, const loghmm_model_t* h_desc, const loghmm_model_t* model,
                       const void* y0, const void* y1, const int64_t* offsets, int64_t B,
                       int64_t N, int64_t max_T, const double* lgamma_lut, int32_t lut_n,
                       int64_t* path, double* log_joint, uint8_t* back, int64_t* flags,
                       void* workspace, size_t workspace_bytes, void* stream) {
  if (!h_desc || !model || !y0 || !offsets || !path || !log_joint || B < 0) return LOGHMM_EINVAL;
  const int K = h_desc->K;
  if (K < 1 || K > LOGHMM_MAX_STATES) return LOGHMM_EINVAL;
  if (h_desc->n_streams > 1 && !y1) return LOGHMM_EINVAL;
  if (B == 0) return LOGHMM_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (workspace_bytes < loghmm_viterbi_workspace_bytes(dtype, K, B, N, max_T))
    return LOGHMM_EWORKSPACE;
  VitArgs a{};
  a.model = model;
  a.y0 = y0;
  a.y1 = h_desc->n_streams > 1 ? y1 : nullptr;
  a.offsets = offsets;
  a.B = B;
  a.lut = lgamma_lut;
  a.lut_n = lut_n;
  a.n_streams = h_desc->n_streams;
  a.path = path;
  a.log_joint = log_joint;
  a.back = back;
  a.flags = flags;
  cudaError_t e;
  int v3_nw = 0;
  size_t v3_smem = 0;
  int fams0 = 0;
  const int cfg0 = cfg_of(h_desc, &fams0);
  if (vit3_ok(K, dtype == LOGHMM_F64 ? 8 : 4, max_T, cfg0, &v3_nw, &v3_smem)) {
    const int cfg = cfg0;
    dim3 grid((unsigned)((B + kV3Seq - 1) / kV3Seq));
    e = dtype == LOGHMM_F64 ? dispatch_vit3<double>(K, a, cfg, v3_nw, grid, v3_smem, st)
                            : dispatch_vit3<float>(K, a, cfg, v3_nw, grid, v3_smem, st);
  } else if (K <= 8) {
    int fams = 0;
    const int cfg = cfg_of(h_desc, &fams);
    const int ns = (cfg == kCfgGammaVM || cfg == kCfgMixed) ? 2 : 1;
    VitGeom g = vit_geom(K, max_T, dtype == LOGHMM_F64 ? 8 : 4, ns);
    a.planes_ws = (uint32_t*)workspace;
    a.plane_words = g.plane_words;
    a.warp_smem_words = g.warp_words;
    const int64_t G = kWarp / K;
    const int64_t warps = (B + G - 1) / G;
    dim3 grid((unsigned)((warps + g.wpb - 1) / g.wpb)), block(32 * g.wpb);
    e = dtype == LOGHMM_F64 ? dispatch_vit_small<double>(K, a, cfg, g.global, grid, block, g.smem, st)
                            : dispatch_vit_small<float>(K, a, cfg, g.global, grid, block, g.smem, st);
  } else {
    const int esz = dtype == LOGHMM_F64 ? 8 : 4;
    const int KM = K <= 16 ? 16 : K <= 32 ? 32 : 64;
    // LOGHMM_VL_SPARSE=0 keeps banded models on the dense recursion (A/B, tests)
    a.sparse_ok = 1;
    if (const char* env = getenv("LOGHMM_VL_SPARSE")) a.sparse_ok = atoi(env) != 0;
    int vlps = 4;  // lanes per destination state (LOGHMM_VL_LPS: 1, 2 or 4)
    if (const char* env = getenv("LOGHMM_VL_LPS")) vlps = atoi(env) >= 4 ? 4 : atoi(env) >= 2 ? 2 : 1;
    const int threads = std::max(32, vlps * KM);
    const size_t smem = std::max<size_t>((size_t)(2 * KM) * esz, (size_t)kBtBlk) + kBtBlk * (size_t)K;
#define LHMM_VL(RR, KMV)                                                                         \
  do {                                                                                           \
    RR* lbw = (RR*)((uint8_t*)workspace + align256((size_t)N * K));                              \
    emission_seq_kernel<RR><<<dim3((unsigned)((max_T + kEmSeqChunk - 1) / kEmSeqChunk), (unsigned)B), 256, 0, st>>>(a, K, lbw); \
    if (vlps == 4) viterbi_large_kernel<RR, KMV, 4><<<(unsigned)B, threads, smem, st>>>(a, K, (uint8_t*)workspace, lbw); \
    else if (vlps == 2) viterbi_large_kernel<RR, KMV, 2><<<(unsigned)B, threads, smem, st>>>(a, K, (uint8_t*)workspace, lbw); \
    else viterbi_large_kernel<RR, KMV, 1><<<(unsigned)B, threads, smem, st>>>(a, K, (uint8_t*)workspace, lbw); \
  } while (0)
    if (dtype == LOGHMM_F64) {
      if (KM == 16) LHMM_VL(double, 16);
      else if (KM == 32) LHMM_VL(double, 32);
      else LHMM_VL(double, 64);
    } else {
      if (KM == 16) LHMM_VL(float, 16);
      else if (KM == 32) LHMM_VL(float, 32);
      else LHMM_VL(float, 64);
    }
#undef LHMM_VL
    e = cudaGetLastError();
  }
  return e == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

int32_t loghmm_reduce_stats(const double* partials, const double* ll, int64_t B, int64_t width,
                            double* totals, void* stream) {
  if (!partials || !ll || !totals || B < 0 || width < 0) return LOGHMM_EINVAL;
  reduce_stats_kernel<<<(unsigned)(width + 1), 256, 0, (cudaStream_t)stream>>>(partials, ll, B,
                                                                                 width, totals);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

// per-block partial sums of the guard / variance passes (after the counter)
static inline size_t kGuardPartBytes(int K) {
  return (size_t)148 * 4 * K * LOGHMM_GUARD_CANDIDATES * sizeof(double);
}

int32_t loghmm_mstep(const loghmm_model_t* model_in, const double* totals, int64_t n_sequences,
                     double collapse_epsilon, double nu_ceiling, double nu_tol, int32_t max_newton,
                     double var_ratio, loghmm_model_t* model_out, int32_t* status,
                     double* guard_state, void* stream) {
  if (!model_in || !totals || !model_out || !status || !guard_state || n_sequences < 1)
    return LOGHMM_EINVAL;
  // the widest statistics vector (K = LOGHMM_MAX_STATES) fits the default
  // 48 KB dynamic shared-memory window
  // + the transition scratch (K*K + K + 1 doubles), sized for K = 64
  const int64_t wmax = (int64_t)loghmm_stats_width(LOGHMM_MAX_STATES, 2) + 1;
  const size_t msm = (size_t)(wmax + LOGHMM_MAX_STATES * LOGHMM_MAX_STATES + LOGHMM_MAX_STATES + 1) *
                     sizeof(double);
  if (cudaFuncSetAttribute(mstep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)msm) !=
      cudaSuccess)
    return LOGHMM_ELAUNCH;
  mstep_kernel<<<1, 256, msm, (cudaStream_t)stream>>>(
      model_in, totals, wmax, n_sequences, collapse_epsilon, nu_ceiling, nu_tol, max_newton,
      model_out, status, guard_state, var_ratio);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

static constexpr int kReduceBlocks = 256;  // upper bound on the reduction grid

// Workspace layouts of the passes that keep an inter-block counter: the
// counter lives in the first 256 bytes (a K- and width-independent place, so
// a workspace reused by calls of different shapes always finds it at zero:
// the buffer is zero-filled once and the last block of every launch resets
// it), the block partials follow at offset kCounterBytes.
static constexpr size_t kCounterBytes = 256;

size_t loghmm_reduce_workspace_bytes(int64_t B, int64_t width) {
  (void)B;
  return kCounterBytes + align256((size_t)kReduceBlocks * (size_t)(width + 1) * sizeof(double));
}

int32_t loghmm_reduce_mstep(const double* partials, const double* ll, int64_t B, int64_t width,
                            double* totals, const loghmm_model_t* model_in, int64_t n_sequences,
                            double collapse_epsilon, double nu_ceiling, double nu_tol,
                            int32_t max_newton, double var_ratio, loghmm_model_t* model_out,
                            int32_t* status, double* guard_state, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!partials || !ll || !totals || B < 1 || width < 0) return LOGHMM_EINVAL;
  const bool do_mstep = model_in != nullptr;
  if (do_mstep && (!model_out || !status || !guard_state || n_sequences < 1)) return LOGHMM_EINVAL;
  if (!workspace || workspace_bytes < loghmm_reduce_workspace_bytes(B, width))
    return LOGHMM_EWORKSPACE;
  unsigned* counter = (unsigned*)workspace;
  double* part = (double*)((char*)workspace + kCounterBytes);
  // totals + one row of column sums per thread group (see the kernel)
  // 1024 threads = G row groups x (width + 1) columns; about sqrt(B) blocks so
  // that both reduction levels keep ~B / (G * sqrt(B)) rows per thread (one
  // batch of independent loads each)
  constexpr int kRedThreads = 1024;
  // (+ the M-step's transition scratch, K*K + K + 1 doubles; K from the
  // statistics width K^2 + 2K + 2K*NSLOT)
  int64_t Ks = 1;
  while (Ks < LOGHMM_MAX_STATES && Ks * Ks + 2 * Ks + 2 * Ks * LOGHMM_NSLOT < width) ++Ks;
  const size_t smem = (size_t)(width + 1 + kRedThreads + Ks * Ks + Ks + 1) * sizeof(double);
  if (smem > 48 * 1024 &&
      cudaFuncSetAttribute(reduce_mstep_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return LOGHMM_ELAUNCH;
  int64_t nbl = 1;
  while (nbl * nbl < B) ++nbl;
  const unsigned nb = (unsigned)std::max<int64_t>(1, std::min<int64_t>(kReduceBlocks, nbl));
  reduce_mstep_kernel<<<nb, kRedThreads, smem, (cudaStream_t)stream>>>(
      partials, ll, B, width, part, counter, totals, model_in, n_sequences, collapse_epsilon,
      nu_ceiling, nu_tol, max_newton, model_out, status, guard_state, var_ratio, do_mstep ? 1 : 0);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

static int32_t variance_launch(int32_t dtype, loghmm_model_t* model_out, const void* y,
                               const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                               const double* guard_state, int32_t* status, double* sums,
                               void* workspace, size_t workspace_bytes, void* stream) {
  if (!model_out || !y || !gamma || !guard_state || K < 1 || K > LOGHMM_MAX_STATES) return LOGHMM_EINVAL;
  if (workspace_bytes < loghmm_guard_workspace_bytes(K, N)) return LOGHMM_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int nblocks = 148 * 2;
  unsigned* counter = (unsigned*)workspace;
  double* part = (double*)((char*)workspace + kCounterBytes);
  if (dtype == LOGHMM_F64)
    variance_pass_kernel<double><<<nblocks, 256, 0, st>>>((const double*)y, (const double*)gamma, N,
                                                          K, stream_index, model_out, guard_state,
                                                          part, counter, status, sums);
  else
    variance_pass_kernel<float><<<nblocks, 256, 0, st>>>((const float*)y, (const float*)gamma, N, K,
                                                         stream_index, model_out, guard_state,
                                                         part, counter, status, sums);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

int32_t loghmm_variance_pass(int32_t dtype, loghmm_model_t* model_out, const void* y,
                             const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                             const double* guard_state, int32_t* status, void* workspace,
                             size_t workspace_bytes, void* stream) {
  if (!status) return LOGHMM_EINVAL;
  return variance_launch(dtype, model_out, y, gamma, N, K, stream_index, guard_state, status, nullptr,
                         workspace, workspace_bytes, stream);
}

int32_t loghmm_variance_partial(int32_t dtype, loghmm_model_t* model_out, const void* y,
                                const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                                const double* guard_state, double* sums, void* workspace,
                                size_t workspace_bytes, void* stream) {
  if (!sums) return LOGHMM_EINVAL;
  return variance_launch(dtype, model_out, y, gamma, N, K, stream_index, guard_state, nullptr, sums,
                         workspace, workspace_bytes, stream);
}

int32_t loghmm_variance_finish(loghmm_model_t* model_out, int32_t K, int32_t stream_index,
                               const double* guard_state, const double* sums, int32_t* status,
                               void* stream) {
  if (!model_out || !guard_state || !sums || !status || K < 1 || K > LOGHMM_MAX_STATES)
    return LOGHMM_EINVAL;
  variance_finish_kernel<<<1, 64, 0, (cudaStream_t)stream>>>(model_out, K, stream_index, guard_state,
                                                             sums, status);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

size_t loghmm_guard_workspace_bytes(int32_t K, int64_t N) {
  (void)N;
  return kCounterBytes + align256(kGuardPartBytes(K));
}

static int32_t guard_launch(int32_t dtype, loghmm_model_t* model_out, const void* y0,
                            const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                            int32_t n_candidates, double* guard_state, int32_t* status,
                            int32_t* need_more, double* sums, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!y0 || !gamma || !guard_state || K < 1 || K > LOGHMM_MAX_STATES || n_candidates < 2 ||
      n_candidates > LOGHMM_GUARD_CANDIDATES)
    return LOGHMM_EINVAL;
  if (workspace_bytes < loghmm_guard_workspace_bytes(K, N)) return LOGHMM_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  const int nblocks = 148 * 4;
  double* part = (double*)((char*)workspace + kCounterBytes);  // (counter area left untouched)
  if (dtype == LOGHMM_F64)
    student_guard_kernel<double><<<nblocks, 256, 0, st>>>((const double*)y0, (const double*)gamma,
                                                          N, K, stream_index, guard_state,
                                                          n_candidates, part);
  else
    student_guard_kernel<float><<<nblocks, 256, 0, st>>>((const float*)y0, (const float*)gamma, N,
                                                         K, stream_index, guard_state,
                                                         n_candidates, part);
  if (sums) {
    guard_fold_kernel<<<1, kGuardSelThreads, 0, st>>>(K, stream_index, guard_state, n_candidates, part, nblocks, sums);
  } else {
    guard_select_kernel<<<1, kGuardSelThreads, 0, st>>>(model_out, K, stream_index, guard_state, n_candidates,
                                          part, nblocks, status, need_more);
  }
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

int32_t loghmm_student_guard(int32_t dtype, loghmm_model_t* model_out, const void* y0,
                             const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                             int32_t n_candidates, double* guard_state, int32_t* status,
                             int32_t* need_more, void* workspace, size_t workspace_bytes,
                             void* stream) {
  if (!model_out || !status || !need_more) return LOGHMM_EINVAL;
  return guard_launch(dtype, model_out, y0, gamma, N, K, stream_index, n_candidates, guard_state,
                      status, need_more, nullptr, workspace, workspace_bytes, stream);
}

int32_t loghmm_ext_fit_pass(int32_t dtype, loghmm_model_t* model_out, const void* y, const void* gamma,
                            int64_t N, int32_t K, int32_t stream_index, double* guard_state,
                            int32_t* status, int32_t* need_more, void* workspace,
                            size_t workspace_bytes, void* stream) {
  if (!model_out || !y || !gamma || !guard_state || !status || !need_more || K < 1 ||
      K > LOGHMM_MAX_STATES)
    return LOGHMM_EINVAL;
  if (!workspace || workspace_bytes < loghmm_guard_workspace_bytes(K, N)) return LOGHMM_EWORKSPACE;
  cudaStream_t st = (cudaStream_t)stream;
  double* part = (double*)((char*)workspace + kCounterBytes);
  if (dtype == LOGHMM_F64)
    ext_pass_kernel<double><<<kExtBlocks, 256, 0, st>>>((const double*)y, (const double*)gamma, N, K,
                                                        stream_index, model_out, guard_state, status, part);
  else
    ext_pass_kernel<float><<<kExtBlocks, 256, 0, st>>>((const float*)y, (const float*)gamma, N, K,
                                                       stream_index, model_out, guard_state, status, part);
  ext_finish_kernel<<<1, 64, 0, st>>>(model_out, K, stream_index, guard_state, status, part, kExtBlocks,
                                      need_more);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

int32_t loghmm_student_guard_partial(int32_t dtype, const void* y0, const void* gamma, int64_t N,
                                     int32_t K, int32_t stream_index, int32_t n_candidates,
                                     const double* guard_state, double* sums, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  if (!sums) return LOGHMM_EINVAL;
  return guard_launch(dtype, nullptr, y0, gamma, N, K, stream_index, n_candidates,
                      const_cast<double*>(guard_state), nullptr, nullptr, sums, workspace,
                      workspace_bytes, stream);
}

int32_t loghmm_student_guard_select(loghmm_model_t* model_out, int32_t K, int32_t stream_index,
                                    int32_t n_candidates, double* guard_state, const double* sums,
                                    int32_t* status, int32_t* need_more, void* stream) {
  if (!model_out || !guard_state || !sums || !status || !need_more || K < 1 ||
      K > LOGHMM_MAX_STATES || n_candidates < 2 || n_candidates > LOGHMM_GUARD_CANDIDATES)
    return LOGHMM_EINVAL;
  guard_select_kernel<<<1, kGuardSelThreads, 0, (cudaStream_t)stream>>>(model_out, K, stream_index, guard_state,
                                                          n_candidates, sums, 1, status, need_more);
  return cudaGetLastError() == cudaSuccess ? LOGHMM_OK : LOGHMM_ELAUNCH;
}

}  // extern "C"
