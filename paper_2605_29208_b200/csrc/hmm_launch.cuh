// hmm_launch.cuh — host-side launch templates, explicitly instantiated per
// (dtype, K) in inst_*.cu so the heavy kernel bodies compile in parallel.
#pragma once

// Translation units that instantiate one kernel family define LHMM_ONLY_FB,
// LHMM_ONLY_VIT or LHMM_ONLY_FBC first, so they depend on (and parse) only
// that family's header; hmm_capi.cu sees every declaration.
#if defined(LHMM_ONLY_FB)
#include "hmm_fb.cuh"
#define LHMM_HAS_FB 1
#elif defined(LHMM_ONLY_VIT)
#include "hmm_viterbi3.cuh"
#define LHMM_HAS_VIT 1
#elif defined(LHMM_ONLY_FBC)
#include "hmm_fbc.cuh"
#define LHMM_HAS_FBC 1
#else
#include "hmm_fb.cuh"
#include "hmm_fbc.cuh"
#include "hmm_viterbi.cuh"
#include "hmm_viterbi3.cuh"
#define LHMM_HAS_FB 1
#define LHMM_HAS_VIT 1
#define LHMM_HAS_FBC 1
#endif

namespace lhmm {

#if defined(LHMM_HAS_FB)
template <typename R, int K, int CFG, bool G>
static cudaError_t launch_fb_one(const FBArgs& a, dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t st) {
  auto fn = fb_small_kernel<R, K, CFG, G>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, block, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename R, int K, bool G>
static cudaError_t launch_fb_cfg(const FBArgs& a, int cfg, dim3 grid, dim3 block, size_t smem,
                                 cudaStream_t st) {
  switch (cfg) {
    case kCfgGauss: return launch_fb_one<R, K, kCfgGauss, G>(a, grid, block, smem, st);
    case kCfgStudent: return launch_fb_one<R, K, kCfgStudent, G>(a, grid, block, smem, st);
    case kCfgGamma: return launch_fb_one<R, K, kCfgGamma, G>(a, grid, block, smem, st);
    case kCfgVonMises: return launch_fb_one<R, K, kCfgVonMises, G>(a, grid, block, smem, st);
    case kCfgPoisson: return launch_fb_one<R, K, kCfgPoisson, G>(a, grid, block, smem, st);
    case kCfgGammaVM: return launch_fb_one<R, K, kCfgGammaVM, G>(a, grid, block, smem, st);
    default: return launch_fb_one<R, K, kCfgMixed, G>(a, grid, block, smem, st);
  }
}

template <typename R, int K>
cudaError_t launch_fb_small(const FBArgs& a, int cfg, bool global, dim3 grid, dim3 block,
                            size_t smem, cudaStream_t st) {
  return global ? launch_fb_cfg<R, K, true>(a, cfg, grid, block, smem, st)
                : launch_fb_cfg<R, K, false>(a, cfg, grid, block, smem, st);
}
#endif  // LHMM_HAS_FB

#if defined(LHMM_HAS_VIT)
template <typename R, int K, int CFG, bool G>
static cudaError_t launch_vit_one(const VitArgs& a, dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t st) {
  auto fn = viterbi_small_kernel<R, K, CFG, G>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  fn<<<grid, block, smem, st>>>(a);
  return cudaGetLastError();
}

template <typename R, int K, bool G>
static cudaError_t launch_vit_cfg(const VitArgs& a, int cfg, dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t st) {
  switch (cfg) {
    case kCfgGauss: return launch_vit_one<R, K, kCfgGauss, G>(a, grid, block, smem, st);
    case kCfgStudent: return launch_vit_one<R, K, kCfgStudent, G>(a, grid, block, smem, st);
    case kCfgGamma: return launch_vit_one<R, K, kCfgGamma, G>(a, grid, block, smem, st);
    case kCfgVonMises: return launch_vit_one<R, K, kCfgVonMises, G>(a, grid, block, smem, st);
    case kCfgPoisson: return launch_vit_one<R, K, kCfgPoisson, G>(a, grid, block, smem, st);
    case kCfgGammaVM: return launch_vit_one<R, K, kCfgGammaVM, G>(a, grid, block, smem, st);
    default: return launch_vit_one<R, K, kCfgMixed, G>(a, grid, block, smem, st);
  }
}

template <typename R, int K>
cudaError_t launch_vit_small(const VitArgs& a, int cfg, bool global, dim3 grid, dim3 block,
                             size_t smem, cudaStream_t st) {
  return global ? launch_vit_cfg<R, K, true>(a, cfg, grid, block, smem, st)
                : launch_vit_cfg<R, K, false>(a, cfg, grid, block, smem, st);
}

template <typename R, int K, int CFG, int NW>
static cudaError_t launch_vit3_one(const VitArgs& a, dim3 grid, size_t smem, cudaStream_t st) {
  if constexpr (K >= 2 && K <= 4) {
    auto fn = viterbi_chain_kernel<R, K, CFG, NW>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, dim3(32 * NW), smem, st>>>(a);
    return cudaGetLastError();
  } else {
    return cudaErrorInvalidValue;
  }
}

template <typename R, int K, int CFG>
static cudaError_t launch_vit3_nw(const VitArgs& a, int nw, dim3 grid, size_t smem, cudaStream_t st) {
  if (nw >= 16) return launch_vit3_one<R, K, CFG, 16>(a, grid, smem, st);
  return launch_vit3_one<R, K, CFG, 8>(a, grid, smem, st);
}

// chain-warp Viterbi (hmm_viterbi3.cuh): nw warps per CTA (8 or 16)
template <typename R, int K>
cudaError_t launch_vit3(const VitArgs& a, int cfg, int nw, dim3 grid, size_t smem, cudaStream_t st) {
  switch (cfg) {
    case kCfgGauss: return launch_vit3_nw<R, K, kCfgGauss>(a, nw, grid, smem, st);
    case kCfgStudent: return launch_vit3_nw<R, K, kCfgStudent>(a, nw, grid, smem, st);
    case kCfgGamma: return launch_vit3_nw<R, K, kCfgGamma>(a, nw, grid, smem, st);
    case kCfgVonMises: return launch_vit3_nw<R, K, kCfgVonMises>(a, nw, grid, smem, st);
    case kCfgPoisson: return launch_vit3_nw<R, K, kCfgPoisson>(a, nw, grid, smem, st);
    case kCfgGammaVM: return launch_vit3_nw<R, K, kCfgGammaVM>(a, nw, grid, smem, st);
    default: return launch_vit3_nw<R, K, kCfgMixed>(a, nw, grid, smem, st);
  }
}
#endif  // LHMM_HAS_VIT

#if defined(LHMM_HAS_FBC)
template <typename R, int K, int CFG>
static cudaError_t launch_fbc_one(const FBCArgs& a, dim3 grid, dim3 block, size_t smem,
                                  cudaStream_t st) {
  if constexpr (K >= 2) {
    auto fn = fb_chunk_kernel<R, K, CFG>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    fn<<<grid, block, smem, st>>>(a);
    return cudaGetLastError();
  } else {
    return cudaErrorInvalidValue;
  }
}

template <typename R, int K>
cudaError_t launch_fb_chunk(const FBCArgs& a, int cfg, dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st) {
  switch (cfg) {
    case kCfgGauss: return launch_fbc_one<R, K, kCfgGauss>(a, grid, block, smem, st);
    case kCfgStudent: return launch_fbc_one<R, K, kCfgStudent>(a, grid, block, smem, st);
    case kCfgGamma: return launch_fbc_one<R, K, kCfgGamma>(a, grid, block, smem, st);
    case kCfgVonMises: return launch_fbc_one<R, K, kCfgVonMises>(a, grid, block, smem, st);
    case kCfgPoisson: return launch_fbc_one<R, K, kCfgPoisson>(a, grid, block, smem, st);
    case kCfgGammaVM: return launch_fbc_one<R, K, kCfgGammaVM>(a, grid, block, smem, st);
    default: return launch_fbc_one<R, K, kCfgMixed>(a, grid, block, smem, st);
  }
}

// shared-memory elements of one warp for chunk length L
template <typename R, int K>
int fb_chunk_warp_elems(int L) { return FBCGeom<R, K>::warp_elems(L); }
#endif  // LHMM_HAS_FBC

#define LHMM_INST_FB(R, K)                                                                   \
  template cudaError_t launch_fb_small<R, K>(const FBArgs&, int, bool, dim3, dim3, size_t,   \
                                             cudaStream_t);
#define LHMM_INST_VIT(R, K)                                                                  \
  template cudaError_t launch_vit_small<R, K>(const VitArgs&, int, bool, dim3, dim3, size_t, \
                                              cudaStream_t);                                 \
  template cudaError_t launch_vit3<R, K>(const VitArgs&, int, int, dim3, size_t, cudaStream_t);
#define LHMM_INST_FBC(R, K)                                                                  \
  template cudaError_t launch_fb_chunk<R, K>(const FBCArgs&, int, dim3, dim3, size_t, cudaStream_t); \
  template int fb_chunk_warp_elems<R, K>(int);

#define LHMM_EXTERN_INST(R, K)                                                                      \
  extern template cudaError_t launch_fb_small<R, K>(const FBArgs&, int, bool, dim3, dim3, size_t,   \
                                                    cudaStream_t);                                  \
  extern template cudaError_t launch_vit_small<R, K>(const VitArgs&, int, bool, dim3, dim3, size_t, \
                                                     cudaStream_t);                                 \
  extern template cudaError_t launch_vit3<R, K>(const VitArgs&, int, int, dim3, size_t, cudaStream_t); \
  extern template cudaError_t launch_fb_chunk<R, K>(const FBCArgs&, int, dim3, dim3, size_t, cudaStream_t); \
  extern template int fb_chunk_warp_elems<R, K>(int);

}  // namespace lhmm
