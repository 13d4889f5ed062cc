/*
 * loghmm_b200.h — C ABI of the B200-native log-space HMM core.
 *
 * This is the drop-in boundary for the data-parallel hot path of the
 * reference `loghmm` package (/root/reference/pkg/src/loghmm).  The
 * reference has no native plugin ABI; its hot path sits
 * behind Python functions.  Each entry point below replaces one of them for a
 * whole batch of sequences at once:
 *
 *   loghmm_emission        <- inference.py:122 emission_log_matrix
 *                             (+ distributions.py:199/256/359/378/526 _log_density)
 *   loghmm_forward_backward<- inference.py:129 _forward_from_log_b,
 *                             inference.py:140 _backward_from_log_b,
 *                             inference.py:161 posteriors (gamma, optional xi),
 *                             training.py:187-210 (E-step accumulation: dead rows,
 *                             LL, first gammas, gamma totals, xi totals) and the
 *                             per-state weighted sums consumed by the fits
 *                             (distributions.py:616-620, 764-786, 874-916, 1031-1087)
 *   loghmm_viterbi         <- inference.py:191 viterbi (backpointers + backtrace)
 *   loghmm_reduce_stats    <- the running sums of training.py:180-210
 *   loghmm_mstep           <- training.py:105 m_step_transitions,
 *                             training.py:130 m_step_emissions, distributions.py:1094 refit
 *   loghmm_student_guard   <- distributions.py:1080-1086 (ECME likelihood guard pass)
 *
 * Conventions:
 *  - every pointer argument is a DEVICE pointer unless its name starts with h_;
 *  - the library allocates nothing and keeps no global mutable state; callers
 *    pass a workspace sized by loghmm_workspace_bytes();
 *  - every call is enqueued on `stream` (a cudaStream_t, NULL = legacy default)
 *    and returns immediately; the return code reports argument / launch errors
 *    only.  Data errors (dead observations, infeasible sequences, NaN input,
 *    fit failures) are written to caller-provided flag buffers so the host can
 *    raise the reference's exceptions with the reference's messages;
 *  - sequences are packed back to back: y[offsets[b] .. offsets[b+1]) is
 *    sequence b (the layout of training.py:172 `np.concatenate(seqs)`); a
 *    [B,T] batch is offsets[b] = b*T.  Per-step outputs are [N, K] row-major
 *    with the same packing (the layout of training.py:221).
 *  - dtype selects the arithmetic type of the recursions and of the per-step
 *    outputs (y, log_alpha, log_beta, gamma, log_b); statistics, likelihoods
 *    and model parameters are always fp64.
 */
#ifndef LOGHMM_B200_H
#define LOGHMM_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LOGHMM_ABI_VERSION 1
#define LOGHMM_MAX_STATES 64
#define LOGHMM_MAX_STREAMS 2
#define LOGHMM_NSLOT 6 /* per-state, per-stream sufficient-statistic slots */

enum loghmm_dtype { LOGHMM_F32 = 0, LOGHMM_F64 = 1 };

/* Emission families on the hot path (distributions.py FAMILIES, :540-559). */
enum loghmm_family {
  LOGHMM_FAM_NONE = 0,
  LOGHMM_FAM_GAUSSIAN = 1,  /* p = {mu, sigma}            distributions.py:187-204 */
  LOGHMM_FAM_STUDENT_T = 2, /* p = {mu, sigma, nu}        distributions.py:512-537 */
  LOGHMM_FAM_GAMMA = 3,     /* p = {shape, rate}          distributions.py:366-389 */
  LOGHMM_FAM_VON_MISES = 4, /* p = {mu, kappa}            distributions.py:343-363 */
  LOGHMM_FAM_POISSON = 5,   /* p = {lambda}               distributions.py:246-263 */
  /* off the benchmarked configurations (runtime-family kernel paths; fits by
   * loghmm_ext_fit_pass); record layouts in distributions.py record() */
  LOGHMM_FAM_LOGNORMAL = 6,   /* p = {mu, sigma}     c = {log sigma, 0.5 LOG_2PI}      :208-227 */
  LOGHMM_FAM_EXPONENTIAL = 7, /* p = {lambda}        c = {log lambda}                  :230-244 */
  LOGHMM_FAM_RAYLEIGH = 8,    /* p = {sigma}         c = {log s2, 2 s2}                :267-283 */
  LOGHMM_FAM_UNIFORM = 9,     /* p = {a, b}          c = {-log(b - a)}                 :286-305 */
  LOGHMM_FAM_CATEGORICAL = 10,/* p, c = log p_0..7, reserved = category count (<= 8)   :308-341 */
  LOGHMM_FAM_BETA = 11,       /* p = {alpha, beta}   c = {log B(alpha, beta)}          :393-413 */
  LOGHMM_FAM_WEIBULL = 12,    /* p = {k, lambda}     c = {log k - log lambda}          :416-439 */
  LOGHMM_FAM_NEGBINOM = 13,   /* p = {r, p}          c = {lgamma r, r log p, log1p(-p)} :442-469 */
  LOGHMM_FAM_CHISQ = 14,      /* p = {nu}            c = {h log 2, lgamma h, h - 1}    :472-489 */
  LOGHMM_FAM_PARETO = 15      /* p = {xm, alpha}     c = {log a + a log xm, a + 1}     :492-510 */
};

/* Return codes. */
enum loghmm_status {
  LOGHMM_OK = 0,
  LOGHMM_EINVAL = 1,       /* bad argument */
  LOGHMM_EUNSUPPORTED = 2, /* shape / family combination not built */
  LOGHMM_ELAUNCH = 3,      /* CUDA launch error (cudaGetLastError) */
  LOGHMM_EWORKSPACE = 4    /* workspace too small */
};

/* Per-state, per-stream emission record.  c[] holds constants the host
 * computes with the reference's own scalar math (math.log, math.lgamma,
 * special.log_bessel_i0) so that IEEE-basic-op families reproduce the
 * reference bit for bit:
 *   gaussian : c0 = (-0.5*LOG_2PI) - log(sigma)                  (:199-201)
 *   student_t: c0 = lg((nu+1)/2) - lg(nu/2) - 0.5*log(nu*pi) - log(sigma),
 *              c1 = (nu+1)/2                                       (:526-534)
 *   gamma    : c0 = shape*log(rate) - lgamma(shape), c1 = shape-1 (:378-386)
 *   von_mises: c0 = LOG_2PI, c1 = log_bessel_i0(kappa)            (:359-360)
 *   poisson  : c0 = log(lambda)                                    (:256-260)  */
typedef struct loghmm_emission {
  int32_t family;
  int32_t reserved;
  double p[4];
  double c[4];
} loghmm_emission_t;

/* Model block (fp64 master copy).  log_pi / log_A are np.log of pi / A as the
 * reference computes them (inference.py:82-88); the host fills them so the
 * Viterbi recursion sees bit-identical inputs.  loghmm_mstep writes a new
 * block in place of its `d_model_out` argument. */
typedef struct loghmm_model {
  int32_t K;
  int32_t n_streams; /* 1, or 2 for joint (factorised) emissions */
  int32_t reserved[2];
  loghmm_emission_t em[LOGHMM_MAX_STREAMS][LOGHMM_MAX_STATES];
  double pi[LOGHMM_MAX_STATES];
  double A[LOGHMM_MAX_STATES * LOGHMM_MAX_STATES];
  double log_pi[LOGHMM_MAX_STATES];
  double log_A[LOGHMM_MAX_STATES * LOGHMM_MAX_STATES];
} loghmm_model_t;

/* Layout of the per-sequence statistics row written by
 * loghmm_forward_backward (all fp64), for K states and S streams:
 *   [0, K*K)          xi totals  sum_{t<T-1} xi_t(i,j)        (training.py:204-210)
 *   [K*K, K*K+K)      gamma totals over t < T-1               (training.py:203)
 *   [K*K+K, K*K+2K)   gamma at t = 0                          (training.py:201)
 *   then for s in streams, for j in states: LOGHMM_NSLOT family slots
 *                     (gamma-weighted sums over ALL t, training.py:221-222)
 * loghmm_stats_width() returns the row width. */
int64_t loghmm_stats_width(int32_t K, int32_t n_streams);

/* Per-sequence flag word (int64 [B, 2]):
 *   flags[2b+0] = first dead observation index of sequence b, or -1
 *                 (training.py:189-194; inference.py:165 for LL = -inf)
 *   flags[2b+1] = bit 0: NaN observation seen (inference.py:117-118)
 *                 bit 1: a log-gamma lookup fell outside the host table
 *                        (Poisson value not bit-exact to math.lgamma)
 *                 bit 2: (K > 8) a posterior step's alpha~ . beta~ or alpha~^T A w underflowed
 *                        the compute precision although the sequence is possible: gamma / xi
 *                        of that step are not representable (fp32 range; use fp64)     */

int32_t loghmm_abi_version(void);
size_t loghmm_model_bytes(void); /* sizeof(loghmm_model_t), for binding checks */

/* Workspace bytes needed by loghmm_forward_backward / loghmm_viterbi for a
 * batch of B sequences, N total observations, longest sequence max_T. */
size_t loghmm_fb_workspace_bytes(int32_t dtype, int32_t K, int64_t B, int64_t N, int64_t max_T);
size_t loghmm_viterbi_workspace_bytes(int32_t dtype, int32_t K, int64_t B, int64_t N, int64_t max_T);

/* Every compute call takes the model twice: `h_desc` is a HOST copy read only
 * for its structure (K, n_streams, em[s][j].family) to pick the kernel;
 * `model` is the DEVICE block whose parameters are used (it may have been
 * written by loghmm_mstep without a host round trip).  A and log_A are packed
 * row-major K x K (the first K*K entries). */

/* emission_log_matrix for the whole batch: log_b[N, K] in dtype, exact
 * reference operation order (no FMA contraction). */
int32_t loghmm_emission(int32_t dtype, const loghmm_model_t* h_desc, const loghmm_model_t* model,
                        const void* y0, const void* y1, int64_t N, const double* lgamma_lut,
                        int32_t lut_n, void* log_b, void* stream);

/* Batched forward-backward + E-step accumulation.  Any of log_alpha,
 * log_beta, gamma, xi, partials, flags may be NULL.  xi is [(N - B), K, K]:
 * the pairwise posteriors of sequence b start at row offsets[b] - b
 * (inference.py:170-181).  ll[B] is always written. */
int32_t loghmm_forward_backward(int32_t dtype, const loghmm_model_t* h_desc,
                                const loghmm_model_t* model, const void* y0, const void* y1,
                                const int64_t* offsets, int64_t B, int64_t N, int64_t max_T,
                                const double* lgamma_lut, int32_t lut_n, void* log_alpha,
                                void* log_beta, void* gamma, void* xi, double* ll,
                                double* partials, int64_t* flags, void* workspace,
                                size_t workspace_bytes, void* stream);

/* Batched Viterbi with on-device backtrace.  path[N] int64, log_joint[B];
 * back[N, K] uint8 (optional, NULL to skip) receives the backpointer table
 * (row t=0 is zero, as inference.py:197 leaves it). */
int32_t loghmm_viterbi(int32_t dtype, const loghmm_model_t* h_desc, const loghmm_model_t* model,
                       const void* y0, const void* y1, const int64_t* offsets, int64_t B,
                       int64_t N, int64_t max_T, const double* lgamma_lut, int32_t lut_n,
                       int64_t* path, double* log_joint, uint8_t* back, int64_t* flags,
                       void* workspace, size_t workspace_bytes, void* stream);

/* Deterministic fixed-order reduction of partials[B, width] -> totals[width]
 * and sum_b ll[b] -> totals[width] (one extra slot at the end). */
int32_t loghmm_reduce_stats(const double* partials, const double* ll, int64_t B, int64_t width,
                            double* totals, void* stream);

/* M-step on the reduced totals: emission refits, collapse guard,
 * m_step_transitions; writes the next model block to model_out and per-state
 * status words to status[n_streams*K] (index s*K + j).
 * n_sequences is B (pi is the mean of first gammas, training.py:117).
 * guard_state: n_streams*K*16 doubles of scratch (Student-t guard, variance pass). */
enum loghmm_mstep_status {
  LOGHMM_MS_UPDATED = 0,
  LOGHMM_MS_COLLAPSED = 1,           /* total weight < epsilon: kept  */
  LOGHMM_MS_ERR_NO_MASS = 16,        /* "fit requires positive total weight" */
  LOGHMM_MS_ERR_SUPPORT = 17,        /* family support violation among w>0 */
  LOGHMM_MS_ERR_GAMMA_VAR = 18,      /* "gamma fit is degenerate: weighted variance is zero" */
  LOGHMM_MS_ERR_GAMMA_GAP = 19,      /* "gamma fit is degenerate: zero log-moment gap" */
  LOGHMM_MS_ERR_NONFINITE = 20,      /* von_mises non-finite angles */
  LOGHMM_MS_ERR_DEGENERATE = 21,     /* exponential / weibull / negative_binomial / pareto degenerate fit */
  LOGHMM_MS_ERR_CAT_CODE = 22,       /* "categorical fit saw code >= m" */
  LOGHMM_MS_WARN_NEWTON = 1 << 8,    /* FitWarning: Newton did not converge */
  LOGHMM_MS_WARN_CEILING = 1 << 9,   /* FitWarning: ceiling clamp */
  LOGHMM_MS_WARN_BOUNDARY = 1 << 10, /* FitWarning: von Mises resultant at boundary / NegBin underdispersed */
  LOGHMM_MS_WARN_ITERCAP = 1 << 11,  /* FitWarning: beta fit hit the iteration cap */
  LOGHMM_MS_STUDENT_GUARD = 1 << 12, /* Student-t state awaiting the LL guard */
  LOGHMM_MS_EXT_FIT = 1 << 13        /* state of families 6..15 awaiting loghmm_ext_fit_pass */
};
int32_t loghmm_mstep(const loghmm_model_t* model_in, const double* totals, int64_t n_sequences,
                     double collapse_epsilon, double nu_ceiling, double nu_tol, int32_t max_newton,
                     double var_ratio, loghmm_model_t* model_out, int32_t* status,
                     double* guard_state, void* stream);

/* Fused single-rank reduction + M-step: the fixed-order block reduction of
 * partials[B, width] / ll[B] into totals[width + 1] followed, in the same
 * launch, by the M-step of loghmm_mstep (model_in == NULL: reduction only).
 * Replaces the loghmm_reduce_stats -> loghmm_mstep pair when no cross-rank
 * all-reduce sits between them.  The workspace (loghmm_reduce_workspace_bytes)
 * must be zero-filled before its first use; the kernel leaves it reusable. */
size_t loghmm_reduce_workspace_bytes(int64_t B, int64_t width);
int32_t loghmm_reduce_mstep(const double* partials, const double* ll, int64_t B, int64_t width,
                            double* totals, const loghmm_model_t* model_in, int64_t n_sequences,
                            double collapse_epsilon, double nu_ceiling, double nu_tol,
                            int32_t max_newton, double var_ratio, loghmm_model_t* model_out,
                            int32_t* status, double* guard_state, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Exact second pass for the variance-type statistics (distributions.py:616-620
 * two-pass variance, :1051 ECME scale).  The E-step accumulates sums shifted
 * about the current parameters; when the M-step finds the new mean moved by
 * more than sqrt(var_ratio) standard deviations from that shift (so the
 * one-pass difference would lose precision) it flags the state and this call
 * recomputes sum_w (y - mean)^2 from y and gamma and finishes the fit.  Cheap
 * no-op when nothing is flagged.  Call after loghmm_mstep, before
 * loghmm_student_guard.  One launch: the last block to finish reduces the
 * block partials and finishes the flagged states; the workspace
 * (loghmm_guard_workspace_bytes) must be zero-filled before its first use. */
int32_t loghmm_variance_pass(int32_t dtype, loghmm_model_t* model_out, const void* y,
                             const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                             const double* guard_state, int32_t* status, void* workspace,
                             size_t workspace_bytes, void* stream);

/* Student-t ECME likelihood guard (distributions.py:1080-1086): one data pass
 * over y and gamma evaluates sum_w log1p(z^2/nu) at the base nu0 and at
 * n_candidates-1 halving candidates per pending Student-t state, then picks
 * the first candidate that passes.  *need_more (device int) becomes nonzero if
 * a state exhausted its candidates without passing; calling again continues
 * the halving sequence (at most 60 candidates, as the reference). */
/* Multi-rank split of loghmm_variance_pass (sequences sharded across ranks,
 * SURVEY.md §8e): the data pass leaves this rank's per-state second-pass sums
 * in sums[K] (fp64; only flagged states are meaningful) instead of finishing
 * the fit; the caller all-reduces them and calls loghmm_variance_finish. */
int32_t loghmm_variance_partial(int32_t dtype, loghmm_model_t* model_out, const void* y,
                                const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                                const double* guard_state, double* sums, void* workspace,
                                size_t workspace_bytes, void* stream);
int32_t loghmm_variance_finish(loghmm_model_t* model_out, int32_t K, int32_t stream_index,
                               const double* guard_state, const double* sums, int32_t* status,
                               void* stream);

#define LOGHMM_GUARD_CANDIDATES 8
size_t loghmm_guard_workspace_bytes(int32_t K, int64_t N);
int32_t loghmm_student_guard(int32_t dtype, loghmm_model_t* model_out, const void* y0,
                             const void* gamma, int64_t N, int32_t K, int32_t stream_index,
                             int32_t n_candidates, double* guard_state, int32_t* status,
                             int32_t* need_more, void* workspace, size_t workspace_bytes,
                             void* stream);

/* Weighted-sample M-step fits of the families LOGHMM_FAM_LOGNORMAL ..
 * LOGHMM_FAM_PARETO (distributions.py:639-723 closed forms, :789-871 Beta and
 * Weibull, :919-973 NegativeBinomial and ChiSquared) for the states
 * loghmm_mstep left pending (status bit LOGHMM_MS_EXT_FIT).  One call = one
 * data pass over y and gamma[:, j] of every pending state of the stream plus
 * a per-state finish step that advances its program (moments -> centred
 * moments -> Newton iterations); *need_more (device int, zeroed by the
 * caller) becomes nonzero while some state needs another pass.  Fits end by
 * writing the parameters and density constants into model_out; failures set
 * the LOGHMM_MS_ERR_* status codes, FitWarnings the LOGHMM_MS_WARN_* bits.
 * At most LOGHMM_EXT_MAX_PASSES calls are needed.  Workspace:
 * loghmm_guard_workspace_bytes. */
#define LOGHMM_EXT_MAX_PASSES 64
int32_t loghmm_ext_fit_pass(int32_t dtype, loghmm_model_t* model_out, const void* y, const void* gamma,
                            int64_t N, int32_t K, int32_t stream_index, double* guard_state,
                            int32_t* status, int32_t* need_more, void* workspace,
                            size_t workspace_bytes, void* stream);

/* Multi-rank split of loghmm_student_guard: the data pass folds this rank's
 * sums of w*log1p(z^2/nu) into sums[K * LOGHMM_GUARD_CANDIDATES] (index
 * j * LOGHMM_GUARD_CANDIDATES + k, k = 0 the base nu0); after the cross-rank
 * all-reduce loghmm_student_guard_select applies the reference's acceptance
 * rule (distributions.py:1080-1086) to the global sums. */
int32_t loghmm_student_guard_partial(int32_t dtype, const void* y0, const void* gamma, int64_t N,
                                     int32_t K, int32_t stream_index, int32_t n_candidates,
                                     const double* guard_state, double* sums, void* workspace,
                                     size_t workspace_bytes, void* stream);
int32_t loghmm_student_guard_select(loghmm_model_t* model_out, int32_t K, int32_t stream_index,
                                    int32_t n_candidates, double* guard_state, const double* sums,
                                    int32_t* status, int32_t* need_more, void* stream);

/* default_initial_model (training.py:239-282) on the device: for the pooled
 * observations SORTED ascending (fp64, N values) and the np.array_split into
 * K bins, one row of LOGHMM_BIN_SLOTS doubles per bin (two-pass moments about
 * the bin mean, as distributions.py _weighted_mean_var):
 *   [0] n  [1] mean  [2] var  [3] mean log y (y>0)  [4] var log y  [5] sum sin y
 *   [6] sum cos y  [7] sum y^2  [8] min  [9] max  [10] #(y<=0)  [11] #(y<0)
 *   [12] #(y outside (0,1))  [13] #(y<0 or non-integral)  [14..21] #(y == c), c < 8 */
#define LOGHMM_BIN_SLOTS 22
int32_t loghmm_bin_moments(const double* pooled_sorted, int64_t N, int32_t K, double* out,
                           void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LOGHMM_B200_H */
