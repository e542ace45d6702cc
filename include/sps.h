/*
 * sps.h -- C ABI of libsps.so, the B200-native (sm_100a) hot path of adaptive
 * sequential posterior simulation (SPS) for binary and multinomial logit
 * models, Geweke, Durham & Xu, arXiv:1304.4333.
 *
 * Conventions (all entry points)
 *  - Status: every call returns sps_status; 0 = SPS_OK.  On error the context
 *    (when there is one) keeps a message readable with sps_last_error().
 *  - Threading: a context is single-owner and not thread-safe.
 *  - Precision: fp64 end to end ("easy to evaluate to
 *    machine accuracy").  For binary models with 64 <= k <= 128 the K1
 *    contraction runs on the INT8 tensor cores as an exact-to-~1e-16 split
 *    (7 x 7 int8 slices with power-of-two row scales, int32 accumulation,
 *    an exact int64 fold); its results agree with the
 *    FP64 DMMA kernel's to rounding (SPS_NO_OZAKI=1 selects the latter).
 *  - Labels: y[t] in [0, C); label 0 is the paper's reference category C
 *    (theta_C = 0).  theta = [theta_1 .. theta_{C-1}]
 *    stacked in blocks of k, d = k (C-1).
 *  - Particles: J groups of N, particle p = j N + n
 *    (group-major), so groups and shards are contiguous.
 *  - Multi-GPU is SPMD group sharding: rank r of G owns groups
 *    [r J/G, (r+1) J/G) (J divisible by G); every call below except
 *    sps_loglik is collective over the ranks of one context family.
 *  - No CPU fallback: every computation runs in the library's CUDA kernels;
 *    without a CUDA device sps_create fails with SPS_E_CUDA.
 *
 * The readings R1..R18 cited below are listed in DESIGN.md.
 */
#ifndef SPS_H
#define SPS_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  SPS_OK = 0,
  SPS_E_CONFIG = 2,  /* invalid configuration or argument                      */
  SPS_E_DATA = 3,    /* invalid data (label out of range, non-finite X)         */
  SPS_E_NUMERIC = 4, /* weight collapse, Cholesky failure after ridge (R13), non-finite loglik */
  SPS_E_MIXING = 5,  /* M phase exceeded max_m_steps (R13)                      */
  SPS_E_CUDA = 6,    /* CUDA runtime error / no device                          */
  SPS_E_NCCL = 7,    /* NCCL error                                              */
  SPS_E_STATE = 8,   /* call out of order (e.g. sps_mphase before any C phase)  */
  SPS_E_GUARD = 9    /* debug: a device buffer's guard zone was overwritten     */
} sps_status;

enum { SPS_DATA_TEMPERING = 0, SPS_POWER_TEMPERING = 1 };
enum { SPS_RESIDUAL = 0, SPS_SYSTEMATIC = 1, SPS_MULTINOMIAL = 2 };

/* Instantiated model shapes (sps_create fails with SPS_E_CONFIG otherwise): binary (C = 2)
 * k <= 128 on the DMMA log-likelihood kernel; C = 3: k <= 16; C = 4: k <= 16; C = 5..8: k <= 8
 * (DFMA kernels).  d = k (C - 1) <= 512; the register-blocked proposal / accept / warp-Cholesky
 * path for d <= 32, generic kernels and a block Cholesky above. */
typedef struct sps_config {
  int32_t n, k, C;         /* observations T, covariates k, outcomes C (2 <= C <= 8)        */
  int32_t J, N;            /* groups (global) and particles per group (N <= 16384)          */
  uint64_t seed;           /* Philox key (R15)                                              */
  int32_t tempering;       /* SPS_DATA_TEMPERING (paper) or SPS_POWER_TEMPERING (R5) */
  int32_t resampling;      /* SPS_RESIDUAL (default), SPS_SYSTEMATIC, SPS_MULTINOMIAL (R7) */
  double ess_frac;         /* 0.5   ESS/(JN) threshold                        */
  double K_inter;          /* 0.35  RNE target, intermediate cycles          */
  double K_final;          /* 0.9   RNE target, final cycle                   */
  int32_t h_init;          /* 50    step scale h in hundredths, PAPER.md:415 (R6)           */
  int32_t h_step;          /* 1                                        */
  int32_t h_min;           /* 10                                                            */
  int32_t h_max;           /* 100                                                           */
  double accept_target;    /* 0.25                                            */
  int32_t max_m_steps;     /* 1000  per M phase (R13)                                       */
  int32_t max_cycles;      /* capacity of the per-cycle trace                               */
  int32_t n_monitors;      /* rows of `monitors`; 0 -> default (R12): C-1 block means       */
  const double* monitors;  /* host, n_monitors x d row-major; copied by sps_create          */
  int32_t pass;            /* stream pass tag (Alg. 3); 0 for a one-pass run                */
  int32_t rank, nranks;    /* group sharding; nranks = 1 for a single GPU                   */
  const void* nccl_id;     /* host, 128-byte ncclUniqueId; required when nranks > 1 (ignored
                            * at nranks = 1 unless SPS_XCHG_1RANK=1: then the one rank runs the
                            * multi-GPU exchange path over a one-rank communicator -- a test /
                            * measurement hook for the NCCL transport on one GPU)               */
  int32_t device;          /* CUDA device ordinal                                           */
  void* stream;            /* cudaStream_t to enqueue on; NULL -> the library creates one   */
} sps_config;

typedef struct sps_report {
  /* outputs */
  int32_t status;
  int32_t L;               /* number of cycles                                              */
  int32_t total_m_steps;
  int32_t h_final;         /* hundredths                                                    */
  double logml, logml_nse; /* PAPER.md:813-816 (R10)                                        */
  double pairs;            /* particle x observation loglik terms evaluated (all ranks)    */
  /* caller-owned per-cycle arrays, capacity cap_cycles (may be NULL)                       */
  int32_t cap_cycles;
  int32_t* t_cycle;        /* t_l (data tempering)                                          */
  double* phi_cycle;       /* phi_l (power tempering)                                       */
  int32_t* R_cycle;        /* M steps of cycle l                                            */
  double* logml_inc;       /* pooled log-ML increment of cycle l                            */
  double* min_rne;         /* min monitor RNE at the end of cycle l                         */
  int32_t* h_cycle;        /* h after cycle l                                               */
  /* reported functionals g_i(theta) = a_i' theta (input rows; NULL -> theta_c' xbar,
   * c = 1..C-1) and their moments (outputs, capacity n_report)           */
  int32_t n_report;
  const double* report_fns;
  double *mean, *sd, *nse, *rne; /* PAPER.md:160-223 with NSE = [(JN)^-1 vhat]^1/2 (R2)     */
  /* caller-owned, capacity n, may be NULL: log predictive likelihoods log p(y_s | y_{1:s-1}),
   * s = 1..T (data tempering; see sps_predictive)                                          */
  double* logpl;
} sps_report;

typedef struct sps_ctx sps_ctx;

/* Fill *cfg with the paper's constants and single-GPU defaults. */
sps_status sps_config_default(sps_config* cfg);

/* Create a context: copies X (n x k row-major, host), y (n, host, labels in
 * [0,C)), the Gaussian prior mean (d) and covariance (d x d SPD) of the
 * normalized parameter to the device, factors the prior
 * covariance, and draws the initial particles theta_jn ~iid p(theta)
 * (Algorithm 1 step 1; INIT stream R15).  In power mode it
 * also evaluates the full-data log-likelihood of every particle.  The caller
 * may free every input on return.  Errors: SPS_E_CONFIG (shapes, constants,
 * non-SPD prior), SPS_E_DATA (labels, non-finite X), SPS_E_CUDA, SPS_E_NCCL. */
sps_status sps_create(const sps_config* cfg, const double* X, const int32_t* y, const double* prior_mean,
                      const double* prior_cov, sps_ctx** out);

/* L_p = sum_{t0 <= t < t1} log P(Y = y_t | x_t, theta_p)  (PAPER.md:115-125 eq.
 * plogit, PAPER.md:233-242 factorization), p = 0..P-1.  theta_dev: device,
 * P rows of ld >= d doubles; out_dev: device, P doubles.  Both caller-owned,
 * not retained; enqueued on the context stream (not synchronized).  Local
 * (not collective).  Errors: SPS_E_CONFIG (ranges, ld < d), returned at once;
 * a non-finite L_p (non-finite or overflowing theta: the model's terms are
 * finite for finite eta) is detected on the device, located
 * there, and returned by the next sps_sync as SPS_E_NUMERIC whose
 * sps_last_error message names the first such particle p and its first
 * non-finite observation t (the device-side check keeps this call async). */
sps_status sps_loglik(sps_ctx* ctx, const double* theta_dev, int64_t P, int32_t ld, int32_t t0, int32_t t1,
                      double* out_dev);

/* Block the host until all work enqueued on the context stream is done.
 * Errors: SPS_E_NUMERIC for a non-finite sps_loglik result since the last sync
 * (message: "particle p = ..., observation t = ..."), SPS_E_CUDA. */
sps_status sps_sync(sps_ctx* ctx);

/* One C phase followed by the S phase (Algorithm 1 step 2(a)-(b),
 * PAPER.md:281-305).  Adaptive (Algorithm 2 step 1) when
 * t_target < 0 (data) / phi_target < 0 (power); otherwise the cycle ends at the
 * given t_target / phi_target (Algorithm 1 with a fixed schedule).  Outputs
 * (host, may be NULL): the new t_l, phi_l and the pooled log-ML increment.
 * Errors: SPS_E_STATE (already at t = T / phi = 1), SPS_E_NUMERIC. */
sps_status sps_cphase(sps_ctx* ctx, int32_t t_target, double phi_target, int32_t* t_new, double* phi_new,
                      double* logml_inc);

/* M phase (Algorithm 2 step 2): Gaussian random-walk
 * Metropolis steps with Sigma = h V (V pooled sample covariance, R11), h
 * adapted by +-0.01 around the 0.25 acceptance target, repeated until the
 * minimum monitor RNE >= K (0.35, or 0.9 once t = T / phi = 1), or exactly
 * R_fixed steps when R_fixed > 0.  Outputs (host, may be NULL): steps taken,
 * final min RNE, h (hundredths).  Errors: SPS_E_STATE, SPS_E_MIXING, SPS_E_NUMERIC. */
sps_status sps_mphase(sps_ctx* ctx, int32_t R_fixed, int32_t* R, double* min_rne, int32_t* h_out);

/* Full adaptive run, Algorithm 2: cycles of sps_cphase +
 * sps_mphase until the final cycle, then the reported moments.  `rep` inputs:
 * cap_cycles + arrays, n_report + report_fns; outputs as documented above. */
sps_status sps_run(sps_ctx* ctx, sps_report* rep);

/* Accumulated log marginal likelihood and its NSE across groups (R10).  Does not
 * change the sampler state (it pulls device-side increments into a host cache). */
sps_status sps_logml(const sps_ctx* ctx, double* logml, double* nse);

/* Posterior moments of m linear functionals a_i' theta (A: host, m x d) over the
 * current particles: grand mean, sd, NSE, RNE (R2). Collective. */
sps_status sps_moments(sps_ctx* ctx, int32_t m, const double* A, double* mean, double* sd, double* nse,
                       double* rne);

/* Copy this rank's particles to the host: theta (P_local x d), cached
 * log-likelihood L and prior kernel lp (P_local each); any pointer may be NULL. */
sps_status sps_get_particles(sps_ctx* ctx, double* theta_host, double* L_host, double* lp_host);

/* Restart Algorithm 2 on the resident data and prior with a new seed / pass
 * tag: redraws theta_jn ~iid p(theta) from the INIT stream of `seed`
 * and clears the cycle state, log ML and trace.  Lets a
 * caller repeat runs (e.g. independent runs A, B, C)
 * without re-uploading data.  Collective. */
sps_status sps_reset(sps_ctx* ctx, uint64_t seed, int32_t pass);

/* Log predictive likelihoods (R18), a
 * by-product of the data-tempering C phase: out[s - s0] = log p(y_{s+1} | y_{1:s})
 * for 0-based observations s0 <= s < s1, each the log ratio of the pooled weight
 * sums after and before absorbing the observation, over the particles of the
 * cycle that absorbed it.  Sum over a cycle = its log-ML increment; sum over all
 * T = log ML.  out: host, s1 - s0 doubles.  Errors: SPS_E_STATE (power tempering,
 * or s1 > observations absorbed so far), SPS_E_CONFIG. */
sps_status sps_predictive(sps_ctx* ctx, int32_t s0, int32_t s1, double* out);

/* ---- Algorithm 3: two passes --------------------------
 * Pass 1 runs Algorithm 2 and records its design: the cycle break points t_l
 * (data tempering) or phi_l (power tempering), the M steps R_l per cycle
 * (sps_run's report) and the proposal variance Sigma_lr = (h_lr/100) V_lr of
 * every M step.  Pass 2 restarts with an independent
 * seed and pass tag 1 (sps_reset) and reruns Algorithm 1 with that design
 * fixed: no ESS rule, no RNE stopping rule, Sigma_lr taken
 * from the record (h is still adapted and reported, and the ridge retry R13
 * uses V = Sigma_lr / (h/100)). */

/* Record Sigma_lr of every M step run from now on (on != 0) into a device
 * buffer indexed by the global M-step number (0-based, counted over the run
 * since sps_create / sps_reset; the record survives sps_reset and is
 * overwritten from step 0 by the next run).  Errors: SPS_E_CUDA. */
sps_status sps_record_sigma(sps_ctx* ctx, int32_t on);

/* Copy recorded Sigma_lr of global M steps [first, first + count) to `out`
 * (host, count x d x d row-major, caller-owned).  Errors: SPS_E_STATE (not
 * recording or steps not yet run), SPS_E_CONFIG. */
sps_status sps_get_sigma(sps_ctx* ctx, int64_t first, int64_t count, double* out);

/* Fix the design of the next sps_run (Algorithm 3 step 2): L cycles with
 * t_cycle[l] (data) or phi_cycle[l] (power; strictly increasing, ending at T /
 * 1 for a run to the posterior), R_cycle[l] >= 1 M steps, and sigma: the
 * sum_l R_l proposal variances d x d row-major in execution order (host; all
 * arrays copied, caller may free on return).  The design stays set across
 * sps_reset; L = 0 clears it (adaptive runs again).  Errors: SPS_E_CONFIG
 * (missing arrays, non-increasing schedule, L > max_cycles), SPS_E_CUDA. */
sps_status sps_set_design(sps_ctx* ctx, int32_t L, const int32_t* t_cycle, const double* phi_cycle,
                          const int32_t* R_cycle, const double* sigma);

typedef struct sps_counters {
  int64_t launches;     /* kernel launches by the library since the last create/reset */
  int64_t k1_launches;  /* log-likelihood (K1) launches                                 */
  double k1_pairs;      /* particle x observation pairs evaluated by K1 launches         */
  double k1_ms;         /* summed CUDA-event duration of K1 launches (profiling on)      */
  int64_t syncs;        /* host synchronizations                                         */
  /* profiling: per-category event time (ms) and count; categories: 0 K1 loglik, 1 propose,
   * 2 accept+moments, 3 moments reduce, 4 gather, 5 finalize, 6 control copy, 7 C phase,
   * 8 resample, 9 other */
  double cat_ms[16];
  int64_t cat_n[16];
} sps_counters;

/* Profiling: when on, every K1 launch is bracketed by CUDA events on the
 * context stream and synchronized (perturbs timing; for measurement runs). */
sps_status sps_set_profiling(sps_ctx* ctx, int32_t on);
sps_status sps_get_counters(const sps_ctx* ctx, sps_counters* out);

/* Local particle count and first global group of this rank. */
sps_status sps_shard(const sps_ctx* ctx, int64_t* P_local, int32_t* group0, int32_t* J_local);

/* Debug memory check (the pool this was built on runs no compute-sanitizer).  With the
 * environment variable SPS_GUARD=1 at sps_create, every device buffer of the context is
 * allocated between two 256-byte guard zones filled with 0xA5; an out-of-bounds write by any
 * kernel (or copy) lands in a zone.  sps_check_guards synchronizes the context's streams and
 * reads every zone back.  *n_corrupt (may be NULL) = overwritten guard bytes.  Returns SPS_OK,
 * SPS_E_GUARD (the last-error message names the first buffer and the byte offset relative to
 * its start: negative = before it, >= its size = past its end), or SPS_E_CONFIG if the context
 * was created without SPS_GUARD=1.  sps_destroy repeats the check on a guarded context, reports a
 * hit on stderr and, with SPS_GUARD_ABORT=1, aborts the process.  Test hook: SPS_GUARD_POKE=<buffer
 * name, e.g. &c->theta> writes 8 bytes past that buffer at create. */
sps_status sps_check_guards(sps_ctx* ctx, int64_t* n_corrupt);

void sps_destroy(sps_ctx* ctx);
const char* sps_last_error(const sps_ctx* ctx);

/* 128-byte NCCL unique id for rank 0 to broadcast (via torch.distributed). */
sps_status sps_nccl_unique_id(void* id128);

/* 128-byte id of an in-process loopback group: passed as cfg.nccl_id instead of an
 * NCCL id, the ranks are contexts of one process (one host thread per rank, any
 * device, e.g. all on one GPU) and each exchange step is staged through host
 * memory at a host barrier.  Exercises the sharded engine without NCCL; slow. */
sps_status sps_loopback_unique_id(void* id128);

/* Test export (host only, no device): one all-gather of the loopback group `id128` (G ranks, one
 * host thread per rank, each calling with its own rank): `send` (bytes, host) of every rank lands in
 * `recv` (G x bytes, host) in rank order, after all G ranks have arrived -- the exchange primitive the
 * sharded engine uses over the loopback transport.  SPS_E_CONFIG on a bad id / rank / G mismatch. */
sps_status sps_test_loopback_allgather(const void* id128, int32_t rank, int32_t G, const void* send, int64_t bytes,
                                       void* recv);

/* Zellner g-prior (PAPER.md:665-668 eq. g-prior_def, exchangeable, normalized
 * by eq. prior_norm): cov (d x d, host) = blocks
 * (2 if i == j else 1) * g T (X'X)^-1.  Computed on the device.  (R9) */
sps_status sps_g_prior(const double* X, int32_t n, int32_t k, int32_t C, double g, int32_t device,
                       double* cov_out);

/* ---- test exports (device computation, host buffers) -------------------- */
/* Philox4x32-10 of n counters (ctr: n x 4 words, key: 2 words) -> out n x 4. */
sps_status sps_test_philox(int32_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out);
/* count standard normals of stream (seed, id, step, tag, pass), R15. */
sps_status sps_test_normals(uint64_t seed, uint32_t id, uint32_t step, uint32_t tag, uint32_t pass,
                            int32_t count, double* out);
/* portable log / exp / sincos(2 pi u) on n inputs: out is n (log, exp) or 2n (sin, cos). */
sps_status sps_test_portable(int32_t which, int32_t n, const double* x, double* out);
/* Integer resampling core (R7) on one group: q (N), a (N 52-bit uniforms) -> anc (N). */
sps_status sps_test_resample_int(int32_t N, const uint64_t* q, int32_t scheme, const uint64_t* a,
                                 int32_t* anc);
/* Resampling of one group from log weights with the RESAMPLE stream (R7, R15). */
sps_status sps_test_resample_group(int32_t N, const double* lw, int32_t scheme, uint64_t seed, uint32_t group,
                                   uint32_t cycle, uint32_t pass, int32_t* anc);
/* Accept decisions plog(u_p) < delta_p for the ACCEPT stream (R16): flags (P). */
sps_status sps_test_accept(int64_t P, const double* delta, uint64_t seed, uint32_t step, uint32_t pass,
                           uint8_t* flags);

#ifdef __cplusplus
}
#endif
#endif /* SPS_H */
