/*
 * oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct CPU oracle for adaptive sequential posterior
 * simulation (SPS) of binary / multinomial logit models, written from
 * Geweke, Durham & Xu, arXiv:1304.4333.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.  The
 * product library (libsps.so) never links, includes or calls anything here,
 * and this file shares no code with it.
 *
 * Every function cites the passage it follows as PAPER.md:<line> (section /
 * equation / algorithm).  Where the paper is silent the reading taken is the
 * one listed in DESIGN.md "Readings of the paper" (R1..R17).
 *
 * Parity pins: see tests/test_oracle_*.py.  Functions without a pin say
 * "parity unpinned" below (none at present).
 */
#ifndef SPS_ORACLE_H
#define SPS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_OK = 0, OR_E_CONFIG = 2, OR_E_DATA = 3, OR_E_NUMERIC = 4, OR_E_MIXING = 5 };
enum { OR_TAG_INIT = 1, OR_TAG_PROPOSAL = 2, OR_TAG_ACCEPT = 3, OR_TAG_RESAMPLE = 4 };
enum { OR_RESIDUAL = 0, OR_SYSTEMATIC = 1, OR_MULTINOMIAL = 2 };
enum { OR_DATA_TEMPERING = 0, OR_POWER_TEMPERING = 1 };

typedef struct {
  int32_t n, k, C, J, N;
  uint64_t seed;
  int32_t tempering;      /* OR_DATA_TEMPERING (paper) or OR_POWER_TEMPERING */
  int32_t resampling;     /* OR_RESIDUAL (default), OR_SYSTEMATIC, OR_MULTINOMIAL */
  double ess_frac;        /* 0.5 */
  double K_inter;         /* 0.35 PAPER.md:421 */
  double K_final;         /* 0.9 */
  int32_t h_init;         /* 50 hundredths = 0.5 */
  int32_t h_step;         /* 1 hundredth = 0.01 */
  int32_t h_min;          /* 10 = 0.1 */
  int32_t h_max;          /* 100 = 1.0 */
  double accept_target;   /* 0.25 */
  int32_t max_m_steps;    /* per M phase safety cap (R13) */
  int32_t max_cycles;     /* capacity of the per-cycle trace arrays */
  int32_t n_monitors;     /* rows of the monitor matrix (test functions g*) */
  int32_t n_report;       /* rows of the reported-functional matrix */
  int32_t pass;           /* stream pass tag (Alg. 3); 0 for a one-pass run */
  int32_t n_threads;      /* OpenMP threads over particles (0 = runtime default) */
} or_config;

typedef struct {
  int32_t status;
  int32_t L;              /* number of cycles */
  int32_t total_m_steps;
  int32_t h_final;        /* hundredths */
  double logml;
  double logml_nse;
  double pairs;           /* particle x observation log-likelihood terms evaluated */
  /* caller-owned arrays, capacity cfg.max_cycles */
  int32_t* t_cycle;       /* t_l (data tempering) */
  double* phi_cycle;      /* phi_l (power tempering) */
  int32_t* R_cycle;       /* M steps in cycle l */
  double* logml_inc;      /* pooled log-ML increment of cycle l */
  double* min_rne;        /* min monitor RNE at the end of cycle l's M phase */
  int32_t* h_cycle;       /* h (hundredths) after cycle l's M phase */
  /* caller-owned arrays, capacity cfg.n_report */
  double* mean;
  double* sd;
  double* nse;
  double* rne;
  /* caller-owned, capacity n, or NULL: log predictive likelihoods (data tempering)
   * logpl[s-1] = log p(y_s | y_{1:s-1}) = log[sum_jn w_jn^(s-1) p(y_s | theta_jn) /
   * sum_jn w_jn^(s-1)] over the particles of the cycle that absorbs s (PAPER.md:532-535,
   * 1413-1416; R18) */
  double* logpl;
  /* Optional adaptive-control trace (test pins of PAPER.md:392-402 cycle end,
   * 443-445 h rule, 447-451 RNE stop, 813-816 log ML); NULL / 0 to skip. */
  int32_t trace_cap;      /* capacity in M steps of step_nacc / step_h / step_minrne */
  int32_t* step_nacc;     /* accepted particles in M step m (global step index) */
  int32_t* step_h;        /* h_lr (hundredths) that M step m used */
  double* step_minrne;    /* min monitor RNE after M step m */
  int32_t snap_cap;       /* capacity in cycles of theta_snap */
  double* theta_snap;     /* theta at the start of cycle l (before its C phase), P x d each */
  double* inc_group;      /* per-group log-ML increment of cycle l, capacity max_cycles x J */
  double* Lj;             /* per-group cumulative log ML L_j, capacity J */
} or_report;

/* ---- random numbers ---------------------- */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
double or_u01(uint32_t hi, uint32_t lo);
/* Portable elementary functions built from IEEE +,-,*,/,sqrt only. */
double or_plog(double x);
double or_pexp(double x);
void or_psincos2pi(double u, double* s, double* c);
/* count standard normals for (id, step, tag, pass) */
void or_normals(uint64_t seed, uint32_t id, uint32_t step, uint32_t tag, uint32_t pass, int32_t count,
                double* z);
/* the uniform of ACCEPT draw / the 52-bit integer of RESAMPLE draw r */
double or_accept_uniform(uint64_t seed, uint32_t p, uint32_t step, uint32_t pass);
uint64_t or_resample_a52(uint64_t seed, uint32_t group, uint32_t cycle, uint32_t pass, uint32_t r);

/* ---- model --------------------------------------------------------------- */
double or_logp(const double* theta, const double* x, int32_t y, int32_t k, int32_t C);
int32_t or_loglik_range(const double* theta, int64_t P, int32_t ld, const double* X, const int32_t* y,
                        int32_t n, int32_t k, int32_t C, int32_t t0, int32_t t1, int32_t n_threads,
                        double* out);
int32_t or_cholesky(int32_t d, const double* A, double* Lo);
double or_prior_quad(int32_t d, const double* Lprior, const double* mu, const double* theta);
int32_t or_g_prior(const double* X, int32_t n, int32_t k, int32_t C, double g, double* cov);

/* ---- SPS pieces --------------------------------------------------------- */
double or_ess(const double* lw, int64_t P);
int32_t or_resample_int(int32_t N, const uint64_t* q, int32_t scheme, const uint64_t* a, int32_t* anc);
int32_t or_resample_group(int32_t N, const double* lw, int32_t scheme, uint64_t seed, uint32_t group,
                          uint32_t cycle, uint32_t pass, int32_t* anc);
void or_group_stats(const double* g, int32_t J, int32_t N, double* mean, double* sd, double* nse, double* rne);
int32_t or_power_search(const double* L, int64_t P, double rem, double ess_frac, double* dphi);

/* ---- Algorithm 2, whole run --------------------------------------------- */
int32_t or_run(const or_config* cfg, const double* X, const int32_t* y, const double* prior_mean,
               const double* prior_cov, const double* monitors, const double* report_fns,
               or_report* rep, double* theta_out);

/* ---- Algorithm 3 (two pass) ---------------------------
 * A fixed design for pass 2: L cycles, their break points t_l (data tempering)
 * or phi_l (power tempering), M steps R_l, and the proposal variance matrices
 * Sigma_lr (d x d, row-major, one per M step in execution order). */
typedef struct {
  int32_t L;
  const int32_t* t_cycle;
  const double* phi_cycle;
  const int32_t* R_cycle;
  const double* sigma;
} or_schedule;

/* or_run with (a) replay != NULL: Algorithm 2 with the cycle break points, M
 * step counts and proposal variances fixed by `replay` (Algorithm 3 step 2 --
 * no ESS rule, no h / V adaptation, no RNE stopping); (b) sigma_out != NULL:
 * the Sigma_lr actually used are recorded (capacity sigma_cap steps; Algorithm
 * 3 step 1).  Everything else as or_run. */
int32_t or_run2(const or_config* cfg, const double* X, const int32_t* y, const double* prior_mean,
                const double* prior_cov, const double* monitors, const double* report_fns,
                const or_schedule* replay, double* sigma_out, int64_t sigma_cap, or_report* rep,
                double* theta_out);

#ifdef __cplusplus
}
#endif
#endif
