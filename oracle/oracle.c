/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * A plain, slow, obviously-correct CPU implementation of what the SPS logit
 * hot path computes, written from Geweke, Durham & Xu, "Bayesian Inference
 * for Logistic Regression Models using Sequential Posterior Simulation",
 * arXiv:1304.4333.  fp64 throughout; scalar loops; OpenMP only
 * over independent particles; every reduction is serial in index order.
 * Compiled with -O2 -ffp-contract=off so that every + - * / is one IEEE op.
 *
 * Shares no code with the CUDA path (paper_1304_4333_b200/csrc).  The random
 * streams are an independent implementation of the same counter-based
 * generator (Philox4x32-10 + the conversions of DESIGN.md "Random streams").
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* ======================================================================
 * Random streams (R15).  Philox4x32-10 of
 * Salmon, Moraes, Dror & Shaw (SC'11): 10 rounds of the 4x32 Philox
 * S-box with multipliers 0xD2511F53 / 0xCD9E8D57 and Weyl key increments
 * 0x9E3779B9 / 0xBB67AE85.  Pinned by the Random123 known-answer tests.
 * ====================================================================== */
void or_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  uint32_t c0 = ctr[0], c1 = ctr[1], c2 = ctr[2], c3 = ctr[3];
  uint32_t k0 = key[0], k1 = key[1];
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    uint64_t p0 = (uint64_t)0xD2511F53u * (uint64_t)c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * (uint64_t)c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    uint32_t n0 = hi1 ^ c1 ^ k0;
    uint32_t n2 = hi0 ^ c3 ^ k1;
    c0 = n0;
    c1 = lo1;
    c2 = n2;
    c3 = lo0;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

/* u = (2*(x>>12)+1) * 2^-53 with x = hi:lo, an exact double in (0,1). */
double or_u01(uint32_t hi, uint32_t lo) {
  uint64_t x = ((uint64_t)hi << 32) | (uint64_t)lo;
  uint64_t m = 2u * (x >> 12) + 1u;
  return (double)m * 0x1p-53;
}

static void stream_block(uint64_t seed, uint32_t i, uint32_t id, uint32_t step, uint32_t tag, uint32_t pass,
                         uint32_t out[4]) {
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  uint32_t ctr[4] = {i, id, step, tag | (pass << 8)};
  or_philox4x32_10(ctr, key, out);
}

static double dbl_from_bits(uint64_t b) {
  double d;
  memcpy(&d, &b, 8);
  return d;
}
static uint64_t bits_from_dbl(double d) {
  uint64_t b;
  memcpy(&b, &d, 8);
  return b;
}

/* Portable log for positive normal x: x = 2^e m, m in (sqrt(2)/2, sqrt(2)],
 * log m = 2 atanh(s), s = (m-1)/(m+1), series to s^23.  Only IEEE + - * / and fma (each
 * a single correctly rounded IEEE operation, so the CUDA library reproduces it bit for bit; R15). */
double or_plog(double x) {
  uint64_t b = bits_from_dbl(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = dbl_from_bits((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull);
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = m * 0.5;
    e = e + 1;
  }
  double f = m - 1.0;
  double s = f / (2.0 + f);
  double z = s * s;
  double R = 0x1.642c8590b2164p-5;     /* 1/23 */
  R = fma(z, R, 0x1.8618618618618p-5);    /* 1/21 */
  R = fma(z, R, 0x1.af286bca1af28p-5);    /* 1/19 */
  R = fma(z, R, 0x1.e1e1e1e1e1e1ep-5);    /* 1/17 */
  R = fma(z, R, 0x1.1111111111111p-4);    /* 1/15 */
  R = fma(z, R, 0x1.3b13b13b13b14p-4);    /* 1/13 */
  R = fma(z, R, 0x1.745d1745d1746p-4);    /* 1/11 */
  R = fma(z, R, 0x1.c71c71c71c71cp-4);    /* 1/9 */
  R = fma(z, R, 0x1.2492492492492p-3);    /* 1/7 */
  R = fma(z, R, 0x1.999999999999ap-3);    /* 1/5 */
  R = fma(z, R, 0x1.5555555555555p-2);    /* 1/3 */
  double two_s = 2.0 * s;
  double logm = fma(two_s, z * R, two_s);
  double ed = (double)e;
  return fma(ed, 0x1.62e42fee00000p-1, fma(ed, 0x1.a39ef35793c76p-33, logm));
}

/* Portable exp for x <= 0 (resampling weights).  x < -708 -> 0 (R8).
 * x = k ln2 + r, |r| <= ln2/2; e^r by the degree-13 Taylor polynomial in
 * Horner form p = 1 + (r/i) p, i = 13..1; result p * 2^k.  Only + - * / floor. */
double or_pexp(double x) {
  if (!(x >= -708.0)) return 0.0;
  double t = x * 0x1.71547652b82fep+0;
  double kf = floor(t + 0.5);
  double r = (x - kf * 0x1.62e42fee00000p-1) - kf * 0x1.a39ef35793c76p-33;
  double p = 1.0;
  for (int i = 13; i >= 1; --i) p = 1.0 + (r / (double)i) * p;
  int k = (int)kf;
  double scale = dbl_from_bits((uint64_t)(k + 1023) << 52);
  return p * scale;
}

/* Portable (sin 2 pi u, cos 2 pi u) for u in (0,1): v = 4u exact, q = nearest
 * quadrant, f = v - q exact in [-1/2, 1/2], a = f pi/2; Taylor to a^17 / a^16, Horner steps
 * as fma (R15). */
void or_psincos2pi(double u, double* s_out, double* c_out) {
  double v = 4.0 * u;
  double q = floor(v + 0.5);
  double f = v - q;
  double a = f * 0x1.921fb54442d18p+0;
  double a2 = a * a;
  double sp = 0x1.952c77030ad4ap-49;
  sp = fma(a2, sp, -0x1.ae7f3e733b81fp-41);
  sp = fma(a2, sp, 0x1.6124613a86d09p-33);
  sp = fma(a2, sp, -0x1.ae64567f544e4p-26);
  sp = fma(a2, sp, 0x1.71de3a556c734p-19);
  sp = fma(a2, sp, -0x1.a01a01a01a01ap-13);
  sp = fma(a2, sp, 0x1.1111111111111p-7);
  sp = fma(a2, sp, -0x1.5555555555555p-3);
  double s = fma(a, a2 * sp, a);
  double cp = 0x1.ae7f3e733b81fp-45;
  cp = fma(a2, cp, -0x1.93974a8c07c9dp-37);
  cp = fma(a2, cp, 0x1.1eed8eff8d898p-29);
  cp = fma(a2, cp, -0x1.27e4fb7789f5cp-22);
  cp = fma(a2, cp, 0x1.a01a01a01a01ap-16);
  cp = fma(a2, cp, -0x1.6c16c16c16c17p-10);
  cp = fma(a2, cp, 0x1.5555555555555p-5);
  cp = fma(a2, cp, -0x1.0000000000000p-1);
  double c = fma(a2, cp, 1.0);
  int qi = ((int)q) & 3;
  if (qi == 0) {
    *s_out = s;
    *c_out = c;
  } else if (qi == 1) {
    *s_out = c;
    *c_out = -s;
  } else if (qi == 2) {
    *s_out = -s;
    *c_out = -c;
  } else {
    *s_out = -c;
    *c_out = s;
  }
}

/* Box-Muller on block i of the (id, step, tag, pass) stream: z_2i, z_2i+1. */
void or_normals(uint64_t seed, uint32_t id, uint32_t step, uint32_t tag, uint32_t pass, int32_t count,
                double* z) {
  for (int32_t i = 0; 2 * i < count; ++i) {
    uint32_t w[4];
    stream_block(seed, (uint32_t)i, id, step, tag, pass, w);
    double u1 = or_u01(w[0], w[1]);
    double u2 = or_u01(w[2], w[3]);
    double r = sqrt(-2.0 * or_plog(u1));
    double s, c;
    or_psincos2pi(u2, &s, &c);
    z[2 * i] = r * c;
    if (2 * i + 1 < count) z[2 * i + 1] = r * s;
  }
}

double or_accept_uniform(uint64_t seed, uint32_t p, uint32_t step, uint32_t pass) {
  uint32_t w[4];
  stream_block(seed, 0u, p, step, OR_TAG_ACCEPT, pass, w);
  return or_u01(w[0], w[1]);
}

uint64_t or_resample_a52(uint64_t seed, uint32_t group, uint32_t cycle, uint32_t pass, uint32_t r) {
  uint32_t w[4];
  stream_block(seed, r >> 1, group, cycle, OR_TAG_RESAMPLE, pass, w);
  uint32_t hi = (r & 1u) ? w[2] : w[0];
  uint32_t lo = (r & 1u) ? w[3] : w[1];
  uint64_t x = ((uint64_t)hi << 32) | (uint64_t)lo;
  return x >> 12;
}

/* ======================================================================
 * Model.  PAPER.md:115-125 eq. (plogit): P(Y=c|x,theta) = exp(theta_c'x) /
 * sum_i exp(theta_i'x), with the normalization theta_C = 0 (PAPER.md:126-128,
 * 649-658).  Our label 0 is the paper's reference category C (R1), so
 * eta_0 = 0 and eta_c = theta_c'x for c = 1..C-1, theta = [theta_1..theta_{C-1}]
 * stacked in blocks of k (d = k(C-1)).
 *
 * log P(Y=y) = eta_y - log sum_c exp(eta_c), evaluated as
 * (eta_y - m) - log1p(sum_{c != c*} exp(eta_c - m)), m = eta_{c*} = max.
 * ====================================================================== */
double or_logp(const double* theta, const double* x, int32_t y, int32_t k, int32_t C) {
  double eta[64];
  eta[0] = 0.0;
  for (int32_t c = 1; c < C; ++c) {
    double acc = 0.0;
    for (int32_t i = 0; i < k; ++i) acc += theta[(c - 1) * k + i] * x[i];
    eta[c] = acc;
  }
  int32_t cstar = 0;
  for (int32_t c = 1; c < C; ++c)
    if (eta[c] > eta[cstar]) cstar = c;
  double m = eta[cstar];
  double rest = 0.0;
  for (int32_t c = 0; c < C; ++c)
    if (c != cstar) rest += exp(eta[c] - m);
  return (eta[y] - m) - log1p(rest);
}

/* L_p = sum_{t0 <= t < t1} log p(y_t | x_t, theta_p): the likelihood
 * factorization of PAPER.md:233-242 (observations conditionally independent). */
int32_t or_loglik_range(const double* theta, int64_t P, int32_t ld, const double* X, const int32_t* y,
                        int32_t n, int32_t k, int32_t C, int32_t t0, int32_t t1, int32_t n_threads,
                        double* out) {
  if (t0 < 0 || t1 < t0 || t1 > n || C < 2 || C > 64 || k < 1) return OR_E_CONFIG;
  int bad = 0;
#ifdef _OPENMP
  int nt = n_threads > 0 ? n_threads : omp_get_max_threads();
#pragma omp parallel for num_threads(nt) schedule(static) reduction(| : bad)
#endif
  for (int64_t p = 0; p < P; ++p) {
    double acc = 0.0;
    for (int32_t t = t0; t < t1; ++t) acc += or_logp(theta + p * ld, X + (int64_t)t * k, y[t], k, C);
    out[p] = acc;
    if (!isfinite(acc)) bad = 1;
  }
  (void)n_threads;
  return bad ? OR_E_NUMERIC : OR_OK;
}

/* Cholesky-Banachiewicz, row-major lower factor Lo with A = Lo Lo'. */
int32_t or_cholesky(int32_t d, const double* A, double* Lo) {
  memset(Lo, 0, sizeof(double) * (size_t)d * (size_t)d);
  for (int32_t j = 0; j < d; ++j) {
    double s = A[j * d + j];
    for (int32_t q = 0; q < j; ++q) s -= Lo[j * d + q] * Lo[j * d + q];
    if (!(s > 0.0) || !isfinite(s)) return OR_E_NUMERIC;
    double ljj = sqrt(s);
    Lo[j * d + j] = ljj;
    for (int32_t i = j + 1; i < d; ++i) {
      double t = A[i * d + j];
      for (int32_t q = 0; q < j; ++q) t -= Lo[i * d + q] * Lo[j * d + q];
      Lo[i * d + j] = t / ljj;
    }
  }
  return OR_OK;
}

/* Gaussian prior kernel (PAPER.md:637-648 eqs. prior_Gauss, prior_norm):
 * log p(theta) = -1/2 (theta-mu)' Sigma^-1 (theta-mu) + const, by forward
 * substitution w = Lprior^-1 (theta - mu).  The constant cancels in every
 * Metropolis ratio and is not needed elsewhere. */
double or_prior_quad(int32_t d, const double* Lprior, const double* mu, const double* theta) {
  double w[512];
  double q = 0.0;
  for (int32_t i = 0; i < d; ++i) {
    double t = theta[i] - mu[i];
    for (int32_t j = 0; j < i; ++j) t -= Lprior[i * d + j] * w[j];
    w[i] = t / Lprior[i * d + i];
    q += w[i] * w[i];
  }
  return -0.5 * q;
}

/* Zellner g-prior PAPER.md:665-668 eq. (g-prior_def): Sigma = g T (X'X)^-1,
 * exchangeable mu_c = 0, Sigma_c = Sigma, normalized with
 * eq. (prior_norm): var(theta_j - theta_C) = 2 Sigma, cov(...) = Sigma
 * (PAPER.md:641-648).  Output: d x d covariance, d = k(C-1).  (R9: the
 * printed formula is used; its log-odds variance is 2gk, not the 2g of
 * PAPER.md:674-678.) */
int32_t or_g_prior(const double* X, int32_t n, int32_t k, int32_t C, double g, double* cov) {
  double* XtX = (double*)calloc((size_t)k * k, sizeof(double));
  double* Lo = (double*)calloc((size_t)k * k, sizeof(double));
  double* inv = (double*)calloc((size_t)k * k, sizeof(double));
  double* col = (double*)calloc((size_t)k, sizeof(double));
  int32_t st = OR_OK;
  for (int32_t a = 0; a < k; ++a)
    for (int32_t b = 0; b < k; ++b) {
      double s = 0.0;
      for (int32_t t = 0; t < n; ++t) s += X[(int64_t)t * k + a] * X[(int64_t)t * k + b];
      XtX[a * k + b] = s;
    }
  if (or_cholesky(k, XtX, Lo) != OR_OK) {
    st = OR_E_DATA;
    goto done;
  }
  /* inverse column by column: solve Lo Lo' x = e_b */
  for (int32_t b = 0; b < k; ++b) {
    for (int32_t i = 0; i < k; ++i) {
      double t = (i == b) ? 1.0 : 0.0;
      for (int32_t j = 0; j < i; ++j) t -= Lo[i * k + j] * col[j];
      col[i] = t / Lo[i * k + i];
    }
    for (int32_t i = k - 1; i >= 0; --i) {
      double t = col[i];
      for (int32_t j = i + 1; j < k; ++j) t -= Lo[j * k + i] * col[j];
      col[i] = t / Lo[i * k + i];
    }
    for (int32_t i = 0; i < k; ++i) inv[i * k + b] = col[i];
  }
  {
    int32_t d = k * (C - 1);
    for (int32_t bi = 0; bi < C - 1; ++bi)
      for (int32_t bj = 0; bj < C - 1; ++bj)
        for (int32_t a = 0; a < k; ++a)
          for (int32_t b = 0; b < k; ++b) {
            double s = g * (double)n * inv[a * k + b];
            cov[(int64_t)(bi * k + a) * d + (bj * k + b)] = (bi == bj) ? 2.0 * s : s;
          }
  }
done:
  free(XtX);
  free(Lo);
  free(inv);
  free(col);
  return st;
}

/* ======================================================================
 * SPS pieces
 * ====================================================================== */

/* PAPER.md:392-397 eq. (ESS_rule): ESS = (sum w)^2 / sum w^2, w = exp(lw),
 * evaluated after subtracting max lw (a common factor that cancels). */
double or_ess(const double* lw, int64_t P) {
  double m = lw[0];
  for (int64_t p = 1; p < P; ++p)
    if (lw[p] > m) m = lw[p];
  double s1 = 0.0, s2 = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    double w = exp(lw[p] - m);
    s1 += w;
    s2 += w * w;
  }
  return s1 * s1 / s2;
}

static int32_t first_above(const uint64_t* cum, int32_t N, uint64_t pos) {
  /* first n with cum[n] > pos (cum inclusive prefix sums, cum[N-1] > pos) */
  for (int32_t n = 0; n < N; ++n)
    if (cum[n] > pos) return n;
  return -1;
}

/* S phase: residual (default; Chopin 2004 Thm 2,
 * PAPER.md:342-344), systematic, or multinomial resampling on integer
 * weights q_n (R7).  a[] are 52-bit uniforms u = (2a+1)2^-53.  Ancestors
 * are written in ascending order. */
int32_t or_resample_int(int32_t N, const uint64_t* q, int32_t scheme, const uint64_t* a, int32_t* anc) {
  if (N < 1 || N > 16384) return OR_E_CONFIG;
  uint64_t Q = 0;
  for (int32_t n = 0; n < N; ++n) Q += q[n];
  if (Q == 0) return OR_E_NUMERIC;
  int32_t* counts = (int32_t*)calloc((size_t)N, sizeof(int32_t));
  uint64_t* cum = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)N);
  if (scheme == OR_RESIDUAL) {
    uint64_t csum = 0, run = 0;
    for (int32_t n = 0; n < N; ++n) {
      uint64_t c = ((uint64_t)N * q[n]) / Q;
      counts[n] = (int32_t)c;
      csum += c;
      run += (uint64_t)N * q[n] - c * Q;
      cum[n] = run;
    }
    uint64_t R = (uint64_t)N - csum;
    uint64_t RQ = R * Q;
    for (uint64_t i = 0; i < R; ++i) {
      uint64_t pos = (uint64_t)(((u128)(2u * a[i] + 1u) * (u128)RQ) >> 53);
      counts[first_above(cum, N, pos)] += 1;
    }
  } else {
    uint64_t run = 0;
    for (int32_t n = 0; n < N; ++n) {
      run += q[n];
      cum[n] = run;
    }
    for (int32_t i = 0; i < N; ++i) {
      uint64_t pos;
      if (scheme == OR_SYSTEMATIC) {
        u128 num = ((u128)(uint64_t)i << 53) + (u128)(2u * a[0] + 1u);
        pos = (uint64_t)(((num * (u128)Q) / (u128)(uint64_t)N) >> 53);
      } else {
        pos = (uint64_t)(((u128)(2u * a[i] + 1u) * (u128)Q) >> 53);
      }
      counts[first_above(cum, N, pos)] += 1;
    }
  }
  int32_t idx = 0;
  for (int32_t n = 0; n < N; ++n)
    for (int32_t c = 0; c < counts[n]; ++c) anc[idx++] = n;
  free(counts);
  free(cum);
  return idx == N ? OR_OK : OR_E_NUMERIC;
}

/* Integer weights of one group: q_n = floor(pexp(lw_n - max lw) 2^32) (R7),
 * then or_resample_int with the RESAMPLE stream of (group, cycle). */
int32_t or_resample_group(int32_t N, const double* lw, int32_t scheme, uint64_t seed, uint32_t group,
                          uint32_t cycle, uint32_t pass, int32_t* anc) {
  if (N < 1 || N > 16384) return OR_E_CONFIG;
  uint64_t* q = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)N);
  uint64_t* a = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)N);
  double m = lw[0];
  for (int32_t n = 1; n < N; ++n)
    if (lw[n] > m) m = lw[n];
  for (int32_t n = 0; n < N; ++n) q[n] = (uint64_t)floor(or_pexp(lw[n] - m) * 4294967296.0);
  for (int32_t r = 0; r < N; ++r) a[r] = or_resample_a52(seed, group, cycle, pass, (uint32_t)r);
  int32_t st = or_resample_int(N, q, scheme, a, anc);
  free(q);
  free(a);
  return st;
}

/* group means (partial_g), grand mean (whole_g), v-hat,
 * NSE (NSE_def, corrected to [(JN)^-1 v-hat]^1/2, R2), RNE (RNE_def);
 * sd = [(JN)^-1 sum (g - gbar)^2]^1/2.  v-hat = 0 -> RNE = +inf (R12). */
void or_group_stats(const double* g, int32_t J, int32_t N, double* mean, double* sd, double* nse, double* rne) {
  double* gj = (double*)malloc(sizeof(double) * (size_t)J);
  for (int32_t j = 0; j < J; ++j) {
    double s = 0.0;
    for (int32_t n = 0; n < N; ++n) s += g[(int64_t)j * N + n];
    gj[j] = s / (double)N;
  }
  double gbar = 0.0;
  for (int32_t j = 0; j < J; ++j) gbar += gj[j];
  gbar = gbar / (double)J;
  double dev = 0.0;
  for (int32_t j = 0; j < J; ++j) dev += (gj[j] - gbar) * (gj[j] - gbar);
  double vhat = ((double)N / (double)(J - 1)) * dev;
  double ss = 0.0;
  for (int64_t i = 0; i < (int64_t)J * N; ++i) ss += (g[i] - gbar) * (g[i] - gbar);
  double var = ss / ((double)J * (double)N);
  if (mean) *mean = gbar;
  if (sd) *sd = sqrt(var);
  if (nse) *nse = sqrt(vhat / ((double)J * (double)N));
  if (rne) *rne = vhat > 0.0 ? var / vhat : INFINITY;
  free(gj);
}

/* Power-tempering increment (north_star; R5): largest dphi on the grid
 * (q 2^-48) rem, q integer, with ESS(dphi) >= ess_frac P, ESS computed on
 * w = exp(dphi (L - max L)); plain integer bisection, 48 halvings. */
static int ess_ok(const double* L, int64_t P, double Lmax, double dphi, double ess_frac) {
  double s1 = 0.0, s2 = 0.0;
  for (int64_t p = 0; p < P; ++p) {
    double w = exp(dphi * (L[p] - Lmax));
    s1 += w;
    s2 += w * w;
  }
  return !(s1 * s1 < ess_frac * (double)P * s2);
}

int32_t or_power_search(const double* L, int64_t P, double rem, double ess_frac, double* dphi) {
  double Lmax = L[0];
  for (int64_t p = 1; p < P; ++p)
    if (L[p] > Lmax) Lmax = L[p];
  if (ess_ok(L, P, Lmax, rem, ess_frac)) {
    *dphi = rem;
    return OR_OK;
  }
  uint64_t lo = 0, hi = (uint64_t)1 << 48;
  while (hi - lo > 1) {
    uint64_t mid = lo + (hi - lo) / 2;
    double dp = ((double)mid * 0x1p-48) * rem;
    if (ess_ok(L, P, Lmax, dp, ess_frac))
      lo = mid;
    else
      hi = mid;
  }
  if (lo == 0) lo = 1;
  *dphi = ((double)lo * 0x1p-48) * rem;
  return OR_OK;
}

/* ======================================================================
 * Algorithm 2 with the phases of Algorithm 1
 * (PAPER.md:266-326).
 * ====================================================================== */
static int nthreads_of(const or_config* cfg) {
#ifdef _OPENMP
  return cfg->n_threads > 0 ? cfg->n_threads : omp_get_max_threads();
#else
  (void)cfg;
  return 1;
#endif
}

int32_t or_run(const or_config* cfg, const double* X, const int32_t* y, const double* prior_mean,
               const double* prior_cov, const double* monitors, const double* report_fns,
               or_report* rep, double* theta_out) {
  return or_run2(cfg, X, y, prior_mean, prior_cov, monitors, report_fns, NULL, NULL, 0, rep, theta_out);
}

int32_t or_run2(const or_config* cfg, const double* X, const int32_t* y, const double* prior_mean,
                const double* prior_cov, const double* monitors, const double* report_fns,
                const or_schedule* replay, double* sigma_out, int64_t sigma_cap, or_report* rep,
                double* theta_out) {
  const int32_t n = cfg->n, k = cfg->k, C = cfg->C, J = cfg->J, N = cfg->N;
  if (n < 1 || k < 1 || C < 2 || C > 64 || J < 2 || N < 2 || N > 16384 || k * (C - 1) > 512 ||
      cfg->n_monitors < 1 || cfg->max_cycles < 1 || cfg->h_min > cfg->h_init || cfg->h_init > cfg->h_max)
    return rep->status = OR_E_CONFIG;
  for (int32_t t = 0; t < n; ++t)
    if (y[t] < 0 || y[t] >= C) return rep->status = OR_E_DATA;
  const int32_t d = k * (C - 1);
  const int64_t P = (int64_t)J * N;
  const int nt = nthreads_of(cfg);
  const int power = cfg->tempering == OR_POWER_TEMPERING;
  int32_t st = OR_OK;

  double* Lprior = (double*)malloc(sizeof(double) * d * d);
  double* theta = (double*)malloc(sizeof(double) * P * d);
  double* theta2 = (double*)malloc(sizeof(double) * P * d);
  double* Lk = (double*)malloc(sizeof(double) * P);   /* cached log-likelihood L_p */
  double* Lk2 = (double*)malloc(sizeof(double) * P);
  double* lp = (double*)malloc(sizeof(double) * P);   /* cached prior kernel */
  double* lp2 = (double*)malloc(sizeof(double) * P);
  double* lw = (double*)malloc(sizeof(double) * P);   /* log weights of the C phase */
  double* mean = (double*)malloc(sizeof(double) * d);
  double* V = (double*)malloc(sizeof(double) * d * d);
  double* Sig = (double*)malloc(sizeof(double) * d * d);
  double* Lprop = (double*)malloc(sizeof(double) * d * d);
  double* g = (double*)malloc(sizeof(double) * P);
  double* Lj = (double*)calloc((size_t)J, sizeof(double)); /* per-group cumulative log ML */
  int32_t* anc = (int32_t*)malloc(sizeof(int32_t) * N);
  unsigned char* acc = (unsigned char*)malloc((size_t)P);

  rep->L = 0;
  rep->total_m_steps = 0;
  rep->logml = 0.0;
  rep->pairs = 0.0;

  if (or_cholesky(d, prior_cov, Lprior) != OR_OK) {
    st = OR_E_CONFIG;
    goto out;
  }

  /* Algorithm 1 step 1: theta_jn ~iid p(theta). */
#pragma omp parallel for num_threads(nt) schedule(static)
  for (int64_t p = 0; p < P; ++p) {
    double z[512];
    or_normals(cfg->seed, (uint32_t)p, 0u, OR_TAG_INIT, (uint32_t)cfg->pass, d, z);
    for (int32_t i = 0; i < d; ++i) {
      double s = prior_mean[i];
      for (int32_t j = 0; j <= i; ++j) s += Lprior[i * d + j] * z[j];
      theta[p * d + i] = s;
    }
    lp[p] = or_prior_quad(d, Lprior, prior_mean, theta + p * d);
  }
  if (power) {
    st = or_loglik_range(theta, P, d, X, y, n, k, C, 0, n, nt, Lk);
    rep->pairs += (double)P * n;
    if (st) goto out;
  } else {
    for (int64_t p = 0; p < P; ++p) Lk[p] = 0.0;
  }

  int32_t t = 0;      /* t_{l-1}: observations absorbed (data tempering) */
  double phi = 0.0;   /* tempering level (power tempering) */
  int32_t h = cfg->h_init;
  uint32_t mstep = 0; /* global M-step counter, keys the PROPOSAL/ACCEPT streams */

  for (int32_t ell = 1;; ++ell) {
    if (ell > cfg->max_cycles) {
      st = OR_E_CONFIG;
      goto out;
    }
    if (rep->theta_snap && ell <= rep->snap_cap)
      memcpy(rep->theta_snap + (int64_t)(ell - 1) * P * d, theta, sizeof(double) * P * d);
    /* ---------------- C phase ------------------------------------------ */
    if (!power) {
      /* PAPER.md:281-295 eq. (C_phase_compute) in log form, with the cycle
       * end rule of PAPER.md:392-402: first s with ESS(s)/(JN) < 0.5, or T. */
      for (int64_t p = 0; p < P; ++p) lw[p] = 0.0;
      int32_t s = t;
      /* log sum_jn w_jn^(s-1): the weights are all 1 after the S phase of the last cycle */
      double lse_prev = log((double)P);
      for (;;) {
        s = s + 1;
        int32_t obs = s - 1;
        int bad = 0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(| : bad)
        for (int64_t p = 0; p < P; ++p) {
          lw[p] += or_logp(theta + p * d, X + (int64_t)obs * k, y[obs], k, C);
          if (!isfinite(lw[p])) bad = 1;
        }
        rep->pairs += (double)P;
        if (bad) {
          st = OR_E_NUMERIC;
          goto out;
        }
        double m = lw[0];
        for (int64_t p = 1; p < P; ++p)
          if (lw[p] > m) m = lw[p];
        double s1 = 0.0, s2 = 0.0;
        for (int64_t p = 0; p < P; ++p) {
          double w = exp(lw[p] - m);
          s1 += w;
          s2 += w * w;
        }
        /* log predictive likelihood of y_s (R18): the ratio of the weight
         * sums after and before absorbing observation s, w^(s) = w^(s-1) p(y_s | theta) */
        {
          const double lse = m + log(s1);
          if (rep->logpl) rep->logpl[obs] = lse - lse_prev;
          lse_prev = lse;
        }
        if (replay ? s == replay->t_cycle[ell - 1]
                   : (s1 * s1 < cfg->ess_frac * (double)P * s2 || s == n))
          break;
      }
      t = s;
      for (int64_t p = 0; p < P; ++p) Lk[p] += lw[p];
    } else {
      double rem = 1.0 - phi;
      double dphi;
      if (replay) {
        dphi = replay->phi_cycle[ell - 1] - phi;
      } else {
        or_power_search(Lk, P, rem, cfg->ess_frac, &dphi);
      }
      for (int64_t p = 0; p < P; ++p) lw[p] = dphi * Lk[p];
      phi = replay ? replay->phi_cycle[ell - 1] : ((dphi == rem) ? 1.0 : phi + dphi);
    }
    /* log marginal likelihood increment (R10):
     * log[(JN)^-1 sum_jn w_jn] pooled and log[N^-1 sum_n w_jn] per group. */
    {
      double m = lw[0];
      for (int64_t p = 1; p < P; ++p)
        if (lw[p] > m) m = lw[p];
      double s1 = 0.0;
      for (int64_t p = 0; p < P; ++p) s1 += exp(lw[p] - m);
      double inc = m + log(s1 / (double)P);
      rep->logml += inc;
      rep->logml_inc[ell - 1] = inc;
      for (int32_t j = 0; j < J; ++j) {
        double mj = lw[(int64_t)j * N];
        for (int32_t q = 1; q < N; ++q)
          if (lw[(int64_t)j * N + q] > mj) mj = lw[(int64_t)j * N + q];
        double sj = 0.0;
        for (int32_t q = 0; q < N; ++q) sj += exp(lw[(int64_t)j * N + q] - mj);
        const double incj = mj + log(sj / (double)N);
        Lj[j] += incj;
        if (rep->inc_group) rep->inc_group[(int64_t)(ell - 1) * J + j] = incj;
      }
    }
    /* ---------------- S phase, per group ------------- */
    for (int32_t j = 0; j < J; ++j) {
      st = or_resample_group(N, lw + (int64_t)j * N, cfg->resampling, cfg->seed, (uint32_t)j, (uint32_t)ell,
                             (uint32_t)cfg->pass, anc);
      if (st) goto out;
      for (int32_t q = 0; q < N; ++q) {
        int64_t dst = (int64_t)j * N + q, src = (int64_t)j * N + anc[q];
        memcpy(theta2 + dst * d, theta + src * d, sizeof(double) * d);
        Lk2[dst] = Lk[src];
        lp2[dst] = lp[src];
      }
    }
    { double* tmp = theta; theta = theta2; theta2 = tmp; }
    { double* tmp = Lk; Lk = Lk2; Lk2 = tmp; }
    { double* tmp = lp; lp = lp2; lp2 = tmp; }

    /* ---------------- M phase ------------------------ */
    const int final_cycle = replay ? (ell == replay->L) : (power ? (phi == 1.0) : (t == n));
    const double K = final_cycle ? cfg->K_final : cfg->K_inter;   /* PAPER.md:418-424, R14 */
    const int32_t r_t1 = power ? n : t;
    const double temper = power ? phi : 1.0;
    int32_t r = 0;
    double minrne = 0.0;
    for (;;) {
      r = r + 1;
      if (r > cfg->max_m_steps) {
        st = OR_E_MIXING;
        goto out;
      }
      /* i. sample variance V_lr of all JN particles (R11) -- pass 2 of
       * Algorithm 3 takes Sigma_lr from the pass-1 record instead */
      double hd = (double)h / 100.0;
      if (replay) {
        memcpy(Sig, replay->sigma + (int64_t)mstep * d * d, sizeof(double) * d * d);
        for (int32_t i = 0; i < d * d; ++i) V[i] = Sig[i] / hd;  /* (only the ridge retry reads V) */
      } else {
      for (int32_t i = 0; i < d; ++i) {
        double s = 0.0;
        for (int64_t p = 0; p < P; ++p) s += theta[p * d + i];
        mean[i] = s / (double)P;
      }
      for (int32_t i = 0; i < d; ++i)
        for (int32_t j = 0; j <= i; ++j) {
          double s = 0.0;
          for (int64_t p = 0; p < P; ++p) s += (theta[p * d + i] - mean[i]) * (theta[p * d + j] - mean[j]);
          V[i * d + j] = V[j * d + i] = s / (double)(P - 1);
        }
      /* Sigma_lr = h_lr V_lr, Cholesky with one ridge retry (R13) */
      for (int32_t i = 0; i < d * d; ++i) Sig[i] = hd * V[i];
      }
      if (sigma_out && (int64_t)mstep < sigma_cap) memcpy(sigma_out + (int64_t)mstep * d * d, Sig, sizeof(double) * d * d);
      if (or_cholesky(d, Sig, Lprop) != OR_OK) {
        double tr = 0.0;
        for (int32_t i = 0; i < d; ++i) tr += V[i * d + i];
        double ridge = 1e-8 * tr / (double)d;
        for (int32_t i = 0; i < d; ++i)
          for (int32_t j = 0; j < d; ++j) Sig[i * d + j] = hd * (V[i * d + j] + (i == j ? ridge : 0.0));
        if (or_cholesky(d, Sig, Lprop) != OR_OK) {
          st = OR_E_NUMERIC;
          goto out;
        }
      }
      /* Gaussian random-walk Metropolis step for every particle */
      int bad = 0;
#pragma omp parallel for num_threads(nt) schedule(static) reduction(| : bad)
      for (int64_t p = 0; p < P; ++p) {
        double z[512], th[512];
        or_normals(cfg->seed, (uint32_t)p, mstep, OR_TAG_PROPOSAL, (uint32_t)cfg->pass, d, z);
        for (int32_t i = 0; i < d; ++i) {
          double s = theta[p * d + i];
          for (int32_t j = 0; j <= i; ++j) s += Lprop[i * d + j] * z[j];
          th[i] = s;
        }
        double lps = or_prior_quad(d, Lprior, prior_mean, th);
        double Ls = 0.0;
        for (int32_t tt = 0; tt < r_t1; ++tt) Ls += or_logp(th, X + (int64_t)tt * k, y[tt], k, C);
        if (!isfinite(Ls)) bad = 1;
        double delta = temper * (Ls - Lk[p]) + (lps - lp[p]);
        double u = or_accept_uniform(cfg->seed, (uint32_t)p, mstep, (uint32_t)cfg->pass);
        acc[p] = 0;
        if (or_plog(u) < delta) {
          acc[p] = 1;
          memcpy(theta + p * d, th, sizeof(double) * d);
          Lk[p] = Ls;
          lp[p] = lps;
        }
      }
      rep->pairs += (double)P * r_t1;
      if (bad) {
        st = OR_E_NUMERIC;
        goto out;
      }
      int64_t nacc = 0;
      for (int64_t p = 0; p < P; ++p) nacc += acc[p];
      const int64_t m_this = mstep;
      if (rep->step_h && m_this < rep->trace_cap) {
        rep->step_h[m_this] = h;
        rep->step_nacc[m_this] = (int32_t)nacc;
      }
      mstep = mstep + 1;
      /* ii. step-scale adaptation (R6) */
      if ((double)nacc > cfg->accept_target * (double)P)
        h = (h + cfg->h_step < cfg->h_max) ? h + cfg->h_step : cfg->h_max;
      else
        h = (h - cfg->h_step > cfg->h_min) ? h - cfg->h_step : cfg->h_min;
      /* iii. RNE of the test functions g* (R12) */
      minrne = INFINITY;
      for (int32_t i = 0; i < cfg->n_monitors; ++i) {
        const double* a = monitors + (int64_t)i * d;
        for (int64_t p = 0; p < P; ++p) {
          double s = 0.0;
          for (int32_t q = 0; q < d; ++q) s += a[q] * theta[p * d + q];
          g[p] = s;
        }
        double rne;
        or_group_stats(g, J, N, NULL, NULL, NULL, &rne);
        if (rne < minrne) minrne = rne;
      }
      if (rep->step_minrne && m_this < rep->trace_cap) rep->step_minrne[m_this] = minrne;
      if (replay ? r == replay->R_cycle[ell - 1] : minrne >= K) break;
    }
    rep->L = ell;
    rep->total_m_steps += r;
    rep->t_cycle[ell - 1] = t;
    rep->phi_cycle[ell - 1] = phi;
    rep->R_cycle[ell - 1] = r;
    rep->min_rne[ell - 1] = minrne;
    rep->h_cycle[ell - 1] = h;
    if (final_cycle) break;
  }
  rep->h_final = h;
  /* reported posterior moments */
  for (int32_t i = 0; i < cfg->n_report; ++i) {
    const double* a = report_fns + (int64_t)i * d;
    for (int64_t p = 0; p < P; ++p) {
      double s = 0.0;
      for (int32_t q = 0; q < d; ++q) s += a[q] * theta[p * d + q];
      g[p] = s;
    }
    or_group_stats(g, J, N, &rep->mean[i], &rep->sd[i], &rep->nse[i], &rep->rne[i]);
  }
  /* NSE of log ML across groups (R10): [sum_j (L_j - Lbar)^2 / (J (J-1))]^1/2 */
  {
    double Lbar = 0.0;
    for (int32_t j = 0; j < J; ++j) Lbar += Lj[j];
    Lbar = Lbar / (double)J;
    double s = 0.0;
    for (int32_t j = 0; j < J; ++j) s += (Lj[j] - Lbar) * (Lj[j] - Lbar);
    rep->logml_nse = sqrt(s / ((double)J * (double)(J - 1)));
    if (rep->Lj) memcpy(rep->Lj, Lj, sizeof(double) * J);
  }
  if (theta_out) memcpy(theta_out, theta, sizeof(double) * P * d);

out:
  rep->status = st;
  free(Lprior);
  free(theta);
  free(theta2);
  free(Lk);
  free(Lk2);
  free(lp);
  free(lp2);
  free(lw);
  free(mean);
  free(V);
  free(Sig);
  free(Lprop);
  free(g);
  free(Lj);
  free(anc);
  free(acc);
  return st;
}
