// loglik.cuh -- K1: particle x observation log-likelihood of the multinomial
// logit (PAPER.md:115-125 eq. plogit; factorization PAPER.md:233-242), fused
// contraction + epilogue + per-particle reduction, fp64 on the FP64 pipe.
//
//   L_p = sum_{t0 <= t < t1} log P(Y = y_t | x_t, theta_p)
//
// B200 design:
//  * DMMA and DFMA share one FP64 pipe on B200 (profiles/r01_fp64_peaks.json:
//    64 FMA/clk/SM either way, no overlap), so the contraction runs as DFMA
//    with theta in registers (PPT particles per thread, no k padding) and x_t
//    broadcast from a shared-memory tile of X staged once per block.
//  * The epilogue dominates with libm (log1p(exp) = ~84 DFMA-equivalents,
//    measured).  Here: log p = -(max(s,0) + log(1 + e^-|s|)) for binary with
//    s = (1-2y) x'theta (y folded into a sign-flipped copy of X), and
//    log p = (eta_y - m) - log(sum_c e^(eta_c - m)) for C > 2.  The logs are
//    deferred: the factors (1 + e^-|s|) / sum_c e^(eta_c-m) in [1, C] are
//    multiplied into a running product with its exponent renormalized every
//    64 observations, and ONE log per particle is taken at the end.  e^-a is
//    a table-driven exp (2^(i/64) table in smem, degree-5 polynomial on
//    |r| <= ln2/128): 10 FP64 ops.  Binary total: 15 FP64 ops per pair + k FMAs.
//  * Grid = particle tiles x observation chunks, chunk count chosen so the
//    block count fills whole waves of 148 SMs x resident blocks; chunk
//    partials are summed in fixed order by the consumer (deterministic).
#pragma once
#include "common.cuh"

namespace sps {

constexpr int LL_THREADS = 128;

__constant__ double c_exp2tab[64] = {
    0x1.0000000000000p+0, 0x1.02c9a3e778061p+0, 0x1.059b0d3158574p+0, 0x1.0874518759bc8p+0,
    0x1.0b5586cf9890fp+0, 0x1.0e3ec32d3d1a2p+0, 0x1.11301d0125b51p+0, 0x1.1429aaea92de0p+0,
    0x1.172b83c7d517bp+0, 0x1.1a35beb6fcb75p+0, 0x1.1d4873168b9aap+0, 0x1.2063b88628cd6p+0,
    0x1.2387a6e756238p+0, 0x1.26b4565e27cddp+0, 0x1.29e9df51fdee1p+0, 0x1.2d285a6e4030bp+0,
    0x1.306fe0a31b715p+0, 0x1.33c08b26416ffp+0, 0x1.371a7373aa9cbp+0, 0x1.3a7db34e59ff7p+0,
    0x1.3dea64c123422p+0, 0x1.4160a21f72e2ap+0, 0x1.44e086061892dp+0, 0x1.486a2b5c13cd0p+0,
    0x1.4bfdad5362a27p+0, 0x1.4f9b2769d2ca7p+0, 0x1.5342b569d4f82p+0, 0x1.56f4736b527dap+0,
    0x1.5ab07dd485429p+0, 0x1.5e76f15ad2148p+0, 0x1.6247eb03a5585p+0, 0x1.6623882552225p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6dfb23c651a2fp+0, 0x1.71f75e8ec5f74p+0, 0x1.75feb564267c9p+0,
    0x1.7a11473eb0187p+0, 0x1.7e2f336cf4e62p+0, 0x1.82589994cce13p+0, 0x1.868d99b4492edp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8f1ae99157736p+0, 0x1.93737b0cdc5e5p+0, 0x1.97d829fde4e50p+0,
    0x1.9c49182a3f090p+0, 0x1.a0c667b5de565p+0, 0x1.a5503b23e255dp+0, 0x1.a9e6b5579fdbfp+0,
    0x1.ae89f995ad3adp+0, 0x1.b33a2b84f15fbp+0, 0x1.b7f76f2fb5e47p+0, 0x1.bcc1e904bc1d2p+0,
    0x1.c199bdd85529cp+0, 0x1.c67f12e57d14bp+0, 0x1.cb720dcef9069p+0, 0x1.d072d4a07897cp+0,
    0x1.d5818dcfba487p+0, 0x1.da9e603db3285p+0, 0x1.dfc97337b9b5fp+0, 0x1.e502ee78b3ff6p+0,
    0x1.ea4afa2a490dap+0, 0x1.efa1bee615a27p+0, 0x1.f50765b6e4540p+0, 0x1.fa7c1819e90d8p+0};

struct LLArgs {
  const double* X;     // n x ldx (binary: rows sign-flipped by (1 - 2 y_t))
  const int32_t* y;    // n labels (C > 2)
  const double* theta; // P rows of ldt doubles
  double* part;        // [nchunks][P] chunk partial sums (or the output when nchunks == 1)
  int64_t ldt;
  int64_t P;
  int32_t t0, t1, chunk;
  int32_t k;           // covariates; theta block stride (K template >= k, zero padded)
  const int* stop;     // speculative M-step launches: return if set
};

// max(s, 0) and min(|s|, 708) with integer ops on the ALU pipe (sm_100a has no
// DMNMX; fmax/fmin on doubles cost a DSETP on the FP64 pipe).  For IEEE
// doubles of one sign the bit patterns order like the values.
__device__ __forceinline__ double relu_bits(double s) {
  const int hi = __double2hiint(s), lo = __double2loint(s);
  const int m = ~(hi >> 31);
  return __hiloint2double(hi & m, lo & m);
}
__device__ __forceinline__ double abs_clamp708(double s) {
  const int hi = __double2hiint(s) & 0x7fffffff, lo = __double2loint(s);
  return hi >= 0x40862000 ? 708.0 : __hiloint2double(hi, lo);  // 708 = 0x4086200000000000
}

// e^-a for 0 <= a <= 708: table-driven, ~1 ulp.  sT = 2^(i/64).
__device__ __forceinline__ double exp_neg(double a, const double* __restrict__ sT) {
  const double t = fma(a, -0x1.71547652b82fep+6, 0x1.8p52);  // MAGIC - round(a 64/ln2)
  const double kd = t - 0x1.8p52;                             // k = -round(a 64/ln2)
  double r = fma(kd, -0x1.62e42fec00000p-7, -a);              // r = -a - k ln2/64 (hi/lo)
  r = fma(kd, -0x1.d1cf79abc9e3bp-38, r);
  const int ki = __double2loint(t);
  const double T = sT[ki & 63];
  const double q = r * fma(fma(fma(fma(r, 1.0 / 120.0, 1.0 / 24.0), r, 1.0 / 6.0), r, 0.5), r, 1.0);
  const double Ts = __hiloint2double(__double2hiint(T) + ((ki >> 6) << 20), __double2loint(T));
  return fma(Ts, q, Ts);
}

// Split a positive running product into mantissa in [1,2) and exponent count.
__device__ __forceinline__ void renorm(double& Pp, int& E) {
  const int hi = __double2hiint(Pp);
  const int e = (hi >> 20) - 1023;
  E += e;
  Pp = __hiloint2double(hi - (e << 20), __double2loint(Pp));
}

template <int K>
__host__ __device__ constexpr int ldx_of() {
  return K + (K & 1);
}

// ---------------------------------------------------------------------------
// Binary (C = 2): s = x~_t' theta with x~_t = (1 - 2 y_t) x_t; log p = -softplus(s).
template <int K, int PPT>
__global__ void __launch_bounds__(LL_THREADS, 2) k_loglik_bin(LLArgs a) {
  constexpr int LDX = ldx_of<K>();
  extern __shared__ __align__(16) double smem[];
  if (a.stop && *a.stop) return;
  double* sT = smem;
  double* sX = smem + 64;
  const int c0 = a.t0 + blockIdx.y * a.chunk;
  const int c1 = min(c0 + a.chunk, a.t1);
  const int nobs = max(c1 - c0, 0);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sT[i] = c_exp2tab[i];
  {
    const double2* src = reinterpret_cast<const double2*>(a.X + (int64_t)c0 * LDX);
    double2* dst = reinterpret_cast<double2*>(sX);
    const int nv = nobs * LDX / 2;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) dst[i] = __ldg(src + i);
  }
  double th[PPT][K];
  const int64_t pbase = (int64_t)blockIdx.x * (LL_THREADS * PPT) + threadIdx.x;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t p = pbase + (int64_t)j * LL_THREADS;
    const double* row = a.theta + (p < a.P ? p : 0) * a.ldt;
#pragma unroll
    for (int i = 0; i < K; ++i) th[j][i] = (p < a.P && i < a.k) ? __ldg(row + i) : 0.0;
  }
  __syncthreads();
  double M[PPT], Pp[PPT];
  int E[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    M[j] = 0.0;
    Pp[j] = 1.0;
    E[j] = 0;
  }
  int t = 0;
  // two observations per iteration: 2 PPT independent FMA chains per thread
  for (; t + 2 <= nobs; t += 2) {
    const double2* x0 = reinterpret_cast<const double2*>(sX + t * LDX);
    const double2* x1 = reinterpret_cast<const double2*>(sX + (t + 1) * LDX);
    double s0[PPT], s1[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) s0[j] = s1[j] = 0.0;
#pragma unroll
    for (int i2 = 0; i2 < LDX / 2; ++i2) {
      const double2 u = x0[i2], v = x1[i2];
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        s0[j] = fma(th[j][2 * i2], u.x, s0[j]);
        s1[j] = fma(th[j][2 * i2], v.x, s1[j]);
        if (2 * i2 + 1 < K) {
          s0[j] = fma(th[j][2 * i2 + 1], u.y, s0[j]);
          s1[j] = fma(th[j][2 * i2 + 1], v.y, s1[j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      M[j] += relu_bits(s0[j]) + relu_bits(s1[j]);
      const double e0 = exp_neg(abs_clamp708(s0[j]), sT), e1 = exp_neg(abs_clamp708(s1[j]), sT);
      Pp[j] *= (1.0 + e0) * (1.0 + e1);
    }
    if ((t & 63) == 62) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) renorm(Pp[j], E[j]);
    }
  }
  for (; t < nobs; ++t) {
    const double2* x0 = reinterpret_cast<const double2*>(sX + t * LDX);
    double s0[PPT];
#pragma unroll
    for (int j = 0; j < PPT; ++j) s0[j] = 0.0;
#pragma unroll
    for (int i2 = 0; i2 < LDX / 2; ++i2) {
      const double2 u = x0[i2];
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        s0[j] = fma(th[j][2 * i2], u.x, s0[j]);
        if (2 * i2 + 1 < K) s0[j] = fma(th[j][2 * i2 + 1], u.y, s0[j]);
      }
    }
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      M[j] += relu_bits(s0[j]);
      Pp[j] *= 1.0 + exp_neg(abs_clamp708(s0[j]), sT);
    }
  }
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t p = pbase + (int64_t)j * LL_THREADS;
    if (p < a.P) {
      renorm(Pp[j], E[j]);
      const double L = -(M[j] + (log(Pp[j]) + (double)E[j] * 0x1.62e42fefa39efp-1));
      a.part[(int64_t)blockIdx.y * a.P + p] = L;
    }
  }
}

// ---------------------------------------------------------------------------
// Multinomial (C = CM1 + 1 >= 3): eta_0 = 0, eta_c = theta_c' x_t;
// log p = (eta_y - m) - log(sum_c e^(eta_c - m)), m = max_c eta_c.
template <int K, int CM1, int PPT>
__global__ void __launch_bounds__(LL_THREADS, 2) k_loglik_mnl(LLArgs a) {
  constexpr int LDX = ldx_of<K>();
  extern __shared__ __align__(16) double smem[];
  if (a.stop && *a.stop) return;
  double* sT = smem;
  double* sX = smem + 64;
  const int c0 = a.t0 + blockIdx.y * a.chunk;
  const int c1 = min(c0 + a.chunk, a.t1);
  const int nobs = max(c1 - c0, 0);
  int* sY = reinterpret_cast<int*>(sX + (size_t)a.chunk * LDX);
  for (int i = threadIdx.x; i < 64; i += blockDim.x) sT[i] = c_exp2tab[i];
  {
    const double2* src = reinterpret_cast<const double2*>(a.X + (int64_t)c0 * LDX);
    double2* dst = reinterpret_cast<double2*>(sX);
    const int nv = nobs * LDX / 2;
    for (int i = threadIdx.x; i < nv; i += blockDim.x) dst[i] = __ldg(src + i);
    for (int i = threadIdx.x; i < nobs; i += blockDim.x) sY[i] = __ldg(a.y + c0 + i);
  }
  double th[PPT][CM1][K];
  const int64_t pbase = (int64_t)blockIdx.x * (LL_THREADS * PPT) + threadIdx.x;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t p = pbase + (int64_t)j * LL_THREADS;
    const double* row = a.theta + (p < a.P ? p : 0) * a.ldt;
#pragma unroll
    for (int c = 0; c < CM1; ++c)
#pragma unroll
      for (int i = 0; i < K; ++i) th[j][c][i] = (p < a.P && i < a.k) ? __ldg(row + c * a.k + i) : 0.0;
  }
  __syncthreads();
  double D[PPT], Pp[PPT];
  int E[PPT];
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    D[j] = 0.0;
    Pp[j] = 1.0;
    E[j] = 0;
  }
  for (int t = 0; t < nobs; ++t) {
    const double2* x0 = reinterpret_cast<const double2*>(sX + t * LDX);
    const int yt = sY[t];
    double eta[PPT][CM1];
#pragma unroll
    for (int j = 0; j < PPT; ++j)
#pragma unroll
      for (int c = 0; c < CM1; ++c) eta[j][c] = 0.0;
#pragma unroll
    for (int i2 = 0; i2 < LDX / 2; ++i2) {
      const double2 u = x0[i2];
#pragma unroll
      for (int j = 0; j < PPT; ++j)
#pragma unroll
        for (int c = 0; c < CM1; ++c) {
          eta[j][c] = fma(th[j][c][2 * i2], u.x, eta[j][c]);
          if (2 * i2 + 1 < K) eta[j][c] = fma(th[j][c][2 * i2 + 1], u.y, eta[j][c]);
        }
    }
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      double m = 0.0, ey = 0.0;
#pragma unroll
      for (int c = 0; c < CM1; ++c) {
        m = fmax(m, eta[j][c]);
        ey = (yt == c + 1) ? eta[j][c] : ey;
      }
      D[j] += m - ey;
      double v = exp_neg(abs_clamp708(m), sT);  // reference category, eta_0 = 0
#pragma unroll
      for (int c = 0; c < CM1; ++c) v += exp_neg(abs_clamp708(m - eta[j][c]), sT);
      Pp[j] *= v;
    }
    if ((t & 63) == 63) {
#pragma unroll
      for (int j = 0; j < PPT; ++j) renorm(Pp[j], E[j]);
    }
  }
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t p = pbase + (int64_t)j * LL_THREADS;
    if (p < a.P) {
      renorm(Pp[j], E[j]);
      const double L = -(D[j] + (log(Pp[j]) + (double)E[j] * 0x1.62e42fefa39efp-1));
      a.part[(int64_t)blockIdx.y * a.P + p] = L;
    }
  }
}

// Sum chunk partials in chunk order: out[p] = sum_c part[c][p].
__global__ void k_sum_chunks(const double* __restrict__ part, int nchunks, int64_t P, double* __restrict__ out) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double s = part[p];
  for (int c = 1; c < nchunks; ++c) s += part[(int64_t)c * P + p];
  out[p] = s;
}

}  // namespace sps
