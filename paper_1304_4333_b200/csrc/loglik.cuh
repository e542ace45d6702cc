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
//    log p = eta_y - log(1 + sum_c e^eta_c) for C > 2 (max-shifted only when
//    some |eta_c| >= 704).  The logs are deferred: the factors (1 + e^-|s|)
//    in [1, 2] / 1 + sum_c e^eta_c are multiplied into a running product with
//    its exponent renormalized every 64 (binary) / every (C > 2) observation,
//    and ONE log per particle is taken at the end.  e^-a is
//    a table-driven exp (2^(i/64) table in smem, degree-5 polynomial on
//    |r| <= ln2/128, one-fma range reduction): 9 FP64 ops.  Binary total (DMMA kernel): 11 FP64
//    ops per pair + k FMAs (exp 9, Pp (1 + e) as one fma, + relu).
//  * Grid = particle tiles x observation chunks, chunk count chosen so the
//    block count fills whole waves of 148 SMs x resident blocks; chunk
//    partials are summed in fixed order by the consumer (deterministic).
#pragma once
#include "common.cuh"

namespace sps {

constexpr int LL_THREADS = 128;

// in global memory (read coalesced through L1/L2: a constant-bank read with 64 distinct addresses
// serializes per address)
__device__ const double c_exp2tab[64] = {
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

__device__ const double c_exp2tab256[256] = {
    0x1.0000000000000p+0, 0x1.00b1afa5abcbfp+0, 0x1.0163da9fb3335p+0, 0x1.02168143b0281p+0,
    0x1.02c9a3e778061p+0, 0x1.037d42e11bbccp+0, 0x1.04315e86e7f85p+0, 0x1.04e5f72f654b1p+0,
    0x1.059b0d3158574p+0, 0x1.0650a0e3c1f89p+0, 0x1.0706b29ddf6dep+0, 0x1.07bd42b72a836p+0,
    0x1.0874518759bc8p+0, 0x1.092bdf66607e0p+0, 0x1.09e3ecac6f383p+0, 0x1.0a9c79b1f3919p+0,
    0x1.0b5586cf9890fp+0, 0x1.0c0f145e46c85p+0, 0x1.0cc922b7247f7p+0, 0x1.0d83b23395decp+0,
    0x1.0e3ec32d3d1a2p+0, 0x1.0efa55fdfa9c5p+0, 0x1.0fb66affed31bp+0, 0x1.1073028d7233ep+0,
    0x1.11301d0125b51p+0, 0x1.11edbab5e2ab6p+0, 0x1.12abdc06c31ccp+0, 0x1.136a814f204abp+0,
    0x1.1429aaea92de0p+0, 0x1.14e95934f312ep+0, 0x1.15a98c8a58e51p+0, 0x1.166a45471c3c2p+0,
    0x1.172b83c7d517bp+0, 0x1.17ed48695bbc0p+0, 0x1.18af9388c8deap+0, 0x1.1972658375d2fp+0,
    0x1.1a35beb6fcb75p+0, 0x1.1af99f8138a1cp+0, 0x1.1bbe084045cd4p+0, 0x1.1c82f95281c6bp+0,
    0x1.1d4873168b9aap+0, 0x1.1e0e75eb44027p+0, 0x1.1ed5022fcd91dp+0, 0x1.1f9c18438ce4dp+0,
    0x1.2063b88628cd6p+0, 0x1.212be3578a819p+0, 0x1.21f49917ddc96p+0, 0x1.22bdda27912d1p+0,
    0x1.2387a6e756238p+0, 0x1.2451ffb82140ap+0, 0x1.251ce4fb2a63fp+0, 0x1.25e85711ece75p+0,
    0x1.26b4565e27cddp+0, 0x1.2780e341ddf29p+0, 0x1.284dfe1f56381p+0, 0x1.291ba7591bb70p+0,
    0x1.29e9df51fdee1p+0, 0x1.2ab8a66d10f13p+0, 0x1.2b87fd0dad990p+0, 0x1.2c57e39771b2fp+0,
    0x1.2d285a6e4030bp+0, 0x1.2df961f641589p+0, 0x1.2ecafa93e2f56p+0, 0x1.2f9d24abd886bp+0,
    0x1.306fe0a31b715p+0, 0x1.31432edeeb2fdp+0, 0x1.32170fc4cd831p+0, 0x1.32eb83ba8ea32p+0,
    0x1.33c08b26416ffp+0, 0x1.3496266e3fa2dp+0, 0x1.356c55f929ff1p+0, 0x1.36431a2de883bp+0,
    0x1.371a7373aa9cbp+0, 0x1.37f26231e754ap+0, 0x1.38cae6d05d866p+0, 0x1.39a401b7140efp+0,
    0x1.3a7db34e59ff7p+0, 0x1.3b57fbfec6cf4p+0, 0x1.3c32dc313a8e5p+0, 0x1.3d0e544ede173p+0,
    0x1.3dea64c123422p+0, 0x1.3ec70df1c5175p+0, 0x1.3fa4504ac801cp+0, 0x1.40822c367a024p+0,
    0x1.4160a21f72e2ap+0, 0x1.423fb2709468ap+0, 0x1.431f5d950a897p+0, 0x1.43ffa3f84b9d4p+0,
    0x1.44e086061892dp+0, 0x1.45c2042a7d232p+0, 0x1.46a41ed1d0057p+0, 0x1.4786d668b3237p+0,
    0x1.486a2b5c13cd0p+0, 0x1.494e1e192aed2p+0, 0x1.4a32af0d7d3dep+0, 0x1.4b17dea6db7d7p+0,
    0x1.4bfdad5362a27p+0, 0x1.4ce41b817c114p+0, 0x1.4dcb299fddd0dp+0, 0x1.4eb2d81d8abffp+0,
    0x1.4f9b2769d2ca7p+0, 0x1.508417f4531eep+0, 0x1.516daa2cf6642p+0, 0x1.5257de83f4eefp+0,
    0x1.5342b569d4f82p+0, 0x1.542e2f4f6ad27p+0, 0x1.551a4ca5d920fp+0, 0x1.56070dde910d2p+0,
    0x1.56f4736b527dap+0, 0x1.57e27dbe2c4cfp+0, 0x1.58d12d497c7fdp+0, 0x1.59c0827ff07ccp+0,
    0x1.5ab07dd485429p+0, 0x1.5ba11fba87a03p+0, 0x1.5c9268a5946b7p+0, 0x1.5d84590998b93p+0,
    0x1.5e76f15ad2148p+0, 0x1.5f6a320dceb71p+0, 0x1.605e1b976dc09p+0, 0x1.6152ae6cdf6f4p+0,
    0x1.6247eb03a5585p+0, 0x1.633dd1d1929fdp+0, 0x1.6434634ccc320p+0, 0x1.652b9febc8fb7p+0,
    0x1.6623882552225p+0, 0x1.671c1c70833f6p+0, 0x1.68155d44ca973p+0, 0x1.690f4b19e9538p+0,
    0x1.6a09e667f3bcdp+0, 0x1.6b052fa75173ep+0, 0x1.6c012750bdabfp+0, 0x1.6cfdcddd47645p+0,
    0x1.6dfb23c651a2fp+0, 0x1.6ef9298593ae5p+0, 0x1.6ff7df9519484p+0, 0x1.70f7466f42e87p+0,
    0x1.71f75e8ec5f74p+0, 0x1.72f8286ead08ap+0, 0x1.73f9a48a58174p+0, 0x1.74fbd35d7cbfdp+0,
    0x1.75feb564267c9p+0, 0x1.77024b1ab6e09p+0, 0x1.780694fde5d3fp+0, 0x1.790b938ac1cf6p+0,
    0x1.7a11473eb0187p+0, 0x1.7b17b0976cfdbp+0, 0x1.7c1ed0130c132p+0, 0x1.7d26a62ff86f0p+0,
    0x1.7e2f336cf4e62p+0, 0x1.7f3878491c491p+0, 0x1.80427543e1a12p+0, 0x1.814d2add106d9p+0,
    0x1.82589994cce13p+0, 0x1.8364c1eb941f7p+0, 0x1.8471a4623c7adp+0, 0x1.857f4179f5b21p+0,
    0x1.868d99b4492edp+0, 0x1.879cad931a436p+0, 0x1.88ac7d98a6699p+0, 0x1.89bd0a478580fp+0,
    0x1.8ace5422aa0dbp+0, 0x1.8be05bad61778p+0, 0x1.8cf3216b5448cp+0, 0x1.8e06a5e0866d9p+0,
    0x1.8f1ae99157736p+0, 0x1.902fed0282c8ap+0, 0x1.9145b0b91ffc6p+0, 0x1.925c353aa2fe2p+0,
    0x1.93737b0cdc5e5p+0, 0x1.948b82b5f98e5p+0, 0x1.95a44cbc8520fp+0, 0x1.96bdd9a7670b3p+0,
    0x1.97d829fde4e50p+0, 0x1.98f33e47a22a2p+0, 0x1.9a0f170ca07bap+0, 0x1.9b2bb4d53fe0dp+0,
    0x1.9c49182a3f090p+0, 0x1.9d674194bb8d5p+0, 0x1.9e86319e32323p+0, 0x1.9fa5e8d07f29ep+0,
    0x1.a0c667b5de565p+0, 0x1.a1e7aed8eb8bbp+0, 0x1.a309bec4a2d33p+0, 0x1.a42c980460ad8p+0,
    0x1.a5503b23e255dp+0, 0x1.a674a8af46052p+0, 0x1.a799e1330b358p+0, 0x1.a8bfe53c12e59p+0,
    0x1.a9e6b5579fdbfp+0, 0x1.ab0e521356ebap+0, 0x1.ac36bbfd3f37ap+0, 0x1.ad5ff3a3c2774p+0,
    0x1.ae89f995ad3adp+0, 0x1.afb4ce622f2ffp+0, 0x1.b0e07298db666p+0, 0x1.b20ce6c9a8952p+0,
    0x1.b33a2b84f15fbp+0, 0x1.b468415b749b1p+0, 0x1.b59728de5593ap+0, 0x1.b6c6e29f1c52ap+0,
    0x1.b7f76f2fb5e47p+0, 0x1.b928cf22749e4p+0, 0x1.ba5b030a1064ap+0, 0x1.bb8e0b79a6f1fp+0,
    0x1.bcc1e904bc1d2p+0, 0x1.bdf69c3f3a207p+0, 0x1.bf2c25bd71e09p+0, 0x1.c06286141b33dp+0,
    0x1.c199bdd85529cp+0, 0x1.c2d1cd9fa652cp+0, 0x1.c40ab5fffd07ap+0, 0x1.c544778fafb22p+0,
    0x1.c67f12e57d14bp+0, 0x1.c7ba88988c933p+0, 0x1.c8f6d9406e7b5p+0, 0x1.ca3405751c4dbp+0,
    0x1.cb720dcef9069p+0, 0x1.ccb0f2e6d1675p+0, 0x1.cdf0b555dc3fap+0, 0x1.cf3155b5bab74p+0,
    0x1.d072d4a07897cp+0, 0x1.d1b532b08c968p+0, 0x1.d2f87080d89f2p+0, 0x1.d43c8eacaa1d6p+0,
    0x1.d5818dcfba487p+0, 0x1.d6c76e862e6d3p+0, 0x1.d80e316c98398p+0, 0x1.d955d71ff6075p+0,
    0x1.da9e603db3285p+0, 0x1.dbe7cd63a8315p+0, 0x1.dd321f301b460p+0, 0x1.de7d5641c0658p+0,
    0x1.dfc97337b9b5fp+0, 0x1.e11676b197d17p+0, 0x1.e264614f5a129p+0, 0x1.e3b333b16ee12p+0,
    0x1.e502ee78b3ff6p+0, 0x1.e653924676d76p+0, 0x1.e7a51fbc74c83p+0, 0x1.e8f7977cdb740p+0,
    0x1.ea4afa2a490dap+0, 0x1.eb9f4867cca6ep+0, 0x1.ecf482d8e67f1p+0, 0x1.ee4aaa2188510p+0,
    0x1.efa1bee615a27p+0, 0x1.f0f9c1cb6412ap+0, 0x1.f252b376bba97p+0, 0x1.f3ac948dd7274p+0,
    0x1.f50765b6e4540p+0, 0x1.f6632798844f8p+0, 0x1.f7bfdad9cbe14p+0, 0x1.f91d802243c89p+0,
    0x1.fa7c1819e90d8p+0, 0x1.fbdba3692d514p+0, 0x1.fd3c22b8f71f1p+0, 0x1.fe9d96b2a23d9p+0};

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
  int32_t sub;         // DMMA kernel: observations per shared-memory sub-chunk (0: whole chunk)
  int32_t tiles;       // DMMA kernel: particle tiles; items = tiles x chunks, item = tile + tiles * chunk
  int32_t nitems;      //   (grid tiles x chunks: one item per block; a persistent grid loops over items)
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

// One m8n8k4 fp64 tensor-core MMA (DMMA): {c0,c1} += A(8x4) B(4x8) fragment.
// Fragments (PTX ISA, mma.m8n8k4 .f64): a = A[lane/4][lane%4],
// b = B[lane%4][lane/4], c0/c1 = C[lane/4][2 (lane%4) + {0,1}].
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// e^-a for 0 <= a <= 708: table-driven, ~1 ulp.  sT = 2^(i/64).  Range reduction by ONE fma
// with ln2/64 rounded to double: its error (1.2e-18) times |k| <= 65600 perturbs r by < 8e-14
// only where e^-a < 1e-300; the absolute error it adds to e^-a is < 4e-17 for every a.
__device__ __forceinline__ double exp_neg(double a, const double* __restrict__ sT) {
  const double t = fma(a, -0x1.71547652b82fep+6, 0x1.8p52);  // MAGIC - round(a 64/ln2)
  const double kd = t - 0x1.8p52;                             // k = -round(a 64/ln2)
  const double r = fma(kd, -0x1.62e42fefa39efp-7, -a);        // r = -a - k ln2/64
  const int ki = __double2loint(t);
  const double T = sT[ki & 63];
  const double q = r * fma(fma(fma(fma(r, 1.0 / 120.0, 1.0 / 24.0), r, 1.0 / 6.0), r, 0.5), r, 1.0);
  const double Ts = __hiloint2double(__double2hiint(T) + ((ki >> 6) << 20), __double2loint(T));
  return fma(Ts, q, Ts);
}

// e^-a for 0 <= a <= 708 with the 2^(i/256) table (sT256 in smem): |r| <= ln2/512,
// degree-4 polynomial (truncation 4e-17): 8 FP64 ops.
__device__ __forceinline__ double exp_neg256(double a, const double* __restrict__ sT) {
  const double t = fma(a, -0x1.71547652b82fep+8, 0x1.8p52);  // MAGIC - round(a 256/ln2)
  const double kd = t - 0x1.8p52;
  const double r = fma(kd, -0x1.62e42fefa39efp-9, -a);  // one fma (see exp_neg)
  const int ki = __double2loint(t);
  const double T = sT[ki & 255];
  const double q = r * fma(fma(fma(r, 1.0 / 24.0, 1.0 / 6.0), r, 0.5), r, 1.0);
  const double Ts = __hiloint2double(__double2hiint(T) + ((ki >> 8) << 20), __double2loint(T));
  return fma(Ts, q, Ts);
}

template <int TAB>
__device__ __forceinline__ double exp_neg_tab(double a, const double* __restrict__ sT) {
  if constexpr (TAB == 256)
    return exp_neg256(a, sT);
  else
    return exp_neg(a, sT);
}

// Split a positive running product into mantissa in [1,2) and exponent count.
__device__ __forceinline__ void renorm(double& Pp, int& E) {
  const int hi = __double2hiint(Pp);
  const int e = (hi >> 20) - 1023;
  E += e;
  Pp = __hiloint2double(hi - (e << 20), __double2loint(Pp));
}

// Row stride of the kernel layout of X: k padded to a multiple of 4 (DMMA k-step).
template <int K>
__host__ __device__ constexpr int ldx_of() {
  return (K + 3) / 4 * 4;
}

// ---------------------------------------------------------------------------
// Binary (C = 2): s = x~_t' theta with x~_t = (1 - 2 y_t) x_t; log p = -softplus(s).
template <int K, int PPT>
__global__ void __launch_bounds__(LL_THREADS, 2) k_loglik_bin(LLArgs a) {
  constexpr int LDX = ldx_of<K>();
  extern __shared__ __align__(16) double smem[];
  if (a.stop && *a.stop) return;
  griddep_wait();  // launched with PDL: theta (the proposal kernel's output) after this
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
    for (int i2 = 0; i2 < (K + 1) / 2; ++i2) {
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
      Pp[j] = fma(Pp[j], e0, Pp[j]);  // Pp (1 + e): one FP64 op instead of an add and a multiply
      Pp[j] = fma(Pp[j], e1, Pp[j]);
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
    for (int i2 = 0; i2 < (K + 1) / 2; ++i2) {
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
      const double e0 = exp_neg(abs_clamp708(s0[j]), sT);
      Pp[j] = fma(Pp[j], e0, Pp[j]);
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
// TAB: exp table 2^(j/64) (9-op exp) or 2^(j/256) (8-op exp; the host reserves 256 doubles).
template <int K, int CM1, int PPT, int TAB = 64, int MINB = 2>
__global__ void __launch_bounds__(LL_THREADS, MINB) k_loglik_mnl(LLArgs a) {
  constexpr int LDX = ldx_of<K>();
  extern __shared__ __align__(16) double smem[];
  if (a.stop && *a.stop) return;
  griddep_wait();  // launched with PDL: theta (the proposal kernel's output) after this
  double* sT = smem;
  double* sX = smem + TAB;
  const int c0 = a.t0 + blockIdx.y * a.chunk;
  const int c1 = min(c0 + a.chunk, a.t1);
  const int nobs = max(c1 - c0, 0);
  int* sY = reinterpret_cast<int*>(sX + (size_t)a.chunk * LDX);
  for (int i = threadIdx.x; i < TAB; i += blockDim.x) sT[i] = TAB == 256 ? c_exp2tab256[i] : c_exp2tab[i];
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
    for (int i2 = 0; i2 < (K + 1) / 2; ++i2) {
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
      // Unshifted form 1 + sum_c e^eta_c (the reference term is e^0 = 1): C-1 exps, no max.
      // Exact as long as every |eta_c| < 704 (no overflow; v < 2^1019); otherwise the
      // max-shifted form below (never taken for the prior / posterior scales of the configs).
      double ey = 0.0, v = 1.0;
      int big = 0;
#pragma unroll
      for (int c = 0; c < CM1; ++c) {
        ey = (yt == c + 1) ? eta[j][c] : ey;
        big |= (__double2hiint(eta[j][c]) & 0x7fffffff) >= 0x40860000;  // |eta| >= 704, inf, nan
        v += exp_neg_tab<TAB>(-eta[j][c], sT);
      }
      D[j] -= ey;
      if (big) {
        double m = 0.0;
#pragma unroll
        for (int c = 0; c < CM1; ++c) m = fmax(m, eta[j][c]);
        v = exp_neg_tab<TAB>(abs_clamp708(m), sT);  // reference category, eta_0 = 0
#pragma unroll
        for (int c = 0; c < CM1; ++c) v += exp_neg_tab<TAB>(abs_clamp708(m - eta[j][c]), sT);
        D[j] += m;
      }
      Pp[j] *= v;
      renorm(Pp[j], E[j]);  // v can reach ~C e^704: keep Pp in [1, 2) every observation (ALU only)
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

// ---------------------------------------------------------------------------
// Binary, contraction on DMMA (mma.sync m8n8k4 f64): M = 8 observations, N =
// 8 particles, K = 4 covariates per instruction.  Warp w owns NTW x 8
// particles whose theta B-fragments (KKD k-steps) stay in registers; each
// 8-observation tile costs KKD shared loads (A fragments of X) + KKD*NTW
// DMMAs, i.e. ~0.2 issue slots per pair for the contraction (the DFMA form
// needs ~31: 25 DFMA + 6 LDS), leaving the issue bandwidth to the epilogue.
// k = 4 KKD + REM: the last REM (<= 2) covariates are DFMAs on the C
// fragment instead of a zero-padded DMMA step (k = 25: 25 FMAs, not 28).
// Lane l holds C[obs = l/4][particle = 2 (l%4) + e] of every n-tile; two
// observation tiles are folded into each product update; per-lane running
// sums are combined over the 8 lanes of a particle column at the end.

// H: 8-observation tiles folded into one product update (1 or 2); TAB: exp table size (64 or 256);
// KS: independent DMMA accumulator chains over k (1 or 2); MINB: min resident blocks (register budget).
template <int KKD, int REM, int NTW, int H = 1, int TAB = 64, int KS = 1, int MINB = 1>
__global__ void __launch_bounds__(128, MINB) k_loglik_bin_mma(LLArgs a) {
  constexpr int KP = 4 * KKD + (REM ? 4 : 0);  // X row stride (k padded to 4)
  extern __shared__ __align__(16) double smem[];
  double* sT = smem;        // TAB
  double* sX = smem + 256;  // 2 x (sub rounded up to 16) x KP
  double tv[TAB / 128 > 0 ? TAB / 128 : 1];  // exp table: loads in flight with the stop-flag load
#pragma unroll
  for (int u = 0; u < (TAB + 127) / 128; ++u) {
    const int i = threadIdx.x + 128 * u;
    tv[u] = i < TAB ? __ldg(TAB == 256 ? c_exp2tab256 + i : c_exp2tab + i) : 0.0;
  }
  if (a.stop && *a.stop) return;
  tl_start(2);
  tl_max(24);  // latest block start (the last wave)
#pragma unroll
  for (int u = 0; u < (TAB + 127) / 128; ++u) {
    const int i = threadIdx.x + 128 * u;
    if (i < TAB) sT[i] = tv[u];
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  const int sub0 = a.sub;  // X sub-chunk rows per shared buffer (0: the whole chunk)
  __shared__ __align__(8) uint64_t xbar[2];
  if (threadIdx.x == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
  }
  __syncthreads();
  griddep_wait();  // theta* (the proposal kernel's output) from here on
  tl_mark(25);     // block (0,0): dependency released
  int it = 0;            // sub-chunk loads issued so far (mbarrier phases)
  int held_chunk = -1;   // chunk whose single sub-chunk is resident in buffer held_buf
  int held_buf = 0;
  const int stride = gridDim.x * gridDim.y;
  for (int item = blockIdx.x + gridDim.x * blockIdx.y; item < a.nitems; item += stride) {
  const int tile = item % a.tiles, cy = item / a.tiles;
  const int c0 = a.t0 + cy * a.chunk;
  const int c1 = min(c0 + a.chunk, a.t1);
  const int ntot = max(c1 - c0, 0);
  const int sub = sub0 > 0 ? sub0 : ntot;
  const int SR = (sub + 15) & ~15;
  const int64_t pw = ((int64_t)tile * 4 + w) * (NTW * 8);  // first particle of this warp
  auto issue = [&](int cs, int buf) {
    const unsigned bytes = (unsigned)(min(sub, ntot - cs) * KP * 8);
    mbar_arrive_expect_tx(&xbar[buf], bytes);
    bulk_g2s(sX + buf * SR * KP, a.X + (int64_t)(c0 + cs) * KP, bytes, &xbar[buf]);
  };
  // one sub-chunk: reuse it while consecutive items share the chunk (persistent grid)
  const bool single = ntot <= sub;
  const bool reuse = single && cy == held_chunk;
  if (!reuse && threadIdx.x == 0 && ntot > 0) issue(0, it & 1);
  double b[NTW][KKD > 0 ? KKD : 1];
  double tr[NTW][2][REM > 0 ? REM : 1];  // remainder covariates of this lane's 2 particles per n-tile
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt) {
    const int64_t p = pw + nt * 8 + ar;
    const double* row = a.theta + (p < a.P ? p : 0) * a.ldt;
#pragma unroll
    for (int kk = 0; kk < KKD; ++kk) {
      const int k = kk * 4 + ac;
      b[nt][kk] = (p < a.P && k < a.k) ? __ldg(row + k) : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t q = pw + nt * 8 + 2 * ac + e;
      const double* rq = a.theta + (q < a.P ? q : 0) * a.ldt;
#pragma unroll
      for (int r = 0; r < REM; ++r) tr[nt][e][r] = q < a.P ? __ldg(rq + 4 * KKD + r) : 0.0;
    }
  }
  __syncthreads();
  if (g_tl) {  // block (0,0): theta fragments loaded (a move of the last-loaded value waits on its scoreboard)
    unsigned long long dep;
    asm volatile("mov.b64 %0, %1;" : "=l"(dep) : "d"(b[NTW - 1][KKD > 0 ? KKD - 1 : 0] + tr[NTW - 1][1][0]) : "memory");
    if (dep != 1ull) tl_mark(26);
    else tl_mark(26);
  }
  double M[NTW][2], Pp[NTW][2];
  int E[NTW][2];
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      M[nt][e] = 0.0;
      Pp[nt][e] = 1.0;
      E[nt][e] = 0;
    }
  int nit = 0;
  // X sub-chunks (sub rows, a multiple of 16) stream through two shared-memory buffers by TMA bulk
  // copies: the next one loads while this one computes.  Rows past a sub-chunk's end hold stale
  // data; their products are masked out below (the per-thread load/store staging these copies
  // replace was ~28% of the stall samples, ncu r01_pa2).
  for (int cs = 0; cs < ntot; cs += sub) {
  const int nobs = min(sub, ntot - cs);
  int buf;
  if (reuse) {
    buf = held_buf;
  } else {
    buf = it & 1;
    if (threadIdx.x == 0 && cs + sub < ntot) issue(cs + sub, buf ^ 1);  // buf ^ 1 released by the barrier below
    mbar_wait(&xbar[buf], (unsigned)(it >> 1) & 1u);
    ++it;
    held_chunk = single ? cy : -1;
    held_buf = buf;
  }
  const double* sXb = sX + buf * SR * KP;
  for (int t0 = 0; t0 < nobs; t0 += 8 * H) {
    double acc[H][NTW][2];
#pragma unroll
    for (int h = 0; h < H; ++h)
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) acc[h][nt][0] = acc[h][nt][1] = 0.0;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const double* xr = sXb + (t0 + 8 * h + ar) * KP;
      if (KS == 2 && KKD >= 2) {
        double acc2[NTW][2];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) acc2[nt][0] = acc2[nt][1] = 0.0;
#pragma unroll
        for (int kk = 0; kk < KKD; ++kk) {
          const double av = xr[kk * 4 + ac];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) {
            if (kk & 1)
              dmma884(acc2[nt][0], acc2[nt][1], av, b[nt][kk]);
            else
              dmma884(acc[h][nt][0], acc[h][nt][1], av, b[nt][kk]);
          }
        }
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) {
          acc[h][nt][0] += acc2[nt][0];
          acc[h][nt][1] += acc2[nt][1];
        }
      } else {
#pragma unroll
        for (int kk = 0; kk < KKD; ++kk) {
          const double av = xr[kk * 4 + ac];
#pragma unroll
          for (int nt = 0; nt < NTW; ++nt) dmma884(acc[h][nt][0], acc[h][nt][1], av, b[nt][kk]);
        }
      }
#pragma unroll
      for (int r = 0; r < REM; ++r) {
        const double xv = xr[4 * KKD + r];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt) {
          acc[h][nt][0] = fma(xv, tr[nt][0][r], acc[h][nt][0]);
          acc[h][nt][1] = fma(xv, tr[nt][1][r], acc[h][nt][1]);
        }
      }
    }
    // padded observations (beyond the chunk) contribute s = -inf: relu 0, e^-|s| = 0
    if (H == 1) {
      if (t0 + ar < nobs) {
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            M[nt][e] += relu_bits(acc[0][nt][e]);
            const double ex = exp_neg_tab<TAB>(abs_clamp708(acc[0][nt][e]), sT);
            Pp[nt][e] = fma(Pp[nt][e], ex, Pp[nt][e]);  // Pp (1 + e) in one FP64 op (11 per pair)
          }
      }
    } else {
      const bool v0 = t0 + ar < nobs, v1 = t0 + 8 + ar < nobs;
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const double s0 = v0 ? acc[0][nt][e] : -1e300, s1 = v1 ? acc[H - 1][nt][e] : -1e300;
          M[nt][e] += relu_bits(s0) + relu_bits(s1);
          const double e0 = exp_neg_tab<TAB>(abs_clamp708(s0), sT), e1 = exp_neg_tab<TAB>(abs_clamp708(s1), sT);
          Pp[nt][e] = fma(Pp[nt][e], e0, Pp[nt][e]);
          Pp[nt][e] = fma(Pp[nt][e], e1, Pp[nt][e]);
        }
    }
    if ((++nit & 31) == 0) {
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt) {
        renorm(Pp[nt][0], E[nt][0]);
        renorm(Pp[nt][1], E[nt][1]);
      }
    }
  }
  __syncthreads();  // every warp is done with buffer `buf` before it is refilled
  }  // sub-chunks
  // combine the 8 lanes (ar = 0..7) of each particle column: sums of M and E, product of P.
  // Reduce-scatter over the lane bits of ar (offsets 4, 8, 16): each round halves the values a
  // lane carries until one is left (then butterfly), so the 2 NTW particles of a column end on
  // different lanes and each lane takes at most one log (not 2 NTW in turn).
  {
    constexpr int V = 2 * NTW;
    double m[V], pp[V];
    int ex[V];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        renorm(Pp[nt][e], E[nt][e]);
        m[nt * 2 + e] = M[nt][e];
        pp[nt * 2 + e] = Pp[nt][e];
        ex[nt * 2 + e] = E[nt][e];
      }
    int jsel = 0;  // index (nt * 2 + e) of the value this lane keeps
    int cnt = V;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int o = 4 << r;
      const int bit = (ar >> r) & 1;
      if (cnt > 1) {  // keep half (upper if bit), add the partner's copy of it
        const int h = cnt / 2;
#pragma unroll
        for (int q = 0; q < V / 2; ++q) {
          if (q < h) {
            const double sm = bit ? m[q] : m[q + h], sp = bit ? pp[q] : pp[q + h];
            const int se = bit ? ex[q] : ex[q + h];
            const double km = bit ? m[q + h] : m[q], kp = bit ? pp[q + h] : pp[q];
            const int ke = bit ? ex[q + h] : ex[q];
            m[q] = km + __shfl_xor_sync(0xffffffffu, sm, o);
            pp[q] = kp * __shfl_xor_sync(0xffffffffu, sp, o);  // 8 factors in [1,2): < 2^8
            ex[q] = ke + __shfl_xor_sync(0xffffffffu, se, o);
          }
        }
        jsel += bit * h;
        cnt = h;
      } else {
        m[0] += __shfl_xor_sync(0xffffffffu, m[0], o);
        pp[0] *= __shfl_xor_sync(0xffffffffu, pp[0], o);
        ex[0] += __shfl_xor_sync(0xffffffffu, ex[0], o);
      }
    }
    // lanes whose remaining ar bits are 0 hold a distinct (nt, e) each
    const int rest = ar >> (V == 8 ? 3 : V == 4 ? 2 : 1);
    const int64_t p = pw + (jsel >> 1) * 8 + 2 * ac + (jsel & 1);
    if (rest == 0 && p < a.P) {
      double pv = pp[0];
      int xv = ex[0];
      renorm(pv, xv);
      a.part[(int64_t)cy * a.P + p] = -(m[0] + (log(pv) + (double)xv * 0x1.62e42fefa39efp-1));
    }
  }
  }  // items
  tl_mark(27);  // block (0,0): done
  griddep_launch();
  tl_end(2);
}

// ---------------------------------------------------------------------------
// Multinomial (C = CM1 + 1 >= 3), contraction on DMMA (mma.sync m8n8k4 f64): each warp owns
// NTW x 8 particles; class c = 1..C-1 of those particles is its own n-tile (B = theta_c
// fragments in registers), so one A fragment of X (8 observations x 4 covariates, from shared
// memory) feeds NTW x CM1 DMMAs and lane (ar, ac) ends with eta_c of observation ar and
// particles 2 ac, 2 ac + 1 of every n-tile, for all classes at once.  k = 4 KKD + REM: the
// last REM (<= 2) covariates are DFMAs on the accumulators (as in the binary kernel).
// Epilogue per (observation, particle): log p = eta_y - log(1 + sum_c e^eta_c), the logs deferred
// into a running product (renormalised every observation: 1 + sum e^eta can reach C e^704), the
// max-shifted form only when some |eta_c| >= 704 (R17).  X streams through two shared-memory
// sub-chunk buffers by TMA bulk copies; the labels of a sub-chunk ride along in a small array.
template <int KKD, int REM, int CM1, int NTW = 2, int MINB = 4>
__global__ void __launch_bounds__(128, MINB) k_loglik_mnl_mma(LLArgs a) {
  constexpr int KP = 4 * KKD + (REM ? 4 : 0);
  extern __shared__ __align__(16) double smem[];
  double* sT = smem;        // 64: exp table 2^(i/64) (256 reserved)
  double* sX = smem + 256;  // 2 x SR x KP
  __shared__ int sY[2][64];
  __shared__ __align__(8) uint64_t xbar[2];
  const double tv = threadIdx.x < 64 ? __ldg(c_exp2tab + threadIdx.x) : 0.0;
  if (a.stop && *a.stop) return;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  const int tile = blockIdx.x, cy = blockIdx.y;
  const int c0 = a.t0 + cy * a.chunk;
  const int c1 = min(c0 + a.chunk, a.t1);
  const int ntot = max(c1 - c0, 0);
  const int sub = a.sub > 0 ? a.sub : ntot;
  const int SR = (sub + 15) & ~15;
  if (threadIdx.x < 64) sT[threadIdx.x] = tv;
  if (threadIdx.x == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
  }
  auto issue = [&](int cs, int buf) {
    const unsigned bytes = (unsigned)(min(sub, ntot - cs) * KP * 8);
    mbar_arrive_expect_tx(&xbar[buf], bytes);
    bulk_g2s(sX + buf * SR * KP, a.X + (int64_t)(c0 + cs) * KP, bytes, &xbar[buf]);
  };
  if (threadIdx.x < 64 && threadIdx.x < ntot && threadIdx.x < sub) sY[0][threadIdx.x] = __ldg(a.y + c0 + threadIdx.x);
  __syncthreads();
  if (threadIdx.x == 0 && ntot > 0) issue(0, 0);  // X does not depend on the predecessor
  griddep_wait();  // theta (the proposal kernel's output) from here on
  const int64_t pw = ((int64_t)tile * 4 + w) * (NTW * 8);
  double b[NTW][CM1][KKD > 0 ? KKD : 1];
  double tr[NTW][CM1][2][REM > 0 ? REM : 1];
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt) {
    const int64_t p = pw + nt * 8 + ar;
    const double* row = a.theta + (p < a.P ? p : 0) * a.ldt;
#pragma unroll
    for (int c = 0; c < CM1; ++c)
#pragma unroll
      for (int kk = 0; kk < KKD; ++kk) {
        const int k = kk * 4 + ac;
        b[nt][c][kk] = (p < a.P && k < a.k) ? __ldg(row + c * a.k + k) : 0.0;
      }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t q = pw + nt * 8 + 2 * ac + e;
      const double* rq = a.theta + (q < a.P ? q : 0) * a.ldt;
#pragma unroll
      for (int c = 0; c < CM1; ++c)
#pragma unroll
        for (int r = 0; r < REM; ++r) tr[nt][c][e][r] = q < a.P ? __ldg(rq + c * a.k + 4 * KKD + r) : 0.0;
    }
  }
  double D[NTW][2], Pp[NTW][2];
  int E[NTW][2];
#pragma unroll
  for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      D[nt][e] = 0.0;
      Pp[nt][e] = 1.0;
      E[nt][e] = 0;
    }
  int it = 0;
  for (int cs = 0; cs < ntot; cs += sub) {
    const int nobs = min(sub, ntot - cs);
    const int buf = it & 1;
    if (cs + sub < ntot) {
      if (threadIdx.x == 0) issue(cs + sub, buf ^ 1);  // buf ^ 1 released by the barrier below
      const int nn = min(sub, ntot - cs - sub);
      if (threadIdx.x < nn) sY[buf ^ 1][threadIdx.x] = __ldg(a.y + c0 + cs + sub + threadIdx.x);
    }
    mbar_wait(&xbar[buf], (unsigned)(it >> 1) & 1u);
    ++it;
    const double* sXb = sX + buf * SR * KP;
    for (int t0 = 0; t0 < nobs; t0 += 8) {
      double acc[NTW][CM1][2];
#pragma unroll
      for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
        for (int c = 0; c < CM1; ++c) acc[nt][c][0] = acc[nt][c][1] = 0.0;
      const double* xr = sXb + (t0 + ar) * KP;
#pragma unroll
      for (int kk = 0; kk < KKD; ++kk) {
        const double av = xr[kk * 4 + ac];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
          for (int c = 0; c < CM1; ++c) dmma884(acc[nt][c][0], acc[nt][c][1], av, b[nt][c][kk]);
      }
#pragma unroll
      for (int r = 0; r < REM; ++r) {
        const double xv = xr[4 * KKD + r];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
          for (int c = 0; c < CM1; ++c) {
            acc[nt][c][0] = fma(xv, tr[nt][c][0][r], acc[nt][c][0]);
            acc[nt][c][1] = fma(xv, tr[nt][c][1][r], acc[nt][c][1]);
          }
      }
      if (t0 + ar < nobs) {  // rows past the sub-chunk hold stale data
        const int yt = sY[buf][t0 + ar];
#pragma unroll
        for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            // unshifted 1 + sum_c e^eta_c (reference class: e^0 = 1), C - 1 exps, no max
            double ey = 0.0, v = 1.0;
            int big = 0;
#pragma unroll
            for (int c = 0; c < CM1; ++c) {
              const double eta = acc[nt][c][e];
              ey = (yt == c + 1) ? eta : ey;
              big |= (__double2hiint(eta) & 0x7fffffff) >= 0x40860000;  // |eta| >= 704, inf, nan
              v += exp_neg(-eta, sT);
            }
            D[nt][e] -= ey;
            if (big) {
              double m = 0.0;
#pragma unroll
              for (int c = 0; c < CM1; ++c) m = fmax(m, acc[nt][c][e]);
              v = exp_neg(abs_clamp708(m), sT);
#pragma unroll
              for (int c = 0; c < CM1; ++c) v += exp_neg(abs_clamp708(m - acc[nt][c][e]), sT);
              D[nt][e] += m;
            }
            Pp[nt][e] *= v;
            renorm(Pp[nt][e], E[nt][e]);
          }
      }
    }
    __syncthreads();  // every warp is done with buffer `buf` (and its labels) before they are refilled
  }
  {  // combine the 8 lanes of each particle column (the binary kernel's reduce-scatter)
    constexpr int V = 2 * NTW;
    double m[V], pp[V];
    int ex[V];
#pragma unroll
    for (int nt = 0; nt < NTW; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        renorm(Pp[nt][e], E[nt][e]);
        m[nt * 2 + e] = D[nt][e];
        pp[nt * 2 + e] = Pp[nt][e];
        ex[nt * 2 + e] = E[nt][e];
      }
    int jsel = 0, cnt = V;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      const int o = 4 << r;
      const int bit = (ar >> r) & 1;
      if (cnt > 1) {
        const int h = cnt / 2;
#pragma unroll
        for (int q = 0; q < V / 2; ++q) {
          if (q < h) {
            const double sm = bit ? m[q] : m[q + h], sp = bit ? pp[q] : pp[q + h];
            const int se = bit ? ex[q] : ex[q + h];
            const double km = bit ? m[q + h] : m[q], kp = bit ? pp[q + h] : pp[q];
            const int ke = bit ? ex[q + h] : ex[q];
            m[q] = km + __shfl_xor_sync(0xffffffffu, sm, o);
            pp[q] = kp * __shfl_xor_sync(0xffffffffu, sp, o);  // 8 factors in [1,2): < 2^8
            ex[q] = ke + __shfl_xor_sync(0xffffffffu, se, o);
          }
        }
        jsel += bit * h;
        cnt = h;
      } else {
        m[0] += __shfl_xor_sync(0xffffffffu, m[0], o);
        pp[0] *= __shfl_xor_sync(0xffffffffu, pp[0], o);
        ex[0] += __shfl_xor_sync(0xffffffffu, ex[0], o);
      }
    }
    const int rest = ar >> (V == 8 ? 3 : V == 4 ? 2 : 1);
    const int64_t p = pw + (jsel >> 1) * 8 + 2 * ac + (jsel & 1);
    if (rest == 0 && p < a.P) {
      double pv = pp[0];
      int xv = ex[0];
      renorm(pv, xv);
      a.part[(int64_t)cy * a.P + p] = -(m[0] + (log(pv) + (double)xv * 0x1.62e42fefa39efp-1));
    }
  }
  griddep_launch();
}

// Sum chunk partials in chunk order: out[p] = sum_c part[c][p].  bad (may be null):
// the smallest p whose sum is not finite (sps_loglik's error check).
__global__ void k_sum_chunks(const double* __restrict__ part, int nchunks, int64_t P, double* __restrict__ out,
                             int* bad = nullptr) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  double s = part[p];
  for (int c = 1; c < nchunks; ++c) s += part[(int64_t)c * P + p];
  out[p] = s;
  if (bad && !isfinite(s)) atomicMin(bad, (int)(p < 0x7ffffffe ? p : 0x7ffffffe));
}

// sps_loglik error path (the log-likelihood is finite for finite theta): if
// k_sum_chunks flagged particle *pending, find the first observation t in [t0, t1) whose term
// log P(y_t | x_t, theta_p) is not finite (eta_c = x_t' theta_c, max-shifted log-sum-exp as in
// K1's fallback branch, so a term is non-finite iff some eta_c is) and record (p, t) in the
// mapped host pair rec (first error sticks until sps_sync reports it); clears *pending.
__global__ void k_ll_locate(const double* __restrict__ theta, int ld, const double* __restrict__ X,
                            const int32_t* __restrict__ y, int k, int C, int t0, int t1, int* pending,
                            volatile int* rec) {
  __shared__ int tmin;
  const int p = *pending;
  if (p == 0x7fffffff) return;
  if (threadIdx.x == 0) tmin = 0x7fffffff;
  __syncthreads();
  const double* th = theta + (int64_t)p * ld;
  for (int t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
    const double* x = X + (int64_t)t * k;
    bool bad = false;
    double m = 0.0, ey = 0.0;
    for (int c = 1; c < C; ++c) {
      double e = 0.0;
      for (int i = 0; i < k; ++i) e = fma(x[i], th[(c - 1) * k + i], e);
      bad |= !isfinite(e);
      m = fmax(m, e);
      if (c == y[t]) ey = e;
    }
    double s = exp(-m);
    for (int c = 1; c < C; ++c) {
      double e = 0.0;
      for (int i = 0; i < k; ++i) e = fma(x[i], th[(c - 1) * k + i], e);
      s += exp(e - m);
    }
    const double term = ey - m - log(s);
    if (bad || !isfinite(term)) atomicMin(&tmin, t);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (rec[0] == 0x7fffffff) {
      rec[1] = tmin == 0x7fffffff ? -1 : tmin;
      __threadfence_system();
      rec[0] = p;
    }
    *pending = 0x7fffffff;
  }
}

}  // namespace sps
