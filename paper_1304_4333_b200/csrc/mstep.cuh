// mstep.cuh -- M phase kernels (Algorithm 2 step 2) and
// the prior draw, B200 layout: every per-particle stage is spread over all
// threads of a block (no long per-thread serial chains), every reduction is
// a fixed tree/order (deterministic), and kernels of a speculatively launched
// step return immediately once the device stop flag is set.
#pragma once
#include "common.cuh"
#include "kernels.cuh"
#include "loglik.cuh"

namespace sps {

// ---------------------------------------------------------------- K8 / K10
// theta* = base + Lz z (z: Box-Muller pairs of the stream (id = p0 + p, step,
// tag), R15) and lp* = -1/2 (theta* - mu)' Sinv (theta* - mu).  INIT: base =
// mu, Lz = Lprior (Algorithm 1 step 1); PROPOSAL: base =
// theta, Lz = chol(h V).
constexpr int PR_TILE = 64;  // particles per block (8 DMMA row tiles)
struct DrawArgs {
  const double* base;  // P x d, or nullptr -> mu
  const double* Lz;    // lower factor, padded NP x KP (NP = round_up(d, 8), KP = round_up(d, 4))
  const double* Sinv;  // prior precision, padded NP x KP
  const double* mu;
  const double* Z;  // P x 2 ceil(d/2) standard normals (k_normals)
  double* out;
  double* lp_out;
  Ctl* ctl;
  const int* stop;
  int64_t P, p0;
  int d;
};

// Standard normals of the streams (id = p0 + p, step, tag) for every local
// particle: Z[p][2 pr + {0,1}] = Box-Muller pair pr (R15).  One thread per
// (particle, pair).  Independent of the particle state, so the engine runs it
// one M step ahead on a side stream, overlapped with the latency-bound kernels.
// With `logu` (PROPOSAL streams), also plog of the step's ACCEPT uniform of each
// particle (R16), so the accept test on the critical path is one comparison.
__global__ void __launch_bounds__(256) k_normals(int64_t P, int64_t p0, int np, int ldz, uint64_t seed, uint32_t step,
                                                 uint32_t tag, uint32_t pass, double* __restrict__ Z,
                                                 double* __restrict__ logu) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= P * np) return;
  const int64_t p = t / np;
  const int pr = (int)(t - p * np);
  double z0, z1;
  normal_pair(seed, (uint32_t)pr, (uint32_t)(p0 + p), step, tag, pass, &z0, &z1);
  reinterpret_cast<double2*>(Z + p * ldz)[pr] = make_double2(z0, z1);
  if (logu && pr == 0) {
    const u4 w = stream_block(seed, 0u, (uint32_t)(p0 + p), step, TAG_ACCEPT, pass);
    logu[p] = plog(u01(w.x, w.y));
  }
}


__host__ __device__ constexpr int round_up(int x, int m) { return (x + m - 1) / m * m; }

// theta* = base + Z Lz' and lp* = -1/2 rowsum(Delta .* (Delta Sinv)), Delta =
// theta* - mu, for PR_TILE particles per block, both products on DMMA
// (K = d padded to 4, N = d padded to 8; padding is zero).  z precomputed by
// k_normals.  STAGE: Lz / Sinv staged in shared memory.
template <bool STAGE>
__global__ void __launch_bounds__(256) k_propose(DrawArgs a) {
  extern __shared__ double sm[];
  if (a.stop && *a.stop) return;
  const int d = a.d, np = (d + 1) / 2, d2 = 2 * np, KP = round_up(d, 4), NP = round_up(d, 8), NT = NP / 8;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* Zs = sm;                  // PR_TILE x KP
  double* Ds = Zs + PR_TILE * KP;   // PR_TILE x KP  (theta* - mu)
  double* qp = Ds + PR_TILE * KP;   // PR_TILE x NT  quad partials
  double* smu = qp + PR_TILE * NT;  // KP
  double* sL = smu + KP;                    // NP x KP (STAGE)
  double* sS = sL + NP * KP;                // NP x KP (STAGE)
  double* Bs = STAGE ? sS + NP * KP : sL;   // PR_TILE x d base rows (theta)
  // mu; Lz and Sinv arrive in the padded DMMA layout (NP x KP, zeros outside d x d) -> bulk copies
  for (int i = threadIdx.x; i < KP; i += blockDim.x) smu[i] = i < d ? a.mu[i] : 0.0;
  auto Lf = [&](int i, int j) -> double { return STAGE ? sL[i * KP + j] : __ldg(a.Lz + i * KP + j); };
  auto Sf = [&](int i, int j) -> double { return STAGE ? sS[i * KP + j] : __ldg(a.Sinv + i * KP + j); };
  const int MT = PR_TILE / 8, ntiles = MT * NT;
  const int ar = lane >> 2, ac = lane & 3;
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();
  const int64_t ntl = (a.P + PR_TILE - 1) / PR_TILE;
  unsigned phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntl; tile += gridDim.x) {
    const int64_t pb = tile * PR_TILE;
    const int cnt = (int)min((int64_t)PR_TILE, a.P - pb);
    __syncthreads();  // previous tile done with Zs / Ds / Bs / qp
    if (threadIdx.x == 0) {  // TMA bulk copies: Z tile (rows of KP, zero padded in memory), theta tile, Lz, Sinv
      const unsigned zb = (unsigned)(PR_TILE * KP * 8);
      const unsigned bb = a.base ? (unsigned)(round_up(cnt * d, 2) * 8) : 0u;
      const unsigned mb = (STAGE && phase == 0) ? (unsigned)(NP * KP * 8) : 0u;
      mbar_arrive_expect_tx(&bar, zb + bb + 2 * mb);
      bulk_g2s(Zs, a.Z + pb * KP, zb, &bar);
      if (a.base) bulk_g2s(Bs, a.base + pb * d, bb, &bar);
      if (mb) {
        bulk_g2s(sL, a.Lz, mb, &bar);
        bulk_g2s(sS, a.Sinv, mb, &bar);
      }
    }
    mbar_wait(&bar, phase);
    phase ^= 1u;
    __syncthreads();
    // theta* = base + Z L'  (C[p][i] = sum_j Z[p][j] L[i][j])
    for (int t = w; t < ntiles; t += 8) {
      const int mt = t / NT, nt = t - mt * NT;
      double c0 = 0.0, c1 = 0.0;
      for (int k0 = 0; k0 < KP; k0 += 4)
        dmma884(c0, c1, Zs[(mt * 8 + ar) * KP + k0 + ac], Lf(nt * 8 + ar, k0 + ac));
      const int p = mt * 8 + ar;
      const int i0 = nt * 8 + 2 * ac;
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = i0 + e;
        if (i < KP) {
          double dv = 0.0;
          if (i < d && p < cnt) {
            const double v = (a.base ? Bs[p * d + i] : smu[i]) + (e ? c1 : c0);
            a.out[(pb + p) * d + i] = v;
            dv = v - smu[i];
          }
          Ds[p * KP + i] = dv;
        }
      }
    }
    __syncthreads();
    // U = Delta Sinv; q_p = sum_i Delta[p][i] U[p][i]
    for (int t = w; t < ntiles; t += 8) {
      const int mt = t / NT, nt = t - mt * NT;
      double c0 = 0.0, c1 = 0.0;
      for (int k0 = 0; k0 < KP; k0 += 4)
        dmma884(c0, c1, Ds[(mt * 8 + ar) * KP + k0 + ac], Sf(nt * 8 + ar, k0 + ac));
      const int p = mt * 8 + ar, i0 = nt * 8 + 2 * ac;
      double q = 0.0;
      if (i0 < KP) q = fma(Ds[p * KP + i0], c0, q);
      if (i0 + 1 < KP) q = fma(Ds[p * KP + i0 + 1], c1, q);
      q += __shfl_xor_sync(0xffffffffu, q, 1);
      q += __shfl_xor_sync(0xffffffffu, q, 2);
      if (ac == 0) qp[p * NT + nt] = q;
    }
    __syncthreads();
    for (int p = threadIdx.x; p < cnt; p += blockDim.x) {
      double q = 0.0;
      for (int nt = 0; nt < NT; ++nt) q += qp[p * NT + nt];
      if (!isfinite(q)) atomicExch(&a.ctl->err, ERR_NUMERIC);
      a.lp_out[pb + p] = -0.5 * q;
    }
  }
}


// Register-blocked variant for d <= 32 (KK = round_up(d,4)/4 k-steps, NT =
// round_up(d,8)/8 column tiles): warp w owns particle rows 8w..8w+7 of the
// tile; all Lz and Sinv B-fragments live in registers (2 NT KK doubles), so a
// DMMA costs one shared load of its A fragment (the two-operand smem version
// is shared-memory-bandwidth bound: 512 B of LDS per 4-cycle DMMA).
template <int KK>
__global__ void __launch_bounds__(256, 2) k_propose_rb(DrawArgs a) {
  constexpr int KP = 4 * KK, NT = (KP + 7) / 8, NP = 8 * NT;
  extern __shared__ double sm[];
  if (a.stop && *a.stop) return;
  const int d = a.d;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  double* Zs = sm;                  // PR_TILE x KP
  double* Ds = Zs + PR_TILE * KP;   // PR_TILE x KP (theta* - mu)
  double* smu = Ds + PR_TILE * KP;  // KP
  double* sL = smu + KP;            // NP x KP
  double* sS = sL + NP * KP;        // NP x KP
  double* Bs = sS + NP * KP;        // PR_TILE x d
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  for (int i = threadIdx.x; i < KP; i += blockDim.x) smu[i] = i < d ? a.mu[i] : 0.0;
  __syncthreads();
  const int64_t ntl = (a.P + PR_TILE - 1) / PR_TILE;
  double bL[NT][KK];  // Lz B-fragments in registers; Sinv fragments are read from shared memory
  unsigned phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntl; tile += gridDim.x) {
    const int64_t pb = tile * PR_TILE;
    const int cnt = (int)min((int64_t)PR_TILE, a.P - pb);
    __syncthreads();  // previous tile's readers of Zs / Bs are done
    if (threadIdx.x == 0) {
      const unsigned zb = (unsigned)(PR_TILE * KP * 8);
      const unsigned bb = a.base ? (unsigned)(round_up(cnt * d, 2) * 8) : 0u;
      const unsigned mb = phase == 0 ? (unsigned)(NP * KP * 8) : 0u;
      mbar_arrive_expect_tx(&bar, zb + bb + 2 * mb);
      bulk_g2s(Zs, a.Z + pb * KP, zb, &bar);
      if (a.base) bulk_g2s(Bs, a.base + pb * d, bb, &bar);
      if (mb) {
        bulk_g2s(sL, a.Lz, mb, &bar);
        bulk_g2s(sS, a.Sinv, mb, &bar);
      }
    }
    mbar_wait(&bar, phase & 1u);
    if (phase == 0) {
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int kk = 0; kk < KK; ++kk) {
          bL[nt][kk] = sL[(nt * 8 + ar) * KP + kk * 4 + ac];
        }
    }
    ++phase;
    const int p = w * 8 + ar;  // this lane's particle row (A / C fragments)
    double c[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const double av = Zs[p * KP + kk * 4 + ac];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(c[nt][0], c[nt][1], av, bL[nt][kk]);
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = nt * 8 + 2 * ac + e;
        if (i < KP) {
          double dv = 0.0;
          if (i < d && p < cnt) {
            const double v = (a.base ? Bs[p * d + i] : smu[i]) + c[nt][e];
            a.out[(pb + p) * d + i] = v;
            dv = v - smu[i];
          }
          Ds[p * KP + i] = dv;
        }
      }
    __syncwarp();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const double av = Ds[p * KP + kk * 4 + ac];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) dmma884(c[nt][0], c[nt][1], av, sS[(nt * 8 + ar) * KP + kk * 4 + ac]);
    }
    double q = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = nt * 8 + 2 * ac + e;
        if (i < KP) q = fma(Ds[p * KP + i], c[nt][e], q);
      }
    q += __shfl_xor_sync(0xffffffffu, q, 1);
    q += __shfl_xor_sync(0xffffffffu, q, 2);
    if (ac == 0 && p < cnt) {
      if (!isfinite(q)) atomicExch(&a.ctl->err, ERR_NUMERIC);
      a.lp_out[pb + p] = -0.5 * q;
    }
  }
}

// ---------------------------------------------------------------- K9 + K6
// Accept (R16) and moments of the updated particles in one pass.  Block = tp
// consecutive particles of one group (tp divides N).  Outputs per block:
// [group-sum partial (d) | shifted second moment, lower triangle (ntri) | accepts].
// `decide` = false: moments only (the resampled particles, before the first step).
struct AccArgs {
  double* theta;
  double* L;
  double* lp;
  const double* theta_s;
  const double* part;
  const double* lp_s;
  const double* shift;
  const double* logu;  // plog of the ACCEPT uniforms of this step (precomputed), or nullptr
  double* bpart;
  Ctl* ctl;
  const int* stop;
  int64_t P, p0;
  double temper;
  uint64_t seed;
  int nchunks, d, tp, decide;
  uint32_t step, pass;
};

// Block = tp (<= 256, divides N) particles of one group, 256 threads.
// Output row: [group-sum partial (d) | sum (theta - c)(theta - c)' (d x d) | accepts].
__global__ void __launch_bounds__(256) k_accept_mom(AccArgs a) {
  extern __shared__ double sm[];
  __shared__ int red_i[32];
  if (a.stop && *a.stop) return;
  const int d = a.d, NP = round_up(d, 8), NT = NP / 8, W = d + d * d + 1;
  const int LT = NP + 4;  // padded row stride of Ts (2-way bank pattern for the DMMA fragments)
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int tp = a.tp, TK = round_up(tp, 4);
  double* Ts = sm;                                                   // TK x LT  (theta - c), zero padded
  double* gsp = sm + TK * LT;                                        // 8 x d group-sum partials
  unsigned char* acc = reinterpret_cast<unsigned char*>(gsp + 8 * d);  // tp flags
  const int64_t pbase = (int64_t)blockIdx.x * tp;
  int nacc = 0;
  for (int q = threadIdx.x; q < tp; q += blockDim.x) {
    unsigned char ok = 0;
    if (a.decide) {
      const int64_t p = pbase + q;
      double Ls = a.part[p];
      for (int c = 1; c < a.nchunks; ++c) Ls += a.part[(int64_t)c * a.P + p];
      const double Lc = a.L[p], lpc = a.lp[p], lps = a.lp_s[p];
      if (!isfinite(Ls)) atomicExch(&a.ctl->err, ERR_NUMERIC);
      const double delta = a.temper * (Ls - Lc) + (lps - lpc);
      double lu;
      if (a.logu) {
        lu = a.logu[p];
      } else {
        const u4 wv = stream_block(a.seed, 0u, (uint32_t)(a.p0 + p), a.step, TAG_ACCEPT, a.pass);
        lu = plog(u01(wv.x, wv.y));
      }
      if (lu < delta) {
        ok = 1;
        a.L[p] = Ls;
        a.lp[p] = lps;
        ++nacc;
      }
    }
    acc[q] = ok;
  }
  nacc = block_sum(nacc, red_i);  // includes a __syncthreads: acc[] visible
  // stage the updated particle rows (accepted -> theta*, else theta) in one cp.async round;
  // flat (q, i) loops with incremental row/column (no integer division)
  const int64_t off0 = pbase * d;
  const int sr = 256 / d, sc = 256 - sr * d;
  {
    int q = threadIdx.x / d, i = threadIdx.x - q * d;
    for (; q < tp;) {
      cp_async8(Ts + q * LT + i, (acc[q] ? a.theta_s : a.theta) + off0 + (int64_t)q * d + i);
      q += sr;
      i += sc;
      if (i >= d) {
        i -= d;
        ++q;
      }
    }
  }
  for (int q = w; q < TK; q += 8)  // zero padding columns / rows
    for (int i = d + lane; i < LT; i += 32) Ts[q * LT + i] = 0.0;
  for (int q = tp + w; q < TK; q += 8)
    for (int i = lane; i < d; i += 32) Ts[q * LT + i] = 0.0;
  cp_async_wait_all();
  __syncthreads();
  {  // write accepted rows back to theta; center on the shift
    int q = threadIdx.x / d, i = threadIdx.x - q * d;
    for (; q < tp;) {
      const double v = Ts[q * LT + i];
      if (acc[q]) a.theta[off0 + (int64_t)q * d + i] = v;
      Ts[q * LT + i] = v - a.shift[i];
      q += sr;
      i += sc;
      if (i >= d) {
        i -= d;
        ++q;
      }
    }
  }
  __syncthreads();
  double* out = a.bpart + (int64_t)blockIdx.x * W;
  // group-sum partial: 8 interleaved row sets per coordinate, then fixed-order combine
  for (int i = lane; i < d; i += 32) {
    const int part = w;
    double g0 = 0.0, g1 = 0.0;
    int q = part;
    for (; q + 8 < tp; q += 16) {
      g0 += Ts[q * LT + i];
      g1 += Ts[(q + 8) * LT + i];
    }
    if (q < tp) g0 += Ts[q * LT + i];
    gsp[part * d + i] = g0 + g1;
  }
  // lower-triangle tiles (mt >= nt) of T' T on DMMA: A[i][p] = T[p][i], B[p][l] = T[p][l]
  const int ar = lane >> 2, ac = lane & 3;
  const int ntri_t = NT * (NT + 1) / 2;
  for (int t = w; t < ntri_t; t += 8) {
    int mt = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while (mt * (mt + 1) / 2 > t) --mt;
    while ((mt + 1) * (mt + 2) / 2 <= t) ++mt;
    const int nt = t - mt * (mt + 1) / 2;
    double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};  // 4 independent DMMA chains over k
    int k0 = 0;
    for (; k0 + 16 <= TK; k0 += 16) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int kk = k0 + 4 * u + ac;
        dmma884(c[u][0], c[u][1], Ts[kk * LT + mt * 8 + ar], Ts[kk * LT + nt * 8 + ar]);
      }
    }
    for (; k0 < TK; k0 += 4) dmma884(c[0][0], c[0][1], Ts[(k0 + ac) * LT + mt * 8 + ar], Ts[(k0 + ac) * LT + nt * 8 + ar]);
    const double c0 = (c[0][0] + c[1][0]) + (c[2][0] + c[3][0]);
    const double c1 = (c[0][1] + c[1][1]) + (c[2][1] + c[3][1]);
    const int i = mt * 8 + ar, l0 = nt * 8 + 2 * ac;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int l = l0 + e;
      if (i < d && l < d) {
        const double v = e ? c1 : c0;
        out[d + i * d + l] = v;
        if (mt != nt) out[d + l * d + i] = v;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < d) {
    double g = 0.0;
    for (int part = 0; part < 8; ++part) g += gsp[part * d + threadIdx.x];
    out[threadIdx.x] = g + (double)tp * a.shift[threadIdx.x];
  }
  if (threadIdx.x == 0) out[W - 1] = (double)nacc;
}


// Register-blocked accept + moments for d <= 32 (NT = round_up(d,8)/8 <= 4):
// K (particles) split over the 8 warps; for each k-step one shared load per
// index tile serves as both the A and the B fragment of T'T (they coincide),
// feeding the NT(NT+1)/2 lower-triangle DMMAs; warp partials are combined in
// fixed order (deterministic).
template <int NT>
__global__ void __launch_bounds__(256) k_accept_mom_rb(AccArgs a) {
  extern __shared__ double sm[];
  __shared__ int red_i[32];
  if (a.stop && *a.stop) return;
  constexpr int NTRI = NT * (NT + 1) / 2;
  const int d = a.d, W = d + d * d + 1;
  constexpr int LT = 8 * NT + 4;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  const int tp = a.tp, TK = round_up(tp, 32);
  double* Ts = sm;                                                     // TK x LT
  double* gsp = sm + TK * LT;                                          // 8 x d
  unsigned char* acc = reinterpret_cast<unsigned char*>(gsp + 8 * d);  // tp flags
  const int64_t pbase = (int64_t)blockIdx.x * tp;
  int nacc = 0;
  for (int q = threadIdx.x; q < tp; q += blockDim.x) {
    unsigned char ok = 0;
    if (a.decide) {
      const int64_t p = pbase + q;
      double Ls = a.part[p];
      for (int c = 1; c < a.nchunks; ++c) Ls += a.part[(int64_t)c * a.P + p];
      const double Lc = a.L[p], lpc = a.lp[p], lps = a.lp_s[p];
      if (!isfinite(Ls)) atomicExch(&a.ctl->err, ERR_NUMERIC);
      const double delta = a.temper * (Ls - Lc) + (lps - lpc);
      double lu;
      if (a.logu) {
        lu = a.logu[p];
      } else {
        const u4 wv = stream_block(a.seed, 0u, (uint32_t)(a.p0 + p), a.step, TAG_ACCEPT, a.pass);
        lu = plog(u01(wv.x, wv.y));
      }
      if (lu < delta) {
        ok = 1;
        a.L[p] = Ls;
        a.lp[p] = lps;
        ++nacc;
      }
    }
    acc[q] = ok;
  }
  nacc = block_sum(nacc, red_i);
  const int64_t off0 = pbase * d;
  const int sr = 256 / d, sc = 256 - sr * d;
  {
    int q = threadIdx.x / d, i = threadIdx.x - q * d;
    for (; q < tp;) {
      cp_async8(Ts + q * LT + i, (acc[q] ? a.theta_s : a.theta) + off0 + (int64_t)q * d + i);
      q += sr;
      i += sc;
      if (i >= d) {
        i -= d;
        ++q;
      }
    }
  }
  for (int q = w; q < TK; q += 8)
    for (int i = (q < tp ? d : 0) + lane; i < LT; i += 32) Ts[q * LT + i] = 0.0;
  cp_async_wait_all();
  __syncthreads();
  {
    int q = threadIdx.x / d, i = threadIdx.x - q * d;
    for (; q < tp;) {
      const double v = Ts[q * LT + i];
      if (acc[q]) a.theta[off0 + (int64_t)q * d + i] = v;
      Ts[q * LT + i] = v - a.shift[i];
      q += sr;
      i += sc;
      if (i >= d) {
        i -= d;
        ++q;
      }
    }
  }
  __syncthreads();
  for (int i = lane; i < d; i += 32) {
    double g0 = 0.0, g1 = 0.0;
    int q = w;
    for (; q + 8 < tp; q += 16) {
      g0 += Ts[q * LT + i];
      g1 += Ts[(q + 8) * LT + i];
    }
    if (q < tp) g0 += Ts[q * LT + i];
    gsp[w * d + i] = g0 + g1;
  }
  // T'T: warp w takes k-steps k0 = 4 (w + 8 m)
  double cacc[NTRI][2];
#pragma unroll
  for (int t = 0; t < NTRI; ++t) cacc[t][0] = cacc[t][1] = 0.0;
  for (int k0 = 4 * w; k0 < TK; k0 += 32) {
    double f[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) f[t] = Ts[(k0 + ac) * LT + t * 8 + ar];
    int tt = 0;
#pragma unroll
    for (int mt = 0; mt < NT; ++mt)
#pragma unroll
      for (int nt = 0; nt <= mt; ++nt) {
        dmma884(cacc[tt][0], cacc[tt][1], f[mt], f[nt]);
        ++tt;
      }
  }
  __syncthreads();  // Ts free: reuse it for the warp partials
  double* wp = Ts;  // 8 x NTRI x 64
#pragma unroll
  for (int t = 0; t < NTRI; ++t) {
    wp[(w * NTRI + t) * 64 + lane * 2] = cacc[t][0];
    wp[(w * NTRI + t) * 64 + lane * 2 + 1] = cacc[t][1];
  }
  __syncthreads();
  double* out = a.bpart + (int64_t)blockIdx.x * W;
  for (int idx = threadIdx.x; idx < NTRI * 64; idx += blockDim.x) {
    const int t = idx >> 6, e = idx & 63, ln = e >> 1, ee = e & 1;
    double v = 0.0;
    for (int ww = 0; ww < 8; ++ww) v += wp[(ww * NTRI + t) * 64 + e];
    int mt = 0, rem = t;
    while (rem > mt) {
      rem -= mt + 1;
      ++mt;
    }
    const int nt = rem;
    const int i = mt * 8 + (ln >> 2), l = nt * 8 + 2 * (ln & 3) + ee;
    if (i < d && l < d) {
      out[d + i * d + l] = v;
      if (mt != nt) out[d + l * d + i] = v;
    }
  }
  if (threadIdx.x < d) {
    double g = 0.0;
    for (int part = 0; part < 8; ++part) g += gsp[part * d + threadIdx.x];
    out[threadIdx.x] = g + (double)tp * a.shift[threadIdx.x];
  }
  if (threadIdx.x == 0) out[W - 1] = (double)nacc;
}

// Deterministic reduction of the block partials into this rank's stats slice
// [Jl x d group sums | d x d second moment | accepts | error].  Blocks
// [0, nm): 32 moment entries each (8 warps x 8 independent rows per round,
// fixed-order combine); blocks [nm, nm + ng): group sums; last block: accepts.
__global__ void __launch_bounds__(256) k_mom_reduce(const double* __restrict__ bpart, int nblk, int bpg, int Jl,
                                                    int d, Ctl* ctl, double* __restrict__ slice,
                                                    const int* __restrict__ stop) {
  __shared__ double part[8][33];
  if (stop && *stop) return;
  const int dd = d * d, W = d + dd + 1;
  const int nm = (dd + 31) / 32, ng = (Jl * d + 255) / 256;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if ((int)blockIdx.x < nm) {
    const int e = blockIdx.x * 32 + lane;
    double acc8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (e < dd) {
      for (int b0 = w; b0 < nblk; b0 += 64) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int b = b0 + 8 * u;
          if (b < nblk) acc8[u] += bpart[(int64_t)b * W + d + e];
        }
      }
    }
    part[w][lane] = ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
    __syncthreads();
    if (w == 0 && e < dd) {
      double t = part[0][lane];
      for (int q = 1; q < 8; ++q) t += part[q][lane];
      slice[Jl * d + e] = t;
    }
  } else if ((int)blockIdx.x < nm + ng) {
    const int idx = (blockIdx.x - nm) * 256 + threadIdx.x;
    if (idx < Jl * d) {
      const int j = idx / d, c = idx % d;
      double s = 0.0;
      for (int b = 0; b < bpg; ++b) s += bpart[(int64_t)(j * bpg + b) * W + c];
      slice[idx] = s;
    }
  } else {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 256) s += bpart[(int64_t)b * W + W - 1];
    __shared__ double red[32];
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      slice[Jl * d + dd] = s;
      slice[Jl * d + dd + 1] = (double)ctl->err;
    }
  }
}

// Cholesky of a d x d SPD matrix (d <= D <= 32, D a multiple of 4 known at
// compile time; rows/cols d..D-1 are identity padding) by ONE warp, rows in
// registers (lane i holds row i).  Column j: every lane takes rsqrt of the
// pivot broadcast by shuffle (measured B200 latencies: rsqrt ~67 cycles,
// 64-bit shuffle ~31, DFMA 8); the column goes through shared memory for the
// off-diagonal updates, each lane's own diagonal stays in registers, so the
// pivot chain is ~110 cycles per column.  A: row-major d x d (read),
// Lout: lower factor (write), colbuf: 32 doubles of shared memory.
// 1/sqrt(x) without a slow-path call: MUFU approximation + 2 Newton steps
// (relative error ~1 ulp); non-positive / non-finite x give non-finite results.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double h = 0.5 * x;
  y = fma(y, fma(-h * y, y, 0.5), y);
  y = fma(y, fma(-h * y, y, 0.5), y);
  return y;
}

template <int D>
__device__ bool warp_cholesky(const double* A, int d, double scale, double ridge, double* Lout, double* colbuf,
                              int ldo, bool write = true) {
  const int lane = threadIdx.x & 31;
  double a[D];
#pragma unroll
  for (int l = 0; l < D; ++l)
    a[l] = (lane < d && l < d) ? scale * (A[lane * d + l] + (lane == l ? ridge : 0.0)) : (lane == l ? 1.0 : 0.0);
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double r = rsqrt_nr(__shfl_sync(0xffffffffu, a[j], j));
    const double lij = lane >= j ? a[j] * r : 0.0;  // L[lane][j]; lane j: sqrt(pivot)
    a[j] = lij;
    if (j + 1 < D) {
      colbuf[lane] = lij;
      __syncwarp();
      // branch-free: lanes < j carry lij = 0; entries above the diagonal are scratch
#pragma unroll
      for (int l = j + 1; l < D; ++l) a[l] = fma(-lij, (lane == l) ? lij : colbuf[l], a[l]);
      __syncwarp();
    }
  }
  // a non-positive or non-finite pivot leaves a non-finite or non-positive diagonal
  double diag = 1.0;
#pragma unroll
  for (int l = 0; l < D; ++l)
    if (lane == l) diag = a[l];
  const bool ok = __all_sync(0xffffffffu, lane >= d || (diag > 0.0 && isfinite(diag)));
  if (write && lane < d)
#pragma unroll
    for (int l = 0; l < D; ++l)
      if (l < d) Lout[lane * ldo + l] = l <= lane ? a[l] : 0.0;
  return ok;
}


// chol((h/100) V) for d <= 32 by one warp (no divergent enclosing code, so
// shuffles need no convergence barriers); one ridge retry (R13).
template <int D>
__global__ void __launch_bounds__(32) k_chol_warp(const double* __restrict__ V, int d, Ctl* ctl,
                                                  double* __restrict__ Lout, const int* __restrict__ stop_in) {
  __shared__ double sV[D * D];
  __shared__ double col[32];
  if (stop_in && *stop_in) return;
  for (int i = threadIdx.x; i < d * d; i += 32) sV[i] = V[i];
  __syncwarp();
  const double hd = (double)ctl->h / 100.0;
  const int ld = round_up(d, 4);  // padded (DMMA) layout of the factor
  bool ok = warp_cholesky<D>(sV, d, hd, 0.0, Lout, col, ld);
  if (!ok) {
    double tr = 0.0;
    for (int i = 0; i < d; ++i) tr += sV[i * d + i];
    ok = warp_cholesky<D>(sV, d, hd, 1e-8 * tr / (double)d, Lout, col, ld);
    if (threadIdx.x == 0) {
      ctl->chol_ridge = 1;
      if (!ok) ctl->err = ERR_NUMERIC;
    }
  } else if (threadIdx.x == 0) {
    ctl->chol_ridge = 0;
  }
}

// ---------------------------------------------------------------- K7
// theta-bar, pooled V (R11), h update (R6), monitor RNEs + stop flag (R12,
// R14), chol((h/100) V) with one ridge retry (R13), new shift.  One block;
// every rank computes the identical result from the gathered stats.  All
// inputs are first staged into shared memory with independent loads (the
// kernel is latency-bound: one block, a handful of dependent phases).
template <int D>  // D > 0: d <= D <= 32, Cholesky by the warps redundantly (no divergent region); D = 0: block path
__global__ void __launch_bounds__(256) k_finalize2(FinArgs f) {
  extern __shared__ double sm[];
  __shared__ int flag;
  __shared__ double red[32];
  if (f.stop_in && *f.stop_in) return;
  const int d = f.d, J = f.J, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gs_len = f.Jl * d;
  double* sV = sm;                 // d x d
  double* sbar = sV + d * d;       // d
  double* sA = sbar + d;           // d x d (Cholesky work of the block path; also the summed M)
  double* sg = sA + d * d;         // nmon x J group means + nmon RNEs
  double* sshift = sg + f.nmon * J + f.nmon;  // d
  double* smon = sshift + d;       // nmon x d
  double* sS = smon + f.nmon * d;  // J x d group sums (rank order == group order), when staged
  double* sM = sA;                 // consumed (into V) before sA is written
  const double P = (double)J * (double)f.N;
  auto S = [&](int j, int i) -> double {
    return f.stage_S ? sS[j * d + i] : f.gath[(int64_t)(j / f.Jl) * f.slice_len + (int64_t)(j % f.Jl) * d + i];
  };
  // ---- stage (one cp.async round)
  for (int i = threadIdx.x; i < d; i += blockDim.x) cp_async8(sshift + i, f.shift + i);
  for (int i = threadIdx.x; i < f.nmon * d; i += blockDim.x) cp_async8(smon + i, f.mon + i);
  if (f.stage_S)
    for (int r = 0; r < f.G; ++r)
      for (int off = threadIdx.x; off < gs_len; off += blockDim.x)
        cp_async8(sS + (int64_t)r * gs_len + off, f.gath + (int64_t)r * f.slice_len + off);
  if (f.G == 1)
    for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) cp_async8(sM + idx, f.gath + gs_len + idx);
  cp_async_wait_all();
  if (f.G > 1)
    for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
      double m = 0.0;
      for (int r = 0; r < f.G; ++r) m += f.gath[(int64_t)r * f.slice_len + gs_len + idx];
      sM[idx] = m;
    }
  __syncthreads();
  if (f.trace && threadIdx.x == 0) f.trace[1] = clock64();
  // ---- theta-bar: warp per coordinate, lanes over groups, fixed shuffle tree
  for (int i = w; i < d; i += nw) {
    double s = 0.0;
    for (int j = lane; j < J; j += 32) s += S(j, i);
    s = warp_sum(s);
    if (lane == 0) sbar[i] = s / P;
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int i = idx / d, l = idx - i * d;
    const double ci = sbar[i] - sshift[i], cl = sbar[l] - sshift[l];
    sV[idx] = (sM[idx] - P * ci * cl) / (P - 1.0);
  }
  __syncthreads();
  if (f.trace && threadIdx.x == 0) f.trace[2] = clock64();
  // warp 0: h update (from the pooled acceptance) then chol((h/100) V) in registers (d <= 32);
  // warps 1..: monitor RNEs, one warp per monitor (lanes over groups / V entries)
  __shared__ int s_h;
  __shared__ double s_col[8 * 32];
  if (w == 0) {
    int h = f.ctl->h;
    if (f.mode == 1) {
      double acc = 0.0, err = 0.0;
      for (int r = 0; r < f.G; ++r) {
        acc += f.gath[(int64_t)r * f.slice_len + gs_len + d * d];
        err = fmax(err, f.gath[(int64_t)r * f.slice_len + gs_len + d * d + 1]);
      }
      h = (acc > f.accept_target * P) ? min(h + f.h_step, f.h_max) : max(h - f.h_step, f.h_min);
      if (lane == 0) {
        if (err > 0.0) f.ctl->err = (int)err;
        f.ctl->h = h;
        f.ctl->acc = (unsigned long long)acc;
      }
    }
    if (lane == 0) s_h = h;
  } else if (f.mode == 1 && w - 1 < f.nmon) {
    for (int m = w - 1; m < f.nmon; m += nw - 1) {
      const double* av = smon + m * d;
      double gp = 0.0;
      for (int j = lane; j < J; j += 32) {
        double s0 = 0.0, s1 = 0.0;
        int i = 0;
        for (; i + 2 <= d; i += 2) {
          s0 = fma(av[i], S(j, i), s0);
          s1 = fma(av[i + 1], S(j, i + 1), s1);
        }
        if (i < d) s0 = fma(av[i], S(j, i), s0);
        const double g = (s0 + s1) / (double)f.N;
        sg[m * J + j] = g;
        gp += g;
      }
      const double gbar = warp_sum(gp) / (double)J;
      double dev = 0.0;
      for (int j = lane; j < J; j += 32) {
        const double t = sg[m * J + j] - gbar;
        dev = fma(t, t, dev);
      }
      dev = warp_sum(dev);
      double quad = 0.0;
      for (int idx = lane; idx < d * d; idx += 32) {
        const int i = idx / d;
        quad += av[i] * sV[idx] * av[idx - i * d];
      }
      quad = warp_sum(quad);
      const double vhat = (double)f.N / (double)(J - 1) * dev;
      const double var = quad * (P - 1.0) / P;
      if (lane == 0) sg[f.nmon * J + m] = vhat > 0.0 ? var / vhat : INFINITY;
    }
  }
  __syncthreads();
  if (f.mode == 1 && threadIdx.x == 0) {
    double minrne = INFINITY;
    for (int m = 0; m < f.nmon; ++m) {
      const double rne = sg[f.nmon * J + m];
      if (f.rne_out) f.rne_out[m] = rne;
      minrne = fmin(minrne, rne);
    }
    f.ctl->minrne = minrne;
    f.ctl->stop = (f.K > 0.0 && minrne >= f.K) ? 1 : 0;
    f.ctl->steps_done += 1;
  }
  const double hd = (double)s_h / 100.0;
  if (f.trace && threadIdx.x == 0) f.trace[3] = clock64();
  if constexpr (D > 0) {
    // every warp factors (h/100) V (identical results, no divergent region around the
    // shuffles); warp 0 writes the padded factor (ld = round_up(d, 4))
    const int ld = round_up(d, 4);
    bool ok = warp_cholesky<D>(sV, d, hd, 0.0, f.Lprop, s_col + 32 * w, ld, w == 0);
    int ridge_used = 0;
    if (!ok) {
      double tr = 0.0;
      for (int i = 0; i < d; ++i) tr += sV[i * d + i];
      ok = warp_cholesky<D>(sV, d, hd, 1e-8 * tr / (double)d, f.Lprop, s_col + 32 * w, ld, w == 0);
      ridge_used = 1;
    }
    if (threadIdx.x == 0) {
      f.ctl->chol_ridge = ridge_used;
      if (!ok) f.ctl->err = ERR_NUMERIC;
    }
  } else {  // block Cholesky (larger d)
    for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) sA[idx] = hd * sV[idx];
    __syncthreads();
    bool ok = block_cholesky(sA, d, &flag);
    if (threadIdx.x == 0) f.ctl->chol_ridge = ok ? 0 : 1;
    if (!ok) {
      double tr = 0.0;
      for (int i = 0; i < d; ++i) tr += sV[i * d + i];
      const double ridge = 1e-8 * tr / (double)d;
      for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x)
        sA[idx] = hd * (sV[idx] + ((idx / d == idx % d) ? ridge : 0.0));
      __syncthreads();
      ok = block_cholesky(sA, d, &flag);
      if (!ok) {
        if (threadIdx.x == 0) f.ctl->err = ERR_NUMERIC;
        return;
      }
    }
    for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) f.Lprop[(idx / d) * round_up(d, 4) + idx % d] = sA[idx];
  }
  if (f.trace && threadIdx.x == 0) f.trace[4] = clock64();
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) f.V[idx] = sV[idx];
  if (f.trace && threadIdx.x == 0) f.trace[5] = clock64();
  for (int i = threadIdx.x; i < d; i += blockDim.x) f.shift[i] = sbar[i];
  __syncthreads();
  if (f.host_out && threadIdx.x == 0) *f.host_out = *f.ctl;  // into mapped pinned host memory (visible at kernel end)
  if (f.trace && threadIdx.x == 0) f.trace[6] = clock64();
}

// Prior precision Sinv = Lprior^-T Lprior^-1 (one block; smem: Linv d x d).
__global__ void k_prior_precision(const double* __restrict__ Lp, int d, double* __restrict__ Sinv) {
  extern __shared__ double sInv[];
  for (int b = threadIdx.x; b < d; b += blockDim.x) {  // column b of Lp^-1 (lower)
    for (int i = 0; i < d; ++i) {
      double t = (i == b) ? 1.0 : 0.0;
      for (int j = b; j < i; ++j) t -= Lp[i * d + j] * sInv[j * d + b];
      sInv[i * d + b] = (i < b) ? 0.0 : t / Lp[i * d + i];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int r = idx / d, c = idx % d;
    double s = 0.0;
    for (int k = max(r, c); k < d; ++k) s += sInv[k * d + r] * sInv[k * d + c];
    Sinv[idx] = s;
  }
}

}  // namespace sps
