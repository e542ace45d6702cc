// mstep.cuh -- M phase kernels (Algorithm 2 step 2) and
// the prior draw, B200 layout: every per-particle stage is spread over all
// threads of a block (no long per-thread serial chains), every reduction is
// a fixed tree/order (deterministic), and kernels of a speculatively launched
// step return immediately once the device stop flag is set.
#pragma once
#include <cooperative_groups.h>

#include "common.cuh"
#include "kernels.cuh"
#include "loglik.cuh"

namespace sps {

// Slice layout (one rank): [Jl x d group sums S | d x d second moment | accepts | error |
// nmon x Jl monitor group means a_m' S_j / N | d column sums of S].
__host__ __device__ inline int slice_off_G(int Jl, int d) { return Jl * d + d * d + 2; }
__host__ __device__ inline int slice_off_C(int Jl, int d, int nmon) { return slice_off_G(Jl, d) + nmon * Jl; }
__host__ __device__ inline int slice_length(int Jl, int d, int nmon) { return slice_off_C(Jl, d, nmon) + d; }
// k_mom_reduce grid: nm moment blocks (32 lower-triangle / column-sum entries each), ng group blocks
// (whole groups: gpb = max(1, 256 / d) per block), one accepts block.
__host__ __device__ inline int red_nm(int d) { return (d * (d + 1) / 2 + d + 31) / 32; }
__host__ __device__ inline int red_gpb(int d) { return d <= 256 ? 256 / d : 1; }
__host__ __device__ inline int red_ng(int Jl, int d) { return (Jl + red_gpb(d) - 1) / red_gpb(d); }

// ---------------------------------------------------------------- K8 / K10
// theta* = base + Lz z (z: Box-Muller pairs of the stream (id = p0 + p, step,
// tag), R15) and lp* = -1/2 (theta* - mu)' Sinv (theta* - mu).  INIT: base =
// mu, Lz = Lprior (Algorithm 1 step 1); PROPOSAL: base =
// theta, Lz = chol(h V).
constexpr int PR_TILE = 64;  // particles per block (8 DMMA row tiles)
struct DrawArgs {
  const double* base;  // P x d, or nullptr -> mu
  const double* Lz;    // lower factor, padded NP x KP (NP = round_up(d, 8), KP = round_up(d, 4))
  const double* Sinv;  // prior precision, padded NP x KP (k_propose)
  const double* Rp;    // prior whitening factor Lprior^-1 (lower), padded NP x KP (k_propose_rb)
  const double* mu;
  const double* Z;  // P x 2 ceil(d/2) standard normals (k_normals)
  double* out;
  double* lp_out;
  Ctl* ctl;
  const int* stop;
  int64_t P, p0;
  int d;
  uint32_t step0;  // set_step: ctl->step_cur = step0 + ctl->steps_done (device-resident step of a graph replay)
  int set_step;
  const double* Zalt;  // device-side loop: Z of odd steps (Z: even steps), chosen by the parity of step_cur
};

// Standard normals of the streams (id = p0 + p, step, tag) for every local
// particle: Z[p][2 pr + {0,1}] = Box-Muller pair pr (R15).  One thread per
// (particle, pair).  Independent of the particle state, so the engine runs it
// one M step ahead on a side stream, overlapped with the latency-bound kernels.
// With `logu` (PROPOSAL streams), also plog of the step's ACCEPT uniform of each
// particle (R16), so the accept test on the critical path is one comparison.
// With `sctl` (M steps replayed from a CUDA graph) the step is device-resident:
// step = sctl->step_cur + 1, written by the proposal kernel of the running step.
// Zalt / logualt (device-side loop): the outputs of odd steps (Z / logu: even steps).
__global__ void __launch_bounds__(256) k_normals(int64_t P, int64_t p0, int np, uint64_t npmagic, int ldz, uint64_t seed,
                                                 uint32_t step,
                                                 uint32_t tag, uint32_t pass, double* __restrict__ Z,
                                                 double* __restrict__ logu, const Ctl* sctl, const int* stop,
                                                 double* Zalt, double* logualt) {
  // grid-stride over (particle, pair) tasks: the engine launches a small persistent grid so
  // the side-stream normals share SMs with the critical path instead of filling them
  if (stop && *stop) return;
  if (sctl) step = sctl->step_cur + 1u;
  if (sctl) tl_start(1);
  if (Zalt && (step & 1u)) {
    Z = Zalt;
    if (logu) logu = logualt;
  }
  const int64_t ntask = P * np;
  const int64_t gstride = (int64_t)gridDim.x * blockDim.x, g0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // t / np as the high half of t * npmagic, npmagic = floor(2^64 / np) + 1 (exact for every t < 2^64 / np;
  // computed on the host): the 64-bit division was a subroutine call per normal pair
  for (int64_t t = g0; t < ntask; t += gstride) {
    const int64_t p = np == 1 ? t : (int64_t)__umul64hi((uint64_t)t, npmagic);
    const int pr = (int)(t - p * np);
    double z0, z1;
    normal_pair(seed, (uint32_t)pr, (uint32_t)(p0 + p), step, tag, pass, &z0, &z1);
    reinterpret_cast<double2*>(Z + p * ldz)[pr] = make_double2(z0, z1);
  }
  // the accept log-uniforms in a pass of their own: as a branch of the loop above (pr == 0) every
  // warp paid one plog for its ~2.5 particle-leading lanes -- ~40% of the kernel's FP64 issue
  if (logu)
    for (int64_t p = g0; p < P; p += gstride) {
      const u4 w = stream_block(seed, 0u, (uint32_t)(p0 + p), step, TAG_ACCEPT, pass);
      logu[p] = plog(u01(w.x, w.y));
    }
  if (sctl) tl_end(1);
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
  if (a.set_step && blockIdx.x == 0 && threadIdx.x == 0) a.ctl->step_cur = a.step0 + (uint32_t)a.ctl->steps_done;
  const double* Zsrc = a.Z;
  if (a.Zalt && ((a.step0 + (uint32_t)a.ctl->steps_done) & 1u)) Zsrc = a.Zalt;
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
      bulk_g2s(Zs, Zsrc + pb * KP, zb, &bar);
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
// tile (A / C fragments in registers; Lz, Rp fragments from shared memory;
// k-steps above the lower-triangular factors skipped).  Persistent (3 blocks
// per SM) and double-buffered:
// the TMA loads of the block's next tile (Z rows, base rows) are in flight
// while the current tile computes; theta* is assembled in shared memory over
// the base rows and leaves as one TMA bulk store (contiguous rows).
template <int KK, int TILE>  // TILE particles per tile = TILE / 8 warps of 8 rows (blockDim = 4 TILE)
__global__ void __launch_bounds__(4 * TILE, TILE == 32 ? 5 : 3) k_propose_rb(DrawArgs a) {
  constexpr int KP = 4 * KK, NT = (KP + 7) / 8, NP = 8 * NT;
  extern __shared__ __align__(16) double sm[];
  // Launched with programmatic dependent launch after the previous step's reduce + finalize, which
  // triggers once the accept kernel is complete: theta (base rows) and Z (side stream, a full graph
  // edge) may be loaded before griddep_wait; Lz, Rp, the stop flag and the step counter (written by
  // the finalize) only after it.  With a static Z buffer (a.Zalt null) the first tile's Z / theta
  // loads are issued before that wait.
  const bool early = a.Zalt == nullptr;
  if (!early) {
    griddep_wait();
    if (a.stop && *a.stop) return;
  }
  const double* Zsrc = a.Z;
  if (a.Zalt && ((a.step0 + (uint32_t)a.ctl->steps_done) & 1u)) Zsrc = a.Zalt;
  const int d = a.d, BS = round_up(TILE * d, 2);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  double* Zs0 = sm;                     // 2 x TILE x KP: Z rows, then (theta* - mu) rows (per warp, in place)
  double* Bs0 = Zs0 + 2 * TILE * KP;  // 2 x BS: base rows, overwritten with theta*
  double* smu = Bs0 + 2 * BS;           // KP
  double* sL = smu + KP;                // NP x KP
  double* sS = sL + NP * KP;            // NP x KP (Rp)
  __shared__ __align__(8) uint64_t bar[2], barL;
  const int64_t ntl = (a.P + TILE - 1) / TILE;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_init(&barL, 1);
  }
  for (int i = threadIdx.x; i < KP; i += blockDim.x) smu[i] = i < d ? a.mu[i] : 0.0;
  __syncthreads();
  // thread 0: TMA loads of `tile` into buffer `buf`
  auto issue = [&](int64_t tile, int buf) {
    const int64_t pb = tile * TILE;
    const int cnt = (int)min((int64_t)TILE, a.P - pb);
    const unsigned zb = (unsigned)(TILE * KP * 8);
    const unsigned bb = a.base ? (unsigned)(round_up(cnt * d, 2) * 8) : 0u;
    mbar_arrive_expect_tx(&bar[buf], zb + bb);
    bulk_g2s(Zs0 + buf * TILE * KP, Zsrc + pb * KP, zb, &bar[buf]);
    if (a.base) bulk_g2s(Bs0 + buf * BS, a.base + pb * d, bb, &bar[buf]);
  };
  if (threadIdx.x == 0 && (int64_t)blockIdx.x < ntl) issue(blockIdx.x, 0);
  griddep_wait();  // the previous step's finalize: Lz, the stop flag, the step counter
  if (threadIdx.x == 0) {  // Lz, Rp (padded NP x KP) under their own barrier -- issued before the stop
    const unsigned mb = (unsigned)(NP * KP * 8);  // flag is read, so that its load overlaps them
    mbar_arrive_expect_tx(&barL, 2 * mb);
    bulk_g2s(sL, a.Lz, mb, &barL);
    bulk_g2s(sS, a.Rp, mb, &barL);
  }
  if (early && a.stop && *a.stop) {  // speculative step after the stop: drain the loads, exit
    if (threadIdx.x == 0) {
      if ((int64_t)blockIdx.x < ntl) mbar_wait(&bar[0], 0u);
      mbar_wait(&barL, 0u);
    }
    return;
  }
  if (a.set_step && blockIdx.x == 0 && threadIdx.x == 0) a.ctl->step_cur = a.step0 + (uint32_t)a.ctl->steps_done;
  if (a.set_step) tl_start(0);
  griddep_launch();  // persistent grid (all CTAs resident): K1's CTAs may start their prologue
  mbar_wait(&barL, 0u);
  int it = 0;
  for (int64_t tile = blockIdx.x; tile < ntl; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    const int64_t pb = tile * TILE;
    const int cnt = (int)min((int64_t)TILE, a.P - pb);
    if (threadIdx.x == 0 && tile + gridDim.x < ntl) {
      bulk_wait_read();  // the bulk store of iteration it-1 has read buffer buf^1
      issue(tile + gridDim.x, buf ^ 1);
    }
    mbar_wait(&bar[buf], (unsigned)(it >> 1) & 1u);
    double* Zs = Zs0 + buf * TILE * KP;
    double* Ds = Zs;  // a warp's Z rows are dead once its first product is done
    double* Bs = Bs0 + buf * BS;
    const int p = w * 8 + ar;  // this lane's particle row (A / C fragments)
    double c[NT][2];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const double av = Zs[p * KP + kk * 4 + ac];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)  // Lz lower: k-steps above the tile vanish
        if (kk <= 2 * nt + 1) dmma884(c[nt][0], c[nt][1], av, sL[(nt * 8 + ar) * KP + kk * 4 + ac]);
    }
    __syncwarp();  // all lanes' Z reads of these rows precede the (theta* - mu) writes over them
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = nt * 8 + 2 * ac + e;
        if (i < KP) {
          double dv = 0.0;
          if (i < d && p < cnt) {
            const double v = (a.base ? Bs[p * d + i] : smu[i]) + c[nt][e];
            Bs[p * d + i] = v;  // same thread read the base element
            dv = v - smu[i];
          }
          Ds[p * KP + i] = dv;
        }
      }
    __syncwarp();
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) c[nt][0] = c[nt][1] = 0.0;
    // W = Delta Rp' (Rp = Lprior^-1 lower, same triangular skip); q = |W|^2 = Delta' Sinv Delta
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const double av = Ds[p * KP + kk * 4 + ac];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        if (kk <= 2 * nt + 1) dmma884(c[nt][0], c[nt][1], av, sS[(nt * 8 + ar) * KP + kk * 4 + ac]);
    }
    double q = 0.0;
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) q = fma(c[nt][e], c[nt][e], q);  // padding columns of W are zero
    q += __shfl_xor_sync(0xffffffffu, q, 1);
    q += __shfl_xor_sync(0xffffffffu, q, 2);
    if (ac == 0 && p < cnt) {
      if (!isfinite(q)) atomicExch(&a.ctl->err, ERR_NUMERIC);
      a.lp_out[pb + p] = -0.5 * q;
    }
    __syncthreads();  // theta* tile complete; Zs / Ds consumed
    if (threadIdx.x == 0) {
      bulk_fence_smem();
      bulk_s2g(a.out + pb * d, Bs, (unsigned)(round_up(cnt * d, 2) * 8));
    }
  }
  if (threadIdx.x == 0) bulk_wait_all();
  if (a.set_step) tl_end(0);
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
  unsigned long long* trace;  // debug (SPS_TRACE): block-0 phase clocks [64..69], latest block end [70]
  Ctl* ctl;
  const int* stop;
  int64_t P, p0;
  double temper;
  uint64_t seed;
  int nchunks, d, tp, decide;
  uint32_t step, pass;
  uint64_t dmagic, pmagic;  // ceil(2^32 / d), ceil(2^32 / (LT - d)): e / m = (e * magic) >> 32 for e < 2^16
  const double* logualt;    // device-side loop: log u of odd steps (step = step0 + ctl->steps_done)
  uint32_t step0;
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
        lu = (a.logualt && ((a.step0 + (uint32_t)a.ctl->steps_done) & 1u)) ? a.logualt[p] : a.logu[p];
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
        lu = (a.logualt && ((a.step0 + (uint32_t)a.ctl->steps_done) & 1u)) ? a.logualt[p] : a.logu[p];
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
  // the tile's rows are contiguous in theta / theta*: flat element order e = q d + i (coalesced),
  // q = e / d by multiply-shift (a.dmagic, exact for e < 2^16), one cp.async round
  const int64_t off0 = pbase * d;
  const int ne = tp * d;
#pragma unroll 5
  for (int e = threadIdx.x; e < ne; e += 256) {
    const int q = (int)(((uint64_t)e * a.dmagic) >> 32), i = e - q * d;
    cp_async8(Ts + q * LT + i, (acc[q] ? a.theta_s : a.theta) + off0 + e);
  }
  // zero padding: columns [d, LT) of every row, full rows beyond tp
  const int padw = LT - d;
  for (int e = threadIdx.x; e < TK * padw; e += 256) {
    const int q = (int)(((uint64_t)e * a.pmagic) >> 32);
    const int i = d + e - q * padw;
    Ts[q * LT + i] = 0.0;
  }
  for (int e = threadIdx.x; e < (TK - tp) * d; e += 256) {
    const int q = (int)(((uint64_t)e * a.dmagic) >> 32);
    Ts[(tp + q) * LT + e - q * d] = 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  // accepted rows back to theta (same flat order), center on the shift
#pragma unroll 5
  for (int e = threadIdx.x; e < ne; e += 256) {
    const int q = (int)(((uint64_t)e * a.dmagic) >> 32), i = e - q * d;
    const double v = Ts[q * LT + i];
    if (acc[q]) a.theta[off0 + e] = v;
    Ts[q * LT + i] = v - a.shift[i];
  }
  __syncthreads();
  // group-sum partials: warp w sums rows w, w + 8, ... (lane = coordinate), fixed order
  if (lane < d) {
    double g0 = 0.0, g1 = 0.0;
    int q = w;
    for (; q + 8 < tp; q += 16) {
      g0 += Ts[q * LT + lane];
      g1 += Ts[(q + 8) * LT + lane];
    }
    if (q < tp) g0 += Ts[q * LT + lane];
    gsp[w * d + lane] = g0 + g1;
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
#pragma unroll 1
  for (int idx = threadIdx.x; idx < NTRI * 64; idx += blockDim.x) {
    const int t = idx >> 6, e = idx & 63, ln = e >> 1, ee = e & 1;
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += wp[(ww * NTRI + t) * 64 + e];
    // lower-triangle tile t -> (mt, nt), t = mt (mt + 1) / 2 + nt, NT <= 4
    const int mt = t >= 6 ? 3 : (t >= 3 ? 2 : (t >= 1 ? 1 : 0));
    const int nt = t - mt * (mt + 1) / 2;
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

// Accept + moments, tile layout (d <= 8 NT - 1, tp and tp d even).  One thread
// issues TMA bulk copies of everything the block needs at its start -- the
// tile's theta and theta* rows (contiguous), L, lp, lp*, log u -- under one
// mbarrier (the working set of an M step is L2-resident, so reading both row
// tiles costs L2, not HBM, bandwidth); the chunk partials of K1 are loaded
// into registers meanwhile.  The decision then runs from shared memory,
// accepted rows go back to theta in flat coalesced order, and T'T is built by
// DMMA with fragments formed on the fly, T[q][i] = (acc_q ? theta* : theta)[q][i]
// - c_i, plus a constant-1 column at index d whose row of T'T is the group-sum
// partial.  Output row: the NT(NT+1)/2 lower 8x8 tiles of T'T (fragment order
// = row-major within the tile) | accepts.  Short chain: one load round, one
// decision, one DMMA pass, one combine.
template <int NT>
__global__ void __launch_bounds__(256) k_accept_tile(AccArgs a) {
  constexpr int NTRI = NT * (NT + 1) / 2;
  extern __shared__ __align__(16) double sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ int red_i[32];
  const bool tr = a.trace && blockIdx.x == 0 && threadIdx.x == 0;
  if (tr) a.trace[64] = gtimer();
  const bool early = a.logualt == nullptr;  // static log-u buffer: loads issued before the stop flag is read
  if (!early && a.stop && *a.stop) return;
  const int d = a.d, tp = a.tp, lane = threadIdx.x & 31, w = threadIdx.x >> 5, ar = lane >> 2, ac = lane & 3;
  const int TD = tp * d;
  const bool dec = a.decide != 0;
  const int treg = max(TD, 8 * NTRI * 64);  // row tile (updated rows), later the warp partials
  double* sTh = sm;                          // tp x d
  double* sv = sm + treg;                    // [L | lp | lp* | log u] x tp
  unsigned char* acc = reinterpret_cast<unsigned char*>(sv + 4 * tp);
  const int64_t pbase = (int64_t)blockIdx.x * tp;
  const double* logu = a.logu;
  if (a.logualt && ((a.step0 + (uint32_t)a.ctl->steps_done) & 1u)) logu = a.logualt;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    const unsigned rb = (unsigned)TD * 8u, vb = (unsigned)tp * 8u;
    mbar_arrive_expect_tx(&bar, rb + (dec ? (a.logu ? 4u : 3u) * vb : 0u));
    bulk_g2s(sTh, a.theta + pbase * d, rb, &bar);
    if (dec) {
      bulk_g2s(sv, a.L + pbase, vb, &bar);
      bulk_g2s(sv + tp, a.lp + pbase, vb, &bar);
      bulk_g2s(sv + 2 * tp, a.lp_s + pbase, vb, &bar);
      if (logu) bulk_g2s(sv + 3 * tp, logu + pbase, vb, &bar);
    }
  }
  if (early && a.stop && *a.stop) {  // speculative step after the stop: drain the loads, exit
    if (threadIdx.x == 0) mbar_wait(&bar, 0u);
    return;
  }
  if (a.decide) tl_start(3);
  double shv[NT];  // c_i of this lane's fragment columns
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    const int i = t * 8 + ar;
    shv[t] = i < d ? a.shift[i] : 0.0;
  }
  double Ls = 0.0;  // K1 chunk partials of this thread's particle (sum in chunk order)
  const int q0 = threadIdx.x;
  griddep_wait();    // K1's chunk partials from here on (the bulk copies above read older data)
  griddep_launch();  // one wave: the reduce may start its launch
  if (dec && q0 < tp) {
    const int64_t p = pbase + q0;
    Ls = a.part[p];
    for (int c = 1; c < a.nchunks; ++c) Ls += a.part[(int64_t)c * a.P + p];
  }
  __syncthreads();  // barrier initialised
  mbar_wait(&bar, 0);
  if (tr) a.trace[65] = gtimer();
  if (dec) tl_mark(12);
  int nacc = 0;
  for (int q = q0; q < tp; q += blockDim.x) {
    unsigned char ok = 0;
    if (dec) {
      const int64_t p = pbase + q;
      if (q != q0) {
        Ls = a.part[p];
        for (int c = 1; c < a.nchunks; ++c) Ls += a.part[(int64_t)c * a.P + p];
      }
      if (!isfinite(Ls)) atomicExch(&a.ctl->err, ERR_NUMERIC);
      const double delta = a.temper * (Ls - sv[q]) + (sv[2 * tp + q] - sv[tp + q]);
      double lu;
      if (a.logu) {
        lu = sv[3 * tp + q];
      } else {
        const u4 wv = stream_block(a.seed, 0u, (uint32_t)(a.p0 + p), a.step, TAG_ACCEPT, a.pass);
        lu = plog(u01(wv.x, wv.y));
      }
      if (lu < delta) {
        ok = 1;
        a.L[p] = Ls;
        a.lp[p] = sv[2 * tp + q];
        ++nacc;
      }
    }
    acc[q] = ok;
  }
  nacc = block_sum(nacc, red_i);  // (barrier) acc visible
  if (tr) a.trace[66] = gtimer();
  if (dec) tl_mark(13);
  if (dec) {  // accepted rows only: theta* over the staged rows (one cp.async round), then back to theta
    // compact the accepted rows first (ballot prefix; tp <= blockDim): the copy loops then touch
    // nacc d elements instead of predicating all tp d (~1/4 accept)
    __shared__ int s_list[256];
    __shared__ int s_wc[8];
    const bool okq = q0 < tp && acc[q0];
    const unsigned bal = __ballot_sync(0xffffffffu, okq);
    if (lane == 0) s_wc[w] = __popc(bal);
    __syncthreads();
    int off = 0;
    for (int ww = 0; ww < w; ++ww) off += s_wc[ww];
    if (okq) s_list[off + __popc(bal & ((1u << lane) - 1u))] = q0;
    __syncthreads();
    const double* ts = a.theta_s + pbase * d;
    double* th = a.theta + pbase * d;
    const int ne = nacc * d;
#pragma unroll 4
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
      const int j = (int)(((uint64_t)e * a.dmagic) >> 32);
      const int o = s_list[j] * d + (e - j * d);
      cp_async8(sTh + o, ts + o);
    }
    cp_async_wait_all();
    __syncthreads();
#pragma unroll 4
    for (int e = threadIdx.x; e < ne; e += blockDim.x) {
      const int j = (int)(((uint64_t)e * a.dmagic) >> 32);
      const int o = s_list[j] * d + (e - j * d);
      th[o] = sTh[o];
    }
  }
  // T'T, lower tiles; warp w takes k-steps k0 = 4 (w + 8 m)
  double cacc[NTRI][2];
#pragma unroll
  for (int t = 0; t < NTRI; ++t) cacc[t][0] = cacc[t][1] = 0.0;
  for (int k0 = 4 * w; k0 < tp; k0 += 32) {
    const int q = k0 + ac;
    const bool valid = q < tp;
    const double* row = sTh + (valid ? q : 0) * d;
    double f[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = t * 8 + ar;
      f[t] = !valid ? 0.0 : (i < d ? row[i] - shv[t] : (i == d ? 1.0 : 0.0));
    }
    int tt = 0;
#pragma unroll
    for (int mt = 0; mt < NT; ++mt)
#pragma unroll
      for (int nt = 0; nt <= mt; ++nt) {
        dmma884(cacc[tt][0], cacc[tt][1], f[mt], f[nt]);
        ++tt;
      }
  }
  __syncthreads();  // row tiles consumed: the region holds the warp partials
  if (tr) a.trace[67] = gtimer();
  if (dec) tl_mark(14);
  double* wp = sm;  // 8 x NTRI x 64
#pragma unroll
  for (int t = 0; t < NTRI; ++t) {
    wp[(w * NTRI + t) * 64 + lane * 2] = cacc[t][0];
    wp[(w * NTRI + t) * 64 + lane * 2 + 1] = cacc[t][1];
  }
  __syncthreads();
  double* out = a.bpart + (int64_t)blockIdx.x * (NTRI * 64 + 1);
  for (int idx = threadIdx.x; idx < NTRI * 64; idx += blockDim.x) {
    double v = 0.0;
#pragma unroll
    for (int ww = 0; ww < 8; ++ww) v += wp[ww * NTRI * 64 + idx];
    out[idx] = v;  // fragment index e = 2 lane + j = 8 r + c: row-major within the tile
  }
  if (threadIdx.x == 0) out[NTRI * 64] = (double)nacc;
  if (a.trace && threadIdx.x == 0) {
    const unsigned long long t = gtimer();
    if (tr) a.trace[68] = t;
    atomicMax(&a.trace[70], t);
  }
  if (a.decide) tl_end(3);
}

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

// Cholesky (lower) of the d x d SPD matrix held in shared memory as Ap (row stride lda >= d;
// entries beyond d unused) by ONE warp, rows in registers (lane i holds row i), columns fully
// unrolled for D = d exactly (a round_up(d, 4) identity padding cost d = 25 three extra pivot steps):
// per column a 64-bit shuffle of the pivot, rsqrt + 2 Newton steps, then the column through shared
// memory for the trailing update (tools/chol_bench3.cu: ~250 cycles per column, ~3x faster than
// run-time-loop shared-memory variants, whose row updates serialize on shared-memory ordering).  One
// out-of-line copy per d serves both factorization attempts (code size: this runs once per M step
// from a cold instruction cache).  Writes the lower factor with row stride ldo (zeros above the
// diagonal) for rows and columns < d; the caller's padding of Lout stays as it is (zero).
// Returns false if a pivot is not positive and finite.
template <int D>
__device__ __noinline__ bool warp_cholesky(const double* Ap, int lda, double* Lout, int ldo) {
  __shared__ double colbuf[32];
  const int lane = threadIdx.x & 31, row = lane < D ? lane : D - 1;
  double a[D];
#pragma unroll
  for (int l = 0; l < D; ++l) a[l] = Ap[row * lda + l];
  bool ok = true;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double piv = __shfl_sync(0xffffffffu, a[j], j);
    ok = ok && piv > 0.0 && isfinite(piv);
    const double r = rsqrt_nr(piv);
    const double lij = lane >= j ? a[j] * r : 0.0;  // lane j: sqrt(pivot)
    a[j] = lij;
    if (j + 1 < D) {
      colbuf[lane] = lij;
      __syncwarp();
#pragma unroll
      for (int l = j + 1; l < D; ++l) a[l] = fma(-lij, colbuf[l], a[l]);
      __syncwarp();
    }
  }
  if (lane < D)
#pragma unroll
    for (int l = 0; l < D; ++l) Lout[lane * ldo + l] = l <= lane ? a[l] : 0.0;
  return ok;
}

__device__ bool warp_cholesky_d(const double* Ap, int lda, double* Lout, int ldo, int d) {
  switch (d) {
#define WCH(D_) \
  case D_: return warp_cholesky<D_>(Ap, lda, Lout, ldo);
    WCH(1) WCH(2) WCH(3) WCH(4) WCH(5) WCH(6) WCH(7) WCH(8) WCH(9) WCH(10) WCH(11) WCH(12) WCH(13) WCH(14)
    WCH(15) WCH(16) WCH(17) WCH(18) WCH(19) WCH(20) WCH(21) WCH(22) WCH(23) WCH(24) WCH(25) WCH(26) WCH(27)
    WCH(28) WCH(29) WCH(30) WCH(31)
#undef WCH
    default: return warp_cholesky<32>(Ap, lda, Lout, ldo);
  }
}

// n doubles global -> shared through L2 (ld.global.cg: coherent with the other
// blocks' writes of the same kernel), 4 independent loads in flight per thread.
__device__ __forceinline__ void stage_cg(double* dst, const double* src, int n) {
  for (int i0 = threadIdx.x; i0 < n; i0 += 4 * blockDim.x) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      v[u] = i < n ? __ldcg(src + i) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int i = i0 + u * blockDim.x;
      if (i < n) dst[i] = v[u];
    }
  }
}

// Group sum S_j[i] read from the gathered slices (when J x d is too large to stage).
__device__ __noinline__ double group_sum_global(const FinArgs& f, int j, int i) {
  return __ldcg(f.gath + (int64_t)(j / f.Jl) * f.slice_len + (int64_t)(j % f.Jl) * f.d + i);
}

// chol((h/100) V) by the whole block for d > 32 (sA: d x d, (h/100) V), one
// ridge retry (R13); factor -> f.Lprop (row stride ldp).
// The ridge base V: the pooled covariance, or Sigma_lr / (h/100) when Sigma_lr comes from a fixed
// design (Algorithm 3 pass 2; the oracle's reading of R13 there).
__device__ __forceinline__ double ridge_base(const double* sV, const double* sig, double hd, int idx) {
  return sig ? __ldcg(sig + idx) / hd : sV[idx];
}

__device__ __noinline__ void block_factor(const FinArgs& f, double* sA, const double* sV, double hd, int ldp, int* s_flag,
                                          const double* sig) {
  const int d = f.d, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  bool ok = block_cholesky(sA, d, s_flag);
  if (threadIdx.x == 0) f.ctl->chol_ridge = ok ? 0 : 1;
  if (!ok) {
    double tr = 0.0;
    for (int i = 0; i < d; ++i) tr += ridge_base(sV, sig, hd, i * d + i);
    const double ridge = 1e-8 * tr / (double)d;
    for (int i = w; i < d; i += nw)
      for (int l = lane; l < d; l += 32)
        sA[i * d + l] = hd * (ridge_base(sV, sig, hd, i * d + l) + (i == l ? ridge : 0.0));
    __syncthreads();
    ok = block_cholesky(sA, d, s_flag);
    if (!ok) {
      if (threadIdx.x == 0) f.ctl->err = ERR_NUMERIC;
      return;
    }
  }
  for (int i = w; i < d; i += nw)
    for (int l = lane; l < d; l += 32) f.Lprop[i * ldp + l] = sA[i * d + l];
}

// Three segments global -> shared through L2, every load of a thread issued
// before its first store (one latency round for up to 12 x blockDim doubles).
__device__ void stage3(double* d0, const double* s0, int n0, double* d1, const double* s1, int n1, double* d2,
                       const double* s2, int n2) {
  const int p1 = n0, p2 = n0 + n1, tot = p2 + n2;
#pragma unroll 1
  for (int base = threadIdx.x; base < tot; base += 12 * blockDim.x) {
    double v[12];
#pragma unroll
    for (int u = 0; u < 12; ++u) {
      const int idx = base + u * blockDim.x;
      const double* src = idx < p1 ? s0 + idx : (idx < p2 ? s1 + (idx - p1) : s2 + (idx - p2));
      v[u] = idx < tot ? __ldcg(src) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 12; ++u) {
      const int idx = base + u * blockDim.x;
      double* dst = idx < p1 ? d0 + idx : (idx < p2 ? d1 + (idx - p1) : d2 + (idx - p2));
      if (idx < tot) *dst = v[u];
    }
  }
}

// Dynamic shared memory of finalize_body (doubles).
__host__ __device__ inline int64_t fin_smem_doubles(int d, int J, int nmon, bool stage_S) {
  const int D = (d + 3) / 4 * 4;
  return (int64_t)2 * d * d + (d > 32 ? 0 : (int64_t)D * D) + 2 * d + (int64_t)nmon * d + (int64_t)nmon * J + nmon +
         4 + (stage_S ? (int64_t)J * d : 0);
}

// ---------------------------------------------------------------- K7
// theta-bar, pooled V (R11), h update (R6), monitor RNEs + stop flag (R12,
// R14), chol((h/100) V) with one ridge retry (R13), new shift, from the
// gathered stats [Jl x d group sums | d x d second moment | accepts | error]
// of the G ranks (rank order == group order).  One block of 256 threads; every
// rank computes the identical result.  Latency-bound: one staging round, then
// warp 0 factors while warps 1.. compute the monitor RNEs (d <= 32).
__device__ void finalize_body(const FinArgs& f, double* sm) {
  const int d = f.d, J = f.J, dd = d * d, lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int gs_len = f.Jl * d, D = round_up(d, 4), ldc = d > 32 ? d : D;
  const double P = (double)J * (double)f.N;
  double* sS = sm;                                // J x d group sums (staged) -- contiguous with sM:
  double* sM = sS + (f.stage_S ? J * d : 0);      // d x d second moment (one rank: one copy of [S | M])
  double* sV = sM + dd;                           // d x d pooled covariance
  // (h/100) V: d <= 32: D x D, identity-padded (warp_cholesky input); d > 32:
  // d x d factored in place, overlaying sM (each (i, l) entry is read from sM
  // and written to sA by the same thread)
  double* sA = d > 32 ? sM : sV + dd;
  double* sbar = sV + dd + (d > 32 ? 0 : D * D);  // d
  double* sshift = sbar + d;                      // d
  double* smon = sshift + d;                      // nmon x d
  double* sg = smon + f.nmon * d;                 // nmon x J group means, then nmon RNEs
  double* sxtra = sg + f.nmon * J + f.nmon;       // [accepts, error, h] (preloaded by the cluster reduce)
  __shared__ int s_h, s_flag;
  __shared__ double s_part[8][32];
  if (f.trace && threadIdx.x == 0) f.trace[0] = gtimer();
  // ---- stage: one round of independent L2 loads
  if (f.preloaded) {
    // S, M, accepts, error (other CTAs, DSMEM) and shift, monitors, h (this CTA, prefetched at its
    // start) are already in shared memory
  } else if (f.G == 1) {
    if (f.stage_S)
      stage3(sS, f.gath, gs_len + dd, sshift, f.shift, d, smon, f.mon, f.nmon * d);
    else
      stage3(sM, f.gath + gs_len, dd, sshift, f.shift, d, smon, f.mon, f.nmon * d);
  } else {
    stage3(sshift, f.shift, d, smon, f.mon, f.nmon * d, sM, f.gath + gs_len, 0);
    if (f.stage_S)
#pragma unroll 1
      for (int r = 0; r < f.G; ++r) stage_cg(sS + (int64_t)r * gs_len, f.gath + (int64_t)r * f.slice_len, gs_len);
#pragma unroll 1
    for (int idx = threadIdx.x; idx < dd; idx += blockDim.x) {
      double m = 0.0;
#pragma unroll 1
      for (int r = 0; r < f.G; ++r) m += __ldcg(f.gath + (int64_t)r * f.slice_len + gs_len + idx);
      sM[idx] = m;
    }
  }
  if (threadIdx.x == 0) {  // h update from the pooled acceptance (R6)
    int h = f.preloaded ? (int)sxtra[2] : f.ctl->h;
    if (f.mode == 1) {
      double acc = 0.0, err = 0.0;
      if (f.preloaded) {
        acc = sxtra[0];
        err = sxtra[1];
      } else {
#pragma unroll 1
        for (int r = 0; r < f.G; ++r) {
          acc += __ldcg(f.gath + (int64_t)r * f.slice_len + gs_len + dd);
          err = fmax(err, __ldcg(f.gath + (int64_t)r * f.slice_len + gs_len + dd + 1));
        }
      }
      h = (acc > f.accept_target * P) ? min(h + f.h_step, f.h_max) : max(h - f.h_step, f.h_min);
      if (err > 0.0) f.ctl->err = (int)err;
      f.ctl->h = h;
      f.ctl->acc = (unsigned long long)acc;
    }
    s_h = h;
  }
  __syncthreads();
  if (f.trace && threadIdx.x == 0) f.trace[1] = gtimer();
  if (f.mode == 1 && threadIdx.x == 0) tl_mark_any(16);
  auto S = [&](int j, int i) -> double { return f.stage_S ? sS[j * d + i] : group_sum_global(f, j, i); };
  // ---- theta-bar: lane = coordinate, warp = group subset, fixed-order combine (S staged); otherwise
  // from the per-rank column sums of S that k_mom_reduce put in the slices (large J: S stays in L2)
  if (!f.stage_S) {
    const int offC = slice_off_C(f.Jl, d, f.nmon), offG = slice_off_G(f.Jl, d);
#pragma unroll 1
    for (int i = threadIdx.x; i < d; i += blockDim.x) {
      double t = 0.0;
#pragma unroll 1
      for (int r = 0; r < f.G; ++r) t += __ldcg(f.gath + (int64_t)r * f.slice_len + offC + i);
      sbar[i] = t / P;
    }
    // monitor group means (nmon x J) into sg, 4 independent loads in flight per thread
    const int nG = f.nmon * J;
#pragma unroll 1
    for (int i0 = threadIdx.x; i0 < nG; i0 += 4 * blockDim.x) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int idx = i0 + u * blockDim.x;
        const int m = idx / J, j = idx - m * J;
        v[u] = idx < nG ? __ldcg(f.gath + (int64_t)(j / f.Jl) * f.slice_len + offG + m * f.Jl + (j % f.Jl)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (i0 + u * blockDim.x < nG) sg[i0 + u * blockDim.x] = v[u];
    }
    __syncthreads();
  } else
#pragma unroll 1
  for (int i0 = 0; i0 < d; i0 += 32) {
    const int i = i0 + lane;
    double s = 0.0;
    if (i < d) {
#pragma unroll 4
      for (int j = w; j < J; j += nw) s += sS[j * d + i];
    }
    s_part[w][lane] = s;
    __syncthreads();
    if (w == 0 && i < d) {
      double t = s_part[0][lane];
#pragma unroll 1
      for (int q = 1; q < nw; ++q) t += s_part[q][lane];
      sbar[i] = t / P;
    }
    __syncthreads();
  }
  if (f.trace && threadIdx.x == 0) f.trace[2] = gtimer();
  if (f.mode == 1 && threadIdx.x == 0) tl_mark_any(17);
  // ---- V (R11) and the factorization input (h/100) V, identity-padded to D x D
  const double hd = (double)s_h / 100.0;
  const double rPm1 = 1.0 / (P - 1.0);
  const int DA = d > 32 ? d : D;
  // Algorithm 3: Sigma of the step this factor serves, from / into the design record
  // (the device step is read only when a record / design is attached: a global load here is on
  // the M step's critical path)
  const int64_t sstep = (!f.sig_in && !f.sig_rec) ? 0
                        : f.sig_step >= 0 ? f.sig_step : (int64_t)__ldcg(&f.ctl->step_cur) + 1;
  const double* sig = (f.sig_in && sstep < f.sig_in_n) ? f.sig_in + sstep * dd : nullptr;
  double* srec = (f.sig_rec && sstep < f.sig_rec_cap) ? f.sig_rec + sstep * dd : nullptr;
#pragma unroll 2
  for (int i = w; i < DA; i += nw) {
    const double ci = i < d ? sbar[i] - sshift[i] : 0.0;
#pragma unroll 1
    for (int l = lane; l < DA; l += 32) {
      if (i < d && l < d) {
        const double cl = sbar[l] - sshift[l];
        const double v = (sM[i * d + l] - P * ci * cl) * rPm1;  // / (JN - 1) (R11), as one multiply
        sV[i * d + l] = v;
        const double a = sig ? __ldcg(sig + i * d + l) : hd * v;  // Sigma_lr = (h/100) V_lr
        sA[i * ldc + l] = a;
        if (srec) srec[i * d + l] = a;
      } else {
        sA[i * ldc + l] = i == l ? 1.0 : 0.0;
      }
    }
  }
  __syncthreads();
  if (f.trace && threadIdx.x == 0) f.trace[3] = gtimer();
  if (f.mode == 1 && threadIdx.x == 0) tl_mark_any(18);
  const int ldp = round_up(d, 4);  // padded (DMMA) layout of the factor
  if (w == 0 && d <= 32) {         // chol((h/100) V), one ridge retry (R13)
    bool ok = warp_cholesky_d(sA, ldc, f.Lprop, ldp, d);
    int ridge_used = 0;
    if (!ok) {
      double tr = 0.0;
#pragma unroll 1
      for (int i = 0; i < d; ++i) tr += ridge_base(sV, sig, hd, i * d + i);
      const double ridge = 1e-8 * tr / (double)d;
      if (lane < d)
#pragma unroll 1
        for (int l = 0; l < d; ++l)
          sA[lane * ldc + l] = hd * (ridge_base(sV, sig, hd, lane * d + l) + (lane == l ? ridge : 0.0));
      __syncwarp();
      ok = warp_cholesky_d(sA, ldc, f.Lprop, ldp, d);
      ridge_used = 1;
    }
    if (lane == 0) {
      f.ctl->chol_ridge = ridge_used;
      if (!ok) f.ctl->err = ERR_NUMERIC;
      if (f.mode == 1) tl_mark_any(15);  // (debug timeline: Cholesky done)
    }
  } else if (w > 0 && f.mode == 1) {  // monitor RNEs: warp per monitor, lanes over groups
#pragma unroll 1
    for (int m = w - 1; m < f.nmon; m += nw - 1) {
      const double* av = smon + m * d;
      double gp = 0.0;
#pragma unroll 1
      for (int j = lane; j < J; j += 32) {
        double g;
        if (f.stage_S) {
          double s0 = 0.0, s1 = 0.0;
          int i = 0;
          for (; i + 2 <= d; i += 2) {
            s0 = fma(av[i], S(j, i), s0);
            s1 = fma(av[i + 1], S(j, i + 1), s1);
          }
          if (i < d) s0 = fma(av[i], S(j, i), s0);
          g = (s0 + s1) / (double)f.N;
          sg[m * J + j] = g;
        } else {  // the same value, formed by k_mom_reduce's group blocks and staged above
          g = sg[m * J + j];
        }
        gp += g;
      }
      const double gbar = warp_sum(gp) / (double)J;
      double dev = 0.0;
#pragma unroll 1
      for (int j = lane; j < J; j += 32) {
        const double t = sg[m * J + j] - gbar;
        dev = fma(t, t, dev);
      }
      dev = warp_sum(dev);
      double quad = 0.0;
#pragma unroll 2
      for (int i = 0; i < d; ++i)
#pragma unroll 1
        for (int l = lane; l < d; l += 32) quad += av[i] * sV[i * d + l] * av[l];
      quad = warp_sum(quad);
      const double vhat = (double)f.N / (double)(J - 1) * dev;
      const double var = quad * (P - 1.0) / P;
      if (lane == 0) sg[f.nmon * J + m] = vhat > 0.0 ? var / vhat : INFINITY;
    }
    if (threadIdx.x == 32 && f.mode == 1) tl_mark_any(21);  // (debug timeline: warp 1's RNEs done)
  }
  __syncthreads();
  if (f.trace && threadIdx.x == 0) f.trace[4] = gtimer();
  if (f.mode == 1 && threadIdx.x == 0) tl_mark_any(19);
  if (d > 32) {  // block Cholesky (larger d)
    block_factor(f, sA, sV, hd, ldp, &s_flag, sig);
  }
  if (f.mode == 1 && threadIdx.x == 0) {
    double minrne = INFINITY;
#pragma unroll 1
    for (int m = 0; m < f.nmon; ++m) {
      const double rne = sg[f.nmon * J + m];
      if (f.rne_out) f.rne_out[m] = rne;
      minrne = fmin(minrne, rne);
    }
    f.ctl->minrne = minrne;
    const int done = f.ctl->steps_done + 1;
    // stop: 1 = min RNE >= K; 2 = the device-side loop reached its step cap
    const int stop = (f.K > 0.0 && minrne >= f.K) ? 1 : ((f.loop && done >= f.rmax) ? 2 : 0);
    f.ctl->stop = stop;
    f.ctl->steps_done = done;
    // device-side M phase (a WHILE graph node, two steps per body): the condition is 1 from the
    // launch on and is cleared once, on the stopping step (a device-side set costs ~2 us)
    if (f.loop && stop != 0) cudaGraphSetConditional(f.cond, 0u);
  }
  if (f.V)
#pragma unroll 1
    for (int idx = threadIdx.x; idx < dd; idx += blockDim.x) f.V[idx] = sV[idx];
  for (int i = threadIdx.x; i < d; i += blockDim.x) f.shift[i] = sbar[i];
  __syncthreads();
  if (f.trace && threadIdx.x == 0) f.trace[5] = gtimer();
  if (f.mode == 1 && threadIdx.x == 0) tl_mark_any(20);
  // into mapped pinned host memory (visible at kernel end); in the device-side loop the host reads
  // it after the phase: written on the stopping step only
  if (f.host_out && threadIdx.x == 0 && (!f.loop || f.ctl->stop != 0)) *f.host_out = *f.ctl;
  if (f.trace && threadIdx.x == 0) f.trace[6] = gtimer();
}

// Block-partial layouts: full (k_accept_mom*): [d | d x d | accepts] (group
// sums of theta, the shift added per block); tile (k_accept_tile, tnt > 0):
// [tnt(tnt+1)/2 lower 8x8 tiles of T'T with the ones row at index d | accepts].
struct RedArgs {
  const double* bpart;
  int nblk, bpg, Jl, d, W;
  int tnt;             // tile layout: tiles per side (0: full layout)
  int N;               // particles per group (tile layout: group sums += N c)
  const double* shift;
  const double* mon;   // nmon x d monitors: k_mom_reduce also writes the monitor group means and the
  int nmon;            // column sums of S into the slice (finalize_body reads them when S is not staged)
};
__device__ __forceinline__ int red_col(const RedArgs& r, int i, int l) {  // entry (i, l), i >= l, of T'T
  if (!r.tnt) return r.d + i * r.d + l;
  const int mt = i >> 3, nt = l >> 3;
  return (mt * (mt + 1) / 2 + nt) * 64 + (i & 7) * 8 + (l & 7);
}

// Deterministic reduction of the block partials into this rank's stats slice
// [Jl x d group sums | d x d second moment | accepts | error].  Blocks
// [0, nm): 32 lower-triangle moment entries each (8 warps x 32 rows in flight,
// fixed-order combine, mirrored on write); blocks [nm, nm + ng): group sums;
// last block: accepts.  With f.ticket (one rank: the slice is the gathered
// stats) the last block to finish runs finalize_body on them (saves a launch
// and a dependent-launch gap).
__global__ void __launch_bounds__(256) k_mom_reduce(RedArgs r, Ctl* ctl, double* __restrict__ slice,
                                                    const int* __restrict__ stop, FinArgs f) {
  extern __shared__ double fin_sm[];
  __shared__ double part[8][33];
  __shared__ int s_last;
  if (f.trace && threadIdx.x == 0) f.trace[8 + blockIdx.x] = gtimer();
  if (stop && *stop) return;
  if (f.mode == 1) tl_start(4);
  griddep_wait();    // the accept kernel's block partials
  griddep_launch();  // the next step's proposal may start its launch and theta / Z loads (accept is done)
  const int d = r.d, Jl = r.Jl, W = r.W, nblk = r.nblk, dd = d * d, nl = d * (d + 1) / 2;
  const int nm = red_nm(d), ng = red_ng(Jl, d), gpb = red_gpb(d);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if ((int)blockIdx.x < nm) {
    // entries e < nl: (i, l) of the lower triangle of the second moment; nl <= e < nl + d: column sum
    // l = e - nl of the group sums over all blocks (the ones row of the tile layout)
    const int e = blockIdx.x * 32 + lane;
    int i = 0, l = 0, col = 0;
    if (e < nl) {  // e = i (i + 1) / 2 + l
      i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > e) --i;
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      l = e - i * (i + 1) / 2;
      col = red_col(r, i, l);
    } else if (e < nl + d) {
      l = e - nl;
      col = r.tnt ? red_col(r, d, l) : l;
    }
    double acc8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (e < nl + d) {
#pragma unroll 1
      for (int b0 = w; b0 < nblk; b0 += 256) {
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int b = b0 + 8 * u;
          v[u] = b < nblk ? r.bpart[(int64_t)b * W + col] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) acc8[u & 7] += v[u];
      }
    }
    part[w][lane] = ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
    __syncthreads();
    if (w == 0 && e < nl + d) {
      double t = part[0][lane];
      for (int q = 1; q < 8; ++q) t += part[q][lane];
      if (e < nl) {
        slice[Jl * d + i * d + l] = t;
        slice[Jl * d + l * d + i] = t;
      } else {
        slice[slice_off_C(Jl, d, r.nmon) + l] = r.tnt ? t + (double)Jl * (double)r.N * r.shift[l] : t;
      }
    }
  } else if ((int)blockIdx.x < nm + ng) {
    // whole groups j0 .. j0 + gpb - 1: their sums S_j, then the monitor group means a_m' S_j / N (the
    // finalize_body arithmetic, two interleaved fma chains)
    __shared__ double sgrp[512];
    const int j0 = (blockIdx.x - nm) * gpb;
#pragma unroll 1
    for (int t = threadIdx.x; t < gpb * d; t += blockDim.x) {
      const int j = j0 + t / d, c = t % d;
      if (j < Jl) {
        const int col = r.tnt ? red_col(r, d, c) : c;
        double s = 0.0;
        for (int b = 0; b < r.bpg; ++b) s += r.bpart[(int64_t)(j * r.bpg + b) * W + col];
        if (r.tnt) s += (double)r.N * r.shift[c];
        slice[j * d + c] = s;
        if (t < 512) sgrp[t] = s;
      }
    }
    __syncthreads();
    if (r.mon && gpb * d <= 512)
#pragma unroll 1
      for (int t = threadIdx.x; t < r.nmon * gpb; t += blockDim.x) {
        const int m = t / gpb, jj = t % gpb, j = j0 + jj;
        if (j < Jl) {
          const double* av = r.mon + m * d;
          const double* Sj = sgrp + jj * d;
          double s0 = 0.0, s1 = 0.0;
          int i = 0;
          for (; i + 2 <= d; i += 2) {
            s0 = fma(av[i], Sj[i], s0);
            s1 = fma(av[i + 1], Sj[i + 1], s1);
          }
          if (i < d) s0 = fma(av[i], Sj[i], s0);
          slice[slice_off_G(Jl, d) + m * Jl + j] = (s0 + s1) / (double)r.N;
        }
      }
  } else {
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 256) s += r.bpart[(int64_t)b * W + W - 1];
    __shared__ double red[32];
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      slice[Jl * d + dd] = s;
      slice[Jl * d + dd + 1] = (double)ctl->err;
    }
  }
  if (!f.ticket) return;
  __threadfence();  // this block's slice writes before its ticket
  __syncthreads();
  if (f.trace && threadIdx.x == 0) f.trace[8 + gridDim.x + blockIdx.x] = gtimer();
  if (f.mode == 1) tl_end(4);
  if (threadIdx.x == 0) s_last = atomicAdd(f.ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (threadIdx.x == 0) *f.ticket = 0u;  // re-armed for the next launch (stream order)
  unsigned long long* tl = g_tl;
  int tlr = -1;
  if (tl && threadIdx.x == 0 && f.mode == 1) {
    tlr = *g_tl_steps;  // before finalize_body increments steps_done
    if (tlr >= 0 && tlr < TL_ROWS) tl[tlr * TL_W + 10] = gtimer();
  }
  finalize_body(f, fin_sm);
  if (tlr >= 0 && tlr < TL_ROWS) tl[tlr * TL_W + 11] = gtimer();
}

// Reduce + finalize as ONE thread-block cluster (one rank): CTA r reduces moment groups r, r + ncta,
// ... (32 lower-triangle entries, 8 warps over the block partial rows) and a share of the group sums,
// writing the results straight into CTA 0's finalize shared memory (DSMEM); after one cluster
// barrier CTA 0 runs finalize_body on them -- no global stats slice, no ticket, no staging round.
__global__ void __launch_bounds__(256) k_mom_reduce_cl(RedArgs r, Ctl* ctl, const int* __restrict__ stop, FinArgs f) {
  namespace cg = cooperative_groups;
  extern __shared__ double fin_sm[];
  __shared__ double part[8][33];
  __shared__ double red[32];
  cg::cluster_group cl = cg::this_cluster();
  const int rank = (int)cl.block_rank(), ncta = (int)cl.num_blocks();
  if (stop && *stop) return;  // uniform over the cluster
  if (f.mode == 1 && rank == 0) tl_start(4);
  griddep_wait();    // the accept kernel's block partials
  griddep_launch();  // the next step's proposal may start its launch and theta / Z loads (accept is done)
  const int d = r.d, Jl = r.Jl, W = r.W, nblk = r.nblk, nl = d * (d + 1) / 2, nm = (nl + 31) / 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double* sS0 = cl.map_shared_rank(fin_sm, 0);  // CTA 0's finalize layout: [S (J x d) | M (d x d) | ...]
  double* sM0 = sS0 + (int64_t)f.J * d;
  double* sx0 = sM0 + fin_smem_doubles(d, f.J, f.nmon, true) - (int64_t)f.J * d - 4;  // [accepts, error, h]
  if (rank == 0) {  // prefetch the finalize inputs that do not depend on this step's partials
    const int D = round_up(d, 4);
    double* sshift = sM0 + 2 * d * d + (d > 32 ? 0 : D * D) + d;  // (layout of finalize_body)
    double* smon = sshift + d;
    for (int i = threadIdx.x; i < d; i += blockDim.x) sshift[i] = f.shift[i];
    for (int i = threadIdx.x; i < f.nmon * d; i += blockDim.x) smon[i] = f.mon[i];
    if (threadIdx.x == 0) fin_sm[sx0 - sS0 + 2] = (double)f.ctl->h;
  }
  for (int g = rank; g < nm; g += ncta) {
    const int e = g * 32 + lane;
    int i = 0, l = 0;
    if (e < nl) {
      i = (int)((sqrt(8.0 * e + 1.0) - 1.0) * 0.5);
      while (i * (i + 1) / 2 > e) --i;
      while ((i + 1) * (i + 2) / 2 <= e) ++i;
      l = e - i * (i + 1) / 2;
    }
    const int col = red_col(r, i, l);
    double acc8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (e < nl) {
#pragma unroll 1
      for (int b0 = w; b0 < nblk; b0 += 256) {
        double v[32];
#pragma unroll
        for (int u = 0; u < 32; ++u) {
          const int b = b0 + 8 * u;
          v[u] = b < nblk ? r.bpart[(int64_t)b * W + col] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 32; ++u) acc8[u & 7] += v[u];
      }
    }
    part[w][lane] = ((acc8[0] + acc8[1]) + (acc8[2] + acc8[3])) + ((acc8[4] + acc8[5]) + (acc8[6] + acc8[7]));
    __syncthreads();
    if (w == 0 && e < nl) {
      double t = part[0][lane];
      for (int q = 1; q < 8; ++q) t += part[q][lane];
      sM0[i * d + l] = t;
      sM0[l * d + i] = t;
    }
    __syncthreads();
  }
  for (int idx = rank * 256 + threadIdx.x; idx < Jl * d; idx += ncta * 256) {  // group sums
    const int j = idx / d, c = idx % d;
    const int col = r.tnt ? red_col(r, d, c) : c;
    double s = 0.0;
    for (int b = 0; b < r.bpg; ++b) s += r.bpart[(int64_t)(j * r.bpg + b) * W + col];
    if (r.tnt) s += (double)r.N * r.shift[c];
    sS0[idx] = s;
  }
  if (rank == ncta - 1) {  // accepts
    double s = 0.0;
    for (int b = threadIdx.x; b < nblk; b += 256) s += r.bpart[(int64_t)b * W + W - 1];
    s = block_sum(s, red);
    if (threadIdx.x == 0) {
      sx0[0] = s;
      sx0[1] = (double)ctl->err;
    }
  }
  cl.sync();  // every DSMEM write into CTA 0 is visible
  if (f.mode == 1 && rank == 0) tl_end(4);
  if (rank != 0) return;
  unsigned long long* tl = g_tl;
  int tlr = -1;
  if (tl && threadIdx.x == 0 && f.mode == 1) {
    tlr = *g_tl_steps;
    if (tlr >= 0 && tlr < TL_ROWS) tl[tlr * TL_W + 10] = gtimer();
  }
  finalize_body(f, fin_sm);
  if (tlr >= 0 && tlr < TL_ROWS) tl[tlr * TL_W + 11] = gtimer();
}

// Finalize as its own launch (G > 1: after the all-gather of the slices; mode 0).
__global__ void __launch_bounds__(256) k_finalize(FinArgs f) {
  extern __shared__ double fin_sm[];
  if (f.stop_in && *f.stop_in) return;
  finalize_body(f, fin_sm);
}

// Prior precision Sinv = Lprior^-T Lprior^-1 and the whitening factor Linv =
// Lprior^-1 (lower; one block; smem: Linv d x d).
__global__ void k_prior_precision(const double* __restrict__ Lp, int d, double* __restrict__ Sinv,
                                  double* __restrict__ Linv) {
  extern __shared__ double sInv[];
  for (int b = threadIdx.x; b < d; b += blockDim.x) {  // column b of Lp^-1 (lower)
    for (int i = 0; i < d; ++i) {
      double t = (i == b) ? 1.0 : 0.0;
      for (int j = b; j < i; ++j) t -= Lp[i * d + j] * sInv[j * d + b];
      sInv[i * d + b] = (i < b) ? 0.0 : t / Lp[i * d + i];
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) Linv[idx] = sInv[idx];
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int r = idx / d, c = idx % d;
    double s = 0.0;
    for (int k = max(r, c); k < d; ++k) s += sInv[k * d + r] * sInv[k * d + c];
    Sinv[idx] = s;
  }
}

}  // namespace sps
