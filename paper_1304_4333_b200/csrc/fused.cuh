// fused.cuh -- one M step of the binary model with d = k <= 32 (the configs[1] shape) as ONE
// kernel up to the moment reduction: proposal (K8), proposal log-likelihood (K1), Metropolis
// accept (K9) and the moment partials (K6) (Algorithm 2 step 2(c)).
//
// Grid = particle tiles of 64 x observation chunks of [0, t1) (the K1 plan).  Every block
//  (B) forms theta* = theta + Lz z for its tile in shared memory, in place over the tile's
//      normals (DMMA, the k_propose_rb arithmetic: the same values in every chunk block of the
//      tile, so theta* never goes to global memory; Lz / Rp fragments through L1) and
//      lp* = -1/2 |Rp (theta* - mu)|^2, while the first X sub-chunk already streams in;
//  (C) runs the K1 contraction + epilogue of its observation chunk (k_loglik_bin_mma with
//      NTW = 2, H = 1) and writes the chunk partial;
//  (D) takes a ticket; the LAST block of the tile to finish (the tail) sums the tile's chunk
//      partials in chunk order, decides accept (R16; plog(u) precomputed by k_normals), writes
//      the accepted theta* rows, L and lp, and builds the tile's shifted T'T (+ ones column =
//      group-sum partial, accept count) on DMMA -- the k_accept_tile row layout.  With TPR > 1
//      tiles per reduce row, the last tile tail of the row sums the TPR tile rows in order.
// It removes the proposal and accept launches (~9.7 + ~7.7 us per cfg2 step), their dependent-launch
// gaps and the theta* / lp* round trips through L2 -- and measured SLOWER, so it is opt-in
// (SPS_FUSED=1, instantiated for k = 4 and 25): cfg2 run 167.6 vs 149.4 ms.  ncu (full-data step, t = 1000,
// S = 4 chunk blocks per tile): 172.6 vs 125.7 us for K1 alone; the phase-B latency (theta / Z
// loads, two dependent DMMA passes) is paid by all S blocks of a tile while each holds one of
// the SM's 4 register-limited slots, and the tile tails (~8 us of dependent loads, barriers and
// tickets) stretch the last wave; at t <= 32 (S = 1, two waves of 1024 blocks) the kernel takes
// as long as proposal + K1 + accept did (29.4 us from start to the last tail).
#pragma once
#include "mstep.cuh"

namespace sps {

struct FusedArgs {
  const double* X;      // n x KP kernel layout (binary: sign-flipped rows)
  double* theta;        // P x d: read; the accepted rows are overwritten by the tile tails
  double* L;            // P cached log-likelihood (accepted: L*)
  double* lp;           // P prior kernel (accepted: lp*)
  const double* Z;      // P x KP standard normals of this step (R15)
  const double* logu;   // P plog(u) of this step's ACCEPT uniforms
  const double* Lz;     // NP x KP lower factor of Sigma = h V (padded, zeros outside d x d)
  const double* Rp;     // NP x KP Lprior^-1 (padded)
  const double* mu;     // d prior mean
  const double* shift;  // d moment shift c
  double* part;         // [S][P] chunk partials
  double* tpart;        // [tiles][W] tile rows (TPR > 1)
  double* bpart;        // [P / (64 TPR)][W] reduce rows (the k_accept_tile layout)
  unsigned* tick;       // [tiles] chunk tickets, then [rows] row tickets; zero between launches
  Ctl* ctl;
  const int* stop;
  int64_t P;
  double temper;
  uint64_t dmagic;      // ceil(2^32 / d): e / d = (e dmagic) >> 32 for e < 2^16
  int32_t d, t1, chunk, sub, S, TPR;
  uint32_t step0;       // ctl->step_cur = step0 + ctl->steps_done (graph replays)
  int32_t set_step;
};

constexpr int FU_TILE = 64;  // particles per tile (4 warps x 2 n-tiles of 8)

// exp table | X buffer 0 | Z / theta* / X buffer 1 | theta rows (then the rows T) | lp*
__host__ __device__ constexpr int fused_smem_doubles(int KP, int d) {
  return 64 + 2 * FU_TILE * KP + FU_TILE * ((d + 1) & ~1) + FU_TILE;
}

// Ticket increment with acquire-release semantics at GPU scope: the block's earlier global writes
// (ordered before it by the preceding __syncthreads) are visible to whoever observes the new count,
// and the last arrival sees every other block's writes -- no separate MEMBAR.SC.GPU.
__device__ __forceinline__ unsigned ticket_acq_rel(unsigned* p) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.u32 %0, [%1], 1;" : "=r"(old) : "l"(p) : "memory");
  return old;
}

template <int KKD, int REM, int NT>
__global__ void __launch_bounds__(128, 4) k_mstep_bin(FusedArgs a) {
  constexpr int KP = 4 * KKD + (REM ? 4 : 0);  // = round_up(d, 4): X, Z, theta* row stride
  constexpr int KK = KP / 4, NTP = (KP + 7) / 8;
  constexpr int NTRI = NT * (NT + 1) / 2, W = NTRI * 64 + 1;
  static_assert(4 * NTRI * 64 <= 2 * FU_TILE * KP, "T'T warp partials must fit in the two row buffers");
  extern __shared__ __align__(16) double smem[];
  double* sT = smem;                      // 64: exp table 2^(i/64)
  const int d = a.d;
  double* sXa = smem + 64;                // 64 x KP: X sub-chunk buffer 0 (C); warp partials (D)
  double* sZ = sXa + FU_TILE * KP;        // 64 x KP: Z, then theta* in place (B); X buffer 1 (C)
  double* sTh = sZ + FU_TILE * KP;        // 64 x d: theta rows (B), then the rows T (D)
  double* slps = sTh + FU_TILE * ((d + 1) & ~1);  // 64 lp*
  __shared__ __align__(8) uint64_t bar[4];  // 0, 1: X sub-chunks; 2: Z; 3: theta
  __shared__ double smu[KP], shs[KP];
  __shared__ int s_tail;
  __shared__ unsigned char s_acc[FU_TILE];
  __shared__ int red_i[32];
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5, ar = lane >> 2, ac = lane & 3;
  const int tile = blockIdx.x, cy = blockIdx.y;
  const int64_t pb = (int64_t)tile * FU_TILE;
  // this block's observation chunk of [0, t1), streamed in sub-chunks of <= 64 rows
  const int c0 = cy * a.chunk;
  const int c1 = min(c0 + a.chunk, a.t1);
  const int ntot = max(c1 - c0, 0);
  const int sub = a.sub > 0 ? a.sub : ntot;
  auto xbuf = [&](int buf) { return buf ? sZ : sXa; };
  auto issue = [&](int cs, int buf) {
    const unsigned bytes = (unsigned)(min(sub, ntot - cs) * KP * 8);
    mbar_arrive_expect_tx(&bar[buf], bytes);
    bulk_g2s(xbuf(buf), a.X + (int64_t)(c0 + cs) * KP, bytes, &bar[buf]);
  };
  const double tv = tid < 64 ? __ldg(c_exp2tab + tid) : 0.0;
  if (tid == 0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) mbar_init(&bar[i], 1);
    // independent of the predecessor: this step's normals (side stream, complete before this launch)
    // and the first X sub-chunk (loads while theta* is formed)
    mbar_arrive_expect_tx(&bar[2], FU_TILE * KP * 8u);
    bulk_g2s(sZ, a.Z + pb * KP, FU_TILE * KP * 8u, &bar[2]);
    if (ntot > 0) issue(0, 0);
  }
  griddep_wait();  // (programmatic launch) Lz, theta, L, lp of the previous step from here on
  if (a.stop && *a.stop) {  // speculative step after the stop: drain the loads, exit
    if (tid == 0) {
      mbar_wait(&bar[2], 0u);
      if (ntot > 0) mbar_wait(&bar[0], 0u);
    }
    return;
  }
  if (tid == 0) {
    // the tile's theta rows (the previous step's result: after the dependency wait)
    const unsigned tb = (unsigned)(FU_TILE * d * 8);
    mbar_arrive_expect_tx(&bar[3], tb);
    bulk_g2s(sTh, a.theta + pb * d, tb, &bar[3]);
    if (a.set_step && tile == 0 && cy == 0) a.ctl->step_cur = a.step0 + (uint32_t)a.ctl->steps_done;
  }
  if (cy == 0 && tile == 0) tl_start(0);  // (debug timeline: "propose" = phase B)
  if (tid < 64) sT[tid] = tv;
  for (int i = tid; i < KP; i += blockDim.x) {
    smu[i] = i < d ? a.mu[i] : 0.0;
    shs[i] = i < d ? a.shift[i] : 0.0;
  }
  __syncthreads();  // barriers initialised, mu / table staged
  mbar_wait(&bar[2], 0u);
  mbar_wait(&bar[3], 0u);
  // ---- (B) theta* = theta + Z Lz' (in place over the warp's own Z rows) and
  //      lp* = -1/2 |(theta* - mu) Rp'|^2; warp w: rows 16 w .. 16 w + 15.  Lz / Rp B-fragments through
  //      L1 (__ldg: the same 2 x NP x KP doubles for every block of the SM).  The k_propose_rb arithmetic.
#pragma unroll
  for (int rt = 0; rt < 2; ++rt) {
    const int q = w * 16 + rt * 8 + ar;
    double c[NTP][2];
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt) c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const double av = sZ[q * KP + kk * 4 + ac];
#pragma unroll
      for (int nt = 0; nt < NTP; ++nt)  // Lz lower: k-steps above the tile vanish
        if (kk <= 2 * nt + 1) dmma884(c[nt][0], c[nt][1], av, __ldg(a.Lz + (nt * 8 + ar) * KP + kk * 4 + ac));
    }
    __syncwarp();  // the warp's Z reads of these rows precede the theta* writes over them
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = nt * 8 + 2 * ac + e;
        if (i < KP) sZ[q * KP + i] = i < d ? sTh[q * d + i] + c[nt][e] : 0.0;
      }
    __syncwarp();
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt) c[nt][0] = c[nt][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < KK; ++kk) {
      const double av = sZ[q * KP + kk * 4 + ac] - smu[kk * 4 + ac];  // theta* - mu (padding: 0 - 0)
#pragma unroll
      for (int nt = 0; nt < NTP; ++nt)
        if (kk <= 2 * nt + 1) dmma884(c[nt][0], c[nt][1], av, __ldg(a.Rp + (nt * 8 + ar) * KP + kk * 4 + ac));
    }
    double qq = 0.0;
#pragma unroll
    for (int nt = 0; nt < NTP; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) qq = fma(c[nt][e], c[nt][e], qq);
    qq += __shfl_xor_sync(0xffffffffu, qq, 1);
    qq += __shfl_xor_sync(0xffffffffu, qq, 2);
    if (ac == 0) {
      if (!isfinite(qq)) atomicExch(&a.ctl->err, ERR_NUMERIC);
      slps[q] = -0.5 * qq;
    }
  }
  __syncwarp();
  // K1 B-fragments of theta* (registers for the whole chunk; the tail writes them back as rows T)
  double b[2][KKD > 0 ? KKD : 1];
  double tr[2][2][REM > 0 ? REM : 1];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int q = w * 16 + nt * 8 + ar;
#pragma unroll
    for (int kk = 0; kk < KKD; ++kk) b[nt][kk] = sZ[q * KP + kk * 4 + ac];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int qe = w * 16 + nt * 8 + 2 * ac + e;
#pragma unroll
      for (int r = 0; r < REM; ++r) tr[nt][e][r] = sZ[qe * KP + 4 * KKD + r];
    }
  }
  __syncthreads();  // every warp holds its fragments: the Z / theta* rows become X buffer 1
  tl_end(0);
  if (cy == 0 && tile == 0) tl_start(2);
  // ---- (C) K1 on theta* over this block's observation chunk (X buffer 0 already loading)
  if (tid == 0) bulk_fence_smem();  // generic-proxy accesses of the Z / theta* rows precede async-proxy writes
  double M[2][2], Pp[2][2];
  int E[2][2];
#pragma unroll
  for (int nt = 0; nt < 2; ++nt)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      M[nt][e] = 0.0;
      Pp[nt][e] = 1.0;
      E[nt][e] = 0;
    }
  int nit = 0, it = 0;
  for (int cs = 0; cs < ntot; cs += sub) {
    const int nobs = min(sub, ntot - cs);
    const int buf = it & 1;
    if (tid == 0 && cs + sub < ntot) issue(cs + sub, buf ^ 1);  // buf ^ 1 released by the barrier below
    mbar_wait(&bar[buf], (unsigned)(it >> 1) & 1u);
    ++it;
    const double* sXb = xbuf(buf);
    for (int t0 = 0; t0 < nobs; t0 += 8) {
      double acc[2][2];
      acc[0][0] = acc[0][1] = acc[1][0] = acc[1][1] = 0.0;
      const double* xr = sXb + (t0 + ar) * KP;
#pragma unroll
      for (int kk = 0; kk < KKD; ++kk) {
        const double av = xr[kk * 4 + ac];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) dmma884(acc[nt][0], acc[nt][1], av, b[nt][kk]);
      }
#pragma unroll
      for (int r = 0; r < REM; ++r) {
        const double xv = xr[4 * KKD + r];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          acc[nt][0] = fma(xv, tr[nt][0][r], acc[nt][0]);
          acc[nt][1] = fma(xv, tr[nt][1][r], acc[nt][1]);
        }
      }
      if (t0 + ar < nobs) {  // rows past the sub-chunk hold stale data
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            M[nt][e] += relu_bits(acc[nt][e]);
            const double ex = exp_neg(abs_clamp708(acc[nt][e]), sT);
            Pp[nt][e] = fma(Pp[nt][e], ex, Pp[nt][e]);
          }
      }
      if ((++nit & 31) == 0) {
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          renorm(Pp[nt][0], E[nt][0]);
          renorm(Pp[nt][1], E[nt][1]);
        }
      }
    }
    __syncthreads();  // every warp is done with buffer `buf` before it is refilled
  }
  {  // combine the 8 lanes of each particle column (the K1 reduce-scatter, V = 4 values per lane)
    constexpr int V = 4;
    double m[V], pp[V];
    int ex[V];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        renorm(Pp[nt][e], E[nt][e]);
        m[nt * 2 + e] = M[nt][e];
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
            pp[q] = kp * __shfl_xor_sync(0xffffffffu, sp, o);
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
    const int rest = ar >> 2;
    const int q = w * 16 + (jsel >> 1) * 8 + 2 * ac + (jsel & 1);
    if (rest == 0) {
      double pv = pp[0];
      int xv = ex[0];
      renorm(pv, xv);
      a.part[(int64_t)cy * a.P + pb + q] = -(m[0] + (log(pv) + (double)xv * 0x1.62e42fefa39efp-1));
    }
  }
  tl_end(2);
  // ---- (D) the last chunk block of the tile accepts and emits the tile's moment partials
  __syncthreads();
  if (tid == 0) s_tail = a.S == 1 || ticket_acq_rel(&a.tick[tile]) == (unsigned)(a.S - 1);
  __syncthreads();
  if (!s_tail) return;
  griddep_launch();  // the reduce may start its launch
  if (tid == 0 && a.S > 1) a.tick[tile] = 0u;  // re-armed for the next launch (stream order)
  // (thread 0's acquire + the barrier above order the chunk-partial loads below after the other blocks' writes)
  if (tile == 0 && tid == 0 && g_tl) {  // (debug timeline: "accept" = tile 0's tail)
    const int r = *g_tl_steps;
    if (r >= 0 && r < TL_ROWS) g_tl[r * TL_W + 6] = gtimer();
  }
  int ok = 0;
  if (tid < FU_TILE) {
    const int64_t p = pb + tid;
    double Ls = __ldcg(a.part + p);
    for (int c = 1; c < a.S; ++c) Ls += __ldcg(a.part + (int64_t)c * a.P + p);
    if (!isfinite(Ls)) atomicExch(&a.ctl->err, ERR_NUMERIC);
    const double delta = a.temper * (Ls - __ldcg(a.L + p)) + (slps[tid] - __ldcg(a.lp + p));
    if (__ldcg(a.logu + p) < delta) {  // R16: accept iff plog(u) < Delta
      ok = 1;
      a.L[p] = Ls;
      a.lp[p] = slps[tid];
    }
    s_acc[tid] = (unsigned char)ok;
  }
  const int nacc = block_sum(ok, red_i);  // (barrier) s_acc visible
  // rows T in place of the staged theta rows: the accepted ones take theta* from the K1 fragments ...
#pragma unroll
  for (int nt = 0; nt < 2; ++nt) {
    const int q = w * 16 + nt * 8 + ar;
    if (s_acc[q]) {
#pragma unroll
      for (int kk = 0; kk < KKD; ++kk)
        if (kk * 4 + ac < d) sTh[q * d + kk * 4 + ac] = b[nt][kk];
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int qe = w * 16 + nt * 8 + 2 * ac + e;
      if (s_acc[qe]) {
#pragma unroll
        for (int r = 0; r < REM; ++r) sTh[qe * d + 4 * KKD + r] = tr[nt][e][r];
      }
    }
  }
  __syncthreads();
  // ... and go back to theta (flat coalesced over the accepted rows' elements)
  {
    double* th = a.theta + pb * d;
    const int ne = FU_TILE * d;
    for (int e = tid; e < ne; e += blockDim.x) {
      const int q = (int)(((uint64_t)e * a.dmagic) >> 32);
      if (s_acc[q]) th[e] = sTh[e];
    }
  }
  // T'T lower tiles on DMMA, warp w: k-steps over particles k0 = 4 (w + 4 m)
  double shv[NT];
#pragma unroll
  for (int t = 0; t < NT; ++t) shv[t] = shs[min(t * 8 + ar, KP - 1)];
  double cacc[NTRI][2];
#pragma unroll
  for (int t = 0; t < NTRI; ++t) cacc[t][0] = cacc[t][1] = 0.0;
#pragma unroll
  for (int m = 0; m < FU_TILE / 16; ++m) {
    const int q = 4 * (w + 4 * m) + ac;
    const double* row = sTh + q * d;
    double f[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {
      const int i = t * 8 + ar;
      f[t] = i < d ? row[i] - shv[t] : (i == d ? 1.0 : 0.0);
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
  double* wp = sXa;  // 4 x NTRI x 64 warp partials over both row buffers (consumed X buffers)
#pragma unroll
  for (int t = 0; t < NTRI; ++t) {
    wp[(w * NTRI + t) * 64 + lane * 2] = cacc[t][0];
    wp[(w * NTRI + t) * 64 + lane * 2 + 1] = cacc[t][1];
  }
  __syncthreads();
  const int row = tile / a.TPR;
  double* out = a.TPR == 1 ? a.bpart + (int64_t)row * W : a.tpart + (int64_t)tile * W;
  for (int idx = tid; idx < NTRI * 64; idx += blockDim.x)
    out[idx] = ((wp[idx] + wp[NTRI * 64 + idx]) + wp[2 * NTRI * 64 + idx]) + wp[3 * NTRI * 64 + idx];
  if (tid == 0) out[NTRI * 64] = (double)nacc;
  if (a.TPR == 1) {
    tl_end(3);
    return;
  }
  __syncthreads();
  if (tid == 0) s_tail = ticket_acq_rel(&a.tick[gridDim.x + row]) == (unsigned)(a.TPR - 1);
  __syncthreads();
  if (!s_tail) return;
  if (tid == 0) a.tick[gridDim.x + row] = 0u;
  const double* tp0 = a.tpart + (int64_t)row * a.TPR * W;
  double* ob = a.bpart + (int64_t)row * W;
  for (int idx = tid; idx < W; idx += blockDim.x) {
    double s = __ldcg(tp0 + idx);
    for (int u = 1; u < a.TPR; ++u) s += __ldcg(tp0 + (int64_t)u * W + idx);
    ob[idx] = s;
  }
  tl_end(3);
}

}  // namespace sps
