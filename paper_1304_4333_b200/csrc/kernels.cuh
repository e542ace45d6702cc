// kernels.cuh -- SPS phase kernels of libsps.so (sm_100a): data preparation,
// prior draws (K10), C phase (K2/K3 data tempering, K4 power tempering),
// S phase (K5 integer resampling + gather), M phase (K6 moments, K7 finalize
// with Cholesky, K8 propose, K9 accept) and accounting (K11).
// Citations: PAPER.md line numbers; readings R1..R17 in DESIGN.md.
#pragma once
#include "common.cuh"

namespace sps {

enum : int { ERR_NONE = 0, ERR_DATA = 3, ERR_NUMERIC = 4 };

// Device control block: scalars shared between kernels and read back by the host.
struct Ctl {
  int h;           // step scale, hundredths (R6)
  int stop;        // M phase: min RNE >= K after the last step
  int err;         // sticky error code (ERR_*)
  int s_star;      // C phase: first crossing observation (1-based), -1 = none in chunk
  int chol_ridge;  // the last Cholesky needed the ridge retry
  int steps_done;  // M steps executed since the phase began (speculative launches skip)
  unsigned long long acc;  // accepted proposals, this rank, last step
  double minrne;   // min monitor RNE after the last step
  double logml_inc;
  double dphi;     // power tempering increment of the last C phase
  double ess;      // ESS at the cycle end (diagnostic)
  unsigned long long q_lo, q_hi;  // power search bracket on the 2^-48 grid
  int q_ok_full;   // ESS(1 - phi) >= threshold
  uint32_t step_cur;  // M step of the running proposal (written by K8; the next step's normals use step_cur + 1)
};

// ============================================================ data preparation
// Kernel layout of X: n x ldx.  Binary: row t multiplied by (1 - 2 y_t) (exact
// sign flip, R17); padding columns zero.  Validates labels and finiteness.
__global__ void k_prep_X(const double* __restrict__ X, const int32_t* __restrict__ y, int n, int k, int C, int ldx,
                         double* __restrict__ Xs, Ctl* ctl) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)n * ldx) return;
  const int t = (int)(idx / ldx), i = (int)(idx % ldx);
  const int yt = y[t];
  if (i == 0 && (yt < 0 || yt >= C)) atomicExch(&ctl->err, ERR_DATA);
  double v = 0.0;
  if (i < k) {
    v = X[(int64_t)t * k + i];
    if (!isfinite(v)) atomicExch(&ctl->err, ERR_DATA);
    if (C == 2 && yt == 1) v = -v;
  }
  Xs[idx] = v;
}

// Column means xbar of X (default monitors / reported functionals, R12).
__global__ void k_colmeans(const double* __restrict__ X, int n, int k, double* __restrict__ xbar) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= k) return;
  double s = 0.0;
  for (int t = 0; t < n; ++t) s += X[(int64_t)t * k + i];
  xbar[i] = s / (double)n;
}

// Default monitor rows (R12): one per coefficient block c = 1..C-1, the block's
// coordinate mean k^-1 sum_i theta_{c,i} -- not the reported log-odds functionals
// theta_c' xbar.
__global__ void k_default_monitors(int k, int C, double* __restrict__ mon) {
  const int d = k * (C - 1);
  for (int idx = threadIdx.x; idx < (C - 1) * d; idx += blockDim.x) {
    const int row = idx / d, col = idx % d;
    mon[idx] = (col / k == row) ? 1.0 / (double)k : 0.0;
  }
}

// In-place Cholesky (lower) of a d x d row-major matrix in shared memory, one
// block.  Returns false (on all threads) if a pivot is not positive.
__device__ bool block_cholesky(double* A, int d, int* sflag) {
  if (threadIdx.x == 0) *sflag = 1;
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    if (threadIdx.x == 0) {
      const double piv = A[j * d + j];
      if (!(piv > 0.0) || !isfinite(piv))
        *sflag = 0;
      else
        A[j * d + j] = sqrt(piv);
    }
    __syncthreads();
    if (!*sflag) return false;
    const double rjj = 1.0 / A[j * d + j];
    for (int i = j + 1 + threadIdx.x; i < d; i += blockDim.x) A[i * d + j] *= rjj;
    __syncthreads();
    const int m = d - j - 1;
    for (int idx = threadIdx.x; idx < m * m; idx += blockDim.x) {
      const int i = j + 1 + idx / m, l = j + 1 + idx % m;
      if (l <= i) A[i * d + l] -= A[i * d + j] * A[l * d + j];
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x)
    if (idx % d > idx / d) A[idx] = 0.0;
  __syncthreads();
  return true;
}

// Factor the prior covariance (one block; dynamic smem d*d doubles).
__global__ void k_chol_prior(const double* __restrict__ S, int d, double* __restrict__ L, Ctl* ctl) {
  extern __shared__ double sA[];
  __shared__ int flag;
  for (int i = threadIdx.x; i < d * d; i += blockDim.x) sA[i] = S[i];
  __syncthreads();
  const bool ok = block_cholesky(sA, d, &flag);
  if (!ok) {
    if (threadIdx.x == 0) ctl->err = ERR_NUMERIC;
    return;
  }
  for (int i = threadIdx.x; i < d * d; i += blockDim.x) L[i] = sA[i];
}

// g-prior helper (R9): XtX = X'X (k x k), one thread per entry.
__global__ void k_xtx(const double* __restrict__ X, int n, int k, double* __restrict__ out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= k * k) return;
  const int a = idx / k, b = idx % k;
  double s = 0.0;
  for (int t = 0; t < n; ++t) s += X[(int64_t)t * k + a] * X[(int64_t)t * k + b];
  out[idx] = s;
}

// Sigma = g T (X'X)^-1 by Cholesky solves (one block), expanded to the
// normalized d x d prior covariance: block (i, j) = (i == j ? 2 : 1) Sigma.
__global__ void k_g_prior(const double* __restrict__ XtX, int n, int k, int C, double g, double* __restrict__ cov,
                          Ctl* ctl) {
  extern __shared__ double sA[];  // k*k factor + k*k inverse
  __shared__ int flag;
  double* inv = sA + k * k;
  for (int i = threadIdx.x; i < k * k; i += blockDim.x) sA[i] = XtX[i];
  __syncthreads();
  if (!block_cholesky(sA, k, &flag)) {
    if (threadIdx.x == 0) ctl->err = ERR_DATA;
    return;
  }
  for (int b = threadIdx.x; b < k; b += blockDim.x) {  // column b of the inverse
    for (int i = 0; i < k; ++i) {
      double t = (i == b) ? 1.0 : 0.0;
      for (int j = 0; j < i; ++j) t -= sA[i * k + j] * inv[j * k + b];
      inv[i * k + b] = t / sA[i * k + i];
    }
    for (int i = k - 1; i >= 0; --i) {
      double t = inv[i * k + b];
      for (int j = i + 1; j < k; ++j) t -= sA[j * k + i] * inv[j * k + b];
      inv[i * k + b] = t / sA[i * k + i];
    }
  }
  __syncthreads();
  const int d = k * (C - 1);
  for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
    const int r = idx / d, c = idx % d;
    const double s = g * (double)n * inv[(r % k) * k + (c % k)];
    cov[idx] = (r / k == c / k) ? 2.0 * s : s;
  }
}

struct FinArgs {
  const double* gath;  // G slices of `slice_len` doubles (rank order)
  int G, slice_len;
  int J, Jl, N, d;
  double* shift;       // in: c used by the moments; out: new c = theta-bar
  double* Lprop;       // out: chol((h/100) V)
  double* V;           // out: pooled covariance (d x d), or null
  const double* mon;   // monitors (nmon x d)
  int nmon;
  int mode;            // 0: moments of resampled particles (no h / RNE); 1: after an M step
  double K;            // RNE target; <= 0: never stop (fixed number of steps)
  int h_step, h_min, h_max;
  double accept_target;
  Ctl* ctl;
  const int* stop_in;  // skip if already stopped (speculative launches)
  double* rne_out;     // nmon RNEs (may be null)
  Ctl* host_out;       // mapped pinned host slot for the control block (may be null)
  unsigned* ticket;    // k_mom_reduce: arrival counter; the last block runs the finalize (null: separate launch)
  unsigned long long* trace;  // debug (SPS_TRACE): %globaltimer at phase boundaries, or null
  int preloaded;                // cluster reduce: group sums, second moment, accepts, error already in shared memory
  int loop;                     // inside a device-side WHILE node: set its condition after the step
  int rmax;                     // step cap of the M phase (adaptive: max_m_steps; fixed: R)
  cudaGraphConditionalHandle cond;
  int stage_S;         // group sums staged in shared memory (else read from gath)
  // Algorithm 3: the proposal variance Sigma_lr of global M step s (computed here
  // for the step that follows: s = sig_step if >= 0, else ctl->step_cur + 1) is recorded into
  // sig_rec[s] (pass 1) or taken from sig_in[s] instead of (h/100) V (pass 2, fixed design)
  double* sig_rec;     // d x d per step, capacity sig_rec_cap steps (null: not recording)
  int64_t sig_rec_cap;
  const double* sig_in;  // d x d per step, sig_in_n steps (null: adaptive Sigma = (h/100) V)
  int64_t sig_in_n;
  int64_t sig_step;
};

// Reported functional moments (K11) from the gathered
// stats: mean, sd, NSE = [vhat/(JN)]^1/2 (R2), RNE.  One block.
__global__ void __launch_bounds__(256) k_functional_stats(const double* __restrict__ gath, int G, int slice_len, int J,
                                                          int Jl, int N, int d, const double* __restrict__ shift,
                                                          const double* __restrict__ A, int m,
                                                          double* __restrict__ out /* m x 4 */) {
  extern __shared__ double sm[];
  __shared__ double red[32];
  double* sbar = sm;
  double* sg = sm + d;
  const double P = (double)J * (double)N;
  const int gs_len = Jl * d;
  for (int i = threadIdx.x; i < d; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < J; ++j) s += gath[(int64_t)(j / Jl) * slice_len + (j % Jl) * d + i];
    sbar[i] = s / P;
  }
  __syncthreads();
  for (int q = 0; q < m; ++q) {
    const double* a = A + (int64_t)q * d;
    for (int j = threadIdx.x; j < J; j += blockDim.x) {
      const double* S = gath + (int64_t)(j / Jl) * slice_len + (j % Jl) * d;
      double s = 0.0;
      for (int i = 0; i < d; ++i) s = fma(a[i], S[i], s);
      sg[j] = s / (double)N;
    }
    __syncthreads();
    double gp = 0.0;
    for (int j = threadIdx.x; j < J; j += blockDim.x) gp += sg[j];
    const double gbar = block_sum(gp, red) / (double)J;
    double dev = 0.0;
    for (int j = threadIdx.x; j < J; j += blockDim.x) dev += (sg[j] - gbar) * (sg[j] - gbar);
    dev = block_sum(dev, red);
    // sum_p (g - gbar)^2 = a' [M - P (bar - c)(bar - c)'] a
    double quad = 0.0;
    for (int idx = threadIdx.x; idx < d * d; idx += blockDim.x) {
      const int i = idx / d, l = idx % d;
      double mm = 0.0;
      for (int r = 0; r < G; ++r) mm += gath[(int64_t)r * slice_len + gs_len + idx];
      mm -= P * (sbar[i] - shift[i]) * (sbar[l] - shift[l]);
      quad += a[i] * mm * a[l];
    }
    quad = block_sum(quad, red);
    if (threadIdx.x == 0) {
      const double vhat = (double)N / (double)(J - 1) * dev;
      const double var = quad / P;
      out[q * 4 + 0] = gbar;
      out[q * 4 + 1] = sqrt(fmax(var, 0.0));
      out[q * 4 + 2] = sqrt(vhat / P);
      out[q * 4 + 3] = vhat > 0.0 ? var / vhat : INFINITY;
    }
    __syncthreads();
  }
}

// ============================================================ C phase, data tempering (K2/K3)
// K2: cumulative log weights over observations [s0, s0 + B) for every
// particle (PAPER.md:281-295 eq. C_phase_compute in log form):
// lwbuf[b][p] = lw_p(s0 + b + 1).  A block holds SCAN_PB particles and
// SCAN_Q warps: warp q evaluates log p(y_t | theta_p) for its contiguous
// 1/SCAN_Q of the chunk (the latency-bound exp/log1p chains spread over
// SCAN_Q x the threads; cfg2 C phase per run: 9.8 ms at 1 warp, 8.9 at 4, 8.6
// at 8, 8.7 at 16) and stores the terms; then one warp accumulates them per particle
// in observation order (the same serial sum as one thread per particle).
// theta staged transposed in shared memory (d x SCAN_PB).
constexpr int SCAN_PB = 32, SCAN_Q = 8;
constexpr int SCAN_LD = SCAN_PB + 1;  // row stride of the transposed theta tile (odd: conflict-free transposing stores)

__device__ __forceinline__ double scan_term_bin(const double* __restrict__ x, const double* __restrict__ sth, int k,
                                                int pl) {
  double a0 = 0.0, a1 = 0.0;
  int i = 0;
  for (; i + 2 <= k; i += 2) {
    a0 = fma(sth[i * SCAN_LD + pl], __ldg(x + i), a0);
    a1 = fma(sth[(i + 1) * SCAN_LD + pl], __ldg(x + i + 1), a1);
  }
  if (i < k) a0 = fma(sth[i * SCAN_LD + pl], __ldg(x + i), a0);
  const double s = a0 + a1;
  return -(fmax(s, 0.0) + log1p(exp(-fabs(s))));
}

__global__ void __launch_bounds__(SCAN_PB * SCAN_Q) k_cphase_scan(
    const double* __restrict__ Xs, const int32_t* __restrict__ y, int ldx, int k, int C,
    const double* __restrict__ theta, int d, int64_t P, int s0, int B, double* __restrict__ lw_cur,
    double* __restrict__ lwbuf) {
  extern __shared__ double sth[];  // d x SCAN_LD (transposed)
  const int pl = threadIdx.x % SCAN_PB, q = threadIdx.x / SCAN_PB;
  const int64_t p0 = (int64_t)blockIdx.x * SCAN_PB;
  const int np = (int)min((int64_t)SCAN_PB, P - p0);
  {  // the block's np contiguous theta rows, read coalesced (4 loads in flight per thread), stored
     // transposed (a transposed, row-strided read was 20% of the kernel's stall samples)
    const double* src = theta + p0 * d;
    const int tot = np * d;
    for (int e0 = threadIdx.x; e0 < d * SCAN_PB; e0 += 4 * blockDim.x) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * blockDim.x;
        v[u] = e < tot ? src[e] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * blockDim.x;
        if (e < d * SCAN_PB) {
          const int j = e / d, i = e - j * d;  // row j (particle), column i
          sth[i * SCAN_LD + j] = v[u];
        }
      }
    }
  }
  __syncthreads();
  const int64_t p = p0 + pl;
  const bool valid = pl < np;
  const int per = (B + SCAN_Q - 1) / SCAN_Q;
  const int b0 = min(B, q * per), b1 = min(B, b0 + per);
  if (valid) {
    int b = b0;
    if (C == 2) {  // binary: two observations per iteration (ILP)
      for (; b + 2 <= b1; b += 2) {
        const double* x0 = Xs + (int64_t)(s0 + b) * ldx;
        const double la = scan_term_bin(x0, sth, k, pl);
        const double lc = scan_term_bin(x0 + ldx, sth, k, pl);
        lwbuf[(int64_t)b * P + p] = la;
        lwbuf[(int64_t)(b + 1) * P + p] = lc;
      }
      if (b < b1) lwbuf[(int64_t)b * P + p] = scan_term_bin(Xs + (int64_t)(s0 + b) * ldx, sth, k, pl);
    } else {
      for (; b < b1; ++b) {
        const int t = s0 + b;
        const double* x = Xs + (int64_t)t * ldx;
        double eta[8];
        eta[0] = 0.0;
        double m = 0.0;
        for (int c = 1; c < C; ++c) {
          double s = 0.0;
          for (int i = 0; i < k; ++i) s = fma(sth[((c - 1) * k + i) * SCAN_LD + pl], __ldg(x + i), s);
          eta[c] = s;
          m = fmax(m, s);
        }
        int cstar = 0;
        for (int c = 1; c < C; ++c)
          if (eta[c] > eta[cstar]) cstar = c;
        double rest = 0.0;
        for (int c = 0; c < C; ++c)
          if (c != cstar) rest += exp(eta[c] - m);
        lwbuf[(int64_t)b * P + p] = (eta[y[t]] - m) - log1p(rest);
      }
    }
  }
  __syncthreads();  // the block's terms (global, written by this block) visible to warp 0
  if (q != 0 || !valid) return;
  double lw = lw_cur[p];
  int b = 0;
  for (; b + 8 <= B; b += 8) {  // loads batched ahead of the serial adds
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = lwbuf[(int64_t)(b + u) * P + p];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      lw += v[u];
      lwbuf[(int64_t)(b + u) * P + p] = lw;
    }
  }
  for (; b < B; ++b) {
    lw += lwbuf[(int64_t)b * P + p];
    lwbuf[(int64_t)b * P + p] = lw;
  }
  lw_cur[p] = lw;
}

// Per (tile, b): (m, S1 = sum e^(lw - m), S2 = sum e^(2 (lw - m))) over a tile of particles.
__global__ void __launch_bounds__(256) k_ess_partials(const double* __restrict__ lwbuf, int64_t P, int tile,
                                                      double* __restrict__ out /* [B][ntiles][3] */) {
  __shared__ double red[32];
  const int b = blockIdx.y, ti = blockIdx.x, ntiles = gridDim.x;
  const double* v = lwbuf + (int64_t)b * P + (int64_t)ti * tile;
  const int cnt = (int)min((int64_t)tile, P - (int64_t)ti * tile);
  double m = -INFINITY, s1 = 0.0, s2 = 0.0;
  constexpr int EU = 8;  // a tile of <= 8 x blockDim values: all loads in flight, one pass over memory
  if (cnt <= EU * (int)blockDim.x) {  // (the max waited on one load at a time: 46% of the stall samples)
    double x[EU];
#pragma unroll
    for (int u = 0; u < EU; ++u) {
      const int i = threadIdx.x + u * blockDim.x;
      x[u] = i < cnt ? v[i] : -INFINITY;
    }
#pragma unroll
    for (int u = 0; u < EU; ++u) m = fmax(m, x[u]);
    m = block_max(m, red);
#pragma unroll
    for (int u = 0; u < EU; ++u)
      if (threadIdx.x + u * blockDim.x < cnt) {  // the same terms in the same order as the loop below
        const double w = exp(x[u] - m);
        s1 += w;
        s2 += w * w;
      }
  } else {
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) m = fmax(m, v[i]);
    m = block_max(m, red);
    for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
      const double w = exp(v[i] - m);
      s1 += w;
      s2 += w * w;
    }
  }
  s1 = block_sum(s1, red);
  s2 = block_sum(s2, red);
  if (threadIdx.x == 0) {
    double* o = out + ((int64_t)b * ntiles + ti) * 3;
    o[0] = m;
    o[1] = s1;
    o[2] = s2;
  }
}

__device__ __forceinline__ void combine3(double& M, double& S1, double& S2, double m, double s1, double s2) {
  if (m == -INFINITY) return;
  if (M == -INFINITY) {
    M = m;
    S1 = s1;
    S2 = s2;
    return;
  }
  if (m > M) {
    const double e = exp(M - m);
    S1 = S1 * e + s1;
    S2 = S2 * e * e + s2;
    M = m;
  } else {
    const double e = exp(m - M);
    S1 += s1 * e;
    S2 += s2 * e * e;
  }
}

// Combine tiles in order -> this rank's (m, S1, S2) per b.
// One warp per chunk observation b (8 per block): lane l combines tiles l, l + 32, ... in order, then a
// fixed 5-round shuffle tree (deterministic; was one thread looping over all tiles: ~18 us per chunk
// in the launch list, a chain of dependent exps).  ESS_RANK_THREADS still caps the chunk size B.
constexpr int ESS_RANK_THREADS = 256;
__global__ void __launch_bounds__(256) k_ess_rank(const double* __restrict__ parts, int ntiles, int B,
                                                  double* __restrict__ slice) {
  const int lane = threadIdx.x & 31;
  const int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (b >= B) return;  // (warp-uniform)
  double M = -INFINITY, S1 = 0.0, S2 = 0.0;
  for (int t = lane; t < ntiles; t += 32) {
    const double* o = parts + ((int64_t)b * ntiles + t) * 3;
    combine3(M, S1, S2, o[0], o[1], o[2]);
  }
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const double m = __shfl_xor_sync(0xffffffffu, M, off);
    const double s1 = __shfl_xor_sync(0xffffffffu, S1, off);
    const double s2 = __shfl_xor_sync(0xffffffffu, S2, off);
    // both partners combine the same pair in the same order (lower lane first): identical results
    if (lane & off) {
      double mm = m, a1 = s1, a2 = s2;
      combine3(mm, a1, a2, M, S1, S2);
      M = mm;
      S1 = a1;
      S2 = a2;
    } else {
      combine3(M, S1, S2, m, s1, s2);
    }
  }
  if (lane == 0) {
    slice[b * 3 + 0] = M;
    slice[b * 3 + 1] = S1;
    slice[b * 3 + 2] = S2;
  }
}

__global__ void k_ess_final(const double* __restrict__ gath, int G, int B, int s0, int n, double ess_frac, double P,
                            Ctl* ctl, int t_fix, int t_start, double* __restrict__ lse, double* __restrict__ logpl) {
  if (blockDim.x != 32) __trap();  // one warp: lane = observation of a 32-observation round
  const int lane = threadIdx.x;
  double carry = lse && s0 != t_start ? lse[s0] : 0.0;  // lse of the observation before the round
  for (int base = 0; base < B; base += 32) {
    const int b = base + lane;
    const bool in = b < B;
    double M = -INFINITY, S1 = 0.0, S2 = 0.0;
    if (in)
      for (int r = 0; r < G; ++r) {
        const double* o = gath + ((int64_t)r * B + b) * 3;
        combine3(M, S1, S2, o[0], o[1], o[2]);
      }
    const int s = s0 + b + 1;
    const bool cross = in && (t_fix >= 0 ? s == t_fix : (S1 * S1 < ess_frac * P * S2 || s == n));
    const unsigned bal = __ballot_sync(0xffffffffu, cross);
    const int last = bal ? __ffs(bal) - 1 : 31;  // lanes <= last are absorbed this round
    if (lse) {
      const double l = in ? M + log(S1) : 0.0;
      double prev = __shfl_up_sync(0xffffffffu, l, 1);
      if (lane == 0) prev = carry;
      if (in && lane <= last) {
        logpl[s - 1] = l - (s - 1 == t_start ? log(P) : prev);
        lse[s] = l;
      }
      carry = __shfl_sync(0xffffffffu, l, 31);
    }
    if (bal) {
      if (lane == last) {
        ctl->s_star = s;
        ctl->ess = S1 * S1 / S2;
      }
      return;
    }
  }
  if (lane == 0) ctl->s_star = -1;  // no crossing in this chunk
}

// lw_p := lwbuf[b*][p] (the cycle's log weights), L_p += lw_p.
__global__ void k_take_lw(const double* __restrict__ lwbuf, int bstar, int64_t P, double* __restrict__ lw,
                          double* __restrict__ L) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double v = lwbuf[(int64_t)bstar * P + p];
  lw[p] = v;
  L[p] += v;
}

// ============================================================ C phase, power tempering (K4, R5)
__global__ void __launch_bounds__(256) k_block_max(const double* __restrict__ v, int64_t P, double* __restrict__ out) {
  __shared__ double red[32];
  double m = -INFINITY;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, v[i]);
  m = block_max(m, red);
  if (threadIdx.x == 0) out[blockIdx.x] = m;
}

__global__ void k_max_reduce(const double* __restrict__ in, int cnt, double* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double m = -INFINITY;
  for (int i = 0; i < cnt; ++i) m = fmax(m, in[i]);
  *out = m;
}

// Candidate increments dphi_i = ((lo + i w) 2^-48) rem, i = 1..ncand (w = (hi-lo)/64),
// or the single candidate rem when ncand == 0.  Per block partial (S1_i, S2_i).
__device__ __forceinline__ double cand_dphi(const Ctl* ctl, int i, int ncand, double rem) {
  if (ncand == 0) return rem;
  const unsigned long long w = (ctl->q_hi - ctl->q_lo) / 64ull;
  return ((double)(ctl->q_lo + (unsigned long long)i * w) * 0x1p-48) * rem;
}

__global__ void __launch_bounds__(256) k_power_partials(const double* __restrict__ L, int64_t P,
                                                        const double* __restrict__ Lmax, const Ctl* ctl, int ncand,
                                                        double rem, double* __restrict__ out /* [nblk][64][2] */) {
  __shared__ double red[32];
  const double lm = *Lmax;
  const int nc = ncand == 0 ? 1 : ncand;
  for (int c = 0; c < nc; ++c) {
    const double dp = cand_dphi(ctl, c + 1, ncand, rem);
    double s1 = 0.0, s2 = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
      const double w = exp(dp * (L[i] - lm));
      s1 += w;
      s2 += w * w;
    }
    s1 = block_sum(s1, red);
    s2 = block_sum(s2, red);
    if (threadIdx.x == 0) {
      out[((int64_t)blockIdx.x * 64 + c) * 2 + 0] = s1;
      out[((int64_t)blockIdx.x * 64 + c) * 2 + 1] = s2;
    }
  }
}

__global__ void k_power_rank(const double* __restrict__ parts, int nblk, int ncand, double* __restrict__ slice) {
  const int c = threadIdx.x;
  const int nc = ncand == 0 ? 1 : ncand;
  if (c >= nc) return;
  double s1 = 0.0, s2 = 0.0;
  for (int b = 0; b < nblk; ++b) {
    s1 += parts[((int64_t)b * 64 + c) * 2 + 0];
    s2 += parts[((int64_t)b * 64 + c) * 2 + 1];
  }
  slice[c * 2 + 0] = s1;
  slice[c * 2 + 1] = s2;
}

// Combine ranks; ok(c) = !(S1^2 < ess_frac P S2).  ncand == 0: test the full
// remaining increment.  Else narrow [lo, hi) to the last ok candidate's cell.
__global__ void k_power_decide(const double* __restrict__ gath, int G, int ncand, double ess_frac, double P,
                               Ctl* ctl) {
  if (threadIdx.x != 0) return;
  const int nc = ncand == 0 ? 1 : ncand;
  int last_ok = 0;
  for (int c = 0; c < nc; ++c) {
    double s1 = 0.0, s2 = 0.0;
    for (int r = 0; r < G; ++r) {
      s1 += gath[((int64_t)r * 64 + c) * 2 + 0];
      s2 += gath[((int64_t)r * 64 + c) * 2 + 1];
    }
    const bool ok = !(s1 * s1 < ess_frac * P * s2);
    if (ncand == 0) {
      ctl->q_ok_full = ok ? 1 : 0;
      if (ok) ctl->ess = s1 * s1 / s2;
      return;
    }
    if (ok) last_ok = c + 1;
  }
  const unsigned long long w = (ctl->q_hi - ctl->q_lo) / 64ull;
  const unsigned long long lo = ctl->q_lo + (unsigned long long)last_ok * w;
  ctl->q_lo = lo;
  ctl->q_hi = lo + w;
}

__global__ void k_power_apply(const double* __restrict__ L, int64_t P, double dphi, double* __restrict__ lw) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p < P) lw[p] = dphi * L[p];
}

// ============================================================ S phase (K5)
// Integer resampling core of one group (R7), executed by one block.  q (N
// integer weights) in `cum` on entry; on exit counts[n] hold the copies of n.
// a(r) supplies the 52-bit uniform of draw r.
template <typename DrawFn>
__device__ void resample_core(int N, uint64_t* cum, int* counts, int scheme, DrawFn a, uint64_t* scratch) {
  // totals
  uint64_t Q = 0;
  {
    uint64_t part = 0;
    for (int n = threadIdx.x; n < N; n += blockDim.x) part += cum[n];
    uint64_t tot;
    // reuse scan helper for the block total
    block_scan_u64(part, scratch, &tot);
    Q = tot;
  }
  __shared__ unsigned long long sR;
  if (scheme == 0) {
    // residual: c_n = floor(N q_n / Q), r_n = N q_n - c_n Q
    uint64_t csum_part = 0;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
      const uint64_t nq = (uint64_t)N * cum[n];
      const uint64_t c = nq / Q;
      counts[n] = (int)c;
      csum_part += c;
      cum[n] = nq - c * Q;
    }
    uint64_t csum;
    block_scan_u64(csum_part, scratch, &csum);
    if (threadIdx.x == 0) sR = (unsigned long long)N - csum;
  } else {
    for (int n = threadIdx.x; n < N; n += blockDim.x) counts[n] = 0;
  }
  __syncthreads();
  // inclusive prefix sums of cum over n (chunks of blockDim, in order)
  {
    uint64_t carry = 0;
    for (int base = 0; base < N; base += blockDim.x) {
      const int n = base + threadIdx.x;
      const uint64_t v = n < N ? cum[n] : 0ull;
      uint64_t tot;
      const uint64_t inc = block_scan_u64(v, scratch, &tot);
      if (n < N) cum[n] = carry + inc;
      carry += tot;
      __syncthreads();
    }
  }
  __syncthreads();
  const uint64_t R = scheme == 0 ? (uint64_t)sR : (uint64_t)N;
  const uint64_t RQ = scheme == 0 ? R * Q : Q;
  for (uint64_t i = threadIdx.x; i < R; i += blockDim.x) {
    uint64_t pos;
    if (scheme == 1) {
      const unsigned __int128 num = ((unsigned __int128)i << 53) + (unsigned __int128)(2ull * a(0) + 1ull);
      pos = (uint64_t)(((num * (unsigned __int128)Q) / (unsigned __int128)(uint64_t)N) >> 53);
    } else {
      const uint64_t x = 2ull * a((uint32_t)i) + 1ull;
      const uint64_t hi = __umul64hi(x, RQ), lo = x * RQ;
      pos = (hi << 11) | (lo >> 53);
    }
    // first n with cum[n] > pos
    int lo_i = 0, hi_i = N - 1;
    while (lo_i < hi_i) {
      const int mid = (lo_i + hi_i) >> 1;
      if (cum[mid] > pos)
        hi_i = mid;
      else
        lo_i = mid + 1;
    }
    atomicAdd(&counts[lo_i], 1);
  }
  __syncthreads();
}

// Expand counts into the ascending ancestor list (block).
__device__ void counts_to_ancestors(int N, const int* counts, int* anc, uint64_t* scratch) {
  uint64_t carry = 0;
  for (int base = 0; base < N; base += blockDim.x) {
    const int n = base + threadIdx.x;
    const uint64_t c = n < N ? (uint64_t)counts[n] : 0ull;
    uint64_t tot;
    const uint64_t inc = block_scan_u64(c, scratch, &tot);
    if (n < N) {
      const int start = (int)(carry + inc - c);
      for (int q = 0; q < (int)c; ++q) anc[start + q] = n;
    }
    carry += tot;
    __syncthreads();
  }
  __syncthreads();
}

// K5: one block per local group.  q_n = floor(pexp(lw_n -
// max) 2^32) (R7, R8), residual/systematic/multinomial draws from the
// RESAMPLE stream of (global group, cycle), ascending ancestors, gather of
// theta / L / lp into the destination buffers.  Also the group's log-ML
// increment m_j + log(sum_n e^(lw - m_j) / N) (R10) and (m_j, s_j) for the pooled one.
__global__ void __launch_bounds__(1024) k_resample(const double* __restrict__ lw, int N, int d, int scheme,
                                                   uint64_t seed, uint32_t cycle, uint32_t pass, int g0,
                                                   const double* __restrict__ th_src, const double* __restrict__ L_src,
                                                   const double* __restrict__ lp_src, double* __restrict__ th_dst,
                                                   double* __restrict__ L_dst, double* __restrict__ lp_dst,
                                                   double* __restrict__ grp_ms /* [Jl][2] */,
                                                   double* __restrict__ Lj, int* __restrict__ anc_out, Ctl* ctl) {
  extern __shared__ unsigned char smraw[];
  uint64_t* cum = reinterpret_cast<uint64_t*>(smraw);
  int* counts = reinterpret_cast<int*>(cum + N);
  int* anc = reinterpret_cast<int*>(cum);  // reuses cum once the draws are done (12 N bytes of smem)
  __shared__ uint64_t scratch[33];
  __shared__ double red[32];
  const int j = blockIdx.x;
  const uint32_t gj = (uint32_t)(g0 + j);
  const double* w = lw + (int64_t)j * N;
  double m = -INFINITY;
  for (int n = threadIdx.x; n < N; n += blockDim.x) m = fmax(m, w[n]);
  m = block_max(m, red);
  double s = 0.0;
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    s += exp(w[n] - m);
    cum[n] = (uint64_t)floor(__dmul_rn(pexp(__dsub_rn(w[n], m)), 4294967296.0));
  }
  s = block_sum(s, red);
  if (threadIdx.x == 0) {
    grp_ms[j * 2 + 0] = m;
    grp_ms[j * 2 + 1] = s;
    Lj[j] += m + log(s / (double)N);
    if (!isfinite(m)) ctl->err = ERR_NUMERIC;
  }
  auto draw = [&](uint32_t r) -> uint64_t {
    const u4 v = stream_block(seed, r >> 1, gj, cycle, TAG_RESAMPLE, pass);
    return (r & 1u) ? a52(v.z, v.w) : a52(v.x, v.y);
  };
  resample_core(N, cum, counts, scheme, draw, scratch);
  counts_to_ancestors(N, counts, anc, scratch);
  if (anc_out)
    for (int n = threadIdx.x; n < N; n += blockDim.x) anc_out[(int64_t)j * N + n] = anc[n];
  const int64_t base = (int64_t)j * N;
  {  // flat (n, c) walk with incremental row / column (no integer division per element); GU loads in
     // flight per thread before their stores (one dependent load-store pair per element left the
     // gather latency-bound: 42% of k_resample's stall samples on one store, ncu r02)
    constexpr int GU = 8;
    const int sr = (int)blockDim.x / d, sc = (int)blockDim.x - sr * d;
    int n = (int)threadIdx.x / d, c = (int)threadIdx.x - n * d;
    double* dst = th_dst + base * d;
    for (int e0 = (int)threadIdx.x; e0 < N * d; e0 += GU * (int)blockDim.x) {
      double v[GU];
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        v[u] = n < N ? th_src[(base + anc[n]) * d + c] : 0.0;
        n += sr;
        c += sc;
        if (c >= d) {
          c -= d;
          ++n;
        }
      }
#pragma unroll
      for (int u = 0; u < GU; ++u) {
        const int e = e0 + u * (int)blockDim.x;
        if (e < N * d) dst[e] = v[u];
      }
    }
  }
  for (int n = threadIdx.x; n < N; n += blockDim.x) {
    L_dst[base + n] = L_src[base + anc[n]];
    lp_dst[base + n] = lp_src[base + anc[n]];
  }
}

// Pooled log-ML increment from all groups' (m_j, s_j) in group order (R10).
// One warp: lanes take the max and the exps; lane 0 adds the terms in group order.
__global__ void k_logml_pooled(const double* __restrict__ gath_ms, int J, double P, Ctl* ctl, double* inc_out) {
  if (blockDim.x != 32) __trap();  // one warp (full-mask shuffles)
  const int lane = threadIdx.x;
  double M = -INFINITY;
  for (int j = lane; j < J; j += 32) M = fmax(M, gath_ms[j * 2]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmax(M, __shfl_xor_sync(0xffffffffu, M, o));
  double S = 0.0;
  for (int base = 0; base < J; base += 32) {
    const int j = base + lane;
    const double t = j < J ? gath_ms[j * 2 + 1] * exp(gath_ms[j * 2] - M) : 0.0;
    const int cnt = min(32, J - base);
    for (int u = 0; u < cnt; ++u) {
      const double v = __shfl_sync(0xffffffffu, t, u);
      if (lane == 0) S += v;
    }
  }
  if (lane != 0) return;
  ctl->logml_inc = M + log(S / P);
  if (inc_out) *inc_out = ctl->logml_inc;  // per-cycle record, read by the host when needed
}

// NSE of log ML across groups (R10) from the gathered per-group L_j.
__global__ void k_logml_nse(const double* __restrict__ Lj, int J, double* __restrict__ out) {
  if (threadIdx.x != 0) return;
  double s = 0.0;
  for (int j = 0; j < J; ++j) s += Lj[j];
  const double bar = s / (double)J;
  double v = 0.0;
  for (int j = 0; j < J; ++j) v += (Lj[j] - bar) * (Lj[j] - bar);
  *out = sqrt(v / ((double)J * (double)(J - 1)));
}

// ============================================================ test-export kernels
__global__ void k_test_philox(int n, const uint32_t* ctr, uint32_t k0, uint32_t k1, uint32_t* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const u4 r = philox4x32_10(u4{ctr[4 * i], ctr[4 * i + 1], ctr[4 * i + 2], ctr[4 * i + 3]}, k0, k1);
  out[4 * i] = r.x;
  out[4 * i + 1] = r.y;
  out[4 * i + 2] = r.z;
  out[4 * i + 3] = r.w;
}

__global__ void k_test_normals(uint64_t seed, uint32_t id, uint32_t step, uint32_t tag, uint32_t pass, int count,
                               double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i >= count) return;
  double z0, z1;
  normal_pair(seed, (uint32_t)i, id, step, tag, pass, &z0, &z1);
  out[2 * i] = z0;
  if (2 * i + 1 < count) out[2 * i + 1] = z1;
}

__global__ void k_test_portable(int which, int n, const double* x, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (which == 0) out[i] = plog(x[i]);
  if (which == 1) out[i] = pexp(x[i]);
  if (which == 2) psincos2pi(x[i], &out[2 * i], &out[2 * i + 1]);
}

__global__ void __launch_bounds__(1024) k_test_resample_int(int N, const uint64_t* q, int scheme, const uint64_t* a,
                                                            int* anc_out) {
  extern __shared__ unsigned char smraw[];
  uint64_t* cum = reinterpret_cast<uint64_t*>(smraw);
  int* counts = reinterpret_cast<int*>(cum + N);
  int* anc = reinterpret_cast<int*>(cum);
  __shared__ uint64_t scratch[33];
  for (int n = threadIdx.x; n < N; n += blockDim.x) cum[n] = q[n];
  __syncthreads();
  auto draw = [&](uint32_t r) -> uint64_t { return a[r]; };
  resample_core(N, cum, counts, scheme, draw, scratch);
  counts_to_ancestors(N, counts, anc, scratch);
  for (int n = threadIdx.x; n < N; n += blockDim.x) anc_out[n] = anc[n];
}

__global__ void k_test_accept(int64_t P, const double* delta, uint64_t seed, uint32_t step, uint32_t pass,
                              uint8_t* flags) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const u4 w = stream_block(seed, 0u, (uint32_t)p, step, TAG_ACCEPT, pass);
  flags[p] = plog(u01(w.x, w.y)) < delta[p] ? 1 : 0;
}

}  // namespace sps
