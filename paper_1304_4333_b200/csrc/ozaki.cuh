// ozaki.cuh -- K1 for the binary model with 64 <= k <= 128 (configs[3]: k = 100) on the 5th-generation
// tensor cores: the FP64 contraction eta_tp = x~_t' theta_p is reproduced from INT8 tcgen05 MMAs with
// int32 accumulators in TMEM (Ozaki-style splitting), then the same deferred-log
// softplus epilogue as the DMMA kernels.  PAPER.md:129-131 asks for the likelihood "to machine
// accuracy": the split below keeps the contraction error ~1e-13 relative (bar 1e-10 on L_p).
//
// Splitting (exact FP64 steps: scaling by powers of two and subtracting integers):
//   row scale sigma = 2^e, e = ilogb(max_i |v_i|) + 1, so |v_i| / sigma < 1;
//   r = v / sigma; V_0 = rint(64 r), r = 64 r - V_0; V_a = rint(128 r), r = 128 r - V_a (a >= 1)
//   => v = sigma * sum_{a < S} V_a 2^(-6 - 7a) + O(sigma 2^(-6 - 7S)),  |V_a| <= 64 (int8).
// Product: eta = sigma_t tau_p sum_{a,b} X_a T_b 2^(-12 - 7(a + b)); the int8 GEMMs of one level
// L = a + b share a TMEM accumulator (|C_L| <= 7 * 128 * 64^2 < 2^22); levels L > LMAX = S - 1 are
// dropped (their weight <= 2^(-12 - 7 S) k); the epilogue folds adjacent levels in int32
// (C_l 2^7 + C_{l+1} < 2^29) and those exactly in int64 (< 2^62), one rounding to double:
// eta = (double)(sum_L C_L 2^(7 (6 - L))) * sigma_t * tau_p * 2^-54.
//
// Operand images (built by k_oz_slice: one thread per row, 16-byte stores, coalesced) are the UMMA
// K-major SWIZZLE_NONE canonical layout -- core matrices of 8 rows x 16 bytes, row groups at SBO =
// 128 B, 16-byte K chunks at LBO -- so one 1-D bulk copy lands a tile in shared memory ready for
// the MMA descriptors:
//   particle tile (M = 128 rows): [128 doubles tau][S slices][2 KB chunks][16 groups][8][16 B]
//   observation tile (32 rows): [32 doubles sigma][2 KB chunks][S slices][4 groups][8][16 B]
// so one MMA per (K block, theta slice b) takes X slices 0 .. LMAX - b together as its N = 32 (S - b)
// rows and writes D at TMEM column 32 b: the product X_a T_b lands in the column block of its level
// a + b (7 MMAs per K block instead of 28; the A tile is read from shared memory once per MMA).
// Kernel (one CTA per 128-particle tile x observation chunk, 10 warps, warp-specialised):
//   warp 0: producer -- bulk copies of observation tiles through a 3-stage ring;
//   warp 1: TMEM owner + MMA issuer -- per observation tile, KB x S tcgen05.mma.kind::i8
//           (M = 128 particles, N = 32 (S - b), K = 32) into the level accumulators of one of two
//           TMEM buffers (2 x S x 32 columns);
//   warps 2-9: epilogue -- two warps per TMEM lane quarter (thread = particle = TMEM lane, 16 of
//           the 32 columns each): tcgen05.ld of the S levels, fold, scale, branch-free softplus into
//           two per-particle deferred-log products, release the buffer; halves combined at the end.
#pragma once
#include "loglik.cuh"

namespace sps {

constexpr int OZ_S = 7;              // slices per operand
constexpr int OZ_LMAX = OZ_S - 1;    // highest level kept
constexpr int OZ_MT = 128;           // particles per tile (MMA M, TMEM lanes)
constexpr int OZ_NT = 32;            // observations per tile (MMA N)
constexpr int OZ_STAGES = 3;
constexpr int OZ_NPAIR = OZ_S * (OZ_S + 1) / 2;
constexpr int OZ_EW = 8;                 // epilogue warps: 2 per TMEM lane quarter, 16 columns each
constexpr int OZ_THREADS = 64 + 32 * OZ_EW;
static_assert(OZ_S == 7, "the epilogue folds levels (0), (1,2), (3,4), (5,6)");

__host__ __device__ constexpr int oz_slice_bytes(int rows, int KB) { return rows * KB * 32; }
__host__ __device__ constexpr int oz_tile_bytes(int rows, int KB) { return rows * 8 + OZ_S * oz_slice_bytes(rows, KB); }

// Split `rows` rows of v (row stride ld, k used columns) into tile images (rows per tile R = 128 or 32).
// inter = 0 (particle tiles, the A operand): [slice][chunk][row group]; inter = 1 (observation tiles,
// the B operand): [chunk][slice][row group], so that for one K chunk the row groups of slices
// 0 .. m-1 are consecutive (SBO apart) and ONE MMA with N = 32 m covers all of them.
// amax (may be null, X only): per K block, the highest slice index with a nonzero entry in any row
// (atomicMax; zero-initialised by the caller) -- 0/1 covariate columns are exact in slice 0.
__global__ void k_oz_slice(const double* __restrict__ v, int64_t rows, int64_t ld, int k, int KB, int R, int inter,
                           int64_t row0, uint8_t* __restrict__ out, const int* stop, int* amax = nullptr) {
  if (stop && *stop) return;  // speculative M step after the stop
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // image row (row0 + r is the data row)
  const int64_t ntile = (rows + R - 1) / R;
  if (r >= ntile * R) return;
  const int64_t tile = r / R;
  const int rr = (int)(r % R);
  const int64_t drow = row0 + r;
  const bool valid = r < rows;
  const double* src = v + (valid ? drow : 0) * ld;
  double mx = 0.0;
  bool finite = true;
  if (valid)
    for (int i = 0; i < k; ++i) {
      mx = fmax(mx, fabs(src[i]));
      finite = finite && isfinite(src[i]);
    }
  const int e = mx > 0.0 ? ilogb(mx) + 1 : 0;
  uint8_t* tb = out + tile * (int64_t)oz_tile_bytes(R, KB);
  // a non-finite entry makes the row's scale NaN, so every eta of the row -- and L_p -- is NaN, as in
  // the FP64 kernels (sps_loglik's non-finite check, the M phase's numerical-failure flag)
  reinterpret_cast<double*>(tb)[rr] = finite ? ldexp(1.0, e) : __longlong_as_double(0x7ff8000000000000ll);
  const int ngrp = R / 8, nch = 2 * KB;
  double rem[16];
  for (int c = 0; c < nch; ++c) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int i = c * 16 + j;
      rem[j] = (valid && i < k && finite) ? ldexp(src[i], -e) : 0.0;
    }
    int anz = 0;  // highest slice of this chunk with a nonzero entry
#pragma unroll 1
    for (int a = 0; a < OZ_S; ++a) {
      uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const double s = rem[j] * (a == 0 ? 64.0 : 128.0);
        const double q = rint(s);
        rem[j] = s - q;
        w[j >> 2] |= (uint32_t)(uint8_t)(int8_t)(int)q << (8 * (j & 3));
      }
      if (w[0] | w[1] | w[2] | w[3]) anz = a;
      const int64_t grp = inter ? ((int64_t)c * OZ_S + a) * ngrp + rr / 8
                                : (int64_t)a * nch * ngrp + (int64_t)c * ngrp + rr / 8;
      uint8_t* dst = tb + R * 8 + grp * 128 + (rr % 8) * 16;
      *reinterpret_cast<uint4*>(dst) = make_uint4(w[0], w[1], w[2], w[3]);
    }
    if (amax && anz > 0) atomicMax(&amax[c >> 1], anz);
  }
}

// UMMA shared-memory descriptor, K-major SWIZZLE_NONE (version 1, base offset 0).
__device__ __forceinline__ uint64_t oz_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = (uint64_t)(smem_u32(smem) >> 4) & 0x3fffull;
  return a | ((uint64_t)((lbo >> 4) & 0x3fff) << 16) | ((uint64_t)((sbo >> 4) & 0x3fff) << 32) | (1ull << 46);
}
// Instruction descriptor: kind::i8, D = S32, A = B = signed int8, both K-major, M = 128 (N set per MMA,
// bits [17, 23) = N / 8).
constexpr uint32_t OZ_IDESC_BASE = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(OZ_MT >> 4) << 24);

__device__ __forceinline__ void oz_mma(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                       uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(d_tmem),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0u), "r"(0u), "r"(0u), "r"(0u));
}
__device__ __forceinline__ void oz_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void oz_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void oz_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar)) : "memory");
}
// 32 consecutive TMEM columns of this thread's lane (32x32b shape, x32)
// (the registers of tcgen05.ld are defined only after tcgen05.wait::ld: one asm statement, so no use
// of them can be scheduled in between)
__device__ __forceinline__ void oz_tmem_ld32_wait(uint32_t taddr, int32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
// 16 consecutive TMEM columns of this thread's lane at two addresses (32x32b shape, x16), then the wait
__device__ __forceinline__ void oz_tmem_ld16x2_wait(uint32_t ta, uint32_t tb, int32_t (&v)[16], int32_t (&w)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%32];\n\t"
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%33];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(w[0]),
        "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]), "=r"(w[8]), "=r"(w[9]),
        "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
      : "r"(ta), "r"(tb)
      : "memory");
}
__device__ __forceinline__ void oz_tmem_ld16_wait(uint32_t ta, int32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n\t"
      "tcgen05.wait::ld.sync.aligned;\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(ta)
      : "memory");
}
// mbarrier wait that traps instead of hanging (a descriptor or protocol error must fail the launch,
// not wedge the GPU): ~2^31 polls, seconds
__device__ __forceinline__ void oz_wait(uint64_t* bar, unsigned phase) {
  uint32_t done = 0;
  for (uint32_t n = 0;; ++n) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(phase)
                 : "memory");
    if (done) return;
    if (n > (1u << 31)) __trap();
  }
}

struct OzArgs {
  const uint8_t* Ti;   // particle tile images (this launch's theta)
  const uint8_t* Xi;   // observation tile images (X, static)
  const int* xamax;    // [KB] highest nonzero X slice per K block (k_oz_slice); K block 0 always takes all
  double* part;        // [S][P] chunk partials
  int64_t P;
  int32_t t0, t1, chunk;
  const int* stop;
};

template <int KB>
__host__ __device__ constexpr int oz_smem_bytes() {
  return oz_tile_bytes(OZ_MT, KB) + OZ_STAGES * oz_tile_bytes(OZ_NT, KB);
}

// DBG (tools/k1_oz_ab.py --dbg, timing experiments only): 1 = no softplus in the epilogue, 2 = no MMAs
template <int KB, int DBG = 0>
__global__ void __launch_bounds__(OZ_THREADS, 1) k_oz_loglik(OzArgs a) {
  constexpr int TA = oz_tile_bytes(OZ_MT, KB), TB = oz_tile_bytes(OZ_NT, KB);
  constexpr int SA = oz_slice_bytes(OZ_MT, KB), SB = oz_slice_bytes(OZ_NT, KB);
  constexpr uint32_t LBO_A = (OZ_MT / 8) * 128, LBO_B = OZ_S * (OZ_NT / 8) * 128, SBO = 128;
  extern __shared__ __align__(1024) uint8_t ozs[];
  uint8_t* sA = ozs;
  uint8_t* sB = ozs + TA;
  __shared__ __align__(8) uint64_t a_full, full[OZ_STAGES], empty[OZ_STAGES], tfull[2], tempty[2];
  __shared__ uint32_t s_tmem;
  __shared__ int s_amax[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (a.stop && *a.stop) return;
  griddep_wait();  // theta images of this launch
  const int tile = blockIdx.x, cy = blockIdx.y;
  const int c0 = a.t0 + cy * a.chunk;
  const int c1 = min(c0 + a.chunk, a.t1);
  const int ob0 = c0 / OZ_NT, ob1 = (c1 + OZ_NT - 1) / OZ_NT;  // observation tiles [ob0, ob1)
  const int nob = c1 > c0 ? ob1 - ob0 : 0;
  if (threadIdx.x < KB) s_amax[threadIdx.x] = a.xamax ? a.xamax[threadIdx.x] : OZ_S - 1;
  if (threadIdx.x == 0) {
    mbar_init(&a_full, 1);
    for (int s = 0; s < OZ_STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1 + OZ_EW);  // the MMA commit + the epilogue warps (they read the scales)
    }
    for (int u = 0; u < 2; ++u) {
      mbar_init(&tfull[u], 1);
      mbar_init(&tempty[u], OZ_EW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {  // TMEM: 2 buffers x OZ_S levels x 32 columns (<= 512)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&s_tmem)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  oz_fence_before();
  __syncthreads();
  oz_fence_after();
  const uint32_t tmem = s_tmem;
  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(&a_full, (unsigned)TA);
      bulk_g2s(sA, a.Ti + (int64_t)tile * TA, (unsigned)TA, &a_full);
      for (int i = 0; i < nob; ++i) {
        const int s = i % OZ_STAGES;
        if (i >= OZ_STAGES) oz_wait(&empty[s], (unsigned)((i / OZ_STAGES) - 1) & 1u);
        mbar_arrive_expect_tx(&full[s], (unsigned)TB);
        bulk_g2s(sB + s * TB, a.Xi + (int64_t)(ob0 + i) * TB, (unsigned)TB, &full[s]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      oz_wait(&a_full, 0u);
      for (int i = 0; i < nob; ++i) {
        const int s = i % OZ_STAGES, u = i & 1;
        oz_wait(&full[s], (unsigned)(i / OZ_STAGES) & 1u);
        if (i >= 2) oz_wait(&tempty[u], (unsigned)((i >> 1) - 1) & 1u);
        oz_fence_after();
        const uint8_t* bb = sB + s * TB + OZ_NT * 8;
        const uint32_t dbase = tmem + (uint32_t)(u * OZ_S * OZ_NT);
        // theta slice tb against X slices 0 .. LMAX - tb in ONE MMA (N = 32 (LMAX + 1 - tb)): its D starts
        // at column 32 tb, so X_a T_tb lands in the column block of level a + tb; the first MMA of a tile
        // (kb = 0, tb = 0) spans all levels and overwrites, every later one accumulates.  K blocks whose X
        // slices above nx - 1 are all zero (0/1 covariates are exact in slice 0) stop there.
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          const int nx = kb == 0 ? OZ_S : s_amax[kb] + 1;
#pragma unroll
          for (int tb = 0; tb <= OZ_LMAX; ++tb) {
            const int na = min(OZ_LMAX + 1 - tb, nx);
            const uint64_t ad = oz_desc(sA + OZ_MT * 8 + tb * SA + 2 * kb * LBO_A, LBO_A, SBO);
            const uint64_t bd = oz_desc(bb + 2 * kb * LBO_B, LBO_B, SBO);
            const uint32_t idesc = OZ_IDESC_BASE | ((uint32_t)((OZ_NT * na) >> 3) << 17);
            if (DBG != 2) oz_mma(dbase + (uint32_t)(tb * OZ_NT), ad, bd, idesc, (kb > 0 || tb > 0) ? 1u : 0u);
          }
        }
        oz_commit(&empty[s]);  // the stage's operands are consumed once these MMAs complete
        oz_commit(&tfull[u]);  // the accumulators of buffer u are ready
      }
    }
  } else {  // epilogue: warp w accesses TMEM lanes 32 (w % 4) .. + 31, columns 16 h .. + 15 (h = (w - 2) / 4)
    const int q = warp & 3, h = (warp - 2) >> 2;
    const int pl = 32 * q + lane;  // particle of the tile = TMEM lane
    const int64_t p = (int64_t)tile * OZ_MT + pl;
    oz_wait(&a_full, 0u);
    const double wp = reinterpret_cast<const double*>(sA)[pl] * 0x1p-54;  // tau_p 2^-12 2^-42
    __shared__ double sT[64];
    if (warp == 2) {
      sT[lane] = __ldg(c_exp2tab + lane);
      sT[lane + 32] = __ldg(c_exp2tab + lane + 32);
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * OZ_EW) : "memory");  // the epilogue warps
    double M = 0.0, P0 = 1.0, P1 = 1.0;
    int E0 = 0, E1 = 0;
    for (int i = 0; i < nob; ++i) {
      const int s = i % OZ_STAGES, u = i & 1;
      oz_wait(&tfull[u], (unsigned)(i >> 1) & 1u);
      oz_fence_after();
      // levels folded in pairs in int32 (|C_L| < 7 * 2^19: C_l 2^7 + C_{l+1} < 2^29), the pairs in int64 on
      // the ALU (A 2^42 + B 2^28 + C 2^14 + D < 2^62), one conversion: V 2^42 = sum_L C_L 2^(7 (6 - L))
      // (the FP64 pipe is shared with the INT8 MMAs: fold work stays off it)
      const uint32_t tb = tmem + ((uint32_t)(32 * q) << 16) + (uint32_t)(u * OZ_S * OZ_NT + 16 * h);
      double V[16];
      {
        int32_t c0v[16], c1v[16], c2v[16];
        long long acc[16];
        oz_tmem_ld16_wait(tb, c0v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = (long long)c0v[j];
        oz_tmem_ld16x2_wait(tb + 1 * OZ_NT, tb + 2 * OZ_NT, c1v, c2v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = acc[j] * 16384 + (long long)(c1v[j] * 128 + c2v[j]);
        oz_tmem_ld16x2_wait(tb + 3 * OZ_NT, tb + 4 * OZ_NT, c1v, c2v);
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[j] = acc[j] * 16384 + (long long)(c1v[j] * 128 + c2v[j]);
        oz_tmem_ld16x2_wait(tb + 5 * OZ_NT, tb + 6 * OZ_NT, c1v, c2v);
#pragma unroll
        for (int j = 0; j < 16; ++j) V[j] = (double)(acc[j] * 16384 + (long long)(c1v[j] * 128 + c2v[j]));
      }
      oz_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[u]);  // buffer u may take the next tile's MMAs
      const double* sc = reinterpret_cast<const double*>(sB + s * TB) + 16 * h;  // sigma_t of the columns
      const int tb0 = (ob0 + i) * OZ_NT + 16 * h;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int t = tb0 + j;
        // columns outside [c0, c1): s = -1e300 -> relu 0, e^-708 leaves the product unchanged
        const double s_ = (t >= c0 && t < c1) ? V[j] * (wp * sc[j]) : -1e300;  // eta (sign-flipped rows)
        if (DBG == 1) {
          M += s_;
          continue;
        }
        M += relu_bits(s_);
        const double ex = exp_neg(abs_clamp708(s_), sT);
        if (j & 1)
          P1 = fma(P1, ex, P1);
        else
          P0 = fma(P0, ex, P0);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);  // (with the MMA commit) the stage may be refilled
      renorm(P0, E0);
      renorm(P1, E1);
    }
    // per particle: the two halves of its 32 columns live in warps h = 0 and h = 1 (same lane quarter)
    __shared__ double sM[OZ_MT], sPp[OZ_MT];
    __shared__ int sE[OZ_MT];
    double Pp = P0 * P1;  // two factors in [1, 2)
    int E = E0 + E1;
    renorm(Pp, E);
    if (h == 1) {
      sM[pl] = M;
      sPp[pl] = Pp;
      sE[pl] = E;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * OZ_EW) : "memory");
    if (h == 0) {
      M += sM[pl];
      Pp *= sPp[pl];
      E += sE[pl];
      renorm(Pp, E);
      if (p < a.P) a.part[(int64_t)cy * a.P + p] = -(M + (log(Pp) + (double)E * 0x1.62e42fefa39efp-1));
    }
  }
  oz_fence_before();
  __syncthreads();
  if (warp == 1) {
    oz_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
  griddep_launch();
}

}  // namespace sps
