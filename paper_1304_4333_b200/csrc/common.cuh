// common.cuh -- device building blocks of libsps.so (sm_100a).
//
// Philox4x32-10 counter-based streams and the portable elementary functions
// of DESIGN.md R15 (bit-identical to the oracle's independent
// implementation: every + - * / sqrt below is an explicit round-to-nearest
// intrinsic so nvcc cannot contract it into an FMA), plus small reduction
// helpers.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sps {

constexpr uint32_t TAG_INIT = 1, TAG_PROPOSAL = 2, TAG_ACCEPT = 3, TAG_RESAMPLE = 4;

// ----------------------------------------------------------------- Philox
struct u4 {
  uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ u4 philox4x32_10(u4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
  for (int round = 0; round < 10; ++round) {
    if (round > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
#ifdef __CUDA_ARCH__
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
#else
    const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
    const uint32_t lo0 = (uint32_t)p0, hi0 = (uint32_t)(p0 >> 32), lo1 = (uint32_t)p1, hi1 = (uint32_t)(p1 >> 32);
#endif
    c = u4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
  }
  return c;
}

// counter = (block i, id, step, tag | pass << 8), key = seed (R15)
__device__ __forceinline__ u4 stream_block(uint64_t seed, uint32_t i, uint32_t id, uint32_t step, uint32_t tag,
                                           uint32_t pass) {
  return philox4x32_10(u4{i, id, step, tag | (pass << 8)}, (uint32_t)seed, (uint32_t)(seed >> 32));
}

__device__ __forceinline__ uint64_t a52(uint32_t hi, uint32_t lo) { return ((((uint64_t)hi) << 32) | lo) >> 12; }

// u = (2 a + 1) 2^-53, exact
__device__ __forceinline__ double u01(uint32_t hi, uint32_t lo) {
  return __dmul_rn((double)(2ull * a52(hi, lo) + 1ull), 0x1p-53);
}

// ------------------------------------------------- portable elementary functions
// Same operation sequence as oracle/oracle.c or_plog (R15).
__device__ __forceinline__ double plog(double x) {
  const uint64_t b = (uint64_t)__double_as_longlong(x);
  int e = (int)((b >> 52) & 0x7ff) - 1023;
  double m = __longlong_as_double((long long)((b & 0x000fffffffffffffull) | 0x3ff0000000000000ull));
  if (m > 0x1.6a09e667f3bcdp+0) {
    m = __dmul_rn(m, 0.5);
    e = e + 1;
  }
  const double f = __dsub_rn(m, 1.0);
  const double s = __ddiv_rn(f, __dadd_rn(2.0, f));
  const double z = __dmul_rn(s, s);
  double R = 0x1.642c8590b2164p-5;
  R = __fma_rn(z, R, 0x1.8618618618618p-5);
  R = __fma_rn(z, R, 0x1.af286bca1af28p-5);
  R = __fma_rn(z, R, 0x1.e1e1e1e1e1e1ep-5);
  R = __fma_rn(z, R, 0x1.1111111111111p-4);
  R = __fma_rn(z, R, 0x1.3b13b13b13b14p-4);
  R = __fma_rn(z, R, 0x1.745d1745d1746p-4);
  R = __fma_rn(z, R, 0x1.c71c71c71c71cp-4);
  R = __fma_rn(z, R, 0x1.2492492492492p-3);
  R = __fma_rn(z, R, 0x1.999999999999ap-3);
  R = __fma_rn(z, R, 0x1.5555555555555p-2);
  const double two_s = __dmul_rn(2.0, s);
  const double logm = __fma_rn(two_s, __dmul_rn(z, R), two_s);
  const double ed = (double)e;
  return __fma_rn(ed, 0x1.62e42fee00000p-1, __fma_rn(ed, 0x1.a39ef35793c76p-33, logm));
}

// Same operation sequence as or_pexp (x <= 0; x < -708 -> 0, R8).
__device__ __forceinline__ double pexp(double x) {
  if (!(x >= -708.0)) return 0.0;
  const double t = __dmul_rn(x, 0x1.71547652b82fep+0);
  const double kf = floor(__dadd_rn(t, 0.5));
  const double r = __dsub_rn(__dsub_rn(x, __dmul_rn(kf, 0x1.62e42fee00000p-1)), __dmul_rn(kf, 0x1.a39ef35793c76p-33));
  double p = 1.0;
#pragma unroll
  for (int i = 13; i >= 1; --i) p = __dadd_rn(1.0, __dmul_rn(__ddiv_rn(r, (double)i), p));
  const int k = (int)kf;
  const double scale = __longlong_as_double((long long)((uint64_t)(k + 1023) << 52));
  return __dmul_rn(p, scale);
}

// Same operation sequence as or_psincos2pi.
__device__ __forceinline__ void psincos2pi(double u, double* s_out, double* c_out) {
  const double v = __dmul_rn(4.0, u);
  const double q = floor(__dadd_rn(v, 0.5));
  const double f = __dsub_rn(v, q);
  const double a = __dmul_rn(f, 0x1.921fb54442d18p+0);
  const double a2 = __dmul_rn(a, a);
  double sp = 0x1.952c77030ad4ap-49;
  sp = __fma_rn(a2, sp, -0x1.ae7f3e733b81fp-41);
  sp = __fma_rn(a2, sp, 0x1.6124613a86d09p-33);
  sp = __fma_rn(a2, sp, -0x1.ae64567f544e4p-26);
  sp = __fma_rn(a2, sp, 0x1.71de3a556c734p-19);
  sp = __fma_rn(a2, sp, -0x1.a01a01a01a01ap-13);
  sp = __fma_rn(a2, sp, 0x1.1111111111111p-7);
  sp = __fma_rn(a2, sp, -0x1.5555555555555p-3);
  const double s = __fma_rn(a, __dmul_rn(a2, sp), a);
  double cp = 0x1.ae7f3e733b81fp-45;
  cp = __fma_rn(a2, cp, -0x1.93974a8c07c9dp-37);
  cp = __fma_rn(a2, cp, 0x1.1eed8eff8d898p-29);
  cp = __fma_rn(a2, cp, -0x1.27e4fb7789f5cp-22);
  cp = __fma_rn(a2, cp, 0x1.a01a01a01a01ap-16);
  cp = __fma_rn(a2, cp, -0x1.6c16c16c16c17p-10);
  cp = __fma_rn(a2, cp, 0x1.5555555555555p-5);
  cp = __fma_rn(a2, cp, -0x1.0000000000000p-1);
  const double c = __fma_rn(a2, cp, 1.0);
  const int qi = ((int)q) & 3;
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

// Box-Muller pair of block i of stream (seed, id, step, tag, pass).
__device__ __forceinline__ void normal_pair(uint64_t seed, uint32_t i, uint32_t id, uint32_t step, uint32_t tag,
                                            uint32_t pass, double* z0, double* z1) {
  const u4 w = stream_block(seed, i, id, step, tag, pass);
  const double u1 = u01(w.x, w.y), u2 = u01(w.z, w.w);
  const double r = __dsqrt_rn(__dmul_rn(-2.0, plog(u1)));
  double s, c;
  psincos2pi(u2, &s, &c);
  *z0 = __dmul_rn(r, c);
  *z1 = __dmul_rn(r, s);
}

// Debug phase clock (ns); callers place it after a __syncthreads.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t) : : "memory");
  return t;
}

// Debug timeline (SPS_TIMELINE): per M step (row = *g_tl_steps, the step
// index within the phase) and kernel slot k, [2k] = start of block (0,0),
// [2k+1] = latest block end (atomicMax).  Null when disabled.  In constant memory: every kernel
// tests it, and as a __device__ variable that test was a global load on the critical path of every
// thread (ncu: the top stall of the proposal kernel, 9.7% of its samples; K1 after its barrier).
constexpr int TL_W = 28, TL_ROWS = 4096;
__constant__ unsigned long long* g_tl = nullptr;
__constant__ const int* g_tl_steps = nullptr;
__device__ __forceinline__ void tl_start(int k) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    unsigned long long* tl = g_tl;
    if (!tl) return;
    const int r = *g_tl_steps;
    if (r >= 0 && r < TL_ROWS) tl[r * TL_W + 2 * k] = gtimer();
  }
}
__device__ __forceinline__ void tl_mark_any(int slot) {  // calling thread: a phase clock in slot 12..23
  unsigned long long* tl = g_tl;
  if (tl) {
    const int r = *g_tl_steps;
    if (r >= 0 && r < TL_ROWS) tl[r * TL_W + slot] = gtimer();
  }
}
__device__ __forceinline__ void tl_mark(int slot) {  // block (0,0) thread 0: a phase clock in slot 12..23
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    unsigned long long* tl = g_tl;
    if (!tl) return;
    const int r = *g_tl_steps;
    if (r >= 0 && r < TL_ROWS) tl[r * TL_W + slot] = gtimer();
  }
}
__device__ __forceinline__ void tl_max(int slot) {  // thread 0 of every block: latest clock in slot 24..27
  if (threadIdx.x == 0) {
    unsigned long long* tl = g_tl;
    if (!tl) return;
    const int r = *g_tl_steps;
    if (r >= 0 && r < TL_ROWS) atomicMax(&tl[r * TL_W + slot], gtimer());
  }
}
__device__ __forceinline__ void tl_end(int k) {
  if (threadIdx.x == 0) {
    unsigned long long* tl = g_tl;
    if (!tl) return;
    const int r = *g_tl_steps;
    if (r >= 0 && r < TL_ROWS) atomicMax(&tl[r * TL_W + 2 * k + 1], gtimer());
  }
}

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialization may start while its predecessor runs; griddep_wait() blocks
// until the predecessor grid has completed and its writes are visible (a no-op
// without the launch attribute); griddep_launch() lets the successor's CTAs be
// scheduled once every CTA of this grid has called it or exited.
__device__ __forceinline__ void griddep_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

// ----------------------------------------------------------------- async copies
// cp.async (LDGSTS) of 8 bytes global -> shared; all issued copies of a thread
// are waited by cp_async_wait_all (one latency round for a whole staging phase).
__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}

// ----------------------------------------------------------------- TMA bulk copies
// cp.async.bulk global -> shared (one instruction per contiguous tile, bytes a
// multiple of 16, 16-byte aligned), completion counted on an mbarrier.
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// shared -> global bulk copy (TMA; bytes a multiple of 16, both ends 16-byte
// aligned), tracked by the issuing thread's bulk group.  Generic-proxy writes
// of the source must be fenced first (bulk_fence_smem).
__device__ __forceinline__ void bulk_fence_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
// wait until the issuing thread's bulk stores have finished reading shared memory
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ----------------------------------------------------------------- reductions
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Block-wide sum / max; `scratch` holds >= 32 elements; result broadcast to all threads.
template <typename T>
__device__ __forceinline__ T block_sum(T v, T* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    T t = lane < nw ? scratch[lane] : T(0);
    t = warp_sum(t);
    if (lane == 0) scratch[0] = t;
  }
  __syncthreads();
  return scratch[0];
}
__device__ __forceinline__ double block_max(double v, double* scratch) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    double t = lane < nw ? scratch[lane] : -INFINITY;
    t = warp_max(t);
    if (lane == 0) scratch[0] = t;
  }
  __syncthreads();
  return scratch[0];
}

// Inclusive block scan of uint64 (one value per thread); returns the inclusive
// prefix and writes the block total to *total.
__device__ __forceinline__ uint64_t block_scan_u64(uint64_t v, uint64_t* scratch, uint64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  __syncthreads();
  if (lane == 31) scratch[w] = v;
  __syncthreads();
  if (w == 0) {
    uint64_t t = lane < nw ? scratch[lane] : 0ull;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t u = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += u;
    }
    scratch[lane] = t;
  }
  __syncthreads();
  const uint64_t off = w > 0 ? scratch[w - 1] : 0ull;
  *total = scratch[nw - 1];
  __syncthreads();
  return v + off;
}

}  // namespace sps
