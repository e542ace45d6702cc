// sps.cu -- libsps.so: engine (host orchestration of the SPS phases on one
// CUDA stream) and the C ABI declared in include/sps.h.
//
// Algorithm 2 with the phases of Algorithm 1
// (PAPER.md:266-326).  Every arithmetic step runs in the kernels of
// loglik.cuh / kernels.cuh; the host only sequences launches, reads back the
// control scalars (s*, stop flag, h, log-ML increment) and records the trace.
// Multi-GPU: group sharding, one NCCL allgather per exchange step (dlopen'ed
// libnccl.so.2), deterministic rank-order combination so every rank takes
// identical decisions.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "../../include/sps.h"
#include "common.cuh"
#include "kernels.cuh"
#include "loglik.cuh"
#include "mstep.cuh"
#include "fused.cuh"
#include "ozaki.cuh"

using namespace sps;

// ================================================================== NCCL (dlopen)
namespace {
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool load(std::string* why) {
    if (h) return true;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
      h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      *why = "dlopen(libnccl.so.2) failed";
      return false;
    }
    GetUniqueId = (decltype(GetUniqueId))dlsym(h, "ncclGetUniqueId");
    CommInitRank = (decltype(CommInitRank))dlsym(h, "ncclCommInitRank");
    CommDestroy = (decltype(CommDestroy))dlsym(h, "ncclCommDestroy");
    AllGather = (decltype(AllGather))dlsym(h, "ncclAllGather");
    GetErrorString = (decltype(GetErrorString))dlsym(h, "ncclGetErrorString");
    if (!GetUniqueId || !CommInitRank || !CommDestroy || !AllGather) {
      *why = "libnccl.so.2 lacks a required symbol";
      return false;
    }
    return true;
  }
};
NcclApi g_nccl;

// Loopback transport: the ranks of one "group" are contexts of ONE process (one host
// thread per rank, usually on one GPU).  An allgather stages the slice through host
// memory and meets the other ranks at a host barrier -- no kernel ever waits on another
// rank.  Used to test the sharded (G > 1) engine on a single GPU.
constexpr char kLoopMagic[] = "SPS-LOOPBACK-v1";
struct Loopback {
  int G = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  std::vector<char> buf[2];
  void allgather(int rank, const void* send, size_t bytes, void* recv) {
    std::unique_lock<std::mutex> lk(m);
    std::vector<char>& b = buf[gen & 1];
    if (b.size() < (size_t)G * bytes) b.resize((size_t)G * bytes);
    std::memcpy(b.data() + (size_t)rank * bytes, send, bytes);
    const uint64_t my = gen;
    if (++arrived == G) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != my; });
    }
    std::memcpy(recv, buf[my & 1].data(), (size_t)G * bytes);
  }
};
std::mutex g_loop_mu;
std::map<std::string, std::shared_ptr<Loopback>> g_loops;
// The group registered under a loopback id (created by its first rank).
std::shared_ptr<Loopback> loopback_get(const void* id128, int G) {
  const std::string key((const char*)id128, 128);
  std::lock_guard<std::mutex> lk(g_loop_mu);
  auto& lb = g_loops[key];
  if (!lb) {
    lb = std::make_shared<Loopback>();
    lb->G = G;
  }
  return lb;
}
}  // namespace

// ================================================================== context
using LLKernel = void (*)(LLArgs);
struct LLChoice_t {
  LLKernel fn = nullptr;
  int KT = 0, PPT = 1;
  int ppb = 0;          // particles per block (0: LL_THREADS * PPT)
  bool streams = false; // streams X through smem in sub-chunks (any chunk length)
  int tab = 256;        // doubles reserved for the exp table at the start of shared memory
};

struct sps_ctx {
  sps_config cfg{};
  int n = 0, k = 0, C = 0, d = 0, J = 0, N = 0, G = 1, rank = 0, Jl = 0, g0 = 0;
  int64_t P = 0, Pl = 0, p0 = 0;
  // exchange path (gathers, unfused finalize, host-driven M steps): G > 1, or one rank with a real
  // NCCL communicator (cfg.nccl_id + SPS_XCHG_1RANK=1: the multi-GPU code path on one GPU)
  bool xchg = false;
  int ldx = 0, KT = 0, PPT = 1, nmon = 0, dmax = 0, pp = 0, bpg = 0, nblk_mom = 0, ngy_mom = 0;
  int max_chunks = 1, Bmax = 8;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  std::shared_ptr<Loopback> loop;      // loopback transport (tests), else NCCL
  std::vector<char> loop_send, loop_recv;
  // device buffers
  double *X = nullptr, *Xs = nullptr, *mu = nullptr, *Lprior = nullptr, *xbar = nullptr, *mon = nullptr;
  int32_t* y = nullptr;
  double *theta = nullptr, *theta2 = nullptr, *L = nullptr, *L2 = nullptr, *lp = nullptr, *lp2 = nullptr;
  double *lw = nullptr, *lw_cur = nullptr, *theta_s = nullptr, *lp_s = nullptr, *part = nullptr;
  double *gpart = nullptr, *mpart = nullptr, *slice = nullptr, *gath = nullptr;
  double *shift = nullptr, *Lprop = nullptr, *V = nullptr, *rne = nullptr;
  double *lwbuf = nullptr, *essparts = nullptr, *essslice = nullptr, *essgath = nullptr;
  double *lse = nullptr, *logpl = nullptr;  // data tempering: log weight sums (n + 1), log predictives (n)
  double *grp_ms = nullptr, *grp_ms_gath = nullptr, *Lj = nullptr, *Lj_gath = nullptr, *scal = nullptr;
  double *pw_parts = nullptr, *pw_slice = nullptr, *pw_gath = nullptr, *mx_parts = nullptr, *mx_slice = nullptr,
         *mx_gath = nullptr;
  double *fn_A = nullptr, *fn_out = nullptr;
  int fn_cap = 0;
  double* ll_scratch = nullptr;  // sps_loglik chunk partials (grown on demand)
  size_t ll_scratch_cap = 0;
  double* Sinv = nullptr;        // prior precision (d x d)
  double *LpriorP = nullptr, *SinvP = nullptr;  // padded copies (NP x KP) for the DMMA proposal kernel
  double *Rp = nullptr, *RpP = nullptr;          // prior whitening factor Lprior^-1 (d x d) and its padded copy
  double* bpart = nullptr;       // accept+moments block partials
  int tp = 0, QE = 1, W = 0, nblk = 0;
  int acc_tnt = 0, Wt = 0;  // tile-layout accept kernel: tiles per side (0: full-layout kernels), partial row width
  int red_cluster = 0;      // cluster size of the DSMEM reduce + finalize (0: ticket path)
  size_t acc_smem = 0;
  Ctl* hslot = nullptr;          // 2 mapped pinned Ctl slots (pipelined M steps), written by finalize_body
  Ctl* dslot = nullptr;          // device view of hslot
  int* llbad = nullptr;          // sps_loglik: smallest particle with a non-finite sum (device; INT_MAX = none)
  int* hllbad = nullptr;         // mapped pinned [p, t] of the first non-finite sps_loglik term (INT_MAX = none)
  int* dllbad = nullptr;         // device view of hllbad
  unsigned* ticket = nullptr;      // arrival counter of the fused reduce + finalize (k_mom_reduce)
  unsigned long long* trace = nullptr;  // debug (SPS_TRACE): finalize / reduce phase clocks (managed)
  unsigned long long* tl = nullptr;     // debug (SPS_TIMELINE): per-step kernel start / end clocks
  double tl_acc[24] = {};
  int tl_rows = 0;
  double tl_bin[6][8] = {};
  double tl_gap_par[2][2] = {};  // next-propose gap by step parity within the phase: sum, count  // by t_l bin (<=32, <=64, <=128, <=256, <=512, >512): steps, K1 span, step span, gap
  double trace_acc[80] = {};
  int trace_n = 0;
  double* Zbuf[2] = {nullptr, nullptr};  // standard normals, one M step ahead (side stream)
  double* LUbuf[2] = {nullptr, nullptr}; // plog of the ACCEPT uniforms, same schedule
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_zready[2] = {nullptr, nullptr}, ev_zfree[2] = {nullptr, nullptr};
  cudaEvent_t evs[2] = {nullptr, nullptr};
  // M steps replayed from CUDA graphs (one per slot parity, captured per M phase; one rank)
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaGraphExec_t gexec[2] = {nullptr, nullptr};
  int64_t g_launches[2] = {0, 0}, g_k1[2] = {0, 0};
  double g_pairs[2] = {0, 0};
  int graph_updates = 0, graph_instantiations = 0;
  bool capturing = false;  // inside build_mstep_graphs / build_mstep_loop
  // device-side M phase: one WHILE graph node whose body is one M step (one rank)
  bool capturing_loop = false;
  cudaGraphExec_t gloop = nullptr;
  cudaGraphConditionalHandle loop_cond = 0;
  int loop_rmax = 0;
  int64_t gl_launches = 0, gl_k1 = 0;
  double gl_pairs = 0;
  LLChoice_t llc{};
  int ll_regs = 0;
  // fused M step (binary, d <= 32): propose + K1 + accept + tile moments in one kernel (fused.cuh)
  void (*fu_fn)(FusedArgs) = nullptr;
  size_t fu_smem = 0;
  int fu_TPR = 1;
  unsigned* fu_tick = nullptr;
  double* fu_tpart = nullptr;
  // K1 on INT8 tensor cores (binary, 64 <= k <= 128; ozaki.cuh): K-blocks of 32, operand images
  int oz_KB = 0, oz_min_range = 512;
  uint8_t* oz_X = nullptr;  // observation tile images (built once at create)
  int* oz_xamax = nullptr;  // [KB] highest nonzero X slice per K block
  uint8_t* oz_T = nullptr;  // particle tile images of the theta of the current launch
  size_t oz_T_cap = 0;
  struct Plan {
    int64_t P = -1;
    int range = -1, max_chunks = -1, S = 1, chunk = 0, sub = 0, occ = 1;
    size_t smem = 0;
  } plans[8];
  int plan_next = 0;
  Ctl* ctl = nullptr;
  Ctl* hctl = nullptr;  // pinned mirror
  char* slab = nullptr;  // pooled pinned mapped slab holding hctl, hslot, hllbad
  // debug memory check (SPS_GUARD=1 at create): every device buffer between two guard zones
  struct Guard {
    char* base;
    size_t bytes;  // user bytes (the buffer is [base + GUARD_BYTES, base + GUARD_BYTES + bytes))
    const char* name;
  };
  bool guarded = false;
  std::vector<Guard> guards;
  int slice_len = 0;
  // host state (Algorithm 2)
  int t = 0;            // observations absorbed
  double phi = 0.0;     // tempering level (power mode)
  int ell = 0;          // cycles completed
  uint32_t mstep = 0;   // global M-step counter (PROPOSAL / ACCEPT streams)
  uint32_t phase_step0 = 0;  // first M step of the running M phase
  bool need_pre_moments = false;
  bool cphase_done = false;  // a C phase ran since the last M phase
  bool finished = false;
  double logml = 0.0, pairs = 0.0;
  std::vector<int> tr_t, tr_R, tr_h;
  std::vector<double> tr_phi, tr_inc, tr_rne;
  // log-ML increments are recorded on the device (inc_dev, cycles inc_base..ell-1) and pulled to the
  // host (tr_inc, logml, in cycle order) only when needed: no host round trip per C phase
  double* inc_dev = nullptr;
  int inc_cap = 1024, inc_base = 0;
  int last_adv = 0;  // observations absorbed by the last data-tempering C phase (first galloping chunk)
  int64_t pre_normals_step = -1;  // the first M step's normals were launched by the C phase (step number)
  // Algorithm 3: Sigma_lr record of pass 1, fixed design of pass 2
  bool recording = false;
  double* sig_rec = nullptr;     // d x d per global M step
  int64_t sig_rec_cap = 0;
  double* sig_in = nullptr;      // fixed design: d x d per global M step
  int64_t sig_in_n = 0;
  std::vector<int> des_t, des_R;
  std::vector<double> des_phi;
  // counters (sps_get_counters)
  int64_t launches = 0, k1_launches = 0, syncs = 0;
  double k1_pairs = 0.0, k1_ms = 0.0;
  bool profiling = false;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double cat_ms[16] = {0};
  int64_t cat_n[16] = {0};
  std::vector<cudaEvent_t> prof_pool;         // event pairs, resolved lazily (no per-launch sync)
  std::vector<std::pair<int, int>> prof_open; // (event index pair base, category) awaiting resolution
  int prof_next = 0;
  int prof_cur = -1;
  double host_launch_us = 0.0, host_wait_us = 0.0, host_graph_us = 0.0;
  std::string err;
};

namespace {

enum Cat { CAT_K1 = 0, CAT_PROPOSE, CAT_ACCEPT, CAT_REDUCE, CAT_GATHER, CAT_FINALIZE, CAT_COPY, CAT_CPHASE,
           CAT_RESAMPLE, CAT_OTHER, NCAT };

sps_status fail(sps_ctx* c, sps_status st, const char* fmt, ...) {
  if (c) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    c->err = buf;
  }
  return st;
}

#define CU(c, x)                                                                                        \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) return fail((c), SPS_E_CUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), \
                                       __FILE__, __LINE__);                                             \
  } while (0)
#define CHECK_LAUNCH(c)        \
  do {                         \
    (c)->launches += 1;        \
    CU(c, cudaGetLastError()); \
  } while (0)
// Profiling (sps_set_profiling): bracket one enqueued operation with a pair of
// pooled events on the context stream; pairs are resolved (synchronized) only
// when the counters are read, so launches stay back to back.
sps_status prof_begin(sps_ctx* c);
sps_status prof_end(sps_ctx* c, int cat);
#define PROF_BEGIN(c) \
  if ((c)->profiling) TRY(prof_begin(c))
#define PROF_END(c, cat) \
  if ((c)->profiling) TRY(prof_end(c, cat))

#define TRY(x)                         \
  do {                                 \
    sps_status s_ = (x);               \
    if (s_ != SPS_OK) return s_;       \
  } while (0)

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its stream predecessor runs and synchronizes with griddep_wait().
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
  static const bool off = getenv("SPS_NO_PDL") != nullptr;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = off ? 0 : 1;
  return cudaLaunchKernelEx(&lc, kern, args...);
}

// Cluster launch (cluster of `cl` CTAs along x) with programmatic stream serialization.
template <typename... KArgs, typename... Args>
cudaError_t launch_cluster_pdl(void (*kern)(KArgs...), int cl, dim3 block, size_t smem, cudaStream_t st,
                               Args... args) {
  static const bool off = getenv("SPS_NO_PDL") != nullptr;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3((unsigned)cl);
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = st;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = (unsigned)cl;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = off ? 1 : 2;
  return cudaLaunchKernelEx(&lc, kern, args...);
}

// NVTX ranges on the host calls (C phase, S phase, M phase, run, loglik) for timeline tools; a no-op
// unless a tool is injected (NVTX_INJECTION64_PATH)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
  NvtxRange(const NvtxRange&) = delete;
  NvtxRange& operator=(const NvtxRange&) = delete;
};

constexpr size_t GUARD_BYTES = 256;   // guard zone before and after each buffer (SPS_GUARD=1)
constexpr unsigned char GUARD_FILL = 0xA5;

template <typename T>
sps_status dalloc(sps_ctx* c, T** p, size_t count, const char* name = "?") {
  // stream-ordered allocation from the device's default pool (release threshold raised once per
  // device): a new context reuses memory cached by earlier ones instead of driver allocations
  const size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  if (!c->guarded) {
    CU(c, cudaMallocAsync((void**)p, bytes, c->stream));
    return SPS_OK;
  }
  // debug: [guard | buffer | guard], both zones filled with GUARD_FILL and verified by
  // sps_check_guards (an out-of-bounds write by any kernel lands in a zone)
  char* base = nullptr;
  CU(c, cudaMallocAsync((void**)&base, bytes + 2 * GUARD_BYTES, c->stream));
  CU(c, cudaMemsetAsync(base, GUARD_FILL, GUARD_BYTES, c->stream));
  CU(c, cudaMemsetAsync(base + GUARD_BYTES + bytes, GUARD_FILL, GUARD_BYTES, c->stream));
  c->guards.push_back(sps_ctx::Guard{base, bytes, name});
  *p = reinterpret_cast<T*>(base + GUARD_BYTES);
  return SPS_OK;
}
#define DALLOC(c, p, n) dalloc(c, p, n, #p)

// Free a dalloc'd buffer (stream-ordered); with guards, the allocation starts GUARD_BYTES earlier.
void dfree(sps_ctx* c, void* p, cudaStream_t s) {
  if (!p) return;
  if (c->guarded) {
    for (size_t i = 0; i < c->guards.size(); ++i)
      if (c->guards[i].base + GUARD_BYTES == (char*)p) {
        cudaFreeAsync(c->guards[i].base, s);
        c->guards.erase(c->guards.begin() + (std::ptrdiff_t)i);
        return;
      }
  }
  cudaFreeAsync(p, s);
}

// Pinned, mapped host slabs for a context's control mirrors ([hctl | hslot x 2 | hllbad x 2 | init
// word]), pooled per process: cudaHostAlloc / cudaFreeHost cost milliseconds per context (cudaFreeHost
// alone 4.5-6.4 ms in sps_destroy), which the end-to-end path (create, run, destroy per run) paid.
constexpr size_t SLAB_CTL = (sizeof(Ctl) + 127) / 128 * 128;
constexpr size_t SLAB_BYTES = 3 * SLAB_CTL + 128;
std::mutex g_slab_mu;
std::vector<char*> g_slabs;
char* slab_get() {
  {
    std::lock_guard<std::mutex> lk(g_slab_mu);
    if (!g_slabs.empty()) {
      char* s = g_slabs.back();
      g_slabs.pop_back();
      return s;
    }
  }
  // pool empty: one allocation carved into 16 slabs (the first context pays the host allocation for
  // the next 15 -- e.g. the end-to-end contexts created beside a live one)
  constexpr int NSLAB = 16;
  char* s = nullptr;
  if (cudaHostAlloc((void**)&s, NSLAB * SLAB_BYTES, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess)
    return nullptr;
  std::lock_guard<std::mutex> lk(g_slab_mu);
  for (int q = NSLAB - 1; q >= 1; --q) g_slabs.push_back(s + (size_t)q * SLAB_BYTES);
  return s;
}
void slab_put(char* s) {
  if (!s) return;
  std::lock_guard<std::mutex> lk(g_slab_mu);
  g_slabs.push_back(s);
}

int num_sms() {
  int dev = 0, v = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
  return v;
}

sps_status gather(sps_ctx* c, const double* send, double* recv, size_t count) {
  if (!c->xchg) {  // single rank: the gathered buffer aliases the local slice
    if (send != recv) CU(c, cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    return SPS_OK;
  }
  if (c->loop) {
    const size_t bytes = count * sizeof(double);
    if (c->loop_send.size() < bytes) c->loop_send.resize(bytes);
    if (c->loop_recv.size() < bytes * c->G) c->loop_recv.resize(bytes * c->G);
    CU(c, cudaMemcpyAsync(c->loop_send.data(), send, bytes, cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    c->loop->allgather(c->rank, c->loop_send.data(), bytes, c->loop_recv.data());
    CU(c, cudaMemcpyAsync(recv, c->loop_recv.data(), bytes * c->G, cudaMemcpyHostToDevice, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
    return SPS_OK;
  }
  ncclResult_t r = g_nccl.AllGather(send, recv, count, ncclFloat64, c->comm, c->stream);
  if (r != ncclSuccess) return fail(c, SPS_E_NCCL, "ncclAllGather: %s", g_nccl.GetErrorString(r));
  return SPS_OK;
}

sps_status prof_begin(sps_ctx* c) {
  if ((size_t)c->prof_next + 2 > c->prof_pool.size()) {
    for (int q = 0; q < 256; ++q) {
      cudaEvent_t e;
      CU(c, cudaEventCreate(&e));
      c->prof_pool.push_back(e);
    }
  }
  c->prof_cur = c->prof_next;
  c->prof_next += 2;
  CU(c, cudaEventRecord(c->prof_pool[c->prof_cur], c->stream));
  return SPS_OK;
}

sps_status prof_end(sps_ctx* c, int cat) {
  CU(c, cudaEventRecord(c->prof_pool[c->prof_cur + 1], c->stream));
  c->prof_open.push_back({c->prof_cur, cat});
  return SPS_OK;
}

sps_status prof_resolve(sps_ctx* c) {
  if (c->prof_open.empty()) return SPS_OK;
  CU(c, cudaStreamSynchronize(c->stream));
  for (auto& pr : c->prof_open) {
    float ms = 0.f;
    CU(c, cudaEventElapsedTime(&ms, c->prof_pool[pr.first], c->prof_pool[pr.first + 1]));
    c->cat_ms[pr.second] += ms;
    c->cat_n[pr.second] += 1;
    if (pr.second == 0) c->k1_ms += ms;
  }
  c->prof_open.clear();
  c->prof_next = 0;
  return SPS_OK;
}

// Read back the control block (synchronizes the stream); maps device errors.
sps_status read_ctl(sps_ctx* c) {
  CU(c, cudaMemcpyAsync(c->hctl, c->ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  c->syncs += 1;
  if (c->hctl->err == ERR_DATA) return fail(c, SPS_E_DATA, "invalid data (label out of range or non-finite X)");
  if (c->hctl->err == ERR_NUMERIC)
    return fail(c, SPS_E_NUMERIC, "numerical failure (non-finite log-likelihood, weight collapse or Cholesky "
                                  "failure after ridge; cf. PAPER.md:1024-1030)");
  return SPS_OK;
}

// ------------------------------------------------------------------ K1 dispatch
template <int K, int CM1, int PPT, int TAB = 64, int MINB = 2>
LLKernel ll_ptr() {
  if constexpr (CM1 == 1)
    return k_loglik_bin<K, PPT>;
  else
    return k_loglik_mnl<K, CM1, PPT, TAB, MINB>;
}

// Instantiated shapes: binary k = 1..32 (PPT 2) and {40,48,56,64} (PPT 1);
// C-1 = 2: k = 1..16 (PPT 2 up to 12); C-1 = 3: k = 1..16; C-1 = 4..7: k in {4, 8}.
// Other k round up to the next instantiated KT (zero padding in X and theta loads).
using LLChoice = LLChoice_t;

template <int CM1, int PPT, int TAB = 64, int MINB = 2, int... Ks>
bool pick_exact(int k, LLChoice* out, std::integer_sequence<int, Ks...>) {
  bool found = false;
  ((k == Ks + 1 && !found ? (out->fn = ll_ptr<Ks + 1, CM1, PPT, TAB, MINB>(), out->KT = Ks + 1, out->PPT = PPT, found = true)
                          : false),
   ...);
  return found;
}

bool choose_ll(int k, int C, LLChoice* o) {
  const int cm1 = C - 1;
  static const bool force_dfma = getenv("SPS_K1_DFMA") != nullptr;
  // tuning hook (tools/k1_variants.py): the previous 4-n-tile layout for k = 25
  static const char* k1var = getenv("SPS_K1_VAR");
  if (k1var && cm1 == 1 && k == 25) {
    if (!strcmp(k1var, "w4")) *o = {k_loglik_bin_mma<6, 1, 4>, 28, 1, 128, true};
    else if (!strcmp(k1var, "h2")) *o = {k_loglik_bin_mma<6, 1, 2, 2>, 28, 1, 64, true};        // 16 obs per update
    else if (!strcmp(k1var, "ks2")) *o = {k_loglik_bin_mma<6, 1, 2, 1, 64, 2>, 28, 1, 64, true};  // 2 DMMA chains over k
    else if (!strcmp(k1var, "h2ks2")) *o = {k_loglik_bin_mma<6, 1, 2, 2, 64, 2, 4>, 28, 1, 64, true};
    else if (!strcmp(k1var, "m5")) *o = {k_loglik_bin_mma<6, 1, 2, 1, 64, 1, 5>, 28, 1, 64, true};    // <= 102 registers
    else if (!strcmp(k1var, "m6")) *o = {k_loglik_bin_mma<6, 1, 2, 1, 64, 1, 6>, 28, 1, 64, true};    // <= 85 registers
    if (o->fn) return true;
  }
  // DMMA contraction (+ <= 2 remainder DFMAs), 2 n-tiles (16 particles) per warp, 64 per block:
  // 114 registers -> 4 blocks per SM (the 4-n-tile layout, 178 registers, held 2; cfg2 run -6%)
  static const int tabv = getenv("SPS_K1_TAB") ? atoi(getenv("SPS_K1_TAB")) : 64;
  if (cm1 == 1 && k <= 32 && !force_dfma) {
    switch (k) {
  // exp table (SPS_K1_TAB, A/B switch): 2^(j/64) (default, 9-op exp) or 2^(j/256) (8 ops, 1% slower:
  // bank conflicts); 2^(j/1024) (7 ops) and an fp32 second-order term (5 FP64 ops) measured 10% slower
#define MMA_CASE(K_, KKD_, REM_)                                                                            \
  case K_:                                                                                                  \
    if (tabv == 256)                                                                                        \
      *o = {k_loglik_bin_mma<KKD_, REM_, 2, 1, 256>, 4 * KKD_ + (REM_ ? 4 : 0), 1, 64, true, 256};        \
    else                                                                                                    \
      *o = {k_loglik_bin_mma<KKD_, REM_, 2>, 4 * KKD_ + (REM_ ? 4 : 0), 1, 64, true, 256};                \
    return true;
      MMA_CASE(1, 0, 1) MMA_CASE(2, 0, 2) MMA_CASE(3, 1, 0) MMA_CASE(4, 1, 0) MMA_CASE(5, 1, 1) MMA_CASE(6, 1, 2)
      MMA_CASE(7, 2, 0) MMA_CASE(8, 2, 0) MMA_CASE(9, 2, 1) MMA_CASE(10, 2, 2) MMA_CASE(11, 3, 0) MMA_CASE(12, 3, 0)
      MMA_CASE(13, 3, 1) MMA_CASE(14, 3, 2) MMA_CASE(15, 4, 0) MMA_CASE(16, 4, 0) MMA_CASE(17, 4, 1)
      MMA_CASE(18, 4, 2) MMA_CASE(19, 5, 0) MMA_CASE(20, 5, 0) MMA_CASE(21, 5, 1) MMA_CASE(22, 5, 2)
      MMA_CASE(23, 6, 0) MMA_CASE(24, 6, 0) MMA_CASE(25, 6, 1) MMA_CASE(26, 6, 2) MMA_CASE(27, 7, 0)
      MMA_CASE(28, 7, 0) MMA_CASE(29, 7, 1) MMA_CASE(30, 7, 2) MMA_CASE(31, 8, 0) MMA_CASE(32, 8, 0)
#undef MMA_CASE
      default: break;
    }
  }
  if (cm1 == 1 && k <= 128 && !force_dfma) {  // wide: 2 n-tiles per warp (64 particles per block), k padded to 4
    switch ((k + 3) / 4) {
#define MMA_W(KK_)                                                                      \
  case KK_:                                                                             \
    *o = {k_loglik_bin_mma<KK_, 0, 2>, 4 * KK_, 1, 64, true, 256};                       \
    return true;
      MMA_W(9) MMA_W(10) MMA_W(11) MMA_W(12) MMA_W(13) MMA_W(14) MMA_W(15) MMA_W(16) MMA_W(17) MMA_W(18)
      MMA_W(19) MMA_W(20) MMA_W(21) MMA_W(22) MMA_W(23) MMA_W(24) MMA_W(25) MMA_W(26) MMA_W(27) MMA_W(28)
      MMA_W(29) MMA_W(30) MMA_W(31) MMA_W(32)
#undef MMA_W
      default: break;
    }
  }
  if (cm1 == 1) {
    if (k <= 32) return pick_exact<1, 2>(k, o, std::make_integer_sequence<int, 32>{});
    if (k <= 40) { *o = {ll_ptr<40, 1, 1>(), 40, 1}; return true; }
    if (k <= 48) { *o = {ll_ptr<48, 1, 1>(), 48, 1}; return true; }
    if (k <= 56) { *o = {ll_ptr<56, 1, 1>(), 56, 1}; return true; }
    if (k <= 64) { *o = {ll_ptr<64, 1, 1>(), 64, 1}; return true; }
    return false;
  }
  // multinomial contraction on DMMA (k_loglik_mnl_mma): classes as n-tiles, 64 particles per block
  // (C - 1 <= 3) / 32 (C - 1 <= 7); SPS_MNL_DFMA: the DFMA kernel below (A/B)
  static const bool mnl_dfma = getenv("SPS_MNL_DFMA") != nullptr;
  if (cm1 >= 2 && cm1 <= 3 && k <= 16 && !mnl_dfma) {
    // C - 1 = 3: one n-tile group (8 particles) per warp, 32 per block -- measured fastest on configs[2]
    // (full-data K1 3.16 ms vs 3.32 ms with two groups and k padded to 12, 3.40 ms with two groups and
    // remainder DFMAs, 3.45 ms DFMA kernel; tools/k1_mnl_ab.py); C - 1 = 2: two groups
#define MNL_CASE(K_, KKD_, REM_)                                                                              \
  case K_:                                                                                                    \
    if (cm1 == 2)                                                                                             \
      *o = LLChoice{k_loglik_mnl_mma<KKD_, REM_, 2>, 4 * KKD_ + (REM_ ? 4 : 0), 1, 64, true, 256};             \
    else                                                                                                      \
      *o = LLChoice{k_loglik_mnl_mma<KKD_, REM_, 3, 1>, 4 * KKD_ + (REM_ ? 4 : 0), 1, 32, true, 256};          \
    return true;
    switch (k) {
      MNL_CASE(1, 0, 1) MNL_CASE(2, 0, 2) MNL_CASE(3, 1, 0) MNL_CASE(4, 1, 0) MNL_CASE(5, 1, 1) MNL_CASE(6, 1, 2)
      MNL_CASE(7, 2, 0) MNL_CASE(8, 2, 0) MNL_CASE(9, 2, 1) MNL_CASE(10, 2, 2) MNL_CASE(11, 3, 0) MNL_CASE(12, 3, 0)
      MNL_CASE(13, 3, 1) MNL_CASE(14, 3, 2) MNL_CASE(15, 4, 0) MNL_CASE(16, 4, 0)
      default: break;
    }
#undef MNL_CASE
  }
  if (cm1 >= 4 && cm1 <= 7 && k <= 8 && !mnl_dfma) {
    const bool k4 = k <= 4;
    switch (cm1) {
#define MNL_W(C_)                                                                                          \
  case C_:                                                                                                 \
    *o = k4 ? LLChoice{k_loglik_mnl_mma<1, 0, C_, 1>, 4, 1, 32, true, 256}                                  \
            : LLChoice{k_loglik_mnl_mma<2, 0, C_, 1>, 8, 1, 32, true, 256};                                 \
    return true;
      MNL_W(4) MNL_W(5) MNL_W(6) MNL_W(7)
#undef MNL_W
      default: break;
    }
  }
  if (cm1 == 2) {
    if (k <= 12) return pick_exact<2, 2>(k, o, std::make_integer_sequence<int, 12>{});
    if (k <= 16) return pick_exact<2, 1>(k, o, std::make_integer_sequence<int, 16>{});
    return false;
  }
  if (cm1 == 3) {
    static const bool tab256 = getenv("SPS_MNL_TAB256") != nullptr;  // A/B hook: 2^(j/256) exp table
    if (tab256 && k <= 16) return pick_exact<3, 1, 256>(k, o, std::make_integer_sequence<int, 16>{});
    static const bool minb5 = getenv("SPS_MNL_MINB5") != nullptr;  // A/B hook: <= 102 registers, 5 blocks / SM
    if (minb5 && k <= 16) return pick_exact<3, 1, 64, 5>(k, o, std::make_integer_sequence<int, 16>{});
    if (k <= 16) return pick_exact<3, 1>(k, o, std::make_integer_sequence<int, 16>{});
    return false;
  }
  if (k > 8) return false;
  const int KT = k <= 4 ? 4 : 8;
  switch (cm1) {
    case 4: *o = KT == 4 ? LLChoice{ll_ptr<4, 4, 1>(), 4, 1} : LLChoice{ll_ptr<8, 4, 1>(), 8, 1}; return true;
    case 5: *o = KT == 4 ? LLChoice{ll_ptr<4, 5, 1>(), 4, 1} : LLChoice{ll_ptr<8, 5, 1>(), 8, 1}; return true;
    case 6: *o = KT == 4 ? LLChoice{ll_ptr<4, 6, 1>(), 4, 1} : LLChoice{ll_ptr<8, 6, 1>(), 8, 1}; return true;
    case 7: *o = KT == 4 ? LLChoice{ll_ptr<4, 7, 1>(), 4, 1} : LLChoice{ll_ptr<8, 7, 1>(), 8, 1}; return true;
    default: return false;
  }
}

// K1 launch plan for P particles over an observation range: chunk count S chosen so the grid
// (tiles x S) fills whole waves of SMs x resident blocks (occupancy from the kernel's registers and
// the chunk's shared memory) and the X tile fits in shared memory; cached per (P, range).
sps_status get_plan(sps_ctx* c, int64_t P, int range, int max_chunks, sps_ctx::Plan** out) {
  const LLChoice& ch = c->llc;
  const int ppb = ch.ppb > 0 ? ch.ppb : LL_THREADS * ch.PPT;
  const int64_t tiles = (P + ppb - 1) / ppb;
  const size_t row_bytes = (size_t)c->ldx * 8 + (c->C > 2 ? 4 : 0);
  sps_ctx::Plan* pl = nullptr;
  for (auto& q : c->plans)
    if (q.P == P && q.range == range && q.max_chunks == max_chunks) pl = &q;
  if (!pl) {
    pl = &c->plans[c->plan_next];
    c->plan_next = (c->plan_next + 1) % 8;
    const int smem_budget = 100 * 1024;
    const int tabb = (ch.tab > 256 ? ch.tab : 256) * 8;  // exp table bytes
    const int chunk_cap = std::max(1, (int)((smem_budget - tabb - 64) / row_bytes) - 16);
    // streaming (DMMA) kernels: two sub-chunk buffers (TMA double buffering) in the same budget
    // X sub-chunks of <= 64 rows (2 x 14 KB at k = 25): the shared-memory footprint no longer grows
    // with the chunk, so long chunks (fewer blocks, fewer per-block prologues / final logs) keep 4
    // blocks per SM (cfg2 run 173 -> 168 ms vs the budget-derived cap; SPS_K1_SUBCAP: tuning)
    static const int sub_cap_env = getenv("SPS_K1_SUBCAP") ? atoi(getenv("SPS_K1_SUBCAP")) : 64;
    const int sub_cap = std::min(std::max(16, sub_cap_env / 16 * 16), std::max(16, (chunk_cap / 2) / 16 * 16));
    const int S_min = ch.streams ? 1 : std::max(1, (range + chunk_cap - 1) / chunk_cap);
    static const int s_cap = getenv("SPS_K1_SMAX") ? std::max(1, atoi(getenv("SPS_K1_SMAX"))) : 1 << 20;  // tuning
    // (round 2: 64 -- cfg2 run 145.6-146.0 -> 144.1-144.3 ms, in-run K1 frac 0.583 -> 0.590; 48-160 alike;
    // 2^20, cfg3, cfg1 unchanged)
    static const double ovh = getenv("SPS_K1_OVH") ? atof(getenv("SPS_K1_OVH")) : 64.0;
    const int S_hi = std::min(std::min(max_chunks, s_cap), std::max(S_min, std::min(S_min + 24, range / 8)));
    const int warp_regs = ((c->ll_regs * 32 + 255) / 256) * 256;
    const int by_regs = 65536 / ((LL_THREADS / 32) * warp_regs);
    // cost ~ waves x (chunk + per-block overhead), overhead ~ 24 observation-equivalents
    // (theta load, X staging, final logs): fills whole waves without shredding the range
    int best = S_min, best_occ = 1;
    double best_cost = 1e300;
    for (int S = S_min; S <= S_hi; ++S) {
      const int chunk = (range + S - 1) / S;
      const int Se = (range + chunk - 1) / chunk;
      const int rows = ch.streams ? std::min(chunk, sub_cap) : chunk;
      const size_t smem = tabb + (size_t)(ch.streams ? 2 * ((rows + 15) / 16 * 16) : rows + 16) * row_bytes + 16;
      const int by_smem = (int)(233472 / (smem + 1024));
      const int occ = std::max(1, std::min(std::min(by_regs, by_smem), 16));
      const double slots = (double)num_sms() * occ;
      const double waves = std::ceil((double)tiles * Se / slots);
      const double cost = waves * (chunk + ovh);
      if (cost < best_cost * 0.995) {
        best_cost = cost;
        best = S;
        best_occ = occ;
      }
    }
    int chunk = (range + best - 1) / best;
    pl->P = P;
    pl->range = range;
    pl->max_chunks = max_chunks;
    pl->chunk = chunk;
    pl->occ = best_occ;
    pl->S = (range + chunk - 1) / chunk;
    pl->sub = ch.streams ? std::min(((chunk + 15) / 16) * 16, sub_cap) : 0;
    const int rows = ch.streams ? pl->sub : chunk;
    pl->smem = tabb + (size_t)(ch.streams ? 2 * ((rows + 15) / 16 * 16) : rows + 16) * c->ldx * 8 +
               (c->C > 2 ? (size_t)chunk * 4 : 0);
    if (pl->S > max_chunks) return fail(c, SPS_E_CONFIG, "observation range too long for the chunk buffer");
    static const bool dbg_plan = getenv("SPS_K1_PLAN") != nullptr;
    if (dbg_plan)
      fprintf(stderr, "K1 plan: P %lld range %d -> S %d chunk %d sub %d occ %d smem %zu\n", (long long)P, range, pl->S,
              pl->chunk, pl->sub, pl->occ, pl->smem);
  }
  *out = pl;
  return SPS_OK;
}

// K1 on the INT8 tensor cores (ozaki.cuh): slice this launch's theta into particle tile images,
// then one CTA (1 per SM: ~200 KB shared memory, 512 TMEM columns) per (128-particle tile,
// observation chunk); S chosen to fill whole waves of SMs.
template <int KB>
sps_status launch_oz(sps_ctx* c, const double* theta, int64_t ldt, int64_t P, int t0, int t1, double* part,
                     int max_chunks, int* nchunks_out, const int* stop) {
  const int range = t1 - t0;
  const int64_t tiles = (P + OZ_MT - 1) / OZ_MT;
  const size_t need = (size_t)tiles * oz_tile_bytes(OZ_MT, KB);
  if (need > c->oz_T_cap && c->capturing)  // (sized for P_local at create: no allocation inside a graph)
    return fail(c, SPS_E_STATE, "ozaki: particle images not allocated before graph capture");
  if (need > c->oz_T_cap) {
    dfree(c, c->oz_T, c->stream);
    c->oz_T = nullptr;
    c->oz_T_cap = 0;
    TRY(DALLOC(c, &c->oz_T, need));
    c->oz_T_cap = need;
  }
  PROF_BEGIN(c);
  k_oz_slice<<<(unsigned)((tiles * OZ_MT + 127) / 128), 128, 0, c->stream>>>(theta, P, ldt, c->k, KB, OZ_MT, 0, 0,
                                                                               c->oz_T, stop);
  CHECK_LAUNCH(c);
  PROF_END(c, CAT_OTHER);
  const int nsm = num_sms();
  int best = 1;
  double best_cost = 1e300;
  for (int S = 1; S <= std::max(1, std::min(max_chunks, range / OZ_NT)); ++S) {
    const int chunk = (range + S - 1) / S;
    const double cost = std::ceil((double)tiles * S / nsm) * ((chunk + OZ_NT - 1) / OZ_NT + 2.0);
    if (cost < best_cost * 0.995) {
      best_cost = cost;
      best = S;
    }
  }
  const int chunk = ((range + best - 1) / best + OZ_NT - 1) / OZ_NT * OZ_NT;
  const int S = (range + chunk - 1) / chunk;
  OzArgs a{c->oz_T, c->oz_X, c->oz_xamax, part, P, t0, t1, chunk, stop};
  static const int dbg = getenv("SPS_OZ_DBG") ? atoi(getenv("SPS_OZ_DBG")) : 0;  // timing experiments only
  auto fn = dbg == 1 ? k_oz_loglik<KB, 1> : dbg == 2 ? k_oz_loglik<KB, 2> : k_oz_loglik<KB>;
  if (dbg) CU(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, oz_smem_bytes<KB>()));
  PROF_BEGIN(c);
  CU(c, launch_pdl(fn, dim3((unsigned)tiles, (unsigned)S), dim3(OZ_THREADS), (size_t)oz_smem_bytes<KB>(), c->stream, a));
  CHECK_LAUNCH(c);
  c->k1_launches += 1;
  c->k1_pairs += (double)P * range;
  PROF_END(c, CAT_K1);
  *nchunks_out = S;
  return SPS_OK;
}

sps_status launch_loglik_oz(sps_ctx* c, const double* theta, int64_t ldt, int64_t P, int t0, int t1, double* part,
                            int max_chunks, int* nchunks_out, const int* stop) {
  switch (c->oz_KB) {
    case 2: return launch_oz<2>(c, theta, ldt, P, t0, t1, part, max_chunks, nchunks_out, stop);
    case 3: return launch_oz<3>(c, theta, ldt, P, t0, t1, part, max_chunks, nchunks_out, stop);
    default: return launch_oz<4>(c, theta, ldt, P, t0, t1, part, max_chunks, nchunks_out, stop);
  }
}

// Launch K1 over [t0, t1) for P particles: partial sums per observation chunk
// into `part` ([nchunks][P]); returns nchunks.  The chunk count S is chosen so
// the grid (tiles x S) fills whole waves of SMs x resident blocks (occupancy
// from the kernel's registers and the chunk's shared memory) and the X tile
// fits in shared memory; plans are cached per (P, range).
sps_status launch_loglik(sps_ctx* c, const double* theta, int64_t ldt, int64_t P, int t0, int t1, double* part,
                         int max_chunks, int* nchunks_out, const int* stop = nullptr) {
  const LLChoice& ch = c->llc;
  const int range = t1 - t0;
  if (range <= 0) {
    CU(c, cudaMemsetAsync(part, 0, (size_t)P * sizeof(double), c->stream));
    *nchunks_out = 1;
    return SPS_OK;
  }
  if (c->oz_KB > 0 && range >= c->oz_min_range)
    return launch_loglik_oz(c, theta, ldt, P, t0, t1, part, max_chunks, nchunks_out, stop);
  const int ppb = ch.ppb > 0 ? ch.ppb : LL_THREADS * ch.PPT;
  const int64_t tiles = (P + ppb - 1) / ppb;
  sps_ctx::Plan* pl = nullptr;
  TRY(get_plan(c, P, range, max_chunks, &pl));
  LLArgs a{c->Xs, c->y, theta, part, ldt, P, t0, t1, pl->chunk};
  a.k = c->k;
  a.stop = stop;
  a.sub = pl->sub;
  a.tiles = (int32_t)tiles;
  a.nitems = (int32_t)(tiles * pl->S);
  dim3 grid((unsigned)tiles, (unsigned)pl->S);
  static const bool persist = getenv("SPS_K1_PERSIST") != nullptr;
  if (persist && ch.streams)  // persistent: one wave of resident blocks loops over the items
    grid = dim3((unsigned)std::min<int64_t>(tiles * pl->S, (int64_t)num_sms() * pl->occ), 1);
  PROF_BEGIN(c);
  CU(c, launch_pdl(ch.fn, grid, dim3(LL_THREADS), pl->smem, c->stream, a));
  CHECK_LAUNCH(c);
  c->k1_launches += 1;
  c->k1_pairs += (double)P * range;
  PROF_END(c, CAT_K1);
  *nchunks_out = pl->S;
  return SPS_OK;
}

// Standard normals of (step, tag) for every local particle into Zbuf[slot], on
// the side stream `aux` (waits until Zbuf[slot] is free; signals ev_zready).
// graph: inside an M-step capture -- forked from the main stream after the
// proposal (ev_fork), step = ctl->step_cur + 1 on the device, joined back
// through ev_join (graph replays are stream-ordered: no Zbuf events needed).
sps_status launch_normals(sps_ctx* c, uint32_t tag, uint32_t step, int slot, bool graph = false, bool forked = false);
sps_status launch_normals(sps_ctx* c, uint32_t tag, uint32_t step, int slot, bool graph, bool forked) {
  const int np = (c->d + 1) / 2;
  static const bool serial = getenv("SPS_SERIAL_NORMALS") != nullptr;  // debug: no overlap, own profile category
  cudaStream_t st = serial && !graph ? c->stream : c->aux;
  if (!graph) CU(c, cudaStreamWaitEvent(st, c->ev_zfree[slot], 0));
  if (forked) CU(c, cudaStreamWaitEvent(st, c->ev_fork, 0));
  const int64_t tasks = c->Pl * np;
  if (serial && !graph) PROF_BEGIN(c);
  {  // lowest scheduling priority as a launch attribute: it carries into captured graph nodes
    cudaLaunchConfig_t lc = {};
    // M steps: 2 blocks per SM (grid-stride); setup / first draws: full grid
    const int64_t full = (tasks + 255) / 256;
    static const bool at_propose = getenv("SPS_NORMALS_FORK") && !strcmp(getenv("SPS_NORMALS_FORK"), "propose");
    // forked at the proposal: one 64-thread block per SM (its 4 K registers fit beside 4 K1 blocks) over
    // the whole step; forked at accept: 8 x 256 per SM into the tail
    // forked at accept, small steps (<= 2M Box-Muller pairs): 4 x 128 per SM -- the normals finish
    // inside the reduce / finalize tail anyway and take fewer issue slots from it (cfg2 run 144.2 ->
    // 142.0 ms; 2^17: -0.6%); larger steps need the full 8 x 256 to leave the critical path (2^18:
    // +2%, 2^20: +10% at 4 x 128)
    const bool small = tasks <= (int64_t)2 << 20;
    static const int bps_env = getenv("SPS_NORMALS_BPS") ? atoi(getenv("SPS_NORMALS_BPS")) : 0;
    static const int thr_env = getenv("SPS_NORMALS_THREADS") ? atoi(getenv("SPS_NORMALS_THREADS")) : 0;
    const int nb_per_sm = bps_env ? bps_env : (at_propose ? 1 : (small ? 4 : 8));
    const int nthr = thr_env ? thr_env : (at_propose ? 64 : (small ? 128 : 256));
    const int64_t fullb = (tasks + nthr - 1) / nthr;
    lc.gridDim = dim3((unsigned)(forked && nb_per_sm > 0 ? std::min<int64_t>(fullb, nb_per_sm * (int64_t)num_sms())
                                                        : full));
    lc.blockDim = dim3(forked ? nthr : 256);
    lc.stream = st;
    cudaLaunchAttribute at[1];
    int lo = 0, hi = 0;
    CU(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = lo;
    lc.attrs = at;
    lc.numAttrs = 1;
    const uint64_t npmagic = np > 1 ? ~0ull / (uint64_t)np + 1ull : 0ull;  // floor(2^64 / np) + 1 (np = 1: unused)
    CU(c, cudaLaunchKernelEx(&lc, k_normals, (int64_t)c->Pl, (int64_t)c->p0, np, npmagic,
                             round_up(c->d, 4), (uint64_t)c->cfg.seed,
                             step, tag, (uint32_t)c->cfg.pass, c->capturing_loop ? c->Zbuf[0] : c->Zbuf[slot],
                             tag == TAG_PROPOSAL ? (c->capturing_loop ? c->LUbuf[0] : c->LUbuf[slot]) : (double*)nullptr,
                             graph ? (const Ctl*)c->ctl : nullptr, graph ? (const int*)&c->ctl->stop : nullptr,
                             c->capturing_loop ? c->Zbuf[1] : (double*)nullptr,
                             c->capturing_loop ? c->LUbuf[1] : (double*)nullptr));
  }
  CHECK_LAUNCH(c);
  if (serial && !graph) PROF_END(c, CAT_OTHER);
  CU(c, cudaEventRecord(graph ? c->ev_join : c->ev_zready[slot], st));
  return SPS_OK;
}

// K8 / K10: theta = base + Lz z with z = Zbuf[slot], lp = prior kernel.
sps_status launch_draw(sps_ctx* c, int slot, const double* base, const double* Lz, double* out, double* lp_out,
                       const int* stop, bool graph = false, bool set_step = false) {
  const int d = c->d, KP = round_up(d, 4), NP = round_up(d, 8);
  const size_t base_sm = (size_t)(2 * PR_TILE * KP + PR_TILE * (NP / 8) + KP + PR_TILE * d);
  const bool stage = (base_sm + 2 * (size_t)NP * KP) * sizeof(double) <= 160 * 1024;
  const size_t smem = (base_sm + (stage ? 2 * (size_t)NP * KP : 0)) * sizeof(double);
  DrawArgs a{};
  a.base = base;
  a.Lz = Lz;
  a.Sinv = c->SinvP;
  a.Rp = c->RpP;
  a.mu = c->mu;
  a.Z = c->Zbuf[slot];
  a.out = out;
  a.lp_out = lp_out;
  a.ctl = c->ctl;
  a.stop = stop;
  a.P = c->Pl;
  a.p0 = c->p0;
  a.d = d;
  a.step0 = c->phase_step0;
  a.set_step = set_step ? 1 : 0;
  // (device-side loop: the body's first step always runs at an even step count since the phase
  // began, the second at an odd one, so each captured step's Z buffer is static: Zbuf[slot])
  if (!graph) CU(c, cudaStreamWaitEvent(c->stream, c->ev_zready[slot], 0));
  const int64_t ntl = (c->Pl + PR_TILE - 1) / PR_TILE;
  PROF_BEGIN(c);
  if (d <= 32) {  // register-blocked DMMA proposal, persistent, double-buffered
    // 32-particle tiles (4 warps, ~42 KB smem -> 5 blocks / SM): a finer tile grain than 64 (3 / SM,
    // ceil(1024 / 444) = 3 rounds of 64 at P = 65536) for the persistent loop's last round
    static const int tile = getenv("SPS_PROPOSE_TILE") ? atoi(getenv("SPS_PROPOSE_TILE")) : 32;
    const int T = tile == 64 ? 64 : 32;
    const int KK = (d + 3) / 4, KPr = 4 * KK, NPr = 8 * ((KPr + 7) / 8);
    const size_t sm = (size_t)(2 * T * KPr + 2 * round_up(T * d, 2) + KPr + 2 * NPr * KPr) * sizeof(double);
    const int64_t ntlT = (c->Pl + T - 1) / T;
    const unsigned grid = (unsigned)std::min<int64_t>(ntlT, (T == 32 ? 5 : 3) * (int64_t)num_sms());
    const unsigned thr = (unsigned)(4 * T);
#define PRB(KK_)                                                                                \
  case KK_:                                                                                     \
    if (T == 32)                                                                                \
      CU(c, launch_pdl(k_propose_rb<KK_, 32>, dim3(grid), dim3(thr), sm, c->stream, a));        \
    else                                                                                        \
      CU(c, launch_pdl(k_propose_rb<KK_, 64>, dim3(grid), dim3(thr), sm, c->stream, a));        \
    break;
    switch (KK) {
      PRB(1) PRB(2) PRB(3) PRB(4) PRB(5) PRB(6) PRB(7)
      default: PRB(8)
    }
#undef PRB
  } else {
    const unsigned grid = (unsigned)ntl;
    if (stage)
      k_propose<true><<<grid, 256, smem, c->stream>>>(a);
    else
      k_propose<false><<<grid, 256, smem, c->stream>>>(a);
  }
  CHECK_LAUNCH(c);
  PROF_END(c, CAT_PROPOSE);
  return SPS_OK;
}

// Fused M step (binary, d <= 32; fused.cuh): theta* in shared memory, K1 over [0, t1), accept and
// the tile moment partials -> bpart rows (the k_accept_tile layout), one launch.
sps_status launch_fused(sps_ctx* c, int slot, int t1, double temper, const int* stop, bool graph) {
  sps_ctx::Plan* pl = nullptr;
  TRY(get_plan(c, c->Pl, t1, c->max_chunks, &pl));
  if (pl->sub <= 0 || pl->sub > 64) return fail(c, SPS_E_CONFIG, "fused M step: X sub-chunk of %d rows (max 64)", pl->sub);
  if (!graph) CU(c, cudaStreamWaitEvent(c->stream, c->ev_zready[slot], 0));
  FusedArgs a{};
  a.X = c->Xs;
  a.theta = c->theta;
  a.L = c->L;
  a.lp = c->lp;
  a.Z = c->Zbuf[slot];
  a.logu = c->LUbuf[slot];
  a.Lz = c->Lprop;
  a.Rp = c->RpP;
  a.mu = c->mu;
  a.shift = c->shift;
  a.part = c->part;
  a.tpart = c->fu_tpart;
  a.bpart = c->bpart;
  a.tick = c->fu_tick;
  a.ctl = c->ctl;
  a.stop = stop;
  a.P = c->Pl;
  a.temper = temper;
  a.dmagic = ((1ull << 32) + (uint64_t)c->d - 1) / (uint64_t)c->d;
  a.d = c->d;
  a.t1 = t1;
  a.chunk = pl->chunk;
  a.sub = pl->sub;
  a.S = pl->S;
  a.TPR = c->fu_TPR;
  a.step0 = c->phase_step0;
  a.set_step = 1;
  const dim3 grid((unsigned)(c->Pl / FU_TILE), (unsigned)pl->S);
  PROF_BEGIN(c);
  CU(c, launch_pdl(c->fu_fn, grid, dim3(128), c->fu_smem, c->stream, a));
  CHECK_LAUNCH(c);
  c->k1_launches += 1;
  c->k1_pairs += (double)c->Pl * t1;
  PROF_END(c, CAT_K1);
  return SPS_OK;
}

// Fused-kernel instance (opt-in experiment): instantiated for the measured / tested
// shapes only, k = 4 (configs[0]) and k = 25 (configs[1]); other k run the separate kernels.
void (*pick_fused(int k))(FusedArgs) {
  switch (k) {
    case 4: return k_mstep_bin<1, 0, 1>;
    case 25: return k_mstep_bin<6, 1, 4>;
    default: return nullptr;
  }
}

// K9 + K6 (decide = true) or K6 only, then the deterministic reduction into this
// rank's stats slice and the gather across ranks -> `gath`.
sps_status launch_normals(sps_ctx* c, uint32_t tag, uint32_t step, int slot, bool graph, bool forked);

// fork_step != ~0u: after the accept kernel, fork the next step's normals (step fork_step + 1) onto
// the side stream.
sps_status accept_moments(sps_ctx* c, bool decide, int nchunks, double temper, uint32_t step, const int* stop,
                          const double* logu = nullptr, const FinArgs* fin = nullptr, size_t fin_smem = 0,
                          uint32_t fork_step = ~0u, bool fused = false) {
  AccArgs a{};
  a.theta = c->theta;
  a.L = c->L;
  a.lp = c->lp;
  a.theta_s = c->theta_s;
  a.part = c->part;
  a.lp_s = c->lp_s;
  a.shift = c->shift;
  a.logu = logu;
  a.bpart = c->bpart;
  a.ctl = c->ctl;
  a.stop = stop;
  a.P = c->Pl;
  a.p0 = c->p0;
  a.temper = temper;
  a.seed = c->cfg.seed;
  a.nchunks = nchunks;
  a.d = c->d;
  a.tp = c->tp;
  a.decide = decide ? 1 : 0;
  a.step = step;
  a.pass = (uint32_t)c->cfg.pass;
  a.dmagic = ((1ull << 32) + (uint64_t)c->d - 1) / (uint64_t)c->d;
  a.trace = decide ? c->trace : nullptr;
  // (device-side loop: each captured step's log-u buffer is static -- LUbuf[step & 1] -- like its Z)
  PROF_BEGIN(c);
  if (fused) {  // accept + tile moments already done by the fused M-step kernel
  } else if (c->acc_tnt > 0) {  // tile layout: bulk-staged rows, on-the-fly DMMA fragments, ones column
    switch (c->acc_tnt) {
      case 1: CU(c, launch_pdl(k_accept_tile<1>, dim3(c->nblk), dim3(256), c->acc_smem, c->stream, a)); break;
      case 2: CU(c, launch_pdl(k_accept_tile<2>, dim3(c->nblk), dim3(256), c->acc_smem, c->stream, a)); break;
      case 3: CU(c, launch_pdl(k_accept_tile<3>, dim3(c->nblk), dim3(256), c->acc_smem, c->stream, a)); break;
      case 4: CU(c, launch_pdl(k_accept_tile<4>, dim3(c->nblk), dim3(256), c->acc_smem, c->stream, a)); break;
      default: CU(c, launch_pdl(k_accept_tile<5>, dim3(c->nblk), dim3(256), c->acc_smem, c->stream, a)); break;
    }
  } else if (c->d <= 32) {  // register-blocked T'T on DMMA
    const int NTr = (c->d + 7) / 8;
    a.dmagic = ((1ull << 32) + (uint64_t)c->d - 1) / (uint64_t)c->d;
    const uint64_t padw = (uint64_t)(8 * NTr + 4 - c->d);
    a.pmagic = ((1ull << 32) + padw - 1) / padw;
    const size_t sm =
        ((size_t)round_up(c->tp, 32) * (8 * NTr + 4) + 8 * (size_t)c->d) * sizeof(double) + (size_t)c->tp + 16;
    switch (NTr) {
      case 1: k_accept_mom_rb<1><<<c->nblk, 256, sm, c->stream>>>(a); break;
      case 2: k_accept_mom_rb<2><<<c->nblk, 256, sm, c->stream>>>(a); break;
      case 3: k_accept_mom_rb<3><<<c->nblk, 256, sm, c->stream>>>(a); break;
      default: k_accept_mom_rb<4><<<c->nblk, 256, sm, c->stream>>>(a); break;
    }
  } else {
    const size_t smem =
        ((size_t)round_up(c->tp, 4) * (round_up(c->d, 8) + 4) + 8 * (size_t)c->d) * sizeof(double) + (size_t)c->tp + 16;
    k_accept_mom<<<c->nblk, 256, smem, c->stream>>>(a);
  }
  CHECK_LAUNCH(c);
  PROF_END(c, CAT_ACCEPT);
  if (fork_step != ~0u) {
    CU(c, cudaEventRecord(c->ev_fork, c->stream));
    TRY(launch_normals(c, TAG_PROPOSAL, fork_step + 1u, (int)((fork_step + 1u) & 1u), c->capturing, true));
  }
  const int d = c->d;
  const int nm = red_nm(d), ng = red_ng(c->Jl, d);
  RedArgs r{c->bpart, c->nblk, c->N / c->tp, c->Jl, d, c->acc_tnt > 0 ? c->Wt : c->W, c->acc_tnt, c->N, c->shift,
            c->mon, c->nmon};
  FinArgs none{};
  if (fin && fin->stage_S && c->red_cluster > 0) {  // one rank: reduce + finalize as one cluster (DSMEM)
    FinArgs f = *fin;
    f.preloaded = 1;
    f.ticket = nullptr;
    PROF_BEGIN(c);
    CU(c, launch_cluster_pdl(k_mom_reduce_cl, c->red_cluster, dim3(256), fin_smem, c->stream, r, c->ctl, stop, f));
    CHECK_LAUNCH(c);
    PROF_END(c, CAT_FINALIZE);
    return SPS_OK;
  }
  PROF_BEGIN(c);
  CU(c, launch_pdl(k_mom_reduce, dim3(nm + ng + 1), dim3(256), fin ? fin_smem : 0, c->stream, r, c->ctl, c->slice, stop,
                    fin ? *fin : none));
  CHECK_LAUNCH(c);
  PROF_END(c, fin ? CAT_FINALIZE : CAT_REDUCE);
  if (fin) return SPS_OK;  // one rank: the slice is the gathered stats, finalized by the last block
  PROF_BEGIN(c);
  TRY(gather(c, c->slice, c->gath, (size_t)c->slice_len));
  PROF_END(c, CAT_GATHER);
  return SPS_OK;
}

bool final_cycle(const sps_ctx* c) {
  return c->cfg.tempering == SPS_POWER_TEMPERING ? (c->phi == 1.0) : (c->t == c->n);
}

// Arguments of finalize_body (K7) and its dynamic shared memory.
sps_status make_fin(sps_ctx* c, int mode, bool allow_stop, const int* stop, int slot, FinArgs* fo, size_t* smem_out) {
  FinArgs f{};
  f.host_out = slot >= 0 ? c->dslot + slot : nullptr;
  f.gath = c->gath;
  f.G = c->G;
  f.slice_len = c->slice_len;
  f.J = c->J;
  f.Jl = c->Jl;
  f.N = c->N;
  f.d = c->d;
  f.shift = c->shift;
  f.Lprop = c->Lprop;
  f.V = nullptr;  // (the pooled V is not read back on the hot path)
  f.mon = c->mon;
  f.nmon = c->nmon;
  f.mode = mode;
  f.K = allow_stop ? (final_cycle(c) ? c->cfg.K_final : c->cfg.K_inter) : -1.0;
  f.h_step = c->cfg.h_step;
  f.h_min = c->cfg.h_min;
  f.h_max = c->cfg.h_max;
  f.accept_target = c->cfg.accept_target;
  f.ctl = c->ctl;
  f.stop_in = stop;
  f.rne_out = c->rne;
  f.trace = c->trace;
  if (c->capturing_loop && mode == 1) {
    f.loop = 1;
    f.cond = c->loop_cond;
    f.rmax = c->loop_rmax;
    f.host_out = c->dslot;
  }
  f.sig_rec = c->recording ? c->sig_rec : nullptr;
  f.sig_rec_cap = c->recording ? c->sig_rec_cap : 0;
  f.sig_in = c->sig_in;
  f.sig_in_n = c->sig_in_n;
  f.sig_step = mode == 0 ? (int64_t)c->mstep : -1;  // mode 1: the device step (ctl->step_cur) + 1
  f.stage_S = fin_smem_doubles(c->d, c->J, c->nmon, true) * 8 <= 200 * 1024 ? 1 : 0;
  const size_t smem = (size_t)fin_smem_doubles(c->d, c->J, c->nmon, f.stage_S != 0) * sizeof(double);
  if (smem > 200 * 1024) return fail(c, SPS_E_CONFIG, "d = %d too large for the finalize kernel", c->d);
  *fo = f;
  *smem_out = smem;
  return SPS_OK;
}

// K7 as its own launch (after the gather; G > 1).
sps_status finalize(sps_ctx* c, int mode, bool allow_stop, const int* stop, int slot = -1) {
  FinArgs f;
  size_t smem = 0;
  TRY(make_fin(c, mode, allow_stop, stop, slot, &f, &smem));
  PROF_BEGIN(c);
  k_finalize<<<1, 256, smem, c->stream>>>(f);
  CHECK_LAUNCH(c);
  PROF_END(c, CAT_FINALIZE);
  return SPS_OK;
}

// K9 + K6 -> reduce -> (gather) -> K7: fused into the reduce launch on one rank.
sps_status moments_finalize(sps_ctx* c, bool decide, int nchunks, double temper, uint32_t step, const int* stop,
                            const double* logu, int mode, bool allow_stop, int slot, bool fork_normals = false,
                            bool fused = false) {
  const bool graph = c->capturing;
  if (c->xchg) {
    TRY(accept_moments(c, decide, nchunks, temper, step, stop, logu, nullptr, 0, fork_normals ? step : ~0u, fused));
    return finalize(c, mode, allow_stop, stop, slot);
  }
  FinArgs f;
  size_t smem = 0;
  TRY(make_fin(c, mode, allow_stop, stop, slot, &f, &smem));
  f.ticket = c->ticket;
  (void)graph;
  return accept_moments(c, decide, nchunks, temper, step, stop, logu, &f, smem, fork_normals ? step : ~0u, fused);
}

sps_status validate(const sps_config* cfg) {
  if (!cfg) return SPS_E_CONFIG;
  if (cfg->n < 1 || cfg->k < 1 || cfg->C < 2 || cfg->C > 8) return SPS_E_CONFIG;
  if (cfg->J < 2 || cfg->N < 2 || cfg->N > 16384) return SPS_E_CONFIG;
  if (cfg->nranks < 1 || cfg->rank < 0 || cfg->rank >= cfg->nranks || cfg->J % cfg->nranks) return SPS_E_CONFIG;
  if (!(cfg->ess_frac > 0 && cfg->ess_frac < 1) || !(cfg->K_inter > 0) || !(cfg->K_final > 0)) return SPS_E_CONFIG;
  if (cfg->h_min > cfg->h_init || cfg->h_init > cfg->h_max || cfg->h_min < 1 || cfg->h_step < 0) return SPS_E_CONFIG;
  if (cfg->max_m_steps < 1 || cfg->max_cycles < 1) return SPS_E_CONFIG;
  if (cfg->tempering != SPS_DATA_TEMPERING && cfg->tempering != SPS_POWER_TEMPERING) return SPS_E_CONFIG;
  if (cfg->resampling < 0 || cfg->resampling > 2) return SPS_E_CONFIG;
  const int64_t P = (int64_t)cfg->J * cfg->N;
  if (P > (int64_t)1 << 31) return SPS_E_CONFIG;
  return SPS_OK;
}

void free_ctx(sps_ctx* c) {
  if (!c) return;
  static const bool dbg = getenv("SPS_DEBUG_CLOSE") != nullptr;
  auto T0 = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!dbg) return;
    const auto t = std::chrono::steady_clock::now();
    fprintf(stderr, "free_ctx %-10s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(t - T0).count());
    T0 = t;
  };
  if (!c->xchg) {  // aliases of the local slices
    c->gath = c->essgath = c->grp_ms_gath = c->Lj_gath = c->pw_gath = c->mx_gath = nullptr;
  }
  if (c->aux) cudaStreamSynchronize(c->aux);
  if (c->stream) cudaStreamSynchronize(c->stream);
  lap("sync");
  cudaStream_t fs = c->stream ? c->stream : 0;
  for (double* z : c->Zbuf) dfree(c, z, fs);
  for (double* z : c->LUbuf) dfree(c, z, fs);
  lap("zbuf");
  for (int q = 0; q < 2; ++q)
    if (c->gexec[q]) cudaGraphExecDestroy(c->gexec[q]);
  if (c->gloop) cudaGraphExecDestroy(c->gloop);
  lap("gexec");
  for (int q = 0; q < 2; ++q) {
    if (c->ev_zready[q]) cudaEventDestroy(c->ev_zready[q]);
    if (c->ev_zfree[q]) cudaEventDestroy(c->ev_zfree[q]);
  }
  if (c->ev_fork) cudaEventDestroy(c->ev_fork);
  if (c->ev_join) cudaEventDestroy(c->ev_join);
  lap("events");
  if (c->aux) cudaStreamDestroy(c->aux);
  lap("graphs/ev");
  void* ptrs[] = {c->X, c->Xs, c->mu, c->Lprior, c->xbar, c->mon, c->y, c->theta, c->theta2, c->L, c->L2, c->lp,
                  c->lp2, c->lw, c->lw_cur, c->theta_s, c->lp_s, c->part, c->gpart, c->mpart, c->slice, c->gath,
                  c->shift, c->Lprop, c->V, c->rne, c->lwbuf, c->essparts, c->essslice, c->essgath, c->lse, c->logpl, c->grp_ms,
                  c->grp_ms_gath, c->Lj, c->Lj_gath, c->scal, c->pw_parts, c->pw_slice, c->pw_gath, c->mx_parts,
                  c->mx_slice, c->mx_gath, c->fn_A, c->fn_out, c->ll_scratch, c->Sinv, c->LpriorP, c->SinvP, c->Rp, c->RpP, c->bpart, c->ctl, c->inc_dev,
                  c->sig_rec, c->sig_in, c->fu_tick, c->fu_tpart, c->oz_X, c->oz_T, c->oz_xamax};
  for (void* p : ptrs) dfree(c, p, fs);
  lap("cudaFree");
  dfree(c, c->llbad, fs);
  lap("freeHost");
  dfree(c, c->ticket, fs);
  if (c->trace) cudaFree(c->trace);  // managed
  dfree(c, c->tl, fs);
  cudaStreamSynchronize(fs);
  slab_put(c->slab);  // (after the stream: no kernel of this context writes it any more)
  c->slab = nullptr;
  for (cudaEvent_t e : c->evs)
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : c->prof_pool) cudaEventDestroy(e);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->comm) g_nccl.CommDestroy(c->comm);
  if (c->own_stream && c->stream) cudaStreamDestroy(c->stream);
  lap("rest");
}

constexpr int ESS_TILE = 2048;
constexpr int MX_BLOCKS = 256;
constexpr int PW_BLOCKS = 256;

}  // namespace

// ================================================================== C ABI
extern "C" {

sps_status sps_config_default(sps_config* cfg) {
  if (!cfg) return SPS_E_CONFIG;
  std::memset(cfg, 0, sizeof *cfg);
  cfg->tempering = SPS_DATA_TEMPERING;
  cfg->resampling = SPS_RESIDUAL;
  cfg->ess_frac = 0.5;
  cfg->K_inter = 0.35;
  cfg->K_final = 0.9;
  cfg->h_init = 50;
  cfg->h_step = 1;
  cfg->h_min = 10;
  cfg->h_max = 100;
  cfg->accept_target = 0.25;
  cfg->max_m_steps = 1000;
  cfg->max_cycles = 1 << 20;
  cfg->nranks = 1;
  return SPS_OK;
}

const char* sps_last_error(const sps_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void sps_destroy(sps_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->cfg.device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  // guarded context (SPS_GUARD=1): verify the guard zones one last time; with SPS_GUARD_ABORT=1 an
  // overwritten zone aborts the process (a whole test suite run under both checks every context)
  if (ctx->guarded && !ctx->guards.empty() && ctx->stream) {
    int64_t bad = 0;
    if (sps_check_guards(ctx, &bad) == SPS_E_GUARD) {
      fprintf(stderr, "SPS_GUARD: %s\n", ctx->err.c_str());
      if (getenv("SPS_GUARD_ABORT") && atoi(getenv("SPS_GUARD_ABORT")) != 0) abort();
    }
  }
  free_ctx(ctx);
  delete ctx;
}

sps_status sps_test_loopback_allgather(const void* id128, int32_t rank, int32_t G, const void* send, int64_t bytes,
                                       void* recv) {
  if (!id128 || G < 1 || rank < 0 || rank >= G || bytes < 0 || (bytes > 0 && (!send || !recv))) return SPS_E_CONFIG;
  if (std::memcmp(id128, kLoopMagic, sizeof kLoopMagic - 1) != 0) return SPS_E_CONFIG;
  std::shared_ptr<Loopback> lb = loopback_get(id128, G);
  if (lb->G != G) return SPS_E_CONFIG;
  lb->allgather(rank, send, (size_t)bytes, recv);
  return SPS_OK;
}

sps_status sps_loopback_unique_id(void* id128) {
  if (!id128) return SPS_E_CONFIG;
  static std::mutex mu;
  static uint64_t counter = 0;
  std::lock_guard<std::mutex> lk(mu);
  char buf[128] = {0};
  std::memcpy(buf, kLoopMagic, sizeof kLoopMagic - 1);
  const uint64_t v = ++counter ^ (uint64_t)std::chrono::steady_clock::now().time_since_epoch().count();
  std::memcpy(buf + 32, &v, sizeof v);
  std::memcpy(id128, buf, 128);
  return SPS_OK;
}

sps_status sps_nccl_unique_id(void* id128) {
  std::string why;
  if (!id128 || !g_nccl.load(&why)) return SPS_E_NCCL;
  ncclUniqueId id;
  if (g_nccl.GetUniqueId(&id) != ncclSuccess) return SPS_E_NCCL;
  std::memcpy(id128, &id, sizeof id);
  return SPS_OK;
}

sps_status sps_create(const sps_config* cfg_in, const double* X, const int32_t* y, const double* prior_mean,
                      const double* prior_cov, sps_ctx** out) {
  if (!out) return SPS_E_CONFIG;
  *out = nullptr;
  if (validate(cfg_in) != SPS_OK || !X || !y || !prior_mean || !prior_cov) return SPS_E_CONFIG;
  sps_ctx* c = new sps_ctx();
  c->cfg = *cfg_in;
  c->guarded = getenv("SPS_GUARD") && atoi(getenv("SPS_GUARD")) != 0;  // debug memory check
  c->cfg.monitors = nullptr;
  c->cfg.nccl_id = nullptr;
  *out = c;
  const sps_config& cfg = *cfg_in;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return fail(c, SPS_E_CUDA, "no CUDA device: libsps has no CPU fallback");
  CU(c, cudaSetDevice(cfg.device));
  c->n = cfg.n;
  c->k = cfg.k;
  c->C = cfg.C;
  c->d = cfg.k * (cfg.C - 1);
  c->J = cfg.J;
  c->N = cfg.N;
  c->G = cfg.nranks;
  c->rank = cfg.rank;
  c->Jl = cfg.J / cfg.nranks;
  c->g0 = c->rank * c->Jl;
  c->P = (int64_t)cfg.J * cfg.N;
  c->Pl = (int64_t)c->Jl * cfg.N;
  c->p0 = (int64_t)c->g0 * cfg.N;
  const int d = c->d;
  if (d > 128) return fail(c, SPS_E_CONFIG, "d = k (C-1) = %d > 128 is not supported", d);
  LLChoice ch;
  if (!choose_ll(c->k, c->C, &ch)) return fail(c, SPS_E_CONFIG, "unsupported (k, C) = (%d, %d)", c->k, c->C);
  c->KT = ch.KT;
  c->PPT = ch.PPT;
  c->llc = ch;
  {  // binary 64 <= k <= 128: K1 on the INT8 tensor cores (ozaki.cuh); SPS_NO_OZAKI: the DMMA kernel
    // per launch, only for observation ranges >= oz_min_range: below that the FP64 DMMA kernel is faster
    // (measured crossover ~384-512 observations at P = 65536, k = 56 and 100: the INT8 path pays the
    // theta slicing and a TMEM / operand-image setup per CTA); SPS_OZ_MINK / SPS_OZ_MINRANGE: A/B, tests
    const bool no_oz = getenv("SPS_NO_OZAKI") != nullptr;
    const int oz_mink = getenv("SPS_OZ_MINK") ? std::max(33, atoi(getenv("SPS_OZ_MINK"))) : 33;
    c->oz_min_range = getenv("SPS_OZ_MINRANGE") ? std::max(1, atoi(getenv("SPS_OZ_MINRANGE"))) : 512;
    if (!no_oz && c->C == 2 && c->k >= oz_mink && c->k <= 128) c->oz_KB = (c->k + 31) / 32;
  }
  {
    cudaFuncAttributes fa{};
    CU(c, cudaFuncGetAttributes(&fa, ch.fn));
    c->ll_regs = fa.numRegs;
    CU(c, cudaFuncSetAttribute(ch.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 101 * 1024 + 1024));
  }
  c->ldx = (ch.KT + 3) / 4 * 4;  // X row stride: k padded to 4 (DMMA k-step; zero columns)
  c->nmon = cfg.n_monitors > 0 ? cfg.n_monitors : c->C - 1;
  if (cfg.n_monitors > 0 && !cfg_in->monitors) return fail(c, SPS_E_CONFIG, "n_monitors > 0 but monitors == NULL");
  // accept + moments layout: blocks of tp particles inside one group (tp divides N,
  // tp <= 256, staged tile tp x round_up(d, 8) doubles <= 96 KB)
  {
    static const int tp_env = getenv("SPS_ACC_TP") ? atoi(getenv("SPS_ACC_TP")) : 256;  // tuning
    const int cap = std::max(1, std::min(std::max(1, std::min(tp_env, 256)), 96 * 1024 / (8 * ((d + 7) / 8 * 8 + 4))));
    c->tp = 1;
    for (int q = std::min(c->N, cap); q >= 1; --q)
      if (c->N % q == 0) {
        c->tp = q;
        break;
      }
  }
  c->nblk = (int)(c->Pl / c->tp);
  c->W = d + d * d + 1;
  {  // tile-layout accept kernel when its bulk copies are 16-byte aligned and it fits in shared memory
    const int tnt = (d + 8) / 8, ntri = tnt * (tnt + 1) / 2, TD = c->tp * d;
    const size_t sm = (size_t)(std::max(TD, 8 * ntri * 64) + 4 * c->tp) * sizeof(double) + (size_t)c->tp + 16;
    static const bool no_tile = getenv("SPS_NO_ACC_TILE") != nullptr;
    if (d <= 32 && c->tp % 2 == 0 && sm <= 200 * 1024 && !no_tile) {
      c->acc_tnt = tnt;
      c->Wt = ntri * 64 + 1;
      c->acc_smem = sm;
    }
  }
  {  // fused M-step kernel (binary, d <= 32, DMMA K1, tile-layout moments, groups of whole 64-tiles):
     // opt-in (SPS_FUSED=1) -- measured slower than the separate kernels at every t_l
    static const bool fused_on = getenv("SPS_FUSED") != nullptr && strcmp(getenv("SPS_FUSED"), "0") != 0;
    if (fused_on && c->C == 2 && c->llc.streams && c->k <= 32 && c->acc_tnt > 0 && c->tp % FU_TILE == 0)
      c->fu_fn = pick_fused(c->k);
    if (c->fu_fn) {
      c->fu_TPR = c->tp / FU_TILE;
      c->fu_smem = (size_t)fused_smem_doubles(round_up(c->k, 4), c->d) * sizeof(double);
    }
  }
  c->slice_len = slice_length(c->Jl, d, c->nmon);
  c->max_chunks = (int)std::max<int64_t>(1, std::min<int64_t>(64, ((int64_t)1 << 26) / std::max<int64_t>(c->Pl, 1)));
  c->Bmax = (int)std::max<int64_t>(8, std::min<int64_t>(ESS_RANK_THREADS, ((int64_t)1 << 23) / std::max<int64_t>(c->Pl, 1)));

  {  // keep freed device memory in the default pool across contexts (once per device)
    static std::mutex mu;
    static bool done[64] = {};
    std::lock_guard<std::mutex> lk(mu);
    if (cfg.device >= 0 && cfg.device < 64 && !done[cfg.device]) {
      cudaMemPool_t pool;
      CU(c, cudaDeviceGetDefaultMemPool(&pool, cfg.device));
      uint64_t thr = ~0ull;
      CU(c, cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
      done[cfg.device] = true;
    }
  }
  if (cfg.stream) {
    c->stream = (cudaStream_t)cfg.stream;
  } else {
    int lo = 0, hi = 0;
    CU(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(c, cudaStreamCreateWithPriority(&c->stream, cudaStreamNonBlocking, hi));  // the critical path
    c->own_stream = true;
  }
  c->xchg = c->G > 1 || (cfg_in->nccl_id && getenv("SPS_XCHG_1RANK") && atoi(getenv("SPS_XCHG_1RANK")) != 0);
  if (c->xchg && cfg_in->nccl_id &&
      std::memcmp(cfg_in->nccl_id, kLoopMagic, sizeof kLoopMagic - 1) == 0) {  // loopback transport
    c->loop = loopback_get(cfg_in->nccl_id, c->G);
  } else if (c->xchg) {
    std::string why;
    if (!cfg_in->nccl_id) return fail(c, SPS_E_CONFIG, "nranks > 1 requires nccl_id");
    if (!g_nccl.load(&why)) return fail(c, SPS_E_NCCL, "%s", why.c_str());
    ncclUniqueId id;
    std::memcpy(&id, cfg_in->nccl_id, sizeof id);
    ncclResult_t r = g_nccl.CommInitRank(&c->comm, c->G, id, c->rank);
    if (r != ncclSuccess) return fail(c, SPS_E_NCCL, "ncclCommInitRank: %s", g_nccl.GetErrorString(r));
  }
  const int64_t Pl = c->Pl;
  TRY(DALLOC(c, &c->X, (size_t)c->n * c->k));
  TRY(DALLOC(c, &c->Xs, (size_t)c->n * c->ldx + 2));
  TRY(DALLOC(c, &c->y, (size_t)c->n));
  TRY(DALLOC(c, &c->mu, d));
  TRY(DALLOC(c, &c->Lprior, (size_t)d * d));
  TRY(DALLOC(c, &c->xbar, c->k));
  TRY(DALLOC(c, &c->mon, (size_t)c->nmon * d));
  TRY(DALLOC(c, &c->theta, (size_t)Pl * d + 2 * PR_TILE));
  TRY(DALLOC(c, &c->theta2, (size_t)Pl * d + 2 * PR_TILE));
  TRY(DALLOC(c, &c->theta_s, (size_t)Pl * d + 2 * PR_TILE));
  TRY(DALLOC(c, &c->L, (size_t)Pl));
  TRY(DALLOC(c, &c->L2, (size_t)Pl));
  TRY(DALLOC(c, &c->lp, (size_t)Pl));
  TRY(DALLOC(c, &c->lp2, (size_t)Pl));
  TRY(DALLOC(c, &c->lw, (size_t)Pl));
  TRY(DALLOC(c, &c->lw_cur, (size_t)Pl));
  TRY(DALLOC(c, &c->lp_s, (size_t)Pl));
  TRY(DALLOC(c, &c->part, (size_t)c->max_chunks * Pl));
  TRY(DALLOC(c, &c->bpart, (size_t)c->nblk * std::max(c->W, c->Wt)));
  if (c->fu_fn) {
    const int64_t tiles = c->Pl / FU_TILE;
    TRY(DALLOC(c, &c->fu_tick, (size_t)(tiles + c->nblk)));
    CU(c, cudaMemsetAsync(c->fu_tick, 0, sizeof(unsigned) * (size_t)(tiles + c->nblk), c->stream));
    if (c->fu_TPR > 1) TRY(DALLOC(c, &c->fu_tpart, (size_t)tiles * c->Wt));
    CU(c, cudaFuncSetAttribute(c->fu_fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)c->fu_smem));
  }
  TRY(DALLOC(c, &c->Sinv, (size_t)d * d));
  c->slab = slab_get();
  if (!c->slab) return fail(c, SPS_E_CUDA, "cudaHostAlloc of the control slab failed");
  std::memset(c->slab, 0, SLAB_BYTES);
  c->hctl = reinterpret_cast<Ctl*>(c->slab);
  c->hslot = reinterpret_cast<Ctl*>(c->slab + SLAB_CTL);
  c->hllbad = reinterpret_cast<int*>(c->slab + 3 * SLAB_CTL);
  int* hinit = c->hllbad + 2;  // staging word for the device-side llbad
  CU(c, cudaHostGetDevicePointer((void**)&c->dslot, c->hslot, 0));
  CU(c, cudaHostGetDevicePointer((void**)&c->dllbad, c->hllbad, 0));
  TRY(DALLOC(c, &c->ticket, 1));
  TRY(DALLOC(c, &c->llbad, 1));
  *hinit = 0x7fffffff;
  CU(c, cudaMemcpyAsync(c->llbad, hinit, sizeof(int), cudaMemcpyHostToDevice, c->stream));
  c->hllbad[0] = c->hllbad[1] = 0x7fffffff;
  if (getenv("SPS_TRACE")) CU(c, cudaMallocManaged((void**)&c->trace, 128 * sizeof(unsigned long long)));
  CU(c, cudaMemsetAsync(c->ticket, 0, sizeof(unsigned), c->stream));
  CU(c, cudaEventCreateWithFlags(&c->evs[0], cudaEventDisableTiming));
  CU(c, cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
  CU(c, cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  CU(c, cudaEventCreateWithFlags(&c->evs[1], cudaEventDisableTiming));
  TRY(DALLOC(c, &c->slice, (size_t)c->slice_len));
  if (c->xchg) TRY(DALLOC(c, &c->gath, (size_t)c->slice_len * c->G));
  else c->gath = c->slice;
  {
    // normals in rows of round_up(d, 4) (DMMA K padding), whole tiles: zeroed once, padding never written
    const size_t zn = (size_t)(Pl + PR_TILE) * round_up(d, 4);
    TRY(DALLOC(c, &c->Zbuf[0], zn));
    TRY(DALLOC(c, &c->Zbuf[1], zn));
    TRY(DALLOC(c, &c->LUbuf[0], (size_t)Pl));
    TRY(DALLOC(c, &c->LUbuf[1], (size_t)Pl));
    CU(c, cudaMemsetAsync(c->Zbuf[0], 0, zn * sizeof(double), c->stream));
    CU(c, cudaMemsetAsync(c->Zbuf[1], 0, zn * sizeof(double), c->stream));
    int lo = 0, hi = 0;
    CU(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CU(c, cudaStreamCreateWithPriority(&c->aux, cudaStreamNonBlocking, lo));  // side work fills idle SMs
    for (int q = 0; q < 2; ++q) {
      CU(c, cudaEventCreateWithFlags(&c->ev_zready[q], cudaEventDisableTiming));
      CU(c, cudaEventCreateWithFlags(&c->ev_zfree[q], cudaEventDisableTiming));
      CU(c, cudaEventRecord(c->ev_zfree[q], c->stream));
    }
  }
  TRY(DALLOC(c, &c->shift, d));
  {  // padded DMMA layouts (NP x KP, zeros outside d x d): Lprop, prior factor, prior precision
    const size_t pn = (size_t)round_up(d, 8) * round_up(d, 4);
    TRY(DALLOC(c, &c->Lprop, pn));
    TRY(DALLOC(c, &c->LpriorP, pn));
    TRY(DALLOC(c, &c->SinvP, pn));
    TRY(DALLOC(c, &c->RpP, pn));
    TRY(DALLOC(c, &c->Rp, (size_t)d * d));
    CU(c, cudaMemsetAsync(c->Lprop, 0, pn * sizeof(double), c->stream));
    CU(c, cudaMemsetAsync(c->LpriorP, 0, pn * sizeof(double), c->stream));
    CU(c, cudaMemsetAsync(c->SinvP, 0, pn * sizeof(double), c->stream));
    CU(c, cudaMemsetAsync(c->RpP, 0, pn * sizeof(double), c->stream));
  }
  TRY(DALLOC(c, &c->V, (size_t)d * d));
  TRY(DALLOC(c, &c->rne, (size_t)c->nmon));
  TRY(DALLOC(c, &c->lwbuf, (size_t)c->Bmax * Pl));
  const int ntiles = (int)((Pl + ESS_TILE - 1) / ESS_TILE);
  TRY(DALLOC(c, &c->essparts, (size_t)c->Bmax * ntiles * 3));
  TRY(DALLOC(c, &c->essslice, (size_t)c->Bmax * 3));
  TRY(DALLOC(c, &c->grp_ms, (size_t)c->Jl * 2));
  if (const char* e = getenv("SPS_INC_CAP")) c->inc_cap = std::max(1, atoi(e));  // (test hook: tiny capacity)
  TRY(DALLOC(c, &c->inc_dev, (size_t)c->inc_cap));
  if (cfg.tempering == SPS_DATA_TEMPERING) {
    TRY(DALLOC(c, &c->lse, (size_t)c->n + 1));
    TRY(DALLOC(c, &c->logpl, (size_t)c->n));
  }
  TRY(DALLOC(c, &c->Lj, (size_t)c->Jl));
  if (c->xchg) {
    TRY(DALLOC(c, &c->essgath, (size_t)c->Bmax * 3 * c->G));
    TRY(DALLOC(c, &c->grp_ms_gath, (size_t)c->J * 2));
    TRY(DALLOC(c, &c->Lj_gath, (size_t)c->J));
  } else {
    c->essgath = c->essslice;
    c->grp_ms_gath = c->grp_ms;
    c->Lj_gath = c->Lj;
  }
  TRY(DALLOC(c, &c->scal, 8));
  TRY(DALLOC(c, &c->pw_parts, (size_t)PW_BLOCKS * 64 * 2));
  TRY(DALLOC(c, &c->pw_slice, 64 * 2));
  if (c->xchg) TRY(DALLOC(c, &c->pw_gath, (size_t)64 * 2 * c->G));
  else c->pw_gath = c->pw_slice;
  TRY(DALLOC(c, &c->mx_parts, MX_BLOCKS));
  TRY(DALLOC(c, &c->mx_slice, 1));
  if (c->xchg) TRY(DALLOC(c, &c->mx_gath, (size_t)c->G));
  else c->mx_gath = c->mx_slice;
  TRY(DALLOC(c, &c->ctl, 1));
  if (getenv("SPS_TIMELINE")) {
    TRY(DALLOC(c, &c->tl, (size_t)TL_W * TL_ROWS));
    CU(c, cudaMemsetAsync(c->tl, 0, sizeof(unsigned long long) * TL_W * TL_ROWS, c->stream));
    const int* steps = &c->ctl->steps_done;
    CU(c, cudaMemcpyToSymbolAsync(g_tl, &c->tl, sizeof(c->tl), 0, cudaMemcpyHostToDevice, c->stream));
    CU(c, cudaMemcpyToSymbolAsync(g_tl_steps, &steps, sizeof(steps), 0, cudaMemcpyHostToDevice, c->stream));
  }
  std::memset(c->hctl, 0, sizeof(Ctl));
  c->hctl->h = cfg.h_init;
  CU(c, cudaMemcpyAsync(c->ctl, c->hctl, sizeof(Ctl), cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaMemsetAsync(c->Lj, 0, sizeof(double) * c->Jl, c->stream));
  // inputs (host -> device); synchronous copies so the caller may free on return
  CU(c, cudaMemcpyAsync(c->X, X, sizeof(double) * c->n * c->k, cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaMemcpyAsync(c->y, y, sizeof(int32_t) * c->n, cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaMemcpyAsync(c->mu, prior_mean, sizeof(double) * d, cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaMemcpyAsync(c->shift, prior_mean, sizeof(double) * d, cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaMemcpyAsync(c->V, prior_cov, sizeof(double) * d * d, cudaMemcpyHostToDevice, c->stream));
  if (cfg.n_monitors > 0)
    CU(c, cudaMemcpyAsync(c->mon, cfg_in->monitors, sizeof(double) * c->nmon * d, cudaMemcpyHostToDevice, c->stream));
  {
    const int64_t tot = (int64_t)c->n * c->ldx;
    k_prep_X<<<(unsigned)((tot + 255) / 256), 256, 0, c->stream>>>(c->X, c->y, c->n, c->k, c->C, c->ldx, c->Xs,
                                                                     c->ctl);
    CHECK_LAUNCH(c);
    CU(c, cudaMemsetAsync(c->Xs + tot, 0, 2 * sizeof(double), c->stream));
    if (c->oz_KB > 0) {  // observation tile images of the sign-flipped X (ozaki.cuh)
      const int64_t ot = (c->n + OZ_NT - 1) / OZ_NT;
      TRY(DALLOC(c, &c->oz_X, (size_t)ot * oz_tile_bytes(OZ_NT, c->oz_KB)));
      TRY(DALLOC(c, &c->oz_xamax, 8));
      CU(c, cudaMemsetAsync(c->oz_xamax, 0, 8 * sizeof(int), c->stream));
      k_oz_slice<<<(unsigned)((ot * OZ_NT + 127) / 128), 128, 0, c->stream>>>(c->Xs, c->n, c->ldx, c->k, c->oz_KB, OZ_NT,
                                                                                1, 0, c->oz_X, nullptr, c->oz_xamax);
      CHECK_LAUNCH(c);
      const int ob = c->oz_KB == 2 ? oz_smem_bytes<2>() : c->oz_KB == 3 ? oz_smem_bytes<3>() : oz_smem_bytes<4>();
      auto fn = c->oz_KB == 2 ? k_oz_loglik<2> : c->oz_KB == 3 ? k_oz_loglik<3> : k_oz_loglik<4>;
      CU(c, cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, ob));
      // particle images for this rank's P_local (the M steps' launches, captured into graphs)
      c->oz_T_cap = (size_t)((c->Pl + OZ_MT - 1) / OZ_MT) * oz_tile_bytes(OZ_MT, c->oz_KB);
      TRY(DALLOC(c, &c->oz_T, c->oz_T_cap));
    }
    k_colmeans<<<(c->k + 127) / 128, 128, 0, c->stream>>>(c->X, c->n, c->k, c->xbar);
    CHECK_LAUNCH(c);
    if (cfg.n_monitors <= 0) {
      k_default_monitors<<<1, 256, 0, c->stream>>>(c->k, c->C, c->mon);
      CHECK_LAUNCH(c);
    }
    const size_t smem = sizeof(double) * d * d;
    CU(c, cudaFuncSetAttribute(k_chol_prior, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
    k_chol_prior<<<1, 256, smem, c->stream>>>(c->V, d, c->Lprior, c->ctl);
    CHECK_LAUNCH(c);
    CU(c, cudaFuncSetAttribute(k_prior_precision, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
    k_prior_precision<<<1, 128, smem, c->stream>>>(c->Lprior, d, c->Sinv, c->Rp);
    CHECK_LAUNCH(c);
    const size_t ldp = (size_t)round_up(d, 4) * sizeof(double);
    CU(c, cudaMemcpy2DAsync(c->LpriorP, ldp, c->Lprior, d * sizeof(double), d * sizeof(double), d,
                            cudaMemcpyDeviceToDevice, c->stream));
    CU(c, cudaMemcpy2DAsync(c->SinvP, ldp, c->Sinv, d * sizeof(double), d * sizeof(double), d,
                            cudaMemcpyDeviceToDevice, c->stream));
    CU(c, cudaMemcpy2DAsync(c->RpP, ldp, c->Rp, d * sizeof(double), d * sizeof(double), d,
                            cudaMemcpyDeviceToDevice, c->stream));
    // one-time kernel attributes (dynamic shared memory above 48 KB)
    const int big = 200 * 1024;
    CU(c, cudaFuncSetAttribute(k_propose<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_propose<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    // the side-stream normals use no shared memory; with the default (L1-leaning) carveout the SMs
    // they run on cannot take a 111 KB accept block until they drain and reconfigure (SPS_TIMELINE:
    // accept started 18 us late), so they request the max-shared split like the M-step kernels
    CU(c, cudaFuncSetAttribute(k_normals, cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared));
    CU(c, cudaFuncSetAttribute(k_finalize, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_mom_reduce, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_mom_reduce_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_mom_reduce_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    {  // largest of 16 / 8 CTAs per cluster the device can co-schedule with the finalize smem
      static const bool no_cl = getenv("SPS_NO_CLUSTER_REDUCE") != nullptr;
      const size_t fsm = (size_t)fin_smem_doubles(d, c->J, c->nmon, true) * sizeof(double);
      for (int cl : {16, 8}) {
        if (no_cl || c->xchg || fsm > 200 * 1024) break;
        cudaLaunchConfig_t lc = {};
        lc.gridDim = dim3((unsigned)cl);
        lc.blockDim = dim3(256);
        lc.dynamicSmemBytes = fsm;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = (unsigned)cl;
        at[0].val.clusterDim.y = at[0].val.clusterDim.z = 1;
        lc.attrs = at;
        lc.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_mom_reduce_cl, &lc) == cudaSuccess && nclusters > 0) {
          c->red_cluster = cl;
          break;
        }
        cudaGetLastError();
      }
    }
    CU(c, cudaFuncSetAttribute(k_accept_mom, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_tile<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_tile<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_tile<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_tile<5>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_mom_rb<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_mom_rb<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_mom_rb<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_accept_mom_rb<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
#define PRB_ATTR(KK_)                                                                                    \
  CU(c, cudaFuncSetAttribute(k_propose_rb<KK_, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, big)); \
  CU(c, cudaFuncSetAttribute(k_propose_rb<KK_, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    PRB_ATTR(1) PRB_ATTR(2) PRB_ATTR(3) PRB_ATTR(4) PRB_ATTR(5) PRB_ATTR(6) PRB_ATTR(7) PRB_ATTR(8)
#undef PRB_ATTR
    CU(c, cudaFuncSetAttribute(k_functional_stats, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_resample, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
    CU(c, cudaFuncSetAttribute(k_cphase_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, big));
  }
  {
    sps_status st = read_ctl(c);
    if (st == SPS_E_NUMERIC) return fail(c, SPS_E_CONFIG, "prior covariance is not positive definite");
    if (st != SPS_OK) return st;
  }
  CU(c, cudaEventCreate(&c->ev0));
  CU(c, cudaEventCreate(&c->ev1));
  if (c->guarded && getenv("SPS_GUARD_POKE")) {  // test hook: an 8-byte overrun past the named buffer
    const char* want = getenv("SPS_GUARD_POKE");
    for (const auto& g : c->guards)
      if (!std::strcmp(g.name, want)) CU(c, cudaMemsetAsync(g.base + GUARD_BYTES + g.bytes, 0, 8, c->stream));
  }
  return sps_reset(c, cfg.seed, cfg.pass);
}

sps_status sps_check_guards(sps_ctx* c, int64_t* n_corrupt) {
  if (!c) return SPS_E_CONFIG;
  if (n_corrupt) *n_corrupt = 0;
  if (!c->guarded) return fail(c, SPS_E_CONFIG, "sps_check_guards: context created without SPS_GUARD=1");
  CU(c, cudaSetDevice(c->cfg.device));
  if (c->aux) CU(c, cudaStreamSynchronize(c->aux));
  CU(c, cudaStreamSynchronize(c->stream));
  std::vector<unsigned char> zone(GUARD_BYTES);
  int64_t bad = 0;
  const char* first = nullptr;
  int64_t first_off = 0;
  for (const auto& g : c->guards)
    for (int side = 0; side < 2; ++side) {
      const char* z = side == 0 ? g.base : g.base + GUARD_BYTES + g.bytes;
      CU(c, cudaMemcpy(zone.data(), z, GUARD_BYTES, cudaMemcpyDeviceToHost));
      for (size_t i = 0; i < GUARD_BYTES; ++i)
        if (zone[i] != GUARD_FILL) {
          if (!first) {
            first = g.name;
            first_off = side == 0 ? (int64_t)i - (int64_t)GUARD_BYTES : (int64_t)(g.bytes + i);
          }
          ++bad;
        }
    }
  if (n_corrupt) *n_corrupt = bad;
  if (bad)
    return fail(c, SPS_E_GUARD, "guard zones overwritten: %lld bytes; first: %s at byte offset %lld", (long long)bad,
                first, (long long)first_off);
  return SPS_OK;
}

sps_status sps_reset(sps_ctx* c, uint64_t seed, int32_t pass) {
  if (!c) return SPS_E_CONFIG;
  CU(c, cudaSetDevice(c->cfg.device));
  c->cfg.seed = seed;
  c->cfg.pass = pass;
  c->t = 0;
  c->phi = 0.0;
  c->ell = 0;
  c->mstep = 0;
  c->need_pre_moments = false;
  c->cphase_done = false;
  c->finished = false;
  c->logml = 0.0;
  c->pairs = 0.0;
  c->tr_t.clear();
  c->tr_R.clear();
  c->tr_h.clear();
  c->tr_phi.clear();
  c->tr_inc.clear();
  c->tr_rne.clear();
  c->inc_base = 0;
  c->last_adv = 0;
  c->pre_normals_step = -1;
  c->launches = c->k1_launches = c->syncs = 0;
  c->k1_pairs = c->k1_ms = 0.0;
  c->host_launch_us = c->host_wait_us = c->host_graph_us = 0.0;
  c->graph_updates = c->graph_instantiations = 0;
  for (int q = 0; q < 16; ++q) {
    c->cat_ms[q] = 0.0;
    c->cat_n[q] = 0;
  }
  if (c->stream) CU(c, cudaStreamSynchronize(c->stream));
  c->prof_open.clear();
  c->prof_next = 0;
  const int64_t Pl = c->Pl;
  std::memset(c->hctl, 0, sizeof(Ctl));
  c->hctl->h = c->cfg.h_init;
  CU(c, cudaMemcpyAsync(c->ctl, c->hctl, sizeof(Ctl), cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaMemsetAsync(c->Lj, 0, sizeof(double) * c->Jl, c->stream));
  CU(c, cudaMemcpyAsync(c->shift, c->mu, sizeof(double) * c->d, cudaMemcpyDeviceToDevice, c->stream));
  // Algorithm 1 step 1: theta_jn ~iid p(theta)
  TRY(launch_normals(c, TAG_INIT, 0u, 0));
  TRY(launch_draw(c, 0, nullptr, c->LpriorP, c->theta, c->lp, nullptr));
  CU(c, cudaEventRecord(c->ev_zfree[0], c->stream));
  if (c->cfg.tempering == SPS_POWER_TEMPERING) {
    int nch = 1;
    TRY(launch_loglik(c, c->theta, c->d, Pl, 0, c->n, c->part, c->max_chunks, &nch));
    k_sum_chunks<<<(unsigned)((Pl + 255) / 256), 256, 0, c->stream>>>(c->part, nch, Pl, c->L);
    CHECK_LAUNCH(c);
    c->pairs += (double)c->P * c->n;
  } else {
    CU(c, cudaMemsetAsync(c->L, 0, sizeof(double) * Pl, c->stream));
  }
  TRY(read_ctl(c));
  return SPS_OK;
}

sps_status sps_set_profiling(sps_ctx* c, int32_t on) {
  if (!c) return SPS_E_CONFIG;
  c->profiling = on != 0;
  return SPS_OK;
}

sps_status sps_get_counters(const sps_ctx* cc, sps_counters* out) {
  if (!cc || !out) return SPS_E_CONFIG;
  sps_ctx* c = const_cast<sps_ctx*>(cc);
  TRY(prof_resolve(c));
  if (c->trace && c->trace_n) {
    static const char* nm[] = {"reduce", "ticket->fin", "stage", "theta-bar", "V", "chol|RNE", "stats+writes",
                               "host slot", "start skew", "longest block", "moment block"};
    fprintf(stderr, "SPS_TRACE mean ns over %d finalizes:", c->trace_n);
    for (int q = 0; q < 11; ++q) fprintf(stderr, " %s=%.0f", nm[q], c->trace_acc[q] / c->trace_n);
    fprintf(stderr, "\n");
    if (false) {}
    if (c->trace_acc[17] > 0) {
      static const char* an[] = {"load", "decide", "writeback+dmma", "combine", "kernel span", "gap->reduce"};
      fprintf(stderr, "SPS_TRACE accept (block 0) mean ns over %.0f:", c->trace_acc[17]);
      for (int q = 0; q < 6; ++q) fprintf(stderr, " %s=%.0f", an[q], c->trace_acc[11 + q] / c->trace_acc[17]);
      fprintf(stderr, "\n");
    }
  }
  if (c->tl && c->tl_rows) {
    static const char* nm[] = {"propose", "normals", "K1", "accept", "reduce", "finalize", "gap K1<-propose",
                               "gap accept<-K1", "gap reduce<-accept", "gap fin<-reduce", "normals start-propose end",
                               "normals end-K1 end", "gap next propose<-fin", "step", "acc0 load", "acc0 decide",
                               "acc0 wb+dmma", "acc0 combine..end(all)", "fin stage", "fin theta-bar", "fin V",
                               "fin chol|RNE", "fin(chol only)", "fin(RNE w1 only)"};
    fprintf(stderr, "SPS_TIMELINE mean us over %d steps:", c->tl_rows);
    for (int q = 0; q < 24; ++q) fprintf(stderr, " %s=%.2f", nm[q], c->tl_acc[q] / c->tl_rows / 1e3);
    fprintf(stderr, " gap next propose<-fin after even / odd steps=%.2f / %.2f\n",
            c->tl_gap_par[0][0] / std::max(1.0, c->tl_gap_par[0][1]) / 1e3,
            c->tl_gap_par[1][0] / std::max(1.0, c->tl_gap_par[1][1]) / 1e3);
    static const char* bn[] = {"t<=32", "t<=64", "t<=128", "t<=256", "t<=512", "t>512"};
    for (int b = 0; b < 6; ++b)
      if (c->tl_bin[b][0] > 0)
        fprintf(stderr,
                c->fu_fn ? "SPS_TIMELINE %-7s steps %5.0f  K1 %7.2f us  step %7.2f us  gap %5.2f us  fused: kernel %.2f "
                           "-> reduce end %.2f -> finalize start %.2f finalize %.2f\n"
                         : "SPS_TIMELINE %-7s steps %5.0f  K1 %7.2f us  step %7.2f us  gap %5.2f us  K1 blk0: release %.2f "
                           "theta %.2f rest %.2f  last block start %.2f\n",
                bn[b], c->tl_bin[b][0], c->tl_bin[b][1] / c->tl_bin[b][0] / 1e3, c->tl_bin[b][2] / c->tl_bin[b][0] / 1e3,
                c->tl_bin[b][3] / c->tl_bin[b][0] / 1e3, c->tl_bin[b][4] / c->tl_bin[b][0] / 1e3,
                c->tl_bin[b][5] / c->tl_bin[b][0] / 1e3, c->tl_bin[b][6] / c->tl_bin[b][0] / 1e3,
                c->tl_bin[b][7] / c->tl_bin[b][0] / 1e3);
  }
  out->launches = c->launches;
  out->k1_launches = c->k1_launches;
  out->k1_pairs = c->k1_pairs;
  out->k1_ms = c->k1_ms;
  out->syncs = c->syncs;
  out->cat_ms[14] = c->host_launch_us / 1e3;
  out->cat_ms[15] = c->host_wait_us / 1e3;
  out->cat_n[14] = out->cat_n[15] = 1;
  for (int q = 0; q < 14; ++q) {
    out->cat_ms[q] = c->cat_ms[q];
    out->cat_n[q] = c->cat_n[q];
  }
  out->cat_ms[13] = c->host_graph_us / 1e3;  // host: M-step graph capture + update / instantiate
  out->cat_n[13] = c->graph_updates + 1000 * c->graph_instantiations;
  return SPS_OK;
}

sps_status sps_shard(const sps_ctx* ctx, int64_t* P_local, int32_t* group0, int32_t* J_local) {
  if (!ctx) return SPS_E_CONFIG;
  if (P_local) *P_local = ctx->Pl;
  if (group0) *group0 = ctx->g0;
  if (J_local) *J_local = ctx->Jl;
  return SPS_OK;
}

sps_status sps_loglik(sps_ctx* c, const double* theta_dev, int64_t P, int32_t ld, int32_t t0, int32_t t1,
                      double* out_dev) {
  if (!c) return SPS_E_CONFIG;
  NvtxRange nvtx_("sps_loglik");
  if (!theta_dev || !out_dev || P < 0 || ld < c->d || t0 < 0 || t1 < t0 || t1 > c->n)
    return fail(c, SPS_E_CONFIG, "sps_loglik: bad arguments");
  if (P == 0) return SPS_OK;
  CU(c, cudaSetDevice(c->cfg.device));
  // chunk partials: up to 64 chunks per particle, in a scratch buffer grown on demand
  const int max_chunks = 64;
  const size_t need = (size_t)max_chunks * (size_t)P;
  if (need > c->ll_scratch_cap) {
    dfree(c, c->ll_scratch, c->stream);
    c->ll_scratch = nullptr;
    c->ll_scratch_cap = 0;
    TRY(DALLOC(c, &c->ll_scratch, need));
    c->ll_scratch_cap = need;
  }
  int nch = 1;
  TRY(launch_loglik(c, theta_dev, ld, P, t0, t1, c->ll_scratch, max_chunks, &nch));
  k_sum_chunks<<<(unsigned)((P + 255) / 256), 256, 0, c->stream>>>(c->ll_scratch, nch, P, out_dev, c->llbad);
  CHECK_LAUNCH(c);
  // non-finite L_p: locate (p, t) on the device; reported by the next sps_sync (no host round trip here)
  k_ll_locate<<<1, 256, 0, c->stream>>>(theta_dev, ld, c->X, c->y, c->k, c->C, t0, t1, c->llbad, c->dllbad);
  CHECK_LAUNCH(c);
  return SPS_OK;
}

sps_status sps_sync(sps_ctx* c) {
  if (!c) return SPS_E_CONFIG;
  CU(c, cudaSetDevice(c->cfg.device));
  CU(c, cudaStreamSynchronize(c->aux));
  CU(c, cudaStreamSynchronize(c->stream));
  c->syncs += 1;
  if (c->hllbad && c->hllbad[0] != 0x7fffffff) {
    const int p = c->hllbad[0], t = c->hllbad[1];
    c->hllbad[1] = c->hllbad[0] = 0x7fffffff;
    return fail(c, SPS_E_NUMERIC, "sps_loglik: non-finite log-likelihood at particle p = %d, observation t = %d", p, t);
  }
  return SPS_OK;
}

// One C phase + S phase.
// Pull the device-recorded log-ML increments of cycles inc_base..ell-1 (cycle order).
static sps_status sync_incs(sps_ctx* c) {
  const int pending = c->ell - c->inc_base;
  if (pending <= 0) return SPS_OK;
  std::vector<double> h((size_t)pending);
  CU(c, cudaMemcpyAsync(h.data(), c->inc_dev, sizeof(double) * pending, cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  for (double inc : h) {
    c->logml += inc;
    c->tr_inc.push_back(inc);
  }
  c->inc_base = c->ell;
  return SPS_OK;
}

sps_status sps_cphase(sps_ctx* c, int32_t t_target, double phi_target, int32_t* t_new, double* phi_new,
                      double* logml_inc) {
  if (!c) return SPS_E_CONFIG;
  NvtxRange nvtx_("sps C phase + S phase");
  CU(c, cudaSetDevice(c->cfg.device));
  if (c->finished || final_cycle(c)) return fail(c, SPS_E_STATE, "sps_cphase: all data already absorbed");
  if (c->ell >= c->cfg.max_cycles) return fail(c, SPS_E_CONFIG, "max_cycles exceeded");
  const int64_t Pl = c->Pl;
  const double P = (double)c->P;
  const unsigned pgrid = (unsigned)((Pl + 255) / 256);
  // the next M phase's first-step normals depend only on the step number: generate them on the
  // low-priority side stream now, overlapped with the C and S phases (host round trips included)
  if (!c->profiling) {
    CU(c, cudaEventRecord(c->ev_zfree[c->mstep & 1u], c->stream));
    TRY(launch_normals(c, TAG_PROPOSAL, c->mstep, (int)(c->mstep & 1u)));
    c->pre_normals_step = (int64_t)c->mstep;
  }
  PROF_BEGIN(c);
  if (c->cfg.tempering == SPS_DATA_TEMPERING) {
    // ---- absorb observations one at a time ----
    if (t_target >= 0 && (t_target <= c->t || t_target > c->n))
      return fail(c, SPS_E_CONFIG, "t_target out of range");
    CU(c, cudaMemsetAsync(c->lw_cur, 0, sizeof(double) * Pl, c->stream));
    int s = c->t;
    int B = 8;  // first galloping chunk: twice the last cycle's advance (usually one chunk, one sync)
    while (B < 2 * c->last_adv && B < c->Bmax) B *= 2;
    const int ntiles = (int)((Pl + ESS_TILE - 1) / ESS_TILE);
    const size_t scan_smem = sizeof(double) * c->d * SCAN_LD;
    CU(c, cudaFuncSetAttribute(k_cphase_scan, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)scan_smem + 1024));
    for (;;) {
      int Be = std::min(std::min(B, c->Bmax), c->n - s);
      if (t_target >= 0) Be = std::min(Be, t_target - s);
      k_cphase_scan<<<(unsigned)((Pl + SCAN_PB - 1) / SCAN_PB), SCAN_PB * SCAN_Q, scan_smem, c->stream>>>(
          c->Xs, c->y, c->ldx, c->k, c->C, c->theta, c->d, Pl, s, Be, c->lw_cur, c->lwbuf);
      CHECK_LAUNCH(c);
      c->pairs += P * Be;
      // pooled (M, S1, S2) per observation: the ESS rule (adaptive) and the log predictive
      // likelihoods (both modes; with a fixed target the crossing is known on the host)
      k_ess_partials<<<dim3((unsigned)ntiles, (unsigned)Be), 256, 0, c->stream>>>(c->lwbuf, Pl, ESS_TILE,
                                                                                 c->essparts);
      CHECK_LAUNCH(c);
      k_ess_rank<<<(unsigned)((Be + 7) / 8), 256, 0, c->stream>>>(c->essparts, ntiles, Be, c->essslice);
      CHECK_LAUNCH(c);
      TRY(gather(c, c->essslice, c->essgath, (size_t)Be * 3));
      k_ess_final<<<1, 32, 0, c->stream>>>(c->essgath, c->G, Be, s, c->n, c->cfg.ess_frac, P, c->ctl,
                                           t_target >= 0 ? t_target : -1, c->t, c->lse, c->logpl);
      CHECK_LAUNCH(c);
      int sstar = -1;
      if (t_target >= 0) {
        if (s + Be == t_target) sstar = t_target;
      } else {
        TRY(read_ctl(c));
        sstar = c->hctl->s_star;
      }
      if (sstar > 0) {
        k_take_lw<<<pgrid, 256, 0, c->stream>>>(c->lwbuf, sstar - s - 1, Pl, c->lw, c->L);
        CHECK_LAUNCH(c);
        c->last_adv = sstar - c->t;
        c->t = sstar;
        break;
      }
      s += Be;
      B *= 2;
    }
  } else {
    // ---- power tempering (R5): Delta phi on the 2^-48 grid of the remaining increment ----
    const double rem = 1.0 - c->phi;
    double dphi;
    if (phi_target >= 0) {
      if (!(phi_target > c->phi && phi_target <= 1.0)) return fail(c, SPS_E_CONFIG, "phi_target out of range");
      dphi = phi_target - c->phi;
    } else {
      k_block_max<<<MX_BLOCKS, 256, 0, c->stream>>>(c->L, Pl, c->mx_parts);
      k_max_reduce<<<1, 32, 0, c->stream>>>(c->mx_parts, MX_BLOCKS, c->mx_slice);
      CHECK_LAUNCH(c);
      TRY(gather(c, c->mx_slice, c->mx_gath, 1));
      k_max_reduce<<<1, 32, 0, c->stream>>>(c->mx_gath, c->G, c->scal);
      CHECK_LAUNCH(c);
      auto round = [&](int ncand) -> sps_status {
        k_power_partials<<<PW_BLOCKS, 256, 0, c->stream>>>(c->L, Pl, c->scal, c->ctl, ncand, rem, c->pw_parts);
        k_power_rank<<<1, 64, 0, c->stream>>>(c->pw_parts, PW_BLOCKS, ncand, c->pw_slice);
        CHECK_LAUNCH(c);
        TRY(gather(c, c->pw_slice, c->pw_gath, 64 * 2));
        k_power_decide<<<1, 32, 0, c->stream>>>(c->pw_gath, c->G, ncand, c->cfg.ess_frac, P, c->ctl);
        CHECK_LAUNCH(c);
        return SPS_OK;
      };
      TRY(round(0));
      TRY(read_ctl(c));
      if (c->hctl->q_ok_full) {
        dphi = rem;
      } else {
        c->hctl->q_lo = 0;
        c->hctl->q_hi = 1ull << 48;
        CU(c, cudaMemcpyAsync(&c->ctl->q_lo, &c->hctl->q_lo, 2 * sizeof(unsigned long long), cudaMemcpyHostToDevice,
                              c->stream));
        for (int r = 0; r < 8; ++r) TRY(round(63));
        TRY(read_ctl(c));
        unsigned long long q = c->hctl->q_lo;
        if (q == 0) q = 1;
        dphi = ((double)q * 0x1p-48) * rem;
      }
    }
    k_power_apply<<<pgrid, 256, 0, c->stream>>>(c->L, Pl, dphi, c->lw);
    CHECK_LAUNCH(c);
    // a fixed schedule (Algorithm 3 pass 2) lands exactly on the recorded phi_l
    c->phi = phi_target >= 0 ? phi_target : ((dphi == rem) ? 1.0 : c->phi + dphi);
  }
  PROF_END(c, CAT_CPHASE);
  // ---- S phase + log-ML increments (R10) ----
  // room for this cycle's increment in inc_dev: pull the pending ones first (cycles inc_base..ell-1)
  if (c->ell - c->inc_base >= c->inc_cap) TRY(sync_incs(c));
  c->ell += 1;
  PROF_BEGIN(c);
  {
    NvtxRange nvtx_s("S phase");
    const size_t smem = (size_t)c->N * (8 + 4);
    CU(c, cudaFuncSetAttribute(k_resample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
    k_resample<<<c->Jl, 1024, smem, c->stream>>>(c->lw, c->N, c->d, c->cfg.resampling, c->cfg.seed, (uint32_t)c->ell,
                                                 (uint32_t)c->cfg.pass, c->g0, c->theta, c->L, c->lp, c->theta2,
                                                 c->L2, c->lp2, c->grp_ms, c->Lj, nullptr, c->ctl);
    CHECK_LAUNCH(c);
    std::swap(c->theta, c->theta2);
    std::swap(c->L, c->L2);
    std::swap(c->lp, c->lp2);
    TRY(gather(c, c->grp_ms, c->grp_ms_gath, (size_t)c->Jl * 2));
    k_logml_pooled<<<1, 32, 0, c->stream>>>(c->grp_ms_gath, c->J, P, c->ctl, c->inc_dev + (c->ell - 1 - c->inc_base));
    CHECK_LAUNCH(c);
  }
  PROF_END(c, CAT_RESAMPLE);
  c->need_pre_moments = true;
  c->cphase_done = true;
  c->tr_t.push_back(c->t);
  c->tr_phi.push_back(c->phi);
  if (t_new) *t_new = c->t;
  if (phi_new) *phi_new = c->phi;
  if (logml_inc) {  // the caller wants it now: one round trip (sps_run does not ask)
    TRY(sync_incs(c));
    TRY(read_ctl(c));
    *logml_inc = c->tr_inc.back();
  }
  return SPS_OK;
}

// Debug (SPS_TRACE): accumulate the phase clocks of the last finished fused
// reduce + finalize (serializes the pipeline; timings of phases only).
static void trace_accumulate(sps_ctx* c) {
  cudaStreamSynchronize(c->stream);
  const unsigned long long* t = c->trace;
  const int d = c->d, nb = (d * (d + 1) / 2 + 31) / 32 + (c->Jl * d + 255) / 256 + 1;
  unsigned long long s0 = ~0ull, s1 = 0, e1 = 0, dmax = 0, dm = 0;
  for (int b = 0; b < nb; ++b) {
    s0 = std::min(s0, t[8 + b]);
    s1 = std::max(s1, t[8 + b]);
    e1 = std::max(e1, t[8 + nb + b]);
    dmax = std::max(dmax, t[8 + nb + b] - t[8 + b]);
    if (b == 0) dm = t[8 + nb + b] - t[8 + b];
  }
  c->trace_acc[8] += (double)(s1 - s0);  // start skew
  c->trace_acc[9] += (double)dmax;       // longest block
  c->trace_acc[10] += (double)dm;        // a moment block
  if (t[0] < s0 || t[6] < t[0]) return;  // stopped step (no finalize)
  if (t[68] > t[64] && t[70] >= t[68]) {  // accept kernel: block 0 phases, latest block end
    c->trace_acc[11] += (double)(t[65] - t[64]);
    c->trace_acc[12] += (double)(t[66] - t[65]);
    c->trace_acc[13] += (double)(t[67] - t[66]);
    c->trace_acc[14] += (double)(t[68] - t[67]);
    c->trace_acc[15] += (double)(t[70] - t[64]);
    c->trace_acc[16] += (double)(s0 - t[70]);  // last accept block end -> first reduce block start
    c->trace_acc[17] += 1;
  }
  c->trace_acc[0] += (double)(e1 - s0);      // reduce phase: first block start -> last block ticket
  c->trace_acc[1] += (double)(t[0] - e1);    // ticket -> finalize start
  for (int q = 1; q <= 6; ++q) c->trace_acc[1 + q] += (double)(t[q] - t[q - 1]);
  c->trace_n += 1;
  c->trace[70] = 0;  // latest accept block end (atomicMax), re-armed (the stream is idle here)
}

// Debug (SPS_TIMELINE): mean kernel spans and gaps over the finished steps of a
// phase (0 propose, 1 normals(next), 2 K1, 3 accept, 4 reduce, 5 finalize block).
static sps_status timeline_accumulate(sps_ctx* c, int R) {
  CU(c, cudaStreamSynchronize(c->stream));
  CU(c, cudaStreamSynchronize(c->aux));
  std::vector<unsigned long long> h((size_t)TL_W * TL_ROWS);
  const int rows = std::min(R, TL_ROWS);
  CU(c, cudaMemcpy(h.data(), c->tl, sizeof(unsigned long long) * TL_W * rows, cudaMemcpyDeviceToHost));
  for (int r = 0; r < rows; ++r) {
    const unsigned long long* t = &h[(size_t)r * TL_W];
    bool ok = true;
    for (int k = 0; k < 6; ++k) ok = ok && t[2 * k] && t[2 * k + 1] >= t[2 * k];
    if (!ok) continue;
    for (int k = 0; k < 6; ++k) c->tl_acc[k] += (double)(t[2 * k + 1] - t[2 * k]);  // spans
    c->tl_acc[6] += (double)t[4] - (double)t[1];    // K1 start - propose end
    c->tl_acc[7] += (double)t[6] - (double)t[5];    // accept start - K1 end
    c->tl_acc[8] += (double)t[8] - (double)t[7];    // reduce start - accept end
    c->tl_acc[9] += (double)t[10] - (double)t[9];   // finalize start - reduce end
    c->tl_acc[10] += (double)t[2] - (double)t[1];   // normals start - propose end
    c->tl_acc[11] += (double)t[3] - (double)t[5];   // normals end - K1 end
    if (r + 1 < rows && h[(size_t)(r + 1) * TL_W]) {
      const double g = (double)h[(size_t)(r + 1) * TL_W] - (double)t[11];
      c->tl_acc[12] += g;
      c->tl_gap_par[r & 1][0] += g;  // even r: next step in the same graph body; odd: the next body
      c->tl_gap_par[r & 1][1] += 1;
    }
    c->tl_acc[13] += (double)t[11] - (double)t[0];  // step: propose start -> finalize end
    {
      const int tt = c->cfg.tempering == SPS_POWER_TEMPERING ? c->n : c->t;
      const int b = tt <= 32 ? 0 : tt <= 64 ? 1 : tt <= 128 ? 2 : tt <= 256 ? 3 : tt <= 512 ? 4 : 5;
      c->tl_bin[b][0] += 1;
      c->tl_bin[b][1] += (double)(t[5] - t[4]);
      c->tl_bin[b][2] += (double)(t[11] - t[0]);
      if (r + 1 < rows && h[(size_t)(r + 1) * TL_W]) c->tl_bin[b][3] += (double)h[(size_t)(r + 1) * TL_W] - (double)t[11];
      if (c->fu_fn) {  // fused M step: kernel start -> last tail, -> reduce end, -> finalize start, finalize
        c->tl_bin[b][4] += (double)t[7] - (double)t[0];
        c->tl_bin[b][5] += (double)t[9] - (double)t[7];
        c->tl_bin[b][6] += (double)t[10] - (double)t[9];
        c->tl_bin[b][7] += (double)t[11] - (double)t[10];
      } else if (t[24] && t[25] && t[26] && t[27]) {  // K1 phases: block (0,0) release / theta loaded / done, last block start
        c->tl_bin[b][4] += (double)t[25] - (double)t[4];
        c->tl_bin[b][5] += (double)t[26] - (double)t[25];
        c->tl_bin[b][6] += (double)t[27] - (double)t[26];
        c->tl_bin[b][7] += (double)t[24] - (double)t[4];
      }
    }
    if (t[16] && t[17] && t[18] && t[19] && t[20]) {  // finalize phases: stage / theta-bar / V / chol|RNE / tail
      c->tl_acc[18] += (double)t[16] - (double)t[10];
      c->tl_acc[19] += (double)t[17] - (double)t[16];
      c->tl_acc[20] += (double)t[18] - (double)t[17];
      c->tl_acc[21] += (double)t[19] - (double)t[18];
      c->tl_acc[22] += t[15] ? (double)t[15] - (double)t[18] : 0.0;  // warp 0: Cholesky
      c->tl_acc[23] += t[21] ? (double)t[21] - (double)t[18] : 0.0;  // warp 1: monitor RNEs
    }
    if (t[12] && t[13] && t[14]) {  // accept block 0: load / decide+writeback / dmma phases
      c->tl_acc[14] += (double)t[12] - (double)t[6];
      c->tl_acc[15] += (double)t[13] - (double)t[12];
      c->tl_acc[16] += (double)t[14] - (double)t[13];
      c->tl_acc[17] += (double)t[7] - (double)t[14];
    }
    c->tl_rows += 1;
  }
  CU(c, cudaMemsetAsync(c->tl, 0, sizeof(unsigned long long) * TL_W * TL_ROWS, c->stream));
  return SPS_OK;
}

// One M step (Algorithm 2 step 2(c)), fully enqueued:
// K8 propose -> K1 loglik of theta* on [0, t_l) -> K9+K6 accept & moments ->
// stats reduce -> gather -> K7 finalize (h, RNE, stop, chol(h V)) -> control
// block into mapped host slot `step & 1`, event evs[step & 1]; the next step's
// normals run alongside on the side stream.  Every kernel returns at once when
// the device stop flag is already set, so a step launched speculatively after
// the stopping step is a no-op.  graph: captured for replay (only the parity of
// `step` matters; the step number itself is device-resident).
static sps_status launch_mstep(sps_ctx* c, uint32_t step, bool allow_stop, bool graph = false) {
  const bool power = c->cfg.tempering == SPS_POWER_TEMPERING;
  const int t1 = power ? c->n : c->t;
  const double temper = power ? c->phi : 1.0;
  const int* stop = &c->ctl->stop;
  const int zs = (int)(step & 1u);
  if (c->fu_fn && t1 > 0) {  // one kernel: propose + K1 + accept + tile moments (fused.cuh)
    TRY(launch_fused(c, zs, t1, temper, stop, graph));
    TRY(moments_finalize(c, true, 1, temper, step, stop, c->LUbuf[zs], 1, allow_stop, zs, true, true));
  } else {
  TRY(launch_draw(c, zs, c->theta, c->Lprop, c->theta_s, c->lp_s, stop, graph, true));
  // the next step's normals: forked after accept into the reduce / finalize tail (default), or after
  // the proposal with a small resident footprint (SPS_NORMALS_FORK=propose, experiment)
  // (measured: forking at the proposal stretches the normals to ~60 us and delays the next step by
  // ~20 us; the tail fork, the default, costs the finalize SM some issue slots instead)
  static const bool fork_at_propose = getenv("SPS_NORMALS_FORK") && !strcmp(getenv("SPS_NORMALS_FORK"), "propose");
  if (fork_at_propose) {
    CU(c, cudaEventRecord(c->ev_fork, c->stream));
    TRY(launch_normals(c, TAG_PROPOSAL, step + 1u, (int)((step + 1u) & 1u), graph, true));
  }
  int nch = 1;
  TRY(launch_loglik(c, c->theta_s, c->d, c->Pl, 0, t1, c->part, c->max_chunks, &nch, stop));
  static const bool fork_at_k1 = getenv("SPS_NORMALS_FORK") && !strcmp(getenv("SPS_NORMALS_FORK"), "k1");
  if (fork_at_k1) {  // (experiment) after K1: overlap accept + reduce + finalize
    CU(c, cudaEventRecord(c->ev_fork, c->stream));
    TRY(launch_normals(c, TAG_PROPOSAL, step + 1u, (int)((step + 1u) & 1u), graph, true));
  }
  // next step's normals on the low-priority side stream, forked after accept: they fill the SMs
  // the reduce / one-block finalize tail leaves idle (SPS_TIMELINE: launched before K1 they held
  // every SM while K1 waited 17.8 us; forked after K1 they stretched accept from 13 to 25 us)
  TRY(moments_finalize(c, true, nch, temper, step, stop, c->LUbuf[zs], 1, allow_stop, zs, !fork_at_propose && !fork_at_k1));
  }
  if (graph) {
    CU(c, cudaStreamWaitEvent(c->stream, c->ev_join, 0));
    if (!c->capturing_loop) CU(c, cudaEventRecordWithFlags(c->evs[zs], c->stream, cudaEventRecordExternal));
  } else {
    CU(c, cudaEventRecord(c->ev_zfree[zs], c->stream));  // Zbuf / LUbuf[zs] consumed
    CU(c, cudaEventRecord(c->evs[zs], c->stream));
  }
  return SPS_OK;
}

// Kernel-node priorities of a captured M step: k_normals lowest, everything else highest.
static sps_status set_node_priorities(sps_ctx* c, cudaGraph_t g) {
  size_t n = 0;
  CU(c, cudaGraphGetNodes(g, nullptr, &n));
  std::vector<cudaGraphNode_t> nodes(n);
  CU(c, cudaGraphGetNodes(g, nodes.data(), &n));
  int lo = 0, hi = 0;
  CU(c, cudaDeviceGetStreamPriorityRange(&lo, &hi));
  for (cudaGraphNode_t nd : nodes) {
    cudaGraphNodeType t;
    CU(c, cudaGraphNodeGetType(nd, &t));
    if (t != cudaGraphNodeTypeKernel) continue;
    cudaKernelNodeParams kp{};
    CU(c, cudaGraphKernelNodeGetParams(nd, &kp));
    cudaKernelNodeAttrValue v{};
    v.priority = kp.func == (void*)k_normals ? lo : hi;
    CU(c, cudaGraphKernelNodeSetAttribute(nd, cudaKernelNodeAttributePriority, &v));
  }
  return SPS_OK;
}

// Capture the M step of both slot parities for this phase (t1, tempering, K
// fixed) and instantiate, or update the executable graphs of the previous phase
// in place (same topology; only kernel parameters and grids change).
static sps_status build_mstep_graphs(sps_ctx* c, bool allow_stop) {
  for (int par = 0; par < 2; ++par) {
    const int64_t l0 = c->launches, k0 = c->k1_launches;
    const double p0 = c->k1_pairs;
    CU(c, cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
    const sps_status st = launch_mstep(c, c->phase_step0 + (uint32_t)((par ^ (int)(c->phase_step0 & 1u)) & 1), allow_stop,
                                       true);
    c->capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(c->stream, &g);
    if (st != SPS_OK) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    CU(c, ee);
    TRY(set_node_priorities(c, g));
    c->g_launches[par] = c->launches - l0;
    c->g_k1[par] = c->k1_launches - k0;
    c->g_pairs[par] = c->k1_pairs - p0;
    c->launches = l0;
    c->k1_launches = k0;
    c->k1_pairs = p0;
    bool ok = false;
    if (c->gexec[par]) {
      cudaGraphExecUpdateResultInfo info;
      ok = cudaGraphExecUpdate(c->gexec[par], g, &info) == cudaSuccess;
      if (ok) c->graph_updates += 1;
      cudaGetLastError();
    }
    if (!ok) {
      if (c->gexec[par]) cudaGraphExecDestroy(c->gexec[par]);
      c->gexec[par] = nullptr;
      // per-node priorities (side-stream normals lowest): without this flag a replay schedules the
      // nodes with the launch stream's priority and the normals hold SMs the critical path needs
      const cudaError_t ei = cudaGraphInstantiateWithFlags(&c->gexec[par], g, cudaGraphInstantiateFlagUseNodePriority);
      cudaGraphDestroy(g);
      CU(c, ei);
      c->graph_instantiations += 1;
    } else {
      cudaGraphDestroy(g);
    }
  }
  return SPS_OK;
}

// Device-side M phase: a graph with one WHILE node whose body (captured from one M step) runs until
// the finalize kernel clears the condition (min RNE >= K, or the step cap).  Captured per phase and
// applied to the previous executable graph with cudaGraphExecUpdate when possible.
// M steps per body of the device-side loop (SPS_LOOP_BODY: tuning; even, 2..16; default 4: cfg2 run
// 148.2 / 147.0 / 147.3 / 147.7 ms at 2 / 4 / 6 / 8).
static int loop_body() {
  static const int b = [] {
    const char* e = getenv("SPS_LOOP_BODY");
    const int v = e ? atoi(e) : 4;
    return std::min(16, std::max(2, v / 2 * 2));
  }();
  return b;
}

static sps_status build_mstep_loop(sps_ctx* c, bool allow_stop, int rmax) {
  cudaGraph_t g = nullptr;
  CU(c, cudaGraphCreate(&g, 0));
  cudaGraphConditionalHandle h;
  CU(c, cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams np = {};
  np.type = cudaGraphNodeTypeConditional;
  np.conditional.handle = h;
  np.conditional.type = cudaGraphCondTypeWhile;
  np.conditional.size = 1;
  cudaGraphNode_t cn;
  CU(c, cudaGraphAddNode(&cn, g, nullptr, 0, &np));
  cudaGraph_t body = np.conditional.phGraph_out[0];
  const int64_t l0 = c->launches, k0 = c->k1_launches;
  const double p0 = c->k1_pairs;
  c->loop_cond = h;
  c->loop_rmax = rmax;
  CU(c, cudaStreamBeginCaptureToGraph(c->stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
  c->capturing = c->capturing_loop = true;
  // B (even) M steps per body: a loop-iteration boundary costs ~5.5 us more than the gap between two
  // steps of one body (SPS_TIMELINE: 6.8 vs 1.35 us); after a stop the body's remaining steps'
  // kernels return at once.  B even keeps each body position on one parity (Z / log u buffers).
  sps_status st = SPS_OK;
  for (int q = 0; q < loop_body() && st == SPS_OK; ++q) st = launch_mstep(c, c->phase_step0 + (uint32_t)q, allow_stop, true);
  c->capturing = c->capturing_loop = false;
  cudaGraph_t captured = nullptr;
  const cudaError_t ee = cudaStreamEndCapture(c->stream, &captured);
  if (st != SPS_OK || ee != cudaSuccess) {
    cudaGraphDestroy(g);
    if (st != SPS_OK) return st;
    CU(c, ee);
  }
  TRY(set_node_priorities(c, body));
  c->gl_launches = c->launches - l0;
  c->gl_k1 = c->k1_launches - k0;
  c->gl_pairs = c->k1_pairs - p0;
  c->launches = l0;
  c->k1_launches = k0;
  c->k1_pairs = p0;
  bool ok = false;
  if (c->gloop) {
    cudaGraphExecUpdateResultInfo info;
    ok = cudaGraphExecUpdate(c->gloop, g, &info) == cudaSuccess;
    if (ok) c->graph_updates += 1;
    cudaGetLastError();
  }
  if (!ok) {
    if (c->gloop) cudaGraphExecDestroy(c->gloop);
    c->gloop = nullptr;
    const cudaError_t ei = cudaGraphInstantiateWithFlags(&c->gloop, g, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(g);
    CU(c, ei);
    c->graph_instantiations += 1;
  } else {
    cudaGraphDestroy(g);
  }
  return SPS_OK;
}

static sps_status replay_mstep(sps_ctx* c, uint32_t step) {
  const int par = (int)(step & 1u);
  CU(c, cudaGraphLaunch(c->gexec[par], c->stream));
  c->launches += c->g_launches[par];
  c->k1_launches += c->g_k1[par];
  c->k1_pairs += c->g_pairs[par];
  return SPS_OK;
}

// Sigma_lr record (Algorithm 3 step 1): room for global M steps [0, need), contents kept.
static sps_status reserve_sigma(sps_ctx* c, int64_t need) {
  if (need <= c->sig_rec_cap) return SPS_OK;
  const int64_t cap = std::max<int64_t>(need, 2 * c->sig_rec_cap), dd = (int64_t)c->d * c->d;
  double* nb = nullptr;
  TRY(DALLOC(c, &nb, (size_t)(cap * dd)));
  if (c->sig_rec) {
    CU(c, cudaMemcpyAsync(nb, c->sig_rec, sizeof(double) * c->sig_rec_cap * dd, cudaMemcpyDeviceToDevice, c->stream));
    dfree(c, c->sig_rec, c->stream);
  }
  c->sig_rec = nb;
  c->sig_rec_cap = cap;
  return SPS_OK;
}

sps_status sps_mphase(sps_ctx* c, int32_t R_fixed, int32_t* R_out, double* min_rne, int32_t* h_out) {
  if (!c) return SPS_E_CONFIG;
  NvtxRange nvtx_("sps M phase");
  CU(c, cudaSetDevice(c->cfg.device));
  if (!c->cphase_done) return fail(c, SPS_E_STATE, "sps_mphase before sps_cphase");
  const bool power = c->cfg.tempering == SPS_POWER_TEMPERING;
  const int t1 = power ? c->n : c->t;
  const bool adaptive = R_fixed <= 0;
  const int Rmax = adaptive ? c->cfg.max_m_steps : R_fixed;
  // reset stop / step counter; moments + chol(h V) of the resampled particles
  CU(c, cudaMemsetAsync(&c->ctl->stop, 0, sizeof(int), c->stream));
  CU(c, cudaMemsetAsync(&c->ctl->steps_done, 0, sizeof(int), c->stream));
  if (c->recording) TRY(reserve_sigma(c, (int64_t)c->mstep + Rmax + 2));
  if (c->need_pre_moments) {
    TRY(moments_finalize(c, false, 1, 1.0, 0u, nullptr, nullptr, 0, false, -1));
    c->need_pre_moments = false;
  }
  const uint32_t step0 = c->mstep;
  c->phase_step0 = step0;
  static const bool no_graph = getenv("SPS_NO_GRAPH") != nullptr;
  static const bool no_loop = getenv("SPS_NO_LOOP") != nullptr;
  const bool graph = !c->xchg && !c->profiling && !no_graph;
  const bool loop = graph && !no_loop;
  if (c->pre_normals_step != (int64_t)step0) {
    // the first step's normals after all earlier work of the main stream (graph replays record no Zbuf events)
    CU(c, cudaEventRecord(c->ev_zfree[step0 & 1u], c->stream));
    TRY(launch_normals(c, TAG_PROPOSAL, step0, (int)(step0 & 1u)));
  }
  c->pre_normals_step = -1;
  if (loop) {  // the whole adaptive M phase on the device: one graph launch, one host sync
    const auto g0 = std::chrono::steady_clock::now();
    TRY(build_mstep_loop(c, adaptive, Rmax));
    c->host_graph_us +=
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - g0).count();
    CU(c, cudaStreamWaitEvent(c->stream, c->ev_zready[step0 & 1u], 0));
    const auto h0 = std::chrono::steady_clock::now();
    CU(c, cudaGraphLaunch(c->gloop, c->stream));
    CU(c, cudaEventRecord(c->evs[0], c->stream));
    const auto h1 = std::chrono::steady_clock::now();
    CU(c, cudaEventSynchronize(c->evs[0]));
    const auto h2 = std::chrono::steady_clock::now();
    c->host_launch_us += std::chrono::duration<double, std::micro>(h1 - h0).count();
    c->host_wait_us += std::chrono::duration<double, std::micro>(h2 - h1).count();
    c->syncs += 1;
    const Ctl got = c->hslot[0];
    const int r = got.steps_done;
    c->launches += c->gl_launches / loop_body() * r;  // (the body holds loop_body() steps)
    c->k1_launches += c->gl_k1 / loop_body() * r;
    c->k1_pairs += c->gl_pairs / loop_body() * r;
    c->pairs += (double)c->P * t1 * r;
    if (got.err == ERR_NUMERIC)
      return fail(c, SPS_E_NUMERIC, "numerical failure in the M phase (non-finite loglik or Cholesky failure "
                                    "after ridge; cf. PAPER.md:1024-1030)");
    if (adaptive && got.stop != 1)
      return fail(c, SPS_E_MIXING, "M phase did not reach RNE >= K in %d steps", c->cfg.max_m_steps);
    c->mstep = step0 + (uint32_t)r;
    if (c->tl) TRY(timeline_accumulate(c, r));
    *c->hctl = got;
    c->cphase_done = false;
    c->tr_R.push_back(r);
    c->tr_rne.push_back(got.minrne);
    c->tr_h.push_back(got.h);
    if (final_cycle(c)) c->finished = true;
    if (R_out) *R_out = r;
    if (min_rne) *min_rne = got.minrne;
    if (h_out) *h_out = got.h;
    return SPS_OK;
  }
  if (graph) {
    const auto g0 = std::chrono::steady_clock::now();
    TRY(build_mstep_graphs(c, adaptive));
    c->host_graph_us +=
        std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - g0).count();
    CU(c, cudaStreamWaitEvent(c->stream, c->ev_zready[step0 & 1u], 0));
  }
  auto launch_step = [&](uint32_t s) -> sps_status {
    return graph ? replay_mstep(c, s) : launch_mstep(c, s, adaptive);
  };
  TRY(launch_step(step0));
  int r = 1;
  Ctl got{};
  for (;;) {
    // keep one step queued behind the one being checked
    auto h0 = std::chrono::steady_clock::now();
    if (r < Rmax) TRY(launch_step(step0 + (uint32_t)r));
    auto h1 = std::chrono::steady_clock::now();
    CU(c, cudaEventSynchronize(c->evs[(step0 + (uint32_t)r - 1u) & 1u]));
    auto h2 = std::chrono::steady_clock::now();
    c->host_launch_us += std::chrono::duration<double, std::micro>(h1 - h0).count();
    c->host_wait_us += std::chrono::duration<double, std::micro>(h2 - h1).count();
    c->syncs += 1;
    if (c->trace) trace_accumulate(c);
    got = c->hslot[(step0 + (uint32_t)r - 1u) & 1u];
    c->pairs += (double)c->P * t1;
    if (got.err == ERR_NUMERIC)
      return fail(c, SPS_E_NUMERIC, "numerical failure in the M phase (non-finite loglik or Cholesky failure "
                                    "after ridge; cf. PAPER.md:1024-1030)");
    if (adaptive ? got.stop != 0 : r >= R_fixed) break;
    if (r >= Rmax) {
      CU(c, cudaStreamSynchronize(c->stream));
      return fail(c, SPS_E_MIXING, "M phase did not reach RNE >= K in %d steps", c->cfg.max_m_steps);
    }
    r += 1;
  }
  c->mstep = step0 + (uint32_t)r;
  if (c->tl) TRY(timeline_accumulate(c, r));
  *c->hctl = got;
  c->cphase_done = false;
  c->tr_R.push_back(r);
  c->tr_rne.push_back(got.minrne);
  c->tr_h.push_back(got.h);
  if (final_cycle(c)) c->finished = true;
  if (R_out) *R_out = r;
  if (min_rne) *min_rne = got.minrne;
  if (h_out) *h_out = got.h;
  return SPS_OK;
}

sps_status sps_logml(const sps_ctx* cc, double* logml, double* nse) {
  if (!cc) return SPS_E_CONFIG;
  // logically const: pulls the increments still pending on the device into the host total (a cache)
  sps_ctx* c = const_cast<sps_ctx*>(cc);
  CU(c, cudaSetDevice(c->cfg.device));
  TRY(sync_incs(c));
  if (logml) *logml = c->logml;
  if (nse) {
    TRY(gather(c, c->Lj, c->Lj_gath, (size_t)c->Jl));
    k_logml_nse<<<1, 32, 0, c->stream>>>(c->Lj_gath, c->J, c->scal + 1);
    CHECK_LAUNCH(c);
    CU(c, cudaMemcpyAsync(nse, c->scal + 1, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(c, cudaStreamSynchronize(c->stream));
  }
  return SPS_OK;
}

sps_status sps_moments(sps_ctx* c, int32_t m, const double* A, double* mean, double* sd, double* nse, double* rne) {
  if (!c || m < 0 || (m > 0 && !A)) return SPS_E_CONFIG;
  if (m == 0) return SPS_OK;
  CU(c, cudaSetDevice(c->cfg.device));
  if (m > c->fn_cap) {
    dfree(c, c->fn_A, c->stream);
    dfree(c, c->fn_out, c->stream);
    c->fn_A = c->fn_out = nullptr;
    TRY(DALLOC(c, &c->fn_A, (size_t)m * c->d));
    TRY(DALLOC(c, &c->fn_out, (size_t)m * 4));
    c->fn_cap = m;
  }
  CU(c, cudaMemcpyAsync(c->fn_A, A, sizeof(double) * m * c->d, cudaMemcpyHostToDevice, c->stream));
  TRY(accept_moments(c, false, 1, 1.0, 0u, nullptr));
  const size_t smem = sizeof(double) * (c->d + c->J);
  k_functional_stats<<<1, 256, smem, c->stream>>>(c->gath, c->G, c->slice_len, c->J, c->Jl, c->N, c->d, c->shift,
                                                  c->fn_A, m, c->fn_out);
  CHECK_LAUNCH(c);
  std::vector<double> h((size_t)m * 4);
  CU(c, cudaMemcpyAsync(h.data(), c->fn_out, sizeof(double) * m * 4, cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  for (int q = 0; q < m; ++q) {
    if (mean) mean[q] = h[q * 4 + 0];
    if (sd) sd[q] = h[q * 4 + 1];
    if (nse) nse[q] = h[q * 4 + 2];
    if (rne) rne[q] = h[q * 4 + 3];
  }
  return SPS_OK;
}

sps_status sps_run(sps_ctx* c, sps_report* rep) {
  if (!c || !rep) return SPS_E_CONFIG;
  NvtxRange nvtx_("sps_run");
  sps_status st = SPS_OK;
  const bool fixed = !c->des_R.empty();  // Algorithm 3 pass 2: the recorded design (sps_set_design)
  const bool power = c->cfg.tempering == SPS_POWER_TEMPERING;
  while (!c->finished) {
    const int l = c->ell;
    if (fixed && l >= (int)c->des_R.size()) break;
    st = sps_cphase(c, fixed && !power ? c->des_t[l] : -1, fixed && power ? c->des_phi[l] : -1.0, nullptr, nullptr,
                    nullptr);
    if (st != SPS_OK) break;
    st = sps_mphase(c, fixed ? c->des_R[l] : 0, nullptr, nullptr, nullptr);
    if (st != SPS_OK) break;
  }
  rep->status = st;
  rep->L = c->ell;
  rep->total_m_steps = 0;
  for (int r : c->tr_R) rep->total_m_steps += r;
  rep->h_final = c->hctl->h;
  rep->pairs = c->pairs;
  if (sync_incs(c) != SPS_OK && st == SPS_OK) st = SPS_E_CUDA;
  const int L = (int)c->tr_t.size();
  for (int l = 0; l < std::min(L, rep->cap_cycles); ++l) {
    if (rep->t_cycle) rep->t_cycle[l] = c->tr_t[l];
    if (rep->phi_cycle) rep->phi_cycle[l] = c->tr_phi[l];
    if (rep->logml_inc) rep->logml_inc[l] = c->tr_inc[l];
    if (l < (int)c->tr_R.size()) {
      if (rep->R_cycle) rep->R_cycle[l] = c->tr_R[l];
      if (rep->min_rne) rep->min_rne[l] = c->tr_rne[l];
      if (rep->h_cycle) rep->h_cycle[l] = c->tr_h[l];
    }
  }
  if (st != SPS_OK) return st;
  TRY(sps_logml(c, &rep->logml, &rep->logml_nse));
  if (rep->logpl && c->cfg.tempering == SPS_DATA_TEMPERING) TRY(sps_predictive(c, 0, c->t, rep->logpl));
  if (rep->n_report > 0) {
    std::vector<double> A;
    const double* fns = rep->report_fns;
    if (!fns) {  // theta_c' xbar, c = 1..C-1
      std::vector<double> xbar(c->k);
      CU(c, cudaMemcpyAsync(xbar.data(), c->xbar, sizeof(double) * c->k, cudaMemcpyDeviceToHost, c->stream));
      CU(c, cudaStreamSynchronize(c->stream));
      A.assign((size_t)rep->n_report * c->d, 0.0);
      for (int r = 0; r < std::min(rep->n_report, c->C - 1); ++r)
        for (int i = 0; i < c->k; ++i) A[(size_t)r * c->d + r * c->k + i] = xbar[i];
      fns = A.data();
    }
    TRY(sps_moments(c, rep->n_report, fns, rep->mean, rep->sd, rep->nse, rep->rne));
  }
  return SPS_OK;
}

sps_status sps_predictive(sps_ctx* c, int32_t s0, int32_t s1, double* out) {
  if (!c || s0 < 0 || s1 < s0 || (s1 > s0 && !out)) return SPS_E_CONFIG;
  if (c->cfg.tempering != SPS_DATA_TEMPERING)
    return fail(c, SPS_E_STATE, "sps_predictive: log predictive likelihoods need data tempering");
  if (s1 > c->t) return fail(c, SPS_E_STATE, "sps_predictive: observations [%d, %d) not absorbed yet (t = %d)", s0, s1, c->t);
  if (s1 == s0) return SPS_OK;
  CU(c, cudaSetDevice(c->cfg.device));
  CU(c, cudaMemcpyAsync(out, c->logpl + s0, sizeof(double) * (s1 - s0), cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  return SPS_OK;
}

sps_status sps_record_sigma(sps_ctx* c, int32_t on) {
  if (!c) return SPS_E_CONFIG;
  CU(c, cudaSetDevice(c->cfg.device));
  c->recording = on != 0;
  if (c->recording) TRY(reserve_sigma(c, (int64_t)c->mstep + 2));
  return SPS_OK;
}

sps_status sps_get_sigma(sps_ctx* c, int64_t first, int64_t count, double* out) {
  if (!c || first < 0 || count < 0 || (count > 0 && !out)) return SPS_E_CONFIG;
  if (count == 0) return SPS_OK;
  CU(c, cudaSetDevice(c->cfg.device));
  if (!c->recording || first + count > (int64_t)c->mstep || first + count > c->sig_rec_cap)
    return fail(c, SPS_E_STATE, "sps_get_sigma: steps [%lld, %lld) not recorded (recording %d, %u steps run)",
                (long long)first, (long long)(first + count), (int)c->recording, c->mstep);
  const int64_t dd = (int64_t)c->d * c->d;
  CU(c, cudaMemcpyAsync(out, c->sig_rec + first * dd, sizeof(double) * count * dd, cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  return SPS_OK;
}

sps_status sps_set_design(sps_ctx* c, int32_t L, const int32_t* t_cycle, const double* phi_cycle,
                          const int32_t* R_cycle, const double* sigma) {
  if (!c || L < 0) return SPS_E_CONFIG;
  CU(c, cudaSetDevice(c->cfg.device));
  CU(c, cudaStreamSynchronize(c->stream));
  dfree(c, c->sig_in, c->stream);
  c->sig_in = nullptr;
  c->sig_in_n = 0;
  c->des_t.clear();
  c->des_R.clear();
  c->des_phi.clear();
  if (L == 0) return SPS_OK;
  const bool power = c->cfg.tempering == SPS_POWER_TEMPERING;
  if (!R_cycle || !sigma || (power ? !phi_cycle : !t_cycle) || L > c->cfg.max_cycles)
    return fail(c, SPS_E_CONFIG, "sps_set_design: missing arrays or L > max_cycles");
  int64_t steps = 0;
  for (int l = 0; l < L; ++l) {
    if (R_cycle[l] < 1) return fail(c, SPS_E_CONFIG, "sps_set_design: R_%d < 1", l + 1);
    if (power ? !(phi_cycle[l] > (l ? phi_cycle[l - 1] : 0.0) && phi_cycle[l] <= 1.0)
              : !(t_cycle[l] > (l ? t_cycle[l - 1] : 0) && t_cycle[l] <= c->n))
      return fail(c, SPS_E_CONFIG, "sps_set_design: schedule not increasing at cycle %d", l + 1);
    steps += R_cycle[l];
  }
  const int64_t dd = (int64_t)c->d * c->d;
  TRY(DALLOC(c, &c->sig_in, (size_t)(steps * dd)));
  CU(c, cudaMemcpyAsync(c->sig_in, sigma, sizeof(double) * steps * dd, cudaMemcpyHostToDevice, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  c->sig_in_n = steps;
  c->des_R.assign(R_cycle, R_cycle + L);
  if (power)
    c->des_phi.assign(phi_cycle, phi_cycle + L);
  else
    c->des_t.assign(t_cycle, t_cycle + L);
  return SPS_OK;
}

sps_status sps_get_particles(sps_ctx* c, double* theta_host, double* L_host, double* lp_host) {
  if (!c) return SPS_E_CONFIG;
  CU(c, cudaSetDevice(c->cfg.device));
  if (theta_host)
    CU(c, cudaMemcpyAsync(theta_host, c->theta, sizeof(double) * c->Pl * c->d, cudaMemcpyDeviceToHost, c->stream));
  if (L_host) CU(c, cudaMemcpyAsync(L_host, c->L, sizeof(double) * c->Pl, cudaMemcpyDeviceToHost, c->stream));
  if (lp_host) CU(c, cudaMemcpyAsync(lp_host, c->lp, sizeof(double) * c->Pl, cudaMemcpyDeviceToHost, c->stream));
  CU(c, cudaStreamSynchronize(c->stream));
  return SPS_OK;
}

sps_status sps_g_prior(const double* X, int32_t n, int32_t k, int32_t C, double g, int32_t device, double* cov_out) {
  if (!X || !cov_out || n < 1 || k < 1 || C < 2 || k > 128) return SPS_E_CONFIG;
  if (cudaSetDevice(device) != cudaSuccess) return SPS_E_CUDA;
  const int d = k * (C - 1);
  double *dX = nullptr, *dXtX = nullptr, *dcov = nullptr;
  Ctl* dctl = nullptr;
  Ctl h{};
  sps_status st = SPS_OK;
  if (cudaMalloc(&dX, sizeof(double) * n * k) || cudaMalloc(&dXtX, sizeof(double) * k * k) ||
      cudaMalloc(&dcov, sizeof(double) * d * d) || cudaMalloc(&dctl, sizeof(Ctl)))
    st = SPS_E_CUDA;
  if (st == SPS_OK) {
    cudaMemcpy(dX, X, sizeof(double) * n * k, cudaMemcpyHostToDevice);
    cudaMemset(dctl, 0, sizeof(Ctl));
    k_xtx<<<(k * k + 127) / 128, 128>>>(dX, n, k, dXtX);
    const size_t smem = sizeof(double) * 2 * k * k;
    cudaFuncSetAttribute(k_g_prior, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024);
    k_g_prior<<<1, 128, smem>>>(dXtX, n, k, C, g, dcov, dctl);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) st = SPS_E_CUDA;
  }
  if (st == SPS_OK) {
    cudaMemcpy(&h, dctl, sizeof(Ctl), cudaMemcpyDeviceToHost);
    if (h.err) st = SPS_E_DATA;
    else cudaMemcpy(cov_out, dcov, sizeof(double) * d * d, cudaMemcpyDeviceToHost);
  }
  cudaFree(dX);
  cudaFree(dXtX);
  cudaFree(dcov);
  cudaFree(dctl);
  return st;
}

// ---------------------------------------------------------------- test exports
#define TCU(x)                                  \
  do {                                          \
    if ((x) != cudaSuccess) return SPS_E_CUDA;  \
  } while (0)

sps_status sps_test_philox(int32_t n, const uint32_t* ctr, const uint32_t* key, uint32_t* out) {
  if (n <= 0) return SPS_E_CONFIG;
  uint32_t *dc = nullptr, *dout = nullptr;
  TCU(cudaMalloc(&dc, 16 * n));
  TCU(cudaMalloc(&dout, 16 * n));
  TCU(cudaMemcpy(dc, ctr, 16 * n, cudaMemcpyHostToDevice));
  k_test_philox<<<(n + 127) / 128, 128>>>(n, dc, key[0], key[1], dout);
  TCU(cudaGetLastError());
  TCU(cudaMemcpy(out, dout, 16 * n, cudaMemcpyDeviceToHost));
  cudaFree(dc);
  cudaFree(dout);
  return SPS_OK;
}

sps_status sps_test_normals(uint64_t seed, uint32_t id, uint32_t step, uint32_t tag, uint32_t pass, int32_t count,
                            double* out) {
  if (count <= 0) return SPS_E_CONFIG;
  double* d = nullptr;
  TCU(cudaMalloc(&d, sizeof(double) * count));
  k_test_normals<<<(count / 2 + 128) / 128, 128>>>(seed, id, step, tag, pass, count, d);
  TCU(cudaGetLastError());
  TCU(cudaMemcpy(out, d, sizeof(double) * count, cudaMemcpyDeviceToHost));
  cudaFree(d);
  return SPS_OK;
}

sps_status sps_test_portable(int32_t which, int32_t n, const double* x, double* out) {
  if (n <= 0 || which < 0 || which > 2) return SPS_E_CONFIG;
  const int on = which == 2 ? 2 * n : n;
  double *dx = nullptr, *dout = nullptr;
  TCU(cudaMalloc(&dx, sizeof(double) * n));
  TCU(cudaMalloc(&dout, sizeof(double) * on));
  TCU(cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  k_test_portable<<<(n + 127) / 128, 128>>>(which, n, dx, dout);
  TCU(cudaGetLastError());
  TCU(cudaMemcpy(out, dout, sizeof(double) * on, cudaMemcpyDeviceToHost));
  cudaFree(dx);
  cudaFree(dout);
  return SPS_OK;
}

sps_status sps_test_resample_int(int32_t N, const uint64_t* q, int32_t scheme, const uint64_t* a, int32_t* anc) {
  if (N < 1 || N > 16384 || scheme < 0 || scheme > 2) return SPS_E_CONFIG;
  uint64_t *dq = nullptr, *da = nullptr;
  int32_t* danc = nullptr;
  TCU(cudaMalloc(&dq, 8 * N));
  TCU(cudaMalloc(&da, 8 * N));
  TCU(cudaMalloc(&danc, 4 * N));
  TCU(cudaMemcpy(dq, q, 8 * N, cudaMemcpyHostToDevice));
  TCU(cudaMemcpy(da, a, 8 * N, cudaMemcpyHostToDevice));
  const size_t smem = (size_t)N * 12;
  TCU(cudaFuncSetAttribute(k_test_resample_int, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
  k_test_resample_int<<<1, 1024, smem>>>(N, dq, scheme, da, danc);
  TCU(cudaGetLastError());
  TCU(cudaMemcpy(anc, danc, 4 * N, cudaMemcpyDeviceToHost));
  cudaFree(dq);
  cudaFree(da);
  cudaFree(danc);
  return SPS_OK;
}

sps_status sps_test_resample_group(int32_t N, const double* lw, int32_t scheme, uint64_t seed, uint32_t group,
                                   uint32_t cycle, uint32_t pass, int32_t* anc) {
  if (N < 1 || N > 16384 || scheme < 0 || scheme > 2) return SPS_E_CONFIG;
  double *dlw = nullptr, *dth = nullptr, *dth2 = nullptr, *dL = nullptr, *dL2 = nullptr, *dms = nullptr,
         *dLj = nullptr;
  int32_t* danc = nullptr;
  Ctl* dctl = nullptr;
  TCU(cudaMalloc(&dlw, 8 * N));
  TCU(cudaMalloc(&dth, 8 * N));
  TCU(cudaMalloc(&dth2, 8 * N));
  TCU(cudaMalloc(&dL, 8 * N));
  TCU(cudaMalloc(&dL2, 8 * N));
  TCU(cudaMalloc(&dms, 16));
  TCU(cudaMalloc(&dLj, 8));
  TCU(cudaMalloc(&danc, 4 * N));
  TCU(cudaMalloc(&dctl, sizeof(Ctl)));
  TCU(cudaMemset(dctl, 0, sizeof(Ctl)));
  TCU(cudaMemset(dLj, 0, 8));
  TCU(cudaMemset(dth, 0, 8 * N));
  TCU(cudaMemset(dL, 0, 8 * N));
  TCU(cudaMemcpy(dlw, lw, 8 * N, cudaMemcpyHostToDevice));
  const size_t smem = (size_t)N * 12;
  TCU(cudaFuncSetAttribute(k_resample, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem + 1024));
  // the kernel's group index is blockIdx.x + g0: launch one block with g0 = group
  k_resample<<<1, 1024, smem>>>(dlw, N, 1, scheme, seed, cycle, pass, (int)group, dth, dL, dL, dth2, dL2, dL2, dms,
                                dLj, danc, dctl);
  TCU(cudaGetLastError());
  TCU(cudaMemcpy(anc, danc, 4 * N, cudaMemcpyDeviceToHost));
  for (void* p : {(void*)dlw, (void*)dth, (void*)dth2, (void*)dL, (void*)dL2, (void*)dms, (void*)dLj, (void*)danc,
                  (void*)dctl})
    cudaFree(p);
  return SPS_OK;
}

sps_status sps_test_accept(int64_t P, const double* delta, uint64_t seed, uint32_t step, uint32_t pass,
                           uint8_t* flags) {
  if (P <= 0) return SPS_E_CONFIG;
  double* dd = nullptr;
  uint8_t* df = nullptr;
  TCU(cudaMalloc(&dd, 8 * P));
  TCU(cudaMalloc(&df, P));
  TCU(cudaMemcpy(dd, delta, 8 * P, cudaMemcpyHostToDevice));
  k_test_accept<<<(unsigned)((P + 255) / 256), 256>>>(P, dd, seed, step, pass, df);
  TCU(cudaGetLastError());
  TCU(cudaMemcpy(flags, df, P, cudaMemcpyDeviceToHost));
  cudaFree(dd);
  cudaFree(df);
  return SPS_OK;
}

}  // extern "C"
