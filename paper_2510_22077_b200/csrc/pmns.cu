// libpmns: B200-native gPLMM-preconditioned Newton-FGMRES (arXiv 2510.22077).
// Unity build of the kernels + host orchestration + the C ABI (include/pmns.h).
#include <cuda_runtime.h>
#include <cuda_profiler_api.h>
#include <nccl.h>   // types only: the functions are resolved at run time (nccl_api)
#include <dlfcn.h>
#include <functional>
#include <future>

#include <array>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <exception>
#include <thread>
#include <unordered_map>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/pmns.h"
#include "kernels.cuh"
#include "setup.hpp"

namespace pmns {
constexpr int kMaxK = 64;
// Optional fused gathers/scatters of the nested-dissection sweeps (nd.inc):
// staged x_q -= sum_{e in [uptr[p], uptr[p+1])} U[usrc[e]] with p = xoff + q
// (the descendants' boundary updates), and y written to Y[yidx[yoff + r]].
struct GemvFuse {
  const int64_t *uptr = nullptr, *usrc = nullptr;
  const double *U = nullptr;
  const int64_t *yidx = nullptr;
};
struct GemvTask {
  int64_t aoff;   // offset of the block in A
  int64_t xoff;   // offset of the block's input segment in X
  int64_t yoff;   // output offset of the block's row 0 in Y
  int32_t n;      // number of columns (= input length)
  int32_t ld;     // row stride (even)
  int32_t r0, r1; // row tile
};
// Pinned host staging, pooled process-wide in size-keyed free lists:
// cudaMallocHost / cudaFreeHost cost tens of ms per 100 MB (page pinning, and
// the free synchronises the device), which a fresh context would otherwise
// pay on its first build and on destroy.  Flushed by pmns_release_cache.
struct PinCache {
  std::mutex mu;
  std::unordered_map<void *, size_t> live;
  std::map<size_t, std::vector<void *>> freel;
};
static PinCache &g_pc() {
  static PinCache d;
  return d;
}
static void *hpin_alloc(size_t bytes) {
  PinCache &d = g_pc();
  size_t B = std::max<size_t>(4096, (bytes + 65535) / 65536 * 65536);
  {
    std::lock_guard<std::mutex> lk(d.mu);
    auto it = d.freel.find(B);
    if (it != d.freel.end() && !it->second.empty()) {
      void *p = it->second.back();
      it->second.pop_back();
      d.live[p] = B;
      return p;
    }
  }
  void *p = nullptr;
  if (cudaMallocHost(&p, B) != cudaSuccess) {
    cudaGetLastError();
    throw std::runtime_error("ENOMEM: cudaMallocHost of " + std::to_string(B) + " bytes");
  }
  std::lock_guard<std::mutex> lk(d.mu);
  d.live[p] = B;
  return p;
}
static void hpin_free(void *p) {
  if (!p) return;
  PinCache &d = g_pc();
  std::lock_guard<std::mutex> lk(d.mu);
  auto it = d.live.find(p);
  if (it == d.live.end()) {
    cudaFreeHost(p);
    return;
  }
  d.freel[it->second].push_back(p);
  d.live.erase(it);
}
static void hpin_flush() {
  PinCache &d = g_pc();
  std::lock_guard<std::mutex> lk(d.mu);
  for (auto &kv : d.freel)
    for (void *p : kv.second) cudaFreeHost(p);
  d.freel.clear();
}

// Host copy of a probed ELL operator in pinned memory (fast D2H; reused
// across builds, buffers from the pinned pool).
struct HostEll {
  int width = 0;
  int32_t *col = nullptr, *cnt = nullptr;
  double *val = nullptr;
  size_t rows = 0;
  HostEll() = default;
  HostEll(const HostEll &) = delete;
  HostEll &operator=(const HostEll &) = delete;
  ~HostEll() {
    hpin_free(col);
    hpin_free(cnt);
    hpin_free(val);
  }
};

struct ProbeGeom {
  int64_t N;
  const uint32_t *rowpos;
  int nx, ny, nz, pyflag, pzflag;
  int px, py, pz;
  int reach;                 // stencil reach of the probed operator (2; 1 at the zero state)
  int fx[3], fy[3], fz[3];
  const int32_t *fmap[3];
  const int32_t *cmap;
};
}  // namespace pmns

#include "linalg_kernels.cu"
#include "mac_kernels.cu"

struct pmns_ctx;

namespace pmns {

static thread_local std::string g_err;

// host phase timers (PMNS_TRACE=1 prints them after each build)
struct Trace {
  std::map<std::string, double> t;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  std::mutex mu;
  void lap(const std::string &k) {
    std::lock_guard<std::mutex> lk(mu);
    auto now = std::chrono::steady_clock::now();
    t[k] += std::chrono::duration<double>(now - t0).count();
    t0 = now;
  }
};
static Trace *g_trace = nullptr;
static bool g_verbose = getenv("PMNS_VERBOSE") != nullptr;
static inline void TLAP(const char *k) {
  if (g_trace) g_trace->lap(k);
}
static int env_int(const char *name, int dflt);

// NCCL is resolved at run time from the process's libnccl.so.2 (normally the
// one PyTorch already loaded), so linking the library never pins a second,
// different NCCL into the process.
struct NcclApi {
  ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*allReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  // point-to-point (halo exchanges of the multi-GPU Krylov phase; optional)
  ncclResult_t (*groupStart)() = nullptr;
  ncclResult_t (*groupEnd)() = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
};
static const NcclApi &nccl_api() {
  static NcclApi api = []() {
    NcclApi a;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.getUniqueId = (decltype(a.getUniqueId))dlsym(h, "ncclGetUniqueId");
    a.commInitRank = (decltype(a.commInitRank))dlsym(h, "ncclCommInitRank");
    a.allReduce = (decltype(a.allReduce))dlsym(h, "ncclAllReduce");
    a.commDestroy = (decltype(a.commDestroy))dlsym(h, "ncclCommDestroy");
    a.groupStart = (decltype(a.groupStart))dlsym(h, "ncclGroupStart");
    a.groupEnd = (decltype(a.groupEnd))dlsym(h, "ncclGroupEnd");
    a.send = (decltype(a.send))dlsym(h, "ncclSend");
    a.recv = (decltype(a.recv))dlsym(h, "ncclRecv");
    return a;
  }();
  if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy)
    throw std::runtime_error("ECUDA: libnccl.so.2 not available");
  return api;
}

#define CK(x)                                                                                  \
  do {                                                                                         \
    cudaError_t e_ = (x);                                                                      \
    if (e_ != cudaSuccess)                                                                     \
      throw std::runtime_error(std::string("ECUDA: ") + cudaGetErrorString(e_) + " at " #x); \
  } while (0)

// Caching device allocator: builds free and re-allocate the same block sizes
// every time (GBs of local operators); cudaMalloc/cudaFree would synchronise
// the device and stall the concurrent build threads.  Blocks are kept in free
// lists keyed by (device, size bucket) -- a block freed by a context on one
// device is only ever handed to an allocation on the same device -- and
// flushed on allocation failure.
constexpr size_t kWasteCap = (size_t)12 << 30;   // oversize hand-outs may hold at most 12 GiB beyond their requests
struct DevCache {
  std::mutex mu;
  int64_t misses = 0;    // cudaMalloc calls (cache misses) and their host time
  double miss_ms = 0.0;
  int64_t oversize_hits = 0;   // requests served by a larger cached block
  size_t waste = 0;            // bytes live blocks hold beyond their requests (oversize hand-outs)
  size_t live_bytes = 0, total = 0;   // bytes of live blocks (their buckets); device memory (first use)
  std::unordered_map<void *, size_t> wasted;   // per oversize live block
  std::unordered_map<void *, std::pair<int, size_t>> live;   // block -> (device, bucket)
  std::map<std::pair<int, size_t>, std::vector<void *>> freel;
};
static DevCache &g_dc() {
  static DevCache d;
  return d;
}
static size_t dbucket(size_t b) {
  b = std::max<size_t>(b, 256);
  size_t p2 = 1;
  while (p2 < b) p2 <<= 1;
  size_t step = std::max<size_t>(4096, p2 >> 4);
  return (b + step - 1) / step * step;
}
static int cur_device() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    dev = 0;
  }
  return dev;
}
// frees every cached block (each on its own device)
static void dflush() {
  DevCache &d = g_dc();
  std::lock_guard<std::mutex> lk(d.mu);
  const int dev0 = cur_device();
  for (auto &kv : d.freel) {
    cudaSetDevice(kv.first.first);
    for (void *p : kv.second) cudaFree(p);
  }
  cudaSetDevice(dev0);
  d.freel.clear();
}
// bytes held in the free lists (reusable without cudaMalloc)
static size_t dcached_bytes() {
  DevCache &d = g_dc();
  std::lock_guard<std::mutex> lk(d.mu);
  size_t t = 0;
  for (auto &kv : d.freel) t += kv.first.second * kv.second.size();
  return t;
}
// (caller holds d.mu) may an oversize hand-out hold `extra` more bytes?  The
// total waste stays below `cap` and below a quarter of the memory that is not
// live: on a nearly full device (config 4h) the waste would be exactly what
// the next large request misses.
static bool waste_ok(DevCache &d, size_t extra, size_t cap) {
  if (d.waste + extra > cap) return false;
  if (d.total == 0) {
    size_t fr = 0, tot = 0;
    if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    d.total = tot;
  }
  const size_t head = d.total > d.live_bytes ? d.total - d.live_bytes : 0;
  return (d.waste + extra) * 4 <= head;
}
static void *dmalloc(size_t bytes) {
  DevCache &d = g_dc();
  const std::pair<int, size_t> key(cur_device(), dbucket(bytes));
  {
    std::lock_guard<std::mutex> lk(d.mu);
    auto it = d.freel.find(key);
    if (it != d.freel.end() && !it->second.empty()) {
      void *p = it->second.back();
      it->second.pop_back();
      d.live[p] = key;
      d.live_bytes += key.second;
      return p;
    }
    // no block of this bucket: take the smallest cached block up to 1.5x the
    // request (the level buffers of a factorisation differ from level to level;
    // a cudaMalloc / cudaFree pair of a multi-GB block costs tens of ms and
    // synchronises the device).  The block keeps its own bucket when freed.
    // The bytes such hand-outs hold beyond their requests are capped (kWasteCap):
    // they count against what a later large request can get.
    if (key.second >= (size_t)(1u << 20)) {
      const size_t cap = key.second + key.second / 2;
      for (auto jt = d.freel.upper_bound(key); jt != d.freel.end() && jt->first.first == key.first &&
                                               jt->first.second <= cap; ++jt)
        if (!jt->second.empty() && waste_ok(d, jt->first.second - key.second, kWasteCap)) {
          void *p = jt->second.back();
          jt->second.pop_back();
          d.live[p] = jt->first;
          d.live_bytes += jt->first.second;
          d.wasted[p] = jt->first.second - key.second;
          d.waste += jt->first.second - key.second;
          d.oversize_hits++;
          return p;
        }
    }
  }
  void *p = nullptr;
  const auto tm0 = std::chrono::steady_clock::now();
  if (cudaMalloc(&p, key.second) != cudaSuccess) {
    cudaGetLastError();
    // evict cached blocks of this device, largest first, only until the
    // request fits (flushing the whole cache would make every later request of
    // the build a miss: ~1k cudaMalloc/cudaFree pairs of GB blocks per build)
    bool ok = false;
    {
      // device memory is full of cached blocks: before freeing any, hand out
      // the smallest cached block that holds the request if it is at most 4x
      // too large (it returns to its own bucket when freed) -- a cudaFree +
      // cudaMalloc pair of GB blocks costs 20-100 ms and waits for the device
      std::lock_guard<std::mutex> lk(d.mu);
      const size_t cap = key.second * 4;
      for (auto jt = d.freel.lower_bound(key); jt != d.freel.end() && jt->first.first == key.first &&
                                               jt->first.second <= cap; ++jt)
        if (!jt->second.empty() && waste_ok(d, jt->first.second - key.second, kWasteCap / 2)) {
          void *q = jt->second.back();
          jt->second.pop_back();
          d.live[q] = jt->first;
          d.live_bytes += jt->first.second;
          d.wasted[q] = jt->first.second - key.second;
          d.waste += jt->first.second - key.second;
          d.oversize_hits++;
          return q;
        }
    }
    while (!ok) {
      void *victim = nullptr;
      {
        std::lock_guard<std::mutex> lk(d.mu);
        // best fit: the smallest cached block at least as large as the request,
        // else the largest cached block
        for (auto it = d.freel.lower_bound(key); it != d.freel.end() && it->first.first == key.first; ++it)
          if (!it->second.empty()) {
            victim = it->second.back();
            it->second.pop_back();
            break;
          }
        if (!victim)
          for (auto it = d.freel.rbegin(); it != d.freel.rend(); ++it)
            if (it->first.first == key.first && !it->second.empty()) {
              victim = it->second.back();
              it->second.pop_back();
              break;
            }
      }
      if (!victim) break;
      cudaFree(victim);
      ok = cudaMalloc(&p, key.second) == cudaSuccess;
      if (!ok) cudaGetLastError();
    }
    if (!ok) {
      dflush();
      if (cudaMalloc(&p, key.second) != cudaSuccess) {
        cudaGetLastError();
        throw std::runtime_error("ENOMEM: cudaMalloc of " + std::to_string(key.second) + " bytes");
      }
    }
  }
  std::lock_guard<std::mutex> lk(d.mu);
  d.live[p] = key;
  d.live_bytes += key.second;
  d.misses++;
  d.miss_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tm0).count();
  return p;
}
static void dfree(void *p) {
  if (!p) return;
  DevCache &d = g_dc();
  std::lock_guard<std::mutex> lk(d.mu);
  auto it = d.live.find(p);
  if (it == d.live.end()) {
    cudaFree(p);
    return;
  }
  d.live_bytes -= std::min(d.live_bytes, it->second.second);
  auto wt = d.wasted.find(p);
  if (wt != d.wasted.end()) {
    d.waste -= wt->second;
    d.wasted.erase(wt);
  }
  d.freel[it->second].push_back(p);
  d.live.erase(it);
}

template <class T>
static T *dalloc(size_t n) {
  if (n == 0) n = 1;
  return (T *)dmalloc(n * sizeof(T));
}
static int64_t *g_h2d_counter = nullptr;
template <class T>
static T *dupload(const std::vector<T> &v, cudaStream_t s) {
  T *p = dalloc<T>(v.size());
  if (g_h2d_counter) *g_h2d_counter += (int64_t)(v.size() * sizeof(T));
  if (!v.empty()) CK(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return p;
}

static inline unsigned nblk(int64_t n, int bs = 256) { return (unsigned)std::max<int64_t>(1, (n + bs - 1) / bs); }

struct Ell {
  int width = 40;
  int32_t *col = nullptr;
  double *val = nullptr;
  int32_t *cnt = nullptr;
};

struct GemvSet {
  std::vector<GemvTask> tasks;
  GemvTask *d_tasks = nullptr;
  int maxn = 0;
  double *A = nullptr;
  int64_t bytes = 0;
};


// nested-dissection multifrontal local solver (nd.inc): numeric part of one
// build; the symbolic layout (NDLayout) is cached in the context
struct NDLayout;
struct NDSolver {
  const NDLayout *lay = nullptr;
  int64_t slot0 = 0, nslots = 0;
  double *St = nullptr;            // stored operator (F11^{-1}, F21, W12 of every front)
  int64_t st_elems = 0;
  const int64_t *d_piv = nullptr;  // level-ordered pivot slots, relative to slot0 (layout)
  const int64_t *d_bnd = nullptr;  // level-ordered boundary slots, relative to slot0 (layout)
  struct Level {
    GemvSet finv, w12;             // A pointers = St, tasks shared with the layout
    int64_t p0 = 0, p1 = 0;
    int64_t nupd = 0;
    const int64_t *d_uidx = nullptr, *d_uptr = nullptr, *d_usrc = nullptr;
  };
  std::vector<Level> lv;
  double *T = nullptr, *X = nullptr, *v = nullptr, *xp = nullptr;   // v = [v | u]
  int64_t bytes = 0;               // algorithmic bytes of one apply
  int pool_base = 0;
  cudaGraphExec_t gexec = nullptr;   // captured level sweeps (apply_nd)
  int64_t gnodes = 0;
  bool f21raw = false;               // F21 kept per level instead of L21 (multi-RHS-only solvers)
  std::vector<double *> f21lv;       // per level F21 buffers (dmalloc'd, owned)
};

struct Build {
  const double *d_xb = nullptr;   // the build state x_b (lives in allocs)
  bool ok = false;
  bool mg_only = false;   // built for the coarse-scale solver: no M_L
  // M_p (nested-dissection fronts of the primary blocks of J(x_b)) and the
  // folded Abar (build only: shape / correction vectors)
  NDSolver mpn, abarn;
  bool use_md_nd = false;            // M_d through nested dissection of each dual grid (PMNS_MD_ND)
  NDSolver mdn;
  // M_d
  GemvSet md;
  int64_t nd_total = 0;
  int64_t *d_dgather = nullptr;      // flattened dual slots
  int64_t *d_sc_ptr = nullptr, *d_sc_pos = nullptr;
  double *d_dbuf_in = nullptr, *d_dbuf_out = nullptr;
  // M_G
  int n_coarse = 0, n_kept = 0;
  std::vector<int> kept;             // kept primaries
  GemvSet coarse;                    // A°^{-1} (one block)
  int64_t *d_clo = nullptr, *d_chi = nullptr;   // restriction segments
  double *d_bc = nullptr, *d_xc = nullptr;
  double *d_B = nullptr;             // prolongation columns (per primary col-major)
  int64_t B_bytes = 0;
  int32_t *d_row_blk = nullptr;
  int64_t *d_blk_row0 = nullptr, *d_blk_boff = nullptr, *d_blk_coff = nullptr;
  int32_t *d_blk_ncol = nullptr, *d_cidx = nullptr, *d_cell_iface = nullptr;
  // f rows
  int64_t nfr = 0, f0 = 0;
  int64_t *d_frp = nullptr;
  int32_t *d_fci = nullptr;
  double *d_fcv = nullptr, *d_ft = nullptr;
  int32_t *d_fclus = nullptr, *d_floc = nullptr, *d_fmem = nullptr;
  int64_t *d_fcptr = nullptr, *d_fmoff = nullptr;
  double *d_fminv = nullptr;
  std::vector<void *> allocs;
};

struct DistPlan;   // multi-GPU Krylov phase (dist.inc)

}  // namespace pmns

struct pmns_ctx {
  int device = 0;
  pmns_problem prob;
  pmns::Geometry geo;
  pmns::Decomp dec;
  pmns::Layout lay;
  pmns::DevGeom G;
  int32_t *d_fmap[3] = {nullptr, nullptr, nullptr};
  int32_t *d_cmap = nullptr;
  uint32_t *d_rowpos = nullptr;
  uint8_t *d_mask = nullptr;
  int64_t *d_perm = nullptr;
  int32_t *d_slot_iface = nullptr;   // interface id of each interface-cell slot
  int32_t *d_tab = nullptr;          // per-row stencil codes
  int32_t *d_rec = nullptr;          // cell records of the Krylov-phase J apply (one allocation)
  int64_t n_rec_irregular = 0;       // record rows that fall back to the per-row table
  bool use_jrec = getenv("PMNS_JREC") != nullptr && atoi(getenv("PMNS_JREC")) != 0;   // records: opt-in (slower, see DESIGN)
  int coarse_colours = 0;            // probe passes of the last coarse assembly (0: unit columns)
  double t_setup_ms = 0;             // pmns_create host set-up time
  bool compose_build = getenv("PMNS_COMPOSE") == nullptr || atoi(getenv("PMNS_COMPOSE")) != 0;
  std::vector<int32_t> h_tab;        // host copy (structural pattern of the ND plan)
  pmns::NDLayout *ndl = nullptr;     // cached nested-dissection layout (first build)
  pmns::NDLayout *ndl_md = nullptr;  // same for the dual grids (virtual slot space = flattened duals)
  std::thread layout_th;              // structural ND layouts computed in the background from pmns_create
  std::exception_ptr layout_err;
  pmns::Build B;
  bool have_exec = false;
  // build-time stream pool: independent local factorisations run concurrently
  static constexpr int kPool = 16;   // two groups of kGroup streams (M_p and Abar build concurrently)
  static constexpr int kGroup = 8;
  cudaStream_t pst[kPool] = {};
  cudaStream_t bst[2] = {};          // main streams of the two concurrent build threads
  pmns::HostEll hJ, hW;             // pinned host copies of the probed operators (build only)
  std::vector<uint32_t> h_rowpos;   // host copies of the device-order position tables
  std::vector<int32_t> h_cmap_dev;
  // work vectors
  double *w[8] = {};
  double *d_part = nullptr, *d_scal = nullptr, *d_h = nullptr, *d_y = nullptr;
  int part_blocks = 0;
  // Krylov
  int m_alloc = 0;
  double *d_V = nullptr, *d_Z = nullptr;
  std::atomic<int64_t> launches{0};
  std::mutex mu;                     // build bookkeeping shared by build threads
  double t_mg = 0, t_ml = 0;
  std::map<std::string, std::pair<void *, size_t>> scratch;   // cached build scratch
  int64_t h2d_bytes = 0;
  // multi-GPU: primaries [own_lo, own_hi) are owned by this rank;
  // their M_p / Abar fronts are factorised and applied here, everything else
  // is replicated; the owned M_p output and shape vectors are combined by
  // ncclAllReduce over disjoint supports (exact: x + 0 = x, so every rank
  // holds bit-identical iterates and the Krylov loop needs no other exchange)
  int rank = 0, world = 1;
  int own_lo = 0, own_hi = 0;
  int dual_lo = 0, dual_hi = 0;      // owned dual grids (M_d) [dual_lo, dual_hi)
  std::vector<std::vector<int64_t>> owned_duals;   // copy of the owned range when world > 1
  ncclComm_t comm = nullptr;         // null: single GPU, or partition-only (tests)
  pmns::DistPlan *dist = nullptr;    // distributed Krylov phase (world > 1 with a transport)
  double *d_mpbuf = nullptr;         // owned M_p output over the primary range
  int64_t *d_dgather_c = nullptr, *d_sc_ptr_c = nullptr, *d_sc_pos_c = nullptr;   // cached dual tables
  int64_t nd_total_c = 0;
  std::vector<std::vector<int32_t>> Ci_cache;   // interfaces adjacent to each primary (C^{p_i})
  void *chk_pinned[2] = {nullptr, nullptr};   // pinned staging of the engine's check flags (per stream group)
  size_t chk_pinned_cap[2] = {0, 0};
  // live per-kernel timing (CUDA events on the launching stream), enabled by pmns_profile(ctx, 1)
  bool prof = false;
  struct EvPair { cudaEvent_t a, b; int kind; int64_t bytes; };
  std::vector<EvPair> evs;
  std::vector<cudaEvent_t> evpool;   // recycled timing events (profiling in the timed region)
};

namespace pmns {

// ----------------------------------------------------------------------------
// small helpers
// ----------------------------------------------------------------------------
static void free_build(Build &b) {
  cudaDeviceSynchronize();   // cached blocks are reused at once: no kernel may still read them
  for (NDSolver *nd : {&b.mpn, &b.abarn, &b.mdn})
    if (nd->gexec) cudaGraphExecDestroy(nd->gexec);
  for (void *p : b.allocs) dfree(p);
  b = Build();
}
static std::mutex g_build_mu;   // Build::allocs is appended from concurrent build threads
template <class T>
static T *balloc(Build &b, size_t n) {
  T *p = dalloc<T>(n);
  std::lock_guard<std::mutex> lk(g_build_mu);
  b.allocs.push_back(p);
  return p;
}
template <class T>
static T *bupload(Build &b, const std::vector<T> &v, cudaStream_t s) {
  T *p = dupload(v, s);
  std::lock_guard<std::mutex> lk(g_build_mu);
  b.allocs.push_back(p);
  return p;
}

static int prof_begin(pmns_ctx *c, int kind, int64_t bytes, cudaStream_t s);
static void *scratch_get(pmns_ctx *c, const char *name, int q, size_t bytes);
static void prof_end(pmns_ctx *c, int idx, cudaStream_t s);

static double dot(pmns_ctx *c, const double *a, const double *b, cudaStream_t s) {
  int nb = c->part_blocks;
  multidot_kernel<8><<<nb, 256, 0, s>>>(c->geo.N, 1, a, 0, b, c->d_part);
  reduce_parts_kernel<<<1, 256, 0, s>>>(nb, 1, c->d_part, c->d_scal, nullptr);
  c->launches += 2;
  double h;
  CK(cudaMemcpyAsync(&h, c->d_scal, sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return h;
}

static void apply_op(pmns_ctx *c, int mode, const double *state, const double *up, const double *v, double *y,
                     double alpha, const double *b, double beta, cudaStream_t s) {
  bool pr = c->prof && mode == MODE_JAC;
  // algorithmic bytes of the J apply (SURVEY §8(d) B_J): v and y (N each), state faces (n_f), b if fused
  int pidx = pr ? prof_begin(c, 2, 8 * (2 * c->geo.N + c->geo.n_f) + (b ? 8 * c->geo.N : 0), s) : -1;
  if (mode == MODE_JAC && c->G.n_rec > 0 && c->use_jrec)
    launch_apply_jrec(c->G, state, v, y, alpha, b, beta, s);
  else
    launch_apply(c->G, mode, state, up, v, y, alpha, b, beta, s);
  c->launches++;
  prof_end(c, pidx, s);
}

static int prof_begin(pmns_ctx *c, int kind, int64_t bytes, cudaStream_t s) {
  if (!c->prof) return -1;
  pmns_ctx::EvPair e;
  auto take = [&](cudaEvent_t &ev) {
    if (!c->evpool.empty()) {
      ev = c->evpool.back();
      c->evpool.pop_back();
    } else {
      CK(cudaEventCreate(&ev));
    }
  };
  take(e.a);
  take(e.b);
  e.kind = kind;
  e.bytes = bytes;
  CK(cudaEventRecord(e.a, s));
  c->evs.push_back(e);
  return (int)c->evs.size() - 1;
}
static void prof_end(pmns_ctx *c, int idx, cudaStream_t s) {
  if (!c->prof || idx < 0) return;
  CK(cudaEventRecord(c->evs[idx].b, s));
}

// Kernel launch, optionally as a programmatic dependent launch (PDL: the
// kernel's CTAs start while the stream's previous kernel drains and block in
// pdl_wait(); used for the chains of short level-sweep launches).
// PMNS_PDL=0 disables it.
static bool pdl_on() {
  const char *e = getenv("PMNS_PDL");
  return !(e && atoi(e) == 0);
}
template <typename... KArgs, typename... Args>
static void launch_k(bool pdl, void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  if (!pdl) {
    k<<<grid, block, smem, s>>>(args...);
    return;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k, ((KArgs)args)...));
}

static void gemv(pmns_ctx *c, const GemvSet &g, const double *X, double *Y, const double *E0, const double *E1,
                 int mode, cudaStream_t s, int kind = -1, const int64_t *xidx = nullptr, int variant = 0,
                 GemvFuse fz = GemvFuse()) {
  if (g.tasks.empty()) return;
  int pidx = -1;
  if (kind >= 0) {
    // algorithmic bytes: stored operator + x read + y write (+ two epilogue reads)
    int64_t rows = 0;
    for (auto &t : g.tasks) rows += t.r1 - t.r0;
    pidx = prof_begin(c, kind, g.bytes + 16 * rows + (mode >= 1 ? 16 * rows : 0), s);
  }
  int cap = 26000;
  int smem_n = std::min(g.maxn + 1, cap);
  size_t smem = (size_t)smem_n * sizeof(double);
  int dev_sms = 148;
  if (variant == 1) {
    // many-task sets of short rows (nested-dissection fronts): 4 rows per warp in flight
    // grid = the CTAs that are resident at once (registers bound it to ~3 per SM,
    // not shared memory): a grid beyond one wave leaves a ragged last wave
    // one CTA per tile: ~3 CTAs per SM are resident (registers), and the block
    // scheduler balances the waves better than a grid-stride loop over resident
    // CTAs (measured: M_p apply 65% vs 58% of HBM peak)
    int grid = (int)std::min<size_t>(g.tasks.size(), (size_t)1 << 30);
    launch_k(pdl_on(), gemv_rows_kernel<4>, dim3(grid), dim3(256), smem, s, (const GemvTask *)g.d_tasks,
             (int)g.tasks.size(), (const double *)g.A, X, Y, E0, mode, smem_n, xidx, fz);
  } else {
    int grid = std::min<int>((int)g.tasks.size(), dev_sms * (smem > 100 * 1024 ? 1 : 2));
    gemv_tasks_kernel<<<grid, 512, smem, s>>>(g.d_tasks, (int)g.tasks.size(), g.A, X, Y, E0, E1, mode, smem_n,
                                               xidx);
  }
  c->launches++;
  prof_end(c, pidx, s);
}

// rows x ncols block (row-major, stride ld); square blocks pass ncols = rows
static void make_tasks(GemvSet &g, int64_t aoff, int64_t xoff, int64_t yoff, int rows_total, int ld,
                       int ncols = -1, int max_rows = 1 << 30) {
  if (ncols < 0) ncols = rows_total;
  if (rows_total <= 0 || ncols <= 0) return;
  // tiles of ~2 MB but at least 64 rows (4 per warp), so restaging x in shared
  // memory (8n bytes per tile) stays a few % of the streamed operator bytes;
  // max_rows spreads a single small matrix over several CTAs (coarse solve)
  int64_t row_bytes = (int64_t)ld * 8;
  int rows = (int)std::min<int64_t>(rows_total, std::max<int64_t>(64, (2 << 20) / std::max<int64_t>(row_bytes, 1)));
  rows = std::max(1, std::min(rows, max_rows));
  for (int r = 0; r < rows_total; r += rows)
    g.tasks.push_back({aoff, xoff, yoff, ncols, ld, r, std::min(rows_total, r + rows)});
  g.maxn = std::max(g.maxn, ncols);
}


static void *scratch_get(pmns_ctx *c, const char *name, int q, size_t bytes) {
  std::lock_guard<std::mutex> lk(c->mu);
  std::string key = std::string(name) + "." + std::to_string(q);
  auto it = c->scratch.find(key);
  if (it != c->scratch.end() && it->second.second >= bytes) return it->second.first;
  if (it != c->scratch.end()) {
    dfree(it->second.first);
    c->scratch.erase(it);
  }
  void *p = dmalloc(std::max<size_t>(bytes, 8));
  c->scratch[key] = {p, std::max<size_t>(bytes, 8)};
  return p;
}

static void scratch_release(pmns_ctx *c) {
  std::lock_guard<std::mutex> lk(c->mu);
  for (auto &kv : c->scratch) dfree(kv.second.first);
  c->scratch.clear();
}

}  // namespace pmns
namespace pmns {
#include "host_util.inc"
#include "dgemm.inc"
#include "dense_inv.inc"
#include "nd.inc"
#include "dist.inc"

// ----------------------------------------------------------------------------
// create
// ----------------------------------------------------------------------------
// Cell records of the Krylov-phase J apply (DevGeom::rec_*, jrec_kernel).
// Built on the host from the same face/cell maps as the per-row table and
// checked against that table entry by entry: a row whose codes the record
// chase does not reproduce exactly is flagged to use the table, so the two
// paths give the same operator by construction.
static void build_records(pmns_ctx *c, cudaStream_t s) {
  const Geometry &g = c->geo;
  const Layout &L = c->lay;
  const int64_t N = g.N;
  const int dim = g.dim;
  const int32_t *T = c->h_tab.data();
  // records in device order of the pressure slot
  std::vector<int64_t> rec_of_vox(g.nvox(), -1);
  std::vector<int32_t> rp;
  rp.reserve(g.n_c);
  for (int64_t w = 0; w < N; ++w) {
    uint32_t pp = c->h_rowpos[w];
    if ((pp >> 30) != 3) continue;
    int k = (pp >> 20) & 1023, j = (pp >> 10) & 1023, i = pp & 1023;
    rec_of_vox[g.flat(k, j, i)] = (int64_t)rp.size();
    rp.push_back((int32_t)w);
  }
  const int64_t R = (int64_t)rp.size();
  std::vector<int32_t> rf(3 * R, -1), rn(6 * R, -1), xm;
  std::vector<uint32_t> rc(3 * R, 0u);
  auto face_slot = [&](int a, int k, int j, int i) -> int32_t {   // DOF slot or -1
    int32_t id = g.face_code(a, k, j, i);
    return id >= 0 ? (int32_t)L.inv[id] : -1;
  };
  for (int64_t r = 0; r < R; ++r) {
    uint32_t pp = c->h_rowpos[rp[r]];
    int k = (pp >> 20) & 1023, j = (pp >> 10) & 1023, i = pp & 1023;
    for (int a = 0; a < dim; ++a) rf[a * R + r] = face_slot(a, k, j, i);
    for (int b = 0; b < dim; ++b)
      for (int sd = 0; sd < 2; ++sd) {
        int kk = k, jj = j, ii = i;
        const int o = sd ? 1 : -1;
        if (b == 0) ii += o;
        else if (b == 1) jj += o;
        else kk += o;
        int32_t code = -1;
        if (b == 0 && ii < 0) {
          code = -3;
        } else if (b == 0 && ii >= g.nx) {
          code = -4 - (int32_t)xm.size();
          xm.push_back(face_slot(0, k, j, g.nx));
        } else {
          bool out = false;
          if (b == 1) {
            if (g.py) jj = (jj + g.ny) % g.ny;
            else out = jj < 0 || jj >= g.ny;
          } else if (b == 2) {
            if (g.pz) kk = (kk + g.nz) % g.nz;
            else out = kk < 0 || kk >= g.nz;
          }
          if (!out) {
            int64_t q = rec_of_vox[g.flat(kk, jj, ii)];
            code = q >= 0 ? (int32_t)q : -1;
          }
        }
        rn[(2 * b + sd) * R + r] = code;
      }
  }
  // the chase of jrec_kernel, on the host
  auto step = [&](int32_t X, int d) -> int32_t { return X >= 0 ? rn[(int64_t)d * R + X] : -1; };
  auto face_at = [&](int a, int32_t X) -> int32_t {
    if (X >= 0) return rf[(int64_t)a * R + X];
    if (X <= -4 && a == 0) return xm[-4 - X];
    return -1;
  };
  auto norm = [](int32_t code) { return code >= 0 ? code : -1; };   // fl codes: slot or -1
  int64_t irregular = 0;
  std::vector<int32_t> rows;   // rows left to the per-row table
  for (int64_t r = 0; r < R; ++r) {
    // mass row: low/high b-faces
    bool ok = true;
    for (int b = 0; b < dim; ++b) {
      int32_t t0 = T[(2 * b) * N + rp[r]], t1 = T[(2 * b + 1) * N + rp[r]];
      if (norm(t0) != rf[b * R + r] || norm(t1) != face_at(b, rn[(2 * b + 1) * R + r])) ok = false;
    }
    if (!ok) {
      rc[r] |= 1u << 30;
      ++irregular;
      rows.push_back(rp[r]);
    }
    for (int a = 0; a < dim; ++a) {
      const int32_t f = rf[a * R + r];
      if (f < 0) continue;
      uint32_t w = 0;
      bool okf = true;
      for (int b = 0; b < dim; ++b)
        for (int oi = 0; oi < 4; ++oi) {
          const int32_t code = T[(4 * b + oi) * N + f];
          if (code >= 0) {
            const int d = 2 * b + (oi >= 2);
            int32_t X = rn[(int64_t)d * R + r];
            if (oi == 0 || oi == 3) X = step(X, d);
            if (face_at(a, X) != code) okf = false;
          } else if (code >= -3) {
            w |= (uint32_t)(-code) << (2 * (4 * b + oi));
          } else {
            okf = false;
          }
        }
      const int32_t Lr = rn[(2 * a) * R + r];
      const int32_t c0 = Lr >= 0 ? rp[Lr] : Lr;
      if (T[20 * N + f] != c0 || T[21 * N + f] != rp[r]) okf = false;
      if (c->prob.rho != 0.0) {
        int bi = 0;
        for (int b = 0; b < dim; ++b) {
          if (b == a) continue;
          int32_t e[4] = {-1, -1, rf[b * R + r], face_at(b, rn[(2 * b + 1) * R + r])};
          if (Lr >= 0) {
            e[0] = rf[b * R + Lr];
            e[1] = face_at(b, step(Lr, 2 * b + 1));
          }
          for (int q = 0; q < 4; ++q)
            if (T[(12 + 4 * bi + q) * N + f] != e[q]) okf = false;
          ++bi;
        }
      }
      if (!okf) {
        w |= 1u << 31;
        ++irregular;
        rows.push_back(f);
      }
      rc[a * R + r] = w;
    }
  }
  c->n_rec_irregular = irregular;
  for (int32_t f : xm)
    if (f >= 0) rows.push_back(f);
  std::sort(rows.begin(), rows.end());
  // one allocation: rp | rf(3R) | rn(6R) | rc(3R) | xm | rows
  const int64_t nxm = std::max<int64_t>(1, (int64_t)xm.size());
  std::vector<int32_t> all((size_t)(13 * R + nxm + rows.size()), -1);
  std::copy(rp.begin(), rp.end(), all.begin());
  std::copy(rf.begin(), rf.end(), all.begin() + R);
  std::copy(rn.begin(), rn.end(), all.begin() + 4 * R);
  std::memcpy(all.data() + 10 * R, rc.data(), rc.size() * 4);
  std::copy(xm.begin(), xm.end(), all.begin() + 13 * R);
  std::copy(rows.begin(), rows.end(), all.begin() + 13 * R + nxm);
  c->d_rec = dupload(all, s);
  DevGeom &G = c->G;
  G.n_rec = R;
  G.rec_p = c->d_rec;
  G.rec_f = c->d_rec + R;
  G.rec_n = c->d_rec + 4 * R;
  G.rec_c = (const uint32_t *)(c->d_rec + 10 * R);
  G.xm_slot = c->d_rec + 13 * R;
  G.rec_rows = c->d_rec + 13 * R + nxm;
  G.n_rec_rows = (int64_t)rows.size();
  if (g_verbose)
    fprintf(stderr, "[pmns setup] %lld cell records, %lld x-max faces, %lld rows on the per-row table\n",
            (long long)R, (long long)xm.size(), (long long)irregular);
}

// per device slot: packed (type, k, j, i) of the row (host)
static void host_rowpos(pmns_ctx *c) {
  const Geometry &g = c->geo;
  const Layout &L = c->lay;
  std::vector<uint32_t> rp(g.N);
  for (int a = 0; a < g.dim; ++a)
    for (int k = 0; k < g.fz[a]; ++k)
      for (int j = 0; j < g.fy[a]; ++j)
        for (int i = 0; i < g.fx[a]; ++i) {
          int32_t id = g.fmap[a][((int64_t)k * g.fy[a] + j) * g.fx[a] + i];
          if (id >= 0) rp[L.inv[id]] = pack_pos(a, k, j, i);
        }
  for (int k = 0; k < g.nz; ++k)
    for (int j = 0; j < g.ny; ++j)
      for (int i = 0; i < g.nx; ++i) {
        int32_t id = g.cmap[g.flat(k, j, i)];
        if (id >= 0) rp[L.inv[id]] = pack_pos(3, k, j, i);
      }
  c->h_rowpos = std::move(rp);
}

static void setup_device(pmns_ctx *c, cudaStream_t s) {
  Geometry &g = c->geo;
  Layout &L = c->lay;
  // maps in device slots
  for (int a = 0; a < g.dim; ++a) {
    std::vector<int32_t> m(g.fmap[a].size());
    for (size_t q = 0; q < m.size(); ++q) {
      int32_t v = g.fmap[a][q];
      m[q] = v >= 0 ? (int32_t)L.inv[v] : v;
    }
    c->d_fmap[a] = dupload(m, s);
  }
  std::vector<int32_t> cm(g.cmap.size());
  for (size_t q = 0; q < cm.size(); ++q) cm[q] = g.cmap[q] >= 0 ? (int32_t)L.inv[g.cmap[q]] : -1;
  c->d_cmap = dupload(cm, s);
  // row positions
  host_rowpos(c);
  const std::vector<uint32_t> &rp = c->h_rowpos;
  c->d_rowpos = dupload(rp, s);
  c->h_cmap_dev = cm;
  std::vector<uint8_t> mk(g.N, 0);
  for (int64_t f = 0; f < g.n_f; ++f) mk[L.inv[f]] = L.face_mask[f];
  c->d_mask = dupload(mk, s);
  c->d_perm = dupload(L.perm, s);
  // interface id of each interface-cell slot
  int64_t ilo = L.seg[c->dec.n_p], ihi = L.seg[c->dec.n_p + c->dec.n_c];
  std::vector<int32_t> si(std::max<int64_t>(1, ihi - ilo));
  for (int j = 0; j < c->dec.n_c; ++j)
    for (int64_t w = L.seg[c->dec.n_p + j]; w < L.seg[c->dec.n_p + j + 1]; ++w) si[w - ilo] = j;
  c->d_slot_iface = dupload(si, s);
  DevGeom &G = c->G;
  G.dim = g.dim;
  G.nx = g.nx;
  G.ny = g.ny;
  G.nz = g.nz;
  G.py = g.py;
  G.pz = g.pz;
  for (int a = 0; a < 3; ++a) {
    G.fx[a] = g.fx[a];
    G.fy[a] = g.fy[a];
    G.fz[a] = g.fz[a];
    G.fmap[a] = c->d_fmap[a];
  }
  G.cmap = c->d_cmap;
  G.rowpos = c->d_rowpos;
  G.mask = c->d_mask;
  G.N = g.N;
  G.tab = nullptr;
  G.n_rec = 0;
  G.n_rec_rows = 0;
  const pmns_problem &P = c->prob;
  G.h = P.h;
  G.rho = P.rho;
  G.mu = P.mu;
  G.dt = P.dt;
  G.p_in = P.p_in;
  G.p_out = P.p_out;
  for (int a = 0; a < 3; ++a) G.bf[a] = P.body_force[a];
  c->d_tab = dalloc<int32_t>((size_t)kTab * g.N);
  launch_stencil(G, c->d_tab, s);
  G.tab = c->d_tab;
  c->h_tab.resize((size_t)kTab * g.N);
  CK(cudaMemcpyAsync(c->h_tab.data(), c->d_tab, c->h_tab.size() * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  build_records(c, s);
  if (g_verbose) {
    int64_t bad = 0, first = -1;
    for (int64_t r = 0; r < g.N; ++r) {
      if ((c->h_rowpos[r] >> 30) == 3) continue;
      if (c->h_tab[20 * g.N + r] < 0 && c->h_tab[21 * g.N + r] < 0) {
        if (first < 0) first = r;
        ++bad;
      }
    }
    fprintf(stderr, "[pmns setup] stencil table: %lld face rows without a void flank (first %lld)\n", (long long)bad,
            (long long)first);
  }
  for (auto &p : c->w) p = dalloc<double>(g.N);
  CK(cudaFuncSetAttribute(gemv_tasks_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 26000 * 8));
  CK(cudaFuncSetAttribute(gemv_rows_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 26000 * 8));
  CK(cudaFuncSetAttribute(gemv_rows_multi_kernel<4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(gemv_rows_multi_kernel<4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  CK(cudaFuncSetAttribute(gemv_rows_multi_kernel<4, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  // 8 CTAs per SM: about one row per thread at config 2, so every thread has
  // its loads of all the chunk's vectors in flight at once
  c->part_blocks = 8 * 148;
  c->d_part = dalloc<double>((size_t)c->part_blocks * kMaxK);
  c->d_scal = dalloc<double>(kMaxK);
  c->d_h = dalloc<double>(kMaxK * 2);
  c->d_y = dalloc<double>(kMaxK);
}

// ----------------------------------------------------------------------------
// build
// ----------------------------------------------------------------------------
// colour period along an axis for stencil reach R: >= 2R + 1 (offsets -R..R
// distinguishable), dividing n on periodic axes
static int period_for(int n, bool periodic, int reach = 2) {
  const int pmin = 2 * reach + 1;
  if (!periodic) return pmin;
  for (int p = pmin; p <= n; ++p)
    if (n % p == 0) return p;
  return n;  // n < pmin: every position its own color (and n | n)
}

// E2 != null: MODE_DUAL, one pass extracts J(state) into E and J~_w (w = state) into E2
static void probe_ell(pmns_ctx *c, int mode, const double *state, Ell &E, Build &b, cudaStream_t s,
                      Ell *E2 = nullptr, int reach = 2) {
  Geometry &g = c->geo;
  int64_t N = g.N;
  for (Ell *e : {&E, E2}) {
    if (!e) continue;
    e->col = balloc<int32_t>(b, (size_t)N * e->width);
    e->val = balloc<double>(b, (size_t)N * e->width);
    e->cnt = balloc<int32_t>(b, N);
    CK(cudaMemsetAsync(e->cnt, 0, N * sizeof(int32_t), s));
  }
  int *d_over = balloc<int>(b, 8);
  CK(cudaMemsetAsync(d_over, 0, 8 * sizeof(int), s));
  ProbeGeom P;
  P.N = N;
  P.rowpos = c->d_rowpos;
  P.nx = g.nx;
  P.ny = g.ny;
  P.nz = g.nz;
  P.pyflag = g.py;
  P.pzflag = g.pz;
  P.reach = reach;
  P.px = period_for(g.nx, false, reach);
  P.py = period_for(g.ny, g.py, reach);
  P.pz = g.dim == 3 ? period_for(g.nz, g.pz, reach) : 1;
  for (int a = 0; a < 3; ++a) {
    P.fx[a] = g.fx[a];
    P.fy[a] = g.fy[a];
    P.fz[a] = g.fz[a];
    P.fmap[a] = c->d_fmap[a];
  }
  P.cmap = c->d_cmap;
  // colors in batches of up to 64 (one apply launch with gridDim.y = batch)
  int ncolors = (g.dim + 1) * P.px * P.py * P.pz;
  const int kB = 64;
  double *pv = dalloc<double>((size_t)kB * N), *py = dalloc<double>((size_t)kB * N);
  double *py2 = E2 ? dalloc<double>((size_t)kB * N) : nullptr;
  for (int c0 = 0; c0 < ncolors; c0 += kB) {
    int nb_ = std::min(kB, ncolors - c0);
    dim3 grid(nblk(N), nb_);
    probe_fill_kernel<<<grid, 256, 0, s>>>(N, c->d_rowpos, c0, nb_, g.dim, P.px, P.py, P.pz, pv);
    if (E2) launch_apply_dual(c->G, state, pv, py, py2, s, nb_);
    else launch_apply(c->G, mode, state, nullptr, pv, py, 1.0, nullptr, 0.0, s, nb_);
    probe_extract_kernel<<<nblk(N), 256, 0, s>>>(P, c0, nb_, g.dim, py, E.col, E.val, E.cnt, E.width, d_over);
    if (E2)
      probe_extract_kernel<<<nblk(N), 256, 0, s>>>(P, c0, nb_, g.dim, py2, E2->col, E2->val, E2->cnt, E2->width,
                                                   d_over);
    c->launches += E2 ? 4 : 3;
  }
  CK(cudaStreamSynchronize(s));
  dfree(pv);
  dfree(py);
  if (py2) dfree(py2);
  int over[8] = {0};
  CK(cudaMemcpyAsync(over, d_over, sizeof(over), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (over[0]) {
    double v;
    memcpy(&v, over + 4, 8);
    throw std::runtime_error("EINVAL: operator probing failed (code " + std::to_string(over[0]) + ", mode " +
                             std::to_string(mode) + ", first stray entry: row " + std::to_string(over[2]) +
                             " colour " + std::to_string(over[3]) + " value " + std::to_string(v) + ")");
  }
}

// The matrix of Op (or J and J~_w at once, mode MODE_DUAL) as ELL, assembled
// directly from the stencil codes: each row's coefficients are the row
// evaluated on the unit vectors of its stencil columns (assemble_kernel), the
// same entries in the same order as colour probing with the periods of
// `reach` gives (probe_ell, kept as the PMNS_PROBE=1 path and as the test
// reference), at the cost of one pass instead of (dim+1)*px*py*pz applies.
static void jacobian_ell(pmns_ctx *c, int mode, const double *state, Ell &E, Build &b, cudaStream_t s,
                         Ell *E2 = nullptr, int reach = 2) {
  const char *pe = getenv("PMNS_PROBE");
  if (pe && atoi(pe) != 0) {
    probe_ell(c, mode, state, E, b, s, E2, reach);
    return;
  }
  Geometry &g = c->geo;
  int64_t N = g.N;
  for (Ell *e : {&E, E2}) {
    if (!e) continue;
    e->col = balloc<int32_t>(b, (size_t)N * e->width);
    e->val = balloc<double>(b, (size_t)N * e->width);
    e->cnt = balloc<int32_t>(b, N);
  }
  int *d_over = balloc<int>(b, 8);
  CK(cudaMemsetAsync(d_over, 0, 8 * sizeof(int), s));
  const int px = period_for(g.nx, false, reach), py = period_for(g.ny, g.py, reach),
            pz = g.dim == 3 ? period_for(g.nz, g.pz, reach) : 1;
  launch_assemble(c->G, mode, state, px, py, pz, E.col, E.val, E.cnt, E2 ? E2->col : nullptr,
                  E2 ? E2->val : nullptr, E2 ? E2->cnt : nullptr, E.width, d_over, s);
  c->launches++;
  int over[8] = {0};
  CK(cudaMemcpyAsync(over, d_over, sizeof(over), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (over[0]) throw std::runtime_error("EINVAL: Jacobian assembly: a row exceeds the ELL width");
}

// Batched dense-set inversion (M_d): chunk job / row descriptors and kernels.
struct MdJob {
  int64_t set_off;   // into the flattened slot list / positions
  int64_t out_off;   // stored inverse offset
  int32_t n, ld;
};
struct MdRow {
  int32_t b, q;      // matrix in the chunk, local row
};
// D_b[pos[q] * P + pos[l]] = A[set[q]][set[l]] for every row of every matrix of the chunk
__global__ void md_fill_kernel(int64_t nrows, const MdRow *__restrict__ rows, const MdJob *__restrict__ jobs,
                               const int64_t *__restrict__ all, const int32_t *__restrict__ pos,
                               const int32_t *__restrict__ ell_col, const double *__restrict__ ell_val,
                               const int32_t *__restrict__ ell_cnt, int width, double *__restrict__ D, int P) {
  int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const MdRow R = rows[t];
  const MdJob J = jobs[R.b];
  const int64_t *set = all + J.set_off;
  const int32_t *ps = pos + J.set_off;
  const int64_t r = set[R.q];
  double *Db = D + (int64_t)R.b * P * P + (int64_t)ps[R.q] * P;
  const int cnt = ell_cnt[r];
  for (int e = 0; e < cnt; ++e) {
    const int32_t col = ell_col[r * (int64_t)width + e];
    int lo = 0, hi = J.n;
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if (set[mid] < col) lo = mid + 1;
      else hi = mid;
    }
    if (lo < J.n && set[lo] == col) Db[ps[lo]] += ell_val[r * (int64_t)width + e];
  }
}
// identity on the padded tail of every matrix of the chunk
__global__ void md_pad_kernel(const MdJob *__restrict__ jobs, double *__restrict__ D, int P) {
  const MdJob J = jobs[blockIdx.y];
  int i = J.n + blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) D[(int64_t)blockIdx.y * P * P + (int64_t)i * P + i] = 1.0;
}
// stored inverse (row-major, ld) of every matrix of the chunk
__global__ void md_emit_kernel(const MdJob *__restrict__ jobs, const int32_t *__restrict__ pos,
                               const double *__restrict__ X, int P, double *__restrict__ out) {
  const MdJob J = jobs[blockIdx.y];
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)J.n * J.n) return;
  const int64_t a = e / J.n, c = e % J.n;
  const int32_t *ps = pos + J.set_off;
  out[J.out_off + a * J.ld + c] = X[(int64_t)blockIdx.y * P * P + (int64_t)ps[a] * P + ps[c]];
}

// Dense LU inverse of a set of blocks (row-major extraction -> cuSOLVER on
// the transpose -> row-major inverse, reading A20 "exact local solves").
static void build_inverse_set(pmns_ctx *c, Build &b, const Ell &E, const std::vector<std::vector<int64_t>> &sets,
                              GemvSet &out, int64_t xbase_mode, cudaStream_t s, const char *what, int pb = 0) {
  // xbase_mode 0: input/output offsets = block's first slot (contiguous primary segments)
  // xbase_mode 1: offsets into a flattened buffer (duals)
  int nb = (int)sets.size();
  std::vector<int64_t> off(nb + 1, 0), flat(nb + 1, 0);
  int64_t total = 0, maxn = 1;
  for (int q = 0; q < nb; ++q) {
    int64_t n = (int64_t)sets[q].size();
    int64_t ld = (n + 1) & ~1LL;
    off[q] = total;
    total += ld * n;
    flat[q + 1] = flat[q] + n;
    maxn = std::max(maxn, n);
  }
  off[nb] = total;
  out.A = balloc<double>(b, std::max<int64_t>(total, 1));
  // the even-stride pad column is read by the GEMV's paired loads (x pad = 0):
  // it must hold 0, not recycled bytes (0 * NaN = NaN)
  CK(cudaMemsetAsync(out.A, 0, (size_t)std::max<int64_t>(total, 1) * 8, s));
  out.bytes = total * 8;
  if (nb == 0) return;
  // all slot lists and faces-first positions at once (device), then the
  // batched inversion engine (dense_inv.inc) in chunks of equal padded size:
  // one fill, one engine recursion, one check and one emit launch per chunk,
  // enqueued round-robin on the stream pool from this thread, checks read once
  std::vector<int64_t> allslots;
  allslots.reserve(flat[nb]);
  for (auto &S : sets) allslots.insert(allslots.end(), S.begin(), S.end());
  std::vector<int32_t> pos(std::max<int64_t>(flat[nb], 1));
  for (int q = 0; q < nb; ++q) faces_first(c->h_rowpos.data(), sets[q].data(), (int64_t)sets[q].size(), pos.data() + flat[q]);
  int64_t *d_all = dupload(allslots, s);
  int32_t *d_pos = dupload(pos, s);
  cudaEvent_t ev0;
  CK(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
  CK(cudaEventRecord(ev0, s));
  const int NP = std::min(pmns_ctx::kGroup - (pb % pmns_ctx::kGroup), env_int("PMNS_POOL", 4));
  for (int q = 0; q < NP; ++q) CK(cudaStreamWaitEvent(c->pst[pb + q], ev0, 0));
  std::vector<int> ord(nb);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int bb) { return sets[a].size() > sets[bb].size(); });
  struct MdChunk {
    int P = 0;
    std::vector<int> jobs;
    double *orig = nullptr, *X = nullptr, *ws = nullptr, *y = nullptr;
    int *info = nullptr;
    unsigned long long *ev = nullptr;
    MdJob *d_jobs = nullptr;
    MdRow *d_rows = nullptr;
    int64_t nrows = 0, maxn = 0;
    int q = 0;
  };
  std::vector<MdChunk> ch;
  for (int j : ord) {
    int n = (int)sets[j].size();
    int P = (n + kNB - 1) / kNB * kNB;
    if (P == 0) continue;
    int64_t cap = std::min<int64_t>(256, std::max<int64_t>(1, (int64_t)(768ll << 20) / (16ll * P * P)));
    if (ch.empty() || ch.back().P != P || (int64_t)ch.back().jobs.size() >= cap) ch.push_back(MdChunk{});
    ch.back().P = P;
    ch.back().jobs.push_back(j);
  }
  int64_t nlaunch = 0;
  for (size_t ci = 0; ci < ch.size(); ++ci) {
    MdChunk &C = ch[ci];
    C.q = (int)(ci % NP);
    cudaStream_t st = c->pst[pb + C.q];
    const int P = C.P, bt = (int)C.jobs.size();
    const int64_t sP = (int64_t)P * P;
    std::vector<MdJob> hj(bt);
    std::vector<MdRow> hr;
    for (int b2 = 0; b2 < bt; ++b2) {
      int j = C.jobs[b2];
      int n = (int)sets[j].size();
      hj[b2] = MdJob{flat[j], off[j], n, (n + 1) & ~1};
      for (int q = 0; q < n; ++q) hr.push_back(MdRow{b2, q});
      C.maxn = std::max<int64_t>(C.maxn, n);
    }
    C.nrows = (int64_t)hr.size();
    C.d_jobs = dupload(hj, st);
    C.d_rows = dupload(hr, st);
    C.orig = (double *)dmalloc((size_t)bt * sP * 8);
    C.X = (double *)dmalloc((size_t)bt * sP * 8);
    C.ws = (double *)dmalloc((size_t)std::max<int64_t>(1, bt * inv_ws(P)) * 8);
    C.y = (double *)dmalloc((size_t)bt * P * 8);
    C.info = (int *)dmalloc((size_t)bt * 4);
    C.ev = (unsigned long long *)dmalloc((size_t)bt * 16);
    CK(cudaMemsetAsync(C.orig, 0, (size_t)bt * sP * 8, st));
    CK(cudaMemsetAsync(C.info, 0, (size_t)bt * 4, st));
    CK(cudaMemsetAsync(C.ev, 0, (size_t)bt * 16, st));
    md_fill_kernel<<<nblk(C.nrows, 128), 128, 0, st>>>(C.nrows, C.d_rows, C.d_jobs, d_all, d_pos, E.col, E.val,
                                                       E.cnt, E.width, C.orig, P);
    md_pad_kernel<<<dim3(nblk(P, 128), bt), 128, 0, st>>>(C.d_jobs, C.orig, P);
    CK(cudaMemcpyAsync(C.X, C.orig, (size_t)bt * sP * 8, cudaMemcpyDeviceToDevice, st));
    inv_rec(st, C.X, P, bt, 0, P, C.ws, C.info, nlaunch);
    dim3 g(nblk(P, 128), bt);
    chk_xv_kernel<<<g, 128, 0, st>>>(P, C.X, C.y);
    chk_res_kernel<<<g, 128, 0, st>>>(P, C.orig, C.y, C.ev, C.ev + bt);
    md_emit_kernel<<<dim3(nblk(C.maxn * C.maxn), bt), 256, 0, st>>>(C.d_jobs, d_pos, C.X, P, out.A);
    nlaunch += 6;
  }
  // deferred checks (one pinned staging buffer, one sync per stream)
  size_t need = 0;
  for (auto &C : ch) need += C.jobs.size() * 20;
  std::vector<char> flags(std::max<size_t>(need, 1));
  {
    size_t o = 0;
    for (auto &C : ch) {
      const int bt = (int)C.jobs.size();
      cudaStream_t st = c->pst[pb + C.q];
      CK(cudaMemcpyAsync(flags.data() + o, C.info, (size_t)bt * 4, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(flags.data() + o + (size_t)bt * 4, C.ev, (size_t)bt * 16, cudaMemcpyDeviceToHost, st));
      o += (size_t)bt * 20;
    }
    for (int q = 0; q < NP; ++q) CK(cudaStreamSynchronize(c->pst[pb + q]));
  }
  c->launches += nlaunch;
  {
    const double tol = inv_tol();
    size_t o = 0;
    for (auto &C : ch) {
      const int bt = (int)C.jobs.size(), P = C.P;
      const int64_t sP = (int64_t)P * P;
      const int *hinfo = (const int *)(flags.data() + o);
      const unsigned long long *hev = (const unsigned long long *)(flags.data() + o + (size_t)bt * 4);
      o += (size_t)bt * 20;
      for (int b2 = 0; b2 < bt; ++b2) {
        double e, sc;
        memcpy(&e, &hev[b2], 8);
        memcpy(&sc, &hev[bt + b2], 8);
        if (hinfo[b2] == 0 && e <= tol * std::max(sc, 1.0)) continue;
        // pivoted Gauss-Jordan fallback on this block, then re-emit it
        cudaStream_t st = c->pst[pb + C.q];
        const bool okp = pivoted_inverse_sync(st, C.orig + b2 * sP, C.X + b2 * sP, P);
        md_emit_kernel<<<dim3(nblk(C.maxn * C.maxn), 1), 256, 0, st>>>(C.d_jobs + b2, d_pos, C.X + b2 * sP, P,
                                                                      out.A);
        CK(cudaStreamSynchronize(st));
        if (g_verbose) fprintf(stderr, "[pmns inv] %s: block %d fallback to pivoted GJ\n", what, C.jobs[b2]);
        if (!okp) throw std::runtime_error(std::string("ESINGULAR: ") + what + " block " + std::to_string(C.jobs[b2]));
      }
    }
  }
  for (auto &C : ch)
    for (void *p : {(void *)C.orig, (void *)C.X, (void *)C.ws, (void *)C.y, (void *)C.info, (void *)C.ev,
                    (void *)C.d_jobs, (void *)C.d_rows})
      if (p) dfree(p);
  dfree(d_all);
  dfree(d_pos);
  cudaEventDestroy(ev0);
  // tiles sized for >= ~1000 CTAs per launch (the GEMV streams each tile once)
  const int64_t tile_bytes = std::max<int64_t>(128 << 10, out.bytes / 1024);
  for (int q = 0; q < nb; ++q) {
    int n = (int)sets[q].size();
    int64_t xo = xbase_mode == 0 ? sets[q][0] : flat[q];
    int ld = (n + 1) & ~1;
    make_tasks(out, off[q], xo, xo, n, ld, -1, (int)std::max<int64_t>(8, tile_bytes / (8 * (int64_t)ld)));
  }
  out.d_tasks = bupload(b, out.tasks, s);
}

static void host_dense_inverse(std::vector<double> &A, int n) {
  // Gauss-Jordan with partial pivoting (small f-face clusters, reading A14)
  std::vector<double> I(n * n, 0.0);
  for (int q = 0; q < n; ++q) I[q * n + q] = 1.0;
  for (int col = 0; col < n; ++col) {
    int piv = col;
    for (int r = col + 1; r < n; ++r)
      if (std::fabs(A[r * n + col]) > std::fabs(A[piv * n + col])) piv = r;
    if (A[piv * n + col] == 0.0) throw std::runtime_error("ESINGULAR: interface f-face block");
    if (piv != col)
      for (int q = 0; q < n; ++q) {
        std::swap(A[piv * n + q], A[col * n + q]);
        std::swap(I[piv * n + q], I[col * n + q]);
      }
    double d = 1.0 / A[col * n + col];
    for (int q = 0; q < n; ++q) {
      A[col * n + q] *= d;
      I[col * n + q] *= d;
    }
    for (int r = 0; r < n; ++r) {
      if (r == col) continue;
      double f = A[r * n + col];
      if (f == 0.0) continue;
      for (int q = 0; q < n; ++q) {
        A[r * n + q] -= f * A[col * n + q];
        I[r * n + q] -= f * I[col * n + q];
      }
    }
  }
  A.swap(I);
}

static void prolong(pmns_ctx *c, const double *xc, double *z, cudaStream_t s);
static void restrict_(pmns_ctx *c, const double *v, double *bc, int64_t stride, cudaStream_t s);

// Dense R^ Op P^ (row-major, stride ldc): prolong a batch of unit vectors,
// apply the operator at `state` to the whole batch, restrict every column.
// Structurally orthogonal colouring of the coarse columns (A° = R^ J~ P^,
// Remark 1): F(j) = the coarse rows column j can reach (the groups -- primary,
// interface cells, f-face cluster -- P^ e_j is supported on, each mapped through
// the J~ stencil and R^ to coarse rows); columns with disjoint F share a colour,
// so one prolong -> J~ -> restrict pass per colour yields all of them, each
// coarse row read back from the single column of the colour that reaches it.
// Other columns contribute exact zeros there, so the entries equal the
// unit-vector assembly bit for bit.  Cost: n_colours instead of n_coarse
// full-size passes (the O(n_coarse N) build term of round 1).
struct CoarseColours {
  int ncol = 0;
  std::vector<int32_t> colour;   // per coarse column
  std::vector<int32_t> owner;    // ncol x nc: column of colour q that owns coarse row k, or -1
};

static CoarseColours coarse_colouring(int64_t N, int64_t f0, int n_p, int n_c, const std::vector<int64_t> &seg,
                                      const std::vector<int> &kept_idx, const std::vector<std::vector<int32_t>> &Ci,
                                      const HostEll &HW, const std::vector<int64_t> &f_rp,
                                      const std::vector<int32_t> &f_ci, const std::vector<int32_t> &f_clus,
                                      int32_t f_ncl, int nc) {
  CoarseColours out;
  const int64_t ng = (int64_t)n_p + n_c + f_ncl;
  // group of a slot and coarse row of a slot
  std::vector<int32_t> grp(N), crow(N, -1);
  for (int i = 0; i < n_p; ++i)
    for (int64_t w = seg[i]; w < seg[i + 1]; ++w) {
      grp[w] = i;
      if (kept_idx[i] >= 0) crow[w] = n_c + kept_idx[i];
    }
  for (int j = 0; j < n_c; ++j)
    for (int64_t w = seg[n_p + j]; w < seg[n_p + j + 1]; ++w) {
      grp[w] = n_p + j;
      crow[w] = j;
    }
  for (int64_t w = f0; w < N; ++w) grp[w] = n_p + n_c + f_clus[w - f0];
  // NB[g]: coarse rows whose restricted J~ rows read a slot of group g
  std::vector<std::vector<int32_t>> NB(ng);
  for (int64_t r = 0; r < N; ++r) {
    const int32_t k = crow[r];
    if (k < 0) continue;
    for (int e = 0; e < HW.cnt[r]; ++e) {
      auto &v = NB[grp[HW.col[(size_t)r * HW.width + e]]];
      if (v.empty() || v.back() != k) v.push_back(k);
    }
  }
  for (auto &v : NB) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  // CL[g]: f-face clusters whose rows read a slot of (primary / interface) group g
  std::vector<std::vector<int32_t>> CL((size_t)n_p + n_c);
  for (int64_t q = 0; q + 1 < (int64_t)f_rp.size(); ++q)
    for (int64_t e = f_rp[q]; e < f_rp[q + 1]; ++e) {
      auto &v = CL[grp[f_ci[e]]];
      if (v.empty() || v.back() != f_clus[q]) v.push_back(f_clus[q]);
    }
  for (auto &v : CL) {
    std::sort(v.begin(), v.end());
    v.erase(std::unique(v.begin(), v.end()), v.end());
  }
  // primaries of each interface column (j in C^{p_i})
  std::vector<std::vector<int32_t>> prim_of(n_c);
  for (int i = 0; i < n_p; ++i)
    for (int32_t j : Ci[i]) prim_of[j].push_back(i);
  std::vector<int32_t> kept_prim(nc - n_c, -1);
  for (int i = 0; i < n_p; ++i)
    if (kept_idx[i] >= 0) kept_prim[kept_idx[i]] = i;
  // greedy colouring over 64-colour words
  const int kW = 64;
  std::vector<std::vector<uint64_t>> used;   // per word: per coarse row
  out.colour.assign(nc, -1);
  std::vector<int32_t> F, S;
  for (int j = 0; j < nc; ++j) {
    S.clear();
    if (j < n_c) {
      S.push_back(n_p + j);
      for (int32_t i : prim_of[j]) S.push_back(i);
    } else {
      S.push_back(kept_prim[j - n_c]);
    }
    const size_t ns = S.size();
    for (size_t e = 0; e < ns; ++e)
      for (int32_t cl : CL[S[e]]) S.push_back(n_p + n_c + cl);
    F.clear();
    for (int32_t g : S) F.insert(F.end(), NB[g].begin(), NB[g].end());
    std::sort(F.begin(), F.end());
    F.erase(std::unique(F.begin(), F.end()), F.end());
    int q = -1;
    for (size_t wd = 0; q < 0; ++wd) {
      if (wd == used.size()) used.emplace_back(nc, 0ull);
      uint64_t m = 0;
      for (int32_t k : F) m |= used[wd][k];
      if (~m) {
        q = (int)(wd * kW) + __builtin_ctzll(~m);
        for (int32_t k : F) used[wd][k] |= 1ull << (q % kW);
      }
    }
    out.colour[j] = q;
    out.ncol = std::max(out.ncol, q + 1);
    if ((int64_t)out.owner.size() < (int64_t)(q + 1) * nc) out.owner.resize((size_t)(q + 1) * nc, -1);
    for (int32_t k : F) out.owner[(size_t)q * nc + k] = j;
  }
  return out;
}

static void assemble_coarse(pmns_ctx *c, int mode, const double *state, double *Ac, int ldc, cudaStream_t s,
                            const CoarseColours *cc = nullptr) {
  Build &b = c->B;
  const int nc = b.n_coarse;
  const int64_t N = c->geo.N;
  if (nc == 0) return;
  Layout &L = c->lay;
  int64_t np_rows = L.seg[c->dec.n_p], npc_rows = L.seg[c->dec.n_p + c->dec.n_c];
  const int npass = cc ? cc->ncol : nc;   // probe vectors: colours, or unit columns
  // batch: two N-vectors per column, <= ~2 GB of scratch
  int nb = (int)std::max<int64_t>(1, std::min<int64_t>(npass, (int64_t)(2ll << 30) / (16 * std::max<int64_t>(N, 1))));
  nb = std::min(nb, 65535);
  double *X = (double *)dmalloc((size_t)nb * nc * 8), *Z = (double *)dmalloc((size_t)nb * N * 8),
         *Yv = (double *)dmalloc((size_t)nb * N * 8), *Tf = (double *)dmalloc((size_t)nb * std::max<int64_t>(b.nfr, 1) * 8);
  double *Rq = nullptr;
  int32_t *d_col = nullptr, *d_own = nullptr;
  if (cc) {
    Rq = (double *)dmalloc((size_t)nb * nc * 8);
    d_col = dupload(cc->colour, s);
    d_own = dupload(cc->owner, s);
  }
  CK(cudaMemsetAsync(Ac, 0, (size_t)nc * ldc * sizeof(double), s));
  for (int k0 = 0; k0 < npass; k0 += nb) {
    const int kb = std::min(nb, npass - k0);
    if (cc) colour_cols_kernel<<<dim3(nblk(nc), kb), 256, 0, s>>>(nc, k0, d_col, X);
    else unit_cols_kernel<<<dim3(nblk(nc), kb), 256, 0, s>>>(nc, k0, X);
    CK(cudaMemsetAsync(Z, 0, (size_t)kb * N * 8, s));
    if (npc_rows > 0)
      prolong_kernel<<<dim3(nblk(npc_rows), kb), 256, 0, s>>>(np_rows, npc_rows, b.d_row_blk, b.d_blk_row0,
                                                             b.d_blk_boff, b.d_blk_ncol, b.d_blk_coff, b.d_cidx, b.d_B,
                                                             b.d_cell_iface, X, Z, nc, N);
    if (b.nfr > 0) {
      frows_t_kernel<<<dim3(nblk(b.nfr), kb), 256, 0, s>>>(b.nfr, b.f0, b.d_frp, b.d_fci, b.d_fcv, Z, Tf, N);
      frows_solve_kernel<<<dim3(nblk(b.nfr * 32), kb), 256, 0, s>>>(b.nfr, b.f0, b.d_fclus, b.d_floc, b.d_fcptr,
                                                               b.d_fmem, b.d_fmoff, b.d_fminv, Tf, Z, N);
    }
    launch_apply(c->G, mode, state, nullptr, Z, Yv, 1.0, nullptr, 0.0, s, kb);
    if (cc) {
      segsum_kernel<<<dim3(nc, kb), 256, 0, s>>>(b.d_clo, b.d_chi, Yv, Rq, nb, N);
      colour_scatter_kernel<<<dim3(nblk(nc), kb), 256, 0, s>>>(nc, k0, nb, d_own, Rq, Ac, ldc);
      c->launches++;
    } else {
      segsum_kernel<<<dim3(nc, kb), 256, 0, s>>>(b.d_clo, b.d_chi, Yv, Ac + k0, ldc, N);
    }
    c->launches += 6;
  }
  CK(cudaStreamSynchronize(s));
  dfree(X);
  dfree(Z);
  dfree(Yv);
  dfree(Tf);
  if (cc) {
    dfree(Rq);
    dfree(d_col);
    dfree(d_own);
  }
}

// M_d gather list and deterministic scatter CSR (layout-only: cached in the context)
static const std::vector<std::vector<int64_t>> &duals_of(const pmns_ctx *c) {
  return c->world > 1 ? c->owned_duals : c->lay.dual_unknowns;
}

static void dual_tables(pmns_ctx *c, Build &b, cudaStream_t s) {
  if (!c->d_dgather_c) {
    const int64_t N = c->geo.N;
    std::vector<int64_t> gat;
    for (auto &S : duals_of(c)) gat.insert(gat.end(), S.begin(), S.end());
    std::vector<int64_t> ptr(N + 1, 0);
    for (int64_t u : gat) ptr[u + 1]++;
    for (int64_t q = 0; q < N; ++q) ptr[q + 1] += ptr[q];
    std::vector<int64_t> pos(gat.size()), fill(ptr.begin(), ptr.end() - 1);
    for (int64_t q = 0; q < (int64_t)gat.size(); ++q) pos[fill[gat[q]]++] = q;   // ascending q = dual order
    c->nd_total_c = (int64_t)gat.size();
    if (gat.empty()) gat.push_back(0);
    if (pos.empty()) pos.push_back(0);
    c->d_dgather_c = dupload(gat, s);
    c->d_sc_ptr_c = dupload(ptr, s);
    c->d_sc_pos_c = dupload(pos, s);
  }
  b.nd_total = c->nd_total_c;
  b.d_dgather = c->d_dgather_c;
  b.d_sc_ptr = c->d_sc_ptr_c;
  b.d_sc_pos = c->d_sc_pos_c;
}

// Structural nested-dissection layouts (M_p over the owned primaries, M_d over
// the owned dual grids in a virtual slot space).  They depend only on the
// stencil pattern and the decomposition, so pmns_create starts them on a
// background thread; every user of c->ndl / c->ndl_md joins it first.
static pmns::NDLayout *make_md_layout(pmns_ctx *c, cudaStream_t sd) {
  const auto &D = duals_of(c);
  std::vector<std::pair<int64_t, int64_t>> vb;
  std::vector<int64_t> gmap;
  for (auto &S : D) {
    vb.push_back({(int64_t)gmap.size(), (int64_t)S.size()});
    gmap.insert(gmap.end(), S.begin(), S.end());
  }
  // leaf size PMNS_MD_LEAF (256: cheapest build; larger leaves keep more
  // duals as single dense fronts, faster apply but more build flops)
  return nd_layout(c, vb, sd, gmap.data(), env_int("PMNS_MD_LEAF", 256));
}
static void join_layouts(pmns_ctx *c) {
  if (c->layout_th.joinable()) c->layout_th.join();
  if (c->layout_err) {
    std::exception_ptr e = c->layout_err;
    c->layout_err = nullptr;
    std::rethrow_exception(e);
  }
}
static void start_layouts(pmns_ctx *c) {
  if (c->dec.n_p == 0) return;
  const char *em = getenv("PMNS_MD_ND"), *edual = getenv("PMNS_ND_DUAL");
  const bool md = !(em && atoi(em) == 0) && !(edual && atoi(edual) == 0);
  c->layout_th = std::thread([c, md]() {
    try {
      CK(cudaSetDevice(c->device));
      std::exception_ptr emd;
      std::thread tmd;
      if (md)
        tmd = std::thread([&]() {
          try {
            CK(cudaSetDevice(c->device));
            cudaStream_t sd = c->pst[pmns_ctx::kGroup + 4];
            pmns::NDLayout *L = make_md_layout(c, sd);
            CK(cudaStreamSynchronize(sd));
            c->ndl_md = L;
          } catch (...) {
            emd = std::current_exception();
          }
        });
      std::exception_ptr emp;
      try {
        std::vector<std::pair<int64_t, int64_t>> ob;
        for (int i = c->own_lo; i < c->own_hi; ++i) ob.push_back({c->lay.seg[i], c->lay.seg[i + 1] - c->lay.seg[i]});
        cudaStream_t s0 = c->bst[0];
        pmns::NDLayout *L = nd_layout(c, ob, s0);
        CK(cudaStreamSynchronize(s0));
        c->ndl = L;
      } catch (...) {
        emp = std::current_exception();
      }
      if (tmd.joinable()) tmd.join();
      if (emp) std::rethrow_exception(emp);
      if (emd) std::rethrow_exception(emd);
    } catch (...) {
      c->layout_err = std::current_exception();
    }
  });
}

static void dist_allgather(pmns_ctx *c, double *x, cudaStream_t s);
static void dist_coarse_rows(pmns_ctx *c, cudaStream_t s);

static void build(pmns_ctx *c, const double *xb_in, cudaStream_t s, bool mg_only = false, bool algebraic = false) {
  Trace tr;
  g_trace = getenv("PMNS_TRACE") ? &tr : nullptr;
  free_build(c->B);
  Build &b = c->B;
  Geometry &g = c->geo;
  Decomp &d = c->dec;
  Layout &L = c->lay;
  int64_t N = g.N;
  double tA = 0.0;   // wall time of the M_L build thread
  cudaEvent_t e0, e1, e2;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  double *xb = balloc<double>(b, N);
  if (xb_in) CK(cudaMemcpyAsync(xb, xb_in, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  else CK(cudaMemsetAsync(xb, 0, N * sizeof(double), s));
  if (c->dist && xb_in) dist_allgather(c, xb, s);   // multi-GPU: owned parts -> the full build state
  b.d_xb = xb;
  CK(cudaEventRecord(e0, s));
  // Order (nested-dissection path): the M_L factorisation (M_p + M_d, from
  // J(x_b)) starts as soon as J is probed, the M_G local factorisation
  // (folded Abar, from J~_w) as soon as J~_w is probed; the host prepares the
  // shape/correction right-hand sides meanwhile and hands them to the M_G
  // thread for its multi-RHS solves.  The two threads use disjoint stream
  // groups and data.
  std::vector<std::pair<int64_t, int64_t>> pblocks;
  for (int i = 0; i < d.n_p; ++i) pblocks.push_back({L.seg[i], L.seg[i + 1] - L.seg[i]});
  // owned primaries (all of them on one GPU): the local factorisations cover only these
  std::vector<std::pair<int64_t, int64_t>> oblocks(pblocks.begin() + c->own_lo, pblocks.begin() + c->own_hi);
  join_layouts(c);
  if (!c->ndl) c->ndl = nd_layout(c, oblocks, s);   // structural: once per context
  TLAP("start");
  const int mg_mode = algebraic ? MODE_JAC : MODE_JW;   // M_G's matrix: J~_w (gPLMM) or J(x_b) (aPLMM)
  Ell EJ, EW;
  HostEll &HJ = c->hJ, &HW = c->hW;
  Build tmpb;   // folded-solve structures: live only during the build
  // memory: run the two factorisations concurrently only if both fit with margin
  bool serial = getenv("PMNS_BUILD_SERIAL") != nullptr;
  {
    // both operators' stored fronts (F11^{-1}, L21 / F21, W12) plus, per
    // operator, the largest level's transient buffers (F12, U, assembled F21)
    double stored = 0.0;
    std::vector<double> lvl(c->ndl->plan.level.size(), 0.0);
    for (auto &F : c->ndl->plan.f) {
      double m = (double)F.piv.size(), bb = (double)F.bnd.size();
      stored += 8.0 * (m * m + 2.0 * m * bb);
      lvl[F.height] += 8.0 * (2.0 * m * bb + bb * bb);
    }
    const double est = 2.0 * (stored + (lvl.empty() ? 0.0 : *std::max_element(lvl.begin(), lvl.end())));
    size_t fr = 0, totm = 0;
    CK(cudaMemGetInfo(&fr, &totm));
    // beside the fronts: M_d (built concurrently), the engine's chunk buffers
    // (<= 768 MB x 2 per stream), both assembled ELL matrices and the coarse
    // level -- a flat 16 GB allowance (the paper-scale Gyroid at h_m = 0.75
    // estimated 148.8 GB of 189.5 GB free and then failed at a 11.8 GB block)
    const double md_est = c->ndl_md ? 8.0 * (double)c->ndl_md->st_elems : 0.0;
    serial = serial || est * 1.15 + md_est + 16e9 > (double)(fr + dcached_bytes());
    if (g_verbose)
      fprintf(stderr, "[pmns build] concurrent M_p || Abar needs ~%.1f GB, free %.1f GB (+%.1f cached): %s\n",
              est / 1e9, fr / 1e9, dcached_bytes() / 1e9, serial ? "serial" : "concurrent");
  }
  const bool early = !serial;   // concurrent early-start schedule
  std::vector<std::vector<int32_t>> Ci(d.n_p);
  std::vector<int64_t> blk_row0(d.n_p + 1), blk_boff(d.n_p), blk_coff(d.n_p + 1, 0);
  std::vector<int32_t> blk_ncol(d.n_p), cidx;
  std::vector<int64_t> own_boff;     // the owned primaries' shape-vector offsets / column counts
  std::vector<int32_t> own_ncol;
  std::promise<void> rhs_promise;
  std::shared_future<void> rhs_ready = rhs_promise.get_future().share();
  cudaEvent_t evJ, evW, evR;
  CK(cudaEventCreateWithFlags(&evJ, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&evW, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&evR, cudaEventDisableTiming));
  std::exception_ptr errA, errB;
  // ---- M_L thread body: M_p (principal blocks of J(x_b)) and M_d ----
  auto bodyA = [&]() {
    try {
      auto t0 = std::chrono::steady_clock::now();
      CK(cudaSetDevice(c->device));
      cudaStream_t s = c->bst[0];
      CK(cudaStreamWaitEvent(s, evJ, 0));
      double tmp_ = 0.0;
      {
        // M_d on its own stream group, concurrently with M_p
        std::exception_ptr errD;
        std::thread thD([&]() {
          try {
            CK(cudaSetDevice(c->device));
            build_inverse_set(c, b, EJ, duals_of(c), b.md, 1, c->pst[4], "M_d", 4);
          } catch (...) {
            errD = std::current_exception();
          }
        });
        try {
          nd_factor(c, b, *c->ndl, EJ, false, b.mpn, s, "M_p", 0);
        } catch (...) {
          thD.join();
          throw;
        }
        tmp_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        thD.join();
        if (errD) std::rethrow_exception(errD);
      }
      if (g_trace)
        fprintf(stderr, "[pmns timeline] M_L thread: M_p done %.3f s, M_d done %.3f s\n", tmp_,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      // dual gather / deterministic scatter tables
      dual_tables(c, b, s);
      b.d_dbuf_in = balloc<double>(b, b.nd_total);
      b.d_dbuf_out = balloc<double>(b, b.nd_total);
      CK(cudaStreamSynchronize(s));
      tA = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    } catch (...) {
      errA = std::current_exception();
    }
  };
  // ---- M_G thread body: folded Abar local solves (shape + correction vectors) ----
  auto bodyB = [&]() {
    try {
      auto tb0 = std::chrono::steady_clock::now();
      CK(cudaSetDevice(c->device));
      cudaStream_t s = c->bst[1];
      CK(cudaStreamWaitEvent(s, evW, 0));
      nd_factor(c, tmpb, *c->ndl, EW, true, b.abarn, s, "Abar", pmns_ctx::kGroup);
      double tf_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - tb0).count();
      rhs_ready.wait();
      CK(cudaStreamWaitEvent(s, evR, 0));
      solve_nd_multi(c, b.abarn, b.d_B, own_boff, own_ncol, s);
      if (g_trace)
        fprintf(stderr, "[pmns timeline] M_G thread: Abar factor done %.3f s, solves done %.3f s\n", tf_,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - tb0).count());
      for (int i = 0; i < d.n_p; ++i) {
        int64_t n = L.seg[i + 1] - L.seg[i];
        int ncs = (int)Ci[i].size();
        if (ncs > 0) {
          negate_kernel<<<nblk(n * ncs), 256, 0, s>>>(n * ncs, b.d_B + blk_boff[i]);   // B = -Abar^{-1} Abar^p_c
          c->launches++;
        }
      }
      CK(cudaStreamSynchronize(s));
    } catch (...) {
      errB = std::current_exception();
    }
  };
  // ---- dual body: M_p and Abar factorised in lockstep (one level schedule,
  // shared engine chunks), M_d concurrently, then the Abar multi-RHS solves ----
  auto bodyDual = [&]() {
    try {
      auto t0 = std::chrono::steady_clock::now();
      CK(cudaSetDevice(c->device));
      cudaStream_t s = c->bst[0];
      CK(cudaStreamWaitEvent(s, evW, 0));   // evW follows evJ on the probing stream
      std::exception_ptr errD;
      auto md_body = [&]() {
        try {
          CK(cudaSetDevice(c->device));
          auto td0 = std::chrono::steady_clock::now();
          if (b.use_md_nd) {
            cudaStream_t sd = c->pst[pmns_ctx::kGroup + 4];
            CK(cudaStreamWaitEvent(sd, evJ, 0));
            if (!c->ndl_md) c->ndl_md = make_md_layout(c, sd);
            nd_factor_multi(c, {NDOp{&b, &EJ, false, &b.mdn, true}}, *c->ndl_md, sd, "M_d", pmns_ctx::kGroup,
                            pmns_ctx::kGroup / 2);
          } else {
            build_inverse_set(c, b, EJ, duals_of(c), b.md, 1, c->pst[pmns_ctx::kGroup], "M_d", pmns_ctx::kGroup);
          }
          if (getenv("PMNS_GPUTIME"))
            fprintf(stderr, "[pmns gputime] M_d build %.1f ms\n",
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - td0).count());
        } catch (...) {
          errD = std::current_exception();
        }
      };
      // M_d concurrently with M_p + Abar only while the fronts are small: on big
      // problems its allocations miss the block cache while the GPU is busy,
      // and a cudaFree there waits for the whole device (config 3: a 0.5 s stall
      // per build against 0.28 s for the M_d factorisation run afterwards)
      const bool md_after = getenv("PMNS_MD_AFTER") ? atoi(getenv("PMNS_MD_AFTER")) != 0
                                                    : (c->ndl && (double)c->ndl->st_elems * 8.0 > 16e9);
      std::thread thD;
      struct JoinGuard {   // never destroy a joinable thread (an exception below would abort)
        std::thread &t;
        ~JoinGuard() {
          if (t.joinable()) t.join();
        }
      } jg{thD};
      if (!md_after) thD = std::thread(md_body);
      const bool fast_multi = !(getenv("PMNS_FAST_MULTI") && atoi(getenv("PMNS_FAST_MULTI")) == 0);
      nd_factor_multi(c, {NDOp{&b, &EJ, false, &b.mpn, true}, NDOp{&tmpb, &EW, true, &b.abarn, fast_multi}}, *c->ndl, s,
                      "M_p+Abar", 0, pmns_ctx::kGroup);
      if (md_after) thD = std::thread(md_body);
      double tf_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      rhs_ready.wait();
      double tr_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      CK(cudaStreamWaitEvent(s, evR, 0));
      if (!solve_nd_multi_fast(c, b.abarn, b.d_B, own_boff, own_ncol, s))
        solve_nd_multi(c, b.abarn, b.d_B, own_boff, own_ncol, s);
      CK(cudaStreamSynchronize(s));
      double ts_ = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (getenv("PMNS_GPUTIME"))
        fprintf(stderr, "[pmns gputime] dual thread: factor %.1f ms, rhs ready %.1f ms, solves done %.1f ms\n",
                1e3 * tf_, 1e3 * tr_, 1e3 * ts_);
      for (int i = 0; i < d.n_p; ++i) {
        int64_t n = L.seg[i + 1] - L.seg[i];
        int ncs = (int)Ci[i].size();
        if (ncs > 0) {
          negate_kernel<<<nblk(n * ncs), 256, 0, s>>>(n * ncs, b.d_B + blk_boff[i]);   // B = -Abar^{-1} Abar^p_c
          c->launches++;
        }
      }
      thD.join();
      if (errD) std::rethrow_exception(errD);
      if (g_trace)
        fprintf(stderr, "[pmns timeline] dual thread: factorisations done %.3f s, solves + M_d done %.3f s\n", tf_,
                std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count());
      dual_tables(c, b, s);
      b.d_dbuf_in = balloc<double>(b, b.nd_total);
      b.d_dbuf_out = balloc<double>(b, b.nd_total);
      CK(cudaStreamSynchronize(s));
      tA = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    } catch (...) {
      errA = std::current_exception();
    }
  };
  const bool dual = early && !mg_only && !(getenv("PMNS_ND_DUAL") && atoi(getenv("PMNS_ND_DUAL")) == 0);
  b.use_md_nd = dual && !(getenv("PMNS_MD_ND") && atoi(getenv("PMNS_MD_ND")) == 0);   // default on
  std::thread thA, thB;
  // J and J~_w from one probing pass when both are needed (PMNS_DUAL_PROBE=0: two passes)
  const bool dual_probe = !mg_only && mg_mode == MODE_JW &&
                          !(getenv("PMNS_DUAL_PROBE") && atoi(getenv("PMNS_DUAL_PROBE")) == 0);
  if (dual_probe) {
    // at the zero state (the first build of a solve) the convection terms vanish
    // identically, so J and J~_w couple only within +-1 per axis: 3-periodic colours
    const bool zero_state = xb_in == nullptr && !(getenv("PMNS_PROBE_REACH2") && atoi(getenv("PMNS_PROBE_REACH2")));
    if (zero_state) {
      try {
        jacobian_ell(c, MODE_DUAL, xb, EJ, b, s, &EW, 1);
      } catch (const std::runtime_error &e) {
        // a coupling beyond +-1 (cannot happen for the MAC operator at rest): full reach
        if (g_verbose) fprintf(stderr, "[pmns] reach-1 probing failed (%s); probing with reach 2\n", e.what());
        EJ = Ell();
        EW = Ell();
        jacobian_ell(c, MODE_DUAL, xb, EJ, b, s, &EW, 2);
      }
    } else {
      jacobian_ell(c, MODE_DUAL, xb, EJ, b, s, &EW, 2);
    }
    CK(cudaEventRecord(evJ, s));
    CK(cudaEventRecord(evW, s));
    TLAP("probe J+Jw");
    if (early && !dual) thA = std::thread(bodyA);
  } else {
    if (!mg_only) jacobian_ell(c, MODE_JAC, xb, EJ, b, s);   // M_G-only builds (coarse solver) skip M_L
    CK(cudaEventRecord(evJ, s));
    TLAP("probe J");
    if (early && !mg_only && !dual) thA = std::thread(bodyA);
    jacobian_ell(c, mg_mode, xb, EW, b, s);
    CK(cudaEventRecord(evW, s));
    TLAP("probe Jw");
  }
  if (dual) thA = std::thread(bodyDual);
  else if (early) thB = std::thread(bodyB);
  download_ell(EW, N, HW, s);
  TLAP("download J");
  // ---------------- M_G (B1) from J~_w, w = u(x_b) ----------------
  // b_B = -r_steady(0, 0) (reading A16)
  double *bB = balloc<double>(b, N);
  {
    double *zero = c->w[5];
    CK(cudaMemsetAsync(zero, 0, N * sizeof(double), s));
    DevGeom G2 = c->G;
    G2.dt = 0.0;
    launch_apply(G2, MODE_RES, zero, nullptr, zero, bB, -1.0, nullptr, 0.0, s);
    c->launches++;
  }
  std::vector<double> hbB(N);
  CK(cudaMemcpyAsync(hbB.data(), bB, N * sizeof(double), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  b.kept.clear();
  for (int i = 0; i < d.n_p; ++i) {
    bool nz = false;
    for (int64_t w = L.seg[i]; w < L.seg[i + 1] && !nz; ++w) nz = hbB[w] != 0.0;
    if (nz) b.kept.push_back(i);
  }
  b.n_kept = (int)b.kept.size();
  b.n_coarse = d.n_c + b.n_kept;
  std::vector<int> kept_idx(d.n_p, -1);
  for (int k = 0; k < b.n_kept; ++k) kept_idx[b.kept[k]] = k;
  // C^{p_i}: interfaces with a cell face-adjacent to a cell of p_i (layout-only: cached)
  if (!c->Ci_cache.empty() || d.n_p == 0) {
    Ci = c->Ci_cache;
  } else {
    int64_t nv = g.nvox();
    for (int64_t f = 0; f < nv; ++f) {
      if (d.iface[f] < 0) continue;
      int i0 = (int)(f % g.nx);
      int64_t t = f / g.nx;
      int j0 = (int)(t % g.ny), k0 = (int)(t / g.ny);
      for (int bb = 0; bb < g.dim; ++bb)
        for (int o = -1; o <= 1; o += 2) {
          int kk = k0 + (bb == 2 ? o : 0), jj = j0 + (bb == 1 ? o : 0), ii = i0 + (bb == 0 ? o : 0);
          if (ii < 0 || ii >= g.nx) continue;
          if (g.py) jj = (jj + g.ny) % g.ny;
          else if (jj < 0 || jj >= g.ny) continue;
          if (g.dim == 3) {
            if (g.pz) kk = (kk + g.nz) % g.nz;
            else if (kk < 0 || kk >= g.nz) continue;
          }
          int64_t q = g.flat(kk, jj, ii);
          if (d.label[q] >= 0) Ci[d.label[q]].push_back(d.iface[f]);
        }
    }
    for (auto &v : Ci) {
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
    }
    c->Ci_cache = Ci;
  }
  // folded blocks, shape + correction vectors
  int64_t Btot = 0;
  for (int i = 0; i < d.n_p; ++i) {
    blk_row0[i] = L.seg[i];
    int64_t n = L.seg[i + 1] - L.seg[i];
    int nc = (int)Ci[i].size() + (kept_idx[i] >= 0 ? 1 : 0);
    blk_ncol[i] = nc;
    blk_boff[i] = Btot;
    Btot += n * nc;
    blk_coff[i + 1] = blk_coff[i] + nc;
    for (int32_t j : Ci[i]) cidx.push_back(j);
    if (kept_idx[i] >= 0) cidx.push_back(d.n_c + kept_idx[i]);
  }
  blk_row0[d.n_p] = L.seg[d.n_p];
  b.d_B = balloc<double>(b, std::max<int64_t>(Btot, 1));
  b.B_bytes = Btot * 8;
  CK(cudaMemsetAsync(b.d_B, 0, std::max<int64_t>(Btot, 1) * sizeof(double), s));
  {
    // RHS columns on the host: Abar^p_c = A^p_c Q° (interface-cell columns summed per interface)
    int64_t ilo = L.seg[d.n_p], ihi = L.seg[d.n_p + d.n_c];
    std::vector<int32_t> slot_if(std::max<int64_t>(ihi - ilo, 1), 0);
    for (int j = 0; j < d.n_c; ++j)
      for (int64_t w = L.seg[d.n_p + j]; w < L.seg[d.n_p + j + 1]; ++w) slot_if[w - ilo] = j;
    std::vector<double> Bh(std::max<int64_t>(Btot, 1), 0.0);
    for (int i = 0; i < d.n_p; ++i) {
      int64_t n = L.seg[i + 1] - L.seg[i];
      std::unordered_map<int32_t, int> cpos;
      for (size_t q = 0; q < Ci[i].size(); ++q) cpos[Ci[i][q]] = (int)q;
      for (int64_t r = L.seg[i]; r < L.seg[i + 1]; ++r)
        for (int e = 0; e < HW.cnt[r]; ++e) {
          int64_t col = HW.col[(size_t)r * HW.width + e];
          if (col < ilo || col >= ihi) continue;
          auto it = cpos.find(slot_if[col - ilo]);
          if (it != cpos.end()) Bh[blk_boff[i] + (int64_t)it->second * n + (r - L.seg[i])] += HW.val[(size_t)r * HW.width + e];
        }
    }
    CK(cudaMemcpyAsync(b.d_B, Bh.data(), Bh.size() * 8, cudaMemcpyHostToDevice, s));
    for (int i = 0; i < d.n_p; ++i)
      if (kept_idx[i] >= 0) {
        int64_t n = L.seg[i + 1] - L.seg[i];
        copy_kernel<<<nblk(n), 256, 0, s>>>(n, bB + L.seg[i], b.d_B + blk_boff[i] + (int64_t)Ci[i].size() * n);
        c->launches++;
      }
    own_boff.assign(blk_boff.begin() + c->own_lo, blk_boff.begin() + c->own_hi);
    own_ncol.assign(blk_ncol.begin() + c->own_lo, blk_ncol.begin() + c->own_hi);
    CK(cudaEventRecord(evR, s));
    CK(cudaStreamSynchronize(s));   // Bh (pageable) copied before it goes out of scope
    rhs_promise.set_value();
    TLAP("rhs");
    TLAP("plans");
    if (!early) {
      // one-level path or memory-constrained: M_G local solves first, then M_L
      thB = std::thread(bodyB);
      thB.join();
      if (!mg_only) {
        if (serial) {
          free_build(tmpb);
          nd_release(b.abarn);
          scratch_release(c);
          bodyA();
        } else {
          thA = std::thread(bodyA);
          thA.join();
        }
      }
    } else {
      if (thB.joinable()) thB.join();
      if (thA.joinable()) thA.join();
    }
    if (c->dist) {
      // every rank decides together before the first collective of the build
      // (a rank whose local factorisation failed must not leave the others
      // waiting in the shape-vector allreduce)
      double flag = (errA || errB) ? 1.0 : 0.0;
      CK(cudaMemcpyAsync(c->d_scal, &flag, sizeof(double), cudaMemcpyHostToDevice, s));
      c->dist->tr->allreduce(c->d_scal, 1, s);
      CK(cudaMemcpyAsync(&flag, c->d_scal, sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      if (flag > 0.0 && !errA && !errB)
        throw std::runtime_error("ESINGULAR: a local factorisation failed on another rank");
    }
    if (errA) std::rethrow_exception(errA);
    if (errB) std::rethrow_exception(errB);
    if (c->world > 1 && Btot > 0) {
      // the other ranks' blocks still hold their right-hand sides: zero them
      int64_t lo = blk_boff[c->own_lo], hi = c->own_hi < d.n_p ? blk_boff[c->own_hi] : Btot;
      if (lo > 0) CK(cudaMemsetAsync(b.d_B, 0, (size_t)lo * 8, s));
      if (hi < Btot) CK(cudaMemsetAsync(b.d_B + hi, 0, (size_t)(Btot - hi) * 8, s));
    }
    if (c->dist && Btot > 0) {
      // shape / correction vectors of the other ranks' primaries (disjoint supports: exact sum)
      c->dist->tr->allreduce(b.d_B, (size_t)Btot, s);
      CK(cudaStreamSynchronize(s));
    } else if (c->comm && Btot > 0) {
      if (nccl_api().allReduce(b.d_B, b.d_B, (size_t)Btot, ncclDouble, ncclSum, c->comm, s) != ncclSuccess)
        throw std::runtime_error("ENCCL: ncclAllReduce (shape vectors)");
      CK(cudaStreamSynchronize(s));
    }
    free_build(tmpb);
    nd_release(b.abarn);
    cudaEventDestroy(evJ);
    cudaEventDestroy(evW);
    cudaEventDestroy(evR);
    TLAP("M_L || M_G local");
    c->t_ml += 1e3 * tA;
  }

  std::vector<int32_t> row_blk(std::max<int64_t>(L.seg[d.n_p], 1), 0);
  for (int i = 0; i < d.n_p; ++i)
    for (int64_t w = L.seg[i]; w < L.seg[i + 1]; ++w) row_blk[w] = i;
  b.d_row_blk = bupload(b, row_blk, s);
  b.d_blk_row0 = bupload(b, blk_row0, s);
  b.d_blk_boff = bupload(b, blk_boff, s);
  b.d_blk_coff = bupload(b, blk_coff, s);
  b.d_blk_ncol = bupload(b, blk_ncol, s);
  if (cidx.empty()) cidx.push_back(0);
  b.d_cidx = bupload(b, cidx, s);
  {
    int64_t ilo = L.seg[d.n_p], ihi = L.seg[d.n_p + d.n_c];
    std::vector<int32_t> ci(std::max<int64_t>(ihi - ilo, 1), 0);
    for (int j = 0; j < d.n_c; ++j)
      for (int64_t w = L.seg[d.n_p + j]; w < L.seg[d.n_p + j + 1]; ++w) ci[w - ilo] = j;
    b.d_cell_iface = bupload(b, ci, s);
  }
  // f rows (Eq. xf): A^f_{pc} (CSR) and clusters of A^f_f with dense inverses
  b.f0 = L.seg[d.n_p + d.n_c];
  b.nfr = N - b.f0;
  std::vector<int64_t> f_rp;     // f-row structure kept for the coarse colouring
  std::vector<int32_t> f_ci, f_clus;
  int32_t f_ncl = 0;
  if (b.nfr > 0) {
    int W = EW.width;
    std::vector<int32_t> hcol((size_t)b.nfr * W), hcnt(b.nfr);
    std::vector<double> hval((size_t)b.nfr * W);
    CK(cudaMemcpyAsync(hcol.data(), EW.col + b.f0 * W, hcol.size() * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hval.data(), EW.val + b.f0 * W, hval.size() * 8, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(hcnt.data(), EW.cnt + b.f0, hcnt.size() * 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    std::vector<int64_t> rp(b.nfr + 1, 0);
    std::vector<int32_t> ci;
    std::vector<double> cv;
    std::vector<int64_t> uf(b.nfr);
    std::iota(uf.begin(), uf.end(), 0);
    auto find = [&](int64_t x) {
      while (uf[x] != x) {
        uf[x] = uf[uf[x]];
        x = uf[x];
      }
      return x;
    };
    for (int64_t q = 0; q < b.nfr; ++q) {
      for (int e = 0; e < hcnt[q]; ++e) {
        int32_t col = hcol[q * W + e];
        if (col < b.f0) {
          ci.push_back(col);
          cv.push_back(hval[q * W + e]);
        } else {
          int64_t r1 = find(q), r2 = find(col - b.f0);
          if (r1 != r2) uf[std::max(r1, r2)] = std::min(r1, r2);
        }
      }
      rp[q + 1] = (int64_t)ci.size();
    }
    std::map<int64_t, int32_t> cl_id;
    std::vector<int32_t> clus(b.nfr), locq(b.nfr);
    std::vector<std::vector<int32_t>> members;
    for (int64_t q = 0; q < b.nfr; ++q) {
      int64_t r = find(q);
      auto it = cl_id.find(r);
      if (it == cl_id.end()) {
        it = cl_id.emplace(r, (int32_t)members.size()).first;
        members.emplace_back();
      }
      clus[q] = it->second;
      locq[q] = (int32_t)members[it->second].size();
      members[it->second].push_back((int32_t)q);
    }
    std::vector<int64_t> cptr(members.size() + 1, 0), moff(members.size() + 1, 0);
    std::vector<int32_t> mem;
    std::vector<double> minv;
    for (size_t cc = 0; cc < members.size(); ++cc) {
      const auto &M = members[cc];
      int n = (int)M.size();
      std::vector<double> A((size_t)n * n, 0.0);
      std::map<int32_t, int> lpos;
      for (int a = 0; a < n; ++a) lpos[M[a]] = a;
      for (int a = 0; a < n; ++a) {
        int64_t q = M[a];
        for (int e = 0; e < hcnt[q]; ++e) {
          int32_t col = hcol[q * W + e];
          if (col >= b.f0) A[(size_t)a * n + lpos.at(col - (int32_t)b.f0)] += hval[q * W + e];
        }
      }
      host_dense_inverse(A, n);
      moff[cc] = (int64_t)minv.size();
      minv.insert(minv.end(), A.begin(), A.end());
      mem.insert(mem.end(), M.begin(), M.end());
      cptr[cc + 1] = (int64_t)mem.size();
    }
    if (ci.empty()) {
      ci.push_back(0);
      cv.push_back(0.0);
    }
    f_rp = rp;
    f_ci = ci;
    f_clus = clus;
    f_ncl = (int32_t)members.size();
    b.d_frp = bupload(b, rp, s);
    b.d_fci = bupload(b, ci, s);
    b.d_fcv = bupload(b, cv, s);
    b.d_ft = balloc<double>(b, b.nfr);
    b.d_fclus = bupload(b, clus, s);
    b.d_floc = bupload(b, locq, s);
    b.d_fmem = bupload(b, mem, s);
    b.d_fcptr = bupload(b, cptr, s);
    b.d_fmoff = bupload(b, moff, s);
    b.d_fminv = bupload(b, minv, s);
  }
  TLAP("B, f-rows");
  // restriction segments: interface cell ranges, then kept primaries' ranges
  {
    std::vector<int64_t> lo, hi;
    for (int j = 0; j < d.n_c; ++j) {
      lo.push_back(L.seg[d.n_p + j]);
      hi.push_back(L.seg[d.n_p + j + 1]);
    }
    for (int i : b.kept) {
      lo.push_back(L.seg[i]);
      hi.push_back(L.seg[i + 1]);
    }
    if (lo.empty()) {
      lo.push_back(0);
      hi.push_back(0);
    }
    b.d_clo = bupload(b, lo, s);
    b.d_chi = bupload(b, hi, s);
  }
  // coarse matrix A° = R^ J~_w P^ (Remark 1), assembled row-major, column by column
  int nc = b.n_coarse;
  b.d_bc = balloc<double>(b, std::max(nc, 1));
  b.d_xc = balloc<double>(b, std::max(nc, 1));
  const bool partial = c->world > 1 && !c->comm && !c->dist;   // partition-only: owned local solvers, no M_G
  if (nc > 0 && !partial) {
    int ldc = (nc + 1) & ~1;
    double *Ac = balloc<double>(b, (size_t)nc * ldc);
    CK(cudaMemsetAsync(Ac, 0, (size_t)nc * ldc * sizeof(double), s));
    CoarseColours cc;
    if (env_int("PMNS_COARSE_PROBE", 1))
      cc = coarse_colouring(N, b.f0, d.n_p, d.n_c, L.seg, kept_idx, Ci, HW, f_rp, f_ci, f_clus, f_ncl, nc);
    assemble_coarse(c, mg_mode, xb, Ac, ldc, s, cc.ncol > 0 ? &cc : nullptr);
    c->coarse_colours = cc.ncol;
    // invert: Ac row-major == A°^T column-major -> inverse of that == A°^{-1} row-major
    // (blocked Gauss-Jordan with partial pivoting, dense_inv.inc)
    b.coarse.A = balloc<double>(b, (size_t)nc * ldc);
    CK(cudaMemcpyAsync(b.coarse.A, Ac, (size_t)nc * ldc * sizeof(double), cudaMemcpyDeviceToDevice, s));
    double *gw = balloc<double>(b, (size_t)kPW * nc);
    int *gi = balloc<int>(b, nc + 1);
    CK(cudaMemsetAsync(gi + nc, 0, sizeof(int), s));
    gj_pivot_inverse(s, b.coarse.A, nc, ldc, gw, gi, gi + nc);
    int info = 0;
    CK(cudaMemcpyAsync(&info, gi + nc, sizeof(int), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    c->launches += 3 * ((nc + kPW - 1) / kPW) + 1;
    if (info != 0) throw std::runtime_error("ESINGULAR: coarse matrix");
    b.coarse.bytes = (int64_t)nc * ldc * 8;
    make_tasks(b.coarse, 0, 0, 0, nc, ldc, -1, std::max(16, (nc + 147) / 148));
    b.coarse.d_tasks = bupload(b, b.coarse.tasks, s);
  }
  if (c->dist) dist_coarse_rows(c, s);
  CK(cudaEventRecord(e2, s));
  CK(cudaStreamSynchronize(s));
  TLAP("coarse");
  scratch_release(c);   // build scratch is large; give it back to the solve phase
  if (g_trace) {
    for (auto &kv : tr.t) fprintf(stderr, "[pmns build] %-14s %8.3f s\n", kv.first.c_str(), kv.second);
    {
      DevCache &dc = g_dc();
      std::lock_guard<std::mutex> lk(dc.mu);
      fprintf(stderr, "[pmns build] allocator: %lld cudaMalloc calls so far, %.1f ms; %lld oversize-block hits\n",
              (long long)dc.misses, dc.miss_ms, (long long)dc.oversize_hits);
    }
    fprintf(stderr, "[pmns build] M_p stored %lld bytes, %lld fronts\n", (long long)b.mpn.st_elems * 8,
            (long long)(c->ndl ? c->ndl->plan.f.size() : 0));
    g_trace = nullptr;
  }
  // t_ml: wall time of the M_L thread; t_mg: the rest of the build (M_G work not
  // hidden behind M_L: probes, RHS, coarse matrix, and any longer Abar thread)
  float tot = 0;
  CK(cudaEventElapsedTime(&tot, e0, e2));
  c->t_mg += std::max(0.0, (double)tot - 1e3 * tA);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaEventDestroy(e2);
  // the probed ELL lists are build-only: release them
  for (void *p : {(void *)EJ.col, (void *)EJ.val, (void *)EJ.cnt, (void *)EW.col, (void *)EW.val, (void *)EW.cnt}) {
    auto it = std::find(b.allocs.begin(), b.allocs.end(), p);
    if (it != b.allocs.end()) {
      dfree(p);
      b.allocs.erase(it);
    }
  }
  b.mg_only = mg_only;
  b.ok = true;
}

// ----------------------------------------------------------------------------
// apply
// ----------------------------------------------------------------------------
static void restrict_(pmns_ctx *c, const double *v, double *bc, int64_t stride, cudaStream_t s) {
  Build &b = c->B;
  if (b.n_coarse == 0) return;
  segsum_kernel<<<b.n_coarse, 256, 0, s>>>(b.d_clo, b.d_chi, v, bc, stride);
  c->launches++;
}

static void prolong(pmns_ctx *c, const double *xc, double *z, cudaStream_t s) {
  Build &b = c->B;
  Layout &L = c->lay;
  int64_t np_rows = L.seg[c->dec.n_p], npc_rows = L.seg[c->dec.n_p + c->dec.n_c];
  if (npc_rows > 0) {
    prolong_kernel<<<nblk(npc_rows), 256, 0, s>>>(np_rows, npc_rows, b.d_row_blk, b.d_blk_row0, b.d_blk_boff,
                                                  b.d_blk_ncol, b.d_blk_coff, b.d_cidx, b.d_B, b.d_cell_iface, xc, z);
    c->launches++;
  }
  if (b.nfr > 0) {
    frows_t_kernel<<<nblk(b.nfr), 256, 0, s>>>(b.nfr, b.f0, b.d_frp, b.d_fci, b.d_fcv, z, b.d_ft);
    frows_solve_kernel<<<nblk(b.nfr * 32), 256, 0, s>>>(b.nfr, b.f0, b.d_fclus, b.d_floc, b.d_fcptr, b.d_fmem, b.d_fmoff,
                                                   b.d_fminv, b.d_ft, z);
    c->launches += 2;
  }
}

static void apply_mg(pmns_ctx *c, const double *v, double *z, cudaStream_t s) {
  Build &b = c->B;
  if (b.n_coarse == 0 || !b.coarse.A) {   // (partition-only contexts build no coarse solver)
    CK(cudaMemsetAsync(z, 0, c->geo.N * sizeof(double), s));
    return;
  }
  restrict_(c, v, b.d_bc, 1, s);
  gemv(c, b.coarse, b.d_bc, b.d_xc, nullptr, nullptr, 0, s);
  prolong(c, b.d_xc, z, s);
}

// z = M^{-1} v (Eq. mono_struct) composed with J(xk) (reading A18 / DESIGN R9:
// FGMRES passes xk = x_b); uses w[0..3]
static void apply_m(pmns_ctx *c, const double *xk, const double *v, double *z, cudaStream_t s) {
  Build &b = c->B;
  int64_t N = c->geo.N;
  double *zG = c->w[0], *sv = c->w[1], *zd = c->w[2], *t = c->w[3];
  apply_mg(c, v, zG, s);                                                   // a3-a5
  apply_op(c, MODE_JAC, xk, nullptr, zG, sv, -1.0, v, 1.0, s);            // a6: s = v - J zG
  if (b.nd_total > 0) {                                                    // a7: z_d = M_d^{-1} s
    gather_kernel<<<nblk(b.nd_total), 256, 0, s>>>(b.nd_total, b.d_dgather, sv, b.d_dbuf_in);
    if (b.use_md_nd) apply_nd(c, b.mdn, b.d_dbuf_in, b.d_dbuf_out, nullptr, nullptr, s, 1);
    else gemv(c, b.md, b.d_dbuf_in, b.d_dbuf_out, nullptr, nullptr, 0, s, 1, nullptr, 1);
    scatter_sum_kernel<<<nblk(N), 256, 0, s>>>(N, b.d_sc_ptr, b.d_sc_pos, b.d_dbuf_out, zd);
    c->launches += 2;
  } else {
    CK(cudaMemsetAsync(zd, 0, N * sizeof(double), s));
  }
  if (c->comm)   // owned dual grids only on this rank: sum over ranks
    if (nccl_api().allReduce(zd, zd, (size_t)N, ncclDouble, ncclSum, c->comm, s) != ncclSuccess)
      throw std::runtime_error("ENCCL: ncclAllReduce (M_d)");
  apply_op(c, MODE_JAC, xk, nullptr, zd, t, -1.0, sv, 1.0, s);            // a8: t = s - J z_d
  int64_t np_rows = c->lay.seg[c->dec.n_p];
  if (c->world > 1 || c->comm) {
    // owned primaries only, combined over ranks (disjoint supports)
    if (!c->d_mpbuf) c->d_mpbuf = dalloc<double>(std::max<int64_t>(np_rows, 1));
    CK(cudaMemsetAsync(c->d_mpbuf, 0, std::max<int64_t>(np_rows, 1) * 8, s));
    apply_nd(c, b.mpn, t, c->d_mpbuf, nullptr, nullptr, s, 0);
    if (c->comm && np_rows > 0)
      if (nccl_api().allReduce(c->d_mpbuf, c->d_mpbuf, (size_t)np_rows, ncclDouble, ncclSum, c->comm, s) !=
          ncclSuccess)
        throw std::runtime_error("ENCCL: ncclAllReduce (M_p)");
    if (np_rows > 0) {
      add3_kernel<<<nblk(np_rows), 256, 0, s>>>(np_rows, zG, zd, c->d_mpbuf, z);
      c->launches++;
    }
  } else {
    apply_nd(c, b.mpn, t, z, zG, zd, s, 0);                                     // a9: z = zG + zd + M_p^{-1} t
  }
  if (N > np_rows) {
    axpby_kernel<<<nblk(N - np_rows), 256, 0, s>>>(N - np_rows, 1.0, zG + np_rows, 1.0, zd + np_rows, z + np_rows);
    c->launches++;
  }
}

// ----------------------------------------------------------------------------
// FGMRES (a10) and Newton (a11)
// ----------------------------------------------------------------------------
static void ensure_krylov(pmns_ctx *c, int m) {
  if (c->m_alloc >= m) return;
  if (c->d_V) dfree(c->d_V);
  if (c->d_Z) dfree(c->d_Z);
  c->d_V = dalloc<double>((size_t)(m + 1) * c->geo.N);
  c->d_Z = dalloc<double>((size_t)m * c->geo.N);
  c->m_alloc = m;
}

static void multidot(pmns_ctx *c, int K, const double *V, const double *w, double *out, double *accum,
                     cudaStream_t s) {
  int nb = c->part_blocks;
  int64_t N = c->geo.N;
  multidot_kernel<8><<<nb, 256, 0, s>>>(N, K, V, N, w, c->d_part);
  c->launches++;
  reduce_parts_kernel<<<K, 256, 0, s>>>(nb, K, c->d_part, out, accum);
  c->launches++;
}

// Solve J d = rhs (rhs device), d device (output).  Returns iterations.
static int fgmres(pmns_ctx *c, const double *xk, const double *rhs, double *d, double tol_abs, int m, int maxit,
                  bool &ok, cudaStream_t s) {
  int64_t N = c->geo.N;
  ensure_krylov(c, m);
  double *V = c->d_V, *Z = c->d_Z;
  double *r = c->w[4];
  CK(cudaMemsetAsync(d, 0, N * sizeof(double), s));
  CK(cudaMemcpyAsync(r, rhs, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
  double beta = std::sqrt(dot(c, r, r, s));
  int total = 0;
  std::vector<double> H((size_t)(m + 1) * m), cs(m), sn(m), gv(m + 1);
  // Hessenberg column staging in pinned memory (a pageable D2H would go
  // through a driver bounce buffer once per iteration)
  struct PinnedCol {
    double *p;
    explicit PinnedCol(size_t n) : p((double *)hpin_alloc(n * sizeof(double))) {}
    ~PinnedCol() { hpin_free(p); }
  } hcol_buf(m + 2);
  double *hcol = hcol_buf.p;
  ok = false;
  while (true) {
    if (beta <= tol_abs) {
      ok = true;
      return total;
    }
    if (total >= maxit) return total;
    std::fill(H.begin(), H.end(), 0.0);
    std::fill(gv.begin(), gv.end(), 0.0);
    gv[0] = beta;
    axpby_kernel<<<nblk(N), 256, 0, s>>>(N, 1.0 / beta, r, 0.0, nullptr, V);
    c->launches++;
    int jend = 0;
    for (int j = 0; j < m; ++j) {
      double *vj = V + (int64_t)j * N, *zj = Z + (int64_t)j * N, *w = V + (int64_t)(j + 1) * N;
      {
        int pm = prof_begin(c, 5, 0, s);   // whole M^{-1} (bench: SURVEY 8(d) B_M / this time)
        // composed with the build-time A_b = J(x_b) (reading A18 / DESIGN R9);
        // PMNS_COMPOSE=0: with the current J^k (the round-1 reading, ablation)
        apply_m(c, (c->compose_build && c->B.d_xb) ? c->B.d_xb : xk, vj, zj, s);
        prof_end(c, pm, s);
      }
      apply_op(c, MODE_JAC, xk, nullptr, zj, w, 1.0, nullptr, 0.0, s);
      // CGS2: h = V^T w; w -= V h; twice (reading A22)
      CK(cudaMemsetAsync(c->d_h, 0, (j + 2) * sizeof(double), s));
      for (int pass = 0; pass < 2; ++pass) {
        multidot(c, j + 1, V, w, c->d_y, c->d_h, s);
        update_kernel<<<8 * 148, 256, 0, s>>>(N, j + 1, V, N, c->d_y, -1.0, w);
        c->launches++;
      }
      multidot(c, 1, w, w, c->d_scal, nullptr, s);
      normalize_kernel<<<2 * 148, 256, 0, s>>>(N, c->d_scal, w, w, c->d_h + j + 1);
      c->launches++;
      CK(cudaMemcpyAsync(hcol, c->d_h, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int i = 0; i <= j + 1; ++i) H[(size_t)i * m + j] = hcol[i];
      for (int i = 0; i < j; ++i) {
        double a = H[(size_t)i * m + j], bb = H[(size_t)(i + 1) * m + j];
        H[(size_t)i * m + j] = cs[i] * a + sn[i] * bb;
        H[(size_t)(i + 1) * m + j] = -sn[i] * a + cs[i] * bb;
      }
      double a = H[(size_t)j * m + j], bb = H[(size_t)(j + 1) * m + j];
      double den = std::hypot(a, bb);
      cs[j] = a / den;
      sn[j] = bb / den;
      H[(size_t)j * m + j] = den;
      H[(size_t)(j + 1) * m + j] = 0.0;
      gv[j + 1] = -sn[j] * gv[j];
      gv[j] = cs[j] * gv[j];
      ++total;
      jend = j + 1;
      if (g_verbose && (total % 25 == 0))
        fprintf(stderr, "[pmns fgmres] it %d  |g|/tol %.3e  restart-beta %.3e\n", total, std::fabs(gv[j + 1]) / tol_abs,
                beta);
      if (std::fabs(gv[j + 1]) <= tol_abs || total >= maxit) break;
    }
    std::vector<double> y(jend);
    for (int i = jend - 1; i >= 0; --i) {
      double sacc = gv[i];
      for (int q = i + 1; q < jend; ++q) sacc -= H[(size_t)i * m + q] * y[q];
      y[i] = sacc / H[(size_t)i * m + i];
    }
    CK(cudaMemcpyAsync(c->d_y, y.data(), jend * sizeof(double), cudaMemcpyHostToDevice, s));
    update_kernel<<<2 * 148, 256, 0, s>>>(N, jend, Z, N, c->d_y, 1.0, d);
    // true residual r = rhs - J d
    apply_op(c, MODE_JAC, xk, nullptr, d, r, -1.0, rhs, 1.0, s);
    c->launches++;
    beta = std::sqrt(dot(c, r, r, s));
  }
}

static void residual(pmns_ctx *c, const double *x, const double *up, double *r, cudaStream_t s) {
  apply_op(c, MODE_RES, x, up, x, r, 1.0, nullptr, 0.0, s);
}

static double b0_norm(pmns_ctx *c, cudaStream_t s) {
  double *z = c->w[5], *r = c->w[6];
  CK(cudaMemsetAsync(z, 0, c->geo.N * sizeof(double), s));
  residual(c, z, z, r, s);
  return std::sqrt(dot(c, r, r, s));
}

static pmns_status newton(pmns_ctx *c, double *x, const double *up, const pmns_solve_opts &o, pmns_report &rep,
                          int max_newton, double b0n, cudaStream_t s) {
  int64_t N = c->geo.N;
  double *r = c->w[6], *dlt = c->w[7];
  double rmin = 1e300;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0, s));
  pmns_status st = PMNS_ENOCONV;
  for (int k = 0; k <= max_newton; ++k) {
    residual(c, x, up, r, s);
    double rn = std::sqrt(dot(c, r, r, s)) / b0n;
    if (rep.newton_iters < 64) rep.res_hist[rep.newton_iters] = rn;
    if (g_verbose) fprintf(stderr, "[pmns newton] step %d  |r|/|b0| %.6e\n", k, rn);
    if (rn <= o.newton_tol) {
      st = PMNS_OK;
      rep.converged = 1;
      break;
    }
    if (rn > 10.0 * rmin) {
      st = PMNS_EDIVERGED;
      break;
    }
    rmin = std::min(rmin, rn);
    if (k == max_newton) break;
    // rhs = -r
    axpby_kernel<<<nblk(N), 256, 0, s>>>(N, -1.0, r, 0.0, nullptr, r);
    c->launches++;
    bool ok = false;
    int it = fgmres(c, x, r, dlt, o.krylov_tol * b0n, o.restart, o.max_krylov, ok, s);
    if (rep.newton_iters < 64) rep.krylov_iters[rep.newton_iters] = it;
    rep.total_krylov += it;
    rep.newton_iters++;
    axpby_kernel<<<nblk(N), 256, 0, s>>>(N, 1.0, x, 1.0, dlt, x);
    c->launches++;
  }
  CK(cudaEventRecord(e1, s));
  CK(cudaEventSynchronize(e1));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  rep.t_sol_ms += ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return st;
}

#include "dist_ops.inc"

static void fill_defaults(pmns_solve_opts &o) {
  if (o.newton_tol <= 0) o.newton_tol = 1e-8;
  if (o.krylov_tol <= 0) o.krylov_tol = 1e-9;
  if (o.restart <= 0) o.restart = 50;
  if (o.restart > kMaxK - 2) o.restart = kMaxK - 2;
  if (o.max_krylov <= 0) o.max_krylov = 2000;
  if (o.max_newton <= 0) o.max_newton = 30;
}

static pmns_status status_of(const std::exception &e) {
  g_err = e.what();
  std::string m = e.what();
  if (m.rfind("ENONPERC", 0) == 0) return PMNS_ENONPERC;
  if (m.rfind("ESINGULAR", 0) == 0) return PMNS_ESINGULAR;
  if (m.rfind("ENOMEM", 0) == 0) return PMNS_ENOMEM;
  if (m.rfind("EINVAL", 0) == 0) return PMNS_EINVAL;
  if (m.rfind("ENCCL", 0) == 0) return PMNS_ENCCL;
  return PMNS_ECUDA;
}

// report fields common to every solve entry point
static pmns_status finalize_report(pmns_ctx *c, pmns_report *rep, pmns_status st) {
  if (!c || !rep) return st;
  rep->t_setup_ms = c->t_setup_ms;
  const Build &b = c->B;
  const int64_t N = c->geo.N;
  int64_t by = b.mpn.st_elems * 8 + b.mdn.st_elems * 8 + b.coarse.bytes + b.B_bytes + 3 * 8 * (3 * N + c->geo.n_f);
  if (rep->total_krylov > 0) by += 32 * N * 26;   // CGS2 at a mean basis size of ~25
  rep->bytes_per_iter = by;
  rep->failed_subdomain = -1;
  if (st == PMNS_ESINGULAR) {
    const std::string &m = g_err;
    for (const char *key : {" block ", " front "}) {
      size_t p = m.rfind(key);
      if (p != std::string::npos) {
        rep->failed_subdomain = atoi(m.c_str() + p + strlen(key));
        break;
      }
    }
  }
  return st;
}

}  // namespace pmns

using namespace pmns;

#define ABI_TRY try {
#define ABI_CATCH                   \
  }                                 \
  catch (const std::exception &e) { \
    return status_of(e);            \
  }                                 \
  return PMNS_OK;

extern "C" {

const char *pmns_last_error(void) { return g_err.c_str(); }

namespace pmns {
// Process-wide pool of execution resources (the build streams): creating 18
// streams per context costs milliseconds, so a destroyed context hands its set
// back for the next one on the same device.
struct ExecSet {
  int device = -1;
  cudaStream_t bst[2] = {};
  cudaStream_t pst[pmns_ctx::kPool] = {};
};
static std::mutex g_exec_mu;
static std::vector<ExecSet> g_exec_free;

static void acquire_exec(pmns_ctx *c) {
  ExecSet e;
  bool have = false;
  {
    std::lock_guard<std::mutex> lk(g_exec_mu);
    for (size_t q = 0; q < g_exec_free.size(); ++q)
      if (g_exec_free[q].device == c->device) {
        e = g_exec_free[q];
        g_exec_free.erase(g_exec_free.begin() + q);
        have = true;
        break;
      }
  }
  if (!have) {
    e.device = c->device;
    for (int q = 0; q < 2; ++q) CK(cudaStreamCreateWithFlags(&e.bst[q], cudaStreamNonBlocking));
    for (int q = 0; q < pmns_ctx::kPool; ++q) CK(cudaStreamCreateWithFlags(&e.pst[q], cudaStreamNonBlocking));
  }
  for (int q = 0; q < 2; ++q) c->bst[q] = e.bst[q];
  for (int q = 0; q < pmns_ctx::kPool; ++q) c->pst[q] = e.pst[q];
  c->have_exec = true;
}

static void release_exec(pmns_ctx *c) {
  if (!c->have_exec) return;
  cudaDeviceSynchronize();
  ExecSet e;
  e.device = c->device;
  for (int q = 0; q < 2; ++q) e.bst[q] = c->bst[q];
  for (int q = 0; q < pmns_ctx::kPool; ++q) e.pst[q] = c->pst[q];
  c->have_exec = false;
  std::lock_guard<std::mutex> lk(g_exec_mu);
  g_exec_free.push_back(e);
}

static void release_pooled_exec() {
  std::lock_guard<std::mutex> lk(g_exec_mu);
  for (auto &e : g_exec_free) {
    cudaSetDevice(e.device);
    for (int q = 0; q < 2; ++q) cudaStreamDestroy(e.bst[q]);
    for (int q = 0; q < pmns_ctx::kPool; ++q) cudaStreamDestroy(e.pst[q]);
  }
  g_exec_free.clear();
}
}  // namespace pmns

pmns_status pmns_create(const pmns_problem *prob, int32_t device, pmns_ctx **out) {
  if (!prob || !out || !prob->solid || (prob->dim != 2 && prob->dim != 3) || prob->n[0] < 1 || prob->n[1] < 1 ||
      prob->h <= 0 || prob->mu <= 0) {
    g_err = "EINVAL: bad problem";
    return PMNS_EINVAL;
  }
  if (prob->n[0] > 1023 || prob->n[1] > 1023 || prob->n[2] > 1023) {
    g_err = "EINVAL: image extents above 1023 are not supported by the packed row positions";
    return PMNS_EINVAL;
  }
  pmns_ctx *c = new pmns_ctx();
  try {
    c->device = device;
    c->prob = *prob;
    c->prob.solid = nullptr;
    if (device >= 0) CK(cudaSetDevice(device));
    int nz = prob->dim == 3 ? (int)prob->n[2] : 1;
    auto tc0 = std::chrono::steady_clock::now();
    const auto tcs = tc0;
    auto clap = [&](const char *what) {
      if (!getenv("PMNS_TRACE")) return;
      auto t = std::chrono::steady_clock::now();
      fprintf(stderr, "[pmns create] %-14s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(t - tc0).count());
      tc0 = t;
    };
    build_geometry(prob->solid, prob->dim, (int)prob->n[0], (int)prob->n[1], nz, prob->periodic & 1,
                   (prob->periodic >> 1) & 1, c->geo);
    clap("geometry");
    decompose(c->geo, prob->ws_merge_h, prob->ws_min_cells, prob->dual_layers, prob->mask_band, c->dec);
    clap("decompose");
    make_layout(c->geo, c->dec, c->lay);
    c->own_lo = 0;
    c->own_hi = c->dec.n_p;
    c->dual_lo = 0;
    c->dual_hi = c->dec.n_c;
    clap("layout");
    if (device >= 0) {   // device < 0: host-only context (setup + export, for CPU parity tests)
      acquire_exec(c);   // streams + cuBLAS/cuSOLVER handles, pooled across contexts
      clap("handles");
      g_h2d_counter = &c->h2d_bytes;
      setup_device(c, 0);
      g_h2d_counter = nullptr;
      CK(cudaStreamSynchronize(0));
      clap("device setup");
      start_layouts(c);
    }
    c->t_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tcs).count();
  } catch (const std::exception &e) {
    pmns_destroy(c);
    return status_of(e);
  }
  *out = c;
  return PMNS_OK;
}

void pmns_destroy(pmns_ctx *c) {
  if (!c) return;
  if (c->layout_th.joinable()) c->layout_th.join();
  const int dev0 = pmns::cur_device();
  cudaSetDevice(c->device);   // frees and stream syncs below belong to the context's device
  free_build(c->B);
  if (c->dist) {
    dist_free(*c->dist);
    delete c->dist;
    c->dist = nullptr;
  }
  if (c->comm) nccl_api().commDestroy(c->comm);
  if (c->d_mpbuf) dfree(c->d_mpbuf);
  for (void *p : c->chk_pinned) hpin_free(p);
  for (auto &e : c->evs) {
    cudaEventDestroy(e.a);
    cudaEventDestroy(e.b);
  }
  for (auto &e : c->evpool) cudaEventDestroy(e);
  for (void *p : {(void *)c->d_dgather_c, (void *)c->d_sc_ptr_c, (void *)c->d_sc_pos_c})
    if (p) dfree(p);
  pmns::nd_layout_free(c->ndl);
  c->ndl = nullptr;
  pmns::nd_layout_free(c->ndl_md);
  c->ndl_md = nullptr;
  for (int a = 0; a < 3; ++a)
    if (c->d_fmap[a]) dfree(c->d_fmap[a]);
  for (void *p : {(void *)c->d_tab, (void *)c->d_rec, (void *)c->d_cmap, (void *)c->d_rowpos, (void *)c->d_mask, (void *)c->d_perm,
                  (void *)c->d_slot_iface, (void *)c->d_part, (void *)c->d_scal, (void *)c->d_h, (void *)c->d_y,
                  (void *)c->d_V, (void *)c->d_Z})
    if (p) dfree(p);
  for (auto p : c->w)
    if (p) dfree(p);
  for (auto &kv : c->scratch) dfree(kv.second.first);
  release_exec(c);
  delete c;
  cudaSetDevice(dev0);
}

pmns_status pmns_dgemm(int32_t transA, int32_t m, int32_t n, int32_t k, double alpha, const double *A, int32_t lda,
                       int64_t sA, const double *B, int32_t ldb, int64_t sB, double beta, double *C, int32_t ldc,
                       int64_t sC, int32_t batch, void *stream) {
  if (m < 0 || n < 0 || k < 0 || batch < 0 || (k == 0 && beta != 1.0)) return PMNS_EINVAL;
  try {
    pmns::dgemm_sb((cudaStream_t)stream, transA ? 1 : 0, m, n, k, alpha, A, lda, sA, B, ldb, sB, beta, C, ldc, sC,
                   batch);
    CK(cudaGetLastError());
    return PMNS_OK;
  } catch (const std::exception &e) {
    g_err = e.what();
    return status_of(e);
  }
}

pmns_status pmns_dense_inverse(double *A, int32_t n, int32_t ld, void *stream) {
  if (!A || n < 1 || ld < n) return PMNS_EINVAL;
  try {
    cudaStream_t s = (cudaStream_t)stream;
    double *wk = (double *)pmns::dmalloc((size_t)pmns::kPW * n * 8);
    int *ip = (int *)pmns::dmalloc((size_t)(n + 1) * 4);
    CK(cudaMemsetAsync(ip + n, 0, 4, s));
    pmns::gj_pivot_inverse(s, A, n, ld, wk, ip, ip + n);
    int info = 0;
    CK(cudaMemcpyAsync(&info, ip + n, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    pmns::dfree(wk);
    pmns::dfree(ip);
    if (info) throw std::runtime_error("ESINGULAR: dense matrix");
    return PMNS_OK;
  } catch (const std::exception &e) {
    g_err = e.what();
    return status_of(e);
  }
}

// Free the device blocks held by the caching allocator and the pooled
// streams/handles of destroyed contexts (live contexts are unaffected).
void pmns_release_cache(void) {
  pmns::release_pooled_exec();
  pmns::dflush();
  pmns::hpin_flush();
}

pmns_status pmns_profile(pmns_ctx *c, int32_t enable) {
  if (!c) return PMNS_EINVAL;
  for (auto &e : c->evs) {   // back to the pool (re-recorded before any later query)
    c->evpool.push_back(e.a);
    c->evpool.push_back(e.b);
  }
  c->evs.clear();
  c->prof = enable != 0;
  return PMNS_OK;
}

pmns_status pmns_profile_query(pmns_ctx *c, int32_t kind, int64_t *count, double *total_ms, int64_t *total_bytes) {
  if (!c || !count || !total_ms || !total_bytes) return PMNS_EINVAL;
  try {
    *count = 0;
    *total_ms = 0;
    *total_bytes = 0;
    for (auto &e : c->evs) {
      if (e.kind != kind) continue;
      CK(cudaEventSynchronize(e.b));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e.a, e.b));
      *count += 1;
      *total_ms += ms;
      *total_bytes += e.bytes;
    }
  } catch (const std::exception &e) {
    return status_of(e);
  }
  return PMNS_OK;
}

pmns_status pmns_query(const pmns_ctx *c, pmns_sizes *o) {
  if (!c || !o) return PMNS_EINVAL;
  memset(o, 0, sizeof(*o));
  o->n_c = c->geo.n_c;
  o->n_f = c->geo.n_f;
  o->N = c->geo.N;
  o->n_p = c->dec.n_p;
  o->n_iface = c->dec.n_c;
  o->n_coarse = c->B.ok ? c->B.n_coarse : 0;
  o->nx = c->geo.nx;
  o->ny = c->geo.ny;
  o->nz = c->geo.nz;
  int64_t du = 0;
  for (auto &s : c->lay.dual_unknowns) du += (int64_t)s.size();
  o->dual_unknowns = du;
  o->mp_bytes = c->B.mpn.st_elems * 8;
  o->md_bytes = c->B.use_md_nd ? c->B.mdn.st_elems * 8 : c->B.md.bytes;
  o->coarse_bytes = c->B.coarse.bytes;
  o->prolong_bytes = c->B.B_bytes;
  o->raw_basins = c->dec.raw_basins;
  o->h2d_bytes = c->h2d_bytes;
  o->rank = c->rank;
  o->world = c->world;
  o->own_lo = c->own_lo;
  o->own_hi = c->own_hi;
  return PMNS_OK;
}

// Memory plan of the local operators (layout-only: the structural nested-
// dissection plans, no numeric build): what pmns_build_preconditioner will
// store and how many flops one factorisation costs.
pmns_status pmns_memory_plan(pmns_ctx *c, pmns_memplan *o) {
  if (!c || !o) return PMNS_EINVAL;
  memset(o, 0, sizeof(*o));
  if (c->device < 0) {
    g_err = "ESTATE: host-only context";
    return PMNS_ESTATE;
  }
  try {
    join_layouts(c);
    if (c->ndl) {
      o->mp_bytes = c->ndl->st_elems * 8;
      o->mp_flops = c->ndl->flops;
      o->mp_fronts = (int64_t)c->ndl->plan.f.size();
      o->mp_max_pivots = c->ndl->max_m;
      o->mp_max_boundary = c->ndl->max_b;
      o->mp_levels = c->ndl->H + 1;
    }
    if (c->ndl_md) {
      o->md_bytes = c->ndl_md->st_elems * 8;
      o->md_flops = c->ndl_md->flops;
      o->md_fronts = (int64_t)c->ndl_md->plan.f.size();
    }
    const int64_t N = c->geo.N;
    o->krylov_bytes = (int64_t)(2 * 50 + 1) * N * 8;
    o->index_bytes = (int64_t)kTab * N * 4 + 5 * N;
    int64_t big = 0;
    for (int i = 0; i < c->dec.n_p; ++i) big = std::max<int64_t>(big, c->lay.seg[i + 1] - c->lay.seg[i]);
    o->max_primary_unknowns = big;
    // run-length statistics of the per-row stencil table: a run = consecutive
    // rows of one type and mask whose every code is the previous row's + 1 (slot
    // codes) or equal (ZERO / GHOST / MIRROR / absent): what a run-length coded
    // table would store once per run instead of 88 B per row
    if (!c->h_tab.empty() && !c->lay.perm.empty()) {
      const int32_t *T = c->h_tab.data();
      std::vector<uint32_t> rp((size_t)N);
      std::vector<uint8_t> mk((size_t)N);
      CK(cudaMemcpy(rp.data(), c->d_rowpos, (size_t)N * 4, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(mk.data(), c->d_mask, (size_t)N, cudaMemcpyDeviceToHost));
      int64_t runs = 0;
      for (int64_t r = 0; r < N; ++r) {
        bool cont = r > 0 && (rp[r] >> 30) == (rp[r - 1] >> 30) && mk[r] == mk[r - 1];
        const int nq = (rp[r] >> 30) == 3 ? 2 * c->geo.dim : kTab;
        for (int q = 0; cont && q < nq; ++q) {
          const int32_t a = T[(size_t)q * N + r - 1], b2 = T[(size_t)q * N + r];
          cont = a >= 0 ? b2 == a + 1 : b2 == a;
        }
        if (!cont) runs++;
      }
      o->stencil_runs = runs;
    }
    return PMNS_OK;
  } catch (const std::exception &e) {
    g_err = e.what();
    return status_of(e);
  }
}

pmns_status pmns_export_layout(const pmns_ctx *c, int64_t *perm, int32_t *labels, int32_t *iface, int64_t *dual_ptr,
                               int64_t *dual_cells, uint8_t *mask) {
  if (!c) return PMNS_EINVAL;
  if (perm) memcpy(perm, c->lay.perm.data(), c->lay.perm.size() * sizeof(int64_t));
  if (labels) memcpy(labels, c->dec.label.data(), c->dec.label.size() * sizeof(int32_t));
  if (iface) memcpy(iface, c->dec.iface.data(), c->dec.iface.size() * sizeof(int32_t));
  if (dual_ptr) {
    int64_t p = 0;
    dual_ptr[0] = 0;
    for (size_t j = 0; j < c->dec.duals.size(); ++j) {
      if (dual_cells) memcpy(dual_cells + p, c->dec.duals[j].data(), c->dec.duals[j].size() * sizeof(int64_t));
      p += (int64_t)c->dec.duals[j].size();
      dual_ptr[j + 1] = p;
    }
  }
  if (mask) memcpy(mask, c->lay.face_mask.data(), c->lay.face_mask.size());
  return PMNS_OK;
}

pmns_status pmns_permute(pmns_ctx *c, const double *src, double *dst, int32_t dir, void *stream) {
  if (!c || !src || !dst || src == dst) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  ABI_TRY
  cudaStream_t s = (cudaStream_t)stream;
  permute_kernel<<<nblk(c->geo.N), 256, 0, s>>>(c->geo.N, c->d_perm, src, dst, dir);
  c->launches++;
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_residual(pmns_ctx *c, const double *x, const double *up, double *r, void *stream) {
  if (!c || !x || !r) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  ABI_TRY
  residual(c, x, up, r, (cudaStream_t)stream);
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_apply_jacobian(pmns_ctx *c, const double *xk, const double *v, double *y, void *stream) {
  if (!c || !xk || !v || !y) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  ABI_TRY
  apply_op(c, MODE_JAC, xk, nullptr, v, y, 1.0, nullptr, 0.0, (cudaStream_t)stream);
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_apply_jacobian_fused(pmns_ctx *c, const double *xk, const double *v, const double *b, double *y,
                                      void *stream) {
  if (!c || !xk || !v || !b || !y) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  ABI_TRY
  apply_op(c, MODE_JAC, xk, nullptr, v, y, -1.0, b, 1.0, (cudaStream_t)stream);
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_apply_jacobian_modified(pmns_ctx *c, const double *w, const double *v, double *y, void *stream) {
  if (!c || !w || !v || !y) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  ABI_TRY
  apply_op(c, MODE_JW, w, nullptr, v, y, 1.0, nullptr, 0.0, (cudaStream_t)stream);
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_build_preconditioner(pmns_ctx *c, const double *xb, void *stream) {
  if (!c) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  ABI_TRY
  build(c, xb, (cudaStream_t)stream);
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_apply_preconditioner(pmns_ctx *c, const double *xk, const double *v, double *z, void *stream) {
  if (!c || !xk || !v || !z) return PMNS_EINVAL;
  if (c->B.mg_only) return PMNS_ESTATE;
  if (!c->d_rowpos) return PMNS_ESTATE;
  if (!c->B.ok) return PMNS_ESTATE;
  ABI_TRY
  apply_m(c, xk, v, z, (cudaStream_t)stream);
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_comm_unique_id(uint8_t *out128) {
  if (!out128) return PMNS_EINVAL;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ABI_TRY
  ncclUniqueId id;
  if (nccl_api().getUniqueId(&id) != ncclSuccess) throw std::runtime_error("ECUDA: ncclGetUniqueId failed");
  memcpy(out128, &id, 128);
  ABI_CATCH
}

// Contiguous primary ranges of the slab partition: primary ids
// follow the first voxel in z-major order, so contiguous id ranges are z-slabs.
// The cost of a primary of n unknowns is modelled as 0.6 n^2 / sum n^2 (dense
// front flops of a build) + 0.4 n^(4/3) / sum n^(4/3) (bytes its M_p apply
// streams) -- the build : Krylov split of the config-3 step -- and the cuts
// minimise the largest rank cost over all contiguous partitions (binary search
// on the bottleneck, greedy feasibility); a proportional prefix split can leave
// a rank empty next to one oversized primary (config 3 at world 8).  Every rank
// computes the same cuts from the replicated layout.
static std::vector<int> primary_cuts(const pmns_ctx *c, int world) {
  const int np = c->dec.n_p;
  std::vector<double> w(np, 0.0);
  double s2 = 0.0, s43 = 0.0;
  for (int i = 0; i < np; ++i) {
    const double n = (double)(c->lay.seg[i + 1] - c->lay.seg[i]);
    s2 += n * n;
    s43 += std::pow(n, 4.0 / 3.0);
  }
  double tot = 0.0, wmax = 0.0;
  for (int i = 0; i < np; ++i) {
    const double n = (double)(c->lay.seg[i + 1] - c->lay.seg[i]);
    w[i] = (s2 > 0 ? 0.6 * n * n / s2 : 0.0) + (s43 > 0 ? 0.4 * std::pow(n, 4.0 / 3.0) / s43 : 0.0);
    tot += w[i];
    wmax = std::max(wmax, w[i]);
  }
  auto parts_needed = [&](double cap) {   // greedy: fewest contiguous parts with cost <= cap each
    int parts = 1;
    double acc = 0.0;
    for (int i = 0; i < np; ++i) {
      if (acc + w[i] > cap && acc > 0.0) {
        ++parts;
        acc = 0.0;
      }
      acc += w[i];
    }
    return parts;
  };
  double lo = std::max(wmax, tot / std::max(world, 1)), hi = tot;
  for (int it = 0; it < 60 && hi - lo > 1e-12 * std::max(tot, 1e-300); ++it) {
    const double mid = 0.5 * (lo + hi);
    if (parts_needed(mid) <= world) hi = mid;
    else lo = mid;
  }
  std::vector<int> pc(world + 1, np);
  pc[0] = 0;
  int r = 1;
  double acc = 0.0;
  const double cap = hi * (1.0 + 1e-9);
  for (int i = 0; i < np && r < world; ++i) {
    if (acc + w[i] > cap && acc > 0.0) {
      pc[r++] = i;
      acc = 0.0;
    }
    acc += w[i];
  }
  // fewer parts than ranks: split the remaining ranks off the tail one primary at a time
  for (int q = world - 1; q >= r; --q) pc[q] = std::max(pc[r - 1], np - (world - q));
  for (int q = 1; q <= world; ++q) pc[q] = std::max(pc[q], pc[q - 1]);
  pc[world] = np;
  return pc;
}

static pmns_status set_comm_impl(pmns_ctx *c, int32_t rank, int32_t world, const uint8_t *id128, LoopGroup *lg) {
  if (!c || world < 1 || rank < 0 || rank >= world) return PMNS_EINVAL;
  if (lg && lg->world != world) return PMNS_EINVAL;
  ABI_TRY
  if (c->dist) {
    dist_free(*c->dist);
    delete c->dist;
    c->dist = nullptr;
  }
  if (c->comm) {
    nccl_api().commDestroy(c->comm);
    c->comm = nullptr;
  }
  join_layouts(c);
  if (c->d_rowpos) free_build(c->B);
  pmns::nd_layout_free(c->ndl);
  c->ndl = nullptr;
  pmns::nd_layout_free(c->ndl_md);
  c->ndl_md = nullptr;
  c->rank = rank;
  c->world = world;
  // contiguous primary ranges (W order ~ z-slabs): primary_cuts
  const int np = c->dec.n_p;
  const std::vector<int> pcuts = primary_cuts(c, world);
  auto cut = [&](int r) { return pcuts[std::max(0, std::min(world, r))]; };
  c->own_lo = cut(rank);
  c->own_hi = cut(rank + 1);
  if (c->own_hi < c->own_lo) c->own_hi = c->own_lo;
  // dual grids (M_d): contiguous ranges balanced by n_j^2 as well
  {
    const int nd = (int)c->lay.dual_unknowns.size();
    std::vector<double> dp(nd + 1, 0.0);
    for (int j = 0; j < nd; ++j) {
      double n = (double)c->lay.dual_unknowns[j].size();
      dp[j + 1] = dp[j] + n * n;
    }
    auto dcut = [&](int r) {
      if (r <= 0) return 0;
      if (r >= world) return nd;
      return (int)(std::lower_bound(dp.begin(), dp.end(), dp[nd] * r / world) - dp.begin());
    };
    c->dual_lo = std::max(0, std::min(nd, dcut(rank)));
    c->dual_hi = std::max(c->dual_lo, std::min(nd, dcut(rank + 1)));
    c->owned_duals.assign(c->lay.dual_unknowns.begin() + c->dual_lo, c->lay.dual_unknowns.begin() + c->dual_hi);
  }
  for (int64_t **p : {&c->d_dgather_c, &c->d_sc_ptr_c, &c->d_sc_pos_c})
    if (*p) {
      dfree(*p);
      *p = nullptr;
    }
  if (id128 && c->d_rowpos) {   // (world 1 with an id: a 1-rank communicator, for tests of the NCCL path)
    ncclUniqueId id;
    memcpy(&id, id128, 128);
    CK(cudaSetDevice(c->device));
    if (nccl_api().commInitRank(&c->comm, world, id, rank) != ncclSuccess) {
      c->comm = nullptr;
      throw std::runtime_error("ENCCL: ncclCommInitRank failed");
    }
  }
  // distributed Krylov phase: owned slabs, halo exchanges (dist.inc)
  if (world > 1 && c->d_rowpos && (c->comm || lg)) {
    c->dist = new DistPlan();
    DistPlan &D = *c->dist;
    if (lg) {
      D.tr = new LoopTransport(lg, rank);
    } else {
      D.tr = new NcclTransport(c->comm);
    }
    D.own_tr = true;
    const std::vector<int> &pc = pcuts;
    cudaStream_t s0 = c->bst[0];
    try {
      dist_plan(c, D, pc, s0);
      CK(cudaStreamSynchronize(s0));
    } catch (...) {
      dist_free(*c->dist);
      delete c->dist;
      c->dist = nullptr;
      throw;
    }
    // the dual grid of an interface belongs to the interface's owner
    c->dual_lo = D.j_lo;
    c->dual_hi = D.j_hi;
    c->owned_duals.assign(c->lay.dual_unknowns.begin() + c->dual_lo, c->lay.dual_unknowns.begin() + c->dual_hi);
    D.on = true;
  }
  ABI_CATCH
}

pmns_status pmns_set_comm(pmns_ctx *c, int32_t rank, int32_t world, const uint8_t *id128) {
  return set_comm_impl(c, rank, world, id128, nullptr);
}

pmns_status pmns_halo_plan(pmns_ctx *c, int32_t rank, int32_t world, int64_t *counts, int64_t *slots) {
  if (!c || !counts || world < 1 || rank < 0 || rank >= world) return PMNS_EINVAL;
  ABI_TRY
  if (c->h_rowpos.empty()) host_rowpos(c);
  if (c->h_tab.empty()) host_tab(c);
  const std::vector<int> pc = primary_cuts(c, world);
  const int r0 = c->rank, w0 = c->world;
  c->rank = rank;
  c->world = world;
  DistPlan D;
  try {
    dist_plan(c, D, pc, nullptr, false);
  } catch (...) {
    c->rank = r0;
    c->world = w0;
    throw;
  }
  c->rank = r0;
  c->world = w0;
  const HaloList *Ls[4] = {&D.fr, &D.fs, &D.rs, &D.rr};
  int64_t pos = 0;
  for (int p = 0; p < world; ++p)
    for (int q = 0; q < 4; ++q) {
      const HaloList &L = *Ls[q];
      auto it = std::lower_bound(L.peer.begin(), L.peer.end(), p);
      int64_t n = 0, o = 0;
      if (it != L.peer.end() && *it == p) {
        size_t k = (size_t)(it - L.peer.begin());
        o = L.off[k];
        n = L.off[k + 1] - o;
      }
      counts[4 * p + q] = n;
      if (slots)
        for (int64_t e = 0; e < n; ++e) slots[pos++] = L.slots[o + e];
    }
  counts[4 * world] = D.r0[0];   // owned ranges (primaries, interface cells, f-faces)
  counts[4 * world + 1] = D.r1[0];
  counts[4 * world + 2] = D.r0[1];
  counts[4 * world + 3] = D.r1[1];
  counts[4 * world + 4] = D.r0[2];
  counts[4 * world + 5] = D.r1[2];
  ABI_CATCH
}

void *pmns_loopback_create(int32_t world) {
  if (world < 1) return nullptr;
  return new LoopGroup(world);
}

void pmns_loopback_destroy(void *group) { delete (LoopGroup *)group; }

pmns_status pmns_set_comm_loopback(pmns_ctx *c, int32_t rank, int32_t world, void *group) {
  if (!group) return PMNS_EINVAL;
  return set_comm_impl(c, rank, world, nullptr, (LoopGroup *)group);
}

pmns_status pmns_apply_md(pmns_ctx *c, const double *v, double *z, void *stream) {
  if (!c || !v || !z) return PMNS_EINVAL;
  if (!c->d_rowpos || !c->B.ok || c->B.mg_only) return PMNS_ESTATE;
  ABI_TRY
  cudaStream_t s = (cudaStream_t)stream;
  Build &b = c->B;
  const int64_t N = c->geo.N;
  if (b.nd_total > 0) {
    gather_kernel<<<nblk(b.nd_total), 256, 0, s>>>(b.nd_total, b.d_dgather, v, b.d_dbuf_in);
    if (b.use_md_nd) apply_nd(c, b.mdn, b.d_dbuf_in, b.d_dbuf_out, nullptr, nullptr, s, -1);
    else gemv(c, b.md, b.d_dbuf_in, b.d_dbuf_out, nullptr, nullptr, 0, s, -1, nullptr, 1);
    scatter_sum_kernel<<<nblk(N), 256, 0, s>>>(N, b.d_sc_ptr, b.d_sc_pos, b.d_dbuf_out, z);
    c->launches += 2;
  } else {
    CK(cudaMemsetAsync(z, 0, N * sizeof(double), s));
  }
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_apply_mp(pmns_ctx *c, const double *t, double *z, void *stream) {
  if (!c || !t || !z) return PMNS_EINVAL;
  if (!c->d_rowpos || !c->B.ok || c->B.mg_only) return PMNS_ESTATE;
  ABI_TRY
  cudaStream_t s = (cudaStream_t)stream;
  int64_t np_rows = c->lay.seg[c->dec.n_p];
  CK(cudaMemsetAsync(z, 0, c->geo.N * sizeof(double), s));
  apply_nd(c, c->B.mpn, t, z, nullptr, nullptr, s, -1);
  (void)np_rows;
  CK(cudaGetLastError());
  ABI_CATCH
}

pmns_status pmns_apply_mg(pmns_ctx *c, const double *v, double *z, void *stream) {
  if (!c || !v || !z) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  if (!c->B.ok) return PMNS_ESTATE;
  ABI_TRY
  apply_mg(c, v, z, (cudaStream_t)stream);
  CK(cudaGetLastError());
  ABI_CATCH
}

static pmns_status newton_solve_impl(pmns_ctx *c, double *x, const double *up, const pmns_solve_opts *opts,
                              pmns_report *rep, void *stream) {
  if (!c || !x || !rep) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  if (!c->B.ok) return PMNS_ESTATE;
  if (c->prob.dt > 0 && !up) {
    g_err = "EINVAL: transient solve needs u_prev";
    return PMNS_EINVAL;
  }
  pmns_solve_opts o = opts ? *opts : pmns_solve_opts{};
  fill_defaults(o);
  try {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t l0 = c->launches;
    double b0n = b0_norm(c, s);
    rep->b0_norm = b0n;
    pmns_status st = newton_any(c, x, up, o, *rep, o.max_newton, b0n, s);
    if (c->dist) dist_allgather(c, x, s);
    rep->kernel_launches += c->launches - l0;
    CK(cudaGetLastError());
    return st;
  } catch (const std::exception &e) {
    return status_of(e);
  }
}

pmns_status pmns_newton_solve(pmns_ctx *c, double *x, const double *up, const pmns_solve_opts *opts,
                              pmns_report *rep, void *stream) {
  pmns_status st = newton_solve_impl(c, x, up, opts, rep, stream);
  return finalize_report(c, rep, st);
}

static pmns_status solve_steady_impl(pmns_ctx *c, double *x, const pmns_solve_opts *opts, pmns_report *rep, void *stream) {
  if (!c || !x || !rep) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  pmns_solve_opts o = opts ? *opts : pmns_solve_opts{};
  fill_defaults(o);
  memset(rep, 0, sizeof(*rep));
  try {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t l0 = c->launches;
    c->t_mg = c->t_ml = 0;
    CK(cudaMemsetAsync(x, 0, c->geo.N * sizeof(double), s));
    double b0n = b0_norm(c, s);
    rep->b0_norm = b0n;
    build(c, nullptr, s);                                   // M_S = gPLMM(w = 0) = aPLMM_S
    rep->builds++;
    if (o.variant == 1) {                                  // aPLMM_S: never rebuilt
      pmns_status st = newton_any(c, x, nullptr, o, *rep, o.max_newton, b0n, s);
      if (c->dist) dist_allgather(c, x, s);
      rep->t_mg_ms = c->t_mg;
      rep->t_ml_ms = c->t_ml;
      rep->kernel_launches = c->launches - l0;
      CK(cudaGetLastError());
      return st;
    }
    pmns_status st = newton_any(c, x, nullptr, o, *rep, 1, b0n, s);   // Newton step 0: the Stokes solve
    if (!rep->converged && st != PMNS_EDIVERGED) {
      build(c, x, s, false, o.variant == 2);                // wind = Stokes velocity; aPLMM_NS: J(x^1)
      rep->builds++;
      int used = rep->newton_iters;
      // PMNS_PROFILE_KRYLOV=1: bracket the Newton-FGMRES phase for ncu --profile-from-start off
      bool prof_range = getenv("PMNS_PROFILE_KRYLOV") != nullptr;
      if (prof_range) {
        CK(cudaStreamSynchronize(s));
        cudaProfilerStart();
      }
      st = newton_any(c, x, nullptr, o, *rep, o.max_newton - used, b0n, s);
      if (prof_range) {
        CK(cudaStreamSynchronize(s));
        cudaProfilerStop();
      }
    }
    if (c->dist) dist_allgather(c, x, s);   // every rank returns the full solution
    rep->t_mg_ms = c->t_mg;
    rep->t_ml_ms = c->t_ml;
    rep->kernel_launches = c->launches - l0;
    CK(cudaGetLastError());
    return st;
  } catch (const std::exception &e) {
    return status_of(e);
  }
}

pmns_status pmns_solve_steady(pmns_ctx *c, double *x, const pmns_solve_opts *opts, pmns_report *rep, void *stream) {
  pmns_status st = solve_steady_impl(c, x, opts, rep, stream);
  return finalize_report(c, rep, st);
}

static pmns_status solve_transient_impl(pmns_ctx *c, double *x, int32_t n_steps, const pmns_solve_opts *opts,
                                 pmns_report *rep, void *stream) {
  if (!c || !x || !rep || n_steps < 0) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  if (!(c->prob.dt > 0)) {
    g_err = "EINVAL: pmns_solve_transient needs dt > 0";
    return PMNS_EINVAL;
  }
  pmns_solve_opts o = opts ? *opts : pmns_solve_opts{};
  fill_defaults(o);
  memset(rep, 0, sizeof(*rep));
  try {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t N = c->geo.N;
    int64_t l0 = c->launches;
    c->t_mg = c->t_ml = 0;
    double *xs = dalloc<double>(N), *up = dalloc<double>(N);
    // 1) steady Stokes state (Newton step 0 of the steady problem from rest)
    const double dt = c->G.dt;
    c->G.dt = 0.0;
    pmns_report tmp;
    memset(&tmp, 0, sizeof(tmp));
    pmns_status st;
    try {
      CK(cudaMemsetAsync(xs, 0, N * sizeof(double), s));
      double b0s = b0_norm(c, s);
      build(c, nullptr, s);
      st = newton_any(c, xs, nullptr, o, tmp, 1, b0s, s);
    } catch (...) {
      c->G.dt = dt;
      throw;
    }
    c->G.dt = dt;
    // 2) one build for all time steps: wind = Stokes velocity, J(x_S) with rho/dt (reading A19)
    build(c, xs, s);
    rep->builds = 2;
    double b0n = b0_norm(c, s);
    rep->b0_norm = b0n;
    // 3) backward-Euler steps, Newton from x^n with u^n = x^n
    st = PMNS_OK;
    for (int k = 0; k < n_steps; ++k) {
      CK(cudaMemcpyAsync(up, x, N * sizeof(double), cudaMemcpyDeviceToDevice, s));
      int before = rep->newton_iters;
      rep->converged = 0;
      pmns_status sk = newton_any(c, x, up, o, *rep, o.max_newton, b0n, s);
      if (k < 64) rep->step_newton[k] = rep->newton_iters - before;
      rep->n_steps = k + 1;
      if (sk != PMNS_OK) {
        st = sk;
        break;
      }
    }
    if (c->dist) dist_allgather(c, x, s);
    rep->t_mg_ms = c->t_mg;
    rep->t_ml_ms = c->t_ml;
    rep->kernel_launches = c->launches - l0;
    dfree(xs);
    dfree(up);
    CK(cudaGetLastError());
    return st;
  } catch (const std::exception &e) {
    return status_of(e);
  }
}

pmns_status pmns_solve_transient(pmns_ctx *c, double *x, int32_t n_steps, const pmns_solve_opts *opts,
                                 pmns_report *rep, void *stream) {
  pmns_status st = solve_transient_impl(c, x, n_steps, opts, rep, stream);
  return finalize_report(c, rep, st);
}

static pmns_status solve_continuation_impl(pmns_ctx *c, double *x, int32_t n_incr, const pmns_solve_opts *opts,
                                    pmns_report *rep, void *stream) {
  if (!c || !x || !rep || n_incr < 1) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  pmns_solve_opts o = opts ? *opts : pmns_solve_opts{};
  fill_defaults(o);
  const DevGeom G0 = c->G;
  pmns_report tot;
  memset(&tot, 0, sizeof(tot));
  try {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t l0 = c->launches;
    double tmg = 0, tml = 0;
    pmns_status st = PMNS_OK;
    for (int k = 1; k <= n_incr; ++k) {
      double f = (double)k / n_incr;
      c->G.p_in = G0.p_in * f;
      c->G.p_out = G0.p_out * f;
      for (int a = 0; a < 3; ++a) c->G.bf[a] = G0.bf[a] * f;
      c->G.dt = 0.0;
      pmns_report r;
      memset(&r, 0, sizeof(r));
      if (k == 1) {
        st = pmns_solve_steady(c, x, &o, &r, stream);   // Stokes fallback wind (A19)
      } else {
        c->t_mg = c->t_ml = 0;
        r.b0_norm = b0_norm(c, s);
        build(c, x, s);                                  // wind = previous increment's velocity
        r.builds = 1;
        st = newton_any(c, x, nullptr, o, r, o.max_newton, r.b0_norm, s);
        r.t_mg_ms = c->t_mg;
        r.t_ml_ms = c->t_ml;
      }
      // accumulate
      for (int q = 0; q < r.newton_iters && tot.newton_iters + q < 64; ++q)
        tot.krylov_iters[tot.newton_iters + q] = r.krylov_iters[q];
      if (k - 1 < 64) {
        tot.step_newton[k - 1] = r.newton_iters;
        tot.res_hist[k - 1] = r.res_hist[std::min(r.newton_iters, 64)];
      }
      tot.newton_iters += r.newton_iters;
      tot.total_krylov += r.total_krylov;
      tot.builds += r.builds;
      tmg += r.t_mg_ms;
      tml += r.t_ml_ms;
      tot.t_sol_ms += r.t_sol_ms;
      tot.n_steps = k;
      tot.b0_norm = r.b0_norm;
      if (st != PMNS_OK) break;
    }
    c->G = G0;
    if (c->dist) dist_allgather(c, x, s);
    tot.converged = st == PMNS_OK;
    tot.t_mg_ms = tmg;
    tot.t_ml_ms = tml;
    tot.kernel_launches = c->launches - l0;
    *rep = tot;
    CK(cudaGetLastError());
    return st;
  } catch (const std::exception &e) {
    c->G = G0;
    return status_of(e);
  }
}

pmns_status pmns_solve_continuation(pmns_ctx *c, double *x, int32_t n_incr, const pmns_solve_opts *opts,
                                    pmns_report *rep, void *stream) {
  pmns_status st = solve_continuation_impl(c, x, n_incr, opts, rep, stream);
  return finalize_report(c, rep, st);
}

static pmns_status coarse_solve_impl(pmns_ctx *c, double *x, int32_t n_ramp, const pmns_solve_opts *opts,
                              pmns_report *rep, void *stream) {
  if (!c || !x || !rep || n_ramp < 1) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  pmns_solve_opts o = opts ? *opts : pmns_solve_opts{};
  if (o.newton_tol <= 0) o.newton_tol = 1e-6;   // Algorithm 1's ||r_c|| / ||r_c^0|| < 1e-6
  if (o.max_newton <= 0) o.max_newton = 50;
  memset(rep, 0, sizeof(*rep));
  const DevGeom G0 = c->G;
  try {
    cudaStream_t s = (cudaStream_t)stream;
    int64_t N = c->geo.N, l0 = c->launches;
    c->t_mg = c->t_ml = 0;
    CK(cudaMemsetAsync(x, 0, N * sizeof(double), s));
    double *r = c->w[7], *z = c->w[4];
    std::vector<double> rc((size_t)std::max(1, 1));
    c->G.dt = 0.0;   // steady
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    pmns_status st = PMNS_OK;
    for (int k = 1; k <= n_ramp; ++k) {
      // drive increment (the paper ramps Re by raising p_in)
      double f = (double)k / n_ramp;
      c->G.p_in = G0.p_in * f;
      c->G.p_out = G0.p_out * f;
      for (int a = 0; a < 3; ++a) c->G.bf[a] = G0.bf[a] * f;
      // M_G from J~_w with the previous increment's velocity (Stokes fallback: w = 0)
      build(c, k == 1 ? nullptr : x, s, true);
      rep->builds++;
      Build &b = c->B;
      int nc = b.n_coarse;
      if (nc == 0) break;
      int ldc = (nc + 1) & ~1;
      struct DevBuf {   // freed on every exit path
        void *p;
        explicit DevBuf(size_t bytes) : p(dmalloc(bytes)) {}
        ~DevBuf() { dfree(p); }
      };
      DevBuf bJc((size_t)nc * ldc * 8), bgw((size_t)kPW * nc * 8), bgi((size_t)(nc + 1) * 4), btmp((size_t)nc * 8);
      double *Jc = (double *)bJc.p, *gw = (double *)bgw.p, *tmp = (double *)btmp.p;
      int *gi = (int *)bgi.p;
      auto rc_norm = [&]() {
        apply_op(c, MODE_RESM, x, nullptr, x, r, 1.0, nullptr, 0.0, s);   // r~
        restrict_(c, r, b.d_bc, 1, s);                                      // r_c = R^ r~
        std::vector<double> h(nc);
        CK(cudaMemcpyAsync(h.data(), b.d_bc, nc * sizeof(double), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        double a2 = 0;
        for (double v : h) a2 += v * v;
        return std::sqrt(a2);
      };
      CK(cudaEventRecord(e0, s));
      double r0 = rc_norm(), rn = r0;
      int it = 0;
      while (it < o.max_newton && r0 > 0) {
        assemble_coarse(c, MODE_JACM, x, Jc, ldc, s);                      // J_c = R^ J~^k P^
        // Jc row-major == J_c^T column-major; its in-place inverse is (J_c^{-1})^T
        // column-major, so delta_c = -J_c^{-1} r_c = -(that)^T r_c
        CK(cudaMemsetAsync(gi + nc, 0, sizeof(int), s));
        gj_pivot_inverse(s, Jc, nc, ldc, gw, gi, gi + nc);
        int info = 0;
        CK(cudaMemcpyAsync(&info, gi + nc, sizeof(int), cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        if (info != 0) throw std::runtime_error("ESINGULAR: coarse Jacobian J_c (Algorithm 1)");
        negate_kernel<<<nblk(nc), 256, 0, s>>>(nc, b.d_bc);
        gemv_t_kernel<<<nblk((int64_t)nc * 32), 256, 0, s>>>(nc, Jc, ldc, b.d_bc, tmp);
        CK(cudaMemcpyAsync(b.d_bc, tmp, nc * sizeof(double), cudaMemcpyDeviceToDevice, s));
        c->launches += 3 * ((nc + kPW - 1) / kPW) + 3;
        prolong(c, b.d_bc, z, s);                                          // x^ += P^ delta_c
        axpby_kernel<<<nblk(N), 256, 0, s>>>(N, 1.0, x, 1.0, z, x);
        c->launches += 2;
        ++it;
        rn = rc_norm();
        if (rn / r0 < o.newton_tol) break;
      }
      CK(cudaEventRecord(e1, s));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      rep->t_sol_ms += ms;
      if (k - 1 < 64) {
        rep->step_newton[k - 1] = it;
        rep->res_hist[k - 1] = r0 > 0 ? rn / r0 : 0.0;
      }
      rep->newton_iters += it;
      rep->n_steps = k;
      if (r0 > 0 && !(rn / r0 < o.newton_tol)) st = PMNS_ENOCONV;
    }
    rep->converged = st == PMNS_OK;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    c->G = G0;
    rep->t_mg_ms = c->t_mg;
    rep->t_ml_ms = c->t_ml;
    rep->kernel_launches = c->launches - l0;
    CK(cudaGetLastError());
    return st;
  } catch (const std::exception &e) {
    c->G = G0;
    return status_of(e);
  }
}

pmns_status pmns_coarse_solve(pmns_ctx *c, double *x, int32_t n_ramp, const pmns_solve_opts *opts,
                              pmns_report *rep, void *stream) {
  pmns_status st = coarse_solve_impl(c, x, n_ramp, opts, rep, stream);
  return finalize_report(c, rep, st);
}

pmns_status pmns_solve_steady_host(pmns_ctx *c, double *xh, const pmns_solve_opts *opts, pmns_report *rep) {
  return pmns_solve_continuation_host(c, xh, 1, opts, rep);
}

pmns_status pmns_solve_continuation_host(pmns_ctx *c, double *xh, int32_t n_incr, const pmns_solve_opts *opts,
                                         pmns_report *rep) {
  if (!c || !xh || !rep || n_incr < 1) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  try {
    int64_t N = c->geo.N;
    double *xd = dalloc<double>(N), *xc = dalloc<double>(N);
    pmns_status st = n_incr == 1 ? pmns_solve_steady(c, xd, opts, rep, nullptr)
                                 : pmns_solve_continuation(c, xd, n_incr, opts, rep, nullptr);
    if (st == PMNS_OK || st == PMNS_ENOCONV) {
      permute_kernel<<<nblk(N), 256>>>(N, c->d_perm, xd, xc, 1);
      CK(cudaMemcpy(xh, xc, N * sizeof(double), cudaMemcpyDeviceToHost));
    }
    dfree(xd);
    dfree(xc);
    return st;
  } catch (const std::exception &e) {
    return status_of(e);
  }
}

// pmns_solve_transient from rest with HOST output (canonical order): the e2e
// path of the transient pipeline (config 4)
pmns_status pmns_solve_transient_host(pmns_ctx *c, double *xh, int32_t n_steps, const pmns_solve_opts *opts,
                                      pmns_report *rep) {
  if (!c || !xh || !rep || n_steps < 1) return PMNS_EINVAL;
  if (!c->d_rowpos) return PMNS_ESTATE;
  try {
    int64_t N = c->geo.N;
    double *xd = dalloc<double>(N), *xc = dalloc<double>(N);
    CK(cudaMemset(xd, 0, N * sizeof(double)));
    pmns_status st = pmns_solve_transient(c, xd, n_steps, opts, rep, nullptr);
    if (st == PMNS_OK || st == PMNS_ENOCONV) {
      permute_kernel<<<nblk(N), 256>>>(N, c->d_perm, xd, xc, 1);
      CK(cudaMemcpy(xh, xc, N * sizeof(double), cudaMemcpyDeviceToHost));
    }
    dfree(xd);
    dfree(xc);
    return st;
  } catch (const std::exception &e) {
    return status_of(e);
  }
}

}  // extern "C"
