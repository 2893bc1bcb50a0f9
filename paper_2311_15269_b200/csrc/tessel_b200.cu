// tessel_b200.cu — sm_100a kernels and the C ABI (include/tessel_b200.h).
//
// Kernels
//   k_decide_batch  general reference-exact decide, one problem per thread
//                   (replaces repsched._core.decide, kernel_c.pyx:23-508)
//   k_stage         K1: unrank a window of candidate ranks in the reference's
//                   lexicographic order (repetend.py:65-90), entry memory and
//                   memory gate (repetend.py:93-105, 264-268)
//   k_probe         K2: one (candidate, period) repetend probe per thread —
//                   anchored bounds + period-parametric lags
//                   (repetend.py:160-190) + reference-exact decide; SAT rows
//                   are compacted out, the rest stay active for the next
//                   period (the period scan of repetend.py:289-302, run
//                   level-synchronously across the window)
// All arithmetic is int32 on the ALU/FMA pipes; no tensor cores, HBM holds
// only the window's assignments, the active lists and per-thread DFS scratch.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <chrono>
#include <ctime>
#include <functional>
#include <memory>
#include <mutex>
#include <thread>
#include <numeric>
#include <string>
#include <map>
#include <unordered_map>
#include <vector>

#include "../../include/tessel_b200.h"
#include "host_build.hpp"
#include "models.cuh"
#include "dj_solve.cuh"
#include "wrx_dfs.cuh"
#include "wrr_dfs.cuh"
#include "wst_dfs.cuh"
#include "wdj_solve.cuh"
#include "sp_dfs.cuh"
#include "validate.cuh"

#define TSL_VERSION 2

// resident blocks per SM the resolve kernel is compiled for (register cap)
#ifndef RESOLVE_MIN_BLOCKS
#define RESOLVE_MIN_BLOCKS 4
#endif

static thread_local std::string g_err;

// Process-wide accounting for the bench's gpu_launches / e2e byte counts.
#include <atomic>
static std::atomic<long long> g_launches{0}, g_h2d{0}, g_d2h{0};
#define COUNT_LAUNCH() g_launches.fetch_add(1, std::memory_order_relaxed)
#define COUNT_H2D(b) g_h2d.fetch_add((long long)(b), std::memory_order_relaxed)
#define COUNT_D2H(b) g_d2h.fetch_add((long long)(b), std::memory_order_relaxed)

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess)                                                             \
      throw tsl::Error(TSL_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_));    \
  } while (0)

static int set_err(int code, const std::string &m) {
  g_err = m;
  return code;
}

#define API_BEGIN try {
#define API_END                                                  \
  }                                                              \
  catch (const tsl::Error &e) {                                  \
    return set_err(e.code, e.what());                            \
  }                                                              \
  catch (const std::exception &e) {                              \
    return set_err(TSL_EINVAL, e.what());                        \
  }

static void h2d(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s));
  COUNT_H2D(bytes);
}
static void d2h(void *dst, const void *src, size_t bytes, cudaStream_t s) {
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s));
  COUNT_D2H(bytes);
}

// Frees temporary device buffers on every exit path (including errors).
struct DevFree {
  std::vector<void *> ptrs;
  template <class T>
  T *add(T *p) {
    ptrs.push_back((void *)p);
    return p;
  }
  ~DevFree() {
    for (void *p : ptrs)
      if (p) cudaFree(p);
  }
};

// Stream-ordered (de)allocation for buffers that grow while other streams
// run: cudaFree synchronises the whole device, which would serialise the
// asynchronous verification slots behind every buffer growth; the pool's
// release threshold keeps freed memory cached.
// The current device's stream-ordered pool keeps freed memory cached
// (release threshold: never), so buffers are reused across growths and
// across engines.
static void pool_keep() {
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      unsigned long long keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  });
}

// Idle engine buffers, kept per device for the next engine: a dropped
// engine's buffers (its streams synchronised first) go here instead of back
// to the pool, whose cross-stream reuse of freed memory is opportunistic —
// a fresh engine then mapped ~1 GB of new memory every few searches
// (0.3-0.8 s stalls, profiles/r02m_e2e_outliers_*.log).
struct IdleBlocks {
  std::mutex mu;
  std::multimap<std::pair<int, size_t>, void *> idle;  // (device, bytes) -> block
  std::unordered_map<void *, size_t> size;             // every pool block we made
  size_t held = 0;
};
static IdleBlocks &idle_blocks() {
  static IdleBlocks b;
  return b;
}
static constexpr size_t IDLE_MAX = 16ull << 30;  // bytes kept idle per process

// A block of >= bytes: an idle one (at most 2x larger) or a new pool block.
static void *dev_take(size_t bytes, cudaStream_t s) {
  pool_keep();
  int dev = 0;
  CK(cudaGetDevice(&dev));
  IdleBlocks &b = idle_blocks();
  {
    std::lock_guard<std::mutex> g(b.mu);
    auto it = b.idle.lower_bound({dev, bytes});
    if (it != b.idle.end() && it->first.first == dev && it->first.second <= 2 * bytes + (1 << 20)) {
      void *p = it->second;
      b.held -= it->first.second;
      b.idle.erase(it);
      return p;
    }
  }
  void *p = nullptr;
  CK(cudaMallocAsync(&p, bytes, s));
  std::lock_guard<std::mutex> g(b.mu);
  b.size[p] = bytes;
  return p;
}

// Park an idle block (its users' streams are done with it) for a later
// engine, or free it when the idle set is full / it is not ours.
static void dev_park(void *p, cudaStream_t s) {
  if (!p) return;
  int dev = 0;
  cudaGetDevice(&dev);
  IdleBlocks &b = idle_blocks();
  {
    std::lock_guard<std::mutex> g(b.mu);
    auto it = b.size.find(p);
    if (it != b.size.end() && b.held + it->second <= IDLE_MAX) {
      b.idle.insert({{dev, it->second}, p});
      b.held += it->second;
      return;
    }
    if (it != b.size.end()) b.size.erase(it);
  }
  cudaFreeAsync(p, s);
}

static void dev_grow(void **p, size_t bytes, cudaStream_t s) {
  pool_keep();
  if (*p) {
    {
      IdleBlocks &b = idle_blocks();
      std::lock_guard<std::mutex> g(b.mu);
      b.size.erase(*p);
    }
    CK(cudaFreeAsync(*p, s));
  }
  *p = dev_take(bytes, s);
}

static void require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw tsl::Error(TSL_ENODEV, std::string("no CUDA device available (") +
                                     (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                                     "); the B200 path has no CPU fallback");
  }
}

// ------------------------------------------------------------------ kernels

__global__ void __launch_bounds__(32) k_decide_batch(const int *__restrict__ pools,
                                                     const long long *__restrict__ pool_off,
                                                     int count,
                                                     const long long *__restrict__ budgets,
                                                     unsigned long long budget_ns, int *ws_base,
                                                     const long long *__restrict__ ws_off,
                                                     int *status, long long *nodes, int *starts,
                                                     int stride) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int *pool = pools + pool_off[i];
  const GenView g = gen_view(pool);
  RxWs w = rx_ws_carve(ws_base + ws_off[i], g.n_, pool[G_MAXDI]);
  for (int k = 0; k < g.n_; ++k) {
    w.lo[k] = g.lo_[k];
    w.hi[k] = g.hi_[k];
  }
  const unsigned long long t_end = budget_ns ? rx_now_ns() + budget_ns : 0ull;
  long long nd = 0;
  const int st = rx_decide(g, w, budgets[i], t_end, &nd);
  status[i] = st;
  nodes[i] = nd;
  if (st == RX_SAT)
    for (int k = 0; k < g.n_; ++k) starts[(long long)i * stride + k] = w.s[k];
}

// Warp-per-problem variant: lanes cooperate on one reference-exact DFS
// (wrx_dfs.cuh); mutable state in shared memory (fast shared atomics),
// per-depth snapshots in global memory.
__global__ void __launch_bounds__(32) k_decide_warp(const int *__restrict__ pools,
                                                    const long long *__restrict__ pool_off,
                                                    int count,
                                                    const long long *__restrict__ budgets,
                                                    unsigned long long budget_ns, int *ws_base,
                                                    const long long *__restrict__ ws_off,
                                                    int *status, long long *nodes, int *starts,
                                                    int stride) {
  extern __shared__ int sm[];
  const int i = blockIdx.x;
  if (i >= count) return;
  const int lane = threadIdx.x & 31;
  const int *pool = pools + pool_off[i];
  const GenView g = gen_view(pool);
  WWs w = wrx_carve(sm, ws_base + ws_off[i], g.n_, pool[G_MAXDI]);
  for (int k = lane; k < g.n_; k += 32) {
    w.lo[k] = g.lo_[k];
    w.hi[k] = g.hi_[k];
  }
  __syncwarp();
  const unsigned long long t_end = budget_ns ? rx_now_ns() + budget_ns : 0ull;
  long long nd = 0;
  const int st = wrx_decide(g, w, budgets[i], t_end, &nd);
  if (lane == 0) {
    status[i] = st;
    nodes[i] = nd;
  }
  if (st == RX_SAT)
    for (int k = lane; k < g.n_; k += 32) starts[(long long)i * stride + k] = w.s[k];
}

__device__ __forceinline__ void load_pool(int *sp, const int *__restrict__ gpool) {
  const int words = gpool[R_WORDS];
  for (int i = threadIdx.x; i < words; i += blockDim.x) sp[i] = gpool[i];
  __syncthreads();
}

__global__ void __launch_bounds__(128) k_stage(const int *__restrict__ gpool,
                                               const unsigned long long *__restrict__ cnt,
                                               const long long *__restrict__ off, int n_r,
                                               unsigned long long r0, long long W, int cap,
                                               unsigned char *__restrict__ assign,
                                               unsigned char *__restrict__ gate, int *act,
                                               int *n_act) {
  extern __shared__ int sp[];
  load_pool(sp, gpool);
  const int K = sp[R_K], D = sp[R_D];
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long wi = (long long)blockIdx.x * blockDim.x + threadIdx.x; wi < W; wi += stride) {
    unsigned char a[TSL_MAX_STAGES];
    bool pass = rep_unrank(sp, cnt, off, n_r, r0 + (unsigned long long)wi, a);
    if (pass && cap >= 0) {
      // entry memory e_d = sum n_st * m_st over stages on d (repetend.py:93-100)
      for (int d = 0; d < D && pass; ++d) {
        int e = 0;
        for (int p = at_ptr(sp, R_DEVPTR, d); p < at_ptr(sp, R_DEVPTR, d + 1); ++p) {
          const int st = sp[sp[R_DEVITEMS] + p];
          e += (int)a[st] * sp[sp[R_MEM] + st];
        }
        if (e > cap) pass = false;
      }
    }
    unsigned char *dst = assign + wi * K;
    for (int st = 0; st < K; ++st) dst[st] = a[st];
    gate[wi] = pass ? 1 : 0;
    if (pass) act[atomicAdd(n_act, 1)] = (int)wi;
  }
}

// Per-thread scratch of the repetend kernels: RX-DFS or DJ workspace (they
// run one after the other), then dependency-row lags and entry memory.
__host__ __device__ inline long long rep_ws_words(const int *pool) {
  const long long rx = rx_ws_words(pool[R_K], pool[R_MAXDI]);
  const long long dj = dj_ws_words(pool[R_K], pool[R_D], pool[R_NPAIR], pool[R_MAXDI]);
  long long w = (rx > dj ? rx : dj) + (pool[R_NDEP] > 0 ? pool[R_NDEP] : 1) + pool[R_D];
  return (w + 31) / 32 * 32;
}

struct ProbeOut {
  int *act_out, *def_out, *sat_widx, *sat_starts;
  int *counters;  // [0] active, [1] sat, [2] deferred
  unsigned long long *stats;  // probes, root_refuted, nodes, capped, sat, deferred, dj_unsat, dj_nodes
};

__device__ __forceinline__ void emit_sat(const ProbeOut &o, int widx, const int *s, int K) {
  const int k = atomicAdd(&o.counters[1], 1);
  o.sat_widx[k] = widx;
  for (int i = 0; i < K; ++i) o.sat_starts[(long long)k * K + i] = s[i];
}

// K2a root filter, one warp per (candidate, P).  The reference's root step
// (kernel_c.pyx:158-215) is FIFO bound propagation over the difference edges,
// then _mem_ok / _dev_ok on every device; any failure is UNSAT with 0 nodes.
// Its verdict does not depend on the propagation order: the propagation
// reaches the unique greatest bounds-consistent box or fails iff that box is
// empty.  Here the fixpoint is computed lane-parallel
// (lanes over edge rows, atomicMax / atomicMin on shared bounds, rounds until
// no lane changes a bound).  Without a positive cycle every bound settles
// within K-1 rounds (longest simple path), so a change in round K+1 proves a
// positive cycle, i.e. the propagation would push some lo above its hi.
// At the root no item is placed, so _mem_ok's events are only negative
// deltas and it reduces to init_d <= cap; _dev_ok runs the warp rank-based
// check (wrx_dfs.cuh) per device.  Refuted probes stay active; survivors go
// to k_probe's reference-exact DFS.
__host__ __device__ inline int root_warp_words(const int *pool) {
  const int K = pool[R_K];
  const int nmemb = pool[pool[R_DEVPTR] + pool[R_D]];  // device memberships
  return ((wrx_state_words(K, pool[R_MAXDI]) + 3) & ~3) + ((K + 3) & ~3) +
         3 * ((nmemb + 3) & ~3);
}

// Root _dev_ok of every device at once (nothing placed: release a = lo,
// deadline e = hi + dur), one lane per device membership p (dev_items order)
// instead of one device after another: for p's device, the suffix (>= p in
// the stable release order (a, p)) and prefix (<= p in the stable deadline
// order (e, a, p)) sums of kernel_c.pyx:470-508 and the serial-completion
// bound max(sum d, a + suffix d) <= max e.  ea / ee / ed: per-membership
// scratch (3 x nmemb words).  ROOT_MEMB_CHUNKS x 32 memberships at most.
#define ROOT_MEMB_CHUNKS 4
#define ROOT_ROWS 9  // edge rows per lane held in registers by k_root (m <= 288)
__device__ __forceinline__ bool root_devs_ok(const int *sp, const WWs &w, int *ea, int *ee,
                                             int *ed, int nmemb, const int (&q0)[ROOT_MEMB_CHUNKS],
                                             const int (&q1)[ROOT_MEMB_CHUNKS]) {
  const int lane = threadIdx.x & 31;
  const int *items = sp + sp[R_DEVITEMS], *dur = sp + sp[R_DUR];
  for (int p = lane; p < nmemb; p += 32) {
    const int it = items[p], du = dur[it];
    ea[p] = w.lo[it];
    ee[p] = w.hi[it] + du;
    ed[p] = du;
  }
  __syncwarp();
  bool bad = false;
#pragma unroll
  for (int c = 0; c < ROOT_MEMB_CHUNKS; ++c) {
    const int p = 32 * c + lane;
    if (32 * c >= nmemb) break;
    if (p < nmemb) {
      const int ai = ea[p], ei = ee[p];
      int suf_d = 0, suf_e = -(1 << 30), pre_d = 0, pre_a = 1 << 30, lim = -(1 << 30), sd = 0;
      for (int q = q0[c]; q < q1[c]; ++q) {
        const int aj = ea[q], ej = ee[q], dj = ed[q];
        lim = ej > lim ? ej : lim;
        sd += dj;
        const bool ge = aj > ai || (aj == ai && q >= p);
        if (ge) {
          suf_d += dj;
          suf_e = ej > suf_e ? ej : suf_e;
        }
        if (ej < ei || (ej == ei && !(ge && q != p))) {
          pre_d += dj;
          pre_a = aj < pre_a ? aj : pre_a;
        }
      }
      bad |= ai + suf_d > suf_e || pre_a + pre_d > ei || ai + suf_d > lim || sd > lim;
    }
  }
  const bool ok = !__any_sync(WRX_FULL, bad);
  __syncwarp();
  return ok;
}

__global__ void __launch_bounds__(256, 3) k_root(const int *__restrict__ gpool,
                                              const unsigned char *__restrict__ assign,
                                              const int *__restrict__ act_in, int n_in,
                                              ProbeOut o, int *__restrict__ surv, int P, int cap,
                                              long long widx_limit, int devs_serial) {
  extern __shared__ int sp[];
  load_pool(sp, gpool);
  const int K = sp[R_K], D = sp[R_D], m = sp[R_M], ndep = sp[R_NDEP];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  int *mine = sp + ((sp[R_WORDS] + 3) & ~3) + wib * root_warp_words(sp);
  int *av = mine + ((wrx_state_words(K, sp[R_MAXDI]) + 3) & ~3);
  const int nmemb = sp[sp[R_DEVPTR] + D];
  int *ea = av + ((K + 3) & ~3), *ee = ea + ((nmemb + 3) & ~3), *ed = ee + ((nmemb + 3) & ~3);
  WWs w = wrx_carve(mine, nullptr, K, sp[R_MAXDI]);
  const int nw = (K + 31) / 32;
  for (int i = lane; i < nw; i += 32) w.placed[i] = 0u;
  // this lane's memberships: their device's range in dev_items
  const bool batched = nmemb <= 32 * ROOT_MEMB_CHUNKS && !devs_serial;
  int q0[ROOT_MEMB_CHUNKS], q1[ROOT_MEMB_CHUNKS];
#pragma unroll
  for (int c = 0; c < ROOT_MEMB_CHUNKS; ++c) {
    const int p = 32 * c + lane;
    q0[c] = q1[c] = 0;
    if (batched && p < nmemb)
      for (int d = 0; d < D; ++d)
        if (at_ptr(sp, R_DEVPTR, d) <= p && p < at_ptr(sp, R_DEVPTR, d + 1)) {
          q0[c] = at_ptr(sp, R_DEVPTR, d);
          q1[c] = at_ptr(sp, R_DEVPTR, d + 1);
        }
  }
  const int *rsrc = sp + sp[R_RSRC], *rdst = sp + sp[R_RDST], *rbase = sp + sp[R_RBASE];
  const int anchor = (K - 1) * (P + sp[R_MAXDUR]);
  const RepView v = rep_view(sp, P, cap, nullptr, nullptr);
  // Register rows: lane l relaxes the contiguous block [l * per, l * per +
  // per) of the m edge rows, lo forward and hi backward through the block
  // (consecutive rows of a stage chain advance several hops per round
  // instead of one); endpoints kept in registers, lags per probe.
  const int per = (m + 31) / 32;
  const bool regrows = per <= ROOT_ROWS && !devs_serial;
  int rsd[ROOT_ROWS], rl[ROOT_ROWS];  // rsd: src | dst << 16 (-1: no row)
#pragma unroll
  for (int i = 0; i < ROOT_ROWS; ++i) {
    const int r = lane * per + i;
    const bool on = regrows && i < per && r < m;
    rsd[i] = on ? (rsrc[r] | (rdst[r] << 16)) : -1;
    rl[i] = 0;
  }
  unsigned long long s_probe = 0, s_root = 0;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + wib; t < n_in; t += nwarps) {
    const int widx = act_in[t];
    if (widx > widx_limit) continue;  // retired by a lower-index completion-feasible SAT
    const unsigned char *a = assign + (long long)widx * K;
    for (int i = lane; i < K; i += 32) {
      av[i] = a[i];
      w.lo[i] = i == 0 ? anchor : 0;
      w.hi[i] = i == 0 ? anchor : 2 * anchor;
    }
    __syncwarp();
    bool fail = false;
    if (cap >= 0) {  // root _mem_ok: init_d <= cap (entry memory, repetend.py:93-100)
      bool bad = false;
      for (int d = lane; d < D; d += 32) {
        int e = 0;
        for (int p = at_ptr(sp, R_DEVPTR, d); p < at_ptr(sp, R_DEVPTR, d + 1); ++p) {
          const int st = sp[sp[R_DEVITEMS] + p];
          e += av[st] * sp[sp[R_MEM] + st];
        }
        bad |= e > cap;
      }
      fail = __any_sync(WRX_FULL, bad);
    }
    if (regrows && !fail) {
#pragma unroll
      for (int i = 0; i < ROOT_ROWS; ++i) {
        const int r = lane * per + i;
        if (rsd[i] >= 0)
          rl[i] = rbase[r] - (r < ndep ? av[rsd[i] & 0xffff] - av[rsd[i] >> 16] : 1) * P;
      }
      for (int round = 0;; ++round) {
        bool changed = false, bad = false;
#pragma unroll
        for (int i = 0; i < ROOT_ROWS; ++i) {
          if (rsd[i] < 0) continue;
          const int sr = rsd[i] & 0xffff, ds = rsd[i] >> 16;
          const int nl = w.lo[sr] + rl[i];
          if (nl > w.lo[ds]) {
            atomicMax(&w.lo[ds], nl);
            changed = true;
            bad |= nl > w.hi[ds];
          }
        }
#pragma unroll
        for (int i = ROOT_ROWS - 1; i >= 0; --i) {
          if (rsd[i] < 0) continue;
          const int sr = rsd[i] & 0xffff, ds = rsd[i] >> 16;
          const int nh = w.hi[ds] - rl[i];
          if (nh < w.hi[sr]) {
            atomicMin(&w.hi[sr], nh);
            changed = true;
            bad |= nh < w.lo[sr];
          }
        }
        __syncwarp();
        if (__any_sync(WRX_FULL, bad)) {
          fail = true;
          break;
        }
        if (!__any_sync(WRX_FULL, changed)) {  // fixpoint: any crossing left over?
          for (int i = lane; i < K; i += 32) bad |= w.lo[i] > w.hi[i];
          fail = __any_sync(WRX_FULL, bad);
          break;
        }
        if (round >= K) {  // still moving after K+1 rounds: positive cycle
          fail = true;
          break;
        }
      }
    }
    for (int round = 0; !fail && !regrows; ++round) {
      bool changed = false;
      for (int r = lane; r < m; r += 32) {
        const int s = rsrc[r], d = rdst[r];
        const int lag = rbase[r] - (r < ndep ? av[s] - av[d] : 1) * P;
        const int nl = w.lo[s] + lag;
        if (nl > w.lo[d]) {
          atomicMax(&w.lo[d], nl);
          changed = true;
        }
        const int nh = w.hi[d] - lag;
        if (nh < w.hi[s]) {
          atomicMin(&w.hi[s], nh);
          changed = true;
        }
      }
      __syncwarp();
      bool bad = false;
      for (int i = lane; i < K; i += 32) bad |= w.lo[i] > w.hi[i];
      if (__any_sync(WRX_FULL, bad)) fail = true;
      else if (!__any_sync(WRX_FULL, changed)) break;
      else if (round >= K) fail = true;  // still moving after K+1 rounds: positive cycle
    }
    if (!fail) {
      if (batched) fail = !root_devs_ok(sp, w, ea, ee, ed, nmemb, q0, q1);
      else
        for (int d = 0; d < D && !fail; ++d) fail = !wrx_dev_ok(v, w, d);
    }
    ++s_probe;
    if (lane == 0) {
      if (fail) o.act_out[atomicAdd(&o.counters[0], 1)] = widx;
      else surv[atomicAdd(&o.counters[3], 1)] = widx;
    }
    s_root += fail;
    __syncwarp();
  }
  if (lane == 0 && s_probe) {
    atomicAdd(&o.stats[0], s_probe);
    atomicAdd(&o.stats[1], s_root);
  }
}

// K2 level pass: probe (candidate, P) with a small node budget first.
// Outcomes: SAT (exact: found within the small budget <= the reference cap),
// UNSAT / TIMEOUT at the reference cap (exact "not SAT"), or DEFERRED (small
// budget exhausted below the reference cap; settled by k_resolve only if the
// candidate is still below the level's retirement limit).
__global__ void __launch_bounds__(128) k_probe(const int *__restrict__ gpool,
                                               const unsigned char *__restrict__ assign,
                                               const int *__restrict__ act_in, int n_in,
                                               const int *__restrict__ n_in_dev,
                                               ProbeOut o, int P, long long full_budget,
                                               long long small_budget, int cap,
                                               long long widx_limit,
                                               unsigned long long budget_ns, int *ws_base,
                                               long long ws_words) {
  extern __shared__ int sp[];
  // n_in_dev: survivors of k_root (already counted as probes there)
  const bool counted = n_in_dev != nullptr;
  if (counted) n_in = *n_in_dev;
  if ((long long)blockIdx.x * blockDim.x >= n_in) return;
  load_pool(sp, gpool);
  const int K = sp[R_K];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int *mine = ws_base + tid * ws_words;
  RxWs w = rx_ws_carve(mine, K, sp[R_MAXDI]);
  int *deplag = mine + (ws_words - (sp[R_NDEP] > 0 ? sp[R_NDEP] : 1) - sp[R_D]);
  int *init = deplag + (sp[R_NDEP] > 0 ? sp[R_NDEP] : 1);
  // a probe is deferred only when the small budget is strictly below the cap
  const long long first_budget =
      (full_budget == 0 || small_budget < full_budget) ? small_budget : full_budget;
  unsigned long long s_probe = 0, s_root = 0, s_nodes = 0, s_cap = 0, s_sat = 0, s_def = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = tid; t < n_in; t += stride) {
    const int widx = act_in[t];
    if (widx > widx_limit) continue;  // retired by a lower-index completion-feasible SAT
    const unsigned char *a = assign + (long long)widx * K;
    rep_prepare(sp, a, P, deplag, init, w.lo, w.hi);
    const RepView v = rep_view(sp, P, cap, deplag, init);
    const unsigned long long t_end = budget_ns ? rx_now_ns() + budget_ns : 0ull;
    long long nd = 0;
    const int st = rx_decide(v, w, first_budget, t_end, &nd);
    ++s_probe;
    if (st == RX_SAT) {
      s_nodes += (unsigned long long)nd;
      ++s_sat;
      emit_sat(o, widx, w.s, K);
    } else if (st == RX_TIMEOUT && first_budget != full_budget) {
      ++s_def;  // node count settled in k_resolve
      o.def_out[atomicAdd(&o.counters[2], 1)] = widx;
    } else {
      s_nodes += (unsigned long long)nd;
      if (st == RX_TIMEOUT) ++s_cap;
      else if (nd == 0) ++s_root;
      o.act_out[atomicAdd(&o.counters[0], 1)] = widx;
    }
  }
  if (s_probe) {
    if (!counted) atomicAdd(&o.stats[0], s_probe);
    atomicAdd(&o.stats[1], s_root);
    atomicAdd(&o.stats[2], s_nodes);
    atomicAdd(&o.stats[3], s_cap);
    atomicAdd(&o.stats[4], s_sat);
    atomicAdd(&o.stats[5], s_def);
  }
}

// K2 resolution of deferred probes, in escalating stages so that a probe
// above the level's retirement limit never burns the full reference cap:
// the complete disjunctive solver first (an infeasibility proof settles the
// probe as "not SAT", which is what the reference concludes from either its
// UNSAT or its node-capped TIMEOUT); otherwise the reference-exact RX-DFS
// with this stage's budget.  Probes exhausting a stage budget below the
// reference cap are deferred again (def_out) for the next stage.
__global__ void __launch_bounds__(128) k_resolve(const int *__restrict__ gpool,
                                                 const unsigned char *__restrict__ assign,
                                                 const int *__restrict__ def_in, int n_def,
                                                 ProbeOut o, int P, long long full_budget,
                                                 long long stage_budget, long long dj_budget,
                                                 int cap,
                                                 long long widx_limit,
                                                 unsigned long long budget_ns, int *ws_base,
                                                 long long ws_words) {
  extern __shared__ int sp[];
  load_pool(sp, gpool);
  const int K = sp[R_K];
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  int *mine = ws_base + tid * ws_words;
  RxWs w = rx_ws_carve(mine, K, sp[R_MAXDI]);
  DjWs dw = dj_ws_carve(mine, K, sp[R_D], sp[R_NPAIR], sp[R_MAXDI]);
  int *deplag = mine + (ws_words - (sp[R_NDEP] > 0 ? sp[R_NDEP] : 1) - sp[R_D]);
  int *init = deplag + (sp[R_NDEP] > 0 ? sp[R_NDEP] : 1);
  unsigned long long s_nodes = 0, s_cap = 0, s_sat = 0, s_dju = 0, s_djn = 0, s_def = 0;
  const bool partial = stage_budget > 0 && (full_budget == 0 || stage_budget < full_budget);
  const long long rx_budget = partial ? stage_budget : full_budget;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long t = tid; t < n_def; t += stride) {
    const int widx = def_in[t];
    if (widx > widx_limit) continue;  // retired meanwhile: never needed
    const unsigned char *a = assign + (long long)widx * K;
    const unsigned long long t_end = budget_ns ? rx_now_ns() + budget_ns : 0ull;
    rep_prepare(sp, a, P, deplag, init, dw.lo, dw.hi);
    const RepView v = rep_view(sp, P, cap, deplag, init);
    long long dn = 0;
    const int dj = dj_budget > 0 ? dj_decide(v, sp, dw, dj_budget, &dn) : DJ_UNKNOWN;
    s_djn += (unsigned long long)dn;
    if (dj == DJ_UNSAT) {
      ++s_dju;
      o.act_out[atomicAdd(&o.counters[0], 1)] = widx;
      continue;
    }
    if (stage_budget < 0) {  // disjunctive filter only: undecided probes stay deferred
      ++s_def;
      o.def_out[atomicAdd(&o.counters[2], 1)] = widx;
      continue;
    }
    rep_prepare(sp, a, P, deplag, init, w.lo, w.hi);
    long long nd = 0;
    const int st = rx_decide(v, w, rx_budget, t_end, &nd);
    if (st == RX_SAT) {
      s_nodes += (unsigned long long)nd;
      ++s_sat;
      emit_sat(o, widx, w.s, K);
    } else if (st == RX_TIMEOUT && partial) {
      ++s_def;
      o.def_out[atomicAdd(&o.counters[2], 1)] = widx;
    } else {
      s_nodes += (unsigned long long)nd;
      if (st == RX_TIMEOUT) ++s_cap;
      o.act_out[atomicAdd(&o.counters[0], 1)] = widx;
    }
  }
  atomicAdd(&o.stats[5], s_def);
  atomicAdd(&o.stats[2], s_nodes);
  atomicAdd(&o.stats[3], s_cap);
  atomicAdd(&o.stats[4], s_sat);
  atomicAdd(&o.stats[6], s_dju);
  atomicAdd(&o.stats[7], s_djn);
}

// Warp-per-probe resolution stage (same contract as k_resolve): DJ on lane
// 0, then the warp-cooperative reference-exact DFS.  Shared memory per warp:
// WRX state + snapshots + dependency lags + entry memory.
__host__ __device__ inline int rep_warp_smem_words(const int *pool) {
  const int K = pool[R_K];
  const int wrx = ((wrx_state_words(K, pool[R_MAXDI]) + 3) & ~3) + (int)wrx_snap_words(K) +
                  (pool[R_NDEP] > 0 ? pool[R_NDEP] : 1) + pool[R_D] + 2;
  const int wrr = wrr_smem_words(K, pool[R_D]);
  return wrx > wrr ? wrx : wrr;
}

// Reference-exact decide of one repetend probe by the warp: the
// register-resident DFS (wrr_dfs.cuh) when the placement fits it, else the
// shared-memory warp DFS (wrx_dfs.cuh).  The per-warp area `mine_s` holds
// either layout; on SAT the witness is in w.s.
// `full_budget` is the reference's cap for the probe (0 = none, at the load
// bound); `budget` the node budget of this run (a resolve stage may run
// below the cap).  With the strong search (wst_dfs.cuh) first, only a SAT
// found within the cap of a capped probe needs the exact count.
__device__ __forceinline__ int rep_decide_warp(const int *sp, const unsigned char *a, int P,
                                               int cap, int *mine_s, WWs &w, int *deplag,
                                               int *init, long long budget,
                                               unsigned long long t_end, long long *nd,
                                               const int *lim, int widx,
                                               long long full_budget) {
  const int K = sp[R_K];
  if (sp[R_WRR]) {
    unsigned *snap = (unsigned *)mine_s;
    int *vstack = mine_s + (K + 1) * 32 * (K > 32 ? 2 : 1);
    int *winit = vstack + K + 1;
    long long n1 = 0;
    if (sp[R_WST]) {
      const int st = K > 32 ? wst_decide<2>(sp, a, P, cap, snap, vstack, winit, budget, t_end,
                                            &n1, lim, widx, w.s)
                            : wst_decide<1>(sp, a, P, cap, snap, vstack, winit, budget, t_end,
                                            &n1, lim, widx, w.s);
      if (st != RX_SAT || full_budget == 0) {
        *nd = n1;
        return st;
      }
    }
    const int st = K > 32 ? wrr_decide<2>(sp, a, P, cap, snap, vstack, winit, budget, t_end,
                                          nd, lim, widx, w.s)
                          : wrr_decide<1>(sp, a, P, cap, snap, vstack, winit, budget, t_end,
                                          nd, lim, widx, w.s);
    *nd += n1;
    return st;
  }
  if ((threadIdx.x & 31) == 0) rep_prepare(sp, a, P, deplag, init, w.lo, w.hi);
  __syncwarp();
  const RepView v = rep_view(sp, P, cap, deplag, init);
  return wrx_decide(v, w, budget, t_end, nd, lim, widx);
}

__global__ void __launch_bounds__(128, RESOLVE_MIN_BLOCKS) k_resolve_warp(const int *__restrict__ gpool,
                                                      const unsigned char *__restrict__ assign,
                                                      const int *__restrict__ def_in, int n_def,
                                                      const int *__restrict__ n_def_dev,
                                                      ProbeOut o, int P, long long full_budget,
                                                      long long stage_budget,
                                                      long long dj_budget, int cap,
                                                      long long widx_limit,
                                                      unsigned long long budget_ns,
                                                      int *ws_base, long long ws_words,
                                                      int *dev_limit, int dj_warp,
                                                      int *work) {
  extern __shared__ int sp[];
  // n_def_dev: device-side count (k_root survivors; probes counted there)
  if (n_def_dev) n_def = *n_def_dev;
  if ((long long)blockIdx.x * (blockDim.x >> 5) >= n_def) return;
  load_pool(sp, gpool);
  const int K = sp[R_K];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int per_warp = rep_warp_smem_words(sp);
  int *mine_s = sp + ((sp[R_WORDS] + 3) & ~3) + wib * ((per_warp + 3) & ~3);
  const int ndep1 = sp[R_NDEP] > 0 ? sp[R_NDEP] : 1;
  int *snap = mine_s + ((wrx_state_words(K, sp[R_MAXDI]) + 3) & ~3);  // int2-aligned
  int *deplag = snap + (int)wrx_snap_words(K);
  int *init = deplag + ndep1;
  WWs w = wrx_carve(mine_s, snap, K, sp[R_MAXDI]);
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  int *mine_g = ws_base + gw * ws_words;  // lane-0 DJ workspace
  DjWs dw = dj_ws_carve(mine_g, K, sp[R_D], sp[R_NPAIR], sp[R_MAXDI]);
  const bool partial = stage_budget > 0 && (full_budget == 0 || stage_budget < full_budget);
  const long long rx_budget = partial ? stage_budget : full_budget;
  unsigned long long s_nodes = 0, s_cap = 0, s_sat = 0, s_dju = 0, s_djn = 0, s_def = 0;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  // dev_limit: speculative retirement limit of this launch — every SAT lowers
  // it to its index - 1 (assuming its completion check passes); probes above
  // it stop early and go back to the deferred list, so the host re-runs them
  // only if that SAT does not retire them (engine.py).
  auto spec_retired = [&](int widx) {
    int l = 0;
    if (lane == 0) l = dev_limit ? *(volatile int *)dev_limit : (int)0x7fffffff;
    l = __shfl_sync(WRX_FULL, l, 0);
    return widx > l;
  };
  auto defer = [&](int widx) {
    if (lane == 0) {
      ++s_def;
      o.def_out[atomicAdd(&o.counters[2], 1)] = widx;
    }
    __syncwarp();
  };
  // work: the launch's probe counter — each warp takes the next probe when it
  // is done with one (probe costs are heavy-tailed: a static stride leaves
  // most warps idle behind a few long ones); nullptr = static stride
  long long t_static = gw - nwarps;
  auto next = [&]() -> long long {
    if (!work) return t_static += nwarps;
    int v = 0;
    if (lane == 0) v = atomicAdd(work, 1);
    return (long long)__shfl_sync(WRX_FULL, v, 0);
  };
  for (long long t = next(); t < n_def; t = next()) {
    const int widx = def_in[t];
    if (widx > widx_limit) continue;
    if (spec_retired(widx)) {
      defer(widx);
      continue;
    }
    const unsigned char *a = assign + (long long)widx * K;
    const unsigned long long t_end = budget_ns ? rx_now_ns() + budget_ns : 0ull;
    int dj = DJ_UNKNOWN;
    if (dj_budget > 0 && dj_warp) {
      // warp disjunctive filter: shared state carved from the (not yet used)
      // RX snapshot area, per-depth snapshots in this warp's global slice
      WdjWs dw2 = wdj_carve(snap, ws_base + gw * 32 * ws_words, K, sp[R_NPAIR]);
      if (lane == 0) rep_prepare(sp, a, P, deplag, init, dw2.lo, dw2.hi);
      for (int i = lane; i < K; i += 32) dw2.av[i] = a[i];
      __syncwarp();
      long long dn = 0;
      dj = wdj_decide(sp, P, cap, init, dw2, dj_budget, &dn);
      if (lane == 0) s_djn += (unsigned long long)dn;
    } else if (dj_budget > 0) {
      if (lane == 0) {
        rep_prepare(sp, a, P, deplag, init, dw.lo, dw.hi);
        const RepView v = rep_view(sp, P, cap, deplag, init);
        long long dn = 0;
        dj = dj_decide(v, sp, dw, dj_budget, &dn);
        s_djn += (unsigned long long)dn;
      }
      dj = __shfl_sync(WRX_FULL, dj, 0);
    }
    if (dj == DJ_UNSAT) {
      if (lane == 0) {
        ++s_dju;
        o.act_out[atomicAdd(&o.counters[0], 1)] = widx;
      }
      continue;
    }
    if (stage_budget < 0 || spec_retired(widx)) {  // filter only / retired meanwhile
      defer(widx);
      continue;
    }
    long long nd = 0;
    const int st = rep_decide_warp(sp, a, P, cap, mine_s, w, deplag, init, rx_budget, t_end, &nd,
                                   dev_limit, widx, full_budget);
    if (st == RX_SAT) {
      int k = 0;
      if (lane == 0) {
        k = atomicAdd(&o.counters[1], 1);
        if (dev_limit) atomicMin(dev_limit, widx - 1);
      }
      k = __shfl_sync(WRX_FULL, k, 0);
      if (lane == 0) o.sat_widx[k] = widx;
      for (int i = lane; i < K; i += 32) o.sat_starts[(long long)k * K + i] = w.s[i];
      if (lane == 0) {
        s_nodes += (unsigned long long)nd;
        ++s_sat;
      }
    } else if (st == RX_ABORT) {
      defer(widx);
      continue;
    } else if (lane == 0) {
      if (st == RX_TIMEOUT && partial) {
        ++s_def;
        o.def_out[atomicAdd(&o.counters[2], 1)] = widx;
      } else {
        s_nodes += (unsigned long long)nd;
        if (st == RX_TIMEOUT) ++s_cap;
        o.act_out[atomicAdd(&o.counters[0], 1)] = widx;
      }
    }
    __syncwarp();
  }
  if (lane == 0) {
    atomicAdd(&o.stats[5], s_def);
    atomicAdd(&o.stats[2], s_nodes);
    atomicAdd(&o.stats[3], s_cap);
    atomicAdd(&o.stats[4], s_sat);
    atomicAdd(&o.stats[6], s_dju);
    atomicAdd(&o.stats[7], s_djn);
  }
}

// Disjunctive filter alone (wdj_solve.cuh), one warp per deferred probe with
// a small shared footprint so many warps hide its latency: refuted probes
// stay active (exactly "not SAT", see k_resolve); the others go to `keep`
// (count in o.counters[3]) for the reference-exact DFS stage.  Probes above
// the speculative limit (a SAT found meanwhile) are kept too.
__host__ __device__ inline int dj_warp_words(const int *pool) {
  const int ndep1 = pool[R_NDEP] > 0 ? pool[R_NDEP] : 1;
  return (wdj_smem_words(pool[R_K], pool[R_NPAIR]) + ndep1 + pool[R_D] + 3) & ~3;
}

#ifndef DJ_FILTER_MINB
#define DJ_FILTER_MINB 4
#endif
__global__ void __launch_bounds__(256, DJ_FILTER_MINB) k_dj_filter(const int *__restrict__ gpool,
                                                   const unsigned char *__restrict__ assign,
                                                   const int *__restrict__ def_in, int n_def,
                                                   ProbeOut o, int *__restrict__ keep, int P,
                                                   long long dj_budget, int cap,
                                                   long long widx_limit, int *gscratch,
                                                   long long gwords, const int *dev_limit,
                                                   int *next) {
  extern __shared__ int sp[];
  load_pool(sp, gpool);
  const int K = sp[R_K];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int ndep1 = sp[R_NDEP] > 0 ? sp[R_NDEP] : 1;
  int *mine = sp + ((sp[R_WORDS] + 3) & ~3) + wib * dj_warp_words(sp);
  int *deplag = mine + wdj_smem_words(K, sp[R_NPAIR]);
  int *init = deplag + ndep1;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  WdjWs w = wdj_carve(mine, gscratch + gw * gwords, K, sp[R_NPAIR]);
  unsigned long long s_dju = 0, s_djn = 0;
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  // probes handed out through a launch counter (heavy-tailed filter costs),
  // or a static grid stride without one
  for (long long t = gw;; t += nwarps) {
    if (next) {
      int tt = 0;
      if (lane == 0) tt = atomicAdd(next, 1);
      t = __shfl_sync(WRX_FULL, tt, 0);
    }
    if (t >= n_def) break;
    const int widx = def_in[t];
    if (widx > widx_limit) continue;
    int l = 0;
    if (lane == 0) l = dev_limit ? *(volatile const int *)dev_limit : 0x7fffffff;
    l = __shfl_sync(WRX_FULL, l, 0);
    int dj = DJ_UNKNOWN;
    if (widx <= l) {
      const unsigned char *a = assign + (long long)widx * K;
      if (lane == 0) rep_prepare(sp, a, P, deplag, init, w.lo, w.hi);
      for (int i = lane; i < K; i += 32) w.av[i] = a[i];
      __syncwarp();
      long long dn = 0;
      dj = wdj_decide(sp, P, cap, init, w, dj_budget, &dn);
      s_djn += (unsigned long long)dn;
    }
    if (lane == 0) {
      if (dj == DJ_UNSAT) {
        ++s_dju;
        o.act_out[atomicAdd(&o.counters[0], 1)] = widx;
      } else {
        keep[atomicAdd(&o.counters[3], 1)] = widx;
      }
    }
    __syncwarp();
  }
  if (lane == 0 && (s_dju || s_djn)) {
    atomicAdd(&o.stats[6], s_dju);
    atomicAdd(&o.stats[7], s_djn);
  }
}

// Verification of speculated probes: explicit (window index, period)
// pairs, one warp each, reference-exact DFS under the reference cap for that
// period (0 = none at the load bound).  Writes status / nodes / starts per
// pair (no list compaction: the host owns the bookkeeping).
__global__ void __launch_bounds__(128, 1) k_verify_warp(const int *__restrict__ gpool,
                                                     const unsigned char *__restrict__ assign,
                                                     const int *__restrict__ vwidx,
                                                     const int *__restrict__ vper,
                                                     const long long *__restrict__ vbudget,
                                                     int count, int cap, int *vstatus,
                                                     long long *vnodes, int *vstarts,
                                                     int *vlim, int pmin, int nlev,
                                                     const unsigned char *__restrict__ rows,
                                                     const int *__restrict__ vpos,
                                                     int cancel) {
  extern __shared__ int sp[];
  load_pool(sp, gpool);
  const int K = sp[R_K];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int per_warp = rep_warp_smem_words(sp);
  int *mine_s = sp + ((sp[R_WORDS] + 3) & ~3) + wib * ((per_warp + 3) & ~3);
  const int ndep1 = sp[R_NDEP] > 0 ? sp[R_NDEP] : 1;
  int *snap = mine_s + ((wrx_state_words(K, sp[R_MAXDI]) + 3) & ~3);
  int *deplag = snap + (int)wrx_snap_words(K);
  int *init = deplag + ndep1;
  WWs w = wrx_carve(mine_s, snap, K, sp[R_MAXDI]);
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long t = (long long)blockIdx.x * (blockDim.x >> 5) + wib; t < count; t += nwarps) {
    const int P = vper[t], widx = vwidx[t];
    // per-period speculative retirement: a SAT (w, P) retires (w2, P2) with
    // w2 > w and P2 >= P if its completion check passes (the host decides)
    // (cancel = 0: every probe of the launch is resident at once, so a
    // cancelled one would only be re-run later, on the critical path)
    int *lim = vlim + (P - pmin);
    int l = 0x7fffffff;
    if (cancel && lane == 0) l = *(volatile int *)lim;
    l = __shfl_sync(WRX_FULL, l, 0);
    if (widx > l) {
      if (lane == 0) {
        vstatus[t] = RX_ABORT;
        vnodes[t] = 0;
      }
      continue;
    }
    // rows: the window's assignments stashed privately (the staged window
    // may already hold the next one); else the staged window
    const unsigned char *a = rows ? rows + (long long)vpos[t] * K : assign + (long long)widx * K;
    long long nd = 0;
    const int st = rep_decide_warp(sp, a, P, cap, mine_s, w, deplag, init, vbudget[t], 0ull, &nd,
                                   cancel ? lim : nullptr, widx, vbudget[t]);
    if (lane == 0) {
      vstatus[t] = st;
      vnodes[t] = nd;
      if (st == RX_SAT)
        for (int q = P - pmin; q < nlev; ++q) atomicMin(&vlim[q], widx - 1);
    }
    if (st == RX_SAT)
      for (int i = lane; i < K; i += 32) vstarts[t * K + i] = w.s[i];
    __syncwarp();
  }
}

// Diagnostic: the disjunctive filter on explicit (assignment, period) pairs
// (tests check it never refutes a feasible probe).  mode 1 = warp filter
// (wdj_solve.cuh), 0 = one-lane filter (dj_solve.cuh).
__global__ void __launch_bounds__(128) k_dj_batch(const int *__restrict__ gpool,
                                                  const int *__restrict__ assign,
                                                  const int *__restrict__ per, int count, int cap,
                                                  long long budget, int mode, int *gscratch,
                                                  long long gwords, int *status,
                                                  long long *nodes) {
  extern __shared__ int sp[];
  load_pool(sp, gpool);
  const int K = sp[R_K], D = sp[R_D];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int ndep1 = sp[R_NDEP] > 0 ? sp[R_NDEP] : 1;
  const int per_warp = (wdj_smem_words(K, sp[R_NPAIR]) + ndep1 + D + 3) & ~3;
  int *mine = sp + ((sp[R_WORDS] + 3) & ~3) + wib * per_warp;
  int *deplag = mine + wdj_smem_words(K, sp[R_NPAIR]);
  int *init = deplag + ndep1;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  int *g = gscratch + gw * gwords;
  WdjWs w = wdj_carve(mine, g, K, sp[R_NPAIR]);
  DjWs dw = dj_ws_carve(g, K, D, sp[R_NPAIR], sp[R_MAXDI]);
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long t = gw; t < count; t += nwarps) {
    const int *a = assign + t * K;
    const int P = per[t];
    long long dn = 0;
    int st;
    if (mode == 1) {
      if (lane == 0) rep_prepare(sp, a, P, deplag, init, w.lo, w.hi);
      for (int i = lane; i < K; i += 32) w.av[i] = a[i];
      __syncwarp();
      st = wdj_decide(sp, P, cap, init, w, budget, &dn);
    } else {
      st = 0;
      if (lane == 0) {
        rep_prepare(sp, a, P, deplag, init, dw.lo, dw.hi);
        const RepView v = rep_view(sp, P, cap, deplag, init);
        st = dj_decide(v, sp, dw, budget, &dn);
      }
      st = __shfl_sync(WRX_FULL, st, 0);
    }
    if (lane == 0) {
      status[t] = st;
      nodes[t] = dn;
    }
    __syncwarp();
  }
}

__global__ void k_stash_rows(const unsigned char *__restrict__ assign,
                             const int *__restrict__ widx, int count, int K,
                             unsigned char *__restrict__ rows) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)count * K) return;
  rows[t] = assign[(long long)widx[t / K] * K + t % K];
}

__global__ void k_gather_rows(const int *__restrict__ rows, const int *__restrict__ pos, int count,
                              int K, int *__restrict__ out) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (long long)count * K) return;
  const int r = (int)(t / K), i = (int)(t % K);
  out[t] = rows[(long long)pos[r] * K + i];
}

// Ordered SAT walk (north_star kernel 3): the smallest window index above
// `after` among the level's SAT rows — a lexicographic (window index, row
// position) argmin by warp shuffles, a shared-memory pass over the warps and
// one 64-bit atomicMin per block — then its row fetched for the host.  The
// host replays SATs in window order up to the first completion-feasible one
// (completion.py:351-382), so typically one argmin per level crosses PCIe.
__global__ void __launch_bounds__(256) k_sat_min(const int *__restrict__ sat_widx, int n,
                                                 int after, unsigned long long *key) {
  unsigned long long best = ~0ull;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int w = sat_widx[i];
    if (w > after) {
      const unsigned long long k = ((unsigned long long)(unsigned)w << 32) | (unsigned)i;
      best = k < best ? k : best;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other < best ? other : best;
  }
  __shared__ unsigned long long wmin[8];
  if ((threadIdx.x & 31) == 0) wmin[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x < 32) {
    best = threadIdx.x < (blockDim.x >> 5) ? wmin[threadIdx.x] : ~0ull;
    for (int o = 4; o; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
      best = other < best ? other : best;
    }
    if (threadIdx.x == 0 && best != ~0ull) atomicMin(key, best);
  }
}

__global__ void k_sat_fetch(const unsigned long long *__restrict__ key,
                            const int *__restrict__ sat_starts, int K, int *out) {
  const unsigned long long k = *key;
  if (k == ~0ull) {
    if (threadIdx.x == 0) out[0] = -1;
    return;
  }
  const long long pos = (long long)(k & 0xffffffffu);
  if (threadIdx.x == 0) out[0] = (int)(k >> 32);
  for (int i = threadIdx.x; i < K; i += blockDim.x) out[1 + i] = sat_starts[pos * K + i];
}

// ------------------------------------------------------------------ SP-DFS
// Speculative subtree-parallel decide for one long general problem
// (sp_dfs.cuh): the master walk (one warp) and the subtree tasks (one warp
// each).  Shared per warp: the WRX state; snapshots in global memory.
__global__ void __launch_bounds__(32) k_sp_master(const int *__restrict__ pool, int *state,
                                                  int floor, int split, long long budget,
                                                  long long base_nodes, long long pause_nodes,
                                                  int *tasks, long long *pre, int max_tasks,
                                                  const unsigned *ovr, int n_ovr, int *hist,
                                                  long long *out, int k0, int *ck,
                                                  long long *ck_nodes, int ck_every, int ck_have,
                                                  long long ck_base) {
  extern __shared__ int sm[];
  const int lane = threadIdx.x & 31;
  const GenView g = gen_view(pool);
  const int n = g.n_;
  SpState st = sp_state_view(state, n);
  WWs w = wrx_carve(sm, (int *)st.snap, n, pool[G_MAXDI]);
  int depth = 0, v = 0, status = -1;
  long long nodes = 0;
  if (st.hdr[2]) {  // fresh: the reference root step
    for (int k = lane; k < n; k += 32) {
      w.lo[k] = g.lo_[k];
      w.hi[k] = g.hi_[k];
    }
    __syncwarp();
    if (!sp_root(g, w)) status = RX_UNSAT;
    else if (n == 0) status = RX_SAT;
    else v = w.lo[g.order(0)];
  } else {
    sp_load(w, st.lo, st.hi, st.s, st.placed, st.inq, n);
    for (int k = lane; k <= n; k += 32) w.vstack[k] = st.vstack[k];
    depth = st.hdr[0];
    v = st.hdr[1];
    __syncwarp();
  }
  SpSink sink{tasks, pre, k0, max_tasks, ovr, n_ovr, ck, ck_nodes, ck_every, ck_have, ck_base};
  if (status < 0)
    status = sp_explore(g, w, floor, split, depth, v, budget, base_nodes, &nodes,
                        split <= n ? &sink : nullptr, pause_nodes, hist);
  sp_store(w, st.lo, st.hi, st.s, st.placed, st.inq, n);
  for (int k = lane; k <= n; k += 32) st.vstack[k] = w.vstack[k];
  if (lane == 0) {
    st.hdr[0] = depth;
    st.hdr[1] = v;
    st.hdr[2] = 0;
    out[0] = status;
    out[1] = sink.count;
    out[2] = nodes;
  }
}

__global__ void __launch_bounds__(128) k_sp_tasks(const int *__restrict__ pool,
                                                  const int *__restrict__ tasks, int first,
                                                  int count, int split, long long budget,
                                                  int *snaps, int *results, int *info,
                                                  long long *part, const long long *pre,
                                                  long long cut_base, long long cut_budget,
                                                  SpDon dq) {
  extern __shared__ int sm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const GenView g = gen_view(pool);
  const int n = g.n_, nw = sp_nw(n);
  const int per_warp = (wrx_state_words(n, pool[G_MAXDI]) + 3) & ~3;
  const long long gw = (long long)blockIdx.x * (blockDim.x >> 5) + wib;
  WWs w = wrx_carve(sm + wib * per_warp, snaps + gw * 2LL * n * (n + 1), n, pool[G_MAXDI]);
  const long long nwarps = (long long)gridDim.x * (blockDim.x >> 5);
  if (!dq.ctl) {  // static: one warp per task
    for (long long t = first + gw; t < first + count; t += nwarps) {
      const int *rec = tasks + t * sp_task_words(n);
      sp_load(w, rec, rec + n, rec + 2 * n, (const unsigned *)(rec + 3 * n),
              (const unsigned *)(rec + 3 * n + nw), n);
      int v = rec[3 * n + 2 * nw], depth = rec[3 * n + 2 * nw + 1];
      long long nodes = 0;
      SpCut cut{part, pre, cut_base, cut_budget, (int)t, 0};
      const int st = sp_explore(g, w, depth, n + 1, depth, v, budget, 0, &nodes, nullptr, 0,
                                nullptr, cut_budget > 0 ? &cut : nullptr);
      if (lane == 0 && cut_budget > 0) ((volatile long long *)part)[t] = nodes;
      int *res = results + t * sp_result_words(n);
      bool moved = false;  // S_out != S_in: the master's speculation failed here
      for (int i = lane; i < nw; i += 32) moved |= w.inq[i] != (unsigned)rec[3 * n + nw + i];
      moved = __any_sync(WRX_FULL, moved);
      if (lane == 0) {
        res[0] = st;
        res[1] = (int)(nodes & 0xffffffffLL);
        res[2] = (int)(nodes >> 32);
        res[3] = moved ? 1 : 0;
        info[4 * t + 0] = st;
        info[4 * t + 1] = res[1];
        info[4 * t + 2] = res[2];
        info[4 * t + 3] = res[3];
      }
      for (int i = lane; i < nw; i += 32) res[4 + i] = (int)w.inq[i];
      if (st == RX_SAT)
        for (int i = lane; i < n; i += 32) res[4 + nw + i] = w.s[i];
      __syncwarp();
    }
    return;
  }
  // dynamic: claim slots (tasks first, then donated pieces) until every
  // piece of the launch is done (SpDon)
  for (;;) {
    int slot = 0;
    if (lane == 0) slot = (int)atomicAdd(&dq.ctl[0], 1u);
    slot = __shfl_sync(WRX_FULL, slot, 0);
    const int *rec;
    long long t;
    int parent = -1;
    if (slot < count) {
      t = first + slot;
      rec = tasks + t * sp_task_words(n);
    } else {
      const int p = slot - count;
      if (p >= dq.cap) break;
      int ok = 0;
      if (lane == 0) {
        for (;;) {
          if (((volatile int *)dq.pmeta)[4 * p + 3]) {
            ok = 1;
            break;
          }
          if (((volatile unsigned *)dq.ctl)[2] == 0u) break;
          __nanosleep(256);
        }
        __threadfence();
      }
      ok = __shfl_sync(WRX_FULL, ok, 0);
      if (!ok) break;
      rec = dq.precs + (long long)p * sp_task_words(n);
      t = ((volatile int *)dq.pmeta)[4 * p];
      parent = ((volatile int *)dq.pmeta)[4 * p + 1];
    }
    __syncwarp();
    sp_load_cg(w, rec, n);
    int v = __ldcg(rec + 3 * n + 2 * nw), depth = __ldcg(rec + 3 * n + 2 * nw + 1);
    long long nodes = 0;
    SpCut cut{part, pre, cut_base, cut_budget, (int)t, 0};
    SpDon d = dq;
    d.self = slot;
    d.parent = parent;
    d.slot_task = (int)(t - first);
    d.s_in = (const unsigned *)(rec + 3 * n + nw);  // this piece's own speculated set
    const int st = sp_explore(g, w, depth, n + 1, depth, v, budget, 0, &nodes, nullptr, 0,
                              nullptr, &cut, &d, (int)t);
    // the set the next piece in DFS order was started on: the latest
    // donation's (donations come right after the donor's own nodes), else
    // the one after this piece, speculated equal to this piece's S_in
    int lastd = -1;
    if (lane == 0) lastd = ((volatile int *)dq.plast)[slot];
    lastd = __shfl_sync(WRX_FULL, lastd, 0);
    const int *snext = lastd >= 0 ? dq.precs + (long long)(lastd - count) * sp_task_words(n) +
                                        3 * n + nw
                                  : (const int *)d.s_in;
    bool moved = false;  // S_out != that set: the DFS prefix the host can use ends here
    for (int i = lane; i < nw; i += 32) moved |= w.inq[i] != (unsigned)__ldcg(snext + i);
    moved = __any_sync(WRX_FULL, moved);
    if (lane == 0) {
      atomicAdd((unsigned long long *)&part[t], (unsigned long long)(nodes - cut.published));
      ((volatile long long *)dq.pnodes)[slot] = nodes;
      sp_publish_sub(d, nodes - cut.published);
      // the DFS prefix the host can use ends at this piece: every piece after
      // it stops (SP_INVALID) — its sticky set changed (an epoch follows),
      // or the probe is settled here (SAT, cap passed)
      if (moved || st == RX_SAT || st == RX_ABORT) sp_mark_moved(d);
    }
    // a task's own result goes to its task slot, a piece's to its piece slot
    int *res = slot < count ? results + t * sp_result_words(n)
                            : dq.pres + (long long)(slot - count) * sp_pres_words(n);
    const int wit_at = slot < count ? 4 + nw : 4;
    if (lane == 0) {
      res[0] = st;
      res[1] = (int)(nodes & 0xffffffffLL);
      res[2] = (int)(nodes >> 32);
      res[3] = moved ? 1 : 0;
      if (slot < count) {
        info[4 * t + 0] = st;
        info[4 * t + 1] = res[1];
        info[4 * t + 2] = res[2];
        info[4 * t + 3] = res[3];
      }
    }
    if (slot < count)
      for (int i = lane; i < nw; i += 32) res[4 + i] = (int)w.inq[i];
    else
      for (int i = lane; i < nw; i += 32) res[4 + n + i] = (int)w.inq[i];
    if (st == RX_SAT)
      for (int i = lane; i < n; i += 32) res[wit_at + i] = w.s[i];
    __syncwarp();
    if (lane == 0) {
      sp_task_piece_done(dq, (int)(t - first));
      __threadfence();
      atomicSub(&dq.ctl[2], 1u);
    }
  }
}

// Copy task records (scattered over the task and piece arrays) into a
// contiguous task array, with the sticky set replaced by S (sp_host.inc,
// SpRun::epochs).
__global__ void k_sp_gather(const unsigned long long *__restrict__ src, int count, int n,
                            const unsigned *__restrict__ S, int *dst) {
  const int tw = (int)sp_task_words(n), nw = sp_nw(n);
  for (int r = blockIdx.x; r < count; r += gridDim.x) {
    const int *a = (const int *)src[r];
    int *b = dst + (long long)r * tw;
    for (int i = threadIdx.x; i < tw; i += blockDim.x) {
      const int k = i - 3 * n - nw;  // the inq words
      b[i] = (k >= 0 && k < nw) ? (int)S[k] : a[i];
    }
  }
}

// ------------------------------------------------------------------ decide API

namespace {

struct DecideCtx {
  std::mutex mu;
  int device = -1;
  cudaStream_t stream = nullptr;
  char *buf = nullptr;
  size_t cap = 0;

  char *reserve(size_t bytes) {
    if (bytes > cap) {
      size_t want = std::max(bytes, cap * 2);
      dev_grow((void **)&buf, want, stream);
      cap = want;
    }
    return buf;
  }
};

DecideCtx &decide_ctx() {
  static DecideCtx ctx;
  return ctx;
}

cudaStream_t decide_ctx_stream() {
  static thread_local cudaStream_t s = nullptr;
  static thread_local int dev = -1;
  int d = 0;
  CK(cudaGetDevice(&d));
  if (!s || dev != d) {
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    dev = d;
  }
  return s;
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

#include "sp_host.inc"

// TSL_DFS_MODE=thread selects the one-thread-per-probe DFS kernels (kept for
// cross-validation); the default is the warp-cooperative DFS.
// TSL_ROOT_FILTER=0 disables k_root (every probe runs k_probe's thread DFS;
// kept for cross-validation).
bool root_filter_off() {
  const char *m = getenv("TSL_ROOT_FILTER");
  return m && std::string(m) == "0";
}

// TSL_DJ_MODE=lane selects the one-lane disjunctive filter (dj_solve.cuh);
// the default is the warp version (wdj_solve.cuh) when its shared state fits
// in the RX snapshot area and its snapshots in a warp's workspace slice.
bool dj_mode_warp(const int *pool) {
  const char *m = getenv("TSL_DJ_MODE");
  if (m && std::string(m) == "lane") return false;
  return wdj_smem_words(pool[R_K], pool[R_NPAIR]) <= wrx_snap_words(pool[R_K]) &&
         wdj_snap_words(pool[R_K], pool[R_NPAIR]) <= 32 * rep_ws_words(pool);
}

// TSL_DJ_SPLIT=1 runs the disjunctive filter as its own high-occupancy
// launch before the DFS stage.  Off by default: measured slower on C2@4/@8
// (the filter is not occupancy-bound, and the split serialises the DFS of a
// SAT probe behind the whole filter launch).
bool dj_split() {
  const char *m = getenv("TSL_DJ_SPLIT");
  return m && std::string(m) == "1";
}

// TSL_ROOT_DEVS=serial: k_root checks the devices one after another
// (wrx_dev_ok) instead of all memberships at once (cross-validation)
bool root_devs_serial() {
  const char *m = getenv("TSL_ROOT_DEVS");
  return m && std::string(m) == "serial";
}

// TSL_RESOLVE_DYN=0 restores the static grid stride of k_resolve_warp
// (default: probes handed out one at a time through a launch counter)
bool resolve_dynamic() {
  const char *m = getenv("TSL_RESOLVE_DYN");
  return !(m && std::string(m) == "0");
}

bool decide_mode_warp() {
  const char *m = getenv("TSL_DFS_MODE");
  return !(m && std::string(m) == "thread");
}

void run_decide_batch(int count, const tsl_problem *probs, double budget_secs, int32_t *status,
                      int64_t *nodes, int64_t *starts, int stride, bool allow_sp) {
  require_device();
  if (count <= 0) return;
  std::vector<int> pools;
  std::vector<long long> pool_off(count), ws_off(count), budgets(count);
  long long ws_total = 0;
  int max_n = 0, max_state = 0;
  const bool warp_mode = decide_mode_warp();
  for (int i = 0; i < count; ++i) {
    const tsl_problem &p = probs[i];
    std::vector<int> one = tsl::gen_build(p.n, p.dur, p.devmask, p.mem, p.edges, p.m, p.order,
                                          p.lo, p.hi, p.ndev, p.init_mem, p.cap);
    pool_off[i] = (long long)pools.size();
    pools.insert(pools.end(), one.begin(), one.end());
    ws_off[i] = ws_total;
    if (warp_mode) {
      ws_total += (wrx_snap_words(p.n) + 3) / 4 * 4;
      max_state = std::max(max_state, wrx_state_words(p.n, one[G_MAXDI]));
    } else {
      ws_total += (rx_ws_words(p.n, one[G_MAXDI]) + 3) / 4 * 4;
    }
    budgets[i] = p.node_budget < 0 ? 0 : p.node_budget;
    max_n = std::max(max_n, p.n);
  }
  // long problems: a first pass of TSL_SP_BATCH_FIRST nodes here; the ones still open
  // then run subtree-parallel (sp_solve) with their real cap
  // (the subtree-parallel workspace holds 2 n (n + 1) ints per task warp:
  // problems above SP_MAX_N stay one warp each)
  const bool sp = allow_sp && warp_mode && sp_enabled() && max_n <= SP_MAX_N;
  std::vector<long long> real_budget(budgets);
  // (short: the problems it leaves open restart with the subtree-parallel
  // decide's own sample, profiles/r01i_sp_first_sweep.log)
  const long long first = sp ? sp_env("TSL_SP_BATCH_FIRST", 1024) : 0;
  const long long sp_min = sp_env("TSL_SP_MIN_BUDGET", SP_MIN_BUDGET);
  if (sp)
    for (int i = 0; i < count; ++i)
      if (budgets[i] == 0 || budgets[i] >= sp_min) budgets[i] = first;
  if (stride < max_n) throw tsl::Error(TSL_EINVAL, "starts stride smaller than a problem size");
  DecideCtx &ctx = decide_ctx();
  std::lock_guard<std::mutex> lock(ctx.mu);
  int dev = 0;
  CK(cudaGetDevice(&dev));
  if (ctx.device != dev) {
    ctx.device = dev;
    ctx.stream = nullptr;
    ctx.buf = nullptr;
    ctx.cap = 0;
    CK(cudaStreamCreateWithFlags(&ctx.stream, cudaStreamNonBlocking));
  }
  const size_t b_pool = align_up(pools.size() * sizeof(int));
  const size_t b_off = align_up(count * sizeof(long long));
  const size_t b_ws = align_up((size_t)ws_total * sizeof(int));
  const size_t b_st = align_up(count * sizeof(int));
  const size_t b_nd = align_up(count * sizeof(long long));
  const size_t b_starts = align_up((size_t)count * stride * sizeof(int));
  char *base = ctx.reserve(b_pool + 3 * b_off + b_ws + b_st + b_nd + b_starts);
  char *q = base;
  int *d_pools = (int *)q; q += b_pool;
  long long *d_poff = (long long *)q; q += b_off;
  long long *d_woff = (long long *)q; q += b_off;
  long long *d_bud = (long long *)q; q += b_off;
  int *d_ws = (int *)q; q += b_ws;
  int *d_st = (int *)q; q += b_st;
  long long *d_nd = (long long *)q; q += b_nd;
  int *d_starts = (int *)q;
  cudaStream_t s = ctx.stream;
  h2d(d_pools, pools.data(), pools.size() * sizeof(int), s);
  h2d(d_poff, pool_off.data(), count * sizeof(long long), s);
  h2d(d_woff, ws_off.data(), count * sizeof(long long), s);
  h2d(d_bud, budgets.data(), count * sizeof(long long), s);
  const unsigned long long budget_ns =
      budget_secs > 0 ? (unsigned long long)(budget_secs * 1e9) : 0ull;
  const int threads = 32;
  COUNT_LAUNCH();
  if (warp_mode) {
    const size_t smem = (size_t)max_state * sizeof(int);
    if (smem > 48 * 1024)
      CK(cudaFuncSetAttribute(k_decide_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
    k_decide_warp<<<count, 32, smem, s>>>(d_pools, d_poff, count, d_bud, budget_ns, d_ws,
                                          d_woff, d_st, d_nd, d_starts, stride);
  } else {
    k_decide_batch<<<(count + threads - 1) / threads, threads, 0, s>>>(
        d_pools, d_poff, count, d_bud, budget_ns, d_ws, d_woff, d_st, d_nd, d_starts, stride);
  }
  CK(cudaGetLastError());
  std::vector<int> h_st(count);
  std::vector<long long> h_nd(count);
  std::vector<int> h_starts((size_t)count * stride);
  d2h(h_st.data(), d_st, count * sizeof(int), s);
  d2h(h_nd.data(), d_nd, count * sizeof(long long), s);
  d2h(h_starts.data(), d_starts, (size_t)count * stride * sizeof(int), s);
  CK(cudaStreamSynchronize(s));
  // many long problems: they run concurrently (one warp each) at their real
  // cap; a few: one at a time, each subtree-parallel over the whole GPU
  std::vector<int> longs;
  for (int i = 0; i < count; ++i)
    if (sp && h_st[i] == RX_TIMEOUT && budgets[i] != real_budget[i]) longs.push_back(i);
  if ((int)longs.size() > SP_BATCH_MAX) {
    std::vector<tsl_problem> sub;
    for (int i : longs) sub.push_back(probs[i]);
    std::vector<int32_t> st2(longs.size());
    std::vector<int64_t> nd2(longs.size()), s2((size_t)longs.size() * stride);
    run_decide_batch((int)longs.size(), sub.data(), budget_secs, st2.data(), nd2.data(),
                     s2.data(), stride, /*allow_sp=*/false);
    for (size_t k = 0; k < longs.size(); ++k) {
      const int i = longs[k];
      h_st[i] = st2[k];
      h_nd[i] = nd2[k];
      for (int j = 0; j < probs[i].n; ++j)
        h_starts[(size_t)i * stride + j] = (int)s2[k * stride + j];
      budgets[i] = real_budget[i];
    }
  }
  for (int i = 0; i < count; ++i) {
    status[i] = h_st[i];
    nodes[i] = h_nd[i];
    if (sp && h_st[i] == RX_TIMEOUT && budgets[i] != real_budget[i]) {
      std::vector<int> one(pools.begin() + pool_off[i],
                           pools.begin() + pool_off[i] + pools[pool_off[i] + G_WORDS]);
      std::vector<int> sv(std::max(probs[i].n, 1));
      long long nd = 0;
      const int st = sp_solve(one, real_budget[i], budget_secs, s, &nd, sv.data());
      status[i] = st;
      nodes[i] = nd;
      if (starts && st == RX_SAT)
        for (int k = 0; k < probs[i].n; ++k) starts[(size_t)i * stride + k] = sv[k];
      continue;
    }
    if (starts && h_st[i] == RX_SAT)
      for (int k = 0; k < probs[i].n; ++k)
        starts[(size_t)i * stride + k] = h_starts[(size_t)i * stride + k];
  }
}

}  // namespace

// ------------------------------------------------------------------ engine

struct tsl_engine {
  tsl::Placement pl;
  std::vector<int> pool;
  int device = 0;
  bool gpu_ready = false;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, evm = nullptr;
  float last_ms = 0.f, last_root_ms = 0.f;  // root_ms: k_root share of the last probe call
  int *d_pool = nullptr;
  // enumeration tables (host copy per n_r, device copy of the staged n_r)
  int h_nr = -1;
  std::vector<unsigned long long> h_cnt;
  std::vector<long long> h_off;
  int d_nr = -1;
  unsigned long long *d_cnt = nullptr;
  long long *d_off = nullptr;
  size_t d_cnt_cap = 0, d_off_cap = 0;
  // staged window
  long long W = 0, W_cap = 0, n_act = 0;
  int cur = 0;
  unsigned char *d_assign = nullptr, *d_gate = nullptr;
  int *d_act[2] = {nullptr, nullptr};
  int *d_def[2] = {nullptr, nullptr};
  int *d_surv = nullptr;  // k_root survivors of the current level
  int dcur = 0;
  long long n_def = 0, n_sat = 0;
  int *d_sat_widx = nullptr, *d_sat_starts = nullptr;
  int *d_counters = nullptr;
  unsigned long long *d_stats = nullptr;
  // SAT rows of the level: the ordered walk runs on the device
  // (k_sat_min / k_sat_fetch, tsl_engine_sat_next); the host-sorted index is
  // built only for the legacy tsl_engine_sat_rows
  std::vector<int> sat_widx_sorted, sat_pos_sorted;
  bool sat_sorted = false;
  unsigned long long *d_sat_key = nullptr;
  int *d_sat_next = nullptr;
  int *d_gather = nullptr;
  size_t d_gather_cap = 0;
  int *d_stash_idx = nullptr;  // window indices of the rows being stashed
  size_t stash_idx_cap = 0;
  char *d_verify = nullptr;
  size_t d_verify_cap = 0;
  // asynchronous verification slots (windows in flight while the next one
  // is scanned): private assignment rows + their own buffers and stream
  struct VSlot {
    unsigned char *rows = nullptr;
    size_t rows_cap = 0;
    long long n_rows = 0;
    char *buf = nullptr;
    size_t cap = 0;
    long long count = 0;
    int *d_st = nullptr, *d_s = nullptr;
    long long *d_n = nullptr;
    cudaEvent_t ev_go = nullptr, ev0 = nullptr, ev1 = nullptr;
    cudaStream_t st = nullptr;  // the slot's verification stream
  } vslot[TSL_VERIFY_SLOTS];
  // per-thread DFS scratch
  int *d_ws = nullptr;
  long long ws_words = 0;
  int ws_threads = 0;
  int num_sms = 148;
  size_t smem_bytes = 0;

  void host_tables(int n_r) {
    if (h_nr == n_r) return;
    tsl::rep_counts(pool, n_r, h_cnt, h_off);
    h_nr = n_r;
  }

  void ensure_gpu() {
    if (gpu_ready) return;
    require_device();
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&ev0));
    CK(cudaEventCreate(&ev1));
    CK(cudaEventCreate(&evm));
    for (auto &vs : vslot) {
      CK(cudaStreamCreateWithFlags(&vs.st, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&vs.ev_go, cudaEventDisableTiming));
      CK(cudaEventCreate(&vs.ev0));
      CK(cudaEventCreate(&vs.ev1));
    }
    CK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, device));
    // every engine buffer comes from the device's stream-ordered pool
    // (dev_grow keeps its freed memory cached): a fresh engine reuses the
    // previous one's memory, and its teardown never synchronises the device
    pool_keep();
    d_pool = (int *)dev_take(pool.size() * sizeof(int), stream);
    h2d(d_pool, pool.data(), pool.size() * sizeof(int), stream);
    CK(cudaStreamSynchronize(stream));
    d_counters = (int *)dev_take(8 * sizeof(int), stream);  // [4] = speculative retirement limit
    d_stats = (unsigned long long *)dev_take(8 * sizeof(unsigned long long), stream);
    smem_bytes = pool.size() * sizeof(int);
    if (smem_bytes > 48 * 1024) {
      CK(cudaFuncSetAttribute(k_probe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem_bytes));
      CK(cudaFuncSetAttribute(k_resolve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem_bytes));
      CK(cudaFuncSetAttribute(k_stage, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem_bytes));
    }
    const int K = pool[R_K];
    const int ndep = pool[R_NDEP];
    (void)K;
    (void)ndep;
    ws_words = rep_ws_words(pool.data());
    ws_threads = num_sms * 4 * 128;
    d_ws = (int *)dev_take((size_t)ws_threads * ws_words * sizeof(int), stream);
    CK(cudaStreamSynchronize(stream));
    gpu_ready = true;
  }

  void device_tables(int n_r) {
    if (d_nr == n_r) return;
    host_tables(n_r);
    if (h_cnt.size() > d_cnt_cap) {
      dev_grow((void **)&d_cnt, h_cnt.size() * sizeof(unsigned long long), stream);
      d_cnt_cap = h_cnt.size();
    }
    if (h_off.size() > d_off_cap) {
      dev_grow((void **)&d_off, h_off.size() * sizeof(long long), stream);
      d_off_cap = h_off.size();
    }
    h2d(d_cnt, h_cnt.data(), h_cnt.size() * sizeof(unsigned long long), stream);
    h2d(d_off, h_off.data(), h_off.size() * sizeof(long long), stream);
    CK(cudaStreamSynchronize(stream));
    d_nr = n_r;
  }

  void ensure_window(long long w) {
    if (w <= W_cap) return;
    const int K = pool[R_K];
    dev_grow((void **)&d_assign, (size_t)w * K, stream);
    dev_grow((void **)&d_gate, (size_t)w, stream);
    dev_grow((void **)&d_act[0], (size_t)w * sizeof(int), stream);
    dev_grow((void **)&d_act[1], (size_t)w * sizeof(int), stream);
    dev_grow((void **)&d_def[0], (size_t)w * sizeof(int), stream);
    dev_grow((void **)&d_def[1], (size_t)w * sizeof(int), stream);
    dev_grow((void **)&d_surv, (size_t)w * sizeof(int), stream);
    dev_grow((void **)&d_sat_widx, (size_t)w * sizeof(int), stream);
    dev_grow((void **)&d_sat_starts, (size_t)w * K * sizeof(int), stream);
    W_cap = w;
  }

  ~tsl_engine() {
    if (!gpu_ready) return;
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);  // blocks are parked under the engine's device
    // stream-ordered frees back into the pool, after the work queued on the
    // engine's streams (a synchronous cudaFree stalled a caller's next
    // search by up to 0.5 s); stream and event destruction do not block
    // the engine's own streams finish first (normally already idle): its
    // buffers are then parked for the next engine (dev_park)
    for (auto &vs : vslot) cudaStreamSynchronize(vs.st);
    cudaStreamSynchronize(stream);
    for (auto &vs : vslot) {
      dev_park(vs.rows, stream);
      dev_park(vs.buf, stream);
    }
    for (void *p : {(void *)d_pool, (void *)d_cnt, (void *)d_off, (void *)d_assign, (void *)d_gate,
                    (void *)d_act[0], (void *)d_act[1], (void *)d_sat_widx, (void *)d_sat_starts,
                    (void *)d_counters, (void *)d_stats, (void *)d_ws, (void *)d_gather,
                    (void *)d_def[0], (void *)d_def[1], (void *)d_verify, (void *)d_surv,
                    (void *)d_sat_key, (void *)d_sat_next, (void *)d_stash_idx})
      dev_park(p, stream);
    cudaEventDestroy(ev0);
    cudaEventDestroy(ev1);
    cudaEventDestroy(evm);
    for (auto &vs : vslot) {
      cudaEventDestroy(vs.ev_go);
      cudaEventDestroy(vs.ev0);
      cudaEventDestroy(vs.ev1);
      cudaStreamDestroy(vs.st);
    }
    cudaStreamDestroy(stream);
    cudaSetDevice(prev);
  }
};

// ------------------------------------------------------------------ C ABI

#ifdef WDJ_COUNT_ROUNDS
extern "C" void tsl_debug_wdj_rounds(unsigned long long *out) {
  CK(cudaMemcpyFromSymbol(out, g_wdj_rounds, 8));
  CK(cudaMemcpyFromSymbol(out + 1, g_wdj_calls, 8));
  CK(cudaMemcpyFromSymbol(out + 2, g_wdj_rows, 8));
  CK(cudaMemcpyFromSymbol(out + 3, g_wdj_pairs, 8));
}
#endif
extern "C" {

const char *tsl_last_error(void) { return g_err.c_str(); }

int tsl_version(void) { return TSL_VERSION; }

int tsl_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int tsl_set_device(int device) {
  API_BEGIN
  require_device();
  CK(cudaSetDevice(device));
  return TSL_OK;
  API_END
}

int tsl_decide(int n, const int64_t *dur, const uint64_t *devmask, const int64_t *mem,
               const int64_t *edges, int m, const int64_t *order, const int64_t *lo,
               const int64_t *hi, int ndev, const int64_t *init_mem, int64_t cap,
               int64_t node_budget, double budget_secs, int64_t *out_starts,
               int64_t *out_nodes) {
  API_BEGIN
  tsl_problem p;
  p.n = n;
  p.m = m;
  p.ndev = ndev;
  p.dur = dur;
  p.mem = mem;
  p.edges = edges;
  p.order = order;
  p.lo = lo;
  p.hi = hi;
  p.init_mem = init_mem;
  p.devmask = devmask;
  p.cap = cap;
  p.node_budget = node_budget;
  int32_t st = 0;
  int64_t nd = 0;
  run_decide_batch(1, &p, budget_secs, &st, &nd, out_starts, std::max(n, 1), true);
  if (out_nodes) *out_nodes = nd;
  return st;
  API_END
}

int tsl_decide_batch(int count, const tsl_problem *probs, double budget_secs, int32_t *status,
                     int64_t *nodes, int64_t *starts, int stride) {
  API_BEGIN
  if (count < 0) throw tsl::Error(TSL_EINVAL, "negative problem count");
  run_decide_batch(count, probs, budget_secs, status, nodes, starts, stride, true);
  return TSL_OK;
  API_END
}

tsl_engine *tsl_engine_open(int K, int D, const int32_t *dur, const int32_t *mem,
                            const uint64_t *devmask, int n_deps, const int32_t *deps,
                            int device) {
  tsl_engine *e = nullptr;
  try {
    for (int i = 0; i < K; ++i) {
      tsl::ck(dur[i], "dur");
      tsl::ck(mem[i], "mem");
      if (dur[i] < 1) throw tsl::Error(TSL_EINVAL, "time_cost must be >= 1");
    }
    e = new tsl_engine();
    e->pl.K = K;
    e->pl.D = D;
    e->pl.dur.assign(dur, dur + K);
    e->pl.mem.assign(mem, mem + K);
    e->pl.mask.assign(devmask, devmask + K);
    for (int i = 0; i < n_deps; ++i) {
      const int a = deps[2 * i], b = deps[2 * i + 1];
      if (a < 0 || a >= K || b < 0 || b >= K) {
        delete e;
        set_err(TSL_EINVAL, "dependency references a missing stage");
        return nullptr;
      }
      e->pl.deps.push_back({a, b});
    }
    std::sort(e->pl.deps.begin(), e->pl.deps.end());
    e->pool = tsl::rep_build(e->pl);
    e->device = device;
    return e;
  } catch (const tsl::Error &err) {
    delete e;
    set_err(err.code, err.what());
    return nullptr;
  } catch (const std::exception &err) {
    delete e;
    set_err(TSL_EINVAL, err.what());
    return nullptr;
  }
}

void tsl_engine_close(tsl_engine *e) { delete e; }

int tsl_engine_count(tsl_engine *e, int n_r, uint64_t *out_count) {
  API_BEGIN
  if (n_r < 1) throw tsl::Error(TSL_EINVAL, "n_r must be >= 1");
  e->host_tables(n_r);
  const unsigned long long c = e->h_cnt[e->h_off[0] + 0];
  if (c >= (1ULL << 63)) throw tsl::Error(TSL_ERANGE, "candidate count exceeds 2^63");
  *out_count = c;
  return TSL_OK;
  API_END
}

int tsl_engine_unrank(tsl_engine *e, int n_r, uint64_t rank, int32_t *out_assignment) {
  API_BEGIN
  e->host_tables(n_r);
  std::vector<int> av(e->pool[R_K], 0);
  int *a = av.data();
  if (!rep_unrank(e->pool.data(), e->h_cnt.data(), e->h_off.data(), n_r, rank, a))
    throw tsl::Error(TSL_EINVAL, "rank out of range");
  for (size_t i = 0; i < av.size(); ++i) out_assignment[i] = av[i];
  return TSL_OK;
  API_END
}

int tsl_engine_stage(tsl_engine *e, int n_r, uint64_t r0, uint64_t r1, int64_t cap,
                     int64_t *out_active, uint8_t *gate_out) {
  API_BEGIN
  if (r1 < r0) throw tsl::Error(TSL_EINVAL, "empty rank window");
  const long long W = (long long)(r1 - r0);
  if (W > (1LL << 30)) throw tsl::Error(TSL_ERANGE, "window larger than 2^30 ranks");
  e->ensure_gpu();
  CK(cudaSetDevice(e->device));
  e->device_tables(n_r);
  e->ensure_window(std::max(W, 1LL));
  const int icap = cap < 0 ? -1 : (int)std::min<int64_t>(cap, tsl::VMAX - 1);
  CK(cudaMemsetAsync(e->d_counters, 0, 4 * sizeof(int), e->stream));
  const int threads = 128;
  long long blocks = (W + threads - 1) / threads;
  blocks = std::max(1LL, std::min<long long>(blocks, (long long)e->num_sms * 8));
  CK(cudaEventRecord(e->ev0, e->stream));
  COUNT_LAUNCH();
  k_stage<<<(int)blocks, threads, e->smem_bytes, e->stream>>>(
      e->d_pool, e->d_cnt, e->d_off, n_r, r0, W, icap, e->d_assign, e->d_gate, e->d_act[0],
      e->d_counters);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e->ev1, e->stream));
  int n_act = 0;
  d2h(&n_act, e->d_counters, sizeof(int), e->stream);
  if (gate_out)
    d2h(gate_out, e->d_gate, (size_t)W, e->stream);
  CK(cudaStreamSynchronize(e->stream));
  CK(cudaEventElapsedTime(&e->last_ms, e->ev0, e->ev1));
  e->W = W;
  e->n_act = n_act;
  e->cur = 0;
  *out_active = n_act;
  return TSL_OK;
  API_END
}

static void fill_stats(const unsigned long long *st, tsl_level_stats *stats) {
  if (!stats) return;
  stats->probes = (int64_t)st[0];
  stats->root_refuted = (int64_t)st[1];
  stats->nodes = (int64_t)st[2];
  stats->capped = (int64_t)st[3];
  stats->sat = (int64_t)st[4];
  stats->deferred = (int64_t)st[5];
  stats->dj_refuted = (int64_t)st[6];
  stats->dj_nodes = (int64_t)st[7];
}

// Record the level's SAT count and return its first min(n_sat, max_sat)
// rows in window order through the device argmin.
static int finish_level(tsl_engine *e, int n_sat, int64_t max_sat, int64_t *out_nsat,
                        int64_t *sat_widx, int32_t *sat_starts) {
  e->n_sat = n_sat;
  e->sat_sorted = false;
  *out_nsat = n_sat;
  const long long keep = std::min<long long>(n_sat, max_sat < 0 ? 0 : max_sat);
  const int K = e->pool[R_K];
  long long after = -1;
  for (long long r = 0; r < keep; ++r) {
    int64_t w = -1;
    const int rc = tsl_engine_sat_next(e, after, &w, sat_starts + r * K);
    if (rc != TSL_OK) return rc;
    sat_widx[r] = w;
    after = w;
  }
  return TSL_OK;
}

int tsl_engine_probe(tsl_engine *e, int period, int64_t node_budget, int64_t small_budget,
                     int64_t cap, int64_t widx_limit, double budget_secs, int64_t max_sat,
                     int64_t *out_nsat, int64_t *sat_widx, int32_t *sat_starts,
                     int64_t *out_active, int64_t *out_deferred, tsl_level_stats *stats) {
  API_BEGIN
  if (!e->gpu_ready) throw tsl::Error(TSL_EINVAL, "tsl_engine_probe before tsl_engine_stage");
  CK(cudaSetDevice(e->device));
  const int K = e->pool[R_K];
  tsl::ck(2LL * (K - 1) * ((long long)period + e->pool[R_MAXDUR]) + 4LL * e->pool[R_TOTAL],
          "period anchor");
  const int icap = cap < 0 ? -1 : (int)std::min<int64_t>(cap, tsl::VMAX - 1);
  const long long n_in = e->n_act;
  {
    const int init[6] = {0, 0, 0, 0, (int)std::min<int64_t>(widx_limit, 0x7fffffff), 0};
    h2d(e->d_counters, init, sizeof init, e->stream);
  }
  CK(cudaMemsetAsync(e->d_stats, 0, 8 * sizeof(unsigned long long), e->stream));
  const int threads = 128;
  long long blocks = (n_in + threads - 1) / threads;
  blocks = std::max(1LL, std::min<long long>(blocks, (long long)e->ws_threads / threads));
  const unsigned long long budget_ns =
      budget_secs > 0 ? (unsigned long long)(budget_secs * 1e9) : 0ull;
  ProbeOut o;
  o.act_out = e->d_act[1 - e->cur];
  e->dcur = 0;
  o.def_out = e->d_def[0];
  o.sat_widx = e->d_sat_widx;
  o.sat_starts = e->d_sat_starts;
  o.counters = e->d_counters;
  o.stats = e->d_stats;
  CK(cudaEventRecord(e->ev0, e->stream));
  bool root_timed = false;
  if (n_in > 0 && !root_filter_off()) {
    // K2a: warp-per-probe root filter, then the exact DFS on its survivors
    const int wpb = 8;
    const size_t smem = (size_t)(((e->pool.size() + 3) & ~(size_t)3) +
                                 wpb * root_warp_words(e->pool.data())) * sizeof(int);
    if (smem > 48 * 1024)
      CK(cudaFuncSetAttribute(k_root, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    long long rblocks = (n_in + wpb - 1) / wpb;
    rblocks = std::max(1LL, std::min<long long>(rblocks, (long long)e->num_sms * 8));
    COUNT_LAUNCH();
    k_root<<<(int)rblocks, 32 * wpb, smem, e->stream>>>(e->d_pool, e->d_assign,
                                                        e->d_act[e->cur], (int)n_in, o,
                                                        e->d_surv, period, icap, widx_limit,
                                                        root_devs_serial() ? 1 : 0);
    CK(cudaGetLastError());
    CK(cudaEventRecord(e->evm, e->stream));
    root_timed = true;
    // survivors: warp-cooperative reference-exact DFS with the small budget
    // (same outcome contract as k_probe: SAT / settled / deferred)
    const int swpb = 4;
    const size_t ssmem = (size_t)(((e->pool.size() + 3) & ~(size_t)3) +
                                  swpb * ((rep_warp_smem_words(e->pool.data()) + 3) & ~3)) *
                         sizeof(int);
    if (ssmem > 48 * 1024)
      CK(cudaFuncSetAttribute(k_resolve_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)ssmem));
    long long sblocks = (n_in + swpb - 1) / swpb;
    sblocks = std::max(1LL, std::min<long long>(sblocks, (long long)e->ws_threads / (32 * swpb)));
    const long long full = node_budget < 0 ? 0 : node_budget;
    const long long sb = small_budget <= 0 ? 0 : small_budget;
    // a probe is deferred only when the small budget is below the cap
    const long long stage = (full == 0 || sb < full) ? sb : 0;
    COUNT_LAUNCH();
    k_resolve_warp<<<(int)sblocks, 32 * swpb, ssmem, e->stream>>>(
        e->d_pool, e->d_assign, e->d_surv, 0, e->d_counters + 3, o, period, full, stage, 0,
        icap, widx_limit, budget_ns, e->d_ws, e->ws_words, e->d_counters + 4, 0,
        resolve_dynamic() ? e->d_counters + 5 : nullptr);
    CK(cudaGetLastError());
  } else if (n_in > 0) {
    COUNT_LAUNCH();
    k_probe<<<(int)blocks, threads, e->smem_bytes, e->stream>>>(
        e->d_pool, e->d_assign, e->d_act[e->cur], (int)n_in, nullptr, o, period,
        node_budget < 0 ? 0 : node_budget, small_budget <= 0 ? 0 : small_budget, icap,
        widx_limit, budget_ns, e->d_ws, e->ws_words);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(e->ev1, e->stream));
  int counters[4] = {0, 0, 0, 0};
  unsigned long long st[8] = {0};
  d2h(counters, e->d_counters, 4 * sizeof(int), e->stream);
  d2h(st, e->d_stats, 8 * sizeof(unsigned long long), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  CK(cudaEventElapsedTime(&e->last_ms, e->ev0, e->ev1));
  e->last_root_ms = 0.f;
  if (root_timed) CK(cudaEventElapsedTime(&e->last_root_ms, e->ev0, e->evm));
  e->cur = 1 - e->cur;
  e->n_act = counters[0];
  e->n_def = counters[2];
  *out_active = counters[0];
  *out_deferred = counters[2];
  fill_stats(st, stats);
  return finish_level(e, counters[1], max_sat, out_nsat, sat_widx, sat_starts);
  API_END
}

int tsl_engine_resolve(tsl_engine *e, int period, int64_t node_budget, int64_t stage_budget,
                       int64_t dj_budget, int64_t cap, int64_t widx_limit, double budget_secs,
                       int64_t max_sat, int64_t *out_nsat, int64_t *sat_widx,
                       int32_t *sat_starts, int64_t *out_active, int64_t *out_deferred,
                       tsl_level_stats *stats) {
  API_BEGIN
  if (!e->gpu_ready) throw tsl::Error(TSL_EINVAL, "tsl_engine_resolve before tsl_engine_stage");
  CK(cudaSetDevice(e->device));
  const int icap = cap < 0 ? -1 : (int)std::min<int64_t>(cap, tsl::VMAX - 1);
  const long long n_def = e->n_def;
  // continue appending to the level's SAT list and to the active list
  int counters[7] = {(int)e->n_act, (int)e->n_sat, 0, 0,
                     (int)std::min<int64_t>(widx_limit, 0x7fffffff), 0, 0};
  h2d(e->d_counters, counters, 7 * sizeof(int), e->stream);
  CK(cudaMemsetAsync(e->d_stats, 0, 8 * sizeof(unsigned long long), e->stream));
  const int threads = 128;
  long long blocks = (n_def + threads - 1) / threads;
  blocks = std::max(1LL, std::min<long long>(blocks, (long long)e->ws_threads / threads));
  const unsigned long long budget_ns =
      budget_secs > 0 ? (unsigned long long)(budget_secs * 1e9) : 0ull;
  ProbeOut o;
  o.act_out = e->d_act[e->cur];
  o.def_out = e->d_def[1 - e->dcur];
  o.sat_widx = e->d_sat_widx;
  o.sat_starts = e->d_sat_starts;
  o.counters = e->d_counters;
  o.stats = e->d_stats;
  CK(cudaEventRecord(e->ev0, e->stream));
  const int *rx_in = e->d_def[e->dcur];
  const int *rx_count = nullptr;
  if (n_def > 0 && decide_mode_warp() && dj_budget > 0 && dj_mode_warp(e->pool.data()) &&
      dj_split()) {
    // the filter alone first, at high occupancy; its survivors (d_surv,
    // counters[3]) then take the DFS stage below without the filter
    const int wpb = 8;
    const long long gwords = wdj_snap_words(e->pool[R_K], e->pool[R_NPAIR]) + 8;
    long long dblocks = std::max(1LL, std::min<long long>((n_def + wpb - 1) / wpb,
                                                          (long long)e->num_sms * 4));
    dblocks = std::min<long long>(dblocks, (e->ws_threads * e->ws_words) / (gwords * wpb));
    const size_t smem = (size_t)(((e->pool.size() + 3) & ~(size_t)3) +
                                 wpb * dj_warp_words(e->pool.data())) * sizeof(int);
    if (smem > 48 * 1024)
      CK(cudaFuncSetAttribute(k_dj_filter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
    COUNT_LAUNCH();
    k_dj_filter<<<(int)dblocks, 32 * wpb, smem, e->stream>>>(
        e->d_pool, e->d_assign, e->d_def[e->dcur], (int)n_def, o, e->d_surv, period,
        dj_budget, icap, widx_limit, e->d_ws, gwords, e->d_counters + 4,
        resolve_dynamic() ? e->d_counters + 6 : nullptr);
    CK(cudaGetLastError());
    rx_in = e->d_surv;
    rx_count = e->d_counters + 3;
    dj_budget = 0;
  }
  if (n_def > 0 && decide_mode_warp()) {
    const int wpb = 4;
    long long wblocks = (n_def + wpb - 1) / wpb;
    wblocks = std::max(1LL, std::min<long long>(wblocks, (long long)e->ws_threads / (32 * wpb)));
    const size_t smem = (size_t)(((e->pool.size() + 3) & ~(size_t)3) +
                                 wpb * ((rep_warp_smem_words(e->pool.data()) + 3) & ~3)) *
                        sizeof(int);
    if (smem > 48 * 1024)
      CK(cudaFuncSetAttribute(k_resolve_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                              (int)smem));
    COUNT_LAUNCH();
    k_resolve_warp<<<(int)wblocks, 32 * wpb, smem, e->stream>>>(
        e->d_pool, e->d_assign, rx_in, (int)n_def, rx_count, o, period,
        node_budget < 0 ? 0 : node_budget, stage_budget < 0 ? -1 : stage_budget,
        dj_budget < 0 ? 0 : dj_budget, icap, widx_limit, budget_ns, e->d_ws, e->ws_words,
        e->d_counters + 4, dj_mode_warp(e->pool.data()) ? 1 : 0,
        resolve_dynamic() ? e->d_counters + 5 : nullptr);
    CK(cudaGetLastError());
  } else if (n_def > 0) {
    COUNT_LAUNCH();
    k_resolve<<<(int)blocks, threads, e->smem_bytes, e->stream>>>(
        e->d_pool, e->d_assign, e->d_def[e->dcur], (int)n_def, o, period,
        node_budget < 0 ? 0 : node_budget, stage_budget < 0 ? -1 : stage_budget,
        dj_budget < 0 ? 0 : dj_budget, icap, widx_limit, budget_ns, e->d_ws, e->ws_words);
    CK(cudaGetLastError());
  }
  CK(cudaEventRecord(e->ev1, e->stream));
  unsigned long long st[8] = {0};
  d2h(counters, e->d_counters, 4 * sizeof(int), e->stream);
  d2h(st, e->d_stats, 8 * sizeof(unsigned long long), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  CK(cudaEventElapsedTime(&e->last_ms, e->ev0, e->ev1));
  e->n_act = counters[0];
  e->n_def = counters[2];
  e->dcur = 1 - e->dcur;
  *out_active = counters[0];
  *out_deferred = counters[2];
  fill_stats(st, stats);
  return finish_level(e, counters[1], max_sat, out_nsat, sat_widx, sat_starts);
  API_END
}

// Take the deferred list of the last stage (entries <= widx_limit) to the
// host without settling it; the entries leave the device lists.
int tsl_engine_take_deferred(tsl_engine *e, int64_t widx_limit, int64_t max_out,
                             int64_t *widx_out, int64_t *out_count) {
  API_BEGIN
  const long long n = e->n_def;
  std::vector<int> buf(n);
  if (n > 0) {
    d2h(buf.data(), e->d_def[e->dcur], n * sizeof(int), e->stream);
    CK(cudaStreamSynchronize(e->stream));
  }
  std::sort(buf.begin(), buf.end());
  long long k = 0;
  for (long long i = 0; i < n; ++i)
    if (buf[i] <= widx_limit) {
      if (k >= max_out) throw tsl::Error(TSL_EINVAL, "take_deferred: output too small");
      widx_out[k++] = buf[i];
    }
  e->n_def = 0;
  *out_count = k;
  return TSL_OK;
  API_END
}

// Append window indices to the active list (they are probed at the next
// level like any other active candidate).
int tsl_engine_add_active(tsl_engine *e, int64_t count, const int64_t *widx) {
  API_BEGIN
  if (count <= 0) return TSL_OK;
  if (e->n_act + count > e->W_cap) throw tsl::Error(TSL_EINVAL, "active list overflow");
  std::vector<int> buf(widx, widx + count);
  h2d(e->d_act[e->cur] + e->n_act, buf.data(), count * sizeof(int), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  e->n_act += count;
  return TSL_OK;
  API_END
}

// Whether a verification launch lets a SAT cancel the higher probes it may
// retire: only when the launch's warps cannot all be resident at once
// (cancelling then frees a warp slot for a waiting probe); a resident probe
// runs on (an aborted one would be re-run after the launch, adding its whole
// count to the window's critical path).  TSL_VERIFY_CANCEL=1 / 0 forces it.
static int verify_cancel(tsl_engine *e, long long count, int wpb, size_t smem) {
  const char *m = getenv("TSL_VERIFY_CANCEL");
  if (m && std::string(m) == "1") return 1;
  if (m && std::string(m) == "0") return 0;
  int per_sm = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_verify_warp, 32 * wpb, smem));
  return count > (long long)std::max(per_sm, 1) * e->num_sms * wpb ? 1 : 0;
}

int tsl_engine_verify(tsl_engine *e, int64_t count, const int64_t *widx, const int32_t *period,
                      const int64_t *node_budget, int64_t cap, int32_t *status_out,
                      int64_t *nodes_out, int32_t *starts_out) {
  API_BEGIN
  if (!e->gpu_ready) throw tsl::Error(TSL_EINVAL, "tsl_engine_verify before tsl_engine_stage");
  if (count <= 0) return TSL_OK;
  CK(cudaSetDevice(e->device));
  const int K = e->pool[R_K];
  const int icap = cap < 0 ? -1 : (int)std::min<int64_t>(cap, tsl::VMAX - 1);
  std::vector<int> w32(count), p32(count);
  for (long long i = 0; i < count; ++i) {
    if (widx[i] < 0 || widx[i] >= e->W) throw tsl::Error(TSL_EINVAL, "verify: bad window index");
    tsl::ck(2LL * (K - 1) * ((long long)period[i] + e->pool[R_MAXDUR]) + 4LL * e->pool[R_TOTAL],
            "period anchor");
    w32[i] = (int)widx[i];
    p32[i] = period[i];
  }
  const size_t b_i = ((size_t)count * sizeof(int) + 255) / 256 * 256;
  const size_t b_l = ((size_t)count * sizeof(long long) + 255) / 256 * 256;
  int pmin = period[0], pmax = period[0];
  for (long long i = 0; i < count; ++i) {
    pmin = std::min(pmin, period[i]);
    pmax = std::max(pmax, period[i]);
  }
  const int nlev = pmax - pmin + 1;
  const size_t b_lim = ((size_t)nlev * sizeof(int) + 255) / 256 * 256;
  const size_t need = 3 * b_i + 2 * b_l + b_lim + (size_t)count * K * sizeof(int);
  if (need > e->d_verify_cap) {
    dev_grow((void **)&e->d_verify, need, e->stream);
    e->d_verify_cap = need;
  }
  char *q = e->d_verify;
  int *d_w = (int *)q; q += b_i;
  int *d_p = (int *)q; q += b_i;
  int *d_st = (int *)q; q += b_i;
  long long *d_b = (long long *)q; q += b_l;
  long long *d_n = (long long *)q; q += b_l;
  int *d_lim = (int *)q; q += b_lim;
  int *d_s = (int *)q;
  {
    std::vector<int> lim0(nlev, 0x7fffffff);
    h2d(d_lim, lim0.data(), nlev * sizeof(int), e->stream);
  }
  h2d(d_w, w32.data(), count * sizeof(int), e->stream);
  h2d(d_p, p32.data(), count * sizeof(int), e->stream);
  h2d(d_b, node_budget, count * sizeof(long long), e->stream);
  const int wpb = 4;
  const size_t smem = (size_t)(((e->pool.size() + 3) & ~(size_t)3) +
                               wpb * ((rep_warp_smem_words(e->pool.data()) + 3) & ~3)) *
                      sizeof(int);
  if (smem > 48 * 1024)
    CK(cudaFuncSetAttribute(k_verify_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
  long long blocks = (count + wpb - 1) / wpb;
  blocks = std::min<long long>(blocks, (long long)e->num_sms * 16);
  const int cancel = verify_cancel(e, count, wpb, smem);
  CK(cudaEventRecord(e->ev0, e->stream));
  COUNT_LAUNCH();
  k_verify_warp<<<(int)blocks, 32 * wpb, smem, e->stream>>>(e->d_pool, e->d_assign, d_w, d_p,
                                                             d_b, (int)count, icap, d_st, d_n,
                                                             d_s, d_lim, pmin, nlev, nullptr,
                                                             nullptr, cancel);
  CK(cudaGetLastError());
  CK(cudaEventRecord(e->ev1, e->stream));
  d2h(status_out, d_st, count * sizeof(int), e->stream);
  d2h(nodes_out, d_n, count * sizeof(long long), e->stream);
  d2h(starts_out, d_s, (size_t)count * K * sizeof(int), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  CK(cudaEventElapsedTime(&e->last_ms, e->ev0, e->ev1));
  return TSL_OK;
  API_END
}

int tsl_engine_verify_stash(tsl_engine *e, int slot, int64_t count, const int64_t *widx) {
  API_BEGIN
  if (!e->gpu_ready) throw tsl::Error(TSL_EINVAL, "verify_stash before tsl_engine_stage");
  if (slot < 0 || slot >= TSL_VERIFY_SLOTS) throw tsl::Error(TSL_EINVAL, "bad verify slot");
  CK(cudaSetDevice(e->device));
  auto &vs = e->vslot[slot];
  CK(cudaStreamSynchronize(vs.st));  // the slot's previous work is done
  const int K = e->pool[R_K];
  const size_t need = (size_t)std::max<int64_t>(count, 1) * K;
  if (need > vs.rows_cap) {
    dev_grow((void **)&vs.rows, need, e->stream);  // written by k_stash_rows on e->stream
    vs.rows_cap = need;
  }
  vs.n_rows = count;
  if (count > 0) {
    std::vector<int> w32(count);
    for (long long i = 0; i < count; ++i) {
      if (widx[i] < 0 || widx[i] >= e->W) throw tsl::Error(TSL_EINVAL, "stash: bad window index");
      w32[i] = (int)widx[i];
    }
    if ((size_t)count > e->stash_idx_cap) {
      dev_grow((void **)&e->d_stash_idx, (size_t)count * sizeof(int), e->stream);
      e->stash_idx_cap = (size_t)count;
    }
    int *d_w = e->d_stash_idx;
    h2d(d_w, w32.data(), count * sizeof(int), e->stream);
    const long long total = count * K;
    COUNT_LAUNCH();
    k_stash_rows<<<(int)((total + 255) / 256), 256, 0, e->stream>>>(e->d_assign, d_w,
                                                                     (int)count, K, vs.rows);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(e->stream));
  }
  return TSL_OK;
  API_END
}

int tsl_engine_verify_launch(tsl_engine *e, int slot, int64_t count, const int64_t *pos,
                             const int64_t *widx, const int32_t *period,
                             const int64_t *node_budget, int64_t cap) {
  API_BEGIN
  if (slot < 0 || slot >= TSL_VERIFY_SLOTS) throw tsl::Error(TSL_EINVAL, "bad verify slot");
  auto &vs = e->vslot[slot];
  vs.count = count;
  if (count <= 0) return TSL_OK;
  CK(cudaSetDevice(e->device));
  const int K = e->pool[R_K];
  const int icap = cap < 0 ? -1 : (int)std::min<int64_t>(cap, tsl::VMAX - 1);
  std::vector<int> w32(count), p32(count), s32(count);
  int pmin = period[0], pmax = period[0];
  for (long long i = 0; i < count; ++i) {
    if (pos[i] < 0 || pos[i] >= vs.n_rows) throw tsl::Error(TSL_EINVAL, "verify: bad row position");
    tsl::ck(2LL * (K - 1) * ((long long)period[i] + e->pool[R_MAXDUR]) + 4LL * e->pool[R_TOTAL],
            "period anchor");
    w32[i] = (int)widx[i];
    p32[i] = period[i];
    s32[i] = (int)pos[i];
    pmin = std::min(pmin, period[i]);
    pmax = std::max(pmax, period[i]);
  }
  const int nlev = pmax - pmin + 1;
  const size_t b_i = ((size_t)count * sizeof(int) + 255) / 256 * 256;
  const size_t b_l = ((size_t)count * sizeof(long long) + 255) / 256 * 256;
  const size_t b_lim = ((size_t)nlev * sizeof(int) + 255) / 256 * 256;
  const size_t need = 4 * b_i + 2 * b_l + b_lim + (size_t)count * K * sizeof(int);
  CK(cudaStreamSynchronize(vs.st));
  if (need > vs.cap) {
    dev_grow((void **)&vs.buf, need, vs.st);
    vs.cap = need;
  }
  char *q = vs.buf;
  int *d_w = (int *)q; q += b_i;
  int *d_p = (int *)q; q += b_i;
  int *d_pos = (int *)q; q += b_i;
  vs.d_st = (int *)q; q += b_i;
  long long *d_b = (long long *)q; q += b_l;
  vs.d_n = (long long *)q; q += b_l;
  int *d_lim = (int *)q; q += b_lim;
  vs.d_s = (int *)q;
  std::vector<int> lim0(nlev, 0x7fffffff);
  // uploads on the verification stream (synchronous w.r.t. the host buffers)
  h2d(d_lim, lim0.data(), nlev * sizeof(int), vs.st);
  h2d(d_w, w32.data(), count * sizeof(int), vs.st);
  h2d(d_p, p32.data(), count * sizeof(int), vs.st);
  h2d(d_pos, s32.data(), count * sizeof(int), vs.st);
  h2d(d_b, node_budget, count * sizeof(long long), vs.st);
  CK(cudaStreamSynchronize(vs.st));
  const int wpb = 4;
  const size_t smem = (size_t)(((e->pool.size() + 3) & ~(size_t)3) +
                               wpb * ((rep_warp_smem_words(e->pool.data()) + 3) & ~3)) *
                      sizeof(int);
  if (smem > 48 * 1024)
    CK(cudaFuncSetAttribute(k_verify_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)smem));
  long long blocks = std::min<long long>((count + wpb - 1) / wpb, (long long)e->num_sms * 16);
  const int cancel = verify_cancel(e, count, wpb, smem);
  CK(cudaEventRecord(vs.ev0, vs.st));
  COUNT_LAUNCH();
  k_verify_warp<<<(int)blocks, 32 * wpb, smem, vs.st>>>(
      e->d_pool, e->d_assign, d_w, d_p, d_b, (int)count, icap, vs.d_st, vs.d_n, vs.d_s, d_lim,
      pmin, nlev, vs.rows, d_pos, cancel);
  CK(cudaGetLastError());
  CK(cudaEventRecord(vs.ev1, vs.st));
  return TSL_OK;
  API_END
}

int tsl_engine_verify_wait(tsl_engine *e, int slot, int32_t *status_out, int64_t *nodes_out,
                           int32_t *starts_out) {
  API_BEGIN
  if (slot < 0 || slot >= TSL_VERIFY_SLOTS) throw tsl::Error(TSL_EINVAL, "bad verify slot");
  auto &vs = e->vslot[slot];
  if (vs.count <= 0) return TSL_OK;
  CK(cudaSetDevice(e->device));
  const int K = e->pool[R_K];
  d2h(status_out, vs.d_st, vs.count * sizeof(int), vs.st);
  d2h(nodes_out, vs.d_n, vs.count * sizeof(long long), vs.st);
  d2h(starts_out, vs.d_s, (size_t)vs.count * K * sizeof(int), vs.st);
  CK(cudaStreamSynchronize(vs.st));
  CK(cudaEventElapsedTime(&e->last_ms, vs.ev0, vs.ev1));
  return TSL_OK;
  API_END
}

int tsl_engine_sat_next(tsl_engine *e, int64_t after, int64_t *widx_out, int32_t *starts_out) {
  API_BEGIN
  const int K = e->pool[R_K];
  *widx_out = -1;
  if (e->n_sat <= 0) return TSL_OK;
  if (!e->d_sat_key) {
    e->d_sat_key = (unsigned long long *)dev_take(sizeof(unsigned long long), e->stream);
    e->d_sat_next = (int *)dev_take((size_t)(K + 1) * sizeof(int), e->stream);
  }
  CK(cudaMemsetAsync(e->d_sat_key, 0xff, sizeof(unsigned long long), e->stream));
  const long long n = e->n_sat;
  const int blocks = (int)std::min<long long>((n + 255) / 256, 148);
  COUNT_LAUNCH();
  k_sat_min<<<blocks, 256, 0, e->stream>>>(e->d_sat_widx, (int)n,
                                           (int)std::min<int64_t>(after, 0x7fffffff),
                                           e->d_sat_key);
  CK(cudaGetLastError());
  COUNT_LAUNCH();
  k_sat_fetch<<<1, 64, 0, e->stream>>>(e->d_sat_key, e->d_sat_starts, K, e->d_sat_next);
  CK(cudaGetLastError());
  std::vector<int> out(K + 1);
  d2h(out.data(), e->d_sat_next, (K + 1) * sizeof(int), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  *widx_out = out[0];
  if (out[0] >= 0)
    for (int i = 0; i < K; ++i) starts_out[i] = out[1 + i];
  return TSL_OK;
  API_END
}

int tsl_engine_sat_rows(tsl_engine *e, int64_t first, int64_t count, int64_t *widx_out,
                        int32_t *starts_out) {
  API_BEGIN
  if (!e->sat_sorted) {  // legacy path: host-sorted index of the level's SAT list
    const int n_sat = (int)e->n_sat;
    std::vector<int> widx(n_sat);
    if (n_sat > 0) {
      d2h(widx.data(), e->d_sat_widx, n_sat * sizeof(int), e->stream);
      CK(cudaStreamSynchronize(e->stream));
    }
    std::vector<int> perm(n_sat);
    std::iota(perm.begin(), perm.end(), 0);
    std::sort(perm.begin(), perm.end(), [&](int x, int y) { return widx[x] < widx[y]; });
    e->sat_widx_sorted.resize(n_sat);
    e->sat_pos_sorted.resize(n_sat);
    for (int r = 0; r < n_sat; ++r) {
      e->sat_widx_sorted[r] = widx[perm[r]];
      e->sat_pos_sorted[r] = perm[r];
    }
    e->sat_sorted = true;
  }
  const long long n_sat = (long long)e->sat_widx_sorted.size();
  if (first < 0 || count < 0 || first + count > n_sat)
    throw tsl::Error(TSL_EINVAL, "SAT row range out of bounds");
  if (count == 0) return TSL_OK;
  const int K = e->pool[R_K];
  const size_t need = (size_t)count * (K + 1);
  if (need > e->d_gather_cap) {
    dev_grow((void **)&e->d_gather, need * sizeof(int), e->stream);
    e->d_gather_cap = need;
  }
  int *d_pos = e->d_gather, *d_out = e->d_gather + count;
  h2d(d_pos, e->sat_pos_sorted.data() + first, count * sizeof(int), e->stream);
  const long long total = count * K;
  COUNT_LAUNCH();
  k_gather_rows<<<(int)((total + 255) / 256), 256, 0, e->stream>>>(e->d_sat_starts, d_pos,
                                                                    (int)count, K, d_out);
  CK(cudaGetLastError());
  d2h(starts_out, d_out, total * sizeof(int), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  for (long long r = 0; r < count; ++r) widx_out[r] = e->sat_widx_sorted[first + r];
  return TSL_OK;
  API_END
}

int tsl_engine_dj(tsl_engine *e, int64_t count, const int32_t *assignments,
                  const int32_t *period, int64_t cap, int64_t budget, int mode,
                  int32_t *status_out, int64_t *nodes_out) {
  API_BEGIN
  if (count <= 0) return TSL_OK;
  e->ensure_gpu();
  CK(cudaSetDevice(e->device));
  const int K = e->pool[R_K], D = e->pool[R_D];
  for (long long i = 0; i < count; ++i)
    tsl::ck(2LL * (K - 1) * ((long long)period[i] + e->pool[R_MAXDUR]) + 4LL * e->pool[R_TOTAL],
            "period anchor");
  const int icap = cap < 0 ? -1 : (int)std::min<int64_t>(cap, tsl::VMAX - 1);
  const int wpb = 4;
  long long blocks = std::min<long long>((count + wpb - 1) / wpb, (long long)e->num_sms * 4);
  const long long warps = blocks * wpb;
  const long long gwords =
      std::max<long long>(wdj_snap_words(K, e->pool[R_NPAIR]),
                          dj_ws_words(K, D, e->pool[R_NPAIR], e->pool[R_MAXDI])) + 8;
  int *d_a = nullptr, *d_p = nullptr, *d_st = nullptr, *d_g = nullptr;
  long long *d_n = nullptr;
  DevFree guard;
  CK(cudaMalloc(&d_a, count * K * sizeof(int)));
  guard.add(d_a);
  CK(cudaMalloc(&d_p, count * sizeof(int)));
  guard.add(d_p);
  CK(cudaMalloc(&d_st, count * sizeof(int)));
  guard.add(d_st);
  CK(cudaMalloc(&d_n, count * sizeof(long long)));
  guard.add(d_n);
  CK(cudaMalloc(&d_g, warps * gwords * sizeof(int)));
  guard.add(d_g);
  h2d(d_a, assignments, count * K * sizeof(int), e->stream);
  h2d(d_p, period, count * sizeof(int), e->stream);
  const int ndep1 = e->pool[R_NDEP] > 0 ? e->pool[R_NDEP] : 1;
  const int per_warp = (wdj_smem_words(K, e->pool[R_NPAIR]) + ndep1 + D + 3) & ~3;
  const size_t smem = (((e->pool.size() + 3) & ~(size_t)3) + (size_t)wpb * per_warp) * sizeof(int);
  if (smem > 48 * 1024)
    CK(cudaFuncSetAttribute(k_dj_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  COUNT_LAUNCH();
  k_dj_batch<<<(int)blocks, 32 * wpb, smem, e->stream>>>(e->d_pool, d_a, d_p, (int)count, icap,
                                                          budget, mode, d_g, gwords, d_st, d_n);
  CK(cudaGetLastError());
  d2h(status_out, d_st, count * sizeof(int), e->stream);
  d2h(nodes_out, d_n, count * sizeof(long long), e->stream);
  CK(cudaStreamSynchronize(e->stream));
  return TSL_OK;
  API_END
}

int tsl_validate(int K, int D, const int32_t *dur, const int32_t *mem, const uint64_t *devmask,
                 int n_deps, const int32_t *deps, int N, const int32_t *starts,
                 const int64_t *init_mem, int64_t cap, int64_t P, int64_t *out_count,
                 uint64_t *sorted_keys, uint8_t *overlap_flags, uint8_t *memory_flags,
                 int64_t *runs, uint8_t *dep_flags, uint8_t *neg_flags) {
  API_BEGIN
  require_device();
  if (K < 1 || D < 1 || D > TSL_MAX_DEVICES || N < 1) throw tsl::Error(TSL_EINVAL, "bad sizes");
  std::vector<int> dptr(D + 1, 0), dst;
  long long maxE = 0;
  for (int d = 0; d < D; ++d) {
    for (int st = 0; st < K; ++st)
      if ((devmask[st] >> d) & 1) dst.push_back(st);
    dptr[d + 1] = (int)dst.size();
    maxE = std::max(maxE, (long long)(dptr[d + 1] - dptr[d]) * N);
  }
  long long want = 1;
  while (want < std::max(maxE, 1LL)) want <<= 1;
  if (P != want) throw tsl::Error(TSL_EINVAL, "P must be the next power of two >= max events/device");
  if (dst.empty()) dst.push_back(0);
  cudaStream_t s = decide_ctx_stream();
  const long long KN = (long long)K * N, DP = (long long)D * P;
  const long long nd = std::max(n_deps, 1);
  int *d_starts, *d_dptr, *d_dst, *d_dur, *d_mem, *d_deps;
  long long *d_init, *d_runs;
  unsigned long long *d_keys, *d_count;
  unsigned char *d_ov, *d_mf, *d_depf, *d_negf;
  DevFree guard;
  CK(cudaMalloc(&d_starts, KN * sizeof(int)));
  guard.add(d_starts);
  CK(cudaMalloc(&d_dptr, (D + 1) * sizeof(int)));
  guard.add(d_dptr);
  CK(cudaMalloc(&d_dst, dst.size() * sizeof(int)));
  guard.add(d_dst);
  CK(cudaMalloc(&d_dur, K * sizeof(int)));
  guard.add(d_dur);
  CK(cudaMalloc(&d_mem, K * sizeof(int)));
  guard.add(d_mem);
  CK(cudaMalloc(&d_deps, 2 * nd * sizeof(int)));
  guard.add(d_deps);
  CK(cudaMalloc(&d_init, D * sizeof(long long)));
  guard.add(d_init);
  CK(cudaMalloc(&d_runs, DP * sizeof(long long)));
  guard.add(d_runs);
  CK(cudaMalloc(&d_keys, DP * sizeof(unsigned long long)));
  guard.add(d_keys);
  CK(cudaMalloc(&d_count, sizeof(unsigned long long)));
  guard.add(d_count);
  CK(cudaMalloc(&d_ov, DP));
  guard.add(d_ov);
  CK(cudaMalloc(&d_mf, DP));
  guard.add(d_mf);
  CK(cudaMalloc(&d_depf, nd * N));
  guard.add(d_depf);
  CK(cudaMalloc(&d_negf, KN));
  guard.add(d_negf);
  h2d(d_starts, starts, KN * sizeof(int), s);
  h2d(d_dptr, dptr.data(), (D + 1) * sizeof(int), s);
  h2d(d_dst, dst.data(), dst.size() * sizeof(int), s);
  h2d(d_dur, dur, K * sizeof(int), s);
  h2d(d_mem, mem, K * sizeof(int), s);
  if (n_deps > 0) h2d(d_deps, deps, 2 * n_deps * sizeof(int), s);
  h2d(d_init, init_mem, D * sizeof(long long), s);
  CK(cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s));
  const int T = 256;
  COUNT_LAUNCH();
  k_val_keys<<<(int)((DP + T - 1) / T), T, 0, s>>>(d_starts, d_dptr, d_dst, D, N, P, d_keys);
  for (long long k = 2; k <= P; k <<= 1)
    for (long long j = k >> 1; j > 0; j >>= 1) {
      COUNT_LAUNCH();
      k_val_bitonic<<<(int)((DP + T - 1) / T), T, 0, s>>>(d_keys, DP, P, k, j);
    }
  COUNT_LAUNCH();
  k_val_scan<<<D, 1024, 0, s>>>(d_keys, d_dptr, d_dst, d_dur, d_mem, N, P, d_init, cap, d_ov,
                                d_mf, d_runs, d_count);
  const long long items = std::max(KN, nd * N);
  COUNT_LAUNCH();
  k_val_items<<<(int)((items + T - 1) / T), T, 0, s>>>(d_starts, d_dur, d_deps, n_deps, K, N,
                                                        d_depf, d_negf, d_count);
  CK(cudaGetLastError());
  unsigned long long cnt = 0;
  d2h(&cnt, d_count, sizeof cnt, s);
  CK(cudaStreamSynchronize(s));
  *out_count = (int64_t)cnt;
  if (cnt) {
    d2h(sorted_keys, d_keys, DP * sizeof(unsigned long long), s);
    d2h(overlap_flags, d_ov, DP, s);
    d2h(memory_flags, d_mf, DP, s);
    d2h(runs, d_runs, DP * sizeof(long long), s);
    if (n_deps > 0) d2h(dep_flags, d_depf, (long long)n_deps * N, s);
    d2h(neg_flags, d_negf, KN, s);
    CK(cudaStreamSynchronize(s));
  }
  return TSL_OK;
  API_END
}

void tsl_counters(int64_t *launches, int64_t *h2d_bytes, int64_t *d2h_bytes) {
  if (launches) *launches = g_launches.load();
  if (h2d_bytes) *h2d_bytes = g_h2d.load();
  if (d2h_bytes) *d2h_bytes = g_d2h.load();
}

float tsl_engine_last_kernel_ms(tsl_engine *e) { return e ? e->last_ms : 0.f; }
float tsl_engine_last_root_ms(tsl_engine *e) { return e ? e->last_root_ms : 0.f; }

void tsl_sp_stats(double *out) {
  const SpStats &s = sp_stats();
  const double v[12] = {(double)s.solves,       (double)s.rounds,       (double)s.tasks,
                        (double)s.replays,      (double)s.subsolves,    (double)s.master_nodes,
                        s.master_ms,            s.task_ms,              (double)s.pieces,
                        (double)s.undivided,    (double)s.explored,     (double)s.epochs};
  for (int i = 0; i < 12; ++i) out[i] = v[i];
}

}  // extern "C"
