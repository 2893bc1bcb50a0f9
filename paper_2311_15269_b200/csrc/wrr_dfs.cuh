// wrr_dfs.cuh — register-resident warp decide for one repetend probe.
//
// Same contract as wrx_decide on a RepView (status, lex-min witness, node
// count of kernel_c.pyx:23-508 for the probe repetend.py:160-190 builds),
// with every per-item quantity in registers: lane l owns items l and l + 32
// (S = 1 for K <= 32, S = 2 for K <= 64) and keeps their lo / hi / start,
// duration, memory delta and micro-batch index, and the item's own relation
// masks (its dependency predecessors and successors, its device partners);
// the placed / in-queue / queued sets are warp-uniform masks (32-bit for
// S = 1, 64-bit for S = 2).  No shared-memory round trip sits on the
// propagation chain:
//
//   * the FIFO queue is a sequence number per queued item; the pop is one
//     ballot (seq == head); the popped item's bounds and constants come in
//     two packed shuffles;
//   * the popped item a relaxes its edge rows lane-parallel, one lane per
//     partner b, which tests bit a of its own masks.  a's out-list (in-list)
//     is its dependency rows (partners ascending) followed by its window rows
//     (devices of a ascending, each device's stages ascending;
//     repetend.py:133-141), so the reference's sequential order is recovered
//     from two classes: a failure in the dependency class is the lowest
//     failing partner, in the window class the first failing partner in a's
//     window order (ascending for a single-device a, a precomputed "before"
//     mask for a multi-device one); rows before the failure are applied and
//     their first-improved targets enqueued in row order (ranks by
//     popcount), exactly the items the sequential loop enqueues before it
//     breaks — so the sticky in-queue flags of kernel_c.pyx:303-347 are
//     reproduced.  Duplicate window rows of a pair (partners sharing several
//     devices) carry the same lag, so only the first can change anything;
//   * placement tightening (kernel_c.pyx:279-302) in conflict order
//     (ascending), the first failing item cutting the pass and the drain
//     clearing the flags of everything queued (kernel_c.pyx:341-347);
//   * _mem_ok / _dev_ok (kernel_c.pyx:374-508) per item against every other
//     item of the device: running memory at the end of each equal-time
//     group, serial completion, the release-sorted suffix and the
//     deadline-sorted prefix energetic bounds, each as a sum / max / min over
//     the items at or after (before) an item in the stable sort order — the
//     same numbers the insertion sorts produce;
//   * per-depth snapshots: every lane stores its own (lo, hi) pair packed
//     into one word (0 <= lo, hi < 2^15, host_build.hpp R_WRR) — restoring
//     needs no synchronisation.
#pragma once
#include "models.cuh"
#include "rx_dfs.cuh"

#define WRR_FULL 0xffffffffu

namespace wrr {

template <int S>
struct Mask;
template <>
struct Mask<1> {
  typedef unsigned T;
  static __device__ __forceinline__ T ballot(bool b0, bool) { return __ballot_sync(WRR_FULL, b0); }
  static __device__ __forceinline__ int ffs(T m) { return __ffs((int)m) - 1; }
  static __device__ __forceinline__ int popc(T m) { return __popc(m); }
  static __device__ __forceinline__ T load(const int *p) { return (unsigned)p[0]; }
};
template <>
struct Mask<2> {
  typedef unsigned long long T;
  static __device__ __forceinline__ T ballot(bool b0, bool b1) {
    return (T)__ballot_sync(WRR_FULL, b0) | ((T)__ballot_sync(WRR_FULL, b1) << 32);
  }
  static __device__ __forceinline__ int ffs(T m) { return __ffsll((long long)m) - 1; }
  static __device__ __forceinline__ int popc(T m) { return __popcll(m); }
  static __device__ __forceinline__ T load(const int *p) {
    return (T)(unsigned)p[0] | ((T)(unsigned)p[1] << 32);
  }
};
template <class T>
__device__ __forceinline__ bool bit(T m, int i) { return (m >> i) & 1; }
template <class T>
__device__ __forceinline__ T one(int i) { return (T)1 << i; }
// item i's mask row (pool stores two words per row)
template <int S>
__device__ __forceinline__ typename Mask<S>::T row(const int *sp, int off, int i) {
  return Mask<S>::load(sp + sp[off] + 2 * i);
}
// value of item i (uniform) held in slot i >> 5 of lane i & 31
template <int S>
__device__ __forceinline__ int bcast(const int (&r)[S], int i) {
  const int v = (S == 2 && (i >> 5)) ? r[S - 1] : r[0];
  return __shfl_sync(WRR_FULL, v, i & 31);
}
template <int S>
__device__ __forceinline__ unsigned bcastu(const unsigned (&r)[S], int i) {
  const unsigned v = (S == 2 && (i >> 5)) ? r[S - 1] : r[0];
  return __shfl_sync(WRR_FULL, v, i & 31);
}

}  // namespace wrr

// Per-warp shared scratch: snapshots (K + 1) x 32S words, vstack K + 1 words,
// entry memory D words.
__host__ __device__ inline int wrr_smem_words(int K, int D) {
  const int S = K > 32 ? 2 : 1;
  return (K + 1) * 32 * S + (K + 1) + (D > 0 ? D : 1);
}

template <int S>
struct WrrState {
  typedef typename wrr::Mask<S>::T M;
  int lo[S], hi[S], sv[S], seq[S];
  int t[S], m[S], nb[S];
  unsigned cst[S];       // packed constants t | multi << 15 | n << 16 (popped-item broadcast)
  M pred[S], succ[S], conf[S], below[S];  // this item's relation masks
  M placed, inq, queued;
  int qh, qt;
};

// Enqueue the items of `e` in the order given by `before` (for item b: the
// items that precede it).
template <int S>
__device__ __forceinline__ void wrr_enqueue(WrrState<S> &st, typename wrr::Mask<S>::T e,
                                            const typename wrr::Mask<S>::T (&before)[S]) {
  typedef wrr::Mask<S> Mk;
  if (!e) return;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int k = 0; k < S; ++k)
    if (wrr::bit(e, 32 * k + lane)) st.seq[k] = st.qt + Mk::popc(e & before[k]);
  st.qt += Mk::popc(e);
  st.queued |= e;
  st.inq |= e;
}

// One relaxation phase of the popped item a over its out-list (OUT = true:
// lo[b] >= base + lag) or in-list (hi[b] <= base - lag).  isd / isw: this
// lane's item has a dependency / window row with a; nd[k] / nw[k]: the
// candidate bounds.  Returns false on failure (bounds of the rows before it
// applied, their targets enqueued).
template <int S, bool OUT>
__device__ __forceinline__ bool wrr_phase(WrrState<S> &st, const bool (&isd)[S],
                                          const bool (&isw)[S], const int (&nd)[S],
                                          const int (&nw)[S], const int *winb /* or null */) {
  typedef wrr::Mask<S> Mk;
  typedef typename Mk::T M;
  const int lane = threadIdx.x & 31;
  bool dfail[S], dimp[S], any[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    dimp[k] = isd[k] && (OUT ? nd[k] > st.lo[k] : nd[k] < st.hi[k]);
    dfail[k] = dimp[k] && (OUT ? nd[k] > st.hi[k] : nd[k] < st.lo[k]);
    // a window row can only act if it improves on the bound before the
    // dependency rows or the lane's dependency row acts (failures imply
    // improvements): no such lane = nothing changes in this phase
    any[k] = dimp[k] || (isw[k] && (OUT ? nw[k] > st.lo[k] : nw[k] < st.hi[k]));
  }
  if (!Mk::ballot(any[0], any[S - 1])) return true;
  const M DF = Mk::ballot(dfail[0], dfail[S - 1]);
  if (DF) {  // the lowest failing partner cuts the dependency rows
    const int f = Mk::ffs(DF);
    bool e[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const int b = 32 * k + lane;
      const bool app = dimp[k] && b < f;
      if (app) {
        if (OUT) st.lo[k] = nd[k];
        else st.hi[k] = nd[k];
      }
      e[k] = app && !wrr::bit(st.inq, b);
    }
    wrr_enqueue<S>(st, Mk::ballot(e[0], e[S - 1]), st.below);
    return false;
  }
  bool ed[S], wimp[S], wfail[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    if (dimp[k]) {
      if (OUT) st.lo[k] = nd[k];
      else st.hi[k] = nd[k];
    }
    ed[k] = dimp[k] && !wrr::bit(st.inq, 32 * k + lane);
    // window rows against the bounds after the dependency rows
    wimp[k] = isw[k] && (OUT ? nw[k] > st.lo[k] : nw[k] < st.hi[k]);
    wfail[k] = wimp[k] && (OUT ? nw[k] > st.hi[k] : nw[k] < st.lo[k]);
  }
  const M Ed = Mk::ballot(ed[0], ed[S - 1]);
  const M WF = Mk::ballot(wfail[0], wfail[S - 1]);
  M wb[S];
#pragma unroll
  for (int k = 0; k < S; ++k) wb[k] = winb && isw[k] ? Mk::load(winb + 2 * (32 * k + lane)) : st.below[k];
  M cut = ~(M)0;  // partners whose window row precedes the failure
  if (WF) {
    bool first[S];
#pragma unroll
    for (int k = 0; k < S; ++k) first[k] = wfail[k] && !(WF & wb[k]);
    const int f = Mk::ffs(Mk::ballot(first[0], first[S - 1]));
    cut = winb ? Mk::load(winb + 2 * f) : wrr::one<M>(f) - 1;
  }
  bool ew[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int b = 32 * k + lane;
    const bool app = wimp[k] && wrr::bit(cut, b);
    if (app) {
      if (OUT) st.lo[k] = nw[k];
      else st.hi[k] = nw[k];
    }
    ew[k] = app && !ed[k] && !wrr::bit(st.inq, b);
  }
  const M Ew = Mk::ballot(ew[0], ew[S - 1]);
  wrr_enqueue<S>(st, Ed, st.below);
  wrr_enqueue<S>(st, Ew, wb);
  return !WF;
}

// FIFO propagation (kernel_c.pyx:303-340) from the queued items.
template <int S>
__device__ __forceinline__ bool wrr_propagate(const int *sp, WrrState<S> &st, int P) {
  typedef wrr::Mask<S> Mk;
  typedef typename Mk::T M;
  const int lane = threadIdx.x & 31;
  const int K = sp[R_K];
  while (st.queued) {
    bool hit[S];
#pragma unroll
    for (int k = 0; k < S; ++k) hit[k] = st.seq[k] == st.qh && wrr::bit(st.queued, 32 * k + lane);
    const int a = Mk::ffs(Mk::ballot(hit[0], hit[S - 1]));
    ++st.qh;
    const M abit = ~wrr::one<M>(a);
    st.queued &= abit;
    st.inq &= abit;
    unsigned bnd[S];
#pragma unroll
    for (int k = 0; k < S; ++k) bnd[k] = (unsigned)st.lo[k] | ((unsigned)st.hi[k] << 16);
    const unsigned wa = wrr::bcastu<S>(bnd, a), ca = wrr::bcastu<S>(st.cst, a);
    const int la = (int)(wa & 0xffffu), ha = (int)(wa >> 16);
    const int ta = (int)(ca & 0x7fffu), naP = (int)(ca >> 16) * P;
    const int *winb = nullptr;
    if (ca & 0x8000u) winb = sp + sp[R_WINB] + sp[sp[R_MULTI] + a] * 2 * K;
    bool isd[S], isw[S];
    int nd[S], nw[S];
    // out rows a -> b: lag t_a - (n_a - n_b) P (dependency), t_a - P (window)
#pragma unroll
    for (int k = 0; k < S; ++k) {
      isd[k] = wrr::bit(st.pred[k], a);
      isw[k] = wrr::bit(st.conf[k], a);
      nd[k] = la + ta - naP + st.nb[k] * P;
      nw[k] = la + ta - P;
    }
    if (!wrr_phase<S, true>(st, isd, isw, nd, nw, winb)) return false;
    // in rows b -> a: hi[b] <= hi[a] - lag(b -> a)
#pragma unroll
    for (int k = 0; k < S; ++k) {
      isd[k] = wrr::bit(st.succ[k], a);
      nd[k] = ha - st.t[k] + st.nb[k] * P - naP;
      nw[k] = ha - st.t[k] + P;
    }
    if (!wrr_phase<S, false>(st, isd, isw, nd, nw, winb)) return false;
  }
  return true;
}

// _mem_ok(d) (kernel_c.pyx:374-425): events = placed items at s and unplaced
// negative-delta items at lo; the running sum after every equal-time group.
// Device item tables: per device its item mask (two words) and its items
// ascending (dev_ptr / dev_items), so the pairwise loops below have a known
// trip count and independent iterations (unrolled: shuffles overlap).
struct WrrDev {
  const int *itm, *ptr, *items;
};

template <int S>
__device__ __forceinline__ bool wrr_mem_ok(const WrrDev &dv, const WrrState<S> &st, int d,
                                           int init, int cap) {
  typedef wrr::Mask<S> Mk;
  typedef typename Mk::T M;
  if (init > cap) return false;
  const int lane = threadIdx.x & 31;
  const M items = Mk::load(dv.itm + 2 * d);
  int tt[S], dm[S], run[S];
  bool ev[S];
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int b = 32 * k + lane;
    const bool pl = wrr::bit(st.placed, b);
    ev[k] = wrr::bit(items, b) && (pl || st.m[k] < 0);
    tt[k] = pl ? st.sv[k] : st.lo[k];
    dm[k] = ev[k] ? st.m[k] : 0;
    run[k] = init;
  }
  const int pe = dv.ptr[d + 1];
#pragma unroll 4
  for (int p = dv.ptr[d]; p < pe; ++p) {
    const int j = dv.items[p];
    const int tj = wrr::bcast<S>(tt, j), dj = wrr::bcast<S>(dm, j);
#pragma unroll
    for (int k = 0; k < S; ++k) run[k] += tj <= tt[k] ? dj : 0;
  }
  bool bad[S];
#pragma unroll
  for (int k = 0; k < S; ++k) bad[k] = ev[k] && run[k] > cap;
  return !Mk::ballot(bad[0], bad[S - 1]);
}

// _dev_ok(d) (kernel_c.pyx:428-508) over the device's items in the stable
// orders (a, id) and (e, a-rank).
template <int S>
__device__ __forceinline__ bool wrr_dev_ok(const WrrDev &dv, const WrrState<S> &st, int d) {
  typedef wrr::Mask<S> Mk;
  typedef typename Mk::T M;
  const int lane = threadIdx.x & 31;
  const M items = Mk::load(dv.itm + 2 * d);
  if (!items) return true;
  int ra[S], re[S];
  unsigned pk[S];
  bool on[S];
  int suf_d[S], suf_e[S], pre_d[S], pre_a[S];
  int lim = -(1 << 30), sd = 0;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int b = 32 * k + lane;
    on[k] = wrr::bit(items, b);
    const bool pl = wrr::bit(st.placed, b);
    ra[k] = pl ? st.sv[k] : st.lo[k];
    re[k] = (pl ? st.sv[k] : st.hi[k]) + st.t[k];
    pk[k] = (unsigned)ra[k] | ((unsigned)re[k] << 16);  // a, e < 2^16
    suf_d[k] = pre_d[k] = 0;
    suf_e[k] = -(1 << 30);
    pre_a[k] = 1 << 30;
  }
  const int pe = dv.ptr[d + 1];
#pragma unroll 4
  for (int p = dv.ptr[d]; p < pe; ++p) {
    const int j = dv.items[p];
    const unsigned pj = wrr::bcastu<S>(pk, j);
    const int aj = (int)(pj & 0xffffu), ej = (int)(pj >> 16), dj = wrr::bcast<S>(st.t, j);
    lim = ej > lim ? ej : lim;
    sd += dj;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const int b = 32 * k + lane;
      // j at or after b in the stable release order (dev_items ascending)
      const bool ge = aj > ra[k] || (aj == ra[k] && j >= b);
      if (ge) {
        suf_d[k] += dj;
        suf_e[k] = ej > suf_e[k] ? ej : suf_e[k];
      }
      // j at or before b in the stable deadline order of the release-sorted list
      const bool le = ej < re[k] || (ej == re[k] && (j == b || !ge));
      if (le) {
        pre_d[k] += dj;
        pre_a[k] = aj < pre_a[k] ? aj : pre_a[k];
      }
    }
  }
  bool bad[S];
  int c = sd;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    bad[k] = on[k] && (ra[k] + suf_d[k] > suf_e[k] || pre_a[k] + pre_d[k] > re[k]);
    if (on[k]) c = ra[k] + suf_d[k] > c ? ra[k] + suf_d[k] : c;
  }
  c = __reduce_max_sync(WRR_FULL, c);
  return c <= lim && !Mk::ballot(bad[0], bad[S - 1]);
}

// The probe (assignment `asg`, period P, memory cap `cap`; -1 = none).
// Every lane calls it; returns the uniform status; *nodes_out; on SAT the
// witness is written to s_out[0..K) (if non-null).
template <int S>
__device__ int wrr_decide(const int *sp, const unsigned char *asg, int P, int cap,
                          unsigned *snap, int *vstack, int *init, long long budget,
                          unsigned long long t_end_ns, long long *nodes_out,
                          const int *abort_lim, int abort_self, int *s_out) {
  typedef wrr::Mask<S> Mk;
  typedef typename Mk::T M;
  const int K = sp[R_K], D = sp[R_D];
  const int lane = threadIdx.x & 31;
  const int anchor = (K - 1) * (P + sp[R_MAXDUR]);
  WrrState<S> st;
  const M all = K >= 32 * S ? ~(M)0 : wrr::one<M>(K) - 1;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int b = 32 * k + lane;
    const bool v = b < K;
    st.t[k] = v ? sp[sp[R_DUR] + b] : 0;
    st.m[k] = v ? sp[sp[R_MEM] + b] : 0;
    st.nb[k] = v ? (int)asg[b] : 0;
    st.cst[k] = (unsigned)st.t[k] | (v && sp[sp[R_MULTI] + b] >= 0 ? 0x8000u : 0u) |
                ((unsigned)st.nb[k] << 16);
    st.pred[k] = v ? wrr::row<S>(sp, R_PREDM, b) : 0;
    st.succ[k] = v ? wrr::row<S>(sp, R_SUCCM, b) : 0;
    st.conf[k] = v ? wrr::row<S>(sp, R_CONFM, b) : 0;
    st.below[k] = wrr::one<M>(b) - 1;
    st.lo[k] = b == 0 ? anchor : 0;
    st.hi[k] = b == 0 ? anchor : 2 * anchor;
    st.sv[k] = 0;
    st.seq[k] = b;  // root: every item queued in id order (kernel_c.pyx:158-165)
  }
  // entry memory per device (repetend.py:93-100)
  for (int d = 0; d < D; ++d) {
    const M items = wrr::row<S>(sp, R_DEVITM, d);
    int e = 0;
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (wrr::bit(items, 32 * k + lane)) e += st.m[k] * st.nb[k];
    e = __reduce_add_sync(WRR_FULL, e);
    if (lane == 0) init[d] = e;
  }
  __syncwarp();
  st.placed = 0;
  st.inq = st.queued = all;
  st.qh = 0;
  st.qt = K;
  *nodes_out = 0;
  const WrrDev dv{sp + sp[R_DEVITM], sp + sp[R_DEVPTR], sp + sp[R_DEVITEMS]};
  const int *devm = sp + sp[R_DEVM], *dur = sp + sp[R_DUR];
  if (!wrr_propagate<S>(sp, st, P)) return RX_UNSAT;
  if (cap >= 0)
    for (int d = 0; d < D; ++d)
      if (!wrr_mem_ok<S>(dv, st, d, init[d], cap)) return RX_UNSAT;
  for (int d = 0; d < D; ++d)
    if (!wrr_dev_ok<S>(dv, st, d)) return RX_UNSAT;
  if (K == 0) return RX_SAT;

  const int *order = sp + sp[R_ORDER];
  long long nodes = 0;
  int status, depth = 0;
  int v = wrr::bcast<S>(st.lo, order[0]);
  for (;;) {
    if (depth == K) {
      status = RX_SAT;
      break;
    }
    int x = order[depth];
    const int hix = wrr::bcast<S>(st.hi, x);
    if (v > hix) {  // exhausted: back to the previous depth's snapshot
      if (--depth < 0) {
        status = RX_UNSAT;
        break;
      }
      x = order[depth];
      const unsigned *sn = snap + depth * 32 * S;
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const unsigned q = sn[32 * k + lane];
        st.lo[k] = (int)(q & 0xffffu);
        st.hi[k] = (int)(q >> 16);
      }
      st.placed &= ~wrr::one<M>(x);
      v = vstack[depth] + 1;
      continue;
    }
    const int dx = dur[x];
    bool cf[S];
#pragma unroll
    for (int k = 0; k < S; ++k) cf[k] = wrr::bit(st.conf[k], x);
    for (;;) {  // conflict jump: smallest value >= v overlapping no placed partner
      int jump = -(1 << 30);
#pragma unroll
      for (int k = 0; k < S; ++k) {
        if (cf[k] && wrr::bit(st.placed, 32 * k + lane)) {
          const int ey = st.sv[k] + st.t[k];
          if (st.sv[k] - dx < v && v < ey) jump = ey > jump ? ey : jump;
        }
      }
      jump = __reduce_max_sync(WRR_FULL, jump);
      if (jump == -(1 << 30)) break;
      v = jump;
    }
    if (v > hix) continue;
    ++nodes;
    if (budget && nodes > budget) {
      status = RX_TIMEOUT;
      break;
    }
    if (t_end_ns && (nodes & 4095) == 0 && rx_now_ns() > t_end_ns) {
      status = RX_TIMEOUT;
      break;
    }
    if (abort_lim && (nodes & 255) == 0) {
      int l = 0;
      if (lane == 0) l = *(volatile const int *)abort_lim;
      l = __shfl_sync(WRR_FULL, l, 0);
      if (abort_self > l) {
        status = RX_ABORT;
        break;
      }
    }
    {
      unsigned *sn = snap + depth * 32 * S;
#pragma unroll
      for (int k = 0; k < S; ++k)
        sn[32 * k + lane] = (unsigned)st.lo[k] | ((unsigned)st.hi[k] << 16);
    }
    // place x at v; tighten its unplaced partners in ascending order
    const M xbit = wrr::one<M>(x);
    bool chg[S], fail[S], c1[S];
    int nlo[S], nhi[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const int b = 32 * k + lane;
      if (b == x) {
        st.sv[k] = v;
        st.lo[k] = v;
        st.hi[k] = v;
      }
      const bool act = cf[k] && !wrr::bit(st.placed, b);
      const int ty = st.t[k];
      c1[k] = act && v - ty < st.lo[k] && st.lo[k] < v + dx;
      nlo[k] = c1[k] ? v + dx : st.lo[k];
      const bool f1 = c1[k] && nlo[k] > st.hi[k];
      const bool c2 = act && !f1 && v - ty < st.hi[k] && st.hi[k] < v + dx;
      nhi[k] = c2 ? v - ty : st.hi[k];
      fail[k] = f1 || (c2 && nhi[k] < nlo[k]);
      chg[k] = c1[k] || c2;
      c1[k] = c1[k] && !f1;  // the lo part went through (its enqueue happened)
    }
    st.placed |= xbit;
    const M F = Mk::ballot(fail[0], fail[S - 1]);
    bool ok;
    if (F) {
      // items queued before the failing partner f: x, partners below f that
      // changed, and f itself when its lo part went through; the drain
      // clears their flags (kernel_c.pyx:341-347)
      const int f = Mk::ffs(F);
      bool q[S];
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const int b = 32 * k + lane;
        q[k] = !wrr::bit(st.inq, b) && ((b < f && chg[k]) || (b == f && c1[k]));
      }
      st.inq &= ~(Mk::ballot(q[0], q[S - 1]) | xbit);
      ok = false;
    } else {
      bool e[S];
#pragma unroll
      for (int k = 0; k < S; ++k) {
        st.lo[k] = nlo[k];
        st.hi[k] = nhi[k];
        e[k] = chg[k] && !wrr::bit(st.inq, 32 * k + lane);
        if (32 * k + lane == x) st.seq[k] = 0;
      }
      const M E = Mk::ballot(e[0], e[S - 1]);
      // queue: x first (enqueued regardless of its flag), then E ascending
      st.qh = 0;
      st.qt = 1;
      st.queued = xbit;
      st.inq |= xbit;
      wrr_enqueue<S>(st, E, st.below);
      ok = wrr_propagate<S>(sp, st, P);
      st.queued = 0;  // after a failure the leftovers keep their flags (sticky)
    }
    if (ok) {
      const M devs = Mk::load(devm + 2 * x);
      if (cap >= 0)
        for (M dm = devs; dm && ok; dm &= dm - 1) {
          const int d = Mk::ffs(dm);
          ok = wrr_mem_ok<S>(dv, st, d, init[d], cap);
        }
      for (M dm = devs; dm && ok; dm &= dm - 1) ok = wrr_dev_ok<S>(dv, st, Mk::ffs(dm));
    }
    if (ok) {
      if (lane == 0) vstack[depth] = v;
      ++depth;
      __syncwarp();
      if (depth < K) v = wrr::bcast<S>(st.lo, order[depth]);
      continue;
    }
    const unsigned *sn = snap + depth * 32 * S;
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const unsigned q = sn[32 * k + lane];
      st.lo[k] = (int)(q & 0xffffu);
      st.hi[k] = (int)(q >> 16);
    }
    st.placed &= ~xbit;
    ++v;
  }
  *nodes_out = nodes;
  if (status == RX_SAT && s_out) {
#pragma unroll
    for (int k = 0; k < S; ++k)
      if (32 * k + lane < K) s_out[32 * k + lane] = st.sv[k];
  }
  __syncwarp();
  return status;
}
