// wst_dfs.cuh — the "strong" warp search for one repetend probe.
//
// Same branching as the reference decide (kernel_c.pyx:225-371: items in π
// order, values ascending from lo, conflict jumps past placed partners, one
// node per try), but
//   * propagation runs to the full bounds fixpoint, order-free, with no
//     in-queue flags (rounds over the changed items; every lane relaxes its
//     own bounds from each changed item's broadcast bounds);
//   * placement tightening applies the reference's rule (kernel_c.pyx:
//     279-302) to every partner;
//   * the memory check is the reference's _mem_ok (kernel_c.pyx:374-425);
//   * the device check is the interval-overload test: for every pair (i, j)
//     of the device's items, the items released at or after a_i and due by
//     e_j must fit in [a_i, e_j].
//
// Why it may replace the reference's DFS for a repetend probe.  Each of
// these steps is monotone in the bounds and at least as strong as the
// reference's: full propagation reaches a fixpoint contained in any partial
// (sticky-flag) propagation from a looser state; the reference's _dev_ok
// checks (serial completion, release-sorted suffix, deadline-sorted
// prefix) each test the overload of one item set, which the interval test
// also catches on any tighter state (the set's min release and max
// deadline are attained by its members); _mem_ok and the tightening rule
// are monotone.  By induction over the search, every node of this search is
// a node of the reference's search, in the same DFS order, and both reach
// the same first solution (the lex-min one).  So with c = the nodes this
// search needs for its outcome and c_ref the reference's:
//   * SAT at c        -> the reference finds the same witness at c_ref >= c;
//   * UNSAT           -> the reference ends UNSAT or TIMEOUT (not SAT);
//   * > budget nodes  -> the reference has not found a solution within the
//                        budget either (TIMEOUT or UNSAT: not SAT).
// A repetend probe's outcome only matters as "SAT with witness" versus "not
// SAT" (repetend.py:294-299: UNSAT and a capped TIMEOUT both continue the
// scan), so this search settles every probe except a SAT found within the
// cap of a capped probe, where the reference's node count decides and the
// exact DFS (wrr_dfs.cuh) runs.  Uncapped probes (the load bound) are
// settled outright.  Node counts here are this search's, not the
// reference's (engine statistics only).
#pragma once
#include "wrr_dfs.cuh"

// Items per device for the gathered interval test (host_build.hpp R_WRR
// placements with a larger device fall back to the exact DFS).
#define WST_MAXDI 8

template <int S>
struct WstState {
  typedef typename wrr::Mask<S>::T M;
  int lo[S], hi[S], sv[S];
  int t[S], m[S], nb[S];
  unsigned cst[S];
  M pred[S], succ[S], conf[S];
  M placed;
};

// Full propagation from the changed items C: rounds until nothing changes
// (true) or a domain empties (false).
template <int S>
__device__ __forceinline__ bool wst_propagate(WstState<S> &st, typename wrr::Mask<S>::T C,
                                              int P) {
  typedef wrr::Mask<S> Mk;
  const int lane = threadIdx.x & 31;
  while (C) {
    int lo0[S], hi0[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      lo0[k] = st.lo[k];
      hi0[k] = st.hi[k];
    }
    for (typename Mk::T it = C; it; it &= it - 1) {
      const int a = Mk::ffs(it);
      const int la = wrr::bcast<S>(st.lo, a), ha = wrr::bcast<S>(st.hi, a);
      const unsigned ca = wrr::bcastu<S>(st.cst, a);
      const int ta = (int)(ca & 0x7fffu), naP = (int)(ca >> 16) * P;
#pragma unroll
      for (int k = 0; k < S; ++k) {
        const int nbP = st.nb[k] * P;
        if (wrr::bit(st.pred[k], a)) st.lo[k] = max(st.lo[k], la + ta - naP + nbP);
        if (wrr::bit(st.succ[k], a)) st.hi[k] = min(st.hi[k], ha - st.t[k] + nbP - naP);
        if (wrr::bit(st.conf[k], a)) {
          st.lo[k] = max(st.lo[k], la + ta - P);
          st.hi[k] = min(st.hi[k], ha - st.t[k] + P);
        }
      }
    }
    bool chg[S], bad[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      chg[k] = st.lo[k] != lo0[k] || st.hi[k] != hi0[k];
      bad[k] = st.lo[k] > st.hi[k];
    }
    if (Mk::ballot(bad[0], bad[S - 1])) return false;
    C = Mk::ballot(chg[0], chg[S - 1]);
  }
  return true;
}

// Interval overload on device d (<= WST_MAXDI items): lane-parallel over the
// (i, j) pairs; (a, e, d) of the device's items gathered to every lane.
template <int S>
__device__ __forceinline__ bool wst_dev_ok(const WrrDev &dv, const WstState<S> &st, int d) {
  typedef wrr::Mask<S> Mk;
  const int lane = threadIdx.x & 31;
  const int p0 = dv.ptr[d], k = dv.ptr[d + 1] - p0;
  if (k == 0) return true;
  int ra[S], re[S];
#pragma unroll
  for (int s = 0; s < S; ++s) {
    const bool pl = wrr::bit(st.placed, 32 * s + lane);
    ra[s] = pl ? st.sv[s] : st.lo[s];
    re[s] = (pl ? st.sv[s] : st.hi[s]) + st.t[s];
  }
  int ga[WST_MAXDI], ge[WST_MAXDI], gd[WST_MAXDI];
#pragma unroll
  for (int q = 0; q < WST_MAXDI; ++q) {
    if (q < k) {
      const int j = dv.items[p0 + q];
      ga[q] = wrr::bcast<S>(ra, j);
      ge[q] = wrr::bcast<S>(re, j);
      gd[q] = wrr::bcast<S>(st.t, j);
    } else {
      ga[q] = 1 << 30;  // never inside an interval
      ge[q] = -(1 << 30);
      gd[q] = 0;
    }
  }
  bool bad = false;
#pragma unroll
  for (int r = 0; r < (WST_MAXDI * WST_MAXDI + 31) / 32; ++r) {
    const int pr = lane + 32 * r;
    const int i = pr / WST_MAXDI, j = pr % WST_MAXDI;
    if (i < k && j < k) {
      int ai = 0, ej = 0;
#pragma unroll
      for (int q = 0; q < WST_MAXDI; ++q) {
        if (q == i) ai = ga[q];
        if (q == j) ej = ge[q];
      }
      int sum = 0;
#pragma unroll
      for (int q = 0; q < WST_MAXDI; ++q) sum += (ga[q] >= ai && ge[q] <= ej) ? gd[q] : 0;
      bad |= ai <= ej && sum > ej - ai;
    }
  }
  return !__any_sync(WRR_FULL, bad);
}

template <int S>
__device__ __forceinline__ bool wst_mem_ok(const WrrDev &dv, const WstState<S> &st, int d,
                                           int init, int cap) {
  WrrState<S> w;  // the reference check reads lo / sv / m / placed only
#pragma unroll
  for (int k = 0; k < S; ++k) {
    w.lo[k] = st.lo[k];
    w.sv[k] = st.sv[k];
    w.m[k] = st.m[k];
  }
  w.placed = st.placed;
  return wrr_mem_ok<S>(dv, w, d, init, cap);
}

// The probe (assignment `asg`, period P, cap; -1 = none), node budget
// (0 = none).  Returns RX_SAT (witness to s_out), RX_UNSAT, RX_TIMEOUT
// (budget exceeded) or RX_ABORT; *nodes_out = this search's nodes.
template <int S>
__device__ int wst_decide(const int *sp, const unsigned char *asg, int P, int cap,
                          unsigned *snap, int *vstack, int *init, long long budget,
                          unsigned long long t_end_ns, long long *nodes_out,
                          const int *abort_lim, int abort_self, int *s_out) {
  typedef wrr::Mask<S> Mk;
  typedef typename Mk::T M;
  const int K = sp[R_K], D = sp[R_D];
  const int lane = threadIdx.x & 31;
  const int anchor = (K - 1) * (P + sp[R_MAXDUR]);
  WstState<S> st;
  const M all = K >= 32 * S ? ~(M)0 : wrr::one<M>(K) - 1;
#pragma unroll
  for (int k = 0; k < S; ++k) {
    const int b = 32 * k + lane;
    const bool v = b < K;
    st.t[k] = v ? sp[sp[R_DUR] + b] : 0;
    st.m[k] = v ? sp[sp[R_MEM] + b] : 0;
    st.nb[k] = v ? (int)asg[b] : 0;
    st.cst[k] = (unsigned)st.t[k] | ((unsigned)st.nb[k] << 16);
    st.pred[k] = v ? wrr::row<S>(sp, R_PREDM, b) : 0;
    st.succ[k] = v ? wrr::row<S>(sp, R_SUCCM, b) : 0;
    st.conf[k] = v ? wrr::row<S>(sp, R_CONFM, b) : 0;
    st.lo[k] = b == 0 ? anchor : 0;
    st.hi[k] = b == 0 ? anchor : (v ? 2 * anchor : 0);
    st.sv[k] = 0;
  }
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
  *nodes_out = 0;
  const WrrDev dv{sp + sp[R_DEVITM], sp + sp[R_DEVPTR], sp + sp[R_DEVITEMS]};
  const int *devm = sp + sp[R_DEVM], *dur = sp + sp[R_DUR], *order = sp + sp[R_ORDER];
  if (!wst_propagate<S>(st, all, P)) return RX_UNSAT;
  if (cap >= 0)
    for (int d = 0; d < D; ++d)
      if (!wst_mem_ok<S>(dv, st, d, init[d], cap)) return RX_UNSAT;
  for (int d = 0; d < D; ++d)
    if (!wst_dev_ok<S>(dv, st, d)) return RX_UNSAT;
  if (K == 0) return RX_SAT;

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
    if (v > hix) {
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
    for (;;) {  // conflict jump (kernel_c.pyx:245-254)
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
    // place x at v and tighten every unplaced partner (kernel_c.pyx:279-302)
    const M xbit = wrr::one<M>(x);
    bool chg[S], fail[S];
#pragma unroll
    for (int k = 0; k < S; ++k) {
      const int b = 32 * k + lane;
      chg[k] = b == x;
      if (b == x) {
        st.sv[k] = v;
        st.lo[k] = v;
        st.hi[k] = v;
      }
      fail[k] = false;
      if (cf[k] && !wrr::bit(st.placed, b)) {
        const int ty = st.t[k];
        if (v - ty < st.lo[k] && st.lo[k] < v + dx) {
          st.lo[k] = v + dx;
          chg[k] = true;
        }
        if (v - ty < st.hi[k] && st.hi[k] < v + dx) {
          st.hi[k] = v - ty;
          chg[k] = true;
        }
        fail[k] = st.lo[k] > st.hi[k];
      }
    }
    st.placed |= xbit;
    bool ok = !Mk::ballot(fail[0], fail[S - 1]);
    if (ok) ok = wst_propagate<S>(st, Mk::ballot(chg[0], chg[S - 1]), P);
    if (ok) {
      const M devs = Mk::load(devm + 2 * x);
      if (cap >= 0)
        for (M dm = devs; dm && ok; dm &= dm - 1) {
          const int d = Mk::ffs(dm);
          ok = wst_mem_ok<S>(dv, st, d, init[d], cap);
        }
      for (M dm = devs; dm && ok; dm &= dm - 1) ok = wst_dev_ok<S>(dv, st, Mk::ffs(dm));
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
