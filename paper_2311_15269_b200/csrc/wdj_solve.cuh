// wdj_solve.cuh — warp-cooperative disjunctive refutation (one probe per warp).
//
// Decides the same question as dj_solve.cuh (is the repetend probe of
// repetend.py:160-190 feasible at all: anchored box, dependency and
// device-window difference edges, exclusivity of items with intersecting
// device masks, per-device running memory <= cap) by branching on the ORDER
// of each conflicting pair, with all 32 lanes sharing each step:
//   * propagation = rounds in which lanes relax the difference edges (lanes
//     over edge rows), the oriented pairs as precedence edges and the
//     detectable precedences of unoriented pairs (lanes over pairs), with
//     atomicMax / atomicMin on shared bounds, until a round changes nothing.
//     Any order of these monotone, sound rules reaches the same kind of
//     verdict: a failure (lo > hi, or a pair impossible both ways) is a proof;
//     bounds still moving K+1 rounds after the last new orientation prove a
//     positive cycle in a fixed difference system;
//   * memory: once every pair on a device is oriented its items are totally
//     ordered by lo (distinct: oriented x->y forces lo[y] >= lo[x] + t_x), so
//     the running memory at item i is init + sum of mem[j] over lo[j] <= lo[i];
//   * branching: the unoriented pair of smallest slack (lowest index on
//     ties), preferred side first — the same rule as dj_solve.cuh;
//   * per-depth snapshots of bounds and orientation bits in global memory
//     (coalesced copies), restored before a frame's second orientation.
// Used only as a FILTER: DJ_UNSAT proves the probe has no solution, which the
// reference's period scan treats like its own node-capped TIMEOUT or UNSAT
// (repetend.py:289-302).  SAT / undecided probes go to the reference-exact
// RX-DFS.
#pragma once
#include "dj_solve.cuh"
#include "wrx_dfs.cuh"

struct WdjWs {
  int *lo, *hi, *av;       // shared: bounds, candidate assignment
  unsigned *ox, *oy;       // shared: orientation bits (x before y / y before x)
  int *f_pid, *f_pref, *f_tried;  // shared: DFS frames
  int *snap;               // global: per depth 2K + 2NW words
};

__host__ __device__ inline int wdj_nw(int npair) { return (npair > 0 ? npair : 1) / 32 + 1; }
// shared words per warp
__host__ __device__ inline int wdj_smem_words(int K, int npair) {
  const int k = K > 0 ? K : 1, np = npair > 0 ? npair : 1;
  return 3 * k + 2 * wdj_nw(npair) + 3 * (np + 1);
}
// global snapshot words per warp
__host__ __device__ inline long long wdj_snap_words(int K, int npair) {
  const long long k = K > 0 ? K : 1, np = npair > 0 ? npair : 1;
  return (np + 2) * (2 * k + 2 * wdj_nw(npair));
}

__device__ inline WdjWs wdj_carve(int *smem, int *gsnap, int K, int npair) {
  const int k = K > 0 ? K : 1, np = npair > 0 ? npair : 1, nw = wdj_nw(npair);
  WdjWs w;
  int *p = smem;
  w.lo = p; p += k;
  w.hi = p; p += k;
  w.av = p; p += k;
  w.ox = (unsigned *)p; p += nw;
  w.oy = (unsigned *)p; p += nw;
  w.f_pid = p; p += np + 1;
  w.f_pref = p; p += np + 1;
  w.f_tried = p;
  w.snap = gsnap;
  return w;
}

struct WdjCtx {
  const int *rsrc, *rdst, *rbase, *pairx, *pairy, *dur, *mem, *dpptr, *dp, *devptr, *devitems;
  const int *init, *rowcm, *paircm;
  int K, D, m, ndep, npair, nw, P, cap;
};

__device__ __forceinline__ unsigned long long wdj_u64(const int *p) {
  return (unsigned long long)(unsigned)p[0] | ((unsigned long long)(unsigned)p[1] << 32);
}
__device__ __forceinline__ unsigned long long wdj_ibit(int i) {
  return i < 64 ? 1ull << i : ~0ull;
}

__device__ __forceinline__ bool wdj_bit(const unsigned *b, int q) {
  return (b[q >> 5] >> (q & 31)) & 1u;
}

// Propagate to a fixpoint of the sound rules; false = infeasible.  `cur`:
// the items whose bounds or pair orientations changed since the last
// fixpoint (all at the root, the branched pair's two items after an
// orientation); each round relaxes only the 32-row / 32-pair chunks that
// touch a changed item (R_ROWCM / R_PAIRCM) — a row or pair none of whose
// items changed cannot change anything — and collects the items it changed
// for the next round.
#ifdef WDJ_COUNT_ROUNDS  // scripts/dj_rounds.py: propagation statistics
__device__ unsigned long long g_wdj_rounds, g_wdj_calls, g_wdj_rows, g_wdj_pairs;
#endif
__device__ inline bool wdj_propagate(const WdjCtx &c, WdjWs &w, unsigned long long cur) {
  const int lane = wrx_lane();
  int quiet = 0;  // rounds since the last new orientation
#ifdef WDJ_COUNT_ROUNDS
  if (lane == 0) atomicAdd(&g_wdj_calls, 1ull);
#endif
  for (;;) {
#ifdef WDJ_COUNT_ROUNDS
    if (lane == 0) {
      atomicAdd(&g_wdj_rounds, 1ull);
      unsigned long long rc = 0, pc = 0;
      for (int base = 0; base < c.m; base += 32) rc += (wdj_u64(c.rowcm + 2 * (base >> 5)) & cur) != 0;
      for (int base = 0; base < c.npair; base += 32) pc += (wdj_u64(c.paircm + 2 * (base >> 5)) & cur) != 0;
      atomicAdd(&g_wdj_rows, rc);
      atomicAdd(&g_wdj_pairs, pc);
    }
#endif
    bool oriented = false, fail = false;
    unsigned long long mine = 0;
    for (int base = 0; base < c.m; base += 32) {
      if (!(wdj_u64(c.rowcm + 2 * (base >> 5)) & cur)) continue;
      const int r = base + lane;
      if (r >= c.m) continue;
      const int s = c.rsrc[r], d = c.rdst[r];
      const int lag = c.rbase[r] - (r < c.ndep ? w.av[s] - w.av[d] : 1) * c.P;
      const int nl = w.lo[s] + lag;
      if (nl > w.lo[d]) {
        atomicMax(&w.lo[d], nl);
        mine |= wdj_ibit(d);
      }
      const int nh = w.hi[d] - lag;
      if (nh < w.hi[s]) {
        atomicMin(&w.hi[s], nh);
        mine |= wdj_ibit(s);
      }
    }
    for (int base = 0; base < c.npair; base += 32) {
      if (!(wdj_u64(c.paircm + 2 * (base >> 5)) & cur)) continue;
      const int q = base + lane;
      if (q >= c.npair) continue;
      const int x = c.pairx[q], y = c.pairy[q];
      bool xf = wdj_bit(w.ox, q), yf = wdj_bit(w.oy, q);
      if (!xf && !yf) {
        const bool can_xy = w.lo[x] + c.dur[x] <= w.hi[y];
        const bool can_yx = w.lo[y] + c.dur[y] <= w.hi[x];
        if (!can_xy && !can_yx) {
          fail = true;
          continue;
        }
        if (can_xy && can_yx) continue;
        xf = can_xy;
        yf = !can_xy;
        atomicOr(xf ? &w.ox[q >> 5] : &w.oy[q >> 5], 1u << (q & 31));
        oriented = true;
      }
      const int a = xf ? x : y, b = xf ? y : x;  // a before b
      const int nl = w.lo[a] + c.dur[a];
      if (nl > w.lo[b]) {
        atomicMax(&w.lo[b], nl);
        mine |= wdj_ibit(b);
      }
      const int nh = w.hi[b] - c.dur[a];
      if (nh < w.hi[a]) {
        atomicMin(&w.hi[a], nh);
        mine |= wdj_ibit(a);
      }
    }
    __syncwarp();
    for (int i = lane; i < c.K; i += 32) fail |= w.lo[i] > w.hi[i];
    if (__any_sync(WRX_FULL, fail)) return false;
    const bool any_or = __any_sync(WRX_FULL, oriented);
    cur = (unsigned long long)__reduce_or_sync(WRX_FULL, (unsigned)mine) |
          ((unsigned long long)__reduce_or_sync(WRX_FULL, (unsigned)(mine >> 32)) << 32);
    if (!cur && !any_or) return true;
    quiet = any_or ? 0 : quiet + 1;
    if (quiet > c.K + 1) return false;  // positive cycle in a fixed difference system
  }
}

// running memory of every device whose pairs are all oriented (lane per device)
__device__ inline bool wdj_mem_ok(const WdjCtx &c, const WdjWs &w) {
  if (c.cap < 0) return true;
  const int lane = wrx_lane();
  bool bad = false;
  for (int d = lane; d < c.D; d += 32) {
    bool complete = true;
    for (int p = c.dpptr[d]; p < c.dpptr[d + 1] && complete; ++p) {
      const int q = c.dp[p];
      complete = wdj_bit(w.ox, q) || wdj_bit(w.oy, q);
    }
    if (!complete) continue;
    const int run0 = c.init[d];
    if (run0 > c.cap) {
      bad = true;
      continue;
    }
    for (int p = c.devptr[d]; p < c.devptr[d + 1] && !bad; ++p) {
      const int i = c.devitems[p], li = w.lo[i];
      int run = run0;
      for (int p2 = c.devptr[d]; p2 < c.devptr[d + 1]; ++p2) {
        const int j = c.devitems[p2];
        if (w.lo[j] <= li) run += c.mem[j];
      }
      bad = run > c.cap;
    }
  }
  return !__any_sync(WRX_FULL, bad);
}

__device__ inline void wdj_save(const WdjCtx &c, WdjWs &w, int depth) {
  const int lane = wrx_lane();
  int *sn = w.snap + (long long)depth * (2 * c.K + 2 * c.nw);
  for (int i = lane; i < c.K; i += 32) {
    sn[i] = w.lo[i];
    sn[c.K + i] = w.hi[i];
  }
  for (int i = lane; i < c.nw; i += 32) {
    sn[2 * c.K + i] = (int)w.ox[i];
    sn[2 * c.K + c.nw + i] = (int)w.oy[i];
  }
  __syncwarp();
}

__device__ inline void wdj_restore(const WdjCtx &c, WdjWs &w, int depth) {
  const int lane = wrx_lane();
  const int *sn = w.snap + (long long)depth * (2 * c.K + 2 * c.nw);
  for (int i = lane; i < c.K; i += 32) {
    w.lo[i] = sn[i];
    w.hi[i] = sn[c.K + i];
  }
  for (int i = lane; i < c.nw; i += 32) {
    w.ox[i] = (unsigned)sn[2 * c.K + i];
    w.oy[i] = (unsigned)sn[2 * c.K + c.nw + i];
  }
  __syncwarp();
}

// w.lo / w.hi / w.av hold the probe's initial box and assignment (written by
// the caller, visible after __syncwarp).  Returns DJ_SAT / DJ_UNSAT /
// DJ_UNKNOWN; *nodes_out = orientation tries (uniform across the warp).
__device__ inline int wdj_decide(const int *pool, int P, int cap, const int *init, WdjWs &w,
                                 long long budget, long long *nodes_out) {
  const int lane = wrx_lane();
  WdjCtx c;
  c.K = pool[R_K];
  c.D = pool[R_D];
  c.m = pool[R_M];
  c.ndep = pool[R_NDEP];
  c.npair = pool[R_NPAIR];
  c.nw = wdj_nw(c.npair);
  c.P = P;
  c.cap = cap;
  c.rsrc = pool + pool[R_RSRC];
  c.rdst = pool + pool[R_RDST];
  c.rbase = pool + pool[R_RBASE];
  c.pairx = pool + pool[R_PAIRX];
  c.pairy = pool + pool[R_PAIRY];
  c.dur = pool + pool[R_DUR];
  c.mem = pool + pool[R_MEM];
  c.dpptr = pool + pool[R_DPPTR];
  c.dp = pool + pool[R_DP];
  c.devptr = pool + pool[R_DEVPTR];
  c.devitems = pool + pool[R_DEVITEMS];
  c.init = init;
  c.rowcm = pool + pool[R_ROWCM];
  c.paircm = pool + pool[R_PAIRCM];
  *nodes_out = 0;
  for (int i = lane; i < c.nw; i += 32) w.ox[i] = w.oy[i] = 0u;
  __syncwarp();
  if (cap >= 0) {
    bool bad = false;
    for (int d = lane; d < c.D; d += 32) bad |= init[d] > cap;
    if (__any_sync(WRX_FULL, bad)) return DJ_UNSAT;
  }
  if (!wdj_propagate(c, w, ~0ull) || !wdj_mem_ok(c, w)) return DJ_UNSAT;
  long long nodes = 0;
  int depth = 0;
  bool descend = true;
  for (;;) {
    if (descend) {
      // most constrained unoriented pair: smallest slack of its tighter side
      int bs = 0x7fffffff, bq = 0x7fffffff, bp = 1;
      for (int q = lane; q < c.npair; q += 32) {
        if (wdj_bit(w.ox, q) || wdj_bit(w.oy, q)) continue;
        const int x = c.pairx[q], y = c.pairy[q];
        const int sxy = w.hi[y] - (w.lo[x] + c.dur[x]);
        const int syx = w.hi[x] - (w.lo[y] + c.dur[y]);
        const int s = sxy < syx ? sxy : syx;
        if (s < bs) {  // q ascending per lane: keeps the lowest index on ties
          bs = s;
          bq = q;
          bp = sxy >= syx ? 1 : 2;
        }
      }
      // slacks are bounded by the box (|s| < 2^30): shift to unsigned order
      const unsigned key = bq == 0x7fffffff ? 0xffffffffu : (unsigned)(bs + (1 << 30));
      const unsigned kmin = __reduce_min_sync(WRX_FULL, key);
      if (kmin == 0xffffffffu) {
        *nodes_out = nodes;
        return DJ_SAT;
      }
      const unsigned qmin = __reduce_min_sync(WRX_FULL, key == kmin ? (unsigned)bq : 0xffffffffu);
      const int owner = (int)(qmin & 31u);  // pair q is scanned by lane q % 32
      const int pref = __shfl_sync(WRX_FULL, bp, owner);
      if (lane == 0) {
        w.f_pid[depth] = (int)qmin;
        w.f_pref[depth] = pref;
        w.f_tried[depth] = 0;
      }
      wdj_save(c, w, depth);
      descend = false;
    }
    const int tried = w.f_tried[depth];
    if (tried == 2) {
      if (--depth < 0) {
        *nodes_out = nodes;
        return DJ_UNSAT;
      }
      continue;
    }
    if (tried == 1) wdj_restore(c, w, depth);
    const int pref = w.f_pref[depth], pid = w.f_pid[depth];
    const int o = tried == 0 ? pref : 3 - pref;
    __syncwarp();
    if (lane == 0) {
      w.f_tried[depth] = tried + 1;
      atomicOr(o == 1 ? &w.ox[pid >> 5] : &w.oy[pid >> 5], 1u << (pid & 31));
    }
    __syncwarp();
    if (++nodes > budget && budget) {
      *nodes_out = nodes;
      return DJ_UNKNOWN;
    }
    if (wdj_propagate(c, w, wdj_ibit(c.pairx[pid]) | wdj_ibit(c.pairy[pid])) && wdj_mem_ok(c, w)) {
      ++depth;
      descend = true;
    }
  }
}
