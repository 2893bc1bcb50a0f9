// wrx_dfs.cuh — warp-cooperative reference-exact decide (one probe per warp).
//
// Same semantics as rx_dfs.cuh / kernel_c.pyx (status, lex-min witness, node
// count) with the 32 lanes sharing each step:
//   * FIFO propagation keeps ONE popped item at a time (the reference order),
//     but relaxes its out-/in-edges lane-parallel.  Per chunk of 32 edges the
//     first failing edge f is found by ballot; edges before f are applied
//     (atomicMax / atomicMin on shared bounds) and their targets enqueued in
//     edge order, each target once at its first improving edge
//     (__match_any_sync + prefix popcount) — exactly the items the
//     sequential loop would have enqueued before returning on edge f, so the
//     sticky-flag behaviour of kernel_c.pyx:303-347 is preserved;
//   * conflict jump / tightening of conf(x) lane-parallel (kernel_c.pyx:
//     245-302); a tightening failure drains the queue like kernel_c.pyx:341;
//   * _mem_ok / _dev_ok lane-parallel: rank-based evaluation of the same
//     stable orders (a, position) and (e, a-rank) as the insertion sorts of
//     kernel_c.pyx:374-508 (the verdict of each check does not depend on how
//     the order is computed);
//   * per-depth lo/hi snapshots copied by all lanes.
#pragma once
#include "rx_dfs.cuh"

#define WRX_FULL 0xffffffffu

struct WWs {
  int *lo, *hi, *s, *queue, *vstack;
  unsigned *placed, *inq;
  int2 *snap;                 // (n + 1) x n (lo, hi) per depth
  int *ev_a, *ev_d, *ev_e, *ev_k;  // device-check scratch (maxdi each)
};

// words of shared/global scratch for a problem (snapshots counted separately)
__host__ __device__ inline int wrx_state_words(int n, int maxdi) {
  const int nn = n > 0 ? n : 1, md = maxdi > 0 ? maxdi : 1;
  return 4 * nn + (nn + 1) + 2 * ((nn + 31) / 32) + 4 * md;
}
__host__ __device__ inline long long wrx_snap_words(int n) {
  const long long nn = n > 0 ? n : 1;
  return 2 * (nn + 1) * nn;
}

__device__ inline WWs wrx_carve(int *state, int *snap, int n, int maxdi) {
  const int nn = n > 0 ? n : 1, md = maxdi > 0 ? maxdi : 1, nw = (nn + 31) / 32;
  WWs w;
  int *p = state;
  w.lo = p; p += nn;
  w.hi = p; p += nn;
  w.s = p; p += nn;
  w.queue = p; p += nn;
  w.vstack = p; p += nn + 1;
  w.placed = (unsigned *)p; p += nw;
  w.inq = (unsigned *)p; p += nw;
  w.ev_a = p; p += md;
  w.ev_d = p; p += md;
  w.ev_e = p; p += md;
  w.ev_k = p;
  w.snap = (int2 *)snap;
  return w;
}

__device__ __forceinline__ int wrx_lane() { return threadIdx.x & 31; }
__device__ __forceinline__ bool wrx_bit(const unsigned *m, int i) {
  return (m[i >> 5] >> (i & 31)) & 1u;
}

// Append the lanes flagged in `cand` (keys b) to the FIFO in lane order,
// once per distinct b (its lowest flagged lane), setting their inq bits.
// `dedup` = the chunk may hold the same target twice (duplicated edge rows);
// without it every candidate lane is its own leader (no __match_any_sync).
__device__ __forceinline__ void wrx_enqueue(WWs &w, bool cand, int b, int n, int &qt, int &qc,
                                            bool dedup = true) {
  const int lane = wrx_lane();
  __syncwarp();  // bound updates of this chunk visible before the next reads
  const unsigned candm = __ballot_sync(WRX_FULL, cand);
  if (!candm) return;
  bool leader = cand;
  unsigned leadm = candm;
  if (dedup) {
    const unsigned grp = __match_any_sync(WRX_FULL, cand ? b : -1 - lane);
    leader = cand && (__ffs(grp) - 1 == lane);
    leadm = __ballot_sync(WRX_FULL, leader);
  }
  if (leader) {
    int slot = qt + __popc(leadm & ((1u << lane) - 1u));
    if (slot >= n) slot -= n;
    w.queue[slot] = b;
    atomicOr(&w.inq[b >> 5], 1u << (b & 31));
  }
  const int cnt = __popc(leadm);
  qt += cnt;
  if (qt >= n) qt -= n;
  qc += cnt;
  __syncwarp();
}

template <class M>
__device__ bool wrx_propagate(const M &md, WWs &w, int &qh, int &qt, int &qc) {
  const int n = md.n();
  const int lane = wrx_lane();
  while (qc > 0) {
    const int a = w.queue[qh];
    if (++qh == n) qh = 0;
    --qc;
    if (lane == 0) atomicAnd(&w.inq[a >> 5], ~(1u << (a & 31)));
    __syncwarp();
    const int la = w.lo[a], ha = w.hi[a];
    const int ob = md.out_begin(a), no = md.out_end(a) - ob;
    const int ib = md.in_begin(a), ni = md.in_end(a) - ib;
    if (no + ni <= 32 && !md.out_dup(a) && !md.in_dup(a)) {
      // one chunk: lanes [0, no) relax the out-edges, lanes [no, no + ni) the
      // in-edges.  Out-edges only raise lo and in-edges only lower hi, so the
      // sequential order is kept by (1) out failures (nl > hi[b]) against
      // the entry hi, (2) the out updates applied, (3) in failures
      // (nh < lo[b]) against the updated lo, (4) one enqueue in lane order
      // (= out-edge order, then in-edge order).  Neither list repeats a node;
      // a node on both lists (in_twin) is enqueued by its out-lane if that
      // lane enqueues it — the sequential in-edge would then find it queued.
      const bool is_out = lane < no, is_in = !is_out && lane < no + ni;
      int b = 0, nv = 0, lob = 0, hib = 0, tw = -1;
      bool inq = true;
      if (is_out) {
        const int p = ob + lane;
        b = md.out_dst(p);
        nv = la + (p < md.out_dep_end(a) ? md.out_dep_lag(p) : md.out_win_lag(a));
        lob = w.lo[b];
      } else if (is_in) {
        const int p = ib + lane - no;
        b = md.in_src(p);
        nv = ha - (p < md.in_dep_end(a) ? md.in_dep_lag(p) : md.in_win_lag(p));
        tw = md.in_twin(p);
      }
      if (is_out || is_in) {
        hib = w.hi[b];
        inq = wrx_bit(w.inq, b);
      }
      const unsigned failo = __ballot_sync(WRX_FULL, is_out && nv > hib);
      const int fo = failo ? __ffs(failo) - 1 : 32;
      const bool impo = is_out && lane < fo && nv > lob;
      __syncwarp();
      if (impo) atomicMax(&w.lo[b], nv);
      if (failo) {
        wrx_enqueue(w, impo && !inq, b, n, qt, qc, false);
        return false;
      }
      const unsigned ocand = __ballot_sync(WRX_FULL, impo && !inq);
      __syncwarp();  // the out updates visible to the in-lanes
      if (is_in) lob = w.lo[b];
      const unsigned faili = __ballot_sync(WRX_FULL, is_in && nv < lob);
      const int fi = faili ? __ffs(faili) - 1 : 32;
      const bool impi = is_in && lane < fi && nv < hib;
      if (impi) atomicMin(&w.hi[b], nv);
      const bool twin_q = tw >= 0 && ((ocand >> tw) & 1u);
      wrx_enqueue(w, (impo || (impi && !twin_q)) && !inq, b, n, qt, qc, false);
      if (faili) return false;
      continue;
    }
    // out-edges: lo[b] >= lo[a] + lag
    {
      const int pb = md.out_begin(a), pe = md.out_end(a), od = md.out_dep_end(a);
      const int owl = md.out_win_lag(a);
      for (int base = pb; base < pe; base += 32) {
        const int p = base + lane;
        const bool act = p < pe;
        int b = 0, nl = 0, lob = 0, hib = 0;
        bool inq = true;
        if (act) {
          b = md.out_dst(p);
          nl = la + (p < od ? md.out_dep_lag(p) : owl);
          lob = w.lo[b];
          hib = w.hi[b];
          inq = wrx_bit(w.inq, b);
        }
        const unsigned failm = __ballot_sync(WRX_FULL, act && nl > hib);
        const int f = failm ? __ffs(failm) - 1 : 32;
        const bool imp = act && lane < f && nl > lob;
        __syncwarp();
        if (imp) atomicMax(&w.lo[b], nl);
        wrx_enqueue(w, imp && !inq, b, n, qt, qc, md.out_dup(a));
        if (failm) return false;
      }
    }
    // in-edges: hi[b] <= hi[a] - lag
    {
      const int pb = md.in_begin(a), pe = md.in_end(a), id = md.in_dep_end(a);
      for (int base = pb; base < pe; base += 32) {
        const int p = base + lane;
        const bool act = p < pe;
        int b = 0, nh = 0, lob = 0, hib = 0;
        bool inq = true;
        if (act) {
          b = md.in_src(p);
          nh = ha - (p < id ? md.in_dep_lag(p) : md.in_win_lag(p));
          lob = w.lo[b];
          hib = w.hi[b];
          inq = wrx_bit(w.inq, b);
        }
        const unsigned failm = __ballot_sync(WRX_FULL, act && nh < lob);
        const int f = failm ? __ffs(failm) - 1 : 32;
        const bool imp = act && lane < f && nh < hib;
        __syncwarp();
        if (imp) atomicMin(&w.hi[b], nh);
        wrx_enqueue(w, imp && !inq, b, n, qt, qc, md.in_dup(a));
        if (failm) return false;
      }
    }
  }
  return true;
}


// ---- warp sort / scan helpers (one element per lane, 32 lanes) --------
// W = power-of-two width (8, 16 or 32): sorts every aligned group of W lanes
__device__ __forceinline__ void wrx_bitonic(unsigned long long &key, int &p0, int &p1,
                                            int W = 32) {
  const int lane = wrx_lane();
  for (int size = 2; size <= W; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long pk = __shfl_xor_sync(WRX_FULL, key, stride);
      const int q0 = __shfl_xor_sync(WRX_FULL, p0, stride);
      const int q1 = __shfl_xor_sync(WRX_FULL, p1, stride);
      const bool up = (lane & size) == 0, lower = (lane & stride) == 0;
      const bool take = (lower == up) ? (pk < key) : (pk > key);
      if (take) {
        key = pk;
        p0 = q0;
        p1 = q1;
      }
    }
  }
}
// scans over W lanes: exact for lanes < W when lanes >= k hold identities
__device__ __forceinline__ int wrx_scan_add(int v, int W = 32) {  // inclusive prefix sum
  const int lane = wrx_lane();
  for (int o = 1; o < W; o <<= 1) {
    const int t = __shfl_up_sync(WRX_FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}
__device__ __forceinline__ int wrx_rscan_add(int v, int W = 32) {  // inclusive suffix sum
  const int lane = wrx_lane();
  for (int o = 1; o < W; o <<= 1) {
    const int t = __shfl_down_sync(WRX_FULL, v, o);
    if (lane + o < 32) v += t;
  }
  return v;
}
__device__ __forceinline__ int wrx_rscan_max(int v, int W = 32) {
  const int lane = wrx_lane();
  for (int o = 1; o < W; o <<= 1) {
    const int t = __shfl_down_sync(WRX_FULL, v, o);
    if (lane + o < 32) v = t > v ? t : v;
  }
  return v;
}
__device__ __forceinline__ int wrx_scan_min(int v, int W = 32) {
  const int lane = wrx_lane();
  for (int o = 1; o < W; o <<= 1) {
    const int t = __shfl_up_sync(WRX_FULL, v, o);
    if (lane >= o) v = t < v ? t : v;
  }
  return v;
}
// order-preserving 64-bit key from (value, tie) with value in (-2^30, 2^30)
__device__ __forceinline__ unsigned long long wrx_key(int v, int tie) {
  return ((unsigned long long)(unsigned)(v + (1 << 30)) << 32) | (unsigned)tie;
}

// _mem_ok for a device with k <= 32 items: sort events by time, prefix sums,
// check the running sum at the end of every equal-time group.
template <class M>
__device__ bool wrx_mem_ok32(const M &md, WWs &w, int d, int cap, int pb, int k, int W) {
  const int lane = wrx_lane();
  const int init = md.init_mem(d);
  unsigned long long key = ~0ull;
  int m = 0, dummy = 0;
  if (lane < k) {
    const int it = md.dev_item(pb + lane);
    const int mm = md.mem(it);
    const bool pl = wrx_bit(w.placed, it);
    if (pl || mm < 0) {
      key = wrx_key(pl ? w.s[it] : w.lo[it], lane);
      m = mm;
    }
  }
  wrx_bitonic(key, m, dummy, W);
  const int run = init + wrx_scan_add(m, W);
  const unsigned long long nkey = __shfl_down_sync(WRX_FULL, key, 1);
  const bool valid = key != ~0ull;
  const bool group_end = valid && (lane == 31 || nkey == ~0ull || (nkey >> 32) != (key >> 32));
  return !__any_sync(WRX_FULL, group_end && run > cap);
}

// _dev_ok for a device with k <= 32 items: stable orders (a, position) and
// (e, a-rank) by bitonic sorts; serial completion, suffix and prefix
// energetic checks by scans.
template <class M>
__device__ bool wrx_dev_ok32(const M &md, WWs &w, int pb, int k, int W) {
  const int lane = wrx_lane();
  const bool real = lane < k;
  int a = 0, du = 0, e = -(1 << 30);
  if (real) {
    const int it = md.dev_item(pb + lane);
    du = md.dur(it);
    const bool pl = wrx_bit(w.placed, it);
    a = pl ? w.s[it] : w.lo[it];
    e = pl ? a + du : w.hi[it] + du;
  }
  const int lim = __reduce_max_sync(WRX_FULL, e);
  const int sd = __reduce_add_sync(WRX_FULL, du);
  unsigned long long key = real ? wrx_key(a, lane) : ~0ull;
  int pd = du, pe = e;
  wrx_bitonic(key, pd, pe, W);  // lane = rank in the stable a-order
  const bool r2 = key != ~0ull;
  const int ra = (int)(key >> 32) - (1 << 30);
  const int suf_d = wrx_rscan_add(pd, W);
  const int suf_e = wrx_rscan_max(pe, W);
  bool bad = r2 && (ra + suf_d > suf_e);
  int c = r2 ? ra + suf_d : sd;
  c = __reduce_max_sync(WRX_FULL, c > sd ? c : sd);
  bad |= c > lim;
  // stable e-order of the a-sorted sequence: key (e, a-rank)
  unsigned long long key2 = r2 ? wrx_key(pe, lane) : ~0ull;
  int qa = r2 ? ra : (1 << 30), qd = r2 ? pd : 0;
  wrx_bitonic(key2, qa, qd, W);
  const bool r3 = key2 != ~0ull;
  const int qe = (int)(key2 >> 32) - (1 << 30);
  const int pre_d = wrx_scan_add(qd, W);
  const int pre_a = wrx_scan_min(qa, W);
  bad |= r3 && (pre_a + pre_d > qe);
  return !__any_sync(WRX_FULL, bad);
}

// device checks ---------------------------------------------------------
// Load the device's items into the scratch arrays: a (release), d (dur),
// e (deadline) for _dev_ok, or time/delta/event-flag for _mem_ok.

template <class M>
__device__ bool wrx_mem_ok(const M &md, WWs &w, int d, int cap) {
  const int init = md.init_mem(d);
  if (init > cap) return false;
  const int pb = md.dev_begin(d), k = md.dev_end(d) - pb;
  // small devices: the O(k^2) shared-memory form measured faster than a sort
  if (k > 8 && k <= 32) return wrx_mem_ok32(md, w, d, cap, pb, k, k <= 16 ? 16 : 32);
  const int lane = wrx_lane();
  if (k <= 8) {
    // all (i, j) pairs in registers: lane = 8 * (i mod 4) + j, rows i and
    // i + 4 in two passes; run(i) = init + sum of delta_j over events j with
    // time_j <= time_i (delta_j = 0 for non-events), reduced over the 8 lanes
    // of a row by xor shuffles
    const int j = lane & 7;
    int tj = 0, dj = 0;
    bool evj = false;
    if (j < k) {
      const int it = md.dev_item(pb + j);
      const int m = md.mem(it);
      const bool pl = wrx_bit(w.placed, it);
      evj = pl || m < 0;
      tj = pl ? w.s[it] : w.lo[it];
      dj = evj ? m : 0;
    }
    bool bad = false;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = (lane >> 3) + 4 * h;
      const int ti = __shfl_sync(WRX_FULL, tj, i);
      const bool evi = __shfl_sync(WRX_FULL, evj, i);
      int c = (j < k && tj <= ti) ? dj : 0;
      c += __shfl_xor_sync(WRX_FULL, c, 1);
      c += __shfl_xor_sync(WRX_FULL, c, 2);
      c += __shfl_xor_sync(WRX_FULL, c, 4);
      bad |= i < k && evi && init + c > cap;
    }
    return !__any_sync(WRX_FULL, bad);
  }
  for (int i = lane; i < k; i += 32) {
    const int it = md.dev_item(pb + i);
    const int m = md.mem(it);
    const bool pl = wrx_bit(w.placed, it);
    const bool ev = pl || m < 0;
    w.ev_a[i] = pl ? w.s[it] : w.lo[it];
    w.ev_d[i] = ev ? m : 0;
    w.ev_k[i] = ev;
  }
  __syncwarp();
  bool bad = false;
  for (int i = lane; i < k; i += 32) {
    if (!w.ev_k[i]) continue;
    const int t = w.ev_a[i];
    int run = init;
    for (int j = 0; j < k; ++j)
      if (w.ev_k[j] && w.ev_a[j] <= t) run += w.ev_d[j];
    bad |= run > cap;
  }
  const bool fail = __any_sync(WRX_FULL, bad);
  __syncwarp();
  return !fail;
}

template <class M>
__device__ bool wrx_dev_ok(const M &md, WWs &w, int d) {
  const int pb = md.dev_begin(d), k = md.dev_end(d) - pb;
  if (k == 0) return true;
  if (k > 8 && k <= 32) return wrx_dev_ok32(md, w, pb, k, k <= 16 ? 16 : 32);
  const int lane = wrx_lane();
  int lim = -(1 << 30), sd = 0;
  for (int i = lane; i < k; i += 32) {
    const int it = md.dev_item(pb + i);
    const int du = md.dur(it);
    const bool pl = wrx_bit(w.placed, it);
    const int a = pl ? w.s[it] : w.lo[it];
    const int e = pl ? a + du : w.hi[it] + du;
    w.ev_a[i] = a;
    w.ev_d[i] = du;
    w.ev_e[i] = e;
    lim = e > lim ? e : lim;
    sd += du;
  }
  lim = __reduce_max_sync(WRX_FULL, lim);
  sd = __reduce_add_sync(WRX_FULL, sd);
  __syncwarp();
  // stable a-order rank (insertion sort by a over dev_items order)
  for (int i = lane; i < k; i += 32) {
    const int ai = w.ev_a[i];
    int r = 0;
    for (int j = 0; j < k; ++j) {
      const int aj = w.ev_a[j];
      r += (aj < ai) | ((aj == ai) & (j < i));
    }
    w.ev_k[i] = r;
  }
  __syncwarp();
  bool bad = false;
  int cmax = sd;  // serial completion: max(sum d, max_i a_i + suffix_d(i))
  for (int i = lane; i < k; i += 32) {
    const int ri = w.ev_k[i], ai = w.ev_a[i], ei = w.ev_e[i];
    int suf_d = 0, suf_e = -(1 << 30), pre_d = 0, pre_a = 1 << 30;
    for (int j = 0; j < k; ++j) {
      const int rj = w.ev_k[j], dj = w.ev_d[j], ej = w.ev_e[j];
      if (rj >= ri) {
        suf_d += dj;
        suf_e = ej > suf_e ? ej : suf_e;
      }
      // stable e-order over the a-sorted sequence: key (e, a-rank)
      if (ej < ei || (ej == ei && rj <= ri)) {
        pre_d += dj;
        const int aj = w.ev_a[j];
        pre_a = aj < pre_a ? aj : pre_a;
      }
    }
    const int c = ai + suf_d;
    cmax = c > cmax ? c : cmax;
    bad |= (ai + suf_d > suf_e) | (pre_a + pre_d > ei);
  }
  cmax = __reduce_max_sync(WRX_FULL, cmax);
  const bool fail = __any_sync(WRX_FULL, bad) || cmax > lim;
  __syncwarp();
  return !fail;
}

// ---------------------------------------------------------------------
// Caller: every lane calls with the same arguments; w.lo / w.hi hold the
// problem bounds (written and __syncwarp'ed).  Returns the status (uniform);
// *nodes_out uniform; w.s holds the witness on SAT.
template <class M>
__device__ int wrx_decide(const M &md, WWs &w, long long budget, unsigned long long t_end_ns,
                          long long *nodes_out, const int *abort_lim = nullptr,
                          int abort_self = 0) {
  const int n = md.n(), ndev = md.ndev(), cap = md.cap();
  const int lane = wrx_lane();
  const int nw = (n + 31) / 32;
  for (int i = lane; i < n; i += 32) w.queue[i] = i;
  for (int i = lane; i < nw; i += 32) {
    w.placed[i] = 0u;
    const int rem = n - 32 * i;
    w.inq[i] = rem >= 32 ? WRX_FULL : ((1u << rem) - 1u);
  }
  __syncwarp();
  int qh = 0, qt = 0, qc = n;
  *nodes_out = 0;
  if (!wrx_propagate(md, w, qh, qt, qc)) return RX_UNSAT;
  if (cap >= 0)
    for (int d = 0; d < ndev; ++d)
      if (!wrx_mem_ok(md, w, d, cap)) return RX_UNSAT;
  for (int d = 0; d < ndev; ++d)
    if (!wrx_dev_ok(md, w, d)) return RX_UNSAT;
  if (n == 0) return RX_SAT;

  long long nodes = 0;
  int status;
  int depth = 0;
  int v = w.lo[md.order(0)];
  for (;;) {
    if (depth == n) {
      status = RX_SAT;
      break;
    }
    int x = md.order(depth);
    const int dx = md.dur(x);
    if (v > w.hi[x]) {  // exhausted: backtrack and restore the depth's snapshot
      if (--depth < 0) {
        status = RX_UNSAT;
        break;
      }
      x = md.order(depth);
      const int2 *sn = w.snap + (long long)depth * n;
      for (int i = lane; i < n; i += 32) {
        const int2 q = sn[i];
        w.lo[i] = q.x;
        w.hi[i] = q.y;
      }
      if (lane == 0) atomicAnd(&w.placed[x >> 5], ~(1u << (x & 31)));
      v = w.vstack[depth] + 1;
      __syncwarp();
      continue;
    }
    const int cb = md.conf_begin(x), ce = md.conf_end(x);
    for (;;) {  // conflict jump to the smallest non-overlapping value >= v
      int jump = -(1 << 30);
      for (int p = cb + lane; p < ce; p += 32) {
        const int y = md.conf_dst(p);
        if (wrx_bit(w.placed, y)) {
          const int sy = w.s[y], ey = sy + md.dur(y);
          if (sy - dx < v && v < ey) jump = ey > jump ? ey : jump;
        }
      }
      jump = __reduce_max_sync(WRX_FULL, jump);
      if (jump == -(1 << 30)) break;
      v = jump;
    }
    if (v > w.hi[x]) continue;
    ++nodes;
    if (budget && nodes > budget) {
      status = RX_TIMEOUT;
      break;
    }
    if (t_end_ns && (nodes & 4095) == 0 && rx_now_ns() > t_end_ns) {
      status = RX_TIMEOUT;
      break;
    }
    // cooperative cancellation: a lower-index probe found SAT meanwhile
    // (the caller re-runs aborted probes unless that SAT retires them)
    if (abort_lim && (nodes & 255) == 0) {
      int l = 0;
      if (lane == 0) l = *(volatile const int *)abort_lim;
      l = __shfl_sync(WRX_FULL, l, 0);
      if (abort_self > l) {
        status = RX_ABORT;
        break;
      }
    }
    {
      int2 *sn = w.snap + (long long)depth * n;
      for (int i = lane; i < n; i += 32) sn[i] = make_int2(w.lo[i], w.hi[i]);
    }
    __syncwarp();
    if (lane == 0) {
      w.s[x] = v;
      w.lo[x] = v;
      w.hi[x] = v;
      atomicOr(&w.placed[x >> 5], 1u << (x & 31));
      w.queue[0] = x;
      atomicOr(&w.inq[x >> 5], 1u << (x & 31));
    }
    qh = 0;
    qt = n == 1 ? 0 : 1;
    qc = 1;
    __syncwarp();
    // tighten unplaced conflicting items, in conf order, first failure wins
    bool ok = true;
    for (int base = cb; base < ce && ok; base += 32) {
      const int p = base + lane;
      const bool act = p < ce;
      int y = 0, nlo = 0, nhi = 0;
      bool chg = false, fail = false, inq = true;
      if (act) {
        y = md.conf_dst(p);
        if (!wrx_bit(w.placed, y)) {
          const int dy = md.dur(y);
          const int lo_y = w.lo[y], hi_y = w.hi[y];
          nlo = lo_y;
          nhi = hi_y;
          if (v - dy < lo_y && lo_y < v + dx) {
            nlo = v + dx;
            chg = true;
            fail = nlo > hi_y;
          }
          if (!fail && v - dy < hi_y && hi_y < v + dx) {
            nhi = v - dy;
            chg = true;
            fail = nhi < nlo;
          }
          inq = wrx_bit(w.inq, y);
        }
      }
      const unsigned failm = __ballot_sync(WRX_FULL, fail);
      if (failm) {
        ok = false;
        break;
      }
      __syncwarp();
      if (chg) {
        w.lo[y] = nlo;
        w.hi[y] = nhi;
      }
      wrx_enqueue(w, chg && !inq, y, n, qt, qc, false);  // conf lists are duplicate-free
    }
    if (ok) {
      ok = wrx_propagate(md, w, qh, qt, qc);
    } else {  // drain and clear the flags of this pass (kernel_c.pyx:341-347)
      for (int k2 = lane; k2 < qc; k2 += 32) {
        int slot = qh + k2;
        if (slot >= n) slot -= n;
        const int b = w.queue[slot];
        atomicAnd(&w.inq[b >> 5], ~(1u << (b & 31)));
      }
      qc = 0;
      __syncwarp();
    }
    const int fb = md.devof_begin(x), fe = md.devof_end(x);
    if (ok && cap >= 0)
      for (int p = fb; p < fe && ok; ++p) ok = wrx_mem_ok(md, w, md.devof(p), cap);
    if (ok)
      for (int p = fb; p < fe && ok; ++p) ok = wrx_dev_ok(md, w, md.devof(p));
    if (ok) {
      if (lane == 0) w.vstack[depth] = v;
      ++depth;
      __syncwarp();
      if (depth < n) v = w.lo[md.order(depth)];
      continue;
    }
    {
      const int2 *sn = w.snap + (long long)depth * n;
      for (int i = lane; i < n; i += 32) {
        const int2 q = sn[i];
        w.lo[i] = q.x;
        w.hi[i] = q.y;
      }
    }
    if (lane == 0) atomicAnd(&w.placed[x >> 5], ~(1u << (x & 31)));
    ++v;
    __syncwarp();
  }
  *nodes_out = nodes;
  __syncwarp();
  return status;
}
