// rx_dfs.cuh — reference-exact decide (RX-DFS) as a CUDA device routine.
//
// Semantics (verdict, lex-min witness AND node count) are those of the
// reference decide kernel /root/reference/pkg/src/repsched/_core/kernel_c.pyx:
//   root FIFO propagation ........................ kernel_c.pyx:158-206
//   root memory / device checks ................... kernel_c.pyx:208-215
//   lex-first DFS, conflict jump, node accounting . kernel_c.pyx:220-263
//   place + tighten conflicting items ............. kernel_c.pyx:264-302
//   FIFO propagation with sticky flags on failure . kernel_c.pyx:303-347
//   _mem_ok / _dev_ok ............................. kernel_c.pyx:374-508
//
// Design differences that do not change results:
//   * per-depth full lo/hi snapshots are replaced by an undo trail with
//     per-node epoch stamps (each item logged at most once per node);
//   * values are int32 (the host checks every input fits, |v| < 2^30);
//   * the problem is accessed through a Model (compile-time polymorphism),
//     so the repetend probe computes its period-dependent edge lags on the
//     fly (lag = base - coef * P, repetend.py:108-190) instead of
//     materialising an edge array per probe.
#pragma once
#include <stdint.h>

#define RX_UNSAT 0
#define RX_SAT 1
#define RX_TIMEOUT 2
#define RX_ABORT 3  // cancelled by the caller's retirement limit (not a reference status)

#ifdef __CUDACC__
#define RX_HD __host__ __device__ __forceinline__
#else
#define RX_HD inline
#endif

// Per-DFS scratch (one slice of a global workspace per concurrent probe).
struct RxWs {
  int *lo, *hi, *s, *queue, *vstack, *mark;
  int *tr_i, *tr_lo, *tr_hi;
  unsigned *stamp;
  unsigned char *placed, *inq;
  int *ev_t, *ev_m, *ev_e;
};

// Number of int32 words of workspace for a problem of n items whose largest
// device has `maxdi` items (placed/inq are carved as bytes from int words).
RX_HD long long rx_ws_words(int n, int maxdi) {
  long long nn = n > 0 ? n : 1;
  long long md = maxdi > 0 ? maxdi : 1;
  long long trail = nn * nn + nn;
  return 4 * nn /*lo,hi,s,queue*/ + 2 * (nn + 1) /*vstack,mark*/ + 3 * trail + nn /*stamp*/ +
         (2 * nn + 3) / 4 + 1 /*placed,inq*/ + 3 * md;
}

RX_HD RxWs rx_ws_carve(int *base, int n, int maxdi) {
  int nn = n > 0 ? n : 1;
  int md = maxdi > 0 ? maxdi : 1;
  long long trail = (long long)nn * nn + nn;
  RxWs w;
  int *p = base;
  w.lo = p; p += nn;
  w.hi = p; p += nn;
  w.s = p; p += nn;
  w.queue = p; p += nn;
  w.vstack = p; p += nn + 1;
  w.mark = p; p += nn + 1;
  w.tr_i = p; p += trail;
  w.tr_lo = p; p += trail;
  w.tr_hi = p; p += trail;
  w.stamp = (unsigned *)p; p += nn;
  w.ev_t = p; p += md;
  w.ev_m = p; p += md;
  w.ev_e = p; p += md;
  w.placed = (unsigned char *)p;
  w.inq = w.placed + nn;
  return w;
}

#ifdef __CUDACC__
__device__ __forceinline__ unsigned long long rx_now_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#endif

template <class M>
RX_HD bool rx_mem_ok(const M &md, const RxWs &w, int d, int cap) {
  int run = md.init_mem(d);
  if (run > cap) return false;
  int ne = 0;
  const int pe = md.dev_end(d);
  for (int p = md.dev_begin(d); p < pe; ++p) {
    const int i = md.dev_item(p);
    const int tm = md.mem(i);
    int tt;
    if (w.placed[i]) {
      tt = w.s[i];
    } else if (tm < 0) {
      tt = w.lo[i];
    } else {
      continue;
    }
    int j = ne;
    while (j > 0 && w.ev_t[j - 1] > tt) {
      w.ev_t[j] = w.ev_t[j - 1];
      w.ev_m[j] = w.ev_m[j - 1];
      --j;
    }
    w.ev_t[j] = tt;
    w.ev_m[j] = tm;
    ++ne;
  }
  int k = 0;
  while (k < ne) {
    const int t = w.ev_t[k];
    while (k < ne && w.ev_t[k] == t) run += w.ev_m[k++];
    if (run > cap) return false;
  }
  return true;
}

template <class M>
RX_HD bool rx_dev_ok(const M &md, const RxWs &w, int d) {
  const int pb = md.dev_begin(d), pe = md.dev_end(d);
  if (pb == pe) return true;
  int lim = -(1 << 30);
  int ne = 0;
  for (int p = pb; p < pe; ++p) {
    const int i = md.dev_item(p);
    const int du = md.dur(i);
    int a, e;
    if (w.placed[i]) {
      a = w.s[i];
      e = a + du;
    } else {
      a = w.lo[i];
      e = w.hi[i] + du;
    }
    if (e > lim) lim = e;
    int j = ne;
    while (j > 0 && w.ev_t[j - 1] > a) {
      w.ev_t[j] = w.ev_t[j - 1];
      w.ev_m[j] = w.ev_m[j - 1];
      w.ev_e[j] = w.ev_e[j - 1];
      --j;
    }
    w.ev_t[j] = a;
    w.ev_m[j] = du;
    w.ev_e[j] = e;
    ++ne;
  }
  int c = 0;
  for (int p = 0; p < ne; ++p) {
    if (w.ev_t[p] > c) c = w.ev_t[p];
    c += w.ev_m[p];
  }
  if (c > lim) return false;
  int suf_p = 0, suf_e = -(1 << 30);
  for (int p = ne - 1; p >= 0; --p) {
    suf_p += w.ev_m[p];
    if (w.ev_e[p] > suf_e) suf_e = w.ev_e[p];
    if (w.ev_t[p] + suf_p > suf_e) return false;
  }
  for (int p = 0; p < ne; ++p) {  // stable re-sort by e
    const int te = w.ev_e[p], ta = w.ev_t[p], tm = w.ev_m[p];
    int j = p;
    while (j > 0 && w.ev_e[j - 1] > te) {
      w.ev_e[j] = w.ev_e[j - 1];
      w.ev_t[j] = w.ev_t[j - 1];
      w.ev_m[j] = w.ev_m[j - 1];
      --j;
    }
    w.ev_e[j] = te;
    w.ev_t[j] = ta;
    w.ev_m[j] = tm;
  }
  int pre_p = 0, pre_a = w.ev_t[0];
  for (int p = 0; p < ne; ++p) {
    pre_p += w.ev_m[p];
    if (w.ev_t[p] < pre_a) pre_a = w.ev_t[p];
    if (pre_a + pre_p > w.ev_e[p]) return false;
  }
  return true;
}

RX_HD void rx_save(RxWs &w, int i, unsigned ep, int &tn) {
  if (w.stamp[i] != ep) {
    w.stamp[i] = ep;
    w.tr_i[tn] = i;
    w.tr_lo[tn] = w.lo[i];
    w.tr_hi[tn] = w.hi[i];
    ++tn;
  }
}

RX_HD void rx_undo(RxWs &w, int mark, int &tn) {
  while (tn > mark) {
    --tn;
    const int i = w.tr_i[tn];
    w.lo[i] = w.tr_lo[tn];
    w.hi[i] = w.tr_hi[tn];
  }
}

RX_HD void rx_push(RxWs &w, int b, int n, int &qt, int &qc) {
  w.inq[b] = 1;
  w.queue[qt] = b;
  if (++qt == n) qt = 0;
  ++qc;
}

// FIFO propagation (kernel_c.pyx:158-206 / 303-340).  On failure returns
// false immediately: flags of items still queued stay set (sticky).
template <bool LOG, class M>
RX_HD bool rx_propagate(const M &md, RxWs &w, int &qh, int &qt, int &qc, unsigned ep, int &tn) {
  const int n = md.n();
  while (qc > 0) {
    const int a = w.queue[qh];
    if (++qh == n) qh = 0;
    --qc;
    w.inq[a] = 0;
    const int la = w.lo[a], ha = w.hi[a];
    const int oe = md.out_end(a), od = md.out_dep_end(a), owl = md.out_win_lag(a);
    for (int p = md.out_begin(a); p < oe; ++p) {
      const int b = md.out_dst(p);
      const int nl = la + (p < od ? md.out_dep_lag(p) : owl);
      if (nl > w.lo[b]) {
        if (nl > w.hi[b]) return false;
        if (LOG) rx_save(w, b, ep, tn);
        w.lo[b] = nl;
        if (!w.inq[b]) rx_push(w, b, n, qt, qc);
      }
    }
    const int ie = md.in_end(a), id = md.in_dep_end(a);
    for (int p = md.in_begin(a); p < ie; ++p) {
      const int b = md.in_src(p);
      const int nh = ha - (p < id ? md.in_dep_lag(p) : md.in_win_lag(p));
      if (nh < w.hi[b]) {
        if (nh < w.lo[b]) return false;
        if (LOG) rx_save(w, b, ep, tn);
        w.hi[b] = nh;
        if (!w.inq[b]) rx_push(w, b, n, qt, qc);
      }
    }
  }
  return true;
}

// The caller initialises w.lo / w.hi with the problem bounds.  Returns the
// status; *nodes_out gets the reference node count; w.s holds the witness on
// SAT.  `budget` = node cap (0: none); `t_end_ns` = globaltimer deadline
// (0: none), polled every 4096 nodes like kernel_c.pyx:20,261.
template <class M>
RX_HD int rx_decide(const M &md, RxWs &w, long long budget, unsigned long long t_end_ns,
                    long long *nodes_out) {
  const int n = md.n();
  const int ndev = md.ndev();
  const int cap = md.cap();
  for (int i = 0; i < n; ++i) {
    w.placed[i] = 0;
    w.inq[i] = 1;
    w.queue[i] = i;
    w.stamp[i] = 0u;
  }
  int qh = 0, qt = 0, qc = n;
  unsigned ep = 0u;
  int tn = 0;
  *nodes_out = 0;
  if (!rx_propagate<false>(md, w, qh, qt, qc, ep, tn)) return RX_UNSAT;
  if (cap >= 0)
    for (int d = 0; d < ndev; ++d)
      if (!rx_mem_ok(md, w, d, cap)) return RX_UNSAT;
  for (int d = 0; d < ndev; ++d)
    if (!rx_dev_ok(md, w, d)) return RX_UNSAT;
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
    if (v > w.hi[x]) {  // exhausted: backtrack
      --depth;
      if (depth < 0) {
        status = RX_UNSAT;
        break;
      }
      x = md.order(depth);
      rx_undo(w, w.mark[depth], tn);
      w.placed[x] = 0;
      v = w.vstack[depth] + 1;
      continue;
    }
    const int cb = md.conf_begin(x), ce = md.conf_end(x);
    for (bool moved = true; moved;) {  // conflict jump
      moved = false;
      for (int p = cb; p < ce; ++p) {
        const int y = md.conf_dst(p);
        if (w.placed[y]) {
          const int sy = w.s[y];
          const int ey = sy + md.dur(y);
          if (sy - dx < v && v < ey) {
            v = ey;
            moved = true;
          }
        }
      }
    }
    if (v > w.hi[x]) continue;
    ++nodes;
    if (budget && nodes > budget) {
      status = RX_TIMEOUT;
      break;
    }
#ifdef __CUDA_ARCH__
    if (t_end_ns && (nodes & 4095) == 0 && rx_now_ns() > t_end_ns) {
      status = RX_TIMEOUT;
      break;
    }
#endif
    w.mark[depth] = tn;
    if (++ep == 0u) {  // epoch wrap (> 4e9 nodes): re-arm the stamps
      for (int i = 0; i < n; ++i) w.stamp[i] = 0u;
      ep = 1u;
    }
    rx_save(w, x, ep, tn);
    w.s[x] = v;
    w.placed[x] = 1;
    w.lo[x] = v;
    w.hi[x] = v;
    bool ok = true;
    qh = 0;
    qt = 0;
    qc = 0;
    rx_push(w, x, n, qt, qc);  // x is enqueued regardless of its flag
    for (int p = cb; p < ce; ++p) {
      const int y = md.conf_dst(p);
      if (w.placed[y]) continue;
      const int dy = md.dur(y);
      if (v - dy < w.lo[y] && w.lo[y] < v + dx) {
        rx_save(w, y, ep, tn);
        w.lo[y] = v + dx;
        if (w.lo[y] > w.hi[y]) {
          ok = false;
          break;
        }
        if (!w.inq[y]) rx_push(w, y, n, qt, qc);
      }
      if (v - dy < w.hi[y] && w.hi[y] < v + dx) {
        rx_save(w, y, ep, tn);
        w.hi[y] = v - dy;
        if (w.hi[y] < w.lo[y]) {
          ok = false;
          break;
        }
        if (!w.inq[y]) rx_push(w, y, n, qt, qc);
      }
    }
    if (ok) {
      ok = rx_propagate<true>(md, w, qh, qt, qc, ep, tn);
    } else {  // drain and clear the flags of this pass (kernel_c.pyx:341-347)
      while (qc > 0) {
        w.inq[w.queue[qh]] = 0;
        if (++qh == n) qh = 0;
        --qc;
      }
    }
    const int fb = md.devof_begin(x), fe = md.devof_end(x);
    if (ok && cap >= 0)
      for (int p = fb; p < fe; ++p)
        if (!rx_mem_ok(md, w, md.devof(p), cap)) {
          ok = false;
          break;
        }
    if (ok)
      for (int p = fb; p < fe; ++p)
        if (!rx_dev_ok(md, w, md.devof(p))) {
          ok = false;
          break;
        }
    if (ok) {
      w.vstack[depth] = v;
      ++depth;
      if (depth < n) v = w.lo[md.order(depth)];
      continue;
    }
    rx_undo(w, w.mark[depth], tn);
    w.placed[x] = 0;
    ++v;
  }
  *nodes_out = nodes;
  return status;
}
