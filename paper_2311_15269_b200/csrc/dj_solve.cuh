// dj_solve.cuh — complete disjunctive feasibility for one repetend probe.
//
// Decides the SAME question as the reference decide kernel on a repetend
// probe (repetend.py:160-190: anchored box, dependency + device-window
// difference edges, exclusivity of items with intersecting device masks,
// per-device running memory <= cap from the entry memory) but by branching
// on the ORDER of each conflicting pair instead of on start values:
//   * state: lower/upper start bounds (longest-path propagation over the
//     difference edges plus the chosen pair orientations);
//   * detectable precedences: a pair whose one orientation is impossible
//     under the current bounds is oriented the other way; both impossible
//     = failure;
//   * memory: once every pair on a device is oriented, the device's items
//     are totally ordered (no two start together), so the running memory is
//     the prefix sum in that order, checked against cap.
// Complete: every failure is a proof, so DJ_UNSAT means the probe has no
// solution in the box.  The search uses it only as a FILTER: a repetend probe
// proven infeasible is "not SAT", which the reference's period scan treats
// exactly like its own 400k-node TIMEOUT or UNSAT (repetend.py:289-302).
// DJ never produces witnesses or node counts for the reference semantics;
// SAT or undecided probes are replayed by the reference-exact RX-DFS.
#pragma once
#include "models.cuh"

#define DJ_UNSAT 0
#define DJ_SAT 1
#define DJ_UNKNOWN 2

struct DjWs {
  int *lo, *hi, *queue, *stamp;
  int *tr_i, *tr_lo, *tr_hi;    // bound trail (each item once per node)
  int *ptr_pid;                  // pair trail
  int *f_pid, *f_pref, *f_tried, *f_bm, *f_pm;  // DFS frames
  int *devleft, *newdev, *ord;
  unsigned char *inq, *orient;
};

RX_HD long long dj_ws_words(int K, int D, int npair, int maxdi) {
  long long k = K > 0 ? K : 1, np = npair > 0 ? npair : 1, d = D > 0 ? D : 1;
  long long md = maxdi > 0 ? maxdi : 1;
  return 4 * k + 3 * k * (np + 2) + np + 5 * (np + 1) + 2 * d + md + (k + np + 3) / 4 + 2;
}

RX_HD DjWs dj_ws_carve(int *base, int K, int D, int npair, int maxdi) {
  const long long k = K > 0 ? K : 1, np = npair > 0 ? npair : 1, d = D > 0 ? D : 1;
  const long long md = maxdi > 0 ? maxdi : 1;
  DjWs w;
  int *p = base;
  w.lo = p; p += k;
  w.hi = p; p += k;
  w.queue = p; p += k;
  w.stamp = p; p += k;
  w.tr_i = p; p += k * (np + 2);
  w.tr_lo = p; p += k * (np + 2);
  w.tr_hi = p; p += k * (np + 2);
  w.ptr_pid = p; p += np;
  w.f_pid = p; p += np + 1;
  w.f_pref = p; p += np + 1;
  w.f_tried = p; p += np + 1;
  w.f_bm = p; p += np + 1;
  w.f_pm = p; p += np + 1;
  w.devleft = p; p += d;
  w.newdev = p; p += d;
  w.ord = p; p += md;
  w.inq = (unsigned char *)p;
  w.orient = w.inq + k;
  return w;
}

struct DjCtx {
  const int *pairx, *pairy, *pdev_ptr, *pdev, *devnpair, *conf_pid;
  int npair;
  int tn, pn, ep, nnew;
};

RX_HD void dj_save(DjWs &w, DjCtx &c, int i) {
  if (w.stamp[i] != c.ep) {
    w.stamp[i] = c.ep;
    w.tr_i[c.tn] = i;
    w.tr_lo[c.tn] = w.lo[i];
    w.tr_hi[c.tn] = w.hi[i];
    ++c.tn;
  }
}

RX_HD void dj_push(DjWs &w, int K, int b, int &qt, int &qc) {
  if (w.inq[b]) return;
  w.inq[b] = 1;
  w.queue[qt] = b;
  if (++qt == K) qt = 0;
  ++qc;
}

// orient pair pid with `first` before the other item
RX_HD void dj_orient(DjWs &w, DjCtx &c, int pid, bool x_first) {
  w.orient[pid] = x_first ? 1 : 2;
  w.ptr_pid[c.pn++] = pid;
  for (int q = c.pdev_ptr[pid]; q < c.pdev_ptr[pid + 1]; ++q) {
    const int d = c.pdev[q];
    if (--w.devleft[d] == 0) w.newdev[c.nnew++] = d;
  }
}

RX_HD void dj_undo(DjWs &w, DjCtx &c, int bm, int pm) {
  while (c.tn > bm) {
    --c.tn;
    const int i = w.tr_i[c.tn];
    w.lo[i] = w.tr_lo[c.tn];
    w.hi[i] = w.tr_hi[c.tn];
  }
  while (c.pn > pm) {
    const int pid = w.ptr_pid[--c.pn];
    w.orient[pid] = 0;
    for (int q = c.pdev_ptr[pid]; q < c.pdev_ptr[pid + 1]; ++q) ++w.devleft[c.pdev[q]];
  }
}

template <class M>
RX_HD bool dj_propagate(const M &md, DjWs &w, DjCtx &c, int &qh, int &qt, int &qc) {
  const int K = md.n();
  while (qc > 0) {
    const int a = w.queue[qh];
    if (++qh == K) qh = 0;
    --qc;
    w.inq[a] = 0;
    const int la = w.lo[a], ha = w.hi[a], da = md.dur(a);
    const int oe = md.out_end(a), od = md.out_dep_end(a), owl = md.out_win_lag(a);
    for (int p = md.out_begin(a); p < oe; ++p) {
      const int b = md.out_dst(p);
      const int nl = la + (p < od ? md.out_dep_lag(p) : owl);
      if (nl > w.lo[b]) {
        if (nl > w.hi[b]) return false;
        dj_save(w, c, b);
        w.lo[b] = nl;
        dj_push(w, K, b, qt, qc);
      }
    }
    const int ie = md.in_end(a), id = md.in_dep_end(a);
    for (int p = md.in_begin(a); p < ie; ++p) {
      const int b = md.in_src(p);
      const int nh = ha - (p < id ? md.in_dep_lag(p) : md.in_win_lag(p));
      if (nh < w.hi[b]) {
        if (nh < w.lo[b]) return false;
        dj_save(w, c, b);
        w.hi[b] = nh;
        dj_push(w, K, b, qt, qc);
      }
    }
    const int ce = md.conf_end(a);
    for (int p = md.conf_begin(a); p < ce; ++p) {
      const int y = md.conf_dst(p);
      const int pid = c.conf_pid[p];
      const bool a_is_x = c.pairx[pid] == a;
      int o = w.orient[pid];
      if (o == 0) {
        const bool can_ay = la + da <= w.hi[y];
        const bool can_ya = w.lo[y] + md.dur(y) <= ha;
        if (!can_ay && !can_ya) return false;
        if (!can_ay || !can_ya) {
          const bool a_first = can_ay;
          dj_orient(w, c, pid, a_is_x ? a_first : !a_first);
          o = w.orient[pid];
          dj_push(w, K, y, qt, qc);
        } else {
          continue;
        }
      }
      const bool a_first = (o == 1) == a_is_x;
      if (a_first) {
        const int nl = la + da;
        if (nl > w.lo[y]) {
          if (nl > w.hi[y]) return false;
          dj_save(w, c, y);
          w.lo[y] = nl;
          dj_push(w, K, y, qt, qc);
        }
      } else {
        const int nh = ha - md.dur(y);
        if (nh < w.hi[y]) {
          if (nh < w.lo[y]) return false;
          dj_save(w, c, y);
          w.hi[y] = nh;
          dj_push(w, K, y, qt, qc);
        }
      }
    }
  }
  return true;
}

// all pairs on device d are oriented: items are totally ordered by lo
template <class M>
RX_HD bool dj_mem_ok(const M &md, DjWs &w, int d, int cap) {
  int run = md.init_mem(d);
  if (run > cap) return false;
  int ne = 0;
  for (int p = md.dev_begin(d); p < md.dev_end(d); ++p) {
    const int i = md.dev_item(p);
    int j = ne++;
    while (j > 0 && w.lo[w.ord[j - 1]] > w.lo[i]) {
      w.ord[j] = w.ord[j - 1];
      --j;
    }
    w.ord[j] = i;
  }
  for (int k = 0; k < ne; ++k) {
    run += md.mem(w.ord[k]);
    if (run > cap) return false;
  }
  return true;
}

template <class M>
RX_HD bool dj_node_checks(const M &md, DjWs &w, DjCtx &c) {
  bool ok = true;
  if (md.cap() >= 0)
    for (int k = 0; k < c.nnew && ok; ++k) ok = dj_mem_ok(md, w, w.newdev[k], md.cap());
  c.nnew = 0;
  return ok;
}

// lo/hi must hold the probe's initial box (rep_prepare).  `pool` is the
// placement structure pool (pair tables).  Returns DJ_SAT / DJ_UNSAT /
// DJ_UNKNOWN (budget of branching nodes exhausted); *nodes_out = nodes used.
template <class M>
RX_HD int dj_decide(const M &md, const int *pool, DjWs &w, long long budget, long long *nodes_out) {
  const int K = md.n(), D = md.ndev();
  DjCtx c;
  c.pairx = pool + pool[R_PAIRX];
  c.pairy = pool + pool[R_PAIRY];
  c.pdev_ptr = pool + pool[R_PDEVPTR];
  c.pdev = pool + pool[R_PDEV];
  c.devnpair = pool + pool[R_DEVNPAIR];
  c.conf_pid = pool + pool[R_CONFPID];
  c.npair = pool[R_NPAIR];
  c.tn = c.pn = c.nnew = 0;
  c.ep = 1;
  *nodes_out = 0;
  for (int i = 0; i < K; ++i) {
    w.stamp[i] = 0;
    w.inq[i] = 1;
    w.queue[i] = i;
  }
  for (int q = 0; q < c.npair; ++q) w.orient[q] = 0;
  for (int d = 0; d < D; ++d) {
    w.devleft[d] = c.devnpair[d];
    if (md.cap() >= 0 && md.init_mem(d) > md.cap()) return DJ_UNSAT;
    if (w.devleft[d] == 0) w.newdev[c.nnew++] = d;
  }
  int qh = 0, qt = 0, qc = K;
  if (!dj_propagate(md, w, c, qh, qt, qc)) return DJ_UNSAT;
  if (!dj_node_checks(md, w, c)) return DJ_UNSAT;

  long long nodes = 0;
  int depth = 0;
  int cursor = 0;
  bool descend = true;
  for (;;) {
    if (descend) {
      // most constrained unresolved pair: smallest slack of its tighter side
      int best = -1, best_slack = 1 << 30, pref = 1;
      for (int q = 0; q < c.npair; ++q) {
        if (w.orient[q]) continue;
        const int x = c.pairx[q], y = c.pairy[q];
        const int sxy = w.hi[y] - (w.lo[x] + md.dur(x));
        const int syx = w.hi[x] - (w.lo[y] + md.dur(y));
        const int s = sxy < syx ? sxy : syx;
        if (s < best_slack) {
          best_slack = s;
          best = q;
          pref = sxy >= syx ? 1 : 2;
        }
      }
      (void)cursor;
      if (best < 0) {
        *nodes_out = nodes;
        return DJ_SAT;
      }
      w.f_pid[depth] = best;
      w.f_pref[depth] = pref;
      w.f_tried[depth] = 0;
      w.f_bm[depth] = c.tn;
      w.f_pm[depth] = c.pn;
      descend = false;
    }
    // try the next orientation of the frame at `depth`
    if (w.f_tried[depth] == 2) {
      if (--depth < 0) {
        *nodes_out = nodes;
        return DJ_UNSAT;
      }
      dj_undo(w, c, w.f_bm[depth], w.f_pm[depth]);
      continue;
    }
    const int o = w.f_tried[depth] == 0 ? w.f_pref[depth] : 3 - w.f_pref[depth];
    ++w.f_tried[depth];
    if (++nodes > budget && budget) {
      *nodes_out = nodes;
      return DJ_UNKNOWN;
    }
    if (++c.ep == 0) {
      for (int i = 0; i < K; ++i) w.stamp[i] = 0;
      c.ep = 1;
    }
    const int pid = w.f_pid[depth];
    c.nnew = 0;
    dj_orient(w, c, pid, o == 1);
    qh = qt = qc = 0;
    dj_push(w, K, c.pairx[pid], qt, qc);
    dj_push(w, K, c.pairy[pid], qt, qc);
    bool ok = dj_propagate(md, w, c, qh, qt, qc);
    if (!ok) {
      while (qc > 0) {  // clear queue flags
        w.inq[w.queue[qh]] = 0;
        if (++qh == K) qh = 0;
        --qc;
      }
      c.nnew = 0;
    } else {
      ok = dj_node_checks(md, w, c);
    }
    if (ok) {
      ++depth;
      descend = true;
    } else {
      dj_undo(w, c, w.f_bm[depth], w.f_pm[depth]);
    }
  }
}
