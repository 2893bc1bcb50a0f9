// models.cuh — problem views consumed by rx_decide (rx_dfs.cuh).
//
// GenView: one general decide problem (kernel_c.pyx:23-37 inputs) lowered
//   on the host into a flat int32 pool with the reference's CSRs
//   (kernel_c.pyx:54-128: out/in edges in edge-row order, conflicts in
//   ascending item order, device->items ascending, item->devices ascending).
// RepView: one repetend probe (candidate assignment a, period P) over a
//   placement-wide structure pool; edge lags are base - coef * P with coef =
//   a[src] - a[dst] for dependency rows and 1 for device-window rows
//   (repetend.py:108-190).
#pragma once
#include "rx_dfs.cuh"

// ---------------------------------------------------------------- GenView
// pool header (ints): n, ndev, cap, m, nconf, nmemb, maxdi, words
enum { G_N = 0, G_NDEV, G_CAP, G_M, G_NCONF, G_NMEMB, G_MAXDI, G_WORDS, G_HDR };

struct GenView {
  int n_, ndev_, cap_;
  const int *dur_, *mem_, *order_, *lo_, *hi_, *init_;
  const int *out_ptr_, *out_dst_, *out_lag_, *in_ptr_, *in_src_, *in_lag_;
  const int *conf_ptr_, *conf_dst_, *dev_ptr_, *dev_items_, *devof_ptr_, *devof_;
  const int *out_dup_, *in_dup_;  // 1 if the node's edge list repeats a target
  const int *in_twin_;            // host_build.hpp in_twins

  RX_HD int n() const { return n_; }
  RX_HD bool out_dup(int a) const { return out_dup_[a] != 0; }
  RX_HD int in_twin(int p) const { return in_twin_[p]; }
  RX_HD bool in_dup(int a) const { return in_dup_[a] != 0; }
  RX_HD int ndev() const { return ndev_; }
  RX_HD int cap() const { return cap_; }
  RX_HD int dur(int i) const { return dur_[i]; }
  RX_HD int mem(int i) const { return mem_[i]; }
  RX_HD int order(int k) const { return order_[k]; }
  RX_HD int init_mem(int d) const { return init_[d]; }
  RX_HD int out_begin(int a) const { return out_ptr_[a]; }
  RX_HD int out_end(int a) const { return out_ptr_[a + 1]; }
  RX_HD int out_dst(int p) const { return out_dst_[p]; }
  RX_HD int out_lag(int p) const { return out_lag_[p]; }
  // every general edge is treated as a "dependency" edge with a stored lag
  RX_HD int out_dep_end(int a) const { return out_ptr_[a + 1]; }
  RX_HD int out_dep_lag(int p) const { return out_lag_[p]; }
  RX_HD int out_win_lag(int) const { return 0; }
  RX_HD int in_dep_end(int a) const { return in_ptr_[a + 1]; }
  RX_HD int in_dep_lag(int p) const { return in_lag_[p]; }
  RX_HD int in_win_lag(int) const { return 0; }
  RX_HD int in_begin(int a) const { return in_ptr_[a]; }
  RX_HD int in_end(int a) const { return in_ptr_[a + 1]; }
  RX_HD int in_src(int p) const { return in_src_[p]; }
  RX_HD int in_lag(int p) const { return in_lag_[p]; }
  RX_HD int conf_begin(int x) const { return conf_ptr_[x]; }
  RX_HD int conf_end(int x) const { return conf_ptr_[x + 1]; }
  RX_HD int conf_dst(int p) const { return conf_dst_[p]; }
  RX_HD int dev_begin(int d) const { return dev_ptr_[d]; }
  RX_HD int dev_end(int d) const { return dev_ptr_[d + 1]; }
  RX_HD int dev_item(int p) const { return dev_items_[p]; }
  RX_HD int devof_begin(int i) const { return devof_ptr_[i]; }
  RX_HD int devof_end(int i) const { return devof_ptr_[i + 1]; }
  RX_HD int devof(int p) const { return devof_[p]; }
};

RX_HD GenView gen_view(const int *pool) {
  GenView g;
  const int n = pool[G_N], ndev = pool[G_NDEV], m = pool[G_M];
  const int nconf = pool[G_NCONF], nmemb = pool[G_NMEMB];
  g.n_ = n;
  g.ndev_ = ndev;
  g.cap_ = pool[G_CAP];
  const int *p = pool + G_HDR;
  g.dur_ = p; p += n;
  g.mem_ = p; p += n;
  g.order_ = p; p += n;
  g.lo_ = p; p += n;
  g.hi_ = p; p += n;
  g.init_ = p; p += ndev;
  g.out_ptr_ = p; p += n + 1;
  g.out_dst_ = p; p += m;
  g.out_lag_ = p; p += m;
  g.in_ptr_ = p; p += n + 1;
  g.in_src_ = p; p += m;
  g.in_lag_ = p; p += m;
  g.conf_ptr_ = p; p += n + 1;
  g.conf_dst_ = p; p += nconf;
  g.dev_ptr_ = p; p += ndev + 1;
  g.dev_items_ = p; p += nmemb;
  g.devof_ptr_ = p; p += n + 1;
  g.devof_ = p; p += nmemb;
  g.out_dup_ = p; p += n;
  g.in_dup_ = p; p += n;
  g.in_twin_ = p;
  return g;
}

// ---------------------------------------------------------------- RepView
// Placement structure pool: header ints followed by the arrays; offsets in
// the header are relative to the pool start.
enum {
  R_K = 0, R_D, R_NDEP, R_M, R_MAXDUR, R_LB, R_TOTAL, R_MAXDI, R_NPAIR,
  R_DUR, R_MEM, R_ORDER, R_OUTPTR, R_OUTDST, R_OUTROW, R_OUTDEPEND, R_INPTR, R_INSRC, R_INROW,
  R_INDEPEND, R_INSRCDUR,
  R_RBASE, R_RSRC, R_RDST, R_CONFPTR, R_CONFDST, R_CONFPID, R_DEVPTR, R_DEVITEMS, R_DEVOFPTR,
  R_DEVOF,
  // disjunctive pairs {x < y} of items with intersecting device masks, the
  // devices each pair shares, and the number of pairs per device
  R_PAIRX, R_PAIRY, R_PDEVPTR, R_PDEV, R_DEVNPAIR, R_OUTDUP, R_INDUP,
  // enumeration metadata: per stage st, lo sources (succ j < st), hi
  // sources (pred i < st), and the frontier F_{st+1} after assigning st
  R_LSPTR, R_LS, R_HSPTR, R_HS, R_FRPTR, R_FR,
  // device -> disjunctive pairs on it (warp disjunctive filter)
  R_DPPTR, R_DP,
  // per in-entry: position of the out-entry naming the same node, or -1
  R_INTWIN,
  // register-resident warp decide (wrr_dfs.cuh), K <= 64 items and D <= 64:
  // per item u64 masks (lo word, hi word) of dependency successors /
  // predecessors, conflicting items (= device-window partners) and devices;
  // per device its items; per item the index of its window-order table (-1:
  // single-device item, window order = ascending id) and, per multi-device
  // item a, for every partner b the items whose first window row of a
  // precedes b's (repetend.py:133-141 row order)
  R_SUCCM, R_PREDM, R_CONFM, R_DEVM, R_DEVITM, R_MULTI, R_WINB, R_WRR,
  // 1: repetend probes run the strong search first (wst_dfs.cuh)
  R_WST,
  // per 32-row chunk of the edge rows / of the disjunctive pairs: the items
  // they touch (u64, all ones when K > 64) — wdj_propagate skips chunks
  // none of whose items changed
  R_ROWCM, R_PAIRCM,
  R_WORDS, R_HDR
};

// Edge rows are (sorted dependency rows) ++ (device-window rows), and the
// CSRs keep row order, so every node's out-list (in-list) starts with its
// dependency entries.  Window rows x->y carry lag t_x - P (coef 1), so the
// window part needs no per-candidate data: out-lag = dur[a] - P for the
// popped node a, in-lag = dur[src] - P (stored per in-entry as srcdur).
struct RepView {
  const int *dur_, *mem_, *order_, *out_ptr_, *out_dst_, *out_row_, *out_dep_end_;
  const int *in_ptr_, *in_src_, *in_row_, *in_dep_end_, *in_srcdur_;
  const int *conf_ptr_, *conf_dst_, *dev_ptr_, *dev_items_, *devof_ptr_, *devof_;
  const int *out_dup_, *in_dup_, *in_twin_;
  const int *deplag;  // per dependency row: base - (a[src] - a[dst]) * P
  const int *init;    // entry memory per device
  int K, D, P, cap_;

  RX_HD int n() const { return K; }
  RX_HD int ndev() const { return D; }
  RX_HD bool out_dup(int a) const { return out_dup_[a] != 0; }
  RX_HD int in_twin(int p) const { return in_twin_[p]; }
  RX_HD bool in_dup(int a) const { return in_dup_[a] != 0; }
  RX_HD int cap() const { return cap_; }
  RX_HD int dur(int i) const { return dur_[i]; }
  RX_HD int mem(int i) const { return mem_[i]; }
  RX_HD int order(int k) const { return order_[k]; }
  RX_HD int init_mem(int d) const { return init[d]; }
  RX_HD int out_begin(int a) const { return out_ptr_[a]; }
  RX_HD int out_end(int a) const { return out_ptr_[a + 1]; }
  RX_HD int out_dst(int p) const { return out_dst_[p]; }
  RX_HD int out_dep_end(int a) const { return out_dep_end_[a]; }
  RX_HD int out_dep_lag(int p) const { return deplag[out_row_[p]]; }
  RX_HD int out_win_lag(int a) const { return dur_[a] - P; }
  RX_HD int in_begin(int a) const { return in_ptr_[a]; }
  RX_HD int in_end(int a) const { return in_ptr_[a + 1]; }
  RX_HD int in_src(int p) const { return in_src_[p]; }
  RX_HD int in_dep_end(int a) const { return in_dep_end_[a]; }
  RX_HD int in_dep_lag(int p) const { return deplag[in_row_[p]]; }
  RX_HD int in_win_lag(int p) const { return in_srcdur_[p] - P; }
  RX_HD int conf_begin(int x) const { return conf_ptr_[x]; }
  RX_HD int conf_end(int x) const { return conf_ptr_[x + 1]; }
  RX_HD int conf_dst(int p) const { return conf_dst_[p]; }
  RX_HD int dev_begin(int d) const { return dev_ptr_[d]; }
  RX_HD int dev_end(int d) const { return dev_ptr_[d + 1]; }
  RX_HD int dev_item(int p) const { return dev_items_[p]; }
  RX_HD int devof_begin(int i) const { return devof_ptr_[i]; }
  RX_HD int devof_end(int i) const { return devof_ptr_[i + 1]; }
  RX_HD int devof(int p) const { return devof_[p]; }
};

RX_HD RepView rep_view(const int *pool, int P, int cap, const int *deplag, const int *init) {
  RepView v;
  v.K = pool[R_K];
  v.D = pool[R_D];
  v.P = P;
  v.cap_ = cap;
  v.deplag = deplag;
  v.init = init;
  v.dur_ = pool + pool[R_DUR];
  v.mem_ = pool + pool[R_MEM];
  v.order_ = pool + pool[R_ORDER];
  v.out_ptr_ = pool + pool[R_OUTPTR];
  v.out_dst_ = pool + pool[R_OUTDST];
  v.out_row_ = pool + pool[R_OUTROW];
  v.out_dep_end_ = pool + pool[R_OUTDEPEND];
  v.in_ptr_ = pool + pool[R_INPTR];
  v.in_src_ = pool + pool[R_INSRC];
  v.in_row_ = pool + pool[R_INROW];
  v.in_dep_end_ = pool + pool[R_INDEPEND];
  v.in_srcdur_ = pool + pool[R_INSRCDUR];
  v.conf_ptr_ = pool + pool[R_CONFPTR];
  v.conf_dst_ = pool + pool[R_CONFDST];
  v.dev_ptr_ = pool + pool[R_DEVPTR];
  v.dev_items_ = pool + pool[R_DEVITEMS];
  v.devof_ptr_ = pool + pool[R_DEVOFPTR];
  v.devof_ = pool + pool[R_DEVOF];
  v.out_dup_ = pool + pool[R_OUTDUP];
  v.in_dup_ = pool + pool[R_INDUP];
  v.in_twin_ = pool + pool[R_INTWIN];
  return v;
}

// Prepare a repetend probe for assignment a[K] at period P: dependency-row
// lags base - (a[src] - a[dst]) * P, entry memory (repetend.py:93-100) and
// the anchored bounds s_0 = A, s_i in [0, 2A], A = (K-1)(P + max t)
// (repetend.py:162-169).
template <class A>
RX_HD void rep_prepare(const int *pool, const A &a, int P, int *deplag, int *init, int *lo,
                       int *hi) {
  const int K = pool[R_K], D = pool[R_D], ndep = pool[R_NDEP];
  for (int r = 0; r < ndep; ++r)
    deplag[r] = pool[pool[R_RBASE] + r] -
                ((int)a[pool[pool[R_RSRC] + r]] - (int)a[pool[pool[R_RDST] + r]]) * P;
  for (int d = 0; d < D; ++d) init[d] = 0;
  for (int st = 0; st < K; ++st) {
    const int mst = pool[pool[R_MEM] + st] * (int)a[st];
    const int fb = pool[pool[R_DEVOFPTR] + st], fe = pool[pool[R_DEVOFPTR] + st + 1];
    for (int p = fb; p < fe; ++p) init[pool[pool[R_DEVOF] + p]] += mst;
  }
  const int anchor = (K - 1) * (P + pool[R_MAXDUR]);
  for (int i = 0; i < K; ++i) {
    lo[i] = 0;
    hi[i] = 2 * anchor;
  }
  if (K > 0) lo[0] = hi[0] = anchor;
}

RX_HD int at_ptr(const int *pool, int off, int i) { return pool[pool[off] + i]; }

// Unrank a global lexicographic rank at n_r (repetend.py:65-90 order, with
// the min-index-0 filter) using the frontier count tables: cnt + off[st]
// holds, for position st, 2 * n_r^|F_st| completion counts indexed by
// (frontier values in mixed radix n_r, has-zero flag).
template <class A>
RX_HD bool rep_unrank(const int *pool, const unsigned long long *cnt, const long long *off, int n_r,
                      unsigned long long rank, A &a) {
  const int K = pool[R_K];
  int z = 0;
  for (int st = 0; st < K; ++st) {
    int lo = 0, hi = n_r - 1;
    for (int p = at_ptr(pool, R_LSPTR, st); p < at_ptr(pool, R_LSPTR, st + 1); ++p) {
      const int v = (int)a[pool[pool[R_LS] + p]];
      lo = v > lo ? v : lo;
    }
    for (int p = at_ptr(pool, R_HSPTR, st); p < at_ptr(pool, R_HSPTR, st + 1); ++p) {
      const int v = (int)a[pool[pool[R_HS] + p]];
      hi = v < hi ? v : hi;
    }
    long long base = 0, cst = 0, mult = 1;
    for (int p = at_ptr(pool, R_FRPTR, st); p < at_ptr(pool, R_FRPTR, st + 1); ++p) {
      const int u = pool[pool[R_FR] + p];
      if (u == st)
        cst = mult;
      else
        base += (long long)a[u] * mult;
      mult *= n_r;
    }
    const unsigned long long *tab = cnt + off[st + 1];
    int chosen = -1;
    for (int v = lo; v <= hi; ++v) {
      const int z2 = z | (v == 0);
      const unsigned long long c = tab[(base + v * cst) * 2 + z2];
      if (rank < c) {
        chosen = v;
        break;
      }
      rank -= c;
    }
    if (chosen < 0) return false;
    a[st] = chosen;
    z |= (chosen == 0);
  }
  return true;
}
