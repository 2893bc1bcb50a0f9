/*
 * ORACLE — TEST INFRASTRUCTURE ONLY.  Never linked into, loaded by or called
 * from the product path (paper_2311_15269_b200/).  Only tests/, the
 * `cpu_baseline` leg of bench.py and __graft_entry__.smoke() use it, as the
 * checker.
 *
 * Plain-C restatement of the reference decide kernel
 *   /root/reference/pkg/src/repsched/_core/kernel_c.pyx:23-508
 * (lex-first DFS over integer start times with FIFO bound propagation,
 * conflict jumps, memory and energetic device-load pruning, node cap and
 * deadline polling).  Every step below cites the kernel_c line range it
 * restates; data structures follow the reference one-to-one (CSR in edge-row
 * order, full per-depth lo/hi snapshots, sticky `inq` flags on a failed
 * propagation, stable insertion sorts in _mem_ok/_dev_ok) so that the NODE
 * COUNTS match, not only the verdicts.  Pinned against the compiled reference
 * in tests/test_oracle.py (per-probe status, witness and node count).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define OR_UNSAT 0
#define OR_SAT 1
#define OR_TIMEOUT 2
#define OR_CLOCK_EVERY 4096 /* kernel_c.pyx:20 */

static double or_monotonic(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

typedef struct {
  int n, ndev;
  const int64_t *dur, *mem, *init_mem;
  const uint64_t *devmask;
  int64_t *out_ptr, *out_dst, *out_lag, *in_ptr, *in_src, *in_lag;
  int64_t *conf_ptr, *conf_dst, *dev_ptr, *dev_items, *devof_ptr, *devof;
  uint8_t *placed, *inq;
  int64_t *s, *lo, *hi, *queue;
  int64_t *evt_t, *evt_m, *evt_e;
} or_state;

/* _mem_ok: kernel_c.pyx:374-425.  Events = placed items at s plus unplaced
 * negative deltas at lo, insertion-sorted by time (stable), grouped by equal
 * time, running sum checked against cap after each group. */
static int or_mem_ok(const or_state *S, int d, int64_t cap) {
  int64_t run = S->init_mem[d];
  if (run > cap) return 0;
  int ne = 0;
  for (int64_t p = S->dev_ptr[d]; p < S->dev_ptr[d + 1]; p++) {
    int i = (int)S->dev_items[p];
    int64_t tt, tm;
    if (S->placed[i]) {
      tt = S->s[i];
      tm = S->mem[i];
    } else if (S->mem[i] < 0) {
      tt = S->lo[i];
      tm = S->mem[i];
    } else {
      continue;
    }
    int j = ne;
    while (j > 0 && S->evt_t[j - 1] > tt) {
      S->evt_t[j] = S->evt_t[j - 1];
      S->evt_m[j] = S->evt_m[j - 1];
      j--;
    }
    S->evt_t[j] = tt;
    S->evt_m[j] = tm;
    ne++;
  }
  int k = 0;
  while (k < ne) {
    int64_t t = S->evt_t[k];
    while (k < ne && S->evt_t[k] == t) {
      run += S->evt_m[k];
      k++;
    }
    if (run > cap) return 0;
  }
  return 1;
}

/* _dev_ok: kernel_c.pyx:428-508.  (a, dur, e) triples, stable insertion sort
 * by a; serial-completion check; release-sorted suffix energetic check;
 * stable re-sort by e; deadline-sorted prefix energetic check. */
static int or_dev_ok(const or_state *S, int d) {
  int lo_p = (int)S->dev_ptr[d], hi_p = (int)S->dev_ptr[d + 1];
  if (hi_p == lo_p) return 1;
  int64_t lim = -((int64_t)1 << 62);
  int ne = 0;
  for (int p = lo_p; p < hi_p; p++) {
    int i = (int)S->dev_items[p];
    int64_t tt, ee;
    if (S->placed[i]) {
      tt = S->s[i];
      ee = S->s[i] + S->dur[i];
    } else {
      tt = S->lo[i];
      ee = S->hi[i] + S->dur[i];
    }
    if (ee > lim) lim = ee;
    int j = ne;
    while (j > 0 && S->evt_t[j - 1] > tt) {
      S->evt_t[j] = S->evt_t[j - 1];
      S->evt_m[j] = S->evt_m[j - 1];
      S->evt_e[j] = S->evt_e[j - 1];
      j--;
    }
    S->evt_t[j] = tt;
    S->evt_m[j] = S->dur[i];
    S->evt_e[j] = ee;
    ne++;
  }
  int64_t c = 0;
  for (int p = 0; p < ne; p++) {
    if (S->evt_t[p] > c) c = S->evt_t[p];
    c += S->evt_m[p];
  }
  if (c > lim) return 0;
  int64_t suf_p = 0, suf_e = -((int64_t)1 << 62);
  for (int p = ne - 1; p >= 0; p--) {
    suf_p += S->evt_m[p];
    if (S->evt_e[p] > suf_e) suf_e = S->evt_e[p];
    if (S->evt_t[p] + suf_p > suf_e) return 0;
  }
  for (int p = 0; p < ne; p++) {
    int64_t te = S->evt_e[p], ta = S->evt_t[p], tm = S->evt_m[p];
    int j = p;
    while (j > 0 && S->evt_e[j - 1] > te) {
      S->evt_e[j] = S->evt_e[j - 1];
      S->evt_t[j] = S->evt_t[j - 1];
      S->evt_m[j] = S->evt_m[j - 1];
      j--;
    }
    S->evt_e[j] = te;
    S->evt_t[j] = ta;
    S->evt_m[j] = tm;
  }
  int64_t pre_p = 0, pre_a = S->evt_t[0];
  for (int p = 0; p < ne; p++) {
    pre_p += S->evt_m[p];
    if (S->evt_t[p] < pre_a) pre_a = S->evt_t[p];
    if (pre_a + pre_p > S->evt_e[p]) return 0;
  }
  return 1;
}

/* FIFO propagation shared by the root (kernel_c.pyx:158-206) and the DFS
 * (kernel_c.pyx:303-340).  Queue is a ring of capacity n; on the first
 * failure the loop breaks and the flags of still-queued items stay set. */
static int or_propagate(or_state *S, int *qhead, int *qtail, int *qcount) {
  int n = S->n;
  while (*qcount > 0) {
    int a = (int)S->queue[*qhead];
    *qhead = (*qhead + 1) % n;
    (*qcount)--;
    S->inq[a] = 0;
    int64_t la = S->lo[a], ha = S->hi[a];
    for (int64_t p = S->out_ptr[a]; p < S->out_ptr[a + 1]; p++) {
      int b = (int)S->out_dst[p];
      int64_t nl = la + S->out_lag[p];
      if (nl > S->lo[b]) {
        if (nl > S->hi[b]) return 0;
        S->lo[b] = nl;
        if (!S->inq[b]) {
          S->inq[b] = 1;
          S->queue[*qtail] = b;
          *qtail = (*qtail + 1) % n;
          (*qcount)++;
        }
      }
    }
    for (int64_t p = S->in_ptr[a]; p < S->in_ptr[a + 1]; p++) {
      int b = (int)S->in_src[p];
      int64_t nh = ha - S->in_lag[p];
      if (nh < S->hi[b]) {
        if (nh < S->lo[b]) return 0;
        S->hi[b] = nh;
        if (!S->inq[b]) {
          S->inq[b] = 1;
          S->queue[*qtail] = b;
          *qtail = (*qtail + 1) % n;
          (*qcount)++;
        }
      }
    }
  }
  return 1;
}

/* decide(): kernel_c.pyx:23-371.  edges is a flat (m x 3) row-major array of
 * (src, dst, lag) meaning s[dst] >= s[src] + lag.  Returns the status; on SAT
 * the starts are written to out_starts.  *out_nodes receives the node count. */
int oracle_decide(int n, const int64_t *dur, const uint64_t *devmask, const int64_t *mem,
                  const int64_t *edges, int m, const int64_t *order, const int64_t *lo_in,
                  const int64_t *hi_in, int ndev, const int64_t *init_mem, int64_t cap,
                  int64_t node_budget, double deadline, int64_t *out_starts,
                  int64_t *out_nodes) {
  or_state S;
  memset(&S, 0, sizeof S);
  S.n = n;
  S.ndev = ndev;
  S.dur = dur;
  S.mem = mem;
  S.init_mem = init_mem;
  S.devmask = devmask;
  int nn = n > 0 ? n : 1;
  int mm = m > 0 ? m : 1;

  /* CSR for outgoing / incoming edges in edge-row order: kernel_c.pyx:54-81 */
  S.out_ptr = calloc(n + 1, sizeof(int64_t));
  S.in_ptr = calloc(n + 1, sizeof(int64_t));
  S.out_dst = malloc(mm * sizeof(int64_t));
  S.out_lag = malloc(mm * sizeof(int64_t));
  S.in_src = malloc(mm * sizeof(int64_t));
  S.in_lag = malloc(mm * sizeof(int64_t));
  for (int i = 0; i < m; i++) {
    S.out_ptr[edges[3 * i] + 1]++;
    S.in_ptr[edges[3 * i + 1] + 1]++;
  }
  for (int i = 0; i < n; i++) {
    S.out_ptr[i + 1] += S.out_ptr[i];
    S.in_ptr[i + 1] += S.in_ptr[i];
  }
  int64_t *fo = calloc(nn, sizeof(int64_t)), *fi = calloc(nn, sizeof(int64_t));
  for (int i = 0; i < m; i++) {
    int a = (int)edges[3 * i], b = (int)edges[3 * i + 1];
    int64_t lag = edges[3 * i + 2];
    S.out_dst[S.out_ptr[a] + fo[a]] = b;
    S.out_lag[S.out_ptr[a] + fo[a]] = lag;
    fo[a]++;
    S.in_src[S.in_ptr[b] + fi[b]] = a;
    S.in_lag[S.in_ptr[b] + fi[b]] = lag;
    fi[b]++;
  }
  free(fo);
  free(fi);

  /* Conflict CSR, ascending item order: kernel_c.pyx:83-98 */
  S.conf_ptr = calloc(n + 1, sizeof(int64_t));
  int64_t nconf = 0;
  for (int i = 0; i < n; i++)
    for (int j = 0; j < n; j++)
      if (i != j && (devmask[i] & devmask[j])) nconf++;
  S.conf_dst = malloc((nconf > 0 ? nconf : 1) * sizeof(int64_t));
  int64_t k = 0;
  for (int i = 0; i < n; i++) {
    for (int j = 0; j < n; j++)
      if (i != j && (devmask[i] & devmask[j])) S.conf_dst[k++] = j;
    S.conf_ptr[i + 1] = k;
  }

  /* device -> items and item -> devices CSRs: kernel_c.pyx:100-128 */
  S.dev_ptr = calloc(ndev + 1, sizeof(int64_t));
  int64_t nmemb = 0;
  for (int d = 0; d < ndev; d++) {
    for (int i = 0; i < n; i++)
      if ((devmask[i] >> d) & 1) nmemb++;
    S.dev_ptr[d + 1] = nmemb;
  }
  S.dev_items = malloc((nmemb > 0 ? nmemb : 1) * sizeof(int64_t));
  k = 0;
  for (int d = 0; d < ndev; d++)
    for (int i = 0; i < n; i++)
      if ((devmask[i] >> d) & 1) S.dev_items[k++] = i;
  S.devof_ptr = calloc(n + 1, sizeof(int64_t));
  k = 0;
  for (int i = 0; i < n; i++) {
    for (int d = 0; d < ndev; d++)
      if ((devmask[i] >> d) & 1) k++;
    S.devof_ptr[i + 1] = k;
  }
  S.devof = malloc((k > 0 ? k : 1) * sizeof(int64_t));
  k = 0;
  for (int i = 0; i < n; i++)
    for (int d = 0; d < ndev; d++)
      if ((devmask[i] >> d) & 1) S.devof[k++] = d;

  S.placed = calloc(nn, 1);
  S.inq = calloc(nn, 1);
  S.s = calloc(nn, sizeof(int64_t));
  S.queue = malloc(nn * sizeof(int64_t));
  S.lo = malloc(nn * sizeof(int64_t));
  S.hi = malloc(nn * sizeof(int64_t));
  memcpy(S.lo, lo_in, n * sizeof(int64_t));
  memcpy(S.hi, hi_in, n * sizeof(int64_t));
  int maxdi = 1;
  for (int d = 0; d < ndev; d++)
    if (S.dev_ptr[d + 1] - S.dev_ptr[d] > maxdi) maxdi = (int)(S.dev_ptr[d + 1] - S.dev_ptr[d]);
  S.evt_t = malloc(maxdi * sizeof(int64_t));
  S.evt_m = malloc(maxdi * sizeof(int64_t));
  S.evt_e = malloc(maxdi * sizeof(int64_t));
  /* per-depth full snapshots: kernel_c.pyx:147-149 */
  int64_t *snap_lo = malloc((size_t)(n + 1) * nn * sizeof(int64_t));
  int64_t *snap_hi = malloc((size_t)(n + 1) * nn * sizeof(int64_t));
  int64_t *vstack = calloc(n + 1, sizeof(int64_t));

  int64_t nodes = 0;
  int status = OR_UNSAT;
  int qhead = 0, qtail = 0, qcount = 0;

  /* Root propagation, queue seeded with 0..n-1: kernel_c.pyx:158-206 */
  for (int i = 0; i < n; i++) {
    S.queue[i] = i;
    S.inq[i] = 1;
  }
  qcount = n;
  qtail = 0;
  if (!or_propagate(&S, &qhead, &qtail, &qcount)) goto done_unsat;

  /* Root memory / device checks: kernel_c.pyx:208-215 */
  if (cap >= 0)
    for (int d = 0; d < ndev; d++)
      if (!or_mem_ok(&S, d, cap)) goto done_unsat;
  for (int d = 0; d < ndev; d++)
    if (!or_dev_ok(&S, d)) goto done_unsat;
  if (n == 0) {
    status = OR_SAT;
    goto done;
  }

  /* Iterative lex-first DFS: kernel_c.pyx:220-371 */
  {
    int depth = 0;
    int64_t v = S.lo[order[0]];
    for (;;) {
      if (depth == n) {
        status = OR_SAT;
        break;
      }
      int x = (int)order[depth];
      int64_t dx = dur[x];
      if (v > S.hi[x]) { /* exhausted: backtrack (kernel_c.pyx:231-244) */
        depth--;
        if (depth < 0) {
          status = OR_UNSAT;
          break;
        }
        x = (int)order[depth];
        memcpy(S.lo, snap_lo + (size_t)depth * nn, n * sizeof(int64_t));
        memcpy(S.hi, snap_hi + (size_t)depth * nn, n * sizeof(int64_t));
        S.placed[x] = 0;
        v = vstack[depth] + 1;
        continue;
      }
      /* conflict jump (kernel_c.pyx:245-254) */
      int moved = 1;
      while (moved) {
        moved = 0;
        for (int64_t p = S.conf_ptr[x]; p < S.conf_ptr[x + 1]; p++) {
          int y = (int)S.conf_dst[p];
          if (S.placed[y]) {
            int64_t sy = S.s[y];
            if (sy - dx < v && v < sy + dur[y]) {
              v = sy + dur[y];
              moved = 1;
            }
          }
        }
      }
      if (v > S.hi[x]) continue;
      nodes++; /* node accounting and caps (kernel_c.pyx:257-263) */
      if (node_budget && nodes > node_budget) {
        status = OR_TIMEOUT;
        break;
      }
      if (deadline != 0.0 && nodes % OR_CLOCK_EVERY == 0 && or_monotonic() > deadline) {
        status = OR_TIMEOUT;
        break;
      }
      memcpy(snap_lo + (size_t)depth * nn, S.lo, n * sizeof(int64_t));
      memcpy(snap_hi + (size_t)depth * nn, S.hi, n * sizeof(int64_t));
      S.s[x] = v;
      S.placed[x] = 1;
      S.lo[x] = v;
      S.hi[x] = v;
      int ok = 1;
      qhead = qtail = qcount = 0;
      S.queue[qtail] = x; /* enqueue x regardless of its flag (272-278) */
      qtail = (qtail + 1) % n;
      qcount++;
      S.inq[x] = 1;
      /* tighten unplaced conflicting items (kernel_c.pyx:279-302) */
      for (int64_t p = S.conf_ptr[x]; p < S.conf_ptr[x + 1] && ok; p++) {
        int y = (int)S.conf_dst[p];
        if (S.placed[y]) continue;
        int64_t dy = dur[y];
        if (v - dy < S.lo[y] && S.lo[y] < v + dx) {
          S.lo[y] = v + dx;
          if (S.lo[y] > S.hi[y]) {
            ok = 0;
            break;
          }
          if (!S.inq[y]) {
            S.inq[y] = 1;
            S.queue[qtail] = y;
            qtail = (qtail + 1) % n;
            qcount++;
          }
        }
        if (v - dy < S.hi[y] && S.hi[y] < v + dx) {
          S.hi[y] = v - dy;
          if (S.hi[y] < S.lo[y]) {
            ok = 0;
            break;
          }
          if (!S.inq[y]) {
            S.inq[y] = 1;
            S.queue[qtail] = y;
            qtail = (qtail + 1) % n;
            qcount++;
          }
        }
      }
      if (ok) {
        ok = or_propagate(&S, &qhead, &qtail, &qcount); /* 303-340, sticky on fail */
      } else {
        while (qcount > 0) { /* drain + clear flags (341-347) */
          int a = (int)S.queue[qhead];
          qhead = (qhead + 1) % n;
          qcount--;
          S.inq[a] = 0;
        }
      }
      if (ok && cap >= 0) /* 348-353 */
        for (int64_t p = S.devof_ptr[x]; p < S.devof_ptr[x + 1]; p++)
          if (!or_mem_ok(&S, (int)S.devof[p], cap)) {
            ok = 0;
            break;
          }
      if (ok) /* 354-359 */
        for (int64_t p = S.devof_ptr[x]; p < S.devof_ptr[x + 1]; p++)
          if (!or_dev_ok(&S, (int)S.devof[p])) {
            ok = 0;
            break;
          }
      if (ok) { /* descend (360-365) */
        vstack[depth] = v;
        depth++;
        if (depth < n) v = S.lo[order[depth]];
        continue;
      }
      /* failed try: restore and advance (366-371) */
      memcpy(S.lo, snap_lo + (size_t)depth * nn, n * sizeof(int64_t));
      memcpy(S.hi, snap_hi + (size_t)depth * nn, n * sizeof(int64_t));
      S.placed[x] = 0;
      v++;
    }
  }
  goto done;
done_unsat:
  status = OR_UNSAT;
  nodes = 0;
done:
  if (status == OR_SAT && out_starts) memcpy(out_starts, S.s, n * sizeof(int64_t));
  *out_nodes = nodes;
  free(S.out_ptr); free(S.in_ptr); free(S.out_dst); free(S.out_lag); free(S.in_src);
  free(S.in_lag); free(S.conf_ptr); free(S.conf_dst); free(S.dev_ptr); free(S.dev_items);
  free(S.devof_ptr); free(S.devof); free(S.placed); free(S.inq); free(S.s); free(S.queue);
  free(S.lo); free(S.hi); free(S.evt_t); free(S.evt_m); free(S.evt_e);
  free(snap_lo); free(snap_hi); free(vstack);
  return status;
}
