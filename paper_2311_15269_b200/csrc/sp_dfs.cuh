// sp_dfs.cuh — speculative subtree-parallel reference-exact DFS (SP-DFS).
//
// One long reference decide (kernel_c.pyx:220-371; e.g. the 8M-node-capped
// completion probes of solver.py:280, or 400k-node repetend probes) is split
// at a depth ds into SUBTREE TASKS run by many warps at once, with results
// identical to the sequential DFS — status, lex-min witness and node count.
//
// Why this is exact.  Between two nodes the sequential DFS carries only
// (a) bounds / placements, restored from per-depth snapshots on backtrack,
// and (b) the "sticky" in-queue flags S that a failed propagation leaves
// behind (kernel_c.pyx:303-347).  The exploration of the subtree below a
// node at depth ds-1 is therefore a pure function of its entry state
// (bounds, placements) and S_in, returning (nodes, SAT witness or exhausted,
// S_out).  The MASTER walks the shallow part (depths < ds) exactly and, at
// each descent into depth ds, emits a task with its entry state and
// S_in = current S, then continues as if the subtree were exhausted with
// S_out = S_in (speculation).  Helpers run the tasks.  The host then checks
// the speculation task by task in DFS order: while every task returned
// S_out == S_in, the master's walk was the exact one, so node counts add up
// in order and the first SAT task (or the node cap) settles the probe.  At
// the first task with S_out != S_in everything after it is discarded and the
// master's walk is replayed from the round start with that task's true S_out
// (measured: S_out == S_in for all 3,075 / 8,624 subtrees of the two
// 8M-node C3 completion probes and ~99% of repetend subtrees).
//
// Master state records (global memory, int words):
//   [0] depth  [1] v  [2] fresh (root propagation pending)  [3] unused
//   lo[n] hi[n] s[n] vstack[n+1] placed[nw] inq[nw] snap[2 n (n+1)] (int2/depth)
// Task records: lo[n] hi[n] s[n] placed[nw] inq[nw] v depth  (the rest of
//   depth `depth` from value v, and everything below it)
// Task results: status, nodes (2 words), inq_out[nw], s[n]
#pragma once
#include "wrx_dfs.cuh"

#define SP_EXHAUSTED 4  // subtree / sub-range exhausted (backtracked below the floor)
#define SP_PAUSED 5     // master stopped after emitting its task quota
#define SP_INVALID 8    // piece stopped: a piece before it in DFS order ended with another sticky set

__host__ __device__ inline int sp_nw(int n) { return ((n > 0 ? n : 1) + 31) / 32; }
// words before the snapshot area, rounded up so the int2 snapshots are aligned
__host__ __device__ inline long long sp_state_head(int n) {
  const long long nn = n > 0 ? n : 1;
  return (4 + 3 * nn + (nn + 1) + 2 * sp_nw(n) + 3) / 4 * 4;
}
__host__ __device__ inline long long sp_state_words(int n) {
  const long long nn = n > 0 ? n : 1;
  return sp_state_head(n) + 2 * nn * (nn + 1);
}
// task record: lo[n] hi[n] s[n] placed[nw] inq[nw] v depth
__host__ __device__ inline long long sp_task_words(int n) {
  const long long nn = n > 0 ? n : 1;
  return 3 * nn + 2 * sp_nw(n) + 2;
}
// donated piece result: status, nodes (2 words), moved, s[n], inq_out[nw]
__host__ __device__ inline long long sp_pres_words(int n) {
  return 4 + (n > 0 ? n : 1) + sp_nw(n);
}
__host__ __device__ inline long long sp_result_words(int n) {
  const long long nn = n > 0 ? n : 1;
  return 4 + sp_nw(n) + nn;
}

struct SpState {  // views into a master state record
  int *hdr, *lo, *hi, *s, *vstack;
  unsigned *placed, *inq;
  int2 *snap;
};
__host__ __device__ inline SpState sp_state_view(int *base, int n) {
  const int nn = n > 0 ? n : 1, nw = sp_nw(n);
  SpState r;
  int *p = base;
  r.hdr = p; p += 4;
  r.lo = p; p += nn;
  r.hi = p; p += nn;
  r.s = p; p += nn;
  r.vstack = p; p += nn + 1;
  r.placed = (unsigned *)p; p += nw;
  r.inq = (unsigned *)p;
  r.snap = (int2 *)(base + sp_state_head(n));
  return r;
}

#ifdef __CUDACC__
// copy the mutable arrays between a record and the warp's shared state
__device__ inline void sp_load(WWs &w, const int *lo, const int *hi, const int *s,
                               const unsigned *placed, const unsigned *inq, int n) {
  const int lane = wrx_lane(), nw = sp_nw(n);
  for (int i = lane; i < n; i += 32) {
    w.lo[i] = lo[i];
    w.hi[i] = hi[i];
    w.s[i] = s[i];
  }
  for (int i = lane; i < nw; i += 32) {
    w.placed[i] = placed[i];
    w.inq[i] = inq[i];
  }
  __syncwarp();
}
// the same from a record another SM wrote during this launch (L2, not L1)
__device__ inline void sp_load_cg(WWs &w, const int *rec, int n) {
  const int lane = wrx_lane(), nw = sp_nw(n);
  for (int i = lane; i < n; i += 32) {
    w.lo[i] = __ldcg(rec + i);
    w.hi[i] = __ldcg(rec + n + i);
    w.s[i] = __ldcg(rec + 2 * n + i);
  }
  for (int i = lane; i < nw; i += 32) {
    w.placed[i] = (unsigned)__ldcg(rec + 3 * n + i);
    w.inq[i] = (unsigned)__ldcg(rec + 3 * n + nw + i);
  }
  __syncwarp();
}
__device__ inline void sp_store(const WWs &w, int *lo, int *hi, int *s, unsigned *placed,
                                unsigned *inq, int n) {
  const int lane = wrx_lane(), nw = sp_nw(n);
  __syncwarp();
  for (int i = lane; i < n; i += 32) {
    lo[i] = w.lo[i];
    hi[i] = w.hi[i];
    s[i] = w.s[i];
  }
  for (int i = lane; i < nw; i += 32) {
    placed[i] = w.placed[i];
    inq[i] = w.inq[i];
  }
  __syncwarp();
}

// Task sink of the master walk.
struct SpSink {
  int *tasks;          // task records
  long long *pre;      // master nodes counted before each task (this walk)
  int count, max;
  const unsigned *ovr; // true S_out of the first n_ovr tasks (replay after a misprediction)
  int n_ovr;
  // replay checkpoints: the full master state right before emitting task
  // k = j * ck_every (state record j of `ck`, its round-relative node count
  // in ck_nodes[j]), written for j >= ck_have
  int *ck;
  long long *ck_nodes;
  int ck_every, ck_have;
  long long ck_base;
};

// The reference DFS loop of wrx_decide (kernel_c.pyx:225-371) generalised:
// starts at (depth, v) with the live state in w (snapshots of depths
// < depth valid), never backtracks below `floor` (returns SP_EXHAUSTED), and
// — when `sink` is given — turns every descent into depth `split` into a
// task (see the header).  *nodes counts this call's nodes; the cap applies
// to (*nodes + base_nodes).  Returns RX_SAT / RX_TIMEOUT / SP_EXHAUSTED /
// SP_PAUSED with depth / v updated.
// Early stop of a speculative task that can no longer matter: task k's
// nodes are only ever counted after every earlier task of its round, so once
// base + pre[k] + (nodes already explored by tasks 0..k-1) exceeds the cap,
// the probe's verdict is settled before task k (TIMEOUT there, or an earlier
// task's SAT) and task k stops.  Counts are published every 256 nodes.
struct SpCut {
  long long *part;       // per task: nodes explored so far
  const long long *pre;  // per task: master nodes before it (this walk)
  long long base, budget;
  int k;
  long long published;   // (donation mode) own nodes already added to part[k]
};

// Dynamic donation (work splitting inside a task launch).  Idle task warps
// claim queue slots beyond the launch's tasks; a running piece that sees a
// claimed-but-unfilled slot gives away "the rest of depth d from value
// vstack[d] + 1" for the SHALLOWEST depth d >= its floor that still has
// untried values, and clamps d in its own snapshot so that it never returns
// there.  In DFS order a piece's own exploration comes first, then its
// donated pieces, deepest donation first (each later donation is deeper:
// every depth <= the previous donation's is exhausted for the donor).  A
// piece runs on the speculation S_in = the task's S (donation only while the
// donor's sticky set equals it; any piece ending with another set makes the
// host re-run the task undivided).  Every piece explores its own subtree in
// DFS order, so a stopped piece still bounds the DFS prefix: the host walks
// a task's pieces in DFS order (sp_host.inc, sp_combine).
struct SpDon {
  unsigned *ctl;           // [0] claims  [1] slots reserved  [2] pieces outstanding
  int *precs;              // piece records (sp_task_words each)
  int *pmeta;              // per piece: task, parent slot, depth, ready
  int *pres;               // per piece: status, nodes (2 words), moved, witness[n]
  long long *pnodes;       // per slot: own nodes explored so far (published)
  long long *psub;         // per slot: nodes of its subtree of pieces (published)
  int *plast;              // per slot: its latest donation (-1: none)
  int *pprev;              // per piece: its donor's previous donation (-1: none)
  int *pmoved;             // per slot: 1 = ends the usable DFS prefix (sticky set changed,
                           // SAT or cap), 2 = a piece in its subtree does
  int first;               // task index of slot 0
  int count, cap;          // task slots of the launch; piece capacity
  int self, parent;        // this piece's slot; its donor's slot (-1 for a task)
  const unsigned *s_in;    // the task's sticky set
  int every;               // donation check interval (nodes, power of two)
  int force;               // donate at every check (testing)
  int any_s;               // donate on any sticky set (the piece starts on the donor's)
  int *tmade, *tdone;      // per task slot: pieces donated / pieces finished (+1: the task)
  int slot_task;           // this piece's task slot
  int window;              // donate only within this many tasks of the leftmost open one (-1: any)
};

// A piece of task slot ts finished: when it was the task's last one, move the
// leftmost-open-task mark (ctl[3]) past every finished task.  Lane 0 only.
__device__ inline void sp_task_piece_done(const SpDon &d, int ts) {
  __threadfence();
  atomicAdd(&d.tdone[ts], 1);
  for (;;) {
    const unsigned lo = ((volatile unsigned *)d.ctl)[3];
    if (lo >= (unsigned)d.count) break;
    if (((volatile int *)d.tdone)[lo] != ((volatile int *)d.tmade)[lo] + 1) break;
    atomicCAS(&d.ctl[3], lo, lo + 1);
  }
}

// Published nodes that precede this piece in DFS order inside its task:
// for every donor A on its chain, A's own nodes and the subtree totals of
// A's donations made after the one this piece descends from (those come
// first in DFS order).  Lane 0 only.
// *invalid: a piece before it in DFS order (a donor's own part, or a
// preceding donation's subtree) ended with another sticky set.
__device__ inline long long sp_prefix_nodes(const SpDon &d, bool *invalid) {
  long long s = 0;
  for (int b = d.self, a = d.parent; a >= 0;) {
    s += ((volatile long long *)d.pnodes)[a];
    if (((volatile int *)d.pmoved)[a] & 1) *invalid = true;
    for (int c = ((volatile int *)d.plast)[a]; c >= 0 && c != b;
         c = ((volatile int *)d.pprev)[c - d.count]) {
      s += ((volatile long long *)d.psub)[c];
      if (((volatile int *)d.pmoved)[c] & 2) *invalid = true;
    }
    if (a < d.count) break;
    b = a;
    a = ((volatile int *)d.pmeta)[4 * (a - d.count) + 1];
  }
  return s;
}

// A piece ended with another sticky set: flag it and every donor's subtree.
// Lane 0 only.
__device__ inline void sp_mark_moved(const SpDon &d) {
  atomicOr(&d.pmoved[d.self], 3);
  for (int a = d.parent; a >= 0;) {
    atomicOr(&d.pmoved[a], 2);
    if (a < d.count) break;
    a = ((volatile int *)d.pmeta)[4 * (a - d.count) + 1];
  }
}

// Publish `delta` more own nodes of this piece into its subtree total and
// every donor's.  Lane 0 only.
__device__ inline void sp_publish_sub(const SpDon &d, long long delta) {
  if (!delta) return;
  for (int a = d.self; a >= 0;) {
    atomicAdd((unsigned long long *)&d.psub[a], (unsigned long long)delta);
    if (a < d.count) break;
    a = ((volatile int *)d.pmeta)[4 * (a - d.count) + 1];
  }
}

// Give away the rest of the shallowest donatable depth (see SpDon).  Called
// by the whole warp between nodes: depths < depth hold valid snapshots and
// vstack entries.
template <class M>
__device__ void sp_donate(const M &md, WWs &w, SpDon &d, int floor, int depth, int task) {
  const int n = md.n(), nw = sp_nw(n), lane = wrx_lane();
  int want = 0;
  if (lane == 0) {
    const unsigned head = ((volatile unsigned *)d.ctl)[0], tail = ((volatile unsigned *)d.ctl)[1];
    want = (d.force || head > tail) && tail < (unsigned)(d.count + d.cap);
    // help only the leftmost unfinished tasks (DFS order): pieces of later
    // tasks mostly explore beyond the cap position
    if (want && d.window >= 0 && !d.force)
      want = d.slot_task - (int)((volatile unsigned *)d.ctl)[3] <= d.window;
  }
  if (!__shfl_sync(WRX_FULL, want, 0)) return;
  if (!d.any_s) {  // donate only on the piece's own set
    bool diff = false;
    for (int i = lane; i < nw; i += 32) diff |= w.inq[i] != d.s_in[i];
    if (__any_sync(WRX_FULL, diff)) return;
  }
  int dd = -1;
  for (int b = floor; b < depth && dd < 0; b += 32) {
    const int j = b + lane;
    bool ok = false;
    if (j < depth) ok = w.vstack[j] + 1 <= w.snap[(long long)j * n + md.order(j)].y;
    const unsigned m = __ballot_sync(WRX_FULL, ok);
    if (m) dd = b + __ffs(m) - 1;
  }
  if (dd < 0) return;
  int slot = 0;
  if (lane == 0) slot = (int)atomicAdd(&d.ctl[1], 1u);
  slot = __shfl_sync(WRX_FULL, slot, 0);
  const int p = slot - d.count;
  if (p >= d.cap) return;  // raced past the capacity: keep the work
  if (lane == 0) {
    atomicAdd(&d.ctl[2], 1u);
    atomicAdd(&d.tmade[d.slot_task], 1);  // before the piece can finish
  }
  int *rec = d.precs + (long long)p * sp_task_words(n);
  const int2 *sn = w.snap + (long long)dd * n;
  for (int i = lane; i < n; i += 32) {
    const int2 q = sn[i];
    rec[i] = q.x;
    rec[n + i] = q.y;
    rec[2 * n + i] = w.s[i];
  }
  // placed at the piece's entry: the items of depths < dd
  for (int i = lane; i < nw; i += 32) {
    unsigned m = 0;
    for (int j = 0; j < dd; ++j) {
      const int x = md.order(j);
      if ((x >> 5) == i) m |= 1u << (x & 31);
    }
    rec[3 * n + i] = (int)m;
    rec[3 * n + nw + i] = (int)w.inq[i];
  }
  __syncwarp();  // every lane has read the snapshot before lane 0 clamps it
  if (lane == 0) {
    rec[3 * n + 2 * nw] = w.vstack[dd] + 1;
    rec[3 * n + 2 * nw + 1] = dd;
    int *pm = d.pmeta + 4 * p;
    pm[0] = task;
    pm[1] = d.self;
    pm[2] = dd;
    d.pprev[p] = ((volatile int *)d.plast)[d.self];
    // the donor never returns to depth dd: its snapshot's hi of the item
    // placed there ends at the value it holds
    w.snap[(long long)dd * n + md.order(dd)].y = w.vstack[dd];
  }
  __syncwarp();
  if (lane == 0) {
    __threadfence();
    ((volatile int *)d.plast)[d.self] = slot;     // first in DFS order among the donations
    ((volatile int *)d.pmeta)[4 * p + 3] = 1;  // ready
  }
  __syncwarp();
}

template <class M>
__device__ int sp_explore(const M &md, WWs &w, int floor, int split, int &depth, int &v,
                          long long budget, long long base_nodes, long long *nodes_io,
                          SpSink *sink, long long pause_nodes = 0, int *hist = nullptr,
                          SpCut *cut = nullptr, SpDon *don = nullptr, int task = -1) {
  const int n = md.n(), cap = md.cap();
  const int lane = wrx_lane();
  long long nodes = *nodes_io;
  int status;
  int qh = 0, qt = 0, qc = 0;
  for (;;) {
    if (depth == n) {
      status = RX_SAT;
      break;
    }
    if (pause_nodes && nodes >= pause_nodes) {  // a consistent resume point
      status = SP_PAUSED;
      break;
    }
    if (sink && depth >= split) {  // the rest of this depth becomes a task
      // (at a descent into `split` that is a whole subtree; a master standing
      // deeper — after a resume or a split change — climbs back emitting
      // the rest of every depth on its way, deepest first = DFS order)
      if (sink->count == sink->max) {
        status = SP_PAUSED;
        break;
      }
      const int k = sink->count;
      const int nw = sp_nw(n);
      if (sink->ck && k % sink->ck_every == 0 && k / sink->ck_every >= sink->ck_have) {
        const int j = k / sink->ck_every;
        SpState c = sp_state_view(sink->ck + (long long)j * sp_state_words(n), n);
        sp_store(w, c.lo, c.hi, c.s, c.placed, c.inq, n);
        for (int i = lane; i <= n; i += 32) c.vstack[i] = w.vstack[i];
        for (long long i = lane; i < (long long)depth * n; i += 32) c.snap[i] = w.snap[i];
        if (lane == 0) {
          c.hdr[0] = depth;
          c.hdr[1] = v;
          c.hdr[2] = 0;
          sink->ck_nodes[j] = sink->ck_base + nodes;
        }
        __syncwarp();
      }
      int *rec = sink->tasks + (long long)k * sp_task_words(n);
      sp_store(w, rec, rec + n, rec + 2 * n, (unsigned *)(rec + 3 * n),
               (unsigned *)(rec + 3 * n + nw), n);
      // the task is the rest of depth `split` from value v (a fresh descent
      // has v = lo[order(split)]; after a resume or a split change the master
      // can also stand inside depth `split`) and everything below it
      if (lane == 0) {
        sink->pre[k] = nodes;
        rec[3 * n + 2 * nw] = v;
        rec[3 * n + 2 * nw + 1] = depth;
      }
      sink->count = k + 1;
      if (k < sink->n_ovr) {  // replay: the task's true sticky set
        const unsigned *so = sink->ovr + (long long)k * nw;
        for (int i = lane; i < nw; i += 32) w.inq[i] = so[i];
      }
      // speculation: the subtree is exhausted and leaves S unchanged —
      // backtrack exactly like the reference after exhausting depth `split`
      --depth;
      const int x = md.order(depth);
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
    int x = md.order(depth);
    const int dx = md.dur(x);
    if (v > w.hi[x]) {  // exhausted: backtrack and restore the depth's snapshot
      if (depth - 1 < floor) {
        status = SP_EXHAUSTED;
        break;
      }
      --depth;
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
    if (budget && nodes + base_nodes > budget) {
      status = RX_TIMEOUT;
      break;
    }
    if (hist && lane == 0) ++hist[depth];
    if (cut && (nodes & 255) == 0) {
      long long sum = 0;
      for (int j = lane; j < cut->k; j += 32) sum += ((volatile long long *)cut->part)[j];
      for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(WRX_FULL, sum, o);
      if (!don) {
        if (lane == 0) ((volatile long long *)cut->part)[cut->k] = nodes;
        if (cut->budget > 0 && cut->base + cut->pre[cut->k] + sum > cut->budget) {
          status = RX_ABORT;
          break;
        }
      } else {
        // pieces of one task add up in part[k]; the DFS prefix before this
        // node also holds every donor's own nodes and this piece's own
        long long anc = 0;
        bool inval = false;
        if (lane == 0) {
          atomicAdd((unsigned long long *)&cut->part[cut->k],
                    (unsigned long long)(nodes - cut->published));
          ((volatile long long *)don->pnodes)[don->self] = nodes;
          sp_publish_sub(*don, nodes - cut->published);
          anc = sp_prefix_nodes(*don, &inval);
        }
        for (int j = don->first + lane; j < cut->k; j += 32)
          inval |= (((volatile int *)don->pmoved)[j - don->first] & 2) != 0;
        anc = __shfl_sync(WRX_FULL, anc, 0);
        cut->published = nodes;
        if (__any_sync(WRX_FULL, inval)) {
          status = SP_INVALID;
          break;
        }
        if (cut->budget > 0 && cut->base + cut->pre[cut->k] + sum + anc + nodes > cut->budget) {
          status = RX_ABORT;
          break;
        }
      }
    }
    if (don && (nodes & (don->every - 1)) == 0 && depth > floor)
      sp_donate(md, w, *don, floor, depth, task);
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
      wrx_enqueue(w, chg && !inq, y, n, qt, qc, false);
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
  *nodes_io = nodes;
  __syncwarp();
  return status;
}

// Root step of the reference decide (kernel_c.pyx:158-215) on the warp
// state: all items queued and flagged, FIFO propagation, root memory / device
// checks.  Returns false = UNSAT with 0 nodes.
template <class M>
__device__ bool sp_root(const M &md, WWs &w) {
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
  if (!wrx_propagate(md, w, qh, qt, qc)) return false;
  if (cap >= 0)
    for (int d = 0; d < ndev; ++d)
      if (!wrx_mem_ok(md, w, d, cap)) return false;
  for (int d = 0; d < ndev; ++d)
    if (!wrx_dev_ok(md, w, d)) return false;
  return true;
}
#endif
