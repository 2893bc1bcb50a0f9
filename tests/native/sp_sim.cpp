// Test-only host model of the subtree-parallel decide (csrc/sp_dfs.cuh +
// csrc/sp_host.inc): the same master walk / task / in-order verification /
// replay / nested sub-solve algorithm, run sequentially on the CPU with the
// host build of the reference-exact DFS steps (rx_dfs.cuh).  Checks the
// ALGORITHM (exact status, witness and node count for any split depth and
// round sizes) against the oracle, and reports a parallel-time model
// (sum over rounds of master nodes + largest task) to tune the heuristics.
//
// stdin: "G" problems as in rx_host_check.cpp, preceded per problem by
//        "P first tasks pause task_nodes ds0" (ds0 = 0: histogram rule).
// stdout per problem: status nodes rounds tasks replays subsolves model [starts]
#include <cstdio>
#include <cstdlib>
#include <iostream>
#include <vector>

#include "../../paper_2311_15269_b200/csrc/host_build.hpp"

#define SP_EXHAUSTED 4
#define SP_PAUSED 5

template <class T>
static std::vector<T> rd(int k) {
  std::vector<T> v(k);
  for (auto &x : v) {
    long long y;
    std::cin >> y;
    x = (T)y;
  }
  return v;
}

struct St {  // full DFS state (master record or task record)
  std::vector<int> lo, hi, s, vstack;
  std::vector<unsigned char> placed, inq;
  std::vector<int> snlo, snhi;  // per-depth snapshots (n x n)
  int depth = 0, v = 0;
};

struct Sim {
  const GenView &g;
  int n;
  std::vector<int> ws;
  RxWs w;
  long long par_model = 0, rounds = 0, tasks = 0, replays = 0, subsolves = 0;
  long long P_FIRST, P_TASKS, P_PAUSE, P_TASKN;
  std::vector<long long> hist;

  Sim(const GenView &gv, int maxdi) : g(gv), n(gv.n_) {
    ws.assign(rx_ws_words(n, maxdi) + 8, 0);
    w = rx_ws_carve(ws.data(), n, maxdi);
  }
  void load(const St &a) {
    for (int i = 0; i < n; ++i) {
      w.lo[i] = a.lo[i];
      w.hi[i] = a.hi[i];
      w.s[i] = a.s[i];
      w.placed[i] = a.placed[i];
      w.inq[i] = a.inq[i];
    }
  }
  void store(St &a) {
    for (int i = 0; i < n; ++i) {
      a.lo[i] = w.lo[i];
      a.hi[i] = w.hi[i];
      a.s[i] = w.s[i];
      a.placed[i] = w.placed[i];
      a.inq[i] = w.inq[i];
    }
  }
  St blank() {
    St a;
    a.lo.assign(n, 0);
    a.hi.assign(n, 0);
    a.s.assign(n, 0);
    a.vstack.assign(n + 1, 0);
    a.placed.assign(n, 0);
    a.inq.assign(n, 0);
    a.snlo.assign((size_t)n * n + 1, 0);
    a.snhi.assign((size_t)n * n + 1, 0);
    return a;
  }
  bool root(St &a) {
    for (int i = 0; i < n; ++i) {
      w.lo[i] = g.lo_[i];
      w.hi[i] = g.hi_[i];
      w.placed[i] = 0;
      w.inq[i] = 1;
      w.queue[i] = i;
      w.stamp[i] = 0;
    }
    int qh = 0, qt = 0, qc = n, tn = 0;
    bool ok = rx_propagate<false>(g, w, qh, qt, qc, 0u, tn);
    if (ok && g.cap() >= 0)
      for (int d = 0; d < g.ndev() && ok; ++d) ok = rx_mem_ok(g, w, d, g.cap());
    for (int d = 0; d < g.ndev() && ok; ++d) ok = rx_dev_ok(g, w, d);
    store(a);
    return ok;
  }
  void restore_depth(St &a, int d) {
    for (int i = 0; i < n; ++i) {
      w.lo[i] = a.snlo[(size_t)d * n + i];
      w.hi[i] = a.snhi[(size_t)d * n + i];
    }
  }
  // port of sp_explore (sp_dfs.cuh) over the record `a` (live arrays in w)
  long long CK = 64;
  bool debug = false;
  struct Ckpt {
    St st;
    long long nodes;
  };
  std::vector<Ckpt> *ckpts = nullptr;
  size_t k_base = 0;  // index of the first task this walk emits
  long long ck_base = 0;  // round-relative master nodes at the walk's start
  int explore(St &a, int floor, int split, long long budget, long long base, long long *nodes_io,
              std::vector<St> *sink, std::vector<long long> *pre, size_t max_tasks,
              const std::vector<std::vector<unsigned char>> *ovr, long long pause,
              bool do_hist) {
    int &depth = a.depth, &v = a.v;
    long long nodes = *nodes_io;
    int status;
    for (;;) {
      if (depth == n) {
        status = RX_SAT;
        break;
      }
      if (pause && nodes >= pause) {
        status = SP_PAUSED;
        break;
      }
      if (sink && depth >= split) {  // emit the rest of this depth (climbing if deeper)
        if (sink->size() == max_tasks) {
          status = SP_PAUSED;
          break;
        }
        const size_t k = sink->size();
        if (ckpts && k % CK == 0 && k / CK >= ckpts->size()) {  // resume point before task k
          Ckpt c{a, ck_base + nodes};  // absolute within the round
          store(c.st);
          ckpts->push_back(c);
        }
        St t = blank();
        store(t);
        t.depth = depth;
        t.v = v;
        sink->push_back(t);
        pre->push_back(nodes);
        if (ovr && k < ovr->size())
          for (int i = 0; i < n; ++i) w.inq[i] = (*ovr)[k][i];
        --depth;
        restore_depth(a, depth);
        w.placed[g.order(depth)] = 0;
        v = a.vstack[depth] + 1;
        continue;
      }
      int x = g.order(depth);
      const int dx = g.dur(x);
      if (v > w.hi[x]) {
        if (depth - 1 < floor) {
          status = SP_EXHAUSTED;
          break;
        }
        --depth;
        x = g.order(depth);
        restore_depth(a, depth);
        w.placed[x] = 0;
        v = a.vstack[depth] + 1;
        continue;
      }
      const int cb = g.conf_begin(x), ce = g.conf_end(x);
      for (bool moved = true; moved;) {
        moved = false;
        for (int p = cb; p < ce; ++p) {
          const int y = g.conf_dst(p);
          if (w.placed[y]) {
            const int sy = w.s[y], ey = sy + g.dur(y);
            if (sy - dx < v && v < ey) {
              v = ey;
              moved = true;
            }
          }
        }
      }
      if (v > w.hi[x]) continue;
      ++nodes;
      if (budget && nodes + base > budget) {
        status = RX_TIMEOUT;
        break;
      }
      if (do_hist) ++hist[depth];
      for (int i = 0; i < n; ++i) {
        a.snlo[(size_t)depth * n + i] = w.lo[i];
        a.snhi[(size_t)depth * n + i] = w.hi[i];
      }
      w.s[x] = v;
      w.placed[x] = 1;
      w.lo[x] = v;
      w.hi[x] = v;
      bool ok = true;
      int qh = 0, qt = 0, qc = 0, tn = 0;
      rx_push(w, x, n, qt, qc);
      for (int p = cb; p < ce; ++p) {
        const int y = g.conf_dst(p);
        if (w.placed[y]) continue;
        const int dy = g.dur(y);
        if (v - dy < w.lo[y] && w.lo[y] < v + dx) {
          w.lo[y] = v + dx;
          if (w.lo[y] > w.hi[y]) {
            ok = false;
            break;
          }
          if (!w.inq[y]) rx_push(w, y, n, qt, qc);
        }
        if (v - dy < w.hi[y] && w.hi[y] < v + dx) {
          w.hi[y] = v - dy;
          if (w.hi[y] < w.lo[y]) {
            ok = false;
            break;
          }
          if (!w.inq[y]) rx_push(w, y, n, qt, qc);
        }
      }
      if (ok) ok = rx_propagate<false>(g, w, qh, qt, qc, 0u, tn);
      else
        while (qc > 0) {
          w.inq[w.queue[qh]] = 0;
          if (++qh == n) qh = 0;
          --qc;
        }
      const int fb = g.devof_begin(x), fe = g.devof_end(x);
      if (ok && g.cap() >= 0)
        for (int p = fb; p < fe && ok; ++p) ok = rx_mem_ok(g, w, g.devof(p), g.cap());
      for (int p = fb; p < fe && ok; ++p) ok = rx_dev_ok(g, w, g.devof(p));
      if (ok) {
        a.vstack[depth] = v;
        ++depth;
        if (depth < n) v = w.lo[g.order(depth)];
        continue;
      }
      restore_depth(a, depth);
      w.placed[x] = 0;
      ++v;
    }
    *nodes_io = nodes;
    return status;
  }
  int run_master(St &a, int floor, int split, long long budget, long long base, long long pause,
                 std::vector<St> *sink, std::vector<long long> *pre,
                 const std::vector<std::vector<unsigned char>> *ovr, long long *nodes, bool hist) {
    load(a);
    *nodes = 0;
    int st = explore(a, floor, split, budget, base, nodes, sink, pre, (size_t)P_TASKS, ovr, pause,
                     hist);
    store(a);
    return st;
  }
  int run_task(St t, long long budget, long long *nodes, St *out) {
    load(t);
    *nodes = 0;
    int st = explore(t, t.depth, n + 1, budget, 0, nodes, nullptr, nullptr, 0, nullptr, 0, false);
    store(t);
    *out = t;
    return st;
  }
  // port of SpRun::run (sp_host.inc)
  int run(St &a, int floor, int ds, long long budget, long long base, long long *nodes_out,
          std::vector<int> *wit, int lev) {
    for (;;) {
      ++rounds;
      std::vector<std::vector<unsigned char>> ovr;
      std::vector<St> res_state;
      std::vector<int> res_st;
      std::vector<long long> res_n;
      std::vector<Ckpt> cks;
      std::vector<St> tk;
      std::vector<long long> pre;
      long long m_nodes = 0, m_base = 0;
      const int ds_round = ds;
      for (;;) {
        ckpts = &cks;
        ck_base = m_base;
        long long mn = 0;
        const int m_status = run_master(a, floor, ds_round, budget, base, P_PAUSE, &tk, &pre,
                                        &ovr, &mn, false);
        ckpts = nullptr;
        m_nodes = m_base + mn;
        // pre[] of re-walked tasks are relative to the checkpoint: rebase
        for (size_t i = k_base; i < pre.size(); ++i) pre[i] += m_base;
        const long long left = budget ? budget - base : 0;
        const long long tbud = left ? std::min(left, P_TASKN) : P_TASKN;
        long long max_round = 0;
        for (size_t i = res_st.size(); i < tk.size(); ++i) {
          long long tn = 0;
          St out;
          const int st = run_task(tk[i], tbud, &tn, &out);
          res_st.push_back(st);
          res_n.push_back(tn);
          res_state.push_back(out);
          max_round = std::max(max_round, std::min(tn, tbud));
          ++tasks;
        }
        par_model += mn + max_round;
        long long acc = base, max_t = 0;
        int mismatch = -1;
        for (size_t i = 0; i < tk.size(); ++i) {
          long long tn = res_n[i];
          const long long before = acc + pre[i];
          if (budget && before > budget) return *nodes_out = budget + 1, RX_TIMEOUT;
          int st = res_st[i];
          if (st == RX_TIMEOUT && (!budget || tbud < budget - before)) {
            if (tk[i].depth + 1 >= n) {
              std::fprintf(stderr, "nesting limit\n");
              std::exit(3);
            }
            ++subsolves;
            St sub = tk[i];
            long long sn = 0;
            std::vector<int> sw;
            const int fl = tk[i].depth;
            const int ss = run(sub, fl, std::min(n - 1, fl + 2), budget ? budget - before : 0, 0,
                               &sn, &sw, lev + 1);
            if (ss == RX_SAT) {
              const long long tot = before + sn;
              if (budget && tot > budget) return *nodes_out = budget + 1, RX_TIMEOUT;
              *wit = sw;
              *nodes_out = tot;
              return RX_SAT;
            }
            if (ss == RX_TIMEOUT) return *nodes_out = budget + 1, RX_TIMEOUT;
            st = res_st[i] = SP_EXHAUSTED;
            tn = res_n[i] = sn;
            res_state[i] = sub;
          }
          if (st == RX_SAT) {
            const long long tot = before + tn;
            if (budget && tot > budget) return *nodes_out = budget + 1, RX_TIMEOUT;
            *wit = res_state[i].s;
            *nodes_out = tot;
            return RX_SAT;
          }
          if (st == RX_TIMEOUT) return *nodes_out = budget + 1, RX_TIMEOUT;
          acc += tn;
          max_t = std::max(max_t, tn);
          if (debug)
            std::fprintf(stderr, "task %zu depth %d v %d pre %lld tn %lld st %d moved %d\n", i,
                         tk[i].depth, tk[i].v, pre[i], tn, st, (int)(res_state[i].inq != tk[i].inq));
          if (res_state[i].inq != tk[i].inq && i >= ovr.size()) {
            mismatch = (int)i;
            break;
          }
        }
        if (mismatch >= 0) {
          ++replays;
          ovr.clear();
          for (int i = 0; i <= mismatch; ++i) ovr.push_back(res_state[i].inq);
          res_st.resize(mismatch + 1);
          res_n.resize(mismatch + 1);
          res_state.resize(mismatch + 1);
          // resume the walk at the last checkpoint at or before the mismatch
          const size_t c = (size_t)mismatch / CK;
          a = cks[c].st;
          m_base = cks[c].nodes;
          cks.resize(c + 1);
          tk.resize(c * CK);
          pre.resize(c * CK);
          k_base = c * CK;
          continue;
        }
        k_base = 0;
        m_base = 0;
        const long long total = acc + m_nodes;
        if (debug)
          std::fprintf(stderr, "round lev %d ds %d tasks %zu m_nodes %lld max_t %lld status %d\n",
                       lev, ds, tk.size(), m_nodes, max_t, m_status);
        if (m_status == SP_PAUSED) {
          base = total;
          if (tk.empty()) ds = std::max(floor + 1, ds - 2);
          else if (m_nodes > 2 * max_t && ds > floor + 1) --ds;
          else if (max_t > 4 * m_nodes && ds < n - 1) ++ds;
          break;
        }
        if (budget && total > budget) return *nodes_out = budget + 1, RX_TIMEOUT;
        *nodes_out = total;
        if (m_status == RX_SAT) *wit = a.s;
        return m_status;
      }
    }
  }
};

int main() {
  std::string tag;
  while (std::cin >> tag) {
    long long first, ntasks, pause, taskn;
    int ds0;
    std::cin >> first >> ntasks >> pause >> taskn >> ds0;
    std::cin >> tag;  // "G"
    int n, m, ndev;
    long long cap, budget;
    std::cin >> n >> m >> ndev >> cap >> budget;
    auto dur = rd<int64_t>(n), mem = rd<int64_t>(n);
    auto mask = rd<uint64_t>(n);
    auto edges = rd<int64_t>(3 * m);
    auto order = rd<int64_t>(n), lo = rd<int64_t>(n), hi = rd<int64_t>(n);
    auto init = rd<int64_t>(ndev);
    std::vector<int> pool = tsl::gen_build(n, dur.data(), mask.data(), mem.data(), edges.data(), m,
                                           order.data(), lo.data(), hi.data(), ndev, init.data(),
                                           cap);
    GenView g = gen_view(pool.data());
    Sim sim(g, pool[G_MAXDI]);
    sim.P_FIRST = first;
    sim.P_TASKS = ntasks;
    sim.P_PAUSE = pause;
    sim.P_TASKN = taskn;
    sim.hist.assign(n + 2, 0);
    if (getenv("SP_CK")) sim.CK = atoll(getenv("SP_CK"));
    sim.debug = getenv("SP_DEBUG") != nullptr;
    St a = sim.blank();
    int st;
    long long nodes = 0;
    std::vector<int> wit;
    if (!sim.root(a)) {
      st = RX_UNSAT;
    } else if (n == 0) {
      st = RX_SAT;
    } else {
      a.depth = 0;
      a.v = a.lo[g.order(0)];
      long long sn = 0;
      st = sim.run_master(a, 0, n + 1, budget, 0, first, nullptr, nullptr, nullptr, &sn, true);
      sim.par_model += sn;
      nodes = sn;
      if (st == SP_PAUSED) {
        int ds = ds0;
        if (ds <= 0) {  // the shallowest depth at which the sample branched
          ds = n - 1;
          for (int d = 1; d < n; ++d)
            if (sim.hist[d] >= 2) {
              ds = d;
              break;
            }
        }
        if (sim.debug) {
          std::fprintf(stderr, "ds %d depth_after_sample %d hist:", ds, a.depth);
          for (int d = 0; d < n; ++d) if (sim.hist[d]) std::fprintf(stderr, " %d:%lld", d, sim.hist[d]);
          std::fprintf(stderr, "\n");
        }
        st = sim.run(a, 0, ds, budget, sn, &nodes, &wit, 0);
      } else if (st == RX_SAT) {
        wit = a.s;
      }
      if (st == SP_EXHAUSTED) st = RX_UNSAT;
      if (st == RX_TIMEOUT) nodes = budget + 1;
    }
    std::printf("%d %lld %lld %lld %lld %lld %lld", st, nodes, sim.rounds, sim.tasks, sim.replays,
                sim.subsolves, sim.par_model);
    if (st == RX_SAT)
      for (int i = 0; i < n; ++i) std::printf(" %d", wit[i]);
    std::printf("\n");
    std::fflush(stdout);
  }
  return 0;
}
