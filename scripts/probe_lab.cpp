// probe_lab.cpp — host-side analysis of repetend probes (development tool,
// not part of the product).  Compiles the device routines (rx_dfs.cuh,
// dj_solve.cuh) for the host and, for a window of candidate ranks at one
// period, reports how each probe is settled: root refutation, RX-DFS within a
// small budget, disjunctive refutation, or the deep RX-DFS.
//
// stdin: K D ndep dur[K] mem[K] mask[K] deps[2*ndep]  n_r r0 count P cap
//        small_budget dj_budget rx_budget
// stdout: one line per probe that is not settled by the small budget:
//        widx dj_status dj_nodes dj_us rx_status rx_nodes rx_us
//        and a summary line "#" counts.
#include <chrono>
#include <cstdio>
#include <iostream>
#include <vector>

#include "../paper_2311_15269_b200/csrc/host_build.hpp"
#include "../paper_2311_15269_b200/csrc/dj_solve.cuh"

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

static double now_us() {
  return std::chrono::duration<double, std::micro>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int main() {
  tsl::Placement pl;
  int ndep;
  std::cin >> pl.K >> pl.D >> ndep;
  pl.dur = rd<int>(pl.K);
  pl.mem = rd<int>(pl.K);
  pl.mask = rd<uint64_t>(pl.K);
  auto deps = rd<int>(2 * ndep);
  for (int i = 0; i < ndep; ++i) pl.deps.push_back({deps[2 * i], deps[2 * i + 1]});
  std::sort(pl.deps.begin(), pl.deps.end());
  long long n_r, r0, count, P, cap, small_b, dj_b, rx_b;
  std::cin >> n_r >> r0 >> count >> P >> cap >> small_b >> dj_b >> rx_b;
  std::vector<int> pool = tsl::rep_build(pl);
  std::vector<unsigned long long> cnt;
  std::vector<long long> off;
  tsl::rep_counts(pool, (int)n_r, cnt, off);
  const int K = pl.K;
  long long n_gate = 0, n_root = 0, n_small_sat = 0, n_small_other = 0, n_def = 0;
  std::vector<std::string> lines(count);
#pragma omp parallel reduction(+ : n_gate, n_root, n_small_sat, n_small_other, n_def)
  {
    std::vector<int> ws(rx_ws_words(K, pool[R_MAXDI]) + 8), coef(std::max(ndep, 1)), init(pl.D);
    RxWs w = rx_ws_carve(ws.data(), K, pool[R_MAXDI]);
    std::vector<int> dws(dj_ws_words(K, pl.D, pool[R_NPAIR], pool[R_MAXDI]) + 8);
    DjWs dw = dj_ws_carve(dws.data(), K, pl.D, pool[R_NPAIR], pool[R_MAXDI]);
    std::vector<int> a(K);
#pragma omp for schedule(dynamic, 256)
    for (long long i = 0; i < count; ++i) {
      int *ap = a.data();
      if (!rep_unrank(pool.data(), cnt.data(), off.data(), (int)n_r, (unsigned long long)(r0 + i),
                      ap))
        continue;
      const RepView v = rep_view(pool.data(), (int)P, cap < 0 ? -1 : (int)cap, coef.data(),
                                 init.data());
      rep_prepare(pool.data(), ap, (int)P, coef.data(), init.data(), w.lo, w.hi);
      bool gate = true;
      if (cap >= 0)
        for (int d = 0; d < pl.D; ++d) gate &= init[d] <= cap;
      if (!gate) continue;
      ++n_gate;
      long long nodes = 0;
      int st = rx_decide(v, w, small_b, 0ull, &nodes);
      if (st == RX_UNSAT && nodes == 0) {
        ++n_root;
        continue;
      }
      if (st != RX_TIMEOUT) {
        st == RX_SAT ? ++n_small_sat : ++n_small_other;
        if (st == RX_SAT) {
          char buf[64];
          std::snprintf(buf, sizeof buf, "S %lld %lld", i, nodes);
          lines[i] = buf;
        }
        continue;
      }
      ++n_def;
      rep_prepare(pool.data(), ap, (int)P, coef.data(), init.data(), dw.lo, dw.hi);
      long long dn = 0;
      double t0 = now_us();
      const int dj = dj_decide(v, pool.data(), dw, dj_b, &dn);
      double t1 = now_us();
      int rst = -1;
      long long rn = 0;
      double t2 = t1, t3 = t1;
      if (dj != DJ_UNSAT || rx_b < 0) {
        rep_prepare(pool.data(), ap, (int)P, coef.data(), init.data(), w.lo, w.hi);
        t2 = now_us();
        rst = rx_decide(v, w, rx_b < 0 ? -rx_b : rx_b, 0ull, &rn);
        t3 = now_us();
      }
      char buf[256];
      std::snprintf(buf, sizeof buf, "%lld %d %lld %.1f %d %lld %.1f", i, dj, dn, t1 - t0, rst, rn,
                    t3 - t2);
      lines[i] = buf;
    }
  }
  for (auto &l : lines)
    if (!l.empty()) std::printf("%s\n", l.c_str());
  std::printf("# gated %lld root %lld small_sat %lld small_other %lld deferred %lld\n", n_gate,
              n_root, n_small_sat, n_small_other, n_def);
  return 0;
}
