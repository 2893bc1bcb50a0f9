// Test-only host build of the device DFS routine (rx_dfs.cuh / models.cuh
// compiled by g++), so its logic can be checked against the oracle on a
// machine without a GPU.  Not part of the product: the product library runs
// the same routine only on the device.
//
// stdin protocol (whitespace separated integers):
//   "G" n m ndev cap budget  dur[n] mem[n] devmask[n] edges[3m] order[n] lo[n] hi[n] init[ndev]
//   "R" K D ndep  dur[K] mem[K] devmask[K] deps[2*ndep]  nq  { P cap budget a[K] } * nq
// stdout: one line per problem: status nodes [starts...]
#include <cstdio>
#include <iostream>
#include <vector>

#include "../../paper_2311_15269_b200/csrc/host_build.hpp"
#include "../../paper_2311_15269_b200/csrc/dj_solve.cuh"

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

static void emit(int st, long long nodes, const int *s, int n) {
  std::printf("%d %lld", st, nodes);
  if (st == RX_SAT)
    for (int i = 0; i < n; ++i) std::printf(" %d", s[i]);
  std::printf("\n");
}

int main() {
  std::string tag;
  while (std::cin >> tag) {
    if (tag == "G") {
      int n, m, ndev;
      long long cap, budget;
      std::cin >> n >> m >> ndev >> cap >> budget;
      auto dur = rd<int64_t>(n), mem = rd<int64_t>(n);
      auto mask = rd<uint64_t>(n);
      auto edges = rd<int64_t>(3 * m);
      auto order = rd<int64_t>(n), lo = rd<int64_t>(n), hi = rd<int64_t>(n);
      auto init = rd<int64_t>(ndev);
      std::vector<int> pool = tsl::gen_build(n, dur.data(), mask.data(), mem.data(), edges.data(),
                                             m, order.data(), lo.data(), hi.data(), ndev,
                                             init.data(), cap);
      GenView g = gen_view(pool.data());
      std::vector<int> ws(rx_ws_words(n, pool[G_MAXDI]) + 8);
      RxWs w = rx_ws_carve(ws.data(), n, pool[G_MAXDI]);
      for (int k = 0; k < n; ++k) {
        w.lo[k] = g.lo_[k];
        w.hi[k] = g.hi_[k];
      }
      long long nodes = 0;
      int st = rx_decide(g, w, budget, 0ull, &nodes);
      emit(st, nodes, w.s, n);
    } else if (tag == "R" || tag == "J") {
      // "J": same input as "R"; runs the disjunctive refutation (dj_decide)
      // and prints "verdict dj_nodes"
      const bool dj = tag == "J";
      tsl::Placement pl;
      int ndep;
      std::cin >> pl.K >> pl.D >> ndep;
      pl.dur = rd<int>(pl.K);
      pl.mem = rd<int>(pl.K);
      pl.mask = rd<uint64_t>(pl.K);
      auto deps = rd<int>(2 * ndep);
      for (int i = 0; i < ndep; ++i) pl.deps.push_back({deps[2 * i], deps[2 * i + 1]});
      std::sort(pl.deps.begin(), pl.deps.end());
      std::vector<int> pool = tsl::rep_build(pl);
      const int K = pl.K;
      std::vector<int> ws(rx_ws_words(K, pool[R_MAXDI]) + 8), coef(std::max(ndep, 1)),
          init(pl.D);
      RxWs w = rx_ws_carve(ws.data(), K, pool[R_MAXDI]);
      std::vector<int> dws(dj_ws_words(K, pl.D, pool[R_NPAIR], pool[R_MAXDI]) + 8);
      DjWs dw = dj_ws_carve(dws.data(), K, pl.D, pool[R_NPAIR], pool[R_MAXDI]);
      int nq;
      std::cin >> nq;
      for (int q = 0; q < nq; ++q) {
        int P;
        long long cap, budget;
        std::cin >> P >> cap >> budget;
        auto a = rd<int>(K);
        const int *ap = a.data();
        const RepView v =
            rep_view(pool.data(), P, cap < 0 ? -1 : (int)cap, coef.data(), init.data());
        long long nodes = 0;
        if (dj) {
          rep_prepare(pool.data(), ap, P, coef.data(), init.data(), dw.lo, dw.hi);
          const int st = dj_decide(v, pool.data(), dw, budget, &nodes);
          std::printf("%d %lld\n", st, nodes);
          continue;
        }
        rep_prepare(pool.data(), ap, P, coef.data(), init.data(), w.lo, w.hi);
        int st = rx_decide(v, w, budget, 0ull, &nodes);
        emit(st, nodes, w.s, K);
      }
    } else {
      std::fprintf(stderr, "bad tag %s\n", tag.c_str());
      return 2;
    }
  }
  return 0;
}
