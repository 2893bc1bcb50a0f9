// host_build.hpp — host-side lowering for the device views (models.cuh).
//
// gen_build:  one decide problem -> GenView pool (kernel_c.pyx:54-128 CSRs).
// rep_build:  a placement -> RepView structure pool (repetend.py:108-150
//             edge rows: sorted dependency rows, then device-window rows
//             device-major, x-major / y-minor over device_stages(d);
//             branch order sorted by (-|devices|, stage)).
// rep_counts: frontier count tables for unranking repetend.py:65-90.
#pragma once
#include <stdint.h>

#include <algorithm>
#include <stdexcept>
#include <cstdlib>
#include <string>
#include <utility>
#include <vector>

#include "../../include/tessel_b200.h"
#include "models.cuh"

namespace tsl {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

// All problem values must satisfy |v| < 2^28 so every int32 intermediate of
// rx_decide (sums of durations, bound + lag, sentinels at -2^30) is exact.
constexpr long long VMAX = 1LL << 28;

inline int ck(long long v, const char *what) {
  if (v >= VMAX || v <= -VMAX)
    throw Error(TSL_EINVAL, std::string(what) + " value " + std::to_string(v) +
                                " outside the kernel's int32 range (|v| < 2^28)");
  return (int)v;
}

inline int popcount64(uint64_t x) { return __builtin_popcountll(x); }

// 1 per node whose CSR list names the same target more than once
inline std::vector<int> dup_flags(const std::vector<int> &ptr, const std::vector<int> &dst, int n) {
  std::vector<int> out(n > 0 ? n : 1, 0);
  for (int a = 0; a < n; ++a) {
    std::vector<int> t(dst.begin() + ptr[a], dst.begin() + ptr[a + 1]);
    std::sort(t.begin(), t.end());
    out[a] = std::adjacent_find(t.begin(), t.end()) != t.end();
  }
  return out;
}

// per in-list entry p of node a: the position (within a's out-list) of the
// out-entry naming the same node, or -1 — the warp propagation's one-chunk
// path (wrx_dfs.cuh) deduplicates a node on both lists with it
inline std::vector<int> in_twins(const std::vector<int> &out_ptr, const std::vector<int> &out_dst,
                                 const std::vector<int> &in_ptr, const std::vector<int> &in_src,
                                 int n) {
  std::vector<int> tw(in_src.empty() ? 1 : in_src.size(), -1);
  for (int a = 0; a < n; ++a)
    for (int p = in_ptr[a]; p < in_ptr[a + 1]; ++p)
      for (int q = out_ptr[a]; q < out_ptr[a + 1]; ++q)
        if (out_dst[q] == in_src[p]) {
          tw[p] = q - out_ptr[a];
          break;
        }
  return tw;
}

// ------------------------------------------------------------------ GenView
inline std::vector<int> gen_build(int n, const int64_t *dur, const uint64_t *devmask,
                                  const int64_t *mem, const int64_t *edges, int m,
                                  const int64_t *order, const int64_t *lo, const int64_t *hi,
                                  int ndev, const int64_t *init, int64_t cap) {
  if (n < 0 || n > TSL_MAX_ITEMS)
    throw Error(TSL_ERANGE, "n=" + std::to_string(n) + " outside [0, " +
                                std::to_string(TSL_MAX_ITEMS) + "]");
  if (ndev < 0 || ndev > TSL_MAX_DEVICES)
    throw Error(TSL_ERANGE, "ndev=" + std::to_string(ndev) + " outside [0, 64]");
  if (m < 0) throw Error(TSL_EINVAL, "negative edge count");
  long long sdur = 0, smem = 0, sinit = 0;
  for (int i = 0; i < n; ++i) {
    ck(dur[i], "dur");
    ck(mem[i], "mem");
    ck(lo[i], "lo");
    ck(hi[i], "hi");
    sdur += dur[i] > 0 ? dur[i] : -dur[i];
    smem += mem[i] > 0 ? mem[i] : -mem[i];
    if (order[i] < 0 || order[i] >= n) throw Error(TSL_EINVAL, "order entry out of range");
  }
  for (int d = 0; d < ndev; ++d) {
    ck(init[d], "init_mem");
    sinit = std::max(sinit, (long long)(init[d] > 0 ? init[d] : -init[d]));
  }
  ck(sdur, "sum(|dur|)");
  ck(smem + sinit, "memory sum");
  int icap = -1;
  if (cap >= 0) icap = (int)std::min<int64_t>(cap, VMAX - 1);
  for (int e = 0; e < m; ++e) {
    if (edges[3 * e] < 0 || edges[3 * e] >= n || edges[3 * e + 1] < 0 || edges[3 * e + 1] >= n)
      throw Error(TSL_EINVAL, "edge endpoint out of range");
    ck(edges[3 * e + 2], "edge lag");
  }
  // CSRs
  std::vector<int> out_ptr(n + 1, 0), in_ptr(n + 1, 0), out_dst(m), out_lag(m), in_src(m),
      in_lag(m);
  for (int e = 0; e < m; ++e) {
    out_ptr[edges[3 * e] + 1]++;
    in_ptr[edges[3 * e + 1] + 1]++;
  }
  for (int i = 0; i < n; ++i) {
    out_ptr[i + 1] += out_ptr[i];
    in_ptr[i + 1] += in_ptr[i];
  }
  {
    std::vector<int> fo(n, 0), fi(n, 0);
    for (int e = 0; e < m; ++e) {
      const int a = (int)edges[3 * e], b = (int)edges[3 * e + 1], lag = (int)edges[3 * e + 2];
      out_dst[out_ptr[a] + fo[a]] = b;
      out_lag[out_ptr[a] + fo[a]++] = lag;
      in_src[in_ptr[b] + fi[b]] = a;
      in_lag[in_ptr[b] + fi[b]++] = lag;
    }
  }
  std::vector<int> conf_ptr(n + 1, 0), conf_dst;
  for (int i = 0; i < n; ++i) {
    for (int j = 0; j < n; ++j)
      if (i != j && (devmask[i] & devmask[j])) conf_dst.push_back(j);
    conf_ptr[i + 1] = (int)conf_dst.size();
  }
  std::vector<int> dev_ptr(ndev + 1, 0), dev_items, devof_ptr(n + 1, 0), devof;
  int maxdi = 0;
  for (int d = 0; d < ndev; ++d) {
    for (int i = 0; i < n; ++i)
      if ((devmask[i] >> d) & 1) dev_items.push_back(i);
    dev_ptr[d + 1] = (int)dev_items.size();
    maxdi = std::max(maxdi, dev_ptr[d + 1] - dev_ptr[d]);
  }
  for (int i = 0; i < n; ++i) {
    for (int d = 0; d < ndev; ++d)
      if ((devmask[i] >> d) & 1) devof.push_back(d);
    devof_ptr[i + 1] = (int)devof.size();
  }
  std::vector<int> pool(G_HDR, 0);
  pool[G_N] = n;
  pool[G_NDEV] = ndev;
  pool[G_CAP] = icap;
  pool[G_M] = m;
  pool[G_NCONF] = (int)conf_dst.size();
  pool[G_NMEMB] = (int)dev_items.size();
  pool[G_MAXDI] = maxdi;
  auto put = [&](const std::vector<int> &v) { pool.insert(pool.end(), v.begin(), v.end()); };
  auto put64 = [&](const int64_t *p, int k) {
    for (int i = 0; i < k; ++i) pool.push_back((int)p[i]);
  };
  put64(dur, n);
  put64(mem, n);
  put64(order, n);
  put64(lo, n);
  put64(hi, n);
  put64(init, ndev);
  put(out_ptr);
  put(out_dst);
  put(out_lag);
  put(in_ptr);
  put(in_src);
  put(in_lag);
  put(conf_ptr);
  put(conf_dst);
  put(dev_ptr);
  put(dev_items);
  put(devof_ptr);
  put(devof);
  put(dup_flags(out_ptr, out_dst, n));
  put(dup_flags(in_ptr, in_src, n));
  put(in_twins(out_ptr, out_dst, in_ptr, in_src, n));
  pool[G_WORDS] = (int)pool.size();
  return pool;
}

// ------------------------------------------------------------------ RepView
struct Placement {
  int K = 0, D = 0;
  std::vector<int> dur, mem;
  std::vector<uint64_t> mask;
  std::vector<std::pair<int, int>> deps;  // sorted ascending
};

inline std::vector<int> rep_build(const Placement &pl) {
  const int K = pl.K, D = pl.D;
  if (K < 1 || K > TSL_MAX_STAGES) throw Error(TSL_ERANGE, "stage count outside [1, 64]");
  if (D < 1 || D > TSL_MAX_DEVICES) throw Error(TSL_ERANGE, "device count outside [1, 64]");
  std::vector<int> order(K);
  for (int i = 0; i < K; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) {
    return popcount64(pl.mask[a]) > popcount64(pl.mask[b]);
  });
  std::vector<std::pair<int, int>> rows = pl.deps;
  const int ndep = (int)rows.size();
  std::vector<std::vector<int>> dstages(D);
  for (int d = 0; d < D; ++d)
    for (int st = 0; st < K; ++st)
      if ((pl.mask[st] >> d) & 1) dstages[d].push_back(st);
  for (int d = 0; d < D; ++d)
    for (int x : dstages[d])
      for (int y : dstages[d])
        if (x != y) rows.push_back({x, y});
  const int m = (int)rows.size();
  std::vector<int> out_ptr(K + 1, 0), in_ptr(K + 1, 0), out_dst(m), out_row(m), in_src(m),
      in_row(m), rbase(m), rsrc(m), rdst(m);
  for (int r = 0; r < m; ++r) {
    out_ptr[rows[r].first + 1]++;
    in_ptr[rows[r].second + 1]++;
    rsrc[r] = rows[r].first;
    rdst[r] = rows[r].second;
    rbase[r] = pl.dur[rows[r].first];
  }
  for (int i = 0; i < K; ++i) {
    out_ptr[i + 1] += out_ptr[i];
    in_ptr[i + 1] += in_ptr[i];
  }
  {
    std::vector<int> fo(K, 0), fi(K, 0);
    for (int r = 0; r < m; ++r) {
      const int a = rows[r].first, b = rows[r].second;
      out_dst[out_ptr[a] + fo[a]] = b;
      out_row[out_ptr[a] + fo[a]++] = r;
      in_src[in_ptr[b] + fi[b]] = a;
      in_row[in_ptr[b] + fi[b]++] = r;
    }
  }
  std::vector<int> out_dep_end(K), in_dep_end(K), in_srcdur(m);
  for (int a = 0; a < K; ++a) {
    int p = out_ptr[a];
    while (p < out_ptr[a + 1] && out_row[p] < ndep) ++p;
    out_dep_end[a] = p;
    p = in_ptr[a];
    while (p < in_ptr[a + 1] && in_row[p] < ndep) ++p;
    in_dep_end[a] = p;
  }
  for (int p = 0; p < m; ++p) in_srcdur[p] = pl.dur[in_src[p]];
  // disjunctive pairs {x < y} with intersecting masks
  std::vector<int> pairx, pairy, pdev_ptr(1, 0), pdev, devnpair(D, 0);
  std::vector<std::vector<int>> pid(K, std::vector<int>(K, -1));
  for (int x = 0; x < K; ++x)
    for (int y = x + 1; y < K; ++y)
      if (pl.mask[x] & pl.mask[y]) {
        pid[x][y] = pid[y][x] = (int)pairx.size();
        pairx.push_back(x);
        pairy.push_back(y);
        for (int d = 0; d < D; ++d)
          if (((pl.mask[x] & pl.mask[y]) >> d) & 1) {
            pdev.push_back(d);
            devnpair[d]++;
          }
        pdev_ptr.push_back((int)pdev.size());
      }
  std::vector<int> dp_ptr(D + 1, 0), dp;
  for (int d = 0; d < D; ++d) {
    for (size_t q = 0; q < pairx.size(); ++q)
      if (((pl.mask[pairx[q]] & pl.mask[pairy[q]]) >> d) & 1) dp.push_back((int)q);
    dp_ptr[d + 1] = (int)dp.size();
  }
  std::vector<int> conf_ptr(K + 1, 0), conf_dst, conf_pid;
  for (int i = 0; i < K; ++i) {
    for (int j = 0; j < K; ++j)
      if (i != j && (pl.mask[i] & pl.mask[j])) {
        conf_dst.push_back(j);
        conf_pid.push_back(pid[i][j]);
      }
    conf_ptr[i + 1] = (int)conf_dst.size();
  }
  std::vector<int> dev_ptr(D + 1, 0), dev_items, devof_ptr(K + 1, 0), devof;
  int maxdi = 0, lb = 0, total = 0, maxdur = 1;
  for (int d = 0; d < D; ++d) {
    int load = 0;
    for (int st : dstages[d]) {
      dev_items.push_back(st);
      load += pl.dur[st];
    }
    dev_ptr[d + 1] = (int)dev_items.size();
    maxdi = std::max(maxdi, (int)dstages[d].size());
    lb = std::max(lb, load);
  }
  for (int st = 0; st < K; ++st) {
    for (int d = 0; d < D; ++d)
      if ((pl.mask[st] >> d) & 1) devof.push_back(d);
    devof_ptr[st + 1] = (int)devof.size();
    total += pl.dur[st];
    maxdur = std::max(maxdur, pl.dur[st]);
  }
  // enumeration metadata
  std::vector<std::vector<int>> succ(K), pred(K);
  for (auto &e : pl.deps) {
    succ[e.first].push_back(e.second);
    pred[e.second].push_back(e.first);
  }
  for (int st = 0; st < K; ++st) {
    std::sort(succ[st].begin(), succ[st].end());
    std::sort(pred[st].begin(), pred[st].end());
  }
  std::vector<int> ls_ptr(K + 1, 0), ls, hs_ptr(K + 1, 0), hs, fr_ptr(K + 1, 0), fr;
  std::vector<int> last_use(K, -1);  // last stage w that reads u as a bound source
  for (int st = 0; st < K; ++st) {
    for (int j : succ[st])
      if (j < st) {
        ls.push_back(j);
        last_use[j] = std::max(last_use[j], st);
      }
    ls_ptr[st + 1] = (int)ls.size();
    for (int i : pred[st])
      if (i < st) {
        hs.push_back(i);
        last_use[i] = std::max(last_use[i], st);
      }
    hs_ptr[st + 1] = (int)hs.size();
  }
  for (int st = 0; st < K; ++st) {
    for (int u = 0; u <= st; ++u)
      if (last_use[u] > st) fr.push_back(u);
    fr_ptr[st + 1] = (int)fr.size();
  }

  std::vector<int> pool(R_HDR, 0);
  pool[R_K] = K;
  pool[R_D] = D;
  pool[R_NDEP] = ndep;
  pool[R_M] = m;
  pool[R_MAXDUR] = maxdur;
  pool[R_LB] = lb;
  pool[R_TOTAL] = total;
  pool[R_MAXDI] = maxdi;
  pool[R_NPAIR] = (int)pairx.size();
  auto put = [&](int slot, const std::vector<int> &v) {
    pool[slot] = (int)pool.size();
    pool.insert(pool.end(), v.begin(), v.end());
    if (v.empty()) pool.push_back(0);
  };
  put(R_DUR, pl.dur);
  put(R_MEM, pl.mem);
  put(R_ORDER, order);
  put(R_OUTPTR, out_ptr);
  put(R_OUTDST, out_dst);
  put(R_OUTROW, out_row);
  put(R_OUTDEPEND, out_dep_end);
  put(R_INPTR, in_ptr);
  put(R_INSRC, in_src);
  put(R_INROW, in_row);
  put(R_INDEPEND, in_dep_end);
  put(R_INSRCDUR, in_srcdur);
  put(R_RBASE, rbase);
  put(R_RSRC, rsrc);
  put(R_RDST, rdst);
  put(R_CONFPTR, conf_ptr);
  put(R_CONFDST, conf_dst);
  put(R_CONFPID, conf_pid);
  put(R_DEVPTR, dev_ptr);
  put(R_DEVITEMS, dev_items);
  put(R_DEVOFPTR, devof_ptr);
  put(R_DEVOF, devof);
  put(R_PAIRX, pairx);
  put(R_PAIRY, pairy);
  put(R_PDEVPTR, pdev_ptr);
  put(R_PDEV, pdev);
  put(R_DEVNPAIR, devnpair);
  put(R_OUTDUP, dup_flags(out_ptr, out_dst, K));
  put(R_INDUP, dup_flags(in_ptr, in_src, K));
  put(R_LSPTR, ls_ptr);
  put(R_LS, ls);
  put(R_HSPTR, hs_ptr);
  put(R_HS, hs);
  put(R_FRPTR, fr_ptr);
  put(R_FR, fr);
  put(R_DPPTR, dp_ptr);
  put(R_DP, dp);
  {  // chunk item masks for wdj_propagate (u64 as two ints)
    const int nrc = (m + 31) / 32, npc = ((int)pairx.size() + 31) / 32;
    std::vector<int> rowcm(2 * (nrc > 0 ? nrc : 1), 0), paircm(2 * (npc > 0 ? npc : 1), 0);
    auto setc = [&](std::vector<int> &v, int c, int item) {
      if (K > 64) {
        v[2 * c] = v[2 * c + 1] = -1;
      } else {
        v[2 * c + (item >> 5)] |= (int)(1u << (item & 31));
      }
    };
    for (int r = 0; r < m; ++r) {
      setc(rowcm, r / 32, rsrc[r]);
      setc(rowcm, r / 32, rdst[r]);
    }
    for (size_t q = 0; q < pairx.size(); ++q) {
      setc(paircm, (int)q / 32, pairx[q]);
      setc(paircm, (int)q / 32, pairy[q]);
    }
    put(R_ROWCM, rowcm);
    put(R_PAIRCM, paircm);
  }
  put(R_INTWIN, in_twins(out_ptr, out_dst, in_ptr, in_src, K));
  {  // wrr_dfs.cuh tables (u64 masks as two ints, low word first)
    const bool fits = K <= 64 && D <= 64;
    std::vector<int> succm(2 * K, 0), predm(2 * K, 0), confm(2 * K, 0), devm(2 * K, 0),
        devitm(2 * D, 0), multi(K, -1), winb;
    auto setb = [](std::vector<int> &v, int row, int bit) {
      v[2 * row + (bit >> 5)] |= (int)(1u << (bit & 31));
    };
    if (fits) {
      for (auto &e : pl.deps) {
        setb(succm, e.first, e.second);
        setb(predm, e.second, e.first);
      }
      for (int i = 0; i < K; ++i) {
        for (int j = 0; j < K; ++j)
          if (i != j && (pl.mask[i] & pl.mask[j])) setb(confm, i, j);
        for (int d = 0; d < D; ++d)
          if ((pl.mask[i] >> d) & 1) {
            setb(devm, i, d);
            setb(devitm, d, i);
          }
      }
      for (int a = 0; a < K; ++a) {
        if (__builtin_popcountll(pl.mask[a]) < 2) continue;
        // a's window rows: devices of a ascending, partners ascending; the
        // first occurrence of a partner fixes its position
        std::vector<int> pos(K, -1);
        int next = 0;
        for (int d = 0; d < D; ++d)
          if ((pl.mask[a] >> d) & 1)
            for (int y : dstages[d])
              if (y != a && pos[y] < 0) pos[y] = next++;
        multi[a] = (int)(winb.size() / (2 * K));
        std::vector<int> tab(2 * K, 0);
        for (int b = 0; b < K; ++b)
          for (int c = 0; c < K; ++c)
            if (pos[b] >= 0 && pos[c] >= 0 && pos[c] < pos[b]) setb(tab, b, c);
        winb.insert(winb.end(), tab.begin(), tab.end());
      }
    }
    put(R_SUCCM, succm);
    put(R_PREDM, predm);
    put(R_CONFM, confm);
    put(R_DEVM, devm);
    put(R_DEVITM, devitm);
    put(R_MULTI, multi);
    put(R_WINB, winb);
    // bounds pack into 16-bit halves: 0 <= lo, hi <= 2A + max t < 2^15
    const long long a_max = (long long)(K - 1) * (total + maxdur);
    const char *mode = std::getenv("TSL_REP_DFS");  // "wrx": shared-memory warp DFS
    pool[R_WRR] = fits && 2 * a_max + 2LL * maxdur < 32767 &&
                          !(mode && std::string(mode) == "wrx") ? 1 : 0;
    const char *strong = std::getenv("TSL_REP_STRONG");  // "0": exact DFS only
    pool[R_WST] = pool[R_WRR] && maxdi <= 8 && !(strong && std::string(strong) == "0") ? 1 : 0;
  }
  pool[R_WORDS] = (int)pool.size();
  // value-range guard for the int32 device arithmetic: anchors reach
  // 2 (K-1)(P + max t) with P <= total.
  ck(2LL * (K - 1) * (2LL * total + maxdur) + 4LL * total, "repetend anchor");
  return pool;
}

// Frontier count tables for n_r.  off[st] (st = 0..K) indexes cnt; the
// table at position st has 2 * n_r^|F_st| entries.  Returns cnt[off[0] + 0]
// = number of candidates (z = 0 at the start: no zero index yet).
inline void rep_counts(const std::vector<int> &pool, int n_r, std::vector<unsigned long long> &cnt,
                       std::vector<long long> &off) {
  const int K = pool[R_K];
  auto F = [&](int pos, std::vector<int> &out) {  // frontier before assigning `pos`
    out.clear();
    if (pos == 0) return;
    for (int p = at_ptr(pool.data(), R_FRPTR, pos - 1); p < at_ptr(pool.data(), R_FRPTR, pos); ++p)
      out.push_back(pool[pool[R_FR] + p]);
  };
  off.assign(K + 2, 0);
  std::vector<int> f;
  long long total = 0;
  for (int pos = 0; pos <= K; ++pos) {
    F(pos, f);
    long long sz = 2;
    for (size_t k = 0; k < f.size(); ++k) {
      sz *= n_r;
      if (sz > (1LL << 26)) throw Error(TSL_ERANGE, "enumeration frontier too wide for n_r");
    }
    off[pos] = total;
    total += sz;
    if (total > (1LL << 26)) throw Error(TSL_ERANGE, "enumeration tables too large for n_r");
  }
  off[K + 1] = total;
  cnt.assign(total, 0ULL);
  const unsigned long long LIM = 1ULL << 63;
  cnt[off[K] + 0] = 0;
  cnt[off[K] + 1] = 1;
  std::vector<int> fs, fn, vals(K, 0);
  for (int st = K - 1; st >= 0; --st) {
    F(st, fs);
    F(st + 1, fn);
    long long states = (off[st + 1] - off[st]) / 2;
    for (long long s = 0; s < states; ++s) {
      long long q = s;
      for (int u : fs) {
        vals[u] = (int)(q % n_r);
        q /= n_r;
      }
      int lo = 0, hi = n_r - 1;
      for (int p = at_ptr(pool.data(), R_LSPTR, st); p < at_ptr(pool.data(), R_LSPTR, st + 1); ++p)
        lo = std::max(lo, vals[pool[pool[R_LS] + p]]);
      for (int p = at_ptr(pool.data(), R_HSPTR, st); p < at_ptr(pool.data(), R_HSPTR, st + 1); ++p)
        hi = std::min(hi, vals[pool[pool[R_HS] + p]]);
      for (int z = 0; z < 2; ++z) {
        unsigned __int128 acc = 0;
        for (int v = lo; v <= hi; ++v) {
          vals[st] = v;
          long long idx = 0, mult = 1;
          for (int u : fn) {
            idx += (long long)vals[u] * mult;
            mult *= n_r;
          }
          acc += cnt[off[st + 1] + idx * 2 + (z | (v == 0))];
        }
        cnt[off[st] + s * 2 + z] = acc >= LIM ? LIM : (unsigned long long)acc;
      }
    }
  }
}

}  // namespace tsl
