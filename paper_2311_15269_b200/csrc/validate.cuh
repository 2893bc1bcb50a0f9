// validate.cuh — schedule validation on the device:
// the checks of the reference's validate_schedule (schedule.py:77-168) for
// schedules with N up to 10^4+ micro-batches (e.g. extension.extend output):
//   * per device, events (start, stage, mb) sorted lexicographically: a
//     bitonic sort of keys (start, input position) over a padded segment per
//     device — input positions enumerate (stage ascending, mb ascending), so
//     the tie order is the reference's tuple order;
//   * overlap between sorted neighbours, running memory at the end of every
//     equal-start group (block-wide scan per device), dependency and
//     negative-start checks, one thread per item.
// The host formats the reference's Violation list from the flags.
#pragma once
#include <stdint.h>

// key = (start + 2^31) << 32 | position; padding = ~0
__global__ void k_val_keys(const int *__restrict__ starts, const int *__restrict__ dev_stage_ptr,
                           const int *__restrict__ dev_stages, int D, int N, long long P,
                           unsigned long long *__restrict__ keys) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (long long)D * P) return;
  const int d = (int)(gid / P);
  const long long i = gid % P;
  const long long E = (long long)(dev_stage_ptr[d + 1] - dev_stage_ptr[d]) * N;
  if (i >= E) {
    keys[gid] = ~0ull;
    return;
  }
  const int st = dev_stages[dev_stage_ptr[d] + (int)(i / N)];
  const int n = (int)(i % N);
  const int t = starts[(long long)st * N + n];
  keys[gid] = ((unsigned long long)((unsigned)t ^ 0x80000000u) << 32) | (unsigned long long)i;
}

// one compare-exchange step (k, j) of an ascending bitonic sort of every
// length-P segment
__global__ void k_val_bitonic(unsigned long long *__restrict__ keys, long long total, long long P,
                              long long k, long long j) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= total) return;
  const long long i = gid % P, base = gid - i;
  const long long l = i ^ j;
  if (l <= i) return;
  const unsigned long long a = keys[base + i], b = keys[base + l];
  const bool up = (i & k) == 0;
  if ((a > b) == up) {
    keys[base + i] = b;
    keys[base + l] = a;
  }
}

// per device (one block): overlap flags between sorted neighbours and the
// running memory at the end of every equal-start group
__global__ void k_val_scan(const unsigned long long *__restrict__ keys,
                           const int *__restrict__ dev_stage_ptr,
                           const int *__restrict__ dev_stages, const int *__restrict__ dur,
                           const int *__restrict__ mem, int N, long long P,
                           const long long *__restrict__ init_mem, long long cap,
                           unsigned char *__restrict__ ovf, unsigned char *__restrict__ memf,
                           long long *__restrict__ runs, unsigned long long *__restrict__ count) {
  const int d = blockIdx.x;
  const long long E = (long long)(dev_stage_ptr[d + 1] - dev_stage_ptr[d]) * N;
  const unsigned long long *ks = keys + (long long)d * P;
  __shared__ long long warp_sums[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = init_mem[d];
  __syncthreads();
  unsigned long long local = 0;
  for (long long c0 = 0; c0 < E; c0 += blockDim.x) {
    const long long p = c0 + threadIdx.x;
    long long delta = 0;
    int t = 0, st = 0;
    bool act = p < E;
    if (act) {
      const unsigned long long key = ks[p];
      t = (int)((unsigned)(key >> 32) ^ 0x80000000u);
      st = dev_stages[dev_stage_ptr[d] + (int)((key & 0xffffffffull) / N)];
      delta = mem[st];
    }
    // inclusive block scan of delta
    long long v = delta;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 1; o < 32; o <<= 1) {
      const long long u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane == 31) warp_sums[wid] = v;
    __syncthreads();
    if (wid == 0) {
      long long w = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
      for (int o = 1; o < 32; o <<= 1) {
        const long long u = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += u;
      }
      warp_sums[lane] = w;
    }
    __syncthreads();
    const long long run = carry + v + (wid > 0 ? warp_sums[wid - 1] : 0);
    if (act) {
      bool ov = false, group_end = true;
      if (p + 1 < E) {
        const unsigned long long nk = ks[p + 1];
        const int tn = (int)((unsigned)(nk >> 32) ^ 0x80000000u);
        ov = (long long)t + dur[st] > tn;
        group_end = tn != t;
      }
      const bool mv = group_end && run > cap;
      ovf[(long long)d * P + p] = ov;
      memf[(long long)d * P + p] = mv;
      runs[(long long)d * P + p] = run;
      local += ov + mv;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = run;
    __syncthreads();
  }
  if (local) atomicAdd(count, local);
}

// dependency (i -> j, every mb) and negative-start checks
__global__ void k_val_items(const int *__restrict__ starts, const int *__restrict__ dur,
                            const int *__restrict__ deps, int n_deps, int K, int N,
                            unsigned char *__restrict__ depf, unsigned char *__restrict__ negf,
                            unsigned long long *__restrict__ count) {
  const long long gid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long local = 0;
  if (gid < (long long)n_deps * N) {
    const int q = (int)(gid / N), n = (int)(gid % N);
    const int a = deps[2 * q], b = deps[2 * q + 1];
    const bool bad = (long long)starts[(long long)a * N + n] + dur[a] > starts[(long long)b * N + n];
    depf[gid] = bad;
    local += bad;
  }
  if (gid < (long long)K * N) {
    const bool bad = starts[gid] < 0;
    negf[gid] = bad;
    local += bad;
  }
  if (local) atomicAdd(count, local);
}
