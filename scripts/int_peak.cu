// INT32 lane-throughput microbenchmark: IADD3 and LOP3
// issue rates on this B200, measured with CUDA events.  8 independent
// register ring per thread (8 independent ops per step), full
// occupancy, 148 x 8 blocks of 256 threads.  Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_int(int iters, unsigned *out, unsigned seed) {
  unsigned a0 = threadIdx.x ^ seed, a1 = a0 * 3u, a2 = a0 * 5u, a3 = a0 * 7u;
  unsigned a4 = a0 * 11u, a5 = a0 * 13u, a6 = a0 * 17u, a7 = a0 * 19u;
  const unsigned b = seed | 1u, c = seed * 0x9e3779b9u;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    // a ring: every op reads a register the previous op of the ring wrote
    // one step earlier, so ptxas cannot fold them; 8 independent ops / step
    if (OP == 0) {  // IADD3 (one 3-input add each)
      a0 = a0 + a1 + b; a1 = a1 + a2 + c; a2 = a2 + a3 + b; a3 = a3 + a4 + c;
      a4 = a4 + a5 + b; a5 = a5 + a6 + c; a6 = a6 + a7 + b; a7 = a7 + a0 + c;
    } else {  // LOP3 (one 3-input logic op each)
      a0 = (a0 ^ a1) ^ b; a1 = (a1 ^ a2) ^ c; a2 = (a2 ^ a3) ^ b; a3 = (a3 ^ a4) ^ c;
      a4 = (a4 ^ a5) ^ b; a5 = (a5 ^ a6) ^ c; a6 = (a6 ^ a7) ^ b; a7 = (a7 ^ a0) ^ c;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = a0 ^ a1 ^ a2 ^ a3 ^ a4 ^ a5 ^ a6 ^ a7;
}

template <int OP>
double run(int sms, int clk_khz) {
  const int blocks = sms * 8, threads = 256, iters = 1 << 16;
  unsigned *out;
  cudaMalloc(&out, sizeof(unsigned) * blocks * threads);
  k_int<OP><<<blocks, threads>>>(iters / 16, out, 1u);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_int<OP><<<blocks, threads>>>(iters, out, 7u);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  const double ops = 8.0 * iters * (double)blocks * threads;  // thread-level int ops
  return ops / (ms * 1e-3);
}

int main() {
  int dev = 0, sms = 0, clk = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const double add = run<0>(sms, clk), lop = run<1>(sms, clk);
  // per SM per clock at the device's max clock (the bench samples the live clock)
  const double hz = clk * 1e3;
  printf("{\"sms\": %d, \"max_clock_mhz\": %.0f, \"iadd_ops_per_s\": %.4e, \"lop3_ops_per_s\": %.4e, "
         "\"iadd_lanes_per_sm_clk\": %.1f, \"lop3_lanes_per_sm_clk\": %.1f, "
         "\"warp_inst_issue_peak_per_s\": %.4e}\n",
         sms, hz / 1e6, add, lop, add / sms / hz, lop / sms / hz, sms * 4.0 * hz);
  return 0;
}
