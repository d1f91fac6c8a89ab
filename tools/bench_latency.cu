// Micro-benchmark: dependent-chain latency (cycles) of one Philox4x32-10 block
// and of a 64-bit multiply-add, single thread, keys from the kernel parameter
// bank vs shared memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2305_00645_b200/csrc -o tools/bench_latency tools/bench_latency.cu
#include <cstdio>
#include <cstdint>
#include "gt_prg.cuh"
using namespace gt;

__global__ void k_lat(Keys K, int n, uint64_t* out, int mode) {
  __shared__ Keys ks;
  if (threadIdx.x == 0) ks = K;
  __syncthreads();
  if (threadIdx.x != 0) return;
  const Keys& KK = mode ? ks : K;
  uint64_t lane = 1;
  // warm-up
  for (int i = 0; i < 4; ++i) lane = philox(KK.pair[1], 7, 3, lane).a;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) lane = philox(KK.pair[1], 7, 3, lane).a;
  long long t1 = clock64();
  uint64_t m = lane;
  for (int i = 0; i < n; ++i) m = m * 0x9E3779B97F4A7C15ull + lane;
  long long t2 = clock64();
  out[0] = (t1 - t0);
  out[1] = (t2 - t1);
  out[2] = lane + m;
}

int main() {
  Keys K;
  K.dealer = expand_key(1, 2);
  for (int i = 0; i < 3; ++i) K.pair[i] = expand_key(3 + i, 7 + i);
  uint64_t* d;
  cudaMalloc(&d, 64);
  uint64_t h[3];
  for (int mode = 0; mode < 2; ++mode) {
    k_lat<<<1, 32>>>(K, 1000, d, mode);
    cudaMemcpy(h, d, 24, cudaMemcpyDeviceToHost);
    printf("keys %s: philox block %.1f cycles (dependent), u64 mad %.1f cycles\n", mode ? "smem" : "param",
           h[0] / 1000.0, h[1] / 1000.0);
  }
  return 0;
}
