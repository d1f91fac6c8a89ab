// Micro-benchmark: cp.async.bulk global->shared streaming bandwidth per SM
// (one CTA per SM, one producer thread, S-stage ring, consumers only wait).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bench_bulk tools/bench_bulk.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void k_stream(const uint8_t* src, uint64_t bytes_per_cta, int stage_bytes, int stages, int copies) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (tid != 0) return;
  const uint8_t* base = src + (uint64_t)blockIdx.x * bytes_per_cta;
  const int T = (int)(bytes_per_cta / stage_bytes);
  const int cb = stage_bytes / copies;
  auto load = [&](int t) {
    const int st = t % stages;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(stage_bytes));
    for (int k = 0; k < copies; ++k)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + st * stage_bytes + k * cb)),
                   "l"(base + (uint64_t)t * stage_bytes + k * cb), "r"(cb), "r"(sa(&full[st]))
                   : "memory");
  };
  for (int t = 0; t < stages && t < T; ++t) load(t);
  for (int t = 0; t < T; ++t) {
    const int st = t % stages;
    const uint32_t par = (t / stages) & 1;
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
                     sa(&full[st])),
                 "r"(par)
                 : "memory");
    if (t + stages < T) load(t + stages);
  }
}

__global__ void k_stream_wrap(const uint8_t* src, uint64_t bytes_per_cta, uint64_t window, int stage_bytes, int stages,
                              int copies) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[16];
  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int i = 0; i < stages; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  if (tid != 0) return;
  const int T = (int)(bytes_per_cta / stage_bytes);
  const int cb = stage_bytes / copies;
  const uint64_t nwin = window / stage_bytes;
  auto load = [&](int t) {
    const int st = t % stages;
    const uint64_t off = ((uint64_t)(t + blockIdx.x * 7) % nwin) * stage_bytes;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[st])), "r"(stage_bytes));
    for (int k = 0; k < copies; ++k)
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(sm + st * stage_bytes + k * cb)),
                   "l"(src + off + k * cb), "r"(cb), "r"(sa(&full[st]))
                   : "memory");
  };
  for (int t = 0; t < stages && t < T; ++t) load(t);
  for (int t = 0; t < T; ++t) {
    const int st = t % stages;
    const uint32_t par = (t / stages) & 1;
    asm volatile("{\n.reg .pred p;\nW%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W%=;\n}" ::"r"(
                     sa(&full[st])),
                 "r"(par)
                 : "memory");
    if (t + stages < T) load(t + stages);
  }
}

int main() {
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const uint64_t per = 8ull << 20;  // 8 MB per CTA
  uint8_t* buf;
  cudaMalloc(&buf, per * sms);
  cudaMemset(buf, 1, per * sms);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaFuncSetAttribute(k_stream_wrap, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  int cfg[][3] = {{16384, 4, 1}, {45056, 4, 2}, {45056, 4, 1}, {32768, 6, 1}, {16384, 12, 1}, {8192, 24, 1},
                  {4096, 16, 1}, {65536, 3, 1}, {45056, 4, 4}, {16384, 12, 4},
                  {24576, 4, 1}, {24576, 7, 1}};  // the fused count's x-plane stages
  for (auto& c : cfg) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_stream<<<sms, 32, c[0] * c[1]>>>(buf, per, c[0], c[1], c[2]);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("stage %6d B x %2d stages, %d copies: %.1f GB/s total (%.1f GB/s per SM) err=%s\n", c[0], c[1], c[2],
                      per * sms / ms / 1e6, per / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  // L2-resident: every CTA streams the same window (wraps), 8 MB per CTA of traffic
  for (uint64_t win : {48ull << 20, 33ull << 20, 16ull << 20})
  for (auto& c : cfg) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      k_stream_wrap<<<sms, 32, c[0] * c[1]>>>(buf, per, win, c[0], c[1], c[2]);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep) printf("L2 win %3llu MB %6d B x %2d stages, %d copies: %.1f GB/s total (%.1f per SM)\n",
                      (unsigned long long)(win >> 20), c[0], c[1], c[2],
                      per * sms / ms / 1e6, per / ms / 1e6);
    }
  }
  return 0;
}
