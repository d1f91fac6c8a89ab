// Probe of tcgen05.mma.cta_group::2 kind::i8 operand distribution (dev tool).
// A CTA pair (cluster 2x1x1) runs one UMMA M=256 N=32 K=32 issued by the
// leader.  Each CTA holds A rows with A[r][0] = (rank + 1), other bytes 0,
// and 32 B rows with B[n][0] = 64 * rank + n.  D[r][n] = A[r][0] * B'[n][0]
// tells which CTA's B row feeds accumulator column n of each CTA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tools/umma2_probe tools/umma2_probe.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) k_probe(uint32_t* out, int N) {
  __shared__ __align__(1024) uint8_t A[2][16][128];  // [kchunk][row group][8 rows x 16 B]
  __shared__ __align__(1024) uint8_t B[2][4][128];   // 32 rows
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t slot;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 2 * 16 * 128; i += 128) {
    const int kc = i / 2048, rem = i % 2048, k = rem % 16;
    (&A[0][0][0])[i] = (kc == 0 && k == 0) ? (uint8_t)(rank + 1) : 0;
  }
  for (int i = tid; i < 2 * 4 * 128; i += 128) {
    const int kc = i / 512, rem = i % 512, rg = rem / 128, r = (rem % 128) / 16, k = rem % 16;
    (&B[0][0][0])[i] = (kc == 0 && k == 0) ? (uint8_t)(64 * rank + rg * 8 + r) : 0;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(64)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = slot;
  if (rank == 0 && tid == 0) {
    const uint32_t idesc = (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((256u >> 4) << 24);
    const uint64_t ad = desc(smem_u32(&A[0][0][0]), 2048, 128), bd = desc(smem_u32(&B[0][0][0]), 512, 128);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(ad), "l"(bd), "r"(idesc), "r"(0)
        : "memory");
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(&bar)),
        "h"((uint16_t)3)
        : "memory");
  }
  asm volatile(
      "{\n\t.reg .pred p;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
          smem_u32(&bar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t d[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]),
        "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]),
        "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]),
        "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
      : "r"(tmem + ((uint32_t)(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int j = 0; j < 32; ++j) out[(rank * 128 + tid) * 32 + j] = d[j];
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64) : "memory");
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 2 * 128 * 32 * 4);
  cudaMemset(d, 0xff, 2 * 128 * 32 * 4);
  for (int N : {16, 32}) {
    k_probe<<<2, 128>>>(d, N);
    cudaError_t e = cudaDeviceSynchronize();
    static uint32_t h[2 * 128 * 32];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    printf("N=%d err=%s\n", N, cudaGetErrorString(e));
    for (int c = 0; c < 2; ++c)
      for (int r : {0, 1, 64, 127}) {
        printf("cta %d row %3d:", c, r);
        for (int j = 0; j < N; ++j) printf(" %u", h[(c * 128 + r) * 32 + j]);
        printf("\n");
      }
  }
  return 0;
}
