#include <cstdlib>
// Secure batch inference (reference infer_batch, pkg/src/obtree/infer.py:20-35)
// as ONE fused kernel: every query walks all H levels; level t fetches the
// current slot's payload with an oblivious lookup over the 2^t level entries
// and then the query's bit for that feature with a row lookup over its nf
// features; slot = 2 slot + branch + 1.  The encoded tree (3 x (2^H - 1)
// words) sits in shared memory for the whole walk; each query is handled by a
// group of G threads that split the lookup lanes and reduce with warp
// shuffles.  The last level's feature fetch is kept (its slot is returned),
// matching the reference's shape-uniform walk.
#include "gt_common.cuh"
#include "gt_lookup.cuh"

namespace gt {
namespace {

template <int G>
__global__ void __launch_bounds__(256) k_walk(const uint64_t* tree, int depth, const uint64_t* Q, uint64_t n, int nf,
                                              uint64_t base, uint64_t* out, uint64_t* slot_out, Keys K) {
  extern __shared__ uint64_t tab[];  // [3][slots]
  const int slots = (1 << depth) - 1;
  for (int i = threadIdx.x; i < 3 * slots; i += blockDim.x) tab[i] = tree[i];
  __syncthreads();
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t s = gt / G;
  const int t = (int)(gt % G);
  const bool valid = s < n;
  const uint64_t nq = n * (uint64_t)nf;
  A3 slot = a3(0, 0, 0), payload = a3(0, 0, 0);
  for (int lv = 0; lv < depth; ++lv) {
    const int m = 1 << lv, o = m - 1;
    A3 part = a3(0, 0, 0);
    if (valid) {
      const A3 local = add_pub<64>(slot, 0ull - (uint64_t)o);  // infer.py:30
      auto entry = [&](int j) { return a3(tab[o + j], tab[slots + o + j], tab[2 * slots + o + j]); };
      part = lookup_partial<64>(K, op_id(lv, SITE_WALK_OAA), base + s, local, m, t, G, entry);
    }
    payload = group_sum<G, 64>(part);
    A3 part2 = a3(0, 0, 0);
    if (valid) {
      auto entry = [&](int f) { return a3(Q[s * nf + f], Q[nq + s * nf + f], Q[2 * nq + s * nf + f]); };
      part2 = lookup_partial<64>(K, op_id(lv, SITE_WALK_ROW), base + s, payload, nf, t, G, entry);
    }
    const A3 branch = group_sum<G, 64>(part2);
    slot = add_pub<64>(add<64>(mul_pub<64>(slot, 2), branch), 1);  // infer.py:33
  }
  if (valid && t == 0) {
    out[s] = payload.v[0];
    out[n + s] = payload.v[1];
    out[2 * n + s] = payload.v[2];
    if (slot_out) {
      slot_out[s] = slot.v[0];
      slot_out[n + s] = slot.v[1];
      slot_out[2 * n + s] = slot.v[2];
    }
  }
}

template <int G>
int launch_walk(const uint64_t* tree, int depth, const uint64_t* Q, uint64_t n, int nf, uint64_t base, uint64_t* out,
                uint64_t* slot_out, const Keys& K, cudaStream_t s) {
  // 128-thread CTAs: finer residency granularity (96 registers per thread
  // leave room for 5 such CTAs per SM vs 2 of 256), so a grid just above one
  // wave of 256-thread CTAs (C3: 313) does not spill into a second wave
  static const int TPB = getenv("GT_WALK_TPB") ? atoi(getenv("GT_WALK_TPB")) : 128;  // A/B experiments
  const int smem = 3 * ((1 << depth) - 1) * (int)sizeof(uint64_t);
  if (smem > 48 * 1024) GT_CUDA_CHECK(cudaFuncSetAttribute(k_walk<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  const uint64_t threads = n * G;
  k_walk<G><<<(unsigned)((threads + TPB - 1) / TPB), TPB, smem, s>>>(tree, depth, Q, n, nf, base, out, slot_out, K);
  GT_LAUNCH_CHECK("k_walk");
  return GT_OK;
}

}  // namespace
}  // namespace gt

using namespace gt;

extern "C" int gt_infer(int depth, const uint64_t* tree, const uint64_t* queries, uint64_t n, uint64_t nf,
                        uint64_t instance_base, uint64_t* out, uint64_t* slot_out, const gt_keys* keys, void* stream) {
  if (!keys) return fail_inval("gt_infer: NULL keys");
  if (depth < 1 || depth > 13) return fail_inval("depth must be in 1..13");
  if (nf < 1 || nf > 4096) return fail_inval("need 1..4096 features");
  if (n == 0) return GT_OK;
  if (!tree || !queries || !out) return fail_inval("gt_infer: NULL operand");
  const Keys K = to_keys(keys);
  cudaStream_t s = (cudaStream_t)stream;
  int dev = 0, sms = 148;
  GT_CUDA_CHECK(cudaGetDevice(&dev));
  GT_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  // group size G (threads per query): the fewest idle lane-slots over the
  // walk's lookups (sum over levels of ceil(2^t/G) + ceil(nf/G) rounds of G
  // lanes) among the G that still give >= 4 resident warps per SMSP
  const uint64_t target = (uint64_t)sms * 512;
  int best = 32;
  uint64_t best_work = ~0ull;
  for (int G = 1; G <= 32; G <<= 1) {
    uint64_t rounds = 0;
    for (int t = 0; t < depth; ++t) rounds += (((1ull << t) + 1) / 2 + G - 1) / G + ((nf + 1) / 2 + G - 1) / G;
    const uint64_t work = rounds * G;
    if (n * (uint64_t)G >= target && work < best_work) {
      best_work = work;
      best = G;
    }
  }
  static const int forced = getenv("GT_WALK_G") ? atoi(getenv("GT_WALK_G")) : 0;  // A/B experiments
  if (forced >= 1 && forced <= 32 && (forced & (forced - 1)) == 0) best = forced;
  switch (best) {
    case 1: return launch_walk<1>(tree, depth, queries, n, (int)nf, instance_base, out, slot_out, K, s);
    case 2: return launch_walk<2>(tree, depth, queries, n, (int)nf, instance_base, out, slot_out, K, s);
    case 4: return launch_walk<4>(tree, depth, queries, n, (int)nf, instance_base, out, slot_out, K, s);
    case 8: return launch_walk<8>(tree, depth, queries, n, (int)nf, instance_base, out, slot_out, K, s);
    case 16: return launch_walk<16>(tree, depth, queries, n, (int)nf, instance_base, out, slot_out, K, s);
    default: return launch_walk<32>(tree, depth, queries, n, (int)nf, instance_base, out, slot_out, K, s);
  }
}
