// Secure level-wise training on device (reference train_tree,
// pkg/src/obtree/train.py:108-197, heuristic "mpc", fixed/grow policies).
//
// Per level h (n_h = 2^h nodes, W = 2nf+1 sample columns):
//   k_partition   (h > 0)  oaa on level h-1 payloads + row_lookup on features,
//                          m_idx = 2 m_idx + d + 1             train.py:134-139
//   k_count                one lane per (sample, node): eq, and is_leaf, b2a,
//                          W products with reshare, summed over samples
//                          into S[n][w] (+ mask column)        train.py:201-221
//   allreduce(S)           sample-sharded runs only (linear in shares)
//   k_node_hc              one CTA per node: counter assembly, _heuristic_mpc
//                          (division ladder + Newton, masked argmin, budget
//                          clear), replace                      train.py:142-162
//   k_node_stop   (grow)   opened stop bit                     train.py:165-168
//   k_node_finish          split (payload / child type / child counters) or
//                          labels on the last level            train.py:170-192
// Every lane's randomness is keyed by (op, sub, field, global lane), so the
// shares produced are independent of sharding and of launch geometry.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <utility>
#include <vector>

#include "gt_common.cuh"
#include "gt_division.cuh"
#include "gt_lookup.cuh"

namespace gt {
namespace {

constexpr uint64_t F_LEAF = 1, F_DUMMY = 2;  // tree.py:40-42

__device__ __forceinline__ A3 ld3s(const uint64_t* p, uint64_t stride, uint64_t i) {
  return a3(p[i], p[stride + i], p[2 * stride + i]);
}
__device__ __forceinline__ void st3s(uint64_t* p, uint64_t stride, uint64_t i, const A3& a) {
  p[i] = a.v[0];
  p[stride + i] = a.v[1];
  p[2 * stride + i] = a.v[2];
}
// streamed-once operands (the early hit shares: written once, read once):
// evict-first in L2 so they do not push out the level-invariant planes
__device__ __forceinline__ A3 ld3s_cs(const uint64_t* p, uint64_t stride, uint64_t i) {
  return a3(__ldcs(p + i), __ldcs(p + stride + i), __ldcs(p + 2 * stride + i));
}
__device__ __forceinline__ void st3s_cs(uint64_t* p, uint64_t stride, uint64_t i, const A3& a) {
  __stcs(p + i, a.v[0]);
  __stcs(p + stride + i, a.v[1]);
  __stcs(p + 2 * stride + i, a.v[2]);
}
__device__ __forceinline__ B3 ldb3s(const uint64_t* p, uint64_t stride, uint64_t i) {
  B3 b;
  b.v[0] = p[i];
  b.v[1] = p[stride + i];
  b.v[2] = p[2 * stride + i];
  return b;
}

// ---------------------------------------------------------------------------
// init + count:0 products
// ---------------------------------------------------------------------------

__global__ void k_init(uint64_t* f, uint64_t* gam, uint64_t* cst, uint64_t fstride, uint64_t cstride, int cols,
                       int nf) {
  // f_level = const(1), gam = const bits(ones), c_start = 0   (train.py:121-124)
  int t = threadIdx.x;
  if (t < 3) {
    f[t * fstride] = t == 0 ? F_LEAF : 0;
    gam[t * fstride] = t == 0 ? lowmask(nf) : 0;
  }
  for (int e = t; e < 3 * cols; e += blockDim.x)
    for (int c = 0; c < 3; ++c) cst[c * cstride + e] = 0;
}

// count:0 prods = mul(features, labels[:, None])               train.py:115-116
// written straight into the level-invariant sample-column matrix the count
// contraction streams: cols[c][s][0..WC) = x | x*y | y | 0 (mask) | 0 (pad)
// (sample_cols, train.py:117-119).  One thread per (sample, column slot).
__global__ void k_prods(const uint64_t* X, const uint64_t* Y, uint64_t* cols, uint64_t N, int nf, int WC,
                        uint64_t base, Keys K, uint32_t op) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t total = N * (uint64_t)WC, nfx = N * (uint64_t)nf;
  if (e >= total) return;
  const uint64_t s = e / WC;
  const int w = (int)(e % WC);
  A3 v = a3(0, 0, 0);
  if (w < nf) {
    v = ld3s(X, nfx, s * nf + w);
  } else if (w < 2 * nf) {
    v = mul<64>(K, op, 0, (uint32_t)(w - nf), base + s, ld3s(X, nfx, s * nf + (w - nf)), ld3s(Y, N, s));
  } else if (w == 2 * nf) {
    v = ld3s(Y, N, s);
  }
  st3s(cols, total, e, v);
}

// ---------------------------------------------------------------------------
// partition
// ---------------------------------------------------------------------------

// Level-start side work the partition launch carries (no extra launch on the
// chain): zero the level's count sums, and is_leaf = eq(F, LEAF) of the
// level's nodes (train.py:206) for the lane kernel.
struct PartAux {
  uint64_t* S;
  uint64_t swords;
  uint64_t* leaf;      // [3][n_h] bits, or null
  const uint64_t* f;   // [3][n_h] node types of the level
  int n_h;
  uint32_t op_leaf;
};

template <int G>
__global__ void k_partition(const uint64_t* X, uint64_t* midx, const uint64_t* T, uint64_t slots, int m, int nf,
                            uint64_t N, uint64_t base, Keys K, uint32_t op_oaa, uint32_t op_row, PartAux aux) {
  extern __shared__ uint64_t tab[];  // [3][m] level h-1 payload table
  pdl_wait();
  pdl_trigger();
  // zero this level's count sums (the previous level's heuristic has read them)
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < aux.swords;
       i += (uint64_t)gridDim.x * blockDim.x)
    aux.S[i] = 0;
  if (aux.leaf && blockIdx.x == gridDim.x - 1)
    for (int n = threadIdx.x; n < aux.n_h; n += blockDim.x) {
      const B3 z = eqz<64>(K, aux.op_leaf, 0, (uint64_t)n, add_pub<64>(ld3s(aux.f, aux.n_h, n), 0ull - F_LEAF));
#pragma unroll
      for (int c = 0; c < 3; ++c) aux.leaf[c * aux.n_h + n] = z.v[c] & 1ull;
    }
  for (int i = threadIdx.x; i < 3 * m; i += blockDim.x) tab[i] = T[(uint64_t)(i / m) * slots + (m - 1) + (i % m)];
  __syncthreads();
  const uint64_t gt = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t s = gt / G;
  const int t = (int)(gt % G);
  const bool valid = s < N;
  const uint64_t nfx = N * (uint64_t)nf;
  A3 idx = a3(0, 0, 0), part = a3(0, 0, 0);
  if (valid) {
    idx = ld3s(midx, N, s);
    const A3 local = add_pub<64>(idx, 0ull - (uint64_t)(m - 1));
    auto entry = [&](int j) { return a3(tab[j], tab[m + j], tab[2 * m + j]); };
    part = lookup_partial<64>(K, op_oaa, base + s, local, m, t, G, entry);
  }
  const A3 feat = group_sum<G, 64>(part);
  A3 part2 = a3(0, 0, 0);
  if (valid) {
    auto entry = [&](int f) { return ld3s(X, nfx, s * nf + f); };
    part2 = lookup_partial<64>(K, op_row, base + s, feat, nf, t, G, entry);
  }
  const A3 dval = group_sum<G, 64>(part2);
  if (valid && t == 0) st3s(midx, N, s, add_pub<64>(add<64>(mul_pub<64>(idx, 2), dval), 1));
}

// Early oaa lanes of the NEXT level's partition (train.py:135-137): the
// eq / b2a lanes of oaa(payloads_{h-1}, m_idx - (m - 1)) depend only on the
// node index the previous partition produced, not on the payload table the
// heuristic is still choosing, so they run beside the heuristic chain on a
// side stream; the partition then only selects the table entries with them
// (Σ_j ca_j T_j).  One thread per (sample, entry pair); ca[c][j][s] written
// for consecutive samples.  Same lanes and randomness as lookup_pair, so the
// partition's shares are unchanged.
// Work is fetched dynamically (a warp takes OAA_CHUNK x 32 items per atomic
// on *ctr): CTAs resident beside the count start early, the ones that only
// find room after it take the rest.
constexpr int OAA_CHUNK = 4;
__global__ void __launch_bounds__(128) k_oaa_early(const uint64_t* midx, uint64_t* ca, uint64_t N, int m,
                                                   uint64_t base, Keys K, uint32_t op_oaa,
                                                   unsigned long long* ctr, int qe) {
  const int mh = (m + 1) >> 1, lane = threadIdx.x & 31;
  const uint64_t total = N * (uint64_t)min(mh, qe), cs = (uint64_t)m * N;
  for (;;) {
    unsigned long long t0 = 0;
    if (lane == 0) t0 = atomicAdd(ctr, 32ull * OAA_CHUNK);
    t0 = __shfl_sync(0xffffffffu, t0, 0);
    if (t0 >= total) break;
#pragma unroll 1
    for (int k = 0; k < OAA_CHUNK; ++k) {
      const uint64_t t = t0 + (uint64_t)k * 32 + lane;  // consecutive samples across the warp
      if (t >= total) break;
      const int q = (int)(t / N);
      const uint64_t s = t - (uint64_t)q * N;
      const A3 local = add_pub<64>(ld3s(midx, N, s), 0ull - (uint64_t)(m - 1));
      A3 c0, c1;
      lookup_pair_ca<64>(K, op_oaa, base + s, local, m, q, &c0, &c1);
      st3s_cs(ca, cs, (uint64_t)(2 * q) * N + s, c0);
      if (2 * q + 1 < m) st3s_cs(ca, cs, (uint64_t)(2 * q + 1) * N + s, c1);
    }
  }
}

// Split partition: B threads per sample, placed in DIFFERENT warps (thread t
// of the 256-thread CTA serves sample t % S of the CTA's S = 256 / B samples
// as member r = t / S), so every lane of a warp runs the same entry pair q
// at the same time -- uniform trip counts, warp-uniform table entries --
// while the level's lookups get B times the threads of one-thread-per-sample.
// Member r draws the telescope words e = r, r + B, ... and the entry pairs
// q = r, r + B, ...; the B partial sums meet in shared memory.  Same lanes,
// same randomness as lookup_partial (identical shares).
constexpr int PS_TPB = 256;
template <int B>
__global__ void __launch_bounds__(PS_TPB, 3)
    k_partition_split(const uint64_t* X, uint64_t* midx, const uint64_t* T, uint64_t slots, int m, int nf, uint64_t N,
                      uint64_t base, Keys K, uint32_t op_oaa, uint32_t op_row, PartAux aux, int tab_smem,
                      const uint64_t* __restrict__ ca, int qe) {
  constexpr int S = PS_TPB / B;
  __shared__ uint64_t part[B][3][S];  // members' partial sums
  __shared__ uint64_t feat[3][S];     // the sample's fetched feature index (shares)
  extern __shared__ uint64_t tab[];   // [3][m] level payloads (if staged)
  pdl_wait();
  pdl_trigger();
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < aux.swords;
       i += (uint64_t)gridDim.x * blockDim.x)
    aux.S[i] = 0;
  if (aux.leaf && blockIdx.x == gridDim.x - 1)
    for (int n = threadIdx.x; n < aux.n_h; n += blockDim.x) {
      const B3 z = eqz<64>(K, aux.op_leaf, 0, (uint64_t)n, add_pub<64>(ld3s(aux.f, aux.n_h, n), 0ull - F_LEAF));
#pragma unroll
      for (int c = 0; c < 3; ++c) aux.leaf[c * aux.n_h + n] = z.v[c] & 1ull;
    }
  if (tab_smem)
    for (int i = threadIdx.x; i < 3 * m; i += blockDim.x) tab[i] = T[(uint64_t)(i / m) * slots + (m - 1) + (i % m)];
  __syncthreads();
  const uint64_t* tg = T + (m - 1);
  auto entryT = [&](int j) {
    return tab_smem ? a3(tab[j], tab[m + j], tab[2 * m + j])
                    : a3(__ldg(tg + j), __ldg(tg + slots + j), __ldg(tg + 2 * slots + j));
  };
  const int ls = threadIdx.x % S, r = threadIdx.x / S;  // r is warp-uniform
  const uint64_t s = (uint64_t)blockIdx.x * S + ls;
  const bool valid = s < N;
  const uint64_t nfx = N * (uint64_t)nf, g = base + s;
  A3 idx = a3(0, 0, 0), acc = a3(0, 0, 0);
  if (valid) {  // oaa on the level-(h-1) payloads at local = m_idx - (m - 1)   (train.py:135-137)
    idx = ld3s(midx, N, s);
    if (ca) {  // hit shares drawn early (k_oaa_early): the telescope words + the entries' selects
      for (int e = r; e < 6; e += B) acc = add<64>(acc, lookup_word<64>(K, op_oaa, g, m, e));
      const uint64_t F0[3] = {0, 0, 0}, cs = (uint64_t)m * N;
      const int mh = (m + 1) >> 1, je = min(m, 2 * qe);
      for (int j = r; j < je; j += B) acc = add<64>(acc, mul_z<64>(entryT(j), ld3s_cs(ca, cs, (uint64_t)j * N + s), F0));
      if (qe < mh) {  // the pairs the early lanes left: drawn here (same lanes, same randomness)
        const A3 local = add_pub<64>(idx, 0ull - (uint64_t)(m - 1));
        for (int q = qe + r; q < mh; q += B) acc = add<64>(acc, lookup_pair<64>(K, op_oaa, g, local, m, q, entryT));
      }
    } else {
      acc = lookup_partial<64>(K, op_oaa, g, add_pub<64>(idx, 0ull - (uint64_t)(m - 1)), m, r, B, entryT);
    }
  }
  if (B > 1) {
#pragma unroll
    for (int c = 0; c < 3; ++c) part[r][c][ls] = acc.v[c];
    __syncthreads();
    if (r == 0) {
#pragma unroll
      for (int q = 1; q < B; ++q) acc = add<64>(acc, a3(part[q][0][ls], part[q][1][ls], part[q][2][ls]));
#pragma unroll
      for (int c = 0; c < 3; ++c) feat[c][ls] = acc.v[c];
    }
    __syncthreads();
    acc = a3(feat[0][ls], feat[1][ls], feat[2][ls]);
  }
  A3 d = a3(0, 0, 0);
  if (valid) {  // row_lookup of the sample's features at the fetched index   (train.py:138)
    auto entryX = [&](int f) { return ld3s(X, nfx, s * nf + f); };
    if (B == 2 && (((nf + 1) >> 1) & 1)) {
      // an odd number of entry pairs: member 0 takes pairs 0, 2, ... (one
      // more than member 1), member 1 the pairs 1, 3, ... and all six
      // telescope words, so neither member's chain is longer than its pairs
      d = a3(0, 0, 0);
      if (r == 1)
        for (int e = 0; e < 6; ++e) d = add<64>(d, lookup_word<64>(K, op_row, g, nf, e));
      for (int q = r; q < ((nf + 1) >> 1); q += 2) d = add<64>(d, lookup_pair<64>(K, op_row, g, acc, nf, q, entryX));
    } else {
      d = lookup_partial<64>(K, op_row, g, acc, nf, r, B, entryX);
    }
  }
  if (B > 1) {
    __syncthreads();
#pragma unroll
    for (int c = 0; c < 3; ++c) part[r][c][ls] = d.v[c];
    __syncthreads();
    if (r == 0)
#pragma unroll
      for (int q = 1; q < B; ++q) d = add<64>(d, a3(part[q][0][ls], part[q][1][ls], part[q][2][ls]));
  }
  if (valid && r == 0) st3s(midx, N, s, add_pub<64>(add<64>(mul_pub<64>(idx, 2), d), 1));  // train.py:139
}

// ---------------------------------------------------------------------------
// count
// ---------------------------------------------------------------------------

constexpr int CNT_TPB = 256;
constexpr int CNT_NA = 2;  // nodes per contraction thread tile
constexpr int CNT_CB = 4;  // columns per contraction thread tile

// is_leaf = eq(F_level, LEAF) per node (train.py:206) -> leaf[3][n_h] bits
__global__ void k_count_leaf(const uint64_t* f, uint64_t* leaf, int n_h, Keys K, uint32_t op_leaf) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= n_h) return;
  const B3 z = eqz<64>(K, op_leaf, 0, (uint64_t)n, add_pub<64>(ld3s(f, n_h, n), 0ull - F_LEAF));
#pragma unroll
  for (int c = 0; c < 3; ++c) leaf[c * n_h + n] = z.v[c] & 1ull;
}

struct LaneArgs {
  const uint64_t *midx, *leaf;
  uint64_t* la;                   // [3][nblk][cap][nbp]: node-block-major, so a contraction tile is contiguous
  uint64_t N, s0, cn, cap, base;  // shard samples, chunk start, chunk samples, chunk capacity, shard base
  int n_h, off, nb, nbp, nblk;
  Keys K;
  uint32_t op_cnt;
};

// One thread per (sample pair, node) of a sample chunk:
//   la = b2a(eq(m_idx, off+n) & is_leaf[n])                 train.py:214-217
// (dealer material per lane, the two lanes' zero words from one pair block:
// count_lane_pair).  Padding node slots are written as zero shares.
__global__ void __launch_bounds__(256) k_count_lanes(LaneArgs a) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t per = (uint64_t)a.nblk * a.nbp;
  const uint64_t pairs = (a.cn + 1) / 2;
  if (e >= pairs * per) return;
  const uint64_t s = 2 * (e / per);
  const int r = (int)(e % per), blk = r / a.nbp, nn = r % a.nbp, n = blk * a.nb + nn;
  const uint64_t cs = (uint64_t)a.nblk * a.cap * a.nbp;
  uint64_t* out = a.la + ((uint64_t)blk * a.cap + s) * a.nbp + nn;
  const bool v1 = s + 1 < a.cn;
  if (nn >= a.nb || n >= a.n_h) {
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      out[c * cs] = 0;
      if (v1) out[c * cs + a.nbp] = 0;
    }
    return;
  }
  const uint64_t gs = a.s0 + s;
  const uint64_t off = 0ull - (uint64_t)(a.off + n);
  const A3 d0 = add_pub<64>(a3(__ldg(a.midx + gs), __ldg(a.midx + a.N + gs), __ldg(a.midx + 2 * a.N + gs)), off);
  A3 d1 = a3(0, 0, 0);
  if (v1) d1 = add_pub<64>(a3(__ldg(a.midx + gs + 1), __ldg(a.midx + a.N + gs + 1), __ldg(a.midx + 2 * a.N + gs + 1)), off);
  B3 lf;
#pragma unroll
  for (int c = 0; c < 3; ++c) lf.v[c] = __ldg(a.leaf + c * a.n_h + n);
  A3 l0, l1;
  count_lane_pair(a.K, a.op_cnt, a.base + gs, a.n_h, n, d0, d1, true, v1, lf, &l0, &l1);
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    out[c * cs] = l0.v[c];
    if (v1) out[c * cs + a.nbp] = l1.v[c];
  }
}

// --- TMA bulk copies (cp.async.bulk) into shared memory, mbarrier completion
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// The suspend-time hint lets the hardware park a waiting warp until the phase
// completes (or the hint expires) instead of re-issuing the probe: the
// count's single-thread copy / MMA warps otherwise spin on their barriers in
// the producers' issue slots.
constexpr uint32_t MBAR_SUSPEND_NS = 0x989680;
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(MBAR_SUSPEND_NS)
      : "memory");
}

// acc + (x << 32) += a * b (mod 2^64): the low-half product accumulates in
// 64 bits (IMAD.WIDE.U32 with the accumulator as addend), the two cross
// products in a separate 32-bit word (the high x high product vanishes mod
// 2^64); the two are combined once after the sample loop.
__device__ __forceinline__ void mac64(uint64_t& acc, uint32_t& x, uint64_t a, uint64_t b) {
  acc += (uint64_t)(uint32_t)a * (uint32_t)b;
  x += (uint32_t)a * (uint32_t)(b >> 32) + (uint32_t)(a >> 32) * (uint32_t)b;
}

struct MacArgs {
  const uint64_t *la, *cols;  // la [3][nblk][cap][nbp] (chunk), cols [3][N][WC] (shard)
  uint64_t* S;                // [3][n_h][W+1]
  uint64_t N, s0, cn, cap;
  int n_h, W, WC, nb, nbp, nblk, ts, tiles_per_cta;
};

// Count contraction of one sample chunk: each thread owns NA nodes x CB
// columns x 3 components and accumulates the party-local cross terms of
// mul(cols, la) (rss.py:391-395)
//     acc_i += la_i (x_i + x_{i+1}) + la_{i+1} x_i
// over its samples; the mask column (x = 0, u = 1) accumulates la_i itself
// (s_mask, train.py:220).  Tiles of TS samples (la rows of the node block and
// column rows) arrive by cp.async.bulk into a 2-stage ring.  The products'
// reshare zero shares are not drawn here: their per-sample stream telescopes
// (F(t) = H(t+1) - H(t)) and k_count_alpha adds the
// shard's sum once per cell.
__global__ void __launch_bounds__(CNT_TPB, 1) k_count_mac(MacArgs a) {
  extern __shared__ __align__(128) uint64_t sm[];
  __shared__ __align__(8) uint64_t full[2];
  const int W = a.W, WC = a.WC, NBP = a.nbp, TS = a.ts;
  const int tid = threadIdx.x;
  const int blk = blockIdx.y, n0 = blk * a.nb, nb = min(a.nb, a.n_h - n0);
  const int stage_words = 3 * TS * (NBP + WC);
  const uint64_t cs_la = (uint64_t)a.nblk * a.cap * NBP, cs_col = a.N * (uint64_t)WC;
  const uint64_t tile0 = (uint64_t)blockIdx.x * a.tiles_per_cta;
  const uint64_t ntiles = (a.cn + TS - 1) / TS;
  const int my_tiles = (int)min((uint64_t)a.tiles_per_cta, ntiles > tile0 ? ntiles - tile0 : 0);

  auto issue = [&](int t) {  // one elected thread: 6 bulk copies of tile t into stage t & 1
    const uint64_t s0 = (tile0 + t) * (uint64_t)TS;
    const int cnt = (int)min((uint64_t)TS, a.cn - s0);
    uint64_t* st = sm + (t & 1) * stage_words;
    const uint32_t lb = (uint32_t)(cnt * NBP * 8), cb = (uint32_t)(cnt * WC * 8);
    mbar_expect_tx(&full[t & 1], 3 * (lb + cb));
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      bulk_g2s(st + c * TS * NBP, a.la + c * cs_la + ((uint64_t)blk * a.cap + s0) * NBP, lb, &full[t & 1]);
      bulk_g2s(st + 3 * TS * NBP + c * TS * WC, a.cols + c * cs_col + (a.s0 + s0) * WC, cb, &full[t & 1]);
    }
  };
  if (tid == 0) {
    mbar_init(&full[0], 1);
    mbar_init(&full[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    if (my_tiles > 0) issue(0);
    if (my_tiles > 1) issue(1);
  }

  const int CT = WC / CNT_CB, P = (NBP / CNT_NA) * CT;
  const int R = max(1, CNT_TPB / P);  // replicas split a tile's samples
  const bool active = tid < P * R;
  const int item = active ? tid % P : 0, q = tid / P;
  const int nl = (item / CT) * CNT_NA, cl = (item % CT) * CNT_CB;
  uint64_t mflag[CNT_CB];  // 1 on the mask column: u = x_i + x_{i+1} + 1 = 1 there
#pragma unroll
  for (int j = 0; j < CNT_CB; ++j) mflag[j] = (cl + j == W) ? 1ull : 0ull;
  uint64_t acc[3][CNT_NA][CNT_CB];
  uint32_t accx[3][CNT_NA][CNT_CB];
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < CNT_NA; ++i)
#pragma unroll
      for (int j = 0; j < CNT_CB; ++j) acc[c][i][j] = 0, accx[c][i][j] = 0;

  for (int t = 0; t < my_tiles; ++t) {
    const int cnt = (int)min((uint64_t)TS, a.cn - (tile0 + t) * (uint64_t)TS);
    mbar_wait(&full[t & 1], (uint32_t)((t >> 1) & 1));
    const uint64_t* lat = sm + (t & 1) * stage_words;
    const uint64_t* xst = lat + 3 * TS * NBP;
    if (active) {
#pragma unroll 2
      for (int s = q; s < cnt; s += R) {
        uint64_t l[3][CNT_NA], x[3][CNT_CB];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const ulonglong2 lv = *reinterpret_cast<const ulonglong2*>(lat + (c * TS + s) * NBP + nl);
          l[c][0] = lv.x;
          l[c][1] = lv.y;
#pragma unroll
          for (int j = 0; j < CNT_CB; j += 2) {
            const ulonglong2 xv = *reinterpret_cast<const ulonglong2*>(xst + (c * TS + s) * WC + cl + j);
            x[c][j] = xv.x;
            x[c][j + 1] = xv.y;
          }
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int cn = (c + 1) % 3;
#pragma unroll
          for (int j = 0; j < CNT_CB; ++j) {
            const uint64_t u = x[c][j] + x[cn][j] + mflag[j];
#pragma unroll
            for (int i = 0; i < CNT_NA; ++i) {
              mac64(acc[c][i][j], accx[c][i][j], l[c][i], u);
              mac64(acc[c][i][j], accx[c][i][j], l[cn][i], x[c][j]);
            }
          }
        }
      }
    }
    __syncthreads();  // stage t & 1 consumed
    if (tid == 0 && t + 2 < my_tiles) issue(t + 2);
  }
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int i = 0; i < CNT_NA; ++i)
#pragma unroll
      for (int j = 0; j < CNT_CB; ++j) acc[c][i][j] += (uint64_t)accx[c][i][j] << 32;
  // replicas of an item meet in shared memory; one atomic per (cell, component) per CTA
  constexpr int NACC = 3 * CNT_NA * CNT_CB;
  if (R > 1) {
    if (active)
#pragma unroll
      for (int c = 0; c < 3; ++c)
#pragma unroll
        for (int i = 0; i < CNT_NA; ++i)
#pragma unroll
          for (int j = 0; j < CNT_CB; ++j) sm[((uint64_t)q * P + item) * NACC + (c * CNT_NA + i) * CNT_CB + j] = acc[c][i][j];
    __syncthreads();
    if (active && q == 0)
      for (int r = 1; r < R; ++r)
#pragma unroll
        for (int c = 0; c < 3; ++c)
#pragma unroll
          for (int i = 0; i < CNT_NA; ++i)
#pragma unroll
            for (int j = 0; j < CNT_CB; ++j) acc[c][i][j] += sm[((uint64_t)r * P + item) * NACC + (c * CNT_NA + i) * CNT_CB + j];
  }
  if (!active || q != 0 || my_tiles == 0) return;
  const uint64_t Sstride = (uint64_t)a.n_h * (W + 1);
#pragma unroll
  for (int i = 0; i < CNT_NA; ++i) {
    if (nl + i >= nb) continue;
#pragma unroll
    for (int j = 0; j < CNT_CB; ++j) {
      if (cl + j > W) continue;
#pragma unroll
      for (int c = 0; c < 3; ++c)
        atomicAdd((unsigned long long*)&a.S[c * Sstride + (uint64_t)(n0 + nl + i) * (W + 1) + cl + j],
                  (unsigned long long)acc[c][i][j]);
    }
  }
}

}  // namespace
}  // namespace gt
#include "gt_count_tc.cuh"
namespace gt {
namespace {

// ---------------------------------------------------------------------------
// per-node heuristic (_heuristic_mpc, train.py:232-274) + replace, in three
// kernels so no thread waits on another's serial chain:
//   k_hc_pre   one CTA per node: counter assembly; warp 0 runs the short
//              probe/featureless/should_split/new_f chain, warp 1 replace;
//              warps 2-7 truncate + ring_down the counters, form the squares
//              and Q products and the Q==0 fix (pv, qs -> global)
//   k_hc_div   one WARP per (node, column): division_warp (ladder over the
//              lanes, Newton chain from a cooperatively drawn Philox tape)
//   k_hc_post  one CTA per node: scores, masked argmin tournament, budget
//              clear
// ---------------------------------------------------------------------------

// Phase timestamps of the heuristic kernels (diagnostics: GT_HC_TIMING=1
// makes node 0's thread 0 record %globaltimer at each phase boundary).
// Slots 0..63: post/finish (8 per level); 64..127: pre/div (8 per level:
// 0 control start, 1 control tapes in, 2 control end, 3 feature-warp start,
// 4 feature tape in, 5 feature end, 6 div start, 7 div end).
__device__ unsigned long long g_hc_ts[128];
__device__ __forceinline__ void hc_ts_at(int slot, bool on) {
  if (!on) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_hc_ts[slot] = t;
}
__device__ __forceinline__ void hc_ts(int slot, bool on) { hc_ts_at(slot, on && blockIdx.x == 0 && threadIdx.x == 0); }

// The heuristic kernels draw Philox blocks along long dependent chains and,
// in warp-cooperative draws, with lane-dependent keys: stage the expanded
// round keys in shared memory once per CTA (every thread of the CTA calls
// this before diverging) instead of indexing the kernel parameters.
__device__ __forceinline__ const Keys& keys_smem(const Keys& K, Keys& ks) {
  for (int i = threadIdx.x; i < (int)(sizeof(Keys) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&ks)[i] = reinterpret_cast<const uint32_t*>(&K)[i];
  __syncthreads();
  return ks;
}

struct NodeArgs {
  const uint64_t* S;          // [3][n_h][W+1]
  const uint64_t* cst;        // [3][n_h][3][cols]
  const uint64_t* f;          // [3][n_h]
  const uint64_t* gam;        // [3][n_h] feature-budget bit words
  const uint64_t* ceff_prev;  // [3][n_h/2][3][cols]
  uint64_t* ceff;             // [3][n_h][3][cols]
  uint64_t* hc;               // [4][3][n_h]: should_split, sd, new_f, new_gam
  uint64_t* dv;               // [3][3][n_h*cols]: P, Q+[Q==0], division terms
  uint64_t* co_out;           // [3][n_h][3][cols] c_orig for the tee helper (or null)
  const W2* divtape;          // precomputed division blocks of this level (or null: draw live)
  const W2* posttape;         // precomputed epilogue blocks of this level (or null: draw live)
  const W2* nodetape;         // precomputed node-chain blocks of this level's nodes (or null)
  const W2* feattape;         // precomputed prologue feature blocks of this level (or null)
  int n_h, nf, level, last, shift, tau, ts;
  int fuse_div;               // the division runs in k_hc_pre's feature CTAs (needs divtape)
  DivParams d;
  Keys K;
};

__device__ __forceinline__ void bar_workers() { asm volatile("bar.sync 1, 192;" ::: "memory"); }

// ---------------------------------------------------------------------------
// Node tapes: the randomness of the per-node chains of every level (heuristic
// prologue: probe eqs, featureless AND tree, ORs, should_split AND, new_f
// select; replace: eq, b2a, counter selects; split: payload / child type /
// condition selects, child counter selects; labels: lt + b2a), drawn for all
// levels up front like the division tapes and staged per node by one bulk
// copy.  Layout per node (blocks):
//   PRE  [3 eqz x 5][and_reduce 3][or 3][or 3][and 3][select 5]        = 32
//   REP  [eqz 5][b2a 2][select muls 3 x ceil(3 cols / 2)]
//   SPL  [b2a 2 + mul 3][b2a 2 + mul 3][b2a 2][counter muls 3 x ceil(3 cols / 2)]
//   LAB  [lt LtRand<64>][b2a 2]
// Entry: site (8) | key+1 (8) | sub (8) | pidx (16) | lane kind (8: 0 = n,
// 1 = 3n + idx) | idx (8).
struct NodeTape {
  int rep, spl, lab, total;  // segment offsets (PRE at 0)
};
__host__ __device__ inline NodeTape node_tape_plan(int nf) {
  const int mh = (3 * 2 * nf + 1) / 2;  // counter-select blocks per key
  NodeTape t;
  t.rep = 32;
  t.spl = t.rep + 7 + 3 * mh;
  t.lab = t.spl + 12 + 3 * mh;
  t.total = t.lab + LtRand<64>::BLOCKS + 2;
  return t;
}
__device__ __forceinline__ uint64_t node_entry(uint32_t site, int key, uint32_t sub, uint32_t pidx, int kind, int idx) {
  return (uint64_t)site | ((uint64_t)(uint32_t)(key + 1) << 8) | ((uint64_t)sub << 16) | ((uint64_t)pidx << 24) |
         ((uint64_t)kind << 40) | ((uint64_t)idx << 48);
}
__global__ void k_node_table(uint64_t* table, int nf) {
  const NodeTape t = node_tape_plan(nf);
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= t.total) return;
  uint64_t v;
  if (e < t.rep) {  // PRE (op HC)
    if (e < 15) {  // eqz lane 3n + j at sub 0: dealer (0,0) (0,1), pair_i (0,0)
      const int j = e / 5, w = e % 5;
      v = w < 2 ? node_entry(SITE_HC, -1, 0, w, 1, j) : node_entry(SITE_HC, w - 2, 0, 0, 1, j);
    } else if (e < 27) {  // and_reduce (sub 1), or (2), or (3), and (4): pair_i (sub, 0)
      const int q = e - 15;
      v = node_entry(SITE_HC, q % 3, 1 + q / 3, 0, 0, 0);
    } else {  // select at 5: b2a dealer (5,0) (5,1), mul pair_i (6,0)
      const int w = e - 27;
      v = w < 2 ? node_entry(SITE_HC, -1, 5, w, 0, 0) : node_entry(SITE_HC, w - 2, 6, 0, 0, 0);
    }
  } else if (e < t.spl) {  // REP (op REPLACE): eqz at 0, b2a at 1, counter-select muls at 2
    const int q = e - t.rep;
    if (q < 5) v = q < 2 ? node_entry(SITE_REPLACE, -1, 0, q, 0, 0) : node_entry(SITE_REPLACE, q - 2, 0, 0, 0, 0);
    else if (q < 7) v = node_entry(SITE_REPLACE, -1, 1, q - 5, 0, 0);
    else v = node_entry(SITE_REPLACE, (q - 7) % 3, 2, (q - 7) / 3, 0, 0);
  } else if (e < t.lab) {  // SPL (op SPLIT): selects at 0/1, 2/3, b2a at 4, counter-select muls at 5
    const int q = e - t.spl;
    if (q < 10) {
      const int g = q / 5, w = q % 5;
      v = w < 2 ? node_entry(SITE_SPLIT, -1, 2 * g, w, 0, 0) : node_entry(SITE_SPLIT, w - 2, 2 * g + 1, 0, 0, 0);
    } else if (q < 12) {
      v = node_entry(SITE_SPLIT, -1, 4, q - 10, 0, 0);
    } else {
      v = node_entry(SITE_SPLIT, (q - 12) % 3, 5, (q - 12) / 3, 0, 0);
    }
  } else {  // LAB (op LABELS): lt at 0, b2a at 1
    const int q = e - t.lab;
    if (q < LtRand<64>::BLOCKS) {
      int key;
      uint32_t pidx;
      lt_block_id<64>(q, 0, &key, &pidx);
      v = node_entry(SITE_LABELS, key, 0, pidx, 0, 0);
    } else {
      v = node_entry(SITE_LABELS, -1, 1, q - LtRand<64>::BLOCKS, 0, 0);
    }
  }
  table[e] = v;
}
// [global node (2^level - 1 + n)][entry]; one thread per block
__global__ void __launch_bounds__(256) k_node_tape(W2* tape, const uint64_t* __restrict__ table, uint32_t total, int E,
                                                   Keys K) {
  __shared__ Keys ks;
  for (int i = threadIdx.x; i < (int)(sizeof(Keys) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&ks)[i] = reinterpret_cast<const uint32_t*>(&K)[i];
  __syncthreads();
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const uint32_t gn = e / (uint32_t)E;
  const uint64_t t = __ldg(table + (e - gn * (uint32_t)E));
  const int level = 31 - __clz(gn + 1);
  const uint32_t n = gn - ((1u << level) - 1);
  const uint32_t site = (uint32_t)(t & 0xff), sub = (uint32_t)((t >> 16) & 0xff), pidx = (uint32_t)((t >> 24) & 0xffff);
  const int key = (int)((t >> 8) & 0xff) - 1, kind = (int)((t >> 40) & 0xff), idx = (int)((t >> 48) & 0xff);
  const uint64_t lane = kind ? 3ull * n + idx : (uint64_t)n;
  tape[e] = word2(key < 0 ? ks.dealer : ks.pair[key], op_id(level, site), sub, pidx, lane);
}
// stage a node's tape segment [off, off + len) into shared memory by one bulk copy (thread 0 issues; all wait)
__device__ __forceinline__ const W2* stage_node_tape(const W2* g, int len, W2* dst, uint64_t* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(bar, (uint32_t)(len * sizeof(W2)));
    bulk_g2s(dst, g, (uint32_t)(len * sizeof(W2)), bar);
  }
  __syncthreads();
  mbar_wait(bar, 0);
  return dst;
}

// c_orig cell e = (row r, column k) of node n: c_start + the counters
// assembled from the count partials (train.py:142, 336-343)
__device__ __forceinline__ uint64_t co_cell(const NodeArgs& a, int c, int n, int e) {
  const int nf = a.nf, cols = 2 * nf, W = cols + 1, C3 = 3 * cols;
  const uint64_t hs = (uint64_t)a.n_h;
  const int r = e / cols, k = e % cols, i = k >> 1, j = k & 1;
  const uint64_t* Sn = a.S + (uint64_t)c * hs * (W + 1) + (uint64_t)n * (W + 1);
  const uint64_t s1 = Sn[W], sx = Sn[i], sp = Sn[nf + i], sy = Sn[2 * nf];
  uint64_t v;
  if (r == 0) v = j ? sx : s1 - sx;
  else if (r == 1) v = j ? sx - sp : s1 - sx - sy + sp;
  else v = j ? sp : sy - sp;
  return a.cst[(uint64_t)c * hs * C3 + (uint64_t)n * C3 + e] + v;
}

// Heuristic prologue, grid (node, 1 + features):
//  y = 0 (control CTA, 64 threads): counter assembly; warp 0 runs the short
//     probe / featureless / should_split / new_f chain, warp 1 replace
//  y = 1 + i (one warp per feature i): the six counter cells of feature i
//     are truncated by the public shift and ring_down'ed, the squares and the
//     a*tot products formed, then P, Q and the Q == 0 fix for its two
//     columns (train.py:252-267).  The warp first draws every Philox block
//     of the feature (truncations, products, eq, b2a: the live schedule's
//     blocks) into shared memory in parallel, so the serial gadget chain
//     only does arithmetic.
// The Philox blocks of feature fi of node n in the prologue, in consumption
// order: six truncations (cells q = r*2 + j <-> e = r*cols + 2fi + j, sub 7),
// eight products (sub 10; p < 6: cell p squared, p = 6 + j: a * tot), two
// (eqz sub 11, b2a sub 12) for the Q == 0 fix of columns 2fi, 2fi+1.
constexpr int FEAT_BLOCKS = 6 * TruncRand<64>::BLOCKS + 8 * 3 + 2 * 7;
__device__ __forceinline__ void feat_block(int b, int fi, int nf, uint32_t n, int* key, uint32_t* sub, uint32_t* pidx,
                                           uint64_t* lane) {
  constexpr int TB = TruncRand<64>::BLOCKS;
  const int cols = 2 * nf, C3 = 3 * cols;
  auto cell_e = [&](int q) { return (q >> 1) * cols + 2 * fi + (q & 1); };
  auto prod_e = [&](int p) { return p < 6 ? cell_e(p) : C3 + 2 * fi + (p - 6); };
  *key = -1;
  if (b < 6 * TB) {
    trunc_block_id<64>(b % TB, 7, key, sub, pidx);
    *lane = (uint64_t)n * C3 + cell_e(b / TB);
  } else if (b < 6 * TB + 24) {
    const int t = b - 6 * TB;
    *key = t % 3, *sub = 10, *pidx = 0;
    *lane = (uint64_t)n * 4 * cols + prod_e(t / 3);
  } else {
    const int t = b - 6 * TB - 24, j = t / 7, w = t % 7;
    *lane = (uint64_t)n * cols + 2 * fi + j;
    if (w < 2) *key = -1, *sub = 11, *pidx = w;            // eqz dealer (r, Rb0) (Rb1, -)
    else if (w < 5) *key = w - 2, *sub = 11, *pidx = 0;    // eqz zero words
    else *key = -1, *sub = 12, *pidx = w - 5;              // b2a dealer (A0, A1) (bits, -)
  }
}
// every heuristic level's feature tapes: [global node][feature][FEAT_BLOCKS]
__global__ void __launch_bounds__(256) k_feat_tape(W2* tape, uint32_t total, int nf, Keys K) {
  __shared__ Keys ks;
  for (int i = threadIdx.x; i < (int)(sizeof(Keys) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&ks)[i] = reinterpret_cast<const uint32_t*>(&K)[i];
  __syncthreads();
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const uint32_t per = (uint32_t)nf * FEAT_BLOCKS;
  const uint32_t gn = e / per, r = e - gn * per, fi = r / FEAT_BLOCKS, b = r - fi * FEAT_BLOCKS;
  const int level = 31 - __clz(gn + 1);
  const uint32_t n = gn - ((1u << level) - 1);
  int key;
  uint32_t sub, pidx;
  uint64_t lane;
  feat_block((int)b, (int)fi, nf, n, &key, &sub, &pidx, &lane);
  tape[e] = word2(key < 0 ? ks.dealer : ks.pair[key], op_id(level, SITE_HC), sub, pidx, lane);
}

template <int SL>
__device__ __forceinline__ void hc_pre_feature(const NodeArgs& a, int n, int fi, const Keys& K, uint64_t (*pq)[2][3]) {
  constexpr uint64_t MS = Ring<SL>::M;
  constexpr int TB = TruncRand<64>::BLOCKS;
  constexpr int NB = FEAT_BLOCKS;
  __shared__ __align__(128) W2 tape[NB];
  __shared__ __align__(8) uint64_t fbar;
  __shared__ uint64_t c32[3][6], pr[3][8];
  const int wl = threadIdx.x;
  const int nf = a.nf, cols = 2 * nf, C3 = 3 * cols;
  const uint64_t hs = (uint64_t)a.n_h, lanes = hs * cols;
  const uint32_t opH = op_id(a.level, SITE_HC);
  auto cell_e = [&](int q) { return (q >> 1) * cols + 2 * fi + (q & 1); };
  const bool tsw = a.ts && n == 0 && fi == 0 && wl == 0;
  hc_ts_at(64 + 8 * a.level + 3, tsw);
  if (a.feattape) {  // precomputed: one bulk copy
    if (wl == 0) {
      mbar_init(&fbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&fbar, (uint32_t)(NB * sizeof(W2)));
      bulk_g2s(tape, a.feattape + ((uint64_t)n * nf + fi) * NB, (uint32_t)(NB * sizeof(W2)), &fbar);
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    mbar_wait(&fbar, 0);
  } else {
    pdl_wait();
    pdl_trigger();
    for (int b = wl; b < NB; b += 32) {
      if (b < 6 * TB && !a.shift) continue;
      int key;
      uint32_t sub, pidx;
      uint64_t lane;
      feat_block(b, fi, nf, (uint32_t)n, &key, &sub, &pidx, &lane);
      tape[b] = word2(key < 0 ? K.dealer : K.pair[key], opH, sub, pidx, lane);
    }
    __syncwarp();
  }
  hc_ts_at(64 + 8 * a.level + 4, tsw);
  // counters: truncate by the public shift, ring_down      train.py:252-256
  if (wl < 6) {
    const int e = cell_e(wl);
    A3 x = a3(co_cell(a, 0, n, e), co_cell(a, 1, n, e), co_cell(a, 2, n, e));
    if (a.shift) x = trunc_arith<64>(tape + wl * TB, x, a.shift);
#pragma unroll
    for (int c = 0; c < 3; ++c) c32[c][wl] = x.v[c] & MS;
  }
  __syncwarp();
  auto C32 = [&](int q) { return a3(c32[0][q], c32[1][q], c32[2][q]); };
  // prods = mul([c32, a], [c32, tot_rep])                   train.py:257-262
  if (wl < 8) {
    A3 x, y;
    if (wl < 6) {
      x = C32(wl);
      y = x;
    } else {
      x = C32(wl - 6);  // row 0, column 2fi + j
      y = add<SL>(C32(0), C32(1));
    }
    const W2* t = tape + 6 * TB + 3 * wl;
    const uint64_t F[3] = {t[0].a, t[1].a, t[2].a};
    const A3 z = mul_z<SL>(x, y, F);
#pragma unroll
    for (int c = 0; c < 3; ++c) pr[c][wl] = z.v[c];
  }
  __syncwarp();
  // P = a^2 - m0^2 - m1^2, qsafe = Q + b2a(eq(Q, 0))       train.py:263-267
  if (wl < 2) {
    auto PR = [&](int p) { return a3(pr[0][p], pr[1][p], pr[2][p]); };
    const A3 p = diff<SL>(diff<SL>(PR(wl), PR(2 + wl)), PR(4 + wl));
    const A3 q = PR(6 + wl);
    const W2* t = tape + 6 * TB + 24 + 7 * wl;
    const uint64_t Zw[3] = {t[2].a, t[3].a, t[4].a};
    const B3 qz = eq_arith<SL>(q, t[0].a, t[0].b, t[1].a, Zw);
    const A3 qsv = add<SL>(q, b2a_arith<SL>(qz, t[5].a, t[5].b, t[6].a));
    const uint64_t lane = (uint64_t)n * cols + 2 * fi + wl;
    if (pq) {  // the division runs in this CTA
#pragma unroll
      for (int c = 0; c < 3; ++c) pq[wl][0][c] = p.v[c], pq[wl][1][c] = qsv.v[c];
    } else {
      st3s(a.dv, lanes, lane, p);
      st3s(a.dv + 3 * lanes, lanes, lane, qsv);
    }
  }
  hc_ts_at(64 + 8 * a.level + 5, tsw);
}

template <int SL>
__global__ void __launch_bounds__(64) k_hc_pre(NodeArgs a) {
  const int n = blockIdx.x;
  if (blockIdx.y > 0) {  // the feature warp draws with lane-dependent keys: stage them in smem
    __shared__ Keys ks;
    const Keys& Ks = keys_smem(a.K, ks);
    const int fi = (int)blockIdx.y - 1, warp = threadIdx.x >> 5;
    if (!a.fuse_div) {
      if (warp == 0) hc_pre_feature<SL>(a, n, fi, Ks, nullptr);
      return;
    }
    // fused division (train.py:268): warp j divides column 2fi + j from its
    // precomputed lane tape, bulk-copied before the wait for the contraction
    extern __shared__ __align__(128) W2 dts[];  // [2][div_tape_blocks]
    __shared__ __align__(8) uint64_t dbar[2];
    __shared__ uint64_t pq[2][2][3];
    const int TB = div_tape_blocks<SL>(a.d);
    const uint64_t cols = 2 * (uint64_t)a.nf, lanes = (uint64_t)a.n_h * cols;
    const uint64_t li = (uint64_t)n * cols + 2 * fi + warp;
    W2* ts = dts + (size_t)warp * TB;
    if ((threadIdx.x & 31) == 0) {
      mbar_init(&dbar[warp], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&dbar[warp], (uint32_t)(TB * sizeof(W2)));
      bulk_g2s(ts, a.divtape + li * (uint64_t)TB, (uint32_t)(TB * sizeof(W2)), &dbar[warp]);
    }
    if (warp == 0) hc_pre_feature<SL>(a, n, fi, Ks, pq);
    __syncthreads();  // P, qsafe of both columns (warp 0 waited for the predecessor)
    const bool tsd = a.ts && li == 0 && (threadIdx.x & 31) == 0;
    hc_ts_at(64 + 8 * a.level + 6, tsd);
    mbar_wait(&dbar[warp], 0);
    const A3 t = division_warp_staged<SL>(ts, a3(pq[warp][0][0], pq[warp][0][1], pq[warp][0][2]),
                                          a3(pq[warp][1][0], pq[warp][1][1], pq[warp][1][2]), a.d,
                                          tsd ? &g_hc_ts[8 * a.level + 7] : nullptr);
    if ((threadIdx.x & 31) == 0) st3s(a.dv + 6 * lanes, lanes, li, t);
    hc_ts_at(64 + 8 * a.level + 7, tsd);
    return;
  }
  // uniform-key chains read the round keys as constant-bank operands
  const Keys& K = a.K;
  extern __shared__ uint64_t sm[];
  const int tid = threadIdx.x;
  const int nf = a.nf, cols = 2 * nf, C3 = 3 * cols;
  const uint64_t hs = (uint64_t)a.n_h;
  uint64_t* co = sm;  // [3][3*cols] c_orig
  const uint32_t opH = op_id(a.level, SITE_HC), opR = op_id(a.level, SITE_REPLACE);
  const NodeTape NT = node_tape_plan(nf);
  const bool tsc = a.ts && n == 0 && tid == 0;
  hc_ts_at(64 + 8 * a.level + 0, tsc);
  __shared__ __align__(8) uint64_t nbar;
  W2* ntb = reinterpret_cast<W2*>(co + ((3 * C3 + 1) & ~1));
  if (a.nodetape && tid == 0) {  // the prologue + replace segments of this node's tape
    mbar_init(&nbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    mbar_expect_tx(&nbar, (uint32_t)(NT.spl * sizeof(W2)));
    bulk_g2s(ntb, a.nodetape + (uint64_t)n * NT.total, (uint32_t)(NT.spl * sizeof(W2)), &nbar);
  }
  pdl_wait();
  pdl_trigger();
  for (int e = tid; e < 3 * C3; e += blockDim.x) co[e] = co_cell(a, e / C3, n, e % C3);
  __syncthreads();
  const W2* nt = nullptr;
  if (a.nodetape) {
    mbar_wait(&nbar, 0);
    nt = ntb;
  }
  hc_ts_at(64 + 8 * a.level + 1, tsc);
  auto CO = [&](int e) { return a3(co[e], co[C3 + e], co[2 * C3 + e]); };
  if (a.co_out)  // heuristic "tee": hand the counters to the trusted helper
    for (int e = tid; e < C3; e += blockDim.x) st3s(a.co_out, hs * C3, (uint64_t)n * C3 + e, CO(e));

  if (tid < 32) {
    const int wl = tid;
    if (!a.last && !a.co_out) {
      // zeros = eq([psi0, psi1, F - LEAF], 0)                 train.py:239-245
      const A3 fl = ld3s(a.f, hs, n);
      B3 z = {{0, 0, 0}};
      if (wl < 3) {
        A3 v;
        if (wl == 0) v = add<64>(CO(cols + 0), CO(cols + 1));
        else if (wl == 1) v = add<64>(CO(2 * cols + 0), CO(2 * cols + 1));
        else v = add_pub<64>(fl, 0ull - F_LEAF);
        if (nt) {
          const W2* b = nt + 5 * wl;
          const uint64_t Zw[3] = {b[2].a, b[3].a, b[4].a};
          z = eq_arith<64>(v, b[0].a, b[0].b, b[1].a, Zw);
        } else {
          z = eqz<64>(K, opH, 0, (uint64_t)n * 3 + wl, v);
        }
      }
      B3 p0, p1, act;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        p0.v[c] = __shfl_sync(0xffffffffu, z.v[c], 0) & 1ull;
        p1.v[c] = __shfl_sync(0xffffffffu, z.v[c], 1) & 1ull;
        act.v[c] = __shfl_sync(0xffffffffu, z.v[c], 2) & 1ull;
      }
      if (wl == 0) {
        // featureless = and_reduce(~gam), leafish, should_split   train.py:246-250
        const B3 gam = ldb3s(a.gam, hs, n);
        B3 ss;
        A3 nfv;
        if (nt) {
          const uint64_t Zr[3] = {nt[15].a, nt[16].a, nt[17].a};
          const B3 fless = and_reduce_w(bnot(gam, lowmask(nf)), nf, Zr);
          const uint64_t Z2[3] = {nt[18].a & 1ull, nt[19].a & 1ull, nt[20].a & 1ull};
          const B3 o1 = bxor(bxor(p0, p1), and_z(p0, p1, Z2));
          const uint64_t Z3[3] = {nt[21].a & 1ull, nt[22].a & 1ull, nt[23].a & 1ull};
          const B3 leafish = bxor(bxor(o1, fless), and_z(o1, fless, Z3));
          const uint64_t Z4[3] = {nt[24].a & 1ull, nt[25].a & 1ull, nt[26].a & 1ull};
          ss = and_z(act, bnot(leafish, 1ull), Z4);
          nfv = select_arith<64>(nt + 27, fl, a3(0, 0, 0), ss);
        } else {
          const B3 fless = and_reduce(K, opH, 1, 0, n, bnot(gam, lowmask(nf)), nf);
          const B3 o1 = or_gate(K, opH, 2, n, p0, p1, 1ull);
          const B3 leafish = or_gate(K, opH, 3, n, o1, fless, 1ull);
          ss = and_gate(K, opH, 4, 0, n, act, bnot(leafish, 1ull), 1ull);
          nfv = select1<64>(K, opH, 5, n, fl, a3(0, 0, 0), ss);
        }
        for (int c = 0; c < 3; ++c) {
          a.hc[(0 * 3 + c) * hs + n] = ss.v[c] & 1ull;
          a.hc[(2 * 3 + c) * hs + n] = nfv.v[c];
        }
        hc_ts_at(64 + 8 * a.level + 2, tsc);
      }
    }
    return;
  }
  const int wl = tid - 32;
  // replace: empty nodes adopt the parent's effective counters  train.py:155-162
  if (a.level > 0) {
    A3 ca = a3(0, 0, 0);
    const W2* rb = nt ? nt + NT.rep : nullptr;
    if (wl == 0) {
      if (rb) {
        const uint64_t Zw[3] = {rb[2].a, rb[3].a, rb[4].a};
        const B3 hz = eq_arith<64>(add<64>(CO(0), CO(1)), rb[0].a, rb[0].b, rb[1].a, Zw);
        ca = b2a_arith<64>(hz, rb[5].a, rb[5].b, rb[6].a);
      } else {
        ca = b2a<64>(K, opR, 1, n, eqz<64>(K, opR, 0, n, add<64>(CO(0), CO(1))));
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) ca.v[c] = __shfl_sync(0xffffffffu, ca.v[c], 0);
    const uint64_t pn = (uint64_t)(n >> 1);
    for (int e = wl; e < C3; e += 32) {
      const A3 par = ld3s(a.ceff_prev, (hs / 2) * C3, pn * C3 + e);
      A3 out;
      if (rb) {
        const W2* b = rb + 7 + 3 * (e >> 1);
        const uint64_t F[3] = {(e & 1) ? b[0].b : b[0].a, (e & 1) ? b[1].b : b[1].a, (e & 1) ? b[2].b : b[2].a};
        out = add<64>(CO(e), mul_z<64>(diff<64>(par, CO(e)), ca, F));
      } else {
        out = select_with<64>(K, opR, 1, (uint32_t)e, n, CO(e), par, ca);
      }
      st3s(a.ceff, hs * C3, (uint64_t)n * C3 + e, out);
    }
  } else {
    for (int e = wl; e < C3; e += 32) st3s(a.ceff, hs * C3, (uint64_t)n * C3 + e, CO(e));
  }
}

constexpr int DIV_WARPS = 4;  // at most; fewer when the tape is large (score ring Z_2^64)

template <int SL>
__global__ void __launch_bounds__(32 * DIV_WARPS) k_hc_div(NodeArgs a) {
  extern __shared__ __align__(128) W2 tape_sm[];
  const int warp = threadIdx.x >> 5, wpc = blockDim.x >> 5;
  const uint64_t cols = 2 * (uint64_t)a.nf, lanes = (uint64_t)a.n_h * cols;
  const uint64_t li = (uint64_t)blockIdx.x * wpc + warp;
  if (li >= lanes) return;  // whole warp exits together
  hc_ts_at(64 + 8 * a.level + 6, a.ts && li == 0 && threadIdx.x == 0);
  // terms = division(P, qsafe)                              train.py:268
  A3 t;
  if (a.divtape) {
    // the lane's whole precomputed tape (ladder + Newton) comes in by one bulk
    // copy, so neither chain waits on global memory
    __shared__ __align__(8) uint64_t bar[DIV_WARPS];
    const int TB = div_tape_blocks<SL>(a.d);
    W2* ts = tape_sm + (size_t)warp * TB;
    if ((threadIdx.x & 31) == 0) {
      mbar_init(&bar[warp], 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&bar[warp], (uint32_t)(TB * sizeof(W2)));
      bulk_g2s(ts, a.divtape + li * (uint64_t)TB, (uint32_t)(TB * sizeof(W2)), &bar[warp]);
    }
    __syncwarp();
    pdl_wait();
    pdl_trigger();
    const A3 p = ld3s(a.dv, lanes, li), q = ld3s(a.dv + 3 * lanes, lanes, li);
    mbar_wait(&bar[warp], 0);
    t = division_warp_staged<SL>(ts, p, q, a.d);
  } else {
    pdl_wait();
    pdl_trigger();
    const A3 p = ld3s(a.dv, lanes, li), q = ld3s(a.dv + 3 * lanes, lanes, li);
    t = division_warp<SL>(a.K, op_id(a.level, SITE_HC), 13, li, p, q, a.d, tape_sm + (size_t)warp * division_tape_blocks<SL>(a.d));
  }
  if ((threadIdx.x & 31) == 0) st3s(a.dv + 6 * lanes, lanes, li, t);
  hc_ts_at(64 + 8 * a.level + 7, a.ts && li == 0 && threadIdx.x == 0);
}

// All division blocks of every heuristic level (see DivTape).  A per-lane
// schedule table (block -> key, sub, Philox block index; identical for every
// lane) is built once, then one thread per (lane, block) draws its block;
// level h's lanes start at (2^h - 1) * cols.
template <int SL>
__global__ void k_div_table(uint32_t* table, DivParams d) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= div_tape_blocks<SL>(d)) return;
  constexpr int LS = DivTape<SL>::LADDER_STEP, LB = LtRand<SL>::BLOCKS;
  const int nl = d.bound - 1;
  int key = -1;
  uint32_t sub = 0, pidx = 0;  // sub relative to the division's first sub
  if (b < nl * LS) {
    const int j = b / LS, w = b % LS;
    if (w < LB) {
      lt_block_id<SL>(w, 0, &key, &pidx);
      sub = j;
    } else {
      sub = nl + j, pidx = w - LB;
    }
  } else {
    int r = b - nl * LS;
    for (int i = 0; i < newton_steps<SL>(d); ++i) {
      const ChainStep c = newton_step<SL>(i, d);
      const int nb = step_blocks<SL>(c);
      if (r < nb) {
        const uint32_t s0 = 2 * nl + c.sub_off;
        if (c.is_trunc) {
          trunc_block_id<SL>(r, s0, &key, &sub, &pidx);
        } else {
          key = r, sub = s0, pidx = 0;
        }
        break;
      }
      r -= nb;
    }
  }
  table[b] = (sub << 16) | (pidx << 8) | (uint32_t)(key + 1);
}

constexpr int DIV_TAPE_PER = 4;  // blocks per thread of k_div_tape
template <int SL>
__global__ void __launch_bounds__(256) k_div_tape(W2* tape, const uint32_t* __restrict__ table, uint64_t total,
                                                   int cols, int TB, Keys K) {
  // the lanes of a warp draw with different keys: index the round keys in
  // shared memory (a dynamically indexed kernel parameter serialises)
  __shared__ Keys ks;
  for (int i = threadIdx.x; i < (int)(sizeof(Keys) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&ks)[i] = reinterpret_cast<const uint32_t*>(&K)[i];
  __syncthreads();
  // 32-bit index math: the tape is capped at 256 MB (< 2^24 blocks).  Each
  // thread draws DIV_TAPE_PER blocks 32 apart (a warp writes 32 consecutive
  // blocks per store; independent Philox chains in flight together; one index
  // decomposition, then a carry per block)
  const uint32_t lane = threadIdx.x & 31, wg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint32_t e = wg * 32 * DIV_TAPE_PER + lane;
  if (e >= total) return;
  uint32_t g = e / (uint32_t)TB, b = e - g * (uint32_t)TB;
  uint32_t tt[DIV_TAPE_PER], gg[DIV_TAPE_PER];
#pragma unroll
  for (int k = 0; k < DIV_TAPE_PER; ++k) {
    gg[k] = g;
    tt[k] = e + 32 * k < total ? __ldg(table + b) : 0u;
    b += 32;
    while (b >= (uint32_t)TB) b -= (uint32_t)TB, ++g;
  }
#pragma unroll
  for (int k = 0; k < DIV_TAPE_PER; ++k, e += 32) {
    if (e >= total) break;
    const uint32_t nodes = gg[k] / (uint32_t)cols;
    const int level = 31 - __clz(nodes + 1);  // nodes in [2^h - 1, 2^{h+1} - 1)
    const uint64_t li = gg[k] - ((1u << level) - 1) * (uint32_t)cols;
    const uint32_t t = tt[k];
    const int key = (int)(t & 0xff) - 1;
    tape[e] = word2(key < 0 ? ks.dealer : ks.pair[key], op_id(level, SITE_HC), 13 + (t >> 16), (t >> 8) & 0xff, li);
  }
}

// hc_post_body's shared scratch in words: vals/idxs/nvals/nidxs [3][nf], hit
// words, then the per-warp live-draw tapes (8 warps), 16-byte aligned
__host__ __device__ inline int post_scratch_words(int nf) {
  return ((12 * nf + 4) + 2 * 8 * (LtRand<64>::BLOCKS + 10) + 1) & ~1;
}

// ---------------------------------------------------------------------------
// Precomputed randomness of the heuristic epilogue (scores' mask selects, the
// argmin tournament, the budget-clear eqs and AND): one node's blocks, in the
// order hc_post_body consumes them, are identical in structure for every
// node (only the lanes move), so like the division tapes they are drawn for
// every level up front and each node's CTA stages its run with one bulk copy.
//   [scores: nf x (b2a 2 + mul 3)] [rounds r, pairs p: 62 = lt 52 + 2 selects]
//   [budget: nf x eqz 5] [and: 3]
// Entry: key+1 (8 bits) | pidx (8) | sub (16) | lane index (16) | lane kind (8:
// 0 = n*nf + index, 1 = n).
template <int SL>
__host__ __device__ inline int post_rounds_blocks(int nf) {
  int m = nf, b = 0;
  while (m > 1) {
    b += (m / 2) * ArgminPair<SL>::BLOCKS;
    m = m / 2 + (m & 1);
  }
  return b;
}
template <int SL>
__host__ __device__ inline int post_tape_blocks(int nf) { return 5 * nf + post_rounds_blocks<SL>(nf) + 5 * nf + 3; }
__host__ __device__ inline int post_tape_blocks_w(int width, int nf) {
  return width == 32 ? post_tape_blocks<32>(nf) : post_tape_blocks<64>(nf);
}

template <int SL>
__global__ void k_post_table(uint64_t* table, int nf, uint32_t SA) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= post_tape_blocks<SL>(nf)) return;
  constexpr int PB = ArgminPair<SL>::BLOCKS;
  const uint32_t SH = SA + 2 + 5 * 7;
  int key = -1, idx = 0, kind = 0;
  uint32_t sub = 0, pidx = 0;
  int b = e;
  if (b < 5 * nf) {  // score mask select (select1 at SA)
    idx = b / 5;
    select_block_id(b % 5, SA, &key, &sub, &pidx);
  } else if ((b -= 5 * nf) < post_rounds_blocks<SL>(nf)) {
    int m = nf, r = 0;
    while (b >= (m / 2) * PB) {
      b -= (m / 2) * PB;
      m = m / 2 + (m & 1);
      ++r;
    }
    const uint32_t base = SA + 2 + 5 * r;
    idx = b / PB;
    const int j = b % PB;
    constexpr int LB = LtRand<SL>::BLOCKS;
    if (j < LB) {
      lt_block_id<SL>(j, base, &key, &pidx);
      sub = base;
    } else if (j < LB + 5) {
      select_block_id(j - LB, base + 1, &key, &sub, &pidx);
    } else {
      select_block_id(j - LB - 5, base + 3, &key, &sub, &pidx);
    }
  } else if ((b -= post_rounds_blocks<SL>(nf)) < 5 * nf) {  // budget eqz at SH
    idx = b / 5;
    const int w = b % 5;
    sub = SH;
    if (w < 2) key = -1, pidx = w;
    else key = w - 2, pidx = 0;
  } else {  // and_gate at SH+1, field 0, lane n
    b -= 5 * nf;
    key = b, sub = SH + 1, pidx = 0, kind = 1;
  }
  table[e] = (uint64_t)(uint32_t)(key + 1) | ((uint64_t)pidx << 8) | ((uint64_t)sub << 16) | ((uint64_t)idx << 32) |
             ((uint64_t)kind << 48);
}

// every level's epilogue tape: [level][node][post_tape_blocks]; one thread per block
__global__ void __launch_bounds__(256) k_post_tape(W2* tape, const uint64_t* __restrict__ table, uint32_t total,
                                                   int nf, int E, Keys K) {
  __shared__ Keys ks;
  for (int i = threadIdx.x; i < (int)(sizeof(Keys) / 4); i += blockDim.x)
    reinterpret_cast<uint32_t*>(&ks)[i] = reinterpret_cast<const uint32_t*>(&K)[i];
  __syncthreads();
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= total) return;
  const uint32_t gn = e / (uint32_t)E;  // global node = (2^level - 1) + n
  const uint64_t t = __ldg(table + (e - gn * (uint32_t)E));
  const int level = 31 - __clz(gn + 1);
  const uint32_t n = gn - ((1u << level) - 1);
  const int key = (int)(t & 0xff) - 1, kind = (int)((t >> 48) & 0xff);
  const uint32_t pidx = (uint32_t)((t >> 8) & 0xff), sub = (uint32_t)((t >> 16) & 0xffff);
  const uint64_t lane = kind ? (uint64_t)n : (uint64_t)n * nf + (uint32_t)((t >> 32) & 0xffff);
  tape[e] = word2(key < 0 ? ks.dealer : ks.pair[key], op_id(level, SITE_HC), sub, pidx, lane);
}

// What the fused post/split kernel takes over after the argmin: the budget
// clear then runs beside the split chains (see k_hc_post_finish).
struct PostOut {
  A3 sd;
  B3 gam;
  const W2* pb;     // staged budget blocks (or null: draw live)
  uint64_t* hitw;   // [3] shared-memory hit words, zeroed
  uint32_t opH, SH;
};

template <int SL>
__device__ __forceinline__ void hc_post_body(const NodeArgs& a, int n, PostOut* out = nullptr) {
  extern __shared__ uint64_t sm[];
  constexpr uint64_t MS = Ring<SL>::M;
  const int tid = threadIdx.x, bd = blockDim.x;
  const int nf = a.nf, cols = 2 * nf;
  const uint64_t hs = (uint64_t)a.n_h, lanes = hs * cols;
  uint64_t* vals = sm;  // [3][nf]
  uint64_t* idxs = vals + 3 * nf;
  uint64_t* nvals = idxs + 3 * nf;
  uint64_t* nidxs = nvals + 3 * nf;
  uint64_t* hitw = nidxs + 3 * nf;  // [3]
  __shared__ Keys ks;
  const Keys& Ks = keys_smem(a.K, ks);  // lane-dependent keys of the tournament tapes
  const Keys& K = a.K;                  // uniform-key gadgets: constant-bank operands
  const uint32_t opH = op_id(a.level, SITE_HC);
  const uint64_t* terms = a.dv + 6 * lanes;
  auto TM = [&](int k) { return ld3s(terms, lanes, (uint64_t)n * cols + k); };
  // staged epilogue tape (see k_post_table): one bulk copy of this node's run,
  // issued before the wait for the division kernel
  const W2* pt = nullptr;
  __shared__ __align__(8) uint64_t pbar;
  if (a.posttape) {
    W2* pts = reinterpret_cast<W2*>(sm + post_scratch_words(nf));
    const int E = post_tape_blocks<SL>(nf);
    if (tid == 0) {
      mbar_init(&pbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&pbar, (uint32_t)(E * sizeof(W2)));
      bulk_g2s(pts, a.posttape + (uint64_t)n * E, (uint32_t)(E * sizeof(W2)), &pbar);
    }
    pt = pts;
  }
  pdl_wait();
  pdl_trigger();
  const B3 gam = ldb3s(a.gam, hs, n);
  if (pt) {
    __syncthreads();
    mbar_wait(&pbar, 0);
  }
  // scores + masked argmin (tournament)     train.py:269-271, gadgets.py:366-401
  hc_ts(0 + 8 * a.level, a.ts);
  const uint32_t SA = 13 + div_subs(a.d);
  const uint64_t worst = (1ull << (a.tau + 1)) & MS;
  for (int i = tid; i < nf; i += bd) {
    const A3 score = add<SL>(TM(2 * i), TM(2 * i + 1));
    B3 av;
    for (int c = 0; c < 3; ++c) av.v[c] = (gam.v[c] >> i) & 1ull;
    const A3 v = pt ? select_arith<SL>(pt + 5 * i, a3_const(worst), score, av)
                    : select1<SL>(K, opH, SA, (uint64_t)n * nf + i, a3_const(worst), score, av);
    for (int c = 0; c < 3; ++c) {
      vals[c * nf + i] = v.v[c];
      idxs[c * nf + i] = c == 0 ? (uint64_t)i : 0ull;
    }
  }
  if (tid < 3) hitw[tid] = 0;
  __syncthreads();
  int m = nf;
  const int warp = tid >> 5, nwarps = bd >> 5;
  W2* tape = reinterpret_cast<W2*>(hitw + 4) + warp * ArgminPair<SL>::BLOCKS;
  hc_ts(1 + 8 * a.level, a.ts);
  int roff = 5 * nf;  // this round's first block in the staged tape
  // ping-pong buffers: round r reads (vals, idxs) and writes (nvals, nidxs),
  // then the two swap
  uint64_t *cv = vals, *ci = idxs, *nv_ = nvals, *ni_ = nidxs;
  for (int r = 0; m > 1; ++r) {
    const int pairs = m / 2;
    const uint32_t base = SA + 2 + 5 * r;
    uint64_t *vals = cv, *idxs = ci, *nvals = nv_, *nidxs = ni_;
    for (int p = warp; p < pairs; p += nwarps) {  // one warp per tournament pair
      const uint64_t lane = (uint64_t)n * nf + p;
      const A3 av = a3(vals[2 * p], vals[nf + 2 * p], vals[2 * nf + 2 * p]);
      const A3 bv = a3(vals[2 * p + 1], vals[nf + 2 * p + 1], vals[2 * nf + 2 * p + 1]);
      const A3 ai = a3(idxs[2 * p], idxs[nf + 2 * p], idxs[2 * nf + 2 * p]);
      const A3 bi = a3(idxs[2 * p + 1], idxs[nf + 2 * p + 1], idxs[2 * nf + 2 * p + 1]);
      A3 nv, ni;
      if (pt) {
        const W2* b = pt + roff + ArgminPair<SL>::BLOCKS * p;
        constexpr int LB = LtRand<SL>::BLOCKS;
        const B3 cw = lt_arith_warp<SL>(b, bv, av);  // challenger wins iff b < a
        nv = select_arith<SL>(b + LB, av, bv, cw);
        ni = select_arith<64>(b + LB + 5, ai, bi, cw);
      } else {
        argmin_pair_warp<SL>(Ks, opH, base, lane, av, bv, ai, bi, tape, &nv, &ni);
      }
      if ((tid & 31) == 0)
        for (int c = 0; c < 3; ++c) {
          nvals[c * nf + p] = nv.v[c];
          nidxs[c * nf + p] = ni.v[c];
        }
    }
    if (tid == 0 && (m & 1))
      for (int c = 0; c < 3; ++c) {
        nvals[c * nf + pairs] = vals[c * nf + m - 1];
        nidxs[c * nf + pairs] = idxs[c * nf + m - 1];
      }
    __syncthreads();
    roff += ArgminPair<SL>::BLOCKS * pairs;
    m = pairs + (m & 1);
    cv = nvals, ci = nidxs, nv_ = vals, ni_ = idxs;
  }
  hc_ts(2 + 8 * a.level, a.ts);
  const A3 sd = a3(ci[0], ci[nf], ci[2 * nf]);
  // gamma &= ~[sd == k]                                     train.py:272-273
  const uint32_t SH = SA + 2 + 5 * 7;
  const W2* pb = pt ? pt + 5 * nf + post_rounds_blocks<SL>(nf) : nullptr;  // budget blocks
  if (out) {  // the caller runs the budget clear beside the split
    out->sd = sd, out->gam = gam, out->pb = pb, out->hitw = hitw, out->opH = opH, out->SH = SH;
    return;
  }
  // lane f = tid (nf <= 64 <= blockDim): hit bits by warp ballots
  __shared__ uint32_t hbw[2][3];
  if (tid < 64) {
    B3 h = {{0, 0, 0}};
    const int f = tid;
    if (f < nf) {
      if (pb) {
        const W2* b = pb + 5 * f;
        const uint64_t Zw[3] = {b[2].a, b[3].a, b[4].a};
        h = eq_arith<64>(add_pub<64>(sd, 0ull - (uint64_t)f), b[0].a, b[0].b, b[1].a, Zw);
      } else {
        h = eqz<64>(K, opH, SH, (uint64_t)n * nf + f, add_pub<64>(sd, 0ull - (uint64_t)f));
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const uint32_t bits = __ballot_sync(0xffffffffu, (uint32_t)(h.v[c] & 1ull));
      if ((tid & 31) == 0) hbw[tid >> 5][c] = bits;
    }
  }
  __syncthreads();
  if (tid == 0) {
    B3 hw;
    for (int c = 0; c < 3; ++c) hw.v[c] = (uint64_t)hbw[0][c] | ((uint64_t)hbw[1][c] << 32);
    B3 ng;
    if (pb) {
      const W2* b = pb + 5 * nf;
      const uint64_t Z[3] = {b[0].a & lowmask(nf), b[1].a & lowmask(nf), b[2].a & lowmask(nf)};
      ng = and_z(gam, bnot(hw, lowmask(nf)), Z);
    } else {
      ng = and_gate(K, opH, SH + 1, 0, n, gam, bnot(hw, lowmask(nf)), lowmask(nf));
    }
    for (int c = 0; c < 3; ++c) {
      a.hc[(1 * 3 + c) * hs + n] = sd.v[c];
      a.hc[(3 * 3 + c) * hs + n] = ng.v[c];
    }
  }
}

template <int SL>
__global__ void __launch_bounds__(256) k_hc_post(NodeArgs a) {
  hc_post_body<SL>(a, blockIdx.x);
}

// grow policy: all_declined = open(and_reduce(~is_int over nodes)) (train.py:164-168,
// and_reduce gadgets.py:94-109).  One CTA, the level's n_h bit planes per
// component in shared memory; level with k planes ANDs plane j with plane
// j + k/2 (odd last plane carried).  Gate g (counted over all levels) draws
// zero bit g & 63 of pair word (sub 0, field g >> 6, lane 0) -- for n_h <= 64
// exactly the in-word and_reduce schedule.
__global__ void __launch_bounds__(256) k_node_stop(const uint64_t* hc, int n_h, Keys K, uint32_t op, uint64_t* out) {
  extern __shared__ uint8_t planes[];  // [2][3][n_h]
  uint8_t* cur = planes;
  uint8_t* nxt = planes + 3 * n_h;
  for (int n = threadIdx.x; n < n_h; n += blockDim.x)
#pragma unroll
    for (int c = 0; c < 3; ++c) cur[c * n_h + n] = (uint8_t)((hc[c * (uint64_t)n_h + n] & 1ull) ^ (c == 0));  // bnot
  __syncthreads();
  int k = n_h, off = 0;
  while (k > 1) {
    const int half = k >> 1;
    for (int j = threadIdx.x; j < half; j += blockDim.x) {
      const int g = off + j;
      uint8_t z[3], a[3], b[3];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        z[i] = (uint8_t)((word(K.pair[i], op, 0, (uint32_t)(g >> 6), 0) >> (g & 63)) & 1ull);
        a[i] = cur[i * n_h + j];
        b[i] = cur[i * n_h + j + half];
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int q = (i + 1) % 3, p = (i + 2) % 3;
        nxt[i * n_h + j] = (a[i] & b[i]) ^ (a[q] & b[i]) ^ (a[i] & b[q]) ^ z[i] ^ z[p];
      }
    }
    if ((k & 1) && threadIdx.x == 0)
#pragma unroll
      for (int i = 0; i < 3; ++i) nxt[i * n_h + half] = cur[i * n_h + k - 1];
    __syncthreads();
    uint8_t* t = cur;
    cur = nxt;
    nxt = t;
    off += half;
    k = half + (k & 1);
  }
  if (threadIdx.x == 0) out[0] = (cur[0] ^ cur[n_h] ^ cur[2 * n_h]) & 1;  // open_bits
}

struct FinishArgs {
  const uint64_t* hc;      // [4][3][n_h]
  const uint64_t* ceff;    // [3][n_h][3][cols]
  const uint64_t* f;       // [3][n_h]
  const uint64_t* filler;  // public [slots]
  uint64_t *T, *F;         // [3][slots]
  uint64_t *f_nxt, *gam_nxt, *cst_nxt;  // children
  const uint64_t* lab;                  // [3][n_h] helper labels (heuristic tee) or null
  uint64_t slots;
  int n_h, nf, level, labels, ts;
  const W2* nodetape;  // precomputed node-chain blocks of this level's nodes (or null: draw live)
  Keys K;
};

__device__ __forceinline__ void node_finish_body(const FinishArgs& a, int n) {
  __shared__ uint64_t ca[3];
  const int tid = threadIdx.x, bd = blockDim.x;
  const int cols = 2 * a.nf, C3 = 3 * cols;
  const uint64_t hs = (uint64_t)a.n_h, slot = hs - 1 + n;
  const Keys& K = a.K;
  hc_ts(5 + 8 * a.level, a.ts);
  auto CE = [&](int e) { return ld3s(a.ceff, hs * C3, (uint64_t)n * C3 + e); };
  // this node's split (or labels) segment of the precomputed node tape
  const NodeTape NT = node_tape_plan(a.nf);
  __shared__ __align__(128) W2 nsb[16 + 12 + 3 * 64 * 3 + LtRand<64>::BLOCKS];  // >= max segment
  __shared__ __align__(8) uint64_t nbar;
  const W2* nt = nullptr;
  if (a.nodetape && !(a.labels && a.lab)) {
    const int off = a.labels ? NT.lab : NT.spl, len = a.labels ? NT.total - NT.lab : NT.lab - NT.spl;
    nt = stage_node_tape(a.nodetape + (uint64_t)n * NT.total + off, len, nsb, &nbar);
  }
  if (a.labels && a.lab) {  // labels from the trusted helper (train.py:187-188)
    if (tid == 0) {
      st3s(a.T, a.slots, slot, ld3s(a.lab, hs, n));
      st3s(a.F, a.slots, slot, ld3s(a.f, hs, n));
    }
    return;
  }
  if (a.labels) {
    // labels = b2a(lt(psi0, psi1)) on effective counters      train.py:186-192
    if (tid < 32) {  // warp 0 (the staged lt pairs its operands on neighbouring lanes)
      const uint32_t op = op_id(a.level, SITE_LABELS);
      const A3 psi0 = add<64>(CE(cols), CE(cols + 1)), psi1 = add<64>(CE(2 * cols), CE(2 * cols + 1));
      constexpr int LB = LtRand<64>::BLOCKS;
      const A3 lab = nt ? b2a_arith<64>(lt_arith_warp<64>(nt, psi0, psi1), nt[LB].a, nt[LB].b, nt[LB + 1].a)
                        : b2a<64>(K, op, 1, n, lt<64>(K, op, 0, n, psi0, psi1));
      if (tid == 0) {
        st3s(a.T, a.slots, slot, lab);
        st3s(a.F, a.slots, slot, ld3s(a.f, hs, n));
      }
    }
    return;
  }
  const uint32_t op = op_id(a.level, SITE_SPLIT);
  B3 ss;
  for (int c = 0; c < 3; ++c) ss.v[c] = a.hc[(0 * 3 + c) * hs + n];
  const uint64_t cs = 2 * hs;  // children per level
  // the three selects of split:h are independent chains: one per warp
  if (tid == 0) {  // payload T = is_int ? sd : filler        (train.py:173)
    const A3 sd = ld3s(a.hc + 3 * hs, hs, n);
    const uint64_t fl = a.filler[slot];
    const A3 cb = nt ? a3(0, 0, 0) : b2a<64>(K, op, 0, n, ss);
    st3s(a.T, a.slots, slot, nt ? select_arith<64>(nt, a3_const(fl), sd, ss)
                                : select_with<64>(K, op, 0, 0, n, a3_const(fl), sd, cb));
    st3s(a.F, a.slots, slot, ld3s(a.hc + 6 * hs, hs, n));
  } else if (tid == 32) {  // child type = is_int ? LEAF : DUMMY  (train.py:174-175)
    const A3 cf = nt ? select_arith<64>(nt + 5, a3_const(F_DUMMY), a3_const(F_LEAF), ss)
                     : select_with<64>(K, op, 2, 0, n, a3_const(F_DUMMY), a3_const(F_LEAF), b2a<64>(K, op, 2, n, ss));
    const A3 ng = ld3s(a.hc + 9 * hs, hs, n);
    for (int ch = 0; ch < 2; ++ch) {
      st3s(a.f_nxt, cs, 2 * n + ch, cf);
      st3s(a.gam_nxt, cs, 2 * n + ch, ng);
    }
  } else if (tid == 64) {  // child counters' condition
    const A3 c2 = nt ? b2a_arith<64>(ss, nt[10].a, nt[10].b, nt[11].a) : b2a<64>(K, op, 4, n, ss);
    for (int c = 0; c < 3; ++c) ca[c] = c2.v[c];
  }
  __syncthreads();
  hc_ts(6 + 8 * a.level, a.ts);
  // child counters = select(c_eff, 0, is_int)                 train.py:176
  const A3 cav = a3(ca[0], ca[1], ca[2]);
  for (int e = tid; e < C3; e += bd) {
    A3 cc;
    if (nt) {
      const W2* b = nt + 12 + 3 * (e >> 1);
      const uint64_t F[3] = {(e & 1) ? b[0].b : b[0].a, (e & 1) ? b[1].b : b[1].a, (e & 1) ? b[2].b : b[2].a};
      cc = add<64>(CE(e), mul_z<64>(diff<64>(a3(0, 0, 0), CE(e)), cav, F));
    } else {
      cc = select_with<64>(K, op, 4, (uint32_t)e, n, CE(e), a3(0, 0, 0), cav);
    }
    for (int ch = 0; ch < 2; ++ch) st3s(a.cst_nxt, cs * C3, (uint64_t)(2 * n + ch) * C3 + e, cc);
  }
}

__global__ void __launch_bounds__(128) k_node_finish(FinishArgs a) {
  pdl_wait();
  pdl_trigger();
  node_finish_body(a, blockIdx.x);
}

// scores / argmin / budget clear, then split, in one launch per level (fixed
// policy, mpc heuristic): the node's CTA continues from sd to its children
// Budget clear (gamma &= ~[sd == k], train.py:272-273) on warps 0-1 while
// warps 4-6 run the split's three independent chains (payload, child type,
// child-counter condition, train.py:173-176); the children's gamma is stored
// after the join.  Same gadgets and blocks as the sequential path.
template <int SL>
__device__ __forceinline__ void post_split_fused(const NodeArgs& na, const FinishArgs& a, int n, const PostOut& po,
                                                 const W2* nt_staged, uint64_t* nbar) {
  __shared__ uint64_t ca[3], ngs[3];
  const int tid = threadIdx.x, bd = blockDim.x, warp = tid >> 5;
  const int nf = a.nf, cols = 2 * nf, C3 = 3 * cols;
  const uint64_t hs = (uint64_t)a.n_h, slot = hs - 1 + n, cs = 2 * hs;
  const Keys& K = a.K;
  const uint32_t op = op_id(a.level, SITE_SPLIT);
  auto CE = [&](int e) { return ld3s(a.ceff, hs * C3, (uint64_t)n * C3 + e); };
  // the split segment of the node tape was bulk-copied at kernel start
  const W2* nt = nullptr;
  if (nt_staged) {
    mbar_wait(nbar, 0);
    nt = nt_staged;
  }
  // this thread's effective counters, loaded while the chains run
  A3 ce = a3(0, 0, 0);
  if (tid < C3) ce = CE(tid);
  B3 ss;
  for (int c = 0; c < 3; ++c) ss.v[c] = a.hc[(0 * 3 + c) * hs + n];
  hc_ts(3 + 8 * a.level, a.ts);  // budget and split start together (slots 3, 5)
  hc_ts(5 + 8 * a.level, a.ts);
  if (warp < 2) {
    // lane f = tid (nf <= 64): the hit bits gather by warp ballots (no
    // contended shared-memory atomics)
    __shared__ uint32_t hb[2][3];
    B3 h = {{0, 0, 0}};
    const int f = tid;
    if (f < nf) {
      if (po.pb) {
        const W2* b = po.pb + 5 * f;
        const uint64_t Zw[3] = {b[2].a, b[3].a, b[4].a};
        h = eq_arith<64>(add_pub<64>(po.sd, 0ull - (uint64_t)f), b[0].a, b[0].b, b[1].a, Zw);
      } else {
        h = eqz<64>(K, po.opH, po.SH, (uint64_t)n * nf + f, add_pub<64>(po.sd, 0ull - (uint64_t)f));
      }
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const uint32_t bits = __ballot_sync(0xffffffffu, (uint32_t)(h.v[c] & 1ull));
      if ((tid & 31) == 0) hb[warp][c] = bits;
    }
    asm volatile("bar.sync 2, 64;" ::: "memory");
    if (tid == 0) {
      B3 hw;
      for (int c = 0; c < 3; ++c) hw.v[c] = (uint64_t)hb[0][c] | ((uint64_t)hb[1][c] << 32);
      B3 ng;
      if (po.pb) {
        const W2* b = po.pb + 5 * nf;
        const uint64_t Z[3] = {b[0].a & lowmask(nf), b[1].a & lowmask(nf), b[2].a & lowmask(nf)};
        ng = and_z(po.gam, bnot(hw, lowmask(nf)), Z);
      } else {
        ng = and_gate(K, po.opH, po.SH + 1, 0, n, po.gam, bnot(hw, lowmask(nf)), lowmask(nf));
      }
      for (int c = 0; c < 3; ++c) {
        na.hc[(1 * 3 + c) * hs + n] = po.sd.v[c];
        na.hc[(3 * 3 + c) * hs + n] = ng.v[c];
        ngs[c] = ng.v[c];
      }
    }
  } else if (tid == 128) {  // payload T = is_int ? sd : filler        (train.py:173)
    const uint64_t fl = a.filler[slot];
    const A3 cb = nt ? a3(0, 0, 0) : b2a<64>(K, op, 0, n, ss);
    st3s(a.T, a.slots, slot, nt ? select_arith<64>(nt, a3_const(fl), po.sd, ss)
                                : select_with<64>(K, op, 0, 0, n, a3_const(fl), po.sd, cb));
    st3s(a.F, a.slots, slot, ld3s(a.hc + 6 * hs, hs, n));
  } else if (tid == 160) {  // child type = is_int ? LEAF : DUMMY  (train.py:174-175)
    const A3 cf = nt ? select_arith<64>(nt + 5, a3_const(F_DUMMY), a3_const(F_LEAF), ss)
                     : select_with<64>(K, op, 2, 0, n, a3_const(F_DUMMY), a3_const(F_LEAF), b2a<64>(K, op, 2, n, ss));
    for (int ch = 0; ch < 2; ++ch) st3s(a.f_nxt, cs, 2 * n + ch, cf);
  } else if (tid == 192) {  // child counters' condition
    const A3 c2 = nt ? b2a_arith<64>(ss, nt[10].a, nt[10].b, nt[11].a) : b2a<64>(K, op, 4, n, ss);
    for (int c = 0; c < 3; ++c) ca[c] = c2.v[c];
  }
  __syncthreads();
  hc_ts(6 + 8 * a.level, a.ts);
  if (tid < 2)  // children's budget
    st3s(a.gam_nxt, cs, 2 * n + tid, a3(ngs[0], ngs[1], ngs[2]));
  // child counters = select(c_eff, 0, is_int)                 train.py:176
  const A3 cav = a3(ca[0], ca[1], ca[2]);
  for (int e = tid; e < C3; e += bd) {
    const A3 cev = e == tid ? ce : CE(e);
    A3 cc;
    if (nt) {
      const W2* b = nt + 12 + 3 * (e >> 1);
      const uint64_t F[3] = {(e & 1) ? b[0].b : b[0].a, (e & 1) ? b[1].b : b[1].a, (e & 1) ? b[2].b : b[2].a};
      cc = add<64>(cev, mul_z<64>(diff<64>(a3(0, 0, 0), cev), cav, F));
    } else {
      cc = select_with<64>(K, op, 4, (uint32_t)e, n, cev, a3(0, 0, 0), cav);
    }
    for (int ch = 0; ch < 2; ++ch) st3s(a.cst_nxt, cs * C3, (uint64_t)(2 * n + ch) * C3 + e, cc);
  }
}

template <int SL>
__global__ void __launch_bounds__(256) k_hc_post_finish(NodeArgs na, FinishArgs fa) {
  static constexpr bool kFusedBudget = true;
  if (kFusedBudget && blockDim.x >= 256 && na.nf <= 64) {
    // the split segment of the node tape (data-independent) starts coming in
    // now, beside the epilogue tape, before the wait for the division
    __shared__ __align__(128) W2 nsb[16 + 12 + 3 * 64 * 3];  // >= the split segment
    __shared__ __align__(8) uint64_t nbar;
    const NodeTape NT = node_tape_plan(fa.nf);
    if (fa.nodetape && threadIdx.x == 0) {
      const int len = NT.lab - NT.spl;
      mbar_init(&nbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      mbar_expect_tx(&nbar, (uint32_t)(len * sizeof(W2)));
      bulk_g2s(nsb, fa.nodetape + (uint64_t)blockIdx.x * NT.total + NT.spl, (uint32_t)(len * sizeof(W2)), &nbar);
    }
    PostOut po;
    hc_post_body<SL>(na, blockIdx.x, &po);  // its barriers order the mbarrier init before any wait
    post_split_fused<SL>(na, fa, blockIdx.x, po, fa.nodetape ? nsb : nullptr, &nbar);
    __syncthreads();
    hc_ts(4 + 8 * na.level, na.ts);
    return;
  }
  hc_post_body<SL>(na, blockIdx.x);
  hc_ts(3 + 8 * na.level, na.ts);
  __syncthreads();  // hc[sd], hc[new_gam] of this node written by thread 0
  node_finish_body(fa, blockIdx.x);
  __syncthreads();
  hc_ts(4 + 8 * na.level, na.ts);
}

// ---------------------------------------------------------------------------
// workspace
// ---------------------------------------------------------------------------

// Node blocking, chunking and tiling of one level's count (shared by the
// workspace layout and the launches).
struct CountPlan {
  int W, WC, CT, nb, nbp, nblk, ts, R, P;
};
CountPlan count_plan(int nf, int n_h) {
  CountPlan p;
  p.W = 2 * nf + 1;
  p.WC = (p.W + 1 + CNT_CB - 1) / CNT_CB * CNT_CB;
  p.CT = p.WC / CNT_CB;
  // node block: as many nodes as keep the (node pair, column tile) items <= one CTA
  const int nb_max = std::max(CNT_NA, (CNT_TPB / p.CT) * CNT_NA);
  p.nblk = (n_h + nb_max - 1) / nb_max;
  p.nb = (n_h + p.nblk - 1) / p.nblk;
  p.nbp = (p.nb + 1) & ~1;
  p.P = (p.nbp / CNT_NA) * p.CT;
  p.R = std::max(1, CNT_TPB / p.P);
  // tile: ~8 samples per replica, two stages within ~200 KB of shared memory
  int ts = std::max(32, std::min(256, (8 * p.R + 7) / 8 * 8));
  while (ts > 8 && 2 * 3 * ts * (p.nbp + p.WC) * 8 > 200 * 1024) ts -= 8;
  p.ts = ts;
  return p;
}
// la chunk capacity (words): keeps a chunk's lanes L2-resident between the
// lane and contraction kernels, but never below 4096 samples per chunk
uint64_t la_words(uint64_t N, int nf, int depth) {
  const CountPlan p = count_plan(nf, 1 << (depth - 1));
  const uint64_t per = 3ull * p.nblk * p.nbp;
  const uint64_t want = std::max<uint64_t>(8ull << 20, per * 4096);
  return std::min<uint64_t>(want, per * std::max<uint64_t>(N, 1));
}

// la8 chunk capacity in 128-sample blocks (tensor engine): ~256 MB of byte
// planes at the deepest level, at least one block, at most the shard
uint64_t tc_la8_blocks(uint64_t N, int nf, int depth) {
  const TcPlan tp = tc_plan(nf, 1 << (depth - 1));
  const uint64_t per_blk = 3ull * tp.mtiles * TC_ABLK;
  const uint64_t nkb = std::max<uint64_t>(1, (N + TC_KB - 1) / TC_KB);
  // 256 MB per buffer: a C2 level is one chunk; at C4 fewer chunks beat L2
  // residency of the lane planes (measured 32 / 64 / 128 / 256 MB: contraction
  // 14.7 / 11.3 / 11.3 / 10.3 ms per C4 tree); GT_LA8_MB overrides
  static const uint64_t mb = getenv("GT_LA8_MB") ? (uint64_t)atoi(getenv("GT_LA8_MB")) : 256ull;
  return std::max<uint64_t>(1, std::min<uint64_t>(nkb, (mb << 20) / per_blk));
}

// Division tapes of every heuristic level (levels 0 .. depth-2, mpc only),
// in W2 units; 0 when they would exceed 256 MB (then blocks are drawn live).
uint64_t div_tape_words(const gt_train_cfg& c) {
  if (c.heuristic != 0 || c.depth < 2) return 0;
  bool ok = false;
  const DivParams d = div_params(c.score_width, c.tau, &ok);
  if (!ok) return 0;
  const int TB = c.score_width == 32 ? div_tape_blocks<32>(d) : div_tape_blocks<64>(d);
  const uint64_t lanes = ((1ull << (c.depth - 1)) - 1) * 2ull * c.nf;
  const uint64_t w = lanes * (uint64_t)TB;
  return w * 16 > (256ull << 20) ? 0 : w;
}
// Count reshare sums of every level (k_alpha_tape, tensor engine); 0 when over 64 MB
uint64_t alpha_tab_words(const gt_train_cfg& c) {
  if (c.count_engine != 0) return 0;
  const uint64_t w = 3ull * ((1ull << c.depth) - 1) * (uint64_t)(2 * c.nf + 1);
  return w * 8 > (64ull << 20) ? 0 : w;
}
// Prologue feature tapes of every heuristic level (W2 units); 0 when over 256 MB
uint64_t feat_tape_words(const gt_train_cfg& c) {
  static const bool off = getenv("GT_NO_FEAT_TAPE") != nullptr;  // A/B experiments
  if (off || c.heuristic != 0 || c.depth < 2) return 0;
  const uint64_t w = ((1ull << (c.depth - 1)) - 1) * (uint64_t)c.nf * FEAT_BLOCKS;
  return w * 16 > (256ull << 20) ? 0 : w;
}
// Epilogue tapes of every heuristic level (W2 units); 0 when over 256 MB
uint64_t post_tape_words(const gt_train_cfg& c) {
  if (c.heuristic != 0 || c.depth < 2) return 0;
  const uint64_t w = ((1ull << (c.depth - 1)) - 1) * (uint64_t)post_tape_blocks_w(c.score_width, c.nf);
  return w * 16 > (256ull << 20) ? 0 : w;
}
inline uint64_t div_tape_level_off(int level, int nf, int TB) {  // W2 offset of level's tape
  return ((1ull << level) - 1) * 2ull * nf * (uint64_t)TB;
}

bool count_fused_ok(int nf);
// The fused count's mask sums on the tensor cores: two constant x-plane
// columns after the W sample columns (room for them in the 32 columns of a
// CTA pair's M tile: nf <= 14)
bool count_mask_mma(int nf) {
  static const bool off = getenv("GT_NO_MASK_MMA") != nullptr;  // A/B experiments
  return !off && count_fused_ok(nf) && 2 * nf + 1 + 2 <= 32;
}

// Early oaa lanes (k_oaa_early) for the split partition's sample counts, when
// the largest level's hit shares [3][2^(depth-2)][N] fit 256 MB.
bool early_oaa_ok(const gt_train_cfg& c) {
  static const bool off = getenv("GT_NO_EARLY_OAA") != nullptr;  // A/B experiments
  const uint64_t N = c.n_local;
  return !off && c.depth >= 3 && N > 0 && N <= (1ull << 17) && 24ull * (1ull << (c.depth - 2)) * N <= (256ull << 20);
}

struct Layout {
  uint64_t xin, yin, fin, tout, fout, cols, la, cols8, leaf, midx, divtape, divtable, posttape, posttable, nodetape, nodetable, feattape, alphatab, S, f[2], gam[2], cst[2], ceff[2], hc, dv, co, lab, stop, oaa, oaactr, total;  // word offsets
};

Layout layout(const gt_train_cfg& c, bool host_io = false) {
  const uint64_t N = c.n_local, nf = (uint64_t)c.nf, cols = 2 * nf, W = cols + 1;
  const uint64_t nmax = 1ull << (c.depth - 1), ch = 2 * nmax;
  Layout L;
  uint64_t o = 0;
  auto take = [&](uint64_t words) {
    uint64_t r = o;
    o += (words + 31) & ~31ull;  // 256-byte alignment
    return r;
  };
  L.cols = take(c.count_engine == 1 ? 3 * N * (uint64_t)count_plan(c.nf, 1).WC : 0);
  if (c.count_engine == 0) {
    const TcPlan tp = tc_plan(c.nf, (int)nmax);
    const uint64_t nkb = (N + TC_KB - 1) / TC_KB;
    // two chunk buffers (none for the fused count: its lanes never leave shared memory)
    L.la = take(count_fused_ok(c.nf) ? 0 : 2 * tc_la8_blocks(N, c.nf, c.depth) * 3ull * tp.mtiles * TC_ABLK / 8);
    L.cols8 = take(3ull * tp.nbn * nkb * tp.BB / 8);
  } else {
    L.la = take(la_words(N, c.nf, c.depth));
    L.cols8 = take(0);
  }
  L.leaf = take(3 * nmax);
  L.midx = take(3 * N);
  L.divtape = take(2 * div_tape_words(c));
  L.posttape = take(2 * post_tape_words(c));
  L.nodetape = take(c.heuristic == 0 ? 2 * ((1ull << c.depth) - 1) * (uint64_t)node_tape_plan(c.nf).total : 0);
  L.nodetable = take(c.heuristic == 0 ? (uint64_t)node_tape_plan(c.nf).total : 0);
  L.feattape = take(2 * feat_tape_words(c));
  L.alphatab = take(alpha_tab_words(c));
  L.posttable = take(c.heuristic == 0 ? (uint64_t)post_tape_blocks_w(c.score_width, c.nf) : 0);
  {
    bool ok = false;
    const DivParams d = div_params(c.score_width, c.tau, &ok);
    const int TB = !ok ? 0 : c.score_width == 32 ? div_tape_blocks<32>(d) : div_tape_blocks<64>(d);
    L.divtable = take((uint64_t)(TB + 1) / 2);  // TB u32 schedule entries
  }
  L.S = take(3 * nmax * (W + 1));
  for (int i = 0; i < 2; ++i) {
    L.f[i] = take(3 * ch);
    L.gam[i] = take(3 * ch);
    L.cst[i] = take(3 * ch * 3 * cols);
    L.ceff[i] = take(3 * nmax * 3 * cols);
  }
  L.hc = take(12 * nmax);
  L.dv = take(9 * nmax * cols);
  L.co = take(3 * nmax * 3 * cols);
  L.lab = take(3 * nmax);
  L.stop = take(4);
  L.oaa = take(early_oaa_ok(c) ? 3ull * (nmax / 2) * N : 0);
  L.oaactr = take(early_oaa_ok(c) ? 16 : 0);
  // device staging of the host-input entry (gt_train_host)
  const uint64_t slots = (1ull << c.depth) - 1;
  L.xin = take(host_io ? 3 * N * nf : 0);
  L.yin = take(host_io ? 3 * N : 0);
  L.fin = take(host_io ? slots : 0);
  L.tout = take(host_io ? 3 * slots : 0);
  L.fout = take(host_io ? 3 * slots : 0);
  L.total = o;
  return L;
}

// Launch of a level-chain kernel with programmatic stream serialization (see
// pdl_wait); GT_NO_PDL=1 launches them normally (A/B experiments).
template <typename... KArgs, typename... Args>
int launch_chain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                 const cudaLaunchAttribute* extra, Args... args) {
  static const bool pdl = getenv("GT_NO_PDL") == nullptr;
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[2];
  int na = 0;
  if (extra) at[na++] = *extra;
  if (pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  lc.attrs = at;
  lc.numAttrs = (unsigned)na;
  const cudaError_t e = cudaLaunchKernelEx(&lc, kern, args...);
  if (e != cudaSuccess) {
    static thread_local char what[160];
    snprintf(what, sizeof what, "chain launch grid (%u,%u) block %u smem %zu", grid.x, grid.y, block.x, smem);
    return fail_cuda(e, what);
  }
  return GT_OK;
}

template <int SL>
int post_smem_bytes(const NodeArgs& na) {
  return (int)sizeof(uint64_t) * post_scratch_words(na.nf) + (int)sizeof(W2) * post_tape_blocks<SL>(na.nf);
}

// The division runs inside k_hc_pre's feature CTAs when its lane tapes exist
// (GT_NO_FUSED_DIV=1: separate k_hc_div launch, A/B experiments).
bool hc_div_fused(const NodeArgs& na) {
  static const bool no_fuse = getenv("GT_NO_FUSED_DIV") != nullptr;
  return !no_fuse && !na.last && !na.co_out && na.divtape != nullptr;
}

template <int SL>
int launch_node_hc(const NodeArgs& na, cudaStream_t s, bool fuse_post) {
  const int cols = 2 * na.nf;
  const int pre_smem = (int)sizeof(uint64_t) * ((9 * cols + 1) & ~1) + (int)sizeof(W2) * node_tape_plan(na.nf).spl;
  const unsigned gy = (na.last || na.co_out) ? 1u : (unsigned)(1 + na.nf);
  NodeArgs nf_args = na;
  nf_args.fuse_div = hc_div_fused(na);
  const int smem = nf_args.fuse_div ? std::max(pre_smem, 2 * (int)sizeof(W2) * div_tape_blocks<SL>(na.d)) : pre_smem;
  GT_CUDA_CHECK(cudaFuncSetAttribute(k_hc_pre<SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int rc = launch_chain(k_hc_pre<SL>, dim3(na.n_h, gy), dim3(64), (size_t)smem, s, nullptr, nf_args);
  if (rc) return rc;
  GT_LAUNCH_CHECK("k_hc_pre");
  if (na.last || na.co_out) return GT_OK;
  if (!nf_args.fuse_div) {
    const uint64_t lanes = (uint64_t)na.n_h * cols;
    const int per_warp = (int)sizeof(W2) * (na.divtape ? div_tape_blocks<SL>(na.d) : division_tape_blocks<SL>(na.d));
    const int wpc = std::max(1, std::min(DIV_WARPS, (200 * 1024) / per_warp));
    const int div_smem = per_warp * wpc;
    GT_CUDA_CHECK(cudaFuncSetAttribute(k_hc_div<SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, div_smem));
    rc = launch_chain(k_hc_div<SL>, dim3((unsigned)((lanes + wpc - 1) / wpc)), dim3(32 * wpc), (size_t)div_smem, s,
                      nullptr, na);
    if (rc) return rc;
    GT_LAUNCH_CHECK("k_hc_div");
  }
  if (fuse_post) return GT_OK;  // k_hc_post_finish runs it with the split
  const int psm = post_smem_bytes<SL>(na);
  GT_CUDA_CHECK(cudaFuncSetAttribute(k_hc_post<SL>, cudaFuncAttributeMaxDynamicSharedMemorySize, psm));
  k_hc_post<SL><<<na.n_h, 256, psm, s>>>(na);
  GT_LAUNCH_CHECK("k_hc_post");
  return GT_OK;
}

template <int G>
int launch_partition_g(const uint64_t* X, uint64_t* midx, const uint64_t* T, uint64_t slots, int m, int nf,
                       uint64_t N, uint64_t base, const Keys& K, int level, cudaStream_t s, const PartAux& aux) {
  // 128-thread CTAs: 96 registers per thread fit 5 per SM (20 warps) where
  // 256-thread CTAs fit 2 (16 warps)
  static const int TPB = getenv("GT_PART_TPB") ? atoi(getenv("GT_PART_TPB")) : 128;  // A/B experiments
  const uint64_t threads = N * G;
  const unsigned grid = (unsigned)((threads + TPB - 1) / TPB);
  const int smem = 3 * m * (int)sizeof(uint64_t);
  if (smem > 48 * 1024) GT_CUDA_CHECK(cudaFuncSetAttribute(k_partition<G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  int rc = launch_chain(k_partition<G>, dim3(grid), dim3(TPB), (size_t)smem, s, nullptr, X, midx, T, slots, m, nf, N,
                        base, K, op_id(level, SITE_PART_OAA), op_id(level, SITE_PART_ROW), aux);
  if (rc) return rc;
  GT_LAUNCH_CHECK("k_partition");
  return GT_OK;
}

// G threads per sample: the fewest idle lane-slots (ceil(m/G) + ceil(nf/G)
// rounds of G lanes) among the G that keep >= 2 warps per SMSP busy (G = 1
// whenever N allows: no group shuffles, no divergent trip counts; measured
// 181 vs 204 us per C2 tree against G = 2).
int launch_partition(const uint64_t* X, uint64_t* midx, const uint64_t* T, uint64_t slots, int m, int nf, uint64_t N,
                     uint64_t base, const Keys& K, int level, cudaStream_t s, int num_sms, const PartAux& aux,
                     const uint64_t* ca = nullptr, int qe = 1 << 30) {
  // A/B: GT_PART_SPLIT=B (1, 2, 4) forces the split kernel, 0 the group kernel.
  // Default (measured, C2 / C4): the split kernel with B = 2 while the level
  // has fewer than ~700 samples per SM (C2: 0.657 vs 0.669 ms per tree), the
  // one-thread-per-sample group kernel above that (C4: 20.95 vs 21.28 ms).
  static const int forced_split = getenv("GT_PART_SPLIT") ? atoi(getenv("GT_PART_SPLIT")) : -1;
  int split = forced_split >= 0 ? forced_split : (N <= (uint64_t)num_sms * 700 ? 2 : 0);
  if (ca && split != 1 && split != 2 && split != 4) split = 2;  // early oaa lanes: the split kernel reads them
  if ((split == 1 || split == 2 || split == 4) && N) {
    const int S = PS_TPB / split;
    const unsigned grid = (unsigned)((N + S - 1) / S);
    const int tab_smem = 3 * m * 8 <= 24 * 1024;
    const size_t smem = tab_smem ? (size_t)3 * m * sizeof(uint64_t) : 0;
    const uint32_t oo = op_id(level, SITE_PART_OAA), orow = op_id(level, SITE_PART_ROW);
    const dim3 blk(PS_TPB);
    int rc = split == 1 ? launch_chain(k_partition_split<1>, dim3(grid), blk, smem, s, nullptr, X, midx, T, slots, m,
                                       nf, N, base, K, oo, orow, aux, tab_smem, ca, qe)
           : split == 2 ? launch_chain(k_partition_split<2>, dim3(grid), blk, smem, s, nullptr, X, midx, T, slots, m,
                                       nf, N, base, K, oo, orow, aux, tab_smem, ca, qe)
                        : launch_chain(k_partition_split<4>, dim3(grid), blk, smem, s, nullptr, X, midx, T, slots, m,
                                       nf, N, base, K, oo, orow, aux, tab_smem, ca, qe);
    if (rc) return rc;
    GT_LAUNCH_CHECK("k_partition_split");
    return GT_OK;
  }
  const uint64_t target = (uint64_t)num_sms * 256;
  int best = 16;
  uint64_t best_work = ~0ull;
  for (int G = 1; G <= 16; G <<= 1) {
    const uint64_t work = (uint64_t)G * (((m + 1) / 2 + G - 1) / G + ((nf + 1) / 2 + G - 1) / G);
    if (N * (uint64_t)G >= target && work < best_work) {
      best_work = work;
      best = G;
    }
  }
  static const int forced = getenv("GT_PART_G") ? atoi(getenv("GT_PART_G")) : 0;  // A/B experiments
  if (forced == 1 || forced == 2 || forced == 4 || forced == 8 || forced == 16) best = forced;
  switch (best) {
    case 1: return launch_partition_g<1>(X, midx, T, slots, m, nf, N, base, K, level, s, aux);
    case 2: return launch_partition_g<2>(X, midx, T, slots, m, nf, N, base, K, level, s, aux);
    case 4: return launch_partition_g<4>(X, midx, T, slots, m, nf, N, base, K, level, s, aux);
    case 8: return launch_partition_g<8>(X, midx, T, slots, m, nf, N, base, K, level, s, aux);
    default: return launch_partition_g<16>(X, midx, T, slots, m, nf, N, base, K, level, s, aux);
  }
}

// CUDA-event timing of each launch (gt_train_ex with a profile struct).
struct Prof {
  enum Kind { PRODS, PARTITION, COUNT_LANES, COUNT_CONTRACT, NODE_HC, NODE_FINISH, NKIND };
  gt_train_profile* out;
  cudaStream_t s;
  cudaEvent_t first = nullptr, a = nullptr;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> spans;
  uint32_t launches = 0;
  Prof(gt_train_profile* o, cudaStream_t st) : out(o), s(st) {}
  ~Prof() {
    for (auto& e : spans) {
      cudaEventDestroy(e.second.first);
      cudaEventDestroy(e.second.second);
    }
    if (first) cudaEventDestroy(first);
  }
  void begin() {
    if (!out) return;
    cudaEventCreate(&first);
    cudaEventRecord(first, s);
  }
  void count_launch() { ++launches; }
  void start() {
    ++launches;
    if (!out) return;
    cudaEventCreate(&a);
    cudaEventRecord(a, s);
  }
  void stop(int kind) {
    if (!out) return;
    cudaEvent_t b;
    cudaEventCreate(&b);
    cudaEventRecord(b, s);
    spans.push_back({kind, {a, b}});
  }
  int finish() {
    if (!out) return GT_OK;
    GT_CUDA_CHECK(cudaStreamSynchronize(s));
    gt_train_profile p{};
    p.launches = launches;
    float* ms[NKIND] = {&p.ms_prods,     &p.ms_partition, &p.ms_count_lanes, &p.ms_count_contract,
                        &p.ms_node_hc,   &p.ms_node_finish};
    uint32_t* cnt[NKIND] = {&p.n_prods,   &p.n_partition, &p.n_count_lanes, &p.n_count_contract,
                            &p.n_node_hc, &p.n_node_finish};
    cudaEvent_t last = first;
    for (auto& e : spans) {
      float t = 0.f;
      GT_CUDA_CHECK(cudaEventElapsedTime(&t, e.second.first, e.second.second));
      *ms[e.first] += t;
      *cnt[e.first] += 1;
      last = e.second.second;
    }
    GT_CUDA_CHECK(cudaEventElapsedTime(&p.ms_total, first, last));
    p.ms_count = p.ms_count_lanes + p.ms_count_contract;
    p.n_count = p.n_count_lanes + p.n_count_contract;
    *out = p;
    return GT_OK;
  }
};

// Zero shares of the count products, summed over this shard's samples, one
// thread per (node, column):
//  elementwise (count_reshare 0, train.py:219): the product at (sample t,
//    node n, column w) is reshared with F_i(t) = H_i(t+1) - H_i(t),
//    H_i(t) = pair_i word (op_cnt, sub 3, field w, lane t n_h + n), so
//    sum_{t in [t0, t1)} F_i = H_i(t1) - H_i(t0) and sharded sums telescope;
//  dot (count_reshare 1): ONE zero share per cell, F_i at (op_cnt, sub 4,
//    field w, lane n), added by the shard holding sample 0.
// alpha_i = F_i - F_{i-1} (rss.py:302-306).
// The count products' reshare sums of every level, drawn up front (they depend
// only on the keys and the shard's sample range): tab[(2^h - 1) + n][c][w] =
// F_c - F_{c-1}, F as in k_count_alpha.  The contraction's epilogue adds them.
__global__ void __launch_bounds__(256) k_alpha_tape(uint64_t* tab, uint32_t cells, int nf, Keys K, int dot,
                                                    uint64_t t0, uint64_t t1) {
  const int W = 2 * nf + 1;
  const uint32_t e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= cells) return;
  const uint32_t gn = e / W;
  const int w = (int)(e - gn * W);
  const int level = 31 - __clz(gn + 1);
  const uint64_t n = gn - ((1u << level) - 1), n_h = 1ull << level;
  const uint32_t op = op_id(level, SITE_COUNT);
  uint64_t F[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    F[i] = dot ? word(K.pair[i], op, 4, (uint32_t)w, n)
               : word(K.pair[i], op, 3, (uint32_t)w, t1 * n_h + n) - word(K.pair[i], op, 3, (uint32_t)w, t0 * n_h + n);
#pragma unroll
  for (int c = 0; c < 3; ++c) tab[((uint64_t)gn * 3 + c) * W + w] = F[c] - F[(c + 2) % 3];
}

__global__ void k_count_alpha(uint64_t* S, int n_h, int nf, Keys K, uint32_t op_cnt, int dot, uint64_t t0,
                              uint64_t t1) {
  const int W = 2 * nf + 1;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= n_h * W) return;
  const int n = e / W, w = e % W;
  const uint64_t Sstride = (uint64_t)n_h * (W + 1);
  uint64_t F[3];
#pragma unroll
  for (int i = 0; i < 3; ++i)
    F[i] = dot ? word(K.pair[i], op_cnt, 4, (uint32_t)w, (uint64_t)n)
               : word(K.pair[i], op_cnt, 3, (uint32_t)w, t1 * (uint64_t)n_h + n) -
                     word(K.pair[i], op_cnt, 3, (uint32_t)w, t0 * (uint64_t)n_h + n);
#pragma unroll
  for (int c = 0; c < 3; ++c) S[c * Sstride + (uint64_t)n * (W + 1) + w] += F[c] - F[(c + 2) % 3];
}

struct CountLaunch {
  const uint64_t *midx, *f, *cols;
  uint64_t *la, *leaf, *S;
  uint64_t la_cap_words, N, base;
  int nf, n_h, n_h_max;
  Keys K;
  int level;
  const uint64_t* alpha_tab;  // the level's precomputed count reshare sums (tensor engine) or null
  const uint64_t* leafbits;   // is_leaf bits [3][n_h] drawn by the level's partition launch, or null
};

// leaf + per chunk (lanes, contraction); returns the number of launches
int launch_count(const CountLaunch& c, cudaStream_t s, int num_sms, Prof& P) {
  const CountPlan p = count_plan(c.nf, c.n_h);
  P.start();
  k_count_leaf<<<(c.n_h + 127) / 128, 128, 0, s>>>(c.f, c.leaf, c.n_h, c.K, op_id(c.level, SITE_ISLEAF));
  GT_LAUNCH_CHECK("k_count_leaf");
  P.stop(Prof::COUNT_LANES);
  const uint64_t per = 3ull * p.nblk * p.nbp;
  const uint64_t cap = std::max<uint64_t>(1, std::min<uint64_t>(c.N, c.la_cap_words / per));
  const int stage_words = 3 * p.ts * (p.nbp + p.WC);
  const int smem = (int)sizeof(uint64_t) * std::max(2 * stage_words, p.R * p.P * 3 * CNT_NA * CNT_CB);
  if (smem > 48 * 1024)
    GT_CUDA_CHECK(cudaFuncSetAttribute(k_count_mac, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (uint64_t s0 = 0; s0 < c.N; s0 += cap) {
    const uint64_t cn = std::min<uint64_t>(cap, c.N - s0);
    LaneArgs la{};
    la.midx = c.midx;
    la.leaf = c.leaf;
    la.la = c.la;
    la.N = c.N;
    la.s0 = s0;
    la.cn = cn;
    la.cap = cap;
    la.base = c.base;
    la.n_h = c.n_h;
    la.off = c.n_h - 1;
    la.nb = p.nb;
    la.nbp = p.nbp;
    la.nblk = p.nblk;
    la.K = c.K;
    la.op_cnt = op_id(c.level, SITE_COUNT);
    const uint64_t lanes = (cn + 1) / 2 * p.nblk * p.nbp;
    P.start();
    k_count_lanes<<<(unsigned)((lanes + 255) / 256), 256, 0, s>>>(la);
    GT_LAUNCH_CHECK("k_count_lanes");
    P.stop(Prof::COUNT_LANES);
    MacArgs ma{};
    ma.la = c.la;
    ma.cols = c.cols;
    ma.S = c.S;
    ma.N = c.N;
    ma.s0 = s0;
    ma.cn = cn;
    ma.cap = cap;
    ma.n_h = c.n_h;
    ma.W = p.W;
    ma.WC = p.WC;
    ma.nb = p.nb;
    ma.nbp = p.nbp;
    ma.nblk = p.nblk;
    ma.ts = p.ts;
    const uint64_t tiles = (cn + p.ts - 1) / p.ts;
    const uint64_t gx0 = std::max<uint64_t>(1, std::min<uint64_t>(tiles, (uint64_t)std::max(1, num_sms / p.nblk)));
    ma.tiles_per_cta = (int)((tiles + gx0 - 1) / gx0);
    const unsigned gx = (unsigned)((tiles + ma.tiles_per_cta - 1) / ma.tiles_per_cta);
    P.start();
    k_count_mac<<<dim3(gx, (unsigned)p.nblk), CNT_TPB, smem, s>>>(ma);
    GT_LAUNCH_CHECK("k_count_mac");
    P.stop(Prof::COUNT_CONTRACT);
  }
  return GT_OK;
}

// Optional (GT_L2_WINDOW=1): keep the level-invariant B operand (the
// byte-plane sample columns, read by every level's contraction) resident in
// L2 with a persisting access-policy window on the launches that write and
// read it, the carve-out raised once per device (bounded by the device max).
// Measured slower at C2 and C4 (see below); the x-plane loads keep their
// evict_last hint instead.
bool l2_window_attr(const void* base, uint64_t bytes, cudaLaunchAttribute* at) {
  static int max_persist = -1, max_window = 0;
  // off by default: the persisting carve-out (79 MB on B200) costs the rest of
  // the level's traffic more than it saves the x planes (C2 0.566 ms without
  // vs 0.576 ms with, same-call A/B); GT_L2_WINDOW=1 restores it
  static const bool off = getenv("GT_L2_WINDOW") == nullptr;
  if (off) return false;
  if (max_persist < 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&max_window, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess)
      max_persist = 0;
    if (getenv("GT_L2_LIMIT_MB") && max_persist > 0)  // A/B experiments
      max_persist = std::min(max_persist, atoi(getenv("GT_L2_LIMIT_MB")) << 20);
    if (max_persist > 0) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)max_persist);
    cudaGetLastError();
  }
  if (max_persist <= 0 || max_window <= 0 || bytes == 0) return false;
  const uint64_t win = std::min<uint64_t>(bytes, (uint64_t)max_window);
  at->id = cudaLaunchAttributeAccessPolicyWindow;
  at->val.accessPolicyWindow.base_ptr = const_cast<void*>(base);
  at->val.accessPolicyWindow.num_bytes = (size_t)win;
  at->val.accessPolicyWindow.hitRatio = std::min(1.0f, (float)max_persist / (float)win);
  at->val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  at->val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  return true;
}

// A second (side) stream per device for work that can run beside the main
// stream -- the division tapes beside the prologue, a chunk's contraction
// beside the next chunk's lanes -- with reusable fork/join events.  Inside a
// CUDA-graph capture the waits become graph edges.
struct Side {
  cudaStream_t st = nullptr;  // compute side stream (high priority)
  cudaStream_t cp = nullptr;  // host <-> device copies of the host-input entry
  cudaStream_t lo = nullptr;  // early oaa lanes beside the heuristic chain (low priority)
  cudaStream_t st2 = nullptr; // the epilogue / prologue / node tapes beside the division tapes (high priority)
  cudaEvent_t et2[2] = {};    // st2 fork / join
  cudaEvent_t ev[16] = {};
  cudaEvent_t eo[2] = {};     // early oaa fork / join
};
// One Side per device, shared by every trainer on that device: train_impl
// holds the device's side lock for its whole host-side enqueue, so calls
// from concurrent host threads never interleave their fork/join event
// records (and the lazy creation below is race-free).
std::recursive_mutex& side_lock(int dev) {
  static std::recursive_mutex mu[64];
  return mu[dev & 63];
}
int side_of(int dev, Side** out) {
  static Side sides[64];
  if (dev < 0 || dev >= 64) return fail_inval("device index out of range");
  Side& sd = sides[dev];
  if (!sd.st) {
    // highest priority: a contraction's CTAs are dispatched as soon as the
    // lane kernel running beside it frees an SM slot
    int lo = 0, hi = 0;
    GT_CUDA_CHECK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    GT_CUDA_CHECK(cudaStreamCreateWithPriority(&sd.st, cudaStreamNonBlocking, hi));
    GT_CUDA_CHECK(cudaStreamCreateWithFlags(&sd.cp, cudaStreamNonBlocking));
    GT_CUDA_CHECK(cudaStreamCreateWithPriority(&sd.lo, cudaStreamNonBlocking, lo));
    GT_CUDA_CHECK(cudaStreamCreateWithPriority(&sd.st2, cudaStreamNonBlocking, hi));
    for (auto& e : sd.et2) GT_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : sd.ev) GT_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : sd.eo) GT_CUDA_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  *out = &sd;
  return GT_OK;
}
// `to` waits for everything issued so far on `from`
int stream_after(cudaStream_t to, cudaStream_t from, cudaEvent_t ev) {
  GT_CUDA_CHECK(cudaEventRecord(ev, from));
  GT_CUDA_CHECK(cudaStreamWaitEvent(to, ev, 0));
  return GT_OK;
}

// Fused count (21..32 sample columns): one launch per level range, CTA pairs
// of (16-node tile, K range) produce the lanes straight into the tcgen05
// B stages (k_count_fused); no la planes, no chunking.
int launch_count_fused(const CountLaunch& c, const uint8_t* B8, int alpha, uint64_t t0, uint64_t t1, cudaStream_t s,
                       int num_sms, Prof& P, uint64_t lo, uint64_t hi) {
  hi = std::min<uint64_t>(hi, c.N);
  if (hi <= lo) return GT_OK;
  const int NN = std::min(16, c.n_h), NBn = std::max(1, NN / 2), ntiles = (c.n_h + 15) / 16;
  const uint64_t nkb_total = (c.N + TC_KB - 1) / TC_KB;
  const uint32_t kb_lo = (uint32_t)(lo / TC_KB);  // lo is a K-block boundary
  const uint32_t nkb = (uint32_t)((hi - lo + TC_KB - 1) / TC_KB);
  // one CTA per SM: the fewest waves of pairs the K-range bound allows, filled
  // with as many K ranges as fit in them
  const int pairs = std::max(1, num_sms / 2);
  const int nkr_min = (int)((nkb + TC_MAX_KB_PER_CTA - 1) / TC_MAX_KB_PER_CTA);
  const int waves = std::max(1, (ntiles * nkr_min + pairs - 1) / pairs);
  int nkr = std::max(nkr_min, waves * pairs / ntiles);
  nkr = std::min<int>(nkr, (int)nkb);
  const int per = (int)((nkb + nkr - 1) / nkr);
  nkr = (int)((nkb + per - 1) / per);
  FusedArgs fa{};
  fa.midx = c.midx;
  fa.f = c.f;
  fa.leafbits = c.leafbits;
  fa.B8 = B8;
  fa.S = c.S;
  fa.alpha_tab = c.alpha_tab;
  fa.K = c.K;
  fa.op_cnt = op_id(c.level, SITE_COUNT);
  fa.op_leaf = op_id(c.level, SITE_ISLEAF);
  fa.alpha = lo == 0 ? alpha : 0;
  fa.t0 = t0;
  fa.t1 = t1;
  fa.N = c.N;
  fa.base = c.base;
  fa.nkb_total = nkb_total;
  fa.kb_lo = kb_lo;
  fa.nkb = nkb;
  fa.n_h = c.n_h;
  fa.W = 2 * c.nf + 1;
  fa.nkr = nkr;
  fa.NBn = NBn;
  fa.mask_mma = count_mask_mma(c.nf) ? 1 : 0;
  {
    static const bool no_m3 = getenv("GT_FUSED_NO_MODE3") != nullptr;  // A/B experiments
    fa.mode3 = tcf_mode3(NBn) && !no_m3;
  }
  fa.stages = tcf_stages(NBn, fa.mode3);
  {
    static const bool ts = getenv("GT_COUNT_TS") != nullptr;
    fa.ts_level = ts ? c.level : -1;
  }
  {
    static const bool no_xpre = getenv("GT_FUSED_NO_XPRE") != nullptr;  // A/B experiments
    fa.xpre = c.level > 0 && !no_xpre;
  }
  const int smem = tcf_smem(NBn, fa.mode3);
  cudaLaunchAttribute at[1];
  const TcPlan tp = tc_plan(c.nf, c.n_h);
  const bool win = l2_window_attr(B8, 3ull * tp.nbn * nkb_total * tp.BB, at);
  // producer warps: 18 (measured C2 0.615 ms vs 0.618 / 0.625 at 14 / 22; 87
  // registers); A/B: GT_FUSED_PW = 14, GT_FUSED_PF = 1 (node-index prefetch, no gain)
  static const int pw = getenv("GT_FUSED_PW") ? atoi(getenv("GT_FUSED_PW")) : 18;
  static const int pf = getenv("GT_FUSED_PF") ? atoi(getenv("GT_FUSED_PF")) : 0;
  auto go = [&](auto kern, int threads) {
    GT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    return launch_chain(kern, dim3(2, (unsigned)ntiles, (unsigned)nkr), dim3(threads), (size_t)smem, s,
                        win ? at : nullptr, fa);
  };
  P.start();
  int rc = pw == 14 ? go(k_count_fused<14, false>, 512)
         : pf ? go(k_count_fused<18, true>, 640) : go(k_count_fused<18, false>, 640);
  if (rc) return rc;
  P.stop(Prof::COUNT_CONTRACT);
  GT_LAUNCH_CHECK("k_count_fused");
  return GT_OK;
}

bool count_fused_ok(int nf) {
  static const bool off = getenv("GT_NO_FUSED_COUNT") != nullptr;  // A/B experiments
  const TcPlan tp = tc_plan(nf, 1);
  return !off && tp.nbn == 2 && tp.cpb == 16;
}

// tensor engine: leaf + per chunk (byte-plane lanes, tcgen05 contraction)
// Chunks alternate between two la8 buffers (each holds la8_blocks K blocks at
// the deepest level): with a side stream, the contraction of chunk k runs
// beside the lanes of chunk k+1 (ALU-bound lanes, copy-bound contraction),
// and the lanes of chunk k+2 wait for the contraction of chunk k.
int launch_count_tc(const CountLaunch& c, const uint8_t* B8, uint64_t la8_blocks, int alpha, uint64_t t0,
                    uint64_t t1, cudaStream_t s, Side* side, int num_sms, Prof& P, uint64_t lo = 0,
                    uint64_t hi = ~0ull) {
  if (count_fused_ok(c.nf)) return launch_count_fused(c, B8, alpha, t0, t1, s, num_sms, P, lo, hi);
  hi = std::min<uint64_t>(hi, c.N);
  const TcPlan tp = tc_plan(c.nf, c.n_h);
  // two chunk buffers when pipelining across streams, else one of twice the size
  const uint64_t buf_bytes = (side ? 1ull : 2ull) * la8_blocks * 3ull * tc_plan(c.nf, c.n_h_max).mtiles * TC_ABLK;
  const uint64_t nkb_all = (c.N + TC_KB - 1) / TC_KB;
  // shallower levels (fewer M tiles) fit proportionally more samples per buffer;
  // with a side stream, at least two chunks so the pipeline has something to overlap
  la8_blocks = std::min<uint64_t>(buf_bytes / (3ull * tp.mtiles * TC_ABLK), nkb_all);
  if (side && nkb_all >= 2) la8_blocks = std::min<uint64_t>(la8_blocks, (nkb_all + 1) / 2);
  const uint64_t cap = la8_blocks * TC_KB;
  cudaStream_t s2 = side ? side->st : s;
  if (side) {
    int rc = stream_after(s2, s, side->ev[0]);  // the side stream joins after the level's partition
    if (rc) return rc;
  }
  int k = 0;
  const uint64_t nkb_total = (c.N + TC_KB - 1) / TC_KB;
  // n_h <= 8: operand roles swapped (k_count_mma_t; its x-plane A operand
  // reads up to 2 KB past a stage)
  static const bool no_t = getenv("GT_NO_MMA_T") != nullptr;  // A/B experiments
  const bool swapped = c.n_h <= 8 && tp.cpb <= 16 && !no_t;  // the x planes fill at most M = 128 rows
  const int smem = TC_MC_STAGES * (TC_A_HB + 3 * tp.BB / 2) + (swapped ? 2048 : 0);
  GT_CUDA_CHECK(cudaFuncSetAttribute(swapped ? k_count_mma_t : k_count_mma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     smem));
  for (uint64_t s0 = lo; s0 < hi; s0 += cap, ++k) {  // lo is a multiple of TC_KB
    const uint64_t cn = std::min<uint64_t>(cap, hi - s0);
    const uint32_t nkb = (uint32_t)((cn + TC_KB - 1) / TC_KB);
    uint8_t* buf = (uint8_t*)c.la + (side ? (uint64_t)(k & 1) * buf_bytes : 0ull);
    if (side && k >= 2) GT_CUDA_CHECK(cudaStreamWaitEvent(s, side->ev[2 + (k & 1)], 0));  // buffer reuse
    Lanes8Args la{};
    la.midx = c.midx;
    la.f = c.f;
    la.op_leaf = op_id(c.level, SITE_ISLEAF);
    la.la8 = buf;
    la.N = c.N;
    la.s0 = s0;
    la.cn = cn;
    la.base = c.base;
    la.nkbc = la8_blocks;
    la.n_h = c.n_h;
    la.off = c.n_h - 1;
    la.mtiles = tp.mtiles;
    la.K = c.K;
    la.op_cnt = op_id(c.level, SITE_COUNT);
    la.S = c.S;
    la.W = 2 * c.nf + 1;
    la.leafbits = c.leafbits;
    P.start();
    {
      const unsigned hpc = (unsigned)tc_lane_hpc(c.n_h);  // half blocks per CTA
      int rc = launch_chain(k_count_lanes8, dim3((2 * nkb + hpc - 1) / hpc, (unsigned)tp.mtiles), dim3(256), 0, s,
                            nullptr, la);
      if (rc) return rc;
    }
    GT_LAUNCH_CHECK("k_count_lanes8");
    P.stop(Prof::COUNT_LANES);
    if (side) {
      GT_CUDA_CHECK(cudaEventRecord(side->ev[4 + (k & 1)], s));
      GT_CUDA_CHECK(cudaStreamWaitEvent(s2, side->ev[4 + (k & 1)], 0));
    }
    MmaArgs ma{};
    ma.la8 = buf;
    ma.B8 = B8;
    ma.S = c.S;
    ma.nkbc = la8_blocks;
    ma.nkb_total = nkb_total;
    ma.kb_base = s0 / TC_KB;
    ma.nkb = nkb;
    ma.n_h = c.n_h;
    ma.W = 2 * c.nf + 1;
    ma.cpb = tp.cpb;
    ma.nbn = tp.nbn;
    ma.mtiles = tp.mtiles;
    ma.N = tp.N;
    ma.K = c.K;
    ma.op_cnt = op_id(c.level, SITE_COUNT);
    {
      static const int probe = getenv("GT_MMA_PROBE") ? atoi(getenv("GT_MMA_PROBE")) : 0;
      ma.probe = probe;
    }
    ma.alpha = s0 == 0 ? alpha : 0;
    ma.alpha_tab = c.alpha_tab;
    ma.t0 = t0;
    ma.t1 = t1;
    // one CTA per SM (shared memory): the fewest waves the K-range bound
    // allows, filled with as many K ranges as fit in them (a partial second
    // wave would double the kernel's time)
    const int tiles = tp.mtiles * tp.nbn;
    const int nkr_min = (int)((nkb + TC_MAX_KB_PER_CTA - 1) / TC_MAX_KB_PER_CTA);
    const int waves = std::max(1, (tiles * nkr_min + num_sms - 1) / num_sms);
    int nkr = std::max(nkr_min, waves * num_sms / tiles);
    nkr = std::min<int>(nkr, (int)nkb);
    const int per = (int)((nkb + nkr - 1) / nkr);
    ma.nkr = (int)((nkb + per - 1) / per);
    {
      cudaLaunchAttribute at[1];
      const bool win = l2_window_attr(B8, 3ull * tp.nbn * nkb_total * tp.BB, at);
      P.start();
      int rc = launch_chain(swapped ? k_count_mma_t : k_count_mma,
                            dim3((unsigned)tp.mtiles, (unsigned)(ma.nkr * tp.nbn), 1), dim3(256), (size_t)smem, s2,
                            win ? at : nullptr, ma);
      if (rc) return rc;
      P.stop(Prof::COUNT_CONTRACT);
    }
    GT_LAUNCH_CHECK("k_count_mma");
    if (side) GT_CUDA_CHECK(cudaEventRecord(side->ev[2 + (k & 1)], s2));
  }
  if (side) {  // join: the level's heuristic needs every chunk's counters
    int rc = stream_after(s, s2, side->ev[1]);
    if (rc) return rc;
  }
  return GT_OK;
}

// host-side operands of gt_train_host
struct HostIn {
  const uint64_t *X, *Y, *fill;
  uint64_t *T, *F;
};

// tensor-engine prologue over the 64-sample half blocks [hb_lo, hb_hi)
int launch_prep8(const gt_train_cfg& c, const uint64_t* features, const uint64_t* labels, uint64_t* ws,
                 const Layout& L, const Keys& K, uint64_t hb_lo, uint64_t hb_hi, cudaStream_t s) {
  if (hb_hi <= hb_lo) return GT_OK;
  const TcPlan tp = tc_plan(c.nf, 1);
  Prep8Args pa{};
  pa.X = features;
  pa.Y = labels;
  pa.B8 = (uint8_t*)(ws + L.cols8);
  pa.N = c.n_local;
  pa.nkb = (c.n_local + TC_KB - 1) / TC_KB;
  pa.base = c.sample_base;
  pa.hb0 = hb_lo;
  pa.nf = c.nf;
  pa.W = 2 * c.nf + 1;
  pa.cpb = tp.cpb;
  pa.nbn = tp.nbn;
  pa.mask_cols = count_mask_mma(c.nf) ? 1 : 0;
  pa.K = K;
  pa.op_prods = op_id(0, SITE_PRODS);
  const int smem = 3 * (TC_KB / 4) * pa.W * (int)sizeof(uint64_t);  // one CTA per 32-sample quarter block
  GT_CUDA_CHECK(cudaFuncSetAttribute(k_prep8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3((unsigned)(2 * (hb_hi - hb_lo)));
  lc.blockDim = dim3(256);
  lc.dynamicSmemBytes = (size_t)smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  lc.attrs = at;
  lc.numAttrs = l2_window_attr(pa.B8, 3ull * tp.nbn * pa.nkb * tp.BB, at) ? 1 : 0;
  GT_CUDA_CHECK(cudaLaunchKernelEx(&lc, k_prep8, pa));
  GT_LAUNCH_CHECK("k_prep8");
  return GT_OK;
}

int counter_shift(uint64_t n, int score_width, int tau) {  // train.py:75-78
  int headroom = (score_width - tau - 2) / 2;
  int bl = 0;
  while (bl < 64 && (n >> bl)) ++bl;
  return std::max(0, bl - headroom);
}

}  // namespace
}  // namespace gt

using namespace gt;

extern "C" {

uint64_t gt_train_workspace_bytes(const gt_train_cfg* cfg) {
  if (!cfg || cfg->depth < 1 || cfg->depth > 16 || cfg->nf < 1 || cfg->nf > 64) return 0;
  return layout(*cfg).total * sizeof(uint64_t);
}

int gt_train(const gt_train_cfg* cfg, const uint64_t* features, const uint64_t* labels, const uint64_t* filler,
             uint64_t* T, uint64_t* F, int32_t* depth_out, void* workspace, uint64_t workspace_bytes,
             const gt_keys* keys, gt_allreduce_fn allreduce, void* allreduce_user, void* stream) {
  return gt_train_ex(cfg, features, labels, filler, T, F, depth_out, workspace, workspace_bytes, keys, allreduce,
                     allreduce_user, nullptr, nullptr, stream, nullptr);
}

static int train_impl(const gt_train_cfg* cfg, const uint64_t* features, const uint64_t* labels,
                      const uint64_t* filler, uint64_t* T, uint64_t* F, int32_t* depth_out, void* workspace,
                      uint64_t workspace_bytes, const gt_keys* keys, gt_allreduce_fn allreduce, void* allreduce_user,
                      gt_heuristic_fn heuristic, void* heuristic_user, void* stream, gt_train_profile* prof,
                      const HostIn* hin) {
  if (!cfg || !keys) return fail_inval("gt_train: NULL cfg/keys");
  const gt_train_cfg c = *cfg;
  if (c.depth < 1 || c.depth > 16) return fail_inval("depth must be in 1..16");
  if (c.nf < 1 || c.nf > 64) return fail_inval("need 1..64 features");
  if (c.score_width != 32 && c.score_width != 64) return fail_inval("score ring width must be 32 or 64");
  if (c.tau < 0 || c.tau >= c.score_width - 2) return fail_inval("fixed-point precision tau out of range");
  if (c.n_total < 1) return fail_inval("dataset is empty");
  if (c.n_local > c.n_total || c.sample_base + c.n_local > c.n_total) return fail_inval("bad sample shard");
  if (c.policy != 0 && c.policy != 1) return fail_inval("policy must be fixed (0) or grow (1)");
  if (c.heuristic != 0 && c.heuristic != 1) return fail_inval("heuristic must be mpc (0) or tee (1)");
  if (c.count_reshare != 0 && c.count_reshare != 1) return fail_inval("count_reshare must be 0 or 1");
  if (c.count_engine != 0 && c.count_engine != 1) return fail_inval("count_engine must be 0 (tensor) or 1 (cuda)");
  if (c.heuristic == 1 && !heuristic) return fail_inval("heuristic tee needs the trusted-helper callback");
  const bool tee = c.heuristic == 1;
  bool ok = false;
  const DivParams d = div_params(c.score_width, c.tau, &ok);
  if (!ok) return fail_inval("division unsupported at this width/tau");
  const Layout L = layout(c, hin != nullptr);
  if (!workspace || workspace_bytes < L.total * sizeof(uint64_t)) return fail_inval("workspace too small");
  if (hin) {  // host operands: stage through the workspace
    if (c.n_local && (!hin->X || !hin->Y)) return fail_inval("NULL features/labels");
    if (!hin->fill || !hin->T || !hin->F) return fail_inval("NULL filler/T/F");
    features = (const uint64_t*)workspace + L.xin;
    labels = (const uint64_t*)workspace + L.yin;
    filler = (const uint64_t*)workspace + L.fin;
    T = (uint64_t*)workspace + L.tout;
    F = (uint64_t*)workspace + L.fout;
  }
  if (c.n_local && (!features || !labels)) return fail_inval("NULL features/labels");
  if (!filler || !T || !F) return fail_inval("NULL filler/T/F");

  cudaStream_t s = (cudaStream_t)stream;
  Prof P(prof, s);
  int dev = 0, num_sms = 148;
  GT_CUDA_CHECK(cudaGetDevice(&dev));
  GT_CUDA_CHECK(cudaDeviceGetAttribute(&num_sms, cudaDevAttrMultiProcessorCount, dev));
  const Keys K = to_keys(keys);
  uint64_t* ws = (uint64_t*)workspace;
  Side* side = nullptr;
  // A/B switches: GT_NO_SIDE keeps the division tapes on the main stream;
  // the lanes8 + contraction count (shapes the fused count does not take,
  // e.g. C4's 65 sample columns) pipelines its chunks across the two streams,
  // the contraction of chunk k beside the lanes of chunk k+1 (C4: 20.2 vs
  // 20.9 ms per tree); GT_NO_COUNT_OVERLAP=1 runs them in one stream
  static const bool no_side = getenv("GT_NO_SIDE") != nullptr;
  static const bool count_overlap = getenv("GT_NO_COUNT_OVERLAP") == nullptr;
  if (dev < 0 || dev >= 64) return fail_inval("device index out of range");
  std::lock_guard<std::recursive_mutex> side_guard(side_lock(dev));
  {
    int rc = side_of(dev, &side);
    if (rc) return rc;
  }
  const uint64_t N = c.n_local, nf = (uint64_t)c.nf, cols = 2 * nf, W = cols + 1;
  const uint64_t slots = (1ull << c.depth) - 1;
  const int shift = counter_shift(c.n_total, c.score_width, c.tau);
  uint64_t *colm = ws + L.cols, *midx = ws + L.midx, *S = ws + L.S, *hc = ws + L.hc;
  uint64_t *f[2] = {ws + L.f[0], ws + L.f[1]}, *gam[2] = {ws + L.gam[0], ws + L.gam[1]};
  uint64_t *cst[2] = {ws + L.cst[0], ws + L.cst[1]}, *ceff[2] = {ws + L.ceff[0], ws + L.ceff[1]};
  int cur = 0;

  // host filler: on the copy stream ahead of the sample chunks when they are
  // streamed (the chunk joins order it before the first split), else here
  const bool host_chunks = hin && c.count_engine == 0 && N;
  if (hin && !host_chunks)
    GT_CUDA_CHECK(cudaMemcpyAsync((void*)filler, hin->fill, slots * sizeof(uint64_t), cudaMemcpyHostToDevice, s));
  GT_CUDA_CHECK(cudaMemsetAsync(T, 0, 3 * slots * sizeof(uint64_t), s));
  GT_CUDA_CHECK(cudaMemsetAsync(F, 0, 3 * slots * sizeof(uint64_t), s));
  if (N) GT_CUDA_CHECK(cudaMemsetAsync(midx, 0, 3 * N * sizeof(uint64_t), s));  // m_idx = const(0)
  P.begin();
  k_init<<<1, 128, 0, s>>>(f[0], gam[0], cst[0], 1, 3 * cols, (int)cols, c.nf);
  GT_LAUNCH_CHECK("k_init");
  P.count_launch();
  // the count reshare sums of every level (data-independent): beside the
  // prologue, joined before the first count
  const int alpha_mode = c.count_reshare == 0 ? 1 : (c.sample_base == 0 ? 2 : 0);
  bool alpha_forked = false;
  if (alpha_tab_words(c) && alpha_mode && N) {
    cudaStream_t as = s;
    if (!prof && !no_side) {
      int rc = stream_after(side->st, s, side->ev[15]);
      if (rc) return rc;
      as = side->st;
      alpha_forked = true;
    }
    const uint32_t cells = (uint32_t)(alpha_tab_words(c) / 3);
    k_alpha_tape<<<(cells + 255) / 256, 256, 0, as>>>(ws + L.alphatab, cells, c.nf, K, alpha_mode == 2 ? 1 : 0,
                                                      c.sample_base, c.sample_base + N);
    GT_LAUNCH_CHECK("k_alpha_tape");
    P.count_launch();
    if (alpha_forked) GT_CUDA_CHECK(cudaEventRecord(side->ev[15], side->st));
  }
  // the division randomness of every level is data-independent: draw it all now
  const uint64_t tape_words = div_tape_words(c);
  bool tape_forked = false;  // joined before the first heuristic
  if (tape_words) {
    const int cols_i = 2 * c.nf;
    const int TB = c.score_width == 32 ? div_tape_blocks<32>(d) : div_tape_blocks<64>(d);
    uint32_t* table = reinterpret_cast<uint32_t*>(ws + L.divtable);
    W2* tape = reinterpret_cast<W2*>(ws + L.divtape);
    // on the side stream beside the prologue (the first count join orders it
    // before any heuristic); inline when profiling
    cudaStream_t ts = s;
    if (!prof && !no_side && N) {
      int rc = stream_after(side->st, s, side->ev[6]);
      if (rc) return rc;
      ts = side->st;
    }
    // the other tapes on a second stream beside the division tape (their
    // launches overlap instead of queueing behind it), joined back into ts
    cudaStream_t ts2 = ts;
    if (ts != s) {
      GT_CUDA_CHECK(cudaEventRecord(side->et2[0], ts));
      GT_CUDA_CHECK(cudaStreamWaitEvent(side->st2, side->et2[0], 0));
      ts2 = side->st2;
    }
    P.start();
    if (c.score_width == 32) {
      k_div_table<32><<<(TB + 127) / 128, 128, 0, ts>>>(table, d);
      k_div_tape<32><<<(unsigned)((tape_words + 256 * DIV_TAPE_PER - 1) / (256 * DIV_TAPE_PER)), 256, 0, ts>>>(
          tape, table, tape_words, cols_i, TB, K);
    } else {
      k_div_table<64><<<(TB + 127) / 128, 128, 0, ts>>>(table, d);
      k_div_tape<64><<<(unsigned)((tape_words + 256 * DIV_TAPE_PER - 1) / (256 * DIV_TAPE_PER)), 256, 0, ts>>>(
          tape, table, tape_words, cols_i, TB, K);
    }
    const uint64_t post_words = post_tape_words(c);
    if (post_words) {
      const int E = post_tape_blocks_w(c.score_width, c.nf);
      const uint32_t SA = 13 + div_subs(d);
      uint64_t* ptab = ws + L.posttable;
      if (c.score_width == 32)
        k_post_table<32><<<(E + 127) / 128, 128, 0, ts2>>>(ptab, c.nf, SA);
      else
        k_post_table<64><<<(E + 127) / 128, 128, 0, ts2>>>(ptab, c.nf, SA);
      k_post_tape<<<(unsigned)((post_words + 255) / 256), 256, 0, ts2>>>(reinterpret_cast<W2*>(ws + L.posttape), ptab,
                                                                       (uint32_t)post_words, c.nf, E, K);
      GT_LAUNCH_CHECK("k_post_tape");
      P.count_launch();
      P.count_launch();
    }
    if (feat_tape_words(c)) {  // prologue feature tapes
      const uint64_t fw = feat_tape_words(c);
      k_feat_tape<<<(unsigned)((fw + 255) / 256), 256, 0, ts2>>>(reinterpret_cast<W2*>(ws + L.feattape), (uint32_t)fw,
                                                                c.nf, K);
      GT_LAUNCH_CHECK("k_feat_tape");
      P.count_launch();
    }
    {  // node tapes of every level (prologue chains, replace, split, labels)
      const NodeTape NT = node_tape_plan(c.nf);
      const uint64_t nwords = ((1ull << c.depth) - 1) * (uint64_t)NT.total;
      uint64_t* ntab = ws + L.nodetable;
      k_node_table<<<(NT.total + 127) / 128, 128, 0, ts2>>>(ntab, c.nf);
      k_node_tape<<<(unsigned)((nwords + 255) / 256), 256, 0, ts2>>>(reinterpret_cast<W2*>(ws + L.nodetape), ntab,
                                                                    (uint32_t)nwords, NT.total, K);
      GT_LAUNCH_CHECK("k_node_tape");
      P.count_launch();
      P.count_launch();
    }
    if (ts2 != ts) {
      GT_CUDA_CHECK(cudaEventRecord(side->et2[1], ts2));
      GT_CUDA_CHECK(cudaStreamWaitEvent(ts, side->et2[1], 0));
    }
    tape_forked = ts != s;
    P.count_launch();
    GT_LAUNCH_CHECK("k_div_tape");
    P.stop(Prof::NODE_HC);
  }
  // the count of one level over the samples [lo, hi)
  // host operands: join the up-front tapes before the first count (they
  // finished long before, beside the uploads) instead of before the first
  // heuristic, so the level-0 count -> heuristic step keeps its programmatic
  // (PDL) overlap (e2e 0.871 -> 0.868 ms in one A/B, within noise in a second).
  // Device operands keep the late join
  // (there the tapes still run beside the prologue: 0.5551 vs 0.5577 ms).
  // A/B: GT_TAPE_JOIN = 1 early always, 0 late always
  static const int tape_join_env = getenv("GT_TAPE_JOIN") ? atoi(getenv("GT_TAPE_JOIN")) : -1;
  const bool tape_join_early = tape_join_env >= 0 ? tape_join_env == 1 : hin != nullptr;
  auto count_range = [&](int level, int fcur, uint64_t lo, uint64_t hi) -> int {
    if (alpha_forked) {
      GT_CUDA_CHECK(cudaStreamWaitEvent(s, side->ev[15], 0));
      alpha_forked = false;
    }
    if (tape_join_early && tape_forked) {
      int rc = stream_after(s, side->st, side->ev[7]);
      if (rc) return rc;
      tape_forked = false;
    }
    CountLaunch cl{};
    cl.alpha_tab = alpha_tab_words(c) ? ws + L.alphatab + 3ull * ((1ull << level) - 1) * W : nullptr;
    cl.leafbits = (level > 0 && N && c.count_engine == 0) ? ws + L.leaf : nullptr;
    cl.midx = midx;
    cl.f = f[fcur];
    cl.cols = colm;
    cl.la = ws + L.la;
    cl.leaf = ws + L.leaf;
    cl.S = S;
    cl.la_cap_words = la_words(N, c.nf, c.depth);
    cl.N = N;
    cl.base = c.sample_base;
    cl.nf = c.nf;
    cl.n_h = 1 << level;
    cl.n_h_max = 1 << (c.depth - 1);
    cl.K = K;
    cl.level = level;
    return c.count_engine == 0
               ? launch_count_tc(cl, (const uint8_t*)(ws + L.cols8), tc_la8_blocks(N, c.nf, c.depth),
                                 alpha_mode, c.sample_base,
                                 c.sample_base + N, s, (prof || !count_overlap) ? nullptr : side, num_sms, P, lo, hi)
               : launch_count(cl, s, num_sms, P);
  };
  bool count0_done = false;
  if (N) {
    const int WC = count_plan(c.nf, 1).WC;
    const uint64_t tot = N * (uint64_t)WC;
    P.start();
    if (c.count_engine == 0) {  // tensor engine: prods and byte planes in one pass
      const uint64_t nhb = (N + TC_KB / 2 - 1) / (TC_KB / 2);
      if (hin) {
        // host inputs: Q sample chunks go up on the copy stream while the
        // prologue of the chunks already resident runs on the main stream
        // chunks on 128-sample K-block boundaries; the level-0 count (m_idx = 0)
        // of a chunk runs as soon as its planes exist
        const uint64_t nkb = (N + TC_KB - 1) / TC_KB;
        // two chunks measured best on C2 (1 / 2 / 3 / 4 / 8: e2e 1.242 / 1.221 / 1.231 / 1.257 / 1.338 ms):
        // (measured with six copies per chunk; now two 2-D copies, 2 chunks still best: 1.016 / 1.019 / 1.027 ms for 2 / 3 / 4)
        static const int Qenv = getenv("GT_HOST_CHUNKS") ? atoi(getenv("GT_HOST_CHUNKS")) : 2;
        const int Q = (int)std::min<uint64_t>((uint64_t)std::max(1, Qenv), nkb);
        int rc = stream_after(side->cp, s, side->ev[8]);
        if (rc) return rc;
        GT_CUDA_CHECK(cudaMemcpyAsync((void*)filler, hin->fill, slots * sizeof(uint64_t), cudaMemcpyHostToDevice,
                                      side->cp));
        const bool count0 = !prof && c.heuristic == 0;
        if (count0) GT_CUDA_CHECK(cudaMemsetAsync(S, 0, 3ull * 1 * (W + 1) * sizeof(uint64_t), s));
        uint64_t hb_lo = 0;
        for (int q = 0; q < Q; ++q) {
          // the last chunk is the smallest: only its prologue and level-0
          // count are exposed after the final upload (GT_HOST_LAST_PCT: its
          // share of the samples when Q = 2, default 15 %: e2e 1.034 / 1.012 / 1.008 ms at 50 / 25 / 15 %)
          static const int last_pct = getenv("GT_HOST_LAST_PCT") ? atoi(getenv("GT_HOST_LAST_PCT")) : 15;
          const uint64_t kb_end = (q + 1 == Q) ? nkb
                                  : (Q == 2 ? nkb * (uint64_t)(100 - std::min(90, std::max(10, last_pct))) / 100
                                            : nkb * (q + 1) / Q);
          const uint64_t hb_hi = std::min<uint64_t>(nhb, 2 * std::max<uint64_t>(kb_end, 1));
          const uint64_t lo = hb_lo * (TC_KB / 2), hi = std::min<uint64_t>(N, hb_hi * (TC_KB / 2));
          // the chunk's rows of the three components: one 2-D copy per operand
          GT_CUDA_CHECK(cudaMemcpy2DAsync((void*)(features + lo * nf), N * nf * sizeof(uint64_t), hin->X + lo * nf,
                                          N * nf * sizeof(uint64_t), (hi - lo) * nf * sizeof(uint64_t), 3,
                                          cudaMemcpyHostToDevice, side->cp));
          GT_CUDA_CHECK(cudaMemcpy2DAsync((void*)(labels + lo), N * sizeof(uint64_t), hin->Y + lo, N * sizeof(uint64_t),
                                          (hi - lo) * sizeof(uint64_t), 3, cudaMemcpyHostToDevice, side->cp));
          GT_CUDA_CHECK(cudaEventRecord(side->ev[9 + (q % 6)], side->cp));
          GT_CUDA_CHECK(cudaStreamWaitEvent(s, side->ev[9 + (q % 6)], 0));
          rc = launch_prep8(c, features, labels, ws, L, K, hb_lo, hb_hi, s);
          if (rc) return rc;
          if (count0) {
            rc = count_range(0, 0, lo, hi);
            if (rc) return rc;
          }
          hb_lo = hb_hi;
        }
        count0_done = count0;
      } else {
        int rc = launch_prep8(c, features, labels, ws, L, K, 0, nhb, s);
        if (rc) return rc;
      }
    } else {
      if (hin) {
        for (int cc = 0; cc < 3; ++cc) {
          GT_CUDA_CHECK(cudaMemcpyAsync((void*)(features + cc * N * nf), hin->X + cc * N * nf, N * nf * sizeof(uint64_t),
                                        cudaMemcpyHostToDevice, s));
          GT_CUDA_CHECK(cudaMemcpyAsync((void*)(labels + cc * N), hin->Y + cc * N, N * sizeof(uint64_t),
                                        cudaMemcpyHostToDevice, s));
        }
      }
      k_prods<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(features, labels, colm, N, c.nf, WC, c.sample_base, K,
                                                            op_id(0, SITE_PRODS));
      GT_LAUNCH_CHECK("k_prods");
    }
    P.stop(Prof::PRODS);
  }
  int32_t trained = c.depth;
  const bool early_oaa = early_oaa_ok(c);
  bool oaa_forked = false;  // an early oaa launch on side->lo not yet joined
  bool oaa_ready = false;   // the next partition's hit shares are (being) drawn
  // the next partition's oaa lanes (hit shares of m_idx vs its 2^level
  // entries), forked on the low-priority stream right after this level's
  // partition: small CTAs (two warps) fit beside the count's CTAs and take
  // idle issue slots there, more start beside the heuristic chain (at most
  // 16 warps per SM); work is fetched dynamically (k_oaa_early).  Measured
  // on one box, C2: 0.603 ms vs 0.615 launched after the count with 128-thread
  // CTAs, 0.648 at 4 warps per SM; 32 / 96-thread CTAs 0.608 / 0.607
  static const int oaa_max = getenv("GT_OAA_MAXLEVEL") ? atoi(getenv("GT_OAA_MAXLEVEL")) : 99;  // A/B
  static const int oaa_ctas = getenv("GT_OAA_CTAS") ? atoi(getenv("GT_OAA_CTAS")) : 0;          // A/B
  static const bool early_after_count = getenv("GT_OAA_AFTER_COUNT") != nullptr;              // A/B
  static const int oaa_tpb = getenv("GT_OAA_TPB") ? atoi(getenv("GT_OAA_TPB")) : 64;            // A/B
  // the share of a partition's entry pairs drawn early (the rest inline in
  // the partition) for partitions over >= oaa_split_min entries: at C2's last
  // partition (32 entries) the early lanes are on the critical path (pausing
  // them during the divisions costs 7 %); drawing 13 of its 16 pairs early and
  // 3 inline: 0.5595 -> 0.554 ms (same-call A/B; 69-81 % tie, 50 / 88 % and
  // splitting the 16-entry partition too are slower)
  static const int oaa_split_pct = getenv("GT_OAA_SPLITPCT") ? atoi(getenv("GT_OAA_SPLITPCT")) : 80;  // A/B
  static const int oaa_split_min = getenv("GT_OAA_SPLITMIN") ? atoi(getenv("GT_OAA_SPLITMIN")) : 32;    // A/B
  auto oaa_qe = [&](int m) -> int {
    const int mh = (m + 1) / 2;
    if (m < oaa_split_min || oaa_split_pct >= 100) return mh;
    return std::max(1, (mh * oaa_split_pct + 99) / 100);
  };
  if (early_oaa) GT_CUDA_CHECK(cudaMemsetAsync(ws + L.oaactr, 0, 16 * sizeof(uint64_t), s));
  auto early_oaa_launch = [&](int level) -> int {
    const bool early_next = early_oaa && level >= 1 && level + 1 < c.depth && level + 1 <= oaa_max && N;
    if (!early_next) return GT_OK;
    cudaStream_t os = s;
    if (!prof && !no_side) {
      int rc = stream_after(side->lo, s, side->eo[0]);
      if (rc) return rc;
      os = side->lo;
    }
    const int m = 1 << level;
    const uint64_t thr = N * (uint64_t)(m / 2);
    const uint64_t per_cta = (uint64_t)oaa_tpb * OAA_CHUNK;
    uint64_t grid = std::min<uint64_t>((thr + per_cta - 1) / per_cta, (uint64_t)(16 * 32 / oaa_tpb) * num_sms);
    if (oaa_ctas > 0) grid = std::min<uint64_t>(grid, (uint64_t)oaa_ctas);
    k_oaa_early<<<(unsigned)grid, oaa_tpb, 0, os>>>(midx, ws + L.oaa, N, m, c.sample_base, K,
                                                   op_id(level + 1, SITE_PART_OAA),
                                                   reinterpret_cast<unsigned long long*>(ws + L.oaactr) + level,
                                                   oaa_qe(m));
    GT_LAUNCH_CHECK("k_oaa_early");
    P.count_launch();
    if (os != s) {
      GT_CUDA_CHECK(cudaEventRecord(side->eo[1], side->lo));
      oaa_forked = true;
    }
    oaa_ready = true;
    return GT_OK;
  };
  for (int level = 0; level < c.depth; ++level) {
    const int n_h = 1 << level;
    const uint64_t swords = 3ull * n_h * (W + 1);
    if (level > 0 && N) {  // the partition also zeroes this level's count sums
      const uint64_t* ca = nullptr;
      if (oaa_ready) {
        ca = ws + L.oaa;
        if (oaa_forked) GT_CUDA_CHECK(cudaStreamWaitEvent(s, side->eo[1], 0));
        oaa_forked = oaa_ready = false;
      }
      P.start();
      PartAux aux{S, swords, c.count_engine == 0 ? ws + L.leaf : nullptr, f[cur], n_h, op_id(level, SITE_ISLEAF)};
      int rc = launch_partition(features, midx, T, slots, n_h / 2, c.nf, N, c.sample_base, K, level, s, num_sms, aux,
                                ca, oaa_qe(n_h / 2));
      if (rc) return rc;
      P.stop(Prof::PARTITION);
      if (!early_after_count) {
        int rc2 = early_oaa_launch(level);
        if (rc2) return rc2;
      }
    }
    if (!(level == 0 && count0_done)) {  // level 0 may already be counted chunk by chunk (host operands)
      if (!(level > 0 && N)) GT_CUDA_CHECK(cudaMemsetAsync(S, 0, swords * sizeof(uint64_t), s));
      if (N) {
        int rc = count_range(level, cur, 0, N);
        if (rc) return rc;
      }
    }
    if (c.count_engine == 1 && (c.count_reshare == 0 ? N > 0 : c.sample_base == 0)) {  // tensor engine: in k_count_mma
      const int cells = n_h * (int)W;
      k_count_alpha<<<(cells + 127) / 128, 128, 0, s>>>(S, n_h, c.nf, K, op_id(level, SITE_COUNT), c.count_reshare,
                                                       c.sample_base, c.sample_base + N);
      GT_LAUNCH_CHECK("k_count_alpha");
      P.count_launch();
    }
    if (early_after_count) {
      int rc = early_oaa_launch(level);
      if (rc) return rc;
    }
    if (allreduce) {
      int rc = allreduce(S, swords, stream, allreduce_user);
      if (rc) return fail_inval("allreduce callback failed");
    }
    bool last = level == c.depth - 1;
    NodeArgs na{};
    na.S = S;
    na.cst = cst[cur];
    na.f = f[cur];
    na.gam = gam[cur];
    na.ceff_prev = ceff[cur ^ 1];
    na.ceff = ceff[cur];
    na.hc = hc;
    na.dv = ws + L.dv;
    na.co_out = tee ? ws + L.co : nullptr;
    na.feattape = (!tee && tape_words && feat_tape_words(c))
                      ? reinterpret_cast<const W2*>(ws + L.feattape) + ((1ull << level) - 1) * (uint64_t)c.nf * FEAT_BLOCKS
                      : nullptr;
    na.nodetape = (!tee && tape_words) ? reinterpret_cast<const W2*>(ws + L.nodetape) +
                                           ((1ull << level) - 1) * (uint64_t)node_tape_plan(c.nf).total
                                     : nullptr;
    na.posttape = post_tape_words(c) ? reinterpret_cast<const W2*>(ws + L.posttape) +
                                           ((1ull << level) - 1) * (uint64_t)post_tape_blocks_w(c.score_width, c.nf)
                                     : nullptr;
    na.divtape = tape_words ? reinterpret_cast<const W2*>(ws + L.divtape) +
                                  div_tape_level_off(level, c.nf, c.score_width == 32 ? div_tape_blocks<32>(d)
                                                                                      : div_tape_blocks<64>(d))
                            : nullptr;
    na.n_h = n_h;
    na.nf = c.nf;
    na.level = level;
    na.last = last;
    na.shift = shift;
    na.tau = c.tau;
    na.d = d;
    na.K = K;
    {
      static const int ts = getenv("GT_HC_TIMING") ? 1 : 0;
      na.ts = ts;
    }
    P.start();
    if (tape_forked) {
      int rc = stream_after(s, side->st, side->ev[7]);
      if (rc) return rc;
      tape_forked = false;
    }
    const bool fuse = !last && !tee && c.policy == 0;
    int rc = c.score_width == 32 ? launch_node_hc<32>(na, s, fuse) : launch_node_hc<64>(na, s, fuse);
    if (rc) return rc;
    P.stop(Prof::NODE_HC);
    if (!last && !tee) {  // k_hc_div unless fused into k_hc_pre (+ k_hc_post unless fused into the finish launch)
      if (!hc_div_fused(na)) P.count_launch();
      if (!fuse) P.count_launch();
    }
    if (!last && tee) {
      int hrc = heuristic(1, level, n_h, c.nf, ws + L.co, gam[cur], f[cur], hc, stream, heuristic_user);
      if (hrc) return fail_inval("trusted helper (split) failed");
    }
    if (!last && c.policy == 1) {
      const int stop_smem = 6 * n_h;
      if (stop_smem > 48 * 1024)
        GT_CUDA_CHECK(cudaFuncSetAttribute(k_node_stop, cudaFuncAttributeMaxDynamicSharedMemorySize, stop_smem));
      k_node_stop<<<1, 256, stop_smem, s>>>(hc, n_h, K, op_id(level, SITE_STOP), ws + L.stop);
      GT_LAUNCH_CHECK("k_node_stop");
      P.count_launch();
      uint64_t flag = 0;
      GT_CUDA_CHECK(cudaMemcpyAsync(&flag, ws + L.stop, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      GT_CUDA_CHECK(cudaStreamSynchronize(s));
      if (flag) last = true;
    }
    FinishArgs fa{};
    fa.hc = hc;
    fa.ceff = ceff[cur];
    fa.f = f[cur];
    fa.filler = filler;
    fa.T = T;
    fa.F = F;
    fa.f_nxt = f[cur ^ 1];
    fa.gam_nxt = gam[cur ^ 1];
    fa.cst_nxt = cst[cur ^ 1];
    fa.lab = nullptr;
    if (last && tee) {
      int hrc = heuristic(2, level, n_h, c.nf, ceff[cur], nullptr, nullptr, ws + L.lab, stream, heuristic_user);
      if (hrc) return fail_inval("trusted helper (labels) failed");
      fa.lab = ws + L.lab;
    }
    fa.slots = slots;
    fa.ts = na.ts;
    fa.nodetape = na.nodetape;
    fa.n_h = n_h;
    fa.nf = c.nf;
    fa.level = level;
    fa.labels = last;
    fa.K = K;
    P.start();
    if (fuse) {
      const int psm = c.score_width == 32 ? post_smem_bytes<32>(na) : post_smem_bytes<64>(na);
      {  // always opt in: the kernel's static shared memory counts against the 48 KB default
        if (c.score_width == 32)
          GT_CUDA_CHECK(cudaFuncSetAttribute(k_hc_post_finish<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, psm));
        else
          GT_CUDA_CHECK(cudaFuncSetAttribute(k_hc_post_finish<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, psm));
      }
      const int rc = c.score_width == 32
                         ? launch_chain(k_hc_post_finish<32>, dim3(n_h), dim3(256), (size_t)psm, s, nullptr, na, fa)
                         : launch_chain(k_hc_post_finish<64>, dim3(n_h), dim3(256), (size_t)psm, s, nullptr, na, fa);
      if (rc) return rc;
    } else {
      const int rc = launch_chain(k_node_finish, dim3(n_h), dim3(128), 0, s, nullptr, fa);
      if (rc) return rc;
    }
    GT_LAUNCH_CHECK("k_node_finish");
    P.stop(Prof::NODE_FINISH);
    cur ^= 1;
    if (last) {
      trained = level + 1;
      break;
    }
  }
  if (oaa_forked) GT_CUDA_CHECK(cudaStreamWaitEvent(s, side->eo[1], 0));  // a grow stop left one unjoined
  if (hin) {
    GT_CUDA_CHECK(cudaMemcpyAsync(hin->T, T, 3 * slots * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    GT_CUDA_CHECK(cudaMemcpyAsync(hin->F, F, 3 * slots * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  }
  if (depth_out) *depth_out = trained;
  return P.finish();
}

int gt_train_ex(const gt_train_cfg* cfg, const uint64_t* features, const uint64_t* labels, const uint64_t* filler,
                uint64_t* T, uint64_t* F, int32_t* depth_out, void* workspace, uint64_t workspace_bytes,
                const gt_keys* keys, gt_allreduce_fn allreduce, void* allreduce_user, gt_heuristic_fn heuristic,
                void* heuristic_user, void* stream, gt_train_profile* prof) {
  return train_impl(cfg, features, labels, filler, T, F, depth_out, workspace, workspace_bytes, keys, allreduce,
                    allreduce_user, heuristic, heuristic_user, stream, prof, nullptr);
}

uint64_t gt_train_host_workspace_bytes(const gt_train_cfg* cfg) {
  if (!cfg || cfg->depth < 1 || cfg->depth > 16 || cfg->nf < 1 || cfg->nf > 64) return 0;
  return layout(*cfg, true).total * sizeof(uint64_t);
}

int gt_train_host(const gt_train_cfg* cfg, const uint64_t* features_h, const uint64_t* labels_h,
                  const uint64_t* filler_h, uint64_t* T_h, uint64_t* F_h, int32_t* depth_out, void* workspace,
                  uint64_t workspace_bytes, const gt_keys* keys, gt_allreduce_fn allreduce, void* allreduce_user,
                  void* stream) {
  if (cfg && cfg->heuristic != 0) return fail_inval("gt_train_host: heuristic mpc only (use gt_train_ex for tee)");
  const HostIn hin{features_h, labels_h, filler_h, T_h, F_h};
  return train_impl(cfg, nullptr, nullptr, nullptr, nullptr, nullptr, depth_out, workspace, workspace_bytes, keys,
                    allreduce, allreduce_user, nullptr, nullptr, stream, nullptr, &hin);
}

// diagnostics: the fused count's phase timestamps of the last GT_COUNT_TS run (ns)
int gt_diag_count_timestamps(unsigned long long* out, int n) {
  if (!out || n < 0 || n > 128) return fail_inval("gt_diag_count_timestamps: bad output");
  GT_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_cnt_ts, sizeof(unsigned long long) * n));
  return GT_OK;
}

// diagnostics: the heuristic phase timestamps of the last GT_HC_TIMING run (ns)
int gt_diag_hc_timestamps(unsigned long long* out, int n) {
  if (!out || n < 0 || n > 128) return fail_inval("gt_diag_hc_timestamps: bad output");
  GT_CUDA_CHECK(cudaMemcpyFromSymbol(out, g_hc_ts, sizeof(unsigned long long) * n));
  return GT_OK;
}

}  // extern "C"
