// Tensor-core count contraction (count_engine 0): tcgen05.mma kind::i8 over
// an INT8 limb decomposition of the Z_2^64 share products.
//
// The count contraction of one level (_count_level, reference
// pkg/src/obtree/train.py:201-229) is, per share component i, the ring GEMM
//     S_i[n][w] = sum_s la_i x_i + la_i x_{i+1} + la_{i+1} x_i
// (the party-local cross terms of mul(cols, la), rss.py:391-395).  Writing
// every u64 as 8 unsigned bytes, a * b mod 2^64 = sum_{p+q<=7} a_p b_q
// 2^{8(p+q)}, so with rows (node n, limb p) and columns (column w, limb q)
//     D_i[(n,p)][(w,q)] = sum_s la_i,p x_i,q + la_i,p x_{i+1},q + la_{i+1},p x_i,q   (u8 x u8 -> s32)
//     S_i[n][w]         = sum_{p+q<=7} D_i[(n,p)][(w,q)] << 8(p+q)   (mod 2^64)
// One CTA holds the three components' accumulators D_0, D_1, D_2 in TMEM
// (M = 128 rows = 16 nodes x 8 limbs, N = 8 x columns of the block each), so
// every operand plane is streamed once per (M tile, column block): nine UMMAs
// per 32-sample K step over three la planes and three x planes.  Each CTA
// sums at most 64 x 128 samples, so every D entry stays below
// 3 x 8192 x 255^2 < 2^31 (exact in the s32 accumulator).  The mask column
// s_mask = sum_s la (train.py:220) is summed by the lane kernel.
//
// Operands are staged by cp.async.bulk in the canonical K-major
// SWIZZLE_NONE core-matrix layout (8 rows x 16 bytes = 128 contiguous bytes;
// SBO = 128 B between 8-row groups, LBO between the 16-byte K chunks), which
// the producer kernels write directly, so one half block (64 samples) of the
// three components of an operand is one contiguous bulk copy.
#pragma once

namespace gt {
namespace {

constexpr int TC_KB = 128;                // samples per K block
constexpr int TC_ABLK = TC_KB * 128;      // bytes of an A block: 128 rows (16 nodes x 8 limbs) x 128 samples
constexpr int TC_MAX_KB_PER_CTA = 64;     // 3 products x 64 x 128 x 255^2 < 2^31
constexpr int TC_TMEM_COLS = 512;         // three accumulators of N <= 160 columns

// node groups per 16-sample chunk of the la planes: min(16, n_h)
__host__ __device__ inline int tc_groups(int n_h) { return n_h < 16 ? n_h : 16; }
// 64-sample half blocks per lane-kernel CTA: 256-512 (node, sample pair)
// items for its 256 threads -- small CTAs, so the last wave is short
__host__ __device__ inline int tc_lane_hpc(int n_h) { return tc_groups(n_h) < 8 ? 8 / tc_groups(n_h) : 1; }

struct TcPlan {
  int CW;      // sample columns W (the mask column is summed by the lane kernel)
  int nbn;     // column blocks
  int cpb;     // columns per block (even)
  int N;       // UMMA N = 8 * cpb (multiple of 16, <= 160: three accumulators fit TMEM)
  int mtiles;  // 16-node M tiles
  int BB;      // bytes of one component's x plane of a K block (N rows x 128 samples)
};
inline TcPlan tc_plan(int nf, int n_h) {
  TcPlan p;
  p.CW = 2 * nf + 1;
  p.nbn = (p.CW + 19) / 20;
  p.cpb = (p.CW + p.nbn - 1) / p.nbn;
  p.cpb += p.cpb & 1;
  if (p.nbn == 2) p.cpb = 16;  // 21..32 columns: two 16-column blocks, the A halves of the fused CTA pair
  p.N = 8 * p.cpb;
  p.mtiles = (n_h + 15) / 16;
  p.BB = p.N * TC_KB;
  return p;
}

// --- B operand: the level-invariant sample columns as byte planes
// X8[nb][kb][half 2][c 3][kc 4][g cpb][q 8][16 samples]: the three
// components' x planes of a 64-sample half block are one contiguous run.
// Fused prologue for the tensor engine (count:0 prods + the x planes): one CTA
// per 128-sample K block stages the block's features and labels in shared
// memory (coalesced rows), forms count:0's prods = mul(features, labels)
// (train.py:115-116, same Philox schedule as k_prods) next to them, and
// writes the U / X byte planes straight from shared memory: the u64 column
// matrix never goes through HBM.
struct Prep8Args {
  const uint64_t *X, *Y;  // [3][N][nf], [3][N]
  uint8_t* B8;
  uint64_t N, nkb, base, hb0;  // hb0: first 64-sample half block of this launch
  int nf, W, cpb, nbn;
  int mask_cols;  // columns W, W+1 = the public constant 1 as shares (1,0,0) / (0,1,0) (k_count_fused's mask sums)
  Keys K;
  uint32_t op_prods;
};
// 6 CTAs per SM (40 registers): C2 0.5808 vs 0.5846 ms at the default 48
// registers / 5 CTAs (same-call A/B; 8 CTAs at 32 registers: 0.5830)
#ifndef GT_PREP8_MINB
#define GT_PREP8_MINB 6
#endif
__global__ void __launch_bounds__(256, GT_PREP8_MINB) k_prep8(Prep8Args a) {
  // one CTA per 32-sample quarter block (chunks kc = 2 sub, 2 sub + 1 of a
  // 64-sample half block: a grid of many small CTAs leaves no near-empty
  // second wave); shared memory (<= 99 KB at nf = 64): xs[3][HS][nf]
  // features, ps[3][HS][nf] prods, ys[3][HS] labels
  constexpr int HS = TC_KB / 4;
  extern __shared__ __align__(16) uint64_t v[];
  __shared__ __align__(8) uint64_t bar;
  const int nf = a.nf, W = a.W, tid = threadIdx.x;
  uint64_t* xs = v;
  uint64_t* ps = v + 3 * HS * nf;
  uint64_t* ys = v + 6 * HS * nf;
  const uint64_t qb = 2 * a.hb0 + blockIdx.x;
  const uint64_t hb = qb >> 1;
  const uint64_t kb = hb >> 1;
  const int half = (int)(hb & 1), sub = (int)(qb & 1);
  const uint64_t nfx = a.N * (uint64_t)nf;
  const uint64_t s0 = kb * TC_KB + half * (TC_KB / 2) + sub * HS;
  const int cnt = s0 < a.N ? (int)min((uint64_t)HS, a.N - s0) : 0;  // 0: a half block's empty tail quarter
  // the block's feature rows and labels are contiguous runs: bulk copies when
  // every run is 16-byte aligned, plain loads otherwise
  const bool bulk = cnt > 0 && ((reinterpret_cast<uintptr_t>(a.X) | reinterpret_cast<uintptr_t>(a.Y)) & 15) == 0 &&
                    ((nfx | a.N | (uint64_t)cnt * nf | (uint64_t)cnt) & 1) == 0;
  if (bulk) {
    if (tid == 0) {
      mbar_init(&bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      const uint32_t xb = (uint32_t)(cnt * nf * 8), yb = (uint32_t)(cnt * 8);
      mbar_expect_tx(&bar, 3 * (xb + yb));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        bulk_g2s(xs + c * HS * nf, a.X + c * nfx + s0 * nf, xb, &bar);
        bulk_g2s(ys + c * HS, a.Y + c * a.N + s0, yb, &bar);
      }
    }
    __syncthreads();
    mbar_wait(&bar, 0);
  } else {
    for (int e = tid; e < cnt * nf; e += blockDim.x) {
#pragma unroll
      for (int c = 0; c < 3; ++c) xs[c * HS * nf + e] = __ldg(a.X + c * nfx + s0 * nf + e);
    }
    for (int sl = tid; sl < cnt; sl += blockDim.x) {
#pragma unroll
      for (int c = 0; c < 3; ++c) ys[c * HS + sl] = __ldg(a.Y + c * a.N + s0 + sl);
    }
    __syncthreads();
  }
  // one thread per (sample, feature pair): features 2j and 2j+1 take the two
  // words of the same Philox block per key (mul's schedule), drawn once
  const int nfp = (nf + 1) >> 1;
  for (int e = tid; e < cnt * nfp; e += blockDim.x) {
    const int sl = (int)((uint32_t)e / (uint32_t)nfp), fp = e - sl * nfp, f0 = 2 * fp;
    W2 Z[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) Z[i] = word2(a.K.pair[i], a.op_prods, 0, (uint32_t)fp, a.base + s0 + sl);
    const A3 y = a3(ys[sl], ys[HS + sl], ys[2 * HS + sl]);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int f = f0 + h;
      if (f >= nf) break;
      const int ef = sl * nf + f;
      const uint64_t F[3] = {h ? Z[0].b : Z[0].a, h ? Z[1].b : Z[1].a, h ? Z[2].b : Z[2].a};
      const A3 z = mul_z<64>(a3(xs[ef], xs[HS * nf + ef], xs[2 * HS * nf + ef]), y, F);
#pragma unroll
      for (int c = 0; c < 3; ++c) ps[c * HS * nf + ef] = z.v[c];
    }
  }
  __syncthreads();
  // planes: item = (component, 16-sample chunk, column, 4-sample quad); the
  // quad's x words are byte-transposed in registers (4x4 byte_perm
  // transposes) into one 32-bit word of each of the 8 limb rows; the four
  // quads of a row are adjacent threads
  // thread t owns (column g, quad) = t % (4 cpb) and walks the (component,
  // column block, 16-sample chunk) combinations: one division per thread
  const uint64_t HBX = (uint64_t)8 * a.cpb * (TC_KB / 2);
  // (unsigned index math: the runtime divisors cost half the instructions)
  const uint32_t gq = 4u * (uint32_t)a.cpb, combos = 3u * (uint32_t)a.nbn * 2u, nbn = (uint32_t)a.nbn;
  const int g = (int)(((uint32_t)tid % gq) >> 2), quad = tid & 3;
  for (uint32_t cb = (uint32_t)tid / gq; cb < combos; cb += blockDim.x / gq) {
    const int kc = 2 * sub + (int)(cb & 1);
    const uint32_t r = cb >> 1;
    const int nb = (int)(r % nbn), c = (int)(r / nbn);
    const int w = nb * a.cpb + g;
    const uint64_t* p0 = nullptr;
    int stride = nf;
    if (w < nf) p0 = xs + c * HS * nf + w;
    else if (w < 2 * nf) p0 = ps + c * HS * nf + (w - nf);
    else if (w == 2 * nf) p0 = ys + c * HS, stride = 1;
    // the mask columns: component c of the constant is 1 in column W + c (c < 2)
    const uint64_t cval = (a.mask_cols && (w == a.W || w == a.W + 1) && c == w - a.W) ? 1ull : 0ull;
    uint32_t wx[2][4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int sl = (kc & 1) * 16 + quad * 4 + i;
      const uint64_t x = sl < cnt ? (p0 ? p0[sl * stride] : cval) : 0ull;
      wx[0][i] = (uint32_t)x, wx[1][i] = (uint32_t)(x >> 32);
    }
    uint8_t* dst = a.B8 + (((uint64_t)nb * a.nkb + kb) * 2 + half) * 3 * HBX + c * HBX +
                   ((uint64_t)kc * a.cpb + g) * 128 + quad * 4;
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const uint32_t* q4 = wx[hh];
      const uint32_t t0 = __byte_perm(q4[0], q4[1], 0x5140), t1 = __byte_perm(q4[0], q4[1], 0x7362);
      const uint32_t t2 = __byte_perm(q4[2], q4[3], 0x5140), t3 = __byte_perm(q4[2], q4[3], 0x7362);
      uint8_t* d = dst + hh * 4 * 16;
      *reinterpret_cast<uint32_t*>(d) = __byte_perm(t0, t2, 0x5410);
      *reinterpret_cast<uint32_t*>(d + 16) = __byte_perm(t0, t2, 0x7632);
      *reinterpret_cast<uint32_t*>(d + 32) = __byte_perm(t1, t3, 0x5410);
      *reinterpret_cast<uint32_t*>(d + 48) = __byte_perm(t1, t3, 0x7632);
    }
  }
}

// --- A operand: one CTA per (128-sample block, 16-node M tile) of a chunk;
// lanes la = b2a(eq(m_idx, off+n) & is_leaf[n]) (train.py:214-217, the same
// randomness as k_count_lanes: count_lane_pair), two samples of one node
// per work item so each limb row leaves as one packed 32-bit word; the byte
// planes la8[mt][kbc][half][c][kc 4][g 16][p 8][16] are stored straight from
// registers (each warp store covers whole 32-byte sectors).  is_leaf of the tile's 16 nodes (train.py:206) is drawn
// in the CTA (it is keyed by node only).
struct Lanes8Args {
  const uint64_t *midx, *f;
  uint8_t* la8;
  uint64_t* S;  // [3][n_h][W+1]: the mask column s_mask[n] = sum_s la (train.py:220)
  int W;
  const uint64_t* leafbits;  // is_leaf [3][n_h] precomputed by the partition launch, or null: draw per CTA
  uint64_t N, s0, cn, base, nkbc;  // nkbc = chunk capacity in K blocks
  int n_h, off, mtiles;
  Keys K;
  uint32_t op_cnt, op_leaf;
};
#ifndef GT_LANES8_MINB
#define GT_LANES8_MINB 1
#endif
__global__ void __launch_bounds__(256, GT_LANES8_MINB) k_count_lanes8(Lanes8Args a) {
  __shared__ uint64_t leaf[3][16];
  const int mt = blockIdx.y, tid = threadIdx.x;
  pdl_wait();
  pdl_trigger();
  // la8[mt][kbc][half 2][c 3][kc 4][g NG][p 8][16], NG = min(16, n_h) node
  // groups: the three components of a 64-sample half block are one
  // contiguous 1.5 NG KB run (one bulk copy for the contraction).  A CTA
  // covers HPC half blocks (tc_lane_hpc).
  const int NG = tc_groups(a.n_h), HPC = tc_lane_hpc(a.n_h);
  const uint64_t cstride = 512ull * NG;
  if (tid < 16) {
    const int n = mt * 16 + tid;
    B3 z = {{0, 0, 0}};
    if (n < a.n_h && a.leafbits) {
#pragma unroll
      for (int c = 0; c < 3; ++c) z.v[c] = a.leafbits[c * a.n_h + n];
    } else if (n < a.n_h) {
      z = eqz<64>(a.K, a.op_leaf, 0, (uint64_t)n, add_pub<64>(ld3s(a.f, a.n_h, n), 0ull - F_LEAF));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) leaf[c][tid] = z.v[c] & 1ull;
  }
  __syncthreads();
  // one PAIR of samples per thread (their zero words share a pair block); a
  // warp = 64 consecutive samples of one node.  Threads t, t^1 hold samples
  // 4k..4k+3: limb bytes are packed with byte permutes, one shuffle pair per
  // component, and the even thread stores limbs 0..3 of the 4 samples, the
  // odd thread limbs 4..7, one 32-bit word each.
  const bool odd = threadIdx.x & 1;
  for (int e = tid; e < HPC * NG * (TC_KB / 4); e += blockDim.x) {
    const int hbl = e / (NG * (TC_KB / 4)), r = e - hbl * NG * (TC_KB / 4);
    const uint64_t hb = (uint64_t)blockIdx.x * HPC + hbl;
    if (hb >= 2 * a.nkbc) break;  // warp-uniform (a warp's items share hbl)
    const uint64_t kb = hb >> 1;
    const int nn = r / (TC_KB / 4), s2 = (int)(hb & 1) * (TC_KB / 2) + (r % (TC_KB / 4)) * 2;
    uint8_t* blk = a.la8 + ((uint64_t)mt * a.nkbc + kb) * (3072ull * NG);
    const int n = mt * 16 + nn;
    const uint64_t s = kb * TC_KB + s2;
    A3 l0 = a3(0, 0, 0), l1 = a3(0, 0, 0);
    if (n < a.n_h && s < a.cn) {
      const uint64_t gs = a.s0 + s;
      const bool v1 = s + 1 < a.cn;
      const uint64_t off = 0ull - (uint64_t)(a.off + n);
      const A3 d0 = add_pub<64>(a3(__ldg(a.midx + gs), __ldg(a.midx + a.N + gs), __ldg(a.midx + 2 * a.N + gs)), off);
      A3 d1 = a3(0, 0, 0);
      if (v1)
        d1 = add_pub<64>(a3(__ldg(a.midx + gs + 1), __ldg(a.midx + a.N + gs + 1), __ldg(a.midx + 2 * a.N + gs + 1)), off);
      B3 lf;
#pragma unroll
      for (int c = 0; c < 3; ++c) lf.v[c] = leaf[c][nn];
      count_lane_pair(a.K, a.op_cnt, a.base + gs, a.n_h, n, d0, d1, true, v1, lf, &l0, &l1);
    }
    {  // s_mask: the warp's 64 samples of node n, one atomic per component
      // (l1 of a pair past the chunk's end is padding: multiplied by zero
      // columns in the contraction, left out here)
      const bool has1 = kb * TC_KB + s2 + 1 < a.cn;
      A3 m = has1 ? add<64>(l0, l1) : l0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1)
#pragma unroll
        for (int c = 0; c < 3; ++c) m.v[c] += __shfl_xor_sync(0xffffffffu, m.v[c], o);
      if ((tid & 31) == 0 && n < a.n_h)
#pragma unroll
        for (int c = 0; c < 3; ++c)
          atomicAdd((unsigned long long*)&a.S[((uint64_t)c * a.n_h + n) * (a.W + 1) + a.W], (unsigned long long)m.v[c]);
    }
    const int o = (s2 >> 6) * (1536 * NG) + ((((s2 >> 4) & 3) * NG + nn) * 8) * 16 + ((s2 & ~3) & 15);
    const int p0 = odd ? 4 : 0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const uint32_t a_lo = (uint32_t)l0.v[c], a_hi = (uint32_t)(l0.v[c] >> 32);
      const uint32_t b_lo = (uint32_t)l1.v[c], b_hi = (uint32_t)(l1.v[c] >> 32);
      const uint32_t P01 = __byte_perm(a_lo, b_lo, 0x5140), P23 = __byte_perm(a_lo, b_lo, 0x7362);
      const uint32_t P45 = __byte_perm(a_hi, b_hi, 0x5140), P67 = __byte_perm(a_hi, b_hi, 0x7362);
      const uint32_t r0 = __shfl_xor_sync(0xffffffffu, odd ? P01 : P45, 1);
      const uint32_t r1 = __shfl_xor_sync(0xffffffffu, odd ? P23 : P67, 1);
      uint32_t w[4];
      if (!odd) {
        w[0] = __byte_perm(P01, r0, 0x5410);
        w[1] = __byte_perm(P01, r0, 0x7632);
        w[2] = __byte_perm(P23, r1, 0x5410);
        w[3] = __byte_perm(P23, r1, 0x7632);
      } else {
        w[0] = __byte_perm(r0, P45, 0x5410);
        w[1] = __byte_perm(r0, P45, 0x7632);
        w[2] = __byte_perm(r1, P67, 0x5410);
        w[3] = __byte_perm(r1, P67, 0x7632);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) *reinterpret_cast<uint32_t*>(blk + c * cstride + o + (p0 + i) * 16) = w[i];
    }
  }
}

// --- UMMA plumbing
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  // K-major SWIZZLE_NONE: start>>4 [0,14), LBO>>4 [16,30), SBO>>4 [32,46),
  // version 1 [46,48), base offset 0, layout type 0 [61,64)
  return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__device__ __forceinline__ void umma_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate), "r"(0), "r"(0), "r"(0), "r"(0)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

struct MmaArgs {
  const uint8_t *la8, *B8;
  uint64_t* S;  // [3][n_h][W+1]
  Keys K;
  uint32_t op_cnt;
  int alpha;            // 0: none, 1: telescoped elementwise reshare sums, 2: dot-product reshare
  const uint64_t* alpha_tab;  // this level's precomputed sums [n][3][W] (k_alpha_tape) or null: draw them
  uint64_t t0, t1;      // shard sample range for the telescoped sums
  uint64_t nkbc, nkb_total, kb_base;  // chunk capacity (blocks), shard blocks, chunk's first global block
  uint32_t nkb;                       // blocks in this chunk
  int n_h, W, cpb, nbn, mtiles, N, nkr;
  int probe;  // diagnostics only (GT_MMA_PROBE): 1 = loads without MMAs, 2 = MMAs without loads, 3 = neither
};

// One CTA per (K range, M tile, column block): the party-local cross terms
// of all three components
//     D_c = A_c X_c + A_c X_{c+1} + A_{c+1} X_c        (rss.py:391-395)
// A stage is one 64-sample half block brought by TWO contiguous bulk copies
// (the three components' la planes, 24 KB; the three components' x planes,
// 3 x N x 64 B), four stages in flight: bulk copies pay a fixed latency each,
// so few large requests with several in flight keep the SM's copy engine
// streaming.
constexpr int TC_MC_STAGES = 4;
constexpr int TC_A_HB = 3 * TC_ABLK / 2;  // the 3 components' la planes of a half block
__global__ void __launch_bounds__(256, 1) k_count_mma(MmaArgs a) {
  extern __shared__ __align__(1024) uint8_t smt[];
  __shared__ __align__(8) uint64_t full[TC_MC_STAGES], empty[TC_MC_STAGES], done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // grid (M tiles, column blocks x K ranges): the M tiles of one (K range,
  // column block) read the same x planes and are adjacent in launch order
  const int mt = blockIdx.x, nb = blockIdx.y % a.nbn, kr = blockIdx.y / a.nbn;
  const uint32_t per = (a.nkb + a.nkr - 1) / a.nkr;
  const uint32_t kb0 = kr * per, kb1 = min(a.nkb, kb0 + per);
  const int T = kb1 > kb0 ? 2 * (int)(kb1 - kb0) : 0;  // half blocks
  const int HBX = a.N * (TC_KB / 2);                    // one component's x plane of a half block
  const int stage = TC_A_HB + 3 * HBX;
  // la planes with NG node groups per 16-sample chunk (see k_count_lanes8):
  // the UMMA still reads 16 groups (M = 128); rows of absent nodes read
  // other chunks' bytes inside the stage and are never folded
  const int NG = tc_groups(a.n_h);
  const uint32_t AHB = 1536u * NG, ACS = 512u * NG, ALBO = 128u * NG;
  const int NS = (a.N + 31) & ~31;                      // accumulator column stride in TMEM

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(TC_TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int i = 0; i < TC_MC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // the epilogue's precomputed reshare sums (drawn before the level chain):
  // loaded now, so their latency hides behind the main loop
  uint64_t apre[4] = {0, 0, 0, 0};
  if (a.alpha && kr == 0 && a.alpha_tab) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int cell = tid + k * (int)blockDim.x;
      const int nc = cell & 15, cw = cell >> 4, w = cw % a.cpb, c = cw / a.cpb;
      const int n = mt * 16 + nc, wg = nb * a.cpb + w;
      if (cell < 3 * a.cpb * 16 && n < a.n_h && wg < a.W) apre[k] = a.alpha_tab[((uint64_t)n * 3 + c) * a.W + wg];
    }
  }
  pdl_wait();  // the lane planes of the lane kernel

  if (tid == 0 && T > 0 && a.probe < 3) {
    // idesc: S32 accumulator [4,6) = 2, A/B unsigned 8-bit, K-major, N>>3 at 17, M>>4 at 24
    const uint32_t idesc = (2u << 4) | ((uint32_t)(a.N >> 3) << 17) | ((128u >> 4) << 24);
    auto load = [&](int t) {
      const int st = t % TC_MC_STAGES;
      const uint64_t kb = kb0 + (uint32_t)(t >> 1), h = t & 1;
      uint8_t* sb = smt + st * stage;
      mbar_expect_tx(&full[st], AHB + (uint32_t)(3 * HBX));
      bulk_g2s(sb, a.la8 + (((uint64_t)mt * a.nkbc + kb) * 2 + h) * (uint64_t)AHB, AHB, &full[st]);
      bulk_g2s(sb + TC_A_HB, a.B8 + (((uint64_t)nb * a.nkb_total + a.kb_base + kb) * 2 + h) * (uint64_t)(3 * HBX),
               (uint32_t)(3 * HBX), &full[st]);
    };
    if (a.probe != 2)
      for (int t = 0; t < min(TC_MC_STAGES, T); ++t) load(t);
    for (int t = 0; t < T; ++t) {
      const int st = t % TC_MC_STAGES;
      if (a.probe != 2) mbar_wait(&full[st], (uint32_t)((t / TC_MC_STAGES) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = smem_u32(smt + st * stage);
      if (a.probe != 1)
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const uint32_t ao = j * 2 * ALBO, xo = j * 2 * (a.cpb * 128);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const int cn = (c + 1) % 3;
            const uint32_t Ac = base + c * ACS + ao, An = base + cn * ACS + ao;
            const uint32_t Xc = base + TC_A_HB + c * HBX + xo, Xn = base + TC_A_HB + cn * HBX + xo;
            const uint32_t D = tmem + (uint32_t)(c * NS);
            umma_i8(D, umma_desc(Ac, ALBO, 128), umma_desc(Xc, a.cpb * 128, 128), idesc, (t > 0 || j > 0) ? 1u : 0u);
            umma_i8(D, umma_desc(Ac, ALBO, 128), umma_desc(Xn, a.cpb * 128, 128), idesc, 1u);
            umma_i8(D, umma_desc(An, ALBO, 128), umma_desc(Xc, a.cpb * 128, 128), idesc, 1u);
          }
        }
      umma_commit(&empty[st]);
      // refill the previous stage (its MMAs were issued one step earlier)
      if (a.probe != 2 && t >= 1 && t - 1 + TC_MC_STAGES < T) {
        const int pst = (t - 1) % TC_MC_STAGES;
        mbar_wait(&empty[pst], (uint32_t)(((t - 1) / TC_MC_STAGES) & 1));
        load(t - 1 + TC_MC_STAGES);
      }
    }
    umma_commit(&done);
  }
  __syncwarp();
  if (T > 0 && a.probe < 3) mbar_wait(&done, 0);
  pdl_trigger();  // the epilogue overlaps the next kernel's launch
  if (T > 0 && a.probe < 4) {
    // epilogue: thread (node nn, limb p) = TMEM lane r forms, per column w,
    // R_p[w] = sum_q D[(nn,p)][(w,q)] << 8(p+q) from 64-column TMEM loads (8
    // columns each); the eight limb rows of a node are summed through shared
    // memory (the operand ring is idle now), one atomic per (component, node,
    // column)
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // warps w and w + 4 share TMEM lanes 32 (w % 4) ..: they split the loads
    const int r = (warp & 3) * 32 + lane, nn = r >> 3, p = r & 7, grp = warp >> 2;
    uint64_t* red = reinterpret_cast<uint64_t*>(smt);  // [3][cpb][16 nn][8 p]
    const int cpb = a.cpb, nchunk = NS / 64 + (NS % 64 ? 1 : 0);
    for (int it = grp; it < 3 * nchunk; it += 2) {
      const int c = it / nchunk, cb = (it % nchunk) * 64;
      {
        uint32_t d[64];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, %36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, %57, %58, %59, %60, %61, %62, %63}, [%64];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31]), "=r"(d[32]), "=r"(d[33]), "=r"(d[34]), "=r"(d[35]), "=r"(d[36]), "=r"(d[37]), "=r"(d[38]), "=r"(d[39]), "=r"(d[40]), "=r"(d[41]), "=r"(d[42]), "=r"(d[43]), "=r"(d[44]), "=r"(d[45]), "=r"(d[46]), "=r"(d[47]), "=r"(d[48]), "=r"(d[49]), "=r"(d[50]), "=r"(d[51]), "=r"(d[52]), "=r"(d[53]), "=r"(d[54]), "=r"(d[55]), "=r"(d[56]), "=r"(d[57]), "=r"(d[58]), "=r"(d[59]), "=r"(d[60]), "=r"(d[61]), "=r"(d[62]), "=r"(d[63])
            : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * NS + cb)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int wl = 0; wl < 8; ++wl) {
          // sum_q d_q << 8q with constant shifts, then << 8p (the terms with
          // p + q >= 8 leave the ring)
          uint64_t v = 0;
#pragma unroll
          for (int q = 0; q < 8; ++q) v += (uint64_t)d[8 * wl + q] << (8 * q);
          v <<= 8 * p;
          const int w = cb / 8 + wl;
          if (w < cpb) red[((c * cpb + w) * 16 + nn) * 8 + p] = v;
        }
      }
    }
    __syncthreads();
    const uint64_t Sstride = (uint64_t)a.n_h * (a.W + 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int cell = tid + k * (int)blockDim.x;
      if (cell >= 3 * cpb * 16) break;
      const int nc = cell & 15, cw = cell >> 4, w = cw % cpb, c = cw / cpb;
      const int n = mt * 16 + nc, wg = nb * cpb + w;
      if (n >= a.n_h || wg >= a.W) continue;
      const uint4* rp = reinterpret_cast<const uint4*>(red + (uint64_t)cell * 8);
      uint64_t v = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 x = rp[i];
        v += ((uint64_t)x.y << 32 | x.x) + ((uint64_t)x.w << 32 | x.z);
      }
      if (a.alpha && kr == 0 && a.alpha_tab) {
        v += apre[k];
      } else if (a.alpha && kr == 0) {
        // zero shares of the count products summed over the shard (see
        // k_count_alpha): alpha_c = F_c - F_{c-1}
        uint64_t F[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
          const Key& key = a.K.pair[q == 0 ? c : (c + 2) % 3];
          F[q] = a.alpha == 2 ? word(key, a.op_cnt, 4, (uint32_t)wg, (uint64_t)n)
                              : word(key, a.op_cnt, 3, (uint32_t)wg, a.t1 * (uint64_t)a.n_h + n) -
                                    word(key, a.op_cnt, 3, (uint32_t)wg, a.t0 * (uint64_t)a.n_h + n);
        }
        v += F[0] - F[1];
      }
      atomicAdd((unsigned long long*)&a.S[c * Sstride + (uint64_t)n * (a.W + 1) + wg], (unsigned long long)v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TC_TMEM_COLS) : "memory");
  }
}

// Shallow levels (n_h <= 8, at most 16 columns per block): the same contraction with the operand roles
// swapped -- the x planes are the UMMA A operand (M = 128 rows = column x limb
// of the block; rows past 8 cpb read neighbouring bytes and are never
// folded) and the compact la planes the B operand (N = 8 n_h node x limb
// columns, at least 16) -- so the UMMA floor max(M,128) N / 256 scales with
// the level's nodes instead of a fixed 16-node tile:
//     D_c[(w,q)][(n,p)] = sum_s x_c la_c + x_{c+1} la_c + x_c la_{c+1}
// Epilogue: thread (column g, limb q) folds sum_p D << 8p per node, shifts by
// 8q, and the 8 limb rows of a column are summed through shared memory.
__global__ void __launch_bounds__(256, 1) k_count_mma_t(MmaArgs a) {
  extern __shared__ __align__(1024) uint8_t smt[];
  __shared__ __align__(8) uint64_t full[TC_MC_STAGES], empty[TC_MC_STAGES], done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nb = blockIdx.y % a.nbn, kr = blockIdx.y / a.nbn;
  const uint32_t per = (a.nkb + a.nkr - 1) / a.nkr;
  const uint32_t kb0 = kr * per, kb1 = min(a.nkb, kb0 + per);
  const int T = kb1 > kb0 ? 2 * (int)(kb1 - kb0) : 0;
  const int HBX = a.N * (TC_KB / 2);
  const int stage = TC_A_HB + 3 * HBX;
  const int NG = tc_groups(a.n_h);
  const uint32_t AHB = 1536u * NG, ACS = 512u * NG, ALBO = 128u * NG;
  const int NT = NG * 8 < 16 ? 16 : NG * 8;  // UMMA N
  constexpr int TCOLS = 256;                  // three accumulators of <= 64 columns

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(TCOLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int i = 0; i < TC_MC_STAGES; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  uint64_t apre[2] = {0, 0};  // the epilogue's reshare sums, loaded early (see k_count_mma)
  if (a.alpha && kr == 0 && a.alpha_tab) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int cell = tid + k * (int)blockDim.x;
      const int g = cell & 15, cn = cell >> 4, n = cn % NG, c = cn / NG;
      const int wg = nb * a.cpb + g;
      if (cell < 3 * NG * 16 && g < a.cpb && n < a.n_h && wg < a.W)
        apre[k] = a.alpha_tab[((uint64_t)n * 3 + c) * a.W + wg];
    }
  }
  pdl_wait();

  if (tid == 0 && T > 0) {
    const uint32_t idesc = (2u << 4) | ((uint32_t)(NT >> 3) << 17) | ((128u >> 4) << 24);
    auto load = [&](int t) {
      const int st = t % TC_MC_STAGES;
      const uint64_t kb = kb0 + (uint32_t)(t >> 1), h = t & 1;
      uint8_t* sb = smt + st * stage;
      mbar_expect_tx(&full[st], AHB + (uint32_t)(3 * HBX));
      bulk_g2s(sb, a.la8 + (kb * 2 + h) * (uint64_t)AHB, AHB, &full[st]);  // one M tile (n_h <= 8)
      bulk_g2s(sb + TC_A_HB, a.B8 + (((uint64_t)nb * a.nkb_total + a.kb_base + kb) * 2 + h) * (uint64_t)(3 * HBX),
               (uint32_t)(3 * HBX), &full[st]);
    };
    for (int t = 0; t < min(TC_MC_STAGES, T); ++t) load(t);
    for (int t = 0; t < T; ++t) {
      const int st = t % TC_MC_STAGES;
      mbar_wait(&full[st], (uint32_t)((t / TC_MC_STAGES) & 1));
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t base = smem_u32(smt + st * stage);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const uint32_t ao = j * 2 * ALBO, xo = j * 2 * (a.cpb * 128);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int cn = (c + 1) % 3;
          const uint32_t Ac = base + c * ACS + ao, An = base + cn * ACS + ao;
          const uint32_t Xc = base + TC_A_HB + c * HBX + xo, Xn = base + TC_A_HB + cn * HBX + xo;
          const uint32_t D = tmem + (uint32_t)(c * 64);
          umma_i8(D, umma_desc(Xc, a.cpb * 128, 128), umma_desc(Ac, ALBO, 128), idesc, (t > 0 || j > 0) ? 1u : 0u);
          umma_i8(D, umma_desc(Xn, a.cpb * 128, 128), umma_desc(Ac, ALBO, 128), idesc, 1u);
          umma_i8(D, umma_desc(Xc, a.cpb * 128, 128), umma_desc(An, ALBO, 128), idesc, 1u);
        }
      }
      umma_commit(&empty[st]);
      if (t >= 1 && t - 1 + TC_MC_STAGES < T) {
        const int pst = (t - 1) % TC_MC_STAGES;
        mbar_wait(&empty[pst], (uint32_t)(((t - 1) / TC_MC_STAGES) & 1));
        load(t - 1 + TC_MC_STAGES);
      }
    }
    umma_commit(&done);
  }
  __syncwarp();
  if (T > 0) mbar_wait(&done, 0);
  pdl_trigger();
  if (T > 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint64_t* red = reinterpret_cast<uint64_t*>(smt);  // [3][NG][16 g][8 q]
    if (warp < 4) {
      const int r = warp * 32 + lane, g = r >> 3, q = r & 7;
      for (int c = 0; c < 3; ++c) {
        uint32_t d[64];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x64.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
            "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32, %33, %34, %35, "
            "%36, %37, %38, %39, %40, %41, %42, %43, %44, %45, %46, %47, %48, %49, %50, %51, %52, %53, %54, %55, %56, "
            "%57, %58, %59, %60, %61, %62, %63}, [%64];"
            : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
              "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15]),
              "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]), "=r"(d[20]), "=r"(d[21]), "=r"(d[22]),
              "=r"(d[23]), "=r"(d[24]), "=r"(d[25]), "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]),
              "=r"(d[30]), "=r"(d[31]), "=r"(d[32]), "=r"(d[33]), "=r"(d[34]), "=r"(d[35]), "=r"(d[36]),
              "=r"(d[37]), "=r"(d[38]), "=r"(d[39]), "=r"(d[40]), "=r"(d[41]), "=r"(d[42]), "=r"(d[43]),
              "=r"(d[44]), "=r"(d[45]), "=r"(d[46]), "=r"(d[47]), "=r"(d[48]), "=r"(d[49]), "=r"(d[50]),
              "=r"(d[51]), "=r"(d[52]), "=r"(d[53]), "=r"(d[54]), "=r"(d[55]), "=r"(d[56]), "=r"(d[57]),
              "=r"(d[58]), "=r"(d[59]), "=r"(d[60]), "=r"(d[61]), "=r"(d[62]), "=r"(d[63])
            : "r"(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)(c * 64)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          if (n >= NG) break;
          uint64_t v = 0;
#pragma unroll
          for (int p = 0; p < 8; ++p) v += (uint64_t)d[8 * n + p] << (8 * p);
          red[((c * NG + n) * 16 + g) * 8 + q] = v << (8 * q);
        }
      }
    }
    __syncthreads();
    const uint64_t Sstride = (uint64_t)a.n_h * (a.W + 1);
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int cell = tid + k * (int)blockDim.x;
      if (cell >= 3 * NG * 16) break;
      const int g = cell & 15, cn = cell >> 4, n = cn % NG, c = cn / NG;
      const int wg = nb * a.cpb + g;
      if (g >= a.cpb || n >= a.n_h || wg >= a.W) continue;
      const uint4* rp = reinterpret_cast<const uint4*>(red + (uint64_t)cell * 8);
      uint64_t v = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint4 x = rp[i];
        v += ((uint64_t)x.y << 32 | x.x) + ((uint64_t)x.w << 32 | x.z);
      }
      if (a.alpha && kr == 0 && a.alpha_tab) {
        v += apre[k];
      } else if (a.alpha && kr == 0) {
        uint64_t F[2];
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const Key& key = a.K.pair[qq == 0 ? c : (c + 2) % 3];
          F[qq] = a.alpha == 2 ? word(key, a.op_cnt, 4, (uint32_t)wg, (uint64_t)n)
                               : word(key, a.op_cnt, 3, (uint32_t)wg, a.t1 * (uint64_t)a.n_h + n) -
                                     word(key, a.op_cnt, 3, (uint32_t)wg, a.t0 * (uint64_t)a.n_h + n);
        }
        v += F[0] - F[1];
      }
      atomicAdd((unsigned long long*)&a.S[c * Sstride + (uint64_t)n * (a.W + 1) + wg], (unsigned long long)v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(TCOLS) : "memory");
  }
}

// ---------------------------------------------------------------------------
// Fused count (lanes + contraction in one CTA pair, 21..32 sample columns)
// ---------------------------------------------------------------------------
//
// The count of one level without the la planes ever leaving shared memory:
// a cluster of two CTAs (one per SM of a TPC) runs ONE tcgen05.mma.cta_group::2
// stream with the operand roles of k_count_mma_t,
//     D_c[(w,q)][(n,p)] = sum_s X_c[(w,q)][s] la_c[(n,p)][s] + X_{c+1} la_c + X_c la_{c+1},
// M = 256 = 32 sample columns x 8 limbs (CTA r holds the x planes of column
// block r: its own M half), N = 16 NBn = 2 NBn nodes x 8 limbs where CTA r
// holds the la rows of ITS NBn nodes (the B operand of a CTA pair is split
// along N: tools/umma2_probe.cu, profiles/r02c_umma2_probe.txt).  So every
// lane la = b2a(eq(m_idx, off+n) & is_leaf[n]) (train.py:211-217) is computed
// exactly once, by the producer warps of the CTA that owns node n, straight
// into the shared-memory B stage; the MMA reads both CTAs' stages; the
// contraction runs on the tensor pipe under the producers' ALU work.
// Pipeline per CTA: stages of 64 samples; x planes in a 3-deep ring by one
// bulk copy each (xfull / xempty), la bytes by the producer warps in a deep
// ring (full[s] = NBn producer arrivals / empty[s]); the peer relays its
// full[s] to the leader's pfull[s]; the leader's commits multicast empty[s]
// and xempty to both CTAs.  Same lanes, same
// randomness and the same epilogue sums as lanes8 + k_count_mma_t: the
// shares are identical.
constexpr int TCF_MAXS = 16;                      // la stages (the x-plane ring has XS)
constexpr int TCF_MAXXS = 8;                      // x-plane stages (at most)
constexpr int TCF_XB = 3 * 128 * (TC_KB / 2);     // x planes of a stage: 3 components x 128 rows x 64 samples
// Shallow tiles (NBn <= 4) run THREE UMMAs per 32-sample step instead of
// nine: with V_c = la_c + la_{c+1} (the ring sum; its byte planes are those
// of the sum mod 2^64),
//     D_c = X_c V_c + X_{c+1} la_c,
// and the two B operands that meet A = X_c (V_c for D_c, la_{c-1} for
// D_{c-1}) are stacked in one N = 2 x 16 NBn operand B_c = [V_c ; la_{c-1}]
// per CTA half, writing its own accumulator region [D_c | D_{c-1}] (each
// component is then the sum of two regions' halves, folded in the
// epilogue).  Shallow levels are bound by the UMMAs' A reads (x planes,
// 4 KB per UMMA and CTA); deep tiles keep nine UMMAs under the lane math.
__host__ __device__ inline bool tcf_mode3(int nbn_nodes) { return nbn_nodes <= 4; }
__host__ __device__ inline int tcf_la_bytes(int nbn_nodes, bool m3) { return (m3 ? 6 : 3) * 512 * nbn_nodes; }
// x-plane stages: deep where the level has few nodes (the contraction then
// streams the x planes; lane work is small), 3 at 16-node tiles
__host__ __device__ inline int tcf_xstages(int nbn_nodes) { return nbn_nodes <= 2 ? 6 : nbn_nodes <= 4 ? 4 : 3; }
// la stages: a deep ring, so a producer warp that runs ahead of the slowest
// one rarely waits for a slot (each stage needs all NBn node items)
// (a power of two: the producers' stage index and phase are shifts and masks)
__host__ __device__ inline int tcf_stages(int nbn_nodes, bool m3) {
  int s = (200 * 1024 - tcf_xstages(nbn_nodes) * TCF_XB) / tcf_la_bytes(nbn_nodes, m3);
  s = s > TCF_MAXS ? TCF_MAXS : s;
  int p = 1;
  while (2 * p <= s) p *= 2;
  return p;
}
__host__ __device__ inline int tcf_smem(int nbn_nodes, bool m3) {
  return tcf_xstages(nbn_nodes) * TCF_XB + tcf_stages(nbn_nodes, m3) * tcf_la_bytes(nbn_nodes, m3);
}

struct FusedArgs {
  const uint64_t *midx, *f, *leafbits;  // leafbits: is_leaf [3][n_h] from the partition launch, or null
  const uint8_t* B8;                    // x planes (tc_plan nbn = 2, cpb = 16)
  uint64_t* S;                          // [3][n_h][W+1]
  const uint64_t* alpha_tab;            // the level's reshare sums [n][3][W] or null (drawn)
  Keys K;
  uint32_t op_cnt, op_leaf;
  int alpha;                            // 0 none, 1 telescoped, 2 dot
  uint64_t t0, t1;                      // shard sample range (telescoped sums)
  uint64_t N, base;                     // shard samples, global index of shard sample 0
  uint64_t nkb_total, kb_lo;            // shard K blocks; first K block of this launch's range
  uint32_t nkb;                         // K blocks of the range
  int n_h, W, nkr, NBn, stages;
  int mode3;     // three UMMAs per step (shallow tiles, tcf_mode3)
  int ts_level;  // diagnostics (GT_COUNT_TS): phase timestamps of cluster 0 into g_cnt_ts[8 level ..], -1 off
  int mask_mma;  // s_mask from the x planes' constant columns W, W+1 (prep8 mask_cols) instead of warp sums
  int xpre;      // the x planes are complete before this launch's predecessor ran (levels >= 1): the copy
                 // thread fills the first x stages before the PDL wait
};

__device__ unsigned long long g_cnt_ts[128];
__device__ unsigned int g_cnt_done[16];
__device__ __forceinline__ void cnt_ts(const FusedArgs& a, int slot, bool on) {
  if (a.ts_level < 0 || !on || blockIdx.y != 0 || blockIdx.z != 0 || blockIdx.x != 0) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  g_cnt_ts[8 * a.ts_level + slot] = t;
}
// slot 7: the end of the level's LAST CTA (the grid's completion)
__device__ __forceinline__ void cnt_ts_last(const FusedArgs& a) {
  if (a.ts_level < 0 || threadIdx.x != 0) return;
  const unsigned int total = gridDim.x * gridDim.y * gridDim.z;
  if (atomicAdd(&g_cnt_done[a.ts_level], 1u) == total - 1) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_cnt_ts[8 * a.ts_level + 7] = t;
    g_cnt_done[a.ts_level] = 0;
  }
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(MBAR_SUSPEND_NS)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_local(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_rank0(uint64_t* bar) {  // the same barrier in cluster CTA 0
  uint32_t remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(remote) : "r"(smem_u32(bar)));
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
}
__device__ __forceinline__ void umma2_i8(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {  // arrive on `bar` in both CTAs of the pair
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// PW producer warps + a copy warp + an MMA warp; PF: each producer loads its next
// item's node indices before computing the current one (the lane math hides
// their L2 latency)
template <int PW, bool PF>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(32 * (PW + 2), 1) k_count_fused(FusedArgs a) {
  constexpr int TCF_PW = PW, TCF_THREADS = 32 * (PW + 2);
  extern __shared__ __align__(1024) uint8_t smt[];
  __shared__ __align__(8) uint64_t full[TCF_MAXS], empty[TCF_MAXS], pfull[TCF_MAXS], xfull[TCF_MAXXS], xempty[TCF_MAXXS],
      done;
  __shared__ uint32_t tmem_slot;
  __shared__ uint64_t leaf[3][8];
  const uint32_t rank = cluster_rank();
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nt = blockIdx.y, kr = blockIdx.z;
  const int NBn = a.NBn, NU = 16 * NBn, NS = a.stages;  // NU: the pair's UMMA N (2 NBn nodes x 8 limbs)
  // NBn and NS are powers of two: item -> (stage, node) and stage -> (slot,
  // phase) by shifts and masks (runtime divisions cost ~20 instructions each)
  const int nbn_sh = __ffs(NBn) - 1, ns_sh = __ffs(NS) - 1;
  const bool mode3 = a.mode3;
  const int LB = tcf_la_bytes(NBn, mode3);
  const int XS = tcf_xstages(NBn);
  uint8_t* lring = smt + XS * TCF_XB;  // la stages after the x-plane stages
  const uint32_t ACS = 512u * NBn, ALBO = 128u * NBn;  // la: [c][kc 4][g NBn][p 8][16 samples] per stage
  const uint32_t per = (a.nkb + a.nkr - 1) / a.nkr;
  const uint32_t kb0 = kr * per, kb1 = min(a.nkb, kb0 + per);
  const int T = kb1 > kb0 ? 2 * (int)(kb1 - kb0) : 0;  // 64-sample stages
  const int node0 = nt * 16 + (int)rank * NBn;          // this CTA's first node
  const uint32_t tcols = (mode3 ? 6 : 3) * NU <= 256 ? 256u : 512u;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_slot)),
                 "r"(tcols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], NBn);
      mbar_init(&empty[i], 1);
      mbar_init(&pfull[i], 1);
    }
    for (int i = 0; i < XS; ++i) {
      mbar_init(&xfull[i], 1);
      mbar_init(&xempty[i], 1);
    }
    mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both CTAs' barriers exist before any remote arrive / multicast commit
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_slot;
  // the epilogue's precomputed reshare sums: loaded before the wait
  uint64_t apre[4] = {0, 0, 0, 0};
  const int NNt = 2 * NBn, cells = 3 * NNt * 16;
  if (a.alpha && kr == 0 && a.alpha_tab) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int cell = tid + k * TCF_THREADS;
      const int w = cell & 15, cn = cell >> 4, ni = cn % NNt, c = cn / NNt;
      const int n = nt * 16 + ni, wg = (int)rank * 16 + w;
      if (cell < cells && n < a.n_h && wg < a.W) apre[k] = a.alpha_tab[((uint64_t)n * 3 + c) * a.W + wg];
    }
  }
  // the x planes of column block `rank`, stage t (one bulk copy; re-read by
  // every level: kept in L2 with evict_last).  With an even ring (XS even;
  // T is always even) one copy fills the two stages of a 128-sample K block
  // (adjacent in HBM and in the ring) and arms the even slot's barrier: a
  // bulk copy's throughput per SM grows with its size (tools/bench_bulk.cu:
  // 66 GB/s at 24 KB, 115 GB/s at 45 KB per copy, L2-resident)
  const int xstep = (XS & 1) ? 1 : 2;
  auto x_copy = [&](int t, uint64_t pol) {
    const int xs = t % XS;
    const uint64_t kb = a.kb_lo + kb0 + (uint32_t)(t >> 1), h = t & 1;
    const uint32_t bytes = (uint32_t)(xstep * TCF_XB);
    mbar_expect_tx(&xfull[xs], bytes);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(smt + xs * TCF_XB)),
        "l"(a.B8 + (((uint64_t)rank * a.nkb_total + kb) * 2 + h) * (uint64_t)TCF_XB), "r"(bytes),
        "r"(smem_u32(&xfull[xs])), "l"(pol)
        : "memory");
  };
  // levels >= 1: the prologue that wrote the x planes finished before the
  // partition launch passed its own wait (and only then triggered this
  // launch), so the first XS stages stream in while the partition drains
  const int xpre = (a.xpre && T > 0) ? min(XS, T) : 0;
  if (tid == 32 * TCF_PW && xpre) {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    for (int t = 0; t < xpre; t += xstep) x_copy(t, pol);
  }
  cnt_ts(a, 0, tid == 0);
  pdl_wait();  // m_idx, is_leaf, the zeroed sums (partition) and the x planes (prologue)
  cnt_ts(a, 1, tid == 0);
  if (tid < NBn) {
    const int n = node0 + tid;
    B3 z = {{0, 0, 0}};
    if (n < a.n_h && a.leafbits) {
#pragma unroll
      for (int c = 0; c < 3; ++c) z.v[c] = a.leafbits[c * a.n_h + n];
    } else if (n < a.n_h) {
      z = eqz<64>(a.K, a.op_leaf, 0, (uint64_t)n, add_pub<64>(ld3s(a.f, a.n_h, n), 0ull - F_LEAF));
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) leaf[c][tid] = z.v[c] & 1ull;
  }
  __syncthreads();

  if (warp < TCF_PW) {
    // producers: warp item (stage t, node g) = the 64 samples of stage t at
    // node node0 + g, one sample pair per lane (count_lane_pair); bytes as in
    // k_count_lanes8 (pairs of lanes swap limb halves with one shuffle pair)
    const bool odd = lane & 1;
    const int s2 = 2 * lane, items = T * NBn;
    auto sample_of = [&](int i) {
      const int t = i >> nbn_sh;
      return ((uint64_t)a.kb_lo + kb0 + (uint32_t)(t >> 1)) * TC_KB + (t & 1) * (TC_KB / 2) + s2;
    };
    auto load_idx = [&](int i, uint64_t (&m)[6]) {
      const uint64_t s = sample_of(i);
#pragma unroll
      for (int k = 0; k < 6; ++k) m[k] = 0;
      if (i < items && s < a.N) {
#pragma unroll
        for (int c = 0; c < 3; ++c) m[c] = __ldg(a.midx + c * a.N + s);
        if (s + 1 < a.N)
#pragma unroll
          for (int c = 0; c < 3; ++c) m[3 + c] = __ldg(a.midx + c * a.N + s + 1);
      }
    };
    uint64_t mnext[6];
    if (PF) load_idx(warp, mnext);
    for (int i = warp; i < items; i += TCF_PW) {
      const int t = i >> nbn_sh, g = i & (NBn - 1), st = t & (NS - 1);
      uint64_t mc[6];
      if (PF) {
#pragma unroll
        for (int k = 0; k < 6; ++k) mc[k] = mnext[k];
        load_idx(i + TCF_PW, mnext);
      } else {
        load_idx(i, mc);
      }
      if (t >= NS) mbar_wait(&empty[st], (uint32_t)(((t >> ns_sh) - 1) & 1));
      const int n = node0 + g;
      const uint64_t s = sample_of(i);
      A3 l0 = a3(0, 0, 0), l1 = a3(0, 0, 0);
      const bool v0 = n < a.n_h && s < a.N, v1 = v0 && s + 1 < a.N;
      if (v0) {
        const uint64_t off = 0ull - (uint64_t)(a.n_h - 1 + n);
        const A3 d0 = add_pub<64>(a3(mc[0], mc[1], mc[2]), off);
        A3 d1 = a3(0, 0, 0);
        if (v1) d1 = add_pub<64>(a3(mc[3], mc[4], mc[5]), off);
        B3 lf;
#pragma unroll
        for (int c = 0; c < 3; ++c) lf.v[c] = leaf[c][g];
        count_lane_pair(a.K, a.op_cnt, a.base + s, a.n_h, n, d0, d1, true, v1, lf, &l0, &l1);
      }
      if (!a.mask_mma) {  // s_mask (train.py:220): the warp's 64 samples of node n, one atomic per component
        A3 m = v1 ? add<64>(l0, l1) : l0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
#pragma unroll
          for (int c = 0; c < 3; ++c) m.v[c] += __shfl_xor_sync(0xffffffffu, m.v[c], o);
        if (lane == 0 && n < a.n_h)
#pragma unroll
          for (int c = 0; c < 3; ++c)
            atomicAdd((unsigned long long*)&a.S[((uint64_t)c * a.n_h + n) * (a.W + 1) + a.W], (unsigned long long)m.v[c]);
      }
      uint8_t* lb = lring + st * LB;
      const int p0 = odd ? 4 : 0, sub = (s2 & ~3) & 15, kc = (s2 >> 4) & 3;
      // the two samples' words x0, x1 as limb bytes into operand region `reg`
      // (gpk node groups per 16-sample chunk) at node group G
      auto put = [&](uint32_t reg, int gpk, int G, uint64_t x0, uint64_t x1) {
        const uint32_t a_lo = (uint32_t)x0, a_hi = (uint32_t)(x0 >> 32);
        const uint32_t b_lo = (uint32_t)x1, b_hi = (uint32_t)(x1 >> 32);
        const uint32_t P01 = __byte_perm(a_lo, b_lo, 0x5140), P23 = __byte_perm(a_lo, b_lo, 0x7362);
        const uint32_t P45 = __byte_perm(a_hi, b_hi, 0x5140), P67 = __byte_perm(a_hi, b_hi, 0x7362);
        const uint32_t r0 = __shfl_xor_sync(0xffffffffu, odd ? P01 : P45, 1);
        const uint32_t r1 = __shfl_xor_sync(0xffffffffu, odd ? P23 : P67, 1);
        uint32_t w[4];
        if (!odd) {
          w[0] = __byte_perm(P01, r0, 0x5410);
          w[1] = __byte_perm(P01, r0, 0x7632);
          w[2] = __byte_perm(P23, r1, 0x5410);
          w[3] = __byte_perm(P23, r1, 0x7632);
        } else {
          w[0] = __byte_perm(r0, P45, 0x5410);
          w[1] = __byte_perm(r0, P45, 0x7632);
          w[2] = __byte_perm(r1, P67, 0x5410);
          w[3] = __byte_perm(r1, P67, 0x7632);
        }
        uint8_t* dst = lb + reg + ((kc * gpk + G) * 8) * 16 + sub;
#pragma unroll
        for (int k = 0; k < 4; ++k) *reinterpret_cast<uint32_t*>(dst + (p0 + k) * 16) = w[k];
      };
      if (mode3) {  // B_c = [V_c ; la_{c-1}]: V_c at group g, la_c into B_{c+1} at group NBn + g
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const int cn = c == 2 ? 0 : c + 1;
          put((uint32_t)c * 2 * ACS, 2 * NBn, g, l0.v[c] + l0.v[cn], l1.v[c] + l1.v[cn]);
          put((uint32_t)cn * 2 * ACS, 2 * NBn, NBn + g, l0.v[c], l1.v[c]);
        }
      } else {
#pragma unroll
        for (int c = 0; c < 3; ++c) put((uint32_t)c * ACS, NBn, g, l0.v[c], l1.v[c]);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> the tensor pipe's view
      __syncwarp();
      if (lane == 0) mbar_arrive_local(&full[st]);
      cnt_ts(a, 2, lane == 0 && i == 0);
      cnt_ts(a, 3, lane == 0 && i + TCF_PW >= items);
    }
  } else if (warp == TCF_PW && lane == 0 && T > 0) {
    // copy thread: the x planes of column block `rank`, XS stages ahead of
    // the MMAs (a slot is refilled as soon as the pair's MMAs release it);
    // the x planes are re-read by every level: kept in L2 (evict_last)
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    for (int t = xpre; t < T; t += xstep) {
      // the last stage this copy fills: its slot's MMAs completing implies the
      // earlier slot's (a commit tracks all of the thread's prior UMMAs)
      const int tl = t + xstep - 1, xs = tl % XS;
      if (tl >= XS) mbar_wait(&xempty[xs], (uint32_t)(((tl / XS) - 1) & 1));
      x_copy(t, pol);
    }
  } else if (warp == TCF_PW + 1 && lane == 0 && T > 0) {
    // MMA thread (leader) / relay (peer): the leader issues the pair's UMMAs
    // once both CTAs' stage t is full; the peer forwards its full stage
    const uint32_t idesc = (2u << 4) | ((uint32_t)((mode3 ? 2 * NU : NU) >> 3) << 17) | ((256u >> 4) << 24);
    for (int t = 0; t < T; ++t) {
      const int st = t & (NS - 1), xs = t % XS;
      const uint32_t ph = (uint32_t)((t >> ns_sh) & 1);
      mbar_wait(&xfull[xstep == 2 ? (xs & ~1) : xs], (uint32_t)((t / XS) & 1));
      mbar_wait(&full[st], ph);
      if (rank == 0) {
        mbar_wait_cluster(&pfull[st], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t base = smem_u32(smt + xs * TCF_XB), lbase = smem_u32(lring + st * LB);
        if (mode3) {
#pragma unroll
          for (int j = 0; j < 2; ++j)
#pragma unroll
            for (int c = 0; c < 3; ++c)  // region c: [D_c | D_{c-1}] += X_c [V_c ; la_{c-1}]
              umma2_i8(tmem + (uint32_t)(c * 2 * NU), umma_desc(base + c * 8192 + j * 2 * 2048, 2048, 128),
                       umma_desc(lbase + c * 2 * ACS + j * 2 * (2 * ALBO), 2 * ALBO, 128), idesc,
                       (t > 0 || j > 0) ? 1u : 0u);
        } else {
#pragma unroll
          for (int j = 0; j < 2; ++j) {
            const uint32_t xo = j * 2 * 2048, ao = j * 2 * ALBO;
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              const int cn = (c + 1) % 3;
              const uint32_t Xc = base + c * 8192 + xo, Xn = base + cn * 8192 + xo;
              const uint32_t Ac = lbase + c * ACS + ao, An = lbase + cn * ACS + ao;
              const uint32_t D = tmem + (uint32_t)(c * NU);
              umma2_i8(D, umma_desc(Xc, 2048, 128), umma_desc(Ac, ALBO, 128), idesc, (t > 0 || j > 0) ? 1u : 0u);
              umma2_i8(D, umma_desc(Xn, 2048, 128), umma_desc(Ac, ALBO, 128), idesc, 1u);
              umma2_i8(D, umma_desc(Xc, 2048, 128), umma_desc(An, ALBO, 128), idesc, 1u);
            }
          }
        }
        umma2_commit_both(&empty[st]);
        umma2_commit_both(&xempty[xs]);
      } else {
        mbar_arrive_rank0(&pfull[st]);
      }
    }
    if (rank == 0) umma2_commit_both(&done);
    cnt_ts(a, 4, true);
  }
  __syncwarp();
  if (T > 0) mbar_wait(&done, 0);
  cnt_ts(a, 5, tid == 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // [slot][3][NNt nodes][16 w][8 q] (the stages are idle now); mode3 cells get
  // two contributions (regions c and c+1), kept in separate slots
  uint64_t* red = reinterpret_cast<uint64_t*>(smt);
  const int RSLOT = 3 * NNt * 16 * 8;
  if (T > 0) {
    // TMEM lane r = 32 (warp % 4) + lane = (column w, limb q) of this CTA's
    // block; accumulator columns j = node index x 8 + p (node index over the
    // pair).  Every warp takes the 16-column chunks warp / 4, + nq, ... of its
    // lane quarter (nq warps per quarter) and issues them two per
    // tcgen05.wait::ld.
    const int quarter = warp & 3, r = quarter * 32 + lane, w = r >> 3, q = r & 7;
    const int ccols = mode3 ? 2 * NU : NU, per_c = ccols / 16, chunks = 3 * per_c;
    constexpr int nq = TCF_THREADS / 128;
    auto fold = [&](const uint32_t(&d)[16], int ch) {
      const int c = ch / per_c, j0 = (ch % per_c) * 16;
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        uint64_t v = 0;
#pragma unroll
        for (int p = 0; p < 8; ++p) v += (uint64_t)d[8 * k + p] << (8 * p);
        const int col = j0 + 8 * k;
        if (mode3) {  // region c columns: [D_c(CTA 0 nodes) | D_{c-1}(0) | D_c(CTA 1 nodes) | D_{c-1}(1)]
          const int blk = col / (8 * NBn), ni = (blk >= 2 ? NBn : 0) + (col % (8 * NBn)) / 8;
          const int comp = (blk & 1) ? (c + 2) % 3 : c;
          red[(blk & 1) * RSLOT + ((comp * NNt + ni) * 16 + w) * 8 + q] = v << (8 * q);
        } else {
          red[((c * NNt + col / 8) * 16 + w) * 8 + q] = v << (8 * q);
        }
      }
    };
    auto tld = [&](uint32_t(&d)[16], int ch) {
      const int c = ch / per_c, j0 = (ch % per_c) * 16;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
          "%14, %15}, [%16];"
          : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7]),
            "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]), "=r"(d[14]), "=r"(d[15])
          : "r"(tmem + ((uint32_t)(quarter * 32) << 16) + (uint32_t)(c * ccols + j0)));
    };
    for (int ch = warp >> 2; ch < chunks; ch += 2 * nq) {  // warp-uniform trip count
      uint32_t d0[16], d1[16];
      const bool two = ch + nq < chunks;
      tld(d0, ch);
      if (two) tld(d1, ch + nq);
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      fold(d0, ch);
      if (two) fold(d1, ch + nq);
    }
    __syncthreads();
    const uint64_t Sstride = (uint64_t)a.n_h * (a.W + 1);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int cell = tid + k * TCF_THREADS;
      if (cell >= cells) break;
      const int w = cell & 15, cn = cell >> 4, ni = cn % NNt, c = cn / NNt;
      const int n = nt * 16 + ni, wg = (int)rank * 16 + w;
      const bool maskcell = a.mask_mma && ((c == 0 && (wg == a.W || wg == a.W + 1)) || (c == 2 && wg == a.W));
      if (n >= a.n_h || (wg >= a.W && !maskcell)) continue;
      uint64_t v = 0;
      for (int sl = 0; sl < (mode3 ? 2 : 1); ++sl) {
        const uint4* rp = reinterpret_cast<const uint4*>(red + sl * RSLOT + (uint64_t)cell * 8);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint4 x = rp[i];
          v += ((uint64_t)x.y << 32 | x.x) + ((uint64_t)x.w << 32 | x.z);
        }
      }
      if (maskcell) {
        // s_mask (train.py:220) from the constant columns: column W (shares
        // (1,0,0)) gives D_0 = sum la_0 + la_1, D_2 = sum la_2; column W+1
        // ((0,1,0)) gives D_0 = sum la_0 -- so mask_0 = D_0(W+1), mask_1 =
        // D_0(W) - D_0(W+1), mask_2 = D_2(W)
        unsigned long long* Sm = (unsigned long long*)&a.S[(uint64_t)n * (a.W + 1) + a.W];
        if (c == 2) {
          atomicAdd(Sm + 2 * Sstride, (unsigned long long)v);
        } else if (wg == a.W) {
          atomicAdd(Sm + Sstride, (unsigned long long)v);
        } else {
          atomicAdd(Sm, (unsigned long long)v);
          atomicAdd(Sm + Sstride, (unsigned long long)(0ull - v));
        }
        continue;
      }
      if (a.alpha && kr == 0 && a.alpha_tab) {
        v += apre[k];
      } else if (a.alpha && kr == 0) {
        uint64_t F[2];
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const Key& key = a.K.pair[qq == 0 ? c : (c + 2) % 3];
          F[qq] = a.alpha == 2 ? word(key, a.op_cnt, 4, (uint32_t)wg, (uint64_t)n)
                               : word(key, a.op_cnt, 3, (uint32_t)wg, a.t1 * (uint64_t)a.n_h + n) -
                                     word(key, a.op_cnt, 3, (uint32_t)wg, a.t0 * (uint64_t)a.n_h + n);
        }
        v += F[0] - F[1];
      }
      atomicAdd((unsigned long long*)&a.S[c * Sstride + (uint64_t)n * (a.W + 1) + wg], (unsigned long long)v);
    }
  }
  // trigger the heuristic after the epilogue's atomics, not at the MMA's end:
  // its CTAs' prologues then do not share the SMs with the epilogue
  // (C2 0.5465 -> 0.5446 ms, same-call A/B x6)
  pdl_trigger();
  cnt_ts(a, 6, tid == 0);
  cnt_ts_last(a);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();  // both CTAs are past their TMEM reads before the pair's columns are freed
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tcols) : "memory");
  }
}

}  // namespace
}  // namespace gt
