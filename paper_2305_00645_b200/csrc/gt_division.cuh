// Warp-cooperative fixed-point division (reference division, gadgets.py:310-349).
//
// One warp computes one division lane.  The comparison ladder (bound-1 lt +
// b2a, gadgets.py:327-336) is spread over the lanes of the warp, one ladder
// step per lane, and summed with shuffles.  The Newton part is a strictly
// serial chain of 3 + 2*iters multiplications and 2 + 2*iters (+1)
// truncations; its randomness does not depend on the data, so all 32 lanes
// first draw every Philox block of the chain in parallel into a per-warp
// shared-memory tape (~390 blocks at (32, 10)), then each lane runs the
// chain's arithmetic (redundantly, no divergence) reading the tape.  The
// blocks are exactly the live schedule's (same op, sub, field, lane), so the
// result equals division() share for share.
#pragma once
#include "gt_gadgets.cuh"

namespace gt {

// Newton chain steps in execution order (subs relative to s0, the first sub
// after the ladder): see div_newton() in gt_gadgets.cuh.
struct ChainStep {
  uint8_t is_trunc;
  uint8_t sub_off;
};

// number of chain steps and tape blocks
template <int L>
__host__ __device__ inline int newton_steps(const DivParams& d) { return 2 + 4 * d.iters + (d.sigma ? 4 : 3); }

template <int L>
__device__ __forceinline__ ChainStep newton_step(int i, const DivParams& d) {
  // [mul s0, trunc s0+1] then per iteration [mul s, trunc s+1, mul s+4, trunc s+5]
  // then [mul s, (trunc s+1 if sigma), mul s+4, trunc s+5]
  ChainStep c;
  if (i < 2) {
    c.is_trunc = (uint8_t)i;
    c.sub_off = (uint8_t)i;
    return c;
  }
  i -= 2;
  const int base = 4 + 8 * (i / 4 < d.iters ? i / 4 : d.iters);
  if (i < 4 * d.iters) {
    const int r = i % 4;
    c.is_trunc = (uint8_t)(r & 1);
    c.sub_off = (uint8_t)(base + (r >> 1) * 4 + (r & 1));
    return c;
  }
  i -= 4 * d.iters;
  if (!d.sigma) i += (i >= 1) ? 1 : 0;  // skip the sigma truncation
  c.is_trunc = (uint8_t)(i & 1);
  c.sub_off = (uint8_t)(base + (i >> 1) * 4 + (i & 1));
  return c;
}

template <int L>
__device__ __forceinline__ int step_blocks(const ChainStep& c) {
  return c.is_trunc ? TruncRand<L>::BLOCKS : 3;
}

template <int L>
__host__ __device__ inline int newton_blocks(const DivParams& d) {
  const int truncs = 2 + 2 * d.iters + (d.sigma ? 1 : 0);
  const int muls = 3 + 2 * d.iters;
  return truncs * (4 + 3 * Levels<L>::n + 4) + muls * 3;
}

// Fill tape[0 .. newton_blocks) cooperatively (lane, 32 lanes).
template <int L>
__device__ __forceinline__ void newton_tape_fill(const Keys& K, uint32_t op, uint32_t s0, uint64_t lane,
                                                 const DivParams& d, W2* tape, int wl) {
  const int steps = newton_steps<L>(d);
  int off = 0;
  for (int i = 0; i < steps; ++i) {
    const ChainStep c = newton_step<L>(i, d);
    const int nb = step_blocks<L>(c);
    const uint32_t sub = s0 + c.sub_off;
    for (int j = (wl - off) & 31; j < nb; j += 32) {
      if (c.is_trunc) {
        int key;
        uint32_t s, pidx;
        trunc_block_id<L>(j, sub, &key, &s, &pidx);
        tape[off + j] = block_of(K, key, op, s, pidx, lane);
      } else {
        tape[off + j] = word2(K.pair[j], op, sub, 0, lane);
      }
    }
    off += nb;
  }
}

// The Newton chain on tape blocks (gadgets.py:338-349; same steps as div_newton).
template <int L>
__device__ __forceinline__ A3 newton_from_tape(const A3& p, const A3& q, const A3& v, const DivParams& d,
                                               const W2* t) {
  constexpr int TB = TruncRand<L>::BLOCKS;
  auto mulT = [&](const A3& x, const A3& y) {
    const uint64_t F[3] = {t[0].a, t[1].a, t[2].a};
    t += 3;
    return mul_z<L>(x, y, F);
  };
  auto truncT = [&](const A3& x, int k) {
    const A3 r = trunc_arith<L>(t, x, k);
    t += TB;
    return r;
  };
  const A3 qn = mulT(q, v);
  const A3 qnorm = truncT(qn, d.bound - d.ti);
  A3 w = rsub_pub<L>(d.w0, mul_pub<L>(qnorm, 2));
  for (int it = 0; it < d.iters; ++it) {
    const A3 tq = truncT(mulT(qnorm, w), d.ti);
    const A3 e = rsub_pub<L>(1ull << (d.ti + 1), tq);
    w = truncT(mulT(w, e), d.ti);
  }
  A3 pn = mulT(p, v);
  if (d.sigma) pn = truncT(pn, d.sigma);
  const A3 prod = add_pub<L>(mulT(pn, w), 1ull << (d.kf - 1));
  return truncT(prod, d.kf);
}

template <int L>
__host__ __device__ inline int division_tape_blocks(const DivParams& d) {
  return newton_blocks<L>(d);
}

// ---------------------------------------------------------------------------
// Precomputed division randomness (the division's Philox blocks depend only
// on the keys, the op, the subs and the lane, never on data): one wide
// kernel draws every block of every division lane of a level into a global
// tape before the heuristic runs, so the latency-bound division chain only
// does arithmetic.  Per lane: ladder step j (1 <= j < bound) = the lt's
// LtRand blocks at sub s0+j-1 then the b2a dabit blocks (s0+bound-1+j-1,
// 0..1); then the Newton chain's blocks in newton_tape_fill order.  Same
// blocks as the live schedule, so shares are unchanged.
template <int L>
struct DivTape {
  static constexpr int LADDER_STEP = LtRand<L>::BLOCKS + 2;
};
template <int L>
__host__ __device__ inline int div_tape_blocks(const DivParams& d) {
  return (d.bound - 1) * DivTape<L>::LADDER_STEP + newton_blocks<L>(d);
}

template <int L>
__device__ __forceinline__ W2 div_tape_block(const Keys& K, uint32_t op, uint32_t s0, uint64_t lane,
                                             const DivParams& d, int b) {
  constexpr int LS = DivTape<L>::LADDER_STEP, LB = LtRand<L>::BLOCKS;
  const int lbt = (d.bound - 1) * LS;
  if (b < lbt) {
    const int j = b / LS + 1, w = b % LS;
    if (w < LB) {
      int key;
      uint32_t pidx;
      lt_block_id<L>(w, s0 + (j - 1), &key, &pidx);
      return word2(key < 0 ? K.dealer : K.pair[key], op, s0 + (j - 1), pidx, lane);
    }
    return word2(K.dealer, op, s0 + (d.bound - 1) + (j - 1), (uint32_t)(w - LB), lane);
  }
  b -= lbt;
  const uint32_t sn = s0 + 2 * (d.bound - 1);
  const int steps = newton_steps<L>(d);
  for (int i = 0; i < steps; ++i) {
    const ChainStep c = newton_step<L>(i, d);
    const int nb = step_blocks<L>(c);
    if (b < nb) {
      const uint32_t sub = sn + c.sub_off;
      if (c.is_trunc) {
        int key;
        uint32_t s, pidx;
        trunc_block_id<L>(b, sub, &key, &s, &pidx);
        return block_of(K, key, op, s, pidx, lane);
      }
      return word2(K.pair[b], op, sub, 0, lane);
    }
    b -= nb;
  }
  return W2{0, 0};
}

// Division by one warp from its lane tape already staged in shared memory
// (`ts` = ladder blocks then Newton blocks, div_tape_blocks<L>(d) of them).
template <int L>
__device__ __forceinline__ A3 division_warp_staged(const W2* ts, const A3& p, const A3& q, const DivParams& d,
                                                   unsigned long long* ts_out = nullptr) {
  constexpr uint64_t M = Ring<L>::M;
  constexpr int LS = DivTape<L>::LADDER_STEP, LB = LtRand<L>::BLOCKS;
  const int wl = threadIdx.x & 31;
  const int nl = d.bound - 1;
  A3 acc = a3(0, 0, 0);
  for (int j = wl + 1; j <= nl; j += 32) {
    const W2* b = ts + (j - 1) * LS;
    const B3 below = lt_arith<L>(b, q, a3_const((1ull << j) & M));
    const A3 t = b2a_arith<L>(bnot(below, 1ull), b[LB].a, b[LB].b, b[LB + 1].a);
    acc = add<L>(acc, mul_pub<L>(t, 1ull << (d.bound - 1 - j)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) acc.v[i] = (acc.v[i] + __shfl_xor_sync(0xffffffffu, acc.v[i], o)) & M;
  const A3 v = rsub_pub<L>(1ull << (d.bound - 1), acc);
  if (ts_out) {  // diagnostics (GT_HC_TIMING): ladder done
    unsigned long long tt;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));
    *ts_out = tt;
  }
  return newton_from_tape<L>(p, q, v, d, ts + nl * LS);
}

// Whole division lane by one warp; every lane returns the result.  `tape`
// points at this warp's division_tape_blocks() W2 slots of shared memory.
// The ladder's steps run one per lane with in-register Philox (measured
// faster than staging their ~1000 blocks through the tape); the Newton
// chain's blocks are drawn by all 32 lanes into the tape first.
template <int L>
__device__ __forceinline__ A3 division_warp(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const A3& p,
                                            const A3& q, const DivParams& d, W2* tape) {
  const int wl = threadIdx.x & 31;
  const int nl = d.bound - 1;
  // ladder: step j = wl + 1 (+32 ...) on this lane
  A3 acc = a3(0, 0, 0);
  for (int j = wl + 1; j <= nl; j += 32) acc = add<L>(acc, div_ladder_term<L>(K, op, sub, lane, q, j, d));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int i = 0; i < 3; ++i) acc.v[i] = (acc.v[i] + __shfl_xor_sync(0xffffffffu, acc.v[i], o)) & Ring<L>::M;
  const A3 v = rsub_pub<L>(1ull << (d.bound - 1), acc);
  newton_tape_fill<L>(K, op, sub + 2 * nl, lane, d, tape, wl);
  __syncwarp();
  const A3 out = newton_from_tape<L>(p, q, v, d, tape);
  __syncwarp();
  return out;
}

// select_share on one lane from blocks: b2a dealer (sub, 0..1), reshare
// pair_i (sub + 1, 0) (gadgets.py:238-253 with field 0).
__device__ __forceinline__ void select_block_id(int j, uint32_t sub, int* key, uint32_t* s, uint32_t* pidx) {
  if (j < 2) {
    *key = -1, *s = sub, *pidx = j;
  } else {
    *key = j - 2, *s = sub + 1, *pidx = 0;
  }
}

template <int L>
__device__ __forceinline__ A3 select_arith(const W2* b, const A3& w1, const A3& w2, const B3& cond) {
  const A3 ca = b2a_arith<L>(cond, b[0].a, b[0].b, b[1].a);
  const uint64_t F[3] = {b[2].a, b[3].a, b[4].a};
  return add<L>(w1, mul_z<L>(diff<L>(w2, w1), ca, F));
}

// One argmin tournament pair (gadgets.py:389-391) by one warp: the lt at
// `base`, the value select at base+1 and the index select (Z_2^64) at base+3
// draw ARGMIN_PAIR_BLOCKS<L> Philox blocks cooperatively into `tape`.
template <int L>
struct ArgminPair {
  static constexpr int BLOCKS = LtRand<L>::BLOCKS + 10;
};

template <int L>
__device__ __forceinline__ void argmin_pair_warp(const Keys& K, uint32_t op, uint32_t base, uint64_t lane, const A3& av,
                                                 const A3& bv, const A3& ai, const A3& bi, W2* tape, A3* nv, A3* ni) {
  const int wl = threadIdx.x & 31;
  constexpr int LB = LtRand<L>::BLOCKS;
  for (int j = wl; j < ArgminPair<L>::BLOCKS; j += 32) {
    int key;
    uint32_t s, pidx;
    if (j < LB) {
      lt_block_id<L>(j, base, &key, &pidx);
      s = base;
    } else if (j < LB + 5) {
      select_block_id(j - LB, base + 1, &key, &s, &pidx);
    } else {
      select_block_id(j - LB - 5, base + 3, &key, &s, &pidx);
    }
    tape[j] = word2(key < 0 ? K.dealer : K.pair[key], op, s, pidx, lane);
  }
  __syncwarp();
  const B3 cw = lt_arith<L>(tape, bv, av);  // challenger wins iff b < a
  *nv = select_arith<L>(tape + LB, av, bv, cw);
  *ni = select_arith<64>(tape + LB + 5, ai, bi, cw);
  __syncwarp();
}

}  // namespace gt
