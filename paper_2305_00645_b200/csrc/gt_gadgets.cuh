// Per-lane MPC gadgets over 2-out-of-3 replicated secret sharing, all three
// parties co-resident.  One lane = one element of a reference gadget call;
// every function below computes the three parties' local steps for that lane
// and treats each reshare / open as the algebraic identity it is when the
// three parties live in the same register file (the message bytes are
// accounted analytically by the host ledger, paper_2305_00645_b200/ledger.py).
//
// Representation: an arithmetic share is the three additive
// components A3.v[0..2] with x = v0 + v1 + v2 mod 2^L; party p (1-based)
// holds (v[p-1], v[p mod 3]) as (lo, hi) exactly as rss.py:1-9.  A boolean
// share B3 holds three XOR components; inside eq/lt one 64-bit word carries
// all L bit planes of one element (bit j = plane j), so the reference's plane
// loops (gadgets.py:81-185) become in-word shifts and masks.  Public
// constants act on component 0 (party 1 lo / party 3 hi, rss.py:313-367).
#pragma once
#include "gt_prg.cuh"

namespace gt {

template <int L>
struct Ring {
  static constexpr uint64_t M = (L == 64) ? ~0ull : ((1ull << L) - 1ull);
};

struct A3 {
  uint64_t v[3];
};
struct B3 {
  uint64_t v[3];
};

__device__ __forceinline__ uint64_t lowmask(int k) { return k >= 64 ? ~0ull : ((1ull << k) - 1ull); }

__device__ __forceinline__ A3 a3(uint64_t a, uint64_t b, uint64_t c) {
  A3 r;
  r.v[0] = a;
  r.v[1] = b;
  r.v[2] = c;
  return r;
}
__device__ __forceinline__ A3 a3_const(uint64_t c) { return a3(c, 0, 0); }  // const_a, rss.py:313-324

template <int L>
__device__ __forceinline__ A3 add(const A3& x, const A3& y) {
  return a3((x.v[0] + y.v[0]) & Ring<L>::M, (x.v[1] + y.v[1]) & Ring<L>::M, (x.v[2] + y.v[2]) & Ring<L>::M);
}
template <int L>
__device__ __forceinline__ A3 diff(const A3& x, const A3& y) {
  return a3((x.v[0] - y.v[0]) & Ring<L>::M, (x.v[1] - y.v[1]) & Ring<L>::M, (x.v[2] - y.v[2]) & Ring<L>::M);
}
template <int L>
__device__ __forceinline__ A3 add_pub(A3 x, uint64_t c) {  // rss.py:341-348
  x.v[0] = (x.v[0] + c) & Ring<L>::M;
  return x;
}
template <int L>
__device__ __forceinline__ A3 mul_pub(const A3& x, uint64_t c) {  // rss.py:88-90
  return a3((x.v[0] * c) & Ring<L>::M, (x.v[1] * c) & Ring<L>::M, (x.v[2] * c) & Ring<L>::M);
}
template <int L>
__device__ __forceinline__ A3 rsub_pub(uint64_t c, const A3& x) {  // rss.py:355-356
  return add_pub<L>(a3((0 - x.v[0]) & Ring<L>::M, (0 - x.v[1]) & Ring<L>::M, (0 - x.v[2]) & Ring<L>::M), c);
}
template <int L>
__device__ __forceinline__ uint64_t open(const A3& x) {  // open_a, rss.py:371-377
  return (x.v[0] + x.v[1] + x.v[2]) & Ring<L>::M;
}

// ---------------------------------------------------------------------------
// communicating primitives
// ---------------------------------------------------------------------------

// Hadamard product + reshare (PartyEngine.mul, rss.py:386-400):
//   z_i = x_i y_i + x_{i+1} y_i + x_i y_{i+1} + F(k_i) - F(k_{i-1})
template <int L>
__device__ __forceinline__ A3 mul_z(const A3& x, const A3& y, const uint64_t F[3]) {
  A3 z;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3, p = (i + 2) % 3;
    z.v[i] = (y.v[i] * (x.v[i] + x.v[j]) + x.v[i] * y.v[j] + F[i] - F[p]) & Ring<L>::M;
  }
  return z;
}

template <int L>
__device__ __forceinline__ A3 mul(const Keys& K, uint32_t op, uint32_t sub, uint32_t field, uint64_t lane,
                                  const A3& x, const A3& y) {
  uint64_t F[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) F[i] = word(K.pair[i], op, sub, field, lane);
  return mul_z<L>(x, y, F);
}

// AND with reshare (and_bits, rss.py:402-409) on bit-vector words; zero-share
// bits Z_i ^ Z_{i-1} restricted to `zmask`.
__device__ __forceinline__ B3 and_z(const B3& a, const B3& b, const uint64_t Z[3]) {
  B3 z;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3, p = (i + 2) % 3;
    z.v[i] = (a.v[i] & b.v[i]) ^ (a.v[j] & b.v[i]) ^ (a.v[i] & b.v[j]) ^ Z[i] ^ Z[p];
  }
  return z;
}

__device__ __forceinline__ B3 and_gate(const Keys& K, uint32_t op, uint32_t sub, uint32_t field, uint64_t lane,
                                       const B3& a, const B3& b, uint64_t zmask) {
  uint64_t Z[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) Z[i] = word(K.pair[i], op, sub, field, lane) & zmask;
  return and_z(a, b, Z);
}

__device__ __forceinline__ B3 bxor(const B3& a, const B3& b) {
  B3 r;
#pragma unroll
  for (int i = 0; i < 3; ++i) r.v[i] = a.v[i] ^ b.v[i];
  return r;
}
__device__ __forceinline__ B3 bnot(B3 a, uint64_t m) {  // xor_pub(ones), rss.py:358-367
  a.v[0] ^= m;
  return a;
}
// or_bits = x ^ y ^ (x & y), rss.py:411-412
__device__ __forceinline__ B3 or_gate(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const B3& x,
                                      const B3& y, uint64_t zmask) {
  return bxor(bxor(x, y), and_gate(K, op, sub, 0, lane, x, y, zmask));
}

// AND over the low k bit planes of the word (and_reduce, gadgets.py:94-109):
// level with k rows ANDs plane j with plane j+half (j < half), an odd last
// plane is carried to position half.  Gate j of a level draws zero bit
// (off + j) of the pair words Zw; off advances by half per level (<= 63 bits).
__device__ __forceinline__ B3 and_reduce_w(B3 P, int k, const uint64_t Zw[3]) {
  int off = 0;
  while (k > 1) {
    const int half = k >> 1;
    const uint64_t lm = lowmask(half);
    B3 a, b;
    uint64_t Z[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      a.v[i] = P.v[i] & lm;
      b.v[i] = (P.v[i] >> half) & lm;
      Z[i] = (Zw[i] >> off) & lm;
    }
    B3 m = and_z(a, b, Z);
    if (k & 1) {
#pragma unroll
      for (int i = 0; i < 3; ++i) m.v[i] |= ((P.v[i] >> (k - 1)) & 1ull) << half;
    }
    P = m;
    off += half;
    k = half + (k & 1);
  }
  return P;
}

__device__ __forceinline__ B3 and_reduce(const Keys& K, uint32_t op, uint32_t sub, uint32_t field, uint64_t lane,
                                         B3 P, int k) {
  uint64_t Zw[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) Zw[i] = word(K.pair[i], op, sub, field, lane);
  return and_reduce_w(P, k, Zw);
}

// ---------------------------------------------------------------------------
// comparisons (masked opening + boolean circuit on public c vs shared r)
// ---------------------------------------------------------------------------

// [d == 0] from an edabit (r, boolean word shares Rb0, Rb1) and the AND-tree
// zero words Zw (eq, gadgets.py:120-130).  The arithmetic shares of r only
// mask the opening, c = sum_i (d_i + R_i) = d + r, so they are not drawn.
template <int L>
__device__ __forceinline__ B3 eq_arith(const A3& d, uint64_t r, uint64_t Rb0, uint64_t Rb1, const uint64_t Zw[3]) {
  constexpr uint64_t M = Ring<L>::M;
  r &= M;
  Rb0 &= M;
  Rb1 &= M;
  const uint64_t c = (open<L>(d) + r) & M;  // open_a(d + r)
  const uint64_t notc = ~c & M;
  B3 P;
  P.v[0] = Rb0 ^ notc;  // xor_pub(planes, ~c)
  P.v[1] = Rb1;
  P.v[2] = r ^ Rb0 ^ Rb1;  // _value_bit_words, dealer.py:51-57
  return and_reduce_w(P, L, Zw);
}

// One 32-bit AND gate with reshare: z_i = (a_i & b_i) ^ (a_{i+1} & b_i) ^
// (a_i & b_{i+1}) ^ Z_i ^ Z_{i-1} = (b_i & (a_i ^ a_{i+1})) ^ (a_i & b_{i+1}) ^ ...
__device__ __forceinline__ void and3_32(const uint32_t a[3], const uint32_t b[3], const uint32_t z[3], uint32_t o[3]) {
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const int j = (i + 1) % 3, p = (i + 2) % 3;
    o[i] = (b[i] & (a[i] ^ a[j])) ^ (a[i] & b[j]) ^ z[i] ^ z[p];
  }
}

// eq at l = 64 with the AND tree on 32-bit halves: after the first level
// (plane j & plane j+32 = low word & high word) every level fits 32 bits.
// Same zero-bit layout as and_reduce_w: level bits at offsets 0, 32, 48, 56,
// 60, 62 of the pair words.
template <>
__device__ __forceinline__ B3 eq_arith<64>(const A3& d, uint64_t r, uint64_t Rb0, uint64_t Rb1, const uint64_t Zw[3]) {
  const uint64_t c = open<64>(d) + r;
  const uint64_t P[3] = {Rb0 ^ ~c, Rb1, r ^ Rb0 ^ Rb1};
  uint32_t a[3], b[3], z[3], w[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    a[i] = (uint32_t)P[i];
    b[i] = (uint32_t)(P[i] >> 32);
    z[i] = (uint32_t)Zw[i];
  }
  and3_32(a, b, z, w);
  uint32_t zh[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) zh[i] = (uint32_t)(Zw[i] >> 32);
  // (rows >= half of a level's operands are never masked: gate j reads bit
  // j of each operand only, so they cannot reach the rows the next level
  // keeps, and the result is bit 0)
#pragma unroll
  for (int lvl = 1, half = 16, off = 0; lvl < 6; ++lvl, off += half, half >>= 1) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      a[i] = w[i];
      b[i] = w[i] >> half;
      z[i] = zh[i] >> off;
    }
    and3_32(a, b, z, w);
  }
  B3 out;
#pragma unroll
  for (int i = 0; i < 3; ++i) out.v[i] = w[i] & 1u;
  return out;
}

// Two l = 64 eq lanes at once: the first AND level runs per lane on the
// 32-bit halves; from the second level on both lanes share every 32-bit
// register (lane A in the low half, lane B in the high half of each packed
// field, packed with byte permutes), halving the AND-tree instructions.
// Same gates, same zero bits as eq_arith<64> (levels at offsets 0, 32, 48,
// 56, 60, 62 of each lane's zero words).  Returns lane A / lane B in bit 0 of
// hA / hB.
template <bool MASK = true>
__device__ __forceinline__ void eq_arith64_x2(const A3& dA, uint64_t rA, uint64_t Rb0A, uint64_t Rb1A,
                                              const uint64_t ZA[3], const A3& dB, uint64_t rB, uint64_t Rb0B,
                                              uint64_t Rb1B, const uint64_t ZB[3], B3* hA, B3* hB) {
  const uint64_t cA = open<64>(dA) + rA, cB = open<64>(dB) + rB;
  const uint64_t PA[3] = {Rb0A ^ ~cA, Rb1A, rA ^ Rb0A ^ Rb1A};
  const uint64_t PB[3] = {Rb0B ^ ~cB, Rb1B, rB ^ Rb0B ^ Rb1B};
  uint32_t a[3], b[3], z[3], wA[3], wB[3];
  // level 1 (64 -> 32) per lane
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    a[i] = (uint32_t)PA[i];
    b[i] = (uint32_t)(PA[i] >> 32);
    z[i] = (uint32_t)ZA[i];
  }
  and3_32(a, b, z, wA);
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    a[i] = (uint32_t)PB[i];
    b[i] = (uint32_t)(PB[i] >> 32);
    z[i] = (uint32_t)ZB[i];
  }
  and3_32(a, b, z, wB);
  uint32_t zhA[3], zhB[3], w[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    zhA[i] = (uint32_t)(ZA[i] >> 32);
    zhB[i] = (uint32_t)(ZB[i] >> 32);
  }
  // level 2 (32 -> 16): halves 0..15 / 16..31 of each lane, packed A | B << 16
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    a[i] = __byte_perm(wA[i], wB[i], 0x5410);
    b[i] = __byte_perm(wA[i], wB[i], 0x7632);
    z[i] = __byte_perm(zhA[i], zhB[i], 0x5410);  // zero bits 0..15 of each lane's high word
  }
  and3_32(a, b, z, w);  // lane A bits 0..15, lane B bits 16..31
  // level 3 (16 -> 8): bytes [A0 A1 B0 B1] -> a = [A0 B0], b = [A1 B1]
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    a[i] = __byte_perm(w[i], 0, 0x4420);
    b[i] = __byte_perm(w[i], 0, 0x4431);
    z[i] = __byte_perm(zhA[i], zhB[i], 0x4462);  // zero bits 16..23 of each lane
  }
  and3_32(a, b, z, w);  // lane A byte 0, lane B byte 1
  // levels 4..6 (8 -> 4 -> 2 -> 1) within each lane's byte
  uint32_t zz[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) zz[i] = __byte_perm(zhA[i], zhB[i], 0x4473);  // zero bits 24..31
  // MASK = false: unmasked operands (gate j of each byte reads bit j only,
  // and bits j + half, off + j stay inside the byte, so nothing crosses into
  // the rows a level keeps; the results are bits 0 and 8) -- fewer
  // instructions; measured faster in the lookups (walk, partition) and
  // slower in the count lanes, which keep the masks
#pragma unroll
  for (int lvl = 0, half = 4, off = 0; lvl < 3; ++lvl, off += half, half >>= 1) {
    const uint32_t lm = MASK ? ((1u << half) - 1u) * 0x0101u : ~0u;
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      a[i] = w[i] & lm;
      b[i] = (w[i] >> half) & lm;
      z[i] = (zz[i] >> off) & lm;
    }
    and3_32(a, b, z, w);
  }
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    hA->v[i] = w[i] & 1u;
    hB->v[i] = (w[i] >> 8) & 1u;
  }
}

// standalone eq: dealer fields r=0 Rb0=1 Rb1=2; pair field 0 = AND-tree bits.
template <int L>
__device__ __forceinline__ B3 eqz(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const A3& d) {
  const W2 d0 = word2(K.dealer, op, sub, 0, lane);
  const uint64_t Rb1 = word(K.dealer, op, sub, 2, lane);
  uint64_t Zw[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) Zw[i] = word(K.pair[i], op, sub, 0, lane);
  return eq_arith<L>(d, d0.a, d0.b, Rb1, Zw);
}

template <int L>
struct Levels {
  static constexpr int n = (L == 64) ? 6 : (L == 32) ? 5 : 3;  // log2 L
};

// Kogge-Stone borrow prefix on (g, p) words (_prefix_borrow, gadgets.py:137-160).
// Level with shift s: pg = p & (g << s), pp = p & (p << s) for bits >= s (two
// batched AND lanes per row); bits < s keep g and p, as the reference does.
// blk[i * nlev + l] holds key i's zero words of level l: .a for pg, .b for pp
// (= pair fields fb + 2l, fb + 2l + 1 of the live schedule).
template <int L>
__device__ __forceinline__ B3 prefix_borrow_blk(B3 g, B3 p, const W2* blk) {
  constexpr uint64_t M = Ring<L>::M;
  constexpr int NL = Levels<L>::n;
  // g and p stay within M; the shifted words and the zero words are used
  // unmasked and the gates' outputs are cut to the rows >= s (and < L) once,
  // inside the combining LOP3 (the same rows the masked operands give: the
  // AND terms vanish outside them because p does)
#pragma unroll
  for (int lvl = 0; lvl < NL; ++lvl) {
    const int s = 1 << lvl;
    const uint64_t hm = M & ~lowmask(s), lm = lowmask(s);
    B3 gs, ps;
    uint64_t Zg[3], Zp[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      gs.v[i] = g.v[i] << s;
      ps.v[i] = p.v[i] << s;
      Zg[i] = blk[i * NL + lvl].a;
      Zp[i] = blk[i * NL + lvl].b;
    }
    const B3 pg = and_z(p, gs, Zg);
#pragma unroll
    for (int i = 0; i < 3; ++i) g.v[i] ^= pg.v[i] & hm;
    if (lvl + 1 < NL) {  // the last level's propagate gates feed nothing: not computed (same g)
      const B3 pp = and_z(p, ps, Zp);
#pragma unroll
      for (int i = 0; i < 3; ++i) p.v[i] = (p.v[i] & lm) | (pp.v[i] & hm);
    }
  }
  return g;
}

template <int L>
__device__ __forceinline__ B3 prefix_borrow(const Keys& K, uint32_t op, uint32_t sub, uint32_t fb, uint64_t lane,
                                            B3 g, B3 p) {
  constexpr int NL = Levels<L>::n;
  W2 blk[3 * NL];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int l = 0; l < NL; ++l) blk[i * NL + l] = word2(K.pair[i], op, sub, (fb >> 1) + l, lane);
  return prefix_borrow_blk<L>(g, p, blk);
}

// Borrow rows S[i] = [c mod 2^{i+1} < r mod 2^{i+1}] for public c
// (_borrow_scan, gadgets.py:163-171): g = r & ~c, p = r ^ ~c.
template <int L>
__device__ __forceinline__ B3 borrow_scan_blk(uint64_t c, const B3& Rb, const W2* blk) {
  constexpr uint64_t M = Ring<L>::M;
  const uint64_t notc = ~c & M;
  B3 g, p;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    g.v[i] = Rb.v[i] & notc;
    p.v[i] = Rb.v[i];
  }
  p.v[0] ^= notc;
  return prefix_borrow_blk<L>(g, p, blk);
}

template <int L>
__device__ __forceinline__ B3 borrow_scan(const Keys& K, uint32_t op, uint32_t sub, uint32_t fb, uint64_t lane,
                                          uint64_t c, const B3& Rb) {
  constexpr uint64_t M = Ring<L>::M;
  const uint64_t notc = ~c & M;
  B3 g, p;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    g.v[i] = Rb.v[i] & notc;
    p.v[i] = Rb.v[i];
  }
  p.v[0] ^= notc;
  return prefix_borrow<L>(K, op, sub, fb, lane, g, p);
}

// Shared bits of (c - r) (_masked_diff_bits, gadgets.py:174-185).
template <int L>
__device__ __forceinline__ B3 masked_diff_bits(const Keys& K, uint32_t op, uint32_t sub, uint32_t fb, uint64_t lane,
                                               uint64_t c, const B3& Rb) {
  constexpr uint64_t M = Ring<L>::M;
  const B3 s = borrow_scan<L>(K, op, sub, fb, lane, c, Rb);
  B3 d;
#pragma unroll
  for (int i = 0; i < 3; ++i) d.v[i] = Rb.v[i] ^ ((s.v[i] << 1) & M);
  d.v[0] ^= c;
  return d;
}

// [x < y] unsigned (lt, gadgets.py:188-216); result in bit 0.
// Live fields: dealer x-edabit 0..4, y-edabit 5..9; pair x scan [0,12),
// y scan [12,24), generate gate 24, final prefix [26,38).  As Philox blocks
// in tape order (LtRand<L>::BLOCKS): dealer (sub, 0..3); x scan pair_i
// (sub, l); y scan pair_i (sub, 6 + l); generate pair_i (sub, 12); prefix
// pair_i (sub, 13 + l) -- i = 0..2, l = 0..nlev-1.
template <int L>
struct LtRand {
  static constexpr int NL = Levels<L>::n;
  static constexpr int BLOCKS = 4 + 9 * NL + 3;
};

template <int L>
__device__ __forceinline__ void lt_block_id(int j, uint32_t sub, int* key, uint32_t* pidx) {
  constexpr int NL = Levels<L>::n;
  if (j < 4) {
    *key = -1, *pidx = j;
    return;
  }
  j -= 4;
  if (j < 3 * NL) {
    *key = j / NL, *pidx = j % NL;
  } else if (j < 6 * NL) {
    j -= 3 * NL;
    *key = j / NL, *pidx = 6 + j % NL;
  } else if (j < 6 * NL + 3) {
    *key = j - 6 * NL, *pidx = 12;
  } else {
    j -= 6 * NL + 3;
    *key = j / NL, *pidx = 13 + j % NL;
  }
}

template <int L>
__device__ __forceinline__ B3 lt_arith(const W2* b, const A3& x, const A3& y) {
  constexpr uint64_t M = Ring<L>::M;
  constexpr int NL = Levels<L>::n;
  B3 xb, yb;
  {
    const uint64_t r = b[0].a & M;  // fields 0 (r), 1 (Rb0), 2 (Rb1)
    B3 Rb;
    Rb.v[0] = b[0].b & M;
    Rb.v[1] = b[1].a & M;
    Rb.v[2] = r ^ Rb.v[0] ^ Rb.v[1];
    const uint64_t c = (open<L>(x) + r) & M;
    const B3 sc = borrow_scan_blk<L>(c, Rb, b + 4);
#pragma unroll
    for (int i = 0; i < 3; ++i) xb.v[i] = Rb.v[i] ^ ((sc.v[i] << 1) & M);
    xb.v[0] ^= c;  // _masked_diff_bits, gadgets.py:174-185
  }
  {
    const uint64_t r = b[2].b & M;  // fields 5 (r), 6 (Rb0), 7 (Rb1)
    B3 Rb;
    Rb.v[0] = b[3].a & M;
    Rb.v[1] = b[3].b & M;
    Rb.v[2] = r ^ Rb.v[0] ^ Rb.v[1];
    const uint64_t c = (open<L>(y) + r) & M;
    const B3 sc = borrow_scan_blk<L>(c, Rb, b + 4 + 3 * NL);
#pragma unroll
    for (int i = 0; i < 3; ++i) yb.v[i] = Rb.v[i] ^ ((sc.v[i] << 1) & M);
    yb.v[0] ^= c;
  }
  const uint64_t Zg[3] = {b[4 + 6 * NL].a & M, b[5 + 6 * NL].a & M, b[6 + 6 * NL].a & M};
  const B3 g = and_z(yb, bnot(xb, M), Zg);
  const B3 p = bnot(bxor(xb, yb), M);
  B3 rows = prefix_borrow_blk<L>(g, p, b + 7 + 6 * NL);
#pragma unroll
  for (int i = 0; i < 3; ++i) rows.v[i] = (rows.v[i] >> (L - 1)) & 1ull;
  return rows;
}

// lt_arith by a whole warp: even lanes recover the bits of x, odd lanes those
// of y (the same instructions on two operands run side by side), one shuffle
// pair exchanges them, then every lane finishes the comparison.  Same blocks
// and result as lt_arith; all 32 lanes must call it.
template <int L>
__device__ __forceinline__ B3 lt_arith_warp(const W2* b, const A3& x, const A3& y) {
  constexpr uint64_t M = Ring<L>::M;
  constexpr int NL = Levels<L>::n;
  const bool odd = threadIdx.x & 1;
  const A3 v = odd ? y : x;
  const uint64_t r = (odd ? b[2].b : b[0].a) & M;
  B3 Rb;
  Rb.v[0] = (odd ? b[3].a : b[0].b) & M;
  Rb.v[1] = (odd ? b[3].b : b[1].a) & M;
  Rb.v[2] = r ^ Rb.v[0] ^ Rb.v[1];
  const uint64_t c = (open<L>(v) + r) & M;
  const B3 sc = borrow_scan_blk<L>(c, Rb, b + 4 + (odd ? 3 * NL : 0));
  B3 mine;
#pragma unroll
  for (int i = 0; i < 3; ++i) mine.v[i] = Rb.v[i] ^ ((sc.v[i] << 1) & M);
  mine.v[0] ^= c;
  B3 other;
#pragma unroll
  for (int i = 0; i < 3; ++i) other.v[i] = __shfl_xor_sync(0xffffffffu, mine.v[i], 1);
  const B3 xb = odd ? other : mine, yb = odd ? mine : other;
  const uint64_t Zg[3] = {b[4 + 6 * NL].a & M, b[5 + 6 * NL].a & M, b[6 + 6 * NL].a & M};
  const B3 g = and_z(yb, bnot(xb, M), Zg);
  const B3 p = bnot(bxor(xb, yb), M);
  B3 rows = prefix_borrow_blk<L>(g, p, b + 7 + 6 * NL);
#pragma unroll
  for (int i = 0; i < 3; ++i) rows.v[i] = (rows.v[i] >> (L - 1)) & 1ull;
  return rows;
}

template <int L>
__device__ __forceinline__ B3 lt(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const A3& x, const A3& y) {
  W2 b[LtRand<L>::BLOCKS];
#pragma unroll
  for (int j = 0; j < LtRand<L>::BLOCKS; ++j) {
    int key;
    uint32_t pidx;
    lt_block_id<L>(j, sub, &key, &pidx);
    b[j] = word2(key < 0 ? K.dealer : K.pair[key], op, sub, pidx, lane);
  }
  return lt_arith<L>(b, x, y);
}

// Boolean bit -> arithmetic share (b2a, gadgets.py:223-231) from a dabit:
// arithmetic shares (A0, A1, beta - A0 - A1) and boolean shares of beta =
// bit0 of `bits` with Bb0 = bit1, Bb1 = bit2 (_gen_dabits, dealer.py:60-64).
template <int L>
__device__ __forceinline__ A3 b2a_arith(const B3& b, uint64_t A0, uint64_t A1, uint64_t bits) {
  constexpr uint64_t M = Ring<L>::M;
  A0 &= M;
  A1 &= M;
  const uint64_t beta = bits & 1ull;
  const uint64_t A2 = (beta - A0 - A1) & M;
  // open_bits of b ^ beta: the dabit's bit shares Bb0, Bb1, Bb2 = beta ^ Bb0 ^
  // Bb1 (bits 1, 2 of `bits`) cancel in the opened sum, leaving beta
  const uint64_t e = (b.v[0] ^ b.v[1] ^ b.v[2] ^ bits) & 1ull;
  // A * (1 - 2e) as a conditional negate ((A ^ m) - m, m = -e): keeps the
  // IMAD pipe for the Philox rounds and the share products
  const uint64_t m = 0ull - e;
  return a3((((A0 ^ m) - m) + e) & M, ((A1 ^ m) - m) & M, ((A2 ^ m) - m) & M);
}

// standalone b2a: dealer fields A0=0 A1=1 bits=2.
template <int L>
__device__ __forceinline__ A3 b2a(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const B3& b) {
  const W2 w = word2(K.dealer, op, sub, 0, lane);
  return b2a_arith<L>(b, w.a, w.b, word(K.dealer, op, sub, 2, lane));
}

// One fused lookup / count lane (oaa.py:28-34, train.py:214-219): eq + b2a
// draw the lane's dealer material from THREE Philox blocks
//   dealer (sub,0) = (r, Rb0)   (sub,1) = (Rb1, A0)   (sub,2) = (A1, dabit bits)
// while the AND-tree zero words of two neighbouring lanes share ONE pair
// block per key (.a / .b halves; the caller picks the block, see
// lookup_partial and the count lane kernels).  A count lane's leaf-AND zero
// bit is bit 63 of its zero word (the l = 64 AND tree uses bits 0..62).
// One count lane (train.py:214-217) from its dealer material and zero word:
// la = b2a(eq(d, 0) & leaf), the AND gate's zero bit = bit 63 of Zw.
__device__ __forceinline__ A3 count_lane_arith(const A3& d, uint64_t r, uint64_t Rb0, uint64_t Rb1, uint64_t A0,
                                               uint64_t A1, uint64_t bits, const uint64_t Zw[3], const B3& leaf);

struct DealerRand {
  uint64_t r, Rb0, Rb1, A0, A1, bits;
};
__device__ __forceinline__ DealerRand dealer_rand(const Keys& K, uint32_t op, uint64_t lane) {
  DealerRand R;
  const W2 d0 = word2(K.dealer, op, 0, 0, lane);
  const W2 d1 = word2(K.dealer, op, 0, 1, lane);
  const W2 d2 = word2(K.dealer, op, 0, 2, lane);
  R.r = d0.a;
  R.Rb0 = d0.b;
  R.Rb1 = d1.a;
  R.A0 = d1.b;
  R.A1 = d2.a;
  R.bits = d2.b;
  return R;
}

__device__ __forceinline__ A3 count_lane_arith(const A3& d, uint64_t r, uint64_t Rb0, uint64_t Rb1, uint64_t A0,
                                               uint64_t A1, uint64_t bits, const uint64_t Zw[3], const B3& leaf) {
  const B3 hit = eq_arith<64>(d, r, Rb0, Rb1, Zw);
  const uint64_t Z[3] = {Zw[0] >> 63, Zw[1] >> 63, Zw[2] >> 63};
  return b2a_arith<64>(and_z(hit, leaf, Z), A0, A1, bits);
}

// The two count lanes of samples gs, gs+1 (global) at node n: their zero
// words come from pair block (g >> 1) * n_h + n, half g & 1, for g = gs, gs+1
// (one shared block per key when gs is even).
__device__ __forceinline__ void count_lane_pair(const Keys& K, uint32_t op, uint64_t gs, int n_h, int n,
                                                const A3& d0, const A3& d1, bool v0, bool v1, const B3& leaf,
                                                A3* l0, A3* l1) {
  uint64_t Z0[3], Z1[3];
  if ((gs & 1) == 0) {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const W2 z = word2(K.pair[i], op, 0, 0, (gs >> 1) * (uint64_t)n_h + n);
      Z0[i] = z.a;
      Z1[i] = z.b;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      Z0[i] = word2(K.pair[i], op, 0, 0, (gs >> 1) * (uint64_t)n_h + n).b;
      Z1[i] = word2(K.pair[i], op, 0, 0, ((gs + 1) >> 1) * (uint64_t)n_h + n).a;
    }
  }
  // both lanes always computed (the second lane of a shard's odd tail is
  // discarded by the caller)
  (void)v0;
  (void)v1;
  const DealerRand R0 = dealer_rand(K, op, gs * (uint64_t)n_h + n);
  const DealerRand R1 = dealer_rand(K, op, (gs + 1) * (uint64_t)n_h + n);
  B3 h0, h1;
  eq_arith64_x2(d0, R0.r, R0.Rb0, R0.Rb1, Z0, d1, R1.r, R1.Rb0, R1.Rb1, Z1, &h0, &h1);
  const uint64_t Y0[3] = {Z0[0] >> 63, Z0[1] >> 63, Z0[2] >> 63};
  const uint64_t Y1[3] = {Z1[0] >> 63, Z1[1] >> 63, Z1[2] >> 63};
  *l0 = b2a_arith<64>(and_z(h0, leaf, Y0), R0.A0, R0.A1, R0.bits);
  *l1 = b2a_arith<64>(and_z(h1, leaf, Y1), R1.A0, R1.A1, R1.bits);
}

// select_share (gadgets.py:238-253) for one condition lane and one payload
// element: w1 + b2a(c) * (w2 - w1); b2a at `sub`, mul at `sub + 1`, `field`
// = payload index inside the condition's group.
template <int L>
__device__ __forceinline__ A3 select_with(const Keys& K, uint32_t op, uint32_t sub, uint32_t field, uint64_t lane,
                                          const A3& w1, const A3& w2, const A3& ca) {
  return add<L>(w1, mul<L>(K, op, sub + 1, field, lane, diff<L>(w2, w1), ca));
}
template <int L>
__device__ __forceinline__ A3 select1(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const A3& w1,
                                      const A3& w2, const B3& cond) {
  const A3 ca = b2a<L>(K, op, sub, lane, cond);
  return select_with<L>(K, op, sub, 0, lane, w1, w2, ca);
}

// Exact floor(x / 2^k), unsigned (truncate, gadgets.py:260-288).  Uses subs
// sub (opening + borrow scan, dealer fields r=0 Rb0=1 Rb1=2 R0=3 R1=4 S0=5
// S1=6, pair fields 0..2*nlev-1), sub+1 (b2a of the wrap bit), sub+2 (b2a of
// the low borrow).  In Philox blocks (TRUNC_BLOCKS of them, the order of a
// tape): dealer (sub, 0..3), pair_i (sub, 0..nlev-1) for i = 0..2, dealer
// (sub+1, 0..1), dealer (sub+2, 0..1).
template <int L>
struct TruncRand {
  static constexpr int NL = Levels<L>::n;
  static constexpr int BLOCKS = 4 + 3 * NL + 4;
  W2 b[BLOCKS];
};

template <int L>
__device__ __forceinline__ void trunc_block_id(int j, uint32_t sub, int* key, uint32_t* s, uint32_t* pidx) {
  constexpr int NL = Levels<L>::n;
  if (j < 4) {
    *key = -1, *s = sub, *pidx = j;
  } else if (j < 4 + 3 * NL) {
    *key = (j - 4) / NL, *s = sub, *pidx = (j - 4) % NL;
  } else {
    const int r = j - 4 - 3 * NL;
    *key = -1, *s = sub + 1 + (r >> 1), *pidx = r & 1;
  }
}

__device__ __forceinline__ W2 block_of(const Keys& K, int key, uint32_t op, uint32_t s, uint32_t pidx, uint64_t lane) {
  return word2(key < 0 ? K.dealer : K.pair[key], op, s, pidx, lane);
}

template <int L>
__device__ __forceinline__ A3 trunc_arith(const W2* b, const A3& x, int k) {
  constexpr uint64_t M = Ring<L>::M;
  constexpr int NL = Levels<L>::n;
  if (k == 0) return x;
  const uint64_t r = b[0].a & M;
  B3 Rb;
  Rb.v[0] = b[0].b & M;
  Rb.v[1] = b[1].a & M;
  Rb.v[2] = r ^ Rb.v[0] ^ Rb.v[1];
  const uint64_t S0 = b[2].b & M, S1 = b[3].a & M;
  const uint64_t S2 = ((r >> k) - S0 - S1) & M;  // _gen_truncpairs, dealer.py:67-72
  const uint64_t c = (open<L>(x) + r) & M;       // open_a(x + r)
  const B3 s = borrow_scan_blk<L>(c, Rb, b + 4);
  B3 wrap, lowb;
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    wrap.v[i] = (s.v[i] >> (L - 1)) & 1ull;
    lowb.v[i] = (s.v[i] >> (k - 1)) & 1ull;
  }
  const W2* w = b + 4 + 3 * NL;
  const A3 wa = b2a_arith<L>(wrap, w[0].a, w[0].b, w[1].a);
  const A3 ba = b2a_arith<L>(lowb, w[2].a, w[2].b, w[3].a);
  const uint64_t sh = (1ull << (L - k)) & M;
  A3 out = a3((wa.v[0] * sh - S0 - ba.v[0]) & M, (wa.v[1] * sh - S1 - ba.v[1]) & M,
              (wa.v[2] * sh - S2 - ba.v[2]) & M);
  return add_pub<L>(out, c >> k);
}

template <int L>
__device__ __forceinline__ A3 trunc(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const A3& x, int k) {
  if (k == 0) return x;
  W2 b[TruncRand<L>::BLOCKS];
#pragma unroll
  for (int j = 0; j < TruncRand<L>::BLOCKS; ++j) {
    int key;
    uint32_t s, pidx;
    trunc_block_id<L>(j, sub, &key, &s, &pidx);
    b[j] = block_of(K, key, op, s, pidx, lane);
  }
  return trunc_arith<L>(b, x, k);
}

// Public fixed-point division schedule (div_params, gadgets.py:297-307).
struct DivParams {
  int bound, ti, sigma, kf, iters;
  uint64_t w0;
};
// subs consumed by division(): 2*(bound-1) ladder subs + 8*iters + 12
__host__ __device__ inline int div_subs(const DivParams& d) { return 2 * (d.bound - 1) + 8 * d.iters + 12; }

// Ladder step j (1 <= j < bound): t_j = b2a(~[q < 2^j]) (gadgets.py:327-332).
template <int L>
__device__ __forceinline__ A3 div_ladder_term(const Keys& K, uint32_t op, uint32_t sub0, uint64_t lane, const A3& q,
                                              int j, const DivParams& d) {
  constexpr uint64_t M = Ring<L>::M;
  const B3 below = lt<L>(K, op, sub0 + (j - 1), lane, q, a3_const((1ull << j) & M));
  const A3 t = b2a<L>(K, op, sub0 + (d.bound - 1) + (j - 1), lane, bnot(below, 1ull));
  return mul_pub<L>(t, 1ull << (d.bound - 1 - j));
}

// Newton part of division once v = 2^{B - bitlen(q)} is shared
// (gadgets.py:338-349).  `sub` = first sub after the ladder.
template <int L>
__device__ __forceinline__ A3 div_newton(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const A3& p,
                                         const A3& q, const A3& v, const DivParams& d) {
  const A3 qn = mul<L>(K, op, sub, 0, lane, q, v);
  const A3 qnorm = trunc<L>(K, op, sub + 1, lane, qn, d.bound - d.ti);
  sub += 4;
  A3 w = rsub_pub<L>(d.w0, mul_pub<L>(qnorm, 2));
  for (int it = 0; it < d.iters; ++it) {
    const A3 t = trunc<L>(K, op, sub + 1, lane, mul<L>(K, op, sub, 0, lane, qnorm, w), d.ti);
    const A3 e = rsub_pub<L>(1ull << (d.ti + 1), t);
    w = trunc<L>(K, op, sub + 5, lane, mul<L>(K, op, sub + 4, 0, lane, w, e), d.ti);
    sub += 8;
  }
  A3 pn = mul<L>(K, op, sub, 0, lane, p, v);
  if (d.sigma) pn = trunc<L>(K, op, sub + 1, lane, pn, d.sigma);
  const A3 prod = add_pub<L>(mul<L>(K, op, sub + 4, 0, lane, pn, w), 1ull << (d.kf - 1));
  return trunc<L>(K, op, sub + 5, lane, prod, d.kf);
}

// Full serial division for one lane (division, gadgets.py:310-349).
template <int L>
__device__ __forceinline__ A3 division(const Keys& K, uint32_t op, uint32_t sub, uint64_t lane, const A3& p,
                                       const A3& q, const DivParams& d) {
  A3 acc = a3(0, 0, 0);
  for (int j = 1; j < d.bound; ++j) acc = add<L>(acc, div_ladder_term<L>(K, op, sub, lane, q, j, d));
  const A3 v = rsub_pub<L>(1ull << (d.bound - 1), acc);
  return div_newton<L>(K, op, sub + 2 * (d.bound - 1), lane, p, q, v, d);
}

}  // namespace gt
