// Oblivious array access lanes (oaa / row_lookup, reference oaa.py:20-55).
// Each index is compared against the public ramp 0..m-1 with one eq lane per
// entry, the hit bit is converted (b2a) and multiplies the entry (select
// against zero), and the picked shares are summed locally.  There is no
// data-dependent addressing: every lane reads every entry.  Lane numbering
// is (global index) * m + j (randomness schedule: lookup_partial).
#pragma once
#include "gt_gadgets.cuh"

namespace gt {

// Partial sum of one lookup over the entry pairs q = q0, q0 + qs, ...
// (entries 2q, 2q+1; lane = gidx * m + j).  The pair's AND-tree zero words
// come from one pair block per key at lane gidx * ceil(m/2) + q (.a for the
// even entry, .b for the odd one).  The selects' reshare zero shares follow
// the telescoping stream F_i(lane) = H_i(lane + 1) - H_i(lane) (H_i = pair_i
// word at sub 1), so their sum over the lookup's m entries is added once:
// H_i(gidx m + m) - H_i(gidx m) per key, its six words spread over the group.
// `entry(j)` returns the A3 shares of table entry j.

// One telescope endpoint word of a lookup's reshare sum (e = 0..5: key e % 3,
// end point for e < 3, start point otherwise).  Key i's word w adds +w to
// component i and -w to component i+1 (F_i - F_{i-1} per component).
template <int L>
__device__ __forceinline__ A3 lookup_word(const Keys& K, uint32_t op, uint64_t gidx, int m, int e) {
  const int i = e % 3;
  const uint64_t w = word(K.pair[i], op, 1, 0, gidx * (uint64_t)m + (e < 3 ? (uint64_t)m : 0ull));
  const uint64_t v = e < 3 ? w : 0ull - w;
  A3 r;
#pragma unroll
  for (int c = 0; c < 3; ++c)  // compile-time component index: the A3 stays in registers
    r.v[c] = (c == i ? v : (c == (i + 1) % 3 ? 0ull - v : 0ull)) & Ring<L>::M;
  return r;
}

// Entry pair q (entries 2q, 2q+1) of one lookup, data-independent of the
// table: eq lanes vs the public ramp and b2a of the hits (oaa.py:26-32) --
// the arithmetic shares ca0, ca1 of the two hit bits (ca1 = 0 past m).
template <int L>
__device__ __forceinline__ void lookup_pair_ca(const Keys& K, uint32_t op, uint64_t gidx, const A3& idx, int m, int q,
                                               A3* ca0, A3* ca1) {
  const int mh = (m + 1) >> 1;
  W2 Z[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) Z[i] = word2(K.pair[i], op, 0, 0, gidx * (uint64_t)mh + (uint64_t)q);
  *ca1 = a3(0, 0, 0);
  if constexpr (L == 64) {  // both entries' eq trees packed together (eq_arith64_x2)
    const int j0 = 2 * q, j1 = 2 * q + 1;
    const uint64_t lane0 = gidx * (uint64_t)m + (uint64_t)j0;
    const A3 d0 = add_pub<L>(idx, 0ull - (uint64_t)j0), d1 = add_pub<L>(idx, 0ull - (uint64_t)j1);
    const DealerRand R0 = dealer_rand(K, op, lane0), R1 = dealer_rand(K, op, lane0 + 1);
    const uint64_t Z0[3] = {Z[0].a, Z[1].a, Z[2].a}, Z1[3] = {Z[0].b, Z[1].b, Z[2].b};
    B3 h0, h1;
    eq_arith64_x2<false>(d0, R0.r, R0.Rb0, R0.Rb1, Z0, d1, R1.r, R1.Rb0, R1.Rb1, Z1, &h0, &h1);
    *ca0 = b2a_arith<L>(h0, R0.A0, R0.A1, R0.bits);
    if (j1 < m) *ca1 = b2a_arith<L>(h1, R1.A0, R1.A1, R1.bits);
    return;
  } else {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int j = 2 * q + h;
    if (j >= m) break;
    const uint64_t lane = gidx * (uint64_t)m + (uint64_t)j;
    const A3 d = add_pub<L>(idx, (0ull - (uint64_t)j) & Ring<L>::M);
    const DealerRand R = dealer_rand(K, op, lane);
    const uint64_t Zw[3] = {h ? Z[0].b : Z[0].a, h ? Z[1].b : Z[1].a, h ? Z[2].b : Z[2].a};
    const B3 hit = eq_arith<L>(d, R.r, R.Rb0, R.Rb1, Zw);
    *(h ? ca1 : ca0) = b2a_arith<L>(hit, R.A0, R.A1, R.bits);
  }
  }
}

// Entry pair q of one lookup: the hits' shares select the entries against
// zero (select_share(zero, rows, hit): w2 - w1 = rows, oaa.py:33) -- the
// picked shares of this pair, local cross terms only.
template <int L, typename Entry>
__device__ __forceinline__ A3 lookup_pair(const Keys& K, uint32_t op, uint64_t gidx, const A3& idx, int m, int q,
                                          Entry entry) {
  const uint64_t F0[3] = {0, 0, 0};
  A3 ca0, ca1;
  lookup_pair_ca<L>(K, op, gidx, idx, m, q, &ca0, &ca1);
  A3 acc = mul_z<L>(entry(2 * q), ca0, F0);
  if (2 * q + 1 < m) acc = add<L>(acc, mul_z<L>(entry(2 * q + 1), ca1, F0));
  return acc;
}

// The part of one lookup that member q0 of a qs-member group computes: the
// six telescope words e = q0, q0 + qs, ... and the entry pairs starting past
// them (a group of >= 8 has no member holding both a word and the first
// pair); the group sum is the whole lookup.
template <int L, typename Entry>
__device__ __forceinline__ A3 lookup_partial(const Keys& K, uint32_t op, uint64_t gidx, const A3& idx, int m, int q0,
                                             int qs, Entry entry) {
  const int mh = (m + 1) >> 1;
  A3 acc = a3(0, 0, 0);
  for (int e = q0; e < 6; e += qs) acc = add<L>(acc, lookup_word<L>(K, op, gidx, m, e));
  const int first = (q0 + qs - (6 % qs)) % qs;
  for (int q = first; q < mh; q += qs) acc = add<L>(acc, lookup_pair<L>(K, op, gidx, idx, m, q, entry));
  return acc;
}

// xor-butterfly sum over a group of G lanes of a warp (G divides 32).
template <int G, int L>
__device__ __forceinline__ A3 group_sum(A3 a) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
#pragma unroll
    for (int i = 0; i < 3; ++i) a.v[i] = (a.v[i] + __shfl_xor_sync(0xffffffffu, a.v[i], o)) & Ring<L>::M;
  }
  return a;
}

}  // namespace gt
