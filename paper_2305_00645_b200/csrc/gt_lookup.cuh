// Oblivious array access lanes (oaa / row_lookup, reference oaa.py:20-55).
// Each index is compared against the public ramp 0..m-1 with one eq lane per
// entry, the hit bit is converted (b2a) and multiplies the entry (select
// against zero), and the picked shares are summed locally.  There is no
// data-dependent addressing: every lane reads every entry.  Lane numbering
// is (global index) * m + j; the lane's eq, b2a and reshare draw from the six
// Philox blocks of LaneRand at sub 0.
#pragma once
#include "gt_gadgets.cuh"

namespace gt {

// Partial sum over entries j = j0, j0 + js, ... < m of one lookup.
// `entry(j)` returns the A3 shares of table entry j.
template <int L, typename Entry>
__device__ __forceinline__ A3 lookup_partial(const Keys& K, uint32_t op, uint64_t gidx, const A3& idx, int m, int j0,
                                             int js, Entry entry) {
  A3 acc = a3(0, 0, 0);
  for (int j = j0; j < m; j += js) {
    const uint64_t lane = gidx * (uint64_t)m + (uint64_t)j;
    const A3 d = add_pub<L>(idx, (0ull - (uint64_t)j) & Ring<L>::M);
    const LaneRand R = lane_rand(K, op, 0, lane);
    const B3 hit = eq_arith<L>(d, R.r, R.Rb0, R.Rb1, R.Zw);
    const A3 ca = b2a_arith<L>(hit, R.A0, R.A1, R.bits);
    // select_share(zero, rows, hit): w2 - w1 = rows (oaa.py:33)
    acc = add<L>(acc, mul_z<L>(entry(j), ca, R.F));
  }
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
