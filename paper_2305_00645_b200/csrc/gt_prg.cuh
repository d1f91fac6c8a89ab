// Counter-based correlated randomness for the 3-party replicated-sharing
// simulation (B200 device side).
//
// Replaces the reference's AES-128-CTR streams (`AesCtrPrg`,
// reference pkg/src/obtree/transport.py:63-94) for the two randomness roles
// of the protocol:
//   * pairwise zero-shares  alpha_i = F(k_i) - F(k_{i-1})   (rss.py:302-310)
//   * dealer material: edabits / dabits / truncation pairs  (dealer.py:43-84)
// Revealed outputs of every gadget are exact functions of the plaintext
// inputs, so the choice of PRG only changes share values,
// never opened trees or predictions.
//
// Philox4x32-10 (Salmon et al., SC'11).  The counter is
//   (lane_lo, lane_hi, stream, op)
// where `lane` is the GLOBAL index of the lane inside one gadget call (so a
// sample-sharded run on G GPUs produces the same shares as G = 1), `op`
// identifies the gadget call site, and stream = (sub << 8) | (field >> 1)
// selects one 128-bit block; `field & 1` picks its low/high 64-bit word.
// The full keying schedule is specified in DESIGN.md ("Randomness schedule")
// and restated independently by oracle/gtree_oracle.c.
#pragma once
#include <stdint.h>

namespace gt {

// A Philox key with its 10-round schedule expanded once on the host
// (k0 + r*W0, k1 + r*W1), so the round XORs take the round key straight from
// the kernel's constant bank instead of re-deriving it per call.
struct Key {
  uint32_t k0[10], k1[10];
};

__host__ __device__ inline Key expand_key(uint32_t k0, uint32_t k1) {
  Key k;
  for (int r = 0; r < 10; ++r) {
    k.k0[r] = k0 + (uint32_t)r * 0x9E3779B9u;
    k.k1[r] = k1 + (uint32_t)r * 0xBB67AE85u;
  }
  return k;
}

// dealer key + the three pairwise keys; pair[i] is the seed shared by party
// i+1 and its successor (SeedSetup.pair_seeds[i+1], transport.py:113-124).
struct Keys {
  Key dealer;
  Key pair[3];
};

struct W2 {
  uint64_t a, b;
};

__device__ __forceinline__ W2 philox(const Key& key, uint32_t op, uint32_t stream, uint64_t lane) {
#ifdef GT_FAKE_PRG  // timing experiments only: a cheap non-random stand-in
  { W2 w; w.a = lane * 0x9E3779B97F4A7C15ull + stream + key.k0[0]; w.b = w.a ^ ((uint64_t)op << 17); return w; }
#endif
  uint32_t c0 = (uint32_t)lane, c1 = (uint32_t)(lane >> 32), c2 = stream, c3 = op;
#ifdef GT_PHILOX_ROLLED  // latency kernels: a rolled round loop keeps the code hot in the instruction cache
#pragma unroll 1
#else
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;  // IMAD.WIDE.U32
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ key.k0[r];  // LOP3 with a c[] operand
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ key.k1[r];
    c0 = n0;
    c1 = (uint32_t)p1;
    c2 = n2;
    c3 = (uint32_t)p0;
  }
  W2 w;
  w.a = (uint64_t)c0 | ((uint64_t)c1 << 32);
  w.b = (uint64_t)c2 | ((uint64_t)c3 << 32);
  return w;
}

__device__ __forceinline__ uint32_t stream_of(uint32_t sub, uint32_t field) {
  return (sub << 8) | (field >> 1);
}

// One 64-bit word of field `field` (fields 2j and 2j+1 share one Philox call;
// when both are requested in one inlined scope the compiler CSEs the call).
__device__ __forceinline__ uint64_t word(const Key& key, uint32_t op, uint32_t sub, uint32_t field, uint64_t lane) {
  W2 w = philox(key, op, stream_of(sub, field), lane);
  return (field & 1) ? w.b : w.a;
}

// Both words of the block holding fields (2j, 2j+1).
__device__ __forceinline__ W2 word2(const Key& key, uint32_t op, uint32_t sub, uint32_t pair_index, uint64_t lane) {
  return philox(key, op, (sub << 8) | pair_index, lane);
}

}  // namespace gt
