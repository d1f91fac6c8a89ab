// Party-local steps of the three-host deployment: each party
// runs on its own device (or rank) holding ONE replicated pair per shared
// vector -- (lo, hi) = (c_i, c_{i+1}), i = party - 1 (rss.py:1-9) -- and the
// protocol's rounds are real messages on the P_i -> P_{i+1} ring
// (transport.py:374-475, rss.py:371-412), exchanged by the host between
// these kernels:
//   open      : send lo to next, x = lo + hi + (prev's lo)
//   mul / and : z_i = local cross terms + zero share, send z_i to prev, the
//               pair becomes (z_i, z_{i+1})
// Correlated material comes from this party's dealt bank (material.py, OBD1
// banks on the device); zero shares from the two pairwise keys the party
// holds, pair[i] (shared with next) and pair[i-1] (shared with prev):
// alpha_i = F(pair[i]) - F(pair[i-1]) as in the co-resident kernels.
// Pair arrays are [2][L] (lo row, then hi row).
#include "gt_common.cuh"

namespace gt {
namespace {

constexpr int PTPB = 256;
inline unsigned pblocks(uint64_t n) { return (unsigned)((n + PTPB - 1) / PTPB); }

// public constant on component 0: party 1's lo, party 3's hi (rss.py:313-367)
__device__ __forceinline__ void add_pub0(int party, uint64_t& lo, uint64_t& hi, uint64_t c) {
  if (party == 1) lo += c;
  if (party == 3) hi += c;
}
__device__ __forceinline__ void xor_pub0(int party, uint64_t& lo, uint64_t& hi, uint64_t c) {
  if (party == 1) lo ^= c;
  if (party == 3) hi ^= c;
}

// eq lanes vs a public ramp: lane (q, j) opens idx[q] - off - j + r   (gadgets.py:120-130)
__global__ void k_p_eq_mask(int party, const uint64_t* idx, uint64_t nq, uint64_t m, uint64_t off, const uint64_t* r,
                            uint64_t* out) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, L = nq * m;
  if (e >= L) return;
  const uint64_t q = e / m, j = e - q * m;
  uint64_t lo = idx[q] + r[e], hi = idx[nq + q] + r[L + e];
  add_pub0(party, lo, hi, 0ull - off - j);
  out[e] = lo;
  out[L + e] = hi;
}

// c = opened mask; planes = ~(c ^ r_bits) as XOR shares of the 64 bit planes
__global__ void k_p_eq_planes(int party, const uint64_t* masked, const uint64_t* recv, const uint64_t* rbits, uint64_t L,
                              uint64_t* planes) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L) return;
  const uint64_t c = masked[e] + masked[L + e] + recv[e];
  uint64_t lo = rbits[e], hi = rbits[L + e];
  xor_pub0(party, lo, hi, ~c);
  planes[e] = lo;
  planes[L + e] = hi;
}

// one AND level of the in-word tree: the low and high halves of each lane's
// `width` bits are ANDed (and_bits, rss.py:402-412), z = new lo (width / 2 bits)
__global__ void k_p_and_half(int party, const uint64_t* P, uint64_t L, int width, Keys K, uint32_t op, uint32_t sub,
                             uint64_t lane0, uint64_t* z) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L) return;
  const int h = width >> 1;
  const uint64_t msk = h == 64 ? ~0ull : ((1ull << h) - 1);
  const uint64_t alo = P[e] & msk, blo = (P[e] >> h) & msk, ahi = P[L + e] & msk, bhi = (P[L + e] >> h) & msk;
  const int i = party - 1;
  const uint64_t zn = word(K.pair[i], op, sub, 0, lane0 + e), zp = word(K.pair[(i + 2) % 3], op, sub, 0, lane0 + e);
  z[e] = ((alo & blo) ^ (alo & bhi) ^ (ahi & blo) ^ zn ^ zp) & msk;
}

// pack `bits` low bits of each lane into a little-endian bit stream (np.packbits
// sizes: ceil(L bits / 8) bytes), one thread per output byte
__global__ void k_p_pack(const uint64_t* src, uint64_t L, int bits, uint8_t* out) {
  const uint64_t b = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nb = (L * bits + 7) / 8;
  if (b >= nb) return;
  uint32_t v = 0;
  for (int k = 0; k < 8; ++k) {
    const uint64_t bit = 8 * b + k, lane = bit / bits;
    if (lane < L) v |= (uint32_t)((src[lane] >> (bit - lane * bits)) & 1ull) << k;
  }
  out[b] = (uint8_t)v;
}
__global__ void k_p_unpack(const uint8_t* in, uint64_t L, int bits, uint64_t* dst) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L) return;
  uint64_t v = 0;
  for (int k = 0; k < bits; ++k) {
    const uint64_t bit = e * bits + k;
    v |= (uint64_t)((in[bit >> 3] >> (bit & 7)) & 1u) << k;
  }
  dst[e] = v;
}

// b2a, first half: the hit bit masked with the dabit's boolean share (e = open_bits)
__global__ void k_p_b2a_mask(const uint64_t* h, const uint8_t* bb, uint64_t L, uint64_t* e_out) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L) return;
  e_out[e] = (h[e] ^ bb[e]) & 1ull;
  e_out[L + e] = (h[L + e] ^ bb[L + e]) & 1ull;
}
// b2a, second half: out = a (1 - 2e) + e   (gadgets.py:223-231)
__global__ void k_p_b2a_finish(int party, const uint64_t* em, const uint64_t* recv, const uint64_t* a, uint64_t L,
                               uint64_t* out) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= L) return;
  const uint64_t ev = (em[e] ^ em[L + e] ^ recv[e]) & 1ull, coef = 1ull - 2ull * ev;
  uint64_t lo = a[e] * coef, hi = a[L + e] * coef;
  add_pub0(party, lo, hi, ev);
  out[e] = lo;
  out[L + e] = hi;
}

// select against zero (oaa.py:26-34): z_i of ca x entry for lane (q, j);
// entries from a shared m-entry table (per_row = 0) or from row q (per_row = 1)
__global__ void k_p_select_mul(int party, const uint64_t* ca, const uint64_t* tab, uint64_t tab_len, int per_row,
                               uint64_t nq, uint64_t m, Keys K, uint32_t op, uint32_t sub, uint64_t lane0, uint64_t* z) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, L = nq * m;
  if (e >= L) return;
  const uint64_t q = e / m, j = e - q * m, t = per_row ? q * m + j : j;
  const uint64_t xl = tab[t], xh = tab[tab_len + t], yl = ca[e], yh = ca[L + e];
  const int i = party - 1;
  const uint64_t fn = word(K.pair[i], op, sub, 0, lane0 + e), fp = word(K.pair[(i + 2) % 3], op, sub, 0, lane0 + e);
  z[e] = yl * (xl + xh) + xl * yh + fn - fp;
}

// per query: sum of its m lanes' pairs
__global__ void k_p_lane_sum(const uint64_t* pair, uint64_t nq, uint64_t m, uint64_t* out) {
  const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, L = nq * m;
  if (q >= nq) return;
  uint64_t lo = 0, hi = 0;
  for (uint64_t j = 0; j < m; ++j) {
    lo += pair[q * m + j];
    hi += pair[L + q * m + j];
  }
  out[q] = lo;
  out[nq + q] = hi;
}

// slot = 2 slot + branch + 1   (infer.py:33)
__global__ void k_p_slot_step(int party, uint64_t* slot, const uint64_t* branch, uint64_t nq) {
  const uint64_t q = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  uint64_t lo = 2 * slot[q] + branch[q], hi = 2 * slot[nq + q] + branch[nq + q];
  add_pub0(party, lo, hi, 1);
  slot[q] = lo;
  slot[nq + q] = hi;
}

}  // namespace
}  // namespace gt

using namespace gt;

#define GT_PARTY_OK(p) \
  if ((p) < 1 || (p) > 3) return fail_inval("party must be 1, 2 or 3")

extern "C" {

int gt_party_eq_mask(int party, const uint64_t* idx, uint64_t nq, uint64_t m, uint64_t off, const uint64_t* r,
                     uint64_t* out, void* stream) {
  GT_PARTY_OK(party);
  if (!nq || !m) return GT_OK;
  if (!idx || !r || !out) return fail_inval("gt_party_eq_mask: NULL operand");
  k_p_eq_mask<<<pblocks(nq * m), PTPB, 0, (cudaStream_t)stream>>>(party, idx, nq, m, off, r, out);
  GT_LAUNCH_CHECK("gt_party_eq_mask");
  return GT_OK;
}

int gt_party_eq_planes(int party, const uint64_t* masked, const uint64_t* recv, const uint64_t* rbits, uint64_t L,
                       uint64_t* planes, void* stream) {
  GT_PARTY_OK(party);
  if (!L) return GT_OK;
  if (!masked || !recv || !rbits || !planes) return fail_inval("gt_party_eq_planes: NULL operand");
  k_p_eq_planes<<<pblocks(L), PTPB, 0, (cudaStream_t)stream>>>(party, masked, recv, rbits, L, planes);
  GT_LAUNCH_CHECK("gt_party_eq_planes");
  return GT_OK;
}

int gt_party_and_half(int party, const uint64_t* planes, uint64_t L, int width, const gt_keys* keys, uint32_t op,
                      uint32_t sub, uint64_t lane0, uint64_t* z, void* stream) {
  GT_PARTY_OK(party);
  if (width < 2 || width > 64 || (width & 1)) return fail_inval("width must be even, 2..64");
  if (!L) return GT_OK;
  if (!planes || !z || !keys) return fail_inval("gt_party_and_half: NULL operand");
  k_p_and_half<<<pblocks(L), PTPB, 0, (cudaStream_t)stream>>>(party, planes, L, width, to_keys(keys), op, sub, lane0,
                                                               z);
  GT_LAUNCH_CHECK("gt_party_and_half");
  return GT_OK;
}

int gt_party_pack(const uint64_t* src, uint64_t L, int bits, uint8_t* out, void* stream) {
  if (bits < 1 || bits > 64) return fail_inval("bits must be 1..64");
  if (!L) return GT_OK;
  if (!src || !out) return fail_inval("gt_party_pack: NULL operand");
  k_p_pack<<<pblocks((L * bits + 7) / 8), PTPB, 0, (cudaStream_t)stream>>>(src, L, bits, out);
  GT_LAUNCH_CHECK("gt_party_pack");
  return GT_OK;
}

int gt_party_unpack(const uint8_t* in, uint64_t L, int bits, uint64_t* dst, void* stream) {
  if (bits < 1 || bits > 64) return fail_inval("bits must be 1..64");
  if (!L) return GT_OK;
  if (!in || !dst) return fail_inval("gt_party_unpack: NULL operand");
  k_p_unpack<<<pblocks(L), PTPB, 0, (cudaStream_t)stream>>>(in, L, bits, dst);
  GT_LAUNCH_CHECK("gt_party_unpack");
  return GT_OK;
}

int gt_party_b2a_mask(const uint64_t* h, const uint8_t* bb, uint64_t L, uint64_t* e, void* stream) {
  if (!L) return GT_OK;
  if (!h || !bb || !e) return fail_inval("gt_party_b2a_mask: NULL operand");
  k_p_b2a_mask<<<pblocks(L), PTPB, 0, (cudaStream_t)stream>>>(h, bb, L, e);
  GT_LAUNCH_CHECK("gt_party_b2a_mask");
  return GT_OK;
}

int gt_party_b2a_finish(int party, const uint64_t* e, const uint64_t* recv, const uint64_t* a, uint64_t L,
                        uint64_t* out, void* stream) {
  GT_PARTY_OK(party);
  if (!L) return GT_OK;
  if (!e || !recv || !a || !out) return fail_inval("gt_party_b2a_finish: NULL operand");
  k_p_b2a_finish<<<pblocks(L), PTPB, 0, (cudaStream_t)stream>>>(party, e, recv, a, L, out);
  GT_LAUNCH_CHECK("gt_party_b2a_finish");
  return GT_OK;
}

int gt_party_select_mul(int party, const uint64_t* ca, const uint64_t* table, uint64_t table_len, int per_row,
                        uint64_t nq, uint64_t m, const gt_keys* keys, uint32_t op, uint32_t sub, uint64_t lane0,
                        uint64_t* z, void* stream) {
  GT_PARTY_OK(party);
  if (!nq || !m) return GT_OK;
  if (!ca || !table || !z || !keys) return fail_inval("gt_party_select_mul: NULL operand");
  if (table_len < (per_row ? nq * m : m)) return fail_inval("gt_party_select_mul: table too short");
  k_p_select_mul<<<pblocks(nq * m), PTPB, 0, (cudaStream_t)stream>>>(party, ca, table, table_len, per_row, nq, m,
                                                                     to_keys(keys), op, sub, lane0, z);
  GT_LAUNCH_CHECK("gt_party_select_mul");
  return GT_OK;
}

int gt_party_lane_sum(const uint64_t* pair, uint64_t nq, uint64_t m, uint64_t* out, void* stream) {
  if (!nq) return GT_OK;
  if (!pair || !out) return fail_inval("gt_party_lane_sum: NULL operand");
  k_p_lane_sum<<<pblocks(nq), PTPB, 0, (cudaStream_t)stream>>>(pair, nq, m, out);
  GT_LAUNCH_CHECK("gt_party_lane_sum");
  return GT_OK;
}

int gt_party_slot_step(int party, uint64_t* slot, const uint64_t* branch, uint64_t nq, void* stream) {
  GT_PARTY_OK(party);
  if (!nq) return GT_OK;
  if (!slot || !branch) return fail_inval("gt_party_slot_step: NULL operand");
  k_p_slot_step<<<pblocks(nq), PTPB, 0, (cudaStream_t)stream>>>(party, slot, branch, nq);
  GT_LAUNCH_CHECK("gt_party_slot_step");
  return GT_OK;
}

}  // extern "C"
