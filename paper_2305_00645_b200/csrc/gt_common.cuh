// Shared host/device plumbing for the C-ABI library: error reporting,
// op-id layout, launch helpers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/gtree_b200.h"
#include "gt_gadgets.cuh"

namespace gt {

// Op ids: (level << 16) | site.  One site per gadget call site of the
// reference level loop (train.py:108-197, infer.py:20-35).
enum Site : uint32_t {
  SITE_PRODS = 1,     // count:0 features x labels          train.py:115-116
  SITE_PART_OAA = 2,  // partition oaa on level payloads    train.py:135-137
  SITE_PART_ROW = 3,  // partition row_lookup on features   train.py:138
  SITE_ISLEAF = 4,    // count is_leaf = eq(F, LEAF)        train.py:206
  SITE_COUNT = 5,     // count lanes (eq, and, b2a, mul)    train.py:211-221
  SITE_HC = 6,        // _heuristic_mpc                     train.py:232-274
  SITE_REPLACE = 7,   // replace:h                          train.py:155-162
  SITE_SPLIT = 8,     // split:h                            train.py:170-176
  SITE_LABELS = 9,    // labels:h                           train.py:186-192
  SITE_STOP = 10,     // grow-policy stop bit               train.py:165-168
  SITE_WALK_OAA = 16, // walk:t oaa                         infer.py:30-31
  SITE_WALK_ROW = 17, // walk:t row_lookup                  infer.py:32
};
__host__ __device__ inline uint32_t op_id(int level, uint32_t site) { return ((uint32_t)level << 16) | site; }

void set_error(const std::string& msg);
int fail_cuda(cudaError_t e, const char* where);
int fail_inval(const std::string& msg);

inline Keys to_keys(const gt_keys* k) {
  Keys K;
  K.dealer = expand_key(k->dealer.k0, k->dealer.k1);
  for (int i = 0; i < 3; ++i) K.pair[i] = expand_key(k->pair[i].k0, k->pair[i].k1);
  return K;
}

inline DivParams div_params(int width, int tau, bool* ok) {
  // gadgets.py:297-307
  DivParams d;
  d.bound = width - tau - 2;
  d.ti = tau + 4;
  int s = d.bound + d.ti + 5 - width;
  d.sigma = s > 0 ? s : 0;
  d.kf = d.bound + d.ti - d.sigma - tau;
  int it = 2;
  if (tau > 1) {
    int c = 0;
    while ((1 << c) < tau) ++c;  // ceil(log2 tau)
    it = c + 2;
  }
  d.iters = it;
  // round(2.9142 * 2^ti), Python round-half-even on an exact binary product
  double w = 2.9142 * (double)(1ull << d.ti);
  double fl = (double)(uint64_t)w;
  double frac = w - fl;
  uint64_t r = (uint64_t)fl;
  if (frac > 0.5 || (frac == 0.5 && (r & 1))) r += 1;
  d.w0 = r;
  *ok = !(d.ti >= d.bound || d.kf < 1);
  return d;
}

#define GT_CUDA_CHECK(expr)                                     \
  do {                                                          \
    cudaError_t _e = (expr);                                    \
    if (_e != cudaSuccess) return ::gt::fail_cuda(_e, #expr);  \
  } while (0)

#define GT_LAUNCH_CHECK(where)                                  \
  do {                                                          \
    cudaError_t _e = cudaGetLastError();                        \
    if (_e != cudaSuccess) return ::gt::fail_cuda(_e, where);  \
  } while (0)

// Programmatic dependent launch: the level-chain kernels are launched with
// programmatic stream serialization (launch_chain), so a kernel's CTAs start
// -- and issue their precomputed-tape bulk copies -- while its predecessor's
// last wave drains.  pdl_wait() blocks until the predecessor grid has
// completed and its writes are visible (a no-op for normal launches): every
// read of a predecessor's output and every global write comes after it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

}  // namespace gt
