// Standalone gadget entry points of the C ABI (include/gtree_b200.h).  These
// run one reference gadget call (gadgets.py / oaa.py / rss.py) over a batch
// of lanes; the training and inference drivers use the same per-lane device
// functions fused into larger kernels.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "gt_common.cuh"
#include "gt_division.cuh"
#include "gt_lookup.cuh"

namespace gt {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
int fail_cuda(cudaError_t e, const char* where) {
  set_error(std::string(where) + ": " + cudaGetErrorString(e));
  return GT_ECUDA;
}
int fail_inval(const std::string& msg) {
  set_error(msg);
  return GT_EINVAL;
}

namespace {

constexpr int TPB = 256;

inline unsigned blocks_for(uint64_t n) { return (unsigned)((n + TPB - 1) / TPB); }

__device__ __forceinline__ A3 ld3(const uint64_t* p, uint64_t n, uint64_t i) {
  return a3(p[i], p[n + i], p[2 * n + i]);
}
__device__ __forceinline__ void st3(uint64_t* p, uint64_t n, uint64_t i, const A3& a) {
  p[i] = a.v[0];
  p[n + i] = a.v[1];
  p[2 * n + i] = a.v[2];
}
__device__ __forceinline__ B3 ldb(const uint8_t* p, uint64_t n, uint64_t i) {
  B3 b;
  b.v[0] = p[i] & 1;
  b.v[1] = p[n + i] & 1;
  b.v[2] = p[2 * n + i] & 1;
  return b;
}
__device__ __forceinline__ void stb(uint8_t* p, uint64_t n, uint64_t i, const B3& b) {
  p[i] = (uint8_t)(b.v[0] & 1);
  p[n + i] = (uint8_t)(b.v[1] & 1);
  p[2 * n + i] = (uint8_t)(b.v[2] & 1);
}
template <int L>
__device__ __forceinline__ A3 operand_y(const uint64_t* y, const uint64_t* ypub, uint64_t n, uint64_t i) {
  if (y) return ld3(y, n, i);
  return a3_const(ypub ? (ypub[i] & Ring<L>::M) : 0ull);
}

template <int L>
__global__ void k_mul(const uint64_t* x, const uint64_t* y, uint64_t* z, uint64_t n, Keys K, uint32_t op) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  st3(z, n, i, mul<L>(K, op, 0, 0, i, ld3(x, n, i), ld3(y, n, i)));
}

template <int L>
__global__ void k_eq(const uint64_t* x, const uint64_t* y, const uint64_t* ypub, uint8_t* out, uint64_t n, Keys K,
                     uint32_t op) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  stb(out, n, i, eqz<L>(K, op, 0, i, diff<L>(ld3(x, n, i), operand_y<L>(y, ypub, n, i))));
}

template <int L>
__global__ void k_lt(const uint64_t* x, const uint64_t* y, const uint64_t* ypub, uint8_t* out, uint64_t n, Keys K,
                     uint32_t op) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  stb(out, n, i, lt<L>(K, op, 0, i, ld3(x, n, i), operand_y<L>(y, ypub, n, i)));
}

template <int L>
__global__ void k_b2a(const uint8_t* bits, uint64_t* out, uint64_t n, Keys K, uint32_t op) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  st3(out, n, i, b2a<L>(K, op, 0, i, ldb(bits, n, i)));
}

// one thread per payload element; the condition's b2a is recomputed per
// element of its group (same lane/op/sub -> identical dabit).
template <int L>
__global__ void k_select(const uint64_t* w1, const uint64_t* w2, const uint8_t* cond, uint64_t* out, uint64_t ncond,
                         uint64_t group, Keys K, uint32_t op) {
  uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t n = ncond * group;
  if (e >= n) return;
  uint64_t c = e / group, k = e % group;
  const A3 ca = b2a<L>(K, op, 0, c, ldb(cond, ncond, c));
  st3(out, n, e, select_with<L>(K, op, 0, (uint32_t)k, c, ld3(w1, n, e), ld3(w2, n, e), ca));
}

template <int L>
__global__ void k_trunc(const uint64_t* x, uint64_t* out, uint64_t n, int k, Keys K, uint32_t op) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  st3(out, n, i, trunc<L>(K, op, 0, i, ld3(x, n, i), k));
}

// one warp per division lane (gt_division.cuh), 4 warps per CTA
template <int L>
__global__ void k_division(const uint64_t* p, const uint64_t* q, uint64_t* out, uint64_t n, DivParams d, Keys K,
                           uint32_t op) {
  extern __shared__ W2 tape_sm[];
  const int warp = threadIdx.x >> 5;
  const uint64_t i = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
  if (i >= n) return;
  const A3 r = division_warp<L>(K, op, 0, i, ld3(p, n, i), ld3(q, n, i), d, tape_sm + warp * division_tape_blocks<L>(d));
  if ((threadIdx.x & 31) == 0) st3(out, n, i, r);
}

// argmin_masked, one row per thread; subs: 0/1 masking select, round r at
// 2+5r (lt), 3+5r/4+5r (value select), 5+5r/6+5r (index select, Z_2^64).
constexpr int ARGMIN_MAX = 128;
template <int L>
__global__ void k_argmin(const uint64_t* scores, const uint8_t* avail, uint64_t* out, uint64_t n, uint64_t m,
                         uint64_t worst, Keys K, uint32_t op, uint64_t* scratch) {
  uint64_t row = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (row >= n) return;
  const uint64_t nm = n * m;
  uint64_t* vals = scratch + row * (6 * m);  // [3][m] values, [3][m] indices
  uint64_t* idxs = vals + 3 * m;
  for (uint64_t j = 0; j < m; ++j) {
    const uint64_t e = row * m + j;
    const A3 v = select1<L>(K, op, 0, e, a3_const(worst & Ring<L>::M), ld3(scores, nm, e), ldb(avail, nm, e));
    for (int c = 0; c < 3; ++c) {
      vals[c * m + j] = v.v[c];
      idxs[c * m + j] = c == 0 ? j : 0;
    }
  }
  uint64_t cur = m;
  for (int r = 0; cur > 1; ++r) {
    const uint64_t pairs = cur / 2;
    const uint32_t base = 2 + 5 * r;
    for (uint64_t p = 0; p < pairs; ++p) {
      const uint64_t lane = row * m + p;
      const A3 av = a3(vals[2 * p], vals[m + 2 * p], vals[2 * m + 2 * p]);
      const A3 bv = a3(vals[2 * p + 1], vals[m + 2 * p + 1], vals[2 * m + 2 * p + 1]);
      const A3 ai = a3(idxs[2 * p], idxs[m + 2 * p], idxs[2 * m + 2 * p]);
      const A3 bi = a3(idxs[2 * p + 1], idxs[m + 2 * p + 1], idxs[2 * m + 2 * p + 1]);
      const B3 cw = lt<L>(K, op, base, lane, bv, av);
      const A3 nv = select1<L>(K, op, base + 1, lane, av, bv, cw);
      const A3 ni = select1<64>(K, op, base + 3, lane, ai, bi, cw);
      for (int c = 0; c < 3; ++c) {  // p <= 2p: in-place compaction is safe
        vals[c * m + p] = nv.v[c];
        idxs[c * m + p] = ni.v[c];
      }
    }
    if (cur & 1) {
      for (int c = 0; c < 3; ++c) {
        vals[c * m + pairs] = vals[c * m + cur - 1];
        idxs[c * m + pairs] = idxs[c * m + cur - 1];
      }
    }
    cur = pairs + (cur & 1);
  }
  out[row] = idxs[0];
  out[n + row] = idxs[m];
  out[2 * n + row] = idxs[2 * m];
}

template <int L>
__global__ void k_oaa(const uint64_t* table, uint64_t m, const uint64_t* idx, uint64_t* out, uint64_t n, Keys K,
                      uint32_t op) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto entry = [&](int j) { return ld3(table, m, (uint64_t)j); };
  st3(out, n, i, lookup_partial<L>(K, op, i, ld3(idx, n, i), (int)m, 0, 1, entry));
}

template <int L>
__global__ void k_row_lookup(const uint64_t* rows, uint64_t m, const uint64_t* idx, uint64_t* out, uint64_t n, Keys K,
                             uint32_t op) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t nm = n * m;
  auto entry = [&](int j) { return ld3(rows, nm, i * m + (uint64_t)j); };
  st3(out, n, i, lookup_partial<L>(K, op, i, ld3(idx, n, i), (int)m, 0, 1, entry));
}

bool width_ok(int w) { return w == 8 || w == 32 || w == 64; }

__global__ void __launch_bounds__(256) k_diag_philox(uint32_t iters, uint64_t* out, Keys K) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t acc = 0;
  for (uint32_t i = 0; i < iters; i += 4) {
    // four independent blocks per step, like three pair keys + a dealer key
    const W2 a = word2(K.pair[0], i, 1, 0, t);
    const W2 b = word2(K.pair[1], i, 1, 0, t);
    const W2 c = word2(K.pair[2], i, 1, 0, t);
    const W2 d = word2(K.dealer, i, 1, 0, t);
    acc += a.a ^ b.b ^ c.a ^ d.b ^ a.b ^ b.a ^ c.b ^ d.a;
  }
  out[t] = acc;
}

// Deal-directory / material-bank loading (reference rss.py:452-481,
// dealer.py:131-176): party i's little-endian ring words at lo.p[i] (stride
// bytes apart) become component i of out[3][n]; hi.p[i] must equal the next
// party's lo word (replicated sharing), mismatches counted into *bad.
struct Ptr3 {
  const uint8_t* p[3];
};
__device__ __forceinline__ uint64_t le_word(const uint8_t* q, uint32_t wb) {
  if (wb == 8 && (reinterpret_cast<uintptr_t>(q) & 7) == 0) return *reinterpret_cast<const uint64_t*>(q);
  uint64_t v = 0;
  for (uint32_t b = 0; b < wb; ++b) v |= (uint64_t)q[b] << (8 * b);
  return v;
}
__global__ void k_unpack_pairs(Ptr3 lo, Ptr3 hi, uint32_t stride, uint32_t wb, uint64_t n, uint64_t* out,
                               unsigned long long* bad) {
  const uint64_t e = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= 3 * n) return;
  const int i = (int)(e / n);
  const uint64_t k = e - (uint64_t)i * n;
  out[e] = le_word(lo.p[i] + k * stride, wb);
  if (bad && le_word(hi.p[i] + k * stride, wb) != le_word(lo.p[(i + 1) % 3] + k * stride, wb)) atomicAdd(bad, 1ull);
}

}  // namespace
}  // namespace gt

using namespace gt;

#define GT_DISPATCH(width, KERNEL, GRID, ...)                                   \
  do {                                                                          \
    cudaStream_t _s = (cudaStream_t)stream;                                     \
    if ((width) == 64) KERNEL<64><<<(GRID), TPB, 0, _s>>>(__VA_ARGS__);         \
    else if ((width) == 32) KERNEL<32><<<(GRID), TPB, 0, _s>>>(__VA_ARGS__);    \
    else KERNEL<8><<<(GRID), TPB, 0, _s>>>(__VA_ARGS__);                        \
  } while (0)

#define GT_CHECK_COMMON(width, keys)                                             \
  do {                                                                           \
    if (!width_ok(width)) return fail_inval("unsupported ring width");           \
    if (!(keys)) return fail_inval("keys must not be NULL");                     \
  } while (0)

extern "C" {

int gt_abi_version(void) { return GT_ABI_VERSION; }

int gt_unpack_pairs(const void* const* lo, const void* const* hi, uint32_t stride_bytes, uint32_t word_bytes,
                    uint64_t n, uint64_t* out, unsigned long long* mismatches, void* stream) {
  if (!lo || !hi || !out) return fail_inval("gt_unpack_pairs: NULL operand");
  if (word_bytes != 1 && word_bytes != 4 && word_bytes != 8) return fail_inval("word_bytes must be 1, 4 or 8");
  if (stride_bytes < word_bytes) return fail_inval("stride shorter than a word");
  if (n == 0) return GT_OK;
  Ptr3 l, h;
  for (int i = 0; i < 3; ++i) {
    if (!lo[i] || !hi[i]) return fail_inval("gt_unpack_pairs: NULL component");
    l.p[i] = (const uint8_t*)lo[i];
    h.p[i] = (const uint8_t*)hi[i];
  }
  k_unpack_pairs<<<blocks_for(3 * n), TPB, 0, (cudaStream_t)stream>>>(l, h, stride_bytes, word_bytes, n, out,
                                                                       mismatches);
  GT_LAUNCH_CHECK("gt_unpack_pairs");
  return GT_OK;
}

// Host staging of the three parties' replicated pairs (the drop-in's
// rendezvous, rss.py:222-228 consistency): component i = party i+1's lo is
// copied to out + i n; party i+1's hi must equal party i+2's lo word for word.
// Split over host threads in 1 MB slices (memcmp + memcpy stream at memory
// speed); returns GT_ERR_INVALID on an inconsistent pair.
namespace {
// Persistent host workers for the staging copies / checks of the drop-in
// path (a fresh std::thread per worker per call cost ~0.1 ms per call).  One
// job at a time (callers serialise on run_mu); the caller works too.
struct HostPool {
  std::vector<std::thread> th;
  std::mutex mu, run_mu;
  std::condition_variable cv, done_cv;
  std::function<void()> job;
  uint64_t gen = 0;
  unsigned pending = 0;
  explicit HostPool(unsigned n) {
    for (unsigned t = 0; t < n; ++t)
      th.emplace_back([this] {
        uint64_t seen = 0;
        for (;;) {
          std::function<void()> j;
          {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return gen != seen; });
            seen = gen;
            j = job;
          }
          j();
          std::lock_guard<std::mutex> lk(mu);
          if (--pending == 0) done_cv.notify_one();
        }
      });
    for (auto& t : th) t.detach();  // process-lifetime workers
  }
  void run(const std::function<void()>& f) {  // f on every worker and the caller
    std::lock_guard<std::mutex> rl(run_mu);
    {
      std::lock_guard<std::mutex> lk(mu);
      job = f;
      pending = (unsigned)th.size();
      ++gen;
    }
    cv.notify_all();
    f();
    std::unique_lock<std::mutex> lk(mu);
    done_cv.wait(lk, [&] { return pending == 0; });
  }
};
HostPool& host_pool() {
  static HostPool* p = new HostPool(std::max(1u, std::min(8u, std::thread::hardware_concurrency())) - 1u);
  return *p;
}
}  // namespace

int gt_stage_pairs(const uint64_t* const* lo, const uint64_t* const* hi, uint64_t n, uint64_t* out, int check) {
  if (!lo || !hi || (!out && !check)) return fail_inval("gt_stage_pairs: NULL operand");
  for (int i = 0; i < 3; ++i)
    if (n && (!lo[i] || !hi[i])) return fail_inval("gt_stage_pairs: NULL component");
  const uint64_t slice = 1ull << 17;  // words
  const uint64_t nsl = (n + slice - 1) / slice;
  std::atomic<uint64_t> next{0};
  std::atomic<int> bad{0};
  auto work = [&]() {
    for (uint64_t k = next++; k < 3 * nsl && !bad.load(std::memory_order_relaxed); k = next++) {
      const int i = (int)(k / nsl);
      const uint64_t a = (k % nsl) * slice, len = std::min<uint64_t>(slice, n - a);
      if (check && std::memcmp(hi[i] + a, lo[(i + 1) % 3] + a, len * 8) != 0) bad = 1;
      if (out) std::memcpy(out + (uint64_t)i * n + a, lo[i] + a, len * 8);
    }
  };
  if (3 * nsl <= 1) work();
  else host_pool().run(work);
  if (bad) return fail_inval("replication inconsistency between party pairs");
  return GT_OK;
}
const char* gt_last_error(void) { return g_last_error.c_str(); }

int gt_mul(int width, const uint64_t* x, const uint64_t* y, uint64_t* z, uint64_t n, const gt_keys* keys, uint32_t op,
           void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (n == 0) return GT_OK;
  if (!x || !y || !z) return fail_inval("gt_mul: NULL operand");
  GT_DISPATCH(width, k_mul, blocks_for(n), x, y, z, n, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_mul");
  return GT_OK;
}

int gt_eq(int width, const uint64_t* x, const uint64_t* y, const uint64_t* y_pub, uint8_t* out, uint64_t n,
          const gt_keys* keys, uint32_t op, void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (n == 0) return GT_OK;
  if (!x || !out) return fail_inval("gt_eq: NULL operand");
  GT_DISPATCH(width, k_eq, blocks_for(n), x, y, y_pub, out, n, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_eq");
  return GT_OK;
}

int gt_lt(int width, const uint64_t* x, const uint64_t* y, const uint64_t* y_pub, uint8_t* out, uint64_t n,
          const gt_keys* keys, uint32_t op, void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (n == 0) return GT_OK;
  if (!x || !out) return fail_inval("gt_lt: NULL operand");
  GT_DISPATCH(width, k_lt, blocks_for(n), x, y, y_pub, out, n, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_lt");
  return GT_OK;
}

int gt_b2a(int width, const uint8_t* bits, uint64_t* out, uint64_t n, const gt_keys* keys, uint32_t op,
           void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (n == 0) return GT_OK;
  if (!bits || !out) return fail_inval("gt_b2a: NULL operand");
  GT_DISPATCH(width, k_b2a, blocks_for(n), bits, out, n, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_b2a");
  return GT_OK;
}

int gt_select(int width, const uint64_t* w1, const uint64_t* w2, const uint8_t* cond, uint64_t* out, uint64_t n_cond,
              uint64_t group, const gt_keys* keys, uint32_t op, void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (group == 0 || group > 512) return fail_inval("payload size must be a multiple of condition size (group 1..512)");
  if (n_cond == 0) return GT_OK;
  if (!w1 || !w2 || !cond || !out) return fail_inval("gt_select: NULL operand");
  GT_DISPATCH(width, k_select, blocks_for(n_cond * group), w1, w2, cond, out, n_cond, group, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_select");
  return GT_OK;
}

int gt_truncate(int width, const uint64_t* x, uint64_t* out, uint64_t n, int k, const gt_keys* keys, uint32_t op,
                void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (k < 0 || k >= width) return fail_inval("truncation amount out of range for width");
  if (n == 0) return GT_OK;
  if (!x || !out) return fail_inval("gt_truncate: NULL operand");
  GT_DISPATCH(width, k_trunc, blocks_for(n), x, out, n, k, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_truncate");
  return GT_OK;
}

int gt_division(int width, const uint64_t* p, const uint64_t* q, uint64_t* out, uint64_t n, int tau,
                const gt_keys* keys, uint32_t op, void* stream) {
  GT_CHECK_COMMON(width, keys);
  bool ok = false;
  DivParams d = div_params(width, tau, &ok);
  if (!ok || tau < 0 || tau >= width - 2) return fail_inval("division unsupported at this width/tau");
  if (n == 0) return GT_OK;
  if (!p || !q || !out) return fail_inval("gt_division: NULL operand");
  cudaStream_t s = (cudaStream_t)stream;
  const Keys K = to_keys(keys);
  auto launch = [&](auto kern, int blocks) -> int {
    const int per_warp = blocks * (int)sizeof(W2);
    const int wpc = std::max(1, std::min(4, (200 * 1024) / per_warp));
    GT_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, per_warp * wpc));
    kern<<<(unsigned)((n + wpc - 1) / wpc), 32 * wpc, per_warp * wpc, s>>>(p, q, out, n, d, K, op);
    return GT_OK;
  };
  int rc;
  if (width == 64) rc = launch(k_division<64>, division_tape_blocks<64>(d));
  else if (width == 32) rc = launch(k_division<32>, division_tape_blocks<32>(d));
  else rc = launch(k_division<8>, division_tape_blocks<8>(d));
  if (rc) return rc;
  GT_LAUNCH_CHECK("gt_division");
  return GT_OK;
}

uint64_t gt_argmin_scratch_words(uint64_t n, uint64_t m) { return n * 6 * m; }

int gt_argmin(int width, const uint64_t* scores, const uint8_t* avail, uint64_t* out, uint64_t n, uint64_t m,
              uint64_t worst, const gt_keys* keys, uint32_t op, uint64_t* scratch, void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (m == 0 || m > ARGMIN_MAX) return fail_inval("argmin: need 1 <= m <= 128 columns");
  if (n == 0) return GT_OK;
  if (!scores || !avail || !out || !scratch) return fail_inval("gt_argmin: NULL operand");
  GT_DISPATCH(width, k_argmin, blocks_for(n), scores, avail, out, n, m, worst, to_keys(keys), op, scratch);
  GT_LAUNCH_CHECK("gt_argmin");
  return GT_OK;
}

int gt_oaa(int width, const uint64_t* table, uint64_t m, const uint64_t* idx, uint64_t* out, uint64_t n,
           const gt_keys* keys, uint32_t op, void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (n == 0) return GT_OK;
  if (!idx || !out || (m && !table)) return fail_inval("gt_oaa: NULL operand");
  GT_DISPATCH(width, k_oaa, blocks_for(n), table, m, idx, out, n, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_oaa");
  return GT_OK;
}

int gt_row_lookup(int width, const uint64_t* rows, uint64_t m, const uint64_t* idx, uint64_t* out, uint64_t n,
                  const gt_keys* keys, uint32_t op, void* stream) {
  GT_CHECK_COMMON(width, keys);
  if (n == 0) return GT_OK;
  if (!idx || !out || (m && !rows)) return fail_inval("gt_row_lookup: NULL operand");
  GT_DISPATCH(width, k_row_lookup, blocks_for(n), rows, m, idx, out, n, to_keys(keys), op);
  GT_LAUNCH_CHECK("gt_row_lookup");
  return GT_OK;
}

int gt_diag_philox(uint32_t grid, uint32_t iters, uint64_t* out, void* stream) {
  if (!out || grid == 0) return fail_inval("gt_diag_philox: bad arguments");
  gt_keys k{};
  k.dealer.k0 = 1;
  for (int i = 0; i < 3; ++i) k.pair[i].k0 = 2 + i;
  k_diag_philox<<<grid, 256, 0, (cudaStream_t)stream>>>(iters, out, to_keys(&k));
  GT_LAUNCH_CHECK("gt_diag_philox");
  return GT_OK;
}

}  // extern "C"
