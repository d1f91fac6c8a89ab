/*
 * gtree_b200.h -- C ABI of the B200-native GTree (arXiv 2305.00645) MPC
 * decision-tree hot path: three-party 2-out-of-3 replicated secret sharing
 * over Z_2^64 / Z_2^32, all three parties simulated on one device exactly as
 * the reference `obtree` package simulates them on three threads.
 *
 * Conventions (every entry point):
 *   - share arrays are DEVICE pointers to component-major uint64 arrays
 *     [3][...]; component i is party (i+1)'s `lo` (AVec.lo, reference
 *     pkg/src/obtree/rss.py:53-63) and party (i+1) holds (c[i], c[(i+1)%3]);
 *   - boolean share arrays are [3][n] uint8 in {0,1} (BitVec, rss.py:151-160);
 *   - `width` is the ring width l in {8, 32, 64}; values are stored masked;
 *   - `stream` is a cudaStream_t (NULL = legacy default stream); calls are
 *     asynchronous on it, re-entrant per stream, and do not allocate: the
 *     caller owns all memory (workspace / scratch sizes are queried up
 *     front: gt_train_workspace_bytes, gt_argmin_scratch_words, ...);
 *   - return GT_OK, GT_EINVAL (bad arguments -> the reference's
 *     ValueError/UsageError) or GT_ECUDA (launch/runtime failure -> the
 *     reference's protocol errors, CLI exit code 2, cli.py:53-56);
 *     gt_last_error() gives the message of the last failure on this thread;
 *   - `op` values name the gadget call site for the counter-based PRG; the
 *     library's own training/inference drivers use op ids < 2^31, so
 *     standalone gadget calls should use op >= 2^31 to stay disjoint.
 */
#ifndef GTREE_B200_H
#define GTREE_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GT_OK 0
#define GT_EINVAL 1
#define GT_ECUDA 2

#define GT_ABI_VERSION 2

typedef struct {
  uint32_t k0, k1;
} gt_key;

/* dealer key (correlated material, dealer.py:43-84) and the three pairwise
 * keys; pair[i] is the seed party i+1 shares with its successor
 * (SeedSetup.pair_seeds[i+1], transport.py:97-124). */
typedef struct {
  gt_key dealer;
  gt_key pair[3];
} gt_keys;

int gt_abi_version(void);
const char* gt_last_error(void);

/* ---- standalone gadgets (reference pkg/src/obtree/gadgets.py, rss.py) ---- */

/* PartyEngine.mul, rss.py:386-400: z = x*y with one reshare. */
int gt_mul(int width, const uint64_t* x, const uint64_t* y, uint64_t* z, uint64_t n, const gt_keys* keys,
           uint32_t op, void* stream);
/* eq, gadgets.py:120-130: out = [x == y]; y (shared) or y_pub ([n] public) or both NULL (y = 0). */
int gt_eq(int width, const uint64_t* x, const uint64_t* y, const uint64_t* y_pub, uint8_t* out, uint64_t n,
          const gt_keys* keys, uint32_t op, void* stream);
/* lt, gadgets.py:188-216: out = [x < y] unsigned; y shared or y_pub public. */
int gt_lt(int width, const uint64_t* x, const uint64_t* y, const uint64_t* y_pub, uint8_t* out, uint64_t n,
          const gt_keys* keys, uint32_t op, void* stream);
/* b2a, gadgets.py:223-231. */
int gt_b2a(int width, const uint8_t* bits, uint64_t* out, uint64_t n, const gt_keys* keys, uint32_t op,
           void* stream);
/* select_share, gadgets.py:238-253: out = w1 + cond*(w2-w1); payload [3][n_cond*group]. */
int gt_select(int width, const uint64_t* w1, const uint64_t* w2, const uint8_t* cond, uint64_t* out,
              uint64_t n_cond, uint64_t group, const gt_keys* keys, uint32_t op, void* stream);
/* truncate, gadgets.py:260-288 (unsigned, exact floor). */
int gt_truncate(int width, const uint64_t* x, uint64_t* out, uint64_t n, int k, const gt_keys* keys, uint32_t op,
                void* stream);
/* division, gadgets.py:310-349 (width 32 or 64). */
int gt_division(int width, const uint64_t* p, const uint64_t* q, uint64_t* out, uint64_t n, int tau,
                const gt_keys* keys, uint32_t op, void* stream);
/* argmin_masked, gadgets.py:366-401: scores [3][n][m] (width), avail [3][n][m]
 * bits, out [3][n] index shares in Z_2^64; scratch: device memory of
 * gt_argmin_scratch_words(n, m) words (the per-row tournament's values and
 * indices), owned by the caller. */
uint64_t gt_argmin_scratch_words(uint64_t n, uint64_t m);
int gt_argmin(int width, const uint64_t* scores, const uint8_t* avail, uint64_t* out, uint64_t n, uint64_t m,
              uint64_t worst, const gt_keys* keys, uint32_t op, uint64_t* scratch, void* stream);
/* oaa, oaa.py:20-35: out[i] = table[idx[i]] (0 when out of range). */
int gt_oaa(int width, const uint64_t* table, uint64_t m, const uint64_t* idx, uint64_t* out, uint64_t n,
           const gt_keys* keys, uint32_t op, void* stream);
/* row_lookup, oaa.py:38-55: rows [3][n][m]; out[i] = rows[i][idx[i]]. */
int gt_row_lookup(int width, const uint64_t* rows, uint64_t m, const uint64_t* idx, uint64_t* out, uint64_t n,
                  const gt_keys* keys, uint32_t op, void* stream);

/* ---- secure training (train_tree, train.py:108-197, heuristic "mpc") ---- */

typedef struct {
  int32_t depth;       /* resolved depth H (train.py:81-86) */
  int32_t tau;         /* fixed-point bits (TrainConfig.tau) */
  int32_t score_width; /* score ring width, 32 or 64 (TrainConfig.score_ring) */
  int32_t nf;          /* features = n_columns - 1, 1..64 */
  int32_t policy;      /* 0 = fixed, 1 = grow (one opened stop bit per level) */
  int32_t heuristic;   /* 0 = mpc (on device), 1 = tee (trusted helper via callback) */
  uint64_t n_total;     /* global sample count (counter_shift, train.py:75-78) */
  uint64_t n_local;     /* samples resident on this device */
  uint64_t sample_base; /* global index of the first local sample */
  int32_t count_reshare; /* 0 = reshare every (sample, node, column) product as the
                            reference does (train.py:219); 1 = dot-product reshare: the
                            local products are summed over samples first and each counter
                            cell is reshared once (same revealed tree, n_h*W instead of
                            N*n_h*W reshared words per level) */
  int32_t count_engine;  /* count contraction: 0 = tensor cores (tcgen05.mma kind::i8 over
                            INT8 limbs of the Z_2^64 shares), 1 = CUDA cores (64-bit IMAD) --
                            identical shares */
} gt_train_cfg;

/* Sum-allreduce of `count` uint64 words in place (count partials of one
 * level, sample-sharded training).  NULL = single device. */
typedef int (*gt_allreduce_fn)(uint64_t* buf, uint64_t count, void* stream, void* user);

uint64_t gt_train_workspace_bytes(const gt_train_cfg* cfg);

/* features [3][n_local][nf], labels [3][n_local], filler [2^depth-1] public
 * placeholder stream (tree.py:160-169) in device memory; outputs T, F
 * [3][2^depth-1] shares; *depth_out = trained depth (< depth only under the
 * grow policy). */
int gt_train(const gt_train_cfg* cfg, const uint64_t* features, const uint64_t* labels, const uint64_t* filler,
             uint64_t* T, uint64_t* F, int32_t* depth_out, void* workspace, uint64_t workspace_bytes,
             const gt_keys* keys, gt_allreduce_fn allreduce, void* allreduce_user, void* stream);

/* Trusted split helper of heuristic "tee" (reference _heuristic_tee /
 * _labels_tee, train.py:277-301, EnclaveService enclave.py:94-185).  Called
 * synchronously with DEVICE pointers on `stream`:
 *   op 1 (split):  counters [3][n][3][2nf] (c_orig), gamma [3][n] bit words,
 *                  types [3][n]; writes out [4][3][n] = should_split bits,
 *                  best feature, new type, new gamma words (fresh shares);
 *   op 2 (labels): counters = effective counters, gamma/types unused; writes
 *                  out [3][n] majority-label shares.
 * Returns 0 on success. */
typedef int (*gt_heuristic_fn)(int op, int level, int n_nodes, int nf, const uint64_t* counters,
                               const uint64_t* gamma, const uint64_t* types, uint64_t* out, void* stream,
                               void* user);

/* Per-kernel-class device time of one gt_train_ex call, measured with CUDA
 * events recorded on `stream` around every launch (bench / roofline use). */
typedef struct {
  uint32_t launches; /* kernels launched by the call */
  uint32_t n_prods, n_partition, n_count, n_node_hc, n_node_finish;
  float ms_prods, ms_partition, ms_count, ms_node_hc, ms_node_finish;
  float ms_total; /* first to last event */
  /* count split: lane kernels (eq/and/b2a per (sample, node)) and the
     contraction (tcgen05 MMA or CUDA-core MAC); ms_count = their sum */
  uint32_t n_count_lanes, n_count_contract;
  float ms_count_lanes, ms_count_contract;
} gt_train_profile;

/* gt_train plus the tee helper callback (required when cfg->heuristic = 1)
 * and optional profiling (prof may be NULL; when set, the call synchronizes
 * `stream` before returning). */
int gt_train_ex(const gt_train_cfg* cfg, const uint64_t* features, const uint64_t* labels, const uint64_t* filler,
                uint64_t* T, uint64_t* F, int32_t* depth_out, void* workspace, uint64_t workspace_bytes,
                const gt_keys* keys, gt_allreduce_fn allreduce, void* allreduce_user, gt_heuristic_fn heuristic,
                void* heuristic_user, void* stream, gt_train_profile* prof);

/* gt_train with HOST operands (the same arrays as gt_train, in pinned host
 * memory): the sample shares go up in chunks on a copy stream while the
 * prologue of the chunks already resident runs, T and F come back at the end;
 * all work is ordered on `stream` (synchronise it before reading T_h / F_h).
 * The workspace must hold gt_train_host_workspace_bytes(cfg) (device). */
uint64_t gt_train_host_workspace_bytes(const gt_train_cfg* cfg);
int gt_train_host(const gt_train_cfg* cfg, const uint64_t* features_h, const uint64_t* labels_h,
                  const uint64_t* filler_h, uint64_t* T_h, uint64_t* F_h, int32_t* depth_out, void* workspace,
                  uint64_t workspace_bytes, const gt_keys* keys, gt_allreduce_fn allreduce, void* allreduce_user,
                  void* stream);

/* Host staging for the drop-in rendezvous (replaces the reference's per-party
 * share handling, rss.py:222-228 consistency): lo[i] / hi[i] are party i+1's
 * share pair (n words each); component i = lo[i] is written to out + i*n
 * (pinned staging of gt_train_host); check != 0 requires hi[i] == lo[(i+1)%3].
 * out == NULL: the check alone (the drop-in runs it while the device trains).
 * Host threads; no device work.  GT_ERR_INVALID on an inconsistent pair. */
int gt_stage_pairs(const uint64_t* const* lo, const uint64_t* const* hi, uint64_t n, uint64_t* out, int check);

/* Device loading of dealt share files / material banks (reference
 * rss.py:452-481 OBS1, dealer.py:131-176 OBD1): lo[i] / hi[i] are DEVICE
 * pointers to party i+1's little-endian ring words (word_bytes 1/4/8, stride
 * bytes apart: 2 words for OBS1's interleaved pairs); component i of out
 * [3][n] (u64) = party i+1's lo words; if mismatches != NULL (device counter)
 * every hi[i] word is compared with lo[(i+1)%3] and differences counted. */
int gt_unpack_pairs(const void* const* lo, const void* const* hi, uint32_t stride_bytes, uint32_t word_bytes,
                    uint64_t n, uint64_t* out, unsigned long long* mismatches, void* stream);

/* ---- three-host deployment: party-local steps (transport.py:374-475) ----
 * One party (1..3) holds one replicated pair per shared vector, pair arrays
 * [2][L] = (lo, hi) = (c_{p-1}, c_p); the host exchanges the ring messages
 * between these calls (party.py).  keys: the party's two pairwise keys in
 * pair[p-1] (shared with next) and pair[(p+1)%3] (shared with prev); the
 * other slots are ignored.  Material pairs come from the party's dealt bank. */
int gt_party_eq_mask(int party, const uint64_t* idx, uint64_t nq, uint64_t m, uint64_t off, const uint64_t* r,
                     uint64_t* out, void* stream);
int gt_party_eq_planes(int party, const uint64_t* masked, const uint64_t* recv, const uint64_t* rbits, uint64_t L,
                       uint64_t* planes, void* stream);
int gt_party_and_half(int party, const uint64_t* planes, uint64_t L, int width, const gt_keys* keys, uint32_t op,
                      uint32_t sub, uint64_t lane0, uint64_t* z, void* stream);
int gt_party_pack(const uint64_t* src, uint64_t L, int bits, uint8_t* out, void* stream);
int gt_party_unpack(const uint8_t* in, uint64_t L, int bits, uint64_t* dst, void* stream);
int gt_party_b2a_mask(const uint64_t* h, const uint8_t* bb, uint64_t L, uint64_t* e, void* stream);
int gt_party_b2a_finish(int party, const uint64_t* e, const uint64_t* recv, const uint64_t* a, uint64_t L,
                        uint64_t* out, void* stream);
int gt_party_select_mul(int party, const uint64_t* ca, const uint64_t* table, uint64_t table_len, int per_row,
                        uint64_t nq, uint64_t m, const gt_keys* keys, uint32_t op, uint32_t sub, uint64_t lane0,
                        uint64_t* z, void* stream);
int gt_party_lane_sum(const uint64_t* pair, uint64_t nq, uint64_t m, uint64_t* out, void* stream);
int gt_party_slot_step(int party, uint64_t* slot, const uint64_t* branch, uint64_t nq, void* stream);

/* ---- secure inference (infer_batch, infer.py:20-35) ---- */

/* tree [3][2^depth-1] heap-ordered payload shares, queries [3][n][nf];
 * instance_base = global index of query 0 (instance sharding); out [3][n]
 * predicted labels; slot_out [3][n] final heap slot (nullable). */
int gt_infer(int depth, const uint64_t* tree, const uint64_t* queries, uint64_t n, uint64_t nf,
             uint64_t instance_base, uint64_t* out, uint64_t* slot_out, const gt_keys* keys, void* stream);

/* ---- diagnostics ---- */

/* Peak counter-based PRG rate: `grid` x 256 threads each draw `iters`
 * Philox4x32-10 blocks (distinct counters) and fold them into out[grid*256].
 * The caller times it; blocks/s is the integer-ALU roof of the share kernels,
 * whose correlated randomness is drawn the same way. */
int gt_diag_philox(uint32_t grid, uint32_t iters, uint64_t* out, void* stream);
/* diagnostics: per-level heuristic phase timestamps (%globaltimer, ns) of the
   last training run made with GT_HC_TIMING=1 (n <= 128): slots 8*level +
   phase for the scores / argmin / budget / split phases and the division's
   ladder end (phase 7), 64 + 8*level + phase for the prologue and the
   division (tools/hc_timing.py). */
int gt_diag_hc_timestamps(unsigned long long* out, int n);
/* diagnostics: phase timestamps (ns, globaltimer) of the fused count's first
 * cluster per level, 8 slots per level, filled when GT_COUNT_TS is set */
int gt_diag_count_timestamps(unsigned long long* out, int n);

#ifdef __cplusplus
}
#endif

#endif /* GTREE_B200_H */
