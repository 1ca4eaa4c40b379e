/*
 * me.h -- C ABI of libme.so: batched, exact-integer evaluation of the per-GPU
 * memory estimator of Fujii, Watanabe, Yokota, "Accelerating Large Language
 * Model Training with 4D Parallelism and Memory Consumption Estimator"
 * (arXiv 2411.06465) on NVIDIA B200 (sm_100a), with the paper's 80%-of-HBM
 * feasibility filter and order-preserving compaction of the survivors.
 *
 * Citations: P:n = line n of the paper's LaTeX source; Eq.k is the
 * k-th numbered equation in source order; R1..R26 are the readings of the
 * paper listed in DESIGN.md §3.
 *
 * Conventions for every call
 *  - Every call returns an int status (ME_OK = 0); out-parameters are left
 *    untouched on error.  No C++ exception crosses this boundary.
 *  - Inputs are borrowed for the duration of the call (the library copies what
 *    it keeps).  Plans and results are owned by the library until their _free
 *    call; their device memory comes from the caller's allocator callback when
 *    one is given, else from cudaMallocAsync.
 *  - All arithmetic on the device is unsigned 64-bit integer; there is no
 *    floating point and no CPU fallback: without a usable CUDA device the
 *    compute calls return ME_ECUDA.
 *  - Calls are thread-safe on distinct plan / result / comm handles.  Sweeps of
 *    one plan reuse its scratch memory and must be issued on one stream.
 *  - me_last_error_detail() returns a thread-local human-readable message for
 *    the last failing call on the calling thread.
 */
#ifndef ME_H
#define ME_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ME_OK = 0,
    ME_EINVAL = 1,    /* NULL pointer, zero field, k not dividing a, a not dividing h,
                         bad mask or threshold, more than 8 capacities, input
                         outside the exact-u64 domain of the sweep (me_plan_create) */
    ME_EDIV = 2,      /* estimator precondition (R10, Eq.17, R17, R19):
                         t must divide k, v and h_ffn; c must divide s; p <= L;
                         p | L unless allow_uneven_pp; (d*b) | gbs when gbs > 0 */
    ME_EOVERFLOW = 3, /* a term would reach 2^63, or a flat index 2^56 */
    ME_ENOMEM = 4,
    ME_ECUDA = 5,     /* no device, launch or runtime failure */
    ME_ENCCL = 6,
    ME_ERANGE = 7     /* caller buffer too small, or index past the end */
};

/* Model shape, Table "Variable names": h, h_ffn, L, a, k, v.
 * Requires all fields > 0, k | a (GQA groups), a | h. */
typedef struct {
    uint32_t hidden, ffn_hidden, layers, heads, kv_heads, vocab;
} me_model;

/* One training configuration.  dp, tp, pp, cp = d, t, p, c; mbs = b; seq = s.
 *  gbs                 0 = paper mode: p microbatches in flight on stage 0
 *                      (Eq.16); >0 = min(p, gbs/(d*b)) in flight (R17)
 *  first_stage_layers  0 = auto: L if p = 1, L/p if p | L, ceil(L/p) if uneven
 *                      splits are allowed (R19); else explicit, 1..L-(p-1)
 *                      (= L when p = 1)
 *  recompute           1 = full activation recompute (R20, extension)
 *  dist_opt            1 = distributed optimizer, 12 B/param sharded over d*c
 *                      (Eq.5, Eq.10; ceil rule R8); 0 = Eq.4 (18 B/param)
 *  zero_stage          see the field (ME_EINVAL above 3) */
typedef struct {
    uint32_t dp, tp, pp, cp, mbs, seq;
    uint32_t gbs;
    uint32_t first_stage_layers;
    uint8_t recompute, dist_opt, allow_uneven_pp;
    uint8_t zero_stage; /* NEXT-4, with dist_opt: 0/1 = optimizer states sharded
                           over d*c (the paper); 2 = also the FP32 gradients;
                           3 = also the BF16 weights (ZeRO-2/3, extension) */
    /* NEXT-4 variants (extensions; 0 = the paper), DESIGN.md §3:
     *  sp_off   1 = sequence parallelism off (R28: the attention and
     *           FFN inputs and the RMSNorm inputs stay whole on every TP rank)
     *  vpp      virtual pipeline stages per GPU: interleaved 1F1B with vpp
     *           model chunks of L/(p vpp) layers (R29; needs p >= 2, p vpp | L,
     *           no uneven split, with gbs a microbatch count divisible by p);
     *           0 or 1 = the paper's 1F1B
     *  w_bytes, g_bytes, o_bytes  bytes per parameter of weights, gradients,
     *           optimizer states (R30; 0 = 2, 4, 12 of the ledger P:192-199),
     *           e.g. FP8 weights w_bytes = 1; at most 8, 8, 16 */
    uint8_t sp_off, vpp, w_bytes, g_bytes, o_bytes, _pad0, _pad1, _pad2;
} me_parallel;

/* Stage-0 per-GPU bytes (Eq.18 split by the ledger of P:192-199):
 * params = 2 Psi_s (BF16), grads = 4 Psi_s (FP32, not sharded, R9),
 * optim = 12 ceil(Psi_s/(d c)) or 12 Psi_s, act_layers / act_embed / act_head
 * = the three groups of Eq.17, total = their sum. */
typedef struct {
    uint64_t params, grads, optim, act_layers, act_embed, act_head, total;
} me_breakdown;

/* feasible for capacity j <=> total <= floor(cap_j * num / den); the paper's
 * rule is num/den = 4/5 ("at or below 80%": a total equal
 * to the threshold is feasible).  1 <= num, den <= 1024.  Thresholds are
 * computed exactly in 128 bits and clamped to 2^63 (every total is below 2^63,
 * so the clamp never changes a verdict). */
typedef struct {
    uint32_t num, den;
} me_threshold;

typedef struct {
    const me_model* models;
    uint32_t n_models;
} me_model_range;

/* world_sizes: the N axis, in enumeration order.  capacity_bytes: up to 8 HBM
 * capacities in bytes (the paper's "40GB"/"94GB" are GiB, R2: pass GB * 2^30).
 * gpus_per_node > 0 keeps only t <= gpus_per_node. */
typedef struct {
    const uint32_t* world_sizes;
    uint32_t n_world;
    const uint64_t* capacity_bytes;
    uint32_t n_cap;
    uint32_t gpus_per_node;
} me_cluster;

/* The remaining axes.  recompute_mask / dist_opt_mask: bit0 = off, bit1 = on
 * (each must be 1, 2 or 3).  max_tp/max_cp/max_pp: 0 = unlimited.
 * stage_policy: ME_STAGE_FIRST (0) = the paper's first-stage estimate;
 * ME_STAGE_MAX (1) = the largest stage total (NEXT-1: Eq.7/8/9 per stage with
 * the stage's 1F1B occupancy; the record then holds that stage's terms). */
typedef struct {
    const uint32_t* mbs;
    uint32_t n_mbs;
    const uint32_t* seq;
    uint32_t n_seq;
    uint8_t recompute_mask, dist_opt_mask, allow_uneven_pp, stage_policy;
    uint32_t gbs, max_tp, max_cp, max_pp;
    uint32_t zero_stage; /* me_parallel.zero_stage of every configuration (0..3) */
    /* me_parallel.sp_off, vpp, w_bytes, g_bytes, o_bytes of every configuration;
     * vpp >= 2 drops the tuples with p = 1 or p vpp not dividing L (and with a
     * global batch the (b, s) pairs whose microbatch count p does not divide)
     * and excludes allow_uneven_pp and ME_STAGE_MAX (ME_EINVAL) */
    uint8_t sp_off, vpp, w_bytes, g_bytes, o_bytes, _pad0, _pad1, _pad2;
} me_cfg_range;

/* Output modes of a sweep:
 *  COUNT    survivor counts only (total and per capacity)
 *  INDEX    one u64 column: flat index | (capacity mask << 56)
 *  FULL     eight u64 columns (structure of arrays): index|mask, params, grads,
 *           optim, act_layers, act_embed, act_head, total
 *  RECORDS  the same eight values per survivor as one 64-byte me_record row
 *           (array of structures): column 0 only, 8 u64 words per row.  The
 *           fastest FULL-content mode (one contiguous run of whole records per
 *           warp round instead of eight short column runs). */
typedef enum { ME_OUT_COUNT = 0, ME_OUT_INDEX = 1, ME_OUT_FULL = 2, ME_OUT_RECORDS = 3 } me_out_mode;

typedef struct {
    uint64_t index_mask; /* flat index | (capacity mask << 56) */
    uint64_t params, grads, optim, act_layers, act_embed, act_head, total;
} me_record;

enum { ME_STAGE_FIRST = 0, ME_STAGE_MAX = 1 };
#define ME_STAGE_ARGMAX 0xFFFFFFFFu

#define ME_N_COLS 8

/* Allocator callbacks (e.g. PyTorch's caching allocator).  Device memory of
 * `bytes` bytes usable on `stream`; free receives the same stream. */
typedef void* (*me_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*me_free_fn)(void* p, void* stream, void* ctx);

typedef struct me_comm me_comm;
typedef struct me_plan me_plan;
typedef struct me_result me_result;

/* Multi-GPU partition of a sweep (north star (3)):
 *  ME_PART_EVEN    with comm, [begin, end) is split into nranks contiguous
 *                  equal parts, this rank sweeps its own, and the call joins
 *                  them (NCCL allgather of the counts: global offsets)
 *  ME_PART_CYCLIC  this call is one block of a cyclic deal (me_cyclic_block):
 *                  [begin, end) is swept by this rank alone with no
 *                  collective; the blocks of a job are joined afterwards by
 *                  one me_result_join (one allgather for all of them) */
typedef enum { ME_PART_EVEN = 0, ME_PART_CYCLIC = 1 } me_sweep_partition;

typedef struct {
    uint64_t begin, end;   /* flat index range; end = 0 -> end of the space.
                              With comm and ME_PART_EVEN, [begin, end) is split
                              into nranks contiguous equal parts and this rank
                              does its own. */
    me_out_mode mode;
    int device;            /* CUDA device ordinal (me_sweep only; a plan keeps its own) */
    void* stream;          /* cudaStream_t; NULL = the legacy default stream */
    me_alloc_fn alloc;     /* NULL -> cudaMallocAsync / cudaFreeAsync (me_sweep only) */
    me_free_fn free;
    void* alloc_ctx;
    me_comm* comm;         /* NULL = single GPU */
    uint32_t gather;       /* with comm: 1 = every rank receives all ranks'
                              columns in global order (NCCL broadcasts over NVLink) */
    uint32_t _pad;
    /* Optional caller-owned output columns: device pointers, ME_N_COLS of
     * them for FULL, 1 for INDEX, 1 for RECORDS (out_capacity rows of 64 B,
     * 8-byte aligned; 32-byte alignment gives whole-sector stores)
     * (NULL = the library allocates exactly, which
     * synchronises the host once).  With caller columns the call is fully
     * asynchronous: survivors beyond out_capacity are counted but not written
     * and me_result_status() then returns ME_ERANGE. */
    uint64_t* const* out_cols;
    uint64_t out_capacity;
    me_sweep_partition partition; /* ME_PART_EVEN (default) or ME_PART_CYCLIC */
    uint32_t _pad2;
} me_sweep_opts;

/* me_estimate: Eq.18 and its parts for one configuration, evaluated by the same
 * device code as the sweep (one GPU thread; synchronous).  Checks EINVAL then
 * EDIV then EOVERFLOW as listed above.  Uses the current CUDA device. */
int me_estimate(const me_model* model, const me_parallel* cfg, me_breakdown* out);

/* me_estimate_stage: the six terms of pipeline stage `stage` (0 .. p-1) of one
 * configuration (NEXT-1, extension of the paper's first-stage estimate: Eq.6
 * for p = 1, Eq.7 first, Eq.8 middle, Eq.9 last stage with the final norm and
 * the LM head; stage i holds min(m, p - i) in-flight microbatches, m =
 * gbs/(d b) or unbounded when gbs = 0; the embedding input lives on stage 0).
 * stage = ME_STAGE_ARGMAX returns the stage with the largest total (the first
 * such stage) and stores its index in *which (may be NULL).  Stage 0 equals
 * me_estimate.  Layers: stage 0 holds L0 (see me_parallel), the other stages
 * split L - L0 as evenly as possible, earlier stages first.  ME_EINVAL for
 * stage >= p and for interleaved 1F1B (vpp >= 2: no per-stage view). */
int me_estimate_stage(const me_model* model, const me_parallel* cfg, uint32_t stage, me_breakdown* out,
                      uint32_t* which);

/* me_estimate_batch: n configurations, cfgs[i] against models[model_ids[i]]
 * (model_ids may be NULL: model 0).  Every array may be host or device memory
 * (detected per pointer).  out (n rows), cap_mask (n bytes: bit j = feasible for
 * capacity j) and status (n bytes: per-config ME_* code) may each be NULL.
 * Synchronous.  Returns ME_OK, or the first per-config failure when status is
 * NULL. */
int me_estimate_batch(const me_model* models, uint32_t n_models, const uint32_t* model_ids,
                      const me_parallel* cfgs, uint64_t n, const uint64_t* capacity_bytes,
                      uint32_t n_cap, me_threshold thr, me_breakdown* out, uint8_t* cap_mask,
                      uint8_t* status, void* stream);

/* Number of valid configurations of the space (the canonical enumeration of
 * model -> N -> t, c, p ascending with t*c*p | N -> b -> s -> rc
 * -> do; invalid tuples consume no index).  Host-only. */
int me_space_size(const me_model_range* models, const me_cluster* cluster,
                  const me_cfg_range* cfg, uint64_t* n);

/* Configuration at a flat index (host-only).  ME_ERANGE past the end. */
int me_decode(const me_model_range* models, const me_cluster* cluster, const me_cfg_range* cfg,
              uint64_t index, uint32_t* model_id, uint32_t* world_size, me_parallel* out);

/* A plan = the space's enumeration tables resident on one device (built on the
 * host, uploaded once) plus reusable scratch.  Domain of exact u64 evaluation
 * (ME_EINVAL outside it): h <= 2^15, h_ffn <= 2^17, L <= 2^8, v <= 2^19,
 * s <= 2^20, b <= 2^6, N <= 2^20 and < 2^56 configurations; then every term
 * is < 2^58 (with the NEXT-4 variants too: at most 32 bytes per parameter,
 * and interleaving keeps the first GPU's layer-microbatches below 2L). */
int me_plan_create(const me_model_range* models, const me_cluster* cluster,
                   const me_cfg_range* cfg, me_threshold thr, int device, void* stream,
                   me_alloc_fn alloc, me_free_fn free, void* alloc_ctx, me_plan** out);
int me_plan_size(const me_plan* plan, uint64_t* n);
/* bytes of enumeration tables the plan uploaded to the device (H2D) */
int me_plan_table_bytes(const me_plan* plan, uint64_t* bytes);
/* evaluate every configuration of opts->[begin, end), keep those whose
 * capacity mask is non-zero, in ascending index order (the feasible set of
 * the 80% rule) */
int me_plan_sweep(me_plan* plan, const me_sweep_opts* opts, me_result** out);
void me_plan_free(me_plan* plan);

/* one-shot: me_plan_create + me_plan_sweep (+ free of the plan's tables) */
int me_sweep(const me_model_range* models, const me_cluster* cluster, const me_cfg_range* cfg,
             me_threshold thr, const me_sweep_opts* opts, me_result** out);

/* Survivors: this rank's (local) and all ranks' (global) counts; without comm
 * they are equal.  rank_offset = global position of this rank's first row.
 * Waits for the sweep to finish. */
int me_result_counts(me_result* r, uint64_t* local, uint64_t* global, uint64_t* rank_offset);
/* per-capacity survivor counts (n_cap entries), global when comm is set */
int me_result_cap_counts(me_result* r, uint64_t* per_cap);
/* device pointers of the output columns (NULL entries for COUNT mode / unused
 * columns; RECORDS: cols[0] = the me_record array).  With comm+gather these are the gathered global columns, else this
 * rank's.  n_rows = rows visible in those columns. */
int me_result_columns(me_result* r, uint64_t** cols /* ME_N_COLS */, uint64_t* n_rows);
/* copy rows [first, first+n) of the visible columns to host arrays; cols_host[j]
 * receives column j and may be NULL (RECORDS: cols_host[0] receives n records).  ME_ERANGE if out of bounds. */
int me_result_copy_to_host(me_result* r, uint64_t first, uint64_t n, uint64_t* const* cols_host);
/* ME_OK, or ME_ERANGE when caller columns overflowed.  Waits. */
int me_result_status(me_result* r);
/* wait for the result's work on its stream to finish */
int me_result_wait(me_result* r);
/* device time in ms from CUDA events: [0] whole sweep, [1] K0 rows + counts
 * (plan stream; COUNT mode: the caller's stream), [2] scan (~0 in COUNT mode:
 * K0 sums the counts itself), [3] K3 output kernel (0 when not run), summed
 * over the sub-ranges.  Waits. */
int me_result_timing(me_result* r, float* ms4);
void me_result_free(me_result* r);

/* Order-dependent digest of a result's rows, for verifying a whole result (or
 * a sharded one) against an independent enumeration without moving its rows.
 * Not part of the method.  For the row at position j (0-based, in the result's
 * ascending index order) with values r = (index|mask, params, grads, optim,
 * act_layers, act_embed, act_head, total):
 *   digest[0] = sum_j mix(r_0 + C) * M^j                       (mod 2^64)
 *   digest[1] = sum_j g(r) * M^j,  g: h <- C; h <- mix(h ^ r_k), k = 0..7
 * mix = the splitmix64 finaliser (x ^= x >> 30; x *= 0xBF58476D1CE4E5B9;
 * x ^= x >> 27; x *= 0x94D049BB133111EB; x ^= x >> 31), C = 0x9E3779B97F4A7C15,
 * M = 0xD1B54A32D192ED03.  digest[1] = 0 for INDEX results.  A comm result
 * without gather: COLLECTIVE (every rank calls it), the digest of the global
 * result (rank shards merged in rank order: D = sum_r M^offset_r D_r).
 * ME_EINVAL for COUNT results, ME_ERANGE if caller columns overflowed.
 * Synchronous. */
int me_result_digest(me_result* r, uint64_t digest[2]);
/* The digest of consecutive pieces of a result from the pieces' digests:
 * piece i has counts[i] rows and digests[2i], digests[2i+1] (index, record);
 * out = sum_i M^(rows before piece i) D_i.  Host-only. */
int me_digest_merge(uint64_t n, const uint64_t* counts, const uint64_t* digests, uint64_t out[2]);

/* NEXT-2 planner (the search heuristics of
 * P:552-593).  For every (model, N) segment of the plan (n_models * n_world
 * entries, model-major), the k best rows of an INDEX, FULL or RECORDS result
 * by the survey's rank key, smallest first:
 *   1. class green < yellow < red (caption P:420: total <= 80% of the
 *      capacity, <= 100%, above): green = bit green_cap of the row's capacity
 *      mask; yellow = not green but bit yellow_cap (e.g. a second capacity
 *      5C/4 under the 4/5 rule, = C at 100%; ME_RANK_NONE: no yellow class);
 *      red = neither (such rows are in a result only through a third
 *      capacity, e.g. UINT64_MAX bytes, which admits every configuration);
 *   2. t <= gpus_per_node first (0 = no node bound);
 *   3. smallest t*c*p; 4. largest mbs;
 *   5. smallest p (pipeline bubble (p-1)/m); 6. smallest c;
 *   7. smallest t; then recompute off first, then the smallest index.
 * out: host array of n_seg * k rows, segment-major; a segment with fewer
 * than k result rows has index = UINT64_MAX in the rest.  Each row carries its
 * decoded configuration and the 1F1B schedule statistics:
 * microbatches m = gbs/(d*b) (0 when gbs = 0: the paper mode has no global
 * batch) and the bubble fraction (p-1)/m as bubble_num / bubble_den.  A
 * sharded comm result (ME_PART_EVEN without gather): COLLECTIVE -- every rank
 * ranks its own rows, the candidates are allgathered (NCCL) and merged per
 * segment, and every rank receives the global top k.  Synchronous; scratch
 * from the result's allocator. */
#define ME_RANK_NONE 0xFFFFFFFFu
typedef struct {
    uint32_t green_cap, yellow_cap; /* capacity slots (yellow_cap may be ME_RANK_NONE) */
    uint32_t gpus_per_node;         /* 0 = no TP <= node preference */
    uint32_t k;                     /* rows per segment, >= 1 */
} me_rank_opts;
typedef struct {
    uint64_t index;                 /* flat index, UINT64_MAX = no row */
    uint64_t key;                   /* packed rank key (smaller is better) */
    uint32_t model_id, world_size;
    me_parallel cfg;
    uint32_t cls;                   /* 0 green, 1 yellow, 2 red */
    uint32_t microbatches;          /* m = gbs/(d*b); 0 in paper mode (gbs = 0) */
    uint32_t bubble_num, bubble_den; /* (p - 1) / m; 0/0 in paper mode */
    uint32_t _pad;
} me_rank_row;
int me_result_rank(me_result* r, const me_rank_opts* opts, me_rank_row* out);

/* Host logic of the multi-GPU path (host-only, no device needed).
 * me_partition: rank's contiguous share [lo, hi) of [begin, end) with
 * lo = begin + floor(len*rank/nranks), hi likewise for rank + 1.
 * me_join_counts: from every rank's stats row (stride u64 per rank: survivor
 * count then n_cap per-capacity counts, as allgathered by a comm sweep)
 * compute this rank's global row offset, the global count and the global
 * per-capacity counts (cap_global may be NULL). */
int me_partition(uint64_t begin, uint64_t end, int rank, int nranks, uint64_t* lo, uint64_t* hi);
int me_join_counts(const uint64_t* stats, int nranks, uint32_t stride, uint32_t n_cap, int rank,
                   uint64_t* offset, uint64_t* global, uint64_t* cap_global);

/* Cyclic partition (a8): [begin, end) cut into n_blocks blocks of `block`
 * indices (the last may be shorter); block q belongs to rank q mod nranks.
 * me_cyclic_block: this rank's k-th block [lo, hi) (block q = k*nranks + rank)
 * and the number of blocks; ME_ERANGE when the rank has no k-th block.
 * Host-only.  Dealing whole blocks round-robin evens out the survivor density
 * of neighbouring blocks, and no rank waits for another until the join. */
int me_cyclic_block(uint64_t begin, uint64_t end, uint64_t block, int rank, int nranks, uint64_t k, uint64_t* lo,
                    uint64_t* hi, uint64_t* n_blocks);
/* The deferred join of a cyclic partition: results[k] must be the ME_PART_CYCLIC
 * sweep of this rank's k-th block (all of this rank's blocks, one plan and
 * stream).  COLLECTIVE over comm: one ncclAllGather of every block's counts,
 * then an exclusive scan over the blocks in global order on the device.
 * Asynchronous on the results' stream.  Afterwards me_result_counts gives for
 * each result its local count, the job's global count, and the global position
 * of its first row (rank_offset); me_result_cap_counts the job's per-capacity
 * counts.  The results keep the join alive.  A rank with no block (more ranks
 * than blocks) calls it with n = 0 and only takes part in the allgather. */
int me_result_join(me_result* const* results, uint32_t n, uint64_t n_blocks, me_comm* comm);

/* NCCL communicator over nranks processes (one per GPU).  rank 0 creates the
 * unique id with me_comm_unique_id and the caller distributes it (e.g. with
 * torch.distributed); every rank then calls me_comm_init collectively. */
int me_comm_unique_id(uint8_t id[128]);
int me_comm_init(const uint8_t id[128], int rank, int nranks, int device, me_comm** out);
int me_comm_rank(const me_comm* c, int* rank, int* nranks);
void me_comm_destroy(me_comm* c);
/* ME_ENCCL when the communicator recorded an asynchronous error
 * (ncclCommGetAsyncError), else ME_OK. */
int me_comm_check(me_comm* c);

const char* me_strerror(int status);
const char* me_last_error_detail(void);
/* library version string */
const char* me_version(void);

#ifdef __cplusplus
}
#endif
#endif /* ME_H */
