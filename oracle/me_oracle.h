/*
 * me_oracle.h -- plain, slow CPU oracle for the memory estimator of
 * Fujii, Watanabe, Yokota, "Accelerating Large Language Model Training with 4D
 * Parallelism and Memory Consumption Estimator" (arXiv 2411.06465).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load, call or link this
 * code.  The product (paper_2411_06465_b200/, libme.so) shares no code, header,
 * table or constant with it and never calls it.
 *
 * Citations: P:n = PAPER.md line n (LaTeX source order), Eq.k = k-th numbered
 * equation in source order.  Readings R1..R26 are listed in DESIGN.md §3.
 *
 * Every function evaluates the printed equations as exact rationals
 * (__int128 numerator/denominator, reduced by gcd after every step) and only
 * converts to an integer at the end, checking that the value is integral.
 * The one non-integral step the paper leaves open, the optimizer shard when
 * (d*c) does not divide the stage parameter count, uses reading R8
 * (12 * ceil(Psi_s / (d*c))).
 */
#ifndef ME_ORACLE_H
#define ME_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (same numeric meaning as the product ABI, defined independently) */
#define OR_OK 0
#define OR_EINVAL 1    /* zero field, k does not divide a, a does not divide h */
#define OR_EDIV 2      /* estimator precondition (R10, c|s, p<=L, p|L, gbs) */
#define OR_EOVERFLOW 3 /* a term >= 2^63, or a rational overflowed 127 bits */
#define OR_ENOMEM 4
#define OR_ERANGE 7    /* caller buffer too small */

/* Table "Variable names": h, h_ffn, L, a, k, v. */
typedef struct {
    uint32_t h, f, L, a, k, v;
} or_model;

/* One training configuration: Table "Variable names" t, c, p, d, b, s plus the
 * builder extensions: gbs (R17), L0 (R19), rc (R20), dopt (R21). */
typedef struct {
    uint32_t d, t, p, c, b, s;
    uint32_t gbs;     /* 0 = paper mode: p microbatches in flight (Eq.16) */
    uint32_t L0;      /* 0 = auto (L if p=1, L/p if p|L, ceil(L/p) if uneven) */
    uint8_t rc;       /* 1 = full recompute (R20, not in the paper) */
    uint8_t dopt;     /* 1 = distributed optimizer (Eq.5/10), 0 = Eq.4 */
    uint8_t uneven;   /* 1 = allow p not dividing L (R19) */
    uint8_t zero;     /* NEXT-4 (extension): with dopt, 0/1 = optimizer states
                         sharded over d*c (the paper, ZeRO stage 1); 2 = also the
                         FP32 gradients; 3 = also the BF16 weights (ZeRO-2/3) */
    /* NEXT-4 variants (extensions, DESIGN.md §3 R28-R30); 0 = the paper */
    uint8_t sp_off;   /* 1 = sequence parallelism off (the FFN input
                         and the RMSNorms are then not parallelized) */
    uint8_t vpp;      /* virtual pipeline stages per GPU (interleaved 1F1B);
                         0 or 1 = the paper's non-interleaved 1F1B */
    uint8_t wb, gb, ob; /* bytes per parameter of weights, gradients and
                         optimizer states (ledger P:192-199: 2, 4, 12; 0 =
                         that default), e.g. FP8 weights wb = 1 */
} or_cfg;

/* Eq.18 split into the ledger of P:192-199 and the three activation groups. */
typedef struct {
    uint64_t params, grads, optim, act_layers, act_embed, act_head, total;
} or_breakdown;

/* enumerated configuration space (canonical order: DESIGN.md §4) */
typedef struct {
    const or_model* models; uint32_t n_models;
    const uint32_t* world; uint32_t n_world;
    const uint64_t* cap_bytes; uint32_t n_caps;  /* <= 8 */
    uint32_t gpus_per_node;                      /* 0 = no t <= node filter */
    const uint32_t* mbs; uint32_t n_mbs;
    const uint32_t* seq; uint32_t n_seq;
    uint8_t rc_mask, do_mask, uneven, stage_max; /* masks: bit0 = off, bit1 = on;
                                                    stage_max: 1 = largest pipeline stage (NEXT-1) */
    uint32_t gbs, max_t, max_c, max_p;           /* 0 = unlimited */
    uint32_t thr_num, thr_den;                   /* feasible <=> total*den <= cap*num */
    uint32_t zero_stage;                         /* or_cfg.zero of every configuration */
    uint8_t sp_off, vpp, wb, gb, ob, _pad[3];    /* or_cfg's NEXT-4 fields of every configuration */
} or_space;

/* Eq.1, Eq.2, Eq.3 */
int or_attention_params(const or_model* m, uint64_t* out);
int or_ffn_params(const or_model* m, uint64_t* out);
int or_total_params(const or_model* m, uint64_t* out);
/* Eq.6 (p=1) / Eq.7 (p>1) with L/p replaced by the first-stage layer count L0 */
int or_stage0_params(const or_model* m, uint32_t t, uint32_t p, uint32_t L0, uint64_t* out);
/* Eq.12: one layer's activation bytes with no parallelism */
int or_activation_per_layer(const or_model* m, uint32_t s, uint32_t b, uint64_t* out);
/* first-stage layer count L0 (R19); 0 on error */
uint32_t or_first_stage_layers(const or_model* m, const or_cfg* c);
/* Eq.18 + extensions: the six stage-0 terms and their sum */
int or_estimate(const or_model* m, const or_cfg* c, or_breakdown* out);
/* NEXT-1: layers of pipeline stage i, the six terms of stage i (Eq.6-9 with
 * the stage's 1F1B occupancy min(m, p - i)), and the largest stage total */
uint32_t or_stage_layers(const or_model* m, const or_cfg* c, uint32_t i);
int or_estimate_stage(const or_model* m, const or_cfg* c, uint32_t i, or_breakdown* out);
int or_estimate_max(const or_model* m, const or_cfg* c, or_breakdown* out, uint32_t* stage);
/* capacity bitmask: bit j set <=> total * den <= cap_j * num (80% rule) */
uint32_t or_cap_mask(uint64_t total, const uint64_t* cap_bytes, uint32_t n_caps,
                     uint32_t num, uint32_t den);

/* canonical enumeration */
int or_space_size(const or_space* sp, uint64_t* n);
int or_decode(const or_space* sp, uint64_t index, uint32_t* model_id, uint32_t* world,
              or_cfg* cfg);
/* Evaluate every config with index in [begin, end) (end = 0: whole space).
 * Survivors (cap mask != 0) are written in ascending index order to
 * idx_mask[i] = index | mask << 56 and rows[i] (either may be NULL = count
 * only) up to `cap` entries; *count gets the number of survivors, cap_counts
 * (n_caps entries, may be NULL) the number per capacity.  n_threads >= 1.
 * Returns OR_ERANGE (and still the counts) if cap was too small. */
int or_sweep(const or_space* sp, uint64_t begin, uint64_t end, uint64_t* idx_mask,
             or_breakdown* rows, uint64_t cap, uint64_t* count, uint64_t* cap_counts,
             int n_threads);

/* Evaluate the configurations at the given strictly ascending indices (one
 * walk): rows[k] and masks[k] (either may be NULL) for points[k]. */
int or_points(const or_space* sp, const uint64_t* points, uint64_t n, or_breakdown* rows,
              uint32_t* masks);

/* Whole-chunk verification (test infrastructure): [begin, end) (end = 0: the
 * whole space) cut into chunks of `chunk` indices; per chunk c the
 * OR_DIGEST_WORDS words out[c*11 ..]: survivor count, 8 per-capacity counts,
 * the index digest and the record digest of the chunk's survivors in
 * ascending index order, position j = 0, 1, ... within the chunk:
 *   D = sum_j g(r_j) * M^j mod 2^64,  M = 0xD1B54A32D192ED03,
 *   g_index(r)  = mix(r_0 + C),
 *   g_record(r) = h <- C; for k = 0..7: h <- mix(h ^ r_k); h
 * with r = (index | mask << 56, params, grads, optim, act_layers, act_embed,
 * act_head, total), C = 0x9E3779B97F4A7C15 and mix the splitmix64
 * finaliser.  The hash is a verification device, not part of the method. */
#define OR_DIGEST_WORDS 11
int or_digest(const or_space* sp, uint64_t begin, uint64_t end, uint64_t chunk, int n_threads,
              uint64_t* out);

#ifdef __cplusplus
}
#endif
#endif
