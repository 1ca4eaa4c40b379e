// me_kernels.cuh -- device code of the estimator sweep (sm_100a).
//
// One pass of the hot path = decode flat index -> evaluate the six stage-0
// byte terms of Eq.18 in exact u64 -> compare with floor(0.8 * capacity) ->
// compact the survivors in index order.  Integer-only: no tensor cores, no FP.
#pragma once
#include <cstdint>

#include "../../include/me.h"
#include "me_space.hpp"

namespace me {

// Device copy of a model shape with the head dimension h/a precomputed (32 B).
struct DevModel {
    uint32_t hidden, ffn_hidden, layers, heads, kv_heads, vocab, head_dim, _pad;
};

__host__ __device__ inline DevModel dev_model(const me_model& m) {
    return DevModel{m.hidden, m.ffn_hidden, m.layers, m.heads, m.kv_heads, m.vocab,
                    m.heads ? m.hidden / m.heads : 0u, 0u};
}

// Table pointers handed to the kernels (all device memory, read-only).
struct DevSpace {
    const DevModel* models;
    const uint32_t* model_class;
    const uint64_t* seg_prefix;   // n_seg + 1
    const uint64_t* seg_row;      // n_seg + 1: rows before each segment
    const uint32_t* list_off;     // n_class * n_world + 1
    const uint32_t* list_tuple;
    const uint64_t* list_prefix;
    const DevTuple* tuples;
    const DevPair* pairs;
    const uint32_t* pair_b;       // micro-batch size of each pair (planner only)
    const uint32_t* pair_su;      // per pair list: its u values sorted ascending (row-count pipeline)
    const uint32_t* pair_fence;   // per pool: 4 + 16 fences over pair_su (DevTuple::fence_off)
    uint32_t n_fence;             // entries of pair_fence
    uint32_t fenced;              // K0 searches through the fences (every pool <= 128 pairs; ME_K0_FENCE)
    uint32_t n_seg, n_world;
    uint32_t n_pairs;             // pooled (b, s) pairs
    uint32_t lg_rcdo, rcdo_rc, rcdo_do;
    uint32_t n_cap;
    uint32_t gbs_mode;            // 1 = a global batch bounds the in-flight microbatches (R17)
    uint32_t stage_max;           // 1 = feasibility of the largest pipeline stage (NEXT-1)
    uint32_t zero_stage;          // 2 / 3 = gradients / also weights sharded with the optimizer (NEXT-4)
    uint32_t sp_off, vpp;         // NEXT-4: sequence parallelism off (R28); virtual pipeline stages (R29)
    uint32_t wb, gb, ob;          // NEXT-4: bytes per parameter of weights / gradients / optimizer states (R30)
    uint32_t k3_caps;             // per-capacity counts from K3's masks (1) or K0's searches (0)
    uint32_t sparse;              // K3: a row with survivors * sparse < configurations takes the
                                  // two-phase (pair mask) path; 0 = never (ME_SPARSE)
    uint32_t k0_smem;             // count-only K0 stages the sorted-u lists in shared memory (ME_K0_SMEM, 1)
    uint64_t thr[8];              // floor(cap_j * num / den); 0 for unused slots
    uint64_t thr_max;             // the largest threshold: survivor <=> total <= thr_max
    // thr_j + 1 with thr_j clamped to 2^62 (every total is < 2^58): the sweep
    // tests total <= thr_j as the carry out of (thr_j + 1) + ~total
    uint64_t thr1[8];
};

// The estimator's variant policy of a configuration (the paper: all zero /
// default): ZeRO stage (NEXT-4), sequence parallelism off (R28), virtual
// pipeline stages of interleaved 1F1B (R29), bytes per parameter (R30).
struct Policy {
    uint32_t zero, sp_off, vpp, wb, gb, ob;
};

__host__ __device__ inline Policy make_policy(uint32_t zero, uint32_t sp_off, uint32_t vpp, uint32_t wb, uint32_t gb,
                                              uint32_t ob) {
    return Policy{zero, sp_off, vpp < 2 ? 1u : vpp, wb ? wb : 2u, gb ? gb : 4u, ob ? ob : 12u};
}

// In-flight work on the first pipeline stage for m microbatches per step
// (0xFFFFFFFF = unbounded, the paper mode): the microbatch count of the layer
// activations (in units of the row's layers-per-chunk, see lam0) and of the
// embedding input.  1F1B (Eq.16, R17): min(p, m) for both.  Interleaved 1F1B
// (R29, Megatron): the first GPU holds p v + p - 1 chunk-microbatches (m v if
// m = p), min(m, 2p) of them of chunk 0 (the embedding's).
__host__ __device__ inline uint32_t n_layer_mb(uint32_t p, uint32_t vpp, uint32_t m) {
    if (vpp < 2) return p < m ? p : m;
    return m == p ? p * vpp : p * vpp + p - 1;
}
__host__ __device__ inline uint32_t n_embed_mb(uint32_t p, uint32_t vpp, uint32_t m) {
    if (vpp < 2) return p < m ? p : m;
    return m < 2 * p ? m : 2 * p;
}

// Per (model, tuple) coefficients: every estimator term of a config in this
// row is an affine function of its tokens-per-microbatch u and in-flight counts.
template <typename U>
struct RowCoefT {
    U psi;        // Psi_s, Eq.6 (p = 1) / Eq.7 (p > 1) with L/p -> L0
    U optim1;     // ob ceil(Psi_s / (d c))   (Eq.10 + reading R8; ob = 12, R30)
    U par1, gra1; // weight / gradient bytes with the distributed optimizer: wb Psi_s / gb Psi_s
                  // (R9), or wb / gb ceil(Psi_s / (d c)) at ZeRO stage 3 / >= 2 (NEXT-4)
    U ms0, ms1;   // model-state bytes with the distributed optimizer off / on
    U lam0;       // Lx * B_t   (rc = 0 layer bytes per token per in-flight unit; Lx = L0, or
                  //             L/(p v) layers per chunk with interleaving)
    U lam1;       // 2 hx Lx    (rc = 1: kept layer inputs, R20; hx = h/t, or h with SP off)
    U bt;         // B_t = 12 ht + 4 hd k/t + 8 h_ffn/t   (Eq.12 / Eq.15 per token; SP off:
                  //       8 h + 4 ht + 4 hd k/t + 8 h_ffn/t, R28)
    U e8;         // 8 hx       (Eq.13 per token per mb, reading R13)
    U hc;         // [p = 1] 4 (ht + v/t)  (Eq.14, delta_{p,1} of Eq.16; SP off: 4 (h + v/t))
    uint32_t p;
    uint32_t nlay, nemb;  // paper mode (m unbounded): n_layer_mb, n_embed_mb
};
using RowCoef = RowCoefT<uint64_t>;

__host__ __device__ inline uint32_t first_stage_layers_auto(uint32_t L, uint32_t p) {
    // R19: L (p = 1), L/p when p | L, ceil(L/p) otherwise -- one formula
    return (L + p - 1) / p;
}

// x / d, a shift when d is a power of two (every t, c, p of a power-of-two
// world size)
__device__ __forceinline__ uint32_t div_u32(uint32_t x, uint32_t d) {
    return (d & (d - 1)) == 0 ? x >> (__ffs(d) - 1) : x / d;
}

// Row coefficients.  All divisions are exact under the validity rules
// (t | k | a | h, t | v, t | h_ffn, p v | L with interleaving) except the
// optimizer ceil (R8).
template <typename U>
__device__ __forceinline__ void make_row(const DevModel& M, uint32_t t, uint32_t c, uint32_t p,
                                         uint32_t d, uint32_t L0, const Policy& Q, RowCoefT<U>& R) {
    const uint32_t h = M.hidden;
    const uint32_t hd = M.head_dim;
    uint32_t ht, kt, vt, ft;
    if ((t & (t - 1)) == 0) {
        const uint32_t lt = __ffs(t) - 1;
        ht = h >> lt;
        kt = M.kv_heads >> lt;
        vt = M.vocab >> lt;
        ft = M.ffn_hidden >> lt;
    } else {
        ht = h / t;
        kt = M.kv_heads / t;
        vt = M.vocab / t;
        ft = M.ffn_hidden / t;
    }
    // per-layer shard: W_Q + W_O (2 h ht), W_K + W_V (2 h hd k/t), up/gate/down
    // (3 h h_ffn/t), two replicated RMSNorms (2h)  -- Eq.1, Eq.2, Eq.6
    const U per_layer = (U)2 * h * ht + (U)2 * h * hd * kt + (U)3 * h * ft + (U)2 * h;
    const U ends = (p == 1) ? ((U)2 * h * vt + h) : (U)h * vt;
    R.psi = ends + (U)L0 * per_layer;
    const uint32_t dc = d * c;
    U share;
    if ((dc & (dc - 1)) == 0) {
        const uint32_t sh = __ffs(dc) - 1;
        share = (R.psi + dc - 1) >> sh;
    } else {
        share = (R.psi + dc - 1) / dc;
    }
    R.optim1 = (U)Q.ob * share;
    R.par1 = Q.zero >= 3 ? (U)Q.wb * share : (U)Q.wb * R.psi;
    R.gra1 = Q.zero >= 2 ? (U)Q.gb * share : (U)Q.gb * R.psi;
    R.ms0 = (U)(Q.wb + Q.gb + Q.ob) * R.psi;
    R.ms1 = R.par1 + R.gra1 + R.optim1;
    const uint32_t hx = Q.sp_off ? h : ht;  // whole on every TP rank without SP (R28)
    R.bt = (U)12 * ht + (U)4 * hd * kt + (U)8 * ft + (Q.sp_off ? (U)8 * (h - ht) : (U)0);
    const uint32_t Lx = Q.vpp >= 2 ? M.layers / (p * Q.vpp) : L0;
    R.lam0 = (U)Lx * R.bt;
    R.lam1 = (U)2 * hx * Lx;
    R.e8 = (U)8 * hx;
    R.hc = (p == 1) ? (U)4 * ((U)hx + vt) : (U)0;
    R.p = p;
    R.nlay = n_layer_mb(p, Q.vpp, 0xFFFFFFFFu);
    R.nemb = n_embed_mb(p, Q.vpp, 0xFFFFFFFFu);
}

template <typename U>
struct TermsT {
    U params, grads, optim, layers, embed, head, total;
};

// NEXT-1: the six terms of pipeline stage i holding Li layers and n_i in-flight
// microbatches -- Eq.6 (single stage), Eq.7 (first), Eq.8 (middle), Eq.9
// (last: the final norm and the LM head); embedding input on the first stage,
// LM-head activations on the last.  For the first stage this is make_row +
// config_terms term by term.  Non-interleaved 1F1B only.
template <typename U>
__device__ __forceinline__ TermsT<U> stage_terms(const DevModel& M, uint32_t t, uint32_t c, uint32_t d, bool first,
                                                 bool last, uint32_t Li, uint32_t n_i, uint32_t u, uint32_t rc,
                                                 uint32_t dopt, const Policy& Q) {
    const uint32_t h = M.hidden, hd = M.head_dim;
    const uint32_t ht = div_u32(h, t), kt = div_u32(M.kv_heads, t), vt = div_u32(M.vocab, t),
                   ft = div_u32(M.ffn_hidden, t);
    const uint32_t hx = Q.sp_off ? h : ht;
    const U per_layer = (U)2 * h * ht + (U)2 * h * hd * kt + (U)3 * h * ft + (U)2 * h;
    const U ends = first && last ? (U)2 * h * vt + h : (first ? (U)h * vt : (last ? (U)h * vt + h : (U)0));
    const U psi = ends + (U)Li * per_layer;
    const uint32_t dc = d * c;
    const U share = (psi + dc - 1) / dc;
    const U bt = (U)12 * ht + (U)4 * hd * kt + (U)8 * ft + (Q.sp_off ? (U)8 * (h - ht) : (U)0);
    TermsT<U> T;
    T.params = dopt && Q.zero >= 3 ? (U)Q.wb * share : (U)Q.wb * psi;
    T.grads = dopt && Q.zero >= 2 ? (U)Q.gb * share : (U)Q.gb * psi;
    T.optim = dopt ? (U)Q.ob * share : (U)Q.ob * psi;
    T.layers = (U)u * (rc ? (U)2 * hx * n_i * Li + bt : (U)n_i * Li * bt);
    T.embed = first ? (U)u * ((U)8 * hx * n_i) : (U)0;
    T.head = last ? (U)u * ((U)4 * ((U)hx + vt) * n_i) : (U)0;
    T.total = T.params + T.grads + T.optim + T.layers + T.embed + T.head;
    return T;
}

// total only: model states + u * (n_lay lam + mu + n_emb e8 + hc), with the
// in-flight counts of m microbatches (0xFFFFFFFF = paper mode)
__device__ __forceinline__ uint64_t config_total(const RowCoef& R, uint32_t u, uint32_t m, uint32_t rc,
                                                 uint32_t dopt, uint32_t vpp) {
    const uint32_t nl = n_layer_mb(R.p, vpp, m), ne = n_embed_mb(R.p, vpp, m);
    const uint64_t K = (uint64_t)nl * (rc ? R.lam1 : R.lam0) + (rc ? R.bt : 0ull) + (uint64_t)ne * R.e8 + R.hc;
    return (dopt ? R.ms1 : R.ms0) + (uint64_t)u * K;
}

// all six terms (single estimates); total = their sum, equal to config_total
// term by term
template <typename U>
__device__ __forceinline__ TermsT<U> config_terms(const RowCoefT<U>& R, uint32_t u, uint32_t m, uint32_t rc,
                                                  uint32_t dopt, const Policy& Q) {
    const uint32_t nl = n_layer_mb(R.p, Q.vpp, m), ne = n_embed_mb(R.p, Q.vpp, m);
    TermsT<U> T;
    T.params = dopt ? R.par1 : (U)Q.wb * R.psi;
    T.grads = dopt ? R.gra1 : (U)Q.gb * R.psi;
    T.optim = dopt ? R.optim1 : (U)Q.ob * R.psi;
    T.layers = (U)u * (rc ? ((U)nl * R.lam1 + R.bt) : (U)nl * R.lam0);
    T.embed = (U)u * ((U)ne * R.e8);
    T.head = (U)u * R.hc;
    T.total = T.params + T.grads + T.optim + T.layers + T.embed + T.head;
    return T;
}

// ---- row-count pipeline (me_fused.cu) -------------------------------------
// One row of the sub-range table (128 B): the row's RowCoef, first index and
// pair offset; uint4-loadable prefix {w, pair_off, p, two}.
struct __align__(16) RowEnt {
    uint32_t w, pair_off, p, two;  // two: NEXT-1 last stage may decide (stage_max and p >= 2)
    uint32_t nlay, nemb;           // paper-mode in-flight counts (RowCoef)
    uint32_t _r0, _r1;
    uint64_t lam0, lam1;
    uint64_t e8, bt;
    uint64_t hc, psi;
    uint64_t par1, gra1;
    uint64_t optim1, rs;           // rs = flat index of the row's first config
    // survivor bound per (rc, do) digit: total <= thr_max  <=>  u <= umax
    // (paper mode; with the largest stage when stage_max); unused with gbs.
    // Paper mode: floor((thr_max - ms) / K) clamped to 2^32 - 1 (0 = none);
    // NEXT-1: the largest surviving u of the row (0 = none)
    uint32_t umax[4];
};
// NEXT-1: last-stage terms of one row for one (rc, do) digit (64 B)
struct __align__(16) StEnt {
    uint64_t msL, kL, parL, graL, optimL, layL, hcL, _pad;
};
constexpr uint32_t kMaxRows = 1u << 21;  // rows of one sub-range (scratch: 128 B + 4 B per row per set)

// ---- launch wrappers (me_kernels.cu) ------------------------------------
struct Cols {
    uint64_t* c[ME_N_COLS];
};

constexpr int kThreads = 256;
constexpr uint64_t kMaxSub = 1ull << 28;           // indices per sub-range of a sweep

// unit offsets = running total stats[0] + exclusive prefix of the unit
// counts; stats[0] += their total (counts: 16-byte aligned)
cudaError_t launch_scan(const uint32_t* counts, uint32_t n, uint64_t* offs, uint64_t* stats, cudaStream_t st);
// row-count pipeline (me_fused.cu): K0 rows [g0, g0 + n_rows) of the range
// [lo, hi) with their survivor counts (rcnt, per 32-row unit ucnt, per
// capacity into stats[1 + j]); K3 rows with survivors -> output rows
// caps: K0 also counts every capacity; otherwise K3 does.  !write (COUNT
// mode, the sizing pass): K0 alone, totals only (stats[0] and every
// capacity; no row entries, no unit counts, no scan needed); either way in
// at most max_blocks grid-stride blocks (0: one per 128 rows)
cudaError_t launch_rowcount(const DevSpace& S, uint64_t g0, uint32_t n_rows, uint32_t seg_lo, uint32_t n_seg_sub,
                            uint64_t lo, uint64_t hi, RowEnt* rows, StEnt* st, uint32_t* rcnt, uint32_t* ucnt,
                            uint64_t* stats, bool caps, bool write, uint32_t max_blocks, cudaStream_t stream);
// resident blocks per SM of the count-only K0
int rowcount_blocks_per_sm(const DevSpace& S);
cudaError_t launch_fused(const DevSpace& S, const RowEnt* rows, const StEnt* st, const uint32_t* rcnt,
                         const uint32_t* ucnt, const uint64_t* uoff, uint32_t n_rows, uint64_t lo, uint64_t hi,
                         me_out_mode mode, Cols cols, uint64_t capacity, uint32_t n_blocks, int minb,
                         uint32_t* next_unit, uint64_t* stats, cudaStream_t stream);
// resident K3 blocks per SM of the variant budgeted for minb blocks (2 or 3)
int fused_blocks_per_sm(me_out_mode mode, uint32_t n_cap, int minb);
uint32_t fused_units_of(uint32_t n_rows);
// order-dependent digest of a result's rows (me_result_digest): out[0] index
// digest, out[1] record digest (words = 8 for records, cols = FULL columns)
cudaError_t launch_digest(const uint64_t* const* cols, uint32_t n_cols, uint32_t words, uint64_t n, uint64_t* out,
                          cudaStream_t stream);
uint64_t digest_pow_host(uint64_t n);
// a8 deferred join of a cyclic partition (me_result_join): see join_kernel
cudaError_t launch_join(const uint64_t* gathered, int nranks, int rank, uint32_t kmax, uint64_t n_blocks,
                        uint64_t* out, cudaStream_t st);  // M^n mod 2^64 (merging digests of consecutive pieces)
// NEXT-2 planner (me_rank.cu): per result row its packed rank key (keys),
// per segment the k best rows (sel, segment-major), their index|mask words and
// keys (out, 2 words per selected row).  stride = u64 words between rows of the
// index column (8 for RECORDS)
cudaError_t launch_rank(const DevSpace& S, const uint64_t* index_col, uint32_t stride, uint64_t n_rows,
                        uint32_t green, uint32_t yellow, uint32_t gpn, uint32_t k, uint64_t* keys, uint64_t* sel,
                        uint64_t* out, cudaStream_t st);
// one configuration, one stage or (stage = 0xFFFFFFFF) the largest stage (NEXT-1)
cudaError_t launch_estimate_stage(const me_model* model, const me_parallel* cfg, uint32_t stage, me_breakdown* out,
                                  uint32_t* which, int* status, cudaStream_t st);
// single configurations (me_estimate / me_estimate_batch)
cudaError_t launch_estimate(const me_model* models, uint32_t n_models, const uint32_t* ids,
                            const me_parallel* cfgs, uint64_t n, const uint64_t* thr,
                            uint32_t n_cap, me_breakdown* out, uint8_t* mask, uint8_t* status,
                            cudaStream_t st);

}  // namespace me
