/*
 * me_oracle.c -- plain, slow, obviously-correct CPU oracle (see me_oracle.h).
 *
 * TEST INFRASTRUCTURE ONLY (tests/, __graft_entry__.smoke(), bench.py
 * cpu_baseline / --impl reference).  Shares nothing with the CUDA path.
 *
 * Each estimator step below follows the printed equation it cites, as an exact
 * rational; no factoring, hoisting or reordering beyond what the equation says.
 */
#include "me_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef __int128 i128;

/* ------------------------------------------------------------------ */
/* exact rationals                                                     */
/* ------------------------------------------------------------------ */
typedef struct {
    i128 n, d; /* d > 0, gcd(|n|, d) = 1 */
} rat;

static __thread int g_overflow; /* set when a rational step overflows 127 bits */

static i128 gcd128(i128 a, i128 b) {
    if (a < 0) a = -a;
    if (b < 0) b = -b;
    while (b) {
        i128 r = a % b;
        a = b;
        b = r;
    }
    return a;
}

static rat R(i128 n, i128 d) {
    rat r;
    if (d == 0) { g_overflow = 1; r.n = 0; r.d = 1; return r; }
    if (d < 0) { n = -n; d = -d; }
    i128 g = gcd128(n, d);
    if (g == 0) g = 1;
    r.n = n / g;
    r.d = d / g;
    return r;
}
static rat RI(i128 n) { return R(n, 1); }

static i128 mul128(i128 a, i128 b) {
    i128 r;
    if (__builtin_mul_overflow(a, b, &r)) g_overflow = 1;
    return r;
}
static i128 add128(i128 a, i128 b) {
    i128 r;
    if (__builtin_add_overflow(a, b, &r)) g_overflow = 1;
    return r;
}
static rat radd(rat x, rat y) { return R(add128(mul128(x.n, y.d), mul128(y.n, x.d)), mul128(x.d, y.d)); }
static rat rmul(rat x, rat y) {
    /* cross-reduce first so products stay small */
    i128 g1 = gcd128(x.n, y.d), g2 = gcd128(y.n, x.d);
    if (g1 == 0) g1 = 1;
    if (g2 == 0) g2 = 1;
    return R(mul128(x.n / g1, y.n / g2), mul128(x.d / g2, y.d / g1));
}
static rat rdiv(rat x, rat y) { return rmul(x, R(y.d, y.n)); }

/* integer value of an exact rational; sets *bad if it is not an integer or
 * does not fit below 2^63 */
static uint64_t to_u64(rat x, int* bad) {
    if (x.d != 1) { *bad = OR_EDIV; return 0; }
    if (x.n < 0 || x.n >= ((i128)1 << 63)) { *bad = OR_EOVERFLOW; return 0; }
    return (uint64_t)x.n;
}

/* ------------------------------------------------------------------ */
/* parameter counts                                                    */
/* ------------------------------------------------------------------ */

static int model_ok(const or_model* m) {
    if (!m) return OR_EINVAL;
    if (!m->h || !m->f || !m->L || !m->a || !m->k || !m->v) return OR_EINVAL;
    /* SPEC S:38-42 / Table "Variable names": k | a (GQA group size), a | h */
    if (m->a % m->k || m->h % m->a) return OR_EINVAL;
    return OR_OK;
}

/* Eq.1: W_Q, W_O are (h, h); W_K, W_V are (h, h/g), g = a/k.
 * Attention parameters per layer = 2 h^2 (1 + k/a). */
static rat eq1_attention(const or_model* m) {
    rat h = RI(m->h);
    return rmul(RI(2), rmul(rmul(h, h), radd(RI(1), R(m->k, m->a))));
}

/* Eq.2: up (h, h_ffn), gate (h, h_ffn), down (h_ffn, h) = 3 h h_ffn */
static rat eq2_ffn(const or_model* m) { return rmul(RI(3), rmul(RI(m->h), RI(m->f))); }

/* Eq.3, first line: 2hv + L(2h^2(1+k/a) + 3h^2 h_ffn/h + 2h) + h */
static rat eq3_total(const or_model* m) {
    rat h = RI(m->h), v = RI(m->v), L = RI(m->L);
    rat ffn = rmul(RI(3), rmul(rmul(h, h), R(m->f, m->h)));
    rat per_layer = radd(radd(eq1_attention(m), ffn), rmul(RI(2), h));
    return radd(radd(rmul(RI(2), rmul(h, v)), rmul(L, per_layer)), h);
}

int or_attention_params(const or_model* m, uint64_t* out) {
    int st = model_ok(m);
    if (st) return st;
    g_overflow = 0;
    int bad = 0;
    uint64_t r = to_u64(eq1_attention(m), &bad);
    if (g_overflow) return OR_EOVERFLOW;
    if (bad) return bad;
    *out = r;
    return OR_OK;
}
int or_ffn_params(const or_model* m, uint64_t* out) {
    int st = model_ok(m);
    if (st) return st;
    g_overflow = 0;
    int bad = 0;
    uint64_t r = to_u64(eq2_ffn(m), &bad);
    if (g_overflow) return OR_EOVERFLOW;
    if (bad) return bad;
    *out = r;
    return OR_OK;
}
int or_total_params(const or_model* m, uint64_t* out) {
    int st = model_ok(m);
    if (st) return st;
    g_overflow = 0;
    int bad = 0;
    uint64_t r = to_u64(eq3_total(m), &bad);
    if (g_overflow) return OR_EOVERFLOW;
    if (bad) return bad;
    *out = r;
    return OR_OK;
}

/* Stage-0 parameter shard Psi_s.
 *  p = 1: Eq.6  2hv/t + h + 2 L h^2 ((1 + k/a + 3/2 h_ffn/h)/t + 1/h)
 *         (reading R4: both vocab matrices and the final norm live on the only stage;
 *          Eq.18 prints hv/t, which the tables reject)
 *  p > 1: Eq.7  hv/t + 2 (L/p) h^2 ((1 + k/a + 3/2 h_ffn/h)/t + 1/h)
 *         (reading R5: no final norm on the first stage)
 * with L/p replaced by the first-stage layer count L0 (R19; L0 = L/p when p | L). */
static rat psi_stage0(const or_model* m, uint32_t t, uint32_t p, uint32_t L0) {
    rat h = RI(m->h), v = RI(m->v), T = RI(t);
    rat inner = radd(radd(RI(1), R(m->k, m->a)), rmul(R(3, 2), R(m->f, m->h)));
    rat bracket = radd(rdiv(inner, T), R(1, m->h));
    rat layers = rmul(rmul(RI(2), RI(L0)), rmul(rmul(h, h), bracket));
    if (p == 1) return radd(radd(rdiv(rmul(RI(2), rmul(h, v)), T), h), layers);
    return radd(rdiv(rmul(h, v), T), layers);
}

int or_stage0_params(const or_model* m, uint32_t t, uint32_t p, uint32_t L0, uint64_t* out) {
    int st = model_ok(m);
    if (st) return st;
    if (!t || !p || !L0) return OR_EINVAL;
    g_overflow = 0;
    int bad = 0;
    uint64_t r = to_u64(psi_stage0(m, t, p, L0), &bad);
    if (g_overflow) return OR_EOVERFLOW;
    if (bad) return bad;
    *out = r;
    return OR_OK;
}

/* Eq.12: sbh (12 + 4 k/a + 8 h_ffn/h) */
static rat eq12_bracket(const or_model* m) {
    return radd(radd(RI(12), rmul(RI(4), R(m->k, m->a))), rmul(RI(8), R(m->f, m->h)));
}

int or_activation_per_layer(const or_model* m, uint32_t s, uint32_t b, uint64_t* out) {
    int st = model_ok(m);
    if (st) return st;
    g_overflow = 0;
    int bad = 0;
    rat sbh = rmul(rmul(RI(s), RI(b)), RI(m->h));
    uint64_t r = to_u64(rmul(sbh, eq12_bracket(m)), &bad);
    if (g_overflow) return OR_EOVERFLOW;
    if (bad) return bad;
    *out = r;
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* preconditions                                                       */
/* ------------------------------------------------------------------ */

/* R19: first-stage layers.  p = 1 -> L (Eq.6); p | L -> L/p (Eq.7);
 * uneven allowed -> ceil(L/p) (the largest stage of any split); an explicit L0
 * must leave at least one layer for each of the other p-1 stages. */
uint32_t or_first_stage_layers(const or_model* m, const or_cfg* c) {
    if (!m || !c || !c->p || c->p > m->L) return 0;
    if (c->L0) {
        if (c->p == 1) return c->L0 == m->L ? c->L0 : 0;
        if (c->L0 > m->L - (c->p - 1)) return 0;
        return c->L0;
    }
    if (c->p == 1) return m->L;
    if (m->L % c->p == 0) return m->L / c->p;
    if (c->uneven) return (m->L + c->p - 1) / c->p;
    return 0;
}

/* bytes per parameter (R30): the ledger of P:192-199 unless overridden */
static uint32_t w_bytes(const or_cfg* c) { return c->wb ? c->wb : 2; }
static uint32_t g_bytes(const or_cfg* c) { return c->gb ? c->gb : 4; }
static uint32_t o_bytes(const or_cfg* c) { return c->ob ? c->ob : 12; }

static int cfg_check(const or_model* m, const or_cfg* c) {
    int st = model_ok(m);
    if (st) return st;
    if (!c || !c->d || !c->t || !c->p || !c->c || !c->b || !c->s) return OR_EINVAL;
    if (c->zero > 3) return OR_EINVAL;
    if (c->sp_off > 1 || c->wb > 8 || c->gb > 8 || c->ob > 16) return OR_EINVAL;
    /* R29 interleaved 1F1B (Megatron's schedule): p >= 2 stages of v model
     * chunks of L/(p v) layers each, and with a global batch a number of
     * microbatches that is a multiple of p */
    if (c->vpp >= 2) {
        if (c->uneven || c->L0) return OR_EINVAL;
        if (c->p < 2 || m->L % (c->p * c->vpp)) return OR_EDIV;
        if (c->gbs && c->gbs % ((uint64_t)c->d * c->b) == 0 && (c->gbs / ((uint64_t)c->d * c->b)) % c->p)
            return OR_EDIV;
    }
    /* R10: t | k (then t | a because k | a), t | v, t | h_ffn */
    if (m->k % c->t || m->v % c->t || m->f % c->t) return OR_EDIV;
    /* Eq.17: c splits the sequence */
    if (c->s % c->c) return OR_EDIV;
    if (c->p > m->L) return OR_EDIV;
    if (!or_first_stage_layers(m, c)) return OR_EDIV;
    /* R17: with a global batch the DP replicas must split it evenly */
    if (c->gbs && c->gbs % ((uint64_t)c->d * c->b)) return OR_EDIV;
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* Eq.18 with its parts                                                */
/* ------------------------------------------------------------------ */

/* Model-state bytes of a stage holding psi parameters: the ledger of
 * P:192-199 (weight BF16 2 B, gradient FP32 4 B, Adam master / momentum /
 * variance FP32 4 + 4 + 4 B).  Distributed optimizer (Eq.5 / Eq.10): the
 * 12-byte optimizer states are divided among the d*c ranks -- the largest rank
 * holds ceil(psi / (d c)) whole parameters (R8); gradients and weights stay
 * replicated (R9).  Off: Eq.4, 18 B per parameter (R21).  NEXT-4 extension
 * (ZeRO): zero = 2 also divides the gradients, zero = 3 also
 * the weights, with the same ceil rule. */
static void model_state_bytes(rat psi, const or_cfg* c, rat* params, rat* grads, rat* optim) {
    *params = rmul(RI(w_bytes(c)), psi);
    *grads = rmul(RI(g_bytes(c)), psi);
    *optim = rmul(RI(o_bytes(c)), psi);
    if (c->dopt) {
        rat share = rdiv(psi, RI((i128)c->d * c->c)); /* Psi_s / (d c) */
        i128 ceil_share = (share.n + share.d - 1) / share.d;
        *optim = rmul(RI(o_bytes(c)), RI(ceil_share));
        if (c->zero >= 2) *grads = rmul(RI(g_bytes(c)), RI(ceil_share));
        if (c->zero >= 3) *params = rmul(RI(w_bytes(c)), RI(ceil_share));
    }
}

/* Per-layer activation bytes on one TP x CP rank.  SP on (the paper, Eq.15 +
 * Eq.17): sbh/(tc) (12 + 4k/a + 8 h_ffn/h).  SP off (R28: "the
 * input to the FFN cannot be parallelized. Additionally, RMSNorm is not
 * parallelized"): the inputs of the attention and FFN blocks and the two
 * RMSNorm inputs (2 + 2 + 4 = 8 sbh of Eq.11-12) stay whole on every TP rank,
 * the rest is split: sbh/c (8 + (4 + 4k/a + 8 h_ffn/h)/t). */
static rat layer_bytes(const or_model* m, const or_cfg* c) {
    rat sbh_c = R((i128)c->s * c->b * m->h, (i128)c->c);
    if (!c->sp_off) return rmul(rdiv(sbh_c, RI(c->t)), eq12_bracket(m));
    rat split = radd(radd(RI(4), rmul(RI(4), R(m->k, m->a))), rmul(RI(8), R(m->f, m->h)));
    return rmul(sbh_c, radd(RI(8), rdiv(split, RI(c->t))));
}
/* one layer's input, 2sbh (kept per layer under recompute, R20): /t with SP */
static rat layer_input_bytes(const or_model* m, const or_cfg* c) {
    rat x = R((i128)2 * c->s * c->b * m->h, (i128)c->c);
    return c->sp_off ? x : rdiv(x, RI(c->t));
}
/* the embedding input per microbatch, Eq.13 literal (R13): 8sbh, /t with SP */
static rat embed_bytes(const or_model* m, const or_cfg* c) {
    rat x = R((i128)8 * c->s * c->b * m->h, (i128)c->c);
    return c->sp_off ? x : rdiv(x, RI(c->t));
}
/* the LM head per microbatch, Eq.14: FP32 logits 4sbv (vocab-parallel: /t)
 * plus the output RMSNorm and linear inputs 2sbh + 2sbh (/t with SP) */
static rat head_bytes(const or_model* m, const or_cfg* c) {
    rat logits = R((i128)4 * c->s * c->b * m->v, (i128)c->t * c->c);
    rat inputs = R((i128)4 * c->s * c->b * m->h, (i128)c->c);
    return radd(logits, c->sp_off ? inputs : rdiv(inputs, RI(c->t)));
}

/* In-flight work on stage 0.  1F1B (Eq.16; R17): n_inf = p
 * microbatches of L0 layers each, n_inf = min(p, m) with a global batch.
 * Interleaved 1F1B (R29, Megatron's schedule with v chunks of L/(p v) layers
 * per GPU): the first GPU runs 2(p-1) + (v-1)p warm-up forwards and one more
 * before its first backward, so it holds p v + p - 1 chunk-microbatches (all
 * m v of them when m = p), of which min(m, 2p) belong to chunk 0, the one
 * with the embedding.  Returns the (layer x microbatch) count of the layer
 * activations and the microbatch count of the embedding input. */
static void stage0_inflight(const or_model* m, const or_cfg* c, uint32_t L0, uint64_t* layer_mb, uint64_t* embed_mb) {
    uint64_t mb = UINT64_MAX; /* microbatches per step: unbounded in paper mode */
    if (c->gbs) mb = c->gbs / ((uint64_t)c->d * c->b);
    if (c->vpp < 2) {
        uint64_t n_inf = c->p < mb ? c->p : mb;
        *layer_mb = n_inf * L0;
        *embed_mb = n_inf;
        return;
    }
    uint64_t v = c->vpp, p = c->p;
    uint64_t chunks = mb == p ? p * v : p * v + p - 1;
    *layer_mb = chunks * (m->L / (p * v));
    *embed_mb = mb < 2 * p ? mb : 2 * p;
}
int or_estimate(const or_model* m, const or_cfg* c, or_breakdown* out) {
    int st = cfg_check(m, c);
    if (st) return st;
    g_overflow = 0;
    int bad = 0;
    uint32_t L0 = or_first_stage_layers(m, c);

    /* in-flight work on stage 0: Eq.16 holds p microbatches of L0
     * layers; R17 caps it at m = gbs/(d b); R29 interleaved 1F1B */
    uint64_t layer_mb, embed_mb;
    stage0_inflight(m, c, L0, &layer_mb, &embed_mb);

    /* model states: ledger P:192-199 (weight BF16 2 B, grad FP32 4 B, Adam
     * master/momentum/variance FP32 4+4+4 B; R30 other byte policies), sharding
     * Eq.5 / Eq.10 (optimizer over d*c; R9: gradients not sharded), Eq.4 when
     * the distributed optimizer is off (R21) */
    rat psi = psi_stage0(m, c->t, c->p, L0);
    uint64_t psi_s = to_u64(psi, &bad);
    rat params, grads, optim;
    model_state_bytes(psi, c, &params, &grads, &optim);

    /* activations: Eq.17, generalised per DESIGN.md §3:
     *   sbh/(tc) * ( (12 + 4k/a + 8h_ffn/h) n_inf L0 + 8 n_inf + delta_{p,1} 4(1 + v/h) )
     * n_inf L0 = L in paper mode (R16); the 8p embedding term keeps its printed h
     * (R13); the LM-head term only at p = 1 (R14).  Recompute (R20, extension):
     * every layer keeps its input, plus one layer's full set.  SP off (R28):
     * layer_bytes / embed_bytes / head_bytes above. */
    rat layers;
    if (c->rc)
        layers = radd(rmul(RI((i128)layer_mb), layer_input_bytes(m, c)), layer_bytes(m, c));
    else
        layers = rmul(RI((i128)layer_mb), layer_bytes(m, c));
    rat embed = rmul(RI((i128)embed_mb), embed_bytes(m, c));
    rat head = RI(0);
    if (c->p == 1) head = head_bytes(m, c);

    or_breakdown r;
    r.params = to_u64(params, &bad);
    r.grads = to_u64(grads, &bad);
    r.optim = to_u64(optim, &bad);
    r.act_layers = to_u64(layers, &bad);
    r.act_embed = to_u64(embed, &bad);
    r.act_head = to_u64(head, &bad);
    (void)psi_s;
    rat total = radd(radd(radd(params, grads), radd(optim, layers)), radd(embed, head));
    r.total = to_u64(total, &bad);
    if (g_overflow) return OR_EOVERFLOW;
    if (bad) return bad;
    *out = r;
    return OR_OK;
}

/* 80% rule (reading R2/R3): feasible for capacity j iff
 * total <= (num/den) * cap_j, compared exactly */
uint32_t or_cap_mask(uint64_t total, const uint64_t* cap_bytes, uint32_t n_caps, uint32_t num,
                     uint32_t den) {
    uint32_t mask = 0;
    for (uint32_t j = 0; j < n_caps; j++)
        if ((i128)total * den <= (i128)cap_bytes[j] * num) mask |= 1u << j;
    return mask;
}

/* ------------------------------------------------------------------ */
/* every pipeline stage (NEXT-1)                        */
/* ------------------------------------------------------------------ */

/* layers of stage i: stage 0 holds L0 (R19); the other p-1 stages split the
 * remaining L - L0 layers as evenly as possible, earlier stages first */
uint32_t or_stage_layers(const or_model* m, const or_cfg* c, uint32_t i) {
    uint32_t L0 = or_first_stage_layers(m, c);
    if (!L0 || i >= c->p) return 0;
    if (i == 0) return L0;
    uint32_t rest = m->L - L0, q = c->p - 1;
    return rest / q + ((i - 1) < rest % q ? 1u : 0u);
}

/* Stage i's six terms:
 *  parameters: Eq.6 (p = 1), Eq.7 (first), Eq.8 (middle), Eq.9 (last: hv/t + h)
 *              with L/p -> L_i;
 *  activations: Eq.17 with the stage's own 1F1B occupancy n_i = min(m, p - i)
 *              ("the first pipeline stage has up to p microbatches ...
 *              the last stage ... only one"), m = gbs/(d b) or
 *              unbounded in paper mode; the embedding term on stage 0 only
 *              (Eq.13), the LM-head term on the last stage only (Eq.14). */
int or_estimate_stage(const or_model* m, const or_cfg* c, uint32_t i, or_breakdown* out) {
    int st = cfg_check(m, c);
    if (st) return st;
    if (i >= c->p || c->vpp >= 2) return OR_EINVAL; /* per-stage view: non-interleaved 1F1B only */
    g_overflow = 0;
    int bad = 0;
    uint32_t Li = or_stage_layers(m, c, i);
    int first = i == 0, last = i == c->p - 1;
    uint64_t n_i = c->p - i;
    if (c->gbs) {
        uint64_t mb = c->gbs / ((uint64_t)c->d * c->b);
        if (mb < n_i) n_i = mb;
    }
    rat h = RI(m->h), v = RI(m->v), T = RI(c->t);
    rat inner = radd(radd(RI(1), R(m->k, m->a)), rmul(R(3, 2), R(m->f, m->h)));
    rat layer_part = rmul(rmul(RI(2), RI(Li)), rmul(rmul(h, h), radd(rdiv(inner, T), R(1, m->h))));
    rat psi = layer_part;                                          /* Eq.8 */
    if (first && last) psi = radd(radd(rdiv(rmul(RI(2), rmul(h, v)), T), h), layer_part); /* Eq.6 */
    else if (first) psi = radd(rdiv(rmul(h, v), T), layer_part);   /* Eq.7 */
    else if (last) psi = radd(radd(rdiv(rmul(h, v), T), h), layer_part); /* Eq.9 */
    rat params, grads, optim;
    model_state_bytes(psi, c, &params, &grads, &optim);
    rat layers = c->rc ? radd(rmul(RI((i128)n_i * Li), layer_input_bytes(m, c)), layer_bytes(m, c))
                       : rmul(RI((i128)n_i * Li), layer_bytes(m, c));
    rat embed = first ? rmul(RI((i128)n_i), embed_bytes(m, c)) : RI(0);
    rat head = last ? rmul(RI((i128)n_i), head_bytes(m, c)) : RI(0);
    or_breakdown r;
    r.params = to_u64(params, &bad);
    r.grads = to_u64(grads, &bad);
    r.optim = to_u64(optim, &bad);
    r.act_layers = to_u64(layers, &bad);
    r.act_embed = to_u64(embed, &bad);
    r.act_head = to_u64(head, &bad);
    r.total = to_u64(radd(radd(radd(params, grads), radd(optim, layers)), radd(embed, head)), &bad);
    if (g_overflow) return OR_EOVERFLOW;
    if (bad) return bad;
    *out = r;
    return OR_OK;
}

/* the stage with the largest total (the first one on ties) */
int or_estimate_max(const or_model* m, const or_cfg* c, or_breakdown* out, uint32_t* stage) {
    int st = cfg_check(m, c);
    if (st) return st;
    or_breakdown best;
    uint32_t arg = 0;
    for (uint32_t i = 0; i < c->p; i++) {
        or_breakdown r;
        if ((st = or_estimate_stage(m, c, i, &r))) return st;
        if (i == 0 || r.total > best.total) {
            best = r;
            arg = i;
        }
    }
    *out = best;
    if (stage) *stage = arg;
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* canonical enumeration                                */
/* ------------------------------------------------------------------ */
typedef struct {
    uint32_t t, c, p, d;
    uint64_t w; /* configs per (model, N, t, c, p): valid (b, s) pairs x rc x do */
} tup;

typedef struct {
    tup* v;
    uint32_t n;
} tuplist;

static int popc2(uint32_t mask) { return (mask & 1) + ((mask >> 1) & 1); }

/* all (t, c, p) with t*c*p | N in ascending (t, c, p) order and their inner size */
static int build_tuples(const or_space* sp, uint32_t N, tuplist* out) {
    uint32_t cap = 64, n = 0;
    tup* v = (tup*)malloc(cap * sizeof(tup));
    if (!v) return OR_ENOMEM;
    for (uint32_t t = 1; t <= N; t++) {
        if (N % t) continue;
        for (uint32_t c = 1; c <= N / t; c++) {
            if ((N / t) % c) continue;
            for (uint32_t p = 1; p <= N / t / c; p++) {
                if ((N / t / c) % p) continue;
                uint32_t d = N / t / c / p;
                uint64_t pairs = 0;
                for (uint32_t bi = 0; bi < sp->n_mbs; bi++)
                    for (uint32_t si = 0; si < sp->n_seq; si++) {
                        uint32_t b = sp->mbs[bi], s = sp->seq[si];
                        if (s % c) continue;
                        if (sp->gbs && sp->gbs % ((uint64_t)d * b)) continue;
                        if (sp->gbs && sp->vpp >= 2 && (sp->gbs / ((uint64_t)d * b)) % p) continue; /* R29 */
                        pairs++;
                    }
                if (n == cap) {
                    cap *= 2;
                    tup* nv = (tup*)realloc(v, cap * sizeof(tup));
                    if (!nv) { free(v); return OR_ENOMEM; }
                    v = nv;
                }
                v[n].t = t; v[n].c = c; v[n].p = p; v[n].d = d;
                v[n].w = pairs * popc2(sp->rc_mask) * popc2(sp->do_mask);
                n++;
            }
        }
    }
    out->v = v;
    out->n = n;
    return OR_OK;
}

static int valid_static(const or_space* sp, const or_model* m, const tup* u) {
    if (m->k % u->t || m->v % u->t || m->f % u->t) return 0;
    if (u->p > m->L) return 0;
    if (!sp->uneven && m->L % u->p) return 0;
    if (sp->vpp >= 2 && (u->p < 2 || m->L % (u->p * sp->vpp))) return 0; /* R29 */
    if (sp->max_t && u->t > sp->max_t) return 0;
    if (sp->max_c && u->c > sp->max_c) return 0;
    if (sp->max_p && u->p > sp->max_p) return 0;
    if (sp->gpus_per_node && u->t > sp->gpus_per_node) return 0;
    return 1;
}

static int space_ok(const or_space* sp) {
    if (!sp || !sp->models || !sp->n_models || !sp->world || !sp->n_world || !sp->mbs ||
        !sp->n_mbs || !sp->seq || !sp->n_seq)
        return OR_EINVAL;
    if (sp->n_caps > 8 || (sp->n_caps && !sp->cap_bytes)) return OR_EINVAL;
    if (!(sp->rc_mask & 3) || !(sp->do_mask & 3) || sp->zero_stage > 3) return OR_EINVAL;
    if (sp->sp_off > 1 || sp->wb > 8 || sp->gb > 8 || sp->ob > 16) return OR_EINVAL;
    if (sp->vpp >= 2 && (sp->uneven || sp->stage_max)) return OR_EINVAL;
    if (!sp->thr_num || !sp->thr_den || sp->thr_num > 1024 || sp->thr_den > 1024) return OR_EINVAL;
    for (uint32_t i = 0; i < sp->n_models; i++)
        if (model_ok(&sp->models[i])) return OR_EINVAL;
    for (uint32_t i = 0; i < sp->n_world; i++)
        if (!sp->world[i]) return OR_EINVAL;
    for (uint32_t i = 0; i < sp->n_mbs; i++)
        if (!sp->mbs[i]) return OR_EINVAL;
    for (uint32_t i = 0; i < sp->n_seq; i++)
        if (!sp->seq[i]) return OR_EINVAL;
    return OR_OK;
}

typedef struct {
    tuplist* tl; /* one per world size */
    uint32_t n;
} tables;

static void free_tables(tables* T) {
    for (uint32_t i = 0; i < T->n; i++) free(T->tl[i].v);
    free(T->tl);
}
static int build_tables(const or_space* sp, tables* T) {
    T->n = sp->n_world;
    T->tl = (tuplist*)calloc(sp->n_world, sizeof(tuplist));
    if (!T->tl) return OR_ENOMEM;
    for (uint32_t i = 0; i < sp->n_world; i++) {
        int st = build_tuples(sp, sp->world[i], &T->tl[i]);
        if (st) { free_tables(T); return st; }
    }
    return OR_OK;
}

int or_space_size(const or_space* sp, uint64_t* n) {
    int st = space_ok(sp);
    if (st) return st;
    tables T;
    if ((st = build_tables(sp, &T))) return st;
    uint64_t idx = 0;
    for (uint32_t mi = 0; mi < sp->n_models; mi++)
        for (uint32_t ni = 0; ni < sp->n_world; ni++)
            for (uint32_t j = 0; j < T.tl[ni].n; j++)
                if (valid_static(sp, &sp->models[mi], &T.tl[ni].v[j])) idx += T.tl[ni].v[j].w;
    free_tables(&T);
    *n = idx;
    return OR_OK;
}

/* sink for survivors of one contiguous index range */
typedef struct {
    const or_space* sp;
    const tables* T;
    uint64_t begin, end;
    int want_rows;
    int want_digest;          /* or_digest: hash the survivors instead of storing them */
    uint64_t dig_idx, dig_rec, dig_pow; /* running digests and M^n (see or_digest) */
    uint64_t* idx;
    or_breakdown* rows;
    uint64_t n, cap;
    uint64_t cap_counts[8];
    int status;
    /* decode target */
    int decode_only;
    uint32_t dec_model, dec_world;
    or_cfg dec_cfg;
} walk_t;

static uint64_t dig_mix(uint64_t x);
#define DIG_C 0x9E3779B97F4A7C15ull
#define DIG_M 0xD1B54A32D192ED03ull

static int push(walk_t* w, uint64_t idx_mask, const or_breakdown* r) {
    if (w->want_digest) {
        /* survivor j (= w->n) of the piece contributes g(record) * M^j */
        uint64_t v[8] = {idx_mask, r->params, r->grads, r->optim, r->act_layers, r->act_embed, r->act_head, r->total};
        uint64_t gi = dig_mix(idx_mask + DIG_C), gr = DIG_C;
        for (int k = 0; k < 8; k++) gr = dig_mix(gr ^ v[k]);
        w->dig_idx += gi * w->dig_pow;
        w->dig_rec += gr * w->dig_pow;
        w->dig_pow *= DIG_M;
        w->n++;
        return OR_OK;
    }
    if (!w->want_rows) { w->n++; return OR_OK; }
    if (w->n == w->cap) {
        uint64_t nc = w->cap ? w->cap * 2 : 1024;
        uint64_t* ni = (uint64_t*)realloc(w->idx, nc * sizeof(uint64_t));
        if (!ni) return OR_ENOMEM;
        w->idx = ni;
        or_breakdown* nr = (or_breakdown*)realloc(w->rows, nc * sizeof(or_breakdown));
        if (!nr) return OR_ENOMEM;
        w->rows = nr;
        w->cap = nc;
    }
    w->idx[w->n] = idx_mask;
    w->rows[w->n] = *r;
    w->n++;
    return OR_OK;
}

/* The canonical nested loops: model -> N -> (t asc, c asc, p asc) -> b -> s ->
 * rc -> do.  Tuples failing valid_static and (b, s) pairs failing c | s or
 * (d b) | gbs consume no index. */
static void walk(walk_t* w) {
    const or_space* sp = w->sp;
    uint64_t idx = 0;
    for (uint32_t mi = 0; mi < sp->n_models; mi++) {
        const or_model* m = &sp->models[mi];
        for (uint32_t ni = 0; ni < sp->n_world; ni++) {
            const tuplist* tl = &w->T->tl[ni];
            for (uint32_t j = 0; j < tl->n; j++) {
                const tup* u = &tl->v[j];
                if (!valid_static(sp, m, u)) continue;
                if (idx + u->w <= w->begin) { idx += u->w; continue; }
                if (idx >= w->end) return;
                for (uint32_t bi = 0; bi < sp->n_mbs; bi++)
                    for (uint32_t si = 0; si < sp->n_seq; si++) {
                        uint32_t b = sp->mbs[bi], s = sp->seq[si];
                        if (s % u->c) continue;
                        if (sp->gbs && sp->gbs % ((uint64_t)u->d * b)) continue;
                        if (sp->gbs && sp->vpp >= 2 && (sp->gbs / ((uint64_t)u->d * b)) % u->p) continue;
                        for (uint32_t rc = 0; rc < 2; rc++) {
                            if (!((sp->rc_mask >> rc) & 1)) continue;
                            for (uint32_t dopt = 0; dopt < 2; dopt++) {
                                if (!((sp->do_mask >> dopt) & 1)) continue;
                                if (idx >= w->begin && idx < w->end) {
                                    or_cfg c;
                                    memset(&c, 0, sizeof c);
                                    c.d = u->d; c.t = u->t; c.p = u->p; c.c = u->c;
                                    c.b = b; c.s = s; c.gbs = sp->gbs; c.L0 = 0;
                                    c.rc = (uint8_t)rc; c.dopt = (uint8_t)dopt;
                                    c.uneven = sp->uneven;
                                    c.zero = (uint8_t)sp->zero_stage;
                                    c.sp_off = sp->sp_off;
                                    c.vpp = sp->vpp;
                                    c.wb = sp->wb;
                                    c.gb = sp->gb;
                                    c.ob = sp->ob;
                                    if (w->decode_only) {
                                        w->dec_model = mi;
                                        w->dec_world = sp->world[ni];
                                        w->dec_cfg = c;
                                        w->status = OR_OK;
                                        return;
                                    }
                                    or_breakdown r;
                                    int st = sp->stage_max ? or_estimate_max(m, &c, &r, NULL)
                                                           : or_estimate(m, &c, &r);
                                    if (st) { w->status = st; return; }
                                    uint32_t mask = or_cap_mask(r.total, sp->cap_bytes, sp->n_caps,
                                                                sp->thr_num, sp->thr_den);
                                    for (uint32_t q = 0; q < sp->n_caps; q++)
                                        w->cap_counts[q] += (mask >> q) & 1;
                                    if (mask) {
                                        st = push(w, idx | ((uint64_t)mask << 56), &r);
                                        if (st) { w->status = st; return; }
                                    }
                                }
                                idx++;
                                if (idx >= w->end) return;
                            }
                        }
                    }
            }
        }
    }
}

int or_decode(const or_space* sp, uint64_t index, uint32_t* model_id, uint32_t* world, or_cfg* cfg) {
    int st = space_ok(sp);
    if (st) return st;
    tables T;
    if ((st = build_tables(sp, &T))) return st;
    walk_t w;
    memset(&w, 0, sizeof w);
    w.sp = sp; w.T = &T; w.begin = index; w.end = index + 1;
    w.decode_only = 1;
    w.status = OR_ERANGE; /* stays if index is past the end */
    walk(&w);
    free_tables(&T);
    if (w.status) return w.status;
    if (model_id) *model_id = w.dec_model;
    if (world) *world = w.dec_world;
    if (cfg) *cfg = w.dec_cfg;
    return OR_OK;
}

/* The same canonical walk, visiting only the given ascending indices: every
 * visited configuration is evaluated (feasible or not). */
int or_points(const or_space* sp, const uint64_t* points, uint64_t n, or_breakdown* rows,
              uint32_t* masks) {
    int st = space_ok(sp);
    if (st) return st;
    for (uint64_t k = 1; k < n; k++)
        if (points[k] <= points[k - 1]) return OR_EINVAL;
    tables T;
    if ((st = build_tables(sp, &T))) return st;
    uint64_t idx = 0, k = 0;
    for (uint32_t mi = 0; mi < sp->n_models && k < n; mi++) {
        const or_model* m = &sp->models[mi];
        for (uint32_t ni = 0; ni < sp->n_world && k < n; ni++) {
            const tuplist* tl = &T.tl[ni];
            for (uint32_t j = 0; j < tl->n && k < n; j++) {
                const tup* u = &tl->v[j];
                if (!valid_static(sp, m, u)) continue;
                if (idx + u->w <= points[k]) { idx += u->w; continue; }
                for (uint32_t bi = 0; bi < sp->n_mbs; bi++)
                    for (uint32_t si = 0; si < sp->n_seq; si++) {
                        uint32_t b = sp->mbs[bi], s = sp->seq[si];
                        if (s % u->c) continue;
                        if (sp->gbs && sp->gbs % ((uint64_t)u->d * b)) continue;
                        if (sp->gbs && sp->vpp >= 2 && (sp->gbs / ((uint64_t)u->d * b)) % u->p) continue;
                        for (uint32_t rc = 0; rc < 2; rc++) {
                            if (!((sp->rc_mask >> rc) & 1)) continue;
                            for (uint32_t dopt = 0; dopt < 2; dopt++) {
                                if (!((sp->do_mask >> dopt) & 1)) continue;
                                if (k < n && idx == points[k]) {
                                    or_cfg c;
                                    memset(&c, 0, sizeof c);
                                    c.d = u->d; c.t = u->t; c.p = u->p; c.c = u->c;
                                    c.b = b; c.s = s; c.gbs = sp->gbs;
                                    c.rc = (uint8_t)rc; c.dopt = (uint8_t)dopt;
                                    c.uneven = sp->uneven;
                                    c.zero = (uint8_t)sp->zero_stage;
                                    c.sp_off = sp->sp_off;
                                    c.vpp = sp->vpp;
                                    c.wb = sp->wb;
                                    c.gb = sp->gb;
                                    c.ob = sp->ob;
                                    or_breakdown r;
                                    st = sp->stage_max ? or_estimate_max(m, &c, &r, NULL)
                                                       : or_estimate(m, &c, &r);
                                    if (st) { free_tables(&T); return st; }
                                    if (rows) rows[k] = r;
                                    if (masks)
                                        masks[k] = or_cap_mask(r.total, sp->cap_bytes, sp->n_caps,
                                                               sp->thr_num, sp->thr_den);
                                    k++;
                                }
                                idx++;
                            }
                        }
                    }
            }
        }
    }
    free_tables(&T);
    return k == n ? OR_OK : OR_ERANGE;
}

static void* walk_thread(void* arg) {
    walk((walk_t*)arg);
    return NULL;
}

int or_sweep(const or_space* sp, uint64_t begin, uint64_t end, uint64_t* idx_mask,
             or_breakdown* rows, uint64_t cap, uint64_t* count, uint64_t* cap_counts,
             int n_threads) {
    int st = space_ok(sp);
    if (st) return st;
    if (end == 0) {
        /* whole space: its size bounds the range (a given end may also lie
           past the space; the walk then simply stops at its last index) */
        if ((st = or_space_size(sp, &end))) return st;
    }
    if (begin > end) begin = end;
    if (n_threads < 1) n_threads = 1;
    if ((uint64_t)n_threads > end - begin) n_threads = (int)(end - begin ? end - begin : 1);
    tables T;
    if ((st = build_tables(sp, &T))) return st;
    walk_t* ws = (walk_t*)calloc((size_t)n_threads, sizeof(walk_t));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!ws || !th) { free(ws); free(th); free_tables(&T); return OR_ENOMEM; }
    uint64_t len = end - begin;
    for (int i = 0; i < n_threads; i++) {
        ws[i].sp = sp;
        ws[i].T = &T;
        ws[i].begin = begin + len * (uint64_t)i / (uint64_t)n_threads;
        ws[i].end = begin + len * (uint64_t)(i + 1) / (uint64_t)n_threads;
        ws[i].want_rows = (idx_mask || rows) ? 1 : 0;
        if (ws[i].end == ws[i].begin) continue;
        if (n_threads == 1) walk(&ws[i]);
        else pthread_create(&th[i], NULL, walk_thread, &ws[i]);
    }
    if (n_threads > 1)
        for (int i = 0; i < n_threads; i++)
            if (ws[i].end != ws[i].begin) pthread_join(th[i], NULL);
    uint64_t n = 0;
    uint64_t cc[8] = {0};
    int status = OR_OK;
    for (int i = 0; i < n_threads; i++) {
        if (ws[i].status && !status) status = ws[i].status;
        for (uint32_t q = 0; q < sp->n_caps; q++) cc[q] += ws[i].cap_counts[q];
        for (uint64_t r = 0; r < ws[i].n && ws[i].want_rows; r++) {
            if (n + r < cap) {
                if (idx_mask) idx_mask[n + r] = ws[i].idx[r];
                if (rows) rows[n + r] = ws[i].rows[r];
            }
        }
        n += ws[i].n;
        free(ws[i].idx);
        free(ws[i].rows);
    }
    free(ws);
    free(th);
    free_tables(&T);
    if (count) *count = n;
    if (cap_counts)
        for (uint32_t q = 0; q < sp->n_caps; q++) cap_counts[q] = cc[q];
    if (status) return status;
    if ((idx_mask || rows) && n > cap) return OR_ERANGE;
    return OR_OK;
}

/* ------------------------------------------------------------------ */
/* whole-chunk digests (verification of full-size sweeps)              */
/* ------------------------------------------------------------------ */

/* splitmix64 finaliser */
static uint64_t dig_mix(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

static uint64_t dig_pow(uint64_t n) {
    uint64_t r = 1, b = DIG_M;
    while (n) {
        if (n & 1) r *= b;
        b *= b;
        n >>= 1;
    }
    return r;
}

typedef struct {
    walk_t* w;
    uint32_t n_pieces;
    uint32_t next; /* atomically incremented */
} piece_pool;

static void* digest_thread(void* arg) {
    piece_pool* pp = (piece_pool*)arg;
    for (;;) {
        uint32_t k = __atomic_fetch_add(&pp->next, 1u, __ATOMIC_RELAXED);
        if (k >= pp->n_pieces) break;
        if (pp->w[k].end > pp->w[k].begin) walk(&pp->w[k]);
    }
    return NULL;
}

int or_digest(const or_space* sp, uint64_t begin, uint64_t end, uint64_t chunk, int n_threads, uint64_t* out) {
    int st = space_ok(sp);
    if (st) return st;
    if (!out || !chunk) return OR_EINVAL;
    uint64_t size;
    if ((st = or_space_size(sp, &size))) return st;
    if (end == 0 || end > size) end = size;
    if (begin > end) begin = end;
    if (n_threads < 1) n_threads = 1;
    const uint64_t n_chunks = (end - begin + chunk - 1) / chunk;
    const uint32_t per = (uint32_t)n_threads; /* pieces per chunk */
    const uint64_t n_pieces = n_chunks * per;
    tables T;
    if ((st = build_tables(sp, &T))) return st;
    walk_t* ws = (walk_t*)calloc(n_pieces ? n_pieces : 1, sizeof(walk_t));
    pthread_t* th = (pthread_t*)calloc((size_t)n_threads, sizeof(pthread_t));
    if (!ws || !th) { free(ws); free(th); free_tables(&T); return OR_ENOMEM; }
    for (uint64_t c = 0; c < n_chunks; c++) {
        const uint64_t cb = begin + c * chunk, ce = cb + chunk < end ? cb + chunk : end;
        for (uint32_t q = 0; q < per; q++) {
            walk_t* w = &ws[c * per + q];
            w->sp = sp;
            w->T = &T;
            w->begin = cb + (ce - cb) * q / per;
            w->end = cb + (ce - cb) * (q + 1) / per;
            w->want_digest = 1;
            w->dig_pow = 1;
        }
    }
    piece_pool pool = {ws, (uint32_t)n_pieces, 0};
    for (int i = 0; i < n_threads; i++) pthread_create(&th[i], NULL, digest_thread, &pool);
    for (int i = 0; i < n_threads; i++) pthread_join(th[i], NULL);
    int status = OR_OK;
    for (uint64_t c = 0; c < n_chunks; c++) {
        uint64_t* o = out + c * OR_DIGEST_WORDS;
        memset(o, 0, OR_DIGEST_WORDS * sizeof(uint64_t));
        for (uint32_t q = 0; q < per; q++) {
            const walk_t* w = &ws[c * per + q];
            if (w->status && !status) status = w->status;
            /* pieces in order: D(A B) = D(A) + M^|A| D(B) */
            const uint64_t shift = dig_pow(o[0]);
            o[9] += shift * w->dig_idx;
            o[10] += shift * w->dig_rec;
            o[0] += w->n;
            for (uint32_t k = 0; k < 8; k++) o[1 + k] += w->cap_counts[k];
        }
    }
    free(ws);
    free(th);
    free_tables(&T);
    return status;
}
