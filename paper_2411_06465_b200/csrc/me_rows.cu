// me_rows.cu -- the row-table sweep pipeline (sm_100a), DESIGN.md §6.
//
// A row is a run of configurations sharing (model, N, t, c, p, d): every
// estimator term of its configs is an affine function of the pair's tokens
// per microbatch u (and in-flight count), with coefficients fixed per row
// (RowCoef).  Per sub-range of the flat index space:
//
//  K0 row_kernel      one thread per row of the sub-range: its coefficients,
//                     first index and pair offset (RowEnt), the last-stage
//                     terms per (rc, do) digit when the largest stage decides
//                     (StEnt), and the walker checkpoint of every span that
//                     starts inside it;
//  K1 stage_kernel    one warp per span of whole tiles: walks the span with
//                     the row table (a row change is one 80-byte load, not a
//                     re-derivation), tests every config against the
//                     capacities and appends one 8-byte descriptor
//                     {position in row, local row, capacity mask} per
//                     survivor to the span's slice of a descriptor buffer;
//                     stores the span's survivor count;
//  scan               span counts -> output offsets (scan_kernel);
//  K3 expand_kernel   warps take spans in grid-stride order and turn 32
//                     descriptors at a time into output rows: every lane
//                     produces one survivor, so the stores of a warp cover
//                     32 consecutive rows (records: 2 KB contiguous), and the
//                     per-capacity counts come from ballots of the masks.
//
// K1 evaluates every configuration once (no second walk in the write pass);
// K3 touches survivors only.  Counts per capacity are exact: K3 sees every
// survivor once.
#include <cuda_runtime.h>

#include <cstdlib>

#include "me_dev.cuh"
#include "me_kernels.cuh"

namespace me {

namespace {

// lane-constant selections of a row's coefficients for the lane's (rc, do)
struct LaneCoef {
    uint64_t nms;        // ~model-state bytes
    uint64_t na, nb;     // -(per-token activation bytes) = -(n_inf a + b)
    uint64_t nkp;        // -(p a + b)
    uint32_t p;
    bool two;            // NEXT-1: the last stage may decide
    uint64_t nmsL, nkL;  // ~msL, -kL of the last stage
    uint32_t umax;       // FAST walker: survivor <=> u <= umax
};

__device__ __forceinline__ void lane_coef(const uint4 h, const ulonglong2 ms, const ulonglong2 lam,
                                          const ulonglong2 e8bt, const uint64_t hc, uint32_t rc, uint32_t dopt,
                                          LaneCoef& C) {
    const uint32_t p = h.z;
    const uint64_t a = (rc ? lam.y : lam.x) + e8bt.x;
    const uint64_t b = rc ? e8bt.y + hc : hc;
    C.nms = ~(dopt ? ms.y : ms.x);
    C.na = 0ull - a;
    C.nb = 0ull - b;
    C.nkp = 0ull - ((uint64_t)p * a + b);
    C.p = p;
}

// Table walker: lane position = (row k of the sub-range table, offset r).
// FAST: the survivor test is u <= umax (paper mode, no mask): a row change
// loads 32 bytes instead of 80.
template <bool FAST>
struct TWalker {
    uint32_t k, r, w;
    const uint2* pp;
    uint32_t rc, dopt, sel;
    LaneCoef C;

    __device__ __forceinline__ void set_row(const DevSpace& S, const RowEnt* __restrict__ rows,
                                            const StEnt* __restrict__ st) {
        const uint4* e = reinterpret_cast<const uint4*>(rows + k);
        const uint4 h = __ldg(e);
        w = h.x;
        pp = reinterpret_cast<const uint2*>(S.pairs) + h.y + (r >> S.lg_rcdo);
        if (FAST) {
            const uint4 um = __ldg(e + 7);
            C.umax = sel == 0 ? um.x : sel == 1 ? um.y : sel == 2 ? um.z : um.w;
            return;
        }
        const uint4 v1 = __ldg(e + 1), v2 = __ldg(e + 2), v3 = __ldg(e + 3), v4 = __ldg(e + 4);
        const ulonglong2 ms = make_ulonglong2(((uint64_t)v1.y << 32) | v1.x, ((uint64_t)v1.w << 32) | v1.z);
        const ulonglong2 lam = make_ulonglong2(((uint64_t)v2.y << 32) | v2.x, ((uint64_t)v2.w << 32) | v2.z);
        const ulonglong2 eb = make_ulonglong2(((uint64_t)v3.y << 32) | v3.x, ((uint64_t)v3.w << 32) | v3.z);
        const uint64_t hc = ((uint64_t)v4.y << 32) | v4.x;
        lane_coef(h, ms, lam, eb, hc, rc, dopt, C);
        C.two = h.w != 0;
        if (S.stage_max && C.two) {
            const StEnt& x = st[(size_t)k << S.lg_rcdo | sel];
            C.nmsL = ~__ldg(&x.msL);
            C.nkL = 0ull - __ldg(&x.kL);
        }
    }

    __device__ __forceinline__ void restore(const DevSpace& S, const RowEnt* __restrict__ rows,
                                            const StEnt* __restrict__ st, uint2 ck, uint32_t lane) {
        k = ck.x;
        r = ck.y + lane;
        sel = r & ((1u << S.lg_rcdo) - 1u);  // constant along the walk: row lengths are multiples of n_rcdo
        rc = (S.rcdo_rc >> sel) & 1u;
        dopt = (S.rcdo_do >> sel) & 1u;
        set_row(S, rows, st);
        while (r >= w) {
            r -= w;
            ++k;
            set_row(S, rows, st);
        }
    }

    __device__ __forceinline__ void advance32(const DevSpace& S, const RowEnt* __restrict__ rows,
                                              const StEnt* __restrict__ st, uint32_t pstep) {
        r += 32;
        if (r < w) {
            pp += pstep;
        } else {
            do {
                r -= w;
                ++k;
                set_row(S, rows, st);
            } while (r >= w);
        }
    }
};

// ---------------------------------------------------------------- K0
// seg_lo, n_seg_sub: the segments holding rows [g0, g0 + n_rows) are
// seg_lo .. seg_lo + n_seg_sub - 2 (the binary search covers only them)
__global__ void row_kernel(const DevSpace S, const uint64_t g0, const uint32_t n_rows, const uint32_t seg_lo,
                           const uint32_t n_seg_sub, const uint64_t base, const uint64_t hi, const uint32_t span_len,
                           const uint32_t n_spans, RowEnt* __restrict__ rows, StEnt* __restrict__ st,
                           uint2* __restrict__ span_ck) {
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n_rows; k += gridDim.x * blockDim.x) {
        const uint64_t g = g0 + k;
        const uint32_t s = seg_lo + upper_bound_u64(S.seg_row + seg_lo, n_seg_sub, g) - 1;
        const uint32_t m = s / S.n_world, n = s - m * S.n_world;
        const uint4 m0 = __ldg(reinterpret_cast<const uint4*>(S.models + m));
        const uint4 m1 = __ldg(reinterpret_cast<const uint4*>(S.models + m) + 1);
        const DevModel M{m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, 0u};
        const uint32_t cls = __ldg(S.model_class + m);
        const uint32_t j = __ldg(S.list_off + cls * S.n_world + n) + (uint32_t)(g - __ldg(S.seg_row + s));
        const DevTuple tu = S.tuples[__ldg(S.list_tuple + j)];
        const uint64_t rs = __ldg(S.seg_prefix + s) + __ldg(S.list_prefix + j);
        const uint32_t L0 = tu.p == 1 ? M.layers : div_u32(M.layers + tu.p - 1, tu.p);
        RowCoef R;
        make_row(M, tu.t, tu.c, tu.p, tu.d, L0, S.zero_stage, R);
        const bool two = S.stage_max && tu.p >= 2;
        RowEnt e;
        e.w = tu.w;
        e.pair_off = tu.pair_off;
        e.p = tu.p;
        e.two = two ? 1u : 0u;
        e.ms0 = R.ms0;
        e.ms1 = R.ms1;
        e.lam0 = R.lam0;
        e.lam1 = R.lam1;
        e.e8 = R.e8;
        e.bt = R.bt;
        e.hc = R.hc;
        e.psi = R.psi;
        e.par1 = R.par1;
        e.gra1 = R.gra1;
        e.optim1 = R.optim1;
        e.rs = rs;
        // survivor bound per digit: total = ms + u K <= thr_max  <=>  u <= (thr_max - ms) / K
        // (u >= 1: a bound of 0 admits nothing); the last stage's bound too when it may decide
        const uint32_t Ll = two ? (M.layers - L0) / (tu.p - 1) : 0u;
        for (uint32_t sel = 0; sel < 4; sel++) {
            uint64_t U = 0;
            if (sel < (1u << S.lg_rcdo)) {
                const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
                const uint64_t ms = dopt ? R.ms1 : R.ms0;
                const uint64_t K = (uint64_t)tu.p * ((rc ? R.lam1 : R.lam0) + R.e8) + (rc ? R.bt + R.hc : R.hc);
                U = ms > S.thr_max ? 0ull : (S.thr_max - ms) / K;
                if (two) {
                    const TermsT<uint64_t> T =
                        stage_terms<uint64_t>(M, tu.t, tu.c, tu.d, false, true, Ll, 1u, 1u, rc, dopt, S.zero_stage);
                    const uint64_t msL = T.params + T.grads + T.optim, kL = T.layers + T.head;
                    const uint64_t UL = msL > S.thr_max ? 0ull : (S.thr_max - msL) / kL;
                    U = U < UL ? U : UL;
                }
            }
            e.umax[sel] = U > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)U;
        }
        rows[k] = e;
        if (two) {
            // the last stage holds floor((L - L0) / (p - 1)) layers, one microbatch
            const uint32_t Ll = (M.layers - L0) / (tu.p - 1);
            for (uint32_t sel = 0; sel < (1u << S.lg_rcdo); sel++) {
                const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
                const TermsT<uint64_t> T =
                    stage_terms<uint64_t>(M, tu.t, tu.c, tu.d, false, true, Ll, 1u, 1u, rc, dopt, S.zero_stage);
                StEnt x;
                x.msL = T.params + T.grads + T.optim;
                x.kL = T.layers + T.head;
                x.parL = T.params;
                x.graL = T.grads;
                x.optimL = T.optim;
                x.layL = T.layers;
                x.hcL = T.head;
                x._pad = 0;
                st[(size_t)k << S.lg_rcdo | sel] = x;
            }
        }
        // checkpoints of the spans starting inside this row
        const uint64_t lo_r = rs > base ? rs : base;
        const uint64_t hi_r = rs + tu.w < hi ? rs + tu.w : hi;
        if (lo_r < hi_r) {
            uint64_t sp = (lo_r - base + span_len - 1) / span_len;
            for (; sp < n_spans; sp++) {
                const uint64_t ps = base + sp * span_len;
                if (ps >= hi_r) break;
                span_ck[sp] = make_uint2(k, (uint32_t)(ps - rs));
            }
        }
    }
}

// ---------------------------------------------------------------- K1
// Descriptor of a survivor, two formats (the plan picks D32 when no span can
// touch more than 255 rows):
//  D64  bits 0..31 position in its row, 32..55 row of the sub-range table,
//       56..63 capacity mask;
//  D32  bits 0..15 position in the span, 16..23 row - the span's first row,
//       24..31 capacity mask.
// MASK: the descriptor carries the capacity mask (INDEX output, whose expand
// pass computes no totals); otherwise only the survivor test (total <= the
// largest threshold: one carry chain) is made here and the expand kernel
// derives the mask from the total it computes anyway.
template <int NCAP, bool GBS, bool STMAX, bool RAGGED, bool MASK>
__device__ __forceinline__ void stage_span(const DevSpace& S, const RowEnt* __restrict__ rows,
                                           const StEnt* __restrict__ st, uint32_t rounds, uint32_t lo_rel,
                                           uint32_t hi_rel, uint2 ck, uint64_t* __restrict__ desc, bool d32,
                                           uint32_t* __restrict__ count_out, uint32_t lane) {
    // positions relative to the span start; RAGGED: the span is cut by the
    // range [lo, hi) = [lo_rel, hi_rel) (first / last span), a lane past the
    // end is parked on the last index and never advances
    constexpr bool FAST = !GBS && !MASK;
    TWalker<FAST> W;
    W.restore(S, rows, st, ck, !RAGGED || lane < hi_rel ? lane : hi_rel - 1);
    const uint32_t pstep = 32u >> S.lg_rcdo;
    uint32_t cnt = 0;
    uint32_t rel = lane;
    uint32_t dk16 = (W.k - ck.x) << 16;  // D32: row - span's first row, in place
    uint2 pr = __ldg(W.pp);
    for (uint32_t it = 0; it < rounds; it++, rel += 32) {
        const bool more = it + 1 < rounds;
        const bool in_row = W.r + 32 < W.w;
        uint2 prn = pr;
        if (in_row && more) prn = __ldg(W.pp + pstep);  // next round's pair, issued early
        const uint32_t u = pr.x;
        uint32_t mask;
        if (FAST) {
            mask = u <= W.C.umax ? 1u : 0u;
        } else {
            const uint32_t n_inf = GBS ? min(W.C.p, pr.y) : W.C.p;
            const uint64_t nK = GBS ? (uint64_t)n_inf * W.C.na + W.C.nb : W.C.nkp;
            uint64_t ntot = W.C.nms + (uint64_t)u * nK;  // ~total
            if (STMAX && W.C.two) {
                const uint64_t ntl = W.C.nmsL + (uint64_t)u * W.C.nkL;
                ntot = ntl < ntot ? ntl : ntot;
            }
            mask = MASK ? cap_mask_n<NCAP>(S, ntot) : le_shift(0u, ntot, S.thr1c[0]);
        }
        if (RAGGED && (rel < lo_rel || rel >= hi_rel)) mask = 0;
        const uint32_t ballot = __ballot_sync(0xffffffffu, mask != 0);
        if (mask) {
            const uint32_t m = MASK ? mask << 24 : 0u;
            const uint32_t at = cnt + __popc(ballot & ((1u << lane) - 1u));
            if (d32) reinterpret_cast<uint32_t*>(desc)[at] = rel | dk16 | m;
            else desc[at] = ((uint64_t)(W.k | m) << 32) | W.r;
        }
        cnt += __popc(ballot);
        if (more && (!RAGGED || rel + 32 < hi_rel)) {
            if (in_row) {
                W.r += 32;
                W.pp += pstep;
                pr = prn;
            } else {
                W.advance32(S, rows, st, pstep);
                pr = __ldg(W.pp);
                dk16 = (W.k - ck.x) << 16;
            }
        }
    }
    if (lane == 0) *count_out = cnt;
}

template <int NCAP, bool MASK>
__device__ __forceinline__ void stage_one(const DevSpace& S, const RowEnt* __restrict__ rows,
                                          const StEnt* __restrict__ st, uint64_t lo, uint64_t hi, uint32_t span_tiles,
                                          uint32_t sp, const uint2* __restrict__ span_ck, uint64_t* __restrict__ desc,
                                          bool d32, uint32_t* __restrict__ span_count, uint32_t lane);

template <int NCAP, bool MASK>
__global__ void __launch_bounds__(kStageWarps * 32, 24 / kStageWarps) stage_kernel(const DevSpace S, const RowEnt* __restrict__ rows,
                                                            const StEnt* __restrict__ st, const uint64_t lo,
                                                            const uint64_t hi, const uint32_t span_tiles,
                                                            const uint32_t n_spans, const uint2* __restrict__ span_ck,
                                                            uint64_t* __restrict__ desc, const uint32_t d32,
                                                            uint32_t* __restrict__ span_count,
                                                            uint32_t* __restrict__ block_count) {
    __shared__ uint32_t s_cnt[kStageWarps];
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t sp = blockIdx.x * kStageWarps + wid;
    if (sp < n_spans)
        stage_one<NCAP, MASK>(S, rows, st, lo, hi, span_tiles, sp, span_ck, desc, d32 != 0, span_count, lane);
    // the block's survivors (the scan runs over blocks; the expand kernel
    // adds the counts of the earlier spans of its block)
    if (lane == 0) s_cnt[wid] = sp < n_spans ? span_count[sp] : 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < kStageWarps; w++) t += s_cnt[w];
        block_count[blockIdx.x] = t;
    }
}

template <int NCAP, bool MASK>
__device__ __forceinline__ void stage_one(const DevSpace& S, const RowEnt* __restrict__ rows,
                                          const StEnt* __restrict__ st, uint64_t lo, uint64_t hi, uint32_t span_tiles,
                                          uint32_t sp, const uint2* __restrict__ span_ck, uint64_t* __restrict__ desc,
                                          bool d32, uint32_t* __restrict__ span_count, uint32_t lane) {
    const uint64_t base = lo & ~31ull;
    const uint32_t n_tiles = (uint32_t)((hi - base + kTile - 1) / kTile);
    const uint32_t t0 = sp * span_tiles;
    const uint32_t t1 = min(n_tiles, t0 + span_tiles);
    const uint64_t s0 = base + (uint64_t)t0 * kTile;
    const uint64_t e = min(base + (uint64_t)t1 * kTile, hi);
    const uint32_t rounds = (uint32_t)((e - s0 + 31) / 32);
    const uint32_t lo_rel = lo > s0 ? (uint32_t)(lo - s0) : 0u, hi_rel = (uint32_t)(e - s0);
    const bool ragged = lo_rel != 0 || (hi_rel & 31u) != 0;
    const uint2 ck = __ldg(span_ck + sp);
    // the span's slice: span_len slots of the descriptor format
    uint64_t* d = d32 ? reinterpret_cast<uint64_t*>(reinterpret_cast<uint32_t*>(desc) + (size_t)sp * span_tiles * kTile)
                      : desc + (size_t)sp * span_tiles * kTile;
    uint32_t* c = span_count + sp;
#define ME_STAGE(GBS, STMAX)                                                                           \
    (ragged ? stage_span<NCAP, GBS, STMAX, true, MASK>(S, rows, st, rounds, lo_rel, hi_rel, ck, d, d32, c, lane) \
            : stage_span<NCAP, GBS, STMAX, false, MASK>(S, rows, st, rounds, lo_rel, hi_rel, ck, d, d32, c, lane))
    if (S.stage_max) {
        if (S.gbs_mode) ME_STAGE(true, true);
        else ME_STAGE(false, true);
    } else {
        if (S.gbs_mode) ME_STAGE(true, false);
        else ME_STAGE(false, false);
    }
#undef ME_STAGE
}

// ---------------------------------------------------------------- K3
// per-lane capacity counters: 16-bit fields, capacities 4j .. 4j + 3 in word j
// (the mask bits spread to bit 16 i by one multiply)
template <int NCAP>
struct CapPack {
    uint64_t w[(NCAP + 3) / 4];
    __device__ __forceinline__ CapPack() {
#pragma unroll
        for (int j = 0; j < (NCAP + 3) / 4; j++) w[j] = 0;
    }
    __device__ __forceinline__ void add(uint32_t mask) {
#pragma unroll
        for (int j = 0; j < (NCAP + 3) / 4; j++)
            w[j] += ((uint64_t)((mask >> (4 * j)) & 0xFu) * 0x0000200040008001ull) & 0x0001000100010001ull;
    }
    // move the fields into u32 counters (call before a field can reach 2^16)
    __device__ __forceinline__ void flush(uint32_t (&capc)[NCAP]) {
#pragma unroll
        for (int q = 0; q < NCAP; q++) capc[q] += (uint32_t)(w[q / 4] >> (16 * (q % 4))) & 0xFFFFu;
#pragma unroll
        for (int j = 0; j < (NCAP + 3) / 4; j++) w[j] = 0;
    }
};

// one survivor: its output values from the descriptor (MODE 1: index|mask only)
// A survivor's row data, loaded in one batch (6 x 16 B of its RowEnt) so that
// the loads of several survivors are in flight together.
struct RowLoad {
    uint4 h;               // w, pair_off, p, two
    ulonglong2 lam, e8bt;  // lam0, lam1 / e8, bt
    ulonglong2 hcpsi, pg;  // hc, psi / par1, gra1
    ulonglong2 optrs;      // optim1, rs
};

__device__ __forceinline__ ulonglong2 ldg_u2(const void* p) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(p));
    return make_ulonglong2(((uint64_t)x.y << 32) | x.x, ((uint64_t)x.w << 32) | x.z);
}

__device__ __forceinline__ ulonglong2 ld_u2(const void* p) {
    const uint4 x = *reinterpret_cast<const uint4*>(p);
    return make_ulonglong2(((uint64_t)x.y << 32) | x.x, ((uint64_t)x.w << 32) | x.z);
}

// SMEM: e points into the warp's shared-memory copy of the span's rows
template <bool SMEM>
__device__ __forceinline__ void load_row(const RowEnt* __restrict__ e, RowLoad& L) {
    if (SMEM) {
        L.h = *reinterpret_cast<const uint4*>(e);
        L.lam = ld_u2(&e->lam0);
        L.e8bt = ld_u2(&e->e8);
        L.hcpsi = ld_u2(&e->hc);
        L.pg = ld_u2(&e->par1);
        L.optrs = ld_u2(&e->optim1);
    } else {
        L.h = __ldg(reinterpret_cast<const uint4*>(e));
        L.lam = ldg_u2(&e->lam0);
        L.e8bt = ldg_u2(&e->e8);
        L.hcpsi = ldg_u2(&e->hc);
        L.pg = ldg_u2(&e->par1);
        L.optrs = ldg_u2(&e->optim1);
    }
}

// one survivor's output values from its descriptor, row data and pair
// (MODE 1: index|mask only)
// (k, r) = row and position in it, idx = flat index, dmask = the mask the
// stage kernel stored (INDEX only)
template <int MODE, int NCAP, bool GBS, bool STMAX>
__device__ __forceinline__ void expand_vals(const DevSpace& S, const StEnt* __restrict__ st, uint32_t k, uint32_t r,
                                            uint64_t idx, uint32_t dmask, const RowLoad& L, uint2 pr,
                                            uint64_t (&v)[8]) {
    if (MODE == 1) {
        v[0] = idx | ((uint64_t)dmask << 56);
        return;
    }
    const uint32_t sel = r & ((1u << S.lg_rcdo) - 1u);
    const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
    const uint32_t u = pr.x, p = L.h.z;
    const uint32_t n_inf = GBS ? min(p, pr.y) : p;
    const uint64_t psi = L.hcpsi.y;
    const uint64_t lam = rc ? L.lam.y : L.lam.x;
    const uint64_t mu = rc ? L.e8bt.y : 0ull;
    v[1] = dopt ? L.pg.x : 2ull * psi;
    v[2] = dopt ? L.pg.y : 4ull * psi;
    v[3] = dopt ? L.optrs.x : 12ull * psi;
    v[4] = (uint64_t)u * ((uint64_t)n_inf * lam + mu);
    v[5] = (uint64_t)u * ((uint64_t)n_inf * L.e8bt.x);
    v[6] = (uint64_t)u * L.hcpsi.x;
    v[7] = v[1] + v[2] + v[3] + v[4] + v[5] + v[6];
    if (STMAX && L.h.w) {
        const StEnt& x = st[(size_t)k << S.lg_rcdo | sel];
        const uint64_t tl = __ldg(&x.msL) + (uint64_t)u * __ldg(&x.kL);
        if (tl > v[7]) {  // the last stage decides (ties: stage 0)
            v[1] = __ldg(&x.parL);
            v[2] = __ldg(&x.graL);
            v[3] = __ldg(&x.optimL);
            v[4] = (uint64_t)u * __ldg(&x.layL);
            v[5] = 0;
            v[6] = (uint64_t)u * __ldg(&x.hcL);
            v[7] = tl;
        }
    }
    v[0] = idx | ((uint64_t)cap_mask_n<NCAP>(S, ~v[7]) << 56);
}

// Shared memory of the expand kernel: the pairs pool (when it fits) and, per
// warp, a copy of the rows its current span refers to (when they fit):
// the survivors' row and pair reads then cost no global-memory round trip.
constexpr uint32_t kSmemPairs = 2048;  // 16 KB
constexpr uint32_t kSmemRows = 24;     // per warp: 3 KB (C5: a 16-tile span touches <= 23 rows)

// the survivors [0, n) of one span, U per lane per iteration, in phases
// (descriptors, rows, pairs, values + stores) so that each phase's loads are
// in flight together.  SMEM: rows from the warp's shared copy (row k at
// srow[k - k0]); pairs: shared or global (pairs).
template <int MODE, int NCAP, bool GBS, bool STMAX, int U, bool SMEM, bool D32>
__device__ __forceinline__ void expand_span(const DevSpace& S, const RowEnt* __restrict__ rows,
                                            const RowEnt* srow, uint32_t k0, uint32_t kspan, uint64_t s0,
                                            const uint2* pairs, const StEnt* __restrict__ st,
                                            const void* __restrict__ dv, uint32_t n, uint64_t off, const Cols& cols,
                                            uint64_t capacity, CapPack<NCAP>& pk, uint32_t lane) {
    for (uint32_t i0 = 0; i0 < n; i0 += 32 * U) {
        // descriptors -> (row, position in row or index, stored mask); past the end: row k0
        uint32_t k[U], r[U], dm[U];
        uint64_t idx[U];
#pragma unroll
        for (int j = 0; j < U; j++) {
            const uint32_t i = i0 + 32 * j + lane;
            if (D32) {
                const uint32_t x = i < n ? __ldg(reinterpret_cast<const uint32_t*>(dv) + i) : 0u;
                k[j] = i < n ? kspan + ((x >> 16) & 0xFFu) : k0;
                idx[j] = s0 + (x & 0xFFFFu);
                dm[j] = x >> 24;
            } else {
                const uint64_t x = i < n ? __ldg(reinterpret_cast<const uint64_t*>(dv) + i) : ((uint64_t)k0 << 32);
                k[j] = (uint32_t)(x >> 32) & 0xFFFFFFu;
                r[j] = (uint32_t)x;
                dm[j] = (uint32_t)(x >> 56);
            }
        }
        if (SMEM) {
            // rows and pairs in shared memory: the U descriptor loads are the
            // only global round trip
#pragma unroll
            for (int j = 0; j < U; j++) {
                const bool valid = i0 + 32 * j + lane < n;
                RowLoad Lj;
                const RowEnt* e = srow + (k[j] - k0);
                if (MODE != 1) load_row<true>(e, Lj);
                else if (!D32) Lj.optrs.y = e->rs;
                uint32_t rj = r[j];
                uint64_t ij = idx[j];
                if (D32) rj = MODE != 1 && valid ? (uint32_t)(ij - Lj.optrs.y) : 0u;
                else ij = Lj.optrs.y + rj;
                const uint2 pj = MODE == 1 ? make_uint2(0, 0) : pairs[Lj.h.y + (rj >> S.lg_rcdo)];
                uint64_t v[8];
                expand_vals<MODE, NCAP, GBS, STMAX>(S, st, k[j], rj, ij, dm[j], Lj, pj, v);
                pk.add(valid ? (uint32_t)(v[0] >> 56) : 0u);
                const uint64_t o = off + i0 + 32 * j + lane;
                if (valid && o < capacity) {
                    if (MODE == 3) {
                        store_record(cols.c[0] + o * 8, v);
                    } else if (MODE == 2) {
#pragma unroll
                        for (int c = 0; c < 8; c++) cols.c[c][o] = v[c];
                    } else {
                        cols.c[0][o] = v[0];
                    }
                }
            }
        } else {
        // rows from global memory (the span's rows do not fit the shared
        // copy): one survivor at a time, descriptors already loaded
#pragma unroll
        for (int j = 0; j < U; j++) {
            const bool valid = i0 + 32 * j + lane < n;
            RowLoad Lj;
            const RowEnt* e = rows + k[j];
            if (MODE != 1) load_row<false>(e, Lj);
            else if (!D32) Lj.optrs.y = __ldg(&e->rs);
            uint32_t rj = r[j];
            uint64_t ij = idx[j];
            if (D32) rj = MODE != 1 && valid ? (uint32_t)(ij - Lj.optrs.y) : 0u;
            else ij = Lj.optrs.y + rj;
            const uint2 pj = MODE == 1 ? make_uint2(0, 0) : pairs[Lj.h.y + (rj >> S.lg_rcdo)];
            uint64_t v[8];
            expand_vals<MODE, NCAP, GBS, STMAX>(S, st, k[j], rj, ij, dm[j], Lj, pj, v);
            pk.add(valid ? (uint32_t)(v[0] >> 56) : 0u);
            const uint64_t o = off + i0 + 32 * j + lane;
            if (valid && o < capacity) {
                if (MODE == 3) {
                    store_record(cols.c[0] + o * 8, v);
                } else if (MODE == 2) {
#pragma unroll
                    for (int c = 0; c < 8; c++) cols.c[c][o] = v[c];
                } else {
                    cols.c[0][o] = v[0];
                }
            }
        }
        }
    }
}

template <int MODE, int NCAP, bool GBS, bool STMAX, int U>
__device__ __forceinline__ void expand_spans(const DevSpace& S, const RowEnt* __restrict__ rows,
                                             const StEnt* __restrict__ st, uint32_t span_len, uint32_t n_spans,
                                             const uint64_t* __restrict__ desc, bool d32,
                                             const uint2* __restrict__ span_ck, uint64_t base,
                                             const uint32_t* __restrict__ span_count,
                                             const uint64_t* __restrict__ block_off, const Cols& cols,
                                             uint64_t capacity, const uint2* pairs, RowEnt* srow,
                                             uint32_t* next_span, uint32_t (&capc)[NCAP]) {
    const uint32_t lane = threadIdx.x & 31;
    // spans are taken in order from a counter (the survivors per span vary:
    // a static assignment leaves a long tail)
    uint32_t sp = 0;
    while (true) {
        if (lane == 0) sp = atomicAdd(next_span, 1u);
        sp = __shfl_sync(0xffffffffu, sp, 0);
        if (sp >= n_spans) break;
        const uint32_t n = __ldg(span_count + sp);
        if (!n) continue;
        // output row of the span: its block's offset + the earlier spans of the block
        uint64_t off = __ldg(block_off + sp / kStageWarps);
        for (uint32_t q = sp & ~(kStageWarps - 1u); q < sp; q++) off += __ldg(span_count + q);
        // rows of the span: from its first and last survivor (index order)
        const uint2 ck = __ldg(span_ck + sp);
        const uint64_t s0 = base + (uint64_t)sp * span_len;
        const void* dv;
        uint32_t k0, k1;
        if (d32) {
            const uint32_t* d = reinterpret_cast<const uint32_t*>(desc) + (size_t)sp * span_len;
            k0 = ck.x + ((__ldg(d) >> 16) & 0xFFu);
            k1 = ck.x + ((__ldg(d + n - 1) >> 16) & 0xFFu);
            dv = d;
        } else {
            const uint64_t* d = desc + (size_t)sp * span_len;
            k0 = (uint32_t)(__ldg(d) >> 32) & 0xFFFFFFu;
            k1 = (uint32_t)(__ldg(d + n - 1) >> 32) & 0xFFFFFFu;
            dv = d;
        }
        CapPack<NCAP> pk;  // <= span_len / 32 survivors per lane per span: fits 16 bits
#define ME_SPAN(SM, D)                                                                                           \
    expand_span<MODE, NCAP, GBS, STMAX, U, SM, D>(S, rows, srow, k0, ck.x, s0, pairs, st, dv, n, off, cols, capacity, \
                                                  pk, lane)
        const bool smem = k1 - k0 < kSmemRows && !(MODE == 1 && d32);
        if (smem) {
            __syncwarp();  // the previous span's readers are done with srow
            const uint4* src = reinterpret_cast<const uint4*>(rows + k0);
            uint4* dst = reinterpret_cast<uint4*>(srow);
            for (uint32_t c = lane; c < (k1 - k0 + 1) * (sizeof(RowEnt) / 16); c += 32) dst[c] = __ldg(src + c);
            __syncwarp();
            if (d32) ME_SPAN(true, true);
            else ME_SPAN(true, false);
        } else {
            if (d32) ME_SPAN(false, true);
            else ME_SPAN(false, false);
        }
#undef ME_SPAN
        pk.flush(capc);
    }
}

// stats[1 + j] += survivors for capacity j (one atomic per block and capacity)
template <int MODE, int NCAP, int U>
__global__ void __launch_bounds__(kThreads, 2) expand_kernel(const DevSpace S, const RowEnt* __restrict__ rows,
                                                             const StEnt* __restrict__ st, const uint32_t span_len,
                                                             const uint32_t n_spans, const uint64_t* __restrict__ desc,
                                                             const uint32_t d32, const uint2* __restrict__ span_ck,
                                                             const uint64_t base,
                                                             const uint32_t* __restrict__ span_count,
                                                             const uint64_t* __restrict__ block_off, const Cols cols,
                                                             const uint64_t capacity, uint64_t* __restrict__ stats,
                                                             uint32_t* __restrict__ next_span) {
    __shared__ uint32_t s_cap[NCAP];
    __shared__ uint2 s_pairs[kSmemPairs];
    __shared__ __align__(16) RowEnt s_rows[kWarpsPerBlock][kSmemRows];
    if (threadIdx.x < NCAP) s_cap[threadIdx.x] = 0;
    const bool pairs_smem = S.n_pairs <= kSmemPairs;
    if (pairs_smem)
        for (uint32_t i = threadIdx.x; i < S.n_pairs; i += blockDim.x)
            s_pairs[i] = __ldg(reinterpret_cast<const uint2*>(S.pairs) + i);
    __syncthreads();
    const uint2* pairs = pairs_smem ? s_pairs : reinterpret_cast<const uint2*>(S.pairs);
    RowEnt* srow = s_rows[threadIdx.x >> 5];
    uint32_t capc[NCAP];
#pragma unroll
    for (int q = 0; q < NCAP; q++) capc[q] = 0;
#define ME_EXPAND(GBS, STMAX)                                                                              \
    expand_spans<MODE, NCAP, GBS, STMAX, U>(S, rows, st, span_len, n_spans, desc, d32 != 0, span_ck, base,      \
                                            span_count, block_off, cols, capacity, pairs, srow, next_span, capc)
    if (S.stage_max) {
        if (S.gbs_mode) ME_EXPAND(true, true);
        else ME_EXPAND(false, true);
    } else {
        if (S.gbs_mode) ME_EXPAND(true, false);
        else ME_EXPAND(false, false);
    }
#undef ME_EXPAND
#pragma unroll
    for (int q = 0; q < NCAP; q++) {
        const uint32_t c = __reduce_add_sync(0xffffffffu, capc[q]);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(s_cap + q, c);
    }
    __syncthreads();
    if (threadIdx.x < NCAP && s_cap[threadIdx.x])
        atomicAdd((unsigned long long*)(stats + 1 + threadIdx.x), (unsigned long long)s_cap[threadIdx.x]);
}

uint32_t ncap_pad(uint32_t n_cap) { return n_cap <= 1 ? 1 : n_cap <= 2 ? 2 : n_cap <= 4 ? 4 : 8; }

template <int MODE, int U>
void* expand_fn_(uint32_t n_cap) {
    switch (ncap_pad(n_cap)) {
        case 1: return reinterpret_cast<void*>(&expand_kernel<MODE, 1, U>);
        case 2: return reinterpret_cast<void*>(&expand_kernel<MODE, 2, U>);
        case 4: return reinterpret_cast<void*>(&expand_kernel<MODE, 4, U>);
        default: return reinterpret_cast<void*>(&expand_kernel<MODE, 8, U>);
    }
}
// u: survivors per lane per iteration (2 or 4; ME_EXPAND_U)
template <int U>
void* expand_fn_u(me_out_mode mode, uint32_t n_cap) {
    return mode == ME_OUT_RECORDS ? expand_fn_<3, U>(n_cap)
                                  : mode == ME_OUT_FULL ? expand_fn_<2, U>(n_cap) : expand_fn_<1, U>(n_cap);
}
int g_expand_u = 2;
void* expand_fn(me_out_mode mode, uint32_t n_cap) {
    return g_expand_u >= 4 ? expand_fn_u<4>(mode, n_cap) : expand_fn_u<2>(mode, n_cap);
}
template <bool MASK>
void* stage_fn_(uint32_t n_cap) {
    switch (ncap_pad(n_cap)) {
        case 1: return reinterpret_cast<void*>(&stage_kernel<1, MASK>);
        case 2: return reinterpret_cast<void*>(&stage_kernel<2, MASK>);
        case 4: return reinterpret_cast<void*>(&stage_kernel<4, MASK>);
        default: return reinterpret_cast<void*>(&stage_kernel<8, MASK>);
    }
}
void* stage_fn(uint32_t n_cap, bool mask) { return mask ? stage_fn_<true>(n_cap) : stage_fn_<false>(n_cap); }

}  // namespace

int expand_blocks_per_sm(me_out_mode mode, uint32_t n_cap) {
    if (const char* e = getenv("ME_EXPAND_U")) g_expand_u = atoi(e);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, expand_fn(mode, n_cap), kThreads, 0) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_rows(const DevSpace& S, uint64_t g0, uint32_t n_rows, uint32_t seg_lo, uint32_t n_seg_sub,
                        uint64_t lo, uint64_t hi, uint32_t span_tiles, RowEnt* rows, StEnt* st, uint2* span_ck,
                        cudaStream_t stream) {
    const uint64_t base = lo & ~31ull;
    const uint32_t n_tiles = n_tiles_of(lo, hi);
    const uint32_t n_spans = (n_tiles + span_tiles - 1) / span_tiles;
    const uint32_t blocks = (n_rows + 255) / 256;
    row_kernel<<<blocks ? blocks : 1, 256, 0, stream>>>(S, g0, n_rows, seg_lo, n_seg_sub, base, hi,
                                                        span_tiles * kTile, n_spans, rows, st, span_ck);
    return cudaGetLastError();
}

cudaError_t launch_stage(const DevSpace& S, const RowEnt* rows, const StEnt* st, uint64_t lo, uint64_t hi,
                         uint32_t span_tiles, const uint2* span_ck, uint64_t* desc, uint32_t d32, uint32_t* span_count,
                         uint32_t* block_count, me_out_mode mode, cudaStream_t stream) {
    const uint32_t n_tiles = n_tiles_of(lo, hi);
    const uint32_t n_spans = (n_tiles + span_tiles - 1) / span_tiles;
    void* args[] = {(void*)&S,          (void*)&rows,    (void*)&st,      (void*)&lo,   (void*)&hi,
                    (void*)&span_tiles, (void*)&n_spans, (void*)&span_ck, (void*)&desc, (void*)&d32,
                    (void*)&span_count, (void*)&block_count};
    return cudaLaunchKernel(stage_fn(S.n_cap, mode == ME_OUT_INDEX), dim3((n_spans + kStageWarps - 1) / kStageWarps),
                            dim3(kStageWarps * 32), args, 0, stream);
}

cudaError_t launch_expand(const DevSpace& S, const RowEnt* rows, const StEnt* st, uint64_t lo, uint64_t hi,
                          uint32_t span_tiles, const uint64_t* desc, uint32_t d32, const uint2* span_ck,
                          const uint32_t* span_count,
                          const uint64_t* block_off, me_out_mode mode, Cols cols, uint64_t capacity, uint64_t* stats,
                          uint32_t n_blocks, uint32_t* next_span, cudaStream_t stream) {
    const uint32_t n_tiles = n_tiles_of(lo, hi);
    const uint32_t n_spans = (n_tiles + span_tiles - 1) / span_tiles;
    const uint32_t span_len = span_tiles * kTile;
    const uint32_t need = (n_spans + kWarpsPerBlock - 1) / kWarpsPerBlock;
    if (n_blocks > need) n_blocks = need ? need : 1;
    const uint64_t base = lo & ~31ull;
    void* args[] = {(void*)&S,    (void*)&rows,    (void*)&st,   (void*)&span_len,   (void*)&n_spans,
                    (void*)&desc, (void*)&d32,     (void*)&span_ck, (void*)&base,   (void*)&span_count,
                    (void*)&block_off, (void*)&cols, (void*)&capacity, (void*)&stats, (void*)&next_span};
    cudaError_t ce = cudaMemsetAsync(next_span, 0, 4, stream);
    if (ce != cudaSuccess) return ce;
    return cudaLaunchKernel(expand_fn(mode, S.n_cap), dim3(n_blocks), dim3(kThreads), args, 0, stream);
}

}  // namespace me
