// me_kernels.cu -- the sweep kernels (sm_100a).
//
// The index range of one pass is cut into tiles of kTile = 512 consecutive
// indices (16 rounds of 32).  A warp evaluates a round as 32 consecutive
// indices, lane l taking index base + l, so a warp ballot yields the survivors
// of a round in index order.  Each lane keeps an odometer over the canonical
// enumeration (segment -> tuple row -> position in row); rows are entered with
// all their estimator coefficients precomputed (LaneRow), so the per-config work
// is one pair load, one u32 x u64 multiply-add and n_cap u64 compares.
//
// Passes:
//  count  warps walk contiguous spans of whole tiles (one binary search per
//         lane per span) and store, per tile, its survivor count and the
//         walker state of the tile's first index (a checkpoint);
//  scan   one block turns the tile counts into output offsets (adding the
//         running total of earlier sub-ranges) and accumulates the totals;
//  write  warps take tiles in grid-stride order -- at any moment the grid
//         writes one compact window of the output columns, which keeps the
//         DRAM write stream local -- restore the walker from the tile's
//         checkpoint and store the survivors' columns (structure of arrays;
//         the stores of a round are contiguous across the surviving lanes).
#include <cuda_runtime.h>

#include "me_kernels.cuh"

namespace me {

namespace {

__device__ __forceinline__ uint32_t upper_bound_u64(const uint64_t* __restrict__ a, uint32_t n,
                                                    uint64_t x) {
    // first i in [0, n) with a[i] > x (n if none)
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// Per-lane row coefficients.  Lanes advance by 32 and every row length is a
// multiple of the (rc, do) digit count (1, 2 or 4), so a lane's (rc, do) digits
// never change along its walk: the rc / do selections of RowCoef are made once
// per row.  The sweep evaluates the complement of the total,
//   ~total = ~ms + u * (-(n_inf * a + b))      (mod 2^64; n_inf = p in paper mode)
// so each capacity test is one carry chain (le_carry below).
struct LaneRow {
    uint64_t nms;       // ~(params + grads + optim) for this lane's do
    uint64_t na, nb;    // -a, -b: per-token activation bytes = n_inf * a + b (this lane's rc)
    uint64_t nkp;       // -(p * a + b) (paper mode: n_inf = p)
    uint64_t par, gra;  // weight / gradient bytes for this lane's do (and the ZeRO stage)
    uint64_t optim;     // optimizer bytes for this lane's do
    uint64_t lam, mu;   // per-token layer bytes = n_inf * lam + mu
    uint64_t e8, hc;    // per-token embedding bytes = n_inf * e8; head bytes = hc
    uint64_t lay, emb;  // paper mode: p * lam + mu, p * e8
    uint32_t p;
    // NEXT-1 (stage_max): the last pipeline stage (p >= 2), one microbatch in
    // flight: total = msL + u * kL, layers = u * layL, head = u * hcL
    bool two;
    uint64_t nmsL, nkL, parL, graL, optimL, layL, hcL;
};

__device__ __forceinline__ void make_lane_row(const DevModel& M, uint32_t t, uint32_t c, uint32_t p, uint32_t d,
                                              uint32_t rc, uint32_t dopt, bool stage_max, uint32_t zero,
                                              LaneRow& L) {
    RowCoef R;
    const uint32_t L0 = p == 1 ? M.layers : div_u32(M.layers + p - 1, p);
    make_row(M, t, c, p, d, L0, zero, R);
    L.two = stage_max && p >= 2;
    if (L.two) {
        // the last stage holds floor((L - L0) / (p - 1)) layers
        const uint32_t Ll = (M.layers - L0) / (p - 1);
        const TermsT<uint64_t> T = stage_terms<uint64_t>(M, t, c, d, false, true, Ll, 1u, 1u, rc, dopt, zero);
        L.parL = T.params;
        L.graL = T.grads;
        L.optimL = T.optim;
        L.nmsL = ~(T.params + T.grads + T.optim);
        L.layL = T.layers;
        L.hcL = T.head;
        L.nkL = 0ull - (T.layers + T.head);
    }
    const uint64_t a = (rc ? R.lam1 : R.lam0) + R.e8;
    const uint64_t b = rc ? R.bt + R.hc : R.hc;
    L.nms = ~(dopt ? R.ms1 : R.ms0);
    L.na = 0ull - a;
    L.nb = 0ull - b;
    L.nkp = 0ull - ((uint64_t)p * a + b);
    L.par = dopt ? R.par1 : 2ull * R.psi;
    L.gra = dopt ? R.gra1 : 4ull * R.psi;
    L.optim = dopt ? R.optim1 : 12ull * R.psi;
    L.lam = rc ? R.lam1 : R.lam0;
    L.mu = rc ? R.bt : 0ull;
    L.e8 = R.e8;
    L.hc = R.hc;
    L.lay = (uint64_t)p * L.lam + L.mu;
    L.emb = (uint64_t)p * R.e8;
    L.p = p;
}

struct Walker {
    uint32_t seg, j, jend, r, w;
    const uint2* pp;    // this lane's current (b, s) pair
    uint32_t rc, dopt;  // this lane's innermost digits (constant along its walk)
    DevModel M;
    LaneRow L;

    __device__ __forceinline__ void enter_segment(const DevSpace& S, uint32_t s) {
        seg = s;
        const uint32_t m = s / S.n_world, n = s - m * S.n_world;
        const uint4 m0 = __ldg(reinterpret_cast<const uint4*>(S.models + m));
        const uint4 m1 = __ldg(reinterpret_cast<const uint4*>(S.models + m) + 1);
        M = DevModel{m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, 0u};
        const uint32_t cls = __ldg(S.model_class + m);
        j = __ldg(S.list_off + cls * S.n_world + n);
        jend = __ldg(S.list_off + cls * S.n_world + n + 1);
    }

    __device__ __forceinline__ void set_row(const DevSpace& S) {
        const uint32_t tid = __ldg(S.list_tuple + j);
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(S.tuples + tid));      // t c p d
        const uint2 b = __ldg(reinterpret_cast<const uint2*>(S.tuples + tid) + 2);  // w pair_off
        w = b.x;
        pp = reinterpret_cast<const uint2*>(S.pairs) + b.y + (r >> S.lg_rcdo);
        make_lane_row(M, a.x, a.y, a.z, a.w, rc, dopt, S.stage_max != 0, S.zero_stage, L);
    }

    __device__ __forceinline__ void set_digits(const DevSpace& S) {
        const uint32_t sel = r & ((1u << S.lg_rcdo) - 1u);
        rc = (S.rcdo_rc >> sel) & 1u;
        dopt = (S.rcdo_do >> sel) & 1u;
    }

    // leave the current row (r >= w): next tuple of the list, next non-empty
    // segment when the list is exhausted
    __device__ __forceinline__ void next_row(const DevSpace& S) {
        r -= w;
        ++j;
        if (j == jend) {
            uint32_t s = seg;
            do {
                ++s;
            } while (__ldg(S.seg_prefix + s + 1) == __ldg(S.seg_prefix + s));
            enter_segment(S, s);
        }
        set_row(S);
    }

    // position on absolute index pos (< total) by binary search
    __device__ __forceinline__ void seek(const DevSpace& S, uint64_t pos) {
        const uint32_t s = upper_bound_u64(S.seg_prefix, S.n_seg + 1, pos) - 1;
        enter_segment(S, s);
        const uint64_t within = pos - __ldg(S.seg_prefix + s);
        const uint32_t k = upper_bound_u64(S.list_prefix + j, jend - j, within) - 1;
        j += k;
        r = (uint32_t)(within - __ldg(S.list_prefix + j));
        set_digits(S);
        set_row(S);
    }

    // position on checkpoint (state of index x) + lane
    __device__ __forceinline__ void restore(const DevSpace& S, uint4 ck, uint32_t lane) {
        enter_segment(S, ck.x);
        j = ck.y;
        r = ck.z + lane;
        set_digits(S);  // row lengths are multiples of the digit count
        set_row(S);
        while (r >= w) next_row(S);
    }

    // move forward by 32 indices (the caller guarantees the target exists)
    __device__ __forceinline__ void advance32(const DevSpace& S, uint32_t pstep) {
        r += 32;
        if (r < w) {
            pp += pstep;
        } else {
            do {
                next_row(S);
            } while (r >= w);
        }
    }
};

// total <= thr  <=>  the 64-bit sum thr1 + ntot carries out, with thr1 = thr + 1
// and ntot = ~total = 2^64 - 1 - total.  Two chained 32-bit adds produce the
// carry; le_count returns acc + carry, le_shift 2 * acc + carry (a capacity
// mask is built from the last slot down).
__device__ __forceinline__ uint32_t le_count(uint32_t acc, uint64_t ntot, uint64_t thr1) {
    asm("{\n\t.reg .u32 t;\n\t"
        "add.cc.u32 t, %1, %2;\n\t"
        "addc.cc.u32 t, %3, %4;\n\t"
        "addc.u32 %0, %0, 0;\n\t}"
        : "+r"(acc)
        : "r"((uint32_t)ntot), "r"((uint32_t)thr1), "r"((uint32_t)(ntot >> 32)), "r"((uint32_t)(thr1 >> 32)));
    return acc;
}
__device__ __forceinline__ uint32_t le_shift(uint32_t acc, uint64_t ntot, uint64_t thr1) {
    asm("{\n\t.reg .u32 t;\n\t"
        "add.cc.u32 t, %1, %2;\n\t"
        "addc.cc.u32 t, %3, %4;\n\t"
        "addc.u32 %0, %0, %0;\n\t}"
        : "+r"(acc)
        : "r"((uint32_t)ntot), "r"((uint32_t)thr1), "r"((uint32_t)(ntot >> 32)), "r"((uint32_t)(thr1 >> 32)));
    return acc;
}

// capacity mask of a config from ntot = ~total: bit q = (total <= thr_q)
template <int NCAP>
__device__ __forceinline__ uint32_t cap_mask(const DevSpace& S, uint64_t ntot) {
    uint32_t mask = 0;
#pragma unroll
    for (int q = NCAP - 1; q >= 0; q--) mask = le_shift(mask, ntot, S.thr1[q]);
    return mask;
}

// per-lane survivor counters per capacity (count pass)
template <int NCAP>
struct CapAcc {
    uint32_t capc[NCAP];
    __device__ __forceinline__ CapAcc() {
#pragma unroll
        for (int q = 0; q < NCAP; q++) capc[q] = 0;
    }
};

// Evaluate one tile's rounds starting at the walker's position (lane's index
// = pos).  RAGGED: the tile is cut by lo/hi (first or last tile of a range).
// GBS: a global batch bounds the in-flight microbatches (R17).  STMAX: the
// largest pipeline stage decides (NEXT-1; middle stages never exceed stage 0,
// so the larger of stage 0 and the last stage is the maximum).  Leaves the
// walker on the first index after the tile when `advance_out`; returns the
// output row after the tile's survivors (write modes).
//
// Write pass stores: each surviving lane stores its 8-byte value of every
// column at its row; a round's rows are contiguous.  (Measured alternatives on
// B200, scripts/storebench.cu and DESIGN.md §6: shared-memory staging into
// aligned full-line stores lifts the store pattern itself from ~4.1 to ~5.7
// TB/s but costs more issue slots than it saves in this kernel.)
template <int MODE, int NCAP, bool RAGGED, bool GBS, bool STMAX>
__device__ __forceinline__ uint64_t run_tile(const DevSpace& S, Walker& W, uint64_t pos, uint64_t lo,
                                             uint64_t hi, uint32_t rounds, uint32_t lane, CapAcc<NCAP>& acc,
                                             uint64_t out, const Cols& cols, uint64_t capacity, bool advance_out) {
    constexpr int NC = MODE >= 2 ? 8 : 1;
    constexpr bool PREFETCH = MODE != 0;  // the write pass hides the pair load behind a round
    const uint32_t pstep = 32u >> S.lg_rcdo;
    uint2 pr = __ldg(W.pp);
    for (uint32_t it = 0; it < rounds; it++, pos += 32) {
        const bool more = (it + 1 < rounds) || advance_out;
        const bool in_row = W.r + 32 < W.w;
        uint2 prn = pr;
        if (PREFETCH && in_row && more) prn = __ldg(W.pp + pstep);  // next round's pair, issued early

        const uint32_t u = pr.x;
        const uint32_t n_inf = GBS ? min(W.L.p, pr.y) : W.L.p;
        const uint64_t nK = GBS ? (uint64_t)n_inf * W.L.na + W.L.nb : W.L.nkp;
        uint64_t ntot = W.L.nms + (uint64_t)u * nK;  // ~total
        bool last = false;
        if (STMAX && W.L.two) {
            const uint64_t ntl = W.L.nmsL + (uint64_t)u * W.L.nkL;
            last = ntl < ntot;  // the last stage's total is larger
            ntot = last ? ntl : ntot;
        }
        const bool act = !RAGGED || (pos >= lo && pos < hi);
        if (MODE == 0) {
            // counts only: survivors per capacity in count-slot order (slot 0
            // = the largest threshold: its count is the survivor count)
            if (act) {
#pragma unroll
                for (int q = 0; q < NCAP; q++) acc.capc[q] = le_count(acc.capc[q], ntot, S.thr1c[q]);
            }
        } else {
            const uint32_t mask = act ? cap_mask<NCAP>(S, ntot) : 0u;
            const uint32_t ballot = __ballot_sync(0xffffffffu, mask != 0);
            if (mask) {
                const uint64_t o = out + __popc(ballot & ((1u << lane) - 1u));
                if (o < capacity) {
                    uint64_t v[NC];
                    v[0] = pos | ((uint64_t)mask << 56);
                    if (MODE >= 2) {
                        v[1] = STMAX && last ? W.L.parL : W.L.par;
                        v[2] = STMAX && last ? W.L.graL : W.L.gra;
                        v[3] = STMAX && last ? W.L.optimL : W.L.optim;
                        const uint64_t lay = GBS ? (uint64_t)n_inf * W.L.lam + W.L.mu : W.L.lay;
                        const uint64_t emb = GBS ? (uint64_t)n_inf * W.L.e8 : W.L.emb;
                        v[4] = (uint64_t)u * (STMAX && last ? W.L.layL : lay);
                        v[5] = STMAX && last ? 0ull : (uint64_t)u * emb;
                        v[6] = (uint64_t)u * (STMAX && last ? W.L.hcL : W.L.hc);
                        v[7] = ~ntot;
                    }
                    if (MODE == 3) {
                        // records (array of structures): one 64-byte row, two 32-byte stores
                        uint64_t* q = cols.c[0] + o * 8;
                        asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(q), "l"(v[0]), "l"(v[1]),
                                     "l"(v[2]), "l"(v[3])
                                     : "memory");
                        asm volatile("st.global.v4.u64 [%0+32], {%1, %2, %3, %4};" ::"l"(q), "l"(v[4]), "l"(v[5]),
                                     "l"(v[6]), "l"(v[7])
                                     : "memory");
                    } else {
#pragma unroll
                        for (int c = 0; c < NC; c++) cols.c[c][o] = v[c];
                    }
                }
            }
            out += __popc(ballot);
        }
        if (more && (!RAGGED || pos + 32 < hi)) {
            if (in_row) {
                W.r += 32;
                W.pp += pstep;
                pr = PREFETCH ? prn : __ldg(W.pp);
            } else {
                W.advance32(S, pstep);
                pr = __ldg(W.pp);
            }
        }
    }
    return out;
}

struct TileGeom {
    uint64_t lo, hi, base;  // range [lo, hi); tiles start at base = lo & ~31
    uint32_t n_tiles;
    __device__ __forceinline__ uint64_t start(uint32_t t) const { return base + (uint64_t)t * kTile; }
    __device__ __forceinline__ bool ragged(uint32_t t) const {
        return (t == 0 && lo != base) || start(t) + kTile > hi;
    }
    __device__ __forceinline__ uint32_t rounds(uint32_t t) const {
        const uint64_t e = start(t) + kTile < hi ? start(t) + kTile : hi;
        return (uint32_t)((e - start(t) + 31) / 32);
    }
};

__device__ __forceinline__ TileGeom geom(uint64_t lo, uint64_t hi) {
    TileGeom g;
    g.lo = lo;
    g.hi = hi;
    g.base = lo & ~31ull;
    g.n_tiles = (uint32_t)((hi - g.base + kTile - 1) / kTile);
    return g;
}

// count pass over span s = tiles [t0, t1): per tile its checkpoint
// {seg, j, r, s}, its survivor count and its first survivor's rank inside the
// span; returns the span total
template <int NCAP, bool GBS, bool STMAX>
__device__ __forceinline__ uint32_t count_span(const DevSpace& S, const TileGeom& G, uint32_t s, uint32_t t0,
                                               uint32_t t1, uint32_t lane, uint32_t* __restrict__ tile_rel,
                                               uint32_t* __restrict__ tile_cnt, uint4* __restrict__ tile_ck,
                                               CapAcc<NCAP>& acc) {
    Walker W;
    // a lane past the end of the range only takes part in the warp reductions:
    // park it on the last index (its own positions stay inactive)
    const uint64_t p0 = G.start(t0) + lane;
    W.seek(S, p0 < G.hi ? p0 : G.hi - 1);
    uint32_t run = 0, prev = 0;
    for (uint32_t t = t0; t < t1; t++) {
        const uint64_t ts = G.start(t);
        if (lane == 0) {  // lane 0 is at the tile's first index
            tile_ck[t] = make_uint4(W.seg, W.j, W.r, s);
            tile_rel[t] = run;
        }
        const bool last = t + 1 == t1;
        if (G.ragged(t))
            run_tile<0, NCAP, true, GBS, STMAX>(S, W, ts + lane, G.lo, G.hi, G.rounds(t), lane, acc, 0, Cols{},
                                                      0, !last);
        else
            run_tile<0, NCAP, false, GBS, STMAX>(S, W, ts + lane, G.lo, G.hi, kTileRounds, lane, acc, 0,
                                                       Cols{}, 0, !last);
        // survivors = this tile's increase of the lane counter of count slot 0
        const uint32_t cur = acc.capc[0];
        const uint32_t cnt = __reduce_add_sync(0xffffffffu, cur - prev);
        prev = cur;
        if (lane == 0) tile_cnt[t] = cnt;
        run += cnt;
    }
    return run;
}

template <int NCAP>
__global__ void __launch_bounds__(kThreads, 3) count_kernel(const DevSpace S, const uint64_t lo, const uint64_t hi,
                                                            const uint32_t n_spans, uint32_t* __restrict__ tile_rel,
                                                            uint32_t* __restrict__ tile_cnt,
                                                            uint4* __restrict__ tile_ck,
                                                            uint32_t* __restrict__ span_count,
                                                            uint32_t* __restrict__ span_caps) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t n_warps = gridDim.x * kWarpsPerBlock;
    const TileGeom G = geom(lo, hi);
    for (uint32_t s = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); s < n_spans; s += n_warps) {
        const uint32_t t0 = (uint32_t)((uint64_t)G.n_tiles * s / n_spans);
        const uint32_t t1 = (uint32_t)((uint64_t)G.n_tiles * (s + 1) / n_spans);
        CapAcc<NCAP> acc;
        uint32_t n = 0;
        if (t0 < t1) {
            if (S.stage_max) {
                if (S.gbs_mode) n = count_span<NCAP, true, true>(S, G, s, t0, t1, lane, tile_rel, tile_cnt, tile_ck, acc);
                else n = count_span<NCAP, false, true>(S, G, s, t0, t1, lane, tile_rel, tile_cnt, tile_ck, acc);
            } else {
                if (S.gbs_mode) n = count_span<NCAP, true, false>(S, G, s, t0, t1, lane, tile_rel, tile_cnt, tile_ck, acc);
                else n = count_span<NCAP, false, false>(S, G, s, t0, t1, lane, tile_rel, tile_cnt, tile_ck, acc);
            }
        }
        if (lane == 0) span_count[s] = n;
#pragma unroll
        for (int q = 0; q < NCAP; q++) {
            const uint32_t c = __reduce_add_sync(0xffffffffu, acc.capc[q]);
            if (lane == 0) span_caps[(size_t)s * NCAP + S.cslot[q]] = c;
        }
    }
}

template <int MODE, int NCAP, bool GBS, bool STMAX>
__device__ __forceinline__ void write_tile(const DevSpace& S, const TileGeom& G, Walker& W, uint32_t t, uint64_t pos,
                                           uint32_t lane, uint64_t out, const Cols& cols, uint64_t capacity) {
    CapAcc<NCAP> none;
    if (G.ragged(t))
        run_tile<MODE, NCAP, true, GBS, STMAX>(S, W, pos, G.lo, G.hi, G.rounds(t), lane, none, out, cols, capacity,
                                               false);
    else
        run_tile<MODE, NCAP, false, GBS, STMAX>(S, W, pos, G.lo, G.hi, kTileRounds, lane, none, out, cols, capacity,
                                                false);
}

// write pass: tiles in grid-stride order (at any moment the grid writes one
// compact window of the output columns)
template <int MODE, int NCAP>
__global__ void __launch_bounds__(kThreads, MODE == 3 ? 2 : 3) write_kernel(const DevSpace S, const uint64_t lo, const uint64_t hi,
                                                            const uint4* __restrict__ tile_ck,
                                                            const uint32_t* __restrict__ tile_rel,
                                                            const uint32_t* __restrict__ tile_cnt,
                                                            const uint64_t* __restrict__ span_off, const Cols cols,
                                                            const uint64_t capacity) {
    const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint32_t n_warps = gridDim.x * kWarpsPerBlock;
    const TileGeom G = geom(lo, hi);
    for (uint32_t t = blockIdx.x * kWarpsPerBlock + wid; t < G.n_tiles; t += n_warps) {
        if (__ldg(tile_cnt + t) == 0) continue;  // no survivor: nothing to write
        const uint64_t ts = G.start(t);
        const uint64_t pos = ts + lane;
        const uint4 ck = __ldg(tile_ck + t);
        const uint64_t out = __ldg(span_off + ck.w) + __ldg(tile_rel + t);
        Walker W;
        // a lane past the end of the range is parked on the last index: it
        // takes part in the ballots with inactive positions
        W.restore(S, ck, pos < hi ? lane : (uint32_t)(hi - 1 - ts));
        if (S.stage_max) {
            if (S.gbs_mode) write_tile<MODE, NCAP, true, true>(S, G, W, t, pos, lane, out, cols, capacity);
            else write_tile<MODE, NCAP, false, true>(S, G, W, t, pos, lane, out, cols, capacity);
        } else {
            if (S.gbs_mode) write_tile<MODE, NCAP, true, false>(S, G, W, t, pos, lane, out, cols, capacity);
            else write_tile<MODE, NCAP, false, false>(S, G, W, t, pos, lane, out, cols, capacity);
        }
    }
}

// one block: exclusive scan of the span counts into u64 offsets starting at
// the running total stats[0]; stats[0] and stats[1 + q] accumulate the totals
// of this sub-range
__global__ void __launch_bounds__(1024) scan_kernel(const uint32_t* __restrict__ counts, uint32_t n,
                                                    const uint32_t* __restrict__ span_caps, uint32_t n_spans,
                                                    uint32_t ncap_stride, uint32_t n_cap,
                                                    uint64_t* __restrict__ offs, uint64_t* __restrict__ stats) {
    __shared__ uint64_t s_warp[32];
    __shared__ uint64_t s_caps[8][32];
    __shared__ uint64_t s_base;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid == 0) s_base = stats[0];
    const uint32_t chunk = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(n, tid * chunk), hi = min(n, lo + chunk);
    uint64_t sum = 0;
    for (uint32_t i = lo; i < hi; i++) sum += counts[i];
    uint64_t caps[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t s = tid; s < n_spans; s += blockDim.x)
        for (uint32_t q = 0; q < n_cap; q++) caps[q] += span_caps[(size_t)s * ncap_stride + q];
    uint64_t inc = sum;  // inclusive warp scan
    for (int o = 1; o < 32; o <<= 1) {
        uint64_t v = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += v;
    }
    if (lane == 31) s_warp[wid] = inc;
    for (uint32_t q = 0; q < n_cap; q++) {
        uint64_t c = caps[q];
        for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
        if (lane == 0) s_caps[q][wid] = c;
    }
    __syncthreads();
    const uint64_t base = s_base;
    if (wid == 0) {
        const uint32_t nw = blockDim.x >> 5;
        uint64_t v = lane < nw ? s_warp[lane] : 0;
        uint64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane < nw) s_warp[lane] = x - v;  // exclusive
        if (lane == 31) stats[0] = base + x;
        for (uint32_t q = 0; q < n_cap; q++) {
            uint64_t c = lane < nw ? s_caps[q][lane] : 0;
            for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
            if (lane == 0) stats[1 + q] += c;
        }
    }
    __syncthreads();
    uint64_t run = base + s_warp[wid] + inc - sum;
    for (uint32_t i = lo; i < hi; i++) {
        offs[i] = run;
        run += counts[i];
    }
}

// ---- single configurations ----------------------------------------------
__device__ int estimate_one(const me_model& Min, const me_parallel& P, me_breakdown& out) {
    const me_model& M = Min;
    if (!M.hidden || !M.ffn_hidden || !M.layers || !M.heads || !M.kv_heads || !M.vocab)
        return ME_EINVAL;
    if (M.heads % M.kv_heads || M.hidden % M.heads) return ME_EINVAL;
    if (!P.dp || !P.tp || !P.pp || !P.cp || !P.mbs || !P.seq || P.zero_stage > 3) return ME_EINVAL;
    const uint32_t t = P.tp, c = P.cp, p = P.pp, d = P.dp, L = M.layers;
    if (M.kv_heads % t || M.vocab % t || M.ffn_hidden % t) return ME_EDIV;  // R10
    if (P.seq % c) return ME_EDIV;
    if (p > L) return ME_EDIV;
    uint32_t L0;
    if (P.first_stage_layers) {
        L0 = P.first_stage_layers;
        if (p == 1 ? (L0 != L) : (L0 > L - (p - 1))) return ME_EDIV;
    } else {
        if (!P.allow_uneven_pp && L % p) return ME_EDIV;
        L0 = first_stage_layers_auto(L, p);
    }
    if (P.gbs && P.gbs % ((uint64_t)d * P.mbs)) return ME_EDIV;
    if ((uint64_t)(P.seq / c) * P.mbs > 0xFFFFFFFFull) return ME_EOVERFLOW;
    const uint32_t u = (P.seq / c) * P.mbs;
    const uint32_t m = P.gbs ? (uint32_t)(P.gbs / ((uint64_t)d * P.mbs)) : 0xFFFFFFFFu;
    // exact shadow in 128 bits for the overflow verdict; the values returned
    // come from the same u64 code the sweep runs
    const DevModel DM = dev_model(M);
    RowCoefT<unsigned __int128> W;
    make_row(DM, t, c, p, d, L0, (uint32_t)P.zero_stage, W);
    const TermsT<unsigned __int128> T2 = config_terms(W, u, m, P.recompute ? 1u : 0u, P.dist_opt ? 1u : 0u);
    const unsigned __int128 lim = (unsigned __int128)1 << 63;
    if (W.psi >= lim || W.ms0 >= lim || T2.total >= lim) return ME_EOVERFLOW;
    RowCoef R;
    make_row(DM, t, c, p, d, L0, (uint32_t)P.zero_stage, R);
    const TermsT<uint64_t> T = config_terms(R, u, m, P.recompute ? 1u : 0u, P.dist_opt ? 1u : 0u);
    out.params = T.params;
    out.grads = T.grads;
    out.optim = T.optim;
    out.act_layers = T.layers;
    out.act_embed = T.embed;
    out.act_head = T.head;
    out.total = T.total;
    return ME_OK;
}

// NEXT-1: stage `stage` of one configuration, or the largest stage (the first
// of equal totals) when stage == 0xFFFFFFFF
__device__ int estimate_stage_one(const me_model& M, const me_parallel& P, uint32_t stage, me_breakdown& out,
                                  uint32_t& which) {
    me_breakdown b0;
    int st = estimate_one(M, P, b0);  // preconditions, overflow of stage 0
    if (st) return st;
    const uint32_t t = P.tp, c = P.cp, p = P.pp, d = P.dp, L = M.layers;
    if (stage != 0xFFFFFFFFu && stage >= p) return ME_EINVAL;
    const uint32_t L0 = P.first_stage_layers ? P.first_stage_layers : first_stage_layers_auto(L, p);
    const uint32_t u = (P.seq / c) * P.mbs;
    const uint64_t m = P.gbs ? P.gbs / ((uint64_t)d * P.mbs) : 0xFFFFFFFFull;
    const DevModel DM = dev_model(M);
    const unsigned __int128 lim = (unsigned __int128)1 << 63;
    uint32_t lo = stage == 0xFFFFFFFFu ? 0 : stage, hi = stage == 0xFFFFFFFFu ? p : stage + 1;
    bool have = false;
    for (uint32_t i = lo; i < hi; i++) {
        // stage 0 holds L0; the others split L - L0 evenly, earlier stages first
        const uint32_t Li = i == 0 ? L0 : (L - L0) / (p - 1) + ((i - 1) < (L - L0) % (p - 1) ? 1u : 0u);
        const uint32_t n_i = (uint32_t)((uint64_t)(p - i) < m ? (uint64_t)(p - i) : m);
        const uint32_t rc = P.recompute ? 1u : 0u, dopt = P.dist_opt ? 1u : 0u;
        const TermsT<unsigned __int128> W = stage_terms<unsigned __int128>(DM, t, c, d, i == 0, i == p - 1, Li, n_i,
                                                                           u, rc, dopt, P.zero_stage);
        if (W.total >= lim) return ME_EOVERFLOW;
        const TermsT<uint64_t> T = stage_terms<uint64_t>(DM, t, c, d, i == 0, i == p - 1, Li, n_i, u, rc, dopt,
                                                         P.zero_stage);
        if (!have || T.total > out.total) {
            out = me_breakdown{T.params, T.grads, T.optim, T.layers, T.embed, T.head, T.total};
            which = i;
            have = true;
        }
    }
    return ME_OK;
}

__global__ void estimate_stage_kernel(const me_model* __restrict__ model, const me_parallel* __restrict__ cfg,
                                      uint32_t stage, me_breakdown* __restrict__ out, uint32_t* __restrict__ which,
                                      int* __restrict__ status) {
    me_breakdown b = {0, 0, 0, 0, 0, 0, 0};
    uint32_t w = 0;
    *status = estimate_stage_one(*model, *cfg, stage, b, w);
    *out = b;
    *which = w;
}

__global__ void estimate_kernel(const me_model* __restrict__ models, uint32_t n_models,
                                const uint32_t* __restrict__ ids,
                                const me_parallel* __restrict__ cfgs, uint64_t n,
                                const uint64_t* __restrict__ thr, uint32_t n_cap,
                                me_breakdown* __restrict__ out, uint8_t* __restrict__ mask,
                                uint8_t* __restrict__ status) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t id = ids ? ids[i] : 0u;
        me_breakdown b = {0, 0, 0, 0, 0, 0, 0};
        int st = id < n_models ? estimate_one(models[id], cfgs[i], b) : ME_EINVAL;
        uint32_t mk = 0;
        if (st == ME_OK)
            for (uint32_t q = 0; q < n_cap; q++) mk |= (b.total <= thr[q] ? 1u : 0u) << q;
        if (out) out[i] = b;
        if (mask) mask[i] = (uint8_t)mk;
        if (status) status[i] = (uint8_t)st;
    }
}

inline uint32_t ncap_stride_(uint32_t n_cap) { return n_cap <= 1 ? 1 : n_cap <= 2 ? 2 : n_cap <= 4 ? 4 : 8; }

void* count_kernel_for(uint32_t n_cap) {
    switch (ncap_stride_(n_cap)) {
        case 1: return reinterpret_cast<void*>(&count_kernel<1>);
        case 2: return reinterpret_cast<void*>(&count_kernel<2>);
        case 4: return reinterpret_cast<void*>(&count_kernel<4>);
        default: return reinterpret_cast<void*>(&count_kernel<8>);
    }
}

template <int MODE>
void* write_kernel_for(uint32_t n_cap) {
    switch (ncap_stride_(n_cap)) {
        case 1: return reinterpret_cast<void*>(&write_kernel<MODE, 1>);
        case 2: return reinterpret_cast<void*>(&write_kernel<MODE, 2>);
        case 4: return reinterpret_cast<void*>(&write_kernel<MODE, 4>);
        default: return reinterpret_cast<void*>(&write_kernel<MODE, 8>);
    }
}

void* write_fn(me_out_mode mode, uint32_t n_cap) {
    if (mode == ME_OUT_RECORDS) return write_kernel_for<3>(n_cap);
    return mode == ME_OUT_FULL ? write_kernel_for<2>(n_cap) : write_kernel_for<1>(n_cap);
}


}  // namespace

uint32_t ncap_stride(uint32_t n_cap) { return ncap_stride_(n_cap); }

uint32_t n_tiles_of(uint64_t lo, uint64_t hi) {
    const uint64_t base = lo & ~31ull;
    return hi > lo ? (uint32_t)((hi - base + kTile - 1) / kTile) : 0u;
}

// pass 0 count, 1 INDEX write, 2 FULL write, 3 RECORDS write
int sweep_blocks_per_sm(int pass, uint32_t n_cap) {
    const me_out_mode mode = pass == 3 ? ME_OUT_RECORDS : (pass == 2 ? ME_OUT_FULL : ME_OUT_INDEX);
    void* fn = pass == 0 ? count_kernel_for(n_cap) : write_fn(mode, n_cap);
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, 0) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_count(const DevSpace& S, uint64_t lo, uint64_t hi, uint32_t n_spans, uint32_t n_blocks,
                         uint32_t* tile_rel, uint32_t* tile_cnt, uint4* tile_ck, uint32_t* span_count,
                         uint32_t* span_caps, cudaStream_t st) {
    void* args[] = {(void*)&S,       (void*)&lo,         (void*)&hi,       (void*)&n_spans, (void*)&tile_rel,
                    (void*)&tile_cnt, (void*)&tile_ck, (void*)&span_count, (void*)&span_caps};
    return cudaLaunchKernel(count_kernel_for(S.n_cap), dim3(n_blocks), dim3(kThreads), args, 0, st);
}

cudaError_t launch_scan(const uint32_t* span_count, const uint32_t* span_caps, uint32_t n_spans, uint32_t n_cap,
                        uint64_t* span_off, uint64_t* stats, cudaStream_t st) {
    scan_kernel<<<1, 1024, 0, st>>>(span_count, n_spans, span_caps, n_spans, ncap_stride(n_cap), n_cap, span_off,
                                    stats);
    return cudaGetLastError();
}

cudaError_t launch_write(const DevSpace& S, uint64_t lo, uint64_t hi, uint32_t n_blocks, const uint4* tile_ck,
                         const uint32_t* tile_rel, const uint32_t* tile_cnt, const uint64_t* span_off,
                         me_out_mode mode, Cols cols, uint64_t capacity, cudaStream_t st) {
    void* args[] = {(void*)&S,        (void*)&lo,       (void*)&hi,       (void*)&tile_ck, (void*)&tile_rel,
                    (void*)&tile_cnt, (void*)&span_off, (void*)&cols, (void*)&capacity};
    return cudaLaunchKernel(write_fn(mode, S.n_cap), dim3(n_blocks), dim3(kThreads), args, 0, st);
}

cudaError_t launch_estimate_stage(const me_model* model, const me_parallel* cfg, uint32_t stage, me_breakdown* out,
                                  uint32_t* which, int* status, cudaStream_t st) {
    estimate_stage_kernel<<<1, 1, 0, st>>>(model, cfg, stage, out, which, status);
    return cudaGetLastError();
}

cudaError_t launch_estimate(const me_model* models, uint32_t n_models, const uint32_t* ids,
                            const me_parallel* cfgs, uint64_t n, const uint64_t* thr,
                            uint32_t n_cap, me_breakdown* out, uint8_t* mask, uint8_t* status,
                            cudaStream_t st) {
    if (!n) return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    estimate_kernel<<<(unsigned)blocks, 256, 0, st>>>(models, n_models, ids, cfgs, n, thr, n_cap,
                                                      out, mask, status);
    return cudaGetLastError();
}

}  // namespace me
