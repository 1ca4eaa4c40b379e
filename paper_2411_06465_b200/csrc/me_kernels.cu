// me_kernels.cu -- the sweep kernels (sm_100a).
//
// Work decomposition: the index range [begin, end) is split into one
// contiguous span per warp (span boundaries aligned to multiples of 32 in
// absolute index).  A warp walks its span in rounds of 32 consecutive
// indices, lane l taking index base + 32 i + l, so a warp ballot yields the
// survivors of a round in index order.  Each lane keeps an odometer over the
// canonical enumeration (segment -> tuple row -> position in row); the only
// search is one binary search per lane at span start.  Row coefficients
// (Psi_s, model-state bytes, per-token activation coefficients) are computed
// once per row; the per-config work is a pair lookup, a u32 x u64 multiply-add
// and n_cap u64 compares.
//
// Two passes: the count pass stores per-warp survivor counts,
// a one-block scan turns them into per-warp output offsets, and the write
// pass re-walks the spans and stores the survivors' columns (structure of
// arrays, 8-byte stores that are contiguous across the active lanes).
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

struct Walker {
    uint32_t seg, j, jend, r, w, pair_off;
    me_model M;
    RowCoef R;

    __device__ __forceinline__ void enter_segment(const DevSpace& S, uint32_t s) {
        seg = s;
        const uint32_t m = s / S.n_world, n = s - m * S.n_world;
        const uint32_t* mp = reinterpret_cast<const uint32_t*>(S.models + m);
        M.hidden = __ldg(mp + 0);
        M.ffn_hidden = __ldg(mp + 1);
        M.layers = __ldg(mp + 2);
        M.heads = __ldg(mp + 3);
        M.kv_heads = __ldg(mp + 4);
        M.vocab = __ldg(mp + 5);
        const uint32_t cls = __ldg(S.model_class + m);
        j = __ldg(S.list_off + cls * S.n_world + n);
        jend = __ldg(S.list_off + cls * S.n_world + n + 1);
    }

    __device__ __forceinline__ void set_row(const DevSpace& S) {
        const uint32_t tid = __ldg(S.list_tuple + j);
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(S.tuples + tid));      // t c p d
        const uint2 b = __ldg(reinterpret_cast<const uint2*>(S.tuples + tid) + 2);  // w pair_off
        w = b.x;
        pair_off = b.y;
        make_row(M, a.x, a.y, a.z, a.w, first_stage_layers_auto(M.layers, a.z), R);
    }

    // position the walker on absolute index pos (< total)
    __device__ __forceinline__ void seek(const DevSpace& S, uint64_t pos) {
        const uint32_t s = upper_bound_u64(S.seg_prefix, S.n_seg + 1, pos) - 1;
        enter_segment(S, s);
        const uint64_t within = pos - __ldg(S.seg_prefix + s);
        const uint32_t k = upper_bound_u64(S.list_prefix + j, jend - j, within) - 1;
        j += k;
        r = (uint32_t)(within - __ldg(S.list_prefix + j));
        set_row(S);
    }

    // move forward by `step` indices (the caller guarantees the target exists)
    __device__ __forceinline__ void advance(const DevSpace& S, uint32_t step) {
        r += step;
        while (r >= w) next_row(S);
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

    __device__ __forceinline__ uint2 pair(const DevSpace& S, uint32_t lg) const {
        return __ldg(reinterpret_cast<const uint2*>(S.pairs) + pair_off + (r >> lg));
    }
};

// span of global warp gw: [span(gw), span(gw + 1)), 32-aligned in absolute index
__device__ __forceinline__ uint64_t span_start(uint64_t begin, uint64_t end, uint32_t gw,
                                               uint32_t n_warps) {
    if (gw == 0) return begin;
    if (gw >= n_warps) return end;
    const uint64_t len = end - begin;
    const uint64_t q = len / n_warps, rem = len % n_warps;
    uint64_t s = begin + q * gw + (rem * gw) / n_warps;
    s = (s + 31) & ~31ull;
    return s < end ? s : end;
}

template <int NCAP>
__device__ __forceinline__ uint32_t cap_mask(const DevSpace& S, uint64_t total) {
    uint32_t mask = 0;
#pragma unroll
    for (int q = 0; q < NCAP; q++) mask |= (total <= S.thr[q] ? 1u : 0u) << q;
    return mask;
}

// Per-lane accumulators of the count pass: survivor count and 8-bit packed
// per-capacity counters (mask * 0x00204081 spreads bits 0..3 to bytes 0..3).
template <int NCAP>
struct CountAcc {
    uint32_t cnt = 0, lo = 0, hi = 0, round = 0;
    uint32_t capc[NCAP];
    __device__ __forceinline__ CountAcc() {
#pragma unroll
        for (int q = 0; q < NCAP; q++) capc[q] = 0;
    }
    __device__ __forceinline__ void flush() {
#pragma unroll
        for (int q = 0; q < NCAP; q++) capc[q] += ((q < 4 ? lo : hi) >> (8 * (q & 3))) & 255u;
        lo = hi = 0;
    }
    __device__ __forceinline__ void add(uint32_t mask) {
        cnt += mask ? 1u : 0u;
        if (NCAP <= 4) {
            lo += (mask * 0x00204081u) & 0x01010101u;
        } else {
            lo += ((mask & 15u) * 0x00204081u) & 0x01010101u;
            hi += ((mask >> 4) * 0x00204081u) & 0x01010101u;
        }
        if ((++round & 255u) == 0) flush();
    }
};

// One warp span.  RAGGED = the span does not start and end on multiples of 32
// (only the first and last spans of a range), so lanes need range checks.
// The pair of the next round is loaded before the current round is evaluated
// (software pipelining of the only per-config memory access).
template <int MODE, int NCAP, bool RAGGED>
__device__ __forceinline__ void walk_span(const DevSpace& S, uint64_t sb, uint64_t se, uint32_t lane,
                                          CountAcc<NCAP>& acc, uint64_t out, const Cols& cols,
                                          uint64_t capacity) {
    const uint64_t base = sb & ~31ull;
    Walker W;
    uint64_t pos = base + lane;
    if (RAGGED && pos >= se) return;  // this lane never has work (its later positions are >= se too)
    W.seek(S, pos);
    const uint32_t rc_bits = S.rcdo_rc, do_bits = S.rcdo_do, lg = S.lg_rcdo;
    const uint32_t sel_mask = (1u << lg) - 1;
    uint2 pr = W.pair(S, lg);
    for (uint64_t p0 = base; p0 < se; p0 += 32, pos += 32) {
        // issue the next round's pair load first when it stays in this row
        const uint32_t rn = W.r + 32;
        const bool more = pos + 32 < se;
        const bool in_row = rn < W.w;
        uint2 prn = pr;
        if (in_row && more) prn = __ldg(reinterpret_cast<const uint2*>(S.pairs) + W.pair_off + (rn >> lg));

        const bool act = !RAGGED || (pos >= sb && pos < se);
        const uint32_t sel = W.r & sel_mask;
        const uint32_t rc = (rc_bits >> sel) & 1u, dopt = (do_bits >> sel) & 1u;
        const uint64_t total = config_total(W.R, pr.x, pr.y, rc, dopt);
        uint32_t mask = act ? cap_mask<NCAP>(S, total) : 0u;
        if (MODE == 0) {
            acc.add(mask);
        } else {
            const uint32_t ballot = __ballot_sync(0xffffffffu, mask != 0);
            if (mask) {
                const uint64_t o = out + __popc(ballot & ((1u << lane) - 1u));
                if (o < capacity) {
                    cols.c[0][o] = pos | ((uint64_t)mask << 56);
                    if (MODE == 2) {
                        const TermsT<uint64_t> T = config_terms_no_total(W.R, pr.x, pr.y, rc, dopt);
                        cols.c[1][o] = T.params;
                        cols.c[2][o] = T.grads;
                        cols.c[3][o] = T.optim;
                        cols.c[4][o] = T.layers;
                        cols.c[5][o] = T.embed;
                        cols.c[6][o] = T.head;
                        cols.c[7][o] = total;
                    }
                }
            }
            out += __popc(ballot);
        }
        if (more) {
            if (in_row) {
                W.r = rn;
                pr = prn;
            } else {
                W.advance(S, 32);
                pr = W.pair(S, lg);
            }
        }
    }
}

// MODE 0 = count pass, 1 = INDEX write, 2 = FULL write.  The range is cut
// into n_spans spans; warp w of the grid handles spans w, w + n_warps, ...
// (the span decomposition, not the grid, fixes the output offsets, so the
// two passes may run with different grids).
template <int MODE, int NCAP>
__global__ void __launch_bounds__(kThreads) sweep_kernel(const DevSpace S, const uint64_t begin,
                                                         const uint64_t end, const uint32_t n_spans,
                                                         uint32_t* __restrict__ warp_count,
                                                         uint32_t* __restrict__ warp_caps,
                                                         const uint64_t* __restrict__ warp_off,
                                                         const Cols cols, const uint64_t capacity) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t n_warps = gridDim.x * kWarpsPerBlock;
    for (uint32_t gw = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5); gw < n_spans; gw += n_warps) {
        const uint64_t sb = span_start(begin, end, gw, n_spans);
        const uint64_t se = span_start(begin, end, gw + 1, n_spans);
        CountAcc<NCAP> acc;
        uint64_t out = 0;
        if (MODE != 0) out = warp_off[gw];
        if (sb < se) {
            if (((sb | se) & 31ull) == 0)
                walk_span<MODE, NCAP, false>(S, sb, se, lane, acc, out, cols, capacity);
            else
                walk_span<MODE, NCAP, true>(S, sb, se, lane, acc, out, cols, capacity);
        }
        if (MODE == 0) {
            acc.flush();
            const uint32_t cnt = __reduce_add_sync(0xffffffffu, acc.cnt);
            uint32_t capc[NCAP];
#pragma unroll
            for (int q = 0; q < NCAP; q++) capc[q] = __reduce_add_sync(0xffffffffu, acc.capc[q]);
            if (lane == 0) {
                warp_count[gw] = cnt;
#pragma unroll
                for (int q = 0; q < NCAP; q++) warp_caps[(size_t)gw * NCAP + q] = capc[q];
            }
        }
    }
}

// one block: exclusive scan of n warp counts (u32) into u64 offsets + totals
__global__ void __launch_bounds__(1024) scan_kernel(const uint32_t* __restrict__ warp_count,
                                                    const uint32_t* __restrict__ warp_caps,
                                                    uint32_t n, uint32_t ncap_stride,
                                                    uint32_t n_cap, uint64_t* __restrict__ warp_off,
                                                    uint64_t* __restrict__ stats) {
    __shared__ uint64_t s_warp[32];
    __shared__ uint64_t s_caps[8][32];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t chunk = (n + blockDim.x - 1) / blockDim.x;
    const uint32_t lo = min(n, tid * chunk), hi = min(n, lo + chunk);
    uint64_t sum = 0;
    uint64_t caps[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint32_t i = lo; i < hi; i++) {
        sum += warp_count[i];
        for (uint32_t q = 0; q < n_cap; q++) caps[q] += warp_caps[(size_t)i * ncap_stride + q];
    }
    // inclusive warp scan
    uint64_t inc = sum;
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
    if (wid == 0) {
        const uint32_t nw = blockDim.x >> 5;
        uint64_t v = lane < nw ? s_warp[lane] : 0;
        uint64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane < nw) s_warp[lane] = x - v;  // exclusive
        if (lane == 31) stats[0] = x;
        for (uint32_t q = 0; q < n_cap; q++) {
            uint64_t c = lane < nw ? s_caps[q][lane] : 0;
            for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
            if (lane == 0) stats[1 + q] = c;
        }
    }
    __syncthreads();
    uint64_t run = s_warp[wid] + inc - sum;
    for (uint32_t i = lo; i < hi; i++) {
        warp_off[i] = run;
        run += warp_count[i];
    }
    if (tid == blockDim.x - 1) warp_off[n] = s_warp[wid] + inc;
}

// ---- single configurations ----------------------------------------------
__device__ int estimate_one(const me_model& M, const me_parallel& P, me_breakdown& out) {
    if (!M.hidden || !M.ffn_hidden || !M.layers || !M.heads || !M.kv_heads || !M.vocab)
        return ME_EINVAL;
    if (M.heads % M.kv_heads || M.hidden % M.heads) return ME_EINVAL;
    if (!P.dp || !P.tp || !P.pp || !P.cp || !P.mbs || !P.seq) return ME_EINVAL;
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
    RowCoefT<unsigned __int128> W;
    make_row(M, t, c, p, d, L0, W);
    const TermsT<unsigned __int128> T2 = config_terms(W, u, m, P.recompute ? 1u : 0u, P.dist_opt ? 1u : 0u);
    const unsigned __int128 lim = (unsigned __int128)1 << 63;
    if (W.psi >= lim || W.ms0 >= lim || T2.total >= lim) return ME_EOVERFLOW;
    RowCoef R;
    make_row(M, t, c, p, d, L0, R);
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

template <int MODE>
void* kernel_for(uint32_t n_cap) {
    switch (ncap_stride_(n_cap)) {
        case 1: return reinterpret_cast<void*>(&sweep_kernel<MODE, 1>);
        case 2: return reinterpret_cast<void*>(&sweep_kernel<MODE, 2>);
        case 4: return reinterpret_cast<void*>(&sweep_kernel<MODE, 4>);
        default: return reinterpret_cast<void*>(&sweep_kernel<MODE, 8>);
    }
}

template <int MODE>
cudaError_t launch_mode(const DevSpace& S, uint64_t begin, uint64_t end, uint32_t n_spans,
                        uint32_t n_blocks, uint32_t* wc, uint32_t* wcap, const uint64_t* woff, Cols cols,
                        uint64_t capacity, cudaStream_t st) {
    void* args[] = {(void*)&S, (void*)&begin, (void*)&end, (void*)&n_spans, (void*)&wc,
                    (void*)&wcap, (void*)&woff, (void*)&cols, (void*)&capacity};
    return cudaLaunchKernel(kernel_for<MODE>(S.n_cap), dim3(n_blocks), dim3(kThreads), args, 0, st);
}

}  // namespace

uint32_t ncap_stride(uint32_t n_cap) { return ncap_stride_(n_cap); }

int sweep_blocks_per_sm(int pass, uint32_t n_cap) {
    void* fn = pass == 0 ? kernel_for<0>(n_cap) : (pass == 1 ? kernel_for<1>(n_cap) : kernel_for<2>(n_cap));
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, 0) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_count(const DevSpace& S, uint64_t begin, uint64_t end, uint32_t n_spans, uint32_t n_blocks,
                         uint32_t* warp_count, uint32_t* warp_caps, cudaStream_t st) {
    Cols none{};
    return launch_mode<0>(S, begin, end, n_spans, n_blocks, warp_count, warp_caps, nullptr, none, 0, st);
}

cudaError_t launch_scan(const uint32_t* warp_count, const uint32_t* warp_caps, uint32_t n_warps,
                        uint32_t n_cap, uint64_t* warp_off, uint64_t* stats, cudaStream_t st) {
    scan_kernel<<<1, 1024, 0, st>>>(warp_count, warp_caps, n_warps, ncap_stride(n_cap), n_cap,
                                    warp_off, stats);
    return cudaGetLastError();
}

cudaError_t launch_write(const DevSpace& S, uint64_t begin, uint64_t end, uint32_t n_spans, uint32_t n_blocks,
                         const uint64_t* warp_off, me_out_mode mode, Cols cols, uint64_t capacity,
                         cudaStream_t st) {
    if (mode == ME_OUT_FULL)
        return launch_mode<2>(S, begin, end, n_spans, n_blocks, nullptr, nullptr, warp_off, cols, capacity, st);
    return launch_mode<1>(S, begin, end, n_spans, n_blocks, nullptr, nullptr, warp_off, cols, capacity, st);
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
