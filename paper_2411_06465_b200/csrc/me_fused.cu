// me_fused.cu -- the row-count sweep pipeline (sm_100a), DESIGN.md §6.
//
// A row is a run of configurations sharing (model, N, t, c, p, d); its
// configurations are its valid (b, s) pairs x the (rc, do) digits, in that
// order.  For one digit every estimator term is affine in the pair's tokens
// per microbatch u = b s / c (paper mode: the in-flight count is p), so the
// total is strictly increasing in u and "total <= threshold" (the 80% rule,
// P:27) holds exactly for the pairs with u up to a bound.  Per
// sub-range of the flat index space:
//
//  K0 rowcount_kernel  one thread per row: the row's coefficients (make_row,
//                      Eq.6/7/10/12-17), per digit the exact survivor bound
//                      umax = floor((thr - ms) / K) (the largest u whose
//                      total fits), its survivors per capacity -- per digit
//                      a binary search for umax over the row's u values
//                      sorted ascending -- and per 32-row unit the survivor
//                      count;
//                      a global batch (R17: the in-flight count depends on
//                      b) or a row cut by the range is evaluated config by
//                      config instead;
//  scan                unit counts -> output offsets (scan_kernel);
//  K3 fused_kernel     warps take 32-row units in order: per row with
//                      survivors, 32 consecutive configurations per round,
//                      survivor test (u <= umax: one compare), ballot
//                      compaction, the survivors' eight output values and
//                      their stores (records: two 32-byte stores per lane,
//                      one contiguous run per round).
//
// Every configuration is tested once (K3); K0 works per row.  No per-survivor
// intermediate goes through HBM: the only scratch traffic is the 128-byte row
// entry per row with survivors.
#include <cuda_runtime.h>

#include <cstdlib>

#include "me_dev.cuh"
#include "me_kernels.cuh"

namespace me {

namespace {

// one (rc, do) digit of a row: stage 0 total = ms + u K; with NEXT-1 and p >= 2
// also the last stage, msL + u kL
struct Digit {
    uint64_t ms, K, msL, kL;
    bool two;
};

__device__ __forceinline__ bool fits(const Digit& c, uint32_t u, uint64_t thr) {
    if (c.ms + (uint64_t)u * c.K > thr) return false;
    return !c.two || c.msL + (uint64_t)u * c.kL <= thr;
}

// number of leading entries of the ascending su[0, n) that fit under thr
__device__ __forceinline__ uint32_t count_fit(const uint32_t* su, uint32_t n, const Digit& c, uint64_t thr) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (fits(c, su[mid], thr)) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// ---------------------------------------------------------------- K0
// CAPS: count the survivors of every capacity too (COUNT mode; the output
// kernel counts them from the masks it computes anyway in the other modes).
// Blocks of kRowThreads threads at <= 64 registers, so that K0 of the next
// sub-range fits beside the resident output-kernel blocks.  The sorted u
// lists are staged in shared memory when they fit; a row's binary searches
// (one per digit) run in lockstep, so their loads are in flight together.
constexpr uint32_t kRowThreads = 128;
#ifndef ME_K0_COUNT_MINB
#define ME_K0_COUNT_MINB 6
#endif
constexpr int kRowMinbCount = ME_K0_COUNT_MINB;  // count-only K0: resident blocks per SM (register budget)
#ifndef ME_K0_WRITE_MINB
#define ME_K0_WRITE_MINB 8
#endif
constexpr int kRowMinbWrite = ME_K0_WRITE_MINB;  // K0 with row entries: 8 = 64 registers

// The survivor bound of one digit: the largest u with ms + u K <= thr, i.e.
// floor((thr - ms) / K), clamped to 2^32 - 1 (u is 32-bit); 0 when thr < ms
// (u >= 1 admits nothing).  The quotient is estimated in FP64 from rK, the
// rounded reciprocal of K: relative error < 2^-50, so for quotients below
// 2^32 the estimate is within 1 of the exact one, which one exact integer
// step each way then restores (thr <= 2^63 and K < 2^62, so the products
// below do not wrap).
__device__ __forceinline__ uint32_t u_bound(uint64_t ms, uint64_t K, double rK, uint64_t thr) {
    ME_CHECK(thr <= (1ull << 63) && K < (1ull << 62));
    const uint64_t num = thr - ms;  // (wraps when thr < ms: the result is 0 then)
    const double qd = __dmul_rz(__ull2double_rz(num), rK);
    uint32_t q = (uint32_t)fmin(qd, 4294967295.0);
    // exact: q K <= num < (q + 1) K, or q = 2^32 - 1 when (2^32 - 1) K <= num
    uint64_t qk = (uint64_t)q * K;
    const bool over = qk > num;
    q = over ? q - 1 : q;
    qk = over ? qk - K : qk;
    q = num - qk >= K && q != 0xFFFFFFFFu ? q + 1 : q;
    ME_CHECK(thr < ms || K == 0 || ((uint64_t)q * K <= num && (q == 0xFFFFFFFFu || num - (uint64_t)q * K < K)));
    return thr < ms ? 0u : K == 0 ? 0xFFFFFFFFu : q;
}

// per bound j < NQ: the number of entries of the ascending su[0, n) that are
// <= ub_j (n >= 1; u >= 1, so a bound 0 counts none).  Branch-free binary
// search: the length sequence depends on n only, so the NQ searches run in
// lockstep with one trip count and their loads in flight together; every load
// is in su[0, n).
#ifndef ME_K0_GROUP
#define ME_K0_GROUP 4
#endif
constexpr int kCapGroup = ME_K0_GROUP;  // COUNT-mode K0: capacities searched together (x 4 digits)
template <int NQ>
__device__ __forceinline__ void count_le(const uint32_t* __restrict__ su, uint32_t n, const uint32_t (&ub)[NQ],
                                         uint32_t (&out)[NQ]) {
    uint32_t base[NQ];
#pragma unroll
    for (int j = 0; j < NQ; j++) base[j] = 0;
    uint32_t len = n;
    while (len > 1) {
        const uint32_t half = len >> 1;
        uint32_t v[NQ];
#pragma unroll
        for (int j = 0; j < NQ; j++) v[j] = su[base[j] + half - 1];
#pragma unroll
        for (int j = 0; j < NQ; j++) base[j] = v[j] <= ub[j] ? base[j] + half : base[j];
        len -= half;
    }
#pragma unroll
    for (int j = 0; j < NQ; j++) out[j] = base[j] + (su[base[j]] <= ub[j] ? 1u : 0u);
}

// The same counts through the pool's fences (n <= 128): fe[0, 4) = the
// largest u of each 32-entry group, fe[4, 20) = of each 8-entry block
// (0xFFFFFFFF past the pool).  Groups, then blocks, whose largest u is <= ub
// form a prefix, so per bound: g = full groups (4 compares), b = full blocks
// of group g (3 compares on one 16-byte load), then a 3-step search inside
// block 4g + b.  4 scattered 4-byte loads per bound instead of log2(n) + 1:
// fewer shared-memory bank conflicts / L1 wavefronts, the dominant stall of
// the plain search.
template <int NQ>
__device__ __forceinline__ void count_le_f(const uint32_t* __restrict__ su, uint32_t n,
                                           const uint32_t* __restrict__ fe, const uint32_t (&ub)[NQ],
                                           uint32_t (&out)[NQ]) {
    const uint4 g4 = *reinterpret_cast<const uint4*>(fe);
#pragma unroll
    for (int j = 0; j < NQ; j++) {
        const uint32_t x = ub[j];
        const uint32_t g = (g4.x <= x) + (g4.y <= x) + (g4.z <= x) + (g4.w <= x);
        const uint4 b4 = *reinterpret_cast<const uint4*>(fe + 4 + 4 * (g & 3u));
        const uint32_t blk = 4 * g + (g < 4 ? (b4.x <= x) + (b4.y <= x) + (b4.z <= x) : 0u);
        const uint32_t lo = 8 * blk;
        uint32_t len = lo < n ? min(8u, n - lo) : 1u, base = 0;
#pragma unroll
        for (int it = 0; it < 3; it++) {
            const uint32_t half = len >> 1;
            const uint32_t at = lo + base + half;
            const uint32_t v = su[min(at ? at - 1 : 0u, n - 1)];  // (half = 0: unused)
            base = half && v <= x ? base + half : base;
            len -= half;
        }
        out[j] = lo < n ? lo + base + (su[min(lo + base, n - 1)] <= x ? 1u : 0u) : n;  // (index clamped: no load past the pool)
        ME_CHECK(out[j] <= n);
    }
}

// One row: its RowEnt (to *out: global for K0, the warp's shared copy for the
// one-pass kernel), its last-stage terms (NEXT-1, to st[k]), its survivors in
// the window [lo, hi) (returned) and, CAPS, per capacity (into capc).
// su_base: the sorted-u lists (shared memory when staged).
template <int NCAP, bool CAPS>
__device__ __forceinline__ uint32_t row_count(const DevSpace& S, uint64_t g, uint32_t k, uint32_t seg,
                                              uint64_t lo, uint64_t hi, const uint32_t* su_base, const uint32_t* fe_base, RowEnt* out,
                                              StEnt* __restrict__ st, uint32_t (&capc)[NCAP]) {
    uint32_t cnt = 0;
    const RowId I = row_id_from(S, g, seg);
    RowCoef R;
    const Policy Q = policy_of(S);
    make_row(I.M, I.tu.t, I.tu.c, I.tu.p, I.tu.d, I.L0, Q, R);
    const bool two = S.stage_max && I.tu.p >= 2;
    *out = row_entry(I, R, two);  // umax[] below
    uint32_t umax[4] = {0, 0, 0, 0};
    const uint32_t lg = S.lg_rcdo, n_sel = 1u << lg;
    // the row's window of the range: [a, b) of its positions
    const uint32_t a = I.rs < lo ? (uint32_t)(lo - I.rs) : 0u;
    const uint32_t b = I.rs + I.tu.w > hi ? (uint32_t)(hi - I.rs) : I.tu.w;
    const bool full = a == 0 && b == I.tu.w;
    const uint32_t* su = su_base + I.tu.pair_off;
    const uint32_t* fe = fe_base + I.tu.fence_off;
    const DevPair* pp = S.pairs + I.tu.pair_off;
    // per digit: stage-0 total = ms + u K in paper mode
    uint64_t ms[4], K[4];
#pragma unroll
    for (uint32_t sel = 0; sel < 4; sel++) {
        ms[sel] = K[sel] = 0;
        if (sel >= n_sel) continue;
        const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
        ms[sel] = dopt ? R.ms1 : R.ms0;
        // per-token bytes in paper mode: n_lay lam + mu + n_emb e8 + hc
        K[sel] = (uint64_t)R.nlay * (rc ? R.lam1 : R.lam0) + (rc ? R.bt : 0ull) + (uint64_t)R.nemb * R.e8 + R.hc;
        if (two) st[(size_t)k << lg | sel] = last_stage(I, rc, dopt, Q);
    }
    if (!S.gbs_mode && !two) {
        // per digit the exact survivor bound umax (u <= umax <=> total <= thr_max,
        // which is what K3 tests) and the row's survivors: pairs with u <= umax
        const uint32_t np = I.tu.n_pairs;
        ME_CHECK(np >= 1);
        double rK[4];
        uint32_t nm[4];
        // (digits sel >= n_sel keep umax 0: they count none)
#pragma unroll
        for (uint32_t sel = 0; sel < 4; sel++) {
            rK[sel] = sel < n_sel && K[sel] ? __drcp_rn(__ull2double_rn(K[sel])) : 0.0;
            umax[sel] = sel < n_sel ? u_bound(ms[sel], K[sel], rK[sel], S.thr_max) : 0u;
        }
        if (CAPS && full) {
            // every capacity's survivors (the largest threshold's are the
            // row's): up to kCapGroup capacities x 4 digits per lockstep
            // search (all of them when they fit; else one at a time, which
            // keeps 8 capacities free of spills)
            constexpr int G = NCAP <= kCapGroup ? NCAP : 1;
#pragma unroll
            for (int q0 = 0; q0 < NCAP; q0 += G) {
                if (q0 >= (int)S.n_cap) break;
                uint32_t ub[4 * G], nq[4 * G];
#pragma unroll
                for (int j = 0; j < G; j++) {
                    const int q = q0 + j;
                    const bool on = q < (int)S.n_cap;
                    const uint64_t th = on ? S.thr[q] : 0ull;
#pragma unroll
                    for (uint32_t sel = 0; sel < 4; sel++)
                        ub[4 * j + sel] = !on ? 0u : th == S.thr_max ? umax[sel]
                                                                      : (sel < n_sel ? u_bound(ms[sel], K[sel], rK[sel], th) : 0u);
                }
                if (S.fenced) count_le_f<4 * G>(su, np, fe, ub, nq);
                else count_le<4 * G>(su, np, ub, nq);
#pragma unroll
                for (int j = 0; j < G; j++) {
                    const int q = q0 + j;
                    if (q >= (int)S.n_cap) break;
                    const uint32_t c = nq[4 * j] + nq[4 * j + 1] + nq[4 * j + 2] + nq[4 * j + 3];
                    capc[q] += c;
                    if (S.thr[q] == S.thr_max) cnt = c;
                }
            }
        } else if (full) {
            if (S.fenced) count_le_f<4>(su, np, fe, umax, nm);
            else count_le<4>(su, np, umax, nm);
            cnt += nm[0] + nm[1] + nm[2] + nm[3];
        } else {
            // a row cut by the range: its window [a, b) configuration by
            // configuration, one compare each against the digit's bound(s)
            // (a single thread walks it: the per-configuration total would
            // keep it running long after the rest of the launch)
            for (uint32_t sel = 0; sel < n_sel; sel++) {
                const uint32_t um = sel == 0 ? umax[0] : sel == 1 ? umax[1] : sel == 2 ? umax[2] : umax[3];
                const uint64_t msq = sel == 0 ? ms[0] : sel == 1 ? ms[1] : sel == 2 ? ms[2] : ms[3];
                const uint64_t Kq = sel == 0 ? K[0] : sel == 1 ? K[1] : sel == 2 ? K[2] : K[3];
                const double rq = sel == 0 ? rK[0] : sel == 1 ? rK[1] : sel == 2 ? rK[2] : rK[3];
                uint32_t ubc[NCAP];
#pragma unroll
                for (int q = 0; q < NCAP; q++)
                    ubc[q] = !CAPS || q >= (int)S.n_cap ? 0u
                             : S.thr[q] == S.thr_max    ? um
                                                        : u_bound(msq, Kq, rq, S.thr[q]);
                // eight independent loads in flight per step
                constexpr uint32_t kW = 8;
                for (uint32_t p0 = a + ((sel - a) & (n_sel - 1u)); p0 < b; p0 += kW * n_sel) {
                    uint32_t u[kW];
#pragma unroll
                    for (uint32_t i = 0; i < kW; i++) {
                        const uint32_t pos = p0 + i * n_sel;
                        u[i] = pos < b ? __ldg(&pp[pos >> lg].u) : 0u;  // u >= 1: 0 marks "outside"
                    }
#pragma unroll
                    for (uint32_t i = 0; i < kW; i++) {
                        const bool in = u[i] != 0;
                        cnt += in && u[i] <= um ? 1u : 0u;
                        if (CAPS) {
#pragma unroll
                            for (int q = 0; q < NCAP; q++) capc[q] += in && u[i] <= ubc[q] ? 1u : 0u;
                        }
                    }
                }
            }
        }
    } else if (!S.gbs_mode) {
        // NEXT-1: the largest of two stage totals, one digit at a time
        // (unrolled: ms[] and K[] stay in registers)
#pragma unroll
        for (uint32_t sel = 0; sel < 4; sel++) {
            if (sel >= n_sel) break;
            const StEnt* x = st + ((size_t)k << lg | sel);
            Digit c{ms[sel], K[sel], x->msL, x->kL, true};
            const uint32_t nm = count_fit(su, I.tu.n_pairs, c, S.thr_max);
            umax[sel] = nm ? su[nm - 1] : 0u;
            if (full) {
                cnt += nm;
                if (CAPS) {
#pragma unroll
                    for (int q = 0; q < NCAP; q++)
                        if (q < (int)S.n_cap) capc[q] += S.thr[q] >= S.thr_max ? nm : count_fit(su, nm, c, S.thr[q]);
                }
            }
        }
    }
    if (S.gbs_mode || (two && !full)) {
        // config by config over the window: in-flight counts of each
        // pair's m microbatches (R17, R29), or a cut row
#pragma unroll
        for (uint32_t sel = 0; sel < 4; sel++) {
            if (sel >= n_sel) break;
            const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
            for (uint32_t pos = a + ((sel - a) & (n_sel - 1u)); pos < b; pos += n_sel) {
                ME_CHECK((pos >> lg) < I.tu.n_pairs);
                const DevPair pr = pp[pos >> lg];
                uint64_t tot = config_total(R, pr.u, pr.m, rc, dopt, S.vpp);
                if (two) {
                    const StEnt* x = st + ((size_t)k << lg | sel);
                    const uint64_t tl = x->msL + (uint64_t)pr.u * x->kL;
                    tot = tl > tot ? tl : tot;
                }
                cnt += tot <= S.thr_max ? 1u : 0u;
                if (CAPS) {
#pragma unroll
                    for (int q = 0; q < NCAP; q++) capc[q] += (q < (int)S.n_cap && tot <= S.thr[q]) ? 1u : 0u;
                }
            }
        }
    }
    ME_CHECK(cnt <= b - a);
    *reinterpret_cast<uint4*>(&out->umax[0]) = make_uint4(umax[0], umax[1], umax[2], umax[3]);
    return cnt;
}

// WR: write each row's entry and the per-row / per-unit survivor counts for
// K3 (one block per 128 rows); !WR (COUNT mode and the sizing pass): only the
// totals, accumulated into stats[0] and stats[1 + j] by the blocks of a
// grid-stride launch.  SMEM (count-only): each block stages the sorted-u
// lists in shared memory once; otherwise they are read through L1 (staging
// per 128-row block measured slower in RECORDS: 344.3 vs 341.9 ms).  MINB: resident blocks per SM the registers are budgeted for (8: 64
// registers, beside K3; COUNT mode runs alone and takes more registers).
template <int NCAP, bool CAPS, bool WR, int MINB, bool SMEM>
__global__ void __launch_bounds__(kRowThreads, MINB)
    rowcount_kernel(const DevSpace S, const uint64_t g0, const uint32_t n_rows, const uint32_t seg_lo,
                    const uint32_t n_seg_sub, const uint64_t lo, const uint64_t hi, RowEnt* __restrict__ rows,
                    StEnt* __restrict__ st, uint32_t* __restrict__ rcnt, uint32_t* __restrict__ ucnt,
                    uint64_t* __restrict__ stats) {
    __shared__ uint32_t s_cap[NCAP + 1];
    extern __shared__ __align__(16) uint32_t s_su[];
    // (SMEM: the sorted lists, then the fences from a 16-byte boundary)
    const uint32_t fe_at = (S.n_pairs + 3u) & ~3u;
    if (threadIdx.x <= NCAP) s_cap[threadIdx.x] = 0;
    if (SMEM) {
        for (uint32_t i = threadIdx.x; i < S.n_pairs; i += blockDim.x) s_su[i] = __ldg(S.pair_su + i);
        if (S.fenced)
            for (uint32_t i = threadIdx.x; i < S.n_fence; i += blockDim.x) s_su[fe_at + i] = __ldg(S.pair_fence + i);
    }
    __syncthreads();
    const uint32_t* su = SMEM ? s_su : S.pair_su;
    const uint32_t* fe = SMEM ? s_su + fe_at : S.pair_fence;
    uint32_t cnt = 0;
    uint32_t capc[NCAP];
#pragma unroll
    for (int q = 0; q < NCAP; q++) capc[q] = 0;
    for (uint32_t base = blockIdx.x * kRowThreads; base < n_rows; base += gridDim.x * kRowThreads) {
        const uint32_t k = base + threadIdx.x;
        // the segment of the warp's first row (all lanes, before the bounds test)
        const uint64_t gw = g0 + (k & ~31u);
        const uint32_t seg = gw < g0 + n_rows ? warp_segment(S.seg_row, seg_lo, n_seg_sub - 1, gw) : seg_lo;
        uint32_t c = 0;
        if (k < n_rows) {
            RowEnt tmp;
            c = row_count<NCAP, CAPS>(S, g0 + k, k, seg, lo, hi, su, fe, WR ? rows + k : &tmp, st, capc);
            if (WR) rcnt[k] = c;
        }
        if (WR) {
            // survivors per 32-row unit (a unit is one warp of this kernel)
            const uint32_t unit_cnt = __reduce_add_sync(0xffffffffu, c);
            if ((threadIdx.x & 31) == 0 && k < n_rows) ucnt[k >> 5] = unit_cnt;
        }
        cnt += c;
    }
    if (!WR) {
        const uint32_t t = __reduce_add_sync(0xffffffffu, cnt);
        if ((threadIdx.x & 31) == 0 && t) atomicAdd(s_cap + NCAP, t);
    }
    if (CAPS) {
#pragma unroll
        for (int q = 0; q < NCAP; q++) {
            const uint32_t c = __reduce_add_sync(0xffffffffu, capc[q]);
            if ((threadIdx.x & 31) == 0 && c) atomicAdd(s_cap + q, c);
        }
    }
    if (CAPS || !WR) {
        __syncthreads();
        if (threadIdx.x < NCAP && CAPS && s_cap[threadIdx.x])
            atomicAdd((unsigned long long*)(stats + 1 + threadIdx.x), (unsigned long long)s_cap[threadIdx.x]);
        if (threadIdx.x == NCAP && !WR && s_cap[NCAP])
            atomicAdd((unsigned long long*)stats, (unsigned long long)s_cap[NCAP]);
    }
}

// ---------------------------------------------------------------- K3
constexpr uint32_t kUnit = 32;         // rows per unit
constexpr uint32_t kPairsSmem = 2048;  // pairs pool in shared memory when it fits (16 KB)
constexpr uint32_t kFusedWarps = kThreads / 32;
constexpr uint32_t kRowPairsSmem = 128;  // = kRowPairs (defined with the two-phase row path)
constexpr size_t kFusedSmemBytes = kPairsSmem * sizeof(DevPair) + (size_t)kFusedWarps * kUnit * sizeof(RowEnt) +
                                   (size_t)kFusedWarps * kRowPairsSmem * 4 * sizeof(uint16_t);


// Lane-constant values of one row for the lane's (rc, do) digit.
struct Lane {
    uint64_t v1, v2, v3;  // params, grads, optim
    uint64_t ms;          // their sum
    uint64_t lam, mu;     // layer bytes per token: n_lay lam + mu
    uint64_t e8, hc;      // embedding bytes per token per microbatch, LM-head bytes per token
    uint64_t c4, c5, K;   // paper mode: n_lay lam + mu, n_emb e8, c4 + c5 + hc
    uint32_t p, umax;
    // NEXT-1 last stage
    uint64_t msL, kL, parL, graL, optimL, layL, hcL;
};

template <bool GBS, bool STMAX>
__device__ __forceinline__ void lane_of(const DevSpace& S, const RowEnt& R, const StEnt* __restrict__ st,
                                        uint64_t kg, uint32_t sel, Lane& C) {
    const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
    const uint64_t psi = R.psi;
    C.v1 = dopt ? R.par1 : (uint64_t)S.wb * psi;
    C.v2 = dopt ? R.gra1 : (uint64_t)S.gb * psi;
    C.v3 = dopt ? R.optim1 : (uint64_t)S.ob * psi;
    C.ms = C.v1 + C.v2 + C.v3;
    C.lam = rc ? R.lam1 : R.lam0;
    C.mu = rc ? R.bt : 0ull;
    C.e8 = R.e8;
    C.hc = R.hc;
    C.p = R.p;
    C.umax = sel == 0 ? R.umax[0] : sel == 1 ? R.umax[1] : sel == 2 ? R.umax[2] : R.umax[3];
    C.c4 = (uint64_t)R.nlay * C.lam + C.mu;
    C.c5 = (uint64_t)R.nemb * C.e8;
    C.K = C.c4 + C.c5 + C.hc;
    if (STMAX && R.two) {
        const StEnt* x = st + (kg << S.lg_rcdo | sel);
        C.msL = __ldg(&x->msL);
        C.kL = __ldg(&x->kL);
        C.parL = __ldg(&x->parL);
        C.graL = __ldg(&x->graL);
        C.optimL = __ldg(&x->optimL);
        C.layL = __ldg(&x->layL);
        C.hcL = __ldg(&x->hcL);
    }
}

// one row's survivors: rounds of 32 consecutive positions of its window
// per-lane capacity counters: 16-bit fields, capacities 4j .. 4j + 3 in word j
// (the mask bits spread to bit 16 i by one multiply); flushed per unit
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
    __device__ __forceinline__ void flush(uint32_t (&capc)[NCAP]) {
#pragma unroll
        for (int q = 0; q < NCAP; q++) capc[q] += (uint32_t)(w[q / 4] >> (16 * (q % 4))) & 0xFFFFu;
#pragma unroll
        for (int j = 0; j < (NCAP + 3) / 4; j++) w[j] = 0;
    }
};

template <int MODE, int NCAP, bool GBS, bool STMAX>
__device__ __forceinline__ void fused_row(const DevSpace& S, const RowEnt& R, const StEnt* __restrict__ st,
                                          uint64_t kg, const DevPair* __restrict__ pairs, uint64_t lo, uint64_t hi,
                                          uint32_t cnt, uint64_t off, const Cols& cols, uint64_t capacity,
                                          CapPack<NCAP>& pk, uint32_t lane) {
    const uint64_t rs = R.rs;
    const uint32_t w = R.w;
    const uint32_t a = rs < lo ? (uint32_t)(lo - rs) : 0u;
    const uint32_t b = rs + w > hi ? (uint32_t)(hi - rs) : w;
    const bool all = cnt == b - a;  // every configuration of the window survives: no test
    const uint32_t sel = (a + lane) & ((1u << S.lg_rcdo) - 1u);  // 32 is a multiple of the digit count
    Lane C;
    lane_of<GBS, STMAX>(S, R, st, kg, sel, C);
    const bool two = STMAX && R.two;
    const DevPair* pp = pairs + R.pair_off;
    const uint32_t lanes_lt = (1u << lane) - 1u;
    uint32_t done = 0;
    for (uint32_t p0 = a; p0 < b; p0 += 32) {
        const uint32_t pos = p0 + lane;
        const bool valid = pos < b;
        ME_CHECK(!valid || (pos >> S.lg_rcdo) < (w >> S.lg_rcdo));
        const DevPair pr = valid ? pp[pos >> S.lg_rcdo] : DevPair{0u, 0u};
        const uint32_t u = pr.u;
        uint64_t c4 = C.c4, c5 = C.c5, tot;
        if (GBS) {
            // in-flight counts of this pair's m microbatches (R17, R29)
            c4 = (uint64_t)n_layer_mb(C.p, S.vpp, pr.m) * C.lam + C.mu;
            c5 = (uint64_t)n_embed_mb(C.p, S.vpp, pr.m) * C.e8;
            tot = C.ms + (uint64_t)u * (c4 + c5 + C.hc);
        } else {
            tot = C.ms + (uint64_t)u * C.K;
        }
        bool s;
        if (all) {
            s = valid;
        } else if (!GBS) {
            s = valid && u <= C.umax;
        } else {
            uint64_t t2 = tot;
            if (two) {
                const uint64_t tl = C.msL + (uint64_t)u * C.kL;
                t2 = tl > t2 ? tl : t2;
            }
            s = valid && t2 <= S.thr_max;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, s);
        if (s) {
            uint64_t v[8];
            v[1] = C.v1;
            v[2] = C.v2;
            v[3] = C.v3;
            v[4] = (uint64_t)u * c4;
            v[5] = (uint64_t)u * c5;
            v[6] = (uint64_t)u * C.hc;
            v[7] = tot;
            if (two) {
                const uint64_t tl = C.msL + (uint64_t)u * C.kL;
                if (tl > tot) {  // the last stage decides (ties: stage 0)
                    v[1] = C.parL;
                    v[2] = C.graL;
                    v[3] = C.optimL;
                    v[4] = (uint64_t)u * C.layL;
                    v[5] = 0;
                    v[6] = (uint64_t)u * C.hcL;
                    v[7] = tl;
                }
            }
            const uint32_t mask = cap_mask_n<NCAP>(S, ~v[7]);
            if (S.k3_caps) pk.add(mask);
            v[0] = (rs + pos) | ((uint64_t)mask << 56);
            const uint64_t o = off + done + __popc(bal & lanes_lt);
            if (o < capacity) {
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
        done += __popc(bal);
    }
    ME_CHECK(done == cnt);  // K3 finds exactly the survivors K0 counted
}


// The survivors of a whole row with few survivors per round, in two phases
// (DESIGN.md §6): (1) lane l takes pairs l, l + 32, ...: the bit mask of its
// surviving (rc, do) digits and, by a warp scan, the rank of its first
// survivor in the row; it writes the code (pair << 2 | digit) of each of its
// survivors to that rank's slot of the warp's shared list; (2) lane l takes
// survivors l, l + 32, ... of the row from the list, then the eight values
// and the store -- every lane of a round stores (32 consecutive rows of the
// output), whatever the survivor density.  Rows of the window [0, w) only.
constexpr uint32_t kRowPairs = kRowPairsSmem;  // pairs per row handled this way (4 codes each in the list)

template <int MODE, int NCAP, bool GBS, bool STMAX>
__device__ __forceinline__ void fused_row_pairs(const DevSpace& S, const RowEnt& R, const StEnt* __restrict__ st,
                                                uint64_t kg, const DevPair* __restrict__ pairs, uint32_t cnt,
                                                uint64_t off, const Cols& cols, uint64_t capacity,
                                                uint16_t* __restrict__ slist, CapPack<NCAP>& pk, uint32_t lane) {
    const uint32_t lg = S.lg_rcdo, n_sel = 1u << lg;
    const uint32_t n_pairs = R.w >> lg;
    const DevPair* pp = pairs + R.pair_off;
    const bool two = STMAX && R.two;
    const uint64_t psi = R.psi;
    // phase 1: survivor masks per pair -> codes of the survivors in row order
    uint32_t run = 0;
    for (uint32_t j0 = 0; j0 < n_pairs; j0 += 32) {
        const uint32_t j = j0 + lane;
        uint32_t m4 = 0;
        if (j < n_pairs) {
            const DevPair pr = pp[j];
#pragma unroll
            for (uint32_t sel = 0; sel < 4; sel++) {
                if (sel >= n_sel) break;
                bool sv;
                if (!GBS) {
                    sv = pr.u <= R.umax[sel];
                } else {
                    const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
                    const uint64_t K = (uint64_t)n_layer_mb(R.p, S.vpp, pr.m) * (rc ? R.lam1 : R.lam0) +
                                       (rc ? R.bt : 0ull) + (uint64_t)n_embed_mb(R.p, S.vpp, pr.m) * R.e8 + R.hc;
                    const uint64_t ms = dopt ? R.par1 + R.gra1 + R.optim1 : (uint64_t)(S.wb + S.gb + S.ob) * psi;
                    uint64_t t2 = ms + (uint64_t)pr.u * K;
                    if (two) {
                        const StEnt* x = st + (kg << lg | sel);
                        const uint64_t tl = __ldg(&x->msL) + (uint64_t)pr.u * __ldg(&x->kL);
                        t2 = tl > t2 ? tl : t2;
                    }
                    sv = t2 <= S.thr_max;
                }
                m4 |= (sv ? 1u : 0u) << sel;
            }
        }
        // the lanes' survivor counts (0..4) bit-sliced into three ballots:
        // exclusive prefix and warp total by popcounts (no shuffle chain)
        const uint32_t c = __popc(m4);
        const uint32_t b0 = __ballot_sync(0xffffffffu, c & 1u), b1 = __ballot_sync(0xffffffffu, c & 2u),
                       b2 = __ballot_sync(0xffffffffu, c & 4u);
        const uint32_t lt = (1u << lane) - 1u;
        const uint32_t at = run + __popc(b0 & lt) + 2u * __popc(b1 & lt) + 4u * __popc(b2 & lt);
        // the pair's survivor codes in digit order: predicated stores, no loop
#pragma unroll
        for (uint32_t sel = 0; sel < 4; sel++)
            if ((m4 >> sel) & 1u) {
                ME_CHECK(at + __popc(m4 & ((1u << sel) - 1u)) < kRowPairs * 4);
                slist[at + __popc(m4 & ((1u << sel) - 1u))] = (uint16_t)(j << 2 | sel);
            }
        run += __popc(b0) + 2u * __popc(b1) + 4u * __popc(b2);
    }
    __syncwarp();
    ME_CHECK(run == cnt);
    // phase 2: survivor k of the row -> (pair, digit) -> values -> row off + k
    for (uint32_t k0 = 0; k0 < cnt; k0 += 32) {
        const uint32_t k = k0 + lane;
        if (k < cnt) {
            const uint32_t code = slist[k];
            const uint32_t j = code >> 2, sel = code & 3u;
            const uint32_t rc = (S.rcdo_rc >> sel) & 1u, dopt = (S.rcdo_do >> sel) & 1u;
            const DevPair pr = pp[j];
            const uint32_t u = pr.u;
            const uint64_t lam = rc ? R.lam1 : R.lam0, mu = rc ? R.bt : 0ull;
            const uint32_t nl = GBS ? n_layer_mb(R.p, S.vpp, pr.m) : R.nlay;
            const uint32_t ne = GBS ? n_embed_mb(R.p, S.vpp, pr.m) : R.nemb;
            uint64_t v[8];
            v[1] = dopt ? R.par1 : (uint64_t)S.wb * psi;
            v[2] = dopt ? R.gra1 : (uint64_t)S.gb * psi;
            v[3] = dopt ? R.optim1 : (uint64_t)S.ob * psi;
            v[4] = (uint64_t)u * ((uint64_t)nl * lam + mu);
            v[5] = (uint64_t)u * ((uint64_t)ne * R.e8);
            v[6] = (uint64_t)u * R.hc;
            v[7] = v[1] + v[2] + v[3] + v[4] + v[5] + v[6];
            if (two) {
                const StEnt* x = st + (kg << lg | sel);
                const uint64_t tl = __ldg(&x->msL) + (uint64_t)u * __ldg(&x->kL);
                if (tl > v[7]) {  // the last stage decides (ties: stage 0)
                    v[1] = __ldg(&x->parL);
                    v[2] = __ldg(&x->graL);
                    v[3] = __ldg(&x->optimL);
                    v[4] = (uint64_t)u * __ldg(&x->layL);
                    v[5] = 0;
                    v[6] = (uint64_t)u * __ldg(&x->hcL);
                    v[7] = tl;
                }
            }
            const uint32_t mask = cap_mask_n<NCAP>(S, ~v[7]);
            if (S.k3_caps) pk.add(mask);
            v[0] = (R.rs + (j << lg | sel)) | ((uint64_t)mask << 56);
            const uint64_t o = off + k;
            if (o < capacity) {
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
    __syncwarp();  // slist is reused by the next row
}

template <int MODE, int NCAP, bool GBS, bool STMAX>
__device__ __forceinline__ void fused_units(const DevSpace& S, const RowEnt* __restrict__ rows,
                                            const StEnt* __restrict__ st, const uint32_t* __restrict__ rcnt,
                                            const uint32_t* __restrict__ ucnt, const uint64_t* __restrict__ uoff,
                                            uint32_t n_rows, uint32_t n_units, uint64_t lo, uint64_t hi,
                                            const Cols& cols, uint64_t capacity, const DevPair* pairs,
                                            RowEnt* srow, uint16_t* slist, uint32_t* next_unit,
                                            uint32_t (&capc)[NCAP]) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t unit = 0;
    while (true) {
        // units are taken in order from a counter (their survivors vary)
        if (lane == 0) unit = atomicAdd(next_unit, 1u);
        unit = __shfl_sync(0xffffffffu, unit, 0);
        if (unit >= n_units) break;
        if (!__ldg(ucnt + unit)) continue;
        const uint32_t k0 = unit * kUnit;
        ME_CHECK(k0 < n_rows);
        const uint32_t nr = min(kUnit, n_rows - k0);
        // the unit's rows into the warp's shared copy: asynchronous 16-byte
        // copies (cp.async), in flight while the counts and the offset load
        __syncwarp();  // the previous unit's readers are done with srow
        {
            const uint4* src = reinterpret_cast<const uint4*>(rows + k0);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(srow);
            const uint32_t n16 = nr * (uint32_t)(sizeof(RowEnt) / 16);
            for (uint32_t i = lane; i < n16; i += 32)
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + i * 16), "l"(src + i) : "memory");
            asm volatile("cp.async.commit_group;" ::: "memory");
        }
        const uint32_t c = lane < nr ? __ldg(rcnt + k0 + lane) : 0u;
        const uint64_t base = __ldg(uoff + unit);
        uint32_t inc = c;  // inclusive warp scan of the row counts
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncwarp();
        uint32_t nz = __ballot_sync(0xffffffffu, c != 0);
        CapPack<NCAP> pk;  // <= 32 rows x w / 32 survivors per lane per unit: fits 16 bits
        while (nz) {
            const uint32_t i = __ffs(nz) - 1;
            nz &= nz - 1;
            ME_CHECK(i < nr);
            const uint32_t ci = __shfl_sync(0xffffffffu, c, i);
            const uint64_t oi = base + (__shfl_sync(0xffffffffu, inc, i) - ci);
            const RowEnt& R = srow[i];
            // whole rows whose survivors would fill few lanes of a positional
            // round: the two-phase path (every lane stores); else positional
            const bool whole = R.rs >= lo && R.rs + R.w <= hi;
            if (whole && ci != R.w && (R.w >> S.lg_rcdo) <= kRowPairs && S.sparse && ci * S.sparse < R.w)
                fused_row_pairs<MODE, NCAP, GBS, STMAX>(S, R, st, (uint64_t)k0 + i, pairs, ci, oi, cols, capacity,
                                                        slist, pk, lane);
            else
                fused_row<MODE, NCAP, GBS, STMAX>(S, R, st, (uint64_t)k0 + i, pairs, lo, hi, ci, oi, cols,
                                                  capacity, pk, lane);
        }
        pk.flush(capc);
    }
}

// stats[1 + j] += survivors for capacity j (one atomic per block and capacity)
// MINB: resident blocks per SM the registers are budgeted for (2: 16 warps
// and room for K0 of the next sub-range beside them; 3: 24 warps, <= 80
// registers)
template <int MODE, int NCAP, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    fused_kernel(const DevSpace S, const RowEnt* __restrict__ rows, const StEnt* __restrict__ st,
                 const uint32_t* __restrict__ rcnt, const uint32_t* __restrict__ ucnt,
                 const uint64_t* __restrict__ uoff, const uint32_t n_rows, const uint32_t n_units, const uint64_t lo,
                 const uint64_t hi, const Cols cols, const uint64_t capacity, uint32_t* __restrict__ next_unit,
                 uint64_t* __restrict__ stats) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint32_t s_cap[NCAP];
    if (threadIdx.x < NCAP) s_cap[threadIdx.x] = 0;
    DevPair* s_pairs = reinterpret_cast<DevPair*>(smem);
    RowEnt* s_rows = reinterpret_cast<RowEnt*>(smem + kPairsSmem * sizeof(DevPair));
    const bool pairs_smem = S.n_pairs <= kPairsSmem;
    if (pairs_smem)
        for (uint32_t i = threadIdx.x; i < S.n_pairs; i += blockDim.x) s_pairs[i] = S.pairs[i];
    ME_CHECK(kPairsSmem * sizeof(DevPair) + (threadIdx.x >> 5) * kUnit * sizeof(RowEnt) + kUnit * sizeof(RowEnt) <=
             kFusedSmemBytes);
    __syncthreads();
    const DevPair* pairs = pairs_smem ? s_pairs : S.pairs;
    RowEnt* srow = s_rows + (threadIdx.x >> 5) * kUnit;
    uint16_t* slist = reinterpret_cast<uint16_t*>(smem + kPairsSmem * sizeof(DevPair) +
                                                  (size_t)kFusedWarps * kUnit * sizeof(RowEnt)) +
                      (threadIdx.x >> 5) * kRowPairsSmem * 4;
    uint32_t capc[NCAP];
#pragma unroll
    for (int q = 0; q < NCAP; q++) capc[q] = 0;
#define ME_FUSED(GBS, STMAX)                                                                                     \
    fused_units<MODE, NCAP, GBS, STMAX>(S, rows, st, rcnt, ucnt, uoff, n_rows, n_units, lo, hi, cols, capacity, \
                                        pairs, srow, slist, next_unit, capc)
    if (S.stage_max) {
        if (S.gbs_mode) ME_FUSED(true, true);
        else ME_FUSED(false, true);
    } else {
        if (S.gbs_mode) ME_FUSED(true, false);
        else ME_FUSED(false, false);
    }
#undef ME_FUSED
#pragma unroll
    for (int q = 0; q < NCAP; q++) {
        const uint32_t c = __reduce_add_sync(0xffffffffu, capc[q]);
        if ((threadIdx.x & 31) == 0 && c) atomicAdd(s_cap + q, c);
    }
    __syncthreads();
    if (threadIdx.x < NCAP && s_cap[threadIdx.x])
        atomicAdd((unsigned long long*)(stats + 1 + threadIdx.x), (unsigned long long)s_cap[threadIdx.x]);
}

constexpr size_t kFusedSmem = kFusedSmemBytes;

uint32_t ncap_pad3(uint32_t n_cap) { return n_cap <= 1 ? 1 : n_cap <= 2 ? 2 : n_cap <= 4 ? 4 : 8; }

template <int MODE, int MINB>
void* fused_fn_(uint32_t n_cap) {
    switch (ncap_pad3(n_cap)) {
        case 1: return reinterpret_cast<void*>(&fused_kernel<MODE, 1, MINB>);
        case 2: return reinterpret_cast<void*>(&fused_kernel<MODE, 2, MINB>);
        case 4: return reinterpret_cast<void*>(&fused_kernel<MODE, 4, MINB>);
        default: return reinterpret_cast<void*>(&fused_kernel<MODE, 8, MINB>);
    }
}
template <int MINB>
void* fused_fn_m(me_out_mode mode, uint32_t n_cap) {
    return mode == ME_OUT_RECORDS ? fused_fn_<3, MINB>(n_cap)
                                  : mode == ME_OUT_FULL ? fused_fn_<2, MINB>(n_cap) : fused_fn_<1, MINB>(n_cap);
}
void* fused_fn(me_out_mode mode, uint32_t n_cap, int minb) {
    return minb >= 3 ? fused_fn_m<3>(mode, n_cap) : fused_fn_m<2>(mode, n_cap);
}

template <bool CAPS, bool WR, int MINB, bool SMEM>
void* rowcount_fn_(uint32_t n_cap) {
    switch (ncap_pad3(n_cap)) {
        case 1: return reinterpret_cast<void*>(&rowcount_kernel<1, CAPS, WR, MINB, SMEM>);
        case 2: return reinterpret_cast<void*>(&rowcount_kernel<2, CAPS, WR, MINB, SMEM>);
        case 4: return reinterpret_cast<void*>(&rowcount_kernel<4, CAPS, WR, MINB, SMEM>);
        default: return reinterpret_cast<void*>(&rowcount_kernel<8, CAPS, WR, MINB, SMEM>);
    }
}
void* rowcount_fn(uint32_t n_cap, bool caps, bool wr, bool smem) {
    if (!wr) return smem ? rowcount_fn_<true, false, kRowMinbCount, true>(n_cap)
                         : rowcount_fn_<true, false, kRowMinbCount, false>(n_cap);
    return caps ? rowcount_fn_<true, true, kRowMinbWrite, false>(n_cap)
                : rowcount_fn_<false, true, kRowMinbWrite, false>(n_cap);
}
// count-only K0 stages the sorted-u lists when they fit the default 48 KB
size_t rowcount_smem(const DevSpace& S) {
    const size_t b = (((S.n_pairs + 3ull) & ~3ull) + (S.fenced ? S.n_fence : 0u)) * 4ull;
    return S.k0_smem && !S.gbs_mode && b <= 48u * 1024u ? b : 0;
}

}  // namespace

int fused_blocks_per_sm(me_out_mode mode, uint32_t n_cap, int minb) {
    void* fn = fused_fn(mode, n_cap, minb);
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFusedSmem) != cudaSuccess)
        return 1;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, fn, kThreads, kFusedSmem) != cudaSuccess) return 1;
    return nb > 0 ? nb : 1;
}

uint32_t fused_units_of(uint32_t n_rows) { return (n_rows + kUnit - 1) / kUnit; }

cudaError_t launch_rowcount(const DevSpace& S, uint64_t g0, uint32_t n_rows, uint32_t seg_lo, uint32_t n_seg_sub,
                            uint64_t lo, uint64_t hi, RowEnt* rows, StEnt* st, uint32_t* rcnt, uint32_t* ucnt,
                            uint64_t* stats, bool caps, bool write, uint32_t max_blocks, cudaStream_t stream) {
    uint32_t blocks = (n_rows + kRowThreads - 1) / kRowThreads;
    if (max_blocks && blocks > max_blocks) blocks = max_blocks;
    void* args[] = {(void*)&S,  (void*)&g0,   (void*)&n_rows, (void*)&seg_lo, (void*)&n_seg_sub, (void*)&lo,
                    (void*)&hi, (void*)&rows, (void*)&st,     (void*)&rcnt,   (void*)&ucnt,      (void*)&stats};
    const size_t smem = write ? 0 : rowcount_smem(S);
    return cudaLaunchKernel(rowcount_fn(S.n_cap, caps || !write, write, smem != 0), dim3(blocks ? blocks : 1),
                            dim3(kRowThreads), args, smem, stream);
}

int rowcount_blocks_per_sm(const DevSpace& S) {
    int nb = 0;
    const size_t smem = rowcount_smem(S);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, rowcount_fn(S.n_cap, true, false, smem != 0), kRowThreads,
                                                      smem) != cudaSuccess)
        return 1;
    return nb > 0 ? nb : 1;
}

cudaError_t launch_fused(const DevSpace& S, const RowEnt* rows, const StEnt* st, const uint32_t* rcnt,
                         const uint32_t* ucnt, const uint64_t* uoff, uint32_t n_rows, uint64_t lo, uint64_t hi,
                         me_out_mode mode, Cols cols, uint64_t capacity, uint32_t n_blocks, int minb,
                         uint32_t* next_unit, uint64_t* stats, cudaStream_t stream) {
    const uint32_t n_units = fused_units_of(n_rows);
    const uint32_t need = (n_units + kFusedWarps - 1) / kFusedWarps;
    if (n_blocks > need) n_blocks = need ? need : 1;
    void* args[] = {(void*)&S,      (void*)&rows,    (void*)&st, (void*)&rcnt, (void*)&ucnt,
                    (void*)&uoff,   (void*)&n_rows,  (void*)&n_units, (void*)&lo, (void*)&hi,
                    (void*)&cols,   (void*)&capacity, (void*)&next_unit, (void*)&stats};
    cudaError_t ce = cudaMemsetAsync(next_unit, 0, 4, stream);
    if (ce != cudaSuccess) return ce;
    return cudaLaunchKernel(fused_fn(mode, S.n_cap, minb), dim3(n_blocks), dim3(kThreads), args, kFusedSmem, stream);
}

}  // namespace me
