// me_dev.cuh -- small device helpers shared by the sweep kernels (sm_100a).
#pragma once
#include <cstdint>

#include "me_kernels.cuh"

// ME_CHECKS (the checked build, libme_checked.so; build.py): device-side
// bounds assertions on every table, scratch, shared-memory and output index
// the sweep kernels compute -- a failed check traps the kernel (the call then
// returns ME_ECUDA).  compiled out of libme.so.
#ifdef ME_CHECKS
#include <cassert>
#define ME_CHECK(cond) assert(cond)
#else
#define ME_CHECK(cond) ((void)0)
#endif

namespace me {

// total <= thr  <=>  thr1 + ~total carries out of 64 bits (thr1 = thr + 1):
// two 32-bit adds with carry and one add-with-carry into acc (acc = 2 acc + carry)
__device__ __forceinline__ uint32_t le_shift(uint32_t acc, uint64_t ntot, uint64_t thr1) {
    asm("{\n\t.reg .u32 t;\n\t"
        "add.cc.u32 t, %1, %2;\n\t"
        "addc.cc.u32 t, %3, %4;\n\t"
        "addc.u32 %0, %0, %0;\n\t}"
        : "+r"(acc)
        : "r"((uint32_t)ntot), "r"((uint32_t)thr1), "r"((uint32_t)(ntot >> 32)), "r"((uint32_t)(thr1 >> 32)));
    return acc;
}

// capacity mask of a total given as ~total: bit q <=> total <= thr_q (80% rule)
template <int NCAP>
__device__ __forceinline__ uint32_t cap_mask_n(const DevSpace& S, uint64_t ntot) {
    uint32_t mask = 0;
#pragma unroll
    for (int q = NCAP - 1; q >= 0; q--) mask = le_shift(mask, ntot, S.thr1[q]);
    return mask;
}

// one 64-byte record as two 32-byte stores (sm_100 STG.E.ENL2.256).  No
// "memory" clobber: the kernels never read what they store, so later loads may
// be scheduled ahead of these stores.
__device__ __forceinline__ void store_record(uint64_t* q, const uint64_t (&v)[8]) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(q), "l"(v[0]), "l"(v[1]), "l"(v[2]), "l"(v[3]));
    asm volatile("st.global.v4.u64 [%0+32], {%1, %2, %3, %4};" ::"l"(q), "l"(v[4]), "l"(v[5]), "l"(v[6]), "l"(v[7]));
}

__device__ __forceinline__ uint32_t upper_bound_u64(const uint64_t* __restrict__ a, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// the space's variant policy (me_cfg_range)
__device__ __forceinline__ Policy policy_of(const DevSpace& S) {
    return Policy{S.zero_stage, S.sp_off, S.vpp, S.wb, S.gb, S.ob};
}

// The row of sub-range table entry k (global row g): segment by binary search
// over the segments of the sub-range, then its model, tuple and first index.
struct RowId {
    DevModel M;
    DevTuple tu;
    uint64_t rs;  // flat index of the row's first configuration
    uint32_t L0;  // first-stage layers (R19)
};

// The segment holding row gw (seg_row[s] <= gw < seg_row[s + 1]) among
// segments [lo, lo + n): a 32-ary search by the whole warp (each step the 32
// lanes probe 32 evenly spaced segments; ~log32 n dependent loads instead of
// log2 n).  Every lane of the warp calls it with the same gw.
__device__ __forceinline__ uint32_t warp_segment(const uint64_t* __restrict__ seg_row, uint32_t lo, uint32_t n,
                                                 uint64_t gw) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t hi = lo + n;  // answer in [lo, hi)
    while (hi - lo > 1) {
        const uint32_t step = (hi - lo + 31) / 32;
        const uint32_t at = lo + lane * step;
        const bool le = at < hi && __ldg(seg_row + at) <= gw;
        const uint32_t last = 31 - __clz(__ballot_sync(0xffffffffu, le) | 1u);  // lane 0 probes lo: always true
        lo += last * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

// row_id given the segment of the warp's first row: a short forward walk (a
// warp's 32 consecutive rows span few segments)
__device__ __forceinline__ RowId row_id_from(const DevSpace& S, uint64_t g, uint32_t s) {
    RowId R;
    while (__ldg(S.seg_row + s + 1) <= g) s++;
    ME_CHECK(s < S.n_seg && __ldg(S.seg_row + s) <= g && g < __ldg(S.seg_row + s + 1));
    const uint32_t m = s / S.n_world, n = s - m * S.n_world;
    const uint4 m0 = __ldg(reinterpret_cast<const uint4*>(S.models + m));
    const uint4 m1 = __ldg(reinterpret_cast<const uint4*>(S.models + m) + 1);
    R.M = DevModel{m0.x, m0.y, m0.z, m0.w, m1.x, m1.y, m1.z, 0u};
    const uint32_t cls = __ldg(S.model_class + m);
    const uint32_t j = __ldg(S.list_off + cls * S.n_world + n) + (uint32_t)(g - __ldg(S.seg_row + s));
    ME_CHECK(j < __ldg(S.list_off + cls * S.n_world + n + 1));
    R.tu = S.tuples[__ldg(S.list_tuple + j)];
    ME_CHECK(R.tu.pair_off + R.tu.n_pairs <= S.n_pairs && R.tu.w == R.tu.n_pairs << S.lg_rcdo);
    R.rs = __ldg(S.seg_prefix + s) + __ldg(S.list_prefix + j);
    R.L0 = R.tu.p == 1 ? R.M.layers : div_u32(R.M.layers + R.tu.p - 1, R.tu.p);
    return R;
}

__device__ __forceinline__ RowId row_id(const DevSpace& S, uint64_t g, uint32_t seg_lo, uint32_t n_seg_sub) {
    return row_id_from(S, g, seg_lo + upper_bound_u64(S.seg_row + seg_lo, n_seg_sub, g) - 1);
}

// RowEnt of a row: make_row's coefficients, first index and pair slice
__device__ __forceinline__ RowEnt row_entry(const RowId& I, const RowCoef& R, bool two) {
    RowEnt e;
    e.w = I.tu.w;
    e.pair_off = I.tu.pair_off;
    e.p = I.tu.p;
    e.two = two ? 1u : 0u;
    e.nlay = R.nlay;
    e.nemb = R.nemb;
    e._r0 = e._r1 = 0;
    e.lam0 = R.lam0;
    e.lam1 = R.lam1;
    e.e8 = R.e8;
    e.bt = R.bt;
    e.hc = R.hc;
    e.psi = R.psi;
    e.par1 = R.par1;
    e.gra1 = R.gra1;
    e.optim1 = R.optim1;
    e.rs = I.rs;
    e.umax[0] = e.umax[1] = e.umax[2] = e.umax[3] = 0;
    return e;
}

// NEXT-1: the last stage (floor((L - L0)/(p - 1)) layers, one microbatch in
// flight) of a row for digit (rc, do), as per-token coefficients
__device__ __forceinline__ StEnt last_stage(const RowId& I, uint32_t rc, uint32_t dopt, const Policy& Q) {
    const uint32_t Ll = (I.M.layers - I.L0) / (I.tu.p - 1);
    const TermsT<uint64_t> T = stage_terms<uint64_t>(I.M, I.tu.t, I.tu.c, I.tu.d, false, true, Ll, 1u, 1u, rc, dopt, Q);
    StEnt x;
    x.msL = T.params + T.grads + T.optim;
    x.kL = T.layers + T.head;
    x.parL = T.params;
    x.graL = T.grads;
    x.optimL = T.optim;
    x.layL = T.layers;
    x.hcL = T.head;
    x._pad = 0;
    return x;
}

}  // namespace me
