// me_kernels.cu -- scan and single-configuration kernels (sm_100a).
//
//  scan             one block turns per-unit survivor counts into output
//                   offsets (adding the running total of earlier sub-ranges)
//                   and accumulates the totals;
//  estimate kernels me_estimate / me_estimate_batch / me_estimate_stage: one
//                   configuration per thread, the same make_row / config_terms
//                   device code as the sweeps, with an exact 128-bit shadow for
//                   the overflow verdict.
#include <cuda_runtime.h>

#include "me_kernels.cuh"

namespace me {

namespace {

// one block: exclusive scan of the unit counts into u64 offsets starting at
// the running total stats[0], which then holds the new running total.  Tiles
// of 4096 counts: one coalesced 16-byte load per thread, warp and block scans,
// 2 x 16-byte stores of the four offsets; the tile's total carries over.  (It
// sits between K0 and K3 of every sub-range, so its latency counts.)
constexpr uint32_t kScanThreads = 1024;
__global__ void __launch_bounds__(kScanThreads) scan_kernel(const uint32_t* __restrict__ counts, uint32_t n,
                                                           uint64_t* __restrict__ offs,
                                                           uint64_t* __restrict__ stats) {
    __shared__ uint64_t s_warp[32];
    __shared__ uint64_t s_carry;
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // (vector accesses when the caller's allocator returned 16-byte-aligned blocks)
    const bool vec = ((reinterpret_cast<uintptr_t>(counts) | reinterpret_cast<uintptr_t>(offs)) & 15u) == 0;
    if (tid == 0) s_carry = stats[0];
    for (uint32_t t0 = 0; t0 < n; t0 += 4 * kScanThreads) {
        const uint32_t i0 = t0 + 4 * tid;
        uint32_t c[4];
        if (vec && i0 + 3 < n) {
            const uint4 v = *reinterpret_cast<const uint4*>(counts + i0);
            c[0] = v.x, c[1] = v.y, c[2] = v.z, c[3] = v.w;
        } else {
#pragma unroll
            for (int k = 0; k < 4; k++) c[k] = i0 + k < n ? counts[i0 + k] : 0u;
        }
        const uint64_t sum = (uint64_t)c[0] + c[1] + c[2] + c[3];
        uint64_t inc = sum;  // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= (uint32_t)o) inc += y;
        }
        if (lane == 31) s_warp[wid] = inc;
        __syncthreads();  // (also orders s_carry's first write)
        if (wid == 0) {
            const uint64_t v = s_warp[lane];
            uint64_t x = v;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= (uint32_t)o) x += y;
            }
            s_warp[lane] = x - v;  // exclusive over warps
        }
        __syncthreads();
        uint64_t run = s_carry + s_warp[wid] + inc - sum;
        uint64_t o4[4];
#pragma unroll
        for (int k = 0; k < 4; k++) o4[k] = run, run += c[k];
        if (vec && i0 + 3 < n) {
            reinterpret_cast<ulonglong2*>(offs + i0)[0] = make_ulonglong2(o4[0], o4[1]);
            reinterpret_cast<ulonglong2*>(offs + i0)[1] = make_ulonglong2(o4[2], o4[3]);
        } else {
#pragma unroll
            for (int k = 0; k < 4; k++)
                if (i0 + k < n) offs[i0 + k] = o4[k];
        }
        __syncthreads();  // every thread has read s_carry and s_warp
        if (tid == kScanThreads - 1) s_carry = run;
    }
    __syncthreads();
    if (tid == 0) stats[0] = s_carry;
}


// a8 deferred join: g = every rank's per-block stats (nranks x kmax x 9, rank
// r's k-th block is global block q = k * nranks + r); out[0] = global
// survivors, out[1..8] per capacity, out[17 + k] = global position of this
// rank's k-th block (exclusive scan over q < n_blocks in order)
__global__ void __launch_bounds__(1024) join_kernel(const uint64_t* __restrict__ g, uint32_t nranks, uint32_t rank,
                                                    uint32_t kmax, uint64_t n_blocks, uint64_t* __restrict__ out) {
    __shared__ uint64_t s_warp[32];
    __shared__ uint64_t s_caps[8];
    const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (tid < 8) s_caps[tid] = 0;
    const uint64_t chunk = (n_blocks + blockDim.x - 1) / blockDim.x;
    const uint64_t lo = min(n_blocks, tid * chunk), hi = min(n_blocks, lo + chunk);
    auto row = [&](uint64_t q) { return g + ((q % nranks) * (uint64_t)kmax + q / nranks) * 9; };
    uint64_t sum = 0, caps[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (uint64_t q = lo; q < hi; q++) {
        const uint64_t* x = row(q);
        sum += x[0];
        for (int c = 0; c < 8; c++) caps[c] += x[1 + c];
    }
    __syncthreads();
    for (int c = 0; c < 8; c++) {
        uint64_t v = caps[c];
        for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
        if (lane == 0 && v) atomicAdd((unsigned long long*)&s_caps[c], (unsigned long long)v);
    }
    uint64_t inc = sum;
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= (uint32_t)o) inc += y;
    }
    if (lane == 31) s_warp[wid] = inc;
    __syncthreads();
    if (wid == 0) {
        const uint32_t nw = blockDim.x >> 5;
        const uint64_t v = lane < nw ? s_warp[lane] : 0;
        uint64_t x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        if (lane < nw) s_warp[lane] = x - v;
        if (lane == 31) out[0] = x;
    }
    __syncthreads();
    if (tid < 8) out[1 + tid] = s_caps[tid];
    uint64_t run = s_warp[wid] + inc - sum;
    for (uint64_t q = lo; q < hi; q++) {
        if (q % nranks == rank) out[17 + q / nranks] = run;
        run += row(q)[0];
    }
}

// ---- single configurations ----------------------------------------------
__device__ int estimate_one(const me_model& Min, const me_parallel& P, me_breakdown& out) {
    const me_model& M = Min;
    if (!M.hidden || !M.ffn_hidden || !M.layers || !M.heads || !M.kv_heads || !M.vocab)
        return ME_EINVAL;
    if (M.heads % M.kv_heads || M.hidden % M.heads) return ME_EINVAL;
    if (!P.dp || !P.tp || !P.pp || !P.cp || !P.mbs || !P.seq || P.zero_stage > 3) return ME_EINVAL;
    if (P.sp_off > 1 || P.w_bytes > 8 || P.g_bytes > 8 || P.o_bytes > 16) return ME_EINVAL;
    const uint32_t t = P.tp, c = P.cp, p = P.pp, d = P.dp, L = M.layers;
    if (P.vpp >= 2) {  // R29 interleaved 1F1B: p >= 2 stages of vpp chunks of L/(p vpp) layers
        if (P.allow_uneven_pp || P.first_stage_layers) return ME_EINVAL;
        if (p < 2 || L % (p * P.vpp)) return ME_EDIV;
        if (P.gbs && P.gbs % ((uint64_t)d * P.mbs) == 0 && (P.gbs / ((uint64_t)d * P.mbs)) % p) return ME_EDIV;
    }
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
    const Policy Q = make_policy(P.zero_stage, P.sp_off, P.vpp, P.w_bytes, P.g_bytes, P.o_bytes);
    RowCoefT<unsigned __int128> W;
    make_row(DM, t, c, p, d, L0, Q, W);
    const TermsT<unsigned __int128> T2 = config_terms(W, u, m, P.recompute ? 1u : 0u, P.dist_opt ? 1u : 0u, Q);
    const unsigned __int128 lim = (unsigned __int128)1 << 63;
    if (W.psi >= lim || W.ms0 >= lim || T2.total >= lim) return ME_EOVERFLOW;
    RowCoef R;
    make_row(DM, t, c, p, d, L0, Q, R);
    const TermsT<uint64_t> T = config_terms(R, u, m, P.recompute ? 1u : 0u, P.dist_opt ? 1u : 0u, Q);
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
    if (P.vpp >= 2) return ME_EINVAL;  // the per-stage view covers non-interleaved 1F1B
    const Policy Q = make_policy(P.zero_stage, P.sp_off, P.vpp, P.w_bytes, P.g_bytes, P.o_bytes);
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
                                                                           u, rc, dopt, Q);
        if (W.total >= lim) return ME_EOVERFLOW;
        const TermsT<uint64_t> T = stage_terms<uint64_t>(DM, t, c, d, i == 0, i == p - 1, Li, n_i, u, rc, dopt, Q);
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

}  // namespace

cudaError_t launch_scan(const uint32_t* counts, uint32_t n, uint64_t* offs, uint64_t* stats, cudaStream_t st) {
    scan_kernel<<<1, kScanThreads, 0, st>>>(counts, n, offs, stats);
    return cudaGetLastError();
}

cudaError_t launch_join(const uint64_t* gathered, int nranks, int rank, uint32_t kmax, uint64_t n_blocks,
                        uint64_t* out, cudaStream_t st) {
    join_kernel<<<1, 1024, 0, st>>>(gathered, (uint32_t)nranks, (uint32_t)rank, kmax, n_blocks, out);
    return cudaGetLastError();
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
