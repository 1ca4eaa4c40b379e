// me_rank.cu -- NEXT-2 planner on the GPU: the k best configurations of every
// (model, N) segment of a sweep result, by the survey's rank key (SURVEY §8(f)
// NEXT-2; the heuristics of P:552-593):
//   1. class green < yellow < red  (caption P:420: <= 80%, <= 100%, > 100%)
//   2. t <= GPUs per node first
//   3. smallest t*c*p              "minimal combination of TP x CP x PP that does
//                                  not result in out-of-memory"
//   4. largest micro batch b
//   5. smallest p                  pipeline bubble (p-1)/m
//   6. smallest c, 7. smallest t   (TP-only first at equal t*c*p)
//   8. recompute off first, then the smallest flat index (determinism).
// The class comes from two capacity bits of the row's mask (green: feasible
// at the sweep threshold for the green slot; green or yellow: the yellow slot,
// e.g. 5C/4 at 4/5 = C at 100%).  Pass 1 packs the key of every result row
// into a u64 (smaller is better); pass 2 gives each segment (a contiguous run
// of result rows, rows being in index order) to one warp, which selects its k
// smallest (key, row) pairs by k rounds of a warp-wide minimum.
#include <cuda_runtime.h>

#include "me_dev.cuh"
#include "me_kernels.cuh"

namespace me {
namespace {

// packed key: [class:2][node:1][t*c*p:21][63-(b-1):6][p:9][c:21][rc:1][0:3]
__device__ __forceinline__ uint64_t rank_key(const DevSpace& S, uint64_t v, uint32_t green, uint32_t yellow,
                                             uint32_t gpn) {
    const uint64_t index = v & ((1ull << 56) - 1);
    const uint32_t mask = (uint32_t)(v >> 56);
    const uint32_t s = upper_bound_u64(S.seg_prefix, S.n_seg + 1, index) - 1;
    const uint32_t m = s / S.n_world, n = s - m * S.n_world;
    const uint32_t cls = __ldg(S.model_class + m);
    const uint32_t jb = __ldg(S.list_off + cls * S.n_world + n), je = __ldg(S.list_off + cls * S.n_world + n + 1);
    const uint64_t within = index - __ldg(S.seg_prefix + s);
    const uint32_t j = jb + upper_bound_u64(S.list_prefix + jb, je - jb, within) - 1;
    const uint32_t r = (uint32_t)(within - __ldg(S.list_prefix + j));
    const DevTuple tu = S.tuples[__ldg(S.list_tuple + j)];
    const uint32_t b = __ldg(S.pair_b + tu.pair_off + (r >> S.lg_rcdo));
    const uint32_t rc = (S.rcdo_rc >> (r & ((1u << S.lg_rcdo) - 1u))) & 1u;
    const uint64_t klass = (mask >> green) & 1u ? 0u : (yellow < 8 && ((mask >> yellow) & 1u) ? 1u : 2u);
    const uint64_t node = gpn && tu.t > gpn ? 1u : 0u;
    const uint64_t tcp = (uint64_t)tu.t * tu.c * tu.p;
    return (klass << 62) | (node << 61) | ((tcp & 0x1FFFFFu) << 40) | ((uint64_t)(63u - ((b - 1) & 63u)) << 34) |
           ((uint64_t)(tu.p & 511u) << 25) | ((uint64_t)(tu.c & 0x1FFFFFu) << 4) | ((uint64_t)rc << 3);
}

__global__ void rank_keys(const DevSpace S, const uint64_t* __restrict__ col, uint32_t stride, uint64_t n,
                          uint32_t green, uint32_t yellow, uint32_t gpn, uint64_t* __restrict__ keys) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = rank_key(S, __ldg(col + i * stride), green, yellow, gpn);
}

// first row whose flat index is >= x (rows ascending by index)
__device__ __forceinline__ uint64_t lower_row(const uint64_t* __restrict__ col, uint32_t stride, uint64_t n,
                                              uint64_t x) {
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if ((__ldg(col + mid * stride) & ((1ull << 56) - 1)) < x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// one warp per segment: its k best rows (row positions; ~0 past the end)
__global__ void rank_topk(const DevSpace S, const uint64_t* __restrict__ col, uint32_t stride, uint64_t n,
                          const uint64_t* __restrict__ keys, uint32_t k, uint64_t* __restrict__ sel) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t seg = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (seg >= S.n_seg) return;
    const uint64_t r0 = lower_row(col, stride, n, __ldg(S.seg_prefix + seg));
    const uint64_t r1 = lower_row(col, stride, n, __ldg(S.seg_prefix + seg + 1));
    uint64_t last_key = 0, last_row = 0;
    bool have = false;
    for (uint32_t q = 0; q < k; q++) {
        uint64_t bk = ~0ull, br = ~0ull;
        for (uint64_t r = r0 + lane; r < r1; r += 32) {
            const uint64_t kk = __ldg(keys + r);
            // strictly after the previous pick in (key, row) order
            if (have && (kk < last_key || (kk == last_key && r <= last_row))) continue;
            if (kk < bk || (kk == bk && r < br)) bk = kk, br = r;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, o), orow = __shfl_xor_sync(0xffffffffu, br, o);
            if (ok < bk || (ok == bk && orow < br)) bk = ok, br = orow;
        }
        if (lane == 0) sel[(uint64_t)seg * k + q] = br;
        if (br == ~0ull) {
            for (uint32_t z = q + 1; z < k && lane == 0; z++) sel[(uint64_t)seg * k + z] = ~0ull;
            break;
        }
        last_key = bk;
        last_row = br;
        have = true;
    }
}

// the selected rows' index|mask words and keys
__global__ void rank_gather(const uint64_t* __restrict__ col, uint32_t stride, const uint64_t* __restrict__ keys,
                            const uint64_t* __restrict__ sel, uint64_t m, uint64_t* __restrict__ out) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t r = sel[i];
        out[2 * i] = r == ~0ull ? ~0ull : __ldg(col + r * stride);
        out[2 * i + 1] = r == ~0ull ? ~0ull : __ldg(keys + r);
    }
}

}  // namespace

cudaError_t launch_rank(const DevSpace& S, const uint64_t* index_col, uint32_t stride, uint64_t n_rows,
                        uint32_t green, uint32_t yellow, uint32_t gpn, uint32_t k, uint64_t* keys, uint64_t* sel,
                        uint64_t* out, cudaStream_t st) {
    if (n_rows) {
        uint64_t blocks = (n_rows + 255) / 256;
        if (blocks > 148 * 32) blocks = 148 * 32;
        rank_keys<<<(unsigned)blocks, 256, 0, st>>>(S, index_col, stride, n_rows, green, yellow, gpn, keys);
    }
    const uint64_t warps = S.n_seg;
    rank_topk<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(S, index_col, stride, n_rows, keys, k, sel);
    const uint64_t m = (uint64_t)S.n_seg * k;
    uint64_t gb = (m + 255) / 256;
    if (gb > 148 * 32) gb = 148 * 32;
    rank_gather<<<(unsigned)(gb ? gb : 1), 256, 0, st>>>(index_col, stride, keys, sel, m, out);
    return cudaGetLastError();
}

}  // namespace me
