// me_rank.cu -- NEXT-2 planner on the GPU: the best feasible configuration of
// every (model, N) segment of a sweep result, by the paper's search heuristics
// (P:552-593), read as the rank key (reading R27):
//   1. smallest t*c*p          "minimal combination of TP x CP x PP that does
//                              not result in out-of-memory"
//   2. largest micro batch b   increasing MBS "consistently led to improved
//                              throughput"
//   3. smallest p              pipeline bubble (p-1)/m
//   4. smallest t              CP communicates less than TP at equal memory
//
//   5. recompute off first, then the smallest flat index (determinism).
// Rows are decoded from their flat index (one binary search per row); pass 1
// takes the segment minimum of the packed key, pass 2 the smallest index with
// that key.
#include <cuda_runtime.h>

#include "me_kernels.cuh"

namespace me {
namespace {

__device__ __forceinline__ uint32_t ub_u64(const uint64_t* __restrict__ a, uint32_t n, uint64_t x) {
    uint32_t lo = 0, hi = n;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldg(a + mid) <= x) lo = mid + 1;
        else hi = mid;
    }
    return lo;
}

// packed key: [t*c*p : 24][63 - (b - 1) : 6][p : 12][t : 20][rc : 1]; smaller is better
__device__ __forceinline__ bool rank_key(const DevSpace& S, uint64_t index, uint32_t& seg, uint64_t& key) {
    const uint32_t s = ub_u64(S.seg_prefix, S.n_seg + 1, index) - 1;
    const uint32_t m = s / S.n_world, n = s - m * S.n_world;
    const uint32_t cls = __ldg(S.model_class + m);
    const uint32_t jb = __ldg(S.list_off + cls * S.n_world + n), je = __ldg(S.list_off + cls * S.n_world + n + 1);
    const uint64_t within = index - __ldg(S.seg_prefix + s);
    const uint32_t j = jb + ub_u64(S.list_prefix + jb, je - jb, within) - 1;
    const uint32_t r = (uint32_t)(within - __ldg(S.list_prefix + j));
    const DevTuple tu = S.tuples[__ldg(S.list_tuple + j)];
    const uint32_t b = __ldg(S.pair_b + tu.pair_off + (r >> S.lg_rcdo));
    const uint32_t rc = (S.rcdo_rc >> (r & ((1u << S.lg_rcdo) - 1u))) & 1u;
    const uint64_t tcp = (uint64_t)tu.t * tu.c * tu.p;
    seg = s;
    key = (tcp << 39) | ((uint64_t)(63u - ((b - 1) & 63u)) << 33) | ((uint64_t)(tu.p & 4095u) << 21) |
          ((uint64_t)(tu.t & 0xFFFFFu) << 1) | rc;
    return true;
}

__global__ void rank_min_key(const DevSpace S, const uint64_t* __restrict__ col, uint32_t stride, uint64_t n,
                             uint32_t cap, unsigned long long* __restrict__ best_key) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = col[i * stride];
        if (!((v >> (56 + cap)) & 1u)) continue;  // not feasible for capacity `cap`
        uint32_t seg;
        uint64_t key;
        rank_key(S, v & ((1ull << 56) - 1), seg, key);
        atomicMin(best_key + seg, (unsigned long long)key);
    }
}

__global__ void rank_min_index(const DevSpace S, const uint64_t* __restrict__ col, uint32_t stride, uint64_t n,
                               uint32_t cap, const unsigned long long* __restrict__ best_key,
                               unsigned long long* __restrict__ best_index) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t v = col[i * stride];
        if (!((v >> (56 + cap)) & 1u)) continue;
        uint32_t seg;
        uint64_t key;
        const uint64_t index = v & ((1ull << 56) - 1);
        rank_key(S, index, seg, key);
        if (key == best_key[seg]) atomicMin(best_index + seg, (unsigned long long)index);
    }
}

}  // namespace

cudaError_t launch_rank(const DevSpace& S, const uint64_t* index_col, uint32_t stride, uint64_t n_rows, uint32_t cap,
                        uint64_t* best_key, uint64_t* best_index, cudaStream_t st) {
    if (!n_rows) return cudaSuccess;
    uint64_t blocks = (n_rows + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    rank_min_key<<<(unsigned)blocks, 256, 0, st>>>(S, index_col, stride, n_rows, cap, (unsigned long long*)best_key);
    rank_min_index<<<(unsigned)blocks, 256, 0, st>>>(S, index_col, stride, n_rows, cap,
                                                     (const unsigned long long*)best_key,
                                                     (unsigned long long*)best_index);
    return cudaGetLastError();
}

}  // namespace me
