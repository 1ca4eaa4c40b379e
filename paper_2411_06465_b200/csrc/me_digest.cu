// me_digest.cu -- order-dependent digest of a sweep result (me_result_digest).
//
// A verification device, not part of the method: it lets a whole result (or
// every rank's shard of it) be compared with an independent CPU enumeration
// without moving the rows.  Definition (include/me.h): for the row at
// position j with values r = (index|mask, params, grads, optim, act_layers,
// act_embed, act_head, total),
//   D_index  = sum_j mix(r_0 + C) * M^j                    (mod 2^64)
//   D_record = sum_j g(r) * M^j,  g: h <- C; h <- mix(h ^ r_k) for k = 0..7
// with mix the splitmix64 finaliser, C = 0x9E3779B97F4A7C15, M = 0xD1B54A32D192ED03.
// The sum is order-dependent through M^j and mergeable: D(A B) = D(A) + M^|A| D(B).
#include <cuda_runtime.h>

#include "me_kernels.cuh"

namespace me {
namespace {

constexpr uint64_t kDigC = 0x9E3779B97F4A7C15ull;
constexpr uint64_t kDigM = 0xD1B54A32D192ED03ull;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ull;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBull;
    x ^= x >> 31;
    return x;
}

__host__ __device__ __forceinline__ uint64_t pow_m(uint64_t n) {
    uint64_t r = 1, b = kDigM;
    while (n) {
        if (n & 1) r *= b;
        b *= b;
        n >>= 1;
    }
    return r;
}

struct ColPtrs {
    const uint64_t* c[ME_N_COLS];
};

// words = 8: one array of records (cols.c[0]); words = 1: n_cols columns
__global__ void digest_kernel(const ColPtrs cols, uint32_t n_cols, uint32_t words, uint64_t n,
                              unsigned long long* __restrict__ out) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    uint64_t pw = pow_m(j);
    const uint64_t pw_stride = pow_m(stride);
    uint64_t di = 0, dr = 0;
    const bool rec = words == 8 || n_cols == ME_N_COLS;
    for (; j < n; j += stride, pw *= pw_stride) {
        uint64_t r[8];
        if (words == 8) {
            const uint4* q = reinterpret_cast<const uint4*>(cols.c[0] + j * 8);
#pragma unroll
            for (int k = 0; k < 4; k++) {
                const uint4 x = __ldg(q + k);
                r[2 * k] = ((uint64_t)x.y << 32) | x.x;
                r[2 * k + 1] = ((uint64_t)x.w << 32) | x.z;
            }
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) r[k] = (k < (int)n_cols) ? __ldg(cols.c[k] + j) : 0ull;
        }
        di += mix64(r[0] + kDigC) * pw;
        if (rec) {
            uint64_t h = kDigC;
#pragma unroll
            for (int k = 0; k < 8; k++) h = mix64(h ^ r[k]);
            dr += h * pw;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        di += __shfl_down_sync(0xffffffffu, di, o);
        dr += __shfl_down_sync(0xffffffffu, dr, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out, (unsigned long long)di);  // wraps mod 2^64
        atomicAdd(out + 1, (unsigned long long)dr);
    }
}

}  // namespace

uint64_t digest_pow_host(uint64_t n) { return pow_m(n); }

cudaError_t launch_digest(const uint64_t* const* cols, uint32_t n_cols, uint32_t words, uint64_t n, uint64_t* out,
                          cudaStream_t stream) {
    cudaError_t ce = cudaMemsetAsync(out, 0, 16, stream);
    if (ce != cudaSuccess || !n) return ce;
    ColPtrs c{};
    for (uint32_t k = 0; k < n_cols && k < ME_N_COLS; k++) c.c[k] = cols[k];
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    digest_kernel<<<(unsigned)blocks, 256, 0, stream>>>(c, n_cols, words, n, (unsigned long long*)out);
    return cudaGetLastError();
}

}  // namespace me
