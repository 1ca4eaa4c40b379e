// storebench2.cu -- store patterns of 64-byte records (RECORDS output):
//   0: lane l writes record l of a 32-record block: two 32-B stores (v4.u64) at 64 l, 64 l + 32
//   1: the block written as two fully contiguous 1-KB warp stores (lane l: 32 B at 32 l, 1024 + 32 l)
//   2: four fully contiguous 512-B warp stores (lane l: 16 B at 16 l + 512 k)
// Each warp writes `blocks_per_warp` consecutive 2-KB blocks; grid = SMs x 32 warps.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o storebench2 storebench2.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ void st256(uint64_t* q, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(q), "l"(a), "l"(b), "l"(c), "l"(d));
}
__device__ __forceinline__ void st128(uint64_t* q, uint64_t a, uint64_t b) {
    asm volatile("st.global.v2.u64 [%0], {%1, %2};" ::"l"(q), "l"(a), "l"(b));
}

template <int P>
__global__ void __launch_bounds__(256) k(uint64_t* out, uint64_t n_blocks, uint32_t per_warp) {
    const uint32_t lane = threadIdx.x & 31;
    const uint64_t gw = blockIdx.x * 8ull + (threadIdx.x >> 5);
    const uint64_t nw = gridDim.x * 8ull;
    for (uint64_t b0 = gw * per_warp; b0 < n_blocks; b0 += nw * per_warp) {
        for (uint32_t i = 0; i < per_warp && b0 + i < n_blocks; i++) {
            uint64_t* blk = out + (b0 + i) * 256;  // 2 KB = 256 u64
            const uint64_t v = b0 + i + lane;
            if (P == 0) {
                st256(blk + lane * 8, v, v + 1, v + 2, v + 3);
                st256(blk + lane * 8 + 4, v + 4, v + 5, v + 6, v + 7);
            } else if (P == 1) {
                st256(blk + lane * 4, v, v + 1, v + 2, v + 3);
                st256(blk + 128 + lane * 4, v + 4, v + 5, v + 6, v + 7);
            } else {
#pragma unroll
                for (int q = 0; q < 4; q++) st128(blk + q * 64 + lane * 2, v + q, v + q + 1);
            }
        }
    }
}

int main() {
    const uint64_t bytes = 8ull << 30;
    const uint64_t n_blocks = bytes / 2048;
    uint64_t* out;
    cudaMalloc(&out, bytes);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int p = 0; p < 3; p++)
        for (uint32_t per : {1u, 8u, 64u}) {
            float best = 1e30f;
            for (int rep = 0; rep < 4; rep++) {
                cudaEventRecord(e0);
                if (p == 0) k<0><<<sms * 4, 256>>>(out, n_blocks, per);
                else if (p == 1) k<1><<<sms * 4, 256>>>(out, n_blocks, per);
                else k<2><<<sms * 4, 256>>>(out, n_blocks, per);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                if (rep && ms < best) best = ms;
            }
            printf("{\"pattern\": %d, \"blocks_per_warp\": %u, \"gbs\": %.1f}\n", p, per, bytes / (best * 1e6));
        }
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
    return 0;
}
