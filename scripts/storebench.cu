// storebench.cu -- which column-store pattern reaches the HBM write roof?
// Each warp owns a contiguous region of every one of 8 u64 columns (like a
// tile of the write pass) and appends `run` consecutive rows per round to all 8
// columns, starting at row offset `skew` inside its region.
//   pattern 0: STG.64, run rows per round from lanes 0..run-1
//   pattern 1: STG.128, 2 rows per lane (run must be even, region 16-B aligned)
// Prints one JSON line per configuration.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o storebench storebench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

struct Cols {
    uint64_t* c[8];
};

template <int PATTERN>
__global__ void k_store(Cols cols, uint64_t rows_per_warp, uint32_t run, uint32_t skew, uint32_t n_warps_total) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t gw = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
    const uint32_t nw = gridDim.x * (blockDim.x / 32);
    for (uint32_t w = gw; w < n_warps_total; w += nw) {
        uint64_t row = (uint64_t)w * rows_per_warp + skew;
        const uint64_t end = (uint64_t)(w + 1) * rows_per_warp;
        for (; row + run <= end; row += run) {
            if (PATTERN == 0) {
                if (lane < run) {
#pragma unroll
                    for (int c = 0; c < 8; c++) cols.c[c][row + lane] = row + lane + c;
                }
            } else {
                if (2 * lane < run) {
#pragma unroll
                    for (int c = 0; c < 8; c++)
                        reinterpret_cast<ulonglong2*>(cols.c[c] + row)[lane] = make_ulonglong2(row + c, row + lane);
                }
            }
        }
    }
}

int main() {
    const uint64_t rows = 1ull << 27;  // per column (1 GiB each, 8 GiB total)
    Cols cols;
    for (int c = 0; c < 8; c++) cudaMalloc(&cols.c[c], rows * 8);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Cfg {
        int pattern;
        uint32_t run, skew, warps_per_sm;
        uint64_t rows_per_warp;
    };
    const Cfg cfgs[] = {
        {0, 32, 0, 16, 16384}, {0, 32, 1, 16, 16384}, {0, 25, 0, 16, 16384}, {0, 25, 3, 16, 16384},
        {0, 32, 0, 32, 16384}, {0, 25, 3, 32, 16384}, {1, 64, 0, 16, 16384}, {1, 64, 0, 32, 16384},
        {0, 32, 0, 16, 512},   {0, 25, 3, 16, 512},   {0, 32, 0, 16, 1 << 20}, {0, 25, 3, 16, 1 << 20},
    };
    for (const Cfg& c : cfgs) {
        const uint32_t n_warps = (uint32_t)(rows / c.rows_per_warp);
        const uint32_t blocks = sms * c.warps_per_sm / 8;
        float best = 1e30f;
        uint64_t written = 0;
        for (int rep = 0; rep < 4; rep++) {
            cudaEventRecord(e0);
            if (c.pattern == 0) k_store<0><<<blocks, 256>>>(cols, c.rows_per_warp, c.run, c.skew, n_warps);
            else k_store<1><<<blocks, 256>>>(cols, c.rows_per_warp, c.run, c.skew, n_warps);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep && ms < best) best = ms;
        }
        written = (uint64_t)n_warps * ((c.rows_per_warp - c.skew) / c.run) * c.run * 8 * 8;
        printf("{\"pattern\": %d, \"run\": %u, \"skew\": %u, \"warps_per_sm\": %u, \"rows_per_warp\": %llu, "
               "\"gbs\": %.1f}\n",
               c.pattern, c.run, c.skew, c.warps_per_sm, (unsigned long long)c.rows_per_warp,
               written / (best * 1e6));
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
