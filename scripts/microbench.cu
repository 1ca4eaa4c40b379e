// microbench.cu -- roofline denominators measured on this B200 (C-int-bench of
// SURVEY §2.7): HBM write-only / read-only / copy bandwidth with 16-byte
// accesses, and the integer issue rates of the ALU pipe (IADD3/LOP3), the FMA
// pipe (IMAD) and a 1:1 mix.  Prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o microbench microbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__global__ void k_write(uint4* __restrict__ p, size_t n, uint32_t v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(v, v + 1, v + 2, v + 3);
}
__global__ void k_read(const uint4* __restrict__ p, size_t n, uint32_t* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint4 x = __ldcs(p + i);
        acc ^= x.x ^ x.y ^ x.z ^ x.w;
    }
    if (acc == 0x12345678u) *sink = acc;
}
__global__ void k_copy(const uint4* __restrict__ a, uint4* __restrict__ b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        b[i] = __ldcs(a + i);
}
// 8-byte stores at 8-byte granularity (the sweep's column stores)
__global__ void k_write8(uint64_t* __restrict__ p, size_t n, uint64_t v) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = v + i;
}

// integer pipes: 8 independent chains per thread, ITER iterations
template <int KIND>
__global__ void k_int(uint32_t* out, int iters, uint32_t s) {
    uint32_t a[8];
#pragma unroll
    for (int j = 0; j < 8; j++) a[j] = threadIdx.x * (j + 3) + s;
    for (int it = 0; it < iters; it++) {
#pragma unroll
        for (int j = 0; j < 8; j++) {
            if (KIND == 0) {  // ALU: IADD3 / LOP3
                asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(s));
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(a[j]) : "r"(it));
            } else if (KIND == 1) {  // FMA pipe: IMAD
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(s | 1), "r"(it));
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(s | 3), "r"(j));
            } else {  // mix 1:1
                asm volatile("add.u32 %0, %0, %1;" : "+r"(a[j]) : "r"(s));
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(a[j]) : "r"(s | 1), "r"(it));
            }
        }
    }
    uint32_t x = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) x ^= a[j];
    if (x == 0xdeadbeefu) *out = x;
}

static float time_ms(cudaEvent_t a, cudaEvent_t b) {
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const size_t bytes = 8ull << 30;
    const size_t n16 = bytes / 16;
    uint4 *a, *b;
    uint32_t* sink;
    cudaMalloc(&a, bytes);
    cudaMalloc(&b, bytes);
    cudaMalloc(&sink, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int grids[] = {sms * 2, sms * 4, sms * 8, sms * 16, sms * 32};
    double best_w = 0, best_r = 0, best_c = 0, best_w8 = 0;
    for (int g : grids) {
        for (int rep = 0; rep < 4; rep++) {
            cudaEventRecord(e0);
            k_write<<<g, 256>>>(b, n16, rep);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            double gbs = bytes / (time_ms(e0, e1) * 1e6);
            if (rep && gbs > best_w) best_w = gbs;
            cudaEventRecord(e0);
            k_write8<<<g, 256>>>((uint64_t*)b, bytes / 8, rep);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            gbs = bytes / (time_ms(e0, e1) * 1e6);
            if (rep && gbs > best_w8) best_w8 = gbs;
            cudaEventRecord(e0);
            k_read<<<g, 256>>>(b, n16, sink);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            gbs = bytes / (time_ms(e0, e1) * 1e6);
            if (rep && gbs > best_r) best_r = gbs;
            cudaEventRecord(e0);
            k_copy<<<g, 256>>>(a, b, n16 / 2);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            gbs = bytes / (time_ms(e0, e1) * 1e6);  // read + write bytes
            if (rep && gbs > best_c) best_c = gbs;
        }
    }
    // integer issue: warp-instr per SM-cycle, from the measured SM clock
    double rate[3] = {0, 0, 0};
    const int iters = 4096, blocks = sms * 8, threads = 256;
    for (int kind = 0; kind < 3; kind++) {
        for (int rep = 0; rep < 3; rep++) {
            cudaEventRecord(e0);
            if (kind == 0) k_int<0><<<blocks, threads>>>(sink, iters, rep + 1);
            if (kind == 1) k_int<1><<<blocks, threads>>>(sink, iters, rep + 1);
            if (kind == 2) k_int<2><<<blocks, threads>>>(sink, iters, rep + 1);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            const double instr = (double)blocks * threads / 32 * iters * 16;  // warp instructions
            const double r = instr / (time_ms(e0, e1) * 1e-3);                 // warp-instr / s
            if (rep && r > rate[kind]) rate[kind] = r;
        }
    }
    printf("{\"sms\": %d, \"clock_mhz_attr\": %.0f, \"write_only_gbs\": %.1f, \"write8_gbs\": %.1f, "
           "\"read_only_gbs\": %.1f, \"copy_rw_gbs\": %.1f, \"alu_warp_instr_per_s\": %.4e, "
           "\"fma_warp_instr_per_s\": %.4e, \"mix_warp_instr_per_s\": %.4e}\n",
           sms, clk_khz / 1e3, best_w, best_w8, best_r, best_c, rate[0], rate[1], rate[2]);
    return 0;
}
