// tools/microbench.cu -- measures the integer issue rates the roofline uses
// (DESIGN.md section 7): LOP3/IADD3 ALU-pipe throughput, IMAD (FMA pipe), and the
// warp primitives of the walk kernel (MATCH.ANY u32/u64, SHFL, VOTE).
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/microbench tools/microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define ITERS 4096

__global__ void k_lop3(uint32_t *out, uint32_t seed)
{
    uint32_t a = seed ^ threadIdx.x, b = a * 3u, c = a + 7u, d = a ^ 0x55u;
    uint32_t e = a + 1, f = b + 1, g = c + 1, h = d + 1;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a = (a & b) ^ c; b = (b | c) ^ d; c = (c ^ d) & a; d = (d + a) ^ b;
        e = (e & f) ^ g; f = (f | g) ^ h; g = (g ^ h) & e; h = (h + e) ^ f;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d ^ e ^ f ^ g ^ h;
}

__global__ void k_imad(uint32_t *out, uint32_t seed)
{
    uint32_t a = seed ^ threadIdx.x, b = a * 3u, c = a + 7u, d = a ^ 0x55u;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a = a * 0xD2511F53u + b; b = b * 0xCD9E8D57u + c; c = c * 0x9E3779B9u + d; d = d * 0xBB67AE85u + a;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

__global__ void k_match32(uint32_t *out, uint32_t seed)
{
    uint32_t a = (seed ^ threadIdx.x) & 7u, b = a + 1, c = a + 2, d = a + 3;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a = __match_any_sync(0xffffffffu, a) & 15u; b = __match_any_sync(0xffffffffu, b) & 15u;
        c = __match_any_sync(0xffffffffu, c) & 15u; d = __match_any_sync(0xffffffffu, d) & 15u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

__global__ void k_match64(uint32_t *out, uint32_t seed)
{
    unsigned long long a = (seed ^ threadIdx.x) & 7u, b = a + 1, c = a + 2, d = a + 3;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a = __match_any_sync(0xffffffffu, a) & 15u; b = __match_any_sync(0xffffffffu, b) & 15u;
        c = __match_any_sync(0xffffffffu, c) & 15u; d = __match_any_sync(0xffffffffu, d) & 15u;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = (uint32_t)(a ^ b ^ c ^ d);
}

__global__ void k_shfl(uint32_t *out, uint32_t seed)
{
    uint32_t a = seed ^ threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a = __shfl_sync(0xffffffffu, a, b & 31); b = __shfl_sync(0xffffffffu, b, c & 31);
        c = __shfl_sync(0xffffffffu, c, d & 31); d = __shfl_sync(0xffffffffu, d, a & 31);
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

__global__ void k_vote(uint32_t *out, uint32_t seed)
{
    uint32_t a = seed ^ threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a = __ballot_sync(0xffffffffu, a & 1) + b; b = __ballot_sync(0xffffffffu, b & 2) + c;
        c = __ballot_sync(0xffffffffu, c & 4) + d; d = __ballot_sync(0xffffffffu, d & 8) + a;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = a ^ b ^ c ^ d;
}

template <typename K>
double run(K kern, const char *name, double ops_per_iter, int blocks_per_sm, int threads, int sms, uint32_t *buf,
           double base_mhz)
{
    const int blocks = sms * blocks_per_sm;
    kern<<<blocks, threads>>>(buf, 1);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) kern<<<blocks, threads>>>(buf, r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double warp_inst = 5.0 * blocks * (threads / 32) * (double)ITERS * ops_per_iter;
    const double rate = warp_inst / (ms / 1e3);                 // warp-instructions / s
    const double per_clk_sm = rate / (base_mhz * 1e6) / sms;   // warp-instr / clk / SM
    printf("%-10s %8.3f ms  %8.1f G warp-inst/s  %6.3f warp-inst/clk/SM @%.0f MHz  (%6.2f T lane-ops/s)\n",
           name, ms, rate / 1e9, per_clk_sm, base_mhz, rate * 32 / 1e12);
    return per_clk_sm;
}

int main(int argc, char **argv)
{
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    const double mhz = argc > 1 ? atof(argv[1]) : clk_khz / 1000.0;
    uint32_t *buf;
    cudaMalloc(&buf, 1 << 26);
    printf("SMs %d, nominal clock %.0f MHz (rates per clk use %.0f MHz)\n", sms, clk_khz / 1000.0, mhz);
    run(k_lop3, "LOP3/IADD", 171.0 / 16, 8, 256, sms, buf, mhz);
    run(k_imad, "IMAD", 4, 8, 256, sms, buf, mhz);
    run(k_match32, "MATCH.32", 8, 8, 256, sms, buf, mhz);   // match + LOP per op
    run(k_match64, "MATCH.64", 8, 8, 256, sms, buf, mhz);
    run(k_shfl, "SHFL", 8, 8, 256, sms, buf, mhz);          // shfl + LOP per op
    run(k_vote, "VOTE", 306.0 / 16, 8, 256, sms, buf, mhz);
    cudaFree(buf);
    return 0;
}
