// INT-pipe modMAC ceiling of one B200 (SURVEY 8(d) "INT-pipe ceiling: measure with a modMAC
// microbenchmark"): every thread runs independent chains of acc += (u64) a * b (the INT engine's
// delayed-reduction modMAC, IMAD.WIDE.U32 in SASS), 148 x 8 CTAs of 256 threads.
// Prints modMACs/s of the whole GPU and per SM-clock.   nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int CH = 8, ITERS = 1 << 16;

__global__ void k_imad(const uint32_t *in, uint64_t *out)
{
    uint32_t a = in[threadIdx.x & 31] | 1u, b = in[(threadIdx.x + 7) & 31] | 3u;
    uint64_t acc[CH];
#pragma unroll
    for (int c = 0; c < CH; c++) acc[c] = c + threadIdx.x;
    for (int i = 0; i < ITERS; i++) {
#pragma unroll
        for (int c = 0; c < CH; c++) acc[c] += (uint64_t)(a + c) * b;
        a ^= (uint32_t)acc[0];
    }
    uint64_t s = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) s += acc[c];
    if (s == 0x12345) out[0] = s;
}

int main()
{
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    uint32_t *in;
    uint64_t *out;
    cudaMalloc(&in, 128);
    cudaMalloc(&out, 8);
    cudaMemset(in, 0x5a, 128);
    const int grid = sms * 8, block = 256;
    k_imad<<<grid, block>>>(in, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int r = 0; r < 5; r++) {
        cudaEventRecord(e0);
        k_imad<<<grid, block>>>(in, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    const double ops = (double)grid * block * ITERS * CH;
    const double rate = ops / (best / 1e3);
    printf("{\"int_modmac_T_per_s\": %.3f, \"sms\": %d, \"max_clock_mhz\": %d, "
           "\"modmac_per_clk_per_sm_at_max_clock\": %.1f, \"how\": \"acc += (u64)a*b chains, %d x %d threads, best of 5\"}\n",
           rate / 1e12, sms, clk / 1000, rate / sms / (clk * 1e3), grid, block);
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
