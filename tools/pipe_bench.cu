// pipe_bench.cu -- register-only throughput microbenchmarks on B200 (integer / FP64 pipes), used to
// derive the ALU roofline of the NTT.  Build: nvcc -O3 -arch=sm_100a -o pipe_bench pipe_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "../paper_2205_11935_b200/csrc/common.cuh"

#define ITERS 4096
#define CHAINS 16

__global__ void k_dfma(double* out, double a, double b)
{
    double x[CHAINS];
    for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) x[i] = fma(x[i], a, b);
    double s = 0;
    for (int i = 0; i < CHAINS; ++i) s += x[i];
    if (s == 1.2345) out[0] = s;
}

__global__ void k_imad_wide(uint64_t* out, uint32_t a)
{
    uint64_t x[CHAINS];
    for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) x[i] = (uint64_t)(uint32_t)x[i] * a + (x[i] >> 32);
    uint64_t s = 0;
    for (int i = 0; i < CHAINS; ++i) s += x[i];
    if (s == 12345) out[0] = s;
}

__global__ void k_iadd3(uint32_t* out, uint32_t a, uint32_t b)
{
    uint32_t x[CHAINS];
    for (int i = 0; i < CHAINS; ++i) x[i] = threadIdx.x + i;
    for (int it = 0; it < ITERS; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; ++i) x[i] = x[i] + a + (b ^ i);
    uint32_t s = 0;
    for (int i = 0; i < CHAINS; ++i) s += x[i];
    if (s == 12345) out[0] = s;
}

// the NTT's 64-bit Shoup Cooley-Tukey butterfly (BIG class, Harvey lazy)
__global__ void k_butterfly(uint64_t* out, uint64_t q, uint64_t w, uint64_t ws)
{
    uint64_t x[CHAINS];
    for (int i = 0; i < CHAINS; ++i) x[i] = (threadIdx.x * 7919ULL + i) % q;
    const uint64_t q2 = 2 * q;
    for (int it = 0; it < ITERS / 2; ++it)
#pragma unroll
        for (int i = 0; i < CHAINS; i += 2) {
            const uint64_t xx = csub(x[i], q2);
            const uint64_t t = shoup_mul(x[i + 1], w, ws, q);
            x[i] = xx + t;
            x[i + 1] = xx - t + q2;
        }
    uint64_t s = 0;
    for (int i = 0; i < CHAINS; ++i) s += x[i];
    if (s == 12345) out[0] = s;
}

// FP64 tensor-core MMA (DMMA) throughput: m16n8k4 f64 (512 FMA per warp instruction)
__global__ void k_dmma(double* out, double a, double b)
{
    double acc[CHAINS / 4][4];
    for (int c = 0; c < CHAINS / 4; ++c)
        for (int i = 0; i < 4; ++i) acc[c][i] = threadIdx.x + i;
    const double a0 = a + threadIdx.x, a1 = a - threadIdx.x, b0 = b + threadIdx.x;
    for (int it = 0; it < ITERS / 4; ++it)
#pragma unroll
        for (int c = 0; c < CHAINS / 4; ++c)
            asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                         : "+d"(acc[c][0]), "+d"(acc[c][1]), "+d"(acc[c][2]), "+d"(acc[c][3])
                         : "d"(a0), "d"(a1), "d"(b0));
    double s = 0;
    for (int c = 0; c < CHAINS / 4; ++c)
        for (int i = 0; i < 4; ++i) s += acc[c][i];
    if (s == 1.2345) out[0] = s;
}

int main()
{
    int dev = 0, sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
    void* buf;
    cudaMalloc(&buf, 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int blocks = sms * 8, threads = 256;
    const double lanes = (double)blocks * threads;
    auto run = [&](const char* name, auto launch, double ops_per_lane, const char* unit) {
        launch();
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        for (int r = 0; r < 5; ++r) launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double rate = lanes * ops_per_lane * 5 / (ms * 1e-3);
        printf("{\"bench\": \"%s\", \"rate\": %.4g, \"unit\": \"%s\", \"per_sm_per_clk_at_max\": %.2f}\n", name, rate,
               unit, rate / sms / (clk * 1e3));
    };
    run("dfma", [&] { k_dfma<<<blocks, threads>>>((double*)buf, 1.0000001, 1e-9); }, (double)ITERS * CHAINS, "DFMA/s");
    run("imad_wide", [&] { k_imad_wide<<<blocks, threads>>>((uint64_t*)buf, 2654435761u); }, (double)ITERS * CHAINS,
        "IMAD.WIDE(+IADD)/s");
    run("iadd3", [&] { k_iadd3<<<blocks, threads>>>((uint32_t*)buf, 3, 5); }, (double)ITERS * CHAINS, "IADD3/s");
    // per thread: (ITERS/4) x (CHAINS/4) mma, each 512 FMA per warp = 16 per thread
    run("dmma_m16n8k4", [&] { k_dmma<<<blocks, threads>>>((double*)buf, 1.0000001, 1e-9); },
        (double)(ITERS / 4) * (CHAINS / 4) * 16.0, "FP64 tensor FMA/s");
    const uint64_t q = 1099510054913ULL, w = 123456789ULL;
    const uint64_t ws = (uint64_t)(((unsigned __int128)w << 64) / q);
    run("shoup_butterfly_64", [&] { k_butterfly<<<blocks, threads>>>((uint64_t*)buf, q, w, ws); },
        (double)(ITERS / 2) * (CHAINS / 2), "butterflies/s");
    printf("{\"sms\": %d, \"clock_khz\": %d}\n", sms, clk);
    return 0;
}
