// ntt_lab.cu -- timing-only knock-out experiments on the quarter-schedule forward NTT (ntt_q.cuh).
// Build variants with -DKNOCK_TW (constant twiddles), -DKNOCK_LD (no global loads), -DKNOCK_ST (no global
// stores), -DPERSIST (grid = #SMs, loop over limbs), -DKNOCK_FP (no butterflies).  Values are garbage in the
// knock-outs; only the time matters.  nvcc -O3 -arch=sm_100a -I../../paper_2205_11935_b200/csrc ...
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "ntt_c.cuh"

#ifndef LAB_Q
#define LAB_Q 1099511480321ULL   /* a 40-bit prime-like modulus; arithmetic cost does not depend on it */
#endif

#ifndef LAB_MINB
#define LAB_MINB 1
#endif
#ifndef LAB_LOGN
#define LAB_LOGN 14
#endif
template <int LOGN>
__global__ void __launch_bounds__(NttC<LOGN>::NT, LAB_MINB)
k_lab(u64* __restrict__ data, const double2* __restrict__ TW, int nlimbs, DPrime Pr, int never)
{
    extern __shared__ u64 sm[];
    using TQ = NttC<LOGN>;
    {
        const int l = blockIdx.x / TQ::CL, h = blockIdx.x % TQ::CL;
        u64* a = data + (size_t)l * TQ::N;
#ifdef KNOCK_LD
        auto ld = [&](int i) { return (u64)(i + never); };
#else
        auto ld = [&](int i) { return a[i]; };
#endif
        u64* dst = a;
#ifdef LAB_R
        TQ::template forward_fp<true>(sm, h, Pr, TW, ld, dst);
#else
        TQ::template forward_fp<false>(sm, h, Pr, TW, ld, dst);
#endif
    }
}

int main(int argc, char** argv)
{
    constexpr int LOGN = LAB_LOGN;
    using TQ = NttC<LOGN>;
    const int nlimbs = argc > 1 ? atoi(argv[1]) : 8192;
    const int reps = 20;
    u64* d;
    double2* tw;
    cudaMalloc(&d, (size_t)nlimbs * TQ::N * 8);
    cudaMalloc(&tw, (size_t)TQ::N * 16);
    std::vector<u64> h((size_t)nlimbs * TQ::N);
    u64 s = 88172645463325252ULL;
    for (auto& v : h) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; v = s % LAB_Q; }
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    std::vector<double2> htw(TQ::N);
    for (auto& w : htw) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; w.x = (double)(s % LAB_Q); w.y = w.x / (double)LAB_Q; }
    cudaMemcpy(tw, htw.data(), htw.size() * 16, cudaMemcpyHostToDevice);
    DPrime Pr{};
    Pr.q = LAB_Q; Pr.q2 = 2 * LAB_Q; Pr.ninv = 1;
    const size_t smem = TQ::SMEM;
    cudaFuncSetAttribute(k_lab<LOGN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int grid = nlimbs * TQ::CL;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid); cfg.blockDim = dim3(TQ::NT); cfg.dynamicSmemBytes = smem; cfg.stream = 0;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    #ifdef NTTC_DUP
    at[0].val.clusterDim.x = 1;
#else
    at[0].val.clusterDim.x = TQ::CL;
#endif
    at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    for (int i = 0; i < 3; ++i) cudaLaunchKernelEx(&cfg, k_lab<LOGN>, d, (const double2*)tw, nlimbs, Pr, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) cudaLaunchKernelEx(&cfg, k_lab<LOGN>, d, (const double2*)tw, nlimbs, Pr, 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    ms /= reps;
    printf("%-40s %8.4f ms  %7.2f us/limb/SM  %8.1f GB/s  (%s)\n", LAB_NAME, ms, ms * 1e3 / ((double)nlimbs / sms),
           2.0 * nlimbs * TQ::N * 8 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
