// kinternal.cuh -- helpers shared by the kernel translation units (internal).
#pragma once
#include "common.cuh"
#include "ntt.cuh"
#include "ntt_c.cuh"
#include "kernels.h"
#include <algorithm>
#include <cstdlib>
#include <stdexcept>
#include <string>

namespace ck {

// ------------------------------------------------------------------------------------ helpers
__device__ __forceinline__ const u64* twp(const DCtx* dc, int p) { return dc->tw + (size_t)p * CK_TW_WORDS * dc->n; }
// (w, w/q) pair tables of the cluster schedule (ntt_c.cuh): forward, inverse
__device__ __forceinline__ const double2* twq_fwd(const DCtx* dc, int p) { return reinterpret_cast<const double2*>(twp(dc, p) + 8 * dc->n); }
__device__ __forceinline__ const ulonglong2* twq_fwd_int(const DCtx* dc, int p) { return reinterpret_cast<const ulonglong2*>(twp(dc, p) + 12 * dc->n); }
__device__ __forceinline__ const double2* twq_inv(const DCtx* dc, int p) { return reinterpret_cast<const double2*>(twp(dc, p) + 10 * dc->n); }

// NTT-domain automorphism (R3): out[k] = in[src(k)] with 2 brev(src)+1 = g (2 brev(k)+1) mod 2N
__device__ __forceinline__ int galois_src(int k, u32 g, int logn)
{
    const u32 e = 2u * brev32((u32)k, logn) + 1u;
    const u32 eg = (e * g) & ((2u << logn) - 1u);
    return (int)brev32((eg - 1u) >> 1, logn);
}

// g^{-1} mod 2N for an odd g (Newton: x <- x (2 - g x) doubles the correct low bits; g g = 1 mod 8)
__device__ __forceinline__ u32 galois_inv(u32 g, int logn)
{
    u32 x = g;
#pragma unroll
    for (int it = 0; it < 4; ++it) x *= 2u - g * x;
    return x & ((2u << logn) - 1u);
}
// sigma_g of an NTT-domain limb read in ITS OWN order: the value at index i belongs at k with galois_src(k, g) = i,
// i.e. k = galois_src(i, g^{-1}) -- the staging of the whole-limb inverse NTTs scatters in shared memory instead of
// gathering 8-byte words from global memory
__device__ __forceinline__ int galois_dst(int i, u32 ginv, int logn) { return galois_src(i, ginv, logn); }

static void check_launch(const char* what)
{
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

template <class K>
static void allow_smem(K kernel, size_t bytes)
{
    if (bytes > 48 * 1024) {
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    }
}

// launch with thread-block clusters of `cl` CTAs along x (grid.x is a multiple of cl)
template <class... KA, class... A>
static void launch_cluster(void (*kernel)(KA...), dim3 grid, int threads, size_t smem, cudaStream_t st, int cl, A... args)
{
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(threads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cl;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, static_cast<KA>(args)...);
    if (e != cudaSuccess) throw std::runtime_error(std::string("cluster launch: ") + cudaGetErrorString(e));
}

// Threads per CTA of the batched NTT kernel (k_ntt_batch): bit 16 set = 32 residues per thread (N/32 threads)
// for the forward, bit 32 for the inverse; clear = 16 (N/16 threads).  Default 16 (measured,
// tools/ab_nttbatch.sh); CKKS_NTT_WIDE overrides it (tuning experiments only).  The key-switching NTT
// kernels use fixed shapes: ModUp 32 residues per thread (compute-bound), the others 16.
static int ntt_wide_mask()
{
    static int mask = [] {
        const char* e = getenv("CKKS_NTT_WIDE");
        return e ? atoi(e) : 16;
    }();
    return mask;
}

#define NTT_DISPATCH(LOGN_VAR, ...)                                                     \
    switch (LOGN_VAR) {                                                                  \
    case 10: { constexpr int LG = 10; __VA_ARGS__; } break;                                     \
    case 11: { constexpr int LG = 11; __VA_ARGS__; } break;                                     \
    case 12: { constexpr int LG = 12; __VA_ARGS__; } break;                                     \
    case 13: { constexpr int LG = 13; __VA_ARGS__; } break;                                     \
    case 14: { constexpr int LG = 14; __VA_ARGS__; } break;                                     \
    default: throw std::runtime_error("unsupported log_n");                              \
    }

// ------------------------------------------------------------------------------------ PRNG (R15)
__device__ __forceinline__ u64 mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ u64 prng(u64 seed, u64 stream, u64 i)
{
    const u64 k = mix64(seed ^ mix64(stream));
    return mix64(k + (i + 1) * 0x9E3779B97F4A7C15ULL);
}
__device__ __forceinline__ u64 stream_tag(u64 purpose, u64 id, u64 digit, u64 prime)
{
    return (purpose << 56) | ((id & 0xFFFFFFFFFULL) << 20) | ((digit & 0x3FF) << 10) | (prime & 0x3FF);
}
__device__ __forceinline__ long long sample_small(const DCtx* dc, int kind, u64 seed, u64 stream, u64 i)
{
    const u64 r = prng(seed, stream, i);
    if (kind == 0) return (long long)(((r >> 32) * 3ULL) >> 32) - 1;   // ternary (R14)
    const int B = dc->cdt_bound;                                         // CDT Gaussian (R13)
    long long v = -B;
    for (int k = 0; k < 2 * B; ++k) v += (r >= dc->cdt[k]) ? 1 : 0;
    return v;
}
__device__ __forceinline__ u64 signed_to_res(long long x, const DPrime& P)
{
    if (x >= 0) return reduce64((u64)x, P);
    const u64 m = reduce64((u64)(-(x + 1)) + 1ULL, P);
    return m ? P.q - m : 0;
}

// active primes of key-switching digit j at nl data limbs (R9b: a digit is cut at the level)
__device__ __forceinline__ int digit_len_at(const DCtx* __restrict__ dc, int j, int nl)
{
    const int s0 = dc->dig_start[j];
    return min(dc->dig_len[j], nl - s0);
}

// FP64 tensor-core MMA m16n8k4 (exact for the split-operand products used here)
__device__ __forceinline__ void dmma16884(double (&c)[4], double a0, double a1, double b0)
{
    asm("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
        : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
        : "d"(a0), "d"(a1), "d"(b0));
}

}  // namespace ck
