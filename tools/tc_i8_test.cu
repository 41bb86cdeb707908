// tc_i8_test.cu -- standalone check of the sm_100a 5th-generation tensor-core integer MMA used by the exact
// modular contractions (tcgen05.mma.cta_group::1.kind::i8, u8 x u8 -> s32 accumulators in TMEM):
//   (1) correctness: D[128][N] = A[128][K] . B[N][K]^T for K-major canonical (no-swizzle) shared-memory operands
//       against a CPU reference, several N and K;
//   (2) throughput: a persistent loop of MMAs on resident operands (int8 MAC/s per GPU).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tc_i8_test tools/tc_i8_test.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#include <vector>

#define CK(x)                                                                                       \
    do {                                                                                            \
        cudaError_t e_ = (x);                                                                       \
        if (e_ != cudaSuccess) {                                                                    \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);         \
            exit(1);                                                                                \
        }                                                                                           \
    } while (0)

// ---- tcgen05 / mbarrier primitives (PTX ISA 8.7, sm_100a)
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols)
{
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols)
{
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(phase));
}
// Shared-memory matrix descriptor, K-major, no swizzle: core matrices of 8 rows x 16 bytes; lbo = byte
// distance between the two 16-byte K chunks of one MMA, sbo = byte distance between 8-row groups.
__device__ __forceinline__ uint64_t smem_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo)
{
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;   // descriptor version (sm_100)
    return d;                 // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
}
// Instruction descriptor of kind::i8: D s32, A/B unsigned 8-bit, both K-major, N, M = 128
__host__ __device__ constexpr uint32_t idesc_u8(int M, int N)
{
    return (2u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_i8(uint32_t dtmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t acc)
{
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(dtmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar)
{
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void tc_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, uint32_t (&r)[8])
{
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// byte offset of element (row, k) in a K-major no-swizzle tile with KB = K bytes per row:
// 8-row group g at g * (KB * 8), within the group the K chunks of 16 bytes at c * 128, row r at r * 16
__host__ __device__ inline uint32_t kmaj_off(int row, int k, int KB)
{
    return (uint32_t)((row >> 3) * (KB * 8) + (k >> 4) * 128 + (row & 7) * 16 + (k & 15));
}

template <int N, int K>
__global__ void __launch_bounds__(128) k_test(const uint8_t* A, const uint8_t* B, int32_t* D, int reps)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    uint8_t* As = sm;                    // 128 x K
    uint8_t* Bs = sm + 128 * K;          // N x K
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * K; i += 128) As[kmaj_off(i / K, i % K, K)] = A[i];
    for (int i = tid; i < N * K; i += 128) Bs[kmaj_off(i / K, i % K, K)] = B[i];
    if (warp == 0) tmem_alloc(&tbase, N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
    if (tid == 0) mbar_init(&bar, 1);
    fence_async_smem();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t taddr = tbase;
    constexpr uint32_t idesc = idesc_u8(128, N);
    if (tid == 0) {
        const uint32_t a0 = smem_u32(As), b0 = smem_u32(Bs);
        for (int r = 0; r < reps; ++r)
            for (int kk = 0; kk < K / 32; ++kk)
                mma_i8(taddr, smem_desc(a0 + kk * 256, 128, K * 8), smem_desc(b0 + kk * 256, 128, K * 8), idesc,
                       (r | kk) ? 1u : 0u);
        mma_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_after_sync();
    for (int c = 0; c < N; c += 8) {
        uint32_t v[8];
        tmem_ld8(taddr + ((uint32_t)(warp * 32) << 16) + c, v);
        for (int e = 0; e < 8; ++e) D[(warp * 32 + (tid & 31)) * N + c + e] = (int32_t)v[e];
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0) tmem_dealloc(taddr, N <= 32 ? 32 : N <= 64 ? 64 : N <= 128 ? 128 : 256);
}

template <int N, int K>
static bool check(int reps)
{
    std::vector<uint8_t> A(128 * K), B(N * K);
    srand(N * 131 + K);
    for (auto& x : A) x = rand() & 255;
    for (auto& x : B) x = rand() & 255;
    uint8_t *dA, *dB;
    int32_t* dD;
    CK(cudaMalloc(&dA, A.size()));
    CK(cudaMalloc(&dB, B.size()));
    CK(cudaMalloc(&dD, 128 * N * 4));
    CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
    const size_t smem = 128 * K + N * K;
    CK(cudaFuncSetAttribute(k_test<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_test<N, K><<<1, 128, smem>>>(dA, dB, dD, reps);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    std::vector<int32_t> D(128 * N);
    CK(cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            long long s = 0;
            for (int k = 0; k < K; ++k) s += (long long)A[m * K + k] * B[n * K + k];
            s *= reps;
            if (s != D[m * N + n] && bad++ < 5) printf("  mismatch m=%d n=%d got %d want %lld\n", m, n, D[m * N + n], s);
        }
    printf("check N=%d K=%d reps=%d: %s\n", N, K, reps, bad ? "FAIL" : "ok");
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    return bad == 0;
}

// throughput: every CTA issues `reps` x (K/32) MMAs of 128 x N x 32 on resident operands
template <int N, int K>
static void rate(int reps)
{
    uint8_t *dA, *dB;
    int32_t* dD;
    const int ctas = 148 * 2;
    CK(cudaMalloc(&dA, 128 * K));
    CK(cudaMalloc(&dB, N * K));
    CK(cudaMemset(dA, 1, 128 * K));
    CK(cudaMemset(dB, 1, N * K));
    CK(cudaMalloc(&dD, 128 * N * 4));
    const size_t smem = 128 * K + N * K;
    CK(cudaFuncSetAttribute(k_test<N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_test<N, K><<<ctas, 128, smem>>>(dA, dB, dD, 10);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k_test<N, K><<<ctas, 128, smem>>>(dA, dB, dD, reps);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double macs = (double)ctas * reps * 128.0 * N * K;
    printf("rate N=%d K=%d: %.3f ms, %.3f int8 TMAC/s (%.1f%% of 2250 nominal dense)\n", N, K, ms, macs / ms / 1e9,
           macs / ms / 1e9 / 2250.0 * 100);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
}

int main()
{
    bool ok = true;
    ok &= check<16, 32>(1);
    ok &= check<80, 320>(1);
    ok &= check<144, 64>(3);
    ok &= check<256, 128>(1);
    ok &= check<48, 160>(2);
    if (!ok) return 1;
    rate<144, 320>(2000);
    rate<256, 128>(4000);
    rate<80, 320>(4000);
    rate<128, 512>(2000);
    return 0;
}
