// tma_box_bench.cu -- streaming rate of 4D TMA boxes over the baby-step buffer layout of the BSGS MAC
// ([j][b][row][x] u64, N = 16384 coefficients, 20 rows, 256 ciphertexts, 63 baby steps): every CTA streams
// its (x-block, row) column of boxes through a ring of RS slots, doing nothing else, so the measured rate is
// the TMA/DRAM limit of the access pattern.  Boxes (X coefficients, 1 row, BB ciphertexts, J baby steps).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tma_box_bench tools/tma_box_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int RS>
__global__ void __launch_bounds__(128) k_stream(const __grid_constant__ CUtensorMap m, int nbox, int X, int BB, int J,
                                                int bytes, unsigned long long* sink)
{
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bars[RS];
    const int x0 = blockIdx.x * X, row = blockIdx.y;
    if (threadIdx.x == 0) {
        for (int s = 0; s < RS; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bars[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int i) {
        const int b0 = (i % (256 / BB)) * BB, j0 = (i / (256 / BB)) * J;
        uint64_t* bar = &bars[i % RS];
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(bar)), "r"(bytes) : "memory");
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
                "r"(su(sm + (i % RS) * bytes)), "l"(&m), "r"(x0), "r"(row), "r"(b0), "r"(j0), "r"(su(bar))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < RS && i < nbox; ++i) issue(i);
    unsigned long long acc = 0;
    for (int i = 0; i < nbox; ++i) {
        const uint32_t ph = (i / RS) & 1;
        asm volatile(
            "{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(
                su(&bars[i % RS])),
            "r"(ph)
            : "memory");
        acc += reinterpret_cast<const unsigned long long*>(sm + (i % RS) * bytes)[threadIdx.x];
        __syncthreads();
        if (threadIdx.x == 0 && i + RS < nbox) issue(i + RS);
    }
    if (acc == 0x1234567) sink[0] = acc;
}

int main()
{
    const int N = 16384, R = 20, B = 256, Jt = 64;
    const size_t words = (size_t)N * R * B * Jt;
    uint64_t* buf;
    cudaMalloc(&buf, words * 8);
    cudaMemset(buf, 1, words * 8);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)f;
    struct Cfg { int X, BB, J; };
    const Cfg cfgs[] = {{4, 128, 8}, {8, 128, 8}, {16, 128, 4}, {4, 256, 4}, {32, 64, 4}, {16, 64, 8}};
    for (const Cfg& cf : cfgs) {
        CUtensorMap m;
        const cuuint64_t dims[4] = {(cuuint64_t)N, (cuuint64_t)R, (cuuint64_t)B, (cuuint64_t)Jt};
        const cuuint64_t str[3] = {(cuuint64_t)N * 8, (cuuint64_t)N * R * 8, (cuuint64_t)N * R * B * 8};
        const cuuint32_t box[4] = {(cuuint32_t)cf.X, 1, (cuuint32_t)cf.BB, (cuuint32_t)cf.J};
        const cuuint32_t es[4] = {1, 1, 1, 1};
        if (enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
            printf("encode failed X=%d\n", cf.X);
            continue;
        }
        const int bytes = cf.X * cf.BB * cf.J * 8;
        const int nbox = (B / cf.BB) * (Jt / cf.J);
        const dim3 grid(N / cf.X, R);
        const size_t smem = (size_t)3 * bytes;
        cudaFuncSetAttribute(k_stream<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_stream<3><<<grid, 128, smem>>>(m, nbox, cf.X, cf.BB, cf.J, bytes, sink);
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        cudaEventRecord(e0);
        k_stream<3><<<grid, 128, smem>>>(m, nbox, cf.X, cf.BB, cf.J, bytes, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("box X=%2d BB=%3d J=%d (%6d B): %.3f ms, %.0f GB/s  %s\n", cf.X, cf.BB, cf.J, bytes, ms,
               words * 8.0 / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
