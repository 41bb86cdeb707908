// Check of the mma.sync m16n8k4 f64 fragment layout assumed by the DMMA inner-product kernel:
//   A 16x4: a0 = A[gid][tig], a1 = A[gid+8][tig];  B 4x8: b0 = B[tig][gid];
//   C 16x8: c0,c1 = C[gid][2 tig + {0,1}], c2,c3 = C[gid+8][2 tig + {0,1}]   (gid = lane/4, tig = lane%4)
// Build: nvcc -O2 -gencode arch=compute_100a,code=sm_100a -o dmma_layout dmma_layout.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(const double* A, const double* B, double* C)
{
    const int lane = threadIdx.x, gid = lane >> 2, tig = lane & 3;
    double a0 = A[gid * 4 + tig], a1 = A[(gid + 8) * 4 + tig], b0 = B[tig * 8 + gid];
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
                 : "+d"(c0), "+d"(c1), "+d"(c2), "+d"(c3) : "d"(a0), "d"(a1), "d"(b0));
    C[gid * 8 + 2 * tig] = c0;
    C[gid * 8 + 2 * tig + 1] = c1;
    C[(gid + 8) * 8 + 2 * tig] = c2;
    C[(gid + 8) * 8 + 2 * tig + 1] = c3;
}
int main()
{
    double hA[64], hB[32], hC[128], ref[128];
    for (int i = 0; i < 64; ++i) hA[i] = (double)((i * 37) % 101) * 1024.0 + i;
    for (int i = 0; i < 32; ++i) hB[i] = (double)((i * 53) % 97) * 2048.0 + 3 * i;
    for (int r = 0; r < 16; ++r)
        for (int c = 0; c < 8; ++c) {
            double s = 0;
            for (int kk = 0; kk < 4; ++kk) s += hA[r * 4 + kk] * hB[kk * 8 + c];
            ref[r * 8 + c] = s;
        }
    double *dA, *dB, *dC;
    cudaMalloc(&dA, sizeof hA);
    cudaMalloc(&dB, sizeof hB);
    cudaMalloc(&dC, sizeof hC);
    cudaMemcpy(dA, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, hB, sizeof hB, cudaMemcpyHostToDevice);
    k<<<1, 32>>>(dA, dB, dC);
    cudaMemcpy(hC, dC, sizeof hC, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int i = 0; i < 128; ++i) bad += hC[i] != ref[i];
    printf("{\"dmma_m16n8k4_layout\": \"%s\", \"mismatches\": %d}\n", bad ? "MISMATCH" : "ok", bad);
    return bad != 0;
}
