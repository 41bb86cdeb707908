// k_ksqprem.cu -- sm_100a kernel of the CKKS encrypted-dense-layer hot path: the special remainders of Q_l P
// components (double hoisting, R11c).  Layouts as in k_keyswitch.cu / DESIGN.md section 4.
#include "kinternal.cuh"

namespace ck {

// rem[b][c] = iNTT of the special limbs of sigma_g(x_b.c) (K = 2: the CRT pair (a, t) of P_0 P_1) for QP
// components (giant-step digits: one component; the layer's final ModDown: both).  grid (ncomp, B)
template <int LOGN, int NTH, int K>
__global__ void __launch_bounds__(NTH)
k_ks_qp_rem(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
            size_t comp_step, u32 galois, int nl, u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int c = blockIdx.x, b = blockIdx.y, L = dc->n_data;
    u64* d0 = rem + ((size_t)b * gridDim.x + c) * K * T::N;
    const u32 ginv = galois ? galois_inv(galois, LOGN) : 0;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)c * comp_step + (size_t)(nl + k) * T::N;
        u64* dst = d0 + (size_t)k * T::N;
        const DPrime Pr = dc->p[L + k];
        auto ld = [&](int i) { return src[i]; };
        auto place = [&](int i) { return galois ? galois_dst(i, ginv, LOGN) : i; };   // sigma_g in the staging
        auto st = [&](int i, u64 v) {
            if constexpr (K == 1) dst[i] = v;
            else dst[i] = (k == 0) ? v : crt2_t(dc, L, d0[i], v);
        };
        ntt_inverse<T>(sm, Pr, twp(dc, L + k), ld, st, place);
    }
}

void launch_ks_qp_rem(const Launch& L, const uint64_t* in, size_t ct_stride, size_t comp_off, size_t comp_step,
                      uint32_t galois, int nl, int ncomp, int batch, uint64_t* rem)
{
    const size_t smem = sizeof(u64) << L.log_n;
    ProbeScope ps_(L.probe, L.st, "k_ks_qp_rem");
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        auto kr = L.n_special == 2 ? k_ks_qp_rem<LG, NT, 2> : k_ks_qp_rem<LG, NT, 1>;
        allow_smem(kr, smem);
        kr<<<dim3(ncomp, batch), NT, smem, L.st>>>(L.dc, in, ct_stride, comp_off, comp_step, galois, nl, rem);
    });
    check_launch("ks_qp_rem");
}

}  // namespace ck
