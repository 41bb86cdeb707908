// k_ksdigits.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path: key-switching digits (R9, R9b) and the special remainders of Q_l P components (R11c)
// (split from k_keyswitch.cu so the whole-limb NTT instantiations compile in parallel).  Layouts as in
// k_keyswitch.cu / DESIGN.md section 4.
#include "kinternal.cuh"
#ifndef CK_STREAM_STORES
#define CK_STREAM_STORES 0
#endif

namespace ck {

// (1) digits: for every active digit j (grid (nd, B)), the inverse NTTs of its primes of sigma_g(d):
//     first prime: a = iNTT_{q_s}(.) in [0, q_s); second: t = (iNTT_{q_{s+1}}(.) - a) q_s^{-1} mod q_{s+1}.
//     QP input (double hoisting, R11c, rem != null): d is a Q_l P component and the digits are those of
//     ModDown(d): every coefficient residue becomes (iNTT_q(sigma_g(d)[q]) - [r]_q) P^{-1} with r the centred
//     special remainder (rem[b]: iNTT of the special limbs, from k_ks_qp_rem; sigma_g commutes with the
//     centred lift, so r is gathered once).
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_digits(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
            u32 galois, u64* __restrict__ digits, int nl, const u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int j = blockIdx.x, b = blockIdx.y;
    const int s0 = dc->dig_start[j], len = digit_len_at(dc, j, nl), K = dc->n_special;
    const u64* r0 = rem ? rem + (size_t)b * K * T::N : nullptr;
    const u64* r1 = rem ? r0 + (size_t)(K - 1) * T::N : nullptr;
    u64* d0 = digits + ((size_t)b * nl + s0) * T::N;
#pragma unroll 1
    for (int h = 0; h < len; ++h) {
        const int pj = s0 + h;
        const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)pj * T::N;
        u64* dst = d0 + (size_t)h * T::N;
        const DPrime Pr = dc->p[pj];
        const u64 Pinv = dc->pinv[pj], Pinv_sh = dc->pinv_sh[pj];
        auto ld = [&](int i) { return galois ? src[galois_src(i, galois, LOGN)] : src[i]; };
        auto st = [&](int i, u64 v) {
            if (rem) {
                const u64 x = v + Pr.q - special_centered(dc, r0[i], r1[i], Pr, pj);
                v = csub(shoup_mul(x, Pinv, Pinv_sh, Pr.q), Pr.q);
            }
            dst[i] = (h == 0) ? v : crt2_t(dc, s0, d0[i], v);   // d0 written by this CTA (synchronised)
        };
        ntt_inverse<T>(sm, Pr, twp(dc, pj), ld, st);
    }
}

// (1') QP remainder: rem[b][c] = iNTT of the special limbs of sigma_g(x_b.c) (K = 2: the CRT pair (a, t)
//      of P_0 P_1) for QP components (giant-step digits: one component; the layer's final ModDown: both).
//      grid (ncomp, B)
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_qp_rem(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
            size_t comp_step, u32 galois, int nl, u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int c = blockIdx.x, b = blockIdx.y, K = dc->n_special, L = dc->n_data;
    u64* d0 = rem + ((size_t)b * gridDim.x + c) * K * T::N;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)c * comp_step + (size_t)(nl + k) * T::N;
        u64* dst = d0 + (size_t)k * T::N;
        const DPrime Pr = dc->p[L + k];
        auto ld = [&](int i) { return galois ? src[galois_src(i, galois, LOGN)] : src[i]; };
        auto st = [&](int i, u64 v) { dst[i] = (k == 0) ? v : crt2_t(dc, L, d0[i], v); };
        ntt_inverse<T>(sm, Pr, twp(dc, L + k), ld, st);
    }
}

void launch_ks_digits(const Launch& L, const KsIn& in, int nd, int batch, int nl, uint64_t* digits, const uint64_t* rem,
                      bool wide)
{
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        constexpr int NW = NttThreadsWide<LG>::value;
        auto kd = wide ? k_ks_digits<LG, NW> : k_ks_digits<LG, NT>;
        allow_smem(kd, smem);
        ProbeScope ps_(L.probe, L.st, "k_ks_digits");
        kd<<<dim3(nd, batch), wide ? NW : NT, smem, L.st>>>(L.dc, in.base, in.ct_stride, in.comp_off, in.galois, digits,
                                                          nl, rem);
    });
    check_launch("ks_digits");
}

void launch_ks_qp_rem(const Launch& L, const uint64_t* in, size_t ct_stride, size_t comp_off, size_t comp_step,
                      uint32_t galois, int nl, int ncomp, int batch, uint64_t* rem, bool wide)
{
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        constexpr int NW = NttThreadsWide<LG>::value;
        auto kr = wide ? k_ks_qp_rem<LG, NW> : k_ks_qp_rem<LG, NT>;
        allow_smem(kr, smem);
        ProbeScope ps_(L.probe, L.st, "k_ks_qp_rem");
        kr<<<dim3(ncomp, batch), wide ? NW : NT, smem, L.st>>>(L.dc, in, ct_stride, comp_off, comp_step, galois, nl, rem);
    });
    check_launch("ks_qp_rem");
}
}  // namespace ck
