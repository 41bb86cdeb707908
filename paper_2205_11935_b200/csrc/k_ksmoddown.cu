// k_ksmoddown.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path: the ModDown NTT kernels
// (special-row inner product + inverse NTT; centred lift + NTT).  Layouts as in k_keyswitch.cu / DESIGN.md 4.
#include "kinternal.cuh"

namespace ck {

// ModDown, special rows: r_c = iNTT_{P_k}( sum_j D_{j,P_k} key_j.c[P_k] ) for k < K -- the inner product for
// the special primes is computed in the (coalesced, staged) loader of the inverse NTT; K = 2 stores the CRT
// pair (a, t).  grid (2, B, G): one CTA per (component, ciphertext, rotation of the group).
template <int LOGN, int NTH, int K>
__global__ void __launch_bounds__(NTH)
k_ks_moddown_intt(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const KsGroup grp, int nl, int nd,
                  u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int c = blockIdx.x, b = blockIdx.y, g = blockIdx.z, B = gridDim.y;
    const int L = dc->n_data, ne = nl + K, np = L + K;
    const u64* __restrict__ key = grp.key[g];
    u64* d0 = rem + (((size_t)g * B + b) * 2 + c) * K * T::N;
#pragma unroll 1
    for (int k = 0; k < K; ++k) {
        const DPrime Pr = dc->p[L + k];
        u64* dst = d0 + (size_t)k * T::N;
        auto ld = [&](int i) {
            Acc128 a;
            a.zero();
            for (int j = 0; j < nd; ++j)
                a.mac(modup[(((size_t)b * nd + j) * ne + nl + k) * T::N + i],
                      key[(((size_t)j * 2 + c) * np + L + k) * T::N + i]);
            return a.reduce(Pr);
        };
        auto st = [&](int i, u64 v) {
            if constexpr (K == 1) dst[i] = v;
            else dst[i] = (k == 0) ? v : crt2_t(dc, L, d0[i], v);
        };
        ntt_inverse<T>(sm, Pr, twp(dc, L + k), ld, st);
    }
}

// ModDown, data rows: x_g,c[i] = NTT_{q_i}(centred(r_g,c) mod q_i) (R10, R10b).  grid (nl, 2, B*G)
// FUSE (the layer-final ModDown of Q_l P ciphertexts y, G = 1): the storer finishes the ModDown,
// out[b][c][i] = (y[b][c][i] - x) P^{-1} mod q_i, instead of writing x for a combine kernel.
template <int LOGN, int NTH, int K, bool FUSE>
__global__ void __launch_bounds__(NTH)
k_ks_moddown_ntt(const DCtx* __restrict__ dc, const u64* __restrict__ rem, int nl, u64* __restrict__ xo,
                 const u64* __restrict__ y, size_t y_stride, u64* __restrict__ out, size_t out_stride)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int i = blockIdx.x, c = blockIdx.y, gb = blockIdx.z;   // gb = g * B + b
    const DPrime Pr = dc->p[i];
    const u64* r0 = rem + ((size_t)gb * 2 + c) * K * T::N;
    auto ld = [&](int k) {
        if constexpr (K == 1) return centered_to(r0[k], dc->p[dc->n_data].q, dc->pmod[i], Pr);
        else return special_centered(dc, r0[k], r0[T::N + k], Pr, i);
    };
    // K = 2 with every prime below 2^45: the centred remainder mod q_i in FP64 (as the digits' epilogue,
    // k_ksdigits.cu): sign by the exact mixed-radix test, r = a + fmodmul(t, P_0) - [neg] (P mod q), |r| < 2 q
    bool fpl = false;
    if constexpr (K == 2) {
        const u64 lim = 1ULL << 45;
        fpl = Pr.q < lim && dc->p[dc->n_data].q < lim && dc->p[dc->n_data + 1].q < lim;
    }
    const double qd = (double)Pr.q;
    const double p0 = dc->qmod[dc->n_data][i] > Pr.q / 2 ? -(double)(Pr.q - dc->qmod[dc->n_data][i])
                                                         : (double)dc->qmod[dc->n_data][i];
    const double p0q = p0 * Pr.qinv_d, pmd = (double)dc->pmod[i];
    const u64 ha = dc->phalf_a, ht = dc->phalf_t;
    auto ldf = [&](int k) {
        const u64 a = r0[k], t = r0[T::N + k];
        const bool neg = t > ht || (t == ht && a > ha);
        return (u2d(a) + fmodmul(u2d(t), p0, p0q, qd)) - (neg ? pmd : 0.0);
    };
    if constexpr (FUSE) {
        const u64* yy = y + (size_t)gb * y_stride + ((size_t)c * (nl + K) + i) * T::N;
        u64* oo = out + (size_t)gb * out_stride + ((size_t)c * nl + i) * T::N;
        const u64 pinv = dc->pinv[i], pinv_sh = dc->pinv_sh[i];
        auto st = [&](int k, u64 v) { oo[k] = csub(shoup_mul(yy[k] + Pr.q - v, pinv, pinv_sh, Pr.q), Pr.q); };
        if (fpl) T::forward_fp(sm, Pr, twp(dc, i), ldf, st);
        else ntt_forward<T>(sm, Pr, twp(dc, i), ld, st);
    } else {
        u64* o = xo + (((size_t)gb * 2 + c) * (nl + K) + i) * T::N;
        auto st = [&](int k, u64 v) { o[k] = v; };
        if (fpl) T::forward_fp(sm, Pr, twp(dc, i), ldf, st);
        else ntt_forward<T>(sm, Pr, twp(dc, i), ld, st);
    }
}

void launch_ks_moddown_intt(const Launch& L, const uint64_t* modup, const KsGroup& grp, int nl, int nd, int batch,
                            uint64_t* rem)
{
    const size_t smem = sizeof(u64) << L.log_n;
    ProbeScope ps_(L.probe, L.st, "k_ks_moddown_intt");
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        auto ki = L.n_special == 2 ? k_ks_moddown_intt<LG, NT, 2> : k_ks_moddown_intt<LG, NT, 1>;
        allow_smem(ki, smem);
        ki<<<dim3(2, batch, grp.G), NT, smem, L.st>>>(L.dc, modup, grp, nl, nd, rem);
    });
    check_launch("ks_moddown_intt");
}

void launch_ks_moddown_ntt(const Launch& L, const uint64_t* rem, int nl, int gb, uint64_t* xo)
{
    const size_t smem = sizeof(u64) << L.log_n;
    ProbeScope ps_(L.probe, L.st, "k_ks_moddown_ntt");
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        auto kn = L.n_special == 2 ? k_ks_moddown_ntt<LG, NT, 2, false> : k_ks_moddown_ntt<LG, NT, 1, false>;
        allow_smem(kn, smem);
        kn<<<dim3(nl, 2, gb), NT, smem, L.st>>>(L.dc, rem, nl, xo, nullptr, 0, nullptr, 0);
    });
    check_launch("ks_moddown_ntt");
}

void launch_ks_moddown_ntt_fused(const Launch& L, const uint64_t* rem, int nl, int batch, const uint64_t* y,
                                 size_t y_stride, uint64_t* out, size_t out_stride)
{
    const size_t smem = sizeof(u64) << L.log_n;
    ProbeScope ps_(L.probe, L.st, "k_ks_moddown_ntt");
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        auto kn = L.n_special == 2 ? k_ks_moddown_ntt<LG, NT, 2, true> : k_ks_moddown_ntt<LG, NT, 1, true>;
        allow_smem(kn, smem);
        kn<<<dim3(nl, 2, batch), NT, smem, L.st>>>(L.dc, rem, nl, nullptr, y, y_stride, out, out_stride);
    });
    check_launch("ks_moddown_ntt_fused");
}

}  // namespace ck
