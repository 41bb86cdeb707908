// k_ksmoddown.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path: the ModDown NTT kernels (special-row inner product + inverse NTT, centred lift + NTT)
// (split from k_keyswitch.cu so the whole-limb NTT instantiations compile in parallel).  Layouts as in
// k_keyswitch.cu / DESIGN.md section 4.
#include "kinternal.cuh"
#ifndef CK_STREAM_STORES
#define CK_STREAM_STORES 0
#endif

namespace ck {

// (3) ModDown, special rows: r_c = iNTT_{P_k}( sum_j D_{j,P_k} key_j.c[P_k] ) for k < K -- the inner product
//     for the special primes is computed in the (coalesced, staged) loader of the inverse NTT; K = 2 stores
//     the CRT pair (a, t).  grid (2, B, G): one CTA per (component, ciphertext, rotation of the group).
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_moddown_intt(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const KsGroup grp, int nl, int nd,
                  u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int c = blockIdx.x, b = blockIdx.y, g = blockIdx.z, B = gridDim.y;
    const int K = dc->n_special, L = dc->n_data, ne = nl + K, np = L + K;
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
        auto st = [&](int i, u64 v) { dst[i] = (k == 0) ? v : crt2_t(dc, L, d0[i], v); };
        ntt_inverse<T>(sm, Pr, twp(dc, L + k), ld, st);
    }
}

// (4) ModDown, data rows: x_g,c[i] = NTT_{q_i}(centred(r_g,c) mod q_i) (R10, R10b).  grid (nl, 2, B*G)
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_moddown_ntt(const DCtx* __restrict__ dc, const u64* __restrict__ rem, int nl, u64* __restrict__ xo)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int i = blockIdx.x, c = blockIdx.y, gb = blockIdx.z;   // gb = g * B + b
    const int K = dc->n_special;
    const DPrime Pr = dc->p[i];
    const u64* r0 = rem + ((size_t)gb * 2 + c) * K * T::N;
    const u64* r1 = r0 + (size_t)(K - 1) * T::N;
    u64* o = xo + (((size_t)gb * 2 + c) * (nl + K) + i) * T::N;
    auto ld = [&](int k) { return special_centered(dc, r0[k], r1[k], Pr, i); };
    auto st = [&](int k, u64 v) { o[k] = v; };
    ntt_forward<T>(sm, Pr, twp(dc, i), ld, st);
}

void launch_ks_moddown_intt(const Launch& L, const uint64_t* modup, const KsGroup& grp, int nl, int nd, int batch,
                            uint64_t* rem, bool wide)
{
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        constexpr int NW = NttThreadsWide<LG>::value;
        auto ki = wide ? k_ks_moddown_intt<LG, NW> : k_ks_moddown_intt<LG, NT>;
        allow_smem(ki, smem);
        ProbeScope ps_(L.probe, L.st, "k_ks_moddown_intt");
        ki<<<dim3(2, batch, grp.G), wide ? NW : NT, smem, L.st>>>(L.dc, modup, grp, nl, nd, rem);
    });
    check_launch("ks_moddown_intt");
}

void launch_ks_moddown_ntt(const Launch& L, const uint64_t* rem, int nl, int gb, uint64_t* xo, bool wide)
{
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        constexpr int NW = NttThreadsWide<LG>::value;
        auto kn = wide ? k_ks_moddown_ntt<LG, NW> : k_ks_moddown_ntt<LG, NT>;
        allow_smem(kn, smem);
        ProbeScope ps_(L.probe, L.st, "k_ks_moddown_ntt");
        kn<<<dim3(nl, 2, gb), wide ? NW : NT, smem, L.st>>>(L.dc, rem, nl, xo);
    });
    check_launch("ks_moddown_ntt");
}
}  // namespace ck
