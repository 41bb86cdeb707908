// k_ksmodup.cu -- sm_100a kernel of the CKKS encrypted-dense-layer hot path: the key-switching ModUp
// (digit -> every other prime of Q_l P).  Layouts as in k_keyswitch.cu / DESIGN.md section 4.
#include "kinternal.cuh"
#ifndef CK_STREAM_STORES
#define CK_STREAM_STORES 0
#endif

namespace ck {

// ModUp: D_{j,e} = NTT_{p_e}(d_j mod p_e) for every row e of Q_l P outside digit j (all_e: every row -- QP
// digits are not the input limbs, so the inner product cannot read those rows from the input).  One launch
// per digit size ALPHA (1: d_j = a; 2: d_j = a + q_s t, reduced with one Shoup product), grid
// (sum over the set's digits of their target rows, B); 32 residues per thread (the compute-bound NTT).
template <int LOGN, int NTH, int ALPHA>
__global__ void __launch_bounds__(NTH)
k_ks_modup(const DCtx* __restrict__ dc, const u64* __restrict__ digits, u64* __restrict__ modup, int nl, int nd,
           int all_e, const DigitSet set)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int ne = nl + dc->n_special;
    int t = 0;
    while (t + 1 < set.count && (int)blockIdx.x >= set.first[t + 1]) ++t;
    const int x = blockIdx.x - set.first[t], s0 = set.s0[t], j = set.j[t];
    const int e = (!all_e && x >= s0) ? x + ALPHA : x;
    const int b = blockIdx.y;
    const int p = ext_prime_of(e, nl, dc->n_data);
    const DPrime Pr = dc->p[p];
    const u64* src = digits + ((size_t)b * nl + s0) * T::N;
    u64* dst = modup + (((size_t)b * nd + j) * ne + e) * T::N;
    auto ld = [&](int i) {
        if constexpr (ALPHA == 1) return reduce64_lazy(src[i], Pr);
        else return crt2_lazy(dc, s0, src[i], src[T::N + i], Pr, p);
    };
#if CK_STREAM_STORES
    auto st = [&](int i, u64 v) { __stcs(dst + i, v); };   // ModUp words: read once, by the next kernel
#else
    auto st = [&](int i, u64 v) { dst[i] = v; };
#endif
    ntt_forward<T>(sm, Pr, twp(dc, p), ld, st);
}

void launch_ks_modup(const Launch& L, const uint64_t* digits, uint64_t* modup, int nl, bool all_e, int batch)
{
    DigitSet one, two;
    digit_sets(L, nl, all_e, one, two);
    const int nd = L.active_digits(nl);
    const size_t smem = sizeof(u64) << L.log_n;
    ProbeScope ps_(L.probe, L.st, "k_ks_modup");
    NTT_DISPATCH(L.log_n, {
        constexpr int NW = NttThreadsWide<LG>::value;
        if (one.count) {
            allow_smem(k_ks_modup<LG, NW, 1>, smem);
            k_ks_modup<LG, NW, 1><<<dim3(one.first[one.count], batch), NW, smem, L.st>>>(L.dc, digits, modup, nl, nd,
                                                                                      all_e ? 1 : 0, one);
        }
        if (two.count) {
            allow_smem(k_ks_modup<LG, NW, 2>, smem);
            k_ks_modup<LG, NW, 2><<<dim3(two.first[two.count], batch), NW, smem, L.st>>>(L.dc, digits, modup, nl, nd,
                                                                                      all_e ? 1 : 0, two);
        }
    });
    check_launch("ks_modup");
}

}  // namespace ck
