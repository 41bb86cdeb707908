// k_ksmodup.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path: the key-switching ModUp (digit -> every other prime of Q_l P)
// (split from k_keyswitch.cu so the whole-limb NTT instantiations compile in parallel).  Layouts as in
// k_keyswitch.cu / DESIGN.md section 4.
#include "kinternal.cuh"
#ifndef CK_STREAM_STORES
#define CK_STREAM_STORES 0
#endif

namespace ck {

// (2) ModUp: D_{j,e} = NTT_{p_e}(d_j mod p_e) for every row e of Q_l P outside digit j (all_e: every row --
//     QP digits are not the input limbs, so the inner product cannot read those rows from the input).
//     grid (sum over active digits of their target counts, B)
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_modup(const DCtx* __restrict__ dc, const u64* __restrict__ digits, u64* __restrict__ modup, int nl, int nd,
           int all_e)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int K = dc->n_special, ne = nl + K;
    int x = blockIdx.x, j = 0, len = 0;
    for (;; ++j) {
        len = digit_len_at(dc, j, nl);
        const int cnt = all_e ? ne : ne - len;
        if (x < cnt) break;
        x -= cnt;
    }
    const int s0 = dc->dig_start[j];
    const int e = (!all_e && x >= s0) ? x + len : x;
    const int b = blockIdx.y;
    const int p = ext_prime_of(e, nl, dc->n_data);
    const DPrime Pr = dc->p[p];
    const u64* src = digits + ((size_t)b * nl + s0) * T::N;
    u64* dst = modup + (((size_t)b * nd + j) * ne + e) * T::N;
    auto ld = [&](int i) {
        return len == 1 ? reduce64_lazy(src[i], Pr) : crt2_lazy(dc, s0, src[i], src[T::N + i], Pr, p);
    };
#if CK_STREAM_STORES
    auto st = [&](int i, u64 v) { __stcs(dst + i, v); };   // ModUp words: read once, by the next kernel
#else
    auto st = [&](int i, u64 v) { dst[i] = v; };
#endif
    ntt_forward<T>(sm, Pr, twp(dc, p), ld, st);
}

void launch_ks_modup(const Launch& L, const uint64_t* digits, uint64_t* modup, int nl, int nd, bool all_e, int pairs,
                     int batch, bool wide)
{
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        constexpr int NW = NttThreadsWide<LG>::value;
        auto km = wide ? k_ks_modup<LG, NW> : k_ks_modup<LG, NT>;
        allow_smem(km, smem);
        ProbeScope ps_(L.probe, L.st, "k_ks_modup");
        km<<<dim3(pairs, batch), wide ? NW : NT, smem, L.st>>>(L.dc, digits, modup, nl, nd, all_e ? 1 : 0);
    });
    check_launch("ks_modup");
}
}  // namespace ck
