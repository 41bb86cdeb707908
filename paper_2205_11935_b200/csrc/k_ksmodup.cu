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
    // a < q_s0 < 2 q_p (primes of the same size): a itself is the lazy residue the transform accepts ([0, 2q))
    auto ld_small = [&](int i) {
        if constexpr (ALPHA == 1) return src[i];
        else return csub(shoup_mul(src[T::N + i], dc->qmod[s0][p], dc->qmod_sh[s0][p], Pr.q) + src[i], Pr.q2);
    };
#if CK_STREAM_STORES
    auto st = [&](int i, u64 v) { __stcs(dst + i, v); };   // ModUp words: read once, by the next kernel
#else
    auto st = [&](int i, u64 v) { dst[i] = v; };
#endif
    if (dc->p[s0].q < Pr.q2) ntt_forward<T>(sm, Pr, twp(dc, p), ld_small, st);
    else ntt_forward<T>(sm, Pr, twp(dc, p), ld, st);
}

// The same ModUp on the CTA-pair schedule (ntt_c.cuh): grid (CL * targets, B) in clusters of CL CTAs; FP64-class
// targets on the FP64 pipe, integer-class targets (q_0, 60-bit special primes) on the integer pipe in the same
// launch and CTA shape, so CTAs of both kinds share an SM.
template <int LOGN, int ALPHA>
__global__ void __launch_bounds__(NttC<LOGN>::NT, NttC<LOGN>::MINB)
k_ks_modup_c(const DCtx* __restrict__ dc, const u64* __restrict__ digits, u64* __restrict__ modup, int nl, int nd,
             int all_e, const DigitSet set)
{
    extern __shared__ u64 sm[];
    using TC = NttC<LOGN>;
    const int ne = nl + dc->n_special;
    const int item = blockIdx.x / TC::CL, h = blockIdx.x % TC::CL;
    int t = 0;
    while (t + 1 < set.count && item >= set.first[t + 1]) ++t;
    const int x = item - set.first[t], s0 = set.s0[t], j = set.j[t];
    const int e = (!all_e && x >= s0) ? x + ALPHA : x;
    const int b = blockIdx.y;
    const int p = ext_prime_of(e, nl, dc->n_data);
    const DPrime Pr = dc->p[p];
    const int pc = prime_class(Pr.q);
    const u64* src = digits + ((size_t)b * nl + s0) * TC::N;
    u64* dst = modup + (((size_t)b * nd + j) * ne + e) * TC::N;
    auto ld = [&](int i) {
        if constexpr (ALPHA == 1) return reduce64_lazy(src[i], Pr);
        else return crt2_lazy(dc, s0, src[i], src[TC::N + i], Pr, p);
    };
    auto ld_small = [&](int i) {   // q_s0 < 2 q_p: see k_ks_modup
        if constexpr (ALPHA == 1) return src[i];
        else return csub(shoup_mul(src[TC::N + i], dc->qmod[s0][p], dc->qmod_sh[s0][p], Pr.q) + src[i], Pr.q2);
    };
    const bool small = dc->p[s0].q < Pr.q2;
    // 2-prime digit of primes below 2^45 -> FP64-class target of the same size: d mod p = a + (q_s mod p) t with one
    // fmodmul, handed to the transform as a signed double (|.| < 2.6 p) -- 23.4 -> 22.7 ms per B = 256 chunk against the
    // integer Shoup form of ld_small (CK_MODUP_INT_LOADER keeps that form)
#ifndef CK_MODUP_INT_LOADER
    if (pc == PC_FP && ALPHA == 2 && small && dc->p[s0 + 1].q < (1ULL << 45)) {
        const u64 qm = dc->qmod[s0][p];
        const double qd = (double)Pr.q, c = qm > Pr.q / 2 ? -(double)(Pr.q - qm) : (double)qm, cq = c * Pr.qinv_d;
        auto ld_fp = [&](int i) { return u2d(src[i]) + fmodmul(u2d(src[TC::N + i]), c, cq, qd); };
        TC::template forward_fp<false>(sm, h, Pr, twq_fwd(dc, p), ld_fp, dst);
        return;
    }
#endif
    if (pc == PC_FP) {
        if (small) TC::template forward_fp<false>(sm, h, Pr, twq_fwd(dc, p), ld_small, dst);
        else TC::template forward_fp<false>(sm, h, Pr, twq_fwd(dc, p), ld, dst);
    } else if (pc == PC_FPR) {
        if (small) TC::template forward_fp<true>(sm, h, Pr, twq_fwd(dc, p), ld_small, dst);
        else TC::template forward_fp<true>(sm, h, Pr, twq_fwd(dc, p), ld, dst);
    } else {
        TC::forward_int(sm, h, Pr, twq_fwd_int(dc, p), ld, dst);
    }
}

template <int LG>
static bool launch_ks_modup_c(const Launch& L, const uint64_t* digits, uint64_t* modup, int nl, bool all_e, int batch,
                              const DigitSet& one, const DigitSet& two, int nd)
{
    if constexpr (ntt_c_supported(LG)) {
        if (!(get_ntt_q() & (LG == 14 ? NTTQ_MODUP_14 : NTTQ_MODUP))) return false;
        using TC = NttC<LG>;
        if (one.count) {
            allow_smem(k_ks_modup_c<LG, 1>, TC::SMEM_ALL);
            launch_cluster(k_ks_modup_c<LG, 1>, dim3(one.first[one.count] * TC::CL, batch), TC::NT, TC::SMEM_ALL, L.st,
                           TC::CL, L.dc, digits, modup, nl, nd, all_e ? 1 : 0, one);
        }
        if (two.count) {
            allow_smem(k_ks_modup_c<LG, 2>, TC::SMEM_ALL);
            launch_cluster(k_ks_modup_c<LG, 2>, dim3(two.first[two.count] * TC::CL, batch), TC::NT, TC::SMEM_ALL, L.st,
                           TC::CL, L.dc, digits, modup, nl, nd, all_e ? 1 : 0, two);
        }
        return true;
    } else {
        return false;
    }
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
        if (launch_ks_modup_c<LG>(L, digits, modup, nl, all_e, batch, one, two, nd)) break;
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
