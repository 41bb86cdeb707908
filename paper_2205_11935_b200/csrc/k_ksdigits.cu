// k_ksdigits.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path: key-switching digits (R9, R9b).
// Layouts as in k_keyswitch.cu / DESIGN.md section 4.
#include "kinternal.cuh"

namespace ck {

// Digits: for every active digit (grid (set.count, B)) the inverse NTTs of its primes of sigma_g(d):
//   first prime: a = iNTT_{q_s}(.) in [0, q_s); second (ALPHA = 2): t = (iNTT_{q_{s+1}}(.) - a) q_s^{-1} mod
//   q_{s+1}, so d_j = a + q_s t exactly (Garner pair, common.cuh).
// QP input (double hoisting, R11c, QPK = K special primes > 0): d is a Q_l P component and the digits are those
//   of ModDown(d): every coefficient residue becomes (iNTT_q(sigma_g(d)[q]) - [r]_q) P^{-1} with r the centred
//   special remainder (rem[b]: iNTT of the special limbs, from k_ks_qp_rem; sigma_g commutes with the centred
//   lift, so r is gathered once).
template <int LOGN, int NTH, int ALPHA, int QPK>
__global__ void __launch_bounds__(NTH)
k_ks_digits(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
            u32 galois, u64* __restrict__ digits, int nl, const u64* __restrict__ rem, const DigitSet set)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int s0 = set.s0[blockIdx.x], b = blockIdx.y;
    const u64* r0 = QPK ? rem + (size_t)b * QPK * T::N : nullptr;
    const u64* r1 = QPK ? r0 + (size_t)(QPK - 1) * T::N : nullptr;
    u64* d0 = digits + ((size_t)b * nl + s0) * T::N;
    const u32 ginv = galois ? galois_inv(galois, LOGN) : 0;
    const int alpha = ALPHA ? ALPHA : set.first[blockIdx.x];   // ALPHA = 0: digits of both sizes in one launch
#pragma unroll 1
    for (int h = 0; h < alpha; ++h) {
        const int pj = s0 + h;
        const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)pj * T::N;
        u64* dst = d0 + (size_t)h * T::N;
        const DPrime Pr = dc->p[pj];
        auto ld = [&](int i) { return src[i]; };
        auto place = [&](int i) { return galois ? galois_dst(i, ginv, LOGN) : i; };   // sigma_g in the staging
        auto st = [&](int i, u64 v) {
            if constexpr (QPK > 0) {
                const u64 r = QPK == 1 ? centered_to(r0[i], dc->p[dc->n_data].q, dc->pmod[pj], Pr)
                                       : special_centered(dc, r0[i], r1[i], Pr, pj);
                v = csub(shoup_mul(v + Pr.q - r, dc->pinv[pj], dc->pinv_sh[pj], Pr.q), Pr.q);
            }
            if constexpr (ALPHA == 1) dst[i] = v;
            else dst[i] = (h == 0) ? v : crt2_t(dc, s0, d0[i], v);   // d0 written by this CTA (synchronised)
        };
        // QP input with K = 2 special primes, everything below 2^45: the fused ModDown goes on in FP64 from the
        // transform's signed output x (|x| < 0.51 q) -- the integer form (special_centered + two Shoup products,
        // ~55 integer-pipe instructions per coefficient) was 40 % of this kernel's issue slots (ncu source page)
        bool fpe = false;
        if constexpr (QPK == 2) {
            const u64 lim = 1ULL << 45;
            fpe = Pr.q < lim && dc->p[dc->n_data].q < lim && dc->p[dc->n_data + 1].q < lim && (h == 0 || dc->p[s0].q < lim);
        }
        if (fpe) {
            if constexpr (QPK == 2) {
                const double q = (double)Pr.q, qi = Pr.qinv_d;
                auto cen = [&](u64 w) { return w > Pr.q / 2 ? -(double)(Pr.q - w) : (double)w; };
                const double p0 = cen(dc->qmod[dc->n_data][pj]), p0q = p0 * qi;     // P_0 mod q (centred), / q
                const double pm = (double)dc->pmod[pj];                              // P mod q
                const double pv = cen(dc->pinv[pj]), pvq = pv * qi;                  // P^{-1} mod q
                const double dv = h ? cen(dc->dig_inv[pj]) : 0.0, dvq = dv * qi;     // q_s0^{-1} mod q (2nd prime)
                const u64 ha = dc->phalf_a, ht = dc->phalf_t;
                auto stf = [&](int i, double x) {
                    const u64 a = r0[i], t = r1[i];
                    const bool neg = t > ht || (t == ht && a > ha);                  // a + P_0 t > (P - 1) / 2, exactly
                    const double y = fmodmul(u2d(t), p0, p0q, q);                    // P_0 t mod q, |y| < 0.51 q
                    const double z = ((x - u2d(a)) - y) + (neg ? pm : 0.0);          // x - [r]_q, |z| < 2^47
                    double o = fmodmul(z, pv, pvq, q);
                    if (h == 0) {
                        o = o < 0.0 ? o + q : o;
                        dst[i] = d2u(o);
                    } else {                                                         // Garner: (o - d_0) q_s0^{-1} mod q
                        double g = fmodmul(o - u2d(d0[i]), dv, dvq, q);
                        g = g < 0.0 ? g + q : g;
                        dst[i] = d2u(g);
                    }
                };
                T::template inverse_fp<false, true>(sm, Pr, twp(dc, pj), ld, stf, place);
            }
        } else {
            ntt_inverse<T>(sm, Pr, twp(dc, pj), ld, st, place);
        }
    }
}

template <int LG, int ALPHA, int QPK>
static void digits_launch(const Launch& L, const KsIn& in, int nl, int batch, uint64_t* digits, const uint64_t* rem,
                          const DigitSet& set)
{
    if (!set.count) return;
    constexpr int NT = NttThreads<LG>::value;
    const size_t smem = sizeof(u64) << LG;
    auto kd = k_ks_digits<LG, NT, ALPHA, QPK>;
    allow_smem(kd, smem);
    kd<<<dim3(set.count, batch), NT, smem, L.st>>>(L.dc, in.base, in.ct_stride, in.comp_off, in.galois, digits, nl, rem,
                                                   set);
}

void launch_ks_digits(const Launch& L, const KsIn& in, int nl, int batch, uint64_t* digits, const uint64_t* rem)
{
    DigitSet one, two;
    digit_sets(L, nl, false, one, two);
    ProbeScope ps_(L.probe, L.st, "k_ks_digits");
    const int qpk = rem ? L.n_special : 0;
    // both digit sizes present: one launch (ALPHA = 0, the size per CTA in set.first) -- two launches of 2-5 CTAs
    // per ciphertext each end in a partial wave (B = 256: 5.2 and 3.5 waves); two-prime digits first in the grid
    DigitSet mix;
    mix.count = 0;
    if (one.count && two.count) {
        for (int k = 0; k < two.count; ++k, ++mix.count) {
            mix.j[mix.count] = two.j[k];
            mix.s0[mix.count] = two.s0[k];
            mix.first[mix.count] = 2;
        }
        for (int k = 0; k < one.count; ++k, ++mix.count) {
            mix.j[mix.count] = one.j[k];
            mix.s0[mix.count] = one.s0[k];
            mix.first[mix.count] = 1;
        }
    }
    NTT_DISPATCH(L.log_n, {
        if (mix.count) {
            if (qpk == 0) digits_launch<LG, 0, 0>(L, in, nl, batch, digits, rem, mix);
            else if (qpk == 1) digits_launch<LG, 0, 1>(L, in, nl, batch, digits, rem, mix);
            else digits_launch<LG, 0, 2>(L, in, nl, batch, digits, rem, mix);
        } else if (qpk == 0) {
            digits_launch<LG, 1, 0>(L, in, nl, batch, digits, rem, one);
            digits_launch<LG, 2, 0>(L, in, nl, batch, digits, rem, two);
        } else if (qpk == 1) {
            digits_launch<LG, 1, 1>(L, in, nl, batch, digits, rem, one);
            digits_launch<LG, 2, 1>(L, in, nl, batch, digits, rem, two);
        } else {
            digits_launch<LG, 1, 2>(L, in, nl, batch, digits, rem, one);
            digits_launch<LG, 2, 2>(L, in, nl, batch, digits, rem, two);
        }
    });
    check_launch("ks_digits");
}

void digit_sets(const Launch& L, int nl, bool all_e, DigitSet& one, DigitSet& two)
{
    one.count = two.count = 0;
    one.first[0] = two.first[0] = 0;
    const int ne = nl + L.n_special, nd = L.active_digits(nl);
    for (int j = 0; j < nd; ++j) {
        const int s0 = L.dig_start[j], len = std::min(L.dig_len[j], nl - s0);
        DigitSet& d = len == 1 ? one : two;
        d.j[d.count] = j;
        d.s0[d.count] = s0;
        d.first[d.count + 1] = d.first[d.count] + (all_e ? ne : ne - len);
        ++d.count;
    }
}

}  // namespace ck
