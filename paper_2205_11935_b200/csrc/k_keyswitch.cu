// k_keyswitch.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path.
//
// Every operation of SURVEY 8(a) rows a2-a12 is one of these kernels; the host side (api.cu)
// only sequences launches and tracks level/scale.  Modular arithmetic runs on the integer pipes
// (64-bit Shoup/Barrett), on the FP64 pipe (exact error-free products for q < 2^45), and -- for the
// two small modular contractions (key-switch inner product, BSGS inner sums) -- on the FP64 tensor
// cores with exactly split operands.  Layouts:
//   ciphertext  [batch][comp][limb][N]  u64, NTT domain, canonical residues in [0, q)
//   key         [digit j][comp][prime 0..L][N]  (prime L = special P)
//   plaintexts  [t][limb][N]
// This unit: key switching (digits, ModUp, inner products, ModDown), Galois gathers.
#include "kinternal.cuh"
#ifndef CK_STREAM_STORES
#define CK_STREAM_STORES 0
#endif

namespace ck {

// ------------------------------------------------------------------------------------ key switch
// (1) digits: d_j = iNTT_{q_j}(sigma_g(d)[j])  -> [B][nl][N] in [0, q_j)                  (R9)
//     QP input (double hoisting, R11c, rem != null): d is a Q_l P component and the digits are those of
//     ModDown(d): d_j = (iNTT_{q_j}(sigma_g(d)[j]) - [r]_{q_j}) P^{-1} with r = centred iNTT_P(sigma_g(d)[P])
//     (rem[b], from k_ks_qp_rem; sigma_g commutes with the centred lift, so r is gathered once).
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_digits(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
            u32 galois, u64* __restrict__ digits, int nl, const u64* __restrict__ rem, int special)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int j = blockIdx.x, b = blockIdx.y;
    const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)j * T::N;
    u64* dst = digits + ((size_t)b * nl + j) * T::N;
    const DPrime Pr = dc->p[j];
    auto ld = [&](int i) { return galois ? src[galois_src(i, galois, LOGN)] : src[i]; };
    if (rem) {
        const u64* r = rem + (size_t)b * T::N;
        const u64 Pbig = dc->p[special].q, Pmod = dc->qmod[special][j];
        const u64 Pinv = dc->qinv[special][j], Pinv_sh = dc->qinv_sh[special][j];
        auto st = [&](int i, u64 v) {
            const u64 x = v + Pr.q - centered_to(r[i], Pbig, Pmod, Pr);
            dst[i] = csub(shoup_mul(x, Pinv, Pinv_sh, Pr.q), Pr.q);
        };
        ntt_inverse<T>(sm, Pr, twp(dc, j), ld, st);
    } else {
        auto st = [&](int i, u64 v) { dst[i] = v; };
        ntt_inverse<T>(sm, Pr, twp(dc, j), ld, st);
    }
}

// (1') QP remainder: rem[b][c] = iNTT_P(sigma_g(x_b.c)[P]) for the P limb of QP components
//      (giant-step digits: one component; the layer's final ModDown: both).  grid (ncomp, B)
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_qp_rem(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
            size_t comp_step, u32 galois, int nl, int special, u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int c = blockIdx.x, b = blockIdx.y;
    const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)c * comp_step + (size_t)nl * T::N;
    u64* dst = rem + ((size_t)b * gridDim.x + c) * T::N;
    const DPrime Pr = dc->p[special];
    auto ld = [&](int i) { return galois ? src[galois_src(i, galois, LOGN)] : src[i]; };
    auto st = [&](int i, u64 v) { dst[i] = v; };
    ntt_inverse<T>(sm, Pr, twp(dc, special), ld, st);
}

// (2) ModUp: D_{j,e} = NTT_{p_e}(d_j mod p_e) for e != j, e in [0, nl] (nl = special); all_e: e == j too
//     (QP digits are not the input limbs, so the inner product cannot read D_{j,j} from the input)
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_modup(const DCtx* __restrict__ dc, const u64* __restrict__ digits, u64* __restrict__ modup, int nl, int special,
           int all_e)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    int j, e;
    if (all_e) {
        j = blockIdx.x / (nl + 1);
        e = blockIdx.x % (nl + 1);
    } else {
        j = blockIdx.x / nl;
        e = blockIdx.x % nl;
        if (e >= j) ++e;
    }
    const int b = blockIdx.y;
    const int p = (e == nl) ? special : e;
    const DPrime Pr = dc->p[p];
    const u64* src = digits + ((size_t)b * nl + j) * T::N;
    u64* dst = modup + (((size_t)b * nl + j) * (nl + 1) + e) * T::N;
    auto ld = [&](int i) { return reduce64_lazy(src[i], Pr); };
#if CK_STREAM_STORES
    auto st = [&](int i, u64 v) { __stcs(dst + i, v); };   // ModUp words: read once, by the next kernel
#else
    auto st = [&](int i, u64 v) { dst[i] = v; };
#endif
    ntt_forward<T>(sm, Pr, twp(dc, p), ld, st);
}

// (3) ModDown, special-prime row: r_c = iNTT_P( sum_j D_{j,P} key_j.c[P] )  -- the inner product for
//     the special prime is computed in the (coalesced, staged) loader of the inverse NTT.
//     grid (2, B, G): one CTA per (component, ciphertext, rotation of the group).
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_moddown_intt(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const KsGroup grp, int L, int nl,
                  int special, u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int c = blockIdx.x, b = blockIdx.y, g = blockIdx.z, B = gridDim.y;
    const u64* __restrict__ key = grp.key[g];
    const DPrime Pr = dc->p[special];
    u64* dst = rem + (((size_t)g * B + b) * 2 + c) * T::N;
    auto ld = [&](int k) {
        Acc128 a;
        a.zero();
        for (int j = 0; j < nl; ++j)
            a.mac(modup[(((size_t)b * nl + j) * (nl + 1) + nl) * T::N + k],
                  key[(((size_t)j * 2 + c) * (L + 1) + L) * T::N + k]);
        return a.reduce(Pr);
    };
    auto st = [&](int i, u64 v) { dst[i] = v; };
    ntt_inverse<T>(sm, Pr, twp(dc, special), ld, st);
}

// (4) ModDown, data rows: x_g,c[i] = NTT_{q_i}(centered(r_g,c) mod q_i).  grid (nl, 2, B*G)
template <int LOGN, int NTH>
__global__ void __launch_bounds__(NTH)
k_ks_moddown_ntt(const DCtx* __restrict__ dc, const u64* __restrict__ rem, int nl, int special, u64* __restrict__ xo)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int i = blockIdx.x, c = blockIdx.y, gb = blockIdx.z;   // gb = g * B + b
    const DPrime Pr = dc->p[i];
    const u64 Pmod = dc->qmod[special][i];
    const u64 Pbig = dc->p[special].q;
    const u64* r = rem + ((size_t)gb * 2 + c) * T::N;
    u64* o = xo + (((size_t)gb * 2 + c) * (nl + 1) + i) * T::N;
    auto ld = [&](int k) { return centered_to(r[k], Pbig, Pmod, Pr); };
    auto st = [&](int k, u64 v) { o[k] = v; };
    ntt_forward<T>(sm, Pr, twp(dc, i), ld, st);
}

// (5) inner product over the data primes + ModDown combine + output permutation, for every rotation
//     g of the group, one CTA per (ciphertext, limb i, SOURCE block of IPO_BLK NTT-domain indices):
//       u_g,c[k] = sum_j D_{j,i}[k] key_g,j.c[i][k]            (D_{j,i}[k] loaded once for all g)
//       y_g,c[k] = (u_g,c[k] - x_g,c[i][k]) P^{-1} + addend_c[k]
//       out_g,c[i][k'] (+)= y_g,c[src_g(k')]                  (hoisted: out = sigma_g(y))
//     sigma_g maps the block of indices sharing their top log2(N/IPO_BLK) bits onto one block (those bits
//     are the low bits of brev(k), on which sigma_g acts as an affine map) so the permutation is done
//     through 2 x IPO_BLK words of shared memory and every global access is coalesced.
#define IPO_BLK 256
template <int NL>
__global__ void __launch_bounds__(IPO_BLK)
k_ks_ip_out(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ in, size_t ct_stride,
            size_t comp_off, u32 galois, const KsGroup grp, int L, int special, const u64* __restrict__ xo,
            size_t out_stride, const u64* __restrict__ add, size_t add_stride, u32 add_galois, int add_comp1,
            int accumulate, int B)
{
    __shared__ u64 ys[2][IPO_BLK];
    constexpr int nl = NL;
    const int n = dc->n, logn = dc->log_n;
    // grid (B, nl, N/1024): the ciphertext index runs fastest so the key rows of (g, i, block) are
    // read from DRAM once and then hit L2 for every ciphertext
    const int b = blockIdx.x, i = blockIdx.y, blk = blockIdx.z;
    const int t = threadIdx.x;
    const int k = blk * IPO_BLK + t;   // source index
    const DPrime Pr = dc->p[i];
    u64 dv[NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        if (j == i) {
            const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)j * n;
            dv[j] = galois ? src[galois_src(k, galois, logn)] : src[k];
        } else {
            dv[j] = modup[(((size_t)b * nl + j) * (nl + 1) + i) * n + k];
        }
    }
    u64 ad[2] = {0, 0};
    if (add) {
#pragma unroll
        for (int c = 0; c < 2; ++c)
            if (c == 0 || add_comp1) {
                const u64* a = add + (size_t)b * add_stride + ((size_t)c * nl + i) * n;
                ad[c] = add_galois ? a[galois_src(k, add_galois, logn)] : a[k];
            }
    }
    const u64 Pinv = dc->qinv[special][i], Pinv_sh = dc->qinv_sh[special][i];
    for (int g = 0; g < grp.G; ++g) {
        const u64* __restrict__ key = grp.key[g] + (size_t)i * n + k;
        const size_t kstride = (size_t)(L + 1) * n;
        Acc128 a0, a1;
        a0.zero();
        a1.zero();
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            a0.mac(dv[j], key[(size_t)(2 * j + 0) * kstride]);
            a1.mac(dv[j], key[(size_t)(2 * j + 1) * kstride]);
        }
        const u64 u[2] = {a0.reduce(Pr), a1.reduce(Pr)};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const u64 x = xo[((((size_t)g * B + b) * 2 + c) * (nl + 1) + i) * n + k];
            ys[c][t] = addmod(csub(shoup_mul(u[c] + Pr.q - x, Pinv, Pinv_sh, Pr.q), Pr.q), ad[c], Pr.q);
        }
        __syncthreads();
        // destination block of this source block under sigma_g, and the source of each destination
        const u32 gp = grp.scatter[g];
        int dblk = blk, sidx = t;
        if (gp) {
            dblk = galois_src(blk * IPO_BLK, grp.ginv[g], logn) / IPO_BLK;
            sidx = galois_src(dblk * IPO_BLK + t, gp, logn) - blk * IPO_BLK;
        }
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            u64& o = grp.out[g][(size_t)b * out_stride + ((size_t)c * nl + i) * n + (size_t)dblk * IPO_BLK + t];
            u64 v = ys[c][sidx];
            if (accumulate) v = addmod(v, o, Pr.q);
            o = v;
        }
        __syncthreads();
    }
}

// (5') inner product into the Q_l P basis (double hoisting, R11c) for every key switch g of the group,
//      one CTA per (ciphertext, row i in [0, nl], SOURCE block); row nl is the special prime P:
//        u_g,c[i][k] = sum_j D_{j,i}[k] key_g,j.c[p_i][k]
//        y_g,0 = u_g,0 + addend,  y_g,1 = u_g,1;   out_g,c[i][k'] (+)= y_g,c[src_g(k')]
//      baby step (scatter g, add_mulP): addend = P c0 (0 on the P row), out = sigma_g(y) with sigma_{g^-1}
//      permuted keys; giant step (no scatter): addend = sigma_g(w.c0) gathered from the QP input.
//      D_{j,j} comes from the Q input limb (in != null, baby) or from the ModUp buffer (all_e ModUp).
//      Each thread handles IPQ_BB ciphertexts of the same coefficient so every key word is read once
//      per IPQ_BB ciphertexts (the inner product is otherwise L2-bandwidth bound on the key reads).
template <int NL, bool SPLIT, int IPQ_BB>
__device__ __forceinline__ void ipqp_dot(const u64 (&dv)[IPQ_BB][NL], const u64* __restrict__ key, size_t kstride,
                                         const DPrime& Pr, int nb, u64 (&u)[IPQ_BB][2])
{
    if constexpr (SPLIT) {
        Acc3 a[IPQ_BB][2];
#pragma unroll
        for (int bb = 0; bb < IPQ_BB; ++bb) a[bb][0].zero(), a[bb][1].zero();
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const u64 k0 = key[(size_t)(2 * j + 0) * kstride], k1 = key[(size_t)(2 * j + 1) * kstride];
#pragma unroll
            for (int bb = 0; bb < IPQ_BB; ++bb) {
                const u32 x1 = (u32)(dv[bb][j] >> 21), x0 = (u32)dv[bb][j] & 0x1FFFFFu;
                a[bb][0].mac(x1, x0, k0);
                a[bb][1].mac(x1, x0, k1);
            }
        }
#pragma unroll
        for (int bb = 0; bb < IPQ_BB; ++bb)
            if (bb < nb) u[bb][0] = a[bb][0].reduce(Pr), u[bb][1] = a[bb][1].reduce(Pr);
    } else {
        Acc128 a[IPQ_BB][2];
#pragma unroll
        for (int bb = 0; bb < IPQ_BB; ++bb) a[bb][0].zero(), a[bb][1].zero();
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            const u64 k0 = key[(size_t)(2 * j + 0) * kstride], k1 = key[(size_t)(2 * j + 1) * kstride];
#pragma unroll
            for (int bb = 0; bb < IPQ_BB; ++bb) {
                a[bb][0].mac(dv[bb][j], k0);
                a[bb][1].mac(dv[bb][j], k1);
            }
        }
#pragma unroll
        for (int bb = 0; bb < IPQ_BB; ++bb)
            if (bb < nb) u[bb][0] = a[bb][0].reduce(Pr), u[bb][1] = a[bb][1].reduce(Pr);
    }
}

template <int NL, int IPQ_BB>
__global__ void __launch_bounds__(IPO_BLK)
k_ks_ip_qp(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ in, size_t ct_stride,
           size_t comp_off, const KsGroup grp, int L, int special, size_t out_stride, const u64* __restrict__ add,
           size_t add_stride, int add_nl, u32 add_galois, int add_mulP, int accumulate, int B, int allow_split)
{
    __shared__ u64 ys[IPQ_BB][2][IPO_BLK];
    constexpr int nl = NL;
    const int n = dc->n, logn = dc->log_n;
    const int b0 = blockIdx.x * IPQ_BB, i = blockIdx.y, blk = blockIdx.z;
    const int nb = min(IPQ_BB, B - b0);
    const int t = threadIdx.x;
    const int k = blk * IPO_BLK + t;
    const bool prow = (i == nl);
    const int p = prow ? special : i;
    const int krow = prow ? L : i;
    const DPrime Pr = dc->p[p];
    (void)add_nl;
    u64 dv[IPQ_BB][NL];
    u64 ad[IPQ_BB];
#pragma unroll
    for (int bb = 0; bb < IPQ_BB; ++bb) {
        const int b = b0 + (bb < nb ? bb : 0);
#pragma unroll
        for (int j = 0; j < NL; ++j) {
            if (j == i && in) dv[bb][j] = in[(size_t)b * ct_stride + comp_off + (size_t)j * n + k];
            else dv[bb][j] = modup[(((size_t)b * nl + j) * (nl + 1) + i) * n + k];
        }
        ad[bb] = 0;
        if (add) {
            if (add_mulP) {
                if (!prow)
                    ad[bb] = csub(shoup_mul(add[(size_t)b * add_stride + (size_t)i * n + k], dc->qmod[special][i],
                                            dc->qmod_sh[special][i], Pr.q), Pr.q);
            } else {
                const u64* a = add + (size_t)b * add_stride + (size_t)i * n;
                ad[bb] = add_galois ? a[galois_src(k, add_galois, logn)] : a[k];
            }
        }
    }
    // rows of primes < 2^42: split 21-bit IMAD.WIDE products (Acc3); 60-bit rows: 128-bit products
    const bool split = allow_split && Pr.q < SPLIT21_MAXQ;
    const size_t kstride = (size_t)(L + 1) * n;
    for (int g = 0; g < grp.G; ++g) {
        const u64* __restrict__ key = grp.key[g] + (size_t)krow * n + k;
        u64 u[IPQ_BB][2];
        if (split) ipqp_dot<NL, true, IPQ_BB>(dv, key, kstride, Pr, nb, u);
        else ipqp_dot<NL, false, IPQ_BB>(dv, key, kstride, Pr, nb, u);
#pragma unroll
        for (int bb = 0; bb < IPQ_BB; ++bb)
            if (bb < nb) {
                ys[bb][0][t] = addmod(u[bb][0], ad[bb], Pr.q);
                ys[bb][1][t] = u[bb][1];
            }
        __syncthreads();
        const u32 gp = grp.scatter[g];
        int dblk = blk, sidx = t;
        if (gp) {
            dblk = galois_src(blk * IPO_BLK, grp.ginv[g], logn) / IPO_BLK;
            sidx = galois_src(dblk * IPO_BLK + t, gp, logn) - blk * IPO_BLK;
        }
#pragma unroll
        for (int bb = 0; bb < IPQ_BB; ++bb) {
            if (bb >= nb) break;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                u64& o = grp.out[g][(size_t)(b0 + bb) * out_stride + ((size_t)c * (nl + 1) + i) * n +
                                    (size_t)dblk * IPO_BLK + t];
                u64 v = ys[bb][c][sidx];
                if (accumulate) v = addmod(v, o, Pr.q);
                o = v;
            }
        }
        __syncthreads();
    }
}

// layer-final ModDown of QP ciphertexts: out[b][c][i] = (y[b][c][i] - x[b][c][i]) P^{-1} mod q_i
__global__ void __launch_bounds__(256)
k_moddown_combine(const DCtx* __restrict__ dc, const u64* __restrict__ y, size_t y_stride, const u64* __restrict__ xo,
                  u64* __restrict__ out, size_t out_stride, int nl, int special)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x;
    const int i = blockIdx.y, c = blockIdx.z % 2, b = blockIdx.z / 2;
    const DPrime Pr = dc->p[i];
    const u64 yv = y[(size_t)b * y_stride + ((size_t)c * (nl + 1) + i) * n + k];
    const u64 xv = xo[(((size_t)b * 2 + c) * (nl + 1) + i) * n + k];
    out[(size_t)b * out_stride + ((size_t)c * nl + i) * n + k] =
        csub(shoup_mul(yv + Pr.q - xv, dc->qinv[special][i], dc->qinv_sh[special][i], Pr.q), Pr.q);
}

void keyswitch_modup(const Launch& L, const KsIn& in, int batch, int nl, const KsWork& w, bool qp_in)
{
    if (batch <= 0) return;
    const int special = L.n_data;   // special prime is stored after the data primes
    const size_t smem = sizeof(u64) << L.log_n;
    const int ne = qp_in ? nl + 1 : nl;   // ModUp targets per digit
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        constexpr int NW = NttThreadsWide<LG>::value;
        const int wm = ntt_wide_mask();
        auto kd = (wm & 1) ? k_ks_digits<LG, NW> : k_ks_digits<LG, NT>;
        auto km = (wm & 2) ? k_ks_modup<LG, NW> : k_ks_modup<LG, NT>;
        allow_smem(kd, smem);
        allow_smem(km, smem);
        const bool pm = L.probe && L.probe->on(PROBE_MODUP);
        if (L.probe && L.probe->on(PROBE_ALL)) {
            L.probe->bytes_by_kernel["k_ks_modup"] +=
                ((double)batch * nl + (double)batch * nl * ne) * (double)(8 << L.log_n);
            // butterflies per limb NTT: (N/2) log2 N; targets of digit j: every prime but q_j (QP: all)
            const double bf = (double)(1 << (L.log_n - 1)) * L.log_n * batch;
            for (int j = 0; j < nl; ++j)
                for (int e = 0; e <= nl; ++e) {
                    if (e == j && !qp_in) continue;
                    const int p = (e == nl) ? L.n_data : e;
                    if (L.pclass && L.pclass[p] == PC_FP) L.probe->bfly_fp += bf;
                    else L.probe->bfly_int += bf;
                }
        }
        if (qp_in) {
            auto kr = (wm & 1) ? k_ks_qp_rem<LG, NW> : k_ks_qp_rem<LG, NT>;
            allow_smem(kr, smem);
            ProbeScope ps_(L.probe, L.st, "k_ks_qp_rem");
            kr<<<dim3(1, batch), (wm & 1) ? NW : NT, smem, L.st>>>(L.dc, in.base, in.ct_stride, in.comp_off, 0, in.galois,
                                                                    nl, special, w.rem);
        }
        { ProbeScope ps_(L.probe, L.st, "k_ks_digits"); kd<<<dim3(nl, batch), (wm & 1) ? NW : NT, smem, L.st>>>(L.dc, in.base, in.ct_stride, in.comp_off, in.galois,
                                                              w.digits, nl, qp_in ? w.rem : nullptr, special); }
        if (pm) {
            L.probe->mark(L.st);
            // digits read once, nl x ne ModUp limbs written
            L.probe->alg_bytes += ((double)batch * nl + (double)batch * nl * ne) * (double)(8 << L.log_n);
        }
        { ProbeScope ps_(L.probe, L.st, "k_ks_modup"); km<<<dim3(nl * ne, batch), (wm & 2) ? NW : NT, smem, L.st>>>(L.dc, w.digits, w.modup, nl,
                                                                                        special, qp_in ? 1 : 0); }
        if (pm) L.probe->mark(L.st);
    });
    check_launch("keyswitch_modup");
    if (L.counter) *L.counter += qp_in ? 3 : 2;
}

// (5'') the baby-step QP inner product on the FP64 tensor cores (DMMA).  For one row i and one
//      coefficient k the group's inner products are a small matrix product
//        U[b][(g, c)] = sum_j D_{b,j}[k] key_g,j.c[k]       (16 ciphertexts x 2G columns x K = nl)
//      computed EXACTLY with mma.sync m16n8k4 f64 on operands split into 23-bit (q < 2^45) or 20-bit
//      (60-bit primes) parts: every partial product is an integer < 2^46 and every sum < 2^53, so the
//      tensor-core FP64 accumulation is exact.  The split sums are recombined mod q per output.
//      CTA = 16 ciphertexts x IPM_KT coefficients of one row; operands staged through shared memory
//      (XOR-swizzled), results staged per (g, c, b) row and written through the sigma_g block permutation
//      (aligned IPM_KT-blocks map onto aligned blocks, as for IPO_BLK).  Output as k_ks_ip_qp (baby mode).
#define IPM_KT 16
#define IPM_BT 16
#define IPM_THREADS 128

template <int NL, bool INT>
__global__ void __launch_bounds__(IPM_THREADS)
k_ks_ip_mma(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ in, size_t ct_stride,
            size_t comp_off, const KsGroup grp, int L, int special, size_t out_stride, int B)
{
    constexpr int nl = NL;
    constexpr int NLP = (NL + 3) & ~3;               // K padded to the MMA k-step
    constexpr int JS = IPM_KT * 16 + 4;              // j stride (words) of the swizzled operand tiles
    extern __shared__ u64 sm[];
    u64* Ds = sm;                                    // [NLP][KT][16 b]  (b ^ kk swizzle)
    u64* Ks = Ds + NLP * JS;                         // [NLP][KT][16 n]  n = 2 g + c
    u64* As = Ks + NLP * JS;                         // [KT][16 b]      addend P c0
    u64* Os = As + IPM_KT * 16;                      // [8 g][2 c][16 b][KT]
    const int n = dc->n, logn = dc->log_n;
    const int b0 = blockIdx.x * IPM_BT, i = blockIdx.y, k0 = blockIdx.z * IPM_KT;
    const bool prow = (i == nl);
    const int p = prow ? special : i;
    const int krow = prow ? L : i;
    const DPrime Pr = dc->p[p];
    if ((prime_class(Pr.q) != PC_FP) != INT) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int G = grp.G;
    // ---- stage D, keys, addend (coalesced along k); all loads of a thread issued before the stores.
    //      Thread: coefficient kk = tid % KT, rows r0 = tid / KT and r0 + 8 (b for D, n = 2g + c for keys)
    {
        const int kk = tid % IPM_KT, r0 = tid / IPM_KT;
        u64 dvals[NLP][2], kvals[NLP][2];
        const size_t jstride_d = (size_t)(nl + 1) * n, jstride_k = (size_t)2 * (L + 1) * n;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = r0 + 8 * h, b = b0 + r, g = r >> 1, c = r & 1;
            const u64* dsrc = modup + (((size_t)b * nl) * (nl + 1) + i) * n + k0 + kk;
            const u64* isrc = in + (size_t)b * ct_stride + comp_off + (size_t)i * n + k0 + kk;
            const u64* ksrc = g < G ? grp.key[g] + ((size_t)c * (L + 1) + krow) * n + k0 + kk : nullptr;
#pragma unroll
            for (int j = 0; j < NLP; ++j) {
                dvals[j][h] = (j < NL && b < B) ? ((j == i) ? *isrc : dsrc[(size_t)j * jstride_d]) : 0;
                kvals[j][h] = (j < NL && ksrc) ? ksrc[(size_t)j * jstride_k] : 0;
            }
        }
        u64 avals[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = r0 + 8 * h, b = b0 + r;
            avals[h] = (!prow && b < B) ? in[(size_t)b * ct_stride + (size_t)i * n + k0 + kk] : 0;
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int r = r0 + 8 * h;
#pragma unroll
            for (int j = 0; j < NLP; ++j) {
                Ds[j * JS + kk * 16 + (r ^ kk)] = dvals[j][h];
                Ks[j * JS + kk * 16 + (r ^ kk)] = kvals[j][h];
            }
            As[kk * 16 + r] =
                prow ? 0 : csub(shoup_mul(avals[h], dc->qmod[special][i], dc->qmod_sh[special][i], Pr.q), Pr.q);
        }
    }
    __syncthreads();
    // ---- per coefficient: split-operand DMMA over j, recombination mod q
    const int gid = lane >> 2, tig = lane & 3;
    constexpr int KPW = IPM_KT / (IPM_THREADS / 32);
    const double q = (double)Pr.q, qinv = 1.0 / q;
    const double two46 = 70368744177664.0;
    const double w46 = two46 - floor(two46 * qinv) * q, w46q = w46 / q, c23q = 8388608.0 / q;
    (void)w46q; (void)c23q;
    for (int kq = 0; kq < KPW; ++kq) {
        const int kk = warp * KPW + kq;
        // Karatsuba on the split parts: FP 3 products (hi hi, lo lo, (hi+lo)(hi+lo)), INT 6 (three-part)
        constexpr int NS = INT ? 6 : 3;
        double S[NS][2][4];
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e) S[s][t][e] = 0.0;
#pragma unroll
        for (int kb = 0; kb < NLP; kb += 4) {
            const int j = kb + tig;
            const u64 a0 = Ds[j * JS + kk * 16 + (gid ^ kk)], a1 = Ds[j * JS + kk * 16 + ((gid + 8) ^ kk)];
            if constexpr (!INT) {
                const u64 m = (1ULL << 23) - 1;
                const double a0h = u2d(a0 >> 23), a0l = u2d(a0 & m), a1h = u2d(a1 >> 23), a1l = u2d(a1 & m);
                const double a0s = a0h + a0l, a1s = a1h + a1l;
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const u64 bv = Ks[j * JS + kk * 16 + ((t * 8 + gid) ^ kk)];
                    const double bh = u2d(bv >> 23), bl = u2d(bv & m);
                    dmma16884(S[2][t], a0h, a1h, bh);
                    dmma16884(S[0][t], a0l, a1l, bl);
                    dmma16884(S[1][t], a0s, a1s, bh + bl);
                }
            } else {
                const u64 m = (1ULL << 20) - 1;
                const double x0[3] = {u2d(a0 & m), u2d((a0 >> 20) & m), u2d(a0 >> 40)};
                const double x1[3] = {u2d(a1 & m), u2d((a1 >> 20) & m), u2d(a1 >> 40)};
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const u64 bv = Ks[j * JS + kk * 16 + ((t * 8 + gid) ^ kk)];
                    const double y[3] = {u2d(bv & m), u2d((bv >> 20) & m), u2d(bv >> 40)};
                    dmma16884(S[0][t], x0[0], x1[0], y[0]);
                    dmma16884(S[1][t], x0[1], x1[1], y[1]);
                    dmma16884(S[2][t], x0[2], x1[2], y[2]);
                    dmma16884(S[3][t], x0[0] + x0[1], x1[0] + x1[1], y[0] + y[1]);
                    dmma16884(S[4][t], x0[1] + x0[2], x1[1] + x1[2], y[1] + y[2]);
                    dmma16884(S[5][t], x0[0] + x0[2], x1[0] + x1[2], y[0] + y[2]);
                }
            }
        }
        // outputs of this thread: (b = gid + 8 (e >> 1), n = 8 t + 2 tig + (e & 1)) -> g = 4 t + tig, c = e & 1
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const int bl = gid + 8 * (e >> 1), g = 4 * t + tig, c = e & 1;
                u64 u;
                if constexpr (!INT) {
                    // v = s0 + s1 2^23 + s2 2^46 mod q on the (otherwise idle) FP64 pipe: each part reduced to
                    // [-q/2, q/2] (exact), r1 2^23 is an exact scaling, r2 2^46 an exact-product fmodmul
                    const double s0 = S[0][t][e], s2 = S[2][t][e], s1 = S[1][t][e] - s2 - s0;   // Karatsuba middle
                    const double r0 = freduce(s0, q, qinv), r1 = freduce(s1, q, qinv), r2 = freduce(s2, q, qinv);
                    const double k1 = __fma_rn(r1, c23q, CK_RND_MAGIC) - CK_RND_MAGIC;
                    const double t1 = __fma_rn(-k1, q, r1 * 8388608.0);
                    const double t2 = fmodmul(r2, w46, w46q, q);
                    u = fcanon(t2 + t1 + r0, q, qinv);
                } else {
                    // P0 = S0, P1 = S1, P2 = S2, P01 = S3, P12 = S4, P02 = S5 (all exact integers < 2^53)
                    const double P0 = S[0][t][e], P1 = S[1][t][e], P2 = S[2][t][e];
                    const u64 s0 = d2u(P0), s1 = d2u(S[3][t][e] - P0 - P1), s2 = d2u(S[5][t][e] - P0 - P2 + P1),
                              s3 = d2u(S[4][t][e] - P1 - P2), s4 = d2u(P2);
                    // v = s0 + s1 2^20 + s2 2^40 + s3 2^60 + s4 2^80   (each s < 2^48)
                    u64 lo = s0, hi = 0, add;
                    add = s1 << 20; lo += add; hi += (lo < add) + (s1 >> 44);
                    add = s2 << 40; lo += add; hi += (lo < add) + (s2 >> 24);
                    add = s3 << 60; lo += add; hi += (lo < add) + (s3 >> 4);
                    hi += s4 << 16;
                    u = reduce128(hi, lo, Pr);
                }
                if (c == 0) u = addmod(u, As[kk * 16 + bl], Pr.q);
                if (g < G) Os[((g * 2 + c) * 16 + bl) * IPM_KT + (kk ^ ((bl + 4 * g) & 15))] = u;
            }
    }
    __syncthreads();
    // ---- permuted, coalesced write: row (g, c, b) of IPM_KT destination words per 16 lanes; the
    //      destination block and source index of this lane are computed once per g
    {
        const int t = tid % IPM_KT, r0 = tid / IPM_KT;   // r0 in [0, 8): rows r0, r0 + 8, ...
        for (int g = 0; g < G; ++g) {
            const u32 gp = grp.scatter[g];
            int dblk = blockIdx.z, sidx = t;
            if (gp) {
                dblk = galois_src(k0, grp.ginv[g], logn) / IPM_KT;
                sidx = galois_src(dblk * IPM_KT + t, gp, logn) - k0;
            }
            u64* og = grp.out[g] + (size_t)i * n + (size_t)dblk * IPM_KT + t;
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                const int rr = r0 + 8 * h;             // rr = c * 16 + bl
                const int c = rr >> 4, bl = rr & 15, b = b0 + bl;
                if (b < B)
                    og[(size_t)b * out_stride + (size_t)c * (nl + 1) * n] =
                        Os[((g * 2 + c) * 16 + bl) * IPM_KT + (sidx ^ ((bl + 4 * g) & 15))];
            }
        }
    }
}

static size_t ip_mma_smem(int nl)
{
    const int NLP = (nl + 3) & ~3, JS = IPM_KT * 16 + 4;
    return sizeof(u64) * ((size_t)2 * NLP * JS + IPM_KT * 16 + 8 * 2 * 16 * IPM_KT);
}

// QP-basis finish (R11c): inner product over all nl+1 rows, no ModDown.  in (baby: the Q_l input whose
// limb j is D_{j,j}) or null (giant: all_e ModUp); addend per KsOut (add_mulP / add_galois)
void keyswitch_finish_qp(const Launch& L, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                         const KsOut& out, bool baby)
{
    if (batch <= 0 || grp.G <= 0) return;
    if (grp.G > KS_GMAX || nl > KS_LMAX) throw std::runtime_error("keyswitch_finish_qp: group/limb limits");
    const int n = 1 << L.log_n;
    if (n < IPO_BLK) throw std::runtime_error("N >= 1024 required");
    static const int bbv = [] {
        const char* e = getenv("CKKS_IPQ_BB");
        return e ? atoi(e) : 2;
    }();
    static const int spl = [] {
        const char* e = getenv("CKKS_IP_SPLIT");
        return e ? atoi(e) : 1;
    }();
    const u64* ib = baby ? in.base : nullptr;
    static const int use_mma = [] {
        const char* e = getenv("CKKS_IP_MMA");
        return e ? atoi(e) : 2;
    }();
    static const int use_giant = [] {
        const char* e = getenv("CKKS_IP_GIANT");
        return e ? atoi(e) : 1;
    }();
    if (!baby && use_giant && grp.G == 1 && out.accumulate && out.add && !grp.scatter[0] && out.base == grp.out[0]) {
        ip_giant(L, grp.key[0], batch, nl, w, out.base, out.ct_stride, out.add, out.add_stride, out.add_galois);
        return;
    }
    if (baby && use_mma == 2 && grp.G >= 2 && out.add == in.base && !out.accumulate) {
        ip_mma_pipelined(L, in, grp, batch, nl, w, out.ct_stride);
        return;
    }
    if (baby && use_mma && grp.G >= 2 && out.add == in.base && !out.accumulate) {
        const size_t smem = ip_mma_smem(nl);
        const dim3 grid((batch + IPM_BT - 1) / IPM_BT, nl + 1, n / IPM_KT);
#define IPM_CASE(V)                                                                                                  \
    case V: {                                                                                                         \
        allow_smem(k_ks_ip_mma<V, false>, smem);                                                                      \
        allow_smem(k_ks_ip_mma<V, true>, smem);                                                                       \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_mma");                                                                 \
        k_ks_ip_mma<V, false><<<grid, IPM_THREADS, smem, L.st>>>(L.dc, w.modup, in.base, in.ct_stride, in.comp_off,  \
                                                               grp, L.n_data, L.n_data, out.ct_stride, batch);        \
        k_ks_ip_mma<V, true><<<grid, IPM_THREADS, smem, L.st>>>(L.dc, w.modup, in.base, in.ct_stride, in.comp_off,   \
                                                              grp, L.n_data, L.n_data, out.ct_stride, batch);         \
    } break;
        switch (nl) {
            IPM_CASE(1) IPM_CASE(2) IPM_CASE(3) IPM_CASE(4) IPM_CASE(5) IPM_CASE(6) IPM_CASE(7) IPM_CASE(8)
            IPM_CASE(9) IPM_CASE(10) IPM_CASE(11) IPM_CASE(12) IPM_CASE(13) IPM_CASE(14) IPM_CASE(15) IPM_CASE(16)
        default: throw std::runtime_error("nl > 16");
        }
#undef IPM_CASE
        check_launch("keyswitch_finish_qp(mma)");
        if (L.counter) *L.counter += 2;
        return;
    }
#define IPQ_CASE(V)                                                                                                  \
    case V: {                                                                                                         \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_qp");                                                                  \
        if (bbv == 4)                                                                                                 \
            k_ks_ip_qp<V, 4><<<dim3((batch + 3) / 4, nl + 1, n / IPO_BLK), IPO_BLK, 0, L.st>>>(                      \
                L.dc, w.modup, ib, in.ct_stride, in.comp_off, grp, L.n_data, L.n_data, out.ct_stride, out.add,         \
                out.add_stride, nl + 1, out.add_galois, baby ? 1 : 0, out.accumulate, batch, spl);                     \
        else if (bbv == 1)                                                                                            \
            k_ks_ip_qp<V, 1><<<dim3(batch, nl + 1, n / IPO_BLK), IPO_BLK, 0, L.st>>>(                                \
                L.dc, w.modup, ib, in.ct_stride, in.comp_off, grp, L.n_data, L.n_data, out.ct_stride, out.add,         \
                out.add_stride, nl + 1, out.add_galois, baby ? 1 : 0, out.accumulate, batch, spl);                     \
        else                                                                                                          \
            k_ks_ip_qp<V, 2><<<dim3((batch + 1) / 2, nl + 1, n / IPO_BLK), IPO_BLK, 0, L.st>>>(                      \
                L.dc, w.modup, ib, in.ct_stride, in.comp_off, grp, L.n_data, L.n_data, out.ct_stride, out.add,         \
                out.add_stride, nl + 1, out.add_galois, baby ? 1 : 0, out.accumulate, batch, spl);                     \
    } break;
    switch (nl) {
        IPQ_CASE(1) IPQ_CASE(2) IPQ_CASE(3) IPQ_CASE(4) IPQ_CASE(5) IPQ_CASE(6) IPQ_CASE(7) IPQ_CASE(8)
        IPQ_CASE(9) IPQ_CASE(10) IPQ_CASE(11) IPQ_CASE(12) IPQ_CASE(13) IPQ_CASE(14) IPQ_CASE(15) IPQ_CASE(16)
    default: throw std::runtime_error("nl > 16");
    }
#undef IPQ_CASE
    check_launch("keyswitch_finish_qp");
    if (L.counter) *L.counter += 1;
}

// layer-final ModDown of B QP ciphertexts y (stride y_stride) into Q_l ciphertexts out
void moddown_qp(const Launch& L, const uint64_t* y, size_t y_stride, int batch, int nl, const KsWork& w, uint64_t* out,
                size_t out_stride)
{
    if (batch <= 0) return;
    const int special = L.n_data;
    const int n = 1 << L.log_n;
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        allow_smem(k_ks_qp_rem<LG, NT>, smem);
        allow_smem(k_ks_moddown_ntt<LG, NT>, smem);
        { ProbeScope ps_(L.probe, L.st, "k_ks_qp_rem");
          k_ks_qp_rem<LG, NT><<<dim3(2, batch), NT, smem, L.st>>>(L.dc, y, y_stride, 0, (size_t)(nl + 1) * n, 0, nl,
                                                                 special, w.rem); }
        { ProbeScope ps_(L.probe, L.st, "k_ks_moddown_ntt");
          k_ks_moddown_ntt<LG, NT><<<dim3(nl, 2, batch), NT, smem, L.st>>>(L.dc, w.rem, nl, special, w.acc); }
    });
    { ProbeScope ps_(L.probe, L.st, "k_moddown_combine");
      k_moddown_combine<<<dim3(n / 256, nl, 2 * batch), 256, 0, L.st>>>(L.dc, y, y_stride, w.acc, out, out_stride, nl,
                                                                         special); }
    check_launch("moddown_qp");
    if (L.counter) *L.counter += 3;
}

// P ct -> QP basis (a hoisted baby step with g == 1): out[c][i] = P in[c][i], out[c][nl] = 0
__global__ void __launch_bounds__(256)
k_lift_qp(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t in_stride, u64* __restrict__ out,
          size_t out_stride, int nl, int special)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x;
    const int i = blockIdx.y, c = blockIdx.z % 2, b = blockIdx.z / 2;
    u64 v = 0;
    if (i < nl) {
        const DPrime Pr = dc->p[i];
        v = csub(shoup_mul(in[(size_t)b * in_stride + ((size_t)c * nl + i) * n + k], dc->qmod[special][i],
                           dc->qmod_sh[special][i], Pr.q), Pr.q);
    }
    out[(size_t)b * out_stride + ((size_t)c * (nl + 1) + i) * n + k] = v;
}

void lift_qp(const Launch& L, const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, int batch, int nl)
{
    if (batch <= 0) return;
    const int n = 1 << L.log_n;
    k_lift_qp<<<dim3(n / 256, nl + 1, 2 * batch), 256, 0, L.st>>>(L.dc, in, in_stride, out, out_stride, nl, L.n_data);
    check_launch("lift_qp");
    if (L.counter) ++*L.counter;
}

static void launch_ks_ip_out(const Launch& L, const KsWork& w, const KsIn& in, const KsGroup& grp, int batch, int nl,
                             const KsOut& out)
{
    const int n = 1 << L.log_n;
    const dim3 grid(batch, nl, n / IPO_BLK);
#define IP_CASE(V)                                                                                                   \
    case V:                                                                                                           \
        { ProbeScope ps_(L.probe, L.st, "k_ks_ip_out"); k_ks_ip_out<V><<<grid, IPO_BLK, 0, L.st>>>(L.dc, w.modup, in.base, in.ct_stride, in.comp_off, in.galois, grp,  \
                                                   L.n_data, L.n_data, w.acc, out.ct_stride, out.add, out.add_stride, \
                                                   out.add_galois, out.add_comp1, out.accumulate, batch); }             \
        break;
    switch (nl) {
        IP_CASE(1) IP_CASE(2) IP_CASE(3) IP_CASE(4) IP_CASE(5) IP_CASE(6) IP_CASE(7) IP_CASE(8)
        IP_CASE(9) IP_CASE(10) IP_CASE(11) IP_CASE(12) IP_CASE(13) IP_CASE(14) IP_CASE(15) IP_CASE(16)
    default: throw std::runtime_error("nl > 16");
    }
#undef IP_CASE
}

void keyswitch_finish(const Launch& L, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                      const KsOut& out)
{
    if (batch <= 0 || grp.G <= 0) return;
    if (grp.G > KS_GMAX || nl > KS_LMAX) throw std::runtime_error("keyswitch_finish: group/limb limits");
    const int special = L.n_data;
    const size_t smem = sizeof(u64) << L.log_n;
    const int n = 1 << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        constexpr int NW = NttThreadsWide<LG>::value;
        const int wm = ntt_wide_mask();
        auto ki = (wm & 4) ? k_ks_moddown_intt<LG, NW> : k_ks_moddown_intt<LG, NT>;
        auto kn = (wm & 8) ? k_ks_moddown_ntt<LG, NW> : k_ks_moddown_ntt<LG, NT>;
        allow_smem(ki, smem);
        allow_smem(kn, smem);
        { ProbeScope ps_(L.probe, L.st, "k_ks_moddown_intt"); ki<<<dim3(2, batch, grp.G), (wm & 4) ? NW : NT, smem, L.st>>>(L.dc, w.modup, grp, L.n_data, nl, special,
                                                                         w.rem); }
        { ProbeScope ps_(L.probe, L.st, "k_ks_moddown_ntt"); kn<<<dim3(nl, 2, batch * grp.G), (wm & 8) ? NW : NT, smem, L.st>>>(L.dc, w.rem, nl, special, w.acc); }
    });
    if (n < IPO_BLK) throw std::runtime_error("N >= 1024 required");
    launch_ks_ip_out(L, w, in, grp, batch, nl, out);
    check_launch("keyswitch_finish");
    if (L.counter) *L.counter += 3;
}

void keyswitch(const Launch& L, const KsIn& in, const uint64_t* key, int batch, int nl, const KsWork& w,
               const KsOut& out)
{
    const bool pk = L.probe && L.probe->on(PROBE_KEYSWITCH);
    if (pk) {
        L.probe->mark(L.st);
        // switched component + addend in, 2 components out, key rows used once per launch
        L.probe->alg_bytes += (4.0 * batch * nl + 2.0 * nl * (nl + 1)) * (double)(8 << L.log_n);
    }
    keyswitch_modup(L, in, batch, nl, w, false);
    KsGroup grp{};
    grp.key[0] = key;
    grp.out[0] = out.base;
    grp.scatter[0] = 0;
    grp.G = 1;
    keyswitch_finish(L, in, grp, batch, nl, w, out);
    if (pk) L.probe->mark(L.st);
}

__global__ void k_galois_limbs(const DCtx* __restrict__ dc, const u64* __restrict__ in, u64* __restrict__ out, u32 g)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x;
    const size_t limb = blockIdx.y + (size_t)blockIdx.z * gridDim.y;
    out[limb * n + k] = in[limb * n + galois_src(k, g, dc->log_n)];
}

void galois_limbs(const Launch& L, const uint64_t* in, uint64_t* out, size_t limbs, uint32_t g)
{
    const int n = 1 << L.log_n;
    for (size_t done = 0; done < limbs; done += 65535) {
        const unsigned cnt = (unsigned)std::min<size_t>(limbs - done, 65535);
        k_galois_limbs<<<dim3(n / 256, cnt, 1), 256, 0, L.st>>>(L.dc, in + done * n, out + done * n, g);
    }
    check_launch("galois_limbs");
    if (L.counter) ++*L.counter;
}

}  // namespace ck
