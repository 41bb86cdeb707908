// k_ipqp.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path: the key-switch inner products on
// the integer pipes (IMAD): the data-row inner product fused with the ModDown combine and the output
// permutation (non-hoisted / hoisted rotations, relinearisation), and the Q_l P-basis inner product of
// double hoisting for groups the tensor-core kernel does not take (R11c).  Layouts:
//   ModUp output  [b][digit j][row 0..nl+K-1][N]   (rows nl..: the special primes P_0..P_{K-1})
//   key           [digit j][comp][prime 0..L+K-1][N]
#include "kinternal.cuh"

namespace ck {

#define KS_ND_CASES(M) M(1) M(2) M(3) M(4) M(5) M(6) M(7) M(8) M(9) M(10) M(11) M(12) M(13) M(14) M(15) M(16)

// (5) inner product over the data primes + ModDown combine + output permutation, for every rotation
//     g of the group, one CTA per (ciphertext, limb i, SOURCE block of IPO_BLK NTT-domain indices):
//       u_g,c[k] = sum_j D_{j,i}[k] key_g,j.c[i][k]            (D_{j,i}[k] loaded once for all g)
//       y_g,c[k] = (u_g,c[k] - x_g,c[i][k]) P^{-1} + addend_c[k]
//       out_g,c[i][k'] (+)= y_g,c[src_g(k')]                  (hoisted: out = sigma_g(y))
//     D_{j,i} for q_i in digit j is the switched limb itself (d_j = d mod q_i).  sigma_g maps the block of
//     indices sharing their top log2(N/IPO_BLK) bits onto one block (those bits are the low bits of brev(k),
//     on which sigma_g acts as an affine map) so the permutation is done through 2 x IPO_BLK words of shared
//     memory and every global access is coalesced.
#define IPO_BLK 256
template <int ND>
__global__ void __launch_bounds__(IPO_BLK)
k_ks_ip_out(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ in, size_t ct_stride,
            size_t comp_off, u32 galois, const KsGroup grp, int nl, const u64* __restrict__ xo, size_t out_stride,
            const u64* __restrict__ add, size_t add_stride, u32 add_galois, int add_comp1, int accumulate, int B)
{
    __shared__ u64 ys[2][IPO_BLK];
    const int n = dc->n, logn = dc->log_n, K = dc->n_special, ne = nl + K, np = dc->n_data + K;
    // grid (B, nl, N/IPO_BLK): the ciphertext index runs fastest so the key rows of (g, i, block) are
    // read from DRAM once and then hit L2 for every ciphertext
    const int b = blockIdx.x, i = blockIdx.y, blk = blockIdx.z;
    const int t = threadIdx.x;
    const int k = blk * IPO_BLK + t;   // source index
    const DPrime Pr = dc->p[i];
    u64 dv[ND];
#pragma unroll
    for (int j = 0; j < ND; ++j) {
        const int s0 = dc->dig_start[j];
        if (i >= s0 && i < s0 + dc->dig_len[j]) {
            const u64* src = in + (size_t)b * ct_stride + comp_off + (size_t)i * n;
            dv[j] = galois ? src[galois_src(k, galois, logn)] : src[k];
        } else {
            dv[j] = modup[(((size_t)b * ND + j) * ne + i) * n + k];
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
    const u64 Pinv = dc->pinv[i], Pinv_sh = dc->pinv_sh[i];
    for (int g = 0; g < grp.G; ++g) {
        const u64* __restrict__ key = grp.key[g] + (size_t)i * n + k;
        const size_t kstride = (size_t)np * n;
        Acc128 a0, a1;
        a0.zero();
        a1.zero();
#pragma unroll
        for (int j = 0; j < ND; ++j) {
            a0.mac(dv[j], key[(size_t)(2 * j + 0) * kstride]);
            a1.mac(dv[j], key[(size_t)(2 * j + 1) * kstride]);
        }
        const u64 u[2] = {a0.reduce(Pr), a1.reduce(Pr)};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
            const u64 x = xo[((((size_t)g * B + b) * 2 + c) * ne + i) * n + k];
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
//      one CTA per (ciphertext, row i in [0, nl + K), SOURCE block); rows nl.. are the special primes:
//        u_g,c[i][k] = sum_j D_{j,i}[k] key_g,j.c[p_i][k]
//        y_g,0 = u_g,0 + addend,  y_g,1 = u_g,1;   out_g,c[i][k'] (+)= y_g,c[src_g(k')]
//      baby step (scatter g, add_mulP): addend = P c0 (0 on the special rows), out = sigma_g(y) with sigma_{g^-1}
//      permuted keys; giant step (no scatter): addend = sigma_g(w.c0) gathered from the QP input.
//      D_{j,i} for q_i in digit j comes from the Q input limb (in != null, baby) or from the ModUp buffer
//      (all_e ModUp).  Each thread handles IPQ_BB ciphertexts of the same coefficient so every key word is read
//      once per IPQ_BB ciphertexts (the inner product is otherwise L2-bandwidth bound on the key reads).
template <int ND, bool SPLIT, int IPQ_BB>
__device__ __forceinline__ void ipqp_dot(const u64 (&dv)[IPQ_BB][ND], const u64* __restrict__ key, size_t kstride,
                                         const DPrime& Pr, int nb, u64 (&u)[IPQ_BB][2])
{
    if constexpr (SPLIT) {
        Acc3 a[IPQ_BB][2];
#pragma unroll
        for (int bb = 0; bb < IPQ_BB; ++bb) a[bb][0].zero(), a[bb][1].zero();
#pragma unroll
        for (int j = 0; j < ND; ++j) {
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
        for (int j = 0; j < ND; ++j) {
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

template <int ND, int IPQ_BB>
__global__ void __launch_bounds__(IPO_BLK)
k_ks_ip_qp(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ in, size_t ct_stride,
           size_t comp_off, const KsGroup grp, int nl, size_t out_stride, const u64* __restrict__ add,
           size_t add_stride, u32 add_galois, int add_mulP, int accumulate, int B, int allow_split)
{
    __shared__ u64 ys[IPQ_BB][2][IPO_BLK];
    const int n = dc->n, logn = dc->log_n, K = dc->n_special, ne = nl + K, np = dc->n_data + K;
    const int b0 = blockIdx.x * IPQ_BB, i = blockIdx.y, blk = blockIdx.z;
    const int nb = min(IPQ_BB, B - b0);
    const int t = threadIdx.x;
    const int k = blk * IPO_BLK + t;
    const bool srow = (i >= nl);
    const int p = ext_prime_of(i, nl, dc->n_data);   // = the key's prime row
    const DPrime Pr = dc->p[p];
    u64 dv[IPQ_BB][ND];
    u64 ad[IPQ_BB];
#pragma unroll
    for (int bb = 0; bb < IPQ_BB; ++bb) {
        const int b = b0 + (bb < nb ? bb : 0);
#pragma unroll
        for (int j = 0; j < ND; ++j) {
            const int s0 = dc->dig_start[j];
            if (in && i >= s0 && i < s0 + dc->dig_len[j] && !srow)
                dv[bb][j] = in[(size_t)b * ct_stride + comp_off + (size_t)i * n + k];
            else
                dv[bb][j] = modup[(((size_t)b * ND + j) * ne + i) * n + k];
        }
        ad[bb] = 0;
        if (add) {
            if (add_mulP) {
                if (!srow)
                    ad[bb] = csub(shoup_mul(add[(size_t)b * add_stride + (size_t)i * n + k], dc->pmod[i], dc->pmod_sh[i],
                                            Pr.q), Pr.q);
            } else {
                const u64* a = add + (size_t)b * add_stride + (size_t)i * n;
                ad[bb] = add_galois ? a[galois_src(k, add_galois, logn)] : a[k];
            }
        }
    }
    // rows of primes < 2^42: split 21-bit IMAD.WIDE products (Acc3); 60-bit rows: 128-bit products
    const bool split = allow_split && Pr.q < SPLIT21_MAXQ;
    const size_t kstride = (size_t)np * n;
    for (int g = 0; g < grp.G; ++g) {
        const u64* __restrict__ key = grp.key[g] + (size_t)p * n + k;
        u64 u[IPQ_BB][2];
        if (split) ipqp_dot<ND, true, IPQ_BB>(dv, key, kstride, Pr, nb, u);
        else ipqp_dot<ND, false, IPQ_BB>(dv, key, kstride, Pr, nb, u);
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
                u64& o = grp.out[g][(size_t)(b0 + bb) * out_stride + ((size_t)c * ne + i) * n + (size_t)dblk * IPO_BLK + t];
                u64 v = ys[bb][c][sidx];
                if (accumulate) v = addmod(v, o, Pr.q);
                o = v;
            }
        }
        __syncthreads();
    }
}

void ip_out(const Launch& L, const KsWork& w, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsOut& out)
{
    const int n = 1 << L.log_n;
    const dim3 grid(batch, nl, n / IPO_BLK);
#define IP_CASE(V)                                                                                                   \
    case V: {                                                                                                         \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_out");                                                                 \
        k_ks_ip_out<V><<<grid, IPO_BLK, 0, L.st>>>(L.dc, w.modup, in.base, in.ct_stride, in.comp_off, in.galois, grp, \
                                                   nl, w.acc, out.ct_stride, out.add, out.add_stride, out.add_galois, \
                                                   out.add_comp1, out.accumulate, batch);                             \
    } break;
    switch (L.active_digits(nl)) {
        KS_ND_CASES(IP_CASE)
    default: throw std::runtime_error("more than 16 digits");
    }
#undef IP_CASE
}

// host launcher of k_ks_ip_qp: IPQ_BB ciphertexts per thread (bbv), 21-bit split products allowed (spl)
void ip_qp(const Launch& L, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w, const KsOut& out,
           bool baby, int bbv, int spl)
{
    const int n = 1 << L.log_n;
    const u64* ib = baby ? in.base : nullptr;
    const int nd = L.active_digits(nl), ne = nl + L.n_special;
#define IPQ_CASE(V)                                                                                                  \
    case V: {                                                                                                         \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_qp");                                                                  \
        if (bbv == 4)                                                                                                 \
            k_ks_ip_qp<V, 4><<<dim3((batch + 3) / 4, ne, n / IPO_BLK), IPO_BLK, 0, L.st>>>(                          \
                L.dc, w.modup, ib, in.ct_stride, in.comp_off, grp, nl, out.ct_stride, out.add, out.add_stride,        \
                out.add_galois, baby ? 1 : 0, out.accumulate, batch, spl);                                            \
        else if (bbv == 1)                                                                                            \
            k_ks_ip_qp<V, 1><<<dim3(batch, ne, n / IPO_BLK), IPO_BLK, 0, L.st>>>(                                    \
                L.dc, w.modup, ib, in.ct_stride, in.comp_off, grp, nl, out.ct_stride, out.add, out.add_stride,        \
                out.add_galois, baby ? 1 : 0, out.accumulate, batch, spl);                                            \
        else                                                                                                          \
            k_ks_ip_qp<V, 2><<<dim3((batch + 1) / 2, ne, n / IPO_BLK), IPO_BLK, 0, L.st>>>(                          \
                L.dc, w.modup, ib, in.ct_stride, in.comp_off, grp, nl, out.ct_stride, out.add, out.add_stride,        \
                out.add_galois, baby ? 1 : 0, out.accumulate, batch, spl);                                            \
    } break;
    switch (nd) {
        KS_ND_CASES(IPQ_CASE)
    default: throw std::runtime_error("more than 16 digits");
    }
#undef IPQ_CASE
}

}  // namespace ck
