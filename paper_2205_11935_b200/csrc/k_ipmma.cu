// k_ipmma.cu -- sm_100a kernel of the CKKS encrypted-dense-layer hot path: the hoisted baby-step
// key-switch inner product in the Q_l P basis (double hoisting, R11c) on the FP64 tensor
// cores.  Layouts:
//   ModUp output  [b][digit j][row 0..nl+K-1][N]   (rows nl..: the special primes P_0..P_{K-1})
//   key           [digit j][comp][prime 0..L+K-1][N]  (pre-permuted by sigma_g^{-1})
//   baby output   [b][comp][row 0..nl+K-1][N]   (Q_l P basis, sigma_g-permuted)
#include "kinternal.cuh"

namespace ck {

// For one row i (prime) and one coefficient k the group's inner products are a small matrix product
//     U[b][(g, c)] = sum_{j < nd} D_{b,j}[k] key_{g,j,c}[k]     (16 ciphertexts x 2G columns x K = nd digits)
// computed EXACTLY with mma.sync m16n8k4 f64 on split operands: q < 2^45 two 23-bit parts and
// Karatsuba (3 products, every sum < 2^53 for nl <= 16), 60-bit primes three 20-bit parts and 6
// products.  The split sums are recombined mod q per output, the addend P c0 is added, and the
// result is written through the sigma_g block permutation (aligned IP2_KT-blocks of NTT indices map
// onto aligned blocks).
//
// Pipelined form: one CTA owns one row and IP2_KT coefficients and streams every ciphertext of the
// batch in tiles of 16 through a cp.async pipeline (D tile + raw c0 addend per stage), so its key
// tile (all digits, all G rotations, both components) is read once per launch and, for the FP class,
// split once into registers; loads of the next tile overlap the DMMA work and the permuted stores
// of the current one.
#define IP2_KT 16
#define IP2_THREADS 256
#ifndef IP2_ST
#define IP2_ST 3
#endif
// 60-bit rows: 128-bit IMAD products (1; measured slower: 188 vs 168, and at round end 162 vs 140 ms per step) or the 6-product
// DMMA split (0, default)
// FP rows: all coefficients' DMMAs before their epilogues (1), or coefficient by coefficient (0)
#ifndef CK_STREAM_STORES
#define CK_STREAM_STORES 0
#endif
#ifndef IP2_FP_BATCH
#define IP2_FP_BATCH 1
#endif
#ifndef IP2_INT_IMAD
#define IP2_INT_IMAD 0
#endif

__device__ __forceinline__ void ip2_cp8(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void ip2_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void ip2_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

template <int NL>
struct Ip2Shape {                                          // NL = digits (the contraction length)
    static constexpr int NLP = (NL + 3) & ~3;              // K padded to the MMA k-step
    static constexpr int JS = IP2_KT * 16 + 4;             // j stride (words) of the swizzled tiles
    static constexpr int SD = NLP * JS + IP2_KT * 16;      // words per stage: D tile + c0 addend
    static constexpr size_t smem = sizeof(u64) * ((size_t)NLP * JS + (size_t)IP2_ST * SD + 8 * 2 * 16 * IP2_KT + 8);
};

template <int NL, bool INT>
__device__ __forceinline__ void ip2_body(const DCtx* __restrict__ dc, const u64* __restrict__ modup,
                                         const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
                                         const KsGroup& grp, int nl, size_t out_stride, int B, u64* sm,
                                         int i, int cblk, int mac_layout)
{
    constexpr int NLP = Ip2Shape<NL>::NLP, JS = Ip2Shape<NL>::JS, SD = Ip2Shape<NL>::SD;
    constexpr int KPW = IP2_KT / (IP2_THREADS / 32);       // coefficients per warp
    constexpr bool CACHE = !INT && NLP <= 8 && !IP2_FP_BATCH;   // FP class: split key fragments in registers
    u64* Ks = sm;                                          // [NLP][KT][16 n]  n = 2 g + c  (n ^ kk swizzle)
    u64* Dst = Ks + NLP * JS;                              // [ST][ D [NLP][KT][16 b] | c0 [KT][16 b] ]
    u64* Os = Dst + IP2_ST * SD;                           // [8 g][2 c][16 b][KT]
    u64** Ob = reinterpret_cast<u64**>(Os + 8 * 2 * 16 * IP2_KT);   // [8 g] destination block of rotation g
    const int n = dc->n, logn = dc->log_n, K = dc->n_special, ne = nl + K, np = dc->n_data + K;
    const int k0 = cblk * IP2_KT;
    const bool prow = (i >= nl);                           // a special-prime row
    const int p = ext_prime_of(i, nl, dc->n_data);
    const int krow = p;
    const DPrime Pr = dc->p[p];
    int ownj = -1;                                         // the digit whose primes include q_i (D = input limb)
    for (int j = 0; j < NL; ++j)
        if (!prow && i >= dc->dig_start[j] && i < dc->dig_start[j] + dc->dig_len[j]) ownj = j;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int G = grp.G;
    const int nbt = (B + 15) / 16;
    // ---- stage fill: thread = (coefficient fk, ciphertext row fr); digits j stride (nl+K) N
    const int fk = tid % IP2_KT, fr = tid / IP2_KT;
    auto fill = [&](int bt) {
        u64* S = Dst + (bt % IP2_ST) * SD;
        const int b = bt * 16 + fr;
        if (b < B) {
            const u64* dsrc = modup + (((size_t)b * NL) * ne + i) * n + k0 + fk;
            const u64* isrc = in + (size_t)b * ct_stride + (size_t)i * n + k0 + fk;
#pragma unroll
            for (int j = 0; j < NL; ++j)
                ip2_cp8(S + j * JS + fk * 16 + (fr ^ fk), (j == ownj) ? isrc + comp_off : dsrc + (size_t)j * ne * n);
            if (!prow) ip2_cp8(S + NLP * JS + fk * 16 + fr, isrc);
            else S[NLP * JS + fk * 16 + fr] = 0;
        } else {
#pragma unroll
            for (int j = 0; j < NL; ++j) S[j * JS + fk * 16 + (fr ^ fk)] = 0;
            S[NLP * JS + fk * 16 + fr] = 0;
        }
#pragma unroll
        for (int j = NL; j < NLP; ++j) S[j * JS + fk * 16 + (fr ^ fk)] = 0;
    };
    // ---- key tile (once, asynchronously, its own commit group ahead of the first D stages): rows n = 2 g + c
    for (int e = tid; e < NLP * IP2_KT * 16; e += IP2_THREADS) {
        const int j = e / (IP2_KT * 16), rem = e % (IP2_KT * 16), kk = rem % IP2_KT, r = rem / IP2_KT;
        const int g = r >> 1, c = r & 1;
        u64* dst = Ks + j * JS + kk * 16 + (r ^ kk);
        if (j < NL && g < G) ip2_cp8(dst, grp.key[g] + ((size_t)j * 2 * np + (size_t)c * np + krow) * n + k0 + kk);
        else *dst = 0;
    }
    ip2_commit();
    // sigma_g store addressing, fixed for the whole launch: the destination block of rotation g (shared by
    // the CTA) and this thread's source index within it (4 bits per g, packed)
    // write phase: word wt of rows wr.  MAC layout (k_mac_tc.cu: per baby step [c][row][x/4][b][x%4]): a warp
    // writes 4 coefficients x 8 ciphertexts = 256 contiguous bytes; else rows of 16 coefficients
    const int wt = mac_layout ? ((tid >> 6) << 2) | (tid & 3) : tid % IP2_KT;
    const int wr = mac_layout ? (tid >> 2) & 15 : tid / IP2_KT;
    u32 spk = 0;
    for (int g = 0; g < G; ++g) {
        const u32 gp = grp.scatter[g];
        int dblk = cblk, sidx = wt;
        if (gp) {
            dblk = galois_src(k0, grp.ginv[g], logn) / IP2_KT;
            sidx = galois_src(dblk * IP2_KT + wt, gp, logn) - k0;
        }
        spk |= (u32)sidx << (4 * g);
        if (tid == 0)
            Ob[g] = mac_layout ? grp.out[g] + ((size_t)i * (n / 4) + (size_t)dblk * (IP2_KT / 4)) * (4 * (size_t)B)
                               : grp.out[g] + (size_t)i * n + (size_t)dblk * IP2_KT;
    }
    // component stride of an output ciphertext (MAC layout: of the baby step's whole batch)
    const size_t wlimb = mac_layout ? (size_t)ne * n * B : (size_t)ne * n;
#pragma unroll
    for (int s = 0; s < IP2_ST - 1; ++s) {
        if (s < nbt) fill(s);
        ip2_commit();
    }
    ip2_wait<IP2_ST - 1>();                                // the key group (the D stages may still fly)
    __syncthreads();
    const double q = (double)Pr.q, qinv = 1.0 / q;
    const double two46 = 70368744177664.0;
    const double w46 = two46 - floor(two46 * qinv) * q, w46q = w46 / q, c23q = 8388608.0 / q;
    const u64 Pm = prow ? 0 : dc->pmod[i], Pm_sh = prow ? 0 : dc->pmod_sh[i];
    const u64 m23 = (1ULL << 23) - 1;
    // 60-bit rows on IMAD: this thread's 2g + c key column of coefficient ik, in registers
    const int ik = tid % IP2_KT, in_ = tid / IP2_KT;
    u64 kreg[(INT && IP2_INT_IMAD) ? NL : 1];
    if constexpr (INT && IP2_INT_IMAD) {
#pragma unroll
        for (int j = 0; j < NL; ++j) kreg[j] = Ks[j * JS + ik * 16 + (in_ ^ ik)];
    }
    // FP class: split key fragments [kq][kb][t] -> (hi, lo, hi + lo), loaded once
    double kf[CACHE ? KPW : 1][CACHE ? NLP / 4 : 1][2][3];
    if constexpr (CACHE) {
#pragma unroll
        for (int kq = 0; kq < KPW; ++kq) {
            const int kk = warp * KPW + kq;
#pragma unroll
            for (int kb = 0; kb < NLP / 4; ++kb)
#pragma unroll
                for (int t = 0; t < 2; ++t) {
                    const u64 bv = Ks[(kb * 4 + tig) * JS + kk * 16 + ((t * 8 + gid) ^ kk)];
                    const double bh = u2d(bv >> 23), bl = u2d(bv & m23);
                    kf[kq][kb][t][0] = bh;
                    kf[kq][kb][t][1] = bl;
                    kf[kq][kb][t][2] = bh + bl;
                }
        }
    }
    for (int bt = 0; bt < nbt; ++bt) {
        ip2_wait<IP2_ST - 2>();
        __syncthreads();
        if (bt + IP2_ST - 1 < nbt) fill(bt + IP2_ST - 1);
        ip2_commit();
        const u64* Ds = Dst + (bt % IP2_ST) * SD;
        const u64* As = Ds + NLP * JS;
        if constexpr (INT && IP2_INT_IMAD) {
            // 60-bit rows on the integer pipe (128-bit products): thread = (coefficient ik, column in = 2g + c),
            // key words stationary in registers, 16 ciphertexts of the tile in turn.  These CTAs share SMs with
            // the tensor-core CTAs of the FP rows, so the two pipes overlap.
            const int g = in_ >> 1, c = in_ & 1;
#pragma unroll 2
            for (int bl = 0; bl < 16; ++bl) {
                Acc128 a;
                a.zero();
#pragma unroll
                for (int j = 0; j < NL; ++j) a.mac(Ds[j * JS + ik * 16 + (bl ^ ik)], kreg[j]);
                u64 u = a.reduce(Pr);
                if (c == 0 && !prow) u = addmod(u, csub(shoup_mul(As[ik * 16 + bl], Pm, Pm_sh, Pr.q), Pr.q), Pr.q);
                if (g < G) Os[((g * 2 + c) * 16 + bl) * IP2_KT + (ik ^ ((bl + 4 * g) & 15))] = u;
            }
        } else if constexpr (!INT && IP2_FP_BATCH) {
            // FP rows: the DMMAs of all KPW coefficients of the warp first (independent accumulator sets, so
            // the tensor latency of one overlaps the conversions of the next), then all epilogues
            double S[KPW][3][2][4];
#pragma unroll
            for (int kq = 0; kq < KPW; ++kq)
#pragma unroll
                for (int s3 = 0; s3 < 3; ++s3)
#pragma unroll
                    for (int t = 0; t < 2; ++t)
#pragma unroll
                        for (int e = 0; e < 4; ++e) S[kq][s3][t][e] = 0.0;
#pragma unroll
            for (int kb = 0; kb < NLP / 4; ++kb) {
                const int j = kb * 4 + tig;
#pragma unroll
                for (int kq = 0; kq < KPW; ++kq) {
                    const int kk = warp * KPW + kq;
                    const u64 a0 = Ds[j * JS + kk * 16 + (gid ^ kk)], a1 = Ds[j * JS + kk * 16 + ((gid + 8) ^ kk)];
                    const double a0h = p2d(a0 >> 23), a0l = p2d(a0 & m23), a1h = p2d(a1 >> 23), a1l = p2d(a1 & m23);
                    const double a0s = p2d((a0 >> 23) + (a0 & m23)), a1s = p2d((a1 >> 23) + (a1 & m23));
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const u64 bv = Ks[j * JS + kk * 16 + ((t * 8 + gid) ^ kk)];
                        dmma16884(S[kq][2][t], a0h, a1h, p2d(bv >> 23));
                        dmma16884(S[kq][0][t], a0l, a1l, p2d(bv & m23));
                        dmma16884(S[kq][1][t], a0s, a1s, p2d((bv >> 23) + (bv & m23)));
                    }
                }
            }
#pragma unroll
            for (int kq = 0; kq < KPW; ++kq) {
                const int kk = warp * KPW + kq;
                // addend P c0 of this thread's two ciphertexts (the same for every rotation g)
                double addd[2];
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    addd[h] = prow ? 0.0 : (double)csub(shoup_mul(As[kk * 16 + gid + 8 * h], Pm, Pm_sh, Pr.q), Pr.q);
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int bl = gid + 8 * (e >> 1), g = 4 * t + tig, c = e & 1;
                        const double add = (c == 0) ? addd[e >> 1] : 0.0;
                        const double s0 = S[kq][0][t][e], s2 = S[kq][2][t][e], mid = S[kq][1][t][e] - s2 - s0;
                        const double k1 = __fma_rn(mid, c23q, CK_RND_MAGIC) - CK_RND_MAGIC;
                        const double t1 = __fma_rn(-k1, q, mid * 8388608.0);
                        const double t2 = fmodmul(s2, w46, w46q, q);
                        double r = freduce(t2 + t1 + (s0 + add), q, qinv);   // [-q/2, q/2]
                        r = r < 0.0 ? r + q : r;                             // canonical: the byte-plane MAC
                        const u64 u = d2u(r);
                        if (g < G) Os[((g * 2 + c) * 16 + bl) * IP2_KT + (kk ^ ((bl + 4 * g) & 15))] = u;
                    }
            }
        } else
#pragma unroll
        for (int kq = 0; kq < KPW; ++kq) {
            const int kk = warp * KPW + kq;
            constexpr int NS = INT ? 6 : 3;
            double S[NS][2][4];
#pragma unroll
            for (int s = 0; s < NS; ++s)
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) S[s][t][e] = 0.0;
#pragma unroll
            for (int kb = 0; kb < NLP / 4; ++kb) {
                const int j = kb * 4 + tig;
                const u64 a0 = Ds[j * JS + kk * 16 + (gid ^ kk)], a1 = Ds[j * JS + kk * 16 + ((gid + 8) ^ kk)];
                if constexpr (!INT) {
                    const double a0h = p2d(a0 >> 23), a0l = p2d(a0 & m23), a1h = p2d(a1 >> 23), a1l = p2d(a1 & m23);
                    const double a0s = p2d((a0 >> 23) + (a0 & m23)), a1s = p2d((a1 >> 23) + (a1 & m23));
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        double bh, bl, bs;
                        if constexpr (CACHE) {
                            bh = kf[kq][kb][t][0];
                            bl = kf[kq][kb][t][1];
                            bs = kf[kq][kb][t][2];
                        } else {
                            const u64 bv = Ks[j * JS + kk * 16 + ((t * 8 + gid) ^ kk)];
                            bh = u2d(bv >> 23);
                            bl = u2d(bv & m23);
                            bs = bh + bl;
                        }
                        dmma16884(S[2][t], a0h, a1h, bh);
                        dmma16884(S[0][t], a0l, a1l, bl);
                        dmma16884(S[1][t], a0s, a1s, bs);
                    }
                } else {
                    const u64 m = (1ULL << 20) - 1;
                    const double x0[3] = {p2d(a0 & m), p2d((a0 >> 20) & m), p2d(a0 >> 40)};
                    const double x1[3] = {p2d(a1 & m), p2d((a1 >> 20) & m), p2d(a1 >> 40)};
#pragma unroll
                    for (int t = 0; t < 2; ++t) {
                        const u64 bv = Ks[j * JS + kk * 16 + ((t * 8 + gid) ^ kk)];
                        const double y[3] = {p2d(bv & m), p2d((bv >> 20) & m), p2d(bv >> 40)};
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
            u64 addw[2];                                   // addend P c0 of the thread's two ciphertexts
#pragma unroll
            for (int h = 0; h < 2; ++h)
                addw[h] = prow ? 0 : csub(shoup_mul(As[kk * 16 + gid + 8 * h], Pm, Pm_sh, Pr.q), Pr.q);
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int bl = gid + 8 * (e >> 1), g = 4 * t + tig, c = e & 1;
                    u64 u;
                    const u64 add = (c == 0) ? addw[e >> 1] : 0;
                    if constexpr (!INT) {
                        // v = s_hh 2^46 + (s_mid - s_hh - s_ll) 2^23 + s_ll mod q on the FP64 pipe, without
                        // pre-reductions: s_hh < 2^48 goes straight into the exact fmodmul by 2^46 mod q;
                        // mid < 2^51: k1 = rint(mid 2^23 / q), mid 2^23 - k1 q is exact in one FMA (the
                        // scaling by 2^23 is exact and the true remainder is < 1.5 q); s_ll < 2^51; the
                        // signed sum (with the addend) stays < 2^52.  Outputs are canonical (the byte-plane
                        // BSGS MAC reads the residue words as unsigned bytes).
                        const double s0 = S[0][t][e], s2 = S[2][t][e], mid = S[1][t][e] - s2 - s0;
                        const double k1 = __fma_rn(mid, c23q, CK_RND_MAGIC) - CK_RND_MAGIC;
                        const double t1 = __fma_rn(-k1, q, mid * 8388608.0);
                        const double t2 = fmodmul(s2, w46, w46q, q);
                        u = fcanon(t2 + t1 + (s0 + (double)add), q, qinv);
                    } else {
                        const double P0 = S[0][t][e], P1 = S[1][t][e], P2 = S[2][t][e];
                        const u64 s0 = d2u(P0), s1 = d2u(S[3][t][e] - P0 - P1), s2 = d2u(S[5][t][e] - P0 - P2 + P1),
                                  s3 = d2u(S[4][t][e] - P1 - P2), s4 = d2u(P2);
                        u64 lo = s0, hi = 0, a2;
                        a2 = s1 << 20; lo += a2; hi += (lo < a2) + (s1 >> 44);
                        a2 = s2 << 40; lo += a2; hi += (lo < a2) + (s2 >> 24);
                        a2 = s3 << 60; lo += a2; hi += (lo < a2) + (s3 >> 4);
                        hi += s4 << 16;
                        u = addmod(reduce128(hi, lo, Pr), add, Pr.q);
                    }
                    if (g < G) Os[((g * 2 + c) * 16 + bl) * IP2_KT + (kk ^ ((bl + 4 * g) & 15))] = u;
                }
        }
        __syncthreads();
        // ---- permuted, coalesced write: row (g, c = h, b = wr) of IP2_KT destination words per 16 lanes
        {
            const int b = bt * 16 + wr;
            if (b < B) {
                const size_t boff = mac_layout ? (size_t)(wt >> 2) * 4 * B + (size_t)b * 4 + (wt & 3)
                                               : (size_t)b * out_stride + wt;
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    if (g < G) {
                        u64* og = Ob[g] + boff;
                        const int sx = ((spk >> (4 * g)) & 15) ^ ((wr + 4 * g) & 15);
#if CK_STREAM_STORES
                        __stcs(og, Os[((g * 2 + 0) * 16 + wr) * IP2_KT + sx]);
                        __stcs(og + wlimb, Os[((g * 2 + 1) * 16 + wr) * IP2_KT + sx]);
#else
                        og[0] = Os[((g * 2 + 0) * 16 + wr) * IP2_KT + sx];
                        og[wlimb] = Os[((g * 2 + 1) * 16 + wr) * IP2_KT + sx];
#endif
                    }
                }
            }
        }
    }
    ip2_wait<0>();
}

// one launch for both prime classes (rows of either class run side by side, so the FP64-heavy and
// the integer-heavy epilogues share the SMs)
template <int NL>
__global__ void __launch_bounds__(IP2_THREADS, 2)
k_ks_ip_mma2(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ in, size_t ct_stride,
             size_t comp_off, const KsGroup grp, int nl, size_t out_stride, int B, int mac_layout)
{
    extern __shared__ u64 sm[];
    // (tried: rows fastest, so CTAs of both classes share an SM at the same time -- 150 vs 147.5 ms per step)
    const int i = blockIdx.y, cblk = blockIdx.x;
    const u64 q = dc->p[ext_prime_of(i, nl, dc->n_data)].q;
    if (prime_class(q) == PC_FP)
        ip2_body<NL, false>(dc, modup, in, ct_stride, comp_off, grp, nl, out_stride, B, sm, i, cblk, mac_layout);
    else ip2_body<NL, true>(dc, modup, in, ct_stride, comp_off, grp, nl, out_stride, B, sm, i, cblk, mac_layout);
}

// host launcher: both prime classes of a baby-step group (scatter outputs, addend P c0, no accumulation)
void ip_mma_pipelined(const Launch& L, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                      size_t out_stride, bool mac_layout)
{
    const int n = 1 << L.log_n, ne = nl + L.n_special, nd = L.active_digits(nl);
    const dim3 grid(n / IP2_KT, ne);
    if (L.probe && L.probe->kind == PROBE_ALL) {
        // exact split products per modular MAC: 3 (FP class rows), 6 (60-bit rows); MACs per row:
        // B x G x 2 components x nd digits x N.  Bytes: ModUp words and input limbs read, c0 addend,
        // the group's keys, the G rotated outputs written.
        double fl = 0;
        for (int i = 0; i < ne; ++i) {
            const int p = ext_prime_of(i, nl, L.n_data);
            fl += 2.0 * ((L.pclass && L.pclass[p] == PC_FP) ? 3 : 6) * batch * grp.G * 2.0 * nd * n;
        }
        L.probe->flops_by_kernel["k_ks_ip_mma"] += fl;
        L.probe->bytes_by_kernel["k_ks_ip_mma"] +=
            ((double)batch * nd * ne + (double)batch * nl + (double)grp.G * nd * 2 * ne + (double)grp.G * batch * 2 * ne) *
            n * 8.0;
    }
    if (ip_mma3(L, in, grp, batch, nl, w, out_stride, mac_layout)) {   // k_ipmma3.cu (default for <= 5 digits)
        check_launch("ip_mma3");
        if (L.counter) *L.counter += 1;
        return;
    }
#define IP2_CASE(V)                                                                                                  \
    case V: {                                                                                                         \
        const size_t smem = Ip2Shape<V>::smem;                                                                        \
        allow_smem(k_ks_ip_mma2<V>, smem);                                                                            \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_mma");                                                                 \
        k_ks_ip_mma2<V><<<grid, IP2_THREADS, smem, L.st>>>(L.dc, w.modup, in.base, in.ct_stride, in.comp_off, grp,   \
                                                         nl, out_stride, batch, mac_layout ? 1 : 0);                  \
    } break;
    switch (nd) {
        IP2_CASE(1) IP2_CASE(2) IP2_CASE(3) IP2_CASE(4) IP2_CASE(5) IP2_CASE(6) IP2_CASE(7) IP2_CASE(8)
        IP2_CASE(9) IP2_CASE(10) IP2_CASE(11) IP2_CASE(12) IP2_CASE(13) IP2_CASE(14) IP2_CASE(15) IP2_CASE(16)
    default: throw std::runtime_error("more than 16 digits");
    }
#undef IP2_CASE
    check_launch("ip_mma_pipelined");
    if (L.counter) *L.counter += 1;
}

}  // namespace ck
