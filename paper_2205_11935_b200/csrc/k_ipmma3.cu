// k_ipmma3.cu -- sm_100a kernel of the CKKS encrypted-dense-layer hot path: the hoisted baby-step
// key-switch inner product in the Q_l P basis (double hoisting, R11c) on the FP64 tensor
// cores, with the key pre-multiplied so that every output needs ONE modular fold (the r02 form of
// k_ipmma.cu, which used Karatsuba split products and a three-term recombination).
//
// The operation (SV §8(a) a4, PAPER.md L92-96 baby steps of Eq. 1):  for one row i (prime q) and one
// coefficient k,
//     U[b][(g, c)] = sum_{j < nd} D_{b,j}[k] key_{g,j,c}[k]  mod q     (+ P c0_b[k] for c = 0)
// and the result is written through sigma_g (aligned 16-blocks of NTT indices map onto aligned blocks).
//
// Exact split, FP rows (q < 2^45): D = Dh 2^23 + Dl, and with K' = K 2^23 mod q (computed once per key
// word in the prologue)
//     D K == Dh K' + Dl K == [Dh K'l + Dl Kl] + 2^23 [Dh K'h + Dl Kh]        (mod q)
// so the MMA contracts over the K index (j, part) of length 2 nd with TWO accumulators S0, S1
// (products < 2^46, nd <= 16: S0 < 2^50.6, S1 < 2^49.6, exact in FP64), and the epilogue is one exact
// fmodmul (2^23 S1 mod q), one add and one reduction.  60-bit rows (q >= 2^45): D = sum_u D_u 2^{20u},
// K^(u) = K 2^{20u} mod q, D K == sum_u D_u K^(u) = S0 + 2^20 S1 + 2^40 S2 with the K index (j, u) of
// length 3 nd (parts < 2^21, sums < 2^48), recombined in 128 bits and reduced once.
//
// Layouts:
//   ModUp output  [b][digit j][row 0..nl+K-1][N]   (rows nl..: the special primes P_0..P_{K-1})
//   key           [digit j][comp][prime 0..L+K-1][N]  (pre-permuted by sigma_g^{-1})
//   baby output   [b][comp][row 0..nl+K-1][N]   (Q_l P basis, sigma_g-permuted)
//   smem D tile   [stage][j | c0][b 16][k 16 ^ 2 (b & 7)]   (16-byte cp.async chunks, XOR-swizzled)
#include "kinternal.cuh"

namespace ck {

#define IP3_KT 16
#define IP3_THREADS 256
#define IP3_ST 3

__device__ __forceinline__ void ip3_cp16(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void ip3_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void ip3_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

template <int NL>
struct Ip3Shape {                                           // NL = active digits (the contraction length)
    static constexpr int KF = 2 * NL;                       // FP rows: K index (j, part)
    static constexpr int KI = 3 * NL;                       // 60-bit rows: K index (j, u)
    static constexpr int JS = 16 * IP3_KT;                  // words per (j) slice of a stage
    static constexpr int SD = (NL + 1) * JS;                // words per stage: D tile + c0 addend
    static constexpr int KEYW_FP = IP3_KT * KF * 16 * 2;    // double2 (S0 part, S1 part) per (k, kidx, n)
    static constexpr int KEYW_INT = IP3_KT * KI * 16;       // K^(u) words per (k, kidx, n)
    static constexpr int KEYW = KEYW_FP > KEYW_INT ? KEYW_FP : KEYW_INT;
    static constexpr int OSW = 8 * 2 * 16 * IP3_KT;         // [8 g][2 c][16 b][KT] staging of the permuted writes
    static constexpr size_t smem = sizeof(u64) * ((size_t)KEYW + (size_t)IP3_ST * SD + OSW + 8);
};

// word position of (b, k) in a [16 b][16 k] slice: 16-byte chunks (k, k^1) XOR-swizzled by b
__device__ __forceinline__ int ip3_pos(int b, int k) { return b * 16 + (k ^ ((b & 7) << 1)); }
// double2 position of (k index kidx, column n) in coefficient kk's block of the FP key tile: blocks of 4 K
// indices [kb][n 16][kidx % 4] (the last block only KF - 4 kb wide), so the 8 lanes (gid, tig) of a quarter
// warp read 8 consecutive 16-byte units (conflict-free LDS.128)
template <int KF>
__device__ __forceinline__ int ip3_kpos(int kk, int kidx, int n)
{
    const int kb = kidx >> 2, w = (KF - 4 * kb) < 4 ? (KF - 4 * kb) : 4;
    return kk * KF * 16 + kb * 64 + n * w + (kidx & 3);
}
// column of B value (k index kidx, n) in the 60-bit key tile (two 8-word halves alternate with kidx)
__device__ __forceinline__ int ip3_icol(int n, int kidx) { return (n + ((kidx & 1) << 3)) & 15; }

// y * w mod q when the product y w is exact in FP64 (w = 2^23 for q > 2^23: a power of two): no low part
__device__ __forceinline__ double fmodmul_pow2(double y, double w, double wq, double q)
{
    const double k = __fma_rn(y, wq, CK_RND_MAGIC) - CK_RND_MAGIC;
    return __fma_rn(-k, q, y * w);
}

// BIGQ: q > 2^23, so 2^23 mod q = 2^23 and the fold of S1 is fmodmul_pow2 (4 FP64 operations instead of 6)
template <int NL, bool INT, bool MACL, bool BIGQ = false>
__device__ __forceinline__ void ip3_body(const DCtx* __restrict__ dc, const u64* __restrict__ modup,
                                         const u64* __restrict__ in, size_t ct_stride, size_t comp_off,
                                         const KsGroup& grp, int nl, size_t out_stride, int B, u64* sm, int i,
                                         int cblk)
{
    constexpr int mac_layout = MACL ? 1 : 0;
    using S = Ip3Shape<NL>;
    constexpr int JS = S::JS, SD = S::SD;
    constexpr int KPW = IP3_KT / (IP3_THREADS / 32);        // coefficients per warp
    constexpr int KX = INT ? S::KI : S::KF;                 // contraction length
    constexpr int NKB = (KX + 3) / 4;                       // MMA k-steps
    // FP rows with two spare K slots (nd = 1, 3, 5): the addend P c0 rides in them as one more "digit" -- A = the
    // staged c0 slice (what the dead lanes read anyway), B = (P mod q) pre-multiplied like a key word, columns
    // c = 0 only -- instead of a Shoup product per (ciphertext, coefficient) in the epilogue
    constexpr bool ADDK = !INT && (4 * NKB - KX) >= 2;
    u64* Kw = sm;                                           // key tile (FP: double2 [k][kidx][n]; INT: u64)
    u64* Dst = Kw + S::KEYW;
    u64* Os = Dst + IP3_ST * SD;
    u64** Ob = reinterpret_cast<u64**>(Os + S::OSW);
    const int n = dc->n, logn = dc->log_n, K = dc->n_special, ne = nl + K, np = dc->n_data + K;
    const int k0 = cblk * IP3_KT;
    const bool prow = (i >= nl);                            // a special-prime row
    const int p = ext_prime_of(i, nl, dc->n_data);
    const DPrime Pr = dc->p[p];
    int ownj = -1;                                          // the digit whose primes include q_i (D = input limb)
    for (int j = 0; j < NL; ++j)
        if (!prow && i >= dc->dig_start[j] && i < dc->dig_start[j] + dc->dig_len[j]) ownj = j;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int G = grp.G;
    const int nbt = (B + 15) / 16;
    // ---- stage fill: 16-byte chunks; chunk e = (slice jj = D digit or c0, ciphertext row br, chunk ch)
    auto fill = [&](int bt) {
        u64* Sg = Dst + (bt % IP3_ST) * SD;
        for (int e = tid; e < (NL + 1) * 16 * 8; e += IP3_THREADS) {
            const int ch = e & 7, br = (e >> 3) & 15, jj = e >> 7;
            const int b = bt * 16 + br;
            u64* dst = Sg + jj * JS + ip3_pos(br, 2 * ch);
            if (b < B && !(jj == NL && prow)) {
                const u64* isrc = in + (size_t)b * ct_stride + (size_t)i * n + k0 + 2 * ch;
                const u64* src = (jj == NL) ? isrc
                               : (jj == ownj) ? isrc + comp_off
                                              : modup + (((size_t)b * NL + jj) * ne + i) * n + k0 + 2 * ch;
                ip3_cp16(dst, src);
            } else {
                dst[0] = 0;
                dst[1] = 0;
            }
        }
    };
#pragma unroll
    for (int s = 0; s < IP3_ST - 1; ++s) {
        if (s < nbt) fill(s);
        ip3_commit();
    }
    // ---- key tile (once per launch; overlaps the first fills): the pre-multiplied split of section 1
    const u64 m23 = (1ULL << 23) - 1, m20 = (1ULL << 20) - 1;
    for (int e = tid; e < IP3_KT * NL * 16; e += IP3_THREADS) {
        const int kk = e % IP3_KT, r = (e / IP3_KT) & 15, j = e / (IP3_KT * 16);
        const int g = r >> 1, c = r & 1;
        const u64 kv = (g < G) ? __ldg(grp.key[g] + ((size_t)j * 2 * np + (size_t)c * np + p) * n + k0 + kk) : 0;
        if constexpr (!INT) {
            const u64 kp = mulmod(kv, Pr.w23, Pr);                              // K' = K 2^23 mod q
            double2* d = reinterpret_cast<double2*>(Kw);
            d[ip3_kpos<S::KF>(kk, 2 * j, r)] = make_double2((double)(kp & m23), (double)(kp >> 23));     // Dh: K'l, K'h
            d[ip3_kpos<S::KF>(kk, 2 * j + 1, r)] = make_double2((double)(kv & m23), (double)(kv >> 23)); // Dl: Kl, Kh
        } else {
            const u64 ku[3] = {kv, mulmod(kv, Pr.w20, Pr), mulmod(kv, Pr.w40, Pr)};
#pragma unroll
            for (int u = 0; u < 3; ++u) {
                const int kidx = 3 * j + u;
                Kw[(kk * S::KI + kidx) * 16 + ip3_icol(r, kidx)] = ku[u];
            }
        }
    }
    // sigma_g store addressing, fixed for the whole launch: the destination block of rotation g (shared by
    // the CTA) and this thread's source index within it (4 bits per g, packed)
    // write phase: word wt of rows wr.  MAC layout (k_mac_tc.cu: per baby step [c][row][x/4][b][x%4]): a warp
    // writes 4 coefficients x 8 ciphertexts = 256 contiguous bytes; else rows of 16 coefficients
    const int wt = mac_layout ? ((tid >> 6) << 2) | (tid & 3) : tid % IP3_KT;
    const int wr = mac_layout ? (tid >> 2) & 15 : tid / IP3_KT;
    u32 spk = 0;
    for (int g = 0; g < G; ++g) {
        const u32 gp = grp.scatter[g];
        int dblk = cblk, sidx = wt;
        if (gp) {
            dblk = galois_src(k0, grp.ginv[g], logn) / IP3_KT;
            sidx = galois_src(dblk * IP3_KT + wt, gp, logn) - k0;
        }
        spk |= (u32)sidx << (4 * g);
        if (tid == 0)
            Ob[g] = mac_layout ? grp.out[g] + ((size_t)i * (n / 4) + (size_t)dblk * (IP3_KT / 4)) * (4 * (size_t)B)
                               : grp.out[g] + (size_t)i * n + (size_t)dblk * IP3_KT;
    }
    const size_t wlimb = mac_layout ? (size_t)ne * n * B : (size_t)ne * n;
    const double q = (double)Pr.q, qinv = Pr.qinv_d;      // host-computed: no 64-bit division per CTA
    const double w23 = (double)Pr.w23, w23q = Pr.w23q;
    const u64 Pm = prow ? 0 : dc->pmod[i], Pm_sh = prow ? 0 : dc->pmod_sh[i];
    // this lane's K index per k-step: FP (j, part) = (kidx >> 1, kidx & 1); INT (j, u) = (kidx / 3, kidx % 3)
    int kj[NKB], ksh[NKB];
#pragma unroll
    for (int kb = 0; kb < NKB; ++kb) {
        const int kidx = 4 * kb + tig;
        kj[kb] = (kidx < KX) ? (INT ? kidx / 3 : kidx >> 1) : -1;
        ksh[kb] = INT ? 20 * (kidx % 3) : ((kidx & 1) ? 0 : 23);
    }
    const double2* Kd = reinterpret_cast<const double2*>(Kw);
    // ADDK: the B values of this lane's spare K slot (last k-step, K index KX + part) for columns gid and 8 + gid
    double2 addb0 = make_double2(0.0, 0.0), addb1 = make_double2(0.0, 0.0);
    if constexpr (ADDK) {
        const int part = 4 * (NKB - 1) + tig - KX;             // 0: pairs with the high part of c0, 1: with the low part
        if (part >= 0 && part < 2 && !prow) {
            const u64 pm = dc->pmod[i], w = part == 0 ? mulmod(pm, Pr.w23, Pr) : pm;
            const double2 val = make_double2((double)(w & m23), (double)(w >> 23));
            if ((gid & 1) == 0 && (gid >> 1) < G) addb0 = val;             // column n = (g, c) = (n >> 1, n & 1)
            if ((gid & 1) == 0 && ((8 + gid) >> 1) < G) addb1 = val;
        }
    }
    for (int bt = 0; bt < nbt; ++bt) {
        ip3_wait<IP3_ST - 2>();
        __syncthreads();                                   // stage bt landed (and the key tile, at bt = 0)
        if (bt + IP3_ST - 1 < nbt) fill(bt + IP3_ST - 1);
        ip3_commit();
        const u64* Ds = Dst + (bt % IP3_ST) * SD;
        const u64* As = Ds + NL * JS;
        if constexpr (!INT) {
            // FP rows: the DMMAs of both coefficients of the warp first (independent accumulator sets), then
            // the epilogues
            double Sa[KPW][2][2][4];
#pragma unroll
            for (int kq = 0; kq < KPW; ++kq)
#pragma unroll
                for (int v = 0; v < 2; ++v)
#pragma unroll
                    for (int t = 0; t < 2; ++t)
#pragma unroll
                        for (int e = 0; e < 4; ++e) Sa[kq][v][t][e] = 0.0;
#pragma unroll
            for (int kb = 0; kb < NKB; ++kb) {
                const int sh = ksh[kb];
                const bool live = kj[kb] >= 0;
                const int j = live ? kj[kb] : NL;          // dead lanes read the c0 slice, times a zero B value
                const u64 mk = sh ? ~0ULL : m23;
#pragma unroll
                for (int kq = 0; kq < KPW; ++kq) {
                    const int kk = warp * KPW + kq;
                    const u64 a0 = Ds[j * JS + ip3_pos(gid, kk)];
                    const u64 a1 = Ds[j * JS + ip3_pos(gid + 8, kk)];
                    const int kidx = 4 * kb + tig;          // dead lanes' positions stay inside shared memory
                    const double2 v0 = Kd[ip3_kpos<S::KF>(kk, kidx, gid)], v1 = Kd[ip3_kpos<S::KF>(kk, kidx, 8 + gid)];
                    const double2 b0 = live ? v0 : ((ADDK && kb == NKB - 1) ? addb0 : make_double2(0.0, 0.0)),
                                  b1 = live ? v1 : ((ADDK && kb == NKB - 1) ? addb1 : make_double2(0.0, 0.0));
                    const double x0 = p2d((a0 >> sh) & mk), x1 = p2d((a1 >> sh) & mk);
                    dmma16884(Sa[kq][0][0], x0, x1, b0.x);
                    dmma16884(Sa[kq][1][0], x0, x1, b0.y);
                    dmma16884(Sa[kq][0][1], x0, x1, b1.x);
                    dmma16884(Sa[kq][1][1], x0, x1, b1.y);
                }
            }
#pragma unroll
            for (int kq = 0; kq < KPW; ++kq) {
                const int kk = warp * KPW + kq;
                double addd[2];                            // P c0 of this thread's two ciphertexts (ADDK: in S0, S1)
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    addd[h] = (ADDK || prow) ? 0.0
                                             : (double)csub(shoup_mul(As[ip3_pos(gid + 8 * h, kk)], Pm, Pm_sh, Pr.q), Pr.q);
                // output (b = gid + 8 h, column 8 t + 2 tig + c) -> Os[(g = 4 t + tig, c)][b][kk ^ ((b + 4 g) & 15)]:
                // two base addresses per thread (h), the (t, c) offsets are immediates
                u64* ob[2];
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    ob[h] = Os + (2 * tig * 16 + gid + 8 * h) * IP3_KT + (kk ^ ((gid + 8 * h + 4 * tig) & 15));
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int c = e & 1;
                        // U = S0 + 2^23 S1 (+ P c0) mod q: |fmodmul| < 0.51 q, S0 < 2^50.6 -> |v| < 2^51
                        const double hi = BIGQ ? fmodmul_pow2(Sa[kq][1][t][e], w23, w23q, q)
                                               : fmodmul(Sa[kq][1][t][e], w23, w23q, q);
                        const double v = hi + (Sa[kq][0][t][e] + ((c == 0) ? addd[e >> 1] : 0.0));
                        const double r = freduce(v, q, qinv);                    // [-q/2, q/2]
                        // the DMMA BSGS MAC reads signed words (arithmetic-shift split); the byte-plane
                        // tensor-core MAC needs canonical ones.  Rows g >= G are staged but never written out.
                        const u64 u = MACL ? d2u(r < 0.0 ? r + q : r) : d2s(r);
                        ob[e >> 1][(8 * t + c) * 16 * IP3_KT] = u;
                    }
            }
        } else {
#pragma unroll 1
            for (int kq = 0; kq < KPW; ++kq) {
                const int kk = warp * KPW + kq;
                double Sa[3][2][4];
#pragma unroll
                for (int v = 0; v < 3; ++v)
#pragma unroll
                    for (int t = 0; t < 2; ++t)
#pragma unroll
                        for (int e = 0; e < 4; ++e) Sa[v][t][e] = 0.0;
#pragma unroll
                for (int kb = 0; kb < NKB; ++kb) {
                    const int j = kj[kb], sh = ksh[kb];
                    const int kidx = 4 * kb + tig;
                    u64 a0 = 0, a1 = 0, w0 = 0, w1 = 0;
                    if (j >= 0) {
                        a0 = Ds[j * JS + ip3_pos(gid, kk)];
                        a1 = Ds[j * JS + ip3_pos(gid + 8, kk)];
                        w0 = Kw[(kk * S::KI + kidx) * 16 + ip3_icol(gid, kidx)];
                        w1 = Kw[(kk * S::KI + kidx) * 16 + ip3_icol(8 + gid, kidx)];
                    }
                    const u64 msk = (sh == 40) ? ~0ULL : m20;
                    const double x0 = p2d((a0 >> sh) & msk), x1 = p2d((a1 >> sh) & msk);
                    dmma16884(Sa[0][0], x0, x1, p2d(w0 & m20));
                    dmma16884(Sa[1][0], x0, x1, p2d((w0 >> 20) & m20));
                    dmma16884(Sa[2][0], x0, x1, p2d(w0 >> 40));
                    dmma16884(Sa[0][1], x0, x1, p2d(w1 & m20));
                    dmma16884(Sa[1][1], x0, x1, p2d((w1 >> 20) & m20));
                    dmma16884(Sa[2][1], x0, x1, p2d(w1 >> 40));
                }
                u64 addw[2];
#pragma unroll
                for (int h = 0; h < 2; ++h)
                    addw[h] = prow ? 0 : csub(shoup_mul(As[ip3_pos(gid + 8 * h, kk)], Pm, Pm_sh, Pr.q), Pr.q);
#pragma unroll
                for (int t = 0; t < 2; ++t)
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        const int bl = gid + 8 * (e >> 1), g = 4 * t + tig, c = e & 1;
                        // S0 + 2^20 S1 + 2^40 S2 (each < 2^48) as a 128-bit integer, reduced once
                        const u64 s0 = d2u(Sa[0][t][e]), s1 = d2u(Sa[1][t][e]), s2 = d2u(Sa[2][t][e]);
                        const u64 a1v = s1 << 20, a2v = s2 << 40;
                        u64 lo = s0 + a1v, hi = (s1 >> 44) + (s2 >> 24) + (lo < a1v ? 1 : 0);
                        lo += a2v;
                        hi += (lo < a2v ? 1 : 0);
                        const u64 red = Pr.mu90 ? reduce89(hi, lo, Pr) : reduce128(hi, lo, Pr);   // uniform per CTA
                        const u64 u = addmod(red, (c == 0) ? addw[e >> 1] : 0, Pr.q);
                        Os[((g * 2 + c) * 16 + bl) * IP3_KT + (kk ^ ((bl + 4 * g) & 15))] = u;
                    }
            }
        }
        __syncthreads();
        // ---- permuted, coalesced write: row (g, c = h, b = wr) of IP3_KT destination words per 16 lanes
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
                        og[0] = Os[((g * 2 + 0) * 16 + wr) * IP3_KT + sx];
                        og[wlimb] = Os[((g * 2 + 1) * 16 + wr) * IP3_KT + sx];
                    }
                }
            }
        }
    }
    ip3_wait<0>();
}

template <int NL>
__global__ void __launch_bounds__(IP3_THREADS, 2)
k_ks_ip_mma3(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ in, size_t ct_stride,
             size_t comp_off, const KsGroup grp, int nl, size_t out_stride, int B, int mac_layout)
{
    extern __shared__ __align__(16) u64 sm3[];
    const int i = blockIdx.y, cblk = blockIdx.x;
    const u64 q = dc->p[ext_prime_of(i, nl, dc->n_data)].q;
    const bool fp = prime_class(q) == PC_FP;
    const bool bigq = q > (1ULL << 23);
    if (mac_layout) {
        if (fp) ip3_body<NL, false, true>(dc, modup, in, ct_stride, comp_off, grp, nl, out_stride, B, sm3, i, cblk);
        else ip3_body<NL, true, true>(dc, modup, in, ct_stride, comp_off, grp, nl, out_stride, B, sm3, i, cblk);
    } else {
        if (fp && bigq) ip3_body<NL, false, false, true>(dc, modup, in, ct_stride, comp_off, grp, nl, out_stride, B, sm3, i, cblk);
        else if (fp) ip3_body<NL, false, false>(dc, modup, in, ct_stride, comp_off, grp, nl, out_stride, B, sm3, i, cblk);
        else ip3_body<NL, true, false>(dc, modup, in, ct_stride, comp_off, grp, nl, out_stride, B, sm3, i, cblk);
    }
}

// process-wide selection (ckks_set_option("ip_v3", ..)): 1 = this kernel for up to IP3_MAXD digits (default),
// 0 = the r01/r02 Karatsuba kernel k_ks_ip_mma2 (k_ipmma.cu) -- same bits either way
#define IP3_MAXD 5
static int g_ip_v3 = [] {
    const char* e = getenv("CKKS_IP_V3");
    return e ? atoi(e) : 1;
}();
void set_ip_v3(int on) { g_ip_v3 = on; }
int get_ip_v3() { return g_ip_v3; }

bool ip_mma3(const Launch& L, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
             size_t out_stride, bool mac_layout)
{
    const int n = 1 << L.log_n, nd = L.active_digits(nl);
    if (!g_ip_v3 || nd > IP3_MAXD || n % IP3_KT) return false;
    const dim3 grid(n / IP3_KT, nl + L.n_special);
#define IP3_CASE(V)                                                                                                  \
    case V: {                                                                                                         \
        const size_t smem = Ip3Shape<V>::smem;                                                                        \
        allow_smem(k_ks_ip_mma3<V>, smem);                                                                            \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_mma");                                                                 \
        k_ks_ip_mma3<V><<<grid, IP3_THREADS, smem, L.st>>>(L.dc, w.modup, in.base, in.ct_stride, in.comp_off, grp,   \
                                                         nl, out_stride, batch, mac_layout ? 1 : 0);                  \
    } break;
    switch (nd) {
        IP3_CASE(1) IP3_CASE(2) IP3_CASE(3) IP3_CASE(4) IP3_CASE(5)
    default: return false;
    }
#undef IP3_CASE
    return true;
}

}  // namespace ck
