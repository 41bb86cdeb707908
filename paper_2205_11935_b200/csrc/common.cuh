// common.cuh -- device-side types and modular arithmetic for the B200 CKKS path.
//
// Residues are 64-bit words modulo primes q < 2^61 (R1).  Products use the integer pipes:
//   * Shoup multiplication by a precomputed constant w (w' = floor(w 2^64 / q)):
//         shoup(a, w) = a w - floor(a w' / 2^64) q  in [0, 2q)   for any a < 2^64.
//   * 128-bit reduction  x = hi 2^64 + lo  ->  shoup(hi, 2^64 mod q) + shoup(lo, 1)  in [0, 4q).
// Lazy ranges are stated at every use.
#pragma once
#include <cstdint>
#include <vector_types.h>

typedef uint64_t u64;
typedef uint32_t u32;

#define CKKS_MAXP 16
// twiddle words per prime: W, W', IW, IW' (u64), Wd, Wq, IWd, IWq (double), then the pair tables of the cluster
// schedule (ntt_c.cuh): [N] x (w, w/q) forward and inverse (FP64), [N] x (w, w') forward (integer Shoup)
#define CK_TW_WORDS 14

struct DPrime {
    u64 q, q2;
    u64 ninv, ninv_sh;   // N^{-1} mod q and its Shoup companion
    u64 one_sh;          // floor(2^64 / q): Shoup companion of 1
    u64 r64, r64_sh;     // 2^64 mod q and companion
    u64 w20, w23, w40;   // 2^20, 2^23, 2^40 mod q (split-operand recombination, k_ipmma3.cu)
    u64 mu90;            // floor(2^90 / q) for q >= 2^59 (< 2^32: one-word Barrett of values < 2^89), else 0
    double qinv_d;       // fl(1 / q)
    double w23q;         // fl(w23 / q)
};

// Per-context constants, resident in device memory (tables buffer).
struct DCtx {
    int log_n, n, n_data, n_special, n_primes;
    int pad_;
    DPrime p[CKKS_MAXP];
    u64 qmod[CKKS_MAXP][CKKS_MAXP];     // q_a mod q_b
    u64 qinv[CKKS_MAXP][CKKS_MAXP];     // q_a^{-1} mod q_b   (a != b)
    u64 qinv_sh[CKKS_MAXP][CKKS_MAXP];
    u64 qmod_sh[CKKS_MAXP][CKKS_MAXP];  // Shoup constants of qmod
    const u64* tw;                      // [n_primes][CK_TW_WORDS][N]  (bit-reversed psi powers)
    u64 cdt[40];                        // discrete Gaussian CDT thresholds (R13)
    int cdt_bound;
    // key switching (R9b, R10b, R17b): dnum digits of 1 or 2 consecutive data primes; P = the product of
    // the n_special (1 or 2) special primes
    int n_digits;
    int dig_start[CKKS_MAXP], dig_len[CKKS_MAXP];
    u64 dig_inv[CKKS_MAXP], dig_inv_sh[CKKS_MAXP];   // [p]: q_{p-1}^{-1} mod q_p when p is the 2nd prime of
                                                     // a 2-prime group (a digit, or P_1 of P = P_0 P_1)
    u64 pmod[CKKS_MAXP], pmod_sh[CKKS_MAXP];         // P mod q_p (0 for the special primes)
    u64 pinv[CKKS_MAXP], pinv_sh[CKKS_MAXP];         // P^{-1} mod q_i (data primes)
    u64 phalf_lo, phalf_hi;                          // (P - 1) / 2 as a 128-bit integer
    u64 phalf_a, phalf_t;                            // K = 2: (P - 1) / 2 = phalf_a + P_0 phalf_t (mixed radix, as the
                                                     // remainder pairs: comparing (t, a) lexicographically is exact)
    // canonical embedding on the device (k_encode.cu, R3/R4): n = N/2 slots
    const u32* slot_pos;                             // [n] (5^i mod 2N - 1) / 4
    const double2* fft_zeta;                         // [n] zeta^k = e^{i pi k / N}
    const double2* fft_omega;                        // [n/2] omega^p = e^{2 pi i p / n}
};

__device__ __forceinline__ u64 csub(u64 a, u64 m) { return a >= m ? a - m : a; }

__device__ __forceinline__ u64 shoup_mul(u64 a, u64 w, u64 wsh, u64 q)
{
    u64 h = __umul64hi(a, wsh);
    return a * w - h * q;   // [0, 2q)
}

// any 64-bit a -> [0, 2q)
__device__ __forceinline__ u64 reduce64_lazy(u64 a, const DPrime& P)
{
    return a - __umul64hi(a, P.one_sh) * P.q;
}
__device__ __forceinline__ u64 reduce64(u64 a, const DPrime& P) { return csub(reduce64_lazy(a, P), P.q); }

// (hi, lo) 128-bit -> [0, q)
__device__ __forceinline__ u64 reduce128(u64 hi, u64 lo, const DPrime& P)
{
    u64 a = shoup_mul(hi, P.r64, P.r64_sh, P.q);   // [0, 2q)
    u64 b = reduce64_lazy(lo, P);                  // [0, 2q)
    u64 s = a + b;                                 // [0, 4q) < 2^63
    s = csub(s, P.q2);
    return csub(s, P.q);
}

// (hi, lo) < 2^89 -> [0, q) for q in [2^59, 2^61): one-word Barrett.  Th = T >> 58 < 2^31, qe = (Th mu90) >> 32 is
// within 3 of floor(T / q) from below, so T - qe q (mod 2^64) is in [0, 4q)
__device__ __forceinline__ u64 reduce89(u64 hi, u64 lo, const DPrime& P)
{
    const u32 th = (u32)((hi << 6) | (lo >> 58));
    const u32 qe = (u32)(((u64)th * (u32)P.mu90) >> 32);
    const u64 r = lo - (u64)qe * P.q;
    return csub(csub(r, P.q2), P.q);
}

__device__ __forceinline__ u64 mulmod(u64 a, u64 b, const DPrime& P)
{
    return reduce128(__umul64hi(a, b), a * b, P);
}

// 128-bit accumulator
struct Acc128 {
    u64 lo, hi;
    __device__ __forceinline__ void zero() { lo = 0; hi = 0; }
    __device__ __forceinline__ void mac(u64 a, u64 b)
    {
        u64 plo = a * b, phi = __umul64hi(a, b);
        lo += plo;
        hi += phi + (lo < plo ? 1 : 0);
    }
    __device__ __forceinline__ u64 reduce(const DPrime& P) const { return reduce128(hi, lo, P); }
};

// Split accumulator for operands < 2^42 (primes q < 2^42): a = a1 2^21 + a0, b = b1 2^21 + b0 with all
// parts < 2^21, so every partial product is a 32x32->64 IMAD.WIDE.U32 (with accumulate) below 2^42 and
// up to 2^20 terms sum without overflow; value = s11 2^42 + s01 2^21 + s00 (< 2^128 always).
#define SPLIT21_MAXQ (1ULL << 42)
struct Acc3 {
    u64 s00, s01, s11;
    __device__ __forceinline__ void zero() { s00 = s01 = s11 = 0; }
    __device__ __forceinline__ void mac(u32 a1, u32 a0, u64 b)
    {
        const u32 b1 = (u32)(b >> 21), b0 = (u32)b & 0x1FFFFFu;
        s00 += (u64)a0 * b0;
        s01 += (u64)a0 * b1;
        s01 += (u64)a1 * b0;
        s11 += (u64)a1 * b1;
    }
    __device__ __forceinline__ u64 reduce(const DPrime& P) const
    {
        const u64 mlo = s01 << 21, mhi = s01 >> 43;
        const u64 slo = s11 << 42, shi = s11 >> 22;
        const u64 l1 = s00 + mlo;
        const u64 l2 = l1 + slo;
        const u64 hi = mhi + shi + (l1 < s00 ? 1 : 0) + (l2 < l1 ? 1 : 0);
        return reduce128(hi, l2, P);
    }
};

__device__ __forceinline__ u64 addmod(u64 a, u64 b, u64 q) { return csub(a + b, q); }
__device__ __forceinline__ u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }

// centered residue r in [0, m) (m odd) reduced mod prime b: r if r <= (m-1)/2 else r - m  (R10)
__device__ __forceinline__ u64 centered_to(u64 r, u64 m, u64 m_mod_b, const DPrime& B)
{
    if (r <= (m >> 1)) return reduce64(r, B);
    // r - m  ==  r mod b  - (m mod b)
    u64 rb = reduce64(r, B);
    return submod(rb, m_mod_b, B.q);
}

__device__ __forceinline__ u32 brev32(u32 x, int bits) { return __brev(x) >> (32 - bits); }

// ---- 2-prime CRT groups (hybrid key switching, R9b / R10b).  A group {q_s, q_{s+1}} holds an integer
// x in [0, q_s q_{s+1}) as (a, t): a = x mod q_s, t = (x - a) / q_s = (x mod q_{s+1} - a) q_s^{-1} mod q_{s+1}
// (Garner), so x = a + q_s t exactly.
// t from a (< q_s) and b = x mod q_{s+1} (< q_{s+1}); canonical [0, q_{s+1})
__device__ __forceinline__ u64 crt2_t(const DCtx* __restrict__ dc, int s, u64 a, u64 b)
{
    const DPrime& B = dc->p[s + 1];
    const u64 am = reduce64(a, B);
    return csub(shoup_mul(submod(b, am, B.q), dc->dig_inv[s + 1], dc->dig_inv_sh[s + 1], B.q), B.q);
}
// x mod q_pb for x = a + q_s t, in [0, 2 q_pb)
__device__ __forceinline__ u64 crt2_lazy(const DCtx* __restrict__ dc, int s, u64 a, u64 t, const DPrime& B, int pb)
{
    const u64 u = shoup_mul(t, dc->qmod[s][pb], dc->qmod_sh[s][pb], B.q);   // [0, 2q)
    const u64 v = reduce64_lazy(a, B);                                     // [0, 2q)
    return csub(u + v, B.q2);
}
// centred special remainder r (R10 / R10b) reduced mod data prime pb, canonical [0, q_pb):
//   K = 1: r = rem0 in [0, P);  K = 2: r = rem0 + P_0 rem1 in [0, P_0 P_1) (CRT pair); r > (P-1)/2 -> r - P
__device__ __forceinline__ u64 special_centered(const DCtx* __restrict__ dc, u64 rem0, u64 rem1, const DPrime& B, int pb)
{
    const int L = dc->n_data;
    if (dc->n_special == 1) return centered_to(rem0, dc->p[L].q, dc->pmod[pb], B);
    const u64 P0 = dc->p[L].q;
    const u64 lo0 = P0 * rem1, hi0 = __umul64hi(P0, rem1);
    const u64 lo = lo0 + rem0, hi = hi0 + (lo < lo0 ? 1 : 0);
    const bool neg = hi > dc->phalf_hi || (hi == dc->phalf_hi && lo > dc->phalf_lo);
    const u64 v = csub(crt2_lazy(dc, L, rem0, rem1, B, pb), B.q);
    return neg ? submod(v, dc->pmod[pb], B.q) : v;
}
// prime index of row e of a Q_l P polynomial with nl data rows: q_e, then the special primes
__host__ __device__ __forceinline__ int ext_prime_of(int e, int nl, int L) { return e < nl ? e : L + (e - nl); }
