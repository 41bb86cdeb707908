// k_mac.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path.
//
// Every operation of SURVEY 8(a) rows a2-a12 is one of these kernels; the host side (api.cu)
// only sequences launches and tracks level/scale.  Modular arithmetic runs on the integer pipes
// (64-bit Shoup/Barrett), on the FP64 pipe (exact error-free products for q < 2^45), and -- for the
// two small modular contractions (key-switch inner product, BSGS inner sums) -- on the FP64 tensor
// cores with exactly split operands.  Layouts:
//   ciphertext  [batch][comp][limb][N]  u64, NTT domain, canonical residues in [0, q)
//   key         [digit j][comp][prime 0..L+K-1][N]  (primes L.. = the special primes P_k)
//   plaintexts  [t][limb][N]
// This unit: BSGS plaintext-ciphertext MAC (Eq. 1 inner sums).
#include "kinternal.cuh"

namespace ck {

// BSGS inner sums (Eq. 1 inner parenthesis), weights-stationary:
//   w_k[b] = sum_{j<t1} pt_{k t1 + j} o v_j[b],   v_0 = input ct, v_j = rot_j(input).
// Thread (coefficient x, giant index k) keeps its t1 plaintext words in registers and loops over the
// batch, so every plaintext word is read once per launch; v words are shared through L1 by the t2
// threads of the same coefficient.
// FP-class limbs (q < 2^45): split-operand FP64 MAC.  Plaintext words a and ciphertext words y are
// split at 2^23 (a = a1 2^23 + a0, y = y1 2^23 + y0, all parts < 2^23), so every partial product
// is < 2^46 and the three sums  A = sum a1 y1,  B = sum (a1 y0 + a0 y1),  C = sum a0 y0  over t1 <= 32
// terms stay below 2^51: exact in FP64 with one DFMA per partial product (4 per MAC, no per-term
// reduction, accumulator-only dependency chains).  w_k = A 2^46 + B 2^23 + C  mod q at the end.
// CTA = 8 coefficients x 32 ciphertext lanes; the split plaintext tile [t][8] (double2) is staged once.
#define MACF_XT 8
#define MACF_BL 32
#define MACF_KH 8
__global__ void __launch_bounds__(MACF_XT * MACF_BL, 2)
k_bsgs_mac_fp(const DCtx* __restrict__ dc, const u64* __restrict__ pts, int pt_nl, const u64* __restrict__ v0,
              size_t v0_stride, const u64* __restrict__ vb, u64* __restrict__ wout, int t1, int t2, int batch, int nl,
              int qp)
{
    extern __shared__ double2 A2[];
    const int n = dc->n;
    const int l = blockIdx.y;                      // limb; QP: limbs nl.. are the special primes
    const int nlx = nl + (qp ? dc->n_special : 0);
    const int pidx = ext_prime_of(l, nl, dc->n_data);
    const DPrime Pr = dc->p[pidx];
    if (prime_class(Pr.q) != PC_FP) return;
    const int tx = threadIdx.x % MACF_XT, ty = threadIdx.x / MACF_XT;
    const int x0 = blockIdx.x * MACF_XT, x = x0 + tx;
    const int t = t1 * t2;
    const u64 mask23 = (1ULL << 23) - 1;
    for (int i = threadIdx.x; i < t * MACF_XT; i += blockDim.x) {
        const u64 a = pts[((size_t)(i / MACF_XT) * pt_nl + l) * n + x0 + (i % MACF_XT)];
        A2[i] = make_double2(u2d(a >> 23), u2d(a & mask23));
    }
    __syncthreads();
    const double q = (double)Pr.q, qinv = 1.0 / q;
    const double two23 = 8388608.0, two46 = 70368744177664.0;
    const double w46 = two46 - floor(two46 * qinv) * q;                        // 2^46 mod q (exact)
    const double w46q = w46 / q, w23q = two23 / q;
    const size_t ctw = (size_t)2 * nlx * n;
    const u64 Pm = qp ? dc->pmod[l < nl ? l : 0] : 0, Pm_sh = qp ? dc->pmod_sh[l < nl ? l : 0] : 0;
    for (int b = ty; b < batch; b += MACF_BL) {
        for (int c = 0; c < 2; ++c) {
            const size_t off = ((size_t)c * nlx + l) * n + x;
            const size_t off0 = ((size_t)c * nl + l) * n + x;
            for (int k0 = 0; k0 < t2; k0 += MACF_KH) {
                double sA[MACF_KH], sB[MACF_KH], sC[MACF_KH];
#pragma unroll
                for (int z = 0; z < MACF_KH; ++z) sA[z] = sB[z] = sC[z] = 0.0;
                for (int j0 = 0; j0 < t1; j0 += 8) {
                    double y1[8], y0[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + u;
                        u64 y = 0;
                        if (j == 0) {
                            if (!qp) y = v0[(size_t)b * v0_stride + off0];
                            else if (l < nl) y = csub(shoup_mul(v0[(size_t)b * v0_stride + off0], Pm, Pm_sh, Pr.q), Pr.q);
                        } else if (j < t1) {
                            y = vb[((size_t)(j - 1) * batch + b) * ctw + off];
                        }
                        y1[u] = s2d((u64)((long long)y >> 23));   // signed or canonical words
                        y0[u] = u2d(y & mask23);
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + u;
                        if (j < t1) {
#pragma unroll
                            for (int z = 0; z < MACF_KH; ++z) {
                                if (k0 + z < t2) {
                                    const double2 a = A2[((k0 + z) * t1 + j) * MACF_XT + tx];
                                    sA[z] = __fma_rn(a.x, y1[u], sA[z]);
                                    sB[z] = __fma_rn(a.x, y0[u], sB[z]);
                                    sB[z] = __fma_rn(a.y, y1[u], sB[z]);
                                    sC[z] = __fma_rn(a.y, y0[u], sC[z]);
                                }
                            }
                        }
                    }
                }
#pragma unroll
                for (int z = 0; z < MACF_KH; ++z) {
                    if (k0 + z < t2) {
                        const double r = fmodmul(freduce(sA[z], q, qinv), w46, w46q, q) +
                                         fmodmul(freduce(sB[z], q, qinv), two23, w23q, q) + freduce(sC[z], q, qinv);
                        wout[((size_t)(k0 + z) * batch + b) * ctw + off] = fcanon(r, q, qinv);
                    }
                }
            }
        }
    }
}

// BIG-class limbs (60-bit primes): same tiling as k_bsgs_mac_fp with 128-bit integer accumulators.
__global__ void __launch_bounds__(MACF_XT * MACF_BL, 2)
k_bsgs_mac_int(const DCtx* __restrict__ dc, const u64* __restrict__ pts, int pt_nl, const u64* __restrict__ v0,
               size_t v0_stride, const u64* __restrict__ vb, u64* __restrict__ wout, int t1, int t2, int batch, int nl,
               int qp)
{
    extern __shared__ u64 Ai[];
    const int n = dc->n;
    const int l = blockIdx.y;
    const int nlx = nl + (qp ? dc->n_special : 0);
    const int pidx = ext_prime_of(l, nl, dc->n_data);
    const DPrime Pr = dc->p[pidx];
    if (prime_class(Pr.q) == PC_FP) return;
    const int tx = threadIdx.x % MACF_XT, ty = threadIdx.x / MACF_XT;
    const int x0 = blockIdx.x * MACF_XT, x = x0 + tx;
    const int t = t1 * t2;
    for (int i = threadIdx.x; i < t * MACF_XT; i += blockDim.x)
        Ai[i] = pts[((size_t)(i / MACF_XT) * pt_nl + l) * n + x0 + (i % MACF_XT)];
    __syncthreads();
    const size_t ctw = (size_t)2 * nlx * n;
    const u64 Pm = qp ? dc->pmod[l < nl ? l : 0] : 0, Pm_sh = qp ? dc->pmod_sh[l < nl ? l : 0] : 0;
    for (int b = ty; b < batch; b += MACF_BL) {
        for (int c = 0; c < 2; ++c) {
            const size_t off = ((size_t)c * nlx + l) * n + x;
            const size_t off0 = ((size_t)c * nl + l) * n + x;
            for (int k0 = 0; k0 < t2; k0 += MACF_KH) {
                Acc128 s[MACF_KH];
#pragma unroll
                for (int z = 0; z < MACF_KH; ++z) s[z].zero();
                for (int j0 = 0; j0 < t1; j0 += 8) {
                    u64 y[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        const int j = j0 + u;
                        y[u] = 0;
                        if (j == 0) {
                            if (!qp) y[u] = v0[(size_t)b * v0_stride + off0];
                            else if (l < nl) y[u] = csub(shoup_mul(v0[(size_t)b * v0_stride + off0], Pm, Pm_sh, Pr.q), Pr.q);
                        } else if (j < t1) {
                            y[u] = vb[((size_t)(j - 1) * batch + b) * ctw + off];
                        }
                    }
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (j0 + u < t1) {
#pragma unroll
                            for (int z = 0; z < MACF_KH; ++z)
                                if (k0 + z < t2) s[z].mac(Ai[((k0 + z) * t1 + j0 + u) * MACF_XT + tx], y[u]);
                        }
                    }
                }
#pragma unroll
                for (int z = 0; z < MACF_KH; ++z)
                    if (k0 + z < t2) wout[((size_t)(k0 + z) * batch + b) * ctw + off] = s[z].reduce(Pr);
            }
        }
    }
}

// BSGS inner sums on the FP64 tensor cores (DMMA).  For one limb, one component c and one
// coefficient x the inner sums are a small matrix product over the baby-step index j:
//     W[b][k] = sum_{j<t1} V_j[b] pt_{k t1 + j}        (rows b = ciphertexts, columns k = giant index)
// computed EXACTLY with mma.sync m16n8k4 f64 on split operands (as k_ks_ip_mma).  FP class (q < 2^45):
// two parts at 2^23 and Karatsuba (3 products); every product of part sums is < 2^47.2 (< 2^46.1 for
// q < 2^41), and the accumulators are folded mod q every 32 (64) terms, so every sum is an exact
// integer < 2^53.  BIG/MID class (q < 2^61): three 20-bit parts, 6 Karatsuba products, every sum
// < 2^50 for t1 <= 256.  CTA = MACM_XT coefficients (one per warp) x one limb x one component x one
// 8-wide giant-index tile; it streams all ciphertexts in tiles of 16 through a cp.async pipeline of
// MACM_JC-baby-step stages ([MACM_JC][16 b][MACM_XT] words, XOR-swizzled so every fragment load is
// bank-conflict free), keeps its plaintext tile [8][t1][MACM_XT] resident (read once per launch), and
// writes W through shared memory as coalesced 64-byte rows.  Each thread copies the same (b, x) for
// MACM_JC consecutive baby steps, so fill addresses are one pointer plus a constant stride.
// XT = coefficients per CTA (template parameter): 16 = 128-byte rows per (baby step, ciphertext) from HBM, 512 threads,
// one CTA per SM -- faster for the large batched launches (B = 256: 23.7 -> 23.0 ms per chunk); 8 = 64-byte rows,
// 256 threads, two CTAs per SM -- faster for small batches (B = 128 stacks +3 %, single-ciphertext latency +5 %)
#define MACM_JC 16
#ifndef MACM_ST
#define MACM_ST 3   // 4 stages (208 KiB): 26.2 vs 23.0 ms per chunk
#endif

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem)
{
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N)); }

// swizzled word index of V element (jj, bb, x) in a stage and of pt element (k, j, x) in the tile
template <int XT>
__device__ __forceinline__ int macm_vidx(int jj, int bb, int x)
{
    if constexpr (XT == 8) return (jj * 16 + bb) * XT + (x ^ (((jj & 3) << 1) | ((bb >> 1) & 1)));
    // rows of 16 words = all 16 banks: the 16 (tig, gid & 3) lanes of a half-warp need 16 different columns
    else return (jj * 16 + bb) * XT + (x ^ (((jj & 3) << 2) | (bb & 3)));
}
template <int XT>
__device__ __forceinline__ int macm_pidx(int k, int j, int t1, int x)
{
    if constexpr (XT == 8) return (k * t1 + j) * XT + (x ^ (((k & 3) << 1) | ((j >> 1) & 1)));
    else return (k * t1 + j) * XT + (x ^ (((k & 3) << 2) | (j & 3)));
}

// column swizzle of output row (k, bb) in the staging tile
template <int XT>
__device__ __forceinline__ int macm_osw(int row)
{
    if constexpr (XT == 8) return (((row >> 5) & 3) << 1) | ((row >> 1) & 1);
    else return (((row >> 5) & 3) << 2) | (row & 3);
}

template <bool INT, int MACM_XT>
__device__ __forceinline__ void macm_body(const DCtx* __restrict__ dc, const u64* __restrict__ pts, int pt_nl,
                                          const u64* __restrict__ v0, size_t v0_stride, const u64* __restrict__ vb,
                                          u64* __restrict__ wout, int t1, int t2, int batch, int nl, int qp, u64* msm)
{
    constexpr int MACM_THREADS = 32 * MACM_XT;
    constexpr int SV = MACM_JC * 16 * MACM_XT;               // words per stage
    constexpr int EPT = SV / MACM_THREADS;                   // words per thread per stage (= MACM_JC / 2)
    static_assert(MACM_THREADS / MACM_XT == 32 && EPT * 2 == MACM_JC, "fill mapping");
    const int n = dc->n;
    const int l = blockIdx.y;
    const int nlx = nl + (qp ? dc->n_special : 0);
    const int pidx = ext_prime_of(l, nl, dc->n_data);
    const DPrime Pr = dc->p[pidx];
    const int x0 = blockIdx.x * MACM_XT, c = blockIdx.z & 1, k0 = (blockIdx.z >> 1) * 8;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int t1p = (t1 + MACM_JC - 1) / MACM_JC * MACM_JC;
    u64* Ps = msm;                                           // [8][t1p][XT] (k relative to k0)
    u64* Vs = Ps + 8 * t1p * MACM_XT;                        // [ST][SV]
    u64* Os = Vs + MACM_ST * SV;                             // [8 k][16 b][XT]
    // ---- plaintext tile (zero beyond t1 / t2)
    // (8 tile loads in flight per thread before their stores: the tile is latency-, not bandwidth-bound,
    //  and it precedes the pipeline)
    for (int i0 = tid; i0 < 8 * t1p * MACM_XT; i0 += 8 * MACM_THREADS) {
        u64 a[8];
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const int i = i0 + h * MACM_THREADS;
            const int x = i % MACM_XT, j = (i / MACM_XT) % t1p, k = i / (MACM_XT * t1p);
            a[h] = 0;
            if (i < 8 * t1p * MACM_XT && j < t1 && k0 + k < t2)
                a[h] = pts[((size_t)((k0 + k) * t1 + j) * pt_nl + l) * n + x0 + x];
        }
#pragma unroll
        for (int h = 0; h < 8; ++h) {
            const int i = i0 + h * MACM_THREADS;
            if (i >= 8 * t1p * MACM_XT) break;
            const int x = i % MACM_XT, j = (i / MACM_XT) % t1p, k = i / (MACM_XT * t1p);
            Ps[macm_pidx<MACM_XT>(k, j, t1p, x)] = a[h];
        }
    }
    const size_t ctw = (size_t)2 * nlx * n, jstride = (size_t)batch * ctw;
    const u64 Pm = qp ? dc->pmod[l < nl ? l : 0] : 0, Pm_sh = qp ? dc->pmod_sh[l < nl ? l : 0] : 0;
    const int nbt = (batch + 15) / 16, njc = t1p / MACM_JC, iters = nbt * njc;
    // fill mapping: thread -> (x, bb, half) copies baby steps jj = half * EPT + h, h < EPT
    const int fx = tid % MACM_XT, fbb = (tid / MACM_XT) % 16, fhalf = tid / (MACM_XT * 16);
    const size_t foff = ((size_t)c * nlx + l) * n + x0 + fx;
    // stage (bt, jc) of the fill sequence tracked by counters (no runtime division per stage)
    int fbt = 0, fjc = 0;
    auto fill = [&](int it) {
        u64* S = Vs + (it % MACM_ST) * SV;
        const int bt = fbt, jc = fjc;
        if (++fjc == njc) {
            fjc = 0;
            ++fbt;
        }
        const int b = bt * 16 + fbb, jb = jc * MACM_JC + fhalf * EPT;
        const bool fast = b < batch && jb >= 1 && jb + EPT <= t1;
        if (fast) {
            const u64* src = vb + ((size_t)(jb - 1) * batch + b) * ctw + foff;
#pragma unroll
            for (int h = 0; h < EPT; ++h) cp_async8(S + macm_vidx<MACM_XT>(fhalf * EPT + h, fbb, fx), src + h * jstride);
        } else {
#pragma unroll
            for (int h = 0; h < EPT; ++h) {
                const int j = jb + h;
                u64* dst = S + macm_vidx<MACM_XT>(fhalf * EPT + h, fbb, fx);
                if (b >= batch || j >= t1) {
                    *dst = 0;
                } else if (j == 0) {
                    u64 y = 0;
                    if (!qp) y = v0[(size_t)b * v0_stride + ((size_t)c * nl + l) * n + x0 + fx];
                    else if (l < nl)
                        y = csub(shoup_mul(v0[(size_t)b * v0_stride + ((size_t)c * nl + l) * n + x0 + fx], Pm, Pm_sh, Pr.q),
                                 Pr.q);
                    *dst = y;
                } else {
                    cp_async8(dst, vb + ((size_t)(j - 1) * batch + b) * ctw + foff);
                }
            }
        }
    };
#pragma unroll
    for (int s = 0; s < MACM_ST - 1; ++s) {
        if (s < iters) fill(s);
        cp_async_commit();
    }
    const double q = (double)Pr.q, qinv = 1.0 / q;
    // fold interval in k-steps of 4 terms (FP class only): 64 terms for q < 2^41, else 32
    const int fold_ks = Pr.q < (1ULL << 41) ? 16 : 8;
    constexpr int NS = INT ? 6 : 3;
    constexpr int KS = MACM_JC / 4;                          // k-steps per stage
    double S[NS][4];
    const int x = warp;
    // pt swizzle: XT = 8: (j >> 1 & 1 == tig >> 1 & 1); XT = 16: (j & 3 == tig)
    const int xsw = MACM_XT == 8 ? (x ^ (((gid & 3) << 1) | ((tig >> 1) & 1))) : (x ^ (((gid & 3) << 2) | tig));
    const u64* Pw = Ps + (size_t)gid * t1p * MACM_XT + xsw;
    int it = 0;
    for (int bt = 0; bt < nbt; ++bt) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
#pragma unroll
            for (int e = 0; e < 4; ++e) S[s][e] = 0.0;
        for (int jc = 0; jc < njc; ++jc, ++it) {
            cp_async_wait<MACM_ST - 2>();
            __syncthreads();
            if (it + MACM_ST - 1 < iters) fill(it + MACM_ST - 1);
            cp_async_commit();
            const u64* Sv = Vs + (it % MACM_ST) * SV;
#pragma unroll
            for (int kq = 0; kq < KS; ++kq) {
                const int jj = kq * 4 + tig;
                const u64 bv = Pw[(size_t)(jc * MACM_JC + jj) * MACM_XT];
                const u64 a0 = Sv[macm_vidx<MACM_XT>(jj, gid, x)], a1 = Sv[macm_vidx<MACM_XT>(jj, gid + 8, x)];
                if constexpr (!INT) {
                    const u64 m = (1ULL << 23) - 1;
                    const double bh = p2d(bv >> 23), bl = p2d(bv & m);
                    // V words: canonical, or signed [-q/2, q/2] from the tensor-core IP (arithmetic shift)
                    const double a0h = sp2d((long long)a0 >> 23), a0l = p2d(a0 & m),
                                 a1h = sp2d((long long)a1 >> 23), a1l = p2d(a1 & m);
                    dmma16884(S[2], a0h, a1h, bh);
                    dmma16884(S[0], a0l, a1l, bl);
                    // part sums in the integer domain (IADD + I2F instead of a DADD on the shared datapath)
                    dmma16884(S[1], sp2d(((long long)a0 >> 23) + (long long)(a0 & m)),
                              sp2d(((long long)a1 >> 23) + (long long)(a1 & m)), p2d((bv >> 23) + (bv & m)));
                } else {
                    const u64 m = (1ULL << 20) - 1;
                    const double y[3] = {p2d(bv & m), p2d((bv >> 20) & m), p2d(bv >> 40)};
                    const double p[3] = {p2d(a0 & m), p2d((a0 >> 20) & m), p2d(a0 >> 40)};
                    const double r[3] = {p2d(a1 & m), p2d((a1 >> 20) & m), p2d(a1 >> 40)};
                    dmma16884(S[0], p[0], r[0], y[0]);
                    dmma16884(S[1], p[1], r[1], y[1]);
                    dmma16884(S[2], p[2], r[2], y[2]);
                    dmma16884(S[3], p[0] + p[1], r[0] + r[1], y[0] + y[1]);
                    dmma16884(S[4], p[1] + p[2], r[1] + r[2], y[1] + y[2]);
                    dmma16884(S[5], p[0] + p[2], r[0] + r[2], y[0] + y[2]);
                }
                if constexpr (!INT) {
                    const int ks = jc * KS + kq + 1;              // k-steps accumulated so far
                    if (ks % fold_ks == 0 && ks * 4 < t1p) {      // fold (exactness, see above)
#pragma unroll
                        for (int s = 0; s < 3; ++s)
#pragma unroll
                            for (int e = 0; e < 4; ++e) S[s][e] = freduce(S[s][e], q, qinv);
                    }
                }
            }
        }
        // recombine mod q: thread holds (b = gid + 8 (e >> 1), k = 2 tig + (e & 1))
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            u64 u;
            if constexpr (!INT) {
                const double s0 = S[0][e], s2 = S[2][e], s1 = S[1][e] - s2 - s0;
                const double r0 = freduce(s0, q, qinv), r1 = freduce(s1, q, qinv), r2 = freduce(s2, q, qinv);
                const double two46 = 70368744177664.0;
                const double w46 = two46 - floor(two46 * qinv) * q, w46q = w46 / q, c23q = 8388608.0 / q;
                const double k1 = __fma_rn(r1, c23q, CK_RND_MAGIC) - CK_RND_MAGIC;
                const double tt1 = __fma_rn(-k1, q, r1 * 8388608.0);
                const double tt2 = fmodmul(r2, w46, w46q, q);
                u = fcanon(tt2 + tt1 + r0, q, qinv);
            } else {
                const double P0 = S[0][e], P1 = S[1][e], P2 = S[2][e];
                const u64 s0 = d2u(P0), s1 = d2u(S[3][e] - P0 - P1), s2 = d2u(S[5][e] - P0 - P2 + P1),
                          s3 = d2u(S[4][e] - P1 - P2), s4 = d2u(P2);
                u64 lo = s0, hi = 0, add;
                add = s1 << 20; lo += add; hi += (lo < add) + (s1 >> 44);
                add = s2 << 40; lo += add; hi += (lo < add) + (s2 >> 24);
                add = s3 << 60; lo += add; hi += (lo < add) + (s3 >> 4);
                hi += s4 << 16;
                u = reduce128(hi, lo, Pr);
            }
            const int bb = gid + 8 * (e >> 1), k = 2 * tig + (e & 1);
            const int row = k * 16 + bb;
            Os[row * MACM_XT + (x ^ macm_osw<MACM_XT>(row))] = u;
        }
        __syncthreads();
        // coalesced write: row (k, bb) of MACM_XT words
        for (int i = tid; i < 8 * 16 * MACM_XT; i += MACM_THREADS) {
            const int xx = i % MACM_XT, row = i / MACM_XT;
            const int bb = row % 16, k = row / 16, b = bt * 16 + bb;
            if (b < batch && k0 + k < t2)
                wout[((size_t)(k0 + k) * batch + b) * ctw + ((size_t)c * nlx + l) * n + x0 + xx] =
                    Os[row * MACM_XT + (xx ^ macm_osw<MACM_XT>(row))];
        }
    }
    cp_async_wait<0>();
}

// one launch for both limb classes (the 3-product FP rows and the 6-product 60-bit rows share the SMs)
template <int XT>
__global__ void __launch_bounds__(32 * XT, XT == 8 ? 2 : 1)
k_bsgs_mac_mma(const DCtx* __restrict__ dc, const u64* __restrict__ pts, int pt_nl, const u64* __restrict__ v0,
               size_t v0_stride, const u64* __restrict__ vb, u64* __restrict__ wout, int t1, int t2, int batch, int nl,
               int qp)
{
    extern __shared__ u64 msm[];
    const int l = blockIdx.y;
    const u64 q = dc->p[ext_prime_of(l, nl, dc->n_data)].q;
    if (prime_class(q) == PC_FP) macm_body<false, XT>(dc, pts, pt_nl, v0, v0_stride, vb, wout, t1, t2, batch, nl, qp, msm);
    else macm_body<true, XT>(dc, pts, pt_nl, v0, v0_stride, vb, wout, t1, t2, batch, nl, qp, msm);
}

static size_t mac_mma_smem(int t1, int xt)
{
    const int t1p = (t1 + MACM_JC - 1) / MACM_JC * MACM_JC;
    return sizeof(u64) * ((size_t)8 * t1p * xt + (size_t)MACM_ST * MACM_JC * 16 * xt + 8 * 16 * xt);
}

void bsgs_mac(const Launch& L, const uint64_t* pts, int pt_nl, const uint64_t* v0, size_t v0_stride,
              const uint64_t* vbaby, uint64_t* wout, int t1, int t2, int batch, int nl, bool qp, bool mac_layout)
{
    if (mac_layout) {   // double-hoisted baby steps in the tensor-core MAC layout (the producer checked the shape)
        if (!bsgs_mac_tc(L, pts, pt_nl, v0, v0_stride, vbaby, wout, t1, t2, batch, nl))
            throw std::runtime_error("bsgs_mac: MAC layout without the tensor-core MAC");
        return;
    }
    const int nlx = nl + (qp ? L.n_special : 0);
    if (batch <= 0) return;
    const int n = 1 << L.log_n;
    static const int use_mma = [] {
        const char* e = getenv("CKKS_MAC_MMA");
        return e ? atoi(e) : 1;
    }();

    if (use_mma && t1 <= 256 && n >= 16) {
        if (L.probe && L.probe->kind == PROBE_ALL) {
            // per row: B x 2 components x t1 x t2 x N modular MACs, 3 (FP class) or 6 (60-bit) exact
            // split products each; bytes: baby steps + input read, plaintexts read, W written
            for (int l = 0; l < nlx; ++l) {
                const int p = ext_prime_of(l, nl, L.n_data);
                const bool fp = L.pclass && L.pclass[p] == PC_FP;
                const char* nm = "k_bsgs_mac_mma";
                L.probe->flops_by_kernel[nm] += 2.0 * (fp ? 3 : 6) * batch * 2.0 * t1 * t2 * n;
                L.probe->bytes_by_kernel[nm] +=
                    ((double)t1 * batch * 2 + (double)t1 * t2 + (double)t2 * batch * 2) * n * 8.0;
            }
        }
        // 16 coefficients per CTA for the large batched launches, 8 below (see the XT note above)
        static const int xt_batch = [] {
            const char* e = getenv("CKKS_MAC_XT16_BATCH");
            return e ? atoi(e) : 192;
        }();
        ProbeScope ps_(L.probe, L.st, "k_bsgs_mac_mma");
        if (batch >= xt_batch && mac_mma_smem(t1, 16) <= 227 * 1024) {   // (t1 <= 112 fits the 227 KiB)
            const size_t smem = mac_mma_smem(t1, 16);
            allow_smem(k_bsgs_mac_mma<16>, smem);
            k_bsgs_mac_mma<16><<<dim3(n / 16, nlx, 2 * ((t2 + 7) / 8)), 512, smem, L.st>>>(
                L.dc, pts, pt_nl, v0, v0_stride, vbaby, wout, t1, t2, batch, nl, qp ? 1 : 0);
        } else {
            const size_t smem = mac_mma_smem(t1, 8);
            allow_smem(k_bsgs_mac_mma<8>, smem);
            k_bsgs_mac_mma<8><<<dim3(n / 8, nlx, 2 * ((t2 + 7) / 8)), 256, smem, L.st>>>(
                L.dc, pts, pt_nl, v0, v0_stride, vbaby, wout, t1, t2, batch, nl, qp ? 1 : 0);
        }
        check_launch("bsgs_mac_mma");
        if (L.counter) *L.counter += 1;
        return;
    }
    if ((size_t)t1 * t2 * MACF_XT * sizeof(double2) > 200 * 1024)
        throw std::runtime_error("bsgs_mac: plaintext tile too large (t <= 1600)");
    const size_t smem_int = (size_t)t1 * t2 * MACF_XT * sizeof(u64);
    allow_smem(k_bsgs_mac_int, smem_int);
    { ProbeScope ps_(L.probe, L.st, "k_bsgs_mac_int"); k_bsgs_mac_int<<<dim3(n / MACF_XT, nlx), MACF_XT * MACF_BL, smem_int, L.st>>>(L.dc, pts, pt_nl, v0, v0_stride, vbaby, wout, t1, t2, batch, nl, qp ? 1 : 0); }
    const size_t smem_fp = (size_t)t1 * t2 * MACF_XT * sizeof(double2);
    allow_smem(k_bsgs_mac_fp, smem_fp);
    { ProbeScope ps_(L.probe, L.st, "k_bsgs_mac_fp"); k_bsgs_mac_fp<<<dim3(n / MACF_XT, nlx), MACF_XT * MACF_BL, smem_fp, L.st>>>(L.dc, pts, pt_nl, v0, v0_stride, vbaby, wout, t1, t2, batch, nl, qp ? 1 : 0); }
    check_launch("bsgs_mac");
    if (L.counter) *L.counter += 2;
}

}  // namespace ck
