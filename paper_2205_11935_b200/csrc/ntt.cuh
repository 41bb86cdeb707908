// ntt.cuh -- CTA-level negacyclic NTT / iNTT over one limb, radix-2^LOGE register passes.
//
// Definition (R2):  NTT(a)[k] = sum_i a_i psi^{(2 brev(k) + 1) i}  mod q,
// bit-reversed output order.  Stage s (0..LOGN-1) of the forward transform pairs indices that
// differ in bit LOGN-1-s with twiddle W[2^s + block] = psi^{brev(2^s + block)} (Cooley-Tukey);
// the inverse runs the stages backwards with IW = psi^{-brev(.)} (Gentleman-Sande) and N^{-1}.
//
// B200 mapping.  One CTA owns one limb (N <= 16384 words = 128 KiB of shared memory).  Each of
// NT threads holds E = N/NT residues in registers; a "pass" performs K = LOGK = 4 consecutive stages
// entirely in registers on groups of 16 elements (radix-16), so the limb crosses shared memory
// only between passes (4 passes for N=16384).  The first forward pass loads straight
// from the caller's loader (HBM, coalesced: lane <-> consecutive index), the last pass stores
// straight through the caller's storer (each thread owns E contiguous words).  The inverse mirrors
// this.  Shared memory is XOR-swizzled  a ^ (((a >> 4) ^ (a >> 5)) & 15)  -- conflict-free (2 wavefronts per
// 64-bit warp access) for every pass of every supported (LOGN, NT), checked by
// tests/test_ntt_layout.py.  Butterflies are Harvey-lazy: forward values live in [0, 4q), inverse
// values in [0, 2q); loaders must supply values < 2q; storers receive canonical values in [0, q).
#pragma once
#include "common.cuh"
#include <type_traits>

template <int I, int END, class F>
__device__ __forceinline__ void static_for(F&& f)
{
    if constexpr (I < END) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, END>(f);
    }
}

constexpr int ilog2c(int x) { return x <= 1 ? 0 : 1 + ilog2c(x >> 1); }

// Prime classes: the arithmetic and the lazy-reduction schedule are chosen from q (bounds tracked
// per stage).
//   PC_FP     q < 2^45: residues held as exact integers in FP64 registers; butterflies on the
//                       FP64 pipe (8 DFMA-class ops: error-free product + rint quotient), signed
//                       representatives; forward needs no reduction, inverse reduces per pass
//   PC_FPR    q < 2^50: FP64 pipe as PC_FP with a few reductions (twiddles are centred, |w| <= q/2, so
//                       fmodmul takes |y| < 2^52 ~ 4q): the forward reduces the X input of the first stage
//                       of every pass (values < 3.7 q inside a pass of <= 5 stages: 8.6-8.75 FP64 ops per
//                       butterfly), the inverse reduces every other stage's sums (values < 1.2 q, |u - v| <
//                       2.3 q: 9.5 ops) -- bounds in DESIGN.md section 5
//   PC_MID    q < 2^52: 64-bit integer Shoup, forward without reductions, inverse Harvey-lazy
//   PC_BIG    q < 2^61: 64-bit integer Shoup, Harvey-lazy both ways ([0,4q) fwd, [0,2q) inv)
// (key-switch inner products and BSGS sums treat every class but PC_FP as 60-bit: three-part splits)
enum { PC_FP = 0, PC_MID = 1, PC_BIG = 2, PC_SMALL = 3, PC_FPR = 4 };
__host__ __device__ __forceinline__ int prime_class(u64 q)
{
    return q < (1ULL << 45) ? PC_FP : q < (1ULL << 50) ? PC_FPR : (q < (1ULL << 52) ? PC_MID : PC_BIG);
}

// ---- FP64 modular arithmetic on exact integers (|values| < 2^51)
#define CK_RND_MAGIC 6755399441055744.0   /* 1.5 * 2^52: x + M - M = rint(x) for |x| < 2^51 */
#define CK_TWO52 4503599627370496.0
// y * w mod q as a signed representative; wq = fl(w / q), |w| <= q/2 (centred twiddles), |y| < 2^52:
// |y wq| < 2^51 so k = rint(y wq) exactly, |y wq - y w / q| <= |y| 2^-54, so |result| <= (1/2 + |y| 2^-54) q
// (< 0.51 q for |y| < 2^47, < 0.75 q always); ph - k q and the sum with pl are integers < 2^53: exact
__device__ __forceinline__ double fmodmul(double y, double w, double wq, double q)
{
    const double ph = y * w;
    const double pl = __fma_rn(y, w, -ph);                        // exact low part of y*w
    const double k = __fma_rn(y, wq, CK_RND_MAGIC) - CK_RND_MAGIC; // rint(y w / q)
    return __fma_rn(-k, q, ph) + pl;                               // exact integer
}
// v mod q, signed representative in [-q/2, q/2]; qinv = fl(1/q)
__device__ __forceinline__ double freduce(double v, double q, double qinv)
{
    const double k = __fma_rn(v, qinv, CK_RND_MAGIC) - CK_RND_MAGIC;
    return __fma_rn(-k, q, v);
}
__device__ __forceinline__ double u2d(u64 a) { return __longlong_as_double((long long)(a | 0x4330000000000000ULL)) - CK_TWO52; }
// v in [0, 2^52) exact integer -> u64
__device__ __forceinline__ u64 d2u(double v) { return (u64)__double_as_longlong(v + CK_TWO52) & 0xFFFFFFFFFFFFFULL; }
// 32-bit parts -> double by the conversion instruction (I2F.F64), not the FP64 add of u2d: the split
// operands of the tensor-core kernels are converted off the FP64 datapath that DMMA shares
__device__ __forceinline__ double p2d(u64 part) { return __uint2double_rn((unsigned)part); }
__device__ __forceinline__ double sp2d(long long part) { return __int2double_rn((int)part); }
// signed integers |x| < 2^51 <-> double (two's complement int64 in a u64 word)
__device__ __forceinline__ double s2d(u64 a)
{
    return __longlong_as_double((long long)(a + 0x4338000000000000ULL)) - CK_RND_MAGIC;
}
__device__ __forceinline__ u64 d2s(double v) { return (u64)__double_as_longlong(v + CK_RND_MAGIC) - 0x4338000000000000ULL; }
// signed representative with |v| < 2^51 -> canonical [0, q)
__device__ __forceinline__ u64 fcanon(double v, double q, double qinv)
{
    double r = freduce(v, q, qinv);   // [-q/2, q/2]
    r = r < 0.0 ? r + q : r;
    return d2u(r);
}

// forward loaders may return the value as an exact signed double (|v| < 2 q) instead of a word in [0, 2q)
__device__ __forceinline__ double ld_to_fp(u64 a) { return u2d(a); }
__device__ __forceinline__ double ld_to_fp(double v) { return v; }

template <int LOGN_, int NT_>
struct NttCta {
    static constexpr int LOGN = LOGN_;
    static constexpr int NT = NT_;
    static constexpr int N = 1 << LOGN;
    static constexpr int E = N / NT;
    static constexpr int LOGE = ilog2c(E);
    static constexpr int LOGK = 4;                          // stages per pass (radix 16), fixed:
                                                            // the twiddle tables are ordered for it
    static constexpr int NPASS = (LOGN + LOGK - 1) / LOGK;
    static_assert((1 << LOGE) == E, "E must be a power of two");
    static_assert(LOGE >= LOGK && LOGE <= 5, "16 or 32 residues per thread");

    template <int P>
    struct Pass {
        static constexpr int S0 = P * LOGK;
        static constexpr int K = (LOGN - S0 < LOGK) ? (LOGN - S0) : LOGK;
        static constexpr int G = E >> K;          // groups per thread
        static constexpr int SH = LOGN - S0 - K;  // log2(stride between group elements)
    };

    __device__ __forceinline__ static int swz(int a) { return a ^ (((a >> 4) ^ (a >> 5)) & 15); }

    // index of element i of the thread's group g in pass P
    template <int P>
    __device__ __forceinline__ static int index(int tid, int g, int i)
    {
        using G_ = Pass<P>;
        const int gid = g * NT + tid;
        const int b0 = gid >> G_::SH;
        const int o = gid & ((1 << G_::SH) - 1);
        return (b0 << (LOGN - G_::S0)) + (i << G_::SH) + o;
    }

    // Twiddle table position of stage s = S0 + r, block b0 * 2^r + j (tables are stored
    // "pass-ordered", see ntt_tw_position, so lanes with consecutive b0 read consecutive words).
    __device__ __forceinline__ static int tw_index(int S0, int r, int b0, int j) { return (1 << (S0 + r)) + (j << S0) + b0; }

    template <int P, int PC>
    __device__ __forceinline__ static void fwd_compute(u64 (&x)[E], int tid, const u64* __restrict__ W,
                                                       const u64* __restrict__ Wsh, u64 q, u64 q2)
    {
        using G_ = Pass<P>;
        constexpr int K = G_::K;
#pragma unroll
        for (int g = 0; g < G_::G; ++g) {
            const int gid = g * NT + tid;
            const int b0 = gid >> G_::SH;
#pragma unroll
            for (int r = 0; r < K; ++r) {
                const int half = 1 << (K - 1 - r);
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    if (i & half) continue;
                    const int m = tw_index(G_::S0, r, b0, i >> (K - r));
                    const u64 w = __ldg(W + m), ws = __ldg(Wsh + m);
                    u64& X = x[g * (1 << K) + i];
                    u64& Y = x[g * (1 << K) + i + half];
                    const u64 xx = (PC == PC_BIG) ? csub(X, q2) : X;
                    const u64 t = shoup_mul(Y, w, ws, q);
                    X = xx + t;
                    Y = xx - t + q2;
                }
            }
        }
    }

    template <int P, int PC>
    __device__ __forceinline__ static void inv_compute(u64 (&x)[E], int tid, const u64* __restrict__ IW,
                                                       const u64* __restrict__ IWsh, u64 q, u64 q2)
    {
        using G_ = Pass<P>;
        constexpr int K = G_::K;
#pragma unroll
        for (int g = 0; g < G_::G; ++g) {
            const int gid = g * NT + tid;
            const int b0 = gid >> G_::SH;
#pragma unroll
            for (int r = K - 1; r >= 0; --r) {
                const int half = 1 << (K - 1 - r);
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    if (i & half) continue;
                    const int m = tw_index(G_::S0, r, b0, i >> (K - r));
                    const u64 w = __ldg(IW + m), ws = __ldg(IWsh + m);
                    u64& X = x[g * (1 << K) + i];
                    u64& Y = x[g * (1 << K) + i + half];
                    const u64 u = X, v = Y;
                    if constexpr (PC == PC_SMALL) {
                        // both inputs < 2^(c+1) q after c = LOGN - S0 - 1 - r stages: no reduction
                        X = u + v;
                        Y = shoup_mul(u - v + (q << (LOGN - G_::S0 - r)), w, ws, q);
                    } else {
                        X = csub(u + v, q2);
                        Y = shoup_mul(u - v + q2, w, ws, q);
                    }
                }
            }
        }
    }

    // ---- FP64 variants (PC_FP): x holds exact signed integers
    template <int P, bool R>
    __device__ __forceinline__ static void fwd_compute_fp(double (&x)[E], int tid, const double* __restrict__ Wd,
                                                          const double* __restrict__ Wq, double q, double qinv)
    {
        using G_ = Pass<P>;
        constexpr int K = G_::K;
#pragma unroll
        for (int g = 0; g < G_::G; ++g) {
            const int b0 = (g * NT + tid) >> G_::SH;
#pragma unroll
            for (int r = 0; r < K; ++r) {
                const int half = 1 << (K - 1 - r);
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    if (i & half) continue;
                    const int m = tw_index(G_::S0, r, b0, i >> (K - r));
                    const double w = __ldg(Wd + m), wq = __ldg(Wq + m);
                    double& X = x[g * (1 << K) + i];
                    double& Y = x[g * (1 << K) + i + half];
                    const double t = fmodmul(Y, w, wq, q);   // |t| < 0.51 q  (FPR: < (0.5 + |Y| / 16 q) q)
                    const double xx = (R && r == 0) ? freduce(X, q, qinv) : X;
                    X = xx + t;                              // |.| grows by < 0.51 q per stage (FPR: < 0.75 q)
                    Y = xx - t;
                }
            }
        }
    }

    template <int P, bool R>
    __device__ __forceinline__ static void inv_compute_fp(double (&x)[E], int tid, const double* __restrict__ IWd,
                                                          const double* __restrict__ IWq, double q, double qinv)
    {
        using G_ = Pass<P>;
        constexpr int K = G_::K;
        // pass entry: bring every value back to [-q/2, q/2] (the X lineage doubles per stage);
        // FPR reduces every sum instead
        if constexpr (P != NPASS - 1 && !R) {
#pragma unroll
            for (int i = 0; i < E; ++i) x[i] = freduce(x[i], q, qinv);
        }
#pragma unroll
        for (int g = 0; g < G_::G; ++g) {
            const int b0 = (g * NT + tid) >> G_::SH;
#pragma unroll
            for (int r = K - 1; r >= 0; --r) {
                const int half = 1 << (K - 1 - r);
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    if (i & half) continue;
                    const int m = tw_index(G_::S0, r, b0, i >> (K - r));
                    const double w = __ldg(IWd + m), wq = __ldg(IWq + m);
                    double& X = x[g * (1 << K) + i];
                    double& Y = x[g * (1 << K) + i + half];
                    const double u = X, v = Y;
                    // FPR: sums reduced at every other stage, counted from the first one executed (LOGN - 1)
                    X = (R && ((LOGN - 1 - (G_::S0 + r)) & 1)) ? freduce(u + v, q, qinv) : u + v;
                    Y = fmodmul(u - v, w, wq, q);
                }
            }
        }
    }

    template <bool R = false, class Load, class Store>
    __device__ __forceinline__ static void forward_fp(u64* sm, const DPrime& Pr, const u64* __restrict__ tw,
                                                      Load&& ld, Store&& st)
    {
        const int tid = threadIdx.x;
        const double q = (double)Pr.q, qinv = 1.0 / q;
        const double* Wd = reinterpret_cast<const double*>(tw + 4 * N);
        const double* Wq = reinterpret_cast<const double*>(tw + 5 * N);
        double* smd = reinterpret_cast<double*>(sm);
        double x[E];
        static_for<0, NPASS>([&](auto pc) {
            constexpr int P = decltype(pc)::value;
            using G_ = Pass<P>;
            constexpr int K = G_::K;
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    const int idx = index<P>(tid, g, i);
                    if constexpr (P == 0) x[g * (1 << K) + i] = ld_to_fp(ld(idx));   // u64 in [0, 2q) or a signed double
                    else x[g * (1 << K) + i] = smd[swz(idx)];
                }
            fwd_compute_fp<P, R>(x, tid, Wd, Wq, q, qinv);
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) smd[swz(index<P>(tid, g, i))] = x[g * (1 << K) + i];
            __syncthreads();
        });
#pragma unroll 4
        for (int c = 0; c < E; ++c) {
            const int idx = c * NT + tid;
            st(idx, fcanon(smd[swz(idx)], q, qinv));
        }
        __syncthreads();
    }

    // place(idx) = the transform index the value ld(idx) belongs to (a permuted input read in its own order, so
    // the global loads stay coalesced and the permutation happens in the shared-memory staging)
    template <bool R = false, class Load, class Store>
    __device__ __forceinline__ static void inverse_fp(u64* sm, const DPrime& Pr, const u64* __restrict__ tw,
                                                      Load&& ld, Store&& st)
    {
        inverse_fp<R, false>(sm, Pr, tw, ld, st, [](int i) { return i; });
    }
    // SIGNED_ST: st(idx, double) receives the signed representative (|v| < 0.66 q) instead of the canonical word
    // (for epilogues that go on in FP64, k_ksdigits.cu)
    template <bool R = false, bool SIGNED_ST = false, class Load, class Store, class Place>
    __device__ __forceinline__ static void inverse_fp(u64* sm, const DPrime& Pr, const u64* __restrict__ tw,
                                                      Load&& ld, Store&& st, Place&& place)
    {
        const int tid = threadIdx.x;
        const double q = (double)Pr.q, qinv = 1.0 / q;
        const double* IWd = reinterpret_cast<const double*>(tw + 6 * N);
        const double* IWq = reinterpret_cast<const double*>(tw + 7 * N);
        const double ninv = Pr.ninv > Pr.q / 2 ? -(double)(Pr.q - Pr.ninv) : (double)Pr.ninv, ninvq = ninv / q;
        double* smd = reinterpret_cast<double*>(sm);
        double x[E];
#pragma unroll 4
        for (int c = 0; c < E; ++c) {
            const int idx = c * NT + tid;
            smd[swz(place(idx))] = R ? freduce(u2d(ld(idx)), q, qinv) : u2d(ld(idx));
        }
        __syncthreads();
        static_for<0, NPASS>([&](auto pc) {
            constexpr int P = NPASS - 1 - decltype(pc)::value;
            using G_ = Pass<P>;
            constexpr int K = G_::K;
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) x[g * (1 << K) + i] = smd[swz(index<P>(tid, g, i))];
            inv_compute_fp<P, R>(x, tid, IWd, IWq, q, qinv);
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    const int idx = index<P>(tid, g, i);
                    const double v = x[g * (1 << K) + i];
                    if constexpr (P == 0) {
                        double r = fmodmul(v, ninv, ninvq, q);   // (-0.51 q, 0.51 q); FPR: (-0.66 q, 0.66 q)
                        if constexpr (SIGNED_ST) {
                            st(idx, r);
                        } else {
                            r = r < 0.0 ? r + q : r;
                            st(idx, d2u(r));
                        }
                    } else {
                        smd[swz(idx)] = v;
                    }
                }
            __syncthreads();
        });
    }

    // forward outputs: [0, 4q) (BIG) or [0, 30q) (SMALL/MID) -> [0, q)
    template <int PC>
    __device__ __forceinline__ static u64 fwd_final(u64 v, const DPrime& Pr)
    {
        if constexpr (PC == PC_BIG) return csub(csub(v, Pr.q2), Pr.q);
        else return reduce64(v, Pr);
    }

    // Forward NTT of one limb.  ld(idx) -> value in [0, 2q); st(idx, v) receives v in [0, q).
    // `tw` points at this prime's [4][N] table block.  `sm` holds N words (+ nothing else).
    template <int PC = PC_BIG, bool STAGED = true, class Load, class Store>
    __device__ __forceinline__ static void forward(u64* sm, const DPrime& Pr, const u64* __restrict__ tw,
                                                   Load&& ld, Store&& st)
    {
        const int tid = threadIdx.x;
        const u64 q = Pr.q, q2 = Pr.q2;
        const u64* W = tw;
        const u64* Wsh = tw + N;
        u64 x[E];
        static_for<0, NPASS>([&](auto pc) {
            constexpr int P = decltype(pc)::value;
            using G_ = Pass<P>;
            constexpr int K = G_::K;
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    const int idx = index<P>(tid, g, i);
                    if constexpr (P == 0) x[g * (1 << K) + i] = ld(idx);
                    else x[g * (1 << K) + i] = sm[swz(idx)];
                }
            fwd_compute<P, PC>(x, tid, W, Wsh, q, q2);
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    const int idx = index<P>(tid, g, i);
                    u64 v = x[g * (1 << K) + i];
                    if constexpr (P == NPASS - 1) {
                        if constexpr (STAGED) sm[swz(idx)] = v;
                        else st(idx, fwd_final<PC>(v, Pr));
                    } else {
                        sm[swz(idx)] = v;
                    }
                }
            __syncthreads();
        });
        if constexpr (STAGED) {
            // coalesced epilogue: lane <-> consecutive index
#pragma unroll 4
            for (int c = 0; c < E; ++c) {
                const int idx = c * NT + tid;
                st(idx, fwd_final<PC>(sm[swz(idx)], Pr));
            }
            __syncthreads();   // shared memory free again on return
        }
    }

    // Inverse NTT of one limb (includes N^{-1}).  ld(idx) -> value in [0, 2q); st gets [0, q).
    template <int PC = PC_BIG, bool STAGED = true, class Load, class Store>
    __device__ __forceinline__ static void inverse(u64* sm, const DPrime& Pr, const u64* __restrict__ tw,
                                                   Load&& ld, Store&& st)
    {
        inverse<PC, STAGED>(sm, Pr, tw, ld, st, [](int i) { return i; });
    }
    template <int PC = PC_BIG, bool STAGED = true, class Load, class Store, class Place>
    __device__ __forceinline__ static void inverse(u64* sm, const DPrime& Pr, const u64* __restrict__ tw,
                                                   Load&& ld, Store&& st, Place&& place)
    {
        const int tid = threadIdx.x;
        const u64 q = Pr.q, q2 = Pr.q2;
        const u64* IW = tw + 2 * N;
        const u64* IWsh = tw + 3 * N;
        const u64 ninv = Pr.ninv, ninv_sh = Pr.ninv_sh;
        u64 x[E];
        if constexpr (STAGED) {
            // coalesced prologue: lane <-> consecutive index, through shared memory
#pragma unroll 4
            for (int c = 0; c < E; ++c) {
                const int idx = c * NT + tid;
                sm[swz(place(idx))] = ld(idx);
            }
            __syncthreads();
        }
        static_for<0, NPASS>([&](auto pc) {
            constexpr int P = NPASS - 1 - decltype(pc)::value;
            using G_ = Pass<P>;
            constexpr int K = G_::K;
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    const int idx = index<P>(tid, g, i);
                    if constexpr (P == NPASS - 1 && !STAGED) x[g * (1 << K) + i] = ld(idx);
                    else x[g * (1 << K) + i] = sm[swz(idx)];
                }
            inv_compute<P, PC>(x, tid, IW, IWsh, q, q2);
#pragma unroll
            for (int g = 0; g < G_::G; ++g)
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    const int idx = index<P>(tid, g, i);
                    u64 v = x[g * (1 << K) + i];
                    if constexpr (P == 0) st(idx, csub(shoup_mul(v, ninv, ninv_sh, q), q));
                    else sm[swz(idx)] = v;
                }
            __syncthreads();
        });
    }
};

// Runtime dispatch on the prime class (uniform per CTA).
template <class T, class Load, class Store>
__device__ __forceinline__ void ntt_forward(u64* sm, const DPrime& Pr, const u64* tw, Load&& ld, Store&& st)
{
    switch (prime_class(Pr.q)) {
    case PC_FP: T::forward_fp(sm, Pr, tw, ld, st); break;
    case PC_FPR: T::template forward_fp<true>(sm, Pr, tw, ld, st); break;
    case PC_MID: T::template forward<PC_MID>(sm, Pr, tw, ld, st); break;
    default: T::template forward<PC_BIG>(sm, Pr, tw, ld, st); break;
    }
}
template <class T, class Load, class Store, class Place>
__device__ __forceinline__ void ntt_inverse(u64* sm, const DPrime& Pr, const u64* tw, Load&& ld, Store&& st, Place&& place)
{
    const int pc = prime_class(Pr.q);
    if (pc == PC_FP) T::inverse_fp(sm, Pr, tw, ld, st, place);
    else if (pc == PC_FPR) T::template inverse_fp<true>(sm, Pr, tw, ld, st, place);
    else T::template inverse<PC_BIG>(sm, Pr, tw, ld, st, place);
}
template <class T, class Load, class Store>
__device__ __forceinline__ void ntt_inverse(u64* sm, const DPrime& Pr, const u64* tw, Load&& ld, Store&& st)
{
    ntt_inverse<T>(sm, Pr, tw, ld, st, [](int i) { return i; });
}

// Threads per CTA: 16 residues per thread by default (more warps to hide the load latency of
// prologue/epilogue-heavy kernels); NttThreadsWide = 32 residues per thread (more ILP, for the
// compute-bound ModUp).  Passes are radix-16 in both cases (ntt_logk).
__host__ __device__ constexpr int ntt_logk(int logn) { return (void)logn, 4; }
template <int LOGN> struct NttThreads { static constexpr int value = 1 << (LOGN - 4); };
template <int LOGN> struct NttThreadsWide { static constexpr int value = 1 << (LOGN - 5); };

// Host: position of the forward/inverse twiddle of stage s, block m (= b0 2^r + j with
// r = s - S0(s), S0(s) = floor(s / LOGK) LOGK) in the pass-ordered table:  2^s + j 2^S0 + b0.
inline int ntt_tw_position(int logn, int s, int m)
{
    const int logk = ntt_logk(logn);
    const int S0 = (s / logk) * logk, r = s - S0;
    const int b0 = m >> r, j = m & ((1 << r) - 1);
    return (1 << s) + (j << S0) + b0;
}
