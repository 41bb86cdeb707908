// ntt_c.cuh -- CTA-pair (thread-block cluster) NTT / iNTT for the FP64-pipe prime classes (PC_FP, PC_FPR).
//
// Same transform as ntt.cuh (R2: stage s pairs indices differing in bit LOGN-1-s, twiddle W[2^s + block],
// bit-reversed output).  What changes is how much of a limb one CTA holds.  With 32 residues per thread in
// registers a whole N = 16384 limb fills half the register file and 128 KiB of shared memory: one CTA per SM, so
// a limb's global loads, its butterflies and its stores run one after the other (measured, tools/lab: 16.1 us
// per limb of which 9.8 us compute; a pure copy through the same structure reaches 3.5 TB/s).  Here a limb is
// split over a cluster of CL = 2 CTAs of M = N/2 points (N/64 threads, 68 KiB of shared memory each): after
// stage 0 the two halves are independent transforms, so the only traffic between the CTAs is stage 0 itself --
// each CTA loads half of the (x[o], x[o + N/2]) pairs, keeps the results of its own half in registers and
// writes the other 16 per thread into its partner's shared memory (DSMEM) -- and two CTAs of different
// clusters share an SM, one computing while the other loads or stores (5.7 us per 8192-point transform at
// 2 CTAs/SM against 8.1 us at 1, tools/lab).  N <= 8192 limbs use CL = 1 (the same passes, no cluster).
//   stage 0          (CL = 2) in registers across the pair, one cluster barrier
//   pass 0           K1 = LOGM - 8 stages (radix 32 for M = 8192) on o = t + (M/32) i: twiddles uniform per CTA
//   pass 1, pass 2   radix-16 on two groups of 16 per thread, exchanged through padded shared memory
//                    a(o) = o + (o >> 4): conflict-free, every address = thread base + immediate
//   out              16 consecutive outputs per group = one 128-byte line: written as a row of shared memory and
//                    handed to the TMA unit (cp.async.bulk shared -> global, SASS UBLKCP), or (ST_DIRECT) as four
//                    256-bit global stores; measured (tools/lab, limb transforms of a resident batch): N = 16384
//                    0.799 -> 0.773 ms, N = 8192 0.666 -> 0.630 ms, N = 4096 0.627 -> 0.564 ms in favour of TMA
// Twiddles are (w, fl(w/q)) pairs fetched with one 128-bit load from a table ordered for these passes
// (ntt_c_tw_position).  The inverse mirrors the forward (256-bit loads, passes backwards, stage 0 and N^{-1}
// last, stores lane <-> consecutive index).  Arithmetic and lazy bounds are those of ntt.cuh's FP64 classes.
#pragma once
#include "ntt.cuh"
#include <cooperative_groups.h>

// cluster size and pass starts (global stage index) for ring degree 2^logn
__host__ __device__ constexpr int ntt_c_cl(int logn) { return logn >= 14 ? 2 : 1; }
__host__ __device__ constexpr int ntt_c_logm(int logn) { return logn - (ntt_c_cl(logn) == 2 ? 1 : 0); }
__host__ __device__ constexpr int ntt_c_k1(int logn) { return ntt_c_logm(logn) - 8; }
__host__ __device__ constexpr int ntt_c_s0(int logn, int s)
{
    const int sb = ntt_c_cl(logn) == 2 ? 1 : 0, k1 = ntt_c_k1(logn);
    return s < sb ? 0 : (s < sb + k1 ? sb : (s < sb + k1 + 4 ? sb + k1 : sb + k1 + 4));
}
// Host: position of the twiddle pair of stage s, block m (m = b0 2^r + j, r = s - S0(s), b0 = the block index at
// the start of the pass) in the pair table:  2^s + j 2^S0 + b0  (consecutive b0 <-> consecutive lanes)
inline int ntt_c_tw_position(int logn, int s, int m)
{
    const int S0 = ntt_c_s0(logn, s), r = s - S0;
    const int b0 = m >> r, j = m & ((1 << r) - 1);
    return (1 << s) + (j << S0) + b0;
}
__host__ __device__ constexpr bool ntt_c_supported(int logn) { return logn >= 12 && logn <= 14; }

// 256-bit global accesses (sm_100: one full 32-byte sector per thread)
__device__ __forceinline__ void st_global_v4(u64* p, u64 a, u64 b, u64 c, u64 d)
{
    asm volatile("st.global.v4.u64 [%0], {%1, %2, %3, %4};" ::"l"(p), "l"(a), "l"(b), "l"(c), "l"(d) : "memory");
}
__device__ __forceinline__ void ld_global_v4(const u64* p, u64 (&v)[4])
{
    asm volatile("ld.global.v4.u64 {%0, %1, %2, %3}, [%4];" : "=l"(v[0]), "=l"(v[1]), "=l"(v[2]), "=l"(v[3]) : "l"(p));
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

// how the forward writes its outputs (forward_fp<R, ST>)
enum { ST_DIRECT = 0, ST_BULK = 2 };
enum { LD_DIRECT = 0, LD_BULK = 2 };
#ifndef NTTC_LD_DEFAULT
#define NTTC_LD_DEFAULT LD_BULK
#endif
#ifndef NTTC_ST_DEFAULT
#define NTTC_ST_DEFAULT ST_BULK
#endif

// Arithmetic of the forward transform.  ArFp<R>: the FP64 classes of ntt.cuh (exact signed integers in doubles;
// R = PC_FPR, the X input reduced in the first stage of a pass).  ArInt: 64-bit Harvey-lazy Shoup butterflies
// ([0, 4q) values, any q < 2^61) on the integer pipe -- so integer-class limbs run in the same launch and the same
// CTA shape as FP64-class ones, and CTAs of both kinds share an SM (different pipes).
template <bool R>
struct ArFp {
    using V = double;
    using TW = double2;
    double q, qinv;
    __device__ __forceinline__ explicit ArFp(const DPrime& P) : q((double)P.q), qinv(1.0 / (double)P.q) {}
    __device__ __forceinline__ V in(u64 a) const { return u2d(a); }
    __device__ __forceinline__ V in(double v) const { return v; }   // loaders may hand over a signed double
    template <bool FIRST>
    __device__ __forceinline__ void bfly(V& X, V& Y, const TW& w) const
    {
        const double tt = fmodmul(Y, w.x, w.y, q);
        const double xx = (R && FIRST) ? freduce(X, q, qinv) : X;
        X = xx + tt;
        Y = xx - tt;
    }
    __device__ __forceinline__ u64 out(V v) const { return fcanon(v, q, qinv); }
};
struct ArInt {
    using V = u64;
    using TW = ulonglong2;   // (w, floor(w 2^64 / q))
    u64 q, q2;
    __device__ __forceinline__ explicit ArInt(const DPrime& P) : q(P.q), q2(P.q2) {}
    __device__ __forceinline__ V in(u64 a) const { return a; }
    template <bool FIRST>
    __device__ __forceinline__ void bfly(V& X, V& Y, const TW& w) const
    {
        const u64 xx = csub(X, q2);                     // [0, 2q)
        const u64 tt = shoup_mul(Y, w.x, w.y, q);       // [0, 2q) for any Y < 2^64
        X = xx + tt;                                    // [0, 4q)
        Y = xx - tt + q2;
    }
    __device__ __forceinline__ u64 out(V v) const { return csub(csub(v, q2), q); }
};
__device__ __forceinline__ ulonglong2 ldg_pair(const ulonglong2* p) { return __ldg(p); }
__device__ __forceinline__ double2 ldg_pair(const double2* p) { return __ldg(p); }

template <int LOGN_>
struct NttC {
    static constexpr int LOGN = LOGN_;
    static constexpr int N = 1 << LOGN;
    static constexpr int CL = ntt_c_cl(LOGN);        // CTAs per limb
    static constexpr int SB = CL == 2 ? 1 : 0;       // stages done across the cluster
    static constexpr int LOGM = LOGN - SB;
    static constexpr int M = 1 << LOGM;              // points per CTA
    static constexpr int E = 32;
    static constexpr int NT = M / E;                 // threads per CTA
    static constexpr int MPAD = M + M / 16;          // padded region (doubles)
    // forward output staging (ST_BULK): one 128-byte row of 16 outputs per (thread, group), row stride 144 bytes
    // (16-byte aligned for cp.async.bulk; 9 x 16 B, so the 128-bit row writes of 8 lanes hit 8 different banks)
    static constexpr int ROWW = 18;
    static constexpr size_t SMEM_ROWS = (size_t)(M / 16) * ROWW * 8;
    static constexpr size_t SMEM = SMEM_ROWS > (size_t)MPAD * 8 ? SMEM_ROWS : (size_t)MPAD * 8;
    static constexpr size_t SMEM_ALL = SMEM + 16;    // + the inverse's mbarrier (LD_BULK)
    static constexpr int K1 = LOGM - 8;
    static constexpr int MINB = LOGM == 12 ? 4 : 2;  // CTAs per SM the kernels are bounded for (128 registers)
    static_assert(LOGN >= 12 && LOGN <= 14 && K1 >= 4 && K1 <= 5, "supported: N = 4096, 8192, 16384");

    template <int P>
    struct Pass {
        static constexpr int S0 = P == 0 ? 0 : K1 + 4 * (P - 1);   // stage offset inside the CTA's transform
        static constexpr int K = P == 0 ? K1 : 4;
        static constexpr int G = E >> K;
        static constexpr int SH = LOGM - S0 - K;
    };

    __host__ __device__ static constexpr int pad(int o) { return o + (o >> 4); }
    // position (thread part t excluded) of register e in pass 0:  o = t + pos0(e)
    __host__ __device__ static constexpr int pos0(int e) { return ((e & ((1 << K1) - 1)) << 8) + (e >> K1) * NT; }

    // padded thread base of group g in pass P
    template <int P>
    __device__ __forceinline__ static int thread_base(int t, int g)
    {
        using G_ = Pass<P>;
        const int gid = g * NT + t;
        return pad(((gid >> G_::SH) << (G_::SH + G_::K)) + (gid & ((1 << G_::SH) - 1)));
    }
    // twiddle pair index of stage S0 + r of pass P: block (h 2^(S0+r)) + b0 2^r + j
    template <int P>
    __device__ __forceinline__ static int tw_base(int h, int t, int g)
    {
        using G_ = Pass<P>;
        return (h << G_::S0) + ((g * NT + t) >> G_::SH);
    }

    template <int P, class AR>
    __device__ __forceinline__ static void fwd_pass(typename AR::V (&x)[E], int h, int t,
                                                    const typename AR::TW* __restrict__ TW, const AR& ar)
    {
        using G_ = Pass<P>;
        constexpr int K = G_::K, S0g = SB + G_::S0;
#pragma unroll
        for (int g = 0; g < G_::G; ++g) {
            const int b0 = tw_base<P>(h, t, g);
            static_for<0, K>([&](auto rc) {
                constexpr int r = decltype(rc)::value;
                constexpr int half = 1 << (K - 1 - r);
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    if (i & half) continue;
#ifdef KNOCK_TW   /* tools/lab timing experiment only */
                    typename AR::TW w;
                    w.x = (decltype(w.x))(12345 + r + b0);
                    w.y = (decltype(w.y))1;
#else
                    const typename AR::TW w = ldg_pair(TW + ((1 << (S0g + r)) + ((i >> (K - r)) << S0g) + b0));
#endif
                    ar.template bfly<r == 0>(x[g * (1 << K) + i], x[g * (1 << K) + i + half], w);
                }
            });
        }
    }

    template <int P, bool R>
    __device__ __forceinline__ static void inv_pass(double (&x)[E], int h, int t, const double2* __restrict__ TW,
                                                    double q, double qinv)
    {
        using G_ = Pass<P>;
        constexpr int K = G_::K, S0g = SB + G_::S0;
        // pass entry: back to [-q/2, q/2] (the X lineage doubles per stage); FPR reduces every sum instead
        if constexpr (P != 2 && !R) {
#pragma unroll
            for (int i = 0; i < E; ++i) x[i] = freduce(x[i], q, qinv);
        }
#pragma unroll
        for (int g = 0; g < G_::G; ++g) {
            const int b0 = tw_base<P>(h, t, g);
#pragma unroll
            for (int r = K - 1; r >= 0; --r) {
                const int half = 1 << (K - 1 - r);
#pragma unroll
                for (int i = 0; i < (1 << K); ++i) {
                    if (i & half) continue;
                    const double2 w = __ldg(TW + ((1 << (S0g + r)) + ((i >> (K - r)) << S0g) + b0));
                    double& X = x[g * (1 << K) + i];
                    double& Y = x[g * (1 << K) + i + half];
                    const double u = X, v = Y;
                    X = (R && ((LOGN - 1 - (S0g + r)) & 1)) ? freduce(u + v, q, qinv) : u + v;   // as ntt.cuh
                    Y = fmodmul(u - v, w.x, w.y, q);
                }
            }
        }
    }

    // Forward NTT of one limb by the CL CTAs of a cluster (h = this CTA's rank, 0 for CL = 1).
    // ld(idx) -> u64 in [0, 2q), called lane <-> consecutive idx; dst = the output limb (canonical residues),
    // written as ST says.  TW = this prime's forward pair table.
    // Every thread of both CTAs must call it (cluster barriers inside).
    template <bool R, int ST = NTTC_ST_DEFAULT, class Load>
    __device__ __forceinline__ static void forward_fp(u64* sm, int h, const DPrime& Pr, const double2* __restrict__ TW,
                                                      Load&& ld, u64* __restrict__ dst)
    {
        forward<ArFp<R>, ST>(sm, h, ArFp<R>(Pr), TW, ld, dst);
    }
    // the same transform on the integer pipe (any q < 2^61); TW = the (w, w') pair table
    template <int ST = NTTC_ST_DEFAULT, class Load>
    __device__ __forceinline__ static void forward_int(u64* sm, int h, const DPrime& Pr,
                                                       const ulonglong2* __restrict__ TW, Load&& ld,
                                                       u64* __restrict__ dst)
    {
        forward<ArInt, ST>(sm, h, ArInt(Pr), TW, ld, dst);
    }
    template <class AR, int ST, class Load>
    __device__ __forceinline__ static void forward(u64* sm, int h, const AR ar, const typename AR::TW* __restrict__ TW,
                                                   Load&& ld, u64* __restrict__ dst)
    {
        using V = typename AR::V;
        const int t = threadIdx.x;
        V* smd = reinterpret_cast<V*>(sm);
        V x[E];
#ifdef NTTC_DUP   /* tools/lab experiment: no cluster, each CTA loads both halves and does all of stage 0 for its own */
        if constexpr (CL == 2) {
            const typename AR::TW w = ldg_pair(TW + 1);
#pragma unroll
            for (int i = 0; i < E; ++i) {
                V X = ar.in(ld(t + NT * i)), Y = ar.in(ld(t + NT * i + M));
                ar.template bfly<true>(X, Y, w);
                x[i] = h ? Y : X;
            }
        } else
#endif
        if constexpr (CL == 2) {
            // stage 0: this CTA takes the pairs (o, o + M), o = t + NT i, of its half of the i range; X' belongs
            // to rank 0, Y' to rank 1 -- at register i of thread t either way
            cluster_arrive();   // the partner must be running before its shared memory is written
            const int i0 = 16 * h;
            V keep[16], send[16];
            const typename AR::TW w = ldg_pair(TW + 1);
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                keep[k] = ar.in(ld(t + NT * (i0 + k)));
                send[k] = ar.in(ld(t + NT * (i0 + k) + M));
            }
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                V xo = keep[k], yo = send[k];
                ar.template bfly<true>(xo, yo, w);
                keep[k] = h ? yo : xo;
                send[k] = h ? xo : yo;
            }
            cluster_wait();
            V* remote = cooperative_groups::this_cluster().map_shared_rank(smd, h ^ 1);
#pragma unroll
            for (int k = 0; k < 16; ++k) remote[k * NT + t] = send[k];
            cluster_arrive();
            cluster_wait();
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const V got = smd[k * NT + t];
                x[k] = h ? got : keep[k];
                x[16 + k] = h ? keep[k] : got;
            }
            __syncthreads();   // the receive buffer aliases the exchange region
        } else {
#pragma unroll
            for (int i = 0; i < E; ++i) x[i] = ar.in(ld(t + pos0(i)));
        }
        static_for<0, 3>([&](auto pc) {
            constexpr int P = decltype(pc)::value;
            using G_ = Pass<P>;
            constexpr int K = G_::K;
            int T[G_::G];
#pragma unroll
            for (int g = 0; g < G_::G; ++g) {
                T[g] = thread_base<P>(t, g);
                if constexpr (P != 0) {
#pragma unroll
                    for (int i = 0; i < (1 << K); ++i) x[g * (1 << K) + i] = smd[T[g] + pad(i << G_::SH)];
                }
            }
#ifndef KNOCK_FP   /* tools/lab timing experiment only */
            fwd_pass<P, AR>(x, h, t, TW, ar);
#endif
            if constexpr (P != 2) {
#pragma unroll
                for (int g = 0; g < G_::G; ++g)
#pragma unroll
                    for (int i = 0; i < (1 << K); ++i) smd[T[g] + pad(i << G_::SH)] = x[g * (1 << K) + i];
                __syncthreads();
            } else if constexpr (ST == ST_DIRECT) {
                // SH == 0: group g holds the 16 consecutive outputs h M + 16 gid + i; 256-bit stores, one sector each
#pragma unroll
                for (int g = 0; g < G_::G; ++g) {
                    const int base = h * M + ((g * NT + t) << K);
#pragma unroll
                    for (int i = 0; i < (1 << K); i += 4)
                        st_global_v4(dst + base + i, ar.out(x[g * (1 << K) + i]),
                                     ar.out(x[g * (1 << K) + i + 1]), ar.out(x[g * (1 << K) + i + 2]),
                                     ar.out(x[g * (1 << K) + i + 3]));
                }
            } else {
                // ST_BULK: each thread writes its 128-byte output rows into shared memory and hands them to the
                // TMA unit (cp.async.bulk shared -> global): no LSU work per 128-byte line, nothing to wait for but
                // the read of the rows before the CTA exits
                __syncthreads();   // every thread has read its pass-2 operands (the rows alias the exchange region)
#pragma unroll
                for (int g = 0; g < G_::G; ++g) {
                    const int gid = g * NT + t;
                    u64* row = sm + (size_t)gid * ROWW;
#pragma unroll
                    for (int i = 0; i < (1 << K); i += 2)
                        *reinterpret_cast<ulonglong2*>(row + i) =
                            make_ulonglong2(ar.out(x[g * (1 << K) + i]), ar.out(x[g * (1 << K) + i + 1]));
                }
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
#pragma unroll
                for (int g = 0; g < G_::G; ++g) {
                    const int gid = g * NT + t;
                    const u32 srow = (u32)__cvta_generic_to_shared(sm + (size_t)gid * ROWW);
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(dst + h * M + (gid << K)),
                                 "r"(srow)
                                 : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            }
        });
    }

    // Inverse NTT of one limb (includes N^{-1}) by the CL CTAs of a cluster.  src = the input limb (residues < 2q),
    // read as LD says: LD_DIRECT four 256-bit loads per 128-byte row of 16 inputs, LD_BULK one cp.async.bulk
    // global -> shared per row (rows as in the forward's ST_BULK; one mbarrier per CTA, in the 16 bytes after SMEM);
    // st(idx, v) receives canonical residues, called lane <-> consecutive idx.  TW = this prime's inverse pair table.
    template <bool R, int LD = NTTC_LD_DEFAULT, class Store>
    __device__ __forceinline__ static void inverse_fp(u64* sm, int h, const DPrime& Pr, const double2* __restrict__ TW,
                                                      const u64* __restrict__ src, Store&& st)
    {
        const int t = threadIdx.x;
        const double q = (double)Pr.q, qinv = 1.0 / q;
        const double ninv = Pr.ninv > Pr.q / 2 ? -(double)(Pr.q - Pr.ninv) : (double)Pr.ninv, ninvq = ninv / q;
        double* smd = reinterpret_cast<double*>(sm);
        double x[E];
        if constexpr (LD == LD_BULK) {
            const u32 bar = (u32)__cvta_generic_to_shared(reinterpret_cast<char*>(sm) + SMEM);
            if (t == 0) {
                asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
                asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            }
            __syncthreads();
            if (t == 0)
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"((u32)(M * 8)) : "memory");
#pragma unroll
            for (int g = 0; g < E / 16; ++g) {
                const int gid = g * NT + t;
                const u32 srow = (u32)__cvta_generic_to_shared(sm + (size_t)gid * ROWW);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(srow),
                    "l"(src + h * M + (gid << 4)), "r"(bar)
                    : "memory");
            }
            asm volatile(
                "{\n.reg .pred p;\nWAIT_%=:\n"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
                "@p bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}" ::"r"(bar)
                : "memory");
        }
        static_for<0, 3>([&](auto pc) {
            constexpr int P = 2 - decltype(pc)::value;
            using G_ = Pass<P>;
            constexpr int K = G_::K;
            int T[G_::G];
#pragma unroll
            for (int g = 0; g < G_::G; ++g) {
                T[g] = thread_base<P>(t, g);
                if constexpr (P == 2 && LD == LD_DIRECT) {
                    const int base = h * M + ((g * NT + t) << K);
#pragma unroll
                    for (int i = 0; i < (1 << K); i += 4) {
                        u64 v[4];
                        ld_global_v4(src + base + i, v);
#pragma unroll
                        for (int e = 0; e < 4; ++e)
                            x[g * (1 << K) + i + e] = R ? freduce(u2d(v[e]), q, qinv) : u2d(v[e]);
                    }
                } else if constexpr (P == 2) {
                    const u64* row = sm + (size_t)(g * NT + t) * ROWW;
#pragma unroll
                    for (int i = 0; i < (1 << K); i += 2) {
                        const ulonglong2 v = *reinterpret_cast<const ulonglong2*>(row + i);
                        x[g * (1 << K) + i] = R ? freduce(u2d(v.x), q, qinv) : u2d(v.x);
                        x[g * (1 << K) + i + 1] = R ? freduce(u2d(v.y), q, qinv) : u2d(v.y);
                    }
                    if (g == G_::G - 1) __syncthreads();   // the rows alias the exchange region written below
                } else {
#pragma unroll
                    for (int i = 0; i < (1 << K); ++i) x[g * (1 << K) + i] = smd[T[g] + pad(i << G_::SH)];
                }
            }
            if constexpr (P == 0 && CL == 2) {
                // this CTA has read its exchange region for the last time: the partner may now write its stage-0
                // operands there (barrier completes during the pass below)
                __syncthreads();
                cluster_arrive();
            }
            inv_pass<P, R>(x, h, t, TW, q, qinv);
            if constexpr (P != 0) {
#pragma unroll
                for (int g = 0; g < G_::G; ++g)
#pragma unroll
                    for (int i = 0; i < (1 << K); ++i) smd[T[g] + pad(i << G_::SH)] = x[g * (1 << K) + i];
                __syncthreads();
            }
        });
        // x[i] = value at o = t + NT i of this CTA's half
        if constexpr (CL == 2) {
            // stage 0 (Gentleman-Sande): X' = X + Y, Y' = (X - Y) w with X in rank 0's half, Y in rank 1's, same o;
            // rank h does the i in [16 h, 16 h + 16): it needs the partner's registers of that range
            cluster_wait();
            double* remote = cooperative_groups::this_cluster().map_shared_rank(smd, h ^ 1);
#pragma unroll
            for (int k = 0; k < 16; ++k) remote[k * NT + t] = h ? x[k] : x[16 + k];
            cluster_arrive();
            const double2 w = __ldg(TW + 1);
            cluster_wait();
            const int i0 = 16 * h;
#pragma unroll
            for (int k = 0; k < 16; ++k) {
                const double got = smd[k * NT + t];
                double X = h ? got : x[k], Y = h ? x[16 + k] : got;
                if constexpr (!R) { X = freduce(X, q, qinv); Y = freduce(Y, q, qinv); }
                const double s = X + Y, d = fmodmul(X - Y, w.x, w.y, q);
                double r0 = fmodmul(s, ninv, ninvq, q), r1 = fmodmul(d, ninv, ninvq, q);
                r0 = r0 < 0.0 ? r0 + q : r0;
                r1 = r1 < 0.0 ? r1 + q : r1;
                st(t + NT * (i0 + k), d2u(r0));
                st(t + NT * (i0 + k) + M, d2u(r1));
            }
        } else {
#pragma unroll
            for (int i = 0; i < E; ++i) {
                double r = fmodmul(x[i], ninv, ninvq, q);
                r = r < 0.0 ? r + q : r;
                st(t + pos0(i), d2u(r));
            }
        }
    }
};
