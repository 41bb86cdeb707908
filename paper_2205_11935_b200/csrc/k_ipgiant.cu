// k_ipgiant.cu -- sm_100a kernel of the CKKS encrypted-dense-layer hot path: the giant-step
// key-switch inner product of double hoisting (R11c) in the Q_l P basis, accumulated.
// Layouts:
//   ModUp output  [b][digit j][row 0..nl+K-1][N]   (all_e: every row, rows nl.. = special primes)
//   key           [digit j][comp][prime 0..L+K-1][N]
//   accumulator   [b][comp][row 0..nl+K-1][N]   (Q_l P), addend w [b][comp][row][N] (Q_l P)
#include "kinternal.cuh"
#include <cmath>

namespace ck {

// Giant step (R11c):  acc[b][c][i][k] += sum_{j<nd} D_{b,j}[i][k] key_{j,c}[i][k] + [c = 0] sigma_g(w.c0)[i][k].
// Key-stationary form: one thread per (row i, coefficient k) keeps its 2 nl key words in registers
// (split once into 21-bit halves for q < 2^42 rows) and walks the whole batch, so every key word is read
// once per launch (the per-ciphertext-pair CTAs of k_ks_ip_qp re-read the group key B/2 times from L2)
// and the ModUp words stream through with all loads of a ciphertext independent (ILP over b).
// Rows of primes < 2^42: 21-bit split products on IMAD.WIDE.U32 (< 2^42 each, exact 64-bit sums);
// 60-bit rows: 128-bit products.
#define IPG_BLK 128
#ifndef IPG_UNROLL
#define IPG_UNROLL 4
#endif
constexpr int kIpgUnroll = IPG_UNROLL;   // ciphertexts per unrolled batch step
#ifndef IPG_MINB
#define IPG_MINB 4
#endif

template <int NL, bool SPLIT>
__device__ __forceinline__ void ipg_row(const DCtx* __restrict__ dc, const u64* __restrict__ modup,
                                        const u64* __restrict__ key, int nl, u64* __restrict__ acc,
                                        size_t acc_stride, const u64* __restrict__ add, size_t add_stride,
                                        u32 add_galois, int B)
{
    // NL = digits (the contraction length); rows i of Q_l P: q_0..q_{nl-1}, then the special primes
    const int n = dc->n, logn = dc->log_n, ne = nl + dc->n_special, np = dc->n_data + dc->n_special;
    const int i = blockIdx.y, k = blockIdx.x * IPG_BLK + threadIdx.x;
    const int p = ext_prime_of(i, nl, dc->n_data);
    const int krow = p;
    const DPrime Pr = dc->p[p];
    u64 kw[2][NL];
#pragma unroll
    for (int j = 0; j < NL; ++j) {
        kw[0][j] = key[((size_t)(2 * j) * np + krow) * n + k];
        kw[1][j] = key[((size_t)(2 * j + 1) * np + krow) * n + k];
    }
    const int src = add_galois ? galois_src(k, add_galois, logn) : k;
    const size_t dstride = (size_t)ne * n;
    const u64* dbase = modup + (size_t)i * n + k;
    // blockIdx.z = slice of the batch (the grid alone is 2.2 waves of CTAs at N = 16384, 10 rows)
    const int bper = (B + gridDim.z - 1) / gridDim.z;
    const int b_lo = blockIdx.z * bper, b_hi = min(B, b_lo + bper);
#pragma unroll kIpgUnroll
    for (int b = b_lo; b < b_hi; ++b) {
        const u64* d = dbase + (size_t)b * NL * dstride;
        u64 dv[NL];
#pragma unroll
        for (int j = 0; j < NL; ++j) dv[j] = d[(size_t)j * dstride];
        u64* o = acc + (size_t)b * acc_stride + (size_t)i * n + k;
        const u64 a0 = add[(size_t)b * add_stride + (size_t)i * n + src];
        const u64 o0 = o[0], o1 = o[dstride];
        u64 u0, u1;
        if constexpr (SPLIT) {
            u64 s00[2] = {0, 0}, s01[2] = {0, 0}, s11[2] = {0, 0};
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const u32 x1 = (u32)(dv[j] >> 21), x0 = (u32)dv[j] & 0x1FFFFFu;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    const u32 y1 = (u32)(kw[c][j] >> 21), y0 = (u32)kw[c][j] & 0x1FFFFFu;
                    s00[c] += (u64)x0 * y0;
                    s01[c] += (u64)x0 * y1;
                    s01[c] += (u64)x1 * y0;
                    s11[c] += (u64)x1 * y1;
                }
            }
            u64 r[2];
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const u64 mlo = s01[c] << 21, mhi = s01[c] >> 43;
                const u64 slo = s11[c] << 42, shi = s11[c] >> 22;
                const u64 l1 = s00[c] + mlo;
                const u64 l2 = l1 + slo;
                const u64 hi = mhi + shi + (l1 < s00[c] ? 1 : 0) + (l2 < l1 ? 1 : 0);
                r[c] = reduce128(hi, l2, Pr);
            }
            u0 = r[0];
            u1 = r[1];
        } else {
            Acc128 a[2];
            a[0].zero();
            a[1].zero();
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                a[0].mac(dv[j], kw[0][j]);
                a[1].mac(dv[j], kw[1][j]);
            }
            u0 = a[0].reduce(Pr);
            u1 = a[1].reduce(Pr);
        }
        o[0] = addmod(addmod(u0, a0, Pr.q), o0, Pr.q);
        o[dstride] = addmod(u1, o1, Pr.q);
    }
}

template <int NL>
__global__ void __launch_bounds__(IPG_BLK, IPG_MINB)
k_ks_ip_giant(const DCtx* __restrict__ dc, const u64* __restrict__ modup, const u64* __restrict__ key, int nl,
              u64* __restrict__ acc, size_t acc_stride, const u64* __restrict__ add, size_t add_stride,
              u32 add_galois, int B)
{
    const int i = blockIdx.y;
    const u64 q = dc->p[ext_prime_of(i, nl, dc->n_data)].q;
    if (q < SPLIT21_MAXQ)
        ipg_row<NL, true>(dc, modup, key, nl, acc, acc_stride, add, add_stride, add_galois, B);
    else
        ipg_row<NL, false>(dc, modup, key, nl, acc, acc_stride, add, add_stride, add_galois, B);
}

static int g_giant_multi = [] {
    const char* e = getenv("CKKS_GIANT_MULTI");
    return e ? atoi(e) : 1;
}();
void set_giant_multi(int on) { g_giant_multi = on; }
int get_giant_multi() { return g_giant_multi; }

// All giant steps of a layer in one pass over the accumulator (R11c):
//   acc[b][c][i][k] += sum_{g < G} ( sum_{j<nd} D^{(g)}_{b,j}[i][k] key^{(g)}_{j,c}[i][k] + [c = 0] sigma_g(w_g.c0)[i][k] )
// where step g has its own ModUp words (its own digits), key, addend ciphertexts w_g and Galois element.  A CTA owns
// 128 coefficients of one row: the key words of all G steps sit in shared memory ([g][c][j][128], pre-split into
// 21-bit halves for q < 2^42 rows), each thread walks a slice of the batch, and for one ciphertext it sums the split
// products of ALL steps before one recombination and one reduction (35 products of < 2^42 per partial sum: < 2^48;
// 60-bit rows: 128-bit accumulators, 35 products of < 2^120), so the accumulator crosses HBM once per layer instead
// of once per step (dense1: 15.5 GB instead of 23.5 GB for 7 steps) and the modular reductions drop 7-fold.
struct GiantSteps {
    int G;
    const u64* modup[KS_GMAX];
    const u64* key[KS_GMAX];
    const u64* add[KS_GMAX];
    u32 galois[KS_GMAX];
};

template <int NL, bool SPLIT>
__device__ __forceinline__ void ipgm_row(const DCtx* __restrict__ dc, const GiantSteps& gs, int nl, u64* __restrict__ acc,
                                         size_t acc_stride, size_t add_stride, int B, u64* __restrict__ Ks)
{
    const int n = dc->n, logn = dc->log_n, ne = nl + dc->n_special, np = dc->n_data + dc->n_special;
    const int i = blockIdx.y, k = blockIdx.x * IPG_BLK + threadIdx.x, tid = threadIdx.x;
    const int p = ext_prime_of(i, nl, dc->n_data);
    const DPrime Pr = dc->p[p];
    const size_t dstride = (size_t)ne * n;
    const int G = gs.G;
    // key words of every step -> shared memory (this thread's own column: no synchronisation needed)
    for (int g = 0; g < G; ++g)
#pragma unroll
        for (int c = 0; c < 2; ++c)
#pragma unroll
            for (int j = 0; j < NL; ++j) {
                const u64 w = gs.key[g][((size_t)(2 * j + c) * np + p) * n + k];
                // split rows: (y1 + y0) | y1 | y0 in 22 + 21 + 21 bits of one word (Karatsuba: 3 products per MAC)
                const u64 y1 = w >> 21, y0 = w & 0x1FFFFFu;
                Ks[((g * 2 + c) * NL + j) * IPG_BLK + tid] = SPLIT ? (((y1 + y0) << 42) | (y1 << 21) | y0) : w;
            }
    int src[KS_GMAX];
#pragma unroll
    for (int g = 0; g < KS_GMAX; ++g) src[g] = g < G ? galois_src(k, gs.galois[g], logn) : 0;
    const int bper = (B + gridDim.z - 1) / gridDim.z;
    const int b_lo = blockIdx.z * bper, b_hi = min(B, b_lo + bper);
#pragma unroll 1
    for (int b = b_lo; b < b_hi; ++b) {
        u64* o = acc + (size_t)b * acc_stride + (size_t)i * n + k;
        const u64 o0 = o[0], o1 = o[dstride];
        u64 adds = 0;                                          // sum of the addends: < 8 q < 2^64
        u64 s00[2] = {0, 0}, s01[2] = {0, 0}, s11[2] = {0, 0};
        Acc128 a[2];
        a[0].zero();
        a[1].zero();
#pragma unroll
        for (int g = 0; g < KS_GMAX; ++g) {
            if (g < G) {
                const u64* d = gs.modup[g] + (size_t)i * n + k + (size_t)b * NL * dstride;
                u64 dv[NL];
#pragma unroll
                for (int j = 0; j < NL; ++j) dv[j] = d[(size_t)j * dstride];
                adds += gs.add[g][(size_t)b * add_stride + (size_t)i * n + src[g]];
#pragma unroll
                for (int j = 0; j < NL; ++j) {
#pragma unroll
                    for (int c = 0; c < 2; ++c) {
                        const u64 w = Ks[((g * 2 + c) * NL + j) * IPG_BLK + tid];
                        if constexpr (SPLIT) {
                            const u32 x1 = (u32)(dv[j] >> 21), x0 = (u32)dv[j] & 0x1FFFFFu;
                            const u32 y0 = (u32)w & 0x1FFFFFu, y1 = (u32)(w >> 21) & 0x1FFFFFu, ys = (u32)(w >> 42);
                            s00[c] += (u64)x0 * y0;
                            s01[c] += (u64)(x0 + x1) * ys;      // (x0 + x1)(y0 + y1) < 2^44: 40 terms < 2^50
                            s11[c] += (u64)x1 * y1;
                        } else {
                            a[c].mac(dv[j], w);
                        }
                    }
                }
            }
        }
        u64 r[2];
        if constexpr (SPLIT) {
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const u64 mid = s01[c] - s00[c] - s11[c];      // x0 y1 + x1 y0 summed
                const u64 mlo = mid << 21, mhi = mid >> 43;
                const u64 slo = s11[c] << 42, shi = s11[c] >> 22;
                const u64 l1 = s00[c] + mlo;
                const u64 l2 = l1 + slo;
                const u64 hi = mhi + shi + (l1 < s00[c] ? 1 : 0) + (l2 < l1 ? 1 : 0);
                r[c] = reduce128(hi, l2, Pr);
            }
        } else {
            r[0] = a[0].reduce(Pr);
            r[1] = a[1].reduce(Pr);
        }
        o[0] = addmod(addmod(r[0], reduce64(adds, Pr), Pr.q), o0, Pr.q);
        o[dstride] = addmod(r[1], o1, Pr.q);
    }
}

template <int NL>
__global__ void __launch_bounds__(IPG_BLK, 5)
k_ks_ip_giant_multi(const DCtx* __restrict__ dc, const GiantSteps gs, int nl, u64* __restrict__ acc, size_t acc_stride,
                    size_t add_stride, int B)
{
    extern __shared__ u64 ipgm_keys[];
    const u64 q = dc->p[ext_prime_of(blockIdx.y, nl, dc->n_data)].q;
    if (q < SPLIT21_MAXQ) ipgm_row<NL, true>(dc, gs, nl, acc, acc_stride, add_stride, B, ipgm_keys);
    else ipgm_row<NL, false>(dc, gs, nl, acc, acc_stride, add_stride, B, ipgm_keys);
}

bool ip_giant_multi(const Launch& L, int G, const uint64_t* const* modup, const uint64_t* const* key,
                    const uint64_t* const* add, const uint32_t* galois, int batch, int nl, uint64_t* acc,
                    size_t acc_stride, size_t add_stride)
{
    const int n = 1 << L.log_n, nd = L.active_digits(nl);
    if (G < 1 || G > KS_GMAX || nd > 5 || n % IPG_BLK) return false;
    GiantSteps gs;
    gs.G = G;
    for (int g = 0; g < G; ++g) {
        gs.modup[g] = modup[g];
        gs.key[g] = key[g];
        gs.add[g] = add[g];
        gs.galois[g] = galois[g];
    }
    // batch slices in grid.z: enough CTAs for 8+ waves at 3 CTAs per SM, at least 8 ciphertexts per slice
    int split = 1;
    while (split < 16 && batch / (2 * split) >= 8 && (long)(n / IPG_BLK) * (nl + L.n_special) * split < 8L * 5 * 148)
        split *= 2;
    const dim3 grid(n / IPG_BLK, nl + L.n_special, split);
    const size_t smem = (size_t)G * 2 * nd * IPG_BLK * sizeof(u64);
#define IPGM_CASE(V)                                                                                                  \
    case V: {                                                                                                         \
        allow_smem(k_ks_ip_giant_multi<V>, smem);                                                                     \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_giant");                                                               \
        k_ks_ip_giant_multi<V><<<grid, IPG_BLK, smem, L.st>>>(L.dc, gs, nl, acc, acc_stride, add_stride, batch);      \
    } break;
    switch (nd) {
        IPGM_CASE(1) IPGM_CASE(2) IPGM_CASE(3) IPGM_CASE(4) IPGM_CASE(5)
    default: return false;
    }
#undef IPGM_CASE
    check_launch("ip_giant_multi");
    if (L.counter) *L.counter += 1;
    return true;
}

void ip_giant(const Launch& L, const uint64_t* key, int batch, int nl, const KsWork& w, uint64_t* acc,
              size_t acc_stride, const uint64_t* add, size_t add_stride, uint32_t add_galois)
{
    const int n = 1 << L.log_n;
    if (n % IPG_BLK) throw std::runtime_error("N >= 128 required");
    // batch slices: the split (1, 2, 4 or 8, at least 16 ciphertexts each) whose CTA count fills its last wave best
    static const int slots = [] {
        int dev = 0, sms = 148;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        return sms * IPG_MINB;
    }();
    int split = 1;
    double best = 0.0;
    for (int sp = 1; sp <= 8 && batch / sp >= 16; sp *= 2) {
        const double waves = (double)(n / IPG_BLK) * (nl + L.n_special) * sp / slots;
        const double eff = waves / std::ceil(waves);
        if (eff > best + 0.02) {
            best = eff;
            split = sp;
        }
    }
    const dim3 grid(n / IPG_BLK, nl + L.n_special, split);
#define IPG_CASE(V)                                                                                                  \
    case V: {                                                                                                         \
        ProbeScope ps_(L.probe, L.st, "k_ks_ip_giant");                                                               \
        k_ks_ip_giant<V><<<grid, IPG_BLK, 0, L.st>>>(L.dc, w.modup, key, nl, acc, acc_stride, add, add_stride,        \
                                                     add_galois, batch);                                              \
    } break;
    switch (L.active_digits(nl)) {
        IPG_CASE(1) IPG_CASE(2) IPG_CASE(3) IPG_CASE(4) IPG_CASE(5) IPG_CASE(6) IPG_CASE(7) IPG_CASE(8)
        IPG_CASE(9) IPG_CASE(10) IPG_CASE(11) IPG_CASE(12) IPG_CASE(13) IPG_CASE(14) IPG_CASE(15) IPG_CASE(16)
    default: throw std::runtime_error("more than 16 digits");
    }
#undef IPG_CASE
    check_launch("ip_giant");
    if (L.counter) *L.counter += 1;
}

}  // namespace ck
