// kernels.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path.
//
// Every operation of SURVEY 8(a) rows a2-a12 is one of these kernels; the host side (api.cu)
// only sequences launches and tracks level/scale.  Modular arithmetic runs on the integer pipes
// (64-bit Shoup/Barrett), on the FP64 pipe (exact error-free products for q < 2^45), and -- for the
// two small modular contractions (key-switch inner product, BSGS inner sums) -- on the FP64 tensor
// cores with exactly split operands.  Layouts:
//   ciphertext  [batch][comp][limb][N]  u64, NTT domain, canonical residues in [0, q)
//   key         [digit j][comp][prime 0..L+K-1][N]  (primes L.. = the special primes P_k)
//   plaintexts  [t][limb][N]
// This unit: batched NTT, rescale, elementwise ops, decrypt, samplers and keygen.
#include "kinternal.cuh"

namespace ck {

// ------------------------------------------------------------------------------------ NTT batch
template <int LOGN, bool INV, int NTH>
__global__ void __launch_bounds__(NTH)
k_ntt_batch(const DCtx* __restrict__ dc, u64* __restrict__ data, int limbs, int prime0)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NTH>;
    const int l = blockIdx.x, b = blockIdx.y, p = prime0 + l;
    u64* a = data + ((size_t)b * limbs + l) * T::N;
    const DPrime Pr = dc->p[p];
    auto ld = [&](int i) { return a[i]; };
    auto st = [&](int i, u64 v) { a[i] = v; };
    if constexpr (INV) ntt_inverse<T>(sm, Pr, twp(dc, p), ld, st);
    else ntt_forward<T>(sm, Pr, twp(dc, p), ld, st);
}

// CTA-pair schedule (ntt_c.cuh) for FP64-class limbs: grid (limbs * CL, batch) in clusters of CL CTAs; IO = ST_BULK /
// LD_BULK (TMA rows) or ST_DIRECT / LD_DIRECT (256-bit accesses)
template <int LOGN, bool INV, int IO>
__global__ void __launch_bounds__(NttC<LOGN>::NT, NttC<LOGN>::MINB)
k_ntt_batch_c(const DCtx* __restrict__ dc, u64* __restrict__ data, int limbs, int prime0)
{
    extern __shared__ u64 sm[];
    using TC = NttC<LOGN>;
    const int l = blockIdx.x / TC::CL, h = blockIdx.x % TC::CL, b = blockIdx.y, p = prime0 + l;
    u64* a = data + ((size_t)b * limbs + l) * TC::N;
    const DPrime Pr = dc->p[p];
    const int pc = prime_class(Pr.q);
    const bool r = pc == PC_FPR;
    if constexpr (INV) {
        auto st = [&](int i, u64 v) { a[i] = v; };
        if (r) TC::template inverse_fp<true, IO>(sm, h, Pr, twq_inv(dc, p), a, st);
        else TC::template inverse_fp<false, IO>(sm, h, Pr, twq_inv(dc, p), a, st);
    } else {
        auto ld = [&](int i) { return a[i]; };
        if (r) TC::template forward_fp<true, IO>(sm, h, Pr, twq_fwd(dc, p), ld, a);
        else if (pc == PC_FP) TC::template forward_fp<false, IO>(sm, h, Pr, twq_fwd(dc, p), ld, a);
        else TC::template forward_int<IO>(sm, h, Pr, twq_fwd_int(dc, p), ld, a);   // integer-class limb, same launch
    }
}

static int g_nvtx = [] {
    const char* e = getenv("CKKS_NVTX");
    return e ? atoi(e) : 0;
}();
int nvtx_on() { return g_nvtx; }
void set_nvtx(int on) { g_nvtx = on; }

static int g_ntt_q = [] {
    const char* e = getenv("CKKS_NTT_Q");
    return e ? atoi(e) : (int)NTTQ_DEFAULT;
}();
void set_ntt_q(int mask) { g_ntt_q = mask; }
int get_ntt_q() { return g_ntt_q; }

template <int LG, bool INV, int NTH>
static void ntt_batch_run(const Launch& L, uint64_t* data, int batch, int limbs, int l0, int l1, int prime0, bool fp)
{
    // limbs [l0, l1) of every [limbs][N] block: the kernels take the block stride from `limbs`, so the run is
    // addressed by offsetting the base pointer and prime0 and keeping gridDim.x = l1 - l0
    uint64_t* base = data + ((size_t)l0 << LG);
    if constexpr (LG >= 12) {
        if (fp) {
            using TC = NttC<LG>;
            // TMA row copies (UBLKCP) for the forward's outputs at every N and for the inverse's inputs at
            // N <= 8192 (cfg2 inverse at N = 16384: 1.059 ms with the bulk loads vs 1.028 ms with 256-bit loads;
            // N = 8192: 0.129 vs 0.134 ms; forward 0.521 vs 0.530 ms at N = 16384, 0.115 vs 0.121 ms at N = 8192)
            const bool direct = (g_ntt_q & NTTQ_DIRECT_IO) || (INV && LG == 14);
            auto k = direct ? k_ntt_batch_c<LG, INV, ST_DIRECT> : k_ntt_batch_c<LG, INV, ST_BULK>;
            allow_smem(k, TC::SMEM_ALL);
            launch_cluster(k, dim3((l1 - l0) * TC::CL, batch), TC::NT, TC::SMEM_ALL, L.st, TC::CL, L.dc, base, limbs,
                           prime0 + l0);
            return;
        }
    }
    auto k = k_ntt_batch<LG, INV, NTH>;
    allow_smem(k, sizeof(u64) << LG);
    k<<<dim3(l1 - l0, batch), NTH, sizeof(u64) << LG, L.st>>>(L.dc, base, limbs, prime0 + l0);
}

void ntt_batch(const Launch& L, uint64_t* data, int batch, int limbs, int prime0, bool inverse)
{
    if (batch <= 0 || limbs <= 0) return;
    const double bytes = 2.0 * batch * limbs * (double)(8 << L.log_n);   // read + write each limb once
    const bool pr = L.probe && L.probe->on(PROBE_NTT);
    if (L.probe && L.probe->on(PROBE_ALL)) L.probe->bytes_by_kernel["k_ntt_batch"] += bytes;
    if (pr) {
        L.probe->mark(L.st);
        L.probe->alg_bytes += bytes;
    }
    NTT_DISPATCH(L.log_n, {
        ProbeScope ps_(L.probe, L.st, "k_ntt_batch");
        // threads per CTA of the whole-limb kernel: 16 residues per thread (NT0), or 32 (NW): CKKS_NTT_WIDE bit 16
        // (forward, default on: cfg2 1.10 -> 1.04 ms) and bit 32 (inverse, default off: 1.27 vs 1.39 ms)
        constexpr int NT0 = NttThreads<LG>::value, NW = NttThreadsWide<LG>::value;
        const bool wide = (ntt_wide_mask() & (inverse ? 32 : 16)) != 0;
        const bool cl = ntt_c_supported(LG) && (g_ntt_q & (inverse ? NTTQ_BATCH_INV : NTTQ_BATCH_FWD)) != 0;
        // maximal runs of limbs of one kind: FP64-class limbs on the CTA-pair schedule (when selected), the rest
        // (and everything when it is off) on the whole-limb kernel
        for (int l0 = 0; l0 < limbs;) {
            // (the forward handles every class on the cluster schedule; the inverse only the FP64 classes)
            auto is_fp = [&](int l) {
                const int c = L.pclass[prime0 + l];
                return cl && (!inverse || c == PC_FP || c == PC_FPR);
            };
            const bool fp = is_fp(l0);
            int l1 = l0 + 1;
            while (l1 < limbs && is_fp(l1) == fp) ++l1;
            if (inverse) {
                if (wide) ntt_batch_run<LG, true, NW>(L, data, batch, limbs, l0, l1, prime0, fp);
                else ntt_batch_run<LG, true, NT0>(L, data, batch, limbs, l0, l1, prime0, fp);
            } else {
                if (wide) ntt_batch_run<LG, false, NW>(L, data, batch, limbs, l0, l1, prime0, fp);
                else ntt_batch_run<LG, false, NT0>(L, data, batch, limbs, l0, l1, prime0, fp);
            }
            if (L.counter) ++*L.counter;
            l0 = l1;
        }
    });
    if (pr) L.probe->mark(L.st);
    check_launch("ntt_batch");
}

// ------------------------------------------------------------------------------------ rescale
template <int LOGN>
__global__ void __launch_bounds__(NttThreads<LOGN>::value)
k_rescale_intt(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t in_stride, int ncomp, int nl,
               u64* __restrict__ rem)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NttThreads<LOGN>::value>;
    const int c = blockIdx.x, b = blockIdx.y, l = nl - 1;
    const u64* src = in + (size_t)b * in_stride + ((size_t)c * nl + l) * T::N;
    u64* dst = rem + ((size_t)b * ncomp + c) * T::N;
    const DPrime Pr = dc->p[l];
    auto ld = [&](int i) { return src[i]; };
    auto st = [&](int i, u64 v) { dst[i] = v; };
    ntt_inverse<T>(sm, Pr, twp(dc, l), ld, st);
}

template <int LOGN>
__global__ void __launch_bounds__(NttThreads<LOGN>::value)
k_rescale_out(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t in_stride, int ncomp, int nl,
              const u64* __restrict__ rem, u64* __restrict__ out, size_t out_stride, const u64* __restrict__ bias)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NttThreads<LOGN>::value>;
    const int i = blockIdx.x, c = blockIdx.y, b = blockIdx.z, l = nl - 1;
    const DPrime Pr = dc->p[i];
    const u64 qlmod = dc->qmod[l][i];
    const u64 qlinv = dc->qinv[l][i], qlinv_sh = dc->qinv_sh[l][i];
    const u64 ql = dc->p[l].q;
    const u64* r = rem + ((size_t)b * ncomp + c) * T::N;
    const u64* a = in + (size_t)b * in_stride + ((size_t)c * nl + i) * T::N;
    u64* o = out + (size_t)b * out_stride + ((size_t)c * (nl - 1) + i) * T::N;
    const u64* bi = (bias && c == 0) ? bias + (size_t)i * T::N : nullptr;
    auto ld = [&](int k) { return centered_to(r[k], ql, qlmod, Pr); };
    auto st = [&](int k, u64 v) {
        u64 x = csub(shoup_mul(a[k] + Pr.q - v, qlinv, qlinv_sh, Pr.q), Pr.q);
        if (bi) x = addmod(x, bi[k], Pr.q);
        o[k] = x;
    };
    ntt_forward<T>(sm, Pr, twp(dc, i), ld, st);
}

void rescale(const Launch& L, const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, int batch,
             int ncomp, int nl, uint64_t* rem, const uint64_t* bias)
{
    if (batch <= 0) return;
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        allow_smem(k_rescale_intt<LG>, smem);
        allow_smem(k_rescale_out<LG>, smem);
        { ProbeScope ps_(L.probe, L.st, "k_rescale_intt"); k_rescale_intt<LG><<<dim3(ncomp, batch), NT, smem, L.st>>>(L.dc, in, in_stride, ncomp, nl, rem); }
        { ProbeScope ps_(L.probe, L.st, "k_rescale_out"); k_rescale_out<LG><<<dim3(nl - 1, ncomp, batch), NT, smem, L.st>>>(L.dc, in, in_stride, ncomp, nl, rem, out,
                                                                         out_stride, bias); }
    });
    check_launch("rescale");
    if (L.counter) *L.counter += 2;
}

// ------------------------------------------------------------------------------------ elementwise
__global__ void __launch_bounds__(256)
k_tensor(const DCtx* __restrict__ dc, const u64* __restrict__ a, const u64* __restrict__ bb, size_t stride,
         u64* __restrict__ out, size_t out_stride, int nl)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, l = blockIdx.y, b = blockIdx.z;
    const DPrime Pr = dc->p[l];
    const u64* A = a + (size_t)b * stride;
    const u64* B = bb + (size_t)b * stride;
    const size_t i0 = (size_t)l * n + k, i1 = ((size_t)nl + l) * n + k;
    const u64 a0 = A[i0], a1 = A[i1], b0 = B[i0], b1 = B[i1];
    u64* O = out + (size_t)b * out_stride;
    O[i0] = mulmod(a0, b0, Pr);
    Acc128 m;
    m.zero();
    m.mac(a0, b1);
    m.mac(a1, b0);
    O[i1] = m.reduce(Pr);
    O[((size_t)2 * nl + l) * n + k] = mulmod(a1, b1, Pr);
}

void tensor(const Launch& L, const uint64_t* a, const uint64_t* b, size_t stride, uint64_t* out3, size_t out_stride,
            int batch, int nl)
{
    if (batch <= 0) return;
    const int n = 1 << L.log_n;
    { ProbeScope ps_(L.probe, L.st, "k_tensor"); k_tensor<<<dim3(n / 256, nl, batch), 256, 0, L.st>>>(L.dc, a, b, stride, out3, out_stride, nl); }
    check_launch("tensor");
    if (L.counter) ++*L.counter;
}

__global__ void __launch_bounds__(256)
k_add(const DCtx* __restrict__ dc, const u64* __restrict__ a, size_t sa, const u64* __restrict__ bb, size_t sb,
      u64* __restrict__ out, size_t so, int nl)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, cl = blockIdx.y, b = blockIdx.z;
    const int l = cl % nl;
    const u64 q = dc->p[l].q;
    const size_t off = (size_t)cl * n + k;
    out[(size_t)b * so + off] = addmod(a[(size_t)b * sa + off], bb[(size_t)b * sb + off], q);
}

void add(const Launch& L, const uint64_t* a, size_t sa, const uint64_t* b, size_t sb, uint64_t* out, size_t so,
         int batch, int ncomp, int nl)
{
    if (batch <= 0) return;
    const int n = 1 << L.log_n;
    { ProbeScope ps_(L.probe, L.st, "k_add"); k_add<<<dim3(n / 256, ncomp * nl, batch), 256, 0, L.st>>>(L.dc, a, sa, b, sb, out, so, nl); }
    check_launch("add");
    if (L.counter) ++*L.counter;
}

// ------------------------------------------------------------------------------------ decrypt
template <int LOGN>
__global__ void __launch_bounds__(NttThreads<LOGN>::value)
k_decrypt(const DCtx* __restrict__ dc, const u64* __restrict__ ct, size_t ct_stride, const u64* __restrict__ s_ntt,
          u64* __restrict__ out, int nl)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NttThreads<LOGN>::value>;
    const int l = blockIdx.x, b = blockIdx.y;
    const DPrime Pr = dc->p[l];
    const u64* c0 = ct + (size_t)b * ct_stride + (size_t)l * T::N;
    const u64* c1 = ct + (size_t)b * ct_stride + ((size_t)nl + l) * T::N;
    const u64* s = s_ntt + (size_t)l * T::N;
    u64* o = out + ((size_t)b * nl + l) * T::N;
    auto ld = [&](int i) { return addmod(c0[i], mulmod(c1[i], s[i], Pr), Pr.q); };
    auto st = [&](int i, u64 v) { o[i] = v; };
    ntt_inverse<T>(sm, Pr, twp(dc, l), ld, st);
}

void decrypt(const Launch& L, const uint64_t* ct, size_t ct_stride, const uint64_t* s_ntt, uint64_t* out, int batch,
             int nl)
{
    if (batch <= 0) return;
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        allow_smem(k_decrypt<LG>, smem);
        k_decrypt<LG><<<dim3(nl, batch), NT, smem, L.st>>>(L.dc, ct, ct_stride, s_ntt, out, nl);
    });
    check_launch("decrypt");
    if (L.counter) ++*L.counter;
}

// ------------------------------------------------------------------------------------ signed -> NTT
template <int LOGN>
__global__ void __launch_bounds__(NttThreads<LOGN>::value)
k_signed_to_ntt(const DCtx* __restrict__ dc, const long long* __restrict__ coeffs, u64* __restrict__ out, int nl,
                int nlimbs)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NttThreads<LOGN>::value>;
    const int l = blockIdx.x, y = blockIdx.y;
    const int p = ext_prime_of(l, nl, dc->n_data);   // limbs nl..: the special primes
    const DPrime Pr = dc->p[p];
    const long long* src = coeffs + (size_t)y * T::N;
    u64* o = out + ((size_t)y * nlimbs + l) * T::N;
    auto ld = [&](int i) { return signed_to_res(src[i], Pr); };
    auto st = [&](int i, u64 v) { o[i] = v; };
    ntt_forward<T>(sm, Pr, twp(dc, p), ld, st);
}

void signed_to_ntt(const Launch& L, const int64_t* coeffs, uint64_t* out, int count, int nl, bool with_special)
{
    const int nlimbs = nl + (with_special ? L.n_special : 0);
    if (count <= 0) return;
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        allow_smem(k_signed_to_ntt<LG>, smem);
        k_signed_to_ntt<LG><<<dim3(nlimbs, count), NT, smem, L.st>>>(L.dc, (const long long*)coeffs, out, nl, nlimbs);
    });
    check_launch("signed_to_ntt");
    if (L.counter) ++*L.counter;
}

// ------------------------------------------------------------------------------------ samplers / keygen
template <int LOGN>
__global__ void __launch_bounds__(NttThreads<LOGN>::value)
k_sample_ntt(const DCtx* __restrict__ dc, u64* __restrict__ out, int nlimbs, int nl_data, int kind, u64 seed,
             u64 purpose, u64 id0, u64 id_step, u64 digit0, u64 digit_step)
{
    extern __shared__ u64 sm[];
    using T = NttCta<LOGN, NttThreads<LOGN>::value>;
    const int limb = blockIdx.x, y = blockIdx.y;
    const int p = ext_prime_of(limb, nl_data, dc->n_data);
    const DPrime Pr = dc->p[p];
    const u64 stream = stream_tag(purpose, id0 + (u64)y * id_step, digit0 + (u64)y * digit_step, 0);
    u64* o = out + ((size_t)y * nlimbs + limb) * T::N;
    auto ld = [&](int i) { return signed_to_res(sample_small(dc, kind, seed, stream, (u64)i), Pr); };
    auto st = [&](int i, u64 v) { o[i] = v; };
    ntt_forward<T>(sm, Pr, twp(dc, p), ld, st);
}

void sample_ntt(const Launch& L, uint64_t* out, int ny, int nlimbs, int nl_data, int kind, uint64_t seed,
                uint64_t purpose, uint64_t id0, uint64_t id_step, uint64_t digit0, uint64_t digit_step)
{
    const size_t smem = sizeof(u64) << L.log_n;
    NTT_DISPATCH(L.log_n, {
        constexpr int NT = NttThreads<LG>::value;
        allow_smem(k_sample_ntt<LG>, smem);
        k_sample_ntt<LG><<<dim3(nlimbs, ny), NT, smem, L.st>>>(L.dc, out, nlimbs, nl_data, kind, seed, purpose, id0,
                                                               id_step, digit0, digit_step);
    });
    check_launch("sample_ntt");
    if (L.counter) ++*L.counter;
}

__global__ void k_sample_uniform(const DCtx* __restrict__ dc, u64* __restrict__ out, int prime, u64 seed, u64 stream)
{
    const int i = blockIdx.x * 256 + threadIdx.x;
    const DPrime Pr = dc->p[prime];
    const u64 hi = prng(seed, stream, 2 * (u64)i), lo = prng(seed, stream, 2 * (u64)i + 1);
    out[i] = reduce128(hi, lo, Pr);   // (hi 2^64 + lo) mod q, exactly (R15)
}

void sample_uniform(const Launch& L, uint64_t* out, int prime, uint64_t seed, uint64_t purpose, uint64_t id,
                    uint64_t digit)
{
    const int n = 1 << L.log_n;
    // stream tag computed on the host side identically
    const uint64_t stream = (purpose << 56) | ((id & 0xFFFFFFFFFULL) << 20) | ((digit & 0x3FF) << 10) |
                            ((uint64_t)prime & 0x3FF);
    k_sample_uniform<<<n / 256, 256, 0, L.st>>>(L.dc, out, prime, seed, stream);
    check_launch("sample_uniform");
    if (L.counter) ++*L.counter;
}

// key[j][1][p] already holds a_j[p]; e_ntt[j][p][N]; s_ntt[p][N]; sprime[p][N]; np = L + K primes:
//   key[j][0][p] = -a s + e + [p in digit j] (P mod p) s'      (R5, R17b; P = prod of the special primes)
__global__ void k_ks_key_combine(const DCtx* __restrict__ dc, u64* __restrict__ key, const u64* __restrict__ e_ntt,
                                 const u64* __restrict__ s_ntt, const u64* __restrict__ sprime, int np)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, p = blockIdx.y, j = blockIdx.z;
    const DPrime Pr = dc->p[p];
    const size_t row1 = (((size_t)j * 2 + 1) * np + p) * n + k;
    const size_t row0 = (((size_t)j * 2 + 0) * np + p) * n + k;
    const u64 a = key[row1];
    const u64 s = s_ntt[(size_t)p * n + k];
    u64 v = submod(e_ntt[((size_t)j * np + p) * n + k], mulmod(a, s, Pr), Pr.q);
    if (p < dc->n_data && p >= dc->dig_start[j] && p < dc->dig_start[j] + dc->dig_len[j])
        v = addmod(v, mulmod(dc->pmod[p], sprime[(size_t)p * n + k], Pr), Pr.q);   // gadget P mod q_p
    key[row0] = v;
}

void keyswitch_key_combine(const Launch& L, uint64_t* key, const uint64_t* e_ntt, const uint64_t* s_ntt,
                           const uint64_t* sprime, int Ld)
{
    const int n = 1 << L.log_n;
    const int np = Ld + L.n_special;
    k_ks_key_combine<<<dim3(n / 256, np, L.n_digits), 256, 0, L.st>>>(L.dc, key, e_ntt, s_ntt, sprime, np);
    check_launch("ks_key_combine");
    if (L.counter) ++*L.counter;
}

// pk[0][p] = -a s + e ; pk[1][p] = a (already written)
__global__ void k_pk_combine(const DCtx* __restrict__ dc, u64* __restrict__ pk, const u64* __restrict__ e_ntt,
                             const u64* __restrict__ s_ntt, int L)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, p = blockIdx.y;
    const DPrime Pr = dc->p[p];
    const u64 a = pk[((size_t)L + p) * n + k];
    pk[(size_t)p * n + k] = submod(e_ntt[(size_t)p * n + k], mulmod(a, s_ntt[(size_t)p * n + k], Pr), Pr.q);
}

void pk_combine(const Launch& L, uint64_t* pk, const uint64_t* e_ntt, const uint64_t* s_ntt, int Ld)
{
    const int n = 1 << L.log_n;
    k_pk_combine<<<dim3(n / 256, Ld), 256, 0, L.st>>>(L.dc, pk, e_ntt, s_ntt, Ld);
    check_launch("pk_combine");
    if (L.counter) ++*L.counter;
}

__global__ void k_square_ntt(const DCtx* __restrict__ dc, const u64* __restrict__ s, u64* __restrict__ out)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, p = blockIdx.y;
    const u64 v = s[(size_t)p * n + k];
    out[(size_t)p * n + k] = mulmod(v, v, dc->p[p]);
}
void square_ntt(const Launch& L, const uint64_t* s, uint64_t* out, int np)
{
    const int n = 1 << L.log_n;
    k_square_ntt<<<dim3(n / 256, np), 256, 0, L.st>>>(L.dc, s, out);
    check_launch("square_ntt");
    if (L.counter) ++*L.counter;
}

__global__ void k_galois_ntt(const DCtx* __restrict__ dc, const u64* __restrict__ s, u64* __restrict__ out, u32 g)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, p = blockIdx.y;
    out[(size_t)p * n + k] = s[(size_t)p * n + galois_src(k, g, dc->log_n)];
}
void galois_ntt(const Launch& L, const uint64_t* s, uint64_t* out, int np, uint32_t g)
{
    const int n = 1 << L.log_n;
    k_galois_ntt<<<dim3(n / 256, np), 256, 0, L.st>>>(L.dc, s, out, g);
    check_launch("galois_ntt");
    if (L.counter) ++*L.counter;
}

// c0 = pk0 u + e0 + m ; c1 = pk1 u + e1   (R6, R17), all NTT form over the L data primes
__global__ void k_encrypt_combine(const DCtx* __restrict__ dc, const u64* __restrict__ pk, const u64* __restrict__ u,
                                  const u64* __restrict__ e0, const u64* __restrict__ e1, const u64* __restrict__ m,
                                  u64* __restrict__ ct, int L)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, p = blockIdx.y, b = blockIdx.z;
    const DPrime Pr = dc->p[p];
    const size_t off = ((size_t)b * L + p) * n + k;
    const u64 uu = u[off];
    const u64 c0 = addmod(addmod(mulmod(pk[(size_t)p * n + k], uu, Pr), e0[off], Pr.q), m[off], Pr.q);
    const u64 c1 = addmod(mulmod(pk[((size_t)L + p) * n + k], uu, Pr), e1[off], Pr.q);
    ct[((size_t)b * 2 * L + p) * n + k] = c0;
    ct[((size_t)b * 2 * L + L + p) * n + k] = c1;
}

void encrypt_combine(const Launch& L, const uint64_t* pk, const uint64_t* u, const uint64_t* e0, const uint64_t* e1,
                     const uint64_t* m, uint64_t* ct, int batch, int Ld)
{
    const int n = 1 << L.log_n;
    k_encrypt_combine<<<dim3(n / 256, Ld, batch), 256, 0, L.st>>>(L.dc, pk, u, e0, e1, m, ct, Ld);
    check_launch("encrypt_combine");
    if (L.counter) ++*L.counter;
}

// constant plaintexts (cubic activation, R23): NTT of an integer constant m0 is m0 mod q in every slot
__global__ void __launch_bounds__(256)
k_mul_scalar(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t sin, u64* __restrict__ out, size_t sout,
             const u64* __restrict__ res, int nl)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, cl = blockIdx.y, b = blockIdx.z;
    const int l = cl % nl;
    out[(size_t)b * sout + (size_t)cl * n + k] = mulmod(in[(size_t)b * sin + (size_t)cl * n + k], res[l], dc->p[l]);
}
void mul_scalar(const Launch& L, const uint64_t* in, size_t sin, uint64_t* out, size_t sout, const uint64_t* res,
                int batch, int ncomp, int nl)
{
    const int n = 1 << L.log_n;
    k_mul_scalar<<<dim3(n / 256, ncomp * nl, batch), 256, 0, L.st>>>(L.dc, in, sin, out, sout, res, nl);
    check_launch("mul_scalar");
    if (L.counter) ++*L.counter;
}
__global__ void __launch_bounds__(256)
k_add_scalar(const DCtx* __restrict__ dc, u64* __restrict__ ct, size_t stride, const u64* __restrict__ res)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x, l = blockIdx.y, b = blockIdx.z;
    u64& v = ct[(size_t)b * stride + (size_t)l * n + k];
    v = addmod(v, res[l], dc->p[l].q);
}
void add_scalar(const Launch& L, uint64_t* ct, size_t stride, const uint64_t* res, int batch, int nl)
{
    const int n = 1 << L.log_n;
    k_add_scalar<<<dim3(n / 256, nl, batch), 256, 0, L.st>>>(L.dc, ct, stride, res);
    check_launch("add_scalar");
    if (L.counter) ++*L.counter;
}

}  // namespace ck
