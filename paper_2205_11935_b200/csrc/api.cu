// api.cpp -- host side of libckks_b200: the C-ABI of include/ckks.h.
//
// The host only (a) builds constants once per context (prime chain, psi, twiddle tables, CRT
// constants) and (b) sequences kernel launches with level/scale bookkeeping.  Every step of the
// hot path runs in the sm_100a kernels of kernels.cu.  There is no CPU fallback: without a CUDA
// device, compute calls fail with CKKS_E_CUDA.
#include "../../include/ckks.h"
#include "common.cuh"
#include "kernels.h"
#include "ntt.cuh"
#include "ntt_c.cuh"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

typedef unsigned __int128 u128;

namespace {

thread_local std::string g_err;

ckks_status fail(ckks_status s, const std::string& msg)
{
    g_err = msg;
    return s;
}

struct CkksError : std::runtime_error {
    ckks_status st;
    CkksError(ckks_status s, const std::string& m) : std::runtime_error(m), st(s) {}
};

#define CK_TRY(...)                                                                             \
    try {                                                                                         \
        __VA_ARGS__                                                                               \
    } catch (const CkksError& e) {                                                                \
        return fail(e.st, e.what());                                                              \
    } catch (const std::exception& e) {                                                           \
        return fail(CKKS_E_CUDA, e.what());                                                       \
    }

void cuda_ok(cudaError_t e, const char* what)
{
    if (e != cudaSuccess) throw CkksError(CKKS_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

// ------------------------------------------------------------------------------ host number theory
u64 h_mulmod(u64 a, u64 b, u64 m) { return (u64)((u128)a * b % m); }
u64 h_pow(u64 a, u64 e, u64 m)
{
    u64 r = 1 % m;
    a %= m;
    for (; e; e >>= 1) {
        if (e & 1) r = h_mulmod(r, a, m);
        a = h_mulmod(a, a, m);
    }
    return r;
}
bool h_is_prime(u64 n)
{
    if (n < 4) return n >= 2;
    for (u64 p : {2ULL, 3ULL, 5ULL, 7ULL, 11ULL, 13ULL, 17ULL, 19ULL, 23ULL, 29ULL, 31ULL, 37ULL})
        if (n % p == 0) return n == p;
    u64 d = n - 1;
    int s = 0;
    while (!(d & 1)) d >>= 1, ++s;
    for (u64 a : {2ULL, 3ULL, 5ULL, 7ULL, 11ULL, 13ULL, 17ULL, 19ULL, 23ULL, 29ULL, 31ULL, 37ULL}) {
        u64 x = h_pow(a, d, n);
        if (x == 1 || x == n - 1) continue;
        bool witness = true;
        for (int r = 1; r < s && witness; ++r) {
            x = h_mulmod(x, x, n);
            if (x == n - 1) witness = false;
        }
        if (witness) return false;
    }
    return true;
}
u64 h_shoup(u64 w, u64 q) { return (u64)(((u128)w << 64) / q); }
u32 h_brev(u32 x, int bits)
{
    u32 r = 0;
    for (int i = 0; i < bits; ++i) r = (r << 1) | ((x >> i) & 1);
    return r;
}

// R1: largest unused prime below 2^bits congruent to 1 mod 2N, in list order.
std::vector<u64> prime_chain(int log_n, const std::vector<u32>& bits)
{
    const u64 m = 2ULL << log_n;
    std::vector<u64> out;
    for (u32 b : bits) {
        if ((int)b < log_n + 2 || b > 61) throw CkksError(CKKS_E_PARAM, "prime bit size out of range [log_n+2, 61]");
        u64 c = (1ULL << b) + 1 - m;
        while (!(h_is_prime(c) && std::find(out.begin(), out.end(), c) == out.end())) {
            if (c <= m + 1) throw CkksError(CKKS_E_PARAM, "ran out of primes");
            c -= m;
        }
        out.push_back(c);
    }
    return out;
}
// R2: smallest primitive 2N-th root of unity mod q.
u64 min_root(u64 q, int log_n)
{
    const u64 m = 2ULL << log_n, n = 1ULL << log_n;
    u64 g = 0;
    for (u64 x = 2;; ++x) {
        u64 c = h_pow(x, (q - 1) / m, q);
        if (h_pow(c, n, q) == q - 1) {
            g = c;
            break;
        }
    }
    const u64 g2 = h_mulmod(g, g, q);
    u64 best = g, cur = g;
    for (u64 k = 1; k < m; k += 2) {
        best = std::min(best, cur);
        cur = h_mulmod(cur, g2, q);
    }
    return best;
}

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
// device canonical-embedding tables (k_encode.cu): slot positions [n] u32, zeta^k [n], omega^p [n/2] (n = N/2)
size_t embed_table_bytes(int N)
{
    const size_t n = (size_t)N / 2;
    return align256(n * 4) + align256(n * 16) + align256(n / 2 * 16);
}

// ------------------------------------------------------------------------------ FFT (encode/decode)
void fft(std::vector<std::complex<double>>& a, int sign)
{
    const size_t n = a.size();
    for (size_t i = 1, j = 0; i < n; ++i) {
        size_t bit = n >> 1;
        for (; j & bit; bit >>= 1) j ^= bit;
        j ^= bit;
        if (i < j) std::swap(a[i], a[j]);
    }
    for (size_t len = 2; len <= n; len <<= 1) {
        const double ang = sign * 2.0 * M_PI / (double)len;
        for (size_t i = 0; i < n; i += len)
            for (size_t k = 0; k < len / 2; ++k) {
                const std::complex<double> w(std::cos(ang * (double)k), std::sin(ang * (double)k));
                const std::complex<double> u = a[i + k], v = a[i + k + len / 2] * w;
                a[i + k] = u + v;
                a[i + k + len / 2] = u - v;
            }
    }
}

std::vector<u64> slot_exps(int n)
{
    std::vector<u64> e(n / 2);
    u64 v = 1;
    for (int i = 0; i < n / 2; ++i) {
        e[i] = v;
        v = (v * 5) % (2ULL * n);
    }
    return e;
}

// R4: m_k = round_half_away(Re FFT_2N(Z)[k] / N), Z[5^i] = scale z_i, Z[-5^i] = conj.
void encode_host(int n, const double* values, size_t count, double scale, int64_t* out)
{
    if (count > (size_t)n / 2) throw CkksError(CKKS_E_PARAM, "more values than slots");
    std::vector<std::complex<double>> Z(2 * (size_t)n, 0.0);
    const auto e = slot_exps(n);
    for (size_t i = 0; i < count; ++i) {
        Z[e[i]] = scale * values[i];
        Z[(2 * n - e[i]) % (2 * n)] = scale * values[i];
    }
    fft(Z, -1);
    for (int k = 0; k < n; ++k) {
        const double x = Z[k].real() / n;
        const double r = (x < 0 ? -1.0 : 1.0) * std::floor(std::fabs(x) + 0.5);
        if (std::fabs(r) >= 4.6e18) throw CkksError(CKKS_E_PARAM, "encoded coefficient overflows int64");
        out[k] = (int64_t)r;
    }
}

}  // namespace

// ================================================================================== structures
struct ckks_ctx {
    // host-buffer forward: copy streams (H2D, D2H) and the events that order staging-buffer reuse
    cudaStream_t h2d_st = nullptr, d2h_st = nullptr;
    cudaEvent_t ev_h2d[2] = {}, ev_done[2] = {}, ev_d2h[2] = {}, ev_ready = nullptr;
    void ensure_copy_streams()
    {
        if (h2d_st) return;
        cuda_ok(cudaStreamCreateWithFlags(&h2d_st, cudaStreamNonBlocking), "copy stream");
        cuda_ok(cudaStreamCreateWithFlags(&d2h_st, cudaStreamNonBlocking), "copy stream");
        for (int k = 0; k < 2; ++k) {
            cuda_ok(cudaEventCreateWithFlags(&ev_h2d[k], cudaEventDisableTiming), "event");
            cuda_ok(cudaEventCreateWithFlags(&ev_done[k], cudaEventDisableTiming), "event");
            cuda_ok(cudaEventCreateWithFlags(&ev_d2h[k], cudaEventDisableTiming), "event");
        }
        cuda_ok(cudaEventCreateWithFlags(&ev_ready, cudaEventDisableTiming), "event");
    }
    int log_n = 0, n = 0, L = 0, ns = 0, np = 0;
    int nd = 0;                                    // key-switching digits (R9b)
    std::vector<int> dig_start, dig_len;
    // digits with at least one active prime at nl limbs (the last may be cut at the level)
    int active_digits(int nl) const
    {
        int d = 0;
        while (d < nd && dig_start[d] < nl) ++d;
        return d;
    }
    double sigma = 3.2;
    uint32_t max_batch = 1;
    uint32_t bsgs_bx = 0;         // extra baby-step doublings of this context's dense layers (R5b)
    std::vector<u64> primes, psi;
    DCtx host_dc{};
    DCtx* d_dc = nullptr;
    u64* d_tw = nullptr;
    u64* d_s = nullptr;      // [np][N] secret, NTT form
    u64* d_pk = nullptr;     // [2][L][N]
    u64* d_keys = nullptr;   // [nkeys][L][2][L+1][N]
    u64* d_keys_perm = nullptr;   // Galois keys pre-permuted by sigma_{g^-1} (hoisted rotations)
    size_t key_words = 0;    // per switching key
    std::vector<int64_t> key_ids;
    std::map<int64_t, int> key_slot;
    u64* d_work = nullptr;
    size_t work_bytes = 0;
    unsigned long long launches = 0;
    ck::Probe probe;
    std::vector<int> pclass;   // prime class per prime (host copy)

    ck::Launch launch(void* st)
    {
        ck::Launch l;
        l.dc = d_dc;
        l.log_n = log_n;
        l.n_data = L;
        l.n_special = ns;
        l.st = (cudaStream_t)st;
        l.counter = &launches;
        l.probe = &probe;
        l.pclass = pclass.data();
        l.n_digits = nd;
        l.dig_start = dig_start.data();
        l.dig_len = dig_len.data();
        return l;
    }
    size_t ct_words(int nl, int ncomp = 2) const { return (size_t)ncomp * nl * n; }
    const u64* key(int64_t id) const
    {
        auto it = key_slot.find(id);
        if (it == key_slot.end()) return nullptr;
        return d_keys + (size_t)it->second * key_words;
    }
    const u64* key_perm(int64_t id) const
    {
        auto it = key_slot.find(id);
        if (it == key_slot.end() || id == 0) return nullptr;
        return d_keys_perm + (size_t)it->second * key_words;
    }
    uint32_t galois_inv(uint32_t g) const { return (uint32_t)h_pow(g, (u64)n - 1, 2ULL * n); }
    uint32_t galois(int64_t step) const
    {
        const int64_t slots = n / 2;
        const int64_t r = ((step % slots) + slots) % slots;
        return (uint32_t)h_pow(5, (u64)r, 2ULL * n);
    }
    // KS workspace views for `B` ciphertexts (sized for the top level): digits [B][L][N],
    // ModUp [B][dnum][L+K][N], ModDown outputs [G][B][2][L+K][N], remainders [G][B][3][K][N]
    ck::KsWork ks_work(int B) const
    {
        ck::KsWork w;
        u64* p = d_work;
        w.digits = p;
        p += (size_t)B * L * n;
        w.modup = p;
        p += (size_t)B * nd * (L + ns) * n;
        w.acc = p;
        p += (size_t)KS_GMAX * B * 2 * (L + ns) * n;
        w.rem = p;
        return w;
    }
};

// A linear layer  y = sum_k rot_{k g}( sum_j pt_{k,j} o rot_{s_j}(x) ) (+ bias): the BSGS dense
// (Eq. 1, s_j = j, g = t1), the packed-SISO conv1d (R26) and the average pool (R27).
struct ckks_layer {
    int kind = CKKS_LAYER_DENSE;
    uint32_t rows, cols, t, t1, t2, level;
    std::vector<int32_t> baby;     // t1 baby steps, baby[0] == 0
    int32_t giant = 0;
    uint32_t region = 0, items = 1;
    double pt_scale, bias_scale;
    u64* d_pts;     // [t2 * t1][level+1+K][N]  (limbs level+1..: mod P_k, for the double-hoisted Q_l P MAC)
    int hoisting = 0;   // ckks_matvec_diag: 0 plain, 1 hoisted baby steps, 2 double hoisting
    u64* d_bias;    // [level][N] or null
};

struct Stage {
    const ckks_layer* layer;
    int activation;       // after the layer: 0 none, 1 square, 2 cubic
    uint32_t replicate_t; // before the layer: y + rot_{-t}(y) when != 0
};

struct ckks_model {
    std::vector<const ckks_layer*> layers;
    std::vector<Stage> stages;
    std::vector<u64*> d_act_stage;   // per stage: masked c0 plaintext of a cubic activation (or null)
    std::vector<u64*> d_act_const;   // per stage: residues [3][CKKS_MAXP] of the Eq. 2 constants c3, c2, c1
    std::vector<double> act_scale;   // per stage: the activation input scale the constants were encoded for
    int activation;
    int hoisted = 0;        // 0 none, 1 hoisted baby steps (R11b), 2 double hoisting (R11c)  (NEXT f-1)
};

namespace {

// digits + modup + KS_GMAX x (ModDown outputs x + remainders)
size_t ks_work_words(int L, int K, int nd, int n, int B)
{
    return (size_t)B * n * ((size_t)L + (size_t)nd * (L + K) + (size_t)KS_GMAX * (2 * (L + K) + 3 * K));
}
size_t enc_work_words(int L, int n, int B) { return (size_t)B * n * (4 * (size_t)L + 1); }

void check_ct(const ckks_ctx* c, const ckks_ct* x, int ncomp_expect = 2)
{
    if (!x || !x->data) throw CkksError(CKKS_E_PARAM, "null ciphertext");
    if (ncomp_expect && (int)x->n_comp != ncomp_expect) throw CkksError(CKKS_E_SHAPE, "wrong number of components");
    if ((int)x->level >= c->L) throw CkksError(CKKS_E_SHAPE, "level above the chain");
    if (x->batch == 0) throw CkksError(CKKS_E_SHAPE, "empty batch");
}

// R5 (x = 0) / R5b: t1 = min(2^(ceil(lg/2) + x), 2^lg)
void bsgs_split(uint32_t rows, uint32_t cols, uint32_t& t, uint32_t& t1, uint32_t& t2, uint32_t x = 0)
{
    t = std::max(rows, cols);
    int lg = 0;
    while ((1u << lg) < t) ++lg;
    t1 = 1u << std::min<int>(lg, (lg + 1) / 2 + (int)x);
    t = (t + t1 - 1) / t1 * t1;
    t2 = t / t1;
}

// rotate a batch (chunked by max_batch): out = rot_step(in)  [+ out if accumulate]
void rotate_impl(ckks_ctx* c, const u64* in, size_t in_stride, int nl, int batch, int64_t step, u64* out,
                 size_t out_stride, bool accumulate, void* stream)
{
    const uint32_t g = c->galois(step);
    auto L = c->launch(stream);
    if (g == 1) {
        for (int b = 0; b < batch; ++b) {
            if (accumulate)
                ck::add(L, in + b * in_stride, 0, out + b * out_stride, 0, out + b * out_stride, 0, 1, 2, nl);
            else
                cuda_ok(cudaMemcpyAsync(out + b * out_stride, in + b * in_stride, c->ct_words(nl) * 8,
                                        cudaMemcpyDeviceToDevice, (cudaStream_t)stream), "copy");
        }
        return;
    }
    const u64* key = c->key((int64_t)g);
    if (!key) throw CkksError(CKKS_E_NOKEY, "no Galois key for step " + std::to_string(step));
    for (int b0 = 0; b0 < batch; b0 += (int)c->max_batch) {
        const int B = std::min((int)c->max_batch, batch - b0);
        ck::KsIn ki{in + (size_t)b0 * in_stride, in_stride, (size_t)nl * c->n, g};
        ck::KsOut ko{out + (size_t)b0 * out_stride, out_stride, in + (size_t)b0 * in_stride, in_stride, g, 0,
                     accumulate ? 1 : 0};
        ck::keyswitch(L, ki, key, B, nl, c->ks_work(B), ko);
    }
}

// Hoisted rotations (NEXT f-1, R11b): one ModUp of the unrotated c1 shared by every step;
// out_s = sigma_g(c0 + ModDown(sum_j D_j key'_j)),  key' = sigma_{g^-1}(gk_g).
void rotate_hoisted_impl(ckks_ctx* c, const u64* in, size_t in_stride, int nl, int batch, const int64_t* steps,
                         int n_steps, u64* const* outs, size_t out_stride, void* stream)
{
    auto L = c->launch(stream);
    for (int s = 0; s < n_steps; ++s) {
        const uint32_t g = c->galois(steps[s]);
        if (g != 1 && !c->key_perm((int64_t)g))
            throw CkksError(CKKS_E_NOKEY, "no Galois key for step " + std::to_string(steps[s]));
    }
    for (int b0 = 0; b0 < batch; b0 += (int)c->max_batch) {
        const int B = std::min((int)c->max_batch, batch - b0);
        const u64* inb = in + (size_t)b0 * in_stride;
        ck::KsIn ki{inb, in_stride, (size_t)nl * c->n, 0};
        auto w = c->ks_work(B);
        bool have_modup = false;
        ck::KsGroup grp{};
        grp.G = 0;
        auto flush = [&]() {
            if (!grp.G) return;
            ck::KsOut ko{nullptr, out_stride, inb, in_stride, 0, 0, 0};
            ck::keyswitch_finish(L, ki, grp, B, nl, w, ko);
            grp.G = 0;
        };
        for (int s = 0; s < n_steps; ++s) {
            const uint32_t g = c->galois(steps[s]);
            u64* ob = outs[s] + (size_t)b0 * out_stride;
            if (g == 1) {
                cuda_ok(cudaMemcpy2DAsync(ob, out_stride * 8, inb, in_stride * 8, c->ct_words(nl) * 8, B,
                                          cudaMemcpyDeviceToDevice, (cudaStream_t)stream), "copy");
                continue;
            }
            if (!have_modup) {
                ck::keyswitch_modup(L, ki, B, nl, w);
                have_modup = true;
            }
            grp.key[grp.G] = c->key_perm((int64_t)g);
            grp.out[grp.G] = ob;
            grp.scatter[grp.G] = g;
            grp.ginv[grp.G] = c->galois_inv(g);
            if (++grp.G == KS_GMAX) flush();
        }
        flush();
    }
}

// Double hoisting (R11c) baby steps: hoisted rotations of a Q_l input left in the Q_l P basis,
// out_s = sigma_g(P c0 + sum_j D_j key'_j) over nl+1 limbs; batch <= max_batch.
void rotate_hoisted_qp_impl(ckks_ctx* c, const u64* in, size_t in_stride, int nl, int B, const int64_t* steps,
                            int n_steps, u64* const* outs, size_t out_stride, void* stream, bool mac_layout = false)
{
    auto L = c->launch(stream);
    for (int s = 0; s < n_steps; ++s) {
        const uint32_t g = c->galois(steps[s]);
        if (g != 1 && !c->key_perm((int64_t)g))
            throw CkksError(CKKS_E_NOKEY, "no Galois key for step " + std::to_string(steps[s]));
    }
    ck::KsIn ki{in, in_stride, (size_t)nl * c->n, 0};
    auto w = c->ks_work(B);
    bool have_modup = false;
    ck::KsGroup grp{};
    grp.G = 0;
    auto flush = [&]() {
        if (!grp.G) return;
        ck::KsOut ko{nullptr, out_stride, in, in_stride, 0, 0, 0};
        ko.mac_layout = mac_layout ? 1 : 0;
        ck::keyswitch_finish_qp(L, ki, grp, B, nl, w, ko, true);
        grp.G = 0;
    };
    for (int s = 0; s < n_steps; ++s) {
        const uint32_t g = c->galois(steps[s]);
        if (g == 1) {
            if (mac_layout) throw CkksError(CKKS_E_PARAM, "MAC layout with an identity baby step");
            ck::lift_qp(L, in, in_stride, outs[s], out_stride, B, nl);
            continue;
        }
        if (!have_modup) {
            ck::keyswitch_modup(L, ki, B, nl, w, false);
            have_modup = true;
        }
        grp.key[grp.G] = c->key_perm((int64_t)g);
        grp.out[grp.G] = outs[s];
        grp.scatter[grp.G] = g;
        grp.ginv[grp.G] = c->galois_inv(g);
        if (++grp.G == KS_GMAX) flush();
    }
    flush();
}

// Double hoisting (R11c) giant step: acc += (sigma_g(w.c0), 0) + KS_QP(sigma_g(ModDown(w.c1))), all in Q_l P.
void rotate_qp_impl(ckks_ctx* c, const u64* wq, size_t w_stride, int nl, int B, int64_t step, u64* acc,
                    size_t acc_stride, void* stream)
{
    auto L = c->launch(stream);
    const uint32_t g = c->galois(step);
    if (g == 1) throw CkksError(CKKS_E_PARAM, "giant step congruent to 0 mod N/2");
    const u64* key = c->key((int64_t)g);
    if (!key) throw CkksError(CKKS_E_NOKEY, "no Galois key for step " + std::to_string(step));
    auto w = c->ks_work(B);
    ck::KsIn ki{wq, w_stride, (size_t)(nl + c->ns) * c->n, g};
    ck::keyswitch_modup(L, ki, B, nl, w, true);
    ck::KsGroup grp{};
    grp.key[0] = key;
    grp.out[0] = acc;
    grp.scatter[0] = 0;
    grp.G = 1;
    ck::KsOut ko{acc, acc_stride, wq, w_stride, g, 0, 1};
    ck::keyswitch_finish_qp(L, ki, grp, B, nl, w, ko, false);
}

void relin_impl(ckks_ctx* c, const u64* in3, size_t in_stride, int nl, int batch, u64* out, size_t out_stride,
                void* stream)
{
    const u64* key = c->key(0);
    if (!key) throw CkksError(CKKS_E_NOKEY, "no relinearisation key");
    auto L = c->launch(stream);
    for (int b0 = 0; b0 < batch; b0 += (int)c->max_batch) {
        const int B = std::min((int)c->max_batch, batch - b0);
        ck::KsIn ki{in3 + (size_t)b0 * in_stride, in_stride, (size_t)2 * nl * c->n, 0};
        ck::KsOut ko{out + (size_t)b0 * out_stride, out_stride, in3 + (size_t)b0 * in_stride, in_stride, 0, 1, 0};
        ck::keyswitch(L, ki, key, B, nl, c->ks_work(B), ko);
    }
}

void rescale_impl(ckks_ctx* c, const u64* in, size_t in_stride, int ncomp, int nl, int batch, u64* out,
                  size_t out_stride, const u64* bias, void* stream)
{
    if (nl < 2) throw CkksError(CKKS_E_LEVEL, "rescale at level 0 (depth exhausted)");
    auto L = c->launch(stream);
    // [B][<=3][N] remainder scratch: the key-switch region's remainders, or (a context without a special
    // prime has no key-switch region) the start of the workspace, which is at least 3 max_batch N words
    u64* rem = c->ns ? c->ks_work(c->max_batch).rem : c->d_work;
    for (int b0 = 0; b0 < batch; b0 += (int)c->max_batch) {
        const int B = std::min((int)c->max_batch, batch - b0);
        ck::rescale(L, in + (size_t)b0 * in_stride, in_stride, out + (size_t)b0 * out_stride, out_stride, B, ncomp,
                    nl, rem, bias);
    }
}

// Device scalar constant helpers for the cubic activation (R23): constant plaintext m0 at
// coefficient 0 has NTT value m0 mod q_i in every slot.
}  // namespace

namespace ck {
void mul_scalar(const Launch&, const uint64_t* in, size_t sin, uint64_t* out, size_t sout, const uint64_t* res,
                int batch, int ncomp, int nl);
void add_scalar(const Launch&, uint64_t* ct, size_t stride, const uint64_t* res, int batch, int nl);
}  // namespace ck

// ================================================================================== C-ABI
extern "C" {

const char* ckks_last_error(void) { return g_err.c_str(); }

static void sizes_impl(const ckks_params* p, size_t* tb, size_t* kb, size_t* wb, std::vector<u64>* primes_out)
{
    if (!p || !p->prime_bits) throw CkksError(CKKS_E_PARAM, "null params");
    if (p->log_n < 10 || p->log_n > 14) throw CkksError(CKKS_E_PARAM, "log_n must be in [10, 14]");
    if (p->n_data < 1 || p->n_special > 2 || p->n_data + p->n_special > CKKS_MAXP)
        throw CkksError(CKKS_E_PARAM, "need 1 <= n_data, n_special <= 2, n_data + n_special <= 16");
    if (p->n_special == 0 && (p->n_rot_steps || p->want_relin))
        throw CkksError(CKKS_E_PARAM, "key switching needs a special prime");
    if (p->max_batch < 1) throw CkksError(CKKS_E_PARAM, "max_batch >= 1");
    const int n = 1 << p->log_n, L = (int)p->n_data, K = (int)p->n_special, np = L + K;
    std::vector<u32> bits(p->prime_bits, p->prime_bits + np);
    auto primes = prime_chain((int)p->log_n, bits);
    if (primes_out) *primes_out = primes;
    // digits (R9b): 1 or 2 consecutive data primes each
    int nd = L;
    if (p->digit_sizes) {
        uint32_t sum = 0;
        for (uint32_t j = 0; j < p->n_digits; ++j) {
            if (p->digit_sizes[j] < 1 || p->digit_sizes[j] > 2)
                throw CkksError(CKKS_E_PARAM, "digit sizes must be 1 or 2 primes");
            sum += p->digit_sizes[j];
        }
        if (sum != p->n_data || p->n_digits == 0) throw CkksError(CKKS_E_PARAM, "digit sizes must sum to n_data");
        nd = (int)p->n_digits;
    }
    // number of distinct switching keys
    std::vector<int64_t> ids;
    if (p->want_relin) ids.push_back(0);
    for (uint32_t i = 0; i < p->n_rot_steps; ++i) {
        const int64_t slots = n / 2;
        const int64_t r = (((int64_t)p->rot_steps[i] % slots) + slots) % slots;
        const int64_t g = (int64_t)h_pow(5, (u64)r, 2ULL * n);
        if (g != 1 && std::find(ids.begin(), ids.end(), g) == ids.end()) ids.push_back(g);
    }
    const size_t key_words = p->n_special ? (size_t)nd * 2 * np * n : 0;
    *tb = align256(sizeof(DCtx)) + align256((size_t)np * CK_TW_WORDS * n * 8) + embed_table_bytes(n);
    // every switching key, plus a sigma_{g^-1}-permuted copy per key slot (used by hoisted rotations)
    *kb = align256((size_t)np * n * 8) + align256((size_t)2 * L * n * 8) + 2 * ids.size() * key_words * 8;
    const int B = (int)p->max_batch;
    size_t w = std::max(enc_work_words(L, n, B), p->n_special ? ks_work_words(L, K, nd, n, B) : (size_t)0);
    w = std::max(w, (size_t)3 * B * n);   // rescale remainders (rescale_impl)
    // keygen scratch: e_ntt [dnum][L+K][N] + s' [np][N]
    w = std::max(w, (size_t)nd * np * n + (size_t)np * n);
    *wb = align256(w * 8);
}

ckks_status ckks_ctx_sizes(const ckks_params* p, size_t* table_bytes, size_t* key_bytes, size_t* work_bytes)
{
    CK_TRY({
        sizes_impl(p, table_bytes, key_bytes, work_bytes, nullptr);
        return CKKS_OK;
    })
}

ckks_status ckks_ctx_create(const ckks_params* p, void* d_tables, void* d_keys, void* d_work, void* stream,
                            ckks_ctx** out)
{
    CK_TRY({
        if (!out) throw CkksError(CKKS_E_PARAM, "null out");
        int ndev = 0;
        if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw CkksError(CKKS_E_CUDA, "no CUDA device");
        size_t tb, kb, wb;
        std::vector<u64> primes;
        sizes_impl(p, &tb, &kb, &wb, &primes);
        if (!d_tables || !d_keys || !d_work) throw CkksError(CKKS_E_PARAM, "null device buffer");
        auto* c = new ckks_ctx();
        c->log_n = (int)p->log_n;
        c->n = 1 << c->log_n;
        c->L = (int)p->n_data;
        c->ns = (int)p->n_special;
        c->np = c->L + c->ns;
        c->sigma = p->sigma > 0 ? p->sigma : 3.2;
        c->max_batch = p->max_batch;
        if (p->bsgs_baby_extra > 4) throw CkksError(CKKS_E_PARAM, "bsgs_baby_extra must be <= 4");
        c->bsgs_bx = p->bsgs_baby_extra;
        c->primes = primes;
        for (u64 q : primes) c->pclass.push_back(prime_class(q));
        {
            int st = 0;
            const int nd = p->digit_sizes ? (int)p->n_digits : (int)p->n_data;
            for (int j = 0; j < nd; ++j) {
                const int len = p->digit_sizes ? (int)p->digit_sizes[j] : 1;
                c->dig_start.push_back(st);
                c->dig_len.push_back(len);
                st += len;
            }
            c->nd = nd;
        }
        const int n = c->n, np = c->np, L = c->L;
        // ---- constants
        DCtx& h = c->host_dc;
        std::memset(&h, 0, sizeof(DCtx));
        h.log_n = c->log_n;
        h.n = n;
        h.n_data = L;
        h.n_special = c->ns;
        h.n_primes = np;
        std::vector<u64> tw((size_t)np * CK_TW_WORDS * n);
        for (int i = 0; i < np; ++i) {
            const u64 q = primes[i];
            const u64 psi = min_root(q, c->log_n), ipsi = h_pow(psi, q - 2, q);
            c->psi.push_back(psi);
            DPrime& P = h.p[i];
            P.q = q;
            P.q2 = 2 * q;
            P.ninv = h_pow((u64)n % q, q - 2, q);
            P.ninv_sh = h_shoup(P.ninv, q);
            P.one_sh = (u64)(((u128)1 << 64) / q);
            P.r64 = (u64)(((u128)1 << 64) % q);
            P.r64_sh = h_shoup(P.r64, q);
            P.w20 = (1ULL << 20) % q;
            P.w23 = (1ULL << 23) % q;
            P.w40 = (1ULL << 40) % q;
            P.mu90 = q >= (1ULL << 59) ? (u64)((((u128)1) << 90) / q) : 0;
            P.qinv_d = 1.0 / (double)q;
            P.w23q = (double)P.w23 / (double)q;
            // W[idx] = psi^{brev(idx)} (stage s = floor(log2 idx), block idx - 2^s), stored at the
            // pass-ordered position ntt_tw_position (ntt.cuh); same for psi^{-1}.
            u64* W = tw.data() + (size_t)i * CK_TW_WORDS * n;
            std::vector<u64> fw(n), iw(n);
            u64 pw = 1, ipw = 1;
            for (int m = 0; m < n; ++m) {
                const u32 r = h_brev((u32)m, c->log_n);
                fw[r] = pw;
                iw[r] = ipw;
                pw = h_mulmod(pw, psi, q);
                ipw = h_mulmod(ipw, ipsi, q);
            }
            W[0] = fw[0];
            W[n] = h_shoup(fw[0], q);
            W[2 * n] = iw[0];
            W[3 * n] = h_shoup(iw[0], q);
            for (int idx = 1; idx < n; ++idx) {
                int s = 0;
                while ((2 << s) <= idx) ++s;
                const int pos = ntt_tw_position(c->log_n, s, idx - (1 << s));
                W[pos] = fw[idx];
                W[n + pos] = h_shoup(fw[idx], q);
                W[2 * n + pos] = iw[idx];
                W[3 * n + pos] = h_shoup(iw[idx], q);
            }
            // FP64 copies for the FP64-pipe classes: the centred representative w in (-q/2, q/2] and fl(w / q), as
            // raw double bits (|w / q| <= 1/2 doubles the multiplicand range of fmodmul, ntt.cuh)
            auto centred = [q](u64 w) { return w > q / 2 ? -(double)(q - w) : (double)w; };
            for (int pos = 0; pos < n; ++pos) {
                const double wd = centred(W[pos]), iwd = centred(W[2 * n + pos]);
                const double wq = wd / (double)q, iwq = iwd / (double)q;
                std::memcpy(&W[4 * n + pos], &wd, 8);
                std::memcpy(&W[5 * n + pos], &wq, 8);
                std::memcpy(&W[6 * n + pos], &iwd, 8);
                std::memcpy(&W[7 * n + pos], &iwq, 8);
            }
            // pair tables of the cluster schedule (ntt_c.cuh): (w, fl(w/q)) at ntt_c_tw_position, forward then inverse
            for (int idx = 1; idx < n && ntt_c_supported(c->log_n); ++idx) {
                int s = 0;
                while ((2 << s) <= idx) ++s;
                const int pos = ntt_c_tw_position(c->log_n, s, idx - (1 << s));
                const double wd = centred(fw[idx]), iwd = centred(iw[idx]);
                const double wq = wd / (double)q, iwq = iwd / (double)q;
                std::memcpy(&W[8 * n + 2 * pos], &wd, 8);
                std::memcpy(&W[8 * n + 2 * pos + 1], &wq, 8);
                std::memcpy(&W[10 * n + 2 * pos], &iwd, 8);
                std::memcpy(&W[10 * n + 2 * pos + 1], &iwq, 8);
                W[12 * n + 2 * pos] = fw[idx];                      // integer pairs (w, w') for ArInt
                W[12 * n + 2 * pos + 1] = h_shoup(fw[idx], q);
            }
            for (int b = 0; b < np; ++b) {
                h.qmod[i][b] = q % primes[b];
                h.qmod_sh[i][b] = h_shoup(h.qmod[i][b], primes[b]);
                if (b != i) {
                    h.qinv[i][b] = h_pow(q % primes[b], primes[b] - 2, primes[b]);
                    h.qinv_sh[i][b] = h_shoup(h.qinv[i][b], primes[b]);
                }
            }
        }
        // key switching constants (R9b, R10b, R17b): digit table, 2-prime CRT inverses, P = prod P_k
        h.n_digits = c->nd;
        for (int j = 0; j < c->nd; ++j) {
            h.dig_start[j] = c->dig_start[j];
            h.dig_len[j] = c->dig_len[j];
            if (c->dig_len[j] == 2) {
                const int s1 = c->dig_start[j] + 1;
                h.dig_inv[s1] = h_pow(primes[s1 - 1] % primes[s1], primes[s1] - 2, primes[s1]);
                h.dig_inv_sh[s1] = h_shoup(h.dig_inv[s1], primes[s1]);
            }
        }
        if (c->ns == 2) {
            const int s1 = L + 1;
            h.dig_inv[s1] = h_pow(primes[L] % primes[s1], primes[s1] - 2, primes[s1]);
            h.dig_inv_sh[s1] = h_shoup(h.dig_inv[s1], primes[s1]);
        }
        if (c->ns) {
            for (int i = 0; i < np; ++i) {
                u64 pm = 1 % primes[i];
                for (int k = 0; k < c->ns; ++k) pm = h_mulmod(pm, primes[L + k] % primes[i], primes[i]);
                h.pmod[i] = i < L ? pm : 0;
                h.pmod_sh[i] = h_shoup(h.pmod[i], primes[i]);
                if (i < L) {
                    h.pinv[i] = h_pow(pm, primes[i] - 2, primes[i]);
                    h.pinv_sh[i] = h_shoup(h.pinv[i], primes[i]);
                }
            }
            u128 P = 1;
            for (int k = 0; k < c->ns; ++k) P *= primes[L + k];
            const u128 half = (P - 1) / 2;
            h.phalf_lo = (u64)half;
            h.phalf_hi = (u64)(half >> 64);
            h.phalf_a = c->ns == 2 ? (u64)(half % primes[L]) : (u64)half;
            h.phalf_t = c->ns == 2 ? (u64)(half / primes[L]) : 0;
        }
        // R13 CDT, same definition as DESIGN.md (computed here independently)
        {
            const int B = (int)std::floor(6.0 * c->sigma);
            if (2 * B > 40) throw CkksError(CKKS_E_PARAM, "sigma too large");
            std::vector<double> rho(2 * B + 1);
            double total = 0.0;
            for (int x = -B; x <= B; ++x) {
                rho[x + B] = std::exp(-(double)(x * x) / (2.0 * c->sigma * c->sigma));
                total += rho[x + B];
            }
            double cum = 0.0;
            for (int x = -B; x < B; ++x) {
                cum += rho[x + B];
                h.cdt[x + B] = (u64)std::ldexp(cum / total, 64);
            }
            h.cdt_bound = B;
        }
        char* tbase = (char*)d_tables;
        c->d_dc = (DCtx*)tbase;
        c->d_tw = (u64*)(tbase + align256(sizeof(DCtx)));
        h.tw = c->d_tw;
        cudaStream_t st = (cudaStream_t)stream;
        cuda_ok(cudaMemcpyAsync(c->d_tw, tw.data(), tw.size() * 8, cudaMemcpyHostToDevice, st), "upload tables");
        // canonical embedding tables (R3): pos(i) = (5^i mod 2N - 1) / 4, zeta^k, omega^p in long double
        {
            const int ns = n / 2;
            char* eb = tbase + align256(sizeof(DCtx)) + align256((size_t)np * CK_TW_WORDS * n * 8);
            std::vector<u32> pos(ns);
            std::vector<double> zeta(2 * (size_t)ns), omega(ns);
            u64 e = 1;
            for (int i = 0; i < ns; ++i) {
                pos[i] = (u32)((e - 1) / 4);
                e = e * 5 % (2ULL * n);
            }
            const long double pi = 3.141592653589793238462643383279502884L;
            for (int k = 0; k < ns; ++k) {
                zeta[2 * k] = (double)cosl(pi * k / n);
                zeta[2 * k + 1] = (double)sinl(pi * k / n);
            }
            for (int q = 0; q < ns / 2; ++q) {
                omega[2 * q] = (double)cosl(2 * pi * q / ns);
                omega[2 * q + 1] = (double)sinl(2 * pi * q / ns);
            }
            h.slot_pos = (const u32*)eb;
            h.fft_zeta = (const double2*)(eb + align256((size_t)ns * 4));
            h.fft_omega = (const double2*)(eb + align256((size_t)ns * 4) + align256((size_t)ns * 16));
            cuda_ok(cudaMemcpyAsync((void*)h.slot_pos, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, st), "tables");
            cuda_ok(cudaMemcpyAsync((void*)h.fft_zeta, zeta.data(), zeta.size() * 8, cudaMemcpyHostToDevice, st), "tables");
            cuda_ok(cudaMemcpyAsync((void*)h.fft_omega, omega.data(), omega.size() * 8, cudaMemcpyHostToDevice, st),
                    "tables");
            cuda_ok(cudaStreamSynchronize(st), "tables");   // host vectors go out of scope
        }
        cuda_ok(cudaMemcpyAsync(c->d_dc, &h, sizeof(DCtx), cudaMemcpyHostToDevice, st), "upload consts");
        // ---- key buffers
        char* kbase = (char*)d_keys;
        c->d_s = (u64*)kbase;
        c->d_pk = (u64*)(kbase + align256((size_t)np * n * 8));
        c->d_keys = (u64*)(kbase + align256((size_t)np * n * 8) + align256((size_t)2 * L * n * 8));
        c->key_words = c->ns ? (size_t)c->nd * 2 * np * n : 0;
        c->d_work = (u64*)d_work;
        c->work_bytes = wb;
        if (p->want_relin) c->key_ids.push_back(0);
        for (uint32_t i = 0; i < p->n_rot_steps; ++i) {
            const int64_t g = c->galois(p->rot_steps[i]);
            if (g != 1 && std::find(c->key_ids.begin(), c->key_ids.end(), g) == c->key_ids.end())
                c->key_ids.push_back(g);
        }
        for (size_t i = 0; i < c->key_ids.size(); ++i) c->key_slot[c->key_ids[i]] = (int)i;
        c->d_keys_perm = c->d_keys + c->key_ids.size() * c->key_words;
        // ---- keygen on the device (R5, R13-R15; stream tags of DESIGN.md)
        auto Lc = c->launch(stream);
        const u64 seed = p->key_seed;
        ck::sample_ntt(Lc, c->d_s, 1, np, L, 0, seed, 1, 0, 0, 0, 0);                 // s (TAG 1)
        u64* scratch = c->d_work;
        for (int i = 0; i < L; ++i) ck::sample_uniform(Lc, c->d_pk + (size_t)(L + i) * n, i, seed, 2, 0, 0);
        ck::sample_ntt(Lc, scratch, 1, L, L, 1, seed, 3, 0, 0, 0, 0);                 // pk e (TAG 3)
        ck::pk_combine(Lc, c->d_pk, scratch, c->d_s, L);
        if (c->ns) {
            const int nd = c->nd;
            u64* e_ntt = scratch;                               // [dnum][L+K][N]
            u64* sp = scratch + (size_t)nd * np * n;            // [np][N]
            for (size_t ki = 0; ki < c->key_ids.size(); ++ki) {
                const int64_t id = c->key_ids[ki];
                u64* key = c->d_keys + ki * c->key_words;
                if (id == 0) ck::square_ntt(Lc, c->d_s, sp, np);
                else ck::galois_ntt(Lc, c->d_s, sp, np, (uint32_t)id);
                for (int j = 0; j < nd; ++j)
                    for (int pi = 0; pi < np; ++pi)
                        ck::sample_uniform(Lc, key + (((size_t)j * 2 + 1) * np + pi) * n, pi, seed, 4, (u64)id,
                                           (u64)j);
                ck::sample_ntt(Lc, e_ntt, nd, np, L, 1, seed, 5, (u64)id, 0, 0, 1);   // e_j (TAG 5)
                ck::keyswitch_key_combine(Lc, key, e_ntt, c->d_s, sp, L);
                if (id != 0)   // key'_j = sigma_{g^-1}(gk_j): sum_j sigma_g(D_j) gk_j = sigma_g(sum_j D_j key'_j)
                    ck::galois_limbs(Lc, key, c->d_keys_perm + ki * c->key_words, (size_t)nd * 2 * np,
                                     c->galois_inv((uint32_t)id));
            }
        }
        cuda_ok(cudaStreamSynchronize(st), "keygen");
        *out = c;
        return CKKS_OK;
    })
}

void ckks_ctx_destroy(ckks_ctx* ctx)
{
    if (ctx) {
        for (auto e : ctx->probe.ev) cudaEventDestroy(e);
        if (ctx->h2d_st) {
            cudaStreamDestroy(ctx->h2d_st);
            cudaStreamDestroy(ctx->d2h_st);
            for (int k = 0; k < 2; ++k) {
                cudaEventDestroy(ctx->ev_h2d[k]);
                cudaEventDestroy(ctx->ev_done[k]);
                cudaEventDestroy(ctx->ev_d2h[k]);
            }
            cudaEventDestroy(ctx->ev_ready);
        }
    }
    delete ctx;
}

ckks_status ckks_probe_enable(ckks_ctx* c, int32_t kind)
{
    CK_TRY({
        if (!c || kind < 0 || kind > 4) throw CkksError(CKKS_E_PARAM, "probe kind 0..4");
        c->probe.kind = kind;
        c->probe.used = 0;
        c->probe.alg_bytes = 0;
        c->probe.names.clear();
        c->probe.bytes_by_kernel.clear();
        c->probe.flops_by_kernel.clear();
        c->probe.bfly_fp = c->probe.bfly_int = 0;
        while (kind && c->probe.ev.size() < 4096) {
            cudaEvent_t e;
            cuda_ok(cudaEventCreate(&e), "event");
            c->probe.ev.push_back(e);
        }
        return CKKS_OK;
    })
}

ckks_status ckks_probe_read_all(ckks_ctx* c, char* json, size_t cap)
{
    CK_TRY({
        if (!c || !json || cap == 0) throw CkksError(CKKS_E_PARAM, "null");
        const size_t pairs = c->probe.used / 2;
        if (pairs) cuda_ok(cudaEventSynchronize(c->probe.ev[2 * pairs - 1]), "probe sync");
        std::map<std::string, std::pair<double, uint64_t>> per;
        for (size_t i = 0; i < pairs && i < c->probe.names.size(); ++i) {
            float ms = 0;
            cuda_ok(cudaEventElapsedTime(&ms, c->probe.ev[2 * i], c->probe.ev[2 * i + 1]), "elapsed");
            auto& e = per[c->probe.names[i]];
            e.first += ms;
            e.second += 1;
        }
        std::string s = "{";
        for (auto& kv : per) {
            if (s.size() > 1) s += ", ";
            char buf[320];
            const auto it = c->probe.bytes_by_kernel.find(kv.first);
            const auto fl = c->probe.flops_by_kernel.find(kv.first);
            std::snprintf(buf, sizeof(buf),
                          "\"%s\": {\"ms\": %.6f, \"launches\": %llu, \"alg_bytes\": %.1f, \"tensor_flops\": %.1f}",
                          kv.first.c_str(), kv.second.first, (unsigned long long)kv.second.second,
                          it == c->probe.bytes_by_kernel.end() ? 0.0 : it->second,
                          fl == c->probe.flops_by_kernel.end() ? 0.0 : fl->second);
            s += buf;
        }
        {
            char buf[160];
            std::snprintf(buf, sizeof(buf), "%s\"_modup_butterflies\": {\"fp64\": %.1f, \"int\": %.1f}",
                          s.size() > 1 ? ", " : "", c->probe.bfly_fp, c->probe.bfly_int);
            s += buf;
        }
        s += "}";
        if (s.size() + 1 > cap) throw CkksError(CKKS_E_SIZE, "json buffer too small");
        std::memcpy(json, s.c_str(), s.size() + 1);
        return CKKS_OK;
    })
}

ckks_status ckks_probe_read(ckks_ctx* c, double* total_ms, uint64_t* launches, double* alg_bytes)
{
    CK_TRY({
        if (!c || !total_ms || !launches) throw CkksError(CKKS_E_PARAM, "null");
        double tot = 0;
        const size_t pairs = c->probe.used / 2;
        if (pairs) cuda_ok(cudaEventSynchronize(c->probe.ev[2 * pairs - 1]), "probe sync");
        for (size_t i = 0; i < pairs; ++i) {
            float ms = 0;
            cuda_ok(cudaEventElapsedTime(&ms, c->probe.ev[2 * i], c->probe.ev[2 * i + 1]), "elapsed");
            tot += ms;
        }
        *total_ms = tot;
        *launches = pairs;
        if (alg_bytes) *alg_bytes = c->probe.alg_bytes;
        return CKKS_OK;
    })
}

ckks_status ckks_ctx_info(const ckks_ctx* c, ckks_info* o)
{
    if (!c || !o) return fail(CKKS_E_PARAM, "null");
    std::memset(o, 0, sizeof(*o));
    o->log_n = (uint32_t)c->log_n;
    o->n = (uint32_t)c->n;
    o->n_data = (uint32_t)c->L;
    o->n_special = (uint32_t)c->ns;
    o->n_keys = (uint32_t)c->key_ids.size();
    for (int i = 0; i < c->np; ++i) {
        o->primes[i] = c->primes[i];
        o->psi[i] = c->psi[i];
    }
    o->n_digits = (uint32_t)c->nd;
    for (int j = 0; j < c->nd; ++j) o->digit_sizes[j] = (uint32_t)c->dig_len[j];
    return CKKS_OK;
}

uint64_t ckks_launch_count(const ckks_ctx* c) { return c ? c->launches : 0; }

ckks_status ckks_set_option(const char* name, int64_t value)
{
    if (!name) return fail(CKKS_E_PARAM, "null option name");
    if (std::strcmp(name, "mac_tc") == 0) {
        if (value != 0 && value != 1) return fail(CKKS_E_PARAM, "mac_tc is 0 or 1");
        ck::set_mac_tc((int)value);
        return CKKS_OK;
    }
    if (std::strcmp(name, "ip_v3") == 0) {
        if (value != 0 && value != 1) return fail(CKKS_E_PARAM, "ip_v3 is 0 or 1");
        ck::set_ip_v3((int)value);
        return CKKS_OK;
    }
    if (std::strcmp(name, "ntt_q") == 0) {
        if (value < 0 || value > 255) return fail(CKKS_E_PARAM, "ntt_q is a bit mask 0..255");
        ck::set_ntt_q((int)value);
        return CKKS_OK;
    }
    if (std::strcmp(name, "giant_multi") == 0) {
        if (value != 0 && value != 1) return fail(CKKS_E_PARAM, "giant_multi is 0 or 1");
        ck::set_giant_multi((int)value);
        return CKKS_OK;
    }
    if (std::strcmp(name, "nvtx") == 0) {
        if (value != 0 && value != 1) return fail(CKKS_E_PARAM, "nvtx is 0 or 1");
        ck::set_nvtx((int)value);
        return CKKS_OK;
    }
    return fail(CKKS_E_PARAM, std::string("unknown option ") + name);
}

ckks_status ckks_get_option(const char* name, int64_t* value)
{
    if (!name || !value) return fail(CKKS_E_PARAM, "null");
    if (std::strcmp(name, "mac_tc") == 0) {
        *value = ck::get_mac_tc();
        return CKKS_OK;
    }
    if (std::strcmp(name, "ip_v3") == 0) {
        *value = ck::get_ip_v3();
        return CKKS_OK;
    }
    if (std::strcmp(name, "ntt_q") == 0) {
        *value = ck::get_ntt_q();
        return CKKS_OK;
    }
    if (std::strcmp(name, "giant_multi") == 0) {
        *value = ck::get_giant_multi();
        return CKKS_OK;
    }
    if (std::strcmp(name, "nvtx") == 0) {
        *value = ck::nvtx_on();
        return CKKS_OK;
    }
    return fail(CKKS_E_PARAM, std::string("unknown option ") + name);
}

uint64_t ckks_galois_elt(const ckks_ctx* c, int32_t step) { return c ? c->galois(step) : 0; }

static ckks_status ntt_impl(ckks_ctx* c, uint64_t* d, uint32_t batch, uint32_t limbs, void* stream, bool inv)
{
    CK_TRY({
        if (!c) throw CkksError(CKKS_E_PARAM, "null context");
        if (limbs == 0 || (int)limbs > c->np) throw CkksError(CKKS_E_SHAPE, "limbs > number of primes");
        if (batch == 0) return CKKS_OK;   // empty batch: no-op, d may be NULL
        if (!d) throw CkksError(CKKS_E_PARAM, "null data");
        auto L = c->launch(stream);
        // grid.y is limited to 65535 CTAs: chunk the batch
        for (uint32_t b0 = 0; b0 < batch; b0 += 65535) {
            const uint32_t B = std::min<uint32_t>(65535, batch - b0);
            ck::ntt_batch(L, d + (size_t)b0 * limbs * c->n, (int)B, (int)limbs, 0, inv);
        }
        return CKKS_OK;
    })
}
ckks_status ckks_ntt_fwd(ckks_ctx* c, uint64_t* d, uint32_t batch, uint32_t limbs, void* stream)
{
    return ntt_impl(c, d, batch, limbs, stream, false);
}
ckks_status ckks_ntt_inv(ckks_ctx* c, uint64_t* d, uint32_t batch, uint32_t limbs, void* stream)
{
    return ntt_impl(c, d, batch, limbs, stream, true);
}

ckks_status ckks_rotate(ckks_ctx* c, const ckks_ct* in, int32_t step, ckks_ct* out, void* stream)
{
    CK_TRY({
        if (!c || !out || !out->data) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in);
        if (in->data == out->data) throw CkksError(CKKS_E_SHAPE, "rotate: out aliases in");
        const int nl = (int)in->level + 1;
        rotate_impl(c, in->data, c->ct_words(nl), nl, (int)in->batch, step, out->data, c->ct_words(nl), false, stream);
        out->batch = in->batch;
        out->n_comp = 2;
        out->level = in->level;
        out->scale = in->scale;
        return CKKS_OK;
    })
}

ckks_status ckks_rotate_hoisted(ckks_ctx* c, const ckks_ct* in, const int32_t* steps, uint32_t n_steps, ckks_ct* outs,
                                void* stream)
{
    CK_TRY({
        if (!c || !steps || !outs || n_steps == 0) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in);
        const int nl = (int)in->level + 1;
        std::vector<int64_t> st(steps, steps + n_steps);
        std::vector<u64*> o(n_steps);
        for (uint32_t s = 0; s < n_steps; ++s) {
            if (!outs[s].data || outs[s].data == in->data) throw CkksError(CKKS_E_SHAPE, "rotate_hoisted: bad out");
            o[s] = outs[s].data;
        }
        rotate_hoisted_impl(c, in->data, c->ct_words(nl), nl, (int)in->batch, st.data(), (int)n_steps, o.data(),
                            c->ct_words(nl), stream);
        for (uint32_t s = 0; s < n_steps; ++s) {
            outs[s].batch = in->batch;
            outs[s].n_comp = 2;
            outs[s].level = in->level;
            outs[s].scale = in->scale;
        }
        return CKKS_OK;
    })
}

ckks_status ckks_model_set_hoisting(ckks_model* m, int32_t on)
{
    if (!m) return fail(CKKS_E_PARAM, "null");
    if (on < 0 || on > 2) return fail(CKKS_E_PARAM, "hoisting mode must be 0, 1 or 2");
    m->hoisted = on;
    return CKKS_OK;
}

ckks_status ckks_layer_set_hoisting(ckks_layer* l, int32_t mode)
{
    if (!l) return fail(CKKS_E_PARAM, "null");
    if (mode < 0 || mode > 2) return fail(CKKS_E_PARAM, "hoisting mode must be 0, 1 or 2");
    l->hoisting = mode;
    return CKKS_OK;
}

ckks_status ckks_mul(ckks_ctx* c, const ckks_ct* a, const ckks_ct* b, ckks_ct* out3, void* stream)
{
    CK_TRY({
        if (!c || !out3 || !out3->data) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, a);
        check_ct(c, b);
        if (a->level != b->level || a->batch != b->batch) throw CkksError(CKKS_E_SHAPE, "mul: level/batch mismatch");
        const int nl = (int)a->level + 1;
        auto L = c->launch(stream);
        for (uint32_t b0 = 0; b0 < a->batch; b0 += 65535) {
            const int B = (int)std::min<uint32_t>(65535, a->batch - b0);
            ck::tensor(L, a->data + b0 * c->ct_words(nl), b->data + b0 * c->ct_words(nl), c->ct_words(nl),
                       out3->data + b0 * c->ct_words(nl, 3), c->ct_words(nl, 3), B, nl);
        }
        out3->batch = a->batch;
        out3->n_comp = 3;
        out3->level = a->level;
        out3->scale = a->scale * b->scale;
        return CKKS_OK;
    })
}

ckks_status ckks_relinearize(ckks_ctx* c, const ckks_ct* in3, ckks_ct* out, void* stream)
{
    CK_TRY({
        if (!c || !out || !out->data) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in3, 3);
        if (in3->data == out->data) throw CkksError(CKKS_E_SHAPE, "relinearize: out aliases in");
        const int nl = (int)in3->level + 1;
        relin_impl(c, in3->data, c->ct_words(nl, 3), nl, (int)in3->batch, out->data, c->ct_words(nl), stream);
        out->batch = in3->batch;
        out->n_comp = 2;
        out->level = in3->level;
        out->scale = in3->scale;
        return CKKS_OK;
    })
}

ckks_status ckks_rescale(ckks_ctx* c, const ckks_ct* in, ckks_ct* out, void* stream)
{
    CK_TRY({
        if (!c || !out || !out->data) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in, 0);
        if (in->n_comp < 2 || in->n_comp > 3) throw CkksError(CKKS_E_SHAPE, "rescale: 2 or 3 components");
        if (in->data == out->data) throw CkksError(CKKS_E_SHAPE, "rescale: out aliases in");
        const int nl = (int)in->level + 1, nc = (int)in->n_comp;
        rescale_impl(c, in->data, c->ct_words(nl, nc), nc, nl, (int)in->batch, out->data, c->ct_words(nl - 1, nc),
                     nullptr, stream);
        out->batch = in->batch;
        out->n_comp = in->n_comp;
        out->level = in->level - 1;
        out->scale = in->scale / (double)c->primes[in->level];
        return CKKS_OK;
    })
}

ckks_status ckks_add(ckks_ctx* c, const ckks_ct* a, const ckks_ct* b, ckks_ct* out, void* stream)
{
    CK_TRY({
        if (!c || !out || !out->data) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, a, 0);
        check_ct(c, b, 0);
        if (a->level != b->level || a->batch != b->batch || a->n_comp != b->n_comp)
            throw CkksError(CKKS_E_SHAPE, "add: shape mismatch");
        if (std::fabs(a->scale - b->scale) > std::ldexp(std::max(a->scale, b->scale), -40))
            throw CkksError(CKKS_E_SCALE, "add: scale mismatch beyond 2^-40 relative");
        const int nl = (int)a->level + 1, nc = (int)a->n_comp;
        const size_t w = c->ct_words(nl, nc);
        auto L = c->launch(stream);
        for (uint32_t b0 = 0; b0 < a->batch; b0 += 65535) {
            const int B = (int)std::min<uint32_t>(65535, a->batch - b0);
            ck::add(L, a->data + b0 * w, w, b->data + b0 * w, w, out->data + b0 * w, w, B, nc, nl);
        }
        out->batch = a->batch;
        out->n_comp = a->n_comp;
        out->level = a->level;
        out->scale = a->scale;
        return CKKS_OK;
    })
}

// ------------------------------------------------------------------------------------ layers
static size_t layer_dev_bytes(const ckks_ctx* c, size_t count, uint32_t level);

ckks_status ckks_layer_sizes(const ckks_ctx* c, uint32_t rows, uint32_t cols, uint32_t level, size_t* bytes)
{
    CK_TRY({
        if (!c || !bytes || rows == 0 || cols == 0) throw CkksError(CKKS_E_PARAM, "bad layer shape");
        if (level < 1 || (int)level >= c->L) throw CkksError(CKKS_E_LEVEL, "layer level must be in [1, L-1]");
        uint32_t t, t1, t2;
        bsgs_split(rows, cols, t, t1, t2, c->bsgs_bx);
        *bytes = layer_dev_bytes(c, t, level);
        return CKKS_OK;
    })
}

static size_t layer_dev_bytes(const ckks_ctx* c, size_t count, uint32_t level)
{
    return align256(count * (level + 1 + c->ns) * c->n * 8) + align256((size_t)level * c->n * 8) +
           align256((count > 1 ? count : 1) * c->n * 8);   // + staging for the int64 coefficients
}

static ckks_status layer_general(ckks_ctx* c, const ckks_layer_desc* d, const int64_t* pts, const int64_t* bias,
                                 void* dev_buf, void* stream, ckks_layer** out)
{
    if (d->n_baby < 1 || !d->baby_steps || d->baby_steps[0] != 0 || d->t2 < 1)
        throw CkksError(CKKS_E_PARAM, "layer: need n_baby >= 1 with baby_steps[0] == 0 and t2 >= 1");
    if (d->n_baby > 64) throw CkksError(CKKS_E_PARAM, "layer: at most 64 baby steps");
    if (d->level < 1 || (int)d->level >= c->L) throw CkksError(CKKS_E_LEVEL, "layer level must be in [1, L-1]");
    const size_t count = (size_t)d->n_baby * d->t2;
    auto* ly = new ckks_layer();
    ly->kind = d->kind;
    ly->rows = d->rows;
    ly->cols = d->cols;
    ly->t = d->t;
    ly->t1 = d->n_baby;
    ly->t2 = d->t2;
    ly->baby.assign(d->baby_steps, d->baby_steps + d->n_baby);
    ly->giant = d->giant;
    ly->region = d->region;
    ly->items = d->items ? d->items : 1;
    ly->level = d->level;
    ly->pt_scale = d->pt_scale;
    ly->bias_scale = d->bias_scale;
    const uint32_t level = d->level;
    char* base = (char*)dev_buf;
    ly->d_pts = (u64*)base;
    ly->d_bias = bias ? (u64*)(base + align256(count * (level + 1 + c->ns) * c->n * 8)) : nullptr;
    int64_t* stage =
        (int64_t*)(base + align256(count * (level + 1 + c->ns) * c->n * 8) + align256((size_t)level * c->n * 8));
    cudaStream_t st = (cudaStream_t)stream;
    auto L = c->launch(stream);
    cuda_ok(cudaMemcpyAsync(stage, pts, count * c->n * 8, cudaMemcpyHostToDevice, st), "upload plaintexts");
    ck::signed_to_ntt(L, stage, ly->d_pts, (int)count, (int)level + 1, true);
    if (bias) {
        cuda_ok(cudaStreamSynchronize(st), "sync");
        cuda_ok(cudaMemcpyAsync(stage, bias, (size_t)c->n * 8, cudaMemcpyHostToDevice, st), "upload bias");
        ck::signed_to_ntt(L, stage, ly->d_bias, 1, (int)level);
    }
    cuda_ok(cudaStreamSynchronize(st), "layer upload");
    *out = ly;
    return CKKS_OK;
}

static ckks_status layer_from_coeffs(ckks_ctx* c, const int64_t* diag, const int64_t* bias, uint32_t rows,
                                     uint32_t cols, uint32_t level, double pt_scale, double bias_scale, void* dev_buf,
                                     void* stream, ckks_layer** out, uint32_t region = 0, uint32_t items = 1)
{
    uint32_t t, t1, t2;
    bsgs_split(rows, cols, t, t1, t2, c->bsgs_bx);
    if (2 * t > (uint32_t)c->n / 2) throw CkksError(CKKS_E_PARAM, "2t exceeds the slot count");
    if (t1 > 64 || t2 > 64) throw CkksError(CKKS_E_PARAM, "t1, t2 <= 64 supported");
    std::vector<int32_t> baby(t1);
    for (uint32_t j = 0; j < t1; ++j) baby[j] = (int32_t)j;
    ckks_layer_desc d{CKKS_LAYER_DENSE, rows, cols, t, t2, t1, baby.data(), (int32_t)t1, region, items, level,
                      pt_scale, bias_scale};
    return layer_general(c, &d, diag, bias, dev_buf, stream, out);
}

ckks_status ckks_layer_import(ckks_ctx* c, const int64_t* diag_coeffs, const int64_t* bias_coeffs, uint32_t rows,
                              uint32_t cols, uint32_t level, double pt_scale, double bias_scale, void* dev_buf,
                              void* stream, ckks_layer** out)
{
    CK_TRY({
        if (!c || !diag_coeffs || !dev_buf || !out) throw CkksError(CKKS_E_PARAM, "null");
        if (level < 1 || (int)level >= c->L) throw CkksError(CKKS_E_LEVEL, "layer level must be in [1, L-1]");
        return layer_from_coeffs(c, diag_coeffs, bias_coeffs, rows, cols, level, pt_scale, bias_scale, dev_buf,
                                 stream, out);
    })
}

// library-side encodings of the layer plaintexts (NEXT f-2 packing R25: one copy per item region)
static void put_regions(std::vector<double>& v, const double* vals, uint32_t len, uint32_t region, uint32_t items,
                        uint32_t offset)
{
    for (uint32_t r = 0; r < items; ++r)
        for (uint32_t s = 0; s < len; ++s) v[(size_t)r * region + offset + s] = vals[s];
}

ckks_status ckks_dense_create_packed(ckks_ctx* c, const double* W, uint32_t rows, uint32_t cols, const double* bias,
                                     uint32_t region, uint32_t items, uint32_t level, double in_scale, void* dev_buf,
                                     void* stream, ckks_layer** out)
{
    CK_TRY({
        if (!c || !W || !dev_buf || !out) throw CkksError(CKKS_E_PARAM, "null");
        if (level < 1 || (int)level >= c->L) throw CkksError(CKKS_E_LEVEL, "layer level must be in [1, L-1]");
        uint32_t t, t1, t2;
        bsgs_split(rows, cols, t, t1, t2, c->bsgs_bx);
        const int n = c->n, slots = n / 2;
        if (items < 1) items = 1;
        if (items == 1 && region == 0) region = 2 * t;
        if (2 * t > region || (size_t)region * items > (size_t)slots)
            throw CkksError(CKKS_E_PARAM, "regions must hold 2t slots and fit the slot vector");
        const double ptscale = (double)c->primes[level];
        std::vector<int64_t> coeffs((size_t)t * n);
        std::vector<double> v(slots), dg(t);
        for (uint32_t i = 0; i < t; ++i) {
            // diag'_i = rot_{-floor(i/t1) t1}(diag_i): slots [k t1, k t1 + t) of every item (R4)
            std::fill(v.begin(), v.end(), 0.0);
            const uint32_t k = i / t1;
            for (uint32_t s = 0; s < t; ++s) {
                const uint32_t col = (s + i) % t;
                dg[s] = (s < rows && col < cols) ? W[(size_t)s * cols + col] : 0.0;
            }
            put_regions(v, dg.data(), t, region, items, k * t1);
            encode_host(n, v.data(), slots, ptscale, coeffs.data() + (size_t)i * n);
        }
        std::vector<int64_t> bcoef;
        if (bias) {
            std::fill(v.begin(), v.end(), 0.0);
            put_regions(v, bias, rows, region, items, 0);
            bcoef.resize(n);
            encode_host(n, v.data(), slots, in_scale, bcoef.data());
        }
        return layer_from_coeffs(c, coeffs.data(), bias ? bcoef.data() : nullptr, rows, cols, level, ptscale,
                                 in_scale, dev_buf, stream, out, region, items);
    })
}

ckks_status ckks_layer_create(ckks_ctx* c, const double* W, uint32_t rows, uint32_t cols, const double* bias,
                              uint32_t level, double in_scale, void* dev_buf, void* stream, ckks_layer** out)
{
    return ckks_dense_create_packed(c, W, rows, cols, bias, 0, 1, level, in_scale, dev_buf, stream, out);
}

ckks_status ckks_layer_general_sizes(const ckks_ctx* c, uint32_t n_plaintexts, uint32_t level, size_t* bytes)
{
    if (!c || !bytes || n_plaintexts == 0) return fail(CKKS_E_PARAM, "null");
    *bytes = layer_dev_bytes(c, n_plaintexts, level);
    return CKKS_OK;
}

ckks_status ckks_layer_import_general(ckks_ctx* c, const ckks_layer_desc* desc, const int64_t* pt_coeffs,
                                      const int64_t* bias_coeffs, void* dev_buf, void* stream, ckks_layer** out)
{
    CK_TRY({
        if (!c || !desc || !pt_coeffs || !dev_buf || !out) throw CkksError(CKKS_E_PARAM, "null");
        return layer_general(c, desc, pt_coeffs, bias_coeffs, dev_buf, stream, out);
    })
}

// R26: taps ordered centre first (step 0), then i - c for the others; m_i = w_i on every item's [rR, rR + t)
ckks_status ckks_conv1d_create(ckks_ctx* c, const double* w, uint32_t f, double bias, uint32_t t, uint32_t region,
                               uint32_t items, uint32_t level, double in_scale, void* dev_buf, void* stream,
                               ckks_layer** out)
{
    CK_TRY({
        if (!c || !w || !dev_buf || !out || f < 1 || f > 32 || (f & 1) == 0) throw CkksError(CKKS_E_PARAM, "conv1d: odd f in [1, 31]");
        if (level < 1 || (int)level >= c->L) throw CkksError(CKKS_E_LEVEL, "layer level must be in [1, L-1]");
        const int n = c->n, slots = n / 2;
        const uint32_t cc = (f - 1) / 2;
        if (items < 1) items = 1;
        if (region == 0) region = 2 * t + cc;
        if (t + cc > region || (size_t)region * items > (size_t)slots) throw CkksError(CKKS_E_PARAM, "conv1d: regions");
        const double ptscale = (double)c->primes[level];
        std::vector<int32_t> steps;
        std::vector<uint32_t> order;
        order.push_back(cc);
        for (uint32_t i = 0; i < f; ++i)
            if (i != cc) order.push_back(i);
        std::vector<int64_t> coeffs((size_t)f * n);
        std::vector<double> v(slots), tap(t);
        for (uint32_t o = 0; o < f; ++o) {
            steps.push_back((int32_t)order[o] - (int32_t)cc);
            std::fill(v.begin(), v.end(), 0.0);
            std::fill(tap.begin(), tap.end(), w[order[o]]);
            put_regions(v, tap.data(), t, region, items, 0);
            encode_host(n, v.data(), slots, ptscale, coeffs.data() + (size_t)o * n);
        }
        std::vector<int64_t> bcoef(n);
        std::fill(v.begin(), v.end(), 0.0);
        std::fill(tap.begin(), tap.end(), bias);
        put_regions(v, tap.data(), t, region, items, 0);
        encode_host(n, v.data(), slots, in_scale, bcoef.data());
        ckks_layer_desc d{CKKS_LAYER_CONV1D, t, t, t, 1, f, steps.data(), 0, region, items, level, ptscale, in_scale};
        return layer_general(c, &d, coeffs.data(), bcoef.data(), dev_buf, stream, out);
    })
}

// R27: out[k] = (1/f) sum_{i<f} x[k - i] on [f-1, t) of each item; steps 0, -1, .., -(f-1)
ckks_status ckks_avgpool_create(ckks_ctx* c, uint32_t f, uint32_t t, uint32_t region, uint32_t items, uint32_t level,
                                void* dev_buf, void* stream, ckks_layer** out)
{
    CK_TRY({
        if (!c || !dev_buf || !out || f < 1 || f > 32 || f > t) throw CkksError(CKKS_E_PARAM, "avgpool: 1 <= f <= min(32, t)");
        if (level < 1 || (int)level >= c->L) throw CkksError(CKKS_E_LEVEL, "layer level must be in [1, L-1]");
        const int n = c->n, slots = n / 2;
        if (items < 1) items = 1;
        if (region == 0) region = 2 * t;
        if (t > region || (size_t)region * items > (size_t)slots) throw CkksError(CKKS_E_PARAM, "avgpool: regions");
        const double ptscale = (double)c->primes[level];
        std::vector<double> v(slots, 0.0), m(t - (f - 1), 1.0 / f);
        put_regions(v, m.data(), t - (f - 1), region, items, f - 1);
        std::vector<int64_t> one(n), coeffs((size_t)f * n);
        encode_host(n, v.data(), slots, ptscale, one.data());
        std::vector<int32_t> steps;
        for (uint32_t i = 0; i < f; ++i) {
            steps.push_back(-(int32_t)i);
            std::copy(one.begin(), one.end(), coeffs.begin() + (size_t)i * n);
        }
        ckks_layer_desc d{CKKS_LAYER_AVGPOOL, t, t, t, 1, f, steps.data(), 0, region, items, level, ptscale, 0.0};
        return layer_general(c, &d, coeffs.data(), nullptr, dev_buf, stream, out);
    })
}

void ckks_layer_destroy(ckks_layer* l) { delete l; }

// baby [t1-1] + inner sums [t2] ciphertexts in the Q_l P basis (the largest of the three modes) + one
// Q_l ciphertext for the double-hoisted ModDown output
static size_t layer_work_words(const ckks_ctx* c, const ckks_layer* l, int B)
{
    const size_t ctq = c->ct_words((int)l->level + 1 + std::max(c->ns, 1));
    return ((size_t)(l->t1 - 1) + l->t2 + 1) * B * ctq;
}

ckks_status ckks_layer_work_sizes(const ckks_ctx* c, const ckks_layer* l, uint32_t batch, size_t* bytes)
{
    if (!c || !l || !bytes) return fail(CKKS_E_PARAM, "null");
    const int B = (int)std::min<uint32_t>(batch ? batch : 1, c->max_batch);
    *bytes = align256(layer_work_words(c, l, B) * 8);
    return CKKS_OK;
}

// Every Galois / relinearisation key a layer or a model needs, checked before anything is launched
// (ckks.h: "on error nothing has been launched").
static void require_step_key(const ckks_ctx* c, int64_t step)
{
    const uint32_t g = c->galois(step);
    if (g != 1 && !c->key((int64_t)g)) throw CkksError(CKKS_E_NOKEY, "no Galois key for step " + std::to_string(step));
}
static void check_layer_keys(const ckks_ctx* c, const ckks_layer* ly, int hoisting)
{
    for (uint32_t j = 1; j < ly->t1; ++j) require_step_key(c, ly->baby[j]);
    for (uint32_t k = 1; k < ly->t2; ++k) {
        const int64_t step = (int64_t)k * ly->giant;
        if (hoisting == 2 && c->galois(step) == 1) throw CkksError(CKKS_E_PARAM, "giant step congruent to 0 mod N/2");
        require_step_key(c, step);
    }
}
// the scales a forward from in_scale produces must be the ones the cubic constants were encoded for
static void check_model_scales(const ckks_ctx* c, const ckks_model* m, double scale)
{
    int level = (int)m->stages[0].layer->level;
    for (size_t si = 0; si < m->stages.size(); ++si) {
        const auto& sg = m->stages[si];
        scale = scale * sg.layer->pt_scale / (double)c->primes[level];
        level -= 1;
        if (sg.activation == 1) {
            scale = scale * scale / (double)c->primes[level];
            level -= 1;
        } else if (sg.activation == 2) {
            const double S = m->act_scale[si];
            if (std::fabs(scale - S) > std::ldexp(S, -40))
                throw CkksError(CKKS_E_SCALE, "cubic activation input scale differs from the model's encoding");
            scale = (S * S / (double)c->primes[level]) * S / (double)c->primes[level - 1];
            level -= 2;
        }
    }
}

static void check_model_keys(const ckks_ctx* c, const ckks_model* m)
{
    for (const auto& sg : m->stages) {
        if (sg.replicate_t) require_step_key(c, -(int64_t)sg.replicate_t);
        check_layer_keys(c, sg.layer, m->hoisted);
        if (sg.activation && !c->key(0)) throw CkksError(CKKS_E_NOKEY, "no relinearisation key");
    }
}

// matvec on B ciphertexts (B <= max_batch): in -> out (level-1), work holds baby + W.
// hoisting 0: every rotation non-hoisted (R11); 1: baby steps hoisted (R11b); 2: double hoisting (R11c)
static void matvec_chunk(ckks_ctx* c, const ckks_layer* ly, const u64* in, size_t in_stride, int B, u64* out,
                         size_t out_stride, u64* work, void* stream, int hoisting = 0)
{
    const int nl = (int)ly->level + 1;
    auto L = c->launch(stream);
    if (hoisting == 2) {
        const size_t ctq = c->ct_words(nl + c->ns), ctw = c->ct_words(nl);
        u64* baby = work;                                   // [t1-1][B][2][nl+1][N]
        u64* Wk = work + (size_t)(ly->t1 - 1) * B * ctq;    // [t2][B][2][nl+1][N]
        u64* md = Wk + (size_t)ly->t2 * B * ctq;            // [B][2][nl][N]
        std::vector<int64_t> steps;
        std::vector<u64*> outs;
        for (uint32_t j = 1; j < ly->t1; ++j) {
            steps.push_back((int64_t)ly->baby[j]);
            outs.push_back(baby + (size_t)(j - 1) * B * ctq);
        }
        // the tensor-core MAC reads the baby steps in its own layout, which the tensor-core baby-step inner
        // product writes: used when every baby-step group of KS_GMAX rotations has >= 2 members and no baby step
        // is the identity
        bool mac_layout = ck::bsgs_mac_tc_enabled(L, (int)ly->t1, B) && (steps.size() % KS_GMAX) != 1;
        for (int64_t st : steps) mac_layout = mac_layout && c->galois(st) != 1;
        if (!steps.empty())
            rotate_hoisted_qp_impl(c, in, in_stride, nl, B, steps.data(), (int)steps.size(), outs.data(), ctq, stream,
                                   mac_layout);
        ck::bsgs_mac(L, ly->d_pts, nl + c->ns, in, in_stride, baby, Wk, (int)ly->t1, (int)ly->t2, B, nl, true,
                     mac_layout);
        // giant steps: every step's digits / ModUp first (each into its own scratch, carved from the baby-step
        // buffer, which is dead after the inner sums), then ONE pass over the accumulator for up to KS_GMAX steps
        // (k_ks_ip_giant_multi); the per-step form (one accumulator pass per step) when the scratch does not fit
        const int G = (int)ly->t2 - 1, nd = L.active_digits(nl), ne = nl + c->ns;
        const size_t step_words = (size_t)B * c->n * ((size_t)nl + (size_t)nd * ne + (size_t)c->ns);
        const bool multi = ck::get_giant_multi() && G >= 1 && nd <= 5 &&
                           (size_t)std::min(G, IPGM_GMAX) * step_words <= (size_t)(ly->t1 - 1) * B * ctq;
        if (multi) {
            for (int g0 = 0; g0 < G; g0 += IPGM_GMAX) {
                const int gn = std::min(IPGM_GMAX, G - g0);
                const u64 *modup[KS_GMAX], *keys[KS_GMAX], *adds[KS_GMAX];
                uint32_t gal[KS_GMAX];
                for (int gi = 0; gi < gn; ++gi) {
                    const uint32_t k = (uint32_t)(g0 + gi + 1);
                    const int64_t step = (int64_t)k * ly->giant;
                    const uint32_t g = c->galois(step);
                    if (g == 1) throw CkksError(CKKS_E_PARAM, "giant step congruent to 0 mod N/2");
                    const u64* key = c->key((int64_t)g);
                    if (!key) throw CkksError(CKKS_E_NOKEY, "no Galois key for step " + std::to_string(step));
                    ck::KsWork w{};
                    u64* p = baby + (size_t)gi * step_words;
                    w.digits = p;
                    w.modup = p + (size_t)B * nl * c->n;
                    w.rem = w.modup + (size_t)B * nd * ne * c->n;
                    const u64* wk = Wk + (size_t)k * B * ctq;
                    ck::KsIn ki{wk, ctq, (size_t)ne * c->n, g};
                    ck::keyswitch_modup(L, ki, B, nl, w, true);
                    modup[gi] = w.modup;
                    keys[gi] = key;
                    adds[gi] = wk;
                    gal[gi] = g;
                }
                if (!ck::ip_giant_multi(L, gn, modup, keys, adds, gal, B, nl, Wk, ctq, ctq))
                    throw CkksError(CKKS_E_PARAM, "ip_giant_multi not applicable");
            }
        } else {
            for (uint32_t k = 1; k < ly->t2; ++k)
                rotate_qp_impl(c, Wk + (size_t)k * B * ctq, ctq, nl, B, (int64_t)k * ly->giant, Wk, ctq, stream);
        }
        ck::moddown_qp(L, Wk, ctq, B, nl, c->ks_work(B), md, ctw);
        rescale_impl(c, md, ctw, 2, nl, B, out, out_stride, ly->d_bias, stream);
        return;
    }
    const size_t ctw = c->ct_words(nl);
    u64* baby = work;                                   // [t1-1][B][2][nl][N]
    u64* Wk = work + (size_t)(ly->t1 - 1) * B * ctw;    // [t2][B][2][nl][N]
    if (hoisting == 1) {
        std::vector<int64_t> steps;
        std::vector<u64*> outs;
        for (uint32_t j = 1; j < ly->t1; ++j) {
            steps.push_back((int64_t)ly->baby[j]);
            outs.push_back(baby + (size_t)(j - 1) * B * ctw);
        }
        if (!steps.empty())
            rotate_hoisted_impl(c, in, in_stride, nl, B, steps.data(), (int)steps.size(), outs.data(), ctw, stream);
    } else {
        for (uint32_t j = 1; j < ly->t1; ++j)
            rotate_impl(c, in, in_stride, nl, B, (int64_t)ly->baby[j], baby + (size_t)(j - 1) * B * ctw, ctw, false,
                        stream);
    }
    ck::bsgs_mac(L, ly->d_pts, nl + c->ns, in, in_stride, baby, Wk, (int)ly->t1, (int)ly->t2, B, nl, false);
    for (uint32_t k = 1; k < ly->t2; ++k)
        rotate_impl(c, Wk + (size_t)k * B * ctw, ctw, nl, B, (int64_t)k * ly->giant, Wk, ctw, true, stream);
    rescale_impl(c, Wk, ctw, 2, nl, B, out, out_stride, ly->d_bias, stream);
}

ckks_status ckks_matvec_diag(ckks_ctx* c, const ckks_layer* ly, const ckks_ct* in, ckks_ct* out, void* work,
                             void* stream)
{
    CK_TRY({
        if (!c || !ly || !out || !out->data || !work) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in);
        if (in->level != ly->level) throw CkksError(CKKS_E_SHAPE, "input level != layer level");
        check_layer_keys(c, ly, ly->hoisting);
        const int nl = (int)in->level + 1;
        for (uint32_t b0 = 0; b0 < in->batch; b0 += c->max_batch) {
            const int B = (int)std::min<uint32_t>(c->max_batch, in->batch - b0);
            matvec_chunk(c, ly, in->data + (size_t)b0 * c->ct_words(nl), c->ct_words(nl), B,
                         out->data + (size_t)b0 * c->ct_words(nl - 1), c->ct_words(nl - 1), (u64*)work, stream,
                         ly->hoisting);
        }
        out->batch = in->batch;
        out->n_comp = 2;
        out->level = in->level - 1;
        out->scale = in->scale * ly->pt_scale / (double)c->primes[in->level];
        return CKKS_OK;
    })
}

// ------------------------------------------------------------------------------------ model
// residues of a signed integer constant m0 modulo q_0..q_{nl-1} (a constant plaintext at coefficient 0 has
// the NTT value m0 mod q_i in every slot, R23)
static void const_residues(const ckks_ctx* c, int64_t m0, int nl, u64* out)
{
    for (int i = 0; i < nl; ++i) {
        const u64 q = c->primes[i];
        out[i] = m0 >= 0 ? (u64)m0 % q : (q - ((u64)(-(m0 + 1)) + 1) % q) % q;
    }
}

static int64_t round_away(double x) { return (int64_t)((x < 0 ? -1.0 : 1.0) * std::floor(std::fabs(x) + 0.5)); }

// per cubic stage: the masked c0 plaintext [L][N] and the constant residues [3][CKKS_MAXP] of c3, c2, c1
// (computed once at model creation, so the forward issues no host->device copy); + one N-word staging row
#define ACT_CONST_WORDS (3 * CKKS_MAXP)
static size_t stages_dev_words(const ckks_ctx* c, const ckks_stage* st, uint32_t n)
{
    size_t cub = 0;
    for (uint32_t i = 0; i < n; ++i) cub += st[i].activation == 2 ? 1 : 0;
    return cub ? cub * ((size_t)c->L * c->n + ACT_CONST_WORDS) + c->n : 0;
}

static int stage_level_drop(int act) { return act == 1 ? 1 : act == 2 ? 2 : 0; }

static ckks_model* build_model(ckks_ctx* c, const ckks_stage* st, uint32_t n, const int64_t* act_coeffs, void* dev_buf,
                               void* stream)
{
    if (!st || n == 0) throw CkksError(CKKS_E_PARAM, "empty model");
    int lvl = (int)st[0].layer->level;
    for (uint32_t i = 0; i < n; ++i) {
        if (!st[i].layer) throw CkksError(CKKS_E_PARAM, "null layer");
        if (st[i].activation < 0 || st[i].activation > 2) throw CkksError(CKKS_E_PARAM, "activation 0|1|2");
        if ((int)st[i].layer->level != lvl)
            throw CkksError(CKKS_E_LEVEL, "stage " + std::to_string(i) + " encoded for the wrong level");
        lvl -= 1 + stage_level_drop(st[i].activation);
    }
    if (lvl < 0) throw CkksError(CKKS_E_LEVEL, "model deeper than the chain");
    const size_t dw = stages_dev_words(c, st, n);
    if (dw && !dev_buf) throw CkksError(CKKS_E_PARAM, "cubic activation needs the model device buffer");
    auto* m = new ckks_model();
    m->activation = st[0].activation;
    u64* next = (u64*)dev_buf;
    int64_t* stage_buf = dw ? (int64_t*)((u64*)dev_buf + dw - c->n) : nullptr;
    auto L = c->launch(stream);
    cudaStream_t cs = (cudaStream_t)stream;
    std::vector<int64_t> coef(c->n);
    std::vector<double> v(c->n / 2);
    for (uint32_t i = 0; i < n; ++i) {
        m->layers.push_back(st[i].layer);
        m->stages.push_back(Stage{st[i].layer, st[i].activation, st[i].replicate_t});
        u64* dact = nullptr;
        if (st[i].activation == 2) {
            const ckks_layer* ly = st[i].layer;
            const int l = (int)ly->level - 1;   // activation input level
            if (l < 2) throw CkksError(CKKS_E_LEVEL, "cubic activation needs two more levels");
            const double S = ly->bias_scale, ql = (double)c->primes[l], ql1 = (double)c->primes[l - 1];
            const double S3 = (S * S / ql) * S / ql1;
            const int64_t* src = act_coeffs ? act_coeffs + (size_t)i * c->n : nullptr;
            if (!src) {
                // c0 of Eq. 2 on the layer's valid output slots [rR, rR + rows) of every item (R23, R25)
                std::fill(v.begin(), v.end(), 0.0);
                const uint32_t R = ly->region ? ly->region : 2 * ly->t;
                for (uint32_t r = 0; r < ly->items; ++r)
                    for (uint32_t s = 0; s < ly->rows; ++s) v[(size_t)r * R + s] = 0.49383;
                encode_host(c->n, v.data(), v.size(), S3, coef.data());
                src = coef.data();
            }
            dact = next;
            next += (size_t)c->L * c->n;
            // Eq. 2 constants of the R23 schedule: c3 at scale q_l (l + 1 limbs), c2 at S (l limbs), c1 at
            // S3 q_l / S (l + 1 limbs)
            const double c3 = -0.0061728, c2 = 0.092593, c1 = 0.59259;
            u64 cres[ACT_CONST_WORDS] = {};
            const_residues(c, round_away(c3 * ql), l + 1, cres);
            const_residues(c, round_away(c2 * S), l, cres + CKKS_MAXP);
            const_residues(c, round_away(c1 * (S3 * ql / S)), l + 1, cres + 2 * CKKS_MAXP);
            u64* dconst = next;
            next += ACT_CONST_WORDS;
            cuda_ok(cudaMemcpyAsync(stage_buf, src, (size_t)c->n * 8, cudaMemcpyHostToDevice, cs), "act upload");
            ck::signed_to_ntt(L, stage_buf, dact, 1, l - 1);
            cuda_ok(cudaMemcpyAsync(dconst, cres, sizeof(cres), cudaMemcpyHostToDevice, cs), "act upload");
            cuda_ok(cudaStreamSynchronize(cs), "act upload");
            m->d_act_const.push_back(dconst);
            m->act_scale.push_back(S);
        }
        m->d_act_stage.push_back(dact);
        if (!dact) {
            m->d_act_const.push_back(nullptr);
            m->act_scale.push_back(0.0);
        }
    }
    return m;
}

ckks_status ckks_model_sizes(const ckks_ctx* c, uint32_t n_layers, int32_t activation, size_t* bytes)
{
    if (!c || !bytes) return fail(CKKS_E_PARAM, "null");
    std::vector<ckks_stage> st(n_layers ? n_layers : 1);
    for (uint32_t i = 0; i < n_layers; ++i) st[i].activation = (i + 1 < n_layers) ? activation : 0;
    *bytes = align256(stages_dev_words(c, st.data(), n_layers) * 8);
    return CKKS_OK;
}

ckks_status ckks_model_create(ckks_ctx* c, const ckks_layer* const* layers, uint32_t n_layers, int32_t activation,
                              const int64_t* act_coeffs, void* dev_buf, void* stream, ckks_model** out)
{
    CK_TRY({
        if (!c || !layers || !out || n_layers == 0) throw CkksError(CKKS_E_PARAM, "null/empty model");
        if (activation < 0 || activation > 2) throw CkksError(CKKS_E_PARAM, "activation 0|1|2");
        // dense_1 -> act -> replicate -> dense_2 -> ... (PAPER.md L118 shape, BASELINE cfg4)
        std::vector<ckks_stage> st(n_layers);
        for (uint32_t i = 0; i < n_layers; ++i) {
            st[i].layer = layers[i];
            st[i].activation = (i + 1 < n_layers) ? activation : 0;
            st[i].replicate_t = i > 0 ? layers[i]->t : 0;
        }
        *out = build_model(c, st.data(), n_layers, act_coeffs, dev_buf, stream);
        (*out)->activation = activation;
        return CKKS_OK;
    })
}

ckks_status ckks_model_stages_sizes(const ckks_ctx* c, const ckks_stage* stages, uint32_t n, size_t* bytes)
{
    if (!c || !stages || !bytes) return fail(CKKS_E_PARAM, "null");
    *bytes = align256(stages_dev_words(c, stages, n) * 8);
    return CKKS_OK;
}

ckks_status ckks_model_create_stages(ckks_ctx* c, const ckks_stage* stages, uint32_t n, const int64_t* act_coeffs,
                                     void* dev_buf, void* stream, ckks_model** out)
{
    CK_TRY({
        if (!c || !stages || !out || n == 0) throw CkksError(CKKS_E_PARAM, "null/empty model");
        *out = build_model(c, stages, n, act_coeffs, dev_buf, stream);
        return CKKS_OK;
    })
}

void ckks_model_destroy(ckks_model* m) { delete m; }

ckks_status ckks_bsgs_plan(uint32_t rows, uint32_t cols, uint32_t* t, uint32_t* t1, uint32_t* t2)
{
    return ckks_bsgs_plan_x(rows, cols, 0, t, t1, t2);
}

ckks_status ckks_bsgs_plan_x(uint32_t rows, uint32_t cols, uint32_t x, uint32_t* t, uint32_t* t1, uint32_t* t2)
{
    if (!rows || !cols || !t || !t1 || !t2) return fail(CKKS_E_PARAM, "bad shape");
    if (x > 4) return fail(CKKS_E_PARAM, "x must be <= 4");
    bsgs_split(rows, cols, *t, *t1, *t2, x);
    return CKKS_OK;
}

ckks_status ckks_model_steps(uint32_t n_layers, const uint32_t* rows, const uint32_t* cols, uint32_t x, int32_t* steps,
                             uint32_t* n_steps)
{
    CK_TRY({
        if (!rows || !cols || !n_steps || n_layers == 0) throw CkksError(CKKS_E_PARAM, "null");
        if (x > 4) throw CkksError(CKKS_E_PARAM, "x must be <= 4");
        std::vector<int32_t> st;
        for (uint32_t i = 0; i < n_layers; ++i) {
            uint32_t t, t1, t2;
            bsgs_split(rows[i], cols[i], t, t1, t2, x);
            for (uint32_t j = 1; j < t1; ++j) st.push_back((int32_t)j);
            for (uint32_t k = 1; k < t2; ++k) st.push_back((int32_t)(k * t1));
            if (i > 0) st.push_back(-(int32_t)t);
        }
        std::sort(st.begin(), st.end());
        st.erase(std::unique(st.begin(), st.end()), st.end());
        if (steps) {
            if (st.size() > *n_steps) throw CkksError(CKKS_E_SIZE, "steps buffer too small");
            std::copy(st.begin(), st.end(), steps);
        }
        *n_steps = (uint32_t)st.size();
        return CKKS_OK;
    })
}

ckks_status ckks_model_plan(const ckks_ctx* c, uint32_t n_layers, const uint32_t* rows, const uint32_t* cols,
                            int32_t activation, uint32_t in_level, double in_scale, uint32_t* layer_level,
                            double* layer_in_scale, int32_t* steps, uint32_t* n_steps)
{
    CK_TRY({
        if (!c || !rows || !cols || !layer_level || !layer_in_scale || !n_steps || n_layers == 0)
            throw CkksError(CKKS_E_PARAM, "null");
        std::vector<int32_t> st;
        int lvl = (int)in_level;
        double s = in_scale;
        for (uint32_t i = 0; i < n_layers; ++i) {
            uint32_t t, t1, t2;
            bsgs_split(rows[i], cols[i], t, t1, t2, c->bsgs_bx);
            if (lvl < 1) throw CkksError(CKKS_E_LEVEL, "model deeper than the chain");
            layer_level[i] = (uint32_t)lvl;
            layer_in_scale[i] = s;
            for (uint32_t j = 1; j < t1; ++j) st.push_back((int32_t)j);
            for (uint32_t k = 1; k < t2; ++k) st.push_back((int32_t)(k * t1));
            if (i > 0) st.push_back(-(int32_t)t);
            lvl -= 1;                       // dense: pt scale q_l, one rescale -> scale unchanged (R8)
            if (i + 1 < n_layers) {
                if (activation == 1) {
                    s = s * s / (double)c->primes[lvl];
                    lvl -= 1;
                } else if (activation == 2) {
                    const double ql = (double)c->primes[lvl], ql1 = (double)c->primes[lvl - 1];
                    s = (s * s / ql) * s / ql1;
                    lvl -= 2;
                }
            }
        }
        if (lvl < 0) throw CkksError(CKKS_E_LEVEL, "model deeper than the chain");
        std::sort(st.begin(), st.end());
        st.erase(std::unique(st.begin(), st.end()), st.end());
        if (steps) {
            if (st.size() > *n_steps) throw CkksError(CKKS_E_SIZE, "steps buffer too small");
            std::copy(st.begin(), st.end(), steps);
        }
        *n_steps = (uint32_t)st.size();
        return CKKS_OK;
    })
}

static size_t model_work_words(const ckks_ctx* c, const ckks_model* m, int B)
{
    size_t lw = 0;
    for (auto* l : m->layers) lw = std::max(lw, layer_work_words(c, l, B));
    const size_t big = (size_t)B * c->ct_words(c->L, 3);
    return lw + 4 * big;
}
// + host-path staging: one chunk of input and one of output ciphertexts
// host-buffer forward staging: two input and two output chunk buffers (double buffering)
static size_t host_stage_words(const ckks_ctx* c, int B) { return (size_t)2 * B * 2 * c->ct_words(c->L); }

ckks_status ckks_model_work_sizes(const ckks_ctx* c, const ckks_model* m, uint32_t batch, size_t* bytes)
{
    if (!c || !m || !bytes) return fail(CKKS_E_PARAM, "null");
    const int B = (int)std::min<uint32_t>(batch ? batch : 1, c->max_batch);
    *bytes = align256((model_work_words(c, m, B) + host_stage_words(c, B)) * 8);
    return CKKS_OK;
}


// One chunk of B ciphertexts through the model's stages.  in: [B][2][l0+1][N]; out: final level.
static void forward_chunk(ckks_ctx* c, const ckks_model* m, const u64* in, size_t in_stride, int B, double in_scale,
                          u64* out, size_t out_stride, u64* work, void* stream, int* out_level, double* out_scale)
{
    const size_t big = (size_t)B * c->ct_words(c->L, 3);
    size_t lw = 0;
    for (auto* l : m->layers) lw = std::max(lw, layer_work_words(c, l, B));
    u64* lwork = work;
    u64* bufA = work + lw;
    u64* bufB = bufA + big;
    u64* bufC = bufB + big;
    u64* bufD = bufC + big;
    auto L = c->launch(stream);
    const u64* cur = in;
    size_t cur_stride = in_stride;
    double scale = in_scale;
    int level = (int)m->stages[0].layer->level;
    const int nst = (int)m->stages.size();
    for (int si = 0; si < nst; ++si) {
        const Stage& sg = m->stages[si];
        const ckks_layer* ly = sg.layer;
        int nl = level + 1;
        if (sg.replicate_t) {
            // replicate: y + rot_{-t}(y)  (P:L116 duplicated layout)
            const size_t ctw = c->ct_words(nl);
            u64* rep = (cur == bufA) ? bufB : bufA;
            cuda_ok(cudaMemcpy2DAsync(rep, ctw * 8, cur, cur_stride * 8, ctw * 8, B, cudaMemcpyDeviceToDevice,
                                      (cudaStream_t)stream), "replicate copy");
            rotate_impl(c, cur, cur_stride, nl, B, -(int64_t)sg.replicate_t, rep, ctw, true, stream);
            cur = rep;
            cur_stride = ctw;
        }
        const bool last = (si == nst - 1);
        const bool to_out = last && sg.activation == 0;
        u64* dst = to_out ? out : ((cur == bufA) ? bufB : bufA);
        const size_t dst_stride = to_out ? out_stride : c->ct_words(nl - 1);
        matvec_chunk(c, ly, cur, cur_stride, B, dst, dst_stride, lwork, stream, m->hoisted);
        scale = scale * ly->pt_scale / (double)c->primes[level];
        level -= 1;
        nl -= 1;
        cur = dst;
        cur_stride = dst_stride;
        if (sg.activation == 1) {
            // square: rescale(relin(z (x) z))
            const size_t w3 = c->ct_words(nl, 3), w2 = c->ct_words(nl);
            ck::tensor(L, cur, cur, cur_stride, bufC, w3, B, nl);
            relin_impl(c, bufC, w3, nl, B, bufD, w2, stream);
            u64* nxt = last ? out : ((cur == bufA) ? bufB : bufA);
            const size_t ns = last ? out_stride : c->ct_words(nl - 1);
            rescale_impl(c, bufD, w2, 2, nl, B, nxt, ns, nullptr, stream);
            scale = scale * scale / (double)c->primes[level];
            level -= 1;
            cur = nxt;
            cur_stride = ns;
        } else if (sg.activation == 2) {
            // Eq. 2 cubic, schedule R23
            const double S = scale, ql = (double)c->primes[level], ql1 = (double)c->primes[level - 1];
            const size_t w3 = c->ct_words(nl, 3), w2 = c->ct_words(nl), w2m = c->ct_words(nl - 1),
                         w2mm = c->ct_words(nl - 2);
            u64* z = (u64*)cur;   // level l, in bufA or bufB
            u64* other = (cur == bufA) ? bufB : bufA;
            // z2 = rescale(relin(z (x) z)) -> other  (level l-1)
            ck::tensor(L, z, z, cur_stride, bufC, w3, B, nl);
            relin_impl(c, bufC, w3, nl, B, bufD, w2, stream);
            rescale_impl(c, bufD, w2, 2, nl, B, other, w2m, nullptr, stream);
            u64* z2 = other;
            // a = rescale(z o [c3]_{ql}) + [c2]_S  -> bufD (level l-1); constants precomputed at model creation
            const u64* dres = m->d_act_const[si];
            ck::mul_scalar(L, z, cur_stride, bufC, w2, dres, B, 2, nl);
            rescale_impl(c, bufC, w2, 2, nl, B, bufD, w2m, nullptr, stream);
            ck::add_scalar(L, bufD, w2m, dres + CKKS_MAXP, B, nl - 1);
            // h = rescale(relin(z2 (x) a)) (level l-2)
            ck::tensor(L, z2, bufD, w2m, bufC, c->ct_words(nl - 1, 3), B, nl - 1);
            u64* rl = other;   // z2 is dead after the tensor
            relin_impl(c, bufC, c->ct_words(nl - 1, 3), nl - 1, B, rl, w2m, stream);
            u64* h = bufD;   // a no longer needed
            rescale_impl(c, rl, w2m, 2, nl - 1, B, h, w2mm, nullptr, stream);
            const double S3 = (S * S / ql) * S / ql1;
            // g = drop(rescale(z o [c1]_{S3 ql / S})) + [c0]_{S3} -> accumulate into h
            ck::mul_scalar(L, z, cur_stride, bufC, w2, dres + 2 * CKKS_MAXP, B, 2, nl);
            u64* g = other;   // z2 no longer needed
            rescale_impl(c, bufC, w2, 2, nl, B, g, w2m, nullptr, stream);
            // h += drop(g): add the first nl-2 limbs of each component of g
            ck::add(L, h, w2mm, g, w2m, h, w2mm, B, 1, nl - 2);
            ck::add(L, h + (size_t)(nl - 2) * c->n, w2mm, g + (size_t)(nl - 1) * c->n, w2m, h + (size_t)(nl - 2) * c->n,
                    w2mm, B, 1, nl - 2);
            // + c0 on the valid slots (model plaintext, R23)
            ck::add(L, h, w2mm, m->d_act_stage[si], 0, h, w2mm, B, 1, nl - 2);
            u64* nxt = last ? out : ((cur == bufA) ? bufB : bufA);
            const size_t ns = last ? out_stride : w2mm;
            cuda_ok(cudaMemcpy2DAsync(nxt, ns * 8, h, w2mm * 8, w2mm * 8, B, cudaMemcpyDeviceToDevice,
                                      (cudaStream_t)stream), "mv");
            scale = S3;
            level -= 2;
            cur = nxt;
            cur_stride = ns;
        }
    }
    *out_level = level;
    *out_scale = scale;
}

static int model_out_level(const ckks_model* m)
{
    int lvl = (int)m->stages[0].layer->level;
    for (const auto& s : m->stages) lvl -= 1 + stage_level_drop(s.activation);
    return lvl;
}

ckks_status ckks_model_levels(const ckks_model* m, uint32_t* in_level, uint32_t* out_level)
{
    if (!m || !in_level || !out_level) return fail(CKKS_E_PARAM, "null");
    *in_level = m->stages[0].layer->level;
    *out_level = (uint32_t)model_out_level(m);
    return CKKS_OK;
}

ckks_status ckks_encrypted_forward(ckks_ctx* c, const ckks_model* m, const ckks_ct* in, ckks_ct* out, void* work,
                                   void* stream)
{
    CK_TRY({
        if (!c || !m || !out || !out->data || !work) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in);
        if (in->level != m->stages[0].layer->level) throw CkksError(CKKS_E_SHAPE, "input level != first layer level");
        check_model_keys(c, m);
        check_model_scales(c, m, in->scale);
        const int nl_in = (int)in->level + 1, ol = model_out_level(m);
        int lvl = 0;
        double sc = 0;
        for (uint32_t b0 = 0; b0 < in->batch; b0 += c->max_batch) {
            const int B = (int)std::min<uint32_t>(c->max_batch, in->batch - b0);
            forward_chunk(c, m, in->data + (size_t)b0 * c->ct_words(nl_in), c->ct_words(nl_in), B, in->scale,
                          out->data + (size_t)b0 * c->ct_words(ol + 1), c->ct_words(ol + 1), (u64*)work, stream, &lvl,
                          &sc);
        }
        out->batch = in->batch;
        out->n_comp = 2;
        out->level = (uint32_t)lvl;
        out->scale = sc;
        return CKKS_OK;
    })
}

ckks_status ckks_encrypted_forward_host(ckks_ctx* c, const ckks_model* m, const uint64_t* h_in, uint32_t batch,
                                        uint32_t in_level, double in_scale, uint64_t* h_out, uint32_t* out_level,
                                        double* out_scale, void* work, void* stream)
{
    CK_TRY({
        if (!c || !m || !h_in || !h_out || !work) throw CkksError(CKKS_E_PARAM, "null");
        if (in_level != m->stages[0].layer->level) throw CkksError(CKKS_E_SHAPE, "input level != first layer level");
        check_model_keys(c, m);
        check_model_scales(c, m, in_scale);
        const int nl_in = (int)in_level + 1, ol = model_out_level(m);
        if (batch == 0) throw CkksError(CKKS_E_SHAPE, "empty batch");
        // chunks never exceed Bw = min(batch, max_batch): the workspace ckks_model_work_sizes(batch) returns
        // is laid out for Bw ciphertexts (model work, then the staging buffers below)
        const int Bmax = (int)std::min<uint32_t>(batch, c->max_batch);
        // device staging after the model workspace: 2 x [Bmax] input cts + 2 x [Bmax] output cts.  Chunk c
        // uses buffer c % 2; H2D of chunk c+1 and D2H of chunk c-1 run on their own streams (separate
        // copy engines, PCIe full duplex) while chunk c is evaluated on `stream`; events order the reuse.
        const size_t mw = model_work_words(c, m, Bmax);
        const size_t in_w = (size_t)Bmax * c->ct_words(nl_in), out_w = (size_t)Bmax * c->ct_words(ol + 1);
        u64* d_in[2] = {(u64*)work + mw, (u64*)work + mw + in_w};
        u64* d_out[2] = {(u64*)work + mw + 2 * in_w, (u64*)work + mw + 2 * in_w + out_w};
        cudaStream_t st = (cudaStream_t)stream;
        c->ensure_copy_streams();
        cudaStream_t sh = c->h2d_st, sd = c->d2h_st;
        int lvl = 0;
        double sc = 0;
        cuda_ok(cudaEventRecord(c->ev_ready, st), "event");          // work/staging free w.r.t. earlier calls
        cuda_ok(cudaStreamWaitEvent(sh, c->ev_ready, 0), "wait");
        int ci = 0;
        // the first chunk is a quarter chunk, so the exposed H2D before the first evaluation (and, through
        // the shifted boundaries, the D2H after the last) is short; all later chunks are Bmax
        const uint32_t first = batch > (uint32_t)Bmax ? std::max<uint32_t>(1, (uint32_t)Bmax / 4) : (uint32_t)Bmax;
        for (uint32_t b0 = 0; b0 < batch; b0 += (ci == 0 ? first : (uint32_t)Bmax), ++ci) {
            const int B = (int)std::min<uint32_t>(ci == 0 ? first : (uint32_t)Bmax, batch - b0), k = ci & 1;
            if (ci >= 2) cuda_ok(cudaStreamWaitEvent(sh, c->ev_done[k], 0), "wait");          // forward(ci-2) read d_in[k]
            cuda_ok(cudaMemcpyAsync(d_in[k], h_in + (size_t)b0 * c->ct_words(nl_in), (size_t)B * c->ct_words(nl_in) * 8,
                                    cudaMemcpyHostToDevice, sh), "h2d");
            cuda_ok(cudaEventRecord(c->ev_h2d[k], sh), "event");
            cuda_ok(cudaStreamWaitEvent(st, c->ev_h2d[k], 0), "wait");
            if (ci >= 2) cuda_ok(cudaStreamWaitEvent(st, c->ev_d2h[k], 0), "wait");          // D2H(ci-2) read d_out[k]
            forward_chunk(c, m, d_in[k], c->ct_words(nl_in), B, in_scale, d_out[k], c->ct_words(ol + 1), (u64*)work,
                          stream, &lvl, &sc);
            cuda_ok(cudaEventRecord(c->ev_done[k], st), "event");
            cuda_ok(cudaStreamWaitEvent(sd, c->ev_done[k], 0), "wait");
            cuda_ok(cudaMemcpyAsync(h_out + (size_t)b0 * c->ct_words(ol + 1), d_out[k],
                                    (size_t)B * c->ct_words(ol + 1) * 8, cudaMemcpyDeviceToHost, sd), "d2h");
            cuda_ok(cudaEventRecord(c->ev_d2h[k], sd), "event");
        }
        cuda_ok(cudaEventRecord(c->ev_ready, sd), "event");
        cuda_ok(cudaStreamWaitEvent(st, c->ev_ready, 0), "wait");    // the caller's stream sees every copy
        cuda_ok(cudaStreamSynchronize(st), "forward_host");
        if (out_level) *out_level = (uint32_t)lvl;
        if (out_scale) *out_scale = sc;
        return CKKS_OK;
    })
}

// ------------------------------------------------------------------------------------ CUDA graphs
// The launch sequence of one forward (SURVEY 3 stack 4, 8(a) row a12 "launch overhead (CUDA graph)") is
// captured once on a context-owned capture stream and replayed with one cudaGraphLaunch: for a single
// ciphertext (cfg1, cfg4 latency) the ~100-300 kernels are each a few microseconds, so the host launch
// cost would otherwise dominate.  The graph binds the buffers it was captured with.
struct ckks_graph {
    ckks_ctx* ctx = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    unsigned long long kernels = 0;   // kernels per replay (bench gpu_launches)
};

ckks_status ckks_forward_graph_create(ckks_ctx* c, const ckks_model* m, const ckks_ct* in, ckks_ct* out, void* work,
                                      void* stream, ckks_graph** out_graph)
{
    CK_TRY({
        if (!c || !m || !in || !out || !out->data || !work || !out_graph) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in);
        if (in->level != m->stages[0].layer->level) throw CkksError(CKKS_E_SHAPE, "input level != first layer level");
        if (in->batch > c->max_batch) throw CkksError(CKKS_E_SIZE, "graph forward: batch above max_batch");
        check_model_keys(c, m);
        check_model_scales(c, m, in->scale);
        cudaStream_t cap;
        cuda_ok(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
        // the capture stream starts after everything already queued on the caller's stream
        cudaEvent_t ev;
        cuda_ok(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
        cuda_ok(cudaEventRecord(ev, (cudaStream_t)stream), "event");
        cuda_ok(cudaStreamWaitEvent(cap, ev, 0), "wait");
        cuda_ok(cudaStreamSynchronize(cap), "sync");
        cudaEventDestroy(ev);
        const int probe_kind = c->probe.kind;
        c->probe.kind = ck::PROBE_OFF;   // no event records inside the graph
        const unsigned long long l0 = c->launches;
        int lvl = 0;
        double sc = 0;
        auto* gph = new ckks_graph();
        gph->ctx = c;
        cudaError_t e = cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal);
        try {
            if (e != cudaSuccess) throw CkksError(CKKS_E_CUDA, std::string("begin capture: ") + cudaGetErrorString(e));
            const int nl_in = (int)in->level + 1, ol = model_out_level(m);
            forward_chunk(c, m, in->data, c->ct_words(nl_in), (int)in->batch, in->scale, out->data,
                          c->ct_words(ol + 1), (u64*)work, cap, &lvl, &sc);
            cuda_ok(cudaStreamEndCapture(cap, &gph->graph), "end capture");
            cuda_ok(cudaGraphInstantiate(&gph->exec, gph->graph, 0), "instantiate");
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(cap, &g);
            if (g) cudaGraphDestroy(g);
            c->probe.kind = probe_kind;
            c->launches = l0;
            cudaStreamDestroy(cap);
            delete gph;
            throw;
        }
        c->probe.kind = probe_kind;
        gph->kernels = c->launches - l0;
        c->launches = l0;
        cudaStreamDestroy(cap);
        out->batch = in->batch;
        out->n_comp = 2;
        out->level = (uint32_t)lvl;
        out->scale = sc;
        *out_graph = gph;
        return CKKS_OK;
    })
}

ckks_status ckks_graph_launch(ckks_graph* g, void* stream)
{
    CK_TRY({
        if (!g || !g->exec) throw CkksError(CKKS_E_PARAM, "null graph");
        cuda_ok(cudaGraphLaunch(g->exec, (cudaStream_t)stream), "graph launch");
        g->ctx->launches += g->kernels;
        return CKKS_OK;
    })
}

void ckks_graph_destroy(ckks_graph* g)
{
    if (!g) return;
    if (g->exec) cudaGraphExecDestroy(g->exec);
    if (g->graph) cudaGraphDestroy(g->graph);
    delete g;
}

// ------------------------------------------------------------------------------------ client side
ckks_status ckks_encode(const ckks_ctx* c, const double* values, uint32_t count, double scale, int64_t* coeffs)
{
    CK_TRY({
        if (!c || (!values && count) || !coeffs) throw CkksError(CKKS_E_PARAM, "null");
        encode_host(c->n, values, count, scale, coeffs);
        return CKKS_OK;
    })
}

ckks_status ckks_encrypt(ckks_ctx* c, const int64_t* h_coeffs, uint32_t batch, uint64_t enc_seed,
                         uint64_t first_index, double scale, ckks_ct* out, void* stream)
{
    CK_TRY({
        if (!c || !h_coeffs || !out || !out->data) throw CkksError(CKKS_E_PARAM, "null");
        const int L = c->L, n = c->n;
        auto Lc = c->launch(stream);
        cudaStream_t st = (cudaStream_t)stream;
        for (uint32_t b0 = 0; b0 < batch; b0 += c->max_batch) {
            const int B = (int)std::min<uint32_t>(c->max_batch, batch - b0);
            u64* u = c->d_work;
            u64* e0 = u + (size_t)B * L * n;
            u64* e1 = e0 + (size_t)B * L * n;
            u64* mm = e1 + (size_t)B * L * n;
            int64_t* stage = (int64_t*)(mm + (size_t)B * L * n);
            cuda_ok(cudaMemcpyAsync(stage, h_coeffs + (size_t)b0 * n, (size_t)B * n * 8, cudaMemcpyHostToDevice, st),
                    "upload m");
            ck::signed_to_ntt(Lc, stage, mm, B, L);
            ck::sample_ntt(Lc, u, B, L, L, 0, enc_seed, 6, first_index + b0, 1, 0, 0);
            ck::sample_ntt(Lc, e0, B, L, L, 1, enc_seed, 7, first_index + b0, 1, 0, 0);
            ck::sample_ntt(Lc, e1, B, L, L, 1, enc_seed, 8, first_index + b0, 1, 0, 0);
            ck::encrypt_combine(Lc, c->d_pk, u, e0, e1, mm, out->data + (size_t)b0 * c->ct_words(L), B, L);
            cuda_ok(cudaStreamSynchronize(st), "encrypt");   // staging reused by the next chunk
        }
        out->batch = batch;
        out->n_comp = 2;
        out->level = (uint32_t)(L - 1);
        out->scale = scale;
        return CKKS_OK;
    })
}

ckks_status ckks_encode_device(ckks_ctx* c, const double* d_values, uint32_t count, size_t values_stride,
                               uint32_t batch, double scale, int64_t* d_coeffs, void* stream)
{
    CK_TRY({
        if (!c || (!d_values && count) || !d_coeffs) throw CkksError(CKKS_E_PARAM, "null");
        if (count > (uint32_t)c->n / 2) throw CkksError(CKKS_E_PARAM, "more values than slots");
        if (count > values_stride && batch > 1) throw CkksError(CKKS_E_PARAM, "values_stride < count");
        if (!(scale > 0) || scale >= std::ldexp(1.0, 62)) throw CkksError(CKKS_E_PARAM, "scale out of range");
        ck::encode_device(c->launch(stream), d_values, (int)count, values_stride, (int)batch, scale, d_coeffs);
        return CKKS_OK;
    })
}

ckks_status ckks_encrypt_device(ckks_ctx* c, const int64_t* d_coeffs, uint32_t batch, uint64_t enc_seed,
                                uint64_t first_index, double scale, ckks_ct* out, void* stream)
{
    CK_TRY({
        if (!c || !d_coeffs || !out || !out->data) throw CkksError(CKKS_E_PARAM, "null");
        const int L = c->L, n = c->n;
        auto Lc = c->launch(stream);
        for (uint32_t b0 = 0; b0 < batch; b0 += c->max_batch) {
            const int B = (int)std::min<uint32_t>(c->max_batch, batch - b0);
            u64* u = c->d_work;   // stream-ordered reuse of the workspace across chunks (no host sync)
            u64* e0 = u + (size_t)B * L * n;
            u64* e1 = e0 + (size_t)B * L * n;
            u64* mm = e1 + (size_t)B * L * n;
            ck::signed_to_ntt(Lc, d_coeffs + (size_t)b0 * n, mm, B, L);
            ck::sample_ntt(Lc, u, B, L, L, 0, enc_seed, 6, first_index + b0, 1, 0, 0);
            ck::sample_ntt(Lc, e0, B, L, L, 1, enc_seed, 7, first_index + b0, 1, 0, 0);
            ck::sample_ntt(Lc, e1, B, L, L, 1, enc_seed, 8, first_index + b0, 1, 0, 0);
            ck::encrypt_combine(Lc, c->d_pk, u, e0, e1, mm, out->data + (size_t)b0 * c->ct_words(L), B, L);
        }
        out->batch = batch;
        out->n_comp = 2;
        out->level = (uint32_t)(L - 1);
        out->scale = scale;
        return CKKS_OK;
    })
}

ckks_status ckks_decode_device(ckks_ctx* c, const uint64_t* d_residues, uint32_t level, uint32_t batch, double scale,
                               double* d_values, uint32_t count, void* stream)
{
    CK_TRY({
        if (!c || !d_residues || !d_values) throw CkksError(CKKS_E_PARAM, "null");
        if ((int)level >= c->L) throw CkksError(CKKS_E_SHAPE, "level");
        if (count > (uint32_t)c->n / 2) throw CkksError(CKKS_E_PARAM, "count > slots");
        ck::decode_device(c->launch(stream), d_residues, (int)level + 1, (int)batch, scale, d_values, (int)count);
        return CKKS_OK;
    })
}

ckks_status ckks_decrypt(ckks_ctx* c, const ckks_ct* in, uint64_t* d_out, void* stream)
{
    CK_TRY({
        if (!c || !d_out) throw CkksError(CKKS_E_PARAM, "null");
        check_ct(c, in);
        const int nl = (int)in->level + 1;
        auto L = c->launch(stream);
        for (uint32_t b0 = 0; b0 < in->batch; b0 += 65535) {
            const int B = (int)std::min<uint32_t>(65535, in->batch - b0);
            ck::decrypt(L, in->data + (size_t)b0 * c->ct_words(nl), c->ct_words(nl), c->d_s,
                        d_out + (size_t)b0 * nl * c->n, B, nl);
        }
        return CKKS_OK;
    })
}

ckks_status ckks_decode(const ckks_ctx* c, const uint64_t* res, uint32_t level, double scale, double* values,
                        uint32_t count)
{
    CK_TRY({
        if (!c || !res || !values) throw CkksError(CKKS_E_PARAM, "null");
        if ((int)level >= c->L) throw CkksError(CKKS_E_SHAPE, "level");
        const int n = c->n, nl = (int)level + 1;
        if (count > (uint32_t)n / 2) throw CkksError(CKKS_E_PARAM, "count > slots");
        // balanced mixed-radix (Garner) lift: x = sum_i v_i M_i, v_i in (-q_i/2, q_i/2], M_i = q_0..q_{i-1}
        std::vector<std::vector<u64>> inv(nl, std::vector<u64>(nl));
        for (int i = 0; i < nl; ++i)
            for (int k = 0; k < i; ++k) inv[k][i] = h_pow(c->primes[k] % c->primes[i], c->primes[i] - 2, c->primes[i]);
        std::vector<std::complex<double>> M(2 * (size_t)n, 0.0);
        std::vector<int64_t> v(nl);
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < nl; ++i) {
                const u64 q = c->primes[i];
                // t = (x - sum_{j<i} v_j M_j) / M_i mod q, evaluated incrementally
                u64 t = res[(size_t)i * n + k] % q;
                for (int j = 0; j < i; ++j) {
                    const u64 vj = v[j] >= 0 ? (u64)v[j] % q : (q - ((u64)(-v[j]) % q)) % q;
                    t = (t + q - vj) % q;
                    t = h_mulmod(t, inv[j][i], q);
                }
                v[i] = t > q / 2 ? (int64_t)t - (int64_t)q : (int64_t)t;
            }
            long double x = 0, Mi = 1;
            for (int i = 0; i < nl; ++i) {
                x += (long double)v[i] * Mi;
                Mi *= (long double)c->primes[i];
            }
            M[k] = (double)x;
        }
        fft(M, +1);   // M[e] = sum_k m_k exp(+2 pi i e k / 2N)
        const auto e = slot_exps(n);
        for (uint32_t i = 0; i < count; ++i) values[i] = M[e[i]].real() / scale;
        return CKKS_OK;
    })
}

ckks_status ckks_export_key(ckks_ctx* c, int64_t key_id, uint64_t* h_out, void* stream)
{
    CK_TRY({
        if (!c || !h_out) throw CkksError(CKKS_E_PARAM, "null");
        cudaStream_t st = (cudaStream_t)stream;
        if (key_id == -1) {
            cuda_ok(cudaMemcpyAsync(h_out, c->d_s, (size_t)c->np * c->n * 8, cudaMemcpyDeviceToHost, st), "export s");
        } else if (key_id == -2) {
            cuda_ok(cudaMemcpyAsync(h_out, c->d_pk, (size_t)2 * c->L * c->n * 8, cudaMemcpyDeviceToHost, st), "export pk");
        } else {
            const u64* k = c->key(key_id);
            if (!k) throw CkksError(CKKS_E_NOKEY, "no such key");
            cuda_ok(cudaMemcpyAsync(h_out, k, c->key_words * 8, cudaMemcpyDeviceToHost, st), "export key");
        }
        cuda_ok(cudaStreamSynchronize(st), "export");
        return CKKS_OK;
    })
}

}  // extern "C"
