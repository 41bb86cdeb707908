// k_keyswitch.cu -- sm_100a kernels of the CKKS encrypted-dense-layer hot path.
//
// Every operation of SURVEY 8(a) rows a2-a12 is one of these kernels; the host side (api.cu)
// only sequences launches and tracks level/scale.  Modular arithmetic runs on the integer pipes
// (64-bit Shoup/Barrett), on the FP64 pipe (exact error-free products for q < 2^45), and -- for the
// two small modular contractions (key-switch inner product, BSGS inner sums) -- on the FP64 tensor
// cores with exactly split operands.  Layouts:
//   ciphertext  [batch][comp][limb][N]  u64, NTT domain, canonical residues in [0, q)
//   key         [digit j][comp][prime 0..L+K-1][N]  (primes L.. = the special primes P_k)
//   plaintexts  [t][limb][N]
// This unit: key-switching orchestration (digits -> ModUp -> inner products -> ModDown launch sequences,
// k_ksdigits.cu / k_ksmodup.cu / k_ksmoddown.cu / k_ipqp.cu / k_ipmma.cu / k_ipgiant.cu), the QP-basis
// lift and ModDown combine, Galois gathers.
#include "kinternal.cuh"
#ifndef CK_STREAM_STORES
#define CK_STREAM_STORES 0
#endif

namespace ck {

// ------------------------------------------------------------------------------------ key switch
// Digits (R9, R9b).  Digit j covers the data primes dig_start[j] .. + dig_len[j] - 1 (1 or 2 primes; cut at
// the level).  Its value is the integer CRT lift of the primes' coefficient residues, in [0, Q_j); a
// 2-prime digit is stored as the Garner pair (a, t) with d_j = a + q_s t (common.cuh), so the ModUp loader
// reduces it mod any target prime with one Shoup product.  K special primes P_0..P_{K-1}, P = their
// product (R17b); rows of a Q_l P polynomial: q_0..q_{nl-1}, then P_0..P_{K-1}.

void keyswitch_modup(const Launch& L, const KsIn& in, int batch, int nl, const KsWork& w, bool qp_in)
{
    if (batch <= 0) return;
    const int K = L.n_special, ne = nl + K, nd = L.active_digits(nl);
    int pairs = 0;   // (digit, target row) pairs of the ModUp
    for (int j = 0; j < nd; ++j) pairs += qp_in ? ne : ne - std::min(L.dig_len[j], nl - L.dig_start[j]);
    const bool pm = L.probe && L.probe->on(PROBE_MODUP);
    if (L.probe && L.probe->on(PROBE_ALL)) {
        L.probe->bytes_by_kernel["k_ks_modup"] += ((double)batch * nl + (double)batch * pairs) * (double)(8 << L.log_n);
        // butterflies per limb NTT: (N/2) log2 N; targets of digit j: every row but its own (QP: all)
        const double bf = (double)(1 << (L.log_n - 1)) * L.log_n * batch;
        for (int j = 0; j < nd; ++j) {
            const int s0 = L.dig_start[j], len = std::min(L.dig_len[j], nl - s0);
            for (int e = 0; e < ne; ++e) {
                if (!qp_in && e >= s0 && e < s0 + len) continue;
                const int p = e < nl ? e : L.n_data + (e - nl);
                if (L.pclass && L.pclass[p] == PC_FP) L.probe->bfly_fp += bf;
                else L.probe->bfly_int += bf;
            }
        }
    }
    if (qp_in) launch_ks_qp_rem(L, in.base, in.ct_stride, in.comp_off, 0, in.galois, nl, 1, batch, w.rem);
    launch_ks_digits(L, in, nl, batch, w.digits, qp_in ? w.rem : nullptr);
    if (pm) {
        L.probe->mark(L.st);
        // digits read once, one ModUp limb written per (digit, target) pair
        L.probe->alg_bytes += ((double)batch * nl + (double)batch * pairs) * (double)(8 << L.log_n);
    }
    launch_ks_modup(L, w.digits, w.modup, nl, qp_in, batch);
    if (pm) L.probe->mark(L.st);
    check_launch("keyswitch_modup");
    if (L.counter) {
        DigitSet one, two;
        digit_sets(L, nl, qp_in, one, two);
        const int sizes = (one.count ? 1 : 0) + (two.count ? 1 : 0);
        *L.counter += (qp_in ? 1 : 0) + 1 + sizes;   // digits: one launch (both sizes together), ModUp: one per size
    }
}

// QP-basis finish (R11c): inner product over all nl+K rows, no ModDown.  in (baby: the Q_l input whose
// limbs are D_{j,i} for q_i in digit j) or null (giant: all_e ModUp); addend per KsOut (add_mulP / add_galois)
void keyswitch_finish_qp(const Launch& L, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                         const KsOut& out, bool baby)
{
    if (batch <= 0 || grp.G <= 0) return;
    if (grp.G > KS_GMAX || nl > KS_LMAX) throw std::runtime_error("keyswitch_finish_qp: group/limb limits");
    const int n = 1 << L.log_n;
    if (n < 1024) throw std::runtime_error("N >= 1024 required");
    static const int bbv = [] {
        const char* e = getenv("CKKS_IPQ_BB");
        return e ? atoi(e) : 2;
    }();
    static const int spl = [] {
        const char* e = getenv("CKKS_IP_SPLIT");
        return e ? atoi(e) : 1;
    }();
    static const int use_mma = [] {
        const char* e = getenv("CKKS_IP_MMA");
        return e ? atoi(e) : 2;
    }();
    static const int use_giant = [] {
        const char* e = getenv("CKKS_IP_GIANT");
        return e ? atoi(e) : 1;
    }();
    if (!baby && use_giant && grp.G == 1 && out.accumulate && out.add && !grp.scatter[0] && out.base == grp.out[0]) {
        ip_giant(L, grp.key[0], batch, nl, w, out.base, out.ct_stride, out.add, out.add_stride, out.add_galois);
        return;
    }
    if (baby && use_mma && grp.G >= 2 && out.add == in.base && !out.accumulate) {
        ip_mma_pipelined(L, in, grp, batch, nl, w, out.ct_stride, out.mac_layout != 0);
        return;
    }
    if (out.mac_layout) throw std::runtime_error("keyswitch_finish_qp: MAC layout needs the tensor-core IP path");
    ip_qp(L, in, grp, batch, nl, w, out, baby, bbv, spl);
    check_launch("keyswitch_finish_qp");
    if (L.counter) *L.counter += 1;
}

// layer-final ModDown of B QP ciphertexts y (stride y_stride) into Q_l ciphertexts out
void moddown_qp(const Launch& L, const uint64_t* y, size_t y_stride, int batch, int nl, const KsWork& w, uint64_t* out,
                size_t out_stride)
{
    if (batch <= 0) return;
    const int n = 1 << L.log_n;
    launch_ks_qp_rem(L, y, y_stride, 0, (size_t)(nl + L.n_special) * n, 0, nl, 2, batch, w.rem);
    launch_ks_moddown_ntt_fused(L, w.rem, nl, batch, y, y_stride, out, out_stride);   // (y - x) P^{-1} in the storer
    check_launch("moddown_qp");
    if (L.counter) *L.counter += 2;
}

// P ct -> QP basis (a hoisted baby step with g == 1): out[c][i] = P in[c][i], out[c][special rows] = 0
__global__ void __launch_bounds__(256)
k_lift_qp(const DCtx* __restrict__ dc, const u64* __restrict__ in, size_t in_stride, u64* __restrict__ out,
          size_t out_stride, int nl)
{
    const int n = dc->n, ne = nl + dc->n_special;
    const int k = blockIdx.x * 256 + threadIdx.x;
    const int i = blockIdx.y, c = blockIdx.z % 2, b = blockIdx.z / 2;
    u64 v = 0;
    if (i < nl) {
        const DPrime Pr = dc->p[i];
        v = csub(shoup_mul(in[(size_t)b * in_stride + ((size_t)c * nl + i) * n + k], dc->pmod[i], dc->pmod_sh[i], Pr.q),
                 Pr.q);
    }
    out[(size_t)b * out_stride + ((size_t)c * ne + i) * n + k] = v;
}

void lift_qp(const Launch& L, const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, int batch, int nl)
{
    if (batch <= 0) return;
    const int n = 1 << L.log_n;
    k_lift_qp<<<dim3(n / 256, nl + L.n_special, 2 * batch), 256, 0, L.st>>>(L.dc, in, in_stride, out, out_stride, nl);
    check_launch("lift_qp");
    if (L.counter) ++*L.counter;
}

void keyswitch_finish(const Launch& L, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                      const KsOut& out)
{
    if (batch <= 0 || grp.G <= 0) return;
    if (grp.G > KS_GMAX || nl > KS_LMAX) throw std::runtime_error("keyswitch_finish: group/limb limits");
    const int n = 1 << L.log_n, nd = L.active_digits(nl);
    launch_ks_moddown_intt(L, w.modup, grp, nl, nd, batch, w.rem);
    launch_ks_moddown_ntt(L, w.rem, nl, batch * grp.G, w.acc);
    if (n < 1024) throw std::runtime_error("N >= 1024 required");
    ip_out(L, w, in, grp, batch, nl, out);
    check_launch("keyswitch_finish");
    if (L.counter) *L.counter += 3;
}

void keyswitch(const Launch& L, const KsIn& in, const uint64_t* key, int batch, int nl, const KsWork& w,
               const KsOut& out)
{
    const bool pk = L.probe && L.probe->on(PROBE_KEYSWITCH);
    if (pk) {
        L.probe->mark(L.st);
        // switched component + addend in, 2 components out, key rows used once per launch
        L.probe->alg_bytes +=
            (4.0 * batch * nl + 2.0 * L.active_digits(nl) * (nl + L.n_special)) * (double)(8 << L.log_n);
    }
    keyswitch_modup(L, in, batch, nl, w, false);
    KsGroup grp{};
    grp.key[0] = key;
    grp.out[0] = out.base;
    grp.scatter[0] = 0;
    grp.G = 1;
    keyswitch_finish(L, in, grp, batch, nl, w, out);
    if (pk) L.probe->mark(L.st);
}

__global__ void k_galois_limbs(const DCtx* __restrict__ dc, const u64* __restrict__ in, u64* __restrict__ out, u32 g)
{
    const int n = dc->n;
    const int k = blockIdx.x * 256 + threadIdx.x;
    const size_t limb = blockIdx.y + (size_t)blockIdx.z * gridDim.y;
    out[limb * n + k] = in[limb * n + galois_src(k, g, dc->log_n)];
}

void galois_limbs(const Launch& L, const uint64_t* in, uint64_t* out, size_t limbs, uint32_t g)
{
    const int n = 1 << L.log_n;
    for (size_t done = 0; done < limbs; done += 65535) {
        const unsigned cnt = (unsigned)std::min<size_t>(limbs - done, 65535);
        k_galois_limbs<<<dim3(n / 256, cnt, 1), 256, 0, L.st>>>(L.dc, in + done * n, out + done * n, g);
    }
    check_launch("galois_limbs");
    if (L.counter) ++*L.counter;
}

}  // namespace ck
