// kernels.h -- host-side launchers of the sm_100a kernels (internal to the library, not the C-ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>
#include <map>
#include <string>
#include <vector>

struct DCtx;

namespace ck {

// CUDA-event probe around every launch of one kernel class (bench roofline, measured live).
enum ProbeKind { PROBE_OFF = 0, PROBE_MODUP = 1, PROBE_KEYSWITCH = 2, PROBE_NTT = 3, PROBE_ALL = 4 };
struct Probe {
    int kind = PROBE_OFF;
    std::vector<cudaEvent_t> ev;
    std::vector<const char*> names;   // PROBE_ALL: kernel name of each event pair
    size_t used = 0;
    double alg_bytes = 0;   // algorithmic bytes of the probed launches
    std::map<std::string, double> bytes_by_kernel;   // PROBE_ALL: algorithmic bytes per kernel name
    std::map<std::string, double> flops_by_kernel;   // PROBE_ALL: FP64 tensor-core FLOPs (2 per FMA) the exact
                                                     // split products need, per kernel name
    double bfly_fp = 0, bfly_int = 0;                // ModUp butterflies on FP64-class / integer-class primes
    void mark(cudaStream_t s)
    {
        if (used == ev.size()) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            ev.push_back(e);
        }
        cudaEventRecord(ev[used++], s);
    }
    bool on(int k) const { return kind == k; }
};

struct Launch;
// NVTX ranges around every hot-path launch site (ckks_set_option("nvtx", 1) / env CKKS_NVTX=1): names the
// launches of a timeline capture by kernel class; off by default (two host calls per launch site)
int nvtx_on();
void set_nvtx(int on);
// PROBE_ALL: event pair around one launch site, tagged with the kernel name (+ the NVTX range when enabled)
struct ProbeScope {
    Probe* p;
    cudaStream_t st;
    bool nv;
    ProbeScope(Probe* probe, cudaStream_t s, const char* name)
        : p(probe && probe->kind == PROBE_ALL ? probe : nullptr), st(s), nv(nvtx_on() != 0)
    {
        if (nv) nvtxRangePushA(name);
        if (p) {
            p->names.push_back(name);
            p->mark(st);
        }
    }
    ~ProbeScope()
    {
        if (p) p->mark(st);
        if (nv) nvtxRangePop();
    }
};

struct Launch {
    const DCtx* dc;       // device constants
    int log_n;
    int n_data, n_special;
    cudaStream_t st;
    unsigned long long* counter;   // launches issued (for bench gpu_launches)
    Probe* probe;
    const int* pclass;             // host: prime class (ntt.cuh PC_*) of every prime, for probe accounting
    int n_digits;                  // key-switching digits (R9b): host copies of the digit table
    const int* dig_start;
    const int* dig_len;
    // digits with at least one prime among the nl active data primes
    int active_digits(int nl) const
    {
        int d = 0;
        while (d < n_digits && dig_start[d] < nl) ++d;
        return d;
    }
};

// batched in-place NTT over [batch][limbs][N]; limb l uses prime (prime0 + l)
void ntt_batch(const Launch&, uint64_t* data, int batch, int limbs, int prime0, bool inverse);

// ---- key switching, see ks.cu / DESIGN.md section 5
struct KsIn {
    const uint64_t* base;     // first ciphertext
    size_t ct_stride;         // words between consecutive ciphertexts
    size_t comp_off;          // words from a ciphertext to the component being switched
    uint32_t galois;          // 0: no automorphism; else apply sigma_g on load (NTT domain)
};
struct KsOut {
    uint64_t* base;           // [b] at base + b*ct_stride, layout [2][nl][N]
    size_t ct_stride;
    const uint64_t* add;      // optional addend ciphertexts (same layout rules as input)
    size_t add_stride;
    uint32_t add_galois;      // apply sigma_g to the addend on load
    int add_comp1;            // add component 1 of the addend as well (relinearize)
    int accumulate;           // out += result (giant-step accumulation)
    int mac_layout = 0;       // double-hoisted baby steps written in the tensor-core MAC layout (k_mac_tc.cu)
};
struct KsWork {
    uint64_t* digits;         // [B][nl][N]  digit coefficients (2-prime digits: (a, t) CRT pairs, R9b)
    uint64_t* modup;          // [B][nd][nl+K][N]  (row e: q_e for e < nl, then P_0..P_{K-1})
    uint64_t* acc;            // [G][B][2][nl+K][N]   (ModDown NTT outputs x, one block per rotation)
    uint64_t* rem;            // [G][B][3][K][N]  special remainders (K = 2: CRT pairs)
};
#define KS_GMAX 8
#define KS_LMAX 16
// up to KS_GMAX key switches of the SAME ModUp output (hoisted rotations), finished together
struct KsGroup {
    const uint64_t* key[KS_GMAX];
    uint64_t* out[KS_GMAX];
    uint32_t scatter[KS_GMAX];   // 0, or g: write the result permuted by sigma_g (out[k] = y[src_g(k)])
    uint32_t ginv[KS_GMAX];      // g^{-1} mod 2N (when scatter != 0)
    int G;
};
void keyswitch(const Launch&, const KsIn& in, const uint64_t* key, int batch, int nl, const KsWork& w,
               const KsOut& out);
// the two halves of a key switch: ModUp of `in` into w (digits, modup), and the inner product +
// ModDown from w.modup.  scatter_g != 0 writes the result permuted by sigma_{g} where the caller
// passes g^{-1} (hoisted rotation: out = sigma_g(c0 + ModDown(sum_j D_j key'_j))).
void keyswitch_modup(const Launch&, const KsIn& in, int batch, int nl, const KsWork& w, bool qp_in = false);
// double hoisting (R11c): qp_in = the switched component is a Q_l P component (digits of its ModDown,
// ModUp to every prime); keyswitch_finish_qp leaves the result in Q_l P (baby: addend P c0 from `in`,
// output sigma_g-scattered; giant: addend = out.add gathered by out.add_galois, accumulated)
void keyswitch_finish_qp(const Launch&, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                         const KsOut& out, bool baby);
// the baby-step (scatter, addend P c0) QP inner product of a group on the FP64 tensor cores, pipelined
// over the batch (k_ipmma.cu); CKKS_IP_MMA=0 selects the IMAD kernel k_ks_ip_qp
void ip_mma_pipelined(const Launch&, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                      size_t out_stride, bool mac_layout = false);
// the same inner product with the key pre-multiplied by 2^23 (FP rows) / 2^{20u} (60-bit rows): two / three
// accumulators and one modular fold per output (k_ipmma3.cu); false when not applicable (> 5 digits, or
// switched off by ckks_set_option("ip_v3", 0)) -- the caller then launches k_ks_ip_mma2
bool ip_mma3(const Launch&, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
             size_t out_stride, bool mac_layout);
void set_ip_v3(int on);
// CTA-pair (cluster) NTT schedule (ntt_c.cuh), bit mask: 1 batch NTT forward, 2 batch NTT inverse, 4 ModUp at
// N <= 8192, 8 ModUp at N = 16384 (24.2 -> 23.4 ms per B = 256 chunk once the integer-class target rows ran in the
// same launch on the integer pipe; with a launch of their own it was slower, 25.7 ms),
// 64 plain 256-bit global accesses instead of the TMA row copies (A/B)  (ckks_set_option("ntt_q", mask); env
// CKKS_NTT_Q; default NTTQ_DEFAULT)
enum { NTTQ_BATCH_FWD = 1, NTTQ_BATCH_INV = 2, NTTQ_MODUP = 4, NTTQ_MODUP_14 = 8, NTTQ_DIRECT_IO = 64,
       NTTQ_DEFAULT = NTTQ_BATCH_FWD | NTTQ_BATCH_INV | NTTQ_MODUP | NTTQ_MODUP_14 };
void set_ntt_q(int mask);
int get_ntt_q();
int get_ip_v3();
// the giant-step (G = 1, accumulate, addend sigma_g(w.c0)) QP inner product, key-stationary over the
// batch (k_ipgiant.cu); CKKS_IP_GIANT=0 selects the per-ciphertext-pair kernel k_ks_ip_qp
// all G <= KS_GMAX giant steps of a layer in one pass over the accumulator: step g has its own ModUp words, key,
// addend ciphertexts (stride add_stride, sigma_g gathered) and Galois element; false when not applicable (> 5 digits)
bool ip_giant_multi(const Launch&, int G, const uint64_t* const* modup, const uint64_t* const* key,
                    const uint64_t* const* add, const uint32_t* galois, int batch, int nl, uint64_t* acc,
                    size_t acc_stride, size_t add_stride);
#ifndef IPGM_GMAX
#define IPGM_GMAX 4   // giant steps per accumulator pass (shared memory: IPGM_GMAX x 2 nd x 1 KiB of key words per CTA)
#endif
void set_giant_multi(int on);
int get_giant_multi();
void ip_giant(const Launch&, const uint64_t* key, int batch, int nl, const KsWork& w, uint64_t* acc,
              size_t acc_stride, const uint64_t* add, size_t add_stride, uint32_t add_galois);
// y [B][2][nl+1][N] (QP, stride y_stride) -> out [B][2][nl][N]: (y - [y_P]) / P  (one ModDown per layer)
void moddown_qp(const Launch&, const uint64_t* y, size_t y_stride, int batch, int nl, const KsWork& w, uint64_t* out,
                size_t out_stride);
void lift_qp(const Launch&, const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, int batch, int nl);
void keyswitch_finish(const Launch&, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w,
                      const KsOut& out);
// The active key-switching digits of one prime-count class (1- or 2-prime digits) at nl data limbs, passed to
// the digit / ModUp kernels by value (kernel parameter space: no dependent global loads in their prologue).
struct DigitSet {
    int count;                 // digits in the set
    int j[KS_LMAX];            // digit index (its block of the ModUp buffer)
    int s0[KS_LMAX];           // its first data prime
    int first[KS_LMAX + 1];    // ModUp: prefix sums of the target rows per digit (blockIdx.x -> digit)
};
// whole-limb NTT kernels of key switching (k_ksdigits.cu, k_ksqprem.cu, k_ksmodup.cu, k_ksmoddown.cu), one
// instantiation per digit size / special-prime count so every loader and storer is branch-free
void launch_ks_digits(const Launch&, const KsIn& in, int nl, int batch, uint64_t* digits, const uint64_t* rem);
void launch_ks_qp_rem(const Launch&, const uint64_t* in, size_t ct_stride, size_t comp_off, size_t comp_step,
                      uint32_t galois, int nl, int ncomp, int batch, uint64_t* rem);
void launch_ks_modup(const Launch&, const uint64_t* digits, uint64_t* modup, int nl, bool all_e, int batch);
void launch_ks_moddown_intt(const Launch&, const uint64_t* modup, const KsGroup& grp, int nl, int nd, int batch,
                            uint64_t* rem);
void launch_ks_moddown_ntt(const Launch&, const uint64_t* rem, int nl, int gb, uint64_t* xo);
// the same transform with the layer-final ModDown finished in its storer: out = (y - x) P^{-1}
void launch_ks_moddown_ntt_fused(const Launch&, const uint64_t* rem, int nl, int batch, const uint64_t* y,
                                 size_t y_stride, uint64_t* out, size_t out_stride);
// the two DigitSets (1-prime, 2-prime digits) of the active digits at nl limbs; first[] counts ModUp targets
void digit_sets(const Launch&, int nl, bool all_e, DigitSet& one, DigitSet& two);
// the IMAD inner products (k_ipqp.cu): data rows + ModDown combine + permutation (ip_out); Q_l P basis (ip_qp)
void ip_out(const Launch&, const KsWork& w, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsOut& out);
void ip_qp(const Launch&, const KsIn& in, const KsGroup& grp, int batch, int nl, const KsWork& w, const KsOut& out,
           bool baby, int bbv, int spl);
// out limbs[c][N] = in limbs[c][galois_src(k, g)] for `limbs` consecutive limbs (key pre-permutation)
void galois_limbs(const Launch&, const uint64_t* in, uint64_t* out, size_t limbs, uint32_t g);

// rescale: in [B][ncomp][nl][N] (stride in_stride words) -> out [B][ncomp][nl-1][N]; optional
// bias plaintext [nl-1][N] added to component 0.
void rescale(const Launch&, const uint64_t* in, size_t in_stride, uint64_t* out, size_t out_stride, int batch,
             int ncomp, int nl, uint64_t* rem /*[B][ncomp][N]*/, const uint64_t* bias);

void tensor(const Launch&, const uint64_t* a, const uint64_t* b, size_t stride, uint64_t* out3, size_t out_stride,
            int batch, int nl);
void add(const Launch&, const uint64_t* a, size_t sa, const uint64_t* b, size_t sb, uint64_t* out, size_t so,
         int batch, int ncomp, int nl);
// pts [t][pt_nl][N]; qp: v/w in the Q_l P basis (nl+1 limbs, the last mod P), v0 (Q_l) lifted by P on load
void bsgs_mac(const Launch&, const uint64_t* pts, int pt_nl, const uint64_t* v0, size_t v0_stride,
              const uint64_t* vbaby, uint64_t* wout, int t1, int t2, int batch, int nl, bool qp, bool mac_layout = false);
// the same inner sums on the integer tensor cores (tcgen05 kind::i8, k_mac_tc.cu) for double-hoisted baby
// steps stored in the MAC layout: per baby step j >= 1, words [c][row][x / 4][b][x % 4] (contiguous over the
// batch, so a TMA box of 4 coefficients x 64 ciphertexts is one 2 KB row); false = shape not supported
bool bsgs_mac_tc(const Launch&, const uint64_t* pts, int pt_nl, const uint64_t* v0, size_t v0_stride,
                 const uint64_t* vbaby, uint64_t* wout, int t1, int t2, int batch, int nl);
// whether the tensor-core MAC (and so the MAC layout of the baby steps) is used for this shape
bool bsgs_mac_tc_enabled(const Launch&, int t1, int batch);
void set_mac_tc(int on);
int get_mac_tc();
void decrypt(const Launch&, const uint64_t* ct, size_t ct_stride, const uint64_t* s_ntt, uint64_t* out, int batch, int nl);

// client side on the device (k_encode.cu, f-4): canonical-embedding encode of values [batch][count] (row stride
// vstride) at scale -> int64 coefficients [batch][N]; decode of decrypted residues [batch][nl][N] -> [batch][count]
void encode_device(const Launch&, const double* values, int count, size_t vstride, int batch, double scale,
                   int64_t* out);
void decode_device(const Launch&, const uint64_t* res, int nl, int batch, double scale, double* out, int count);
// signed int64 coefficients [count][N] -> NTT residues out[count][nl(+1)][N] over primes 0..nl-1 (and P)
void signed_to_ntt(const Launch&, const int64_t* coeffs, uint64_t* out, int count, int nl, bool with_special = false);

// ---- keygen / encryption samplers (R13-R15; streams as in DESIGN.md)
// out[y][limb][N] = NTT_{p(limb)}(sample_kind(seed, stream(purpose, id0 + y*id_step, digit0 + y*digit_step, 0), i))
// p(limb) = limb < nl_data ? limb : special index.  kind 0 ternary, 1 gaussian.
void sample_ntt(const Launch&, uint64_t* out, int ny, int nlimbs, int nl_data, int kind, uint64_t seed,
                uint64_t purpose, uint64_t id0, uint64_t id_step, uint64_t digit0, uint64_t digit_step);
// out[N] uniform mod prime p with stream (purpose, id, digit, p)
void sample_uniform(const Launch&, uint64_t* out, int prime, uint64_t seed, uint64_t purpose, uint64_t id,
                    uint64_t digit);
// key material combine, see keygen in api.cpp
void keyswitch_key_combine(const Launch&, uint64_t* key, const uint64_t* e_ntt, const uint64_t* s_ntt,
                           const uint64_t* sprime, int L);
void pk_combine(const Launch&, uint64_t* pk, const uint64_t* e_ntt, const uint64_t* s_ntt, int L);
void square_ntt(const Launch&, const uint64_t* s, uint64_t* out, int np);
void galois_ntt(const Launch&, const uint64_t* s, uint64_t* out, int np, uint32_t g);
void encrypt_combine(const Launch&, const uint64_t* pk, const uint64_t* u, const uint64_t* e0, const uint64_t* e1,
                     const uint64_t* m, uint64_t* ct, int batch, int L);

}  // namespace ck
