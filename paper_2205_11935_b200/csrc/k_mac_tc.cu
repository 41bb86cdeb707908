// k_mac_tc.cu -- sm_100a kernel of the CKKS encrypted-dense-layer hot path: the BSGS inner sums of Eq. 1
// (the inner parenthesis) on the 5th-generation tensor cores, integer path
// (tcgen05.mma.kind::i8, u8 x u8 -> s32 accumulators in TMEM).
//
// For one limb (prime q), one component c and one coefficient x the inner sums are a small matrix product
//     W[b][k] = sum_{j < t1} V_j[b] pt_{k t1 + j}   (mod q)      rows b = ciphertexts, columns k = giant index.
// Exact on byte planes: with V = sum_u a_u 256^u and pt = sum_v w_v 256^v (canonical residues, NB bytes),
//     sum_j V_j pt_j = sum_s 256^s T_s,   T_s = sum_j sum_{u + v = s} a_u(j) w_v(j)     (s < 2 NB - 1).
// The A operand is the little-endian 64-bit residue word itself (K index (j, u), u < 8, bytes u >= NB are 0),
// so the ciphertext side needs no conversion at all; the B operand row (s, k) holds, for baby step j, the 8
// bytes w_{s-u}(pt_{k,j}) (tc_shift_bytes: a shift and a byte reversal).  One 128 x (8 NS) x 32 MMA per 4 baby
// steps; T_s < t1 NB 255^2 < 2^31 for t1 <= 256, so the s32 accumulation never wraps.  The epilogue folds
// the NS shift classes into a 128-bit integer and reduces it mod q.
//
// CTA = 4 coefficients (one 32-byte sector of every residue row) x one limb x one component x 8 giant indices x
// 128 ciphertexts, 512 threads.  TMA (cp.async.bulk.tensor, 4D maps over the baby-step buffer and the
// plaintexts, zero fill past the batch / t1 / t2 edges) brings 8 baby steps x 128 ciphertexts x 4 coefficients
// per stage into a 2-3 deep raw ring; the threads transpose each stage into the canonical K-major SWIZZLE_NONE
// operand tiles (16-byte stores, one core matrix per quarter warp) and build the shift-class B tiles; one
// thread issues the MMAs (which run while the next stage is transposed) and the next TMA; accumulators of the
// 4 coefficients live in TMEM (4 x NR <= 512 columns, column 8 s + k).
#include "kinternal.cuh"
#include "tc05.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>

namespace ck {

#define MTC_XT 4          // coefficients per CTA
#define MTC_JS 8          // baby steps per stage (64 K bytes per row)
#define MTC_THREADS 512
#define MTC_KB (MTC_JS * 8)

// B rows per coefficient: n = 8 s + k (s < NS shift classes, k < 8 giant indices), padded to a multiple of 16
__host__ __device__ constexpr int mtc_nr(int nb) { return ((2 * nb - 1) * 8 + 15) / 16 * 16; }
template <int NB>
struct MacTcCfg {
    static constexpr int NS = 2 * NB - 1;
    static constexpr int NR = mtc_nr(NB);
    static constexpr int RS = NB == 8 ? 2 : 3;                       // TMA ring depth (raw stages)
    static constexpr int RAW_V = MTC_JS * 128 * MTC_XT * 8;          // [b / 64][j 8][b % 64][x 4] words = 32 KB
    static constexpr int RAW_P = 8 * MTC_JS * MTC_XT * 8;            // [k 8][j 8][x 4] words = 2 KB
    static constexpr int RAW = RAW_V + RAW_P;
    static constexpr int A_BYTES = 128 * MTC_KB;                     // one coefficient's canonical A (8 KB)
    static constexpr int B_BYTES = NR * MTC_KB;
    static constexpr int CAN = MTC_XT * (A_BYTES + B_BYTES);
    static constexpr int SMEM = RS * RAW + 2 * CAN;
};
__host__ __device__ constexpr size_t mtc_max(size_t a, size_t b) { return a > b ? a : b; }
__host__ __device__ constexpr size_t mac_tc_smem()
{
    return mtc_max(mtc_max(MacTcCfg<7>::SMEM, MacTcCfg<8>::SMEM), MacTcCfg<6>::SMEM) + 128;
}

// byte offset of (row, 16-byte K chunk c) in a K-major SWIZZLE_NONE tile of MTC_KB bytes per row
__device__ __forceinline__ uint32_t mtc_off(int row, int c) { return (row >> 3) * (8 * MTC_KB) + c * 128 + (row & 7) * 16; }

__device__ __forceinline__ void mtc_expect(uint64_t* bar, uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mtc_tma4(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3, uint64_t* bar)
{
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::
            "r"(tc_smem_u32(dst)), "l"(map), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(tc_smem_u32(bar))
        : "memory");
}

template <int NB>
__device__ __forceinline__ void mac_tc_body(const DCtx* __restrict__ dc, const CUtensorMap* vmap, const CUtensorMap* pmap,
                                            const u64* __restrict__ v0, size_t v0_stride, u64* __restrict__ wout,
                                            int t1, int t2, int batch, int nl, int nlx, uint8_t* sm, uint64_t* bars,
                                            uint32_t taddr)
{
    using C = MacTcCfg<NB>;
    constexpr int NS = C::NS, NR = C::NR, RS = C::RS;
    uint64_t* full = bars;            // [RS]  TMA stage landed
    uint64_t* mmad = bars + 4;        // [2]   MMAs of a canonical slot finished
    uint8_t* raw = sm;                // [RS][RAW]
    uint8_t* can = sm + RS * C::RAW;  // [2][CAN]
    const int n = dc->n, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int l = blockIdx.y, x0 = blockIdx.x * MTC_XT;
    const int ngt = (t2 + 7) / 8;
    const int c = blockIdx.z & 1, kt = (blockIdx.z >> 1) % ngt, bt = (blockIdx.z >> 1) / ngt;
    const int pidx = ext_prime_of(l, nl, dc->n_data);
    const DPrime Pr = dc->p[pidx];
    const u64 Pm = l < nl ? dc->pmod[l] : 0, Pm_sh = l < nl ? dc->pmod_sh[l] : 0;
    const size_t ctw = (size_t)2 * nlx * n;
    const size_t roff = ((size_t)c * nlx + l) * n + x0;   // this limb's coefficients in a W (output) ciphertext
    const size_t roff0 = ((size_t)c * nl + l) * n + x0;    // same in the input ciphertext (Q_l basis)
    const int nst = (t1 + MTC_JS - 1) / MTC_JS;
    // TMA of raw stage s: baby steps j = 8 s .. 8 s + 7 (tensor index j - 1; j = 0 and j >= t1 land as zeros)
    // for 128 ciphertexts x 4 coefficients (two boxes of 64 ciphertexts: rows of 2 KB in the MAC layout), and the
    // plaintexts pt_{k, j} for the CTA's 8 giant indices
    auto tma = [&](int s) {
        uint8_t* r = raw + (s % RS) * C::RAW;
        mtc_expect(&full[s % RS], C::RAW);
        mtc_tma4(r, vmap, bt * 512, x0 / 4, c * nlx + l, s * MTC_JS - 1, &full[s % RS]);
        mtc_tma4(r + C::RAW_V / 2, vmap, bt * 512 + 256, x0 / 4, c * nlx + l, s * MTC_JS - 1, &full[s % RS]);
        mtc_tma4(r + C::RAW_V, pmap, x0, l, s * MTC_JS, kt * 8, &full[s % RS]);
    };
    if (tid == 0)
        for (int s = 0; s < RS && s < nst; ++s) tma(s);
    // zero the padding rows NS*8 .. NR-1 of both B tiles once (never written by the fills)
    for (int cs = 0; cs < 2; ++cs)
        for (int i = tid; i < MTC_XT * (NR - NS * 8) * (MTC_KB / 16); i += MTC_THREADS) {
            const int ch = i % (MTC_KB / 16), r = i / (MTC_KB / 16);
            const int row = NS * 8 + r % (NR - NS * 8), xc = r / (NR - NS * 8);
            uint8_t* Bt = can + cs * C::CAN + MTC_XT * C::A_BYTES + xc * C::B_BYTES;
            *reinterpret_cast<uint4*>(Bt + mtc_off(row, ch)) = make_uint4(0, 0, 0, 0);
        }
    constexpr uint32_t idesc = tc_idesc_u8(128, NR);
    for (int st = 0; st < nst; ++st) {
        const uint8_t* r = raw + (st % RS) * C::RAW;
        const u64* rv = reinterpret_cast<const u64*>(r);              // [b / 64][j][b % 64][x]
        const u64* rp = reinterpret_cast<const u64*>(r + C::RAW_V);   // [k][j][x]
        uint8_t* cn = can + (st & 1) * C::CAN;
        tc_mbar_wait(&full[st % RS], (uint32_t)((st / RS) & 1));
        if (st >= 2) tc_mbar_wait(&mmad[st & 1], (uint32_t)(((st >> 1) - 1) & 1));
        // A: unit (b, x, jp): lane = 8 x' + b' (b fastest); words (j, j+1) -> one 16-byte canonical store
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const int u = tid + it * MTC_THREADS;
            const int b = (u & 7) | ((u >> 5) & 15) << 3, x = (u >> 3) & 3, jp = u >> 9;
            const u64* rb = rv + (b >> 6) * (MTC_JS * 64 * MTC_XT) + (b & 63) * MTC_XT + x;
            u64 w0 = rb[(2 * jp) * 64 * MTC_XT];
            const u64 w1 = rb[(2 * jp + 1) * 64 * MTC_XT];
            if (st == 0 && jp == 0) {                                   // j = 0: the input, times P (Q_l P basis)
                const int bg = bt * 128 + b;
                w0 = 0;
                if (bg < batch && l < nl)
                    w0 = csub(shoup_mul(v0[(size_t)bg * v0_stride + roff0 + x], Pm, Pm_sh, Pr.q), Pr.q);
            }
            *reinterpret_cast<ulonglong2*>(cn + x * C::A_BYTES + mtc_off(b, jp)) = make_ulonglong2(w0, w1);
        }
        // B: lane = (giant index k, chunk jp), warp = (coefficient xc, shift classes sg, sg + 4, ..); one store
        // instruction covers the 8 rows 8 s + k of one aligned group x 4 chunks = 4 whole core matrices
        {
            // read the plaintext block conflict-free (lane L: k = L >> 2, j pair L & 3, all 4 coefficients =
            // 64 contiguous bytes), keep this warp's coefficient, then shuffle to the store mapping
            // (k = L & 7, chunk jp = L >> 3)
            const int xc = warp >> 2, sg = warp & 3;
            const ulonglong2* rq = reinterpret_cast<const ulonglong2*>(rp) + lane * 4;
            const ulonglong2 q0 = rq[(xc >> 1)], q1 = rq[2 + (xc >> 1)];
            const u64 a0 = (xc & 1) ? q0.y : q0.x, a1 = (xc & 1) ? q1.y : q1.x;
            const int k = lane & 7, jp = lane >> 3, src = k * 4 + jp;
            const u64 p0 = __shfl_sync(0xffffffffu, a0, src), p1 = __shfl_sync(0xffffffffu, a1, src);
            uint8_t* Bt = cn + MTC_XT * C::A_BYTES + xc * C::B_BYTES;
#pragma unroll
            for (int s = sg; s < NS; s += 4)
                *reinterpret_cast<ulonglong2*>(Bt + mtc_off(8 * s + k, jp)) =
                    make_ulonglong2(tc_shift_bytes(p0, s), tc_shift_bytes(p1, s));
        }
        tc_fence_smem();
        __syncthreads();
        if (tid == 0) {
            tc_after_sync();
            const uint32_t sb = tc_smem_u32(cn);
#pragma unroll
            for (int xc = 0; xc < MTC_XT; ++xc)
#pragma unroll
                for (int kk = 0; kk < MTC_KB / 32; ++kk) {
                    const uint64_t ad = tc_desc(sb + xc * C::A_BYTES + kk * 256, 128, 8 * MTC_KB);
                    const uint64_t bd = tc_desc(sb + MTC_XT * C::A_BYTES + xc * C::B_BYTES + kk * 256, 128, 8 * MTC_KB);
                    tc_mma_u8(taddr + xc * NR, ad, bd, idesc, (st | kk) ? 1u : 0u);
                }
            tc_commit(&mmad[st & 1]);
            if (st + RS < nst) tma(st + RS);                           // raw slot consumed by every thread
        }
    }
    tc_mbar_wait(&mmad[(nst - 1) & 1], (uint32_t)(((nst - 1) >> 1) & 1));   // every MMA done
    tc_after_sync();
    // ---- epilogue: warp w reads TMEM lanes 32 (w & 3) + lane (= ciphertext row b) of coefficient w >> 2;
    //      column 8 s + k holds T_s of giant index k
    u64* Os = reinterpret_cast<u64*>(can);                   // [8 k][128 b][4 xc]  (the ring is free now)
    const int b = 32 * (warp & 3) + lane, xc = warp >> 2;
    u64 g[8][3];
#pragma unroll
    for (int k = 0; k < 8; ++k) g[k][0] = g[k][1] = g[k][2] = 0;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        uint32_t T[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(T[0]), "=r"(T[1]), "=r"(T[2]), "=r"(T[3]), "=r"(T[4]), "=r"(T[5]), "=r"(T[6]), "=r"(T[7])
                     : "r"(taddr + ((uint32_t)(32 * (warp & 3)) << 16) + xc * NR + 8 * s));
        tc_ld_wait();
#pragma unroll
        for (int k = 0; k < 8; ++k) g[k][s / 5] += (u64)T[k] << (8 * (s % 5));
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        // x = g0 + g1 2^40 + g2 2^80 (each < 2^60): y = g1 + g2 2^40 mod q, then x = g0 + y 2^40 mod q
        u64 lo = g[k][1] + (g[k][2] << 40), hi = (g[k][2] >> 24) + (lo < g[k][1] ? 1 : 0);
        const u64 y = reduce128(hi, lo, Pr);
        lo = g[k][0] + (y << 40);
        hi = (y >> 24) + (lo < g[k][0] ? 1 : 0);
        Os[((size_t)k * 128 + b) * MTC_XT + xc] = reduce128(hi, lo, Pr);
    }
    tc_before_sync();
    __syncthreads();
    // coalesced write: 32 bytes (4 coefficients) per (k, b)
    for (int i = tid; i < 8 * 128; i += MTC_THREADS) {
        const int k = i >> 7, bb = i & 127, kg = kt * 8 + k, bg = bt * 128 + bb;
        if (kg < t2 && bg < batch) {
            const ulonglong2* src = reinterpret_cast<const ulonglong2*>(Os + (size_t)i * MTC_XT);
            ulonglong2* dst = reinterpret_cast<ulonglong2*>(wout + ((size_t)kg * batch + bg) * ctw + roff);
            dst[0] = src[0];
            dst[1] = src[1];
        }
    }
}

__global__ void __launch_bounds__(MTC_THREADS, 1)
k_bsgs_mac_tc(const DCtx* __restrict__ dc, const __grid_constant__ CUtensorMap vmap, const __grid_constant__ CUtensorMap pmap,
              const u64* __restrict__ v0, size_t v0_stride, u64* __restrict__ wout, int t1, int t2, int batch, int nl)
{
    extern __shared__ __align__(1024) uint8_t msm[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(msm + mac_tc_smem() - 128);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 8);
    const int warp = threadIdx.x >> 5;
    if (warp == 0) tc_tmem_alloc(tslot, 512);
    if (threadIdx.x == 0)
        for (int s = 0; s < 8; ++s) tc_mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    tc_before_sync();
    __syncthreads();
    tc_after_sync();
    const uint32_t taddr = *tslot;
    const int nlx = nl + dc->n_special;
    const int l = blockIdx.y;
    const u64 q = dc->p[ext_prime_of(l, nl, dc->n_data)].q;
    const int nb = (64 - __clzll((long long)q) + 7) / 8;   // bytes of a residue
    switch (nb) {
    case 1: case 2: case 3: mac_tc_body<3>(dc, &vmap, &pmap, v0, v0_stride, wout, t1, t2, batch, nl, nlx, msm, bars, taddr); break;
    case 4: mac_tc_body<4>(dc, &vmap, &pmap, v0, v0_stride, wout, t1, t2, batch, nl, nlx, msm, bars, taddr); break;
    case 5: mac_tc_body<5>(dc, &vmap, &pmap, v0, v0_stride, wout, t1, t2, batch, nl, nlx, msm, bars, taddr); break;
    case 6: mac_tc_body<6>(dc, &vmap, &pmap, v0, v0_stride, wout, t1, t2, batch, nl, nlx, msm, bars, taddr); break;
    case 7: mac_tc_body<7>(dc, &vmap, &pmap, v0, v0_stride, wout, t1, t2, batch, nl, nlx, msm, bars, taddr); break;
    default: mac_tc_body<8>(dc, &vmap, &pmap, v0, v0_stride, wout, t1, t2, batch, nl, nlx, msm, bars, taddr); break;
    }
    tc_before_sync();
    __syncthreads();
    if (warp == 0) tc_tmem_dealloc(taddr, 512);
}

// 4D tensor map over u64 words (dims d0 innermost), strides in bytes of d1..d3, box (b0, b1, b2, b3)
static bool encode_map4(CUtensorMap* m, const void* base, const uint64_t dims[4], const uint64_t strides[3],
                        const uint32_t box[4])
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            f = nullptr;
        return (PFN_cuTensorMapEncodeTiled_v12000)f;
    }();
    if (!fn) return false;
    const cuuint32_t es[4] = {1, 1, 1, 1};
    return fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 4, const_cast<void*>(base), (const cuuint64_t*)dims,
              (const cuuint64_t*)strides, (const cuuint32_t*)box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// process-wide selection (ckks_set_option("mac_tc", ..)): the measured A/B of DESIGN.md section 5 keeps the FP64
// tensor-core MAC as the default (the integer tensor-core kernel is exact but data-movement bound, slower here)
static int g_mac_tc = [] {
    const char* e = getenv("CKKS_MAC_TC");
    return e ? atoi(e) : 0;
}();
void set_mac_tc(int on) { g_mac_tc = on; }
int get_mac_tc() { return g_mac_tc; }

bool bsgs_mac_tc_enabled(const Launch& L, int t1, int batch)
{
    return g_mac_tc && t1 >= 2 && t1 <= 256 && batch > 0 && (1 << L.log_n) % (4 * MTC_XT) == 0;
}

// host launcher (Q_l P basis, double hoisting; baby steps in the MAC layout); false if the shape is unsupported
bool bsgs_mac_tc(const Launch& L, const uint64_t* pts, int pt_nl, const uint64_t* v0, size_t v0_stride,
                 const uint64_t* vbaby, uint64_t* wout, int t1, int t2, int batch, int nl)
{
    const int n = 1 << L.log_n;
    if (!bsgs_mac_tc_enabled(L, t1, batch)) return false;
    const int nlx = nl + L.n_special;
    const int ngt = (t2 + 7) / 8, nbt = (batch + 127) / 128;
    // baby steps V_j (j >= 1) in the MAC layout: [j - 1][row = c nlx + l][x / 4][b][x % 4] -> 4D map with
    // d0 = (b, x % 4) (4 batch words), d1 = x / 4, d2 = row, d3 = j - 1; plaintexts [k][j][row l of pt_nl][x]
    CUtensorMap vmap, pmap;
    const uint64_t vd[4] = {(uint64_t)4 * batch, (uint64_t)(n / 4), (uint64_t)(2 * nlx), (uint64_t)(t1 - 1)};
    const uint64_t vs[3] = {(uint64_t)4 * batch * 8, (uint64_t)n * batch * 8, (uint64_t)2 * nlx * n * batch * 8};
    const uint32_t vbx[4] = {256, 1, 1, MTC_JS};
    const uint64_t pd[4] = {(uint64_t)n, (uint64_t)pt_nl, (uint64_t)t1, (uint64_t)t2};
    const uint64_t ps[3] = {(uint64_t)n * 8, (uint64_t)pt_nl * n * 8, (uint64_t)t1 * pt_nl * n * 8};
    const uint32_t pbx[4] = {MTC_XT, 1, MTC_JS, 8};
    if (!encode_map4(&vmap, vbaby, vd, vs, vbx) || !encode_map4(&pmap, pts, pd, ps, pbx)) return false;
    if (L.probe && L.probe->kind == PROBE_ALL) {
        // algorithmic bytes: baby steps + input + plaintexts read, W written (as k_bsgs_mac_mma)
        L.probe->bytes_by_kernel["k_bsgs_mac_tc"] +=
            nlx * ((double)t1 * batch * 2 + (double)t1 * t2 + (double)t2 * batch * 2) * n * 8.0;
    }
    const size_t smem = mac_tc_smem();
    allow_smem(k_bsgs_mac_tc, smem);
    const dim3 grid(n / MTC_XT, nlx, 2 * ngt * nbt);
    {
        ProbeScope ps_(L.probe, L.st, "k_bsgs_mac_tc");
        k_bsgs_mac_tc<<<grid, MTC_THREADS, smem, L.st>>>(L.dc, vmap, pmap, v0, v0_stride, wout, t1, t2, batch, nl);
    }
    check_launch("bsgs_mac_tc");
    if (L.counter) *L.counter += 1;
    return true;
}

}  // namespace ck
