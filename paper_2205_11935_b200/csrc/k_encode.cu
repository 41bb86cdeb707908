// k_encode.cu -- sm_100a kernels of the client side of CryptoTL on the device: the
// canonical-embedding encode of a batch of real vectors (R4, R16) and the decode of decrypted residues.
//
// Slots (R3): slot i <-> the root zeta^{5^i mod 2N}, zeta = e^{i pi / N}, n = N/2 slots.  Because 5^i = 1 mod 4,
// zeta^{n 5^i} = i, so with w_k = m_k + i m_{k+n} (k < n) the slot values are
//     z_i = sum_{k<N} m_k zeta^{k 5^i} = sum_{k<n} w_k zeta^{k 5^i} = DFT_n(w_k zeta^k)[pos(i)],
// pos(i) = (5^i mod 2N - 1) / 4 (the roots zeta^{1 + 4j}, j < n, are exactly the slot roots), DFT_n with the
// positive exponent omega = e^{2 pi i / n}.  Encode is the inverse: u[pos(i)] = scale z_i, w = zeta^{-k}
// IDFT_n(u) / n, m_k = round_half_away(Re w_k), m_{k+n} = round_half_away(Im w_k) -- the same numbers as
// R4's m_k = round(scale (2/N) Re sum_i z_i zeta^{-k 5^i}) (1/n = 2/N), computed in FP64 in a different
// order, so a coefficient can differ by 1 from the host/oracle encoder when it sits within rounding error of
// a half-integer (tests bound the fraction).  One CTA per vector: the n complex values (128 KiB at
// N = 16384) live in shared memory for the log2(n) radix-2 stages.
#include "kinternal.cuh"

namespace ck {

#define ENC_THREADS 512

__device__ __forceinline__ double2 cmul(double2 a, double2 b)
{
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// iterative radix-2 DIT over n = 2^lgn values held in bit-reversed order in a[]: A_k = sum_j a_j omega^{s j k}
// (s = +1 forward, -1 inverse); omega[p] = e^{2 pi i p / n}, p < n/2.  Output in natural order.
__device__ __forceinline__ void smem_fft(double2* a, const double2* __restrict__ omega, int lgn, bool inverse)
{
    const int n = 1 << lgn;
    for (int lh = 0; lh < lgn; ++lh) {
        const int half = 1 << lh, step = n >> (lh + 1);
        for (int t = threadIdx.x; t < n / 2; t += blockDim.x) {
            const int pos = t & (half - 1), i = ((t >> lh) << (lh + 1)) + pos, j = i + half;
            double2 w = omega[pos * step];
            if (inverse) w.y = -w.y;
            const double2 u = a[i], v = cmul(a[j], w);
            a[i] = make_double2(u.x + v.x, u.y + v.y);
            a[j] = make_double2(u.x - v.x, u.y - v.y);
        }
        __syncthreads();
    }
}

__device__ __forceinline__ long long round_half_away(double x)
{
    return x < 0.0 ? -(long long)floor(-x + 0.5) : (long long)floor(x + 0.5);
}

// values [B][count] (row stride vstride doubles) -> coefficients out [B][N] int64
__global__ void __launch_bounds__(ENC_THREADS)
k_encode(const DCtx* __restrict__ dc, const double* __restrict__ values, int count, size_t vstride, double scale,
         long long* __restrict__ out)
{
    extern __shared__ double2 a2[];
    const int lgn = dc->log_n - 1, n = 1 << lgn, b = blockIdx.x;
    for (int i = threadIdx.x; i < n; i += blockDim.x) a2[i] = make_double2(0.0, 0.0);
    __syncthreads();
    const double* v = values + (size_t)b * vstride;
    for (int i = threadIdx.x; i < count; i += blockDim.x)
        a2[brev32(dc->slot_pos[i], lgn)] = make_double2(scale * v[i], 0.0);
    __syncthreads();
    smem_fft(a2, dc->fft_omega, lgn, true);
    const double inv_n = 1.0 / (double)n;
    long long* o = out + ((size_t)b << dc->log_n);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        double2 z = dc->fft_zeta[k];
        z.y = -z.y;
        const double2 w = cmul(a2[k], z);
        o[k] = round_half_away(w.x * inv_n);
        o[k + n] = round_half_away(w.y * inv_n);
    }
}

// Balanced mixed-radix (Garner) lift of the coefficient residues of one coefficient k over nl primes to a
// double: x = sum_i v_i q_0 ... q_{i-1}, v_i in (-q_i/2, q_i/2]  (the centred CRT lift, as the host decode).
__device__ __forceinline__ double crt_lift_double(const DCtx* __restrict__ dc, const u64* __restrict__ r, int nl, int k)
{
    long long v[CKKS_MAXP];
    double x = 0.0, M = 1.0;
    for (int i = 0; i < nl; ++i) {
        const DPrime& P = dc->p[i];
        u64 t = r[((size_t)i << dc->log_n) + k];
        for (int j = 0; j < i; ++j) {
            const u64 vj = v[j] >= 0 ? reduce64((u64)v[j], P) : csub(P.q - reduce64((u64)(-v[j]), P), P.q);
            t = csub(shoup_mul(submod(t, vj, P.q), dc->qinv[j][i], dc->qinv_sh[j][i], P.q), P.q);
        }
        v[i] = t > (P.q >> 1) ? (long long)t - (long long)P.q : (long long)t;
        x += (double)v[i] * M;
        M *= (double)P.q;
    }
    return x;
}

// decrypted residues [B][nl][N] (coefficient domain, c0 + c1 s) -> slot values out [B][count] / scale
__global__ void __launch_bounds__(ENC_THREADS)
k_decode(const DCtx* __restrict__ dc, const u64* __restrict__ res, int nl, double scale, double* __restrict__ out,
         int count)
{
    extern __shared__ double2 a2[];
    const int lgn = dc->log_n - 1, n = 1 << lgn, b = blockIdx.x;
    const u64* r = res + ((size_t)b * nl << dc->log_n);
    for (int k = threadIdx.x; k < n; k += blockDim.x) {
        const double2 w = make_double2(crt_lift_double(dc, r, nl, k), crt_lift_double(dc, r, nl, k + n));
        a2[brev32(k, lgn)] = cmul(w, dc->fft_zeta[k]);
    }
    __syncthreads();
    smem_fft(a2, dc->fft_omega, lgn, false);
    const double inv = 1.0 / scale;
    for (int i = threadIdx.x; i < count; i += blockDim.x)
        out[(size_t)b * count + i] = a2[dc->slot_pos[i]].x * inv;
}

void encode_device(const Launch& L, const double* values, int count, size_t vstride, int batch, double scale,
                   int64_t* out)
{
    if (batch <= 0) return;
    const size_t smem = sizeof(double2) << (L.log_n - 1);
    allow_smem(k_encode, smem);
    for (int b0 = 0; b0 < batch; b0 += 65535) {
        const int B = std::min(65535, batch - b0);
        ProbeScope ps_(L.probe, L.st, "k_encode");
        k_encode<<<B, ENC_THREADS, smem, L.st>>>(L.dc, values + (size_t)b0 * vstride, count, vstride, scale,
                                                 (long long*)out + ((size_t)b0 << L.log_n));
    }
    check_launch("encode_device");
    if (L.counter) ++*L.counter;
}

void decode_device(const Launch& L, const uint64_t* res, int nl, int batch, double scale, double* out, int count)
{
    if (batch <= 0) return;
    const size_t smem = sizeof(double2) << (L.log_n - 1);
    allow_smem(k_decode, smem);
    for (int b0 = 0; b0 < batch; b0 += 65535) {
        const int B = std::min(65535, batch - b0);
        ProbeScope ps_(L.probe, L.st, "k_decode");
        k_decode<<<B, ENC_THREADS, smem, L.st>>>(L.dc, res + ((size_t)b0 * nl << L.log_n), nl, scale,
                                                 out + (size_t)b0 * count, count);
    }
    check_launch("decode_device");
    if (L.counter) ++*L.counter;
}

}  // namespace ck
