/*
 * ckks_oracle.c -- plain, slow, scalar CPU oracle for the CKKS encrypted-dense-layer path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2205_11935_b200/) may include,
 * link, load or execute this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference leg may use it.  It shares no code, header, table or
 * constant generator with the CUDA library: every table below is recomputed here from the
 * definitions.
 *
 * Citation key:  P:Lx = /root/reference/PAPER.md line x (the paper, arXiv 2205.11935);
 *                S:Lx = /root/reference/SPEC.md line x;  R# = reading
 *                (where the paper is silent and defers to SEAL).
 *
 * Arithmetic style: every modular product is `(unsigned __int128)a*b % q`; no Barrett, no
 * Shoup, no lazy reduction, no SIMD, no threads.  The NTT is the textbook iterative radix-2
 * Cooley-Tukey / Gentleman-Sande pair with bit-reversed powers of psi (S:L38-46, S:L92
 * "iterative radix-2 with precomputed bit-reversed twiddles; negacyclic folding via psi").
 * Its output is pinned in tests against the O(N^2) evaluation definition
 *     NTT(a)[k] = sum_i a_i psi^{(2 brev(k) + 1) i}  (mod q)                      (R2)
 * and against schoolbook negacyclic convolution.
 *
 * All residues handed in or out are canonical, in [0, q).
 *
 * Key switching generalises to the hybrid form of SURVEY 8(f) row f-3 (readings R9b, R17b,
 * R10b): the data primes are partitioned into dnum digits of consecutive primes (default: one digit per
 * prime) and there are K >= 1 special primes with P = their product.  Digit values are integers
 * (CRT lifts, up to 2^126) held in `__int128`.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

typedef uint64_t u64;
typedef unsigned __int128 u128;

#define OR_MAXP 64
#define OR_MAXKEYS 512
#define OR_MAXSP 4

typedef __int128 i128;

/* ------------------------------------------------------------------ scalar modular arithmetic */

static u64 mulmod(u64 a, u64 b, u64 q) { return (u64)(((u128)a * b) % q); }
/* a, b in [0, q), q < 2^62: no overflow */
static u64 addmod(u64 a, u64 b, u64 q) { u64 s = a + b; return s >= q ? s - q : s; }
static u64 submod(u64 a, u64 b, u64 q) { return a >= b ? a - b : a + q - b; }
static u64 negmod(u64 a, u64 q) { return a == 0 ? 0 : q - a; }
static u64 powmod(u64 a, u64 e, u64 q)
{
    u64 r = 1 % q;
    a %= q;
    while (e) {
        if (e & 1) r = mulmod(r, a, q);
        a = mulmod(a, a, q);
        e >>= 1;
    }
    return r;
}
/* a^{-1} mod q for prime q (Fermat). */
static u64 invmod(u64 a, u64 q) { return powmod(a, q - 2, q); }
/* signed integer -> residue */
static u64 from_signed(int64_t x, u64 q)
{
    if (x >= 0) return (u64)x % q;
    u64 m = (u64)(-(x + 1)) + 1; /* |x| without overflow */
    return negmod(m % q, q);
}

/* Deterministic Miller-Rabin for 64-bit n (bases 2..37 suffice for n < 3.3e24). */
static int is_prime_u64(u64 n)
{
    static const u64 bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    u64 d = n - 1;
    int r = 0;
    while ((d & 1) == 0) { d >>= 1; r++; }
    for (int i = 0; i < 12; i++) {
        u64 x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int k = 1; k < r; k++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

static u64 bitrev(u64 x, int bits)
{
    u64 r = 0;
    for (int i = 0; i < bits; i++) { r = (r << 1) | (x & 1); x >>= 1; }
    return r;
}

/* ------------------------------------------------------------------ counter-based PRNG (R15) */
/* SplitMix64 finaliser over (seed, stream, index).  Not a CSPRNG (benchmark only). */
static u64 mix64(u64 z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
u64 or_prng(u64 seed, u64 stream, u64 i)
{
    u64 k = mix64(seed ^ mix64(stream));
    return mix64(k + (i + 1) * 0x9E3779B97F4A7C15ULL);
}
/* stream tag: purpose(8 bits) | id(36) | digit(10) | prime(10)  (R15 tag table) */
u64 or_stream(u64 purpose, u64 id, u64 digit, u64 prime)
{
    return (purpose << 56) | ((id & 0xFFFFFFFFFULL) << 20) | ((digit & 0x3FF) << 10) | (prime & 0x3FF);
}
enum { TAG_SECRET = 1, TAG_PK_A = 2, TAG_PK_E = 3, TAG_KS_A = 4, TAG_KS_E = 5,
       TAG_ENC_U = 6, TAG_ENC_E0 = 7, TAG_ENC_E1 = 8 };

/* ternary in {-1,0,1}: floor(3 * hi32 / 2^32) - 1  (R14; bias 2^-32, accepted) */
void or_sample_ternary(u64 seed, u64 stream, int8_t* out, int64_t n)
{
    for (int64_t i = 0; i < n; i++) {
        u64 r = or_prng(seed, stream, (u64)i);
        out[i] = (int8_t)((int)(((r >> 32) * 3ULL) >> 32) - 1);
    }
}
/* uniform in [0,q): (draw(2i) * 2^64 + draw(2i+1)) mod q  (R15) */
void or_sample_uniform(u64 seed, u64 stream, u64 q, u64* out, int64_t n)
{
    for (int64_t i = 0; i < n; i++) {
        u128 hi = or_prng(seed, stream, 2 * (u64)i);
        u128 lo = or_prng(seed, stream, 2 * (u64)i + 1);
        out[i] = (u64)(((hi << 64) | lo) % q);
    }
}

/* ------------------------------------------------------------------ context */
typedef struct or_ctx {
    int log_n, n, n_data, n_special;
    double sigma;
    u64 q[OR_MAXP];
    u64 psi[OR_MAXP];
    u64* psi_rev[OR_MAXP];  /* psi^{brev(m)}, m < N               */
    u64* ipsi_rev[OR_MAXP]; /* psi^{-brev(m)}, m < N              */
    u64 n_inv[OR_MAXP];
    u64 cdt[64];            /* discrete-Gaussian CDT thresholds (R13) */
    int cdt_bound;          /* support [-bound, bound]                */
    /* key-switching digits (R9b): digit j = data primes dig_start[j] .. dig_start[j] + dig_len[j] - 1 */
    int n_digits;
    int dig_start[OR_MAXP], dig_len[OR_MAXP];
    /* keys */
    int have_sk;
    int8_t* s;              /* secret coefficients                      */
    u64* s_ntt;             /* [n_data + n_special][N] NTT form         */
    u64* pk;                /* [2][n_data][N] NTT form, top level        */
    int n_keys;
    int64_t key_id[OR_MAXKEYS];
    u64* key[OR_MAXKEYS];   /* [n_digits][2][n_data + n_special][N] NTT form */
} or_ctx;

static void default_digits(or_ctx* c)
{
    c->n_digits = c->n_data;
    for (int j = 0; j < c->n_data; j++) { c->dig_start[j] = j; c->dig_len[j] = 1; }
}

/* Digit partition (R9b): sizes[0..count-1] consecutive data primes per digit, summing to n_data.  Must be
 * called before any switching key is generated.  Returns -1 on a bad partition. */
int or_set_digits(or_ctx* c, const int* sizes, int count)
{
    if (c->n_keys || count < 1 || count > c->n_data) return -1;
    int start = 0;
    for (int j = 0; j < count; j++) {
        if (sizes[j] < 1) return -1;
        double bits = 0;
        for (int k = 0; k < sizes[j] && start + k < c->n_data; k++) bits += log2((double)c->q[start + k]);
        if (bits > 125.0) return -1;       /* digit values must fit a signed 128-bit integer */
        c->dig_start[j] = start;
        c->dig_len[j] = sizes[j];
        start += sizes[j];
    }
    if (start != c->n_data) return -1;
    c->n_digits = count;
    return 0;
}
int or_n_digits(const or_ctx* c) { return c->n_digits; }
int or_n_special(const or_ctx* c) { return c->n_special; }

int or_n(const or_ctx* c) { return c->n; }
int or_n_data(const or_ctx* c) { return c->n_data; }
u64 or_prime(const or_ctx* c, int i) { return c->q[i]; }
u64 or_psi(const or_ctx* c, int i) { return c->psi[i]; }

/*
 * Prime chain (R1): for each requested bit size b in list order, the largest
 * prime q < 2^b with q = 1 (mod 2N) that is not already in the chain.  The data primes come
 * first, the special prime P (if any) last.
 */
static int gen_chain(or_ctx* c, const int* bits, int count)
{
    u64 two_n = 2ULL * (u64)c->n;
    for (int i = 0; i < count; i++) {
        if (bits[i] < c->log_n + 2 || bits[i] > 61) return -1;
        u64 q = (1ULL << bits[i]) - two_n + 1;
        for (;;) {
            int used = 0;
            for (int k = 0; k < i; k++) if (c->q[k] == q) used = 1;
            if (!used && is_prime_u64(q)) break;
            if (q <= two_n + 1) return -1;
            q -= two_n;
        }
        c->q[i] = q;
    }
    return 0;
}

/*
 * psi = the smallest primitive 2N-th root of unity mod q (R2).  A primitive 2N-th root is an
 * x with x^N = -1.  Take one such root g = x^((q-1)/2N) for the first x that works; every
 * primitive 2N-th root is g^k for odd k < 2N; return the minimum over those N values.
 */
static u64 min_primitive_2n_root(u64 q, int n)
{
    u64 two_n = 2ULL * (u64)n;
    u64 g = 0;
    for (u64 x = 2; x < q; x++) {
        u64 cand = powmod(x, (q - 1) / two_n, q);
        if (powmod(cand, (u64)n, q) == q - 1) { g = cand; break; }
    }
    u64 best = g, g2 = mulmod(g, g, q), cur = g;
    for (u64 k = 1; k < two_n; k += 2) {
        if (cur < best) best = cur;
        cur = mulmod(cur, g2, q);
    }
    return best;
}

/*
 * Discrete Gaussian CDT (R13): rho(x) = exp(-(x*x) / (2 sigma^2)) on |x| <= floor(6 sigma),
 * cumulative sums in increasing x, T_k = floor(2^64 * C_k / C_total) for k = -B..B-1.
 * A draw r maps to  -B + #{k : r >= T_k}.
 */
static void build_cdt(or_ctx* c)
{
    int B = (int)floor(6.0 * c->sigma);
    double rho[128], total = 0.0;
    for (int x = -B; x <= B; x++) {
        rho[x + B] = exp(-(double)(x * x) / (2.0 * c->sigma * c->sigma));
        total += rho[x + B];
    }
    double cum = 0.0;
    for (int x = -B; x < B; x++) {
        cum += rho[x + B];
        c->cdt[x + B] = (u64)ldexp(cum / total, 64);
    }
    c->cdt_bound = B;
}
void or_sample_gaussian(const or_ctx* c, u64 seed, u64 stream, int64_t* out, int64_t n)
{
    int B = c->cdt_bound;
    for (int64_t i = 0; i < n; i++) {
        u64 r = or_prng(seed, stream, (u64)i);
        int64_t v = -B;
        for (int k = 0; k < 2 * B; k++) if (r >= c->cdt[k]) v++;
        out[i] = v;
    }
}
u64 or_cdt(const or_ctx* c, int k) { return c->cdt[k]; }
int or_cdt_bound(const or_ctx* c) { return c->cdt_bound; }

or_ctx* or_ctx_new(int log_n, int n_data, int n_special, const int* bits, double sigma)
{
    if (log_n < 1 || log_n > 17 || n_data < 1 || n_special < 0 || n_special > OR_MAXSP ||
        n_data + n_special > OR_MAXP)
        return NULL;
    or_ctx* c = (or_ctx*)calloc(1, sizeof(or_ctx));
    c->log_n = log_n;
    c->n = 1 << log_n;
    c->n_data = n_data;
    c->n_special = n_special;
    c->sigma = sigma;
    default_digits(c);
    int np = n_data + n_special;
    if (gen_chain(c, bits, np) != 0) { free(c); return NULL; }
    {
        double pbits = 0;   /* P = product of the special primes must fit a signed 128-bit integer */
        for (int k = 0; k < n_special; k++) pbits += log2((double)c->q[n_data + k]);
        if (pbits > 125.0) { free(c); return NULL; }
    }
    for (int i = 0; i < np; i++) {
        u64 q = c->q[i];
        c->psi[i] = min_primitive_2n_root(q, c->n);
        u64 ipsi = invmod(c->psi[i], q);
        c->psi_rev[i] = (u64*)malloc(sizeof(u64) * c->n);
        c->ipsi_rev[i] = (u64*)malloc(sizeof(u64) * c->n);
        u64 p = 1, ip = 1;
        for (int m = 0; m < c->n; m++) {
            u64 r = bitrev((u64)m, log_n);
            c->psi_rev[i][r] = p;
            c->ipsi_rev[i][r] = ip;
            p = mulmod(p, c->psi[i], q);
            ip = mulmod(ip, ipsi, q);
        }
        c->n_inv[i] = invmod((u64)c->n % q, q);
    }
    build_cdt(c);
    return c;
}

/* Test-only constructor with an explicit prime list (for the N=8, q=17 worked example). */
or_ctx* or_ctx_new_primes(int log_n, int n_data, int n_special, const u64* primes, double sigma)
{
    if (log_n < 1 || log_n > 17 || n_data < 1 || n_special < 0 || n_special > OR_MAXSP ||
        n_data + n_special > OR_MAXP)
        return NULL;
    or_ctx* c = (or_ctx*)calloc(1, sizeof(or_ctx));
    c->log_n = log_n;
    c->n = 1 << log_n;
    c->n_data = n_data;
    c->n_special = n_special;
    c->sigma = sigma;
    default_digits(c);
    for (int i = 0; i < n_data + n_special; i++) {
        u64 q = primes[i];
        if (!is_prime_u64(q) || (q - 1) % (2ULL * (u64)c->n) != 0) { free(c); return NULL; }
        c->q[i] = q;
        c->psi[i] = min_primitive_2n_root(q, c->n);
        u64 ipsi = invmod(c->psi[i], q);
        c->psi_rev[i] = (u64*)malloc(sizeof(u64) * c->n);
        c->ipsi_rev[i] = (u64*)malloc(sizeof(u64) * c->n);
        u64 p = 1, ip = 1;
        for (int m = 0; m < c->n; m++) {
            u64 r = bitrev((u64)m, log_n);
            c->psi_rev[i][r] = p;
            c->ipsi_rev[i][r] = ip;
            p = mulmod(p, c->psi[i], q);
            ip = mulmod(ip, ipsi, q);
        }
        c->n_inv[i] = invmod((u64)c->n % q, q);
    }
    build_cdt(c);
    return c;
}

void or_ctx_free(or_ctx* c)
{
    if (!c) return;
    for (int i = 0; i < c->n_data + c->n_special; i++) { free(c->psi_rev[i]); free(c->ipsi_rev[i]); }
    free(c->s);
    free(c->s_ntt);
    free(c->pk);
    for (int k = 0; k < c->n_keys; k++) free(c->key[k]);
    free(c);
}

/* ------------------------------------------------------------------ NTT (R2) */
/* Forward negacyclic NTT, in place, natural-order input, bit-reversed-order output:
 * Cooley-Tukey with psi^{brev(m+i)} (the Longa-Naehrig / SEAL textbook loop). */
void or_ntt(const or_ctx* c, int pi, u64* a)
{
    u64 q = c->q[pi];
    const u64* W = c->psi_rev[pi];
    int n = c->n;
    int t = n;
    for (int m = 1; m < n; m <<= 1) {
        t >>= 1;
        for (int i = 0; i < m; i++) {
            int j1 = 2 * i * t;
            u64 S = W[m + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j];
                u64 V = mulmod(a[j + t], S, q);
                a[j] = addmod(U, V, q);
                a[j + t] = submod(U, V, q);
            }
        }
    }
}
/* Inverse: Gentleman-Sande with psi^{-brev(m+i)}, then multiply by N^{-1}. */
void or_intt(const or_ctx* c, int pi, u64* a)
{
    u64 q = c->q[pi];
    const u64* W = c->ipsi_rev[pi];
    int n = c->n;
    int t = 1;
    for (int m = n >> 1; m >= 1; m >>= 1) {
        int j1 = 0;
        for (int i = 0; i < m; i++) {
            u64 S = W[m + i];
            for (int j = j1; j < j1 + t; j++) {
                u64 U = a[j];
                u64 V = a[j + t];
                a[j] = addmod(U, V, q);
                a[j + t] = mulmod(submod(U, V, q), S, q);
            }
            j1 += 2 * t;
        }
        t <<= 1;
    }
    for (int j = 0; j < n; j++) a[j] = mulmod(a[j], c->n_inv[pi], q);
}

/* ------------------------------------------------------------------ automorphism (R3) */
/* Coefficient domain: a(X) -> a(X^g), X^N = -1: coefficient i moves to i*g mod 2N, negated if >= N. */
void or_automorphism_coef(const or_ctx* c, int pi, const u64* a, u64 g, u64* out)
{
    u64 q = c->q[pi];
    u64 n = (u64)c->n, two_n = 2 * n;
    for (u64 i = 0; i < n; i++) {
        u64 e = (i * g) % two_n;
        if (e < n) out[e] = a[i];
        else out[e - n] = negmod(a[i], q);
    }
}
/* NTT domain, computed the obviously-correct way: iNTT -> coefficient map -> NTT. */
void or_automorphism_ntt(const or_ctx* c, int pi, const u64* a, u64 g, u64* out)
{
    int n = c->n;
    u64* tmp = (u64*)malloc(sizeof(u64) * n);
    memcpy(tmp, a, sizeof(u64) * n);
    or_intt(c, pi, tmp);
    or_automorphism_coef(c, pi, tmp, g, out);
    or_ntt(c, pi, out);
    free(tmp);
}

/* Galois element of a left rotation by `step` slots (R3): g = 5^(step mod n) mod 2N, n = N/2. */
u64 or_galois_elt(const or_ctx* c, int64_t step)
{
    int64_t slots = c->n / 2;
    int64_t r = ((step % slots) + slots) % slots;
    return powmod(5, (u64)r, 2ULL * (u64)c->n);
}

/* ------------------------------------------------------------------ keys (R5) */
static u64* sp(const or_ctx* c, const u64* base, int limb) { return (u64*)base + (size_t)limb * c->n; }

/* small signed coefficients -> NTT residues mod prime pi */
static void small_to_ntt(const or_ctx* c, int pi, const int64_t* x, u64* out)
{
    for (int k = 0; k < c->n; k++) out[k] = from_signed(x[k], c->q[pi]);
    or_ntt(c, pi, out);
}

/* secret key s (ternary, stream TAG_SECRET) and public key pk = (-a s + e, a) over the data primes */
int or_keygen(or_ctx* c, u64 seed)
{
    int n = c->n, np = c->n_data + c->n_special;
    c->s = (int8_t*)malloc(n);
    or_sample_ternary(seed, or_stream(TAG_SECRET, 0, 0, 0), c->s, n);
    c->s_ntt = (u64*)malloc(sizeof(u64) * (size_t)np * n);
    int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * n);
    for (int k = 0; k < n; k++) tmp[k] = c->s[k];
    for (int p = 0; p < np; p++) small_to_ntt(c, p, tmp, sp(c, c->s_ntt, p));
    /* pk */
    c->pk = (u64*)malloc(sizeof(u64) * 2 * (size_t)c->n_data * n);
    or_sample_gaussian(c, seed, or_stream(TAG_PK_E, 0, 0, 0), tmp, n);
    u64* e = (u64*)malloc(sizeof(u64) * n);
    for (int p = 0; p < c->n_data; p++) {
        u64 q = c->q[p];
        u64* a = sp(c, c->pk, c->n_data + p);   /* component 1 */
        u64* b = sp(c, c->pk, p);               /* component 0 */
        or_sample_uniform(seed, or_stream(TAG_PK_A, 0, 0, (u64)p), q, a, n);
        small_to_ntt(c, p, tmp, e);
        const u64* s = sp(c, c->s_ntt, p);
        for (int k = 0; k < n; k++) b[k] = addmod(negmod(mulmod(a[k], s[k], q), q), e[k], q);
    }
    free(e);
    free(tmp);
    c->have_sk = 1;
    c->n_keys = 0;
    return 0;
}

static int find_key(const or_ctx* c, int64_t id)
{
    for (int k = 0; k < c->n_keys; k++) if (c->key_id[k] == id) return k;
    return -1;
}

/* P = product of the special primes, reduced mod q (R17b) */
static u64 special_product_mod(const or_ctx* c, u64 q)
{
    u64 r = 1 % q;
    for (int k = 0; k < c->n_special; k++) r = mulmod(r, c->q[c->n_data + k] % q, q);
    return r;
}

/*
 * Key-switching key from s' to s (R5, R17b): for every digit j < n_digits (one digit per data prime by
 * default; groups of consecutive primes in the hybrid form, R9b) and every prime p in
 * {q_0..q_{L-1}, P_0..P_{K-1}}:
 *     b_j[p] = -a_j[p] s[p] + e_j[p] + [p in digit j] (P mod p) s'[p],      a_j[p] uniform (NTT form),
 * P = P_0 ... P_{K-1}: the gadget is P times the CRT idempotent of digit j (1 mod the digit's primes,
 * 0 mod every other prime), so sum_j d_j g_j = P d mod Q for digits d_j = d mod Q_j.
 * id 0 -> s' = s^2 (relinearisation key); id = g (odd) -> s' = sigma_g(s) (Galois key).
 * Layout: [digit j][component c][prime p = 0..L+K-1][N], special primes last.
 */
int or_gen_switch_key(or_ctx* c, u64 seed, int64_t id)
{
    if (!c->have_sk || c->n_special < 1) return -1;
    if (find_key(c, id) >= 0) return 0;
    if (c->n_keys >= OR_MAXKEYS) return -1;
    int n = c->n, L = c->n_data, np = L + c->n_special, D = c->n_digits;
    /* s' in NTT form over all primes */
    u64* sprime = (u64*)malloc(sizeof(u64) * (size_t)np * n);
    if (id == 0) {
        for (int p = 0; p < np; p++)
            for (int k = 0; k < n; k++) {
                u64 v = sp(c, c->s_ntt, p)[k];
                sp(c, sprime, p)[k] = mulmod(v, v, c->q[p]);
            }
    } else {
        if ((id & 1) == 0) { free(sprime); return -1; }
        u64* coef = (u64*)malloc(sizeof(u64) * n);
        for (int p = 0; p < np; p++) {
            for (int k = 0; k < n; k++) coef[k] = from_signed(c->s[k], c->q[p]);
            or_automorphism_coef(c, p, coef, (u64)id, sp(c, sprime, p));
            or_ntt(c, p, sp(c, sprime, p));
        }
        free(coef);
    }
    u64* key = (u64*)malloc(sizeof(u64) * (size_t)D * 2 * np * n);
    int64_t* ecoef = (int64_t*)malloc(sizeof(int64_t) * n);
    u64* e = (u64*)malloc(sizeof(u64) * n);
    for (int j = 0; j < D; j++) {
        or_sample_gaussian(c, seed, or_stream(TAG_KS_E, (u64)id, (u64)j, 0), ecoef, n);
        for (int p = 0; p < np; p++) {
            u64 q = c->q[p];
            u64* b = key + (((size_t)j * 2 + 0) * np + p) * n;
            u64* a = key + (((size_t)j * 2 + 1) * np + p) * n;
            or_sample_uniform(seed, or_stream(TAG_KS_A, (u64)id, (u64)j, (u64)p), q, a, n);
            small_to_ntt(c, p, ecoef, e);
            const u64* s = sp(c, c->s_ntt, p);
            int in_digit = p < L && p >= c->dig_start[j] && p < c->dig_start[j] + c->dig_len[j];
            u64 gadget = in_digit ? special_product_mod(c, q) : 0;
            for (int k = 0; k < n; k++) {
                u64 v = addmod(negmod(mulmod(a[k], s[k], q), q), e[k], q);
                if (gadget) v = addmod(v, mulmod(gadget, sp(c, sprime, p)[k], q), q);
                b[k] = v;
            }
        }
    }
    free(e);
    free(ecoef);
    free(sprime);
    c->key_id[c->n_keys] = id;
    c->key[c->n_keys] = key;
    c->n_keys++;
    return 0;
}

int or_export_key(const or_ctx* c, int64_t id, u64* out)
{
    int k = find_key(c, id);
    if (k < 0) return -3;
    size_t np = (size_t)c->n_data + c->n_special;
    memcpy(out, c->key[k], sizeof(u64) * (size_t)c->n_digits * 2 * np * c->n);
    return 0;
}
int or_export_secret(const or_ctx* c, int8_t* out)
{
    if (!c->have_sk) return -1;
    memcpy(out, c->s, c->n);
    return 0;
}
int or_export_pk(const or_ctx* c, u64* out)
{
    if (!c->have_sk) return -1;
    memcpy(out, c->pk, sizeof(u64) * 2 * (size_t)c->n_data * c->n);
    return 0;
}

/* ------------------------------------------------------------------ encrypt / decrypt (R6, R17) */
/* Plaintext from integer coefficients m (the rounded, scaled encoding) to NTT residues at level l. */
void or_plain_from_coeffs(const or_ctx* c, const int64_t* m, int level, u64* out)
{
    for (int p = 0; p <= level; p++) small_to_ntt(c, p, m, sp(c, out, p));
}

/*
 * Public-key encryption at the top level (level = n_data - 1), R17:
 *   u ternary, e0, e1 Gaussian (streams TAG_ENC_* with id = index), c = (pk0 u + e0 + m, pk1 u + e1).
 * out: [2][n_data][N] NTT form.
 */
int or_encrypt(const or_ctx* c, const int64_t* m, u64 enc_seed, u64 index, u64* out)
{
    if (!c->have_sk) return -1;
    int n = c->n, L = c->n_data;
    int8_t* u = (int8_t*)malloc(n);
    int64_t* e0 = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* e1 = (int64_t*)malloc(sizeof(int64_t) * n);
    int64_t* ut = (int64_t*)malloc(sizeof(int64_t) * n);
    or_sample_ternary(enc_seed, or_stream(TAG_ENC_U, index, 0, 0), u, n);
    or_sample_gaussian(c, enc_seed, or_stream(TAG_ENC_E0, index, 0, 0), e0, n);
    or_sample_gaussian(c, enc_seed, or_stream(TAG_ENC_E1, index, 0, 0), e1, n);
    for (int k = 0; k < n; k++) ut[k] = u[k];
    u64* un = (u64*)malloc(sizeof(u64) * n);
    u64* en = (u64*)malloc(sizeof(u64) * n);
    u64* mn = (u64*)malloc(sizeof(u64) * n);
    for (int p = 0; p < L; p++) {
        u64 q = c->q[p];
        small_to_ntt(c, p, ut, un);
        small_to_ntt(c, p, m, mn);
        const u64* pk0 = sp(c, c->pk, p);
        const u64* pk1 = sp(c, c->pk, L + p);
        u64* c0 = sp(c, out, p);
        u64* c1 = sp(c, out, L + p);
        small_to_ntt(c, p, e0, en);
        for (int k = 0; k < n; k++) c0[k] = addmod(addmod(mulmod(pk0[k], un[k], q), en[k], q), mn[k], q);
        small_to_ntt(c, p, e1, en);
        for (int k = 0; k < n; k++) c1[k] = addmod(mulmod(pk1[k], un[k], q), en[k], q);
    }
    free(u); free(e0); free(e1); free(ut); free(un); free(en); free(mn);
    return 0;
}

/* Decrypt (R6): c0 + c1 s over the level's primes; returns COEFFICIENT residues [level+1][N].
 * Size-3 ciphertexts are not accepted (the caller passes exactly two components). */
int or_decrypt(const or_ctx* c, const u64* ct, int level, u64* out)
{
    if (!c->have_sk) return -1;
    int n = c->n, nl = level + 1;
    for (int p = 0; p < nl; p++) {
        u64 q = c->q[p];
        const u64* c0 = sp(c, ct, p);
        const u64* c1 = sp(c, ct, nl + p);
        const u64* s = sp(c, c->s_ntt, p);
        u64* o = sp(c, out, p);
        for (int k = 0; k < n; k++) o[k] = addmod(c0[k], mulmod(c1[k], s[k], q), q);
        or_intt(c, p, o);
    }
    return 0;
}

/* ------------------------------------------------------------------ elementwise (R7) */
void or_add(const or_ctx* c, const u64* a, const u64* b, int level, int ncomp, u64* out)
{
    int nl = level + 1;
    for (int comp = 0; comp < ncomp; comp++)
        for (int p = 0; p < nl; p++)
            for (int k = 0; k < c->n; k++) {
                size_t idx = ((size_t)comp * nl + p) * c->n + k;
                out[idx] = addmod(a[idx], b[idx], c->q[p]);
            }
}
/* (c0 m, c1 m) with m in NTT form at the same level */
void or_mul_plain(const or_ctx* c, const u64* ct, const u64* pt, int level, u64* out)
{
    int nl = level + 1;
    for (int comp = 0; comp < 2; comp++)
        for (int p = 0; p < nl; p++)
            for (int k = 0; k < c->n; k++) {
                size_t idx = ((size_t)comp * nl + p) * c->n + k;
                out[idx] = mulmod(ct[idx], pt[(size_t)p * c->n + k], c->q[p]);
            }
}
/* (c0 + m, c1) */
void or_add_plain(const or_ctx* c, const u64* ct, const u64* pt, int level, u64* out)
{
    int nl = level + 1;
    size_t half = (size_t)nl * c->n;
    memcpy(out + half, ct + half, sizeof(u64) * half);
    for (int p = 0; p < nl; p++)
        for (int k = 0; k < c->n; k++) {
            size_t idx = (size_t)p * c->n + k;
            out[idx] = addmod(ct[idx], pt[idx], c->q[p]);
        }
}
/* tensor product (a0 b0, a0 b1 + a1 b0, a1 b1) */
void or_tensor(const or_ctx* c, const u64* a, const u64* b, int level, u64* out3)
{
    int nl = level + 1;
    size_t h = (size_t)nl * c->n;
    for (int p = 0; p < nl; p++)
        for (int k = 0; k < c->n; k++) {
            u64 q = c->q[p];
            size_t i = (size_t)p * c->n + k;
            u64 a0 = a[i], a1 = a[h + i], b0 = b[i], b1 = b[h + i];
            out3[i] = mulmod(a0, b0, q);
            out3[h + i] = addmod(mulmod(a0, b1, q), mulmod(a1, b0, q), q);
            out3[2 * h + i] = mulmod(a1, b1, q);
        }
}

/* centered representative of r in [0, m) -> residue mod q  (R10: round to nearest, m odd) */
static u64 centered_mod(u64 r, u64 m, u64 q)
{
    if (r <= (m - 1) / 2) return r % q;
    return negmod((m - r) % q, q);
}

/* ------------------------------------------------------------------ key switching (R5, R9-R12) */
/* signed 128-bit integer -> residue mod q */
static u64 from_i128(i128 x, u64 q)
{
    i128 r = x % (i128)q;
    return (u64)(r < 0 ? r + (i128)q : r);
}
/* CRT lift (Garner, R9b) of residues r[0..k-1] modulo m[0..k-1] (distinct primes) to the unique integer
 * in [0, m_0 ... m_{k-1}); the product must stay below 2^127. */
static i128 crt_lift(const u64* r, const u64* m, int k)
{
    unsigned __int128 x = r[0], M = m[0];
    for (int i = 1; i < k; i++) {
        u64 xm = (u64)(x % m[i]);
        u64 t = mulmod(submod(r[i], xm, m[i]), invmod((u64)(M % m[i]), m[i]), m[i]);
        x += M * t;
        M *= m[i];
    }
    return (i128)x;
}
static unsigned __int128 special_product(const or_ctx* c)
{
    unsigned __int128 P = 1;
    for (int k = 0; k < c->n_special; k++) P *= c->q[c->n_data + k];
    return P;
}
/* prime index of limb e of a Q_l P (extended-basis) polynomial: data primes 0..l, then P_0..P_{K-1} */
static int ext_prime(const or_ctx* c, int level, int e) { return e <= level ? e : c->n_data + (e - level - 1); }
/* number of active digits at level l and the active primes of digit j (a digit is cut at the level) */
static int active_digits(const or_ctx* c, int level)
{
    int d = 0;
    while (d < c->n_digits && c->dig_start[d] <= level) d++;
    return d;
}
static int digit_len_at(const or_ctx* c, int j, int level)
{
    int end = c->dig_start[j] + c->dig_len[j];
    if (end > level + 1) end = level + 1;
    return end - c->dig_start[j];
}

/*
 * Key switch from explicit digit polynomials (signed integer coefficients, one per active digit j),
 * R-KS steps 2-4:
 *   2. ModUp: D_{j,p} = NTT_p(digit_j mod p) for every p in {q_0..q_l, P_0..P_{K-1}}
 *   3. inner product  u~_c[p] = sum_j D_{j,p} key_j.c[p]   mod p
 *   4. ModDown: r = centered(CRT_P(iNTT(u~_c[P_k]))),  u_c[i] = (u~_c[i] - NTT_{q_i}(r mod q_i)) P^{-1} mod q_i
 */
/* steps 2-3 into the extended basis: acc [2][l+1+K][N]  (no ModDown) */
static void ks_ip_qp(const or_ctx* c, const i128* digit, int level, int kidx, u64* acc)
{
    int n = c->n, L = c->n_data, nl = level + 1, np_key = L + c->n_special;
    const u64* key = c->key[kidx];
    int ne = nl + c->n_special, nd = active_digits(c, level);
    memset(acc, 0, sizeof(u64) * (size_t)2 * ne * n);
    u64* D = (u64*)malloc(sizeof(u64) * n);
    for (int j = 0; j < nd; j++) {
        for (int e = 0; e < ne; e++) {
            int p = ext_prime(c, level, e);
            u64 q = c->q[p];
            for (int k = 0; k < n; k++) D[k] = from_i128(digit[(size_t)j * n + k], q);
            or_ntt(c, p, D);
            for (int comp = 0; comp < 2; comp++) {
                const u64* kv = key + (((size_t)j * 2 + comp) * np_key + p) * n;
                u64* a = acc + ((size_t)comp * ne + e) * n;
                for (int k = 0; k < n; k++) a[k] = addmod(a[k], mulmod(D[k], kv[k], q), q);
            }
        }
    }
    free(D);
}

/* step 4 on one component: in [l+1+K][N] (QP basis) -> out [l+1][N] */
static void moddown_comp(const or_ctx* c, const u64* in, int level, u64* out)
{
    int n = c->n, L = c->n_data, nl = level + 1, K = c->n_special;
    unsigned __int128 P = special_product(c);
    u64* rs = (u64*)malloc(sizeof(u64) * (size_t)K * n);   /* coefficient residues mod P_k */
    u64 pm[OR_MAXSP];
    for (int k = 0; k < K; k++) {
        memcpy(rs + (size_t)k * n, in + (size_t)(nl + k) * n, sizeof(u64) * n);
        or_intt(c, L + k, rs + (size_t)k * n);
        pm[k] = c->q[L + k];
    }
    /* r = the centred representative of the CRT of the special residues, (-P/2, P/2) (R10b) */
    i128* r = (i128*)malloc(sizeof(i128) * n);
    for (int k = 0; k < n; k++) {
        u64 v[OR_MAXSP];
        for (int m = 0; m < K; m++) v[m] = rs[(size_t)m * n + k];
        unsigned __int128 x = (unsigned __int128)crt_lift(v, pm, K);
        r[k] = x <= (P - 1) / 2 ? (i128)x : -(i128)(P - x);
    }
    u64* t = (u64*)malloc(sizeof(u64) * n);
    for (int i = 0; i < nl; i++) {
        u64 q = c->q[i];
        u64 pinv = invmod(special_product_mod(c, q), q);
        for (int k = 0; k < n; k++) t[k] = from_i128(r[k], q);
        or_ntt(c, i, t);
        const u64* a = in + (size_t)i * n;
        u64* o = out + (size_t)i * n;
        for (int k = 0; k < n; k++) o[k] = mulmod(submod(a[k], t[k], q), pinv, q);
    }
    free(rs); free(r); free(t);
}

static int ks_from_digits(const or_ctx* c, const i128* digit, int level, int64_t key_id, u64* out)
{
    int kidx = find_key(c, key_id);
    if (kidx < 0) return -3;
    int n = c->n, nl = level + 1, ne = nl + c->n_special;
    u64* acc = (u64*)malloc(sizeof(u64) * (size_t)2 * ne * n);
    ks_ip_qp(c, digit, level, kidx, acc);
    for (int comp = 0; comp < 2; comp++)
        moddown_comp(c, acc + (size_t)comp * ne * n, level, out + (size_t)comp * nl * n);
    free(acc);
    return 0;
}

/* digits of d (NTT form, l+1 limbs) (R9, R9b): d_j = the CRT lift of iNTT_{q}(d[q]) over the active
 * primes q of digit j, an integer in [0, prod q) (unsigned lift); [n_active_digits][N] */
static i128* digits_of(const or_ctx* c, const u64* d, int level)
{
    int n = c->n, nd = active_digits(c, level);
    i128* digit = (i128*)malloc(sizeof(i128) * (size_t)nd * n);
    u64* tmp = (u64*)malloc(sizeof(u64) * (size_t)(level + 1) * n);
    for (int i = 0; i <= level; i++) {
        memcpy(tmp + (size_t)i * n, d + (size_t)i * n, sizeof(u64) * n);
        or_intt(c, i, tmp + (size_t)i * n);
    }
    for (int j = 0; j < nd; j++) {
        int s0 = c->dig_start[j], len = digit_len_at(c, j, level);
        for (int k = 0; k < n; k++) {
            u64 r[OR_MAXP], m[OR_MAXP];
            for (int i = 0; i < len; i++) { r[i] = tmp[(size_t)(s0 + i) * n + k]; m[i] = c->q[s0 + i]; }
            digit[(size_t)j * n + k] = crt_lift(r, m, len);
        }
    }
    free(tmp);
    return digit;
}
/* sigma_g on signed integer digit polynomials (coefficient i -> i g mod 2N, negated if >= N) */
static i128* sigma_digits(const or_ctx* c, const i128* digit, int nd, u64 g)
{
    int n = c->n;
    i128* sd = (i128*)calloc((size_t)nd * n, sizeof(i128));   /* sigma_g is a bijection */
    u64 two_n = 2ULL * (u64)n;
    for (int j = 0; j < nd; j++)
        for (u64 i = 0; i < (u64)n; i++) {
            u64 e = (i * g) % two_n;
            i128 v = digit[(size_t)j * n + i];
            if (e < (u64)n) sd[(size_t)j * n + e] = v;
            else sd[(size_t)j * n + (e - n)] = -v;
        }
    return sd;
}

/* KS(d; key) at level l with the unsigned digits of d (R-KS step 1 + ks_from_digits). */
int or_keyswitch(const or_ctx* c, const u64* d, int level, int64_t key_id, u64* out)
{
    if (find_key(c, key_id) < 0) return -3;
    if (level < 0 || level >= c->n_data) return -2;
    i128* digit = digits_of(c, d, level);
    int st = ks_from_digits(c, digit, level, key_id, out);
    free(digit);
    return st;
}

/* Relinearize (R-composite): (c0, c1, c2) -> (c0, c1) + KS(c2; rlk).  in3: [3][l+1][N]. */
int or_relinearize(const or_ctx* c, const u64* in3, int level, u64* out)
{
    int nl = level + 1;
    size_t h = (size_t)nl * c->n;
    u64* u = (u64*)malloc(sizeof(u64) * 2 * h);
    int st = or_keyswitch(c, in3 + 2 * h, level, 0, u);
    if (st) { free(u); return st; }
    or_add(c, in3, u, level, 2, out);
    free(u);
    return 0;
}

/* Rotate left by `step` slots, non-hoisted (R11):
 *   (sigma_g(c0), sigma_g(c1)) -> (sigma_g(c0), 0) + KS(sigma_g(c1); gk_g). */
int or_rotate(const or_ctx* c, const u64* ct, int level, int64_t step, u64* out)
{
    int n = c->n, nl = level + 1;
    size_t h = (size_t)nl * n;
    u64 g = or_galois_elt(c, step);
    if (g == 1) { memcpy(out, ct, sizeof(u64) * 2 * h); return 0; }
    if (find_key(c, (int64_t)g) < 0) return -3;
    u64* rc = (u64*)malloc(sizeof(u64) * 2 * h);
    for (int comp = 0; comp < 2; comp++)
        for (int p = 0; p < nl; p++)
            or_automorphism_ntt(c, p, ct + comp * h + (size_t)p * n, g, rc + comp * h + (size_t)p * n);
    u64* u = (u64*)malloc(sizeof(u64) * 2 * h);
    int st = or_keyswitch(c, rc + h, level, (int64_t)g, u);
    if (st == 0) {
        for (int p = 0; p < nl; p++)
            for (int k = 0; k < n; k++) {
                size_t i = (size_t)p * n + k;
                out[i] = addmod(rc[i], u[i], c->q[p]);
                out[h + i] = u[h + i];
            }
    }
    free(rc);
    free(u);
    return st;
}

/*
 * Hoisted rotation (NEXT f-1; reading R11b): the digits are taken from the UNROTATED c1 and the
 * automorphism is applied to them as signed integer polynomials,
 *     d_j = digits of c1 (R9 / R9b, unsigned lift),   d'_j = sigma_g(d_j)  (coefficient i -> i g mod 2N,
 *     negated if >= N, as a signed integer: -d, not Q_j - d),
 *     (sigma_g(c0), 0) + ModDown(sum_j ModUp(d'_j) key_j).
 * All rotations of one ciphertext can then share ModUp(d_j) (sigma_g commutes with NTT_p).  The
 * result differs from the non-hoisted one by an encryption of a small value (different rounding
 * of the digit lift), so it has its own pins.
 */
int or_rotate_hoisted(const or_ctx* c, const u64* ct, int level, int64_t step, u64* out)
{
    int n = c->n, nl = level + 1;
    size_t h = (size_t)nl * n;
    u64 g = or_galois_elt(c, step);
    if (g == 1) { memcpy(out, ct, sizeof(u64) * 2 * h); return 0; }
    if (find_key(c, (int64_t)g) < 0) return -3;
    i128* digit = digits_of(c, ct + h, level);
    i128* sd = sigma_digits(c, digit, active_digits(c, level), g);
    u64* u = (u64*)malloc(sizeof(u64) * 2 * h);
    int st = ks_from_digits(c, sd, level, (int64_t)g, u);
    if (st == 0) {
        u64* rc0 = (u64*)malloc(sizeof(u64) * h);
        for (int p = 0; p < nl; p++) or_automorphism_ntt(c, p, ct + (size_t)p * n, g, rc0 + (size_t)p * n);
        for (int p = 0; p < nl; p++)
            for (int k = 0; k < n; k++) {
                size_t i = (size_t)p * n + k;
                out[i] = addmod(rc0[i], u[i], c->q[p]);
                out[h + i] = u[h + i];
            }
        free(rc0);
    }
    free(digit); free(sd); free(u);
    return st;
}

/* ------------------------------------------------------------------ QP-basis (double hoisting, R11c) */
/*
 * NEXT f-1 second stage (R11c, "double hoisting"): the BSGS baby-step rotations are left in
 * the extended basis Q_l P (no ModDown), the inner sums and the giant-step rotations are accumulated
 * there, and ONE ModDown per layer brings the sum back to Q_l.  A QP ciphertext at level l has l+1+K
 * limbs per component: q_0..q_l, then P_0..P_{K-1}.
 */
static u64 ext_q(const or_ctx* c, int level, int e) { return c->q[ext_prime(c, level, e)]; }

/* step 4 (ModDown) on ncomp components: in [ncomp][l+1+K][N] -> out [ncomp][l+1][N] */
void or_moddown(const or_ctx* c, const u64* in_qp, int level, int ncomp, u64* out)
{
    int n = c->n, nl = level + 1, ne = nl + c->n_special;
    for (int comp = 0; comp < ncomp; comp++)
        moddown_comp(c, in_qp + (size_t)comp * ne * n, level, out + (size_t)comp * nl * n);
}

/* P * ct in the QP basis: residues P c mod q_i on the data limbs, 0 mod every P_k */
void or_lift_qp(const or_ctx* c, const u64* ct, int level, int ncomp, u64* out)
{
    int n = c->n, nl = level + 1, ne = nl + c->n_special;
    for (int comp = 0; comp < ncomp; comp++) {
        for (int i = 0; i < nl; i++) {
            u64 pm = special_product_mod(c, c->q[i]);
            for (int k = 0; k < n; k++)
                out[((size_t)comp * ne + i) * n + k] = mulmod(ct[((size_t)comp * nl + i) * n + k], pm, c->q[i]);
        }
        memset(out + ((size_t)comp * ne + nl) * n, 0, sizeof(u64) * (size_t)c->n_special * n);
    }
}

/* plaintext of integer coefficients m over q_0..q_l, P_0..P_{K-1} (NTT form) */
void or_plain_qp(const or_ctx* c, const int64_t* m, int level, u64* out)
{
    int n = c->n, ne = level + 1 + c->n_special;
    for (int e = 0; e < ne; e++) {
        int p = ext_prime(c, level, e);
        u64* o = out + (size_t)e * n;
        for (int k = 0; k < n; k++) o[k] = from_signed(m[k], c->q[p]);
        or_ntt(c, p, o);
    }
}

void or_mul_plain_qp(const or_ctx* c, const u64* ct, const u64* pt, int level, u64* out)
{
    int n = c->n, ne = level + 1 + c->n_special;
    for (int comp = 0; comp < 2; comp++)
        for (int e = 0; e < ne; e++) {
            u64 q = ext_q(c, level, e);
            for (int k = 0; k < n; k++) {
                size_t idx = ((size_t)comp * ne + e) * n + k;
                out[idx] = mulmod(ct[idx], pt[(size_t)e * n + k], q);
            }
        }
}

void or_add_qp(const or_ctx* c, const u64* a, const u64* b, int level, int ncomp, u64* out)
{
    int n = c->n, ne = level + 1 + c->n_special;
    for (int comp = 0; comp < ncomp; comp++)
        for (int e = 0; e < ne; e++) {
            u64 q = ext_q(c, level, e);
            for (int k = 0; k < n; k++) {
                size_t idx = ((size_t)comp * ne + e) * n + k;
                out[idx] = addmod(a[idx], b[idx], q);
            }
        }
}

/* Baby step (R11c): the hoisted rotation of R11b without its ModDown,
 *   (P sigma_g(c0) + sum_j ModUp(d'_j) gk_j.c0,  sum_j ModUp(d'_j) gk_j.c1)  over Q_l P,
 * d'_j = sigma_g(d_j) as signed integers, d_j the digits of c1.  step 0: P ct. */
int or_rotate_hoisted_qp(const or_ctx* c, const u64* ct, int level, int64_t step, u64* out)
{
    int n = c->n, nl = level + 1;
    size_t h = (size_t)nl * n;
    u64 g = or_galois_elt(c, step);
    if (g == 1) { or_lift_qp(c, ct, level, 2, out); return 0; }
    int kidx = find_key(c, (int64_t)g);
    if (kidx < 0) return -3;
    i128* digit = digits_of(c, ct + h, level);
    i128* sd = sigma_digits(c, digit, active_digits(c, level), g);
    ks_ip_qp(c, sd, level, kidx, out);
    u64* rc0 = (u64*)malloc(sizeof(u64) * n);
    for (int p = 0; p < nl; p++) {
        u64 q = c->q[p];
        u64 pm = special_product_mod(c, q);
        or_automorphism_ntt(c, p, ct + (size_t)p * n, g, rc0);
        u64* o = out + (size_t)p * n;                       /* component 0, limb p */
        for (int k = 0; k < n; k++) o[k] = addmod(o[k], mulmod(rc0[k], pm, q), q);
    }
    free(rc0); free(digit); free(sd);
    return 0;
}

/* Giant step (R11c) on a QP ciphertext w:
 *   c1' = ModDown(w.c1),  digits d_j of sigma_g(c1') (unsigned, as R9 / R9b),
 *   (sigma_g(w.c0) + sum_j ModUp(d_j) gk_j.c0,  sum_j ModUp(d_j) gk_j.c1)  over Q_l P.  step 0: w. */
int or_rotate_qp(const or_ctx* c, const u64* w, int level, int64_t step, u64* out)
{
    int n = c->n, nl = level + 1, ne = nl + c->n_special;
    size_t hq = (size_t)ne * n, h = (size_t)nl * n;
    u64 g = or_galois_elt(c, step);
    if (g == 1) { memcpy(out, w, sizeof(u64) * 2 * hq); return 0; }
    int kidx = find_key(c, (int64_t)g);
    if (kidx < 0) return -3;
    u64* c1 = (u64*)malloc(sizeof(u64) * h);
    moddown_comp(c, w + hq, level, c1);
    u64* rc1 = (u64*)malloc(sizeof(u64) * h);
    for (int p = 0; p < nl; p++) or_automorphism_ntt(c, p, c1 + (size_t)p * n, g, rc1 + (size_t)p * n);
    i128* digit = digits_of(c, rc1, level);
    ks_ip_qp(c, digit, level, kidx, out);
    u64* r0 = (u64*)malloc(sizeof(u64) * n);
    for (int e = 0; e < ne; e++) {
        int p = ext_prime(c, level, e);
        u64 q = c->q[p];
        or_automorphism_ntt(c, p, w + (size_t)e * n, g, r0);
        u64* o = out + (size_t)e * n;
        for (int k = 0; k < n; k++) o[k] = addmod(o[k], r0[k], q);
    }
    free(c1); free(rc1); free(digit); free(r0);
    return 0;
}

/* Rescale (R10, "rescaling ... equivalent to rounding"):
 *   r = centered(iNTT_{q_l}(c[l])),  out[i] = (c[i] - NTT_{q_i}(r mod q_i)) q_l^{-1} mod q_i, i < l.
 * in: [ncomp][l+1][N] -> out: [ncomp][l][N]. */
int or_rescale(const or_ctx* c, const u64* in, int level, int ncomp, u64* out)
{
    if (level < 1) return -2;
    int n = c->n, nl = level + 1;
    u64 ql = c->q[level];
    u64* r = (u64*)malloc(sizeof(u64) * n);
    u64* t = (u64*)malloc(sizeof(u64) * n);
    for (int comp = 0; comp < ncomp; comp++) {
        memcpy(r, in + ((size_t)comp * nl + level) * n, sizeof(u64) * n);
        or_intt(c, level, r);
        for (int i = 0; i < level; i++) {
            u64 q = c->q[i];
            u64 inv = invmod(ql % q, q);
            for (int k = 0; k < n; k++) t[k] = centered_mod(r[k], ql, q);
            or_ntt(c, i, t);
            const u64* a = in + ((size_t)comp * nl + i) * n;
            u64* o = out + ((size_t)comp * level + i) * n;
            for (int k = 0; k < n; k++) o[k] = mulmod(submod(a[k], t[k], q), inv, q);
        }
    }
    free(r);
    free(t);
    return 0;
}

/* Drop the top limbs without scaling (mod-switch): residues of the kept primes unchanged. */
void or_drop_level(const or_ctx* c, const u64* in, int level, int new_level, int ncomp, u64* out)
{
    int n = c->n;
    for (int comp = 0; comp < ncomp; comp++)
        for (int p = 0; p <= new_level; p++)
            memcpy(out + ((size_t)comp * (new_level + 1) + p) * n,
                   in + ((size_t)comp * (level + 1) + p) * n, sizeof(u64) * n);
}
