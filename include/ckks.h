/*
 * ckks.h -- C-ABI of the B200 CKKS encrypted-dense-layer library (libckks_b200.so).
 *
 * What it computes: the server side of CryptoTL (arXiv 2205.11935): dense layers with plaintext
 * weights applied to a CKKS ciphertext by the baby-step/giant-step diagonal method (PAPER.md L92-96,
 * Eq. 1), the polynomial activation (square, or Eq. 2 at PAPER.md L112) and rescaling (PAPER.md
 * L85), over an RNS ring Z_Q[X]/(X^N + 1).  CKKS internals the paper leaves to SEAL
 * follow the readings R1-R24 of DESIGN.md section 3.
 *
 * Conventions shared by every call
 *   - All device memory is owned by the caller (e.g. torch tensors).  The context BORROWS the
 *     tables/keys/workspace buffers passed to ckks_ctx_create; layers and models borrow theirs.
 *     Nothing is allocated on the device by the library after creation.
 *   - Ciphertext layout: `data` = device pointer to [batch][n_comp][level+1][N] uint64 words,
 *     NTT (evaluation) domain, residue of limb i modulo q_i in canonical range [0, q_i).
 *     n_comp is 2 (or 3 between ckks_mul and ckks_relinearize).
 *   - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream).
 *     Preconditions (level, scale, key presence, shapes) are checked on the host before launch.
 *   - Calls on one ckks_ctx must be stream-ordered (one stream, or events inserted by the caller):
 *     key switching, hoisted rotations and rescale use scratch space inside the context's workspace
 *     buffer, so two calls on the same context running concurrently on different streams would race.
 *   - SECURITY: keys and encryption randomness come from a seeded counter-based generator (SplitMix64,
 *     reading R15 of DESIGN.md) so that the CPU oracle can reproduce them bit for bit.  It is NOT a
 *     CSPRNG: anyone who knows the 64-bit seed recovers the secret key.  TEST/BENCHMARK USE ONLY.
 *   - Return value: CKKS_OK (0) or a negative ckks_status; ckks_last_error() gives a message
 *     (thread-local).  On error nothing has been launched.
 *   - There is no CPU fallback: without a CUDA device every compute call returns CKKS_E_CUDA.
 */
#ifndef CKKS_B200_H
#define CKKS_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    CKKS_OK = 0,
    CKKS_E_PARAM = -1,  /* bad N / chain / scale / argument            */
    CKKS_E_LEVEL = -2,  /* depth exhausted: rescale at level 0          */
    CKKS_E_NOKEY = -3,  /* rotation step without a Galois key, or no relin key       */
    CKKS_E_SCALE = -4,  /* scales of an addition differ by more than 2^-40 relative   */
    CKKS_E_DOMAIN = -5, /* representation misuse                                              */
    CKKS_E_SHAPE = -6,  /* level / batch / component mismatch, aliasing not allowed            */
    CKKS_E_CUDA = -7,   /* CUDA error or no device                                             */
    CKKS_E_SIZE = -8    /* caller buffer too small / batch above the context's max_batch       */
} ckks_status;

typedef struct ckks_ctx ckks_ctx;
typedef struct ckks_model ckks_model;

/* Scheme parameters (R1, R13-R15).  Primes: for each entry of prime_bits in order, the largest
 * unused prime q < 2^bits with q = 1 mod 2N; the first n_data are q_0..q_{L-1}, then the special
 * primes P_0..P_{K-1} (K = n_special) used by key switching, P = P_0 ... P_{K-1}.  Keys are generated
 * on the device from key_seed.
 * Key switching (readings R9b/R10b/R17b): the data primes are split into dnum
 * digits of consecutive primes (digit_sizes, each 1 or 2; NULL = one digit per prime);
 * K = 2 special primes with 2-prime digits is the hybrid form (fewer ModUp NTTs: dnum digits instead
 * of L, each lifted by an exact 2-prime CRT).  Switching keys are [dnum][2][L+K][N]. */
typedef struct {
    uint32_t log_n;             /* 10..14 (N = 1024 .. 16384; one limb must fit shared memory)     */
    uint32_t n_data;            /* L >= 1 data primes                                              */
    uint32_t n_special;         /* 0 (NTT-only context), 1 or 2 special primes                     */
    const uint32_t* prime_bits; /* n_data + n_special entries, each in [log_n + 2, 61]             */
    double sigma;               /* discrete Gaussian error parameter, 3.2 (R13)                    */
    uint64_t key_seed;          /* seed of the counter-based PRNG for s, pk, relin and Galois keys */
    const int32_t* rot_steps;   /* rotation steps needing Galois keys (left rotation by step)      */
    uint32_t n_rot_steps;
    int32_t want_relin;         /* generate the relinearisation key (s^2 -> s)                     */
    uint32_t max_batch;         /* ciphertexts per internal launch sequence (workspace sizing)     */
    uint32_t bsgs_baby_extra;   /* dense layers of this context use t1 = 2^(ceil(log2 t / 2) + x)   */
                                /* baby steps (x = this, 0..4; R5 is x = 0, see ckks_bsgs_plan_x);  */
                                /* rot_steps must cover the resulting baby/giant steps               */
    const uint32_t* digit_sizes; /* n_digits entries in {1, 2} summing to n_data, or NULL (all 1)     */
    uint32_t n_digits;
} ckks_params;

/* Host-readable context description. */
typedef struct {
    uint32_t log_n, n, n_data, n_special, n_keys;
    uint64_t primes[16];        /* q_0..q_{L-1}, then P_0..P_{K-1}                                 */
    uint64_t psi[16];           /* minimal primitive 2N-th root used by the NTT (R2)               */
    uint32_t n_digits;          /* key-switching digits dnum                                       */
    uint32_t digit_sizes[16];
} ckks_info;

/* Layer kinds (the paper's frozen stack).  Every layer is evaluated as
 *   y = sum_{k<t2} rot_{k giant}( sum_{j<t1} pt_{k t1 + j} o rot_{baby_steps[j]}(x) )  (+ bias)
 * with one rescale: the BSGS dense (Eq. 1), the packed-SISO conv1d (L98, R26) and the
 * average pool (L100-103, R27).  Multi-item packing (L115-116, R25): item r of p lives in slots
 * [r R, r R + t) (R = region size); layer plaintexts hold one copy per item. */
enum { CKKS_LAYER_DENSE = 0, CKKS_LAYER_CONV1D = 1, CKKS_LAYER_AVGPOOL = 2 };
typedef struct {
    int32_t kind;
    uint32_t rows, cols;        /* dense shape; conv/pool: t, t                                    */
    uint32_t t;                 /* item width (distance of a replicate before the next layer)      */
    uint32_t t2;                /* giant steps (1 for conv/pool)                                   */
    uint32_t n_baby;            /* t1 <= 32                                                        */
    const int32_t* baby_steps;  /* n_baby rotation steps, baby_steps[0] == 0                       */
    int32_t giant;              /* giant step (t1 for the dense)                                   */
    uint32_t region, items;     /* R, p (items 1 and region 0 = single item)                       */
    uint32_t level;             /* level of the input ciphertext                                   */
    double pt_scale, bias_scale;
} ckks_layer_desc;

/* One stage of a model: optional replicate y + rot_{-t}(y) before the layer, activation after it. */
typedef struct ckks_layer ckks_layer;
typedef struct {
    const ckks_layer* layer;
    int32_t activation;         /* 0 none, 1 square, 2 cubic (Eq. 2)                               */
    uint32_t replicate_t;       /* 0 = no replicate                                                */
} ckks_stage;

typedef struct {
    uint64_t* data;  /* device [batch][n_comp][level+1][N]                                         */
    uint32_t batch;
    uint32_t n_comp;
    uint32_t level;  /* limbs = level + 1                                                          */
    double scale;    /* tracked scale (real)                                                       */
} ckks_ct;

const char* ckks_last_error(void);

/* ---- context (setup; not on the hot path) -------------------------------------------------- */
/* Byte sizes of the three device buffers ckks_ctx_create needs (each 256-byte aligned). */
ckks_status ckks_ctx_sizes(const ckks_params* p, size_t* table_bytes, size_t* key_bytes, size_t* work_bytes);
/* Builds primes/tables on the host, uploads them, and generates s, pk, relin key and the Galois
 * keys on the device (seeded; synchronises `stream` before returning).  Borrows the buffers. */
ckks_status ckks_ctx_create(const ckks_params* p, void* d_tables, void* d_keys, void* d_work, void* stream,
                            ckks_ctx** out);
void ckks_ctx_destroy(ckks_ctx* ctx);
ckks_status ckks_ctx_info(const ckks_ctx* ctx, ckks_info* out);
/* Process-wide kernel selection for measured A/B runs (not a precision or semantics switch: every choice gives
 * the same bits).  "mac_tc": 1 = the BSGS inner sums of double-hoisted layers on the integer tensor cores
 * (tcgen05.mma kind::i8, TMEM accumulators, TMA operand staging; k_mac_tc.cu), 0 = on the FP64 tensor cores
 * (DMMA, the default: faster in the measured A/B).  "ip_v3": 1 (default) = the baby-step
 * key-switch inner product with the pre-multiplied key (k_ipmma3.cu), 0 = the Karatsuba form (k_ipmma.cu).
 * "ntt_q": bit mask selecting the CTA-pair FP64 NTT schedule (ntt_c.cuh: thread-block clusters, TMA row copies):
 * 1 batch NTT forward, 2 batch NTT inverse, 4 key-switch ModUp at N <= 8192, 8 ModUp at N = 16384, 64 plain 256-bit
 * accesses instead of the TMA copies; default 15.  "giant_multi": 1 (default) = all giant steps of a double-hoisted layer accumulated in one
 * pass (k_ks_ip_giant_multi), 0 = one accumulator pass per step.  "nvtx": 1 = an NVTX range around every hot-path launch site
 * (named by kernel class), default 0 (env CKKS_NVTX).  Takes effect for launches issued after the call.
 * CKKS_E_PARAM for an unknown name or value. */
ckks_status ckks_set_option(const char* name, int64_t value);
ckks_status ckks_get_option(const char* name, int64_t* value);
/* Number of kernels this context has launched so far (bench accounting). */
uint64_t ckks_launch_count(const ckks_ctx* ctx);
/* Measurement probe: from now on record a CUDA event pair, on the launching stream, around every
 * launch of one kernel class: kind 1 = key-switch ModUp NTT kernel, 2 = a whole key switch
 * (5 kernels), 3 = batched NTT (ckks_ntt_fwd/inv); 0 = off.  Resets the accumulated record.
 * ckks_probe_read synchronises on the last event and returns the summed device time (ms) and the
 * number of probed launches, and (alg_bytes, may be NULL) the algorithmic HBM bytes of those launches
 * as defined in DESIGN.md section 7.  Costs two event records per probed launch; off by default. */
ckks_status ckks_probe_enable(ckks_ctx* ctx, int32_t kind);
ckks_status ckks_probe_read(ckks_ctx* ctx, double* total_ms, uint64_t* launches, double* alg_bytes);
/* kind 4 = every hot-path kernel launch (tagged by kernel name).  Writes a JSON object
 * {"<kernel>": {"ms": total, "launches": n, "alg_bytes": b}, ...} into json (capacity cap). */
ckks_status ckks_probe_read_all(ckks_ctx* ctx, char* json, size_t cap);

/* ---- ring: batched negacyclic NTT ---------------------------------------- */
/* In place over d = device [batch][limbs][N]; limb i is reduced modulo prime i.  Forward maps
 * coefficients (any residues in [0, q_i)) to NTT(a)[k] = sum_j a_j psi^{(2 brev(k)+1) j}
 * (bit-reversed order, R2); inverse is its exact inverse.  limbs <= n_data + n_special. */
/* batch == 0 is a no-op (d may be NULL); limbs must be in [1, number of primes] else CKKS_E_SHAPE. */
ckks_status ckks_ntt_fwd(ckks_ctx* ctx, uint64_t* d, uint32_t batch, uint32_t limbs, void* stream);
ckks_status ckks_ntt_inv(ckks_ctx* ctx, uint64_t* d, uint32_t batch, uint32_t limbs, void* stream);

/* ---- CKKS evaluator (rows a3-a5, a8, a10) --------------------------------------------------- */
/* Left rotation of every slot vector by `step`: (sigma_g(c0), 0) +
 * KS(sigma_g(c1); gk_g), g = 5^(step mod N/2) mod 2N, non-hoisted (R11).  out must not alias in;
 * out->data is written, its level/scale/batch/n_comp are set.  CKKS_E_NOKEY if no key for g. */
ckks_status ckks_rotate(ckks_ctx* ctx, const ckks_ct* in, int32_t step, ckks_ct* out, void* stream);
/* Hoisted rotations (R11b): n_steps rotations of the same input
 * sharing one ModUp of the unrotated c1: out_s = (sigma_g(c0), 0) + ModDown(sum_j sigma_g(D_j) gk_j)
 * with D_j = ModUp of the unsigned digits of c1 -- computed as sigma_g(c0 + ModDown(sum_j D_j key'_j))
 * with pre-permuted keys.  Residues differ from ckks_rotate (different digit lift); both decrypt
 * to the rotated slots.  outs: array of n_steps ciphertext descriptors (device data preallocated). */
ckks_status ckks_rotate_hoisted(ckks_ctx* ctx, const ckks_ct* in, const int32_t* steps, uint32_t n_steps,
                                ckks_ct* outs, void* stream);
/* Tensor product (a0 b0, a0 b1 + a1 b0, a1 b1); equal level and batch; out3 has 3 components. */
ckks_status ckks_mul(ckks_ctx* ctx, const ckks_ct* a, const ckks_ct* b, ckks_ct* out3, void* stream);
/* (c0, c1, c2) -> (c0, c1) + KS(c2; rlk).  in3 has 3 components; out must not alias in3. */
ckks_status ckks_relinearize(ckks_ctx* ctx, const ckks_ct* in3, ckks_ct* out, void* stream);
/* Divide by q_l with rounding and drop limb l (R10); scale /= q_l.
 * CKKS_E_LEVEL at level 0.  Works for 2 or 3 components.  out must not alias in. */
ckks_status ckks_rescale(ckks_ctx* ctx, const ckks_ct* in, ckks_ct* out, void* stream);
/* Slot-wise sum; equal level, batch, n_comp and scale (CKKS_E_SCALE beyond 2^-40 relative). */
ckks_status ckks_add(ckks_ctx* ctx, const ckks_ct* a, const ckks_ct* b, ckks_ct* out, void* stream);

/* ---- dense layer (Eq. 1, rows a6, a7, a9) ---------------------------------------------------- */
/* Device bytes of an encoded rows x cols layer whose input ciphertext is at `level`. */
ckks_status ckks_layer_sizes(const ckks_ctx* ctx, uint32_t rows, uint32_t cols, uint32_t level, size_t* dev_bytes);
/* Encode W (host, row-major rows x cols, float64) and bias (host, rows, may be NULL) with the
 * library's own encoder: diag'_i zero-padded to t x t, t1 = 2^ceil(ceil(log2 t)/2)
 * (R5), plaintext scale q_level (R8), bias at scale in_scale and level-1.  Borrows dev_buf. */
ckks_status ckks_layer_create(ckks_ctx* ctx, const double* W, uint32_t rows, uint32_t cols, const double* bias,
                              uint32_t level, double in_scale, void* dev_buf, void* stream, ckks_layer** out);
/* Same layer from already-encoded integer coefficients: diag_coeffs host [t][N] int64 (diag'_i
 * encodings, i < t), bias_coeffs host [N] int64 (may be NULL).  Used to feed both the oracle and
 * the library the same plaintexts (SURVEY 7 hard part 2). */
ckks_status ckks_layer_import(ckks_ctx* ctx, const int64_t* diag_coeffs, const int64_t* bias_coeffs, uint32_t rows,
                              uint32_t cols, uint32_t level, double pt_scale, double bias_scale, void* dev_buf,
                              void* stream, ckks_layer** out);
void ckks_layer_destroy(ckks_layer* layer);
/* f-2 constructors (library encoder).  dense with p items in regions of R slots (R >= 2t); conv1d
 * with f taps ('same', zero padded, centre tap first), scalar bias on [rR, rR + t); avgpool of size f
 * (right-aligned window, 1/f mask on [rR + f - 1, rR + t)).  dev_buf: ckks_layer_general_sizes bytes
 * for t (dense), f (conv, pool) plaintexts. */
ckks_status ckks_dense_create_packed(ckks_ctx* ctx, const double* W, uint32_t rows, uint32_t cols, const double* bias,
                                     uint32_t region, uint32_t items, uint32_t level, double in_scale, void* dev_buf,
                                     void* stream, ckks_layer** out);
ckks_status ckks_conv1d_create(ckks_ctx* ctx, const double* w, uint32_t f, double bias, uint32_t t, uint32_t region,
                               uint32_t items, uint32_t level, double in_scale, void* dev_buf, void* stream,
                               ckks_layer** out);
ckks_status ckks_avgpool_create(ckks_ctx* ctx, uint32_t f, uint32_t t, uint32_t region, uint32_t items, uint32_t level,
                                void* dev_buf, void* stream, ckks_layer** out);
ckks_status ckks_layer_general_sizes(const ckks_ctx* ctx, uint32_t n_plaintexts, uint32_t level, size_t* dev_bytes);
/* Any layer from already-encoded plaintexts: pt_coeffs host [t2 * n_baby][N] int64 in (k, j) order,
 * bias_coeffs host [N] or NULL (parity path: the oracle's encodings). */
ckks_status ckks_layer_import_general(ckks_ctx* ctx, const ckks_layer_desc* desc, const int64_t* pt_coeffs,
                                      const int64_t* bias_coeffs, void* dev_buf, void* stream, ckks_layer** out);
/* Workspace (device bytes) ckks_matvec_diag / ckks_encrypted_forward need for `batch` cts. */
ckks_status ckks_layer_work_sizes(const ckks_ctx* ctx, const ckks_layer* layer, uint32_t batch, size_t* bytes);
/* Rotation schedule ckks_matvec_diag uses for this layer: 0 = every rotation
 * non-hoisted (R11, default); 1 = baby steps hoisted (R11b); 2 = double hoisting (R11c): baby steps,
 * inner sums and giant steps stay in the Q_l P basis and one ModDown per layer returns to Q_l.  The three
 * give different residues (different rounding points) that decrypt to the same slots.  CKKS_E_PARAM
 * for any other mode. */
ckks_status ckks_layer_set_hoisting(ckks_layer* layer, int32_t mode);
/* y = sum_k rot_{k t1}(sum_j diag'_{k t1+j} o rot_j(x)) (Eq. 1), one rescale (R7), + bias.
 * in at the layer's level; out at level-1, scale = in scale.  work: ckks_layer_work_sizes bytes. */
ckks_status ckks_matvec_diag(ckks_ctx* ctx, const ckks_layer* layer, const ckks_ct* in, ckks_ct* out, void* work,
                             void* stream);

/* ---- model / forward (rows a10-a12) --------------------------------------------------------- */
/* activation: 0 none, 1 square (BASELINE cfg4), 2 cubic ReLU approximation (Eq. 2).
 * Layers must be encoded for the levels/scales the forward produces (see ckks_model_plan, R8).
 * The cubic's constant term c0 is added on the previous layer's valid slots [0, rows) only (R23),
 * from a plaintext the model keeps in dev_buf (ckks_model_sizes bytes; NULL/0 for none/square):
 * act_coeffs = host [n_layers-1][N] int64 encodings of those plaintexts, or NULL to encode here. */
ckks_status ckks_model_sizes(const ckks_ctx* ctx, uint32_t n_layers, int32_t activation, size_t* dev_bytes);
ckks_status ckks_model_create(ckks_ctx* ctx, const ckks_layer* const* layers, uint32_t n_layers, int32_t activation,
                              const int64_t* act_coeffs, void* dev_buf, void* stream, ckks_model** out);
/* General stage list (e.g. the paper's depth-6 frozen stack: conv -> [rep] dense+cubic -> pool ->
 * [rep] dense).  act_coeffs: host [n][N], row i = the masked c0 plaintext of stage i when its
 * activation is cubic (NULL: encoded here on the layer's rows of every item). */
ckks_status ckks_model_stages_sizes(const ckks_ctx* ctx, const ckks_stage* stages, uint32_t n, size_t* dev_bytes);
ckks_status ckks_model_create_stages(ckks_ctx* ctx, const ckks_stage* stages, uint32_t n, const int64_t* act_coeffs,
                                     void* dev_buf, void* stream, ckks_model** out);
void ckks_model_destroy(ckks_model* model);
/* Rotation schedule of every layer of the model, as ckks_layer_set_hoisting: 0 none, 1 hoisted baby
 * steps (ckks_rotate_hoisted semantics), 2 double hoisting (R11c).  CKKS_E_PARAM for other values. */
ckks_status ckks_model_set_hoisting(ckks_model* model, int32_t on);
/* BSGS split of a rows x cols layer: t = max(rows, cols) padded to a multiple of
 * t1 = 2^ceil(ceil(log2 t)/2), t2 = t / t1 (R5). */
ckks_status ckks_bsgs_plan(uint32_t rows, uint32_t cols, uint32_t* t, uint32_t* t1, uint32_t* t2);
/* Same with x extra doublings of the baby-step count: t1 = min(2^(ceil(lg/2) + x), 2^lg), lg =
 * ceil(log2 t) (R5b: under double hoisting a baby step costs ~1/6 of a giant step, so x = 1 is
 * cheaper; every split computes the same Eq. 1 product).  CKKS_E_PARAM for x > 4. */
ckks_status ckks_bsgs_plan_x(uint32_t rows, uint32_t cols, uint32_t x, uint32_t* t, uint32_t* t1, uint32_t* t2);
/* Level/scale schedule of a forward (R8): for each layer the level and scale its input has, and
 * the sorted set of rotation steps the forward needs (baby 1..t1-1, giant k t1, replicate -t).
 * steps may be NULL to query the count; *n_steps is its capacity on input, the count on output. */
ckks_status ckks_model_plan(const ckks_ctx* ctx, uint32_t n_layers, const uint32_t* rows, const uint32_t* cols,
                            int32_t activation, uint32_t in_level, double in_scale, uint32_t* layer_level,
                            double* layer_in_scale, int32_t* steps, uint32_t* n_steps);
/* The rotation steps ckks_model_plan lists, without a context (needed to choose the Galois keys of the
 * context itself): rows x cols dense layers with x extra baby-step doublings (R5b).  steps may be NULL
 * to query the count; *n_steps is its capacity on input, the count on output (CKKS_E_SIZE if short). */
ckks_status ckks_model_steps(uint32_t n_layers, const uint32_t* rows, const uint32_t* cols, uint32_t x, int32_t* steps,
                             uint32_t* n_steps);
/* Input level of the model's first stage and the level its output ends at. */
ckks_status ckks_model_levels(const ckks_model* model, uint32_t* in_level, uint32_t* out_level);
/* Device workspace bytes for a forward over `batch` ciphertexts (chunked at max_batch). */
ckks_status ckks_model_work_sizes(const ckks_ctx* ctx, const ckks_model* model, uint32_t batch, size_t* bytes);
/* dense_1 -> act -> replicate -> dense_2 -> ... on a batch of independent
 * ciphertexts; out is written at the final level (sets out->level/scale). */
ckks_status ckks_encrypted_forward(ckks_ctx* ctx, const ckks_model* model, const ckks_ct* in, ckks_ct* out,
                                   void* work, void* stream);
/* Same, end to end from HOST buffers: h_in [batch][2][in_level+1][N] (pinned recommended) is
 * copied to the device chunk by chunk, evaluated, and copied back to h_out [batch][2][out_level+1][N].
 * Synchronises the stream before returning. */
ckks_status ckks_encrypted_forward_host(ckks_ctx* ctx, const ckks_model* model, const uint64_t* h_in,
                                        uint32_t batch, uint32_t in_level, double in_scale, uint64_t* h_out,
                                        uint32_t* out_level, double* out_scale, void* work, void* stream);

/* ---- CUDA graph of a forward (launch overhead) -------------------------- */
/* Captures the whole launch sequence of ckks_encrypted_forward(in -> out, work) for in->batch <=
 * max_batch ciphertexts into a CUDA graph (on a context-owned capture stream ordered after `stream`).
 * The graph binds in->data, out->data and work: ckks_graph_launch replays the forward on `stream`
 * over whatever those buffers hold, with one launch.  Sets out->level/scale.  CKKS_E_SIZE if
 * in->batch > max_batch; key/scale/level errors as ckks_encrypted_forward (nothing captured). */
typedef struct ckks_graph ckks_graph;
ckks_status ckks_forward_graph_create(ckks_ctx* ctx, const ckks_model* model, const ckks_ct* in, ckks_ct* out,
                                      void* work, void* stream, ckks_graph** graph);
ckks_status ckks_graph_launch(ckks_graph* graph, void* stream);
void ckks_graph_destroy(ckks_graph* graph);

/* ---- client-side helpers (off the hot path) ------------------------------------------------ */
/* values (count <= N/2 reals) -> int64 coefficients m[N] = round(scale * inverse embedding) (R4). */
ckks_status ckks_encode(const ckks_ctx* ctx, const double* values, uint32_t count, double scale, int64_t* coeffs);
/* Public-key encryption at the top level of host coefficients [batch][N] (R6, R17); the randomness
 * of ciphertext i comes from (enc_seed, first_index + i).  out->data device [batch][2][L][N]. */
ckks_status ckks_encrypt(ckks_ctx* ctx, const int64_t* h_coeffs, uint32_t batch, uint64_t enc_seed,
                         uint64_t first_index, double scale, ckks_ct* out, void* stream);
/* Client side on the device: the same three steps without host round trips.
 * ckks_encode_device: d_values device [batch][values_stride] doubles (the first `count` <= N/2 of each row)
 *   -> d_coeffs device [batch][N] int64 = round_half_away(inverse canonical embedding of scale * values) (R4,
 *   R16), one n-point FFT per vector in FP64 (k_encode.cu); may differ by +-1 from ckks_encode on a
 *   coefficient lying within rounding error of a half-integer.  Requires |scale * value| small enough that
 *   every coefficient fits int64 (not checked on the device).
 * ckks_encrypt_device: as ckks_encrypt, from device coefficients [batch][N]; no host synchronisation.
 * ckks_decode_device: decrypted residues d_residues device [batch][level+1][N] (ckks_decrypt) -> d_values
 *   device [batch][count] real slot values / scale (centred CRT lift in FP64, forward FFT). */
ckks_status ckks_encode_device(ckks_ctx* ctx, const double* d_values, uint32_t count, size_t values_stride,
                               uint32_t batch, double scale, int64_t* d_coeffs, void* stream);
ckks_status ckks_encrypt_device(ckks_ctx* ctx, const int64_t* d_coeffs, uint32_t batch, uint64_t enc_seed,
                                uint64_t first_index, double scale, ckks_ct* out, void* stream);
ckks_status ckks_decode_device(ckks_ctx* ctx, const uint64_t* d_residues, uint32_t level, uint32_t batch,
                               double scale, double* d_values, uint32_t count, void* stream);
/* c0 + c1 s, inverse NTT: d_out device [batch][level+1][N] coefficient residues. */
ckks_status ckks_decrypt(ckks_ctx* ctx, const ckks_ct* in, uint64_t* d_out, void* stream);
/* Host decode of one decrypted [level+1][N] residue block: centered CRT lift, canonical
 * embedding, / scale -> values[count]. */
ckks_status ckks_decode(const ckks_ctx* ctx, const uint64_t* h_residues, uint32_t level, double scale, double* values,
                        uint32_t count);
/* Export key material to host memory (synchronises `stream`):
 *   key_id 0 = relinearisation key, key_id = g (odd) = Galois key: [dnum][2][L+K][N] NTT form;
 *   key_id -1 = secret s in NTT form over all primes [L + n_special][N];
 *   key_id -2 = public key [2][L][N] NTT form.  (Test/parity use only.) */
ckks_status ckks_export_key(ckks_ctx* ctx, int64_t key_id, uint64_t* h_out, void* stream);
/* Galois element of a left rotation by step (R3). */
uint64_t ckks_galois_elt(const ckks_ctx* ctx, int32_t step);

#ifdef __cplusplus
}
#endif
#endif /* CKKS_B200_H */
