"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle, bit-exact on every residue.

Bar (north_star): bit-exact ciphertexts given the same seeded keys, noise and inputs; decrypted
outputs within 1e-3 absolute of the float64 plaintext forward.  Inputs come from `synthetic`; the
oracle's own encoder produces the shared plaintext encodings (SURVEY 7 hard part 2).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle  # noqa: E402
from oracle import circuits as OC  # noqa: E402
from oracle import encoding as OE  # noqa: E402
import synthetic as S  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def gpu_ctx(cfg, steps=(), relin=True, max_batch=4, log_n=None, data_bits=None, special_bits=None):
    return G.Context(log_n or cfg.log_n, data_bits or cfg.data_bits,
                     cfg.special_bits if special_bits is None else special_bits, key_seed=cfg.key_seed,
                     rot_steps=steps, want_relin=relin, max_batch=max_batch)


def oracle_ctx(cfg, steps=(), relin=True, log_n=None, data_bits=None, special_bits=None):
    c = oracle.Context(log_n or cfg.log_n, data_bits or cfg.data_bits,
                       cfg.special_bits if special_bits is None else special_bits)
    c.keygen(cfg.key_seed, steps, relin=relin)
    return c


# ------------------------------------------------------------------------------------------ NTT
@pytest.mark.parametrize("log_n", [10, 11, 12, 13, 14])
def test_ntt_parity_all_sizes(log_n):
    bits = (50,) * 3 + (60,)
    g = G.Context(log_n, bits, (), max_batch=1, want_relin=False)
    o = oracle.Context(log_n, bits, ())
    assert g.primes == o.primes and g.psi == o.psi
    x = S.uniform_residues(11, g.primes, (3,), g.n)          # 3 polys x 4 limbs (ragged vs warps)
    t = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_fwd(t)
    got = u64(t)
    for b in range(3):
        for l in range(4):
            assert np.array_equal(got[b, l], o.ntt(x[b, l], l)), (b, l)
    g.ntt_inv(t)
    assert np.array_equal(u64(t), x)


def test_ntt_cfg2_full_size():
    """BASELINE cfg2 in the bench launch configuration: [1024][8][16384]; sampled limbs vs oracle,
    full inverse round trip; and the inverse on its own vs the oracle on sampled limbs."""
    cfg = S.CFG2
    g = gpu_ctx(cfg, relin=False, max_batch=1)
    o = oracle.Context(cfg.log_n, cfg.data_bits, ())
    assert g.primes == o.primes
    x = S.uniform_residues(cfg.data_seed, g.primes, (cfg.batch,), g.n)
    t = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_fwd(t)
    got = u64(t)
    rng = np.random.default_rng(0)
    for b, l in zip(rng.integers(0, cfg.batch, 6), rng.integers(0, 8, 6)):
        assert np.array_equal(got[b, l], o.ntt(x[b, l], int(l)))
    g.ntt_inv(t)
    assert np.array_equal(u64(t), x)
    t2 = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_inv(t2)
    inv = u64(t2)
    for b, l in zip(rng.integers(0, cfg.batch, 4), rng.integers(0, 8, 4)):
        assert np.array_equal(inv[b, l], o.intt(x[b, l], int(l)))


# ------------------------------------------------------------------------------------------ keys
def test_keys_bit_exact_cfg1():
    cfg = S.CFG1
    steps = (1, 3, -2)
    g = gpu_ctx(cfg, steps)
    o = oracle_ctx(cfg, steps)
    assert g.primes == o.primes and g.psi == o.psi
    s = o.export_secret().astype(np.int64)
    s_ntt = np.stack([o.ntt(np.array([v % q for v in s.tolist()], dtype=np.uint64), i)
                      for i, q in enumerate(o.primes)])
    assert np.array_equal(g.export_key(-1), s_ntt)
    assert np.array_equal(g.export_key(-2), o.export_pk())
    for kid in [0] + [o.galois_elt(st) for st in steps]:
        assert np.array_equal(g.export_key(kid), o.export_key(kid)), kid


# ------------------------------------------------------------------------------------------ scheme
@pytest.fixture(scope="module")
def c1():
    cfg = S.CFG1
    steps = OC.rotation_steps_for(cfg.layers) + [5, -7]
    return cfg, gpu_ctx(cfg, steps, max_batch=2), oracle_ctx(cfg, steps)


def _enc_batch(cfg, o, B, seed=3, scale=2.0 ** 40):
    rng = np.random.default_rng(seed)
    ms = [OE.encode(rng.uniform(-1, 1, o.n // 2), scale, o.n) for _ in range(B)]
    cts = np.stack([o.encrypt(m, cfg.enc_seed, i) for i, m in enumerate(ms)])
    return ms, cts


def test_encrypt_decrypt_parity(c1):
    cfg, g, o = c1
    ms, cts = _enc_batch(cfg, o, 3)
    ct = g.encrypt(np.stack(ms), cfg.enc_seed, 0, 2.0 ** 40)
    assert np.array_equal(u64(ct.data), cts)
    dec = u64(g.decrypt(ct))
    for b in range(3):
        assert np.array_equal(dec[b], o.decrypt(cts[b]))
    # library-side decode of the library-side decryption
    vals = g.decode(dec[0], ct.level, ct.scale)
    ref = OE.decode(o.decrypt(cts[0]), o.primes, 2.0 ** 40, o.n)
    assert np.max(np.abs(vals - ref)) < 1e-9


@pytest.mark.parametrize("step", [1, 3, 5, -7, 56])
def test_rotate_parity_ragged_batch(c1, step):
    cfg, g, o = c1
    ms, cts = _enc_batch(cfg, o, 3, seed=step + 100)       # batch 3 with max_batch 2: ragged chunking
    ct = g.from_numpy(cts, scale=2.0 ** 40)
    out = g.rotate(ct, step)
    got = u64(out.data)
    for b in range(3):
        assert np.array_equal(got[b], o.rotate(cts[b], step)), b


def test_rotate_hoisted_parity(c1):
    """NEXT f-1: hoisted rotations (one ModUp shared by all steps) vs the oracle's hoisted definition."""
    cfg, g, o = c1
    ms, cts = _enc_batch(cfg, o, 3, seed=31)
    ct = g.from_numpy(cts, scale=2.0 ** 40)
    steps = [1, 3, 0, 5, -7, 56]
    outs = g.rotate_hoisted(ct, steps)
    for st, out in zip(steps, outs):
        got = u64(out.data)
        for b in range(3):
            assert np.array_equal(got[b], o.rotate_hoisted(cts[b], st)), (st, b)
    low = o.drop_level(cts[0], 1)
    outs = g.rotate_hoisted(g.from_numpy(low[None], scale=2.0 ** 40), [3])
    assert np.array_equal(u64(outs[0].data)[0], o.rotate_hoisted(low, 3))


def test_rotate_lower_level_and_errors(c1):
    cfg, g, o = c1
    ms, cts = _enc_batch(cfg, o, 1, seed=7)
    low = o.drop_level(cts[0], 1)
    ct = g.from_numpy(low[None], scale=2.0 ** 40)
    assert np.array_equal(u64(g.rotate(ct, 3).data)[0], o.rotate(low, 3))
    with pytest.raises(G.CkksError) as e:
        g.rotate(ct, 11)
    assert e.value.status == G.E_NOKEY
    z = g.from_numpy(o.drop_level(cts[0], 0)[None], scale=2.0 ** 40)
    with pytest.raises(G.CkksError) as e:
        g.rescale(z)
    assert e.value.status == G.E_LEVEL


def test_mul_relin_rescale_parity(c1):
    cfg, g, o = c1
    ms, cts = _enc_batch(cfg, o, 2, seed=9)
    a, b = g.from_numpy(cts[:1], scale=2.0 ** 40), g.from_numpy(cts[1:], scale=2.0 ** 40)
    t3 = g.mul(a, b)
    ref3 = o.tensor(cts[0], cts[1])
    assert np.array_equal(u64(t3.data)[0], ref3)
    r = g.relinearize(t3)
    ref_r = o.relinearize(ref3)
    assert np.array_equal(u64(r.data)[0], ref_r)
    rs = g.rescale(r)
    assert np.array_equal(u64(rs.data)[0], o.rescale(ref_r))
    rs3 = g.rescale(t3)                                      # 3-component rescale
    assert np.array_equal(u64(rs3.data)[0], o.rescale(ref3))
    s = g.add(a, b)
    assert np.array_equal(u64(s.data)[0], o.add(cts[0], cts[1]))
    b.scale = 2.0 ** 41
    with pytest.raises(G.CkksError) as e:
        g.add(a, b)
    assert e.value.status == G.E_SCALE


def test_matvec_cfg1_parity_and_accuracy(c1):
    cfg, g, o = c1
    prob = S.dense_problem(cfg)
    Delta = 2.0 ** cfg.log2_scale
    lay = OC.encode_layer(o, prob["W"][0], prob["b"][0], o.top_level, Delta)
    x = prob["x"][0]
    m = OE.encode(OC.pack_input(x, lay.t, o.n // 2), Delta, o.n)
    ct_o = OC.Ct(o.encrypt(m, cfg.enc_seed, 0), Delta)
    ref = OC.matvec(o, ct_o, lay)
    glay = G.Layer(g, lay.rows, lay.cols, lay.level, diag_coeffs=lay.diag_coeffs, bias_coeffs=lay.bias_coeffs,
                   pt_scale=lay.pt_scale, bias_scale=lay.bias_scale)
    ct = g.from_numpy(ct_o.data[None], scale=Delta)
    out = glay.matvec(ct)
    assert out.level == ref.level and out.scale == ref.scale
    assert np.array_equal(u64(out.data)[0], ref.data)
    dec = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
    assert np.max(np.abs(dec[:16] - (prob["W"][0] @ x + prob["b"][0]))) < 1e-3


def test_library_encoder_vs_oracle_encoder(c1):
    """The library's own encoder (ckks_encode / ckks_layer_create) agrees with the oracle's up to
    +-1 on rare coefficients (float rounding), and its layers decrypt to the float64 result."""
    cfg, g, o = c1
    rng = np.random.default_rng(12)
    v = rng.uniform(-1, 1, o.n // 2)
    a, b = g.encode(v, 2.0 ** 40), OE.encode(v, 2.0 ** 40, o.n)
    d = np.abs(a - b)
    assert d.max() <= 1 and (d > 0).mean() < 1e-3
    prob = S.dense_problem(cfg)
    Delta = 2.0 ** 40
    glay = G.Layer(g, 16, 64, o.top_level, W=prob["W"][0], bias=prob["b"][0], in_scale=Delta)
    m = g.encode(OC.pack_input(prob["x"][0], 64, o.n // 2), Delta)
    ct = g.encrypt(m, cfg.enc_seed, 0, Delta)
    out = glay.matvec(ct)
    dec = u64(g.decrypt(out))[0]
    y = g.decode(dec, out.level, out.scale, 16)
    assert np.max(np.abs(y - (prob["W"][0] @ prob["x"][0] + prob["b"][0]))) < 1e-3


# ------------------------------------------------------------------------------------------ forward
def _model_case(cfg, activation, B, max_batch, data_bits=None, log_n=None, seed_batch=None, hoisted=False, x=0):
    log_n = log_n or cfg.log_n
    data_bits = data_bits or cfg.data_bits
    steps = OC.rotation_steps_for(cfg.layers, x)
    o = oracle.Context(log_n, data_bits, cfg.special_bits)
    o.keygen(cfg.key_seed, steps)
    g = G.Context(log_n, data_bits, cfg.special_bits, key_seed=cfg.key_seed, rot_steps=steps, max_batch=max_batch,
                  bsgs_baby_extra=x)
    prob = S.dense_problem(cfg, batch=B)
    Delta = 2.0 ** cfg.log2_scale
    layers = OC.encode_model(o, prob["W"], prob["b"], o.top_level, Delta, activation, x)
    glayers = [G.Layer(g, l.rows, l.cols, l.level, diag_coeffs=l.diag_coeffs, bias_coeffs=l.bias_coeffs,
                       pt_scale=l.pt_scale, bias_scale=l.bias_scale) for l in layers]
    model = G.Model(g, glayers, {"none": 0, "square": 1, "cubic": 2}[activation],
                    act_coeffs=OC.activation_plaintexts(o, layers, activation))
    if hoisted:
        model.set_hoisting(hoisted)
    ms = np.stack([OE.encode(OC.pack_input(prob["x"][b], layers[0].t, o.n // 2), Delta, o.n) for b in range(B)])
    ct = g.encrypt(ms, cfg.enc_seed, 0, Delta)
    out = model.forward(ct)
    return o, g, prob, layers, ms, ct, out


@pytest.mark.parametrize("activation", ["square", "cubic"])
def test_forward_small_ring_parity(activation):
    """cfg4's two-layer network on a smaller ring (N=4096, 6 data primes) with a ragged batch."""
    cfg = S.CFG4
    o, g, prob, layers, ms, ct, out = _model_case(
        S.Config(name="small", log_n=12, data_bits=(60,) + (40,) * 5, special_bits=(60,), log2_scale=40,
                 layers=((64, 128), (32, 64)), activation=activation, in_dim=128,
                 weight_std=(1 / np.sqrt(128), 1 / np.sqrt(64))), activation, B=3, max_batch=2)
    Delta = 2.0 ** 40
    got = u64(out.data)
    for b in range(3):
        ref = OC.forward(o, OC.Ct(o.encrypt(ms[b], S.CFG4.enc_seed, b), Delta), layers, activation)
        assert out.level == ref.level and abs(out.scale - ref.scale) <= 1e-9 * ref.scale
        assert np.array_equal(got[b], ref.data), b
        dec = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
        W, bb = prob["W"], prob["b"]
        y = OC.plain_forward(prob["x"][b], W, bb, activation)
        assert np.max(np.abs(dec[: y.size] - y)) < 1e-3


def test_forward_cfg4_parity_and_accuracy():
    """BASELINE cfg4 at full size: bit-exact vs the oracle, decrypted within 1e-3 of float64."""
    cfg = S.CFG4
    o, g, prob, layers, ms, ct, out = _model_case(cfg, "square", B=1, max_batch=1)
    Delta = 2.0 ** 40
    ref = OC.forward(o, OC.Ct(o.encrypt(ms[0], cfg.enc_seed, 0), Delta), layers, "square")
    assert np.array_equal(u64(out.data)[0], ref.data)
    dec = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
    y = OC.plain_forward(prob["x"][0], prob["W"], prob["b"], "square")
    assert np.max(np.abs(dec[:128] - y)) < 1e-3
    # the library's own decryption and decoding agree
    gy = g.decode(u64(g.decrypt(out))[0], out.level, out.scale, 128)
    assert np.max(np.abs(gy - y)) < 1e-3


@pytest.mark.parametrize("mode,x", [(1, 0), (2, 0), (2, 1), (0, 2)])
@pytest.mark.parametrize("activation", ["square", "cubic"])
def test_forward_small_ring_hoisted_parity(activation, mode, x):
    o, g, prob, layers, ms, ct, out = _model_case(
        S.Config(name="small", log_n=12, data_bits=(60,) + (40,) * 5, special_bits=(60,), log2_scale=40,
                 layers=((64, 128), (32, 64)), activation=activation, in_dim=128,
                 weight_std=(1 / np.sqrt(128), 1 / np.sqrt(64))), activation, B=3, max_batch=2, hoisted=mode, x=x)
    got = u64(out.data)
    for b in range(3):
        ref = OC.forward(o, OC.Ct(o.encrypt(ms[b], S.CFG4.enc_seed, b), 2.0 ** 40), layers, activation, hoisted=mode)
        assert np.array_equal(got[b], ref.data), b
        y = OC.plain_forward(prob["x"][b], prob["W"], prob["b"], activation)
        dec = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
        assert np.max(np.abs(dec[: y.size] - y)) < 1e-3


@pytest.mark.parametrize("mode,x", [(1, 0), (2, 0), (2, 1)])
def test_forward_cfg4_hoisted_parity_and_accuracy(mode, x):
    """cfg4 at full size (x = 1, mode 2 is the bench's schedule: t1 = 64 / 32, double hoisting)."""
    cfg = S.CFG4
    o, g, prob, layers, ms, ct, out = _model_case(cfg, "square", B=2, max_batch=2, hoisted=mode, x=x)
    for b in range(2):
        ref = OC.forward(o, OC.Ct(o.encrypt(ms[b], cfg.enc_seed, b), 2.0 ** 40), layers, "square", hoisted=mode)
        assert np.array_equal(u64(out.data)[b], ref.data)
        y = OC.plain_forward(prob["x"][b], prob["W"], prob["b"], "square")
        assert np.max(np.abs(OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)[:128] - y)) < 1e-3


def test_rotation_batch_cfg3_sampled():
    """BASELINE cfg3 launch configuration: 256 uniform-residue ciphertexts x 9 steps; sampled outputs
    vs the oracle (uniform residues, so only bit-exact parity is meaningful, R21)."""
    cfg = S.CFG3
    g = gpu_ctx(cfg, cfg.rot_steps, relin=False, max_batch=256)
    o = oracle_ctx(cfg, cfg.rot_steps, relin=False)
    x = S.uniform_residues(cfg.data_seed, g.primes[: g.n_data], (cfg.batch, 2), g.n)
    ct = g.from_numpy(x, scale=2.0 ** 40)
    rng = np.random.default_rng(1)
    for step in cfg.rot_steps:
        out = g.rotate(ct, step)
        got = out.data
        for b in rng.integers(0, cfg.batch, 1):
            assert np.array_equal(u64(got[b]), o.rotate(x[b], step)), (step, b)
    # the hoisted form the bench also times (one ModUp per ciphertext for all 9 steps, R11b)
    outs = g.rotate_hoisted(ct, cfg.rot_steps)
    for step, out in zip(cfg.rot_steps, outs):
        b = int(rng.integers(0, cfg.batch))
        assert np.array_equal(u64(out.data[b]), o.rotate_hoisted(x[b], step)), (step, b)


@pytest.mark.parametrize("bits", [(40,) * 2, (45,) * 2, (50,) * 2, (60,) * 2])
def test_ntt_extreme_residues(bits):
    """Worst cases of the lazy/exactness bounds of every prime class (FP64 q < 2^45, FP64 with
    per-butterfly reduction q < 2^50, 64-bit Shoup above): all-(q-1), alternating 0/(q-1) and
    random limbs at N=16384, forward and inverse vs the oracle, and the round trip."""
    log_n = 14
    g = G.Context(log_n, bits, (), max_batch=1, want_relin=False)
    o = oracle.Context(log_n, bits, ())
    n = g.n
    rng = np.random.default_rng(5)
    rows = []
    for q in g.primes:
        rows.append([np.full(n, q - 1, dtype=np.uint64),
                     np.where(np.arange(n) % 2 == 0, 0, q - 1).astype(np.uint64),
                     rng.integers(0, q, n, dtype=np.uint64)])
    x = np.stack([np.stack([rows[l][k] for l in range(len(bits))]) for k in range(3)])   # [3][limbs][N]
    t = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_fwd(t)
    got = u64(t)
    for b in range(3):
        for l in range(len(bits)):
            assert np.array_equal(got[b, l], o.ntt(x[b, l], l)), (bits, b, l)
    g.ntt_inv(t)
    assert np.array_equal(u64(t), x)
    t2 = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_inv(t2)
    inv = u64(t2)
    for b in range(3):
        for l in range(len(bits)):
            assert np.array_equal(inv[b, l], o.intt(x[b, l], l)), (bits, b, l)


def test_forward_host_buffers_chunked():
    """ckks_encrypted_forward_host (H2D / compute / D2H overlapped on three streams, double-buffered
    staging) on 5 ciphertexts in chunks of 2 (ragged last chunk), twice in a row (staging reuse across
    calls): bit-identical to the device-resident forward and to the oracle."""
    cfg = S.Config(name="small", log_n=12, data_bits=(60,) + (40,) * 5, special_bits=(60,), log2_scale=40,
                   layers=((64, 128), (32, 64)), activation="square", in_dim=128,
                   weight_std=(1 / np.sqrt(128), 1 / np.sqrt(64)))
    steps = OC.rotation_steps_for(cfg.layers, 1)
    o = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    o.keygen(cfg.key_seed, steps)
    g = G.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, key_seed=cfg.key_seed, rot_steps=steps, max_batch=2,
                  bsgs_baby_extra=1)
    B = 5
    prob = S.dense_problem(cfg, batch=B)
    D = 2.0 ** 40
    layers = OC.encode_model(o, prob["W"], prob["b"], o.top_level, D, "square", 1)
    gl = [G.Layer(g, l.rows, l.cols, l.level, diag_coeffs=l.diag_coeffs, bias_coeffs=l.bias_coeffs,
                  pt_scale=l.pt_scale, bias_scale=l.bias_scale) for l in layers]
    model = G.Model(g, gl, G.ACT_SQUARE)
    model.set_hoisting(2)
    ms = np.stack([OE.encode(OC.pack_input(prob["x"][b], layers[0].t, o.n // 2), D, o.n) for b in range(B)])
    ct = g.encrypt(ms, cfg.enc_seed, 0, D)
    work = torch.empty(model.work_bytes(B), dtype=torch.uint8, device="cuda")
    out = model.forward(ct, work=work)
    h_in = torch.empty(tuple(ct.data.shape), dtype=torch.int64, pin_memory=True)
    h_in.copy_(ct.data)
    h_out = torch.empty(tuple(out.data.shape), dtype=torch.int64, pin_memory=True)
    for _ in range(2):
        h_out.zero_()
        lvl, sc = model.forward_host(h_in, ct.level, ct.scale, h_out, work)
        assert lvl == out.level and sc == out.scale
        assert torch.equal(h_out, out.data.cpu())
    ref = OC.forward(o, OC.Ct(o.encrypt(ms[4], cfg.enc_seed, 4), D), layers, "square", hoisted=2)
    assert np.array_equal(h_out.numpy().view(np.uint64)[4], ref.data)
