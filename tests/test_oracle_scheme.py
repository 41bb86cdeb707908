"""Pins of the oracle's CKKS layer: encode/decode definitions, exact big-integer identities for
rescale and key switching, scheme correctness (decrypt within noise), rotation semantics.

Expected values come from: direct-sum definitions (encoding), Python big-integer arithmetic with
schoolbook negacyclic products (rescale / key switch), the worked examples in tests/golden, and
float64 arithmetic on the decoded slots.
"""
import numpy as np
import pytest

import oracle
from oracle import circuits as C
from oracle import encoding as E
import synthetic as S

from test_oracle_ring import schoolbook_negacyclic


def small_ctx(log_n=4, relin=True, steps=(), bits=None):
    bits = bits or (S.CFG1.data_bits, S.CFG1.special_bits)
    ctx = oracle.Context(log_n, bits[0], bits[1])
    ctx.keygen(1234, steps, relin=relin)
    return ctx


def crt(residues, primes):
    Q = 1
    for q in primes:
        Q *= q
    out = []
    for k in range(len(residues[0])):
        x = 0
        for i, q in enumerate(primes):
            Qi = Q // q
            x += int(residues[i][k]) * Qi * pow(Qi, -1, q)
        out.append(x % Q)
    return out, Q


def centered(x, m):
    x %= m
    return x - m if x > m // 2 else x


# ------------------------------------------------------------------------------- encoding
def test_encode_fft_equals_direct_definition():
    rng = np.random.default_rng(0)
    for log_n in (3, 5, 7):
        n = 1 << log_n
        z = rng.uniform(-1, 1, n // 2)
        direct = E.encode_direct(z, 2.0 ** 30, n)
        assert np.array_equal(E.encode(z, 2.0 ** 30, n), E.round_half_away(direct).astype(np.int64))
        m = E.encode(z, 2.0 ** 30, n)
        assert np.allclose(E.decode_coeffs(m, 2.0 ** 30, n), E.decode_direct(m, 2.0 ** 30, n), atol=1e-12)


def test_encode_defining_property():
    """m(zeta^{5^i}) = Delta z_i up to rounding: evaluate the integer polynomial with numpy."""
    n = 64
    z = np.random.default_rng(1).uniform(-1, 1, n // 2)
    m = E.encode(z, 2.0 ** 40, n)
    e = E.slot_exponents(n)
    zeta = np.exp(1j * np.pi / n)
    vals = np.array([np.polyval(m[::-1].astype(np.float64), zeta ** int(ei)) for ei in e])
    assert np.max(np.abs(vals / 2.0 ** 40 - z)) < 1e-9
    assert np.array_equal(E.encode(np.zeros(n // 2), 2.0 ** 40, n), np.zeros(n, dtype=np.int64))


def test_encode_roundtrip_bound(golden):
    g = golden["encode_roundtrip"]
    n = 8192
    v = np.zeros(n // 2)
    v[: len(g["v_head"])] = g["v_head"]
    m = E.encode(v, 2.0 ** g["log2_scale"], n)
    back = E.decode_coeffs(m, 2.0 ** g["log2_scale"], n).real
    assert np.max(np.abs(back - v)) <= g["bound"]


def test_crt_lift():
    primes = [1152921504606830593, 1099511480321, 1099510890497]
    Q = primes[0] * primes[1] * primes[2]
    xs = [0, 1, -1, Q // 2, -(Q // 2), 123456789123456789123456789 % (Q // 2)]
    res = np.array([[x % q for x in xs] for q in primes], dtype=np.uint64)
    assert E.crt_lift_centered(res, primes) == xs


def test_rotation_semantics(golden):
    """sigma_5 on the plaintext polynomial rotates the decoded slots left by 1."""
    g = golden["rotate_left_1"]
    n = 32
    v = np.zeros(n // 2)
    v[: len(g["v_head"])] = g["v_head"]
    m = E.encode(v, 2.0 ** 40, n)
    ctx = oracle.Context(5, (), (), primes=[1152921504606830593])
    q = ctx.primes[0]
    res = np.array([x % q for x in m.tolist()], dtype=np.uint64)
    r = ctx.automorphism_coef(res, 0, ctx.galois_elt(g["step"]))
    out = E.decode(r[None, :], [q], 2.0 ** 40, n)
    assert np.allclose(out[:4], g["expect_head"], atol=1e-9)
    assert abs(out[-1] - g["expect_last"]) < 1e-9


# ------------------------------------------------------------------------------- exact identities
def test_rescale_exact_bigint_identity():
    """R10: CRT(out) = round(CRT(c) / q_l) mod Q_{l-1}, at N=16 with the cfg1 primes."""
    ctx = small_ctx()
    n, primes = ctx.n, ctx.primes[:3]
    rng = np.random.default_rng(5)
    ct = np.stack([np.stack([rng.integers(0, q, n, dtype=np.uint64) for q in primes]) for _ in range(2)])
    out = ctx.rescale(ct)
    for comp in range(2):
        cin, Q = crt([ctx.intt(ct[comp, i], i) for i in range(3)], primes)
        cout, Q2 = crt([ctx.intt(out[comp, i], i) for i in range(2)], primes[:2])
        for x, y in zip(cin, cout):
            xc = centered(x, Q)
            r = centered(xc, primes[2])
            assert (xc - r) % primes[2] == 0
            assert ((xc - r) // primes[2]) % Q2 == y


def _keyswitch_by_bigint(ctx, d_ntt, key, level):
    """KS from its definition: digits d_j (ints in [0,q_j)), U_c = sum_j d_j * key_{j,c} over Q_l P
    with schoolbook products per prime, out_c = round(U_c / P) mod Q_l."""
    n = ctx.n
    L = ctx.n_data
    nl = level + 1
    ext = list(range(nl)) + [L]
    P = ctx.primes[L]
    digits = [[int(v) for v in ctx.intt(d_ntt[j], j)] for j in range(nl)]
    outs = []
    for comp in range(2):
        per_prime = []
        for p in ext:
            q = ctx.primes[p]
            acc = [0] * n
            for j in range(nl):
                kc = [int(v) for v in ctx.intt(key[j, comp, p], p)]
                prod = schoolbook_negacyclic([x % q for x in digits[j]], kc, q)
                acc = [(a + b) % q for a, b in zip(acc, prod)]
            per_prime.append(acc)
        U, QP = crt(per_prime, [ctx.primes[p] for p in ext])
        Ql = QP // P
        res = []
        for x in U:
            r = centered(x, P)
            res.append(((x - r) // P) % Ql)
        outs.append(res)
    return outs


@pytest.mark.parametrize("level", [2, 1])
def test_keyswitch_exact_bigint(level):
    """R-KS: the RNS ModUp/inner-product/ModDown equals the big-integer definition exactly."""
    ctx = small_ctx(steps=(1,))
    n = ctx.n
    rng = np.random.default_rng(9)
    d = np.stack([rng.integers(0, ctx.primes[i], n, dtype=np.uint64) for i in range(level + 1)])
    for key_id in (0, ctx.galois_elt(1)):
        out = ctx.keyswitch(d, key_id)
        ref = _keyswitch_by_bigint(ctx, d, ctx.export_key(key_id), level)
        for comp in range(2):
            got, _ = crt([ctx.intt(out[comp, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
            assert got == ref[comp]


def test_keyswitch_decrypts_to_d_times_sprime():
    """u0 + u1 s = d s' + small, s' = s^2 (relin) or sigma_g(s) (Galois); schoolbook big ints."""
    ctx = small_ctx(log_n=5, steps=(3,))
    n, L = ctx.n, ctx.n_data
    level = L - 1
    s = [int(v) for v in ctx.export_secret()]
    rng = np.random.default_rng(2)
    d = np.stack([rng.integers(0, ctx.primes[i], n, dtype=np.uint64) for i in range(L)])
    primes = ctx.primes[:L]
    g = ctx.galois_elt(3)
    s2 = schoolbook_negacyclic(s, s, 1 << 200)
    s2 = [centered(x, 1 << 200) for x in s2]
    sg = [0] * n
    for i, c in enumerate(s):
        e = (i * g) % (2 * n)
        if e < n:
            sg[e] += c
        else:
            sg[e - n] -= c
    for key_id, sp in ((0, s2), (g, sg)):
        u = ctx.keyswitch(d, key_id)
        for i, q in enumerate(primes):
            u0 = [int(v) for v in ctx.intt(u[0, i], i)]
            u1 = [int(v) for v in ctx.intt(u[1, i], i)]
            dd = [int(v) for v in ctx.intt(d[i], i)]
            lhs = [(a + b) % q for a, b in zip(u0, schoolbook_negacyclic(u1, [x % q for x in s], q))]
            rhs = schoolbook_negacyclic(dd, [x % q for x in sp], q)
            err = [centered(a - b, q) for a, b in zip(lhs, rhs)]
            assert max(abs(e) for e in err) < 2 ** 12


# ------------------------------------------------------------------------------- scheme
def enc_vec(ctx, v, scale, index=0):
    return C.Ct(ctx.encrypt(E.encode(v, scale, ctx.n), 77, index), scale)


def dec_vec(ctx, ct):
    return E.decode(ctx.decrypt(ct.data), ctx.primes, ct.scale, ctx.n)


def test_encrypt_decrypt_roundtrip_and_randomized():
    ctx = small_ctx(log_n=10)
    v = np.random.default_rng(4).uniform(-1, 1, ctx.n // 2)
    a = enc_vec(ctx, v, 2.0 ** 40, 0)
    b = enc_vec(ctx, v, 2.0 ** 40, 1)
    assert not np.array_equal(a.data, b.data)
    assert np.max(np.abs(dec_vec(ctx, a) - v)) < 2 ** -25
    with pytest.raises(oracle.OracleError):
        ctx.decrypt(np.zeros((3, 3, ctx.n), dtype=np.uint64))


def test_multiply_relin_rescale():
    """dec(rescale(relin(enc(u) (x) enc(v)))) ~ u o v; level-0 rescale refused."""
    ctx = small_ctx(log_n=10)
    rng = np.random.default_rng(6)
    u, v = rng.uniform(-1, 1, ctx.n // 2), rng.uniform(-1, 1, ctx.n // 2)
    a, b = enc_vec(ctx, u, 2.0 ** 40), enc_vec(ctx, v, 2.0 ** 40, 1)
    prod = C.Ct(ctx.rescale(ctx.relinearize(ctx.tensor(a.data, b.data))), 2.0 ** 80 / ctx.primes[2])
    assert np.max(np.abs(dec_vec(ctx, prod) - u * v)) < 1e-6
    low = ctx.rescale(ctx.rescale(a.data))
    with pytest.raises(oracle.OracleError):
        ctx.rescale(low)


def test_rotate_semantics_and_missing_key(golden):
    g = golden["rotate_left_1"]
    ctx = small_ctx(log_n=10, steps=(1, 3, -3))
    v = np.zeros(ctx.n // 2)
    v[:4] = g["v_head"]
    ct = enc_vec(ctx, v, 2.0 ** 40)
    r = dec_vec(ctx, C.Ct(ctx.rotate(ct.data, 1), ct.scale))
    assert np.allclose(r[:4], g["expect_head"], atol=1e-6) and abs(r[-1] - g["expect_last"]) < 1e-6
    back = dec_vec(ctx, C.Ct(ctx.rotate(ctx.rotate(ct.data, 3), -3), ct.scale))
    assert np.allclose(back, v, atol=1e-6)
    assert np.array_equal(ctx.rotate(ct.data, 0), ct.data)
    with pytest.raises(oracle.OracleError):
        ctx.rotate(ct.data, 5)


# ------------------------------------------------------------------------------- circuits
def test_relu_approx_values(golden):
    g = golden["relu_approx"]
    assert tuple(g["coeffs_c3_c2_c1_c0"]) == C.RELU_APPROX
    for z, val in zip(g["z"], g["value"]):
        y = C.plain_forward(np.array([z]), [np.eye(1), np.eye(1)], [np.zeros(1), np.zeros(1)], "cubic")
        assert abs(y[0] - val) < g["abs_tol"]


def test_bsgs_split_and_counts(golden):
    for t, t1, t2 in golden["bsgs_counts"]["cases"]:
        assert C.bsgs_split(t, t) == (t, t1, t2)


def _dense_case(ctx, W, b, x, scale=2.0 ** 40):
    lay = C.encode_layer(ctx, W, b, ctx.top_level, scale)
    ct = enc_vec(ctx, C.pack_input(x, lay.t, ctx.n // 2), scale)
    ops = C.OpCount()
    out = C.matvec(ctx, ct, lay, ops)
    return dec_vec(ctx, out), lay, ops, out


def test_bsgs_toy_t4(golden):
    g = golden["bsgs_t4"]
    W = np.array(g["M"], dtype=np.float64)
    ctx = small_ctx(log_n=6, steps=C.rotation_steps_for([W.shape]))
    y, lay, ops, out = _dense_case(ctx, W / 16.0, None, np.array(g["x"], dtype=np.float64))
    assert np.allclose(y[:4] * 16.0, g["y"], atol=1e-5)
    assert ops.rot == lay.t1 + lay.t2 - 2 and ops.mul_plain == lay.t
    assert out.level == ctx.top_level - 1 and out.scale == 2.0 ** 40


def test_bsgs_identity_and_random():
    ctx = small_ctx(log_n=10, steps=C.rotation_steps_for([(64, 64), (16, 64)]))
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, 64)
    y, _, _, _ = _dense_case(ctx, np.eye(64), None, x)
    assert np.max(np.abs(y[:64] - x)) < 1e-6
    W = rng.normal(0, 0.1, (16, 64))
    b = rng.uniform(-0.1, 0.1, 16)
    y, _, ops, _ = _dense_case(ctx, W, b, x)
    assert np.max(np.abs(y[:16] - (W @ x + b))) < 1e-6
    assert np.max(np.abs(y[16:])) < 1e-6
    assert ops.rot == 14 and ops.mul_plain == 64


def test_cubic_activation_encrypted():
    ctx = small_ctx(log_n=10, bits=((60, 40, 40, 40), (60,)))
    z = np.random.default_rng(10).uniform(-3, 3, ctx.n // 2)
    ct = enc_vec(ctx, z, 2.0 ** 40)
    out = C.cubic(ctx, ct)
    assert out.level == ctx.top_level - 2
    c3, c2, c1, c0 = C.RELU_APPROX
    assert np.max(np.abs(dec_vec(ctx, out) - (((c3 * z + c2) * z + c1) * z + c0))) < 1e-5


def _forward_case(cfg, activation):
    ctx = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    ctx.keygen(cfg.key_seed, C.rotation_steps_for(cfg.layers))
    prob = S.dense_problem(cfg, batch=1)
    Delta = 2.0 ** cfg.log2_scale
    layers = C.encode_model(ctx, prob["W"], prob["b"], ctx.top_level, Delta, activation)
    ct = enc_vec(ctx, C.pack_input(prob["x"][0], layers[0].t, ctx.n // 2), Delta)
    out = C.forward(ctx, ct, layers, activation)
    ref = C.plain_forward(prob["x"][0], prob["W"], prob["b"], activation)
    y = dec_vec(ctx, out)
    return y, ref, out


def test_forward_cfg1_vs_float64():
    """north_star: |decrypt(forward) - float64 forward| <= 1e-3 on valid slots (pinned tighter: 1e-6)."""
    y, ref, out = _forward_case(S.CFG1, "none")
    err = np.max(np.abs(y[: ref.size] - ref))
    assert err < 1e-6
    assert np.max(np.abs(y[ref.size:])) < 1e-6
    assert out.level == 1


@pytest.mark.slow
def test_forward_cfg4_vs_float64():
    y, ref, out = _forward_case(S.CFG4, "square")
    assert np.max(np.abs(y[: ref.size] - ref)) < 1e-5
    assert out.level == 4 and out.data.shape[1] == 5


def test_forward_cubic_small_ring_vs_float64():
    """Two dense layers with the Eq. 2 activation between them (R23 masked constant term) on N=4096."""
    cfg = S.Config(name="small", log_n=12, data_bits=(60,) + (40,) * 5, special_bits=(60,), log2_scale=40,
                   layers=((64, 128), (32, 64)), activation="cubic", in_dim=128,
                   weight_std=(1 / np.sqrt(128), 1 / np.sqrt(64)))
    y, ref, out = _forward_case(cfg, "cubic")
    assert np.max(np.abs(y[: ref.size] - ref)) < 1e-5
    assert out.level == 1


# ------------------------------------------------------------------------------- hoisted rotation (f-1)
def _hoisted_ks_by_bigint(ctx, c1_ntt, key, level, g):
    """Definition: digits of the unrotated c1, sigma_g applied as SIGNED integer polynomials, then
    U = sum_j sigma_g(d_j) * key_j over Q_l P (schoolbook), out = round(U / P)."""
    n, L = ctx.n, ctx.n_data
    nl = level + 1
    ext = list(range(nl)) + [L]
    P = ctx.primes[L]
    digits = []
    for j in range(nl):
        d = [int(v) for v in ctx.intt(c1_ntt[j], j)]
        sd = [0] * n
        for i, v in enumerate(d):
            e = (i * g) % (2 * n)
            if e < n:
                sd[e] = v
            else:
                sd[e - n] = -v
        digits.append(sd)
    outs = []
    for comp in range(2):
        per_prime = []
        for p in ext:
            q = ctx.primes[p]
            acc = [0] * n
            for j in range(nl):
                kc = [int(v) for v in ctx.intt(key[j, comp, p], p)]
                prod = schoolbook_negacyclic([x % q for x in digits[j]], kc, q)
                acc = [(a + b) % q for a, b in zip(acc, prod)]
            per_prime.append(acc)
        U, QP = crt(per_prime, [ctx.primes[p] for p in ext])
        Ql = QP // P
        outs.append([((x - centered(x, P)) // P) % Ql for x in U])
    return outs


@pytest.mark.parametrize("level", [2, 1])
def test_hoisted_rotation_exact_bigint(level):
    ctx = small_ctx(steps=(1, 3))
    n = ctx.n
    rng = np.random.default_rng(21 + level)
    ct = np.stack([np.stack([rng.integers(0, ctx.primes[i], n, dtype=np.uint64) for i in range(level + 1)])
                   for _ in range(2)])
    for step in (1, 3):
        g = ctx.galois_elt(step)
        out = ctx.rotate_hoisted(ct, step)
        ref = _hoisted_ks_by_bigint(ctx, ct[1], ctx.export_key(g), level, g)
        got1, _ = crt([ctx.intt(out[1, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
        assert got1 == ref[1]
        # component 0 = sigma_g(c0) + u0
        c0r = np.stack([ctx.automorphism_ntt(ct[0, i], i, g) for i in range(level + 1)])
        u0 = np.stack([(out[0, i].astype(object) - c0r[i].astype(object)) % ctx.primes[i] for i in range(level + 1)])
        got0, _ = crt([ctx.intt(u0[i].astype(np.uint64), i) for i in range(level + 1)], ctx.primes[: level + 1])
        assert got0 == ref[0]


def test_hoisted_rotation_decrypts_and_differs():
    ctx = small_ctx(log_n=10, steps=(1, 5, -3))
    v = np.random.default_rng(5).uniform(-1, 1, ctx.n // 2)
    ct = enc_vec(ctx, v, 2.0 ** 40)
    for step in (1, 5, -3):
        h = ctx.rotate_hoisted(ct.data, step)
        nh = ctx.rotate(ct.data, step)
        assert not np.array_equal(h, nh)                        # different digit lift -> different residues
        dec = dec_vec(ctx, C.Ct(h, ct.scale))
        assert np.max(np.abs(dec - np.roll(v, -step))) < 1e-6


def test_forward_cfg1_hoisted_vs_float64():
    cfg = S.CFG1
    ctx = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    ctx.keygen(cfg.key_seed, C.rotation_steps_for(cfg.layers))
    prob = S.dense_problem(cfg)
    Delta = 2.0 ** 40
    layers = C.encode_model(ctx, prob["W"], prob["b"], ctx.top_level, Delta, "none")
    ct = enc_vec(ctx, C.pack_input(prob["x"][0], layers[0].t, ctx.n // 2), Delta)
    ops = C.OpCount()
    out = C.forward(ctx, ct, layers, "none", ops, hoisted=True)
    y = dec_vec(ctx, out)
    assert np.max(np.abs(y[:16] - (prob["W"][0] @ prob["x"][0] + prob["b"][0]))) < 1e-6
    assert ops.rot == 14
