"""Pins of the oracle's hybrid key switching (readings R9b, R10b, R17b):
dnum < L digits made of consecutive data primes and K = 2 special primes, P = P_0 P_1.

Every expected value is computed here from the definition with Python big integers (CRT of whole digits,
schoolbook negacyclic products per prime, exact division by P with the centred remainder), never from
the oracle's own arithmetic:
  * keys:      key_j.c0 + key_j.c1 s = e_j + [p in digit j] P s'  (mod p, e_j small)           (R17b)
  * digits:    d_j = CRT of the digit's coefficient residues, in [0, Q_j)                          (R9b)
  * KS:        out_c = round(sum_j d_j key_j.c / P) mod Q_l, exactly                              (R10b)
  * ModDown:   (X - [X]_P) / P mod Q_l with the centred residue mod P = P_0 P_1
  * QP steps:  the double-hoisting baby / giant steps (R11c) with the digit groups
  * semantics: KS decrypts to d s' + small; encrypted matvec / forward decrypt to float64.
"""
import numpy as np
import pytest

import oracle
from oracle import circuits as C
from oracle import encoding as E

from test_oracle_ring import schoolbook_negacyclic
from test_oracle_scheme import crt, centered

DATA = (60, 40, 40, 40, 40)
SPECIAL = (40, 40)
DIGITS = (1, 2, 2)


def hctx(log_n=4, steps=(1, 3), digits=DIGITS, data=DATA, special=SPECIAL, relin=True):
    ctx = oracle.Context(log_n, data, special, digits=digits)
    ctx.keygen(4321, steps, relin=relin)
    return ctx


def digit_groups(ctx, level):
    """Active primes of every digit at level l (a digit is cut at the level)."""
    groups, start = [], 0
    for size in ctx.digits:
        prims = [i for i in range(start, start + size) if i <= level]
        if prims:
            groups.append(prims)
        start += size
    return groups


def ext_primes(ctx, level):
    return list(range(level + 1)) + list(range(ctx.n_data, ctx.n_data + ctx.n_special))


def digits_bigint(ctx, d_ntt, level):
    """d_j = CRT over the digit's primes of iNTT_q(d[q]), an integer in [0, Q_j) (R9b)."""
    out = []
    for prims in digit_groups(ctx, level):
        vals, _ = crt([ctx.intt(d_ntt[i], i) for i in prims], [ctx.primes[i] for i in prims])
        out.append(vals)
    return out


def ip_bigint(ctx, digits, key, level):
    ext = ext_primes(ctx, level)
    res = []
    for comp in range(2):
        per_prime = []
        for p in ext:
            q = ctx.primes[p]
            acc = [0] * ctx.n
            for j, d in enumerate(digits):
                kc = [int(v) for v in ctx.intt(key[j, comp, p], p)]
                prod = schoolbook_negacyclic([x % q for x in d], kc, q)
                acc = [(a + b) % q for a, b in zip(acc, prod)]
            per_prime.append(acc)
        U, QP = crt(per_prime, [ctx.primes[p] for p in ext])
        res.append(U)
    return res, QP


def coeffs_qp(ctx, x, level):
    ext = ext_primes(ctx, level)
    return crt([ctx.intt(x[e], p) for e, p in enumerate(ext)], [ctx.primes[p] for p in ext])


def sigma(vals, g, n, M):
    out = [0] * n
    for i, v in enumerate(vals):
        e = (i * g) % (2 * n)
        if e < n:
            out[e] = v % M
        else:
            out[e - n] = (-v) % M
    return out


def test_chain_and_digits():
    """K = 2 special primes after the data primes (R1 scan continues through the 40-bit primes); the
    hybrid cfg5 chain [60, 40x7 | 40, 40] has log2(QP) = 420 <= 438."""
    ctx = hctx()
    assert ctx.n_special == 2 and ctx.n_digits == 3 and ctx.digits == [1, 2, 2]
    assert ctx.primes[5] < ctx.primes[4] and ctx.primes[6] < ctx.primes[5]      # next 40-bit primes
    assert ctx.special_product == ctx.primes[5] * ctx.primes[6]
    full = oracle.Context(14, (60,) + (40,) * 7, (40, 40), digits=(1, 2, 2, 2, 1))
    bits = sum(np.log2(float(q)) for q in full.primes)
    assert 419 < bits <= 438
    with pytest.raises(oracle.OracleError):
        oracle.Context(4, DATA, SPECIAL, digits=(2, 2))                       # does not cover the chain


def test_keys_are_the_gadget_encryptions():
    """key_j.c0 + key_j.c1 s - [p in digit j] (P mod p) s' is the small error e_j on every prime (R17b)."""
    ctx = hctx(steps=(1,))
    n, L = ctx.n, ctx.n_data
    s = [int(v) for v in ctx.export_secret()]
    P = ctx.special_product
    g = ctx.galois_elt(1)
    s2 = [centered(x, 1 << 200) for x in schoolbook_negacyclic(s, s, 1 << 200)]
    sg = [0] * n
    for i, v in enumerate(s):
        e = (i * g) % (2 * n)
        if e < n:
            sg[e] += v
        else:
            sg[e - n] -= v
    groups = digit_groups(ctx, L - 1)
    for key_id, sp in ((0, s2), (g, sg)):
        key = ctx.export_key(key_id)
        assert key.shape == (3, 2, L + 2, n)
        for j, prims in enumerate(groups):
            errs = []
            for p in range(L + ctx.n_special):
                q = ctx.primes[p]
                k0 = [int(v) for v in ctx.intt(key[j, 0, p], p)]
                k1 = [int(v) for v in ctx.intt(key[j, 1, p], p)]
                lhs = [(a + b) % q for a, b in zip(k0, schoolbook_negacyclic(k1, [x % q for x in s], q))]
                gad = (P % q) if p in prims else 0
                errs.append([centered(a - gad * x, q) for a, x in zip(lhs, sp)])
            assert max(abs(e) for row in errs for e in row) <= 19                  # |e| <= 6 sigma (R13)
            assert all(row == errs[0] for row in errs)                            # one e_j over all primes


@pytest.mark.parametrize("level", [4, 3, 2, 0])
def test_hybrid_keyswitch_exact_bigint(level):
    """R-KS with digit groups: the RNS ModUp / inner product / ModDown by P_0 P_1 equals
    round(sum_j d_j key_j / P) mod Q_l exactly; level 3 cuts the digit {q3, q4} to {q3}."""
    ctx = hctx()
    rng = np.random.default_rng(70 + level)
    d = np.stack([rng.integers(0, ctx.primes[i], ctx.n, dtype=np.uint64) for i in range(level + 1)])
    P = ctx.special_product
    for key_id in (0, ctx.galois_elt(3)):
        out = ctx.keyswitch(d, key_id)
        U, QP = ip_bigint(ctx, digits_bigint(ctx, d, level), ctx.export_key(key_id), level)
        Ql = QP // P
        for comp in range(2):
            ref = [((x - centered(x, P)) // P) % Ql for x in U[comp]]
            got, _ = crt([ctx.intt(out[comp, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
            assert got == ref


def test_hybrid_keyswitch_decrypts_to_d_times_sprime():
    """u0 + u1 s = d s' + small for the relinearisation and a Galois key (noise of 80-bit digits over an
    80-bit P stays small)."""
    ctx = hctx(log_n=5, steps=(3,))
    n, L = ctx.n, ctx.n_data
    s = [int(v) for v in ctx.export_secret()]
    rng = np.random.default_rng(3)
    d = np.stack([rng.integers(0, ctx.primes[i], n, dtype=np.uint64) for i in range(L)])
    g = ctx.galois_elt(3)
    s2 = [centered(x, 1 << 200) for x in schoolbook_negacyclic(s, s, 1 << 200)]
    sg = [0] * n
    for i, c in enumerate(s):
        e = (i * g) % (2 * n)
        if e < n:
            sg[e] += c
        else:
            sg[e - n] -= c
    for key_id, sp in ((0, s2), (g, sg)):
        u = ctx.keyswitch(d, key_id)
        for i in range(L):
            q = ctx.primes[i]
            u0 = [int(v) for v in ctx.intt(u[0, i], i)]
            u1 = [int(v) for v in ctx.intt(u[1, i], i)]
            dd = [int(v) for v in ctx.intt(d[i], i)]
            lhs = [(a + b) % q for a, b in zip(u0, schoolbook_negacyclic(u1, [x % q for x in s], q))]
            rhs = schoolbook_negacyclic(dd, [x % q for x in sp], q)
            assert max(abs(centered(a - b, q)) for a, b in zip(lhs, rhs)) < 2 ** 14


@pytest.mark.parametrize("level", [4, 1])
def test_hybrid_moddown_and_lift(level):
    """ModDown by P = P_0 P_1: (X - [X]_P) / P mod Q_l; lift_qp(ct) is P ct (zero on both special limbs)."""
    ctx = hctx()
    rng = np.random.default_rng(80 + level)
    ext = ext_primes(ctx, level)
    x = np.stack([np.stack([rng.integers(0, ctx.primes[p], ctx.n, dtype=np.uint64) for p in ext]) for _ in range(2)])
    P = ctx.special_product
    out = ctx.moddown(x)
    for comp in range(2):
        X, QP = coeffs_qp(ctx, x[comp], level)
        ref = [((v - centered(v, P)) // P) % (QP // P) for v in X]
        got, _ = crt([ctx.intt(out[comp, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
        assert got == ref
    ct = x[:, : level + 1].copy()
    lifted = ctx.lift_qp(ct)
    assert np.all(lifted[:, level + 1:] == 0)
    C0, Ql = crt([ctx.intt(ct[0, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
    assert coeffs_qp(ctx, lifted[0], level)[0] == [(P * centered(v, Ql)) % (Ql * P) for v in C0]
    assert np.array_equal(ctx.moddown(lifted), ct)


@pytest.mark.parametrize("level", [4, 3])
def test_hybrid_qp_baby_and_giant_steps_exact(level):
    """Double hoisting (R11c) with digit groups: baby step (P sigma_g(c0) + U_0, U_1) with the signed
    sigma_g of the unsigned digit lifts; giant step with the digits of sigma_g(ModDown(w.c1))."""
    ctx = hctx(steps=(1, 3))
    rng = np.random.default_rng(90 + level)
    n = ctx.n
    P = ctx.special_product
    ct = np.stack([np.stack([rng.integers(0, ctx.primes[i], n, dtype=np.uint64) for i in range(level + 1)])
                   for _ in range(2)])
    for step in (1, 3):
        g = ctx.galois_elt(step)
        out = ctx.rotate_hoisted_qp(ct, step)
        digits = [sigma(d, g, n, 1 << 300) for d in digits_bigint(ctx, ct[1], level)]
        digits = [[centered(v, 1 << 300) for v in d] for d in digits]         # signed: -d, not Q_j - d
        U, QP = ip_bigint(ctx, digits, ctx.export_key(g), level)
        C0, Ql = crt([ctx.intt(ct[0, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
        c0s = sigma([centered(v, Ql) for v in C0], g, n, QP)
        assert coeffs_qp(ctx, out[0], level)[0] == [(u + P * v) % QP for u, v in zip(U[0], c0s)]
        assert coeffs_qp(ctx, out[1], level)[0] == U[1]
        # giant step on the baby step's output
        w = out
        gout = ctx.rotate_qp(w, step)
        W1, _ = coeffs_qp(ctx, w[1], level)
        c1p = [((v - centered(v, P)) // P) % Ql for v in W1]
        rc1 = sigma(c1p, g, n, Ql)
        gd = []
        for prims in digit_groups(ctx, level):
            Qj = 1
            for i in prims:
                Qj *= ctx.primes[i]
            gd.append([v % Qj for v in rc1])
        U2, _ = ip_bigint(ctx, gd, ctx.export_key(g), level)
        W0, _ = coeffs_qp(ctx, w[0], level)
        assert coeffs_qp(ctx, gout[0], level)[0] == [(u + v) % QP for u, v in zip(U2[0], sigma(W0, g, n, QP))]
        assert coeffs_qp(ctx, gout[1], level)[0] == U2[1]


@pytest.mark.parametrize("hoisted", [0, 1, 2])
def test_hybrid_matvec_vs_float64(hoisted):
    ctx = hctx(log_n=10, steps=C.rotation_steps_for([(16, 64)]))
    rng = np.random.default_rng(13)
    W = rng.normal(0, 0.1, (16, 64))
    b = rng.uniform(-0.1, 0.1, 16)
    x = rng.uniform(-1, 1, 64)
    lay = C.encode_layer(ctx, W, b, ctx.top_level, 2.0 ** 40)
    ct = C.Ct(ctx.encrypt(E.encode(C.pack_input(x, lay.t, ctx.n // 2), 2.0 ** 40, ctx.n), 77, 0), 2.0 ** 40)
    y = C.matvec(ctx, ct, lay, hoisted=hoisted)
    d = E.decode(ctx.decrypt(y.data), ctx.primes, y.scale, ctx.n)
    assert np.max(np.abs(d[:16] - (W @ x + b))) < 1e-6
    assert np.max(np.abs(d[16:])) < 1e-6


def test_hybrid_two_layer_forward_vs_float64():
    """cfg4-shaped network on a small ring with the hybrid chain: dense -> square -> replicate -> dense,
    double hoisting, decrypted within 1e-3 of float64."""
    rng = np.random.default_rng(21)
    shapes = [(32, 64), (16, 32)]
    ctx = hctx(log_n=10, steps=C.rotation_steps_for(shapes, 1))
    Ws = [rng.normal(0, 1 / np.sqrt(c), (r, c)) for r, c in shapes]
    bs = [rng.uniform(-0.1, 0.1, r) for r, _ in shapes]
    x = rng.uniform(-1, 1, 64)
    D = 2.0 ** 40
    layers = C.encode_model(ctx, Ws, bs, ctx.top_level, D, "square", 1)
    ct = C.Ct(ctx.encrypt(E.encode(C.pack_input(x, layers[0].t, ctx.n // 2), D, ctx.n), 5, 0), D)
    y = C.forward(ctx, ct, layers, "square", hoisted=2)
    d = E.decode(ctx.decrypt(y.data), ctx.primes, y.scale, ctx.n)
    ref = C.plain_forward(x, Ws, bs, "square")
    assert np.max(np.abs(d[:16] - ref)) < 1e-3
