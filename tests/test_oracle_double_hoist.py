"""Pins of the oracle's double-hoisting operations (NEXT f-1, R11c): the Q_l P basis baby
step, the QP giant step, ModDown, and the lift / plaintext identities, each against its big-integer
definition (Python ints, schoolbook negacyclic products, CRT), plus the decrypted matvec.
"""
import numpy as np
import pytest

import oracle
from oracle import circuits as C
from oracle import encoding as E
import synthetic as S

from test_oracle_ring import schoolbook_negacyclic
from test_oracle_scheme import small_ctx, crt, centered, enc_vec, dec_vec, _dense_case


def _ext(ctx, level):
    return list(range(level + 1)) + [ctx.n_data]


def _coeffs_qp(ctx, x, level):
    """CRT of the coefficient residues of one QP component [l+2][N] -> ints in [0, Q_l P)."""
    ext = _ext(ctx, level)
    return crt([ctx.intt(x[e], p) for e, p in enumerate(ext)], [ctx.primes[p] for p in ext])


def _sigma(vals, g, n, M):
    """sigma_g on integer coefficients mod M: coefficient i -> i g mod 2N, negated past N."""
    out = [0] * n
    for i, v in enumerate(vals):
        e = (i * g) % (2 * n)
        if e < n:
            out[e] = v % M
        else:
            out[e - n] = (-v) % M
    return out


def _rand_qp(ctx, level, rng, ncomp=2):
    ext = _ext(ctx, level)
    return np.stack([np.stack([rng.integers(0, ctx.primes[p], ctx.n, dtype=np.uint64) for p in ext])
                     for _ in range(ncomp)])


def _ip_bigint(ctx, digits, key, level):
    """U_c = sum_j digit_j * key_{j,c} over every prime of Q_l P (schoolbook), CRT-combined."""
    ext = _ext(ctx, level)
    out = []
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
        out.append(U)
    return out, QP


@pytest.mark.parametrize("level", [2, 1])
def test_moddown_exact_bigint(level):
    """ModDown(X) = (X - [X]_P) / P mod Q_l with [.]_P the centred residue (R10 rounding)."""
    ctx = small_ctx()
    rng = np.random.default_rng(40 + level)
    x = _rand_qp(ctx, level, rng)
    out = ctx.moddown(x)
    P = ctx.primes[ctx.n_data]
    for comp in range(2):
        X, QP = _coeffs_qp(ctx, x[comp], level)
        Ql = QP // P
        ref = [((v - centered(v, P)) // P) % Ql for v in X]
        got, _ = crt([ctx.intt(out[comp, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
        assert got == ref


def test_lift_and_plaintext_identities():
    """ModDown(P ct) = ct and ModDown(P ct o pt) = ct o pt exactly (the P residue of P x is 0)."""
    ctx = small_ctx()
    rng = np.random.default_rng(3)
    level = 2
    ct = np.stack([np.stack([rng.integers(0, ctx.primes[i], ctx.n, dtype=np.uint64) for i in range(level + 1)])
                   for _ in range(2)])
    lifted = ctx.lift_qp(ct)
    assert np.all(lifted[:, level + 1] == 0)
    assert np.array_equal(ctx.moddown(lifted), ct)
    m = rng.integers(-2 ** 40, 2 ** 40, ctx.n)
    prod = ctx.mul_plain_qp(lifted, ctx.plain_qp(m, level))
    assert np.array_equal(ctx.moddown(prod), ctx.mul_plain(ct, ctx.plain(m, level)))
    s = ctx.add_qp(lifted, lifted)
    assert np.array_equal(ctx.moddown(s), ctx.add(ct, ct))
    assert np.array_equal(ctx.plain_qp(m, level)[: level + 1], ctx.plain(m, level))


@pytest.mark.parametrize("level", [2, 1])
def test_rotate_hoisted_qp_exact_bigint(level):
    """Baby step: out = (P sigma_g(c0) + U_0, U_1) over Q_l P, U_c = sum_j sigma_g(d_j) key_j.c with
    the SIGNED automorphism of the unsigned digits d_j = iNTT(c1[j]) (R11b) -- no division by P."""
    ctx = small_ctx(steps=(1, 3))
    rng = np.random.default_rng(50 + level)
    n, L = ctx.n, ctx.n_data
    P = ctx.primes[L]
    ct = np.stack([np.stack([rng.integers(0, ctx.primes[i], n, dtype=np.uint64) for i in range(level + 1)])
                   for _ in range(2)])
    for step in (1, 3):
        g = ctx.galois_elt(step)
        out = ctx.rotate_hoisted_qp(ct, step)
        digits = []
        for j in range(level + 1):
            d = [int(v) for v in ctx.intt(ct[1, j], j)]
            sd = [0] * n
            for i, v in enumerate(d):
                e = (i * g) % (2 * n)
                if e < n:
                    sd[e] = v
                else:
                    sd[e - n] = -v
            digits.append(sd)
        U, QP = _ip_bigint(ctx, digits, ctx.export_key(g), level)
        C0, Ql = crt([ctx.intt(ct[0, i], i) for i in range(level + 1)], ctx.primes[: level + 1])
        c0s = _sigma([centered(v, Ql) for v in C0], g, n, QP)
        ref0 = [(u + P * v) % QP for u, v in zip(U[0], c0s)]
        assert _coeffs_qp(ctx, out[0], level)[0] == ref0
        assert _coeffs_qp(ctx, out[1], level)[0] == U[1]
    assert np.array_equal(ctx.rotate_hoisted_qp(ct, 0), ctx.lift_qp(ct))


@pytest.mark.parametrize("level", [2, 1])
def test_rotate_qp_exact_bigint(level):
    """Giant step: c1' = (W1 - [W1]_P) / P mod Q_l, digits d_j = sigma_g(c1') mod q_j in [0, q_j),
    out = (sigma_g(w.c0) + U_0, U_1) over Q_l P with U_c = sum_j d_j key_j.c."""
    ctx = small_ctx(steps=(2, 5))
    rng = np.random.default_rng(60 + level)
    n, L = ctx.n, ctx.n_data
    P = ctx.primes[L]
    w = _rand_qp(ctx, level, rng)
    for step in (2, 5):
        g = ctx.galois_elt(step)
        out = ctx.rotate_qp(w, step)
        W1, QP = _coeffs_qp(ctx, w[1], level)
        Ql = QP // P
        c1p = [((v - centered(v, P)) // P) % Ql for v in W1]
        rc1 = _sigma(c1p, g, n, Ql)
        digits = [[v % ctx.primes[j] for v in rc1] for j in range(level + 1)]
        U, _ = _ip_bigint(ctx, digits, ctx.export_key(g), level)
        W0, _ = _coeffs_qp(ctx, w[0], level)
        ref0 = [(u + v) % QP for u, v in zip(U[0], _sigma(W0, g, n, QP))]
        assert _coeffs_qp(ctx, out[0], level)[0] == ref0
        assert _coeffs_qp(ctx, out[1], level)[0] == U[1]
    assert np.array_equal(ctx.rotate_qp(w, 0), w)


def test_double_hoisted_rotation_decrypts():
    """moddown(baby step) = R11b hoisted rotation exactly; moddown(giant step of P ct) decrypts to the
    rotated slots."""
    ctx = small_ctx(log_n=10, steps=(1, 5, -3))
    v = np.random.default_rng(5).uniform(-1, 1, ctx.n // 2)
    ct = enc_vec(ctx, v, 2.0 ** 40)
    for step in (1, 5, -3):
        b = ctx.moddown(ctx.rotate_hoisted_qp(ct.data, step))
        gs = ctx.moddown(ctx.rotate_qp(ctx.lift_qp(ct.data), step))
        for r in (b, gs):
            assert np.max(np.abs(dec_vec(ctx, C.Ct(r, ct.scale)) - np.roll(v, -step))) < 1e-6
        # P sigma_g(c0) has residue 0 mod P, so ModDown(baby step) is exactly the R11b hoisted rotation
        assert np.array_equal(b, ctx.rotate_hoisted(ct.data, step))


def test_double_hoisted_matvec_vs_float64():
    ctx = small_ctx(log_n=10, steps=C.rotation_steps_for([(16, 64)]))
    rng = np.random.default_rng(8)
    W = rng.normal(0, 0.1, (16, 64))
    b = rng.uniform(-0.1, 0.1, 16)
    x = rng.uniform(-1, 1, 64)
    lay = C.encode_layer(ctx, W, b, ctx.top_level, 2.0 ** 40)
    ct = enc_vec(ctx, C.pack_input(x, lay.t, ctx.n // 2), 2.0 ** 40)
    ops = C.OpCount()
    y2 = C.matvec(ctx, ct, lay, ops, hoisted=2)
    y1 = C.matvec(ctx, ct, lay, hoisted=1)
    assert ops.rot == 14 and ops.mul_plain == 64
    assert not np.array_equal(y1.data, y2.data)
    d = dec_vec(ctx, y2)
    assert np.max(np.abs(d[:16] - (W @ x + b))) < 1e-6
    assert np.max(np.abs(d[16:])) < 1e-6


def test_bsgs_split_extra_baby_steps():
    """R5b: x extra doublings of t1 (capped at 2^ceil(log2 t)); t1 t2 = t padded to t1 | t."""
    assert C.bsgs_split(256, 512) == (512, 32, 16)
    assert C.bsgs_split(256, 512, 1) == (512, 64, 8)
    assert C.bsgs_split(128, 256, 1) == (256, 32, 8)
    assert C.bsgs_split(766, 766, 1) == (768, 64, 12)
    assert C.bsgs_split(16, 64, 4) == (64, 64, 1)
    assert C.bsgs_split(1, 1, 1) == (1, 1, 1)
    steps = C.rotation_steps_for([(256, 512), (128, 256)], 1)
    assert steps == sorted(set(range(1, 64)) | {64 * k for k in range(1, 8)} | set(range(1, 32))
                           | {32 * k for k in range(1, 8)} | {-256})


@pytest.mark.parametrize("hoisted", [0, 2])
def test_matvec_more_baby_steps_vs_float64(hoisted):
    """Any BSGS split computes the same Eq. 1 product: x = 1 decrypts to W x + b; op counts t1-1 + t2-1."""
    ctx = small_ctx(log_n=10, steps=C.rotation_steps_for([(16, 64)], 1))
    rng = np.random.default_rng(12)
    W = rng.normal(0, 0.1, (16, 64))
    b = rng.uniform(-0.1, 0.1, 16)
    x = rng.uniform(-1, 1, 64)
    lay = C.encode_layer(ctx, W, b, ctx.top_level, 2.0 ** 40, x=1)
    assert (lay.t1, lay.t2) == (16, 4)
    ct = enc_vec(ctx, C.pack_input(x, lay.t, ctx.n // 2), 2.0 ** 40)
    ops = C.OpCount()
    y = C.matvec(ctx, ct, lay, ops, hoisted=hoisted)
    assert ops.rot == 15 + 3 and ops.mul_plain == 64
    d = dec_vec(ctx, y)
    assert np.max(np.abs(d[:16] - (W @ x + b))) < 1e-6
