"""Pins of the oracle's ring layer against definitions that do not come from the oracle.

Each test names what fixes the expected value: the worked examples in tests/golden (SPEC/hand),
the O(N^2) evaluation definition of the negacyclic NTT (R2), schoolbook negacyclic convolution,
sympy's primality test and n-th-root solver, or an algebraic invariant.
"""
import numpy as np
import pytest
import sympy
from sympy.ntheory.residue_ntheory import nthroot_mod

import oracle
import synthetic as S

pytestmark = pytest.mark.filterwarnings("ignore")


def schoolbook_negacyclic(a, b, q):
    n = len(a)
    out = [0] * n
    for i in range(n):
        for j in range(n):
            k = i + j
            v = int(a[i]) * int(b[j])
            if k < n:
                out[k] += v
            else:
                out[k - n] -= v
    return [x % q for x in out]


def brev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def ntt_by_definition(a, q, psi):
    """NTT(a)[k] = a(psi^{2 brev(k) + 1}) mod q  (Horner; R2)."""
    n = len(a)
    bits = n.bit_length() - 1
    out = []
    for k in range(n):
        x = pow(psi, 2 * brev(k, bits) + 1, q)
        acc = 0
        for c in reversed([int(v) for v in a]):
            acc = (acc * x + c) % q
        out.append(acc)
    return out


@pytest.mark.parametrize("cfg", [S.CFG1, S.CFG2, S.CFG4])
def test_prime_chain_is_the_downward_scan(cfg):
    """R1/S:L95: each prime is the largest unused prime < 2^b with q = 1 mod 2N (sympy.isprime)."""
    ctx = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    two_n = 2 * ctx.n
    used = []
    for b, q in zip(cfg.bits, ctx.primes):
        assert sympy.isprime(q) and q % two_n == 1 and q < 2 ** b
        # nothing skipped: every candidate strictly between q and 2^b is composite or already used
        c = 2 ** b - two_n + 1
        while c > q:
            assert (not sympy.isprime(c)) or c in used
            c -= two_n
        used.append(q)
    assert len(set(ctx.primes)) == len(ctx.primes)


@pytest.mark.parametrize("cfg", [S.CFG1, S.CFG4])
def test_psi_is_min_primitive_root(cfg):
    """R2: psi = min of all x with x^N = -1 mod q (sympy nthroot_mod enumerates them)."""
    ctx = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    for q, psi in zip(ctx.primes, ctx.psi):
        roots = nthroot_mod(q - 1, ctx.n, q, all_roots=True)
        assert len(roots) == ctx.n
        assert psi == min(roots)
        assert pow(psi, ctx.n, q) == q - 1


def test_ntt_worked_example_n8_q17(golden):
    g = golden["ntt_n8_q17"]
    ctx = oracle.Context(3, (), (), primes=[g["q"]])
    q = g["q"]
    for a_key, sq_key in (("a", "square_schoolbook"), ("b", "b_square")):
        a = np.array(g[a_key], dtype=np.uint64)
        A = ctx.ntt(a, 0)
        sq = ctx.intt((A * A) % np.uint64(q), 0)
        assert [int(v) for v in sq] == g[sq_key]
        assert [int(v) for v in A] == ntt_by_definition(g[a_key], q, ctx.psi[0])
    assert schoolbook_negacyclic(g["b"], g["b"], q) == g["b_square"]


@pytest.mark.parametrize("primes_of", [S.CFG1, S.CFG2, S.CFG4])
@pytest.mark.parametrize("log_n", [4, 6])
def test_ntt_matches_definition_real_primes(primes_of, log_n):
    """Real 40/50/60-bit chain primes at small N: O(N^2) definition, schoolbook product, inverse."""
    big = oracle.Context(primes_of.log_n, primes_of.data_bits, primes_of.special_bits)
    ctx = oracle.Context(log_n, (), (), primes=big.primes)
    n = ctx.n
    rng = np.random.default_rng(log_n)
    for pi, q in enumerate(ctx.primes):
        a = rng.integers(0, q, size=n, dtype=np.uint64)
        b = rng.integers(0, q, size=n, dtype=np.uint64)
        A, B = ctx.ntt(a, pi), ctx.ntt(b, pi)
        assert [int(v) for v in A] == ntt_by_definition(a, q, ctx.psi[pi])
        prod = np.array([(int(x) * int(y)) % q for x, y in zip(A, B)], dtype=np.uint64)
        assert [int(v) for v in ctx.intt(prod, pi)] == schoolbook_negacyclic(a, b, q)
        assert np.array_equal(ctx.intt(A, pi), a)


@pytest.mark.parametrize("cfg", [S.CFG1, S.CFG4])
def test_ntt_full_size_invariants(cfg):
    """Full N: NTT(1) = all ones, iNTT(NTT(a)) = a, sampled outputs equal the definition."""
    ctx = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    n = ctx.n
    rng = np.random.default_rng(7)
    one = np.zeros(n, dtype=np.uint64)
    one[0] = 1
    for pi in (0, len(ctx.primes) - 1):
        q, psi = ctx.primes[pi], ctx.psi[pi]
        assert np.all(ctx.ntt(one, pi) == 1)
        a = rng.integers(0, q, size=n, dtype=np.uint64)
        A = ctx.ntt(a, pi)
        assert np.array_equal(ctx.intt(A, pi), a)
        bits = ctx.log_n
        coeffs = [int(v) for v in a]
        for k in (0, 1, n // 2 + 3, n - 1):
            x = pow(psi, 2 * brev(k, bits) + 1, q)
            acc = 0
            for c in reversed(coeffs):
                acc = (acc * x + c) % q
            assert int(A[k]) == acc


def test_automorphism_worked_example(golden):
    g = golden["automorphism_n8"]
    ctx = oracle.Context(3, (), (), primes=[g["q"]])
    for src, dst in (("x", "sigma_x"), ("x3", "sigma_x3")):
        out = ctx.automorphism_coef(np.array(g[src], dtype=np.uint64), 0, g["g"])
        assert [int(v) for v in out] == g[dst]


def test_automorphism_invariants():
    """g=1 identity; sigma_g then sigma_{g^-1} identity; ring homomorphism (schoolbook)."""
    big = oracle.Context(S.CFG1.log_n, S.CFG1.data_bits, S.CFG1.special_bits)
    ctx = oracle.Context(5, (), (), primes=big.primes)
    n, q = ctx.n, ctx.primes[1]
    rng = np.random.default_rng(3)
    a = rng.integers(0, q, size=n, dtype=np.uint64)
    b = rng.integers(0, q, size=n, dtype=np.uint64)
    assert np.array_equal(ctx.automorphism_coef(a, 1, 1), a)
    for g in (3, 5, 13, 2 * n - 1, 25):
        gi = pow(g, -1, 2 * n)
        assert np.array_equal(ctx.automorphism_coef(ctx.automorphism_coef(a, 1, g), 1, gi), a)
        lhs = ctx.automorphism_coef(np.array(schoolbook_negacyclic(a, b, q), dtype=np.uint64), 1, g)
        rhs = schoolbook_negacyclic(ctx.automorphism_coef(a, 1, g), ctx.automorphism_coef(b, 1, g), q)
        assert [int(v) for v in lhs] == rhs
        # the NTT-domain automorphism is the coefficient one conjugated by the NTT
        A = ctx.ntt(a, 1)
        assert np.array_equal(ctx.intt(ctx.automorphism_ntt(A, 1, g), 1), ctx.automorphism_coef(a, 1, g))


def test_galois_elements():
    ctx = oracle.Context(4, (), (), primes=[97])
    n = ctx.n
    assert ctx.galois_elt(0) == 1
    assert ctx.galois_elt(1) == 5
    assert ctx.galois_elt(-1) == pow(5, n // 2 - 1, 2 * n)
    assert (ctx.galois_elt(3) * ctx.galois_elt(-3)) % (2 * n) == 1


def test_samplers():
    """determinism, ternary support, Gaussian std within 5% over 1e5 draws; uniform range."""
    ctx = oracle.Context(4, (), (), primes=[97])
    st = oracle.stream(5, 17, 2, 3)
    g1 = ctx.sample_gaussian(11, st, 100000)
    g2 = ctx.sample_gaussian(11, st, 100000)
    assert np.array_equal(g1, g2)
    assert abs(g1.std() - 3.2) / 3.2 < 0.05 and abs(g1.mean()) < 0.05
    assert g1.max() <= 19 and g1.min() >= -19
    t = oracle.sample_ternary(11, st, 100000)
    assert set(np.unique(t).tolist()) == {-1, 0, 1}
    assert all(abs((t == v).mean() - 1 / 3) < 0.01 for v in (-1, 0, 1))
    q = 1099511480321
    u = oracle.sample_uniform(11, st, q, 100000)
    assert u.max() < q and abs(u.astype(np.float64).mean() / q - 0.5) < 0.01
    assert not np.array_equal(u, oracle.sample_uniform(12, st, q, 100000))
    cdt, B = ctx.cdt()
    assert B == 19 and all(cdt[i] < cdt[i + 1] for i in range(len(cdt) - 1))
