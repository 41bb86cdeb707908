"""Worst-case magnitude bounds of the FP64-pipe NTT for 45-50-bit primes (PC_FPR; csrc/ntt.cuh, csrc/ntt_c.cuh),
recomputed here in exact rational arithmetic for every pass structure the kernels use.

Model (units of q, q < 2^50): twiddles are centred, |w| <= q/2, and fl(w/q) has relative error <= 2^-53, so for a
multiplicand |y| = c q the quotient estimate is off by at most c q / 2 * 2^-53 <= c / 16 and
|fmodmul(y, w)| <= (1/2 + c/16) q.  The kernels are exact as long as every multiplicand is below 2^52 (= 4 q at the
top of the class: |y w/q| < 2^51 for the rint trick) and every sum below 2^53; the final representative must be
inside (-q, q) for the single conditional +q.
  forward (Cooley-Tukey):  t = fmodmul(Y), X' = X + t, Y' = X - t; X is reduced to 1/2 in the first stage of a pass
  inverse (Gentleman-Sande): X' = u + v, Y' = fmodmul(u - v); sums reduced at every other stage counted from the
  first one executed (stage LOGN - 1); loaded inputs reduced; N^{-1} (centred) applied last
"""
from fractions import Fraction as F

import pytest

HALF = F(1, 2)
LIMIT = F(4)          # multiplicand bound 2^52 in units of q = 2^50


def t_bound(c):
    return HALF + c / 16


def forward_passes_whole_limb(logn):
    out, s = [], 0
    while s < logn:
        out.append(min(4, logn - s))
        s += out[-1]
    return out


def forward_passes_cluster(logn):
    sb = 1 if logn >= 14 else 0
    return sb, [logn - sb - 8, 4, 4]


def run_forward(passes, v_in, lead_stage=False):
    """returns the largest multiplicand seen; v = bound on every value entering a stage"""
    worst = F(0)
    v = v_in
    if lead_stage:                                   # stage 0 across the CTA pair: X reduced, Y = loaded value
        worst = max(worst, v)
        v = HALF + t_bound(v)
    for k in passes:
        for r in range(k):
            worst = max(worst, v)                    # Y input of this stage
            x = HALF if r == 0 else v
            v = x + t_bound(v)
            assert v < 8                             # sums exact: < 2^53
    return worst, v


@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14])
def test_forward_whole_limb(logn):
    worst, v = run_forward(forward_passes_whole_limb(logn), F(2))        # lazy loads in [0, 2q)
    assert worst < LIMIT and v < LIMIT                                   # fcanon input below 2^52 as well


@pytest.mark.parametrize("logn", [12, 13, 14])
def test_forward_cluster(logn):
    sb, passes = forward_passes_cluster(logn)
    worst, v = run_forward(passes, F(2), lead_stage=bool(sb))
    assert worst < LIMIT and v < LIMIT
    assert passes[0] in (4, 5)


@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14])
def test_inverse(logn):
    v = HALF                                          # loaded inputs are reduced
    for s in range(logn - 1, -1, -1):
        diff = 2 * v                                  # |u - v|: the multiplicand
        assert diff < LIMIT, (logn, s)
        y = t_bound(diff)
        x = HALF if ((logn - 1 - s) & 1) else 2 * v
        v = max(x, y)
        assert 2 * v < 8
    # N^{-1}: one more fmodmul of the X lineage, then a single conditional + q
    assert v < LIMIT and t_bound(v) < 1


def test_inverse_cluster_stage0():
    """N = 16384 on CTA pairs: stage 0 is done after the exchange on unreduced inputs (values of stage 1), and both
    X + Y and (X - Y) w go through the N^{-1} product before the conditional + q."""
    logn, v = 14, HALF
    for s in range(logn - 1, 0, -1):
        y = t_bound(2 * v)
        x = HALF if ((logn - 1 - s) & 1) else 2 * v
        v = max(x, y)
    s_sum, d = 2 * v, t_bound(2 * v)
    assert 2 * v < LIMIT and s_sum < LIMIT
    assert t_bound(s_sum) < 1 and t_bound(d) < 1
