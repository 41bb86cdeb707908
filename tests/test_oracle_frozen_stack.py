"""Pins of the oracle's NEXT f-2 circuits (conv1d, avgpool, multi-item packing, the depth-6 frozen
stack) against float64 definitions, the SPEC's worked cases and the paper's Table 2 p column."""
import numpy as np
import pytest

import oracle
from oracle import circuits as C
from oracle import encoding as E
import synthetic as S


def ctx_with(log_n, data_bits, steps):
    c = oracle.Context(log_n, data_bits, (60,))
    c.keygen(4321, steps)
    return c


def enc(ctx, v, scale=2.0 ** 40, idx=0):
    return C.Ct(ctx.encrypt(E.encode(v, scale, ctx.n), 99, idx), scale)


def dec(ctx, ct):
    return E.decode(ctx.decrypt(ct.data), ctx.primes, ct.scale, ctx.n)


def test_packing_matches_paper_p(golden):
    """P:L116 p = floor(#slots / (2 #neurons)) and Table 2's p column, t = 768."""
    g = golden["paper_presets"]
    for key in ("p1", "p2"):
        n_slots = g[key]["N"] // 2
        p, R = C.packing(n_slots, g["neurons"], conv_half=4)
        assert p == g[key]["p"] == n_slots // (2 * g["neurons"])
        assert R >= 2 * g["neurons"] + 4 and p * R <= n_slots


def test_conv_identity_constant_random():
    t, f = 64, 9
    n = 2048
    p, R = C.packing(n // 2, t, 4)
    ctx = ctx_with(11, (60, 40, 40), list(range(-4, 5)))
    rng = np.random.default_rng(1)
    xs = [rng.uniform(-1, 1, t) for _ in range(p)]
    ct = enc(ctx, C.pack_items(xs, t, R, n // 2))
    # identity filter (delta at the centre) -> output = input (SPEC he-layers enc_conv1d example)
    ident = np.zeros(f)
    ident[4] = 1.0
    lay = C.encode_conv(ctx, ident, 0.0, t, ctx.top_level, ct.scale, R, p)
    ops = C.OpCount()
    y = dec(ctx, C.apply_layer(ctx, ct, lay, ops=ops))
    assert ops.mul_plain == f and ops.rot == f - 1                  # P:L98 counts
    for r in range(p):
        assert np.max(np.abs(y[r * R: r * R + t] - xs[r])) < 1e-6
        assert np.max(np.abs(y[r * R + t:(r + 1) * R])) < 1e-6
    # constant input c, filter of ones: interior slot -> 9c
    c = 0.3
    ctc = enc(ctx, C.pack_items([np.full(t, c)] * p, t, R, n // 2), idx=1)
    y = dec(ctx, C.apply_layer(ctx, ctc, C.encode_conv(ctx, np.ones(f), 0.0, t, ctx.top_level, ctc.scale, R, p)))
    assert abs(y[R + 10] - 9 * c) < 1e-6 and abs(y[0] - 5 * c) < 1e-6
    # random filter vs the float64 'same' convolution
    w, b = rng.normal(0, 0.3, f), 0.05
    y = dec(ctx, C.apply_layer(ctx, ct, C.encode_conv(ctx, w, b, t, ctx.top_level, ct.scale, R, p)))
    for r in range(p):
        assert np.max(np.abs(y[r * R: r * R + t] - C.conv_same(xs[r], w, b))) < 1e-6


def test_avgpool():
    t, f = 32, 3
    n = 1024
    p, R = C.packing(n // 2, t, 0)
    ctx = ctx_with(10, (60, 40, 40), [-1, -2])
    x = np.zeros(t)
    x[:3] = [3, 6, 9]                                     # SPEC avgpool example: mean 6
    rng = np.random.default_rng(2)
    xs = [x] + [rng.uniform(-1, 1, t) for _ in range(p - 1)]
    ct = enc(ctx, C.pack_items(xs, t, R, n // 2))
    ops = C.OpCount()
    y = dec(ctx, C.apply_layer(ctx, ct, C.encode_pool(ctx, f, t, ctx.top_level, R, p), ops=ops))
    assert ops.mul_plain == f and ops.rot == f - 1        # P:L100 (f-1 rotations; one mask per term)
    assert abs(y[2] - 6.0) < 1e-6
    for r in range(p):
        ref = C.pool_valid_right(xs[r], f)
        assert np.max(np.abs(y[r * R + f - 1: r * R + t] - ref)) < 1e-6
        assert np.max(np.abs(y[r * R: r * R + f - 1])) < 1e-6          # masked
        assert np.max(np.abs(y[r * R + t:(r + 1) * R])) < 1e-6


def _stack_weights(t, rng):
    tp = t - 2
    return {"conv_w": rng.normal(0, 0.3, 9), "conv_b": 0.01, "W1": rng.normal(0, 1 / np.sqrt(t), (t, t)),
            "b1": rng.uniform(-0.1, 0.1, t), "W2": rng.normal(0, 1 / np.sqrt(tp), (tp, tp)),
            "b2": rng.uniform(-0.1, 0.1, tp), "f_pool": 3}


def test_frozen_stack_small_ring_vs_float64():
    """Depth-6 stack on N=4096, t=64: p=15 items, level drops by exactly 6."""
    t = 64
    n = 4096
    p, R = C.packing(n // 2, t, 4)
    assert p == 15
    rng = np.random.default_rng(3)
    wts = _stack_weights(t, rng)
    steps = C.frozen_stack_steps(t, [(t, t), (t - 2, t)], 9, 3)
    ctx = ctx_with(12, (60,) + (40,) * 6, steps)
    Delta = 2.0 ** 40
    stages = C.encode_frozen_stack(ctx, wts, ctx.top_level, Delta, R, p)
    xs = [rng.uniform(-1, 1, t) for _ in range(p)]
    ct = enc(ctx, C.pack_items(xs, t, R, n // 2))
    ops = C.OpCount()
    out = C.forward_stages(ctx, ct, stages, R, p, hoisted=True, ops=ops)
    assert out.level == ctx.top_level - 6
    y = dec(ctx, out)
    for r in range(p):
        ref = C.plain_frozen_forward(xs[r], wts)
        assert np.max(np.abs(y[r * R: r * R + ref.size] - ref)) < 1e-3
    # rotations: conv 8 + dense 2 x (t1 + t2 - 2) + pool 2 + 2 replicates
    t1 = 8
    assert ops.rot == 8 + 2 * (t1 + t // t1 - 2) + 2 + 2


def test_multi_item_isolation():
    """Item 0's output does not depend on the other items (SPEC region isolation)."""
    t = 32
    n = 2048
    p, R = C.packing(n // 2, t, 4)
    rng = np.random.default_rng(4)
    ctx = ctx_with(11, (60, 40, 40), list(range(-4, 5)))
    w = rng.normal(0, 0.3, 9)
    x0 = rng.uniform(-1, 1, t)
    a = enc(ctx, C.pack_items([x0] + [rng.uniform(-1, 1, t) for _ in range(p - 1)], t, R, n // 2))
    b = enc(ctx, C.pack_items([x0], t, R, n // 2), idx=1)
    lay = C.encode_conv(ctx, w, 0.0, t, ctx.top_level, a.scale, R, p)
    ya, yb = dec(ctx, C.apply_layer(ctx, a, lay)), dec(ctx, C.apply_layer(ctx, b, lay))
    assert np.max(np.abs(ya[:R] - yb[:R])) < 1e-6
