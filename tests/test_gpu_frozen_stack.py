"""GPU parity for NEXT row f-2 (the paper's frozen stack): conv1d, avgpool, multi-item dense, and the
depth-6 stack conv -> dense+cubic -> pool -> dense, bit-exact vs the oracle on shared encodings, and
decrypted within 1e-3 of the float64 stack."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle  # noqa: E402
from oracle import circuits as OC  # noqa: E402
from oracle import encoding as OE  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402

KIND = {"dense": G.LAYER_DENSE, "conv": G.LAYER_CONV1D, "pool": G.LAYER_AVGPOOL}


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


def pair(log_n, data_bits, steps, max_batch=2, seed=2024):
    o = oracle.Context(log_n, data_bits, (60,))
    o.keygen(seed, steps)
    g = G.Context(log_n, data_bits, (60,), key_seed=seed, rot_steps=steps, max_batch=max_batch)
    assert g.primes == o.primes
    return o, g


def imported(g, lay, region, items):
    return G.GeneralLayer.imported(g, KIND[lay.kind], lay.rows, lay.cols, lay.t, lay.t2, lay.baby_steps, lay.giant,
                                   region, items, lay.level, lay.pt_scale, lay.bias_scale, lay.pt_coeffs,
                                   lay.bias_coeffs)


def weights(t, rng):
    tp = t - 2
    return {"conv_w": rng.normal(0, 0.3, 9), "conv_b": 0.01, "W1": rng.normal(0, 1 / np.sqrt(t), (t, t)),
            "b1": rng.uniform(-0.1, 0.1, t), "W2": rng.normal(0, 1 / np.sqrt(tp), (tp, tp)),
            "b2": rng.uniform(-0.1, 0.1, tp), "f_pool": 3}


@pytest.mark.parametrize("hoisted", [0, 1, 2])
def test_conv_and_pool_layers(hoisted):
    t, n = 64, 2048
    p, R = OC.packing(n // 2, t, 4)
    o, g = pair(11, (60, 40, 40), sorted(set(range(-4, 5)) - {0}), max_batch=2)
    rng = np.random.default_rng(5)
    B = 3
    ms = np.stack([OE.encode(OC.pack_items([rng.uniform(-1, 1, t) for _ in range(p)], t, R, n // 2), 2.0 ** 40, n)
                   for _ in range(B)])
    ct = g.encrypt(ms, 7, 0, 2.0 ** 40)
    for lay in (OC.encode_conv(o, rng.normal(0, 0.3, 9), 0.02, t, o.top_level, 2.0 ** 40, R, p),
                OC.encode_pool(o, 3, t, o.top_level, R, p)):
        gl = imported(g, lay, R, p)
        model = G.Model.from_stages(g, [(gl, G.ACT_NONE, 0)])
        model.set_hoisting(hoisted)
        out = model.forward(ct)
        for b in range(B):
            ref = OC.apply_layer(o, OC.Ct(o.encrypt(ms[b], 7, b), 2.0 ** 40), lay, hoisted=hoisted)
            assert np.array_equal(u64(out.data)[b], ref.data), (lay.kind, b)


@pytest.mark.parametrize("mode", [1, 2])
def test_frozen_stack_small_ring_parity(mode):
    """Depth-6 stack on N=4096, t=64, 15 items per ciphertext, ragged batch over max_batch."""
    t, n = 64, 4096
    p, R = OC.packing(n // 2, t, 4)
    rng = np.random.default_rng(6)
    wts = weights(t, rng)
    steps = OC.frozen_stack_steps(t, [(t, t), (t - 2, t)], 9, 3)
    o, g = pair(12, (60,) + (40,) * 6, steps, max_batch=2)
    Delta = 2.0 ** 40
    stages = OC.encode_frozen_stack(o, wts, o.top_level, Delta, R, p)
    gstages, acts = [], np.zeros((len(stages), o.n), dtype=np.int64)
    for i, (lay, act, rep) in enumerate(stages):
        gstages.append((imported(g, lay, R, p), {"none": 0, "square": 1, "cubic": 2}[act], rep))
        if act == "cubic":
            S = lay.bias_scale
            l = lay.level - 1
            S3 = (S * S / o.primes[l]) * S / o.primes[l - 1]
            acts[i] = OC.cubic_masked_coeffs(o, lay.rows, lay.t, R, p, S3)
    model = G.Model.from_stages(g, gstages, act_coeffs=acts)
    model.set_hoisting(mode)
    B = 3
    items = [[rng.uniform(-1, 1, t) for _ in range(p)] for _ in range(B)]
    ms = np.stack([OE.encode(OC.pack_items(it, t, R, n // 2), Delta, n) for it in items])
    out = model.forward(g.encrypt(ms, 11, 0, Delta))
    assert out.level == o.top_level - 6
    for b in range(B):
        ref = OC.forward_stages(o, OC.Ct(o.encrypt(ms[b], 11, b), Delta), stages, R, p, hoisted=mode)
        assert np.array_equal(u64(out.data)[b], ref.data), b
        y = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
        for r in range(p):
            ref_f = OC.plain_frozen_forward(items[b][r], wts)
            assert np.max(np.abs(y[r * R: r * R + ref_f.size] - ref_f)) < 1e-3


def test_frozen_stack_library_encoders():
    """Same stack built entirely with the library's own encoders (conv1d/avgpool/dense constructors)."""
    t, n = 64, 4096
    p, R = OC.packing(n // 2, t, 4)
    rng = np.random.default_rng(7)
    wts = weights(t, rng)
    steps = OC.frozen_stack_steps(t, [(t, t), (t - 2, t)], 9, 3)
    g = G.Context(12, (60,) + (40,) * 6, (60,), key_seed=77, rot_steps=steps, max_batch=4)
    Delta = 2.0 ** 40
    l0 = g.top_level
    conv = G.GeneralLayer.conv1d(g, wts["conv_w"], wts["conv_b"], t, R, p, l0, Delta)
    d1 = G.GeneralLayer.dense(g, wts["W1"], wts["b1"], R, p, l0 - 1, Delta)
    S3 = (Delta * Delta / g.primes[l0 - 2]) * Delta / g.primes[l0 - 3]
    pool = G.GeneralLayer.avgpool(g, 3, t, R, p, l0 - 4)
    W2 = np.zeros((t - 2, t))
    W2[:, 2:] = wts["W2"]
    d2 = G.GeneralLayer.dense(g, W2, wts["b2"], R, p, l0 - 5, S3)
    model = G.Model.from_stages(g, [(conv, 0, 0), (d1, 2, t), (pool, 0, 0), (d2, 0, t)])
    model.set_hoisting(True)
    items = [rng.uniform(-1, 1, t) for _ in range(p)]
    ct = g.encrypt(g.encode(OC.pack_items(items, t, R, n // 2), Delta), 3, 0, Delta)
    out = model.forward(ct)
    y = g.decode(u64(g.decrypt(out))[0], out.level, out.scale)
    for r in range(p):
        ref_f = OC.plain_frozen_forward(items[r], wts)
        assert np.max(np.abs(y[r * R: r * R + ref_f.size] - ref_f)) < 1e-3


@pytest.mark.parametrize("mode", [1, 2])
def test_paper_stack_t768_parity(mode):
    """The paper's shapes: t = 768, conv f=9, dense 768 + ReLU_approx, pool 3, dense 766, p = 5
    items at N=16384 (Table 2 p column), depth 6 on the [60, 40x7 | 60] chain; bit-exact vs the oracle."""
    t, n = 768, 16384
    p, R = OC.packing(n // 2, t, 4)
    assert p == 5
    rng = np.random.default_rng(8)
    wts = weights(t, rng)
    steps = OC.frozen_stack_steps(t, [(t, t), (t - 2, t)], 9, 3)
    o, g = pair(14, (60,) + (40,) * 7, steps, max_batch=1)
    Delta = 2.0 ** 40
    stages = OC.encode_frozen_stack(o, wts, o.top_level, Delta, R, p)
    gst, acts = [], np.zeros((len(stages), o.n), dtype=np.int64)
    for i, (lay, act, rep) in enumerate(stages):
        gst.append((imported(g, lay, R, p), {"none": 0, "cubic": 2}[act], rep))
        if act == "cubic":
            S = lay.bias_scale
            l = lay.level - 1
            acts[i] = OC.cubic_masked_coeffs(o, lay.rows, lay.t, R, p, (S * S / o.primes[l]) * S / o.primes[l - 1])
    model = G.Model.from_stages(g, gst, act_coeffs=acts)
    model.set_hoisting(mode)
    items = [rng.uniform(-1, 1, t) for _ in range(p)]
    m = OE.encode(OC.pack_items(items, t, R, n // 2), Delta, n)
    out = model.forward(g.encrypt(m, 13, 0, Delta))
    ref = OC.forward_stages(o, OC.Ct(o.encrypt(m, 13, 0), Delta), stages, R, p, hoisted=mode)
    assert np.array_equal(u64(out.data)[0], ref.data)
    y = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
    for r in range(p):
        ref_f = OC.plain_frozen_forward(items[r], wts)
        assert np.max(np.abs(y[r * R: r * R + ref_f.size] - ref_f)) < 1e-3
