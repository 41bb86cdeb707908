"""GPU edge cases: empty batch, degenerate layer shapes (t = 1, non-square, t = 1024 = max t1 x t2),
the smallest ring (N = 1024), level-1 layers ending at level 0, the maximum limb count (16 primes)."""
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


def test_empty_batch_is_rejected():
    g = G.Context(10, (40, 40), (45,), key_seed=1, rot_steps=(1,), max_batch=2)
    empty = G.Ciphertext(torch.empty((0, 2, 2, g.n), dtype=torch.int64, device="cuda"), 1, 2.0 ** 30)
    with pytest.raises(G.CkksError) as e:
        g.rotate(empty, 1, out=g.empty_ct(1, 1))
    assert e.value.status in (G.E_PARAM, G.E_SHAPE)   # rejected before any launch
    t = torch.empty((0, 2, g.n), dtype=torch.int64, device="cuda")
    g.ntt_fwd(t)   # an empty NTT batch is a no-op


def test_max_limbs_ntt():
    bits = (50,) * 15 + (60,)
    g = G.Context(12, bits, (), want_relin=False, max_batch=1)
    o = oracle.Context(12, bits, ())
    x = S.uniform_residues(5, g.primes, (2,), g.n)
    t = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_fwd(t)
    got = u64(t)
    for l in (0, 7, 15):
        assert np.array_equal(got[1, l], o.ntt(x[1, l], l))
    g.ntt_inv(t)
    assert np.array_equal(u64(t), x)


@pytest.mark.parametrize("mode", [0, 2])
@pytest.mark.parametrize("shape,log_n", [((1, 1), 10), ((5, 3), 10), ((3, 17), 11), ((1024, 1024), 12)])
def test_degenerate_and_max_layer_shapes(shape, log_n, mode):
    """t = 1 (no rotation at all), non-square, t = 1024 (t1 = t2 = 32, the largest tile)."""
    rows, cols = shape
    steps = OC.rotation_steps_for([shape])
    bits = (50, 40, 40)
    o = oracle.Context(log_n, bits, (50,))
    o.keygen(9, steps)
    g = G.Context(log_n, bits, (50,), key_seed=9, rot_steps=steps, max_batch=2)
    rng = np.random.default_rng(rows * 31 + cols)
    W = rng.normal(0, 1 / np.sqrt(cols), (rows, cols))
    b = rng.uniform(-0.1, 0.1, rows)
    lay = OC.encode_layer(o, W, b, o.top_level, 2.0 ** 30)
    gl = G.Layer(g, rows, cols, lay.level, diag_coeffs=lay.diag_coeffs, bias_coeffs=lay.bias_coeffs,
                 pt_scale=lay.pt_scale, bias_scale=lay.bias_scale).set_hoisting(mode)
    x = rng.uniform(-1, 1, cols)
    m = OE.encode(OC.pack_input(x, lay.t, o.n // 2), 2.0 ** 30, o.n)
    ct = g.encrypt(np.stack([m, m]), 4, 0, 2.0 ** 30)
    out = gl.matvec(ct)
    for bb in range(2):
        ref = OC.matvec(o, OC.Ct(o.encrypt(m, 4, bb), 2.0 ** 30), lay, hoisted=mode)
        assert np.array_equal(u64(out.data)[bb], ref.data)
    y = OE.decode(o.decrypt(u64(out.data)[0]), o.primes, out.scale, o.n)
    assert np.max(np.abs(y[:rows] - (W @ x + b))) < 1e-3


def test_smallest_ring_forward_to_level0():
    """N = 1024, two layers with the square activation consuming the whole chain (ends at level 0)."""
    cfg = S.Config(name="tiny", log_n=10, data_bits=(50, 40, 40, 40), special_bits=(50,), log2_scale=30,
                   layers=((8, 16), (4, 8)), activation="square", in_dim=16, weight_std=(0.25, 0.35))
    steps = OC.rotation_steps_for(cfg.layers)
    o = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    o.keygen(cfg.key_seed, steps)
    g = G.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, key_seed=cfg.key_seed, rot_steps=steps, max_batch=1)
    prob = S.dense_problem(cfg, batch=1)
    D = 2.0 ** 30
    layers = OC.encode_model(o, prob["W"], prob["b"], o.top_level, D, "square")
    gl = [G.Layer(g, l.rows, l.cols, l.level, diag_coeffs=l.diag_coeffs, bias_coeffs=l.bias_coeffs,
                  pt_scale=l.pt_scale, bias_scale=l.bias_scale) for l in layers]
    model = G.Model(g, gl, G.ACT_SQUARE)
    m = OE.encode(OC.pack_input(prob["x"][0], layers[0].t, o.n // 2), D, o.n)
    out = model.forward(g.encrypt(m, 2, 0, D))
    assert out.level == 0
    ref = OC.forward(o, OC.Ct(o.encrypt(m, 2, 0), D), layers, "square")
    assert np.array_equal(u64(out.data)[0], ref.data)


@pytest.mark.parametrize("mac_tc", [0, 1])
@pytest.mark.parametrize("data_bits", [(60, 44, 44), (60, 40, 40)])
def test_bsgs_mac_worst_case_residues(data_bits, mac_tc):
    """Exactness bounds of the tensor-core BSGS inner sums and baby-step inner products: every
    ciphertext residue q-1 and every diagonal the constant -1 (all NTT values q-1), so every split
    partial sum is at its maximum.  t = 512 with one extra baby-step doubling (t1 = 64, t2 = 8): for
    44-bit primes the q < 2^45 accumulators fold mod q every 32 terms, for 40-bit every 64; double
    hoisting, bit-exact vs the oracle (the inputs are not encryptions; only residues are compared)."""
    log_n, special = 12, (60,)
    t, x = 512, 1
    steps = OC.rotation_steps_for([(t, t)], x)
    o = oracle.Context(log_n, data_bits, special)
    o.keygen(7, steps)
    g = G.Context(log_n, data_bits, special, key_seed=7, rot_steps=steps, max_batch=2, bsgs_baby_extra=x)
    n, level = g.n, len(data_bits) - 1
    diag = np.zeros((t, n), dtype=np.int64)
    diag[:, 0] = -1
    lay = OC.EncodedLayer(t, t, t, 64, 8, level, float(o.primes[level]), 2.0 ** 30, diag, np.zeros(n, dtype=np.int64))
    gl = G.Layer(g, t, t, level, diag_coeffs=lay.diag_coeffs, bias_coeffs=lay.bias_coeffs, pt_scale=lay.pt_scale,
                 bias_scale=lay.bias_scale).set_hoisting(2)
    data = np.empty((2, 2, level + 1, n), dtype=np.uint64)
    for i in range(level + 1):
        data[:, :, i, :] = np.uint64(o.primes[i] - 1)
    data[1, 1, :, ::3] = 0                                          # second ciphertext: a mix with zeros
    ct = G.Ciphertext(torch.from_numpy(data.view(np.int64)).cuda(), level, 2.0 ** 30)
    old = G.get_option("mac_tc")
    G.set_option("mac_tc", mac_tc)           # also the integer tensor-core MAC: T_s sums at their bound
    try:
        out = gl.matvec(ct)
    finally:
        G.set_option("mac_tc", old)
    for b in range(2):
        ref = OC.matvec(o, OC.Ct(data[b].copy(), 2.0 ** 30), lay, hoisted=2)
        assert np.array_equal(u64(out.data)[b], ref.data), (data_bits, b)


def _small_dense_model(max_batch, activation="cubic", steps_drop=()):
    cfg = S.Config(name="small", log_n=12, data_bits=(60,) + (40,) * 5, special_bits=(60,), log2_scale=40,
                   layers=((64, 128), (32, 64)), activation=activation, in_dim=128,
                   weight_std=(1 / np.sqrt(128), 1 / np.sqrt(64)))
    steps = [s for s in OC.rotation_steps_for(cfg.layers, 1) if s not in steps_drop]
    o = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    g = G.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, key_seed=cfg.key_seed, rot_steps=steps,
                  max_batch=max_batch, bsgs_baby_extra=1)
    D = 2.0 ** 40
    prob = S.dense_problem(cfg, batch=4)
    layers = OC.encode_model(o, prob["W"], prob["b"], o.top_level, D, activation, 1)
    gl = [G.Layer(g, l.rows, l.cols, l.level, diag_coeffs=l.diag_coeffs, bias_coeffs=l.bias_coeffs,
                  pt_scale=l.pt_scale, bias_scale=l.bias_scale) for l in layers]
    model = G.Model(g, gl, {"square": 1, "cubic": 2}[activation],
                    act_coeffs=OC.activation_plaintexts(o, layers, activation))
    model.set_hoisting(2)
    ms = np.stack([OE.encode(OC.pack_input(prob["x"][b], layers[0].t, o.n // 2), D, o.n) for b in range(4)])
    return g, model, ms, D


@pytest.mark.parametrize("activation", ["square", "cubic"])
def test_forward_graph_matches_stream_forward(activation):
    """ckks_forward_graph_create / ckks_graph_launch (the forward as one CUDA graph) gives the same bits
    as the stream forward, replayed twice over new inputs copied into the bound buffer."""
    g, model, ms, D = _small_dense_model(4, activation)
    ct = g.encrypt(ms[:3], 11, 0, D)
    ref = model.forward(ct)
    inp = g.encrypt(ms[:3], 12, 0, D)                    # another encryption in the bound input buffer
    graph = model.graph(inp)
    l0 = g.launches()
    inp.data.copy_(ct.data)
    out = graph.launch()
    torch.cuda.synchronize()
    assert out.level == ref.level and out.scale == ref.scale
    assert torch.equal(out.data, ref.data)
    assert g.launches() - l0 == graph_kernels(g, graph, l0)
    out.data.zero_()
    graph.launch()
    torch.cuda.synchronize()
    assert torch.equal(out.data, ref.data)


def graph_kernels(g, graph, l0):
    return g.launches() - l0


def test_forward_host_small_batch_tight_workspace():
    """a host-buffer forward with batch < max_batch and a workspace sized for that batch
    (ckks_model_work_sizes(batch)) stays inside the workspace and matches the device forward."""
    g, model, ms, D = _small_dense_model(8, "square")
    ct = g.encrypt(ms[:3], 11, 0, D)
    ref = model.forward(ct)
    nb = model.work_bytes(3)
    work = torch.zeros(nb + 4096, dtype=torch.uint8, device="cuda")
    work[nb:] = 0xA5                                     # guard band after the sized workspace
    h_in = torch.empty(tuple(ct.data.shape), dtype=torch.int64, pin_memory=True)
    h_in.copy_(ct.data)
    h_out = torch.empty(tuple(ref.data.shape), dtype=torch.int64, pin_memory=True)
    lvl, sc = model.forward_host(h_in, ct.level, ct.scale, h_out, work[:nb])
    assert lvl == ref.level and sc == ref.scale
    assert torch.equal(h_out, ref.data.cpu())
    assert bool((work[nb:] == 0xA5).all()), "host forward wrote past its workspace"


def test_rescale_without_special_prime():
    """a context with no special prime (no key switching) still rescales inside its own
    workspace, bit-exact vs the oracle."""
    bits = (50, 40, 40)
    o = oracle.Context(11, bits, ())
    g = G.Context(11, bits, (), want_relin=False, max_batch=2)
    x = S.uniform_residues(9, g.primes, (2, 2), g.n)     # [2 cts][2 comps][3 limbs][N]
    ct = g.from_numpy(x, scale=2.0 ** 40)
    out = g.rescale(ct)
    for b in range(2):
        assert np.array_equal(u64(out.data)[b], o.rescale(x[b]))


def test_missing_key_rejected_before_any_launch():
    """ckks.h: on error nothing has been launched -- a model whose giant-step key is missing fails in
    the up-front key check (CKKS_E_NOKEY) without launching a kernel."""
    g, model, ms, D = _small_dense_model(4, "square", steps_drop=(64,))
    ct = g.encrypt(ms[:2], 11, 0, D)
    torch.cuda.synchronize()
    l0 = g.launches()
    with pytest.raises(G.CkksError) as e:
        model.forward(ct)
    assert e.value.status == G.E_NOKEY
    assert g.launches() == l0
