"""GPU parity of hybrid key switching (R9b, R10b, R17b, R29): digits of 1 or
2 consecutive data primes (exact 2-prime CRT lifts), K = 1 or 2 special primes with P = P_0 P_1.  Every
kernel of the key-switching path (digits, ModUp, the IMAD / tensor-core / key-stationary inner products,
ModDown, the Q_l P basis MAC and lift) is compared bit-exactly with the CPU oracle's definition.
"""
import dataclasses

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
import oracle_pool as OP  # noqa: E402
from test_gpu_launch_shape import gpu_forward, check  # noqa: E402


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


VARIANTS = {
    # (data bits, special bits, digits)
    "hybrid_k2": ((60, 40, 40, 40, 40), (40, 40), (1, 2, 2)),
    "k2_single_digits": ((60, 40, 40, 40), (40, 40), None),
    "k1_pair_digits": ((60, 40, 40, 40, 40), (60,), (1, 2, 2)),
    "k2_pairs_fpr": ((50, 45, 45, 45, 45), (45, 45), (2, 2, 1)),
}


def pair(variant, log_n=11, steps=(1, 3, -5), max_batch=2, seed=31):
    data, special, digits = VARIANTS[variant]
    o = oracle.Context(log_n, data, special, digits=digits)
    o.keygen(seed, steps)
    g = G.Context(log_n, data, special, key_seed=seed, rot_steps=steps, max_batch=max_batch, digits=digits)
    assert g.primes == o.primes
    assert g.n_digits == o.n_digits and g.digits == o.digits
    return o, g


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_hybrid_keys_bit_exact(variant):
    o, g = pair(variant)
    for kid in [0] + [o.galois_elt(s) for s in (1, 3, -5)]:
        assert np.array_equal(g.export_key(kid), o.export_key(kid)), kid


@pytest.mark.parametrize("variant", list(VARIANTS))
def test_hybrid_rotate_relin_parity_all_levels(variant):
    """Non-hoisted and hoisted rotations and relinearisation at every level (lower levels cut a 2-prime
    digit to one prime), ragged batch of 3 over max_batch 2; uniform residues (bit-exact only)."""
    o, g = pair(variant)
    L = len(o.primes) - o.n_special
    for level in range(L - 1, -1, -1):
        x = S.uniform_residues(level + 7, g.primes[: level + 1], (3, 3), g.n)   # [3 cts][3 comps][l+1][N]
        ct2 = g.from_numpy(np.ascontiguousarray(x[:, :2]), scale=2.0 ** 40)
        for step in (1, -5):
            got = u64(g.rotate(ct2, step).data)
            goth = u64(g.rotate_hoisted(ct2, [step, 3])[0].data)
            for b in range(3):
                assert np.array_equal(got[b], o.rotate(x[b, :2], step)), (level, step, b)
                assert np.array_equal(goth[b], o.rotate_hoisted(x[b, :2], step)), (level, step, b)
        ct3 = g.from_numpy(x, scale=2.0 ** 40)
        got = u64(g.relinearize(ct3).data)
        for b in range(3):
            assert np.array_equal(got[b], o.relinearize(x[b])), (level, b)


@pytest.mark.parametrize("variant", ["hybrid_k2", "k1_pair_digits"])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_hybrid_matvec_parity(variant, mode):
    """One dense layer t = 64 in every rotation schedule (double hoisting: the Q_l P MAC over K special
    rows, the tensor-core baby-step inner product with 2-prime digit rows, the key-stationary giant step)."""
    o, g = pair(variant, log_n=11, steps=OC.rotation_steps_for([(16, 64)]), max_batch=3)
    rng = np.random.default_rng(mode)
    W = rng.normal(0, 0.1, (16, 64))
    b = rng.uniform(-0.1, 0.1, 16)
    lay = OC.encode_layer(o, W, b, o.top_level, 2.0 ** 40)
    gl = G.Layer(g, 16, 64, lay.level, diag_coeffs=lay.diag_coeffs, bias_coeffs=lay.bias_coeffs,
                 pt_scale=lay.pt_scale, bias_scale=lay.bias_scale).set_hoisting(mode)
    xs = [rng.uniform(-1, 1, 64) for _ in range(4)]
    ms = np.stack([OE.encode(OC.pack_input(x, lay.t, o.n // 2), 2.0 ** 40, o.n) for x in xs])
    out = gl.matvec(g.encrypt(ms, 9, 0, 2.0 ** 40))
    for bb in range(4):
        ref = OC.matvec(o, OC.Ct(o.encrypt(ms[bb], 9, bb), 2.0 ** 40), lay, hoisted=mode)
        assert np.array_equal(u64(out.data)[bb], ref.data), bb
        if variant == "hybrid_k2":
            y = OE.decode(o.decrypt(ref.data), o.primes, ref.scale, o.n)
            assert np.max(np.abs(y[:16] - (W @ xs[bb] + b))) < 1e-3


SMALL_HYBRID = S.Config(name="small_ring_hybrid", log_n=12, data_bits=(60,) + (40,) * 5, special_bits=(40, 40),
                        log2_scale=40, layers=((64, 128), (32, 64)), activation="square", in_dim=128,
                        weight_std=(1 / np.sqrt(128), 1 / np.sqrt(64)), digits=(1, 2, 2, 1))


@pytest.mark.parametrize("activation,mode,x", [("square", 2, 1), ("cubic", 2, 1), ("square", 1, 0), ("square", 0, 0)])
def test_hybrid_forward_small_ring_every_ciphertext(activation, mode, x):
    """The cfg4 network shape on N = 4096 with [60, 40x5 | 40, 40] and digits {q0}{q1q2}{q3q4}{q5}, batch
    45 in launch sequences of 40 (2 full batch tiles + ragged): every ciphertext vs the oracle."""
    B, mb = 45, 40
    cfg = dataclasses.replace(SMALL_HYBRID, activation=activation)
    spec = {"kind": "dense", "cfg": cfg, "batch": B, "activation": activation, "hoisting": mode, "x": x}
    _, got, out = gpu_forward(spec, B, mb)
    check(got, out, OP.oracle_forwards(spec, range(B)))


def test_hybrid_cfg4_bench_shape_sampled():
    """R29 at full size in the bench's launch shape: cfg4 network, [60, 40x7 | 40, 40], dnum = 5,
    max_batch = 256, double hoisting, t1 = 64 / 32, B = 260; sampled ciphertexts vs the oracle."""
    B, mb = 260, 256
    spec = {"kind": "dense", "cfg": S.CFG4_HYBRID, "batch": B, "activation": "square", "hoisting": 2, "x": 1}
    _, got, out = gpu_forward(spec, B, mb)
    check(got, out, OP.oracle_forwards(spec, [0, 16, 17, 255, 256, 259]))
