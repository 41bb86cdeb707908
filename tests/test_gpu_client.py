"""GPU parity of the client side on the device: canonical-embedding encode of a batch
(ckks_encode_device) against the oracle's encoder (R4, R16: +-1 on a bounded fraction of coefficients, FP64
rounding order), device encryption from device coefficients (bit-exact with the oracle's encryption of the
same coefficients), device decode against the oracle's decode, and the encode -> encrypt -> decrypt ->
decode round trip (2^-28 at scale 2^40)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle  # noqa: E402
from oracle import encoding as OE  # noqa: E402
import synthetic as S  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402


def u64(t):
    return t.detach().cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("log_n,count", [(10, 512), (12, 1000), (13, 64), (14, 8192), (14, 1024)])
def test_encode_device_vs_oracle_encoder(log_n, count):
    g = G.Context(log_n, (60, 40), (60,), want_relin=False, max_batch=4)
    rng = np.random.default_rng(log_n * 7 + count)
    B = 5
    vals = rng.uniform(-1, 1, (B, count))
    got = g.encode_device(torch.from_numpy(vals).cuda(), 2.0 ** 40).cpu().numpy()
    for b in range(B):
        ref = OE.encode(np.concatenate([vals[b], np.zeros(g.n // 2 - count)]), 2.0 ** 40, g.n)
        d = np.abs(got[b] - ref)
        assert d.max() <= 1 and (d > 0).mean() < 1e-3, (b, d.max(), (d > 0).mean())


def test_encrypt_device_bit_exact_and_decode_device():
    cfg = S.CFG1
    o = oracle.Context(cfg.log_n, cfg.data_bits, cfg.special_bits)
    o.keygen(cfg.key_seed, ())
    g = G.Context(cfg.log_n, cfg.data_bits, cfg.special_bits, key_seed=cfg.key_seed, max_batch=2)
    rng = np.random.default_rng(3)
    B = 3
    vals = rng.uniform(-1, 1, (B, g.n // 2))
    ms = np.stack([OE.encode(v, 2.0 ** 40, g.n) for v in vals])            # the oracle's coefficients
    ct = g.encrypt_device(torch.from_numpy(ms).cuda(), cfg.enc_seed, 0, 2.0 ** 40)
    for b in range(B):
        assert np.array_equal(u64(ct.data)[b], o.encrypt(ms[b], cfg.enc_seed, b)), b
    assert torch.equal(ct.data, g.encrypt(ms, cfg.enc_seed, 0, 2.0 ** 40).data)   # = the host-coefficient path
    dec = g.decrypt(ct)
    y = g.decode_device(dec, ct.level, ct.scale, g.n // 2).cpu().numpy()
    for b in range(B):
        ref = OE.decode(o.decrypt(u64(ct.data)[b]), o.primes, 2.0 ** 40, o.n)
        assert np.max(np.abs(y[b] - ref)) < 1e-9
        assert np.max(np.abs(y[b] - vals[b])) < 2.0 ** -20          # fresh-encryption noise over 2^40


def test_client_round_trip_through_a_forward_level():
    """Device encode -> device encrypt -> rotate -> rescale-level decrypt -> device decode (lower level,
    other scale): the slots come back rotated within 2^-20."""
    g = G.Context(12, (60, 40, 40), (60,), key_seed=5, rot_steps=(3,), max_batch=4)
    rng = np.random.default_rng(8)
    vals = rng.uniform(-1, 1, (4, g.n // 2))
    coeffs = g.encode_device(torch.from_numpy(vals).cuda(), 2.0 ** 40)
    ct = g.encrypt_device(coeffs, 9, 0, 2.0 ** 40)
    r = g.rotate(ct, 3)
    y = g.decode_device(g.decrypt(r), r.level, r.scale, g.n // 2).cpu().numpy()
    assert np.max(np.abs(y - np.roll(vals, -3, axis=1))) < 2.0 ** -20
