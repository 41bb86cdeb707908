"""GPU parity of the CTA-pair NTT schedule (csrc/ntt_c.cuh: thread-block clusters + DSMEM for N = 16384, two
CTAs per SM for N <= 8192, TMA row copies) against the oracle's textbook negacyclic NTT (R2), for every value of
the library option that selects it (ckks_set_option("ntt_q", mask)):
   0   whole-limb kernels only (ntt.cuh)
   3   batch NTT forward + inverse on the cluster schedule (TMA rows where the library picks them)
  67   the same with plain 256-bit global accesses
  15   + the key-switch ModUp on it at every N (N = 16384 is off by default: measured slower)
  79   the same with plain accesses
Prime classes: 22/40-bit (PC_FP), 46/50-bit (PC_FPR, one reduction per butterfly) on the cluster schedule, 60-bit
limbs of the same launch on the whole-limb integer kernel (the launcher splits the limb range by class).
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]

import oracle  # noqa: E402
import synthetic as S  # noqa: E402
from paper_2205_11935_b200 import ckks as G  # noqa: E402
import oracle_pool as OP  # noqa: E402
from test_gpu_launch_shape import SMALL, gpu_forward, check, u64  # noqa: E402


@pytest.fixture
def ntt_q(request):
    old = G.get_option("ntt_q")
    G.set_option("ntt_q", request.param)
    yield request.param
    G.set_option("ntt_q", old)


@pytest.mark.parametrize("ntt_q", [0, 3, 67], indirect=True)
@pytest.mark.parametrize("log_n", [12, 13, 14])
def test_batch_ntt_every_schedule(log_n, ntt_q):
    """Forward and inverse vs the oracle, limb by limb: random residues, all q-1, alternating 0 / q-1, a ragged
    batch (5 polynomials), limb classes interleaved (FP, 60-bit, FP, FPR, FPR, 60-bit) so the launcher's runs of
    equal class have lengths 1, 1, 3, 1."""
    bits = (40, 60, 22, 46, 50, 60)
    g = G.Context(log_n, bits, (), max_batch=1, want_relin=False)
    o = oracle.Context(log_n, bits, ())
    assert g.primes == o.primes and g.psi == o.psi
    x = S.uniform_residues(5, g.primes, (5,), g.n)
    for l, q in enumerate(g.primes):
        x[1, l, :] = q - 1
        x[2, l, 0::2] = 0
        x[2, l, 1::2] = q - 1
        x[3, l, :] = 0
        x[3, l, 1] = 1                                       # X: the transform is the vector of psi powers
    t = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_fwd(t)
    got = u64(t)
    for b in range(5):
        for l in range(len(bits)):
            assert np.array_equal(got[b, l], o.ntt(x[b, l], l)), (b, l)
    g.ntt_inv(t)
    assert np.array_equal(u64(t), x)
    t2 = torch.from_numpy(x.view(np.int64)).cuda()
    g.ntt_inv(t2)
    inv = u64(t2)
    for b in (0, 1, 2):
        for l in range(len(bits)):
            assert np.array_equal(inv[b, l], o.intt(x[b, l], l)), (b, l)


@pytest.mark.parametrize("ntt_q", [0, 15, 79], indirect=True)
def test_modup_schedules_small_ring_every_ciphertext(ntt_q):
    """Double-hoisted forward on the N = 4096 ring (60-bit q0 and special prime: integer-class ModUp rows in their
    own launch beside the cluster kernel), B = 70 in chunks of 40: every ciphertext vs the oracle."""
    B, mb = 70, 40
    spec = {"kind": "dense", "cfg": SMALL, "batch": B, "activation": "square", "hoisting": 2, "x": 1}
    _, got, out = gpu_forward(spec, B, mb)
    check(got, out, OP.oracle_forwards(spec, range(B)))


@pytest.mark.parametrize("ntt_q", [15], indirect=True)
def test_modup_cluster_cfg4_hybrid_sampled(ntt_q):
    """The cluster ModUp at N = 16384 (CTA pairs, DSMEM stage 0) on the hybrid chain (2-prime digits: Garner
    loader, K = 2 special primes), B = 40 in one launch sequence: sampled ciphertexts vs the oracle."""
    B = 40
    spec = {"kind": "dense", "cfg": S.CFG4_HYBRID, "batch": B, "activation": "square", "hoisting": 2, "x": 1}
    _, got, out = gpu_forward(spec, B, B)
    check(got, out, OP.oracle_forwards(spec, [0, 17, 39]))


def test_nvtx_ranges_do_not_change_results():
    """ckks_set_option("nvtx", 1): NVTX ranges around every launch site (host-side only); same bits as the oracle."""
    old = G.get_option("nvtx")
    G.set_option("nvtx", 1)
    try:
        B = 5
        spec = {"kind": "dense", "cfg": SMALL, "batch": B, "activation": "square", "hoisting": 2, "x": 1}
        _, got, out = gpu_forward(spec, B, 4)
        check(got, out, OP.oracle_forwards(spec, range(B)))
    finally:
        G.set_option("nvtx", old)


@pytest.mark.parametrize("giant_multi", [0, 1])
def test_giant_step_accumulation_forms(giant_multi):
    """Double-hoisted forward with the giant steps accumulated per step (k_ks_ip_giant, option giant_multi = 0) and in
    one pass per 4 steps (k_ks_ip_giant_multi, the default: Karatsuba split products summed over the steps, one
    reduction per ciphertext): t2 = 8 giant tiles (7 steps = passes of 4 + 3) on the small ring, B = 37 in chunks of
    20 (ragged batch slices), every ciphertext vs the oracle."""
    old = G.get_option("giant_multi")
    G.set_option("giant_multi", giant_multi)
    try:
        B, mb = 37, 20
        spec = {"kind": "dense", "cfg": SMALL, "batch": B, "activation": "square", "hoisting": 2, "x": 0}
        _, got, out = gpu_forward(spec, B, mb)
        check(got, out, OP.oracle_forwards(spec, range(B)))
    finally:
        G.set_option("giant_multi", old)
