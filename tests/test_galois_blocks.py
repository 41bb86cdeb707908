"""Host-side invariant the tensor-core inner product's output permutation relies on:
the NTT-domain Galois permutation sigma_g (slot index k <-> odd exponent
2 brev(k) + 1, sigma_g multiplies the exponent by g mod 2N) maps every aligned block of KT consecutive NTT
indices onto one aligned block.  `k_ks_ip_mma2` therefore computes each rotation's destination block once
per launch and writes whole blocks, so a permutation that split a block would scatter outputs wrongly.
"""
import numpy as np
import pytest


def brev(x, bits):
    return int(format(x, f"0{bits}b")[::-1], 2) if bits else 0


def galois_index_map(logn, g):
    """dst[k] = NTT index holding the image of index k under X -> X^g (exponent identity of 8(c)3)."""
    n = 1 << logn
    out = np.empty(n, dtype=np.int64)
    for k in range(n):
        e = (2 * brev(k, logn) + 1) * g % (2 * n)
        out[k] = brev((e - 1) // 2, logn)
    return out


@pytest.mark.parametrize("logn", [6, 10, 14])
@pytest.mark.parametrize("kt", [8, 16])
def test_sigma_maps_aligned_blocks_onto_aligned_blocks(logn, kt):
    n = 1 << logn
    steps = [1, 2, 3, 5, 64, n // 2 - 1, -1, -256 % (n // 2)]
    for r in steps:
        g = pow(5, r % (n // 2), 2 * n)
        dst = galois_index_map(logn, g)
        assert sorted(dst.tolist()) == list(range(n))          # a permutation
        blocks = dst.reshape(n // kt, kt) // kt
        assert (blocks == blocks[:, :1]).all()                  # each source block lands in one block
        assert sorted(blocks[:, 0].tolist()) == list(range(n // kt))
    # the conjugation X -> X^{-1} (g = 2N - 1) too
    dst = galois_index_map(logn, 2 * n - 1)
    blocks = dst.reshape(n // kt, kt) // kt
    assert (blocks == blocks[:, :1]).all()
