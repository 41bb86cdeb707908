"""Host-side check of the CUDA NTT's register/shared-memory layout (csrc/ntt.cuh):
  * every pass touches every index exactly once (a permutation), groups follow the stage structure;
  * the XOR swizzle a ^ (((a >> 4) ^ (a >> 5)) & 15) makes every 64-bit warp access conflict-free
    (2 wavefronts = the minimum for 32 x 8 bytes) for every supported (LOGN, threads).
Mirrors NttCta::index / swz exactly."""
import pytest


def ntt_threads(logn):
    return 1 << (logn - 4)        # default 16 residues per thread (ntt.cuh NttThreads)


def passes(logn, loge):
    """radix-16 passes (ntt.cuh LOGK = 4) regardless of the residues per thread"""
    out, s0 = [], 0
    while s0 < logn:
        k = min(4, logn - s0)
        out.append((s0, k))
        s0 += k
    return out


def index(logn, loge, s0, k, tid, g, i, nt):
    sh = logn - s0 - k
    gid = g * nt + tid
    b0, o = gid >> sh, gid & ((1 << sh) - 1)
    return (b0 << (logn - s0)) + (i << sh) + o


def wavefronts(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(half):
            banks.setdefault(a % 16, set()).add(a)
        tot += max(len(v) for v in banks.values())
    return tot


@pytest.mark.parametrize("per_thread", [16, 32])
@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14])
def test_ntt_layout(logn, per_thread):
    nt = (1 << logn) // per_thread
    E = (1 << logn) // nt
    loge = E.bit_length() - 1
    swz = lambda a: a ^ (((a >> 4) ^ (a >> 5)) & 15)
    for s0, k in passes(logn, loge):
        G = E >> k
        seen = set()
        for w in range(0, nt, 32):
            for g in range(G):
                for i in range(1 << k):
                    addrs = [index(logn, loge, s0, k, w + l, g, i, nt) for l in range(32)]
                    seen.update(addrs)
                    assert wavefronts([swz(a) for a in addrs]) == 2
                    # butterfly partner at the pass's first stage differs in bit logn-1-s0
        assert seen == set(range(1 << logn))
        # group elements are spaced by the stage stride
        for tid in range(0, nt, max(1, nt // 7)):
            idx = [index(logn, loge, s0, k, tid, 0, i, nt) for i in range(1 << k)]
            stride = 1 << (logn - s0 - k)
            assert all(b - a == stride for a, b in zip(idx, idx[1:]))


def tw_position(logn, s, m):
    logk = 4
    S0 = (s // logk) * logk
    r = s - S0
    return (1 << s) + ((m & ((1 << r) - 1)) << S0) + (m >> r)


@pytest.mark.parametrize("logn", [10, 13, 14])
def test_twiddle_order_is_a_permutation_and_matches_kernel_lookup(logn):
    """Host table position ntt_tw_position and the kernel's tw_index address the same entry."""
    n = 1 << logn
    nt = ntt_threads(logn)
    loge = ((1 << logn) // nt).bit_length() - 1
    pos = {tw_position(logn, s, m) for s in range(logn) for m in range(1 << s)}
    assert pos == set(range(1, n))
    for s0, k in passes(logn, loge):
        sh = logn - s0 - k
        for tid in range(0, nt, 37):
            for g in range(((1 << loge) >> k)):
                b0 = (g * nt + tid) >> sh
                for r in range(k):
                    for j in range(1 << r):
                        kernel_idx = (1 << (s0 + r)) + (j << s0) + b0
                        assert kernel_idx == tw_position(logn, s0 + r, b0 * (1 << r) + j)
