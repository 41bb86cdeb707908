"""Host-side check of the CUDA NTT's register/shared-memory layout (csrc/ntt.cuh):
  * every pass touches every index exactly once (a permutation), groups follow the stage structure;
  * the XOR swizzle a ^ ((a >> LOGE) & 15) makes every 64-bit warp access conflict-free
    (2 wavefronts = the minimum for 32 x 8 bytes) for every supported (LOGN, threads).
Mirrors NttCta::index / swz exactly."""
import pytest


def ntt_threads(logn):
    return (1 << (logn - 5)) if logn >= 13 else (1 << (logn - 4))


def passes(logn, loge):
    out, s0 = [], 0
    while s0 < logn:
        k = min(loge, logn - s0)
        out.append((s0, k))
        s0 += k
    return out


def index(logn, loge, s0, k, tid, g, i):
    G = (1 << loge) >> k
    sh = logn - s0 - k
    gid = tid * G + g
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


@pytest.mark.parametrize("logn", [10, 11, 12, 13, 14])
def test_ntt_layout(logn):
    nt = ntt_threads(logn)
    E = (1 << logn) // nt
    loge = E.bit_length() - 1
    swz = lambda a: a ^ ((a >> loge) & 15)
    for s0, k in passes(logn, loge):
        G = E >> k
        seen = set()
        for w in range(0, nt, 32):
            for g in range(G):
                for i in range(1 << k):
                    addrs = [index(logn, loge, s0, k, w + l, g, i) for l in range(32)]
                    seen.update(addrs)
                    assert wavefronts([swz(a) for a in addrs]) == 2
                    # butterfly partner at the pass's first stage differs in bit logn-1-s0
        assert seen == set(range(1 << logn))
        # group elements are spaced by the stage stride
        for tid in range(0, nt, max(1, nt // 7)):
            idx = [index(logn, loge, s0, k, tid, 0, i) for i in range(1 << k)]
            stride = 1 << (logn - s0 - k)
            assert all(b - a == stride for a, b in zip(idx, idx[1:]))
