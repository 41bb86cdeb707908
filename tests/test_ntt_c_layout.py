"""Host-side check of the CTA-pair NTT schedule's layout (csrc/ntt_c.cuh), mirrored here index for index:
  * pass structure: stage 0 across the cluster (N = 16384), then K1 = log2(M) - 8 stages, then 4 + 4;
  * every pass's register <-> point map is a permutation of the CTA's M points and groups the 2^K points a
    radix-2^K butterfly network needs (same high bits above the pass, same low bits below it);
  * the padded shared-memory address a(o) = o + (o >> 4) makes every 64-bit warp access of the exchange
    conflict-free (2 wavefronts per 32 x 8 bytes), and the TMA output rows (stride 18 words) are written with
    conflict-free 128-bit accesses (4 wavefronts per 32 x 16 bytes);
  * the pair-table order ntt_c_tw_position is a bijection onto [1, N) and agrees with the kernel's lookup
    (1 << s) + (j << S0) + b0.
"""
import pytest


def cl(logn):
    return 2 if logn >= 14 else 1


def params(logn):
    sb = 1 if cl(logn) == 2 else 0
    logm = logn - sb
    return sb, logm, 1 << logm, (1 << logm) // 32, logm - 8


def pass_cfg(logn, p):
    sb, logm, M, NT, K1 = params(logn)
    s0 = 0 if p == 0 else K1 + 4 * (p - 1)
    k = K1 if p == 0 else 4
    return s0, k, 32 >> k, logm - s0 - k


def pad(o):
    return o + (o >> 4)


def point(logn, p, t, g, i):
    """index (within the CTA's M points) of register g 2^K + i of thread t in pass p"""
    sb, logm, M, NT, K1 = params(logn)
    s0, k, G, sh = pass_cfg(logn, p)
    gid = g * NT + t
    return ((gid >> sh) << (sh + k)) + (gid & ((1 << sh) - 1)) + (i << sh)


def wavefronts64(addrs):
    tot = 0
    for half in (addrs[:16], addrs[16:]):
        banks = {}
        for a in set(half):
            banks.setdefault(a % 16, set()).add(a)
        tot += max(len(v) for v in banks.values())
    return tot


def wavefronts128(addrs16):
    """addresses in 16-byte units; a 128-bit warp access is served 8 lanes at a time over 8 banks of 16 bytes"""
    tot = 0
    for q in range(4):
        banks = {}
        for a in set(addrs16[8 * q: 8 * q + 8]):
            banks.setdefault(a % 8, set()).add(a)
        tot += max(len(v) for v in banks.values())
    return tot


@pytest.mark.parametrize("logn", [12, 13, 14])
def test_passes_are_permutations_and_conflict_free(logn):
    sb, logm, M, NT, K1 = params(logn)
    assert K1 in (4, 5) and sb + K1 + 8 == logn
    for p in range(3):
        s0, k, G, sh = pass_cfg(logn, p)
        seen = set()
        for t in range(NT):
            for g in range(G):
                pts = [point(logn, p, t, g, i) for i in range(1 << k)]
                # one butterfly network: the points differ exactly in bits [sh, sh + k)
                base = pts[0]
                assert all(pt == base + (i << sh) for i, pt in enumerate(pts)) and (base >> sh) % (1 << k) == 0
                seen.update(pts)
        assert seen == set(range(M))
        # shared-memory exchange: register (g, i) of the 32 lanes of a warp in one access
        for w in range(0, NT, 32):
            for g in range(G):
                for i in range(1 << k):
                    assert wavefronts64([pad(point(logn, p, t, g, i)) for t in range(w, w + 32)]) == 2
    # pass 0 covers o = t + pos0(e): lane <-> consecutive o (coalesced global loads)
    s0, k, G, sh = pass_cfg(logn, 0)
    for e in range(32):
        g, i = e >> k, e & ((1 << k) - 1)
        assert [point(logn, 0, t, g, i) for t in range(32)] == list(range(point(logn, 0, 0, g, i),
                                                                          point(logn, 0, 0, g, i) + 32))
    # the last pass leaves 16 consecutive outputs per (thread, group): one 128-byte row each
    s0, k, G, sh = pass_cfg(logn, 2)
    assert sh == 0 and k == 4
    rows = sorted(point(logn, 2, t, g, 0) for t in range(NT) for g in range(G))
    assert rows == list(range(0, M, 16))


@pytest.mark.parametrize("logn", [12, 13, 14])
def test_tma_rows_conflict_free(logn):
    sb, logm, M, NT, K1 = params(logn)
    roww = 18                                                   # words per row (144 bytes, 16-byte aligned)
    assert (roww * 8) % 16 == 0 and roww >= 16
    assert (M // 16) * roww * 8 + 16 <= 113 * 1024              # two CTAs per SM fit the 227 KiB
    for g in range(2):
        for w in range(0, NT, 32):
            for i in range(0, 16, 2):
                a16 = [((g * NT + t) * roww + i) // 2 for t in range(w, w + 32)]
                assert wavefronts128(a16) == 4


def tw_position(logn, s, m):
    sb, logm, M, NT, K1 = params(logn)
    S0 = 0 if s < sb else (sb if s < sb + K1 else (sb + K1 if s < sb + K1 + 4 else sb + K1 + 4))
    r = s - S0
    return (1 << s) + ((m & ((1 << r) - 1)) << S0) + (m >> r)


@pytest.mark.parametrize("logn", [12, 13, 14])
def test_pair_table_order(logn):
    sb, logm, M, NT, K1 = params(logn)
    pos = [tw_position(logn, s, m) for s in range(logn) for m in range(1 << s)]
    assert sorted(pos) == list(range(1, 1 << logn))
    # kernel lookup of stage S0g + r of pass p for the butterfly on registers (i, i + half) of group g, thread t,
    # CTA rank h: block index of that butterfly in the whole transform = (point >> (logm - s_local)) + h 2^(s - sb)
    for h in range(cl(logn)):
        for p in range(3):
            s0, k, G, sh = pass_cfg(logn, p)
            S0g = sb + s0
            for t in (0, 1, NT // 2 + 3, NT - 1):
                for g in range(G):
                    b0 = (h << s0) + ((g * NT + t) >> sh)
                    for r in range(k):
                        half = 1 << (k - 1 - r)
                        for i in range(1 << k):
                            if i & half:
                                continue
                            s = S0g + r
                            pt = point(logn, p, t, g, i)
                            block = (pt >> (logm - (s0 + r))) + (h << (s0 + r))      # block of stage s in the limb
                            assert (1 << s) + ((i >> (k - r)) << S0g) + b0 == tw_position(logn, s, block)
