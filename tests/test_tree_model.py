"""CPU model of the device backward's reduction schedule (qfb_bwd.cu).

The kernel reproduces the reference pairwise tree (tensor.hpp:100-109) by
(1) 2^D leaf groups of <= 16 elements located by descending the recursive
floor split, (2) tiles of 2^g groups reduced by an xor butterfly, (3) the
tiles' partials reduced by a perfect tree. This test executes exactly that
schedule in Python (IEEE doubles) and checks it bitwise against the
reference's own pairwise_sum for many lengths — so the algorithm is proven
on CPU before it runs on the GPU. It also checks the host launch planning
(leaf depth) mirrors qfb_api.cpp:leaf_depth.
"""
import numpy as np
import pytest

LEAF_MAX = 16
GROUPS_LOG = 8


def leaf_depth(n):
    d = 0
    while ((n + (1 << d) - 1) >> d) > LEAF_MAX:
        d += 1
    return d


def descend(lo, m, path, levels):
    for lvl in range(levels - 1, -1, -1):
        h = m >> 1
        if (path >> lvl) & 1:
            lo += h
            m -= h
        else:
            m = h
    return lo, m


def fold(a, start, length):
    acc = 0.0
    for k in range(length):
        acc = acc + a[start + k]
    return acc


def butterfly(vals):
    """xor butterfly over a power-of-two lane count; returns lane 0."""
    v = list(vals)
    lanes = len(v)
    off = 1
    while off < lanes:
        v = [v[i] + v[i ^ off] for i in range(lanes)]
        off <<= 1
    return v[0]


def device_schedule_sum(a):
    n = len(a)
    D = leaf_depth(n)
    g = min(D, GROUPS_LOG)
    tps_log = D - g
    partials = []
    for t in range(1 << tps_log):
        lo, m = descend(0, n, t, tps_log)
        assert m <= LEAF_MAX << GROUPS_LOG
        leaves = []
        for i in range(1 << g):
            glo, gm = descend(lo, m, i, g)
            assert gm <= LEAF_MAX
            if gm <= 8:
                leaves.append(fold(a, glo, gm))
            else:
                h = gm >> 1
                leaves.append(fold(a, glo, h) + fold(a, glo + h, gm - h))
        partials.append(butterfly(leaves))
    if len(partials) == 1:
        return partials[0]
    # finisher warp: each lane tree-reduces `per` consecutive partials, then butterfly
    lanes = min(len(partials), 32)
    per = len(partials) // lanes
    sub = []
    for i in range(lanes):
        chunk = partials[i * per:(i + 1) * per]
        while len(chunk) > 1:
            chunk = [chunk[2 * k] + chunk[2 * k + 1] for k in range(len(chunk) // 2)]
        sub.append(chunk[0])
    return butterfly(sub)


def reference_pairwise(a, lo=0, n=None):
    n = len(a) if n is None else n
    if n <= 8:
        return fold(a, lo, n)
    h = n // 2
    return reference_pairwise(a, lo, h) + reference_pairwise(a, lo + h, n - h)


LENGTHS = list(range(1, 300)) + [511, 512, 513, 1023, 4095, 4096, 4097, 4100, 8191, 8193,
                                 12345, 65536, 65537, 99991]


@pytest.mark.parametrize("chunk", range(4))
def test_schedule_matches_pairwise_tree(orc, chunk):
    rng = np.random.default_rng(100 + chunk)
    for n in LENGTHS[chunk::4]:
        a = (rng.normal(0, 1, n) * np.exp(rng.uniform(-30, 30, n))).tolist()
        got = device_schedule_sum(a)
        want = orc.pairwise_sum(np.array(a))
        assert got == want or (np.isnan(got) and np.isnan(want)), n


def test_schedule_large_rows(orc):
    # config-sized rows: [128,120,160] per-tensor and a 76,800 HW row
    rng = np.random.default_rng(7)
    for n in (76_800, 19_200, 307_200):
        a = rng.normal(0, 1, n).tolist()
        assert device_schedule_sum(a) == orc.pairwise_sum(np.array(a))


def test_leaf_groups_cover_row_exactly():
    for n in [1, 2, 9, 16, 17, 33, 4096, 4097, 100_000]:
        D = leaf_depth(n)
        covered = 0
        for j in range(1 << D):
            lo, m = descend(0, n, j, D)
            assert lo == covered and 0 <= m <= LEAF_MAX
            covered += m
        assert covered == n
