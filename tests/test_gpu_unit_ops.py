"""Batched unit kernels: SPEC acceptance criteria 1 (frequency formula grid)
and 2 (router oracle over 10,000 random usage vectors), plus service time,
the agent-tick min reduction, and the scalar API mirror."""

import math

import numpy as np
import pytest

import paper_2604_16682_b200 as asb
from paper_2604_16682_b200 import ops

pytestmark = pytest.mark.gpu


def test_ac1_frequency_formula_grid(cuda_device):
    """usage in {0..capacity} at 10,001 points x L in 2..16 x alpha in {.5,.75,1}: exact + monotone."""
    capacity = 123_457
    usage = np.unique(np.linspace(0, capacity, 10_001).round().astype(np.int64))
    for L in range(2, 17):
        for alpha in (0.5, 0.75, 1.0):
            n = usage.size
            got = ops.select_level_batch(usage, np.full(n, capacity), np.full(n, L), np.full(n, alpha))
            want = np.array([L if u >= alpha * capacity else math.floor(u / (alpha * capacity) * (L - 1)) + 1
                             for u in usage.tolist()])
            assert np.array_equal(got, want)
            assert (np.diff(got) >= 0).all() and got.min() >= 1 and got.max() <= L


def test_select_level_takes_float_usage(cuda_device):
    """The reference's signature takes floats (controller.py:81): fractional
    usage and capacity are not truncated."""
    rng = np.random.default_rng(4)
    n = 20_000
    usage = rng.uniform(0, 2.0, n)
    cap = rng.uniform(0.1, 1.5, n)
    L = rng.integers(2, 17, n)
    alpha = rng.choice([0.5, 0.75, 1.0], n)
    got = ops.select_level_batch(usage, cap, L, alpha)
    want = [asb.select_frequency_level(u, c, int(lv), a) for u, c, lv, a in zip(usage, cap, L, alpha)]
    assert got.tolist() == want
    assert ops.select_level_batch([0.5], [1.0], [4], [0.75])[0] == 3


def oracle_assign(usages, capacity, theta):
    light = [i for i in range(1, len(usages) + 1) if usages[i - 1] < theta * capacity]
    if light:
        return min(light)
    return min(range(1, len(usages) + 1), key=lambda i: (usages[i - 1], i))


def oracle_reassign(counter, current, usages, interval, ratio):
    counter += 1
    if counter < interval:
        return counter, 0
    j = min(range(1, len(usages) + 1), key=lambda i: (usages[i - 1], i))
    target = j if j != current and usages[current - 1] >= ratio * usages[j - 1] else 0
    return 0, target


def test_ac2_router_oracle_10k_vectors(cuda_device):
    rng = np.random.default_rng(5)
    capacity = 100_000.0
    rows, cur, ctr = [], [], []
    for _ in range(10_000):
        n = int(rng.integers(4, 17))
        rows.append(rng.uniform(1.0, capacity, size=n).tolist())
        cur.append(int(rng.integers(1, n + 1)))
        ctr.append(int(rng.integers(0, 10)))
    got = ops.assign_batch(rows, capacity, 0.5, "context_aware")
    want = [oracle_assign(r, capacity, 0.5) for r in rows]
    assert got.tolist() == want
    tgt, new_ctr = ops.reassign_batch(rows, cur, ctr, 8, 2.0, True, False)
    exp = [oracle_reassign(c, k, r, 8, 2.0) for r, k, c in zip(rows, cur, ctr)]
    assert new_ctr.tolist() == [e[0] for e in exp]
    assert tgt.tolist() == [e[1] for e in exp]
    ll = ops.assign_batch(rows, capacity, 0.5, "least_loaded")
    assert ll.tolist() == [min(range(1, len(r) + 1), key=lambda i: (r[i - 1], i)) for r in rows]


def test_service_time_matches_reference_arithmetic(cuda_device):
    rng = np.random.default_rng(1)
    n = 20_000
    p = rng.integers(1, 32768, n)
    d = rng.integers(1, 8192, n)
    pr = rng.uniform(1000, 20000, n)
    dr = rng.uniform(10, 80, n)
    c = rng.integers(1, 9, n)
    th = rng.integers(0, 2, n)
    got = ops.service_time_batch(p, d, pr, dr, c, th, 0.1, 3.0)
    want = []
    for i in range(n):
        base = int(p[i]) / float(pr[i]) + int(d[i]) / float(dr[i])
        f = 1.0 + 0.1 * max(0, int(c[i]) - 1)
        if th[i]:
            f *= 3.0
        want.append(base * f)
    assert np.array_equal(got, np.array(want))


def test_min_throughput_reduction(cuda_device):
    rng = np.random.default_rng(2)
    n = 50_000
    dec = rng.integers(0, 10_000, n)
    llm = np.where(rng.random(n) < 0.2, 0.0, rng.uniform(0.1, 500, n))
    seg = rng.integers(0, 16, n)
    got = ops.min_throughput_batch(dec, llm, seg, 17)
    for s in range(17):
        vals = [int(dec[i]) / float(llm[i]) for i in np.nonzero((seg == s) & (llm > 0))[0]]
        if vals:
            assert got[s] == min(vals)
        else:
            assert math.isnan(got[s])
