"""CPU checks of the exact Gram-gradient accumulator format (fixed-point int64
limbs, sk_common.cuh FixAcc) through its numpy restatement tests/fixpt_ref.py:
exact and order-independent sums, lossless round trip, integer merging of
partial accumulators (what gram_dist's all-reduce does across GPUs)."""

import math

import numpy as np
import pytest

import fixpt_ref as fx


def _values(rng, n):
    mags = 10.0 ** rng.uniform(-12, 3, n)
    return rng.standard_normal(n) * mags


def test_round_trip_is_lossless():
    """Values whose 53-bit mantissa lies above the lowest limb's unit 2^(E-168)
    come back exactly; smaller ones are rounded to that unit."""
    rng = np.random.default_rng(0)
    E = fx.anchor(1.0, 1024.0)
    for v in _values(rng, 500):
        acc = np.zeros((1, 4), dtype=np.int64)
        fx.accumulate(acc, [v], E)
        got = fx.finalize(acc, E)[0]
        if abs(v) >= 2.0 ** (E - 168 + 53):
            assert got == v
        else:
            assert abs(got - v) <= 2.0 ** (E - 168)


def test_sum_is_order_independent_and_correctly_rounded():
    rng = np.random.default_rng(1)
    vals = _values(rng, 2000)
    E = fx.anchor(1.0, 4096.0)
    results = set()
    for seed in range(5):
        order = np.random.default_rng(seed).permutation(len(vals))
        acc = np.zeros((1, 4), dtype=np.int64)
        for i in order:
            fx.accumulate(acc, [vals[i]], E)
        results.add(float(fx.finalize(acc, E)[0]))
    assert len(results) == 1
    got = results.pop()
    want = math.fsum(vals)
    assert abs(got - want) <= 2 * math.ulp(want)


def test_partial_accumulators_merge_as_integers():
    """Two ranks' limbs added as int64 == one accumulator over all terms (bitwise)."""
    rng = np.random.default_rng(2)
    vals = _values(rng, 64 * 3).reshape(3, 64)
    E = fx.anchor(2.0, 100.0)
    one = np.zeros((64, 4), dtype=np.int64)
    for row in vals:
        fx.accumulate(one, row, E)
    r0 = np.zeros((64, 4), dtype=np.int64)
    r1 = np.zeros((64, 4), dtype=np.int64)
    fx.accumulate(r0, vals[0], E)
    fx.accumulate(r1, vals[1], E)
    fx.accumulate(r1, vals[2], E)
    np.testing.assert_array_equal(fx.finalize(r0 + r1, E), fx.finalize(one, E))


def test_range_guard():
    E = fx.anchor(1.0, 8.0)
    with pytest.raises(OverflowError):
        fx.to_limbs(2.0 ** (E + 3), E)
    assert fx.to_limbs(0.0, E) == (0, 0, 0, 0)
