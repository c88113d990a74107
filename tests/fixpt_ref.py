"""numpy restatement of the exact Gram-gradient accumulator format
(sk_common.cuh FixAcc / fix_add, sk_capi.cu fix_finalize_kernel), used by the
CPU tests to check the format's arithmetic and the host-side exchange logic
(gram_dist) without a GPU.  Test infrastructure only."""

import math

import numpy as np

MASK = (1 << 42) - 1


def anchor(maxc, nscale):
    m = maxc * nscale
    if not (m > 0.0) or not (m < 1e300):
        return 0
    _, e = math.frexp(m)
    e += 64
    return max(-900, min(960, e))


def to_limbs(v, E):
    """One contribution -> its four chunks (c0, c1, c2, c3), exactly as fix_add."""
    v = float(v)
    if v == 0.0:
        return (0, 0, 0, 0)
    x = v * 2.0 ** (42 - E)
    if not abs(x) < 2.0 ** 44:
        raise OverflowError("contribution out of the accumulator's range")
    c3 = math.trunc(x)
    x = (x - c3) * 2.0 ** 42
    c2 = math.trunc(x)
    x = (x - c2) * 2.0 ** 42
    c1 = math.trunc(x)
    x = (x - c1) * 2.0 ** 42
    c0 = round(x)  # round half to even, as rint
    return (c0, c1, c2, c3)


def _normalize(a0, a1, a2, a3):
    a1 = a1 + (a0 >> 42)
    a0 = a0 & MASK
    a2 = a2 + (a1 >> 42)
    a1 = a1 & MASK
    a3 = a3 + (a2 >> 42)
    a2 = a2 & MASK
    return a0, a1, a2, a3


def finalize(limbs, E):
    """(..., 4) int64 limbs -> float64, as the device: carry-normalise, take the
    magnitude (negate and renormalise when negative: all four digits are then
    non-negative, so the fp64 sum has no cancellation), convert, restore the sign."""
    a = _normalize(*(limbs[..., k].astype(np.int64) for k in range(4)))
    neg = a[3] < 0
    b = _normalize(-a[0], -a[1], -a[2], -a[3])
    a0, a1, a2, a3 = (np.where(neg, bk, ak) for ak, bk in zip(a, b))
    u3, u2, u1, u0 = (math.ldexp(1.0, E - s) for s in (42, 84, 126, 168))
    v = (a3.astype(np.float64) * u3
         + (a2.astype(np.float64) * u2
            + (a1.astype(np.float64) * u1 + a0.astype(np.float64) * u0)))
    return np.where(neg, -v, v)


def accumulate(acc, values, E):
    """acc (N, 4) int64 += chunks of every element of values (N,)."""
    for i, v in enumerate(np.asarray(values, dtype=np.float64).ravel()):
        c = to_limbs(v, E)
        for k in range(4):
            acc[i, k] += c[k]
    return acc
