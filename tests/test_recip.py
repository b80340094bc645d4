"""recip_u32 (csrc/sampling.cuh): floor((2^64-1)/d) without the u64 division routine.

The splitmix draws reduce z % deg through this reciprocal (mod_by_recip), so it
must be exact for every degree.  The device function uses only IEEE-exact fp64
operations (__drcp_rn is the correctly rounded 1/d) and wrapping u64 integer
arithmetic, which numpy reproduces operation for operation; this test runs that
restatement over every d < 2^22, both ends of the range and 4M random d < 2^32,
and counts the correction steps the device loops take (bounded, small).
"""
import numpy as np


def recip_u32_restated(d: np.ndarray):
    d = d.astype(np.uint64)
    r = 1.0 / d.astype(np.float64)                       # __drcp_rn((double)d)
    q = (r * 18446744073709551616.0).astype(np.uint64)   # (uint64_t)(r * 2^64)
    full = np.uint64(0xFFFFFFFFFFFFFFFF)
    with np.errstate(over="ignore"):
        rem = (full - q * d).view(np.int64)              # wrapping u64 read as int64
        k = np.floor(rem.astype(np.float64) * r).astype(np.int64)
        q = q + k.view(np.uint64)
        rem = rem - k * d.view(np.int64)
    steps = np.zeros(len(d), dtype=np.int64)
    di = d.view(np.int64)
    for _ in range(8):
        neg = rem < 0
        big = rem >= di
        if not (neg.any() or big.any()):
            break
        steps += neg | big
        with np.errstate(over="ignore"):
            q = np.where(neg, q - np.uint64(1), np.where(big, q + np.uint64(1), q))
        rem = np.where(neg, rem + di, np.where(big, rem - di, rem))
    assert not ((rem < 0) | (rem >= di)).any()
    q = np.where(d == 1, full, q)
    return q, steps


def test_recip_exact_over_degree_range():
    rng = np.random.default_rng(0)
    d = np.concatenate([
        np.arange(1, 1 << 22, dtype=np.uint64),
        np.arange((1 << 32) - 4096, 1 << 32, dtype=np.uint64),
        rng.integers(1 << 22, 1 << 32, size=4_000_000, dtype=np.uint64),
        np.array([(1 << k) + o for k in range(1, 32) for o in (-1, 0, 1)], dtype=np.uint64),
    ])
    got, steps = recip_u32_restated(d)
    want = np.uint64(0xFFFFFFFFFFFFFFFF) // d
    assert np.array_equal(got, want)
    assert steps.max() <= 2
