"""The roofline byte models in bench.py against brute force on
small ranges: per-prime hit counts (multiples coprime to 6 from max(L, p^2)),
the shared-memory model and the bucket-spill hit count (with a small S so the
bucket policy engages), and the config-5 interval starts."""
import math
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


def _hits(p, L, R):
    start = max(L, p * p)
    return sum(1 for m in range(-(-start // p) * p, R, p) if m % 2 and m % 3)


@pytest.mark.parametrize("L,R", [(0, 10**5), (10**6 - 37, 10**6 + 5000), (123_456, 200_001)])
def test_smem_model_matches_brute_force(L, R):
    lo0 = L // 6 * 6
    slots = (R - lo0 + 5) // 6
    W = 2 * ((slots + 31) // 32)
    ps = [p for p in bench.small_primes(math.isqrt(R - 1)) if p >= 17]
    want = 4.0 * (2 * W + sum(min(_hits(int(p), L, R), W) for p in ps))
    assert bench.smem_bytes(L, R) == want


@pytest.mark.parametrize("L,R,S", [(10**7, 10**7 + 3 * 10**5, 64), (0, 2 * 10**6, 16),
                                   (10**5, 10**5 + 10**4, 4096)])
def test_bucket_hits_matches_brute_force(L, R, S):
    B = math.isqrt(R - 1)
    want = 0
    if B >= 8 * S:
        want = sum(_hits(int(p), L, R) for p in bench.small_primes(B) if p >= 2 * S)
    assert bench.bucket_hits(L, R, S) == want


def test_c5_starts_follow_the_survey_convention():
    Ls = bench.splitmix_starts(42, 4096, 2**32, 2**44)
    assert int(Ls[0]) == 378_761_080_469
    assert Ls.dtype == np.uint64 and bool(np.all((Ls >= 2**32) & (Ls < 2**44)))
