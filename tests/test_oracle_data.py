"""Pins for oracle/data.py (C.2): the 1-byte compression (reading R36) and
the N x M block randomisation.  CPU only."""
import numpy as np
import pytest

from oracle import data


def test_compression_error_bound_and_endpoints():
    """|x~ - x| <= step/2 (+ float32 rounding); the column min and max are exact codes 0 and
    255; a constant column decodes exactly (step 0)."""
    rng = np.random.default_rng(0)
    X = (rng.normal(size=(300, 40)) * rng.uniform(0.01, 100, 40)).astype(np.float32)
    X[:, 7] = 3.25
    q, lo, step = data.compress(X)
    assert q.dtype == np.uint8 and q.shape == X.shape
    Xt = data.decompress(q, lo, step)
    err = np.abs(Xt.astype(np.float64) - X.astype(np.float64))
    assert np.all(err <= step[None, :] / 2 + 1e-6 * np.abs(X) + 1e-30)
    assert np.all(Xt[:, 7] == 3.25) and np.all(q[:, 7] == 0)
    for c in range(40):
        if c == 7:
            continue
        assert q[np.argmin(X[:, c]), c] == 0 and q[np.argmax(X[:, c]), c] == 255


def test_compression_is_the_nearest_code():
    """Brute force on a small case: each code is the nearest of the 256 levels."""
    rng = np.random.default_rng(1)
    X = rng.uniform(-2, 5, size=(50, 3)).astype(np.float32)
    q, lo, step = data.compress(X)
    levels = lo[None, :] + step[None, :] * np.arange(256)[:, None]        # [256, D]
    best = np.argmin(np.abs(X.astype(np.float64)[:, None, :] - levels[None, :, :]), axis=1)
    assert np.all(np.abs(best.astype(int) - q.astype(int)) <= 1)
    assert np.mean(best == q) > 0.98                                         # ties only


@pytest.mark.parametrize("F,N,K", [(10_000, 1, 400), (100_003, 4, 3000), (262_144, 8, 32_768), (50, 6, 1000)])
def test_block_randomize_partition(F, N, K):
    blocks = data.block_randomize(F, N, K, seed=7)
    M = data.outer_iterations_per_epoch(F, N, K)
    assert len(blocks) == N and all(len(b) == M for b in blocks)
    allidx = np.concatenate([blk for row in blocks for blk in row])
    assert np.array_equal(np.sort(allidx), np.arange(F))                     # disjoint cover
    sizes = [len(blk) for row in blocks for blk in row]
    assert max(sizes) - min(sizes) <= 1
    if F >= N * K:                                                             # M per the K target
        assert abs(F / (N * M) - K) <= abs(F / (N * (M + 1)) - K) + 1e-9
        assert abs(F / (N * M) - K) <= abs(F / (N * max(M - 1, 1)) - K) + 1e-9


def test_block_randomize_deterministic_and_random_order():
    a = data.block_randomize(1000, 2, 100, seed=3)
    b = data.block_randomize(1000, 2, 100, seed=3)
    c = data.block_randomize(1000, 2, 100, seed=4)
    assert all(np.array_equal(x, y) for ra, rb in zip(a, b) for x, y in zip(ra, rb))
    assert not all(np.array_equal(x, y) for ra, rc in zip(a, c) for x, y in zip(ra, rc))
    assert not np.all(np.diff(a[0][0]) > 0)                                   # randomised inside a block
