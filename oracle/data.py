"""Input side of the training step (C.2) (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

* ``compress`` / ``decompress`` -- "we compress the features on disk to 1 byte per float,
  using a lossy compression method".  The paper gives no format; reading R36:
  per column c, lo = min_r x[r, c], step = (max_r x[r, c] - lo) / 255 (float64 from the
  float32 data), q = clip(round_half_even((x - lo) / step), 0, 255) (0 where step = 0), and
  x~ = float32(lo + step q).  So |x~ - x| <= step / 2 (+ float32 rounding).
* ``block_randomize`` -- the N x M blocks of C.2: N jobs, M outer iterations
  per epoch with M chosen so the samples per job per outer iteration are close to K, the
  data randomly distributed into the N M blocks in a random order inside each block, the
  same order every epoch; job n processes block (n, m) on outer iteration m.
"""
from __future__ import annotations

import numpy as np


def compress(X: np.ndarray):
    """1 byte per float (R36): returns (q uint8 [n, D], lo float64 [D], step float64 [D])."""
    X = np.asarray(X, dtype=np.float32).astype(np.float64)
    lo = X.min(axis=0)
    hi = X.max(axis=0)
    step = (hi - lo) / 255.0
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.where(step > 0.0, (X - lo) / np.where(step > 0.0, step, 1.0), 0.0)
    q = np.clip(np.rint(t), 0, 255).astype(np.uint8)          # rint: round half to even
    return q, lo, step


def decompress(q: np.ndarray, lo: np.ndarray, step: np.ndarray) -> np.ndarray:
    """x~ = float32(lo + step q) (R36)."""
    return (lo[None, :] + step[None, :] * q.astype(np.float64)).astype(np.float32)


def outer_iterations_per_epoch(num_examples: int, n_jobs: int, k_samples: int) -> int:
    """M >= 1 with num_examples / (N M) closest to K."""
    return max(1, int(round(num_examples / float(n_jobs * k_samples))))


def block_randomize(num_examples: int, n_jobs: int, k_samples: int, seed: int):
    """blocks[n][m]: example indices of block (n, m), disjoint, covering every example once,
    sizes differing by at most one, each in a random order."""
    M = outer_iterations_per_epoch(num_examples, n_jobs, k_samples)
    perm = np.random.default_rng(seed).permutation(num_examples)
    chunks = np.array_split(perm, n_jobs * M)
    return [[chunks[m * n_jobs + n] for m in range(M)] for n in range(n_jobs)]
