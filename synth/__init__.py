"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no preconditioning, no network
maths): only random draws shaped like the paper's workloads.  Both sides receive the
same arrays; random numbers the method itself needs (weight init) are drawn here and
passed in.  Recipes are documented in DESIGN.md ("Synthetic inputs").

* ``spliced_frames``   -- speech-like frames: per "utterance" a sticky Markov chain of
  class labels (Zipf(1) prior, mean dwell 8 frames), 40-dim base vectors = class mean
  (N(0, 0.5^2 I)) + unit-variance AR(1) noise (coefficient 0.9), spliced +-4 frames with
  edge replication -> 360 dims (paper: +-4 spliced 40-dim features).
* ``power_law_rows``   -- rows from N(0, Q Lambda Q^T) with Lambda_kk = 1/k and a random
  orthogonal Q (config 2 out side); ``nonneg=True, append_one=True`` gives the
  activation-like in side [|.|, 1].
* ``standard_normals`` -- i.i.d. N(0,1) draws for weight initialisation.
"""
from __future__ import annotations

import numpy as np

BENCH_SEED = 1410


def rank_seed(rank: int, base: int = BENCH_SEED) -> int:
    """Per-rank seed: seed = 1410 + 7455 * rank (disjoint data shard per job)."""
    return base + 7455 * int(rank)


def _zipf_prior(num_classes: int) -> np.ndarray:
    p = 1.0 / np.arange(1, num_classes + 1, dtype=np.float64)
    return p / p.sum()


def spliced_frames(seed: int, n_frames: int, base_dim: int = 40, context: int = 4,
                   num_classes: int = 5000, dwell: float = 8.0, utt_len: int = 300,
                   dtype=np.float32):
    """Return (frames [n_frames, base_dim*(2*context+1)], labels int32 [n_frames])."""
    rng = np.random.default_rng(seed)
    n_utt = -(-n_frames // utt_len)
    means = rng.normal(0.0, 0.5, size=(num_classes, base_dim))
    prior = _zipf_prior(num_classes)
    labels = np.empty((n_utt, utt_len), dtype=np.int64)
    cur = rng.choice(num_classes, size=n_utt, p=prior)
    for t in range(utt_len):
        switch = rng.random(n_utt) < (1.0 / dwell)
        fresh = rng.choice(num_classes, size=n_utt, p=prior)
        cur = np.where(switch, fresh, cur)
        labels[:, t] = cur
    noise = np.empty((n_utt, utt_len, base_dim))
    u = rng.normal(size=(n_utt, base_dim))
    c = np.sqrt(1.0 - 0.9 ** 2)
    for t in range(utt_len):
        u = 0.9 * u + c * rng.normal(size=(n_utt, base_dim))
        noise[:, t, :] = u
    base = means[labels] + noise                                  # (n_utt, T, base_dim)
    if context > 0:
        idx = np.clip(np.arange(utt_len)[:, None] + np.arange(-context, context + 1)[None, :],
                      0, utt_len - 1)                              # edge replication
        spliced = base[:, idx, :].reshape(n_utt, utt_len, -1)
    else:
        spliced = base
    frames = spliced.reshape(n_utt * utt_len, -1)[:n_frames].astype(dtype)
    return np.ascontiguousarray(frames), labels.reshape(-1)[:n_frames].astype(np.int32)


def random_orthogonal(rng: np.random.Generator, dim: int) -> np.ndarray:
    q, r = np.linalg.qr(rng.normal(size=(dim, dim)))
    return q * np.sign(np.diag(r))[None, :]


def power_law_rows(seed: int, n_rows: int, dim: int, n_batches: int = 1, nonneg: bool = False,
                   append_one: bool = False, dtype=np.float64):
    """``n_batches`` minibatches of ``n_rows`` rows ~ N(0, Q diag(1/k) Q^T)."""
    rng = np.random.default_rng(seed)
    q = random_orthogonal(rng, dim)
    scale = 1.0 / np.sqrt(np.arange(1, dim + 1, dtype=np.float64))
    out = []
    for _ in range(n_batches):
        x = (rng.normal(size=(n_rows, dim)) * scale[None, :]) @ q.T
        if nonneg:
            x = np.abs(x)
        if append_one:
            x = np.concatenate([x, np.ones((n_rows, 1))], axis=1)
        out.append(x.astype(dtype))
    return out


def gaussian_rows(seed: int, n_rows: int, dim: int, scale: float = 1.0, dtype=np.float64):
    rng = np.random.default_rng(seed)
    return (scale * rng.normal(size=(n_rows, dim))).astype(dtype)


def standard_normals(seed: int, shapes, dtype=np.float64):
    rng = np.random.default_rng(seed)
    return [rng.normal(size=s).astype(dtype) for s in shapes]


def labels_uniform(seed: int, n: int, num_classes: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.integers(0, num_classes, size=n).astype(np.int32)
