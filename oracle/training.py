"""Scalar training machinery of arXiv 1410.7455, section 3 and C.3 (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import math
from typing import Sequence

import numpy as np


def lr_at(samples_seen: float, total_samples: float, lr_initial: float = 0.01,
          lr_final: float = 0.001) -> float:
    """Exponential schedule, 3.2.1: 'decreases by a factor of 10 during
    training, on an exponential schedule ... starts at 0.01 and ends at 0.001'.
    Reading R17: per minibatch, lr_t = lr0 (lr_end/lr0)^(samples_seen/total)."""
    return lr_initial * (lr_final / lr_initial) ** (float(samples_seen) / float(total_samples))


def job_learning_rate(effective_lr: float, n_jobs: int) -> float:
    """3.1: the per-job rate is the effective rate times the number of jobs."""
    return effective_lr * n_jobs


def max_change_bound(lr: float, gamma_x: float, gamma_y: float,
                     p_x: np.ndarray, p_y: np.ndarray) -> float:
    """eqn:delta_t_approx on the preconditioned rows:
    sum_i lr ||x_bar_i|| ||y_bar_i|| with ||x_bar_i|| = gamma_x sqrt(p_i).
    ``p_x``/``p_y`` are the UNSCALED p_i = ||x_hat_i||^2."""
    return float(lr * gamma_x * gamma_y * np.sum(np.sqrt(p_x * p_y)))


def max_change_scale(bound: float, n: int, max_change_per_sample: float = 0.075) -> float:
    """C.3: alpha_t = min(1, N * max_change_per_sample / bound);
    alpha_t = 1 when the bound is 0 (reading R16)."""
    limit = n * max_change_per_sample
    if bound <= 0.0:
        return 1.0
    return min(1.0, limit / bound)


def tree_sum(values, dtype=np.float64):
    """Fixed pairwise (binary-tree) order over rank index: level by level,
    s[k] <- s[2k] + s[2k+1] (an unpaired last element is carried up unchanged).
    For n = 8: ((x0 + x1) + (x2 + x3)) + ((x4 + x5) + (x6 + x7))."""
    s = [np.asarray(v, dtype=dtype) for v in values]
    while len(s) > 1:
        s = [(s[k] + s[k + 1]).astype(dtype) if k + 1 < len(s) else s[k]
             for k in range(0, len(s), 2)]
    return s[0]


def average_models(models: Sequence[Sequence[np.ndarray]], dtype=np.float64):
    """3.1 'average the parameters across all the jobs': unweighted mean
    (reading R18) W = tree_sum(W^0..W^{n-1}) * (1/n) in a fixed pairwise order, so the
    result is deterministic and n identical models give back the model bit-exactly for
    n a power of two.  ``dtype`` selects the arithmetic precision (float32
    reproduces the GPU arithmetic)."""
    n = len(models)
    inv = dtype(1.0) / dtype(n)
    out = []
    for layer in range(len(models[0])):
        acc = tree_sum([m[layer] for m in models], dtype)
        out.append((acc * inv).astype(dtype))
    return out
