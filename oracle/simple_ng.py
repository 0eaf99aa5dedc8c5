"""Simple natural-gradient preconditioner, Appendix A of arXiv 1410.7455 (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

``precondition_simple``      -- the efficient computation of A.3.
``precondition_simple_brute``-- the definition of A.2: one explicit
                                 held-out D x D inverse per row.
Reading R1: G_i = beta I + (1/(N-1)) sum_{j != i} x_j x_j^T and x_hat_i = G_i^{-1} x_i
(P:815-819 writes the inverse twice; the efficient section fixes the intent).
"""
from __future__ import annotations

import math

import numpy as np

SIMPLE_EPSILON = 1e-20   # P:430, P:811 (reading R9)


def simple_beta(X: np.ndarray, alpha: float = 4.0, epsilon: float = SIMPLE_EPSILON) -> float:
    """beta = alpha max(tr(X^T X), eps) / (N D)."""
    N, D = X.shape
    return alpha * max(float(np.sum(X * X)), epsilon) / (N * D)


def _gamma(X: np.ndarray, X_hat: np.ndarray) -> float:
    """gamma = sqrt(tr(X^T X) / tr(X_hat^T X_hat)), 1 if the denominator is 0."""
    den = float(np.sum(X_hat * X_hat))
    return math.sqrt(float(np.sum(X * X)) / den) if den > 0.0 else 1.0


def precondition_simple(X: np.ndarray, alpha: float = 4.0, epsilon: float = SIMPLE_EPSILON,
                        branch: str | None = None):
    """Efficient simple NG (A.3).  Returns (X_bar, gamma, row_sq=||x_bar_i||^2).

    G = beta I + X^T X / (N-1).  Q = X G^{-1} in column space if N > D,
    else Q = (beta I + X X^T/(N-1))^{-1} X in row space (strict N > D,
    reading R11).  a_i = x_i^T q_i, b_i = 1 + a_i/(N-1-a_i),
    x_hat_i = b_i q_i, X_bar = gamma X_hat.
    """
    X = np.asarray(X, dtype=np.float64)
    N, D = X.shape
    if N < 2:
        raise ValueError("simple NG needs N >= 2 (hold-out needs another row)")
    beta = simple_beta(X, alpha, epsilon)
    if branch is None:
        branch = "column" if N > D else "row"
    if branch == "column":
        G = beta * np.eye(D) + (X.T @ X) / (N - 1)
        Q = np.linalg.solve(G, X.T).T                          # X G^{-1}, G symmetric
    else:
        Gr = beta * np.eye(N) + (X @ X.T) / (N - 1)
        Q = np.linalg.solve(Gr, X)
    a = np.sum(X * Q, axis=1)
    b = 1.0 + a / (N - 1 - a)
    X_hat = b[:, None] * Q
    gamma = _gamma(X, X_hat)
    X_bar = gamma * X_hat
    return X_bar, gamma, np.sum(X_bar * X_bar, axis=1)


def precondition_simple_brute(X: np.ndarray, alpha: float = 4.0, epsilon: float = SIMPLE_EPSILON):
    """Definition A.2: per-row held-out G_i formed and inverted explicitly."""
    X = np.asarray(X, dtype=np.float64)
    N, D = X.shape
    if N < 2:
        raise ValueError("simple NG needs N >= 2")
    beta = simple_beta(X, alpha, epsilon)
    X_hat = np.empty_like(X)
    for i in range(N):
        Gi = beta * np.eye(D)
        for j in range(N):
            if j != i:
                Gi += np.outer(X[j], X[j]) / (N - 1)
        X_hat[i] = np.linalg.inv(Gi) @ X[i]
    gamma = _gamma(X, X_hat)
    X_bar = gamma * X_hat
    return X_bar, gamma, np.sum(X_bar * X_bar, axis=1)
