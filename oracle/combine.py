"""Generalised model combination at the end of training (C.4) (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Given the models of the last P outer iterations (each a list of the L weight matrices),
find per-layer weights w[l, p] (L P parameters) maximising the objective of
the combined network W_l = sum_p w[l, p] W_l^(p) on a data subset, minus a tiny
regulariser 1e-10 ||w||^2.  The optimiser is L-BFGS; the start is
the best of the P + 1 choices: each single model and the plain average.
Reading R37: the paper's Fisher-related preconditioning of the L-BFGS space (P:1569-1570,
unspecified) is omitted -- it only speeds the search up; L-BFGS here is scipy's L-BFGS-B
(a library routine used as one step).  Gradient (chain rule through W_l):
d obj / d w[l, p] = <d obj / d W_l, W_l^(p)>_F, with d obj / d W_l = X_l^T Y_l.
"""
from __future__ import annotations

import numpy as np

from . import nnet

REG = 1e-10


def combine(models, weights):
    """W_l = sum_p w[l, p] W_l^(p)."""
    L, P = weights.shape
    return [sum(weights[l, p] * models[p][l] for p in range(P)) for l in range(L)]


def objective_and_grad(models, weights, cfg, batches):
    """Objective sum_i log p(y_i|x_i) over the batches of the combined model minus
    REG ||w||^2, and its gradient w.r.t. w."""
    L, P = weights.shape
    params = combine(models, weights)
    obj = 0.0
    grad = np.zeros((L, P))
    for frames, labels in batches:
        fb = nnet.forward_backward(params, cfg, frames, labels)
        obj += fb.objective
        for l in range(L):
            G = fb.X[l].T @ fb.Y[l]
            for p in range(P):
                grad[l, p] += float(np.sum(G * models[p][l]))
    obj -= REG * float(np.sum(weights * weights))
    grad -= 2.0 * REG * weights
    return obj, grad


def starting_point(models, cfg, batches):
    """Best of the P + 1 choices: each single model, then the average."""
    P, L = len(models), len(models[0])
    cands = []
    for p in range(P):
        w = np.zeros((L, P))
        w[:, p] = 1.0
        cands.append(w)
    cands.append(np.full((L, P), 1.0 / P))
    objs = [objective_and_grad(models, w, cfg, batches)[0] for w in cands]
    return cands[int(np.argmax(objs))], objs


def combine_lbfgs(models, cfg, batches, iters: int = 20):
    """Maximise with L-BFGS from the best starting point; returns (weights, objective)."""
    from scipy.optimize import minimize
    w0, _ = starting_point(models, cfg, batches)
    shape = w0.shape

    def f(v):
        o, g = objective_and_grad(models, v.reshape(shape), cfg, batches)
        return -o, -g.ravel()

    res = minimize(f, w0.ravel(), jac=True, method="L-BFGS-B", options={"maxiter": iters})
    return res.x.reshape(shape), -float(res.fun)
