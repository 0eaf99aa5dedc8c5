"""p-norm / softmax DNN and the preconditioned minibatch step of arXiv 1410.7455 (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Problem (section 2): frames x in R^D, labels y, maximise sum_i log p(y_i|x_i).
Affine layers carry the bias as the last column of W with a 1 appended to the input
(P:281-283).  Hidden nonlinearity: p-norm with p = 2 over contiguous groups of G
(reading R19).  Optionally (``renorm=True``, reading R32) each
p-norm layer is followed by the renormalisation layer the paper's networks carry
("renormalization layers that follow each p-norm layer"): y = s a with
s = sqrt(D / ||a||^2), i.e. every row rescaled to unit root-mean-square (s = 0 for an
all-zero row).  Gradients are summed
over the minibatch, not averaged.  Backprop of all layers uses
the pre-update weights, then every layer is updated (reading R21).
"""
from __future__ import annotations

import dataclasses
from typing import List, Sequence

import numpy as np

from . import online_ng, simple_ng, training


@dataclasses.dataclass
class NnetConfig:
    input_dim: int
    num_hidden: int
    hidden_dim: int          # p-norm input dimension (e.g. 3000)
    pnorm_group: int         # G (e.g. 10): p-norm output dimension = hidden_dim / G
    num_classes: int
    renorm: bool = False     # renormalisation layer after each p-norm layer (R32)

    @property
    def pnorm_dim(self) -> int:
        return self.hidden_dim // self.pnorm_group

    def layer_shapes(self) -> List[tuple]:
        """(D_out, D_in + 1) per weight matrix, bias column included."""
        shapes = []
        d_in = self.input_dim
        for _ in range(self.num_hidden):
            shapes.append((self.hidden_dim, d_in + 1))
            d_in = self.pnorm_dim
        shapes.append((self.num_classes, d_in + 1))
        return shapes


def init_params(cfg: NnetConfig, normals: Sequence[np.ndarray]) -> List[np.ndarray]:
    """C.6: weights with standard deviation 1/sqrt(fan-in) (reading R20:
    fan-in counts the bias column); softmax layer initialised to zero.  The standard
    normal draws are passed in (``normals[l]`` has the layer's shape)."""
    params = []
    shapes = cfg.layer_shapes()
    for l, (d_out, d_in1) in enumerate(shapes):
        if l == len(shapes) - 1:
            params.append(np.zeros((d_out, d_in1)))
        else:
            params.append(np.asarray(normals[l], dtype=np.float64) / np.sqrt(d_in1))
    return params


def append_one(a: np.ndarray) -> np.ndarray:
    """[a; 1]."""
    return np.concatenate([a, np.ones((a.shape[0], 1))], axis=1)


def pnorm(z: np.ndarray, group: int) -> np.ndarray:
    """p-norm, p = 2: a_j = (sum_{k in group j} z_k^2)^{1/2}."""
    n, d = z.shape
    return np.sqrt(np.sum((z * z).reshape(n, d // group, group), axis=2))


def renorm_scale(a: np.ndarray) -> np.ndarray:
    """Per-row scale of the renormalisation layer (reading R32):
    s = sqrt(D / ||a||^2) so that y = s a has unit root-mean-square; s = 0 if a = 0."""
    ss = np.sum(a * a, axis=1, keepdims=True)
    with np.errstate(divide="ignore"):
        return np.where(ss > 0.0, np.sqrt(a.shape[1] / np.where(ss > 0.0, ss, 1.0)), 0.0)


def log_softmax(z: np.ndarray) -> np.ndarray:
    """log p(y|x) = z_y - log sum_k exp z_k."""
    m = np.max(z, axis=1, keepdims=True)
    return z - m - np.log(np.sum(np.exp(z - m), axis=1, keepdims=True))


@dataclasses.dataclass
class ForwardBackward:
    Y: List[np.ndarray]        # per weight matrix: input with the 1-column, N x (D_in + 1)
    S: List[np.ndarray]        # per hidden layer: renormalisation scale s (N x 1), or None
    Z: List[np.ndarray]        # per weight matrix: output, N x D_out
    X: List[np.ndarray]        # per weight matrix: derivative of objective w.r.t. Z
    objective: float
    logp: np.ndarray


def forward(params: Sequence[np.ndarray], cfg: NnetConfig, frames: np.ndarray):
    """Forward pass; returns (Y list, Z list, S list, log-probs)."""
    Y, Z, S = [], [], []
    a = np.asarray(frames, dtype=np.float64)
    for l, W in enumerate(params):
        y = append_one(a)
        z = y @ W.T                                            # z = W [a; 1]
        Y.append(y)
        Z.append(z)
        if l < len(params) - 1:
            a = pnorm(z, cfg.pnorm_group)
            if cfg.renorm:
                s = renorm_scale(a)
                a = s * a                                      # unit-RMS rows
                S.append(s)
            else:
                S.append(None)
    return Y, Z, S, log_softmax(Z[-1])


def forward_backward(params: Sequence[np.ndarray], cfg: NnetConfig, frames: np.ndarray,
                     labels: np.ndarray) -> ForwardBackward:
    """Objective sum_i log p(y_i|x_i) and, for every weight matrix, the
    derivative X_i w.r.t. its output and its input Y_i."""
    labels = np.asarray(labels)
    Y, Z, S, logp = forward(params, cfg, frames)
    N = logp.shape[0]
    if np.any(labels < 0) or np.any(labels >= cfg.num_classes):
        raise ValueError("label out of range")
    objective = float(np.sum(logp[np.arange(N), labels]))
    L = len(params)
    X = [None] * L
    onehot = np.zeros_like(logp)
    onehot[np.arange(N), labels] = 1.0
    X[L - 1] = onehot - np.exp(logp)                           # d obj / d z_L
    G = cfg.pnorm_group
    for l in range(L - 1, 0, -1):
        W = params[l]
        g = X[l] @ W[:, :-1]                                   # d obj / d a_{l-1} (bias col excluded)
        z = Z[l - 1]
        a = Y[l][:, :-1]
        s = S[l - 1]
        if s is not None:
            # renormalisation backward: y = s a, s = sqrt(D/||a||^2) =>
            # d obj / d a = s (g - y (y^T g) / D)
            g = s * (g - a * np.sum(a * g, axis=1, keepdims=True) / a.shape[1])
            with np.errstate(divide="ignore", invalid="ignore"):
                a = np.where(s > 0.0, a / np.where(s > 0.0, s, 1.0), 0.0)   # the p-norm output
        a_rep = np.repeat(a, G, axis=1)
        g_rep = np.repeat(g, G, axis=1)
        with np.errstate(divide="ignore", invalid="ignore"):
            X[l - 1] = np.where(a_rep > 0.0, g_rep * z / a_rep, 0.0)   # d a_j / d z_k = z_k / a_j
    return ForwardBackward(Y, S, Z, X, objective, logp)


@dataclasses.dataclass
class LayerStats:
    alpha_t: float
    gamma_in: float
    gamma_out: float
    bound: float
    updated_in: bool
    updated_out: bool
    flags_in: tuple = (False, False, False)    # (floored, reorth_checked, reorthogonalized), B.3.1
    flags_out: tuple = (False, False, False)
    margins_in: tuple = (0.0, 0.0)             # (floor_margin, cond_c) of the update, if any
    margins_out: tuple = (0.0, 0.0)


def make_states(cfg: NnetConfig, ng_in: online_ng.OnlineNgConfig, ng_out: online_ng.OnlineNgConfig):
    """2I states, one per side per weight matrix."""
    states = []
    for d_out, d_in1 in cfg.layer_shapes():
        states.append((online_ng.OnlineNgState(d_in1, dataclasses.replace(ng_in)),
                       online_ng.OnlineNgState(d_out, dataclasses.replace(ng_out))))
    return states


def update(params: List[np.ndarray], fb: ForwardBackward, lr: float, states=None,
           precond: str = "online", max_change_per_sample: float = 0.075) -> List[LayerStats]:
    """Preconditioned minibatch update, in place on ``params``.

    For each weight matrix: X_bar = gamma_x X_hat = NG_A(X), Y_bar = gamma_y Y_hat =
    NG_B(Y); alpha_t from the preconditioned row norms (C.3,
    P:1517-1541); W += alpha_t lr X_bar^T Y_bar (eqn:add:w P:1507-1508).
    precond: 'online' (Appendix B), 'simple' (Appendix A) or 'none' (plain SGD).
    """
    stats = []
    for l in range(len(params)):
        X, Y = fb.X[l], fb.Y[l]
        N = X.shape[0]
        upd_in = upd_out = False
        fl_in = fl_out = (False, False, False)
        mg_in = mg_out = (0.0, 0.0)
        if precond == "online":
            s_in, s_out = states[l]
            ox = online_ng.precondition(s_out, X)
            oy = online_ng.precondition(s_in, Y)
            x_hat, gx, px = ox.x_hat, ox.gamma, ox.row_sq / (ox.gamma ** 2)
            y_hat, gy, py = oy.x_hat, oy.gamma, oy.row_sq / (oy.gamma ** 2)
            upd_in, upd_out = oy.updated, ox.updated
            fl_in = (oy.floored, oy.reorth_checked, oy.reorthogonalized)
            fl_out = (ox.floored, ox.reorth_checked, ox.reorthogonalized)
            mg_in, mg_out = (oy.floor_margin, oy.cond_c), (ox.floor_margin, ox.cond_c)
        elif precond == "simple":
            x_hat, gx, _ = simple_ng.precondition_simple(X)
            y_hat, gy, _ = simple_ng.precondition_simple(Y)
            px, py = np.sum(x_hat * x_hat, axis=1), np.sum(y_hat * y_hat, axis=1)
            gx = gy = 1.0
        elif precond == "none":
            x_hat, y_hat, gx, gy = X, Y, 1.0, 1.0
            px, py = np.sum(X * X, axis=1), np.sum(Y * Y, axis=1)
        else:
            raise ValueError(precond)
        bound = training.max_change_bound(lr, gx, gy, px, py)
        alpha_t = training.max_change_scale(bound, N, max_change_per_sample)
        params[l] += (alpha_t * lr * gx * gy) * (x_hat.T @ y_hat)
        stats.append(LayerStats(alpha_t, gy, gx, bound, upd_in, upd_out, fl_in, fl_out, mg_in, mg_out))
    return stats


def train_step(params, cfg, frames, labels, lr, states=None, precond="online",
               max_change_per_sample=0.075):
    """One minibatch: forward/backward with the old weights, then update all layers."""
    fb = forward_backward(params, cfg, frames, labels)
    stats = update(params, fb, lr, states, precond, max_change_per_sample)
    return fb.objective, stats
