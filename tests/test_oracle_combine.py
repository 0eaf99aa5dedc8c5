"""Pins for oracle/combine.py (C.4).  CPU only."""
import numpy as np
import pytest

from oracle import combine, nnet
from synth import gaussian_rows, labels_uniform, standard_normals

CFG = nnet.NnetConfig(input_dim=6, num_hidden=1, hidden_dim=12, pnorm_group=3, num_classes=4, renorm=True)


def _models(P, seed):
    ms = []
    for p in range(P):
        ps = nnet.init_params(CFG, standard_normals(seed + p, CFG.layer_shapes()))
        ps[-1] = 0.3 * standard_normals(seed + 100 + p, [CFG.layer_shapes()[-1]])[0]
        ms.append(ps)
    return ms


def _batches():
    return [(gaussian_rows(1, 20, 6), labels_uniform(2, 20, 4)), (gaussian_rows(3, 15, 6), labels_uniform(4, 15, 4))]


def test_single_model_weights_reproduce_it():
    ms = _models(3, 10)
    w = np.zeros((2, 3))
    w[:, 1] = 1.0
    for a, b in zip(combine.combine(ms, w), ms[1]):
        assert np.array_equal(a, b)


def test_gradient_matches_finite_differences():
    """d obj / d w by central differences (h = 1e-6, relative 1e-5)."""
    ms, bt = _models(3, 20), _batches()
    w = np.random.default_rng(0).uniform(0.1, 0.6, size=(2, 3))
    _, g = combine.objective_and_grad(ms, w, CFG, bt)
    h = 1e-6
    for idx in np.ndindex(w.shape):
        wp, wm = w.copy(), w.copy()
        wp[idx] += h
        wm[idx] -= h
        num = (combine.objective_and_grad(ms, wp, CFG, bt)[0] - combine.objective_and_grad(ms, wm, CFG, bt)[0]) / (2 * h)
        assert num == pytest.approx(g[idx], rel=1e-5, abs=1e-7)


def test_lbfgs_never_worse_than_start_and_reaches_stationarity():
    ms, bt = _models(3, 30), _batches()
    w0, objs = combine.starting_point(ms, CFG, bt)
    w, obj = combine.combine_lbfgs(ms, CFG, bt, iters=50)
    assert obj >= max(objs) - 1e-9
    _, g = combine.objective_and_grad(ms, w, CFG, bt)
    assert np.max(np.abs(g)) <= 1e-3 * max(1.0, abs(obj))
