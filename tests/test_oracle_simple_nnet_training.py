"""Pins for oracle/simple_ng.py, oracle/nnet.py and oracle/training.py: worked
examples (tests/golden/spec_examples.json), per-row held-out brute force, finite
differences, closed forms.  CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import nnet, online_ng, simple_ng, training
from synth import gaussian_rows, labels_uniform, standard_normals

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ---------------------------------------------------------------- simple NG (Appendix A)

def test_simple_beta_golden():
    a, b = GOLD["simple_beta"]["cases"]
    assert simple_ng.simple_beta(np.array(a["X"]), a["alpha"]) == pytest.approx(a["beta"], abs=a["tol"])
    assert simple_ng.simple_beta(np.zeros(b["zeros"]), b["alpha"]) == pytest.approx(b["beta"], abs=b["tol"])


def test_simple_worked_example():
    g = GOLD["simple_pipeline_11"]
    xb, gamma, rs = simple_ng.precondition_simple(np.array(g["X"]))
    assert gamma == pytest.approx(g["gamma"], rel=1e-14)
    assert np.allclose(xb, g["x_bar"], rtol=1e-14)
    assert np.allclose(xb / gamma, g["x_hat"], rtol=1e-14)
    z = GOLD["simple_zero"]
    xb, gamma, _ = simple_ng.precondition_simple(np.zeros(z["zeros"]))
    assert gamma == z["gamma"] and np.all(xb == 0)


def test_simple_matches_heldout_bruteforce():
    """SPEC acceptance 1: efficient (A.3) vs explicit per-row held-out inverses (A.2)."""
    rng = np.random.default_rng(0)
    for _ in range(60):
        N, D = int(rng.integers(2, 40)), int(rng.integers(1, 24))
        X = rng.normal(size=(N, D)) * rng.uniform(0.1, 10)
        a, ga, ra = simple_ng.precondition_simple(X)
        b, gb, rb = simple_ng.precondition_simple_brute(X)
        assert np.max(np.abs(a - b)) <= 1e-10 * np.max(np.abs(b))
        assert ga == pytest.approx(gb, rel=1e-10)
        assert np.linalg.norm(a) == pytest.approx(np.linalg.norm(X), rel=1e-12)


def test_simple_column_row_equivalence():
    """column-space and row-space Q agree (push-through identity)."""
    rng = np.random.default_rng(1)
    for N, D in [(5, 9), (9, 5), (12, 12), (40, 3)]:
        X = rng.normal(size=(N, D))
        a = simple_ng.precondition_simple(X, branch="column")[0]
        b = simple_ng.precondition_simple(X, branch="row")[0]
        assert np.max(np.abs(a - b)) <= 1e-10 * np.max(np.abs(a))


# ---------------------------------------------------------------- DNN (section 2, C.6)

CFG_T = nnet.NnetConfig(input_dim=6, num_hidden=2, hidden_dim=12, pnorm_group=4, num_classes=5)


def _rand_params(cfg, seed, scale=0.7):
    return [scale * w for w in standard_normals(seed, cfg.layer_shapes())]


def test_pnorm_golden():
    g = GOLD["pnorm_34"]
    assert np.allclose(nnet.pnorm(np.array(g["z"]), g["group"]), g["a"])


def test_zero_net_uniform_logprob():
    """zero network -> log p = -log C for every class."""
    params = [np.zeros(s) for s in CFG_T.layer_shapes()]
    _, _, _, logp = nnet.forward(params, CFG_T, gaussian_rows(0, 4, 6))
    assert np.allclose(logp, -np.log(5.0))


def test_softmax_rows_and_bias_gradient_at_uniform():
    """zero net, all labels identical -> final bias-column gradient = sum_i
    (onehot - 1/C)."""
    params = [np.zeros(s) for s in CFG_T.layer_shapes()]
    N = 7
    fb = nnet.forward_backward(params, CFG_T, gaussian_rows(1, N, 6), np.full(N, 2))
    grad_bias = (fb.X[-1].T @ fb.Y[-1])[:, -1]
    expect = -N / 5.0 * np.ones(5)
    expect[2] += N
    assert np.allclose(grad_bias, expect, atol=1e-12)
    assert np.allclose(np.exp(fb.logp).sum(axis=1), 1.0)


@pytest.mark.parametrize("num_hidden", [1, 2, 3])
def test_finite_difference_gradients(num_hidden):
    """SPEC acceptance 6: d objective / d W_l = X_l^T Y_l against central
    differences, h = 1e-5, relative 1e-4."""
    cfg = nnet.NnetConfig(input_dim=5, num_hidden=num_hidden, hidden_dim=8, pnorm_group=2, num_classes=4)
    params = _rand_params(cfg, 10 + num_hidden)
    frames, labels = gaussian_rows(2, 6, 5), labels_uniform(3, 6, 4)
    fb = nnet.forward_backward(params, cfg, frames, labels)
    h = 1e-5
    for l, W in enumerate(params):
        grad = fb.X[l].T @ fb.Y[l]
        num = np.zeros_like(W)
        for idx in np.ndindex(W.shape):
            old = W[idx]
            W[idx] = old + h
            fp = nnet.forward_backward(params, cfg, frames, labels).objective
            W[idx] = old - h
            fm = nnet.forward_backward(params, cfg, frames, labels).objective
            W[idx] = old
            num[idx] = (fp - fm) / (2 * h)
        assert np.max(np.abs(num - grad)) <= 1e-4 * max(1.0, np.max(np.abs(grad))), l


def test_duplicated_minibatch_doubles():
    """Sum convention: duplicating the minibatch doubles the
    objective and every gradient."""
    params = _rand_params(CFG_T, 4)
    f, y = gaussian_rows(5, 5, 6), labels_uniform(6, 5, 5)
    a = nnet.forward_backward(params, CFG_T, f, y)
    b = nnet.forward_backward(params, CFG_T, np.concatenate([f, f]), np.concatenate([y, y]))
    assert b.objective == pytest.approx(2 * a.objective, rel=1e-12)
    for l in range(len(params)):
        assert np.allclose(b.X[l].T @ b.Y[l], 2 * (a.X[l].T @ a.Y[l]), rtol=1e-12, atol=1e-14)


def test_init_statistics():
    """C.6: std 1/sqrt(fan-in) (fan-in includes bias, R20); softmax zero."""
    cfg = nnet.NnetConfig(input_dim=99, num_hidden=1, hidden_dim=400, pnorm_group=10, num_classes=7)
    params = nnet.init_params(cfg, standard_normals(7, cfg.layer_shapes()))
    assert np.std(params[0]) == pytest.approx(0.1, rel=0.02)    # fan-in 100 -> 0.1
    assert np.all(params[-1] == 0)


def test_max_change_guarantee_in_step():
    """SPEC acceptance 7: the applied change satisfies ||alpha Delta||_F <= N * 0.075."""
    cfg = nnet.NnetConfig(input_dim=10, num_hidden=2, hidden_dim=40, pnorm_group=4, num_classes=6)
    params = _rand_params(cfg, 8)
    states = nnet.make_states(cfg, online_ng.OnlineNgConfig(rank=3), online_ng.OnlineNgConfig(rank=5))
    for step in range(6):
        f, y = gaussian_rows(100 + step, 32, 10, scale=3.0), labels_uniform(200 + step, 32, 6)
        before = [w.copy() for w in params]
        _, stats = nnet.train_step(params, cfg, f, y, lr=5.0, states=states)
        for l, st in enumerate(stats):
            delta = np.linalg.norm(params[l] - before[l])
            assert delta <= 32 * 0.075 * (1 + 1e-6)
            assert st.alpha_t <= 1.0
        assert any(st.alpha_t < 1.0 for st in stats)


def test_plain_sgd_reduction():
    """precond='none' with an inactive guard is textbook SGD: the objective improves on a
    fixed minibatch for a small step (gradient ascent)."""
    params = _rand_params(CFG_T, 12)
    f, y = gaussian_rows(13, 16, 6), labels_uniform(14, 16, 5)
    o0 = nnet.forward_backward(params, CFG_T, f, y).objective
    nnet.train_step(params, CFG_T, f, y, lr=1e-3, precond="none")
    assert nnet.forward_backward(params, CFG_T, f, y).objective > o0


# ---------------------------------------------------------------- training scalars

def test_lr_schedule_golden():
    for c in GOLD["lr_schedule"]["cases"]:
        assert training.lr_at(c["frac"], 1.0) == pytest.approx(c["lr"], rel=1e-12)


def test_max_change_golden():
    g = GOLD["max_change"]
    assert g["n"] * g["per_sample"] == pytest.approx(g["limit"])
    for c in g["cases"]:
        assert training.max_change_scale(c["bound"], g["n"], g["per_sample"]) == pytest.approx(c["alpha"])


def test_average_golden_and_identity():
    g = GOLD["average"]
    out = training.average_models([[np.array(m)] for m in g["models"]])
    assert np.allclose(out[0], g["mean"])
    rng = np.random.default_rng(0)
    w = rng.normal(size=(50, 7)).astype(np.float32)
    for n in (2, 4, 8):                        # n identical models -> bit-exact no-op
        assert np.array_equal(training.average_models([[w]] * n, dtype=np.float32)[0], w)
    ws = [rng.normal(size=(9,)) for _ in range(5)]
    m = training.average_models([[x] for x in ws])[0]
    assert np.all(m <= np.max(ws, axis=0) + 1e-15) and np.all(m >= np.min(ws, axis=0) - 1e-15)
