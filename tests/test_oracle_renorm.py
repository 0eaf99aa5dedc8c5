"""Pins for the renormalisation layer of oracle/nnet.py (reading R32): the layers that
"follow each p-norm layer", y = s a with s = sqrt(D / ||a||^2).  CPU only.

What pins it (none of these re-types the formula):
* the paper's own statement that with these layers "the network output is invariant to
  (nonzero) scaling of the parameters of the p-norm layers";
* central finite differences of the objective (the backward pass, incl. the
  s (g - y y^T g / D) term);
* unit root-mean-square rows and the all-zero-row special case.
"""
import numpy as np
import pytest

from oracle import nnet
from synth import gaussian_rows, labels_uniform, standard_normals


def _params(cfg, seed):
    ps = nnet.init_params(cfg, standard_normals(seed, cfg.layer_shapes()))
    rng = np.random.default_rng(seed + 100)
    ps[-1] = rng.normal(size=ps[-1].shape) * 0.3      # non-zero softmax layer: every gradient non-trivial
    return ps


@pytest.mark.parametrize("num_hidden", [1, 2, 3])
def test_output_invariant_to_pnorm_layer_scaling(num_hidden):
    """with renormalisation layers the output is invariant to scaling the
    parameters of a p-norm layer (here: each hidden W_l, bias included, by c != 0)."""
    cfg = nnet.NnetConfig(input_dim=7, num_hidden=num_hidden, hidden_dim=12, pnorm_group=3, num_classes=5,
                          renorm=True)
    params = _params(cfg, 3 + num_hidden)
    frames = gaussian_rows(4, 9, 7)
    ref = nnet.forward(params, cfg, frames)[3]
    for l in range(num_hidden):
        for c in (1e-3, 0.37, -2.5, 1e4):
            scaled = [p.copy() for p in params]
            scaled[l] *= c
            out = nnet.forward(scaled, cfg, frames)[3]
            assert np.max(np.abs(out - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref))), (l, c)
    # and without the layer the output does change (the pin is not vacuous)
    plain = nnet.NnetConfig(7, num_hidden, 12, 3, 5, renorm=False)
    scaled = [p.copy() for p in params]
    scaled[0] *= 2.0
    assert np.max(np.abs(nnet.forward(scaled, plain, frames)[3] - nnet.forward(params, plain, frames)[3])) > 1e-3


def test_rows_have_unit_rms():
    cfg = nnet.NnetConfig(input_dim=6, num_hidden=2, hidden_dim=20, pnorm_group=4, num_classes=3, renorm=True)
    params = _params(cfg, 9)
    Y, _, S, _ = nnet.forward(params, cfg, gaussian_rows(1, 11, 6) * 50.0)
    for l in (1, 2):
        a = Y[l][:, :-1]
        assert np.allclose(np.mean(a * a, axis=1), 1.0, rtol=1e-13)
        assert np.all(Y[l][:, -1] == 1.0)
        assert S[l - 1].shape == (11, 1) and np.all(S[l - 1] > 0)


@pytest.mark.parametrize("num_hidden", [1, 2, 3])
def test_finite_difference_gradients_renorm(num_hidden):
    """d objective / d W_l = X_l^T Y_l through the renormalisation layers, against central
    differences (h = 1e-5, relative 1e-4)."""
    cfg = nnet.NnetConfig(input_dim=5, num_hidden=num_hidden, hidden_dim=8, pnorm_group=2, num_classes=4,
                          renorm=True)
    params = _params(cfg, 20 + num_hidden)
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


def test_zero_row_passes_zero():
    """An all-zero p-norm output row has s = 0: y = [0, ..., 0, 1] and zero derivatives
    below it (no 0/0)."""
    cfg = nnet.NnetConfig(input_dim=4, num_hidden=1, hidden_dim=6, pnorm_group=2, num_classes=3, renorm=True)
    params = _params(cfg, 5)
    params[0][:] = 0.0
    fb = nnet.forward_backward(params, cfg, gaussian_rows(7, 5, 4), labels_uniform(8, 5, 3))
    assert np.all(fb.Y[1][:, :-1] == 0.0) and np.all(fb.Y[1][:, -1] == 1.0)
    assert np.all(fb.X[0] == 0.0) and np.all(np.isfinite(fb.X[1]))
