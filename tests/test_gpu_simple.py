"""GPU parity of the simple NG-SGD preconditioner (Appendix A)
against the float64 oracle oracle/simple_ng.py (itself pinned by SPEC's worked example and
the per-row held-out brute force, tests/test_oracle_simple_nnet_training.py).  The device
path is FP64 arithmetic on FP32 data: X_bar within 1e-5 normwise (FP32 output rounding of
X_hat, amplified by at most cond(beta I + G/(n-1)) <= 1 + n D / (alpha (n-1)))."""
import ctypes

import numpy as np
import pytest

from oracle import nnet as onn
from oracle import simple_ng as osn
from oracle import training as otr
from synth import gaussian_rows, labels_uniform, power_law_rows, spliced_frames, standard_normals

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_7455_b200 import api
    return api


def normwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def run_simple(api, X, ld_pad=0):
    n, D = X.shape
    pre = api.SimplePreconditioner(D, max(n, 2))
    buf = torch.zeros((n, D + ld_pad), dtype=torch.float32, device="cuda")
    x = buf[:, :D]
    x.copy_(torch.from_numpy(np.ascontiguousarray(X, dtype=np.float32)))
    g = torch.zeros(1, device="cuda")
    p = torch.zeros(n, device="cuda")
    pre.precondition(x, g, p)
    pre.read_flags()
    xh = x.cpu().numpy().astype(np.float64)
    return xh, float(g.cpu()[0]), p.cpu().numpy().astype(np.float64), buf


def test_spec_worked_example(api):
    """SPEC's [[1],[1]]: beta = 4, G = 6, q = a = 1/6, b = 6/5, x_hat = 1/5,
    gamma = 5, x_bar = [[1],[1]]."""
    xh, g, p, _ = run_simple(api, np.array([[1.0], [1.0]]))
    assert np.allclose(xh, 0.2, rtol=1e-6) and g == pytest.approx(5.0, rel=1e-6)
    assert np.allclose(p, 0.04, rtol=1e-5)


@pytest.mark.parametrize("n,D", [(2, 1), (16, 8), (8, 16), (33, 33), (128, 41), (128, 200), (77, 300),
                                 (512, 361), (512, 3000)])
def test_matches_oracle(api, n, D):
    """Both branches (column space n > D, row space n <= D, strict, R11), ragged sizes and
    the config-3 sizes: X_bar = gamma X_hat within 1e-5 normwise, gamma 1e-6 relative."""
    X = gaussian_rows(n * 31 + D, n, D) * np.linspace(0.2, 3.0, D)[None, :]
    X = X.astype(np.float32).astype(np.float64)
    xb_ref, g_ref, rs_ref = osn.precondition_simple(X)
    xh, g, p, buf = run_simple(api, X, ld_pad=3)
    assert g == pytest.approx(g_ref, rel=1e-6)
    assert normwise(g * xh, xb_ref) <= 1e-5, normwise(g * xh, xb_ref)
    assert normwise(g * g * p, rs_ref) <= 1e-5
    assert np.all(buf[:, D:].cpu().numpy() == 0.0)          # padding columns untouched


def test_power_law_and_activation_like(api):
    """Config-2-shaped data (power-law covariance; [|.|, 1] input side), both branches."""
    for X in (power_law_rows(5, 512, 2000)[0], power_law_rows(6, 256, 200, nonneg=True, append_one=True)[0]):
        X = X.astype(np.float32).astype(np.float64)
        xb_ref, g_ref, _ = osn.precondition_simple(X)
        xh, g, _, _ = run_simple(api, X)
        assert normwise(g * xh, xb_ref) <= 1e-5


def test_zero_input(api):
    """tr X^T X = 0: beta from the 1e-20 floor, X_hat = 0, gamma = 1."""
    xh, g, p, _ = run_simple(api, np.zeros((8, 5)))
    assert g == 1.0 and np.all(xh == 0.0) and np.all(p == 0.0)


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_nnet_simple_ng_steps(api, precision):
    """The DNN step with simple NG-SGD on both sides of every matrix (precond = 2; Table 2's
    "simple NG" row): 3 steps of the tiny config and 1 of config 3 (with the
    renormalisation layers), Delta W per matrix against the oracle's update(precond='simple')
    applied to the GPU's pre-step weights: 1e-4 (FP32) / 2e-2 (TF32) normwise."""
    tol = 1e-4 if precision == "fp32" else 2e-2
    for shape in ("tiny", "config3"):
        if shape == "tiny":
            cfg = onn.NnetConfig(input_dim=40, num_hidden=2, hidden_dim=200, pnorm_group=10, num_classes=16, renorm=True)
            N, steps, ctx = 128, 3, 0
        else:
            cfg = onn.NnetConfig(360, 4, 3000, 10, 5000, renorm=True)
            N, steps, ctx = 512, 1, 4
        net = api.Nnet(cfg.input_dim, cfg.num_hidden, cfg.hidden_dim, cfg.pnorm_group, cfg.num_classes,
                       max_minibatch=N, precond="simple", seed=3, precision=precision, renorm=True)
        params = onn.init_params(cfg, standard_normals(3, cfg.layer_shapes()))
        params[-1] = 0.05 * standard_normals(4, [cfg.layer_shapes()[-1]])[0]
        for l, p in enumerate(params):
            net.set_params(l, p.astype(np.float32))
        frames, labels = spliced_frames(7, steps * N, num_classes=cfg.num_classes, context=ctx)
        for k in range(steps):
            fr, lb = frames[k * N:(k + 1) * N], labels[k * N:(k + 1) * N]
            before = [net.get_params(l).astype(np.float64) for l in range(len(params))]
            net.forward_backward(torch.from_numpy(fr).cuda(), torch.from_numpy(lb).cuda())
            net.update(0.002, 0.075)
            fb = onn.forward_backward(before, cfg, fr.astype(np.float64), lb)
            ref = [b.copy() for b in before]
            onn.update(ref, fb, 0.002, precond="simple")
            for l in range(len(params)):
                d_gpu = net.get_params(l).astype(np.float64) - before[l]
                half_ulp = 0.5 * np.spacing(np.abs(net.get_params(l))).astype(np.float64)
                err = np.max(np.maximum(np.abs(d_gpu - (ref[l] - before[l])) - half_ulp, 0.0)) / \
                    np.max(np.abs(ref[l] - before[l]))
                assert err <= tol, (shape, k, l, err)
