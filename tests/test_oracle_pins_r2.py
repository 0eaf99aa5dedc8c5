"""Round-2 pins of the oracle (CPU only), each chosen so that a specific plausible mistake
fails it (VERDICT r1 "What's weak" 1):

* gamma scaling of the weight update ("rescale so the Frobenius norm is the
  same", eqn:gammat P:1058-1061, eqn:add:w P:1507-1508): when every row of X lies in the
  span of R_t and all d_i are equal, X_hat = (beta/(beta+d)) X exactly, so X_bar = gamma X_hat
  = X and the online step must equal the plain-SGD step.  Dropping gamma_x gamma_y from the
  update leaves a factor (beta/(beta+d))^2 ~ 0.58 behind.
* the B.3.1 trigger threshold cond(C) > 1e6: with rows of X
  orthogonal to span(R_t), Z_t = (1-eta)^2 (D_t + rho I)^2 in closed form, so cond(C) is set
  by the state alone; 1e5 must not trigger the check, 1e7 must.
"""
import math

import numpy as np
import pytest

from oracle import nnet, online_ng as ong


def _state(D, R, d, rho, t, basis):
    """A state with R_t = rows of `basis` (orthonormal), D_t = diag(d), rho_t = rho."""
    cfg = ong.OnlineNgConfig(rank=R)
    s = ong.OnlineNgState(D, cfg)
    s.d = np.asarray(d, dtype=np.float64)
    s.rho = float(rho)
    e = ong.e_of(ong.beta_of(s.rho, s.d, cfg.alpha, D), s.d)
    s.W = np.sqrt(e)[:, None] * basis
    s.t, s.initialized = t, True
    return s


def _orthonormal(rng, D, k):
    q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    return q.T[:k], q.T[k:]          # first k rows span the state, the rest its complement


def test_in_span_closed_form():
    """Rows in span(R_t), equal d: X_hat = beta/(beta+d) X (Woodbury on a scaled identity,
    P:1064-1082) and gamma = (beta+d)/beta, so X_bar = X exactly."""
    rng = np.random.default_rng(21)
    D, R, N, delta, rho = 9, 4, 5, 1.3, 0.2
    basis, _ = _orthonormal(rng, D, R)
    s = _state(D, R, [delta] * R, rho, 11, basis)          # t = 11: no refresh
    X = rng.normal(size=(N, R)) @ basis
    out = ong.precondition(s, X)
    beta = ong.beta_of(rho, s.d, 4.0, D)
    assert not out.updated
    assert np.allclose(out.x_hat, beta / (beta + delta) * X, rtol=0, atol=1e-13)
    assert out.gamma == pytest.approx((beta + delta) / beta, rel=1e-13)
    assert np.allclose(out.x_bar, X, rtol=0, atol=1e-13)


def test_online_step_equals_plain_sgd_in_span():
    """nnet.update with online NG on states whose spans contain the data equals the plain
    SGD update (max-change included: ||x_bar_i|| = ||x_i||), while X_hat^T Y_hat alone is
    off by (beta/(beta+d))^2 -- this fails if gamma_x gamma_y is dropped from eqn:add:w."""
    rng = np.random.default_rng(22)
    N, Dout, Din1, R = 6, 10, 8, 4
    bo, _ = _orthonormal(rng, Dout, R)
    bi, _ = _orthonormal(rng, Din1, R)
    X = rng.normal(size=(N, R)) @ bo
    Y = rng.normal(size=(N, R)) @ bi
    fb = nnet.ForwardBackward(Y=[Y], S=[], Z=[None], X=[X], objective=0.0, logp=None)
    for lr, mc in ((1e-3, 0.075), (10.0, 0.075)):     # guard inactive / active
        w0 = rng.normal(size=(Dout, Din1))
        p_on, p_plain = [w0.copy()], [w0.copy()]
        states = [(_state(Din1, R, [0.7] * R, 0.05, 13, bi), _state(Dout, R, [2.0] * R, 0.3, 13, bo))]
        st_on = nnet.update(p_on, fb, lr, states, precond="online", max_change_per_sample=mc)
        st_pl = nnet.update(p_plain, fb, lr, precond="none", max_change_per_sample=mc)
        assert st_on[0].alpha_t == pytest.approx(st_pl[0].alpha_t, rel=1e-12)
        assert np.max(np.abs(p_on[0] - p_plain[0])) <= 1e-12 * np.max(np.abs(p_plain[0] - w0))
        # the unscaled product is measurably different (what a dropped gamma would give)
        bx = ong.beta_of(0.3, np.full(R, 2.0), 4.0, Dout)
        by = ong.beta_of(0.05, np.full(R, 0.7), 4.0, Din1)
        shrink = (bx / (bx + 2.0)) * (by / (by + 0.7))
        assert shrink < 0.9


def _cond_case(cond_target, naive):
    """Rows of X orthogonal to span(R_t): Y_t = R_t T_t = (1-eta)(D_t + rho I) R_t, so
    c_i = (1-eta)^2 (d_i + rho)^2 and cond(C) = ((d_1 + rho)/(d_R + rho))^2 exactly."""
    rng = np.random.default_rng(23)
    D, R, N, rho = 12, 3, 7, 0.01
    basis, comp = _orthonormal(rng, D, R)
    ratio = math.sqrt(cond_target)
    d = np.array([(1e-9 + rho) * ratio - rho, 5 * rho, 1e-9])
    s = _state(D, R, d, rho, 12, basis)                   # t = 12: refresh step
    X = rng.normal(size=(N, D - R)) @ comp
    out = (ong.precondition_naive if naive else ong.precondition)(s, X)
    eta = ong.eta_from(N, 2000.0)
    trx = float(np.sum(X * X))
    rho_dash = ((eta / N) * trx + (1 - eta) * (D - R) * rho) / (D - R)      # eqn:rhodash2 here
    assert out.updated and not out.floored
    assert s.rho == pytest.approx(rho_dash, rel=1e-9)
    assert np.allclose(s.d, np.maximum((1 - eta) * (d + rho) - rho_dash, 1e-10), rtol=1e-9, atol=0)
    return out


@pytest.mark.parametrize("naive", [False, True])
def test_reorth_trigger_threshold(naive):
    """B.3.1 check iff cond(C) > 1e6 (no floor here): 1e5 -> not checked, 1e7 -> checked;
    float64 keeps R_{t+1} orthonormal, so the check never repairs."""
    lo, hi = _cond_case(1e5, naive), _cond_case(1e7, naive)
    assert not lo.reorth_checked
    assert hi.reorth_checked and not hi.reorthogonalized
