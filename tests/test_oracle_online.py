"""Pins for oracle/online_ng.py (Appendix B) against things other than itself:
worked examples, the naive D x D defining equations, explicit-inverse brute force,
closed forms and the paper's invariants.  CPU only."""
import json
import math
import os

import numpy as np
import pytest

from oracle import online_ng as ong
from synth import gaussian_rows, power_law_rows

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def _cfg(rank, **kw):
    return ong.OnlineNgConfig(rank=rank, **kw)


def test_eta_golden():
    for c in GOLD["eta"]["cases"]:
        assert abs(ong.eta_from(c["n"], c["S"]) - c["eta"]) <= c["tol"]


def test_paper_defaults():
    g = GOLD["paper_ng_defaults"]
    c = ong.OnlineNgConfig()
    assert (c.alpha, c.s_samples, c.epsilon, c.update_period, c.always_update_first) == \
        (g["alpha"], g["S"], g["epsilon"], g["J"], g["first"])


def test_update_policy():
    """B.5 P:1328-1329: t < 10 or 4 | t."""
    c = ong.OnlineNgConfig()
    upd = [t for t in range(40) if ong.should_update(t, c)]
    assert upd == list(range(10)) + [12, 16, 20, 24, 28, 32, 36]


def test_init_golden():
    g = GOLD["online_init_2000"]
    s = ong.OnlineNgState(4, _cfg(g["rank"]))
    ong.init_state(s, np.array(g["X0"]))
    assert s.rho == pytest.approx(g["rho0"], rel=1e-12)
    assert s.d[0] == pytest.approx(g["d0"], rel=1e-12)
    R = ong.R_of(s)
    assert np.allclose(np.abs(R[0]), g["r0_abs"], atol=1e-12)
    # tr F_0 = tr S_0 when no floor engages (trace-matching of the init)
    assert np.trace(ong.F_of(s)) == pytest.approx(4.0, rel=1e-9)


def test_init_trace_matching_random():
    X = gaussian_rows(3, 40, 12)
    s = ong.OnlineNgState(12, _cfg(5))
    ong.init_state(s, X)
    assert np.trace(ong.F_of(s)) == pytest.approx(np.trace(X.T @ X) / 40, rel=1e-12)
    # the top-R eigenpairs of S_0 are exactly those of F_0's R subspace: compare with eigh
    lam = np.sort(np.linalg.eigvalsh(X.T @ X / 40))[::-1]
    assert np.allclose(s.d + s.rho, lam[:5], rtol=1e-12)
    assert s.rho == pytest.approx(lam[5:].mean(), rel=1e-12)


def test_deferred_init_on_zero_input():
    """Reading R7: an all-zero first minibatch passes through and leaves the state
    uninitialised; t counts it (the schedule is per minibatch)."""
    s = ong.OnlineNgState(6, _cfg(2))
    out = ong.precondition(s, np.zeros((5, 6)))
    assert not s.initialized and s.t == 1 and out.gamma == 1.0
    assert np.all(out.x_hat == 0) and np.all(out.row_sq == 0)


@pytest.mark.parametrize("N,D,R,steps", [(16, 8, 3, 50), (10, 30, 4, 40), (64, 40, 7, 30), (31, 31, 5, 20)])
def test_efficient_matches_naive_defining_form(N, D, R, steps):
    """SPEC acceptance 3: B.5 efficient form vs the B.1-B.2 definitions
    with explicit D x D F_t, T_t, Y_t = R_t T_t, over sequential minibatches
    (covers both L branches: N > D and N <= D)."""
    batches = power_law_rows(11 + N + D, N, D, n_batches=steps)
    se = ong.OnlineNgState(D, _cfg(R))
    sn = ong.OnlineNgState(D, _cfg(R))
    for t, X in enumerate(batches):
        oe = ong.precondition(se, X)
        on = ong.precondition_naive(sn, X)
        assert oe.updated == on.updated
        scale = np.max(np.abs(on.x_bar))
        assert np.max(np.abs(oe.x_bar - on.x_bar)) <= 1e-8 * scale, t
        assert oe.gamma == pytest.approx(on.gamma, rel=1e-8)
        assert se.rho == pytest.approx(sn.rho, rel=1e-8)
        assert np.allclose(se.d, sn.d, rtol=1e-8)
        wtw_e, wtw_n = se.W.T @ se.W, sn.W.T @ sn.W
        assert np.max(np.abs(wtw_e - wtw_n)) <= 1e-8 * np.max(np.abs(wtw_n))
        assert oe.row_sq == pytest.approx(np.sum(oe.x_bar ** 2, axis=1), rel=1e-10)


def test_apply_matches_explicit_inverse():
    """X_bar = gamma X G^{-1} with G formed and solved explicitly versus the
    Woodbury form X - X W^T W."""
    D, R = 25, 6
    s = ong.OnlineNgState(D, _cfg(R))
    for X in power_law_rows(5, 20, D, n_batches=8):
        ong.precondition(s, X)
    X = gaussian_rows(9, 17, D)
    ref = ong.apply_bruteforce(s, X)
    out = ong.precondition(s.copy(), X, update=False)
    assert np.max(np.abs(out.x_bar - ref)) <= 1e-12 * np.max(np.abs(ref))


def test_invariants_over_trajectory():
    """Norm preservation, R R^T = I, trace preservation
    tr F_{t+1} = tr T_t when no floor engages, 0 < e < 1,
    rho, d >= eps, eqn:trxxt (asserted inside precondition)."""
    D, R, N = 60, 8, 48
    s = ong.OnlineNgState(D, _cfg(R))
    for X in power_law_rows(21, N, D, n_batches=60):
        X = X * 3.0
        prev = s.copy() if s.initialized else None
        out = ong.precondition(s, X)
        assert np.linalg.norm(out.x_bar) == pytest.approx(np.linalg.norm(X), rel=1e-12)
        Rm = ong.R_of(s)
        assert np.max(np.abs(Rm @ Rm.T - np.eye(R))) <= 1e-10
        beta = ong.beta_of(s.rho, s.d, s.cfg.alpha, D)
        e = ong.e_of(beta, s.d)
        assert np.all(e > 0) and np.all(e < 1)
        assert s.rho >= 1e-10 and np.all(s.d >= 1e-10)
        if prev is not None and out.updated and not out.floored:
            eta = ong.eta_from(N, s.cfg.s_samples)
            trT = eta * np.trace(X.T @ X) / N + (1 - eta) * np.trace(ong.F_of(prev))
            assert np.trace(ong.F_of(s)) == pytest.approx(trT, rel=1e-10)


def test_non_update_is_pure():
    """update=false leaves (rho, d, W) bit-identical."""
    D = 20
    s = ong.OnlineNgState(D, _cfg(4))
    for X in power_law_rows(2, 30, D, n_batches=3):
        ong.precondition(s, X)
    before = s.copy()
    ong.precondition(s, gaussian_rows(4, 30, D), update=False)
    assert s.rho == before.rho and np.array_equal(s.d, before.d) and np.array_equal(s.W, before.W)
    assert s.t == before.t + 1


def test_rank_zero_is_identity():
    """R = 0 (D = 1 clips R to D - 1 = 0): X_bar = X exactly (reading R27)."""
    s = ong.OnlineNgState(1, _cfg(3))
    X = gaussian_rows(1, 9, 1)
    out = ong.precondition(s, X)
    assert out.gamma == 1.0 and np.array_equal(out.x_bar, X)


def test_textbook_reduction_eta_one_subspace_iteration():
    """eta = 1 with S_t = Sigma fixed: the update is orthogonal (subspace) iteration
    (P:964-968); F converges to the top-R eigen-truncation of Sigma with rho = mean of
    the remaining D - R eigenvalues.  Closed form via eigh."""
    rng = np.random.default_rng(0)
    D, R = 12, 3
    Q, _ = np.linalg.qr(rng.normal(size=(D, D)))
    lam = np.array([10.0, 6.0, 4.0] + list(np.linspace(1.0, 0.2, D - 3)))
    Sigma = Q @ np.diag(lam) @ Q.T
    w, V = np.linalg.eigh(Sigma)
    X_sig = math.sqrt(D) * (V * np.sqrt(np.maximum(w, 0))[None, :]) @ V.T     # X^T X / D = Sigma
    cfg = _cfg(R, s_samples=1e-9)                                              # eta == 1.0
    assert ong.eta_from(D, cfg.s_samples) == 1.0
    s = ong.OnlineNgState(D, cfg)
    ong.init_state(s, gaussian_rows(3, 40, D))                                 # unrelated start
    for _ in range(200):
        ong.precondition(s, X_sig, update=True)
    Ftrunc = sum((lam[i] - lam[R:].mean()) * np.outer(Q[:, i], Q[:, i]) for i in range(R)) \
        + lam[R:].mean() * np.eye(D)
    assert np.max(np.abs(ong.F_of(s) - Ftrunc)) <= 1e-9


def test_reorthogonalize_repairs_perturbation():
    """B.3.1: W perturbed by 1e-2 -> repaired to <= 1e-6 and
    the row space is preserved."""
    D, R = 30, 5
    s = ong.OnlineNgState(D, _cfg(R))
    for X in power_law_rows(8, 40, D, n_batches=12):
        ong.precondition(s, X)
    rng = np.random.default_rng(1)
    s.W = s.W + 1e-2 * rng.normal(size=s.W.shape)
    W_bad = s.W.copy()
    assert ong.reorthogonalize(s)
    Rm = ong.R_of(s)
    assert np.max(np.abs(Rm @ Rm.T - np.eye(R))) <= 1e-6
    P_bad = np.linalg.pinv(W_bad) @ W_bad
    P_new = np.linalg.pinv(s.W) @ s.W
    assert np.max(np.abs(P_bad - P_new)) <= 1e-9
    assert not ong.reorthogonalize(s)          # already orthonormal: no-op


def test_reorth_check_triggers_on_wide_spectrum():
    """A stream whose covariance spans > 1e3 in scale makes cond(C) > 1e6, which
    triggers the B.3.1 orthogonality check; in float64
    the check passes without repair, and the naive form agrees on every output."""
    D, R, N = 16, 6, 40
    rng = np.random.default_rng(4)
    scale = 10.0 ** -np.arange(D)            # 1, 0.1, ..., 1e-15
    se, sn = ong.OnlineNgState(D, _cfg(R)), ong.OnlineNgState(D, _cfg(R))
    flags = []
    for t in range(25):
        X = rng.normal(size=(N, D)) * scale[None, :]
        oe, on = ong.precondition(se, X), ong.precondition_naive(sn, X)
        assert oe.floored == on.floored and oe.reorth_checked == on.reorth_checked
        assert not oe.reorthogonalized
        flags.append(oe.reorth_checked)
        assert np.max(np.abs(oe.x_bar - on.x_bar)) <= 1e-7 * np.max(np.abs(on.x_bar))
    assert any(flags)
