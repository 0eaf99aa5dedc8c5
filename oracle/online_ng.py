"""Online natural-gradient preconditioner, Appendix B of arXiv 1410.7455 (oracle).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Two independent implementations of the same method, both float64:

* ``precondition``        -- the efficient algorithm exactly as summarised in B.5
                             (P:1299-1407), using the sub-expressions of B.3
                             (P:1027-1241).  This is what the CUDA path mirrors.
* ``precondition_naive``  -- the *defining* equations of B.1-B.2:
                             explicit D x D F_t, G_t, S_t, T_t, Y_t = R_t T_t, with
                             ``R_t`` materialised.  Ground truth on small D.

Notation follows the paper: X (N x D) minibatch, R rank, rho, d (= diag D_t),
W (= W_t = E_t^{1/2} R_t, R x D), eta the forgetting factor, alpha the identity
smoothing constant, epsilon the floor.  Readings of ambiguous passages are numbered
as in DESIGN.md section "Readings" (R#).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass
class OnlineNgConfig:
    """B.4 / B.5 typical configuration."""

    rank: int = 20                 # R: 20 input side, 80 output side
    alpha: float = 4.0             # identity smoothing
    s_samples: float = 2000.0      # S, eta = 1 - exp(-N/S)
    update_period: int = 4         # J
    always_update_first: int = 10  # "except on the first 10 minibatches"
    epsilon: float = 1e-10         # floor for rho and d


@dataclasses.dataclass
class OnlineNgState:
    """Per-side state: rho_t, D_t, W_t and the counter t.

    R_t itself is never stored.  ``rank`` is the effective rank
    R = min(R_cfg, D-1) (reading R29: B.1 requires R < D).
    """

    dim: int
    cfg: OnlineNgConfig
    rank: int = 0
    rho: float = 0.0
    d: np.ndarray | None = None     # (R,)   diagonal of D_t, descending
    W: np.ndarray | None = None     # (R, D) W_t = E_t^{1/2} R_t
    t: int = 0
    initialized: bool = False

    def __post_init__(self):
        self.rank = max(0, min(int(self.cfg.rank), self.dim - 1))

    def copy(self) -> "OnlineNgState":
        s = OnlineNgState(self.dim, dataclasses.replace(self.cfg))
        s.rank, s.rho, s.t, s.initialized = self.rank, self.rho, self.t, self.initialized
        s.d = None if self.d is None else self.d.copy()
        s.W = None if self.W is None else self.W.copy()
        return s


@dataclasses.dataclass
class PrecondOutput:
    """X_hat (NOT scaled by gamma), gamma, and row_sq = gamma^2 p_i."""

    x_hat: np.ndarray
    gamma: float
    row_sq: np.ndarray
    updated: bool = False
    floored: bool = False
    reorth_checked: bool = False
    reorthogonalized: bool = False
    tr_xxt: float = 0.0
    # diagnostics of the update's threshold decisions (values the algorithm computes anyway;
    # tests use them to tell a decided threshold from one inside rounding noise)
    floor_margin: float = 0.0     # (min_i c_i - (1-eta)^2 rho^2) / max_i c_i, before flooring
    cond_c: float = 0.0           # max c / min c after flooring (the B.3.1 trigger, > 1e6)

    @property
    def x_bar(self) -> np.ndarray:
        return self.gamma * self.x_hat


# --------------------------------------------------------------------------------------
# scalar helpers
# --------------------------------------------------------------------------------------

def eta_from(n: int, s_samples: float) -> float:
    """eqn:eta:ns: eta = 1 - exp(-N/S).  Recomputed per call from that
    call's N (reading R10: the last minibatch may be short)."""
    return 1.0 - math.exp(-float(n) / float(s_samples))


def beta_of(rho: float, d: np.ndarray, alpha: float, dim: int) -> float:
    """eqn:beta2: beta_t = rho_t (1 + alpha) + (alpha / D) tr(D_t)."""
    return rho * (1.0 + alpha) + (alpha / dim) * float(np.sum(d))


def e_of(beta: float, d: np.ndarray) -> np.ndarray:
    """eqn:etii: e_tii = 1 / (beta_t / d_tii + 1)."""
    return 1.0 / (beta / d + 1.0)


def should_update(t: int, cfg: OnlineNgConfig) -> bool:
    """B.5: update iff t < 10 or J divides t."""
    return t < cfg.always_update_first or (t % cfg.update_period) == 0


def _eigh_descending(m: np.ndarray):
    """Symmetric eigendecomposition, eigenvalues sorted descending (reading R12;
    eigenvalue order 'sorted on i from greatest to least').  Ties keep
    numpy's ascending-index order reversed stably (reading R7)."""
    w, v = np.linalg.eigh(m)
    order = np.argsort(-w, kind="stable")
    return w[order], v[:, order]


# --------------------------------------------------------------------------------------
# initialisation (B.3.2)
# --------------------------------------------------------------------------------------

def init_state(state: OnlineNgState, X0: np.ndarray) -> None:
    """B.3.2 "Initialization", and B.5 P:1318-1322.

    S_0 = X_0^T X_0 / N; the rows of R_0 are the top-R eigenvectors of S_0 with
    eigenvalues lambda_i; rho_0 = max((tr S_0 - sum lambda_i)/(D - R), eps);
    d_0ii = max(eps, lambda_i - rho_0); W_0 = E_0^{1/2} R_0 via eqn:beta2, eqn:etii,
    eqn:wt:def.
    """
    cfg = state.cfg
    X0 = np.asarray(X0, dtype=np.float64)
    N, D = X0.shape
    assert D == state.dim
    R = state.rank
    eps = cfg.epsilon
    S0 = (X0.T @ X0) / N
    lam, V = _eigh_descending(S0)
    lam_r = lam[:R]
    R0 = V[:, :R].T                                            # rows = eigenvectors
    rho0 = max((float(np.trace(S0)) - float(np.sum(lam_r))) / (D - R), eps)
    d0 = np.maximum(eps, lam_r - rho0)
    beta0 = beta_of(rho0, d0, cfg.alpha, D)
    e0 = e_of(beta0, d0)
    state.rho = rho0
    state.d = d0
    state.W = np.sqrt(e0)[:, None] * R0                        # eqn:wt:def
    state.initialized = True                                   # (t is not reset: reading R7)


# --------------------------------------------------------------------------------------
# efficient algorithm (B.5 summary)
# --------------------------------------------------------------------------------------

def precondition(state: OnlineNgState, X: np.ndarray, update: bool | None = None,
                 check_trace: bool = True) -> PrecondOutput:
    """Online NG-SGD, B.5 "Summary of the online natural gradient method".

    Mutates ``state`` (on update steps: rho, d, W; always: t).  Returns X_hat (not
    scaled), gamma and gamma^2 p_i.  ``update=None`` applies the internal policy
    t < 10 or J | t; True/False forces it.
    """
    cfg = state.cfg
    X = np.asarray(X, dtype=np.float64)
    N, D = X.shape
    assert D == state.dim
    R = state.rank

    # Reading R7: defer initialisation until the first minibatch with tr(X^T X) > 0
    # (zero-initialised softmax makes hidden-layer derivatives exactly 0 at step 0,
    # P:1697-1698; eigenvectors of S_0 = 0 are arbitrary).  t still counts the minibatch:
    # the update schedule is per minibatch of the process.
    if not state.initialized:
        if float(np.sum(X * X)) == 0.0:
            state.t += 1
            return PrecondOutput(X.copy(), 1.0, np.zeros(N), tr_xxt=0.0)
        init_state(state, X)

    if R == 0:
        # Degenerate rank: F = rho I, G = (1+alpha) rho I, X_hat = X exactly and
        # gamma = 1 (reading R27: same reduction tree for both traces).
        p = np.sum(X * X, axis=1)
        upd = should_update(state.t, cfg) if update is None else bool(update)
        state.t += 1
        return PrecondOutput(X.copy(), 1.0, p.copy(), updated=upd, tr_xxt=float(np.sum(p)))

    if update is None:
        update = should_update(state.t, cfg)
    eta = eta_from(N, cfg.s_samples)
    W, rho, d = state.W, state.rho, state.d
    alpha, eps = cfg.alpha, cfg.epsilon

    beta = beta_of(rho, d, alpha, D)                           # eqn:beta2
    e = e_of(beta, d)                                          # eqn:etii

    H = X @ W.T                                                # P:1335-1337, eqn:ht

    if not update:
        # "Without updating the Fisher matrix".
        tr_xxt = float(np.sum(np.sum(X * X, axis=1)))          # tr(X^T X) direct
        X_hat = X - H @ W
        p = np.sum(X_hat * X_hat, axis=1)                      # eqn:pi (reading R2)
        sp = float(np.sum(p))
        gamma = math.sqrt(tr_xxt / sp) if sp > 0.0 else 1.0    # eqn:gammat
        state.t += 1
        return PrecondOutput(X_hat, gamma, gamma * gamma * p, updated=False, tr_xxt=tr_xxt)

    # "With updating the Fisher matrix".
    J = H.T @ X
    K = J @ J.T
    if N > D:                                                  # P:1363 (reading R11: strict)
        L = W @ J.T
    else:
        L = H.T @ H

    # E_t, E_t^{0.5}, E_t^{-0.5} and Z_t by eqn:zt:compute.
    e_mhalf = 1.0 / np.sqrt(e)
    dr = d + rho                                               # diag(D_t + rho_t I)
    Kt = e_mhalf[:, None] * K * e_mhalf[None, :]               # E^{-1/2} K E^{-1/2}
    Lt = e_mhalf[:, None] * L * e_mhalf[None, :]               # E^{-1/2} L E^{-1/2}
    Z = ((eta * eta) / (N * N)) * Kt \
        + ((1.0 - eta) ** 2) * np.diag(dr * dr) \
        + (eta * (1.0 - eta) / N) * (Lt * dr[None, :]) \
        + (eta * (1.0 - eta) / N) * (dr[:, None] * Lt)

    c, U = _eigh_descending(Z)                                 # eqn:zt:eig:repeat
    c_floor = ((1.0 - eta) ** 2) * rho * rho                   # P:1125-1128 (reading R13: old rho)
    floored = bool(np.any(c < c_floor))
    floor_margin = float((np.min(c) - c_floor) / np.max(c))
    c = np.maximum(c, c_floor)

    X_hat = X - H @ W
    p = np.sum(X_hat * X_hat, axis=1)                          # eqn:pi
    sp = float(np.sum(p))
    # tr(X X^T): the quantity eqn:gammat and eqn:rhodash2 are defined with, computed by its
    # definition (reading R30).  The paper's shortcut eqn:trxxt is the same
    # number whenever R_t R_t^T = I; it is evaluated and checked here, not used.
    tr_xxt = float(np.sum(np.sum(X * X, axis=1)))
    if check_trace:
        shortcut = sp - float(np.sum(np.diag(L) * e)) + 2.0 * float(np.trace(L))   # eqn:trxxt
        assert abs(shortcut - tr_xxt) <= 1e-8 * max(1.0, abs(tr_xxt)), (shortcut, tr_xxt)
    gamma = math.sqrt(tr_xxt / sp) if sp > 0.0 else 1.0        # eqn:gammat

    sqrt_c = np.sqrt(c)
    rho_dash = ((eta / N) * tr_xxt + (1.0 - eta) * (D * rho + float(np.sum(d)))
                - float(np.sum(sqrt_c))) / (D - R)             # eqn:rhodash2
    d_new = np.maximum(sqrt_c - rho_dash, eps)                 # eqn:dt1, P:1141 (reading R14)
    rho_new = max(eps, rho_dash)                               # eqn:rhot1
    beta_new = beta_of(rho_new, d_new, alpha, D)
    e_new = e_of(beta_new, d_new)

    # W_{t+1} = A_t B_t, eqn:wt1.
    A = (eta / N) * (np.sqrt(e_new)[:, None] * (1.0 / sqrt_c)[:, None] * U.T * e_mhalf[None, :])
    B = J + (N * (1.0 - eta) / eta) * (dr[:, None] * W)
    W_new = A @ B

    # B.3.1 orthogonality check, P:1167-1190 and P:1404-1407 (readings R5, R6).
    cond = float(np.max(c) / np.min(c))
    reorth_checked = floored or cond > 1e6
    reorthogonalized = False
    if reorth_checked:
        W_new, reorthogonalized = _reorthogonalize(W_new, e_new)

    state.W, state.rho, state.d = W_new, rho_new, d_new
    state.t += 1
    return PrecondOutput(X_hat, gamma, gamma * gamma * p, updated=True, floored=floored,
                         reorth_checked=reorth_checked, reorthogonalized=reorthogonalized,
                         tr_xxt=tr_xxt, floor_margin=floor_margin, cond_c=cond)


def _reorthogonalize(W: np.ndarray, e: np.ndarray, tol: float = 1e-3):
    """B.3.1 "Maintaining orthogonality", P:1178-1188 (reading R5: check/repair the
    *new* state with E_{t+1}).  O = E^{-1/2} (W W^T) E^{-1/2}; if any element differs
    from I by more than 1e-3: O = C C^T (Cholesky, lower), M = E^{1/2} C^{-1} E^{-1/2},
    W <- M W.  A non-PD O raises numpy.linalg.LinAlgError (corrupted state)."""
    e_mhalf = 1.0 / np.sqrt(e)
    O = e_mhalf[:, None] * (W @ W.T) * e_mhalf[None, :]
    if float(np.max(np.abs(O - np.eye(O.shape[0])))) <= tol:
        return W, False
    C = np.linalg.cholesky(O)
    M = np.sqrt(e)[:, None] * np.linalg.inv(C) * e_mhalf[None, :]
    return M @ W, True


def reorthogonalize(state: OnlineNgState) -> bool:
    """Apply the B.3.1 check/repair to a state in place; returns True if repaired."""
    beta = beta_of(state.rho, state.d, state.cfg.alpha, state.dim)
    e = e_of(beta, state.d)
    state.W, fixed = _reorthogonalize(state.W, e)
    return fixed


# --------------------------------------------------------------------------------------
# naive defining form (B.1-B.2), explicit D x D matrices
# --------------------------------------------------------------------------------------

def R_of(state: OnlineNgState) -> np.ndarray:
    """R_t = E_t^{-1/2} W_t (inverse of eqn:wt:def)."""
    beta = beta_of(state.rho, state.d, state.cfg.alpha, state.dim)
    e = e_of(beta, state.d)
    return (1.0 / np.sqrt(e))[:, None] * state.W


def F_of(state: OnlineNgState) -> np.ndarray:
    """eqn:low:rank: F_t = R_t^T D_t R_t + rho_t I (D x D)."""
    Rm = R_of(state)
    return Rm.T @ np.diag(state.d) @ Rm + state.rho * np.eye(state.dim)


def precondition_naive(state: OnlineNgState, X: np.ndarray, update: bool | None = None) -> PrecondOutput:
    """The defining equations with explicit D x D matrices (B.1-B.2).

    Apply: G_t = F_t + (alpha tr F_t / D) I; X_hat = beta_t X G_t^{-1}
    (eqn:hatxt) computed with an explicit inverse; gamma by eqn:gammat.
    Update: S_t = X^T X / N; T_t = eta S_t + (1-eta) F_t;
    Y_t = R_t T_t (eqn:yt); Z_t = Y Y^T (eqn:zt:def); Z = U C U^T (eqn:zt:eig);
    floor C at (1-eta)^2 rho^2; R_{t+1} = C^{-1/2} U^T Y (eqn:rt1:def);
    rho' chosen so tr F_{t+1} = tr T_t (eqn:rhodash) -- computed here
    from the explicit trace of T_t; D_{t+1} = max(C^{1/2} - rho', eps);
    rho_{t+1} = max(eps, rho'); W_{t+1} = E_{t+1}^{1/2} R_{t+1}.
    """
    cfg = state.cfg
    X = np.asarray(X, dtype=np.float64)
    N, D = X.shape
    if not state.initialized:
        if float(np.sum(X * X)) == 0.0:
            state.t += 1                                       # reading R7
            return PrecondOutput(X.copy(), 1.0, np.zeros(N))
        init_state(state, X)
    if update is None:
        update = should_update(state.t, cfg)
    R = state.rank
    alpha, eps = cfg.alpha, cfg.epsilon
    F = F_of(state) if R > 0 else state.rho * np.eye(D)
    beta = beta_of(state.rho, state.d if R > 0 else np.zeros(0), alpha, D)
    trF = float(np.trace(F))
    G = F + (alpha * trF / D) * np.eye(D)
    X_hat = beta * X @ np.linalg.inv(G)
    p = np.sum(X_hat * X_hat, axis=1)
    tr_xxt = float(np.trace(X @ X.T))
    sp = float(np.sum(p))
    gamma = math.sqrt(tr_xxt / sp) if sp > 0.0 else 1.0
    out = PrecondOutput(X_hat, gamma, gamma * gamma * p, updated=bool(update), tr_xxt=tr_xxt)
    if not update or R == 0:
        state.t += 1
        return out
    eta = eta_from(N, cfg.s_samples)
    Rm = R_of(state)
    S = X.T @ X / N
    T = eta * S + (1.0 - eta) * F
    Y = Rm @ T
    Z = Y @ Y.T
    c, U = _eigh_descending(Z)
    c_floor = ((1.0 - eta) ** 2) * state.rho ** 2
    out.floored = bool(np.any(c < c_floor))
    c = np.maximum(c, c_floor)
    R_new = np.diag(c ** -0.5) @ U.T @ Y
    rho_dash = (float(np.trace(T)) - float(np.sum(np.sqrt(c)))) / (D - R)
    d_new = np.maximum(np.sqrt(c) - rho_dash, eps)
    rho_new = max(eps, rho_dash)
    beta_new = beta_of(rho_new, d_new, alpha, D)
    e_new = e_of(beta_new, d_new)
    W_new = np.sqrt(e_new)[:, None] * R_new
    cond = float(np.max(c) / np.min(c))
    out.reorth_checked = out.floored or cond > 1e6
    if out.reorth_checked:
        W_new, out.reorthogonalized = _reorthogonalize(W_new, e_new)
    state.W, state.rho, state.d = W_new, rho_new, d_new
    state.t += 1
    return out


def apply_bruteforce(state: OnlineNgState, X: np.ndarray) -> np.ndarray:
    """X_bar = gamma X G^{-1} with G formed explicitly and solved, rescaled to
    ||X_bar||_F = ||X||_F.  Independent of Woodbury."""
    X = np.asarray(X, dtype=np.float64)
    D = X.shape[1]
    F = F_of(state)
    G = F + (state.cfg.alpha * float(np.trace(F)) / D) * np.eye(D)
    Xg = np.linalg.solve(G, X.T).T                              # G symmetric
    nx, ng = np.linalg.norm(X), np.linalg.norm(Xg)
    return Xg * (nx / ng) if ng > 0 else X.copy()
