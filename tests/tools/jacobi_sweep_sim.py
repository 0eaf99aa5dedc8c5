"""CPU study of the refresh eigensolve: capture the Z_t matrices (eqn:zt:compute) the oracle
forms while training the config-3 network from its C.6 initialisation, then run the
circle-method cyclic Jacobi of eig_jacobi.cuh (in numpy, FP64) under several rotation /
stopping rules and report sweeps and the error of what the update consumes:
sqrt(c) (the new D + rho) and the rows C^{-1/2} U^T of A_t, measured through
G = U diag(sqrt(max(c, floor))) U^T.

    python tools/jacobi_sweep_sim.py [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

from oracle import nnet as onn
from oracle import online_ng as ong
from synth import spliced_frames, standard_normals


RULES = [("rel", 1e-7, 0.0), ("mix", 1e-7, 1e-10), ("mix", 1e-7, 1e-8), ("mix", 1e-7, 1e-6), ("mix", 1e-6, 1e-8),
         ("mix", 1e-5, 1e-8), ("abs", 1e-7, 1.0)]
STATS = {r: {"sweeps": [], "werr": [], "derr": [], "xerr": []} for r in RULES}


def jacobi_desc(Z, rule):
    kind, tol, kappa = rule
    n_sw, c, V = jacobi(Z, tol, kappa)
    order = np.argsort(-c, kind="stable")
    return n_sw, c[order], V[:, order]


def run(steps: int):
    orig_eigh = ong._eigh_descending
    orig_pre = ong.precondition

    def pre(state, X, update=None, check_trace=True):
        if not state.initialized or state.rank != 80:
            return orig_pre(state, X, update, check_trace)
        upd = ong.should_update(state.t, state.cfg) if update is None else update
        if not upd:
            return orig_pre(state, X, update, check_trace)
        ref = state.copy()
        out = orig_pre(ref, X, True, False)
        P0 = ref.W.T @ ref.W
        for rule in RULES:
            st = state.copy()
            box = {}

            def hook(m, rule=rule):
                n_sw, c, V = jacobi_desc(m, rule)
                box["sw"] = n_sw
                return c, V
            ong._eigh_descending = hook
            o2 = orig_pre(st, X, True, False)
            ong._eigh_descending = orig_eigh
            S = STATS[rule]
            S["sweeps"].append(box["sw"])
            S["werr"].append(np.linalg.norm(st.W.T @ st.W - P0) / np.linalg.norm(P0))
            S["derr"].append(np.max(np.abs(st.d - ref.d) / np.maximum(ref.d, 1e-300) * (ref.d > 1e-6 * ref.d.max())))
            # next-minibatch action with the new state (same X as a proxy)
            x1 = X - (X @ ref.W.T) @ ref.W
            x2 = X - (X @ st.W.T) @ st.W
            S["xerr"].append(np.linalg.norm(x2 - x1) / np.linalg.norm(x1))
        state.W, state.rho, state.d, state.t = ref.W, ref.rho, ref.d, ref.t
        return out

    ong.precondition = pre
    onn.online_ng.precondition = pre
    cfg = onn.NnetConfig(360, 4, 3000, 10, 5000)
    params = onn.init_params(cfg, standard_normals(1410, cfg.layer_shapes()))
    states = onn.make_states(cfg, ong.OnlineNgConfig(rank=20), ong.OnlineNgConfig(rank=80))
    n = 512
    frames, labels = spliced_frames(1410, 16 * n, num_classes=5000)
    frames = frames.astype(np.float64)
    for k in range(steps):
        i = k % 16
        onn.train_step(params, cfg, frames[i * n:(i + 1) * n], labels[i * n:(i + 1) * n], 0.01 / 6, states,
                       max_change_per_sample=0.075)
    ong.precondition = orig_pre


def pairs_of_round(r, n):
    npad = n + (n & 1)
    m1 = npad - 1
    out = []
    for k in range(npad // 2):
        if k == 0:
            p, q = m1, r
        else:
            p, q = (r + k) % m1, (r - k) % m1
        p, q = min(p, q), max(p, q)
        if q < n:
            out.append((p, q))
    return out


def jacobi(Z, tol, kappa, max_sweeps=30):
    """Rotate (p, q) when a_pq^2 > tol^2 max(a_pp, kappa zmax) max(a_qq, kappa zmax);
    stop after a sweep with no rotation or whose largest such ratio was below tol."""
    A = Z.copy()
    n = A.shape[0]
    V = np.eye(n)
    zmax = np.max(np.abs(np.diag(A)))
    fl = kappa * zmax
    rounds = [np.array(pairs_of_round(r, n)) for r in range(n + (n & 1) - 1)]
    for sweep in range(max_sweeps):
        nrot, offmax = 0, 0.0
        for pr in rounds:
            p, q = pr[:, 0], pr[:, 1]
            app, aqq, apq = A[p, p], A[q, q], A[p, q]
            scale2 = np.maximum(np.abs(app), fl) * np.maximum(np.abs(aqq), fl)
            rot = (apq * apq > tol * tol * scale2) & (apq * apq > (1e-15 * zmax) ** 2)
            if not rot.any():
                continue
            ratio = np.where(rot, apq * apq / np.maximum(scale2, 1e-300), 0.0)
            offmax = max(offmax, ratio.max())
            nrot += int(rot.sum())
            th = (aqq - app) / (2 * np.where(rot, apq, 1.0))
            t = np.sign(th) / (np.abs(th) + np.sqrt(th * th + 1))
            t = np.where(th == 0, 1.0, t)
            c = 1 / np.sqrt(t * t + 1)
            s = t * c
            c = np.where(rot, c, 1.0)
            s = np.where(rot, s, 0.0)
            J = np.eye(n)
            J[p, p] = c
            J[q, q] = c
            J[p, q] = s
            J[q, p] = -s
            A = J.T @ A @ J
            V = V @ J
        if nrot == 0 or offmax < tol:
            return sweep + 1, np.diag(A).copy(), V
    return max_sweeps, np.diag(A).copy(), V


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    run(steps)
    for rule in RULES:
        S = STATS[rule]
        print(f"{rule[0]:4s} tol={rule[1]:.0e} kappa={rule[2]:.0e}: sweeps mean {np.mean(S['sweeps']):.1f} "
              f"max {max(S['sweeps'])}  |dWtW|/|WtW| max {max(S['werr']):.1e}  d rel err max {max(S['derr']):.1e}  "
              f"X_hat rel err max {max(S['xerr']):.1e}")


if __name__ == "__main__":
    main()
