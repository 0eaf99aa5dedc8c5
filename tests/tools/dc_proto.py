"""NumPy prototype of the refresh eigensolver candidate: Householder tridiagonalisation +
divide-and-conquer (Cuppen tearing, LAPACK-style deflation, secular equation solved for the
offset from the nearer pole, Gu-Eisenstat eigenvectors).  Used to validate the numerics on
the oracle's own Z_t matrices before the CUDA port (tests/tools/jacobi_sweep_sim.py captures them).

    python tools/dc_proto.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np

EPS = np.finfo(np.float64).eps


def householder_tridiag(Z):
    """A = Q T Q^T; returns diag a, off-diagonal e, reflectors (v_k, beta_k)."""
    A = Z.copy()
    n = A.shape[0]
    refl = []
    e = np.zeros(max(n - 1, 0))
    for k in range(n - 2):
        x = A[k, k + 1:].copy()
        sigma = float(x[1:] @ x[1:])
        v = x.copy()
        v[0] = 1.0
        if sigma == 0.0:
            beta = 0.0
            e[k] = x[0]
        else:
            mu = np.sqrt(x[0] * x[0] + sigma)
            v0 = x[0] - mu if x[0] <= 0 else -sigma / (x[0] + mu)
            beta = 2.0 * v0 * v0 / (sigma + v0 * v0)
            v[1:] = x[1:] / v0
            e[k] = mu
        refl.append((v, beta))
        if beta != 0.0:
            S = A[k + 1:, k + 1:]
            p = beta * (S @ v)
            K = 0.5 * beta * float(p @ v)
            w = p - K * v
            S -= np.outer(v, w) + np.outer(w, v)
    a = np.diag(A).copy()
    if n >= 2:
        e[n - 2] = A[n - 2, n - 1]
    return a, e, refl


def apply_q(refl, M):
    """Q M for Q = H_0 H_1 ... H_{n-3} (H_k acts on rows k+1..)."""
    M = M.copy()
    for k in reversed(range(len(refl))):
        v, beta = refl[k]
        if beta == 0.0:
            continue
        S = M[k + 1:, :]
        w = v @ S
        S -= beta * np.outer(v, w)
    return M


def secular_root(d, z, rho, j, K):
    """Root j of 1 + rho sum z_i^2/(d_i - lam) = 0, d ascending (K entries).  Returns
    (origin index, tau) with lam = d[origin] + tau."""
    if j < K - 1:
        gap = d[j + 1] - d[j]
        mid = 0.5 * gap
        fmid = 1.0 + rho * np.sum(z * z / ((d - d[j]) - mid))
        if fmid >= 0:
            o, lo, hi = j, 0.0, mid
        else:
            o, lo, hi = j + 1, -mid, 0.0
    else:
        o = K - 1
        lo, hi = 0.0, rho * float(z @ z)
    delta = d - d[o]
    # bisection then safeguarded Newton
    tau = 0.5 * (lo + hi)
    for it in range(200):
        den = delta - tau
        f = 1.0 + rho * np.sum(z * z / den)
        if f > 0:
            hi = tau
        else:
            lo = tau
        fp = rho * np.sum(z * z / (den * den))
        if it < 4:
            tn = 0.5 * (lo + hi)
        else:
            tn = tau - f / fp
            if not (lo < tn < hi):
                tn = 0.5 * (lo + hi)
        if abs(tn - tau) <= 2 * EPS * max(abs(tn), 1e-300) or hi - lo <= 2 * EPS * max(abs(lo), abs(hi)):
            tau = tn
            break
        tau = tn
    return o, tau


def merge(dL, QL, dR, QR, rho_signed):
    """Eigen of [T1 0; 0 T2] + rho v v^T given T1 = QL diag(dL) QL^T etc."""
    nl, nr = len(dL), len(dR)
    k = nl + nr
    rho = abs(rho_signed)
    sgn = 1.0 if rho_signed >= 0 else -1.0
    Q = np.zeros((k, k))
    Q[:nl, :nl] = QL
    Q[nl:, nl:] = QR
    z = np.concatenate([QL[nl - 1, :], sgn * QR[0, :]])
    d = np.concatenate([dL, dR])
    # normalise z (norm sqrt 2): rho *= |z|^2
    zn = np.linalg.norm(z)
    z = z / zn
    rho = rho * zn * zn
    order = np.argsort(d, kind="stable")
    d = d[order]
    z = z[order]
    Q = Q[:, order]
    tol = 8.0 * EPS * max(np.max(np.abs(d)), rho * np.max(np.abs(z)), 1e-300)
    defl = np.zeros(k, bool)
    # type 1
    defl |= rho * np.abs(z) <= tol
    # type 2: consecutive non-deflated pairs with close d
    prev = -1
    for i in range(k):
        if defl[i]:
            continue
        if prev >= 0:
            r = np.hypot(z[prev], z[i])
            c, s = z[i] / r, -z[prev] / r
            if abs((d[i] - d[prev]) * c * s) <= tol:
                # rotate (prev, i) so z[prev] = 0: deflate prev
                t = d[prev] * c * c + d[i] * s * s
                d[i] = d[prev] * s * s + d[i] * c * c
                d[prev] = t
                z[i] = r
                z[prev] = 0.0
                qp, qi = Q[:, prev].copy(), Q[:, i].copy()
                Q[:, prev] = c * qp + s * qi
                Q[:, i] = -s * qp + c * qi
                defl[prev] = True
        prev = i
    nd = np.where(~defl)[0]
    K = len(nd)
    lam = d.copy()
    V = np.eye(k)
    if K > 0:
        dk, zk = d[nd], z[nd]
        roots = [secular_root(dk, zk, rho, j, K) for j in range(K)]
        # Gu-Eisenstat zhat: prod_j (lam_j - d_i) = rho zhat_i^2 prod_{j != i} (d_j - d_i)
        zh = np.zeros(K)
        for i in range(K):
            num = 1.0
            for j in range(K):
                o, tau = roots[j]
                lam_minus_di = (dk[o] - dk[i]) + tau
                num *= lam_minus_di
                if j != i:
                    num /= (dk[j] - dk[i])
            zh[i] = np.copysign(np.sqrt(max(num / rho, 0.0)), zk[i])
        Vk = np.zeros((K, K))
        for j in range(K):
            o, tau = roots[j]
            col = zh / ((dk - dk[o]) - tau)
            Vk[:, j] = col / np.linalg.norm(col)
            lam[nd[j]] = dk[o] + tau
        V[np.ix_(nd, nd)] = Vk
    Qn = Q @ V
    o2 = np.argsort(lam, kind="stable")
    return lam[o2], Qn[:, o2]


def tridiag_dc(a, e):
    """Eigen of the symmetric tridiagonal (a, e) by bottom-up D&C from 1x1 leaves."""
    n = len(a)
    a = a.copy()
    rhos = []
    for b in range(1, n):   # tear every boundary
        r = e[b - 1]
        a[b - 1] -= abs(r)
        a[b] -= abs(r)
        rhos.append(r)
    blocks = [(i, i + 1, np.array([a[i]]), np.eye(1)) for i in range(n)]
    while len(blocks) > 1:
        nb = []
        for t in range(0, len(blocks) - 1, 2):
            (l0, s, dL, QL), (s2, r1, dR, QR) = blocks[t], blocks[t + 1]
            lam, Q = merge(dL, QL, dR, QR, rhos[s - 1])
            nb.append((l0, r1, lam, Q))
        if len(blocks) % 2:
            nb.append(blocks[-1])
        blocks = nb
    return blocks[0][2], blocks[0][3]


def eig_hdc(Z):
    a, e, refl = householder_tridiag(Z)
    lam, Qt = tridiag_dc(a, e)
    U = apply_q(refl, Qt)
    return lam, U


def main():
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    import jacobi_sweep_sim as J
    from oracle import online_ng as ong
    Zs = []
    orig = ong._eigh_descending

    def hook(m):
        if m.shape[0] in (80, 20):
            Zs.append(m.copy())
        return orig(m)
    ong._eigh_descending = hook
    J.RULES = []
    J.run(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
    ong._eigh_descending = orig
    rng = np.random.default_rng(0)
    Zs += [(lambda q, l: (q * l) @ q.T)(np.linalg.qr(rng.normal(size=(80, 80)))[0], l)
           for l in (np.logspace(0, -17, 80), np.r_[np.ones(40), np.full(40, 1e-9)], np.r_[np.arange(1, 71.), np.zeros(10)])]
    worst = 0
    for Z in Zs:
        lam, U = eig_hdc(Z)
        zmax = np.max(np.abs(np.diag(Z)))
        orth = np.max(np.abs(U.T @ U - np.eye(len(lam))))
        resid = np.max(np.abs(Z @ U - U * lam)) / zmax
        l0 = np.linalg.eigvalsh(Z)
        lerr = np.max(np.abs(np.sort(lam) - l0)) / zmax
        worst = max(worst, orth, resid, lerr)
        print(f"n={len(lam)} orth {orth:.1e} resid/zmax {resid:.1e} lam err/zmax {lerr:.1e}")
    print("worst", worst)


if __name__ == "__main__":
    main()
