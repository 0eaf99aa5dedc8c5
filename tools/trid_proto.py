"""Prototype: Householder tridiagonalisation (Q accumulated) + block split + bisection +
twisted-factorisation eigenvectors + V = X Q^T.  Mirrors the planned CUDA order."""
import numpy as np, pickle, sys
EPS = np.finfo(float).eps

def trid(A):
    A = A.copy(); n = A.shape[0]
    Q = np.eye(n); d = np.zeros(n); e = np.zeros(max(n - 1, 0))
    vprev = wprev = None
    # reflector k from column k rows k+1..
    def reflector(x):
        alpha = x[0]; xn = np.linalg.norm(x[1:])
        if xn == 0.0:
            return np.zeros_like(x), 0.0, alpha
        beta = -np.copysign(np.hypot(alpha, xn), alpha)
        tau = (beta - alpha) / beta
        v = x / (alpha - beta); v[0] = 1.0
        return v, tau, beta
    for k in range(n - 2):
        x = A[k + 1:, k]
        v, tau, beta = reflector(x)
        d[k] = A[k, k]; e[k] = beta
        A22 = A[k + 1:, k + 1:]
        p = tau * (A22 @ v)
        w = p - 0.5 * tau * (p @ v) * v
        A[k + 1:, k + 1:] = A22 - np.outer(v, w) - np.outer(w, v)
        # Q <- Q H_k, H_k = I - tau v v^T acting on cols k+1..
        q = Q[:, k + 1:] @ v
        Q[:, k + 1:] -= tau * np.outer(q, v)
    if n >= 2:
        d[n - 2] = A[n - 2, n - 2]; e[n - 2] = A[n - 1, n - 2]
    d[n - 1] = A[n - 1, n - 1]
    return d, e, Q

def sturm(d, e2, lo, hi, x):
    # number of eigenvalues < x of block d[lo:hi]: division-free with rescale
    p0, p1 = 1.0, d[lo] - x
    cnt = 1 if p1 < 0 else 0
    for i in range(lo + 1, hi):
        p = (d[i] - x) * p1 - e2[i - 1] * p0
        if (p < 0) != (p1 < 0) if p != 0 else False: pass
        # sign change counting: sign(p) vs sign(p1), zero takes the opposite of p1 (limit x -> x-)
        s_prev = p1 < 0 if p1 != 0 else True
        s = p < 0 if p != 0 else (not s_prev)
        cnt += (s != s_prev)
        p0, p1 = p1, p
        a = abs(p1)
        if a > 2.0 ** 400 or (a < 2.0 ** -400 and a != 0):
            sc = 2.0 ** -np.floor(np.log2(a)); p0 *= sc; p1 *= sc
    return cnt

def sturm_ratio(d, e2, lo, hi, x, pivmin):
    cnt = 0; q = d[lo] - x
    if abs(q) < pivmin: q = -pivmin
    cnt += q < 0
    for i in range(lo + 1, hi):
        q = (d[i] - x) - e2[i - 1] / q
        if abs(q) < pivmin: q = -pivmin
        cnt += q < 0
    return cnt

def eig_trid(d, e):
    n = len(d)
    tnorm = max(np.max(np.abs(d)), np.max(np.abs(e)) if n > 1 else 0.0)
    e = e.copy()
    # split
    for i in range(n - 1):
        if abs(e[i]) <= EPS * tnorm:   # negligible
            e[i] = 0.0
    blocks = []; s = 0
    for i in range(n - 1):
        if e[i] == 0.0: blocks.append((s, i + 1)); s = i + 1
    blocks.append((s, n))
    e2 = e * e
    pivmin = np.finfo(float).tiny * max(1.0, np.max(e2) if n > 1 else 1.0)
    lam = np.zeros(n); X = np.zeros((n, n)); blk = np.zeros(n, int)
    slot = 0
    for (lo, hi) in blocks:
        nb = hi - lo
        # gershgorin
        gl, gu = np.inf, -np.inf
        for i in range(lo, hi):
            r = (abs(e[i - 1]) if i > lo else 0) + (abs(e[i]) if i < hi - 1 else 0)
            gl = min(gl, d[i] - r); gu = max(gu, d[i] + r)
        bn = max(abs(gl), abs(gu)); gl -= 2 * EPS * bn * nb + 2 * pivmin; gu += 2 * EPS * bn * nb + 2 * pivmin
        for k in range(nb):   # k-th smallest
            a, b = gl, gu
            for it in range(60):
                mid = 0.5 * (a + b)
                if sturm(d, e2, lo, hi, mid) <= k: a = mid
                else: b = mid
            lam[slot] = 0.5 * (a + b)
            blk[slot] = lo * 1000 + hi
            slot += 1
    # eigenvectors by twisted factorisation
    for j in range(n):
        lo, hi = divmod(blk[j], 1000); l = lam[j]
        Dp = np.zeros(n); Dm = np.zeros(n)
        Dp[lo] = d[lo] - l
        for i in range(lo, hi - 1):
            if abs(Dp[i]) < pivmin: Dp[i] = -pivmin
            Dp[i + 1] = d[i + 1] - l - e2[i] / Dp[i]
        if abs(Dp[hi - 1]) < pivmin: Dp[hi - 1] = -pivmin
        Dm[hi - 1] = d[hi - 1] - l
        for i in range(hi - 2, lo - 1, -1):
            if abs(Dm[i + 1]) < pivmin: Dm[i + 1] = -pivmin
            Dm[i] = d[i] - l - e2[i] / Dm[i + 1]
        if abs(Dm[lo]) < pivmin: Dm[lo] = -pivmin
        gam = Dp[lo:hi] + Dm[lo:hi] - (d[lo:hi] - l)
        r = lo + int(np.argmin(np.abs(gam)))
        z = np.zeros(n); z[r] = 1.0
        for i in range(r - 1, lo - 1, -1): z[i] = -(e[i] / Dp[i]) * z[i + 1]
        for i in range(r, hi - 1): z[i + 1] = -(e[i] / Dm[i + 1]) * z[i]
        X[j] = z / np.linalg.norm(z)
    return lam, X, blocks

def eig(Z):
    n = Z.shape[0]
    s = np.max(np.abs(Z)); s = 2.0 ** -np.floor(np.log2(s)) if s > 0 else 1.0
    d, e, Q = trid(Z * s)
    lam, X, blocks = eig_trid(d, e)
    V = X @ Q.T     # rows = eigenvectors of Z
    return lam / s, V, blocks

def check(Z, name):
    lam, V, blocks = eig(Z)
    l0, V0 = np.linalg.eigh(Z)
    zmax = np.max(np.abs(Z))
    o = np.argsort(-lam); lam = lam[o]; V = V[o]
    l0 = l0[::-1]; V0 = V0[:, ::-1]
    orth = np.max(np.abs(V @ V.T - np.eye(len(lam))))
    res = np.max(np.abs(Z @ V.T - V.T * lam)) / zmax
    lerr = np.max(np.abs(lam - l0)) / zmax
    print(f"{name:14s} n={len(lam)} blocks={len(blocks)} orth={orth:.2e} res={res:.2e} lamerr={lerr:.2e}")
    return orth, res

def spd(n, spec, seed):
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.normal(size=(n, n)))
    return (q * spec) @ q.T

if __name__ == "__main__":
    for name, n, spec in [("graded", 80, np.logspace(0, -17, 80)), ("two_clusters", 80, np.r_[np.ones(40), np.full(40, 1e-9)]),
                          ("zeros", 80, np.r_[np.arange(1.0, 72), np.zeros(9)]), ("uniform", 80, np.linspace(1, 2, 80)),
                          ("random_signs", 64, np.random.default_rng(3).normal(size=64)), ("in_side", 20, np.logspace(1, -12, 20)),
                          ("odd", 37, np.logspace(0, -6, 37)), ("tiny", 2, np.array([3.0, 1.0])), ("one", 1, np.array([2.5]))]:
        check(spd(n, spec, n), name)
    check(np.diag(np.r_[np.ones(10), np.full(70, 2.4e-20)]), "diag_degen")
    Zs = pickle.load(open('/tmp/zs.pkl', 'rb'))
    worst = [0, 0]
    for k, Z in enumerate(Zs):
        if k % 10 == 0: o, r = check(Z, f"Z{k}")
