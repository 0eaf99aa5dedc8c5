"""MRRR-lite prototype: Householder T (from trid_proto), relative split, PD LDL^T root
representation per block, per-eigenvalue bisection + safeguarded RQI on the twisted
factorisation, eigenvector from the twist.  No cluster recursion; orthogonality checked."""
import numpy as np, pickle, sys
sys.path.insert(0, __import__('os').path.dirname(__file__))
from trid_proto import trid, spd
EPS = np.finfo(float).eps
TINY = np.finfo(float).tiny

def ldl(d, e, sigma):
    n = len(d); D = np.zeros(n); L = np.zeros(max(n - 1, 0))
    D[0] = d[0] - sigma
    for i in range(n - 1):
        if not D[i] > 0: return None, None
        L[i] = e[i] / D[i]
        D[i + 1] = d[i + 1] - sigma - L[i] * e[i]
    if not D[n - 1] > 0: return None, None
    return D, L

def twisted(D, L, lam, want_vec):
    n = len(D); pivmin = TINY * 1e10
    s = np.zeros(n); Dp = np.zeros(n); Lp = np.zeros(max(n - 1, 0))
    neg = 0
    s[0] = -lam
    for i in range(n - 1):
        Dp[i] = D[i] + s[i]
        if abs(Dp[i]) < pivmin: Dp[i] = -pivmin
        neg += Dp[i] < 0
        Lp[i] = D[i] * L[i] / Dp[i]
        s[i + 1] = Lp[i] * L[i] * s[i] - lam
    Dp[n - 1] = D[n - 1] + s[n - 1]
    if abs(Dp[n - 1]) < pivmin: Dp[n - 1] = -pivmin
    neg += Dp[n - 1] < 0
    if not want_vec: return neg, None, None, None
    p = np.zeros(n); Um = np.zeros(max(n - 1, 0))
    p[n - 1] = D[n - 1] - lam
    for i in range(n - 2, -1, -1):
        Dm = D[i] * L[i] * L[i] + p[i + 1]
        if abs(Dm) < pivmin: Dm = -pivmin
        t = D[i] / Dm
        Um[i] = L[i] * t
        p[i] = p[i + 1] * t - lam
    gam = s + p + lam
    r = int(np.argmin(np.abs(gam)))
    z = np.zeros(n); z[r] = 1.0
    for i in range(r - 1, -1, -1): z[i] = -Lp[i] * z[i + 1]
    for i in range(r, n - 1): z[i + 1] = -Um[i] * z[i]
    return neg, z, gam[r], float(z @ z)

def block_eig(D, L, passes):
    n = len(D)
    # Gershgorin upper bound of LDL^T (tridiagonal: diag D_i + D_{i-1} L_{i-1}^2, off D_i L_i)
    dg = D.copy(); dg[1:] += D[:-1] * L * L
    off = np.abs(D[:-1] * L) if n > 1 else np.zeros(0)
    rad = np.zeros(n); rad[:-1] += off; rad[1:] += off
    gu = float(np.max(dg + rad)) * (1 + 4 * n * EPS)
    lams = np.zeros(n); Z = np.zeros((n, n)); cnt = 0
    if n == 1:
        return D.copy(), np.ones((1, 1))
    for j in range(n):           # j-th smallest
        a, b = gu * 1e-300, gu
        na, nb = 0, n
        lam_c = None; it = 0; z = None
        while True:
            it += 1
            rqi = (na == j and nb == j + 1 and (b - a) <= 0.5 * a)
            if rqi and lam_c is not None and a < lam_c < b: lam = lam_c
            elif b > 4 * a: lam = np.sqrt(a * b)
            else: lam = 0.5 * (a + b)
            neg, zz, g, nz = twisted(D, L, lam, rqi)
            passes[0] += 3 if rqi else 1
            if neg <= j: a, na = lam, neg
            else: b, nb = lam, neg
            if rqi:
                z, lam_c = zz, lam + g / nz
                if abs(g / nz) <= 4 * EPS * lam or (b - a) <= 4 * EPS * a:
                    lams[j] = lam; break
            if it > 200:
                print("  noconv", j, a, b); lams[j] = lam
                if z is None: z = twisted(D, L, lam, True)[1]
                break
        Z[j] = z / np.linalg.norm(z)
    return lams, Z

def eig(Zm, passes):
    n = Zm.shape[0]
    sc = np.max(np.abs(Zm)); sc = 2.0 ** -np.floor(np.log2(sc)) if sc > 0 else 1.0
    d, e, Q = trid(Zm * sc)
    e = e.copy()
    tn0 = max(np.max(np.abs(d)), np.max(np.abs(e)) if n > 1 else 0)
    for i in range(n - 1):
        if abs(e[i]) <= EPS * np.sqrt(abs(d[i]) * abs(d[i + 1])) or abs(e[i]) <= 2 * EPS * tn0: e[i] = 0.0
    blocks = []; s0 = 0
    for i in range(n - 1):
        if e[i] == 0.0: blocks.append((s0, i + 1)); s0 = i + 1
    blocks.append((s0, n))
    tn = max(np.max(np.abs(d)), np.max(np.abs(e)) if n > 1 else 0)
    lam = np.zeros(n); X = np.zeros((n, n)); k = 0
    for lo, hi in blocks:
        sig = 0.0
        while True:
            D, L = ldl(d[lo:hi], e[lo:hi - 1], sig)
            if D is not None: break
            sig = -4 * n * EPS * tn if sig == 0.0 else 2 * sig
        lb, Xb = block_eig(D, L, passes)
        lam[k:k + hi - lo] = lb + sig
        X[k:k + hi - lo, lo:hi] = Xb
        k += hi - lo
    V = X @ Q.T
    return lam / sc, V, blocks

def check(Zm, name):
    passes = [0]
    lam, V, blocks = eig(Zm, passes)
    n = len(lam)
    l0, V0 = np.linalg.eigh(Zm)
    zmax = np.max(np.abs(Zm))
    o = np.argsort(-lam); lam = lam[o]; V = V[o]; l0 = l0[::-1]
    orth = np.max(np.abs(V @ V.T - np.eye(n)))
    res = np.max(np.abs(Zm @ V.T - V.T * lam)) / zmax
    lerr = np.max(np.abs(lam - l0)) / zmax
    print(f"{name:14s} n={n} blocks={len(blocks)} orth={orth:.2e} res={res:.2e} lamerr={lerr:.2e} passes/eig={passes[0]/n:.1f}")

if __name__ == "__main__":
    for name, n, spec in [("graded", 80, np.logspace(0, -17, 80)), ("two_clusters", 80, np.r_[np.ones(40), np.full(40, 1e-9)]),
                          ("zeros", 80, np.r_[np.arange(1.0, 72), np.zeros(9)]), ("uniform", 80, np.linspace(1, 2, 80)),
                          ("random_signs", 64, np.random.default_rng(3).normal(size=64)), ("in_side", 20, np.logspace(1, -12, 20)),
                          ("odd", 37, np.logspace(0, -6, 37)), ("tiny", 2, np.array([3.0, 1.0])), ("one", 1, np.array([2.5]))]:
        check(spd(n, spec, n), name)
    check(np.diag(np.r_[np.ones(10), np.full(70, 2.4e-20)]), "diag_degen")
    Zs = pickle.load(open('/tmp/zs.pkl', 'rb'))
    for k, Z in enumerate(Zs):
        if k % 8 == 0: check(Z, f"Z{k}")

def stat_solve(D, L, lam, b):
    """(L D L^T - lam I) y = b via the stationary factorisation L+ D+ L+^T."""
    n = len(D); pivmin = TINY * 1e10
    s = -lam; Dp = np.zeros(n); Lp = np.zeros(max(n - 1, 0))
    for i in range(n - 1):
        Dp[i] = D[i] + s
        if abs(Dp[i]) < pivmin: Dp[i] = -pivmin
        Lp[i] = D[i] * L[i] / Dp[i]
        s = Lp[i] * L[i] * s - lam
    Dp[n - 1] = D[n - 1] + s
    if abs(Dp[n - 1]) < pivmin: Dp[n - 1] = -pivmin
    y = b.copy()
    for i in range(n - 1): y[i + 1] -= Lp[i] * y[i]
    y /= Dp
    for i in range(n - 2, -1, -1): y[i] -= Lp[i] * y[i + 1]
    return y

def block_eig_cl(D, L, passes, ctol=1e-5):
    lams, Z = block_eig(D, L, passes)
    n = len(D)
    # clusters of consecutive eigenvalues with relgap < ctol; redo members after the first
    j = 0
    while j < n:
        k = j
        while k + 1 < n and abs(lams[k + 1] - lams[k]) <= ctol * abs(lams[k]): k += 1
        for m in range(j + 1, k + 1):
            rng = np.random.default_rng(m)
            y = rng.uniform(-1, 1, n)
            for it in range(2):
                y = stat_solve(D, L, lams[m], y)
                for q in range(j, m): y -= (Z[q] @ y) * Z[q]
                for q in range(j, m): y -= (Z[q] @ y) * Z[q]
                y /= np.linalg.norm(y)
            Z[m] = y
        j = k + 1
    return lams, Z

block_eig_orig = block_eig
