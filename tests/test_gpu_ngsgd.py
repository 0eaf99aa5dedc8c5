"""GPU parity of the online NG-SGD preconditioner (libngsgd.so via the C ABI) against
the float64 oracle (oracle/online_ng.py), element by element on the same seeded inputs.

Tolerance (north_star, FP32 path): normwise max|gpu - oracle| / max|oracle| <= 1e-4 on
X_bar = gamma X_hat and on W^T W (sign-free state comparison, reading R12); scalars
(gamma, rho) relative 1e-4; branch flags exactly equal."""
import numpy as np
import pytest

from oracle import online_ng as ong
from synth import gaussian_rows, power_law_rows

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TOL = 1e-4


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_7455_b200 import api
    return api


def normwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def run_gpu(pre, X, update=-1, ld=None):
    """Precondition X (float32 numpy) on the GPU; return (x_hat, gamma, p)."""
    n, D = X.shape
    ld = ld or D
    buf = torch.zeros((n, ld), dtype=torch.float32, device="cuda")
    buf[:, :D] = torch.from_numpy(X.astype(np.float32))
    if ld > D:
        buf[:, D:] = 7.0                         # must not be touched
    g = torch.zeros(1, dtype=torch.float32, device="cuda")
    p = torch.zeros(n, dtype=torch.float32, device="cuda")
    pre.precondition(buf[:, :D] if ld == D else buf.as_strided((n, D), (ld, 1)), g, p, update)
    torch.cuda.synchronize()
    out = buf.cpu().numpy()
    if ld > D:
        assert np.all(out[:, D:] == 7.0)
    return out[:, :D].astype(np.float64), float(g.item()), p.cpu().numpy().astype(np.float64)


def compare_state(pre, s, tol=TOL):
    st = pre.get_state()
    assert st["initialized"] == s.initialized and st["t"] == s.t
    if not s.initialized or s.rank == 0:
        return st
    assert st["rho"] == pytest.approx(s.rho, rel=tol, abs=1e-9)
    assert normwise(st["d"], s.d) <= tol
    W = st["W"].astype(np.float64)
    assert normwise(W.T @ W, s.W.T @ s.W) <= tol
    return st


def inject(pre, s):
    pre.set_state(s.rho, s.d, s.W.astype(np.float32), s.t, s.initialized)


def synthetic_state(D, R, seed, t=10, spread=1e2, d=None, rho=0.3):
    """A valid state (orthonormal R, descending d > 0) from random draws; W = E^{1/2} R."""
    rng = np.random.default_rng(seed)
    q, _ = np.linalg.qr(rng.normal(size=(D, R)))
    s = ong.OnlineNgState(D, ong.OnlineNgConfig(rank=R))
    s.d = np.sort(rng.uniform(1.0, spread, size=s.rank))[::-1].copy() if d is None else np.asarray(d, float)
    s.rho = rho
    e = ong.e_of(ong.beta_of(s.rho, s.d, 4.0, D), s.d)
    s.W = np.sqrt(e)[:, None] * q[:, :s.rank].T
    s.t, s.initialized = t, True
    return s


@pytest.mark.parametrize("N,D,R,steps", [(64, 40, 6, 24), (48, 300, 20, 24), (512, 2000, 80, 12), (512, 2001, 20, 12),
                                         (37, 130, 9, 16)])
def test_trajectory_from_init(api, N, D, R, steps):
    """From an uninitialised state: init on the first minibatch (B.3.2) then the B.5
    policy (update on t < 10 and 4 | t) -- per-step X_bar, gamma, flags and state."""
    batches = power_law_rows(100 + D, N, D, n_batches=steps, nonneg=(D % 2 == 1), append_one=False)
    batches = [b.astype(np.float32).astype(np.float64) for b in batches]
    pre = api.OnlinePreconditioner(D, N, rank=R)
    s = ong.OnlineNgState(D, ong.OnlineNgConfig(rank=R))
    for t, X in enumerate(batches):
        o = ong.precondition(s, X)
        xh, g, p = run_gpu(pre, X)
        assert g == pytest.approx(o.gamma, rel=TOL), t
        assert normwise(g * xh, o.x_bar) <= TOL, t
        assert normwise(p, o.row_sq / o.gamma ** 2) <= TOL, t
        st = compare_state(pre, s)
        assert st["updated"] == o.updated and st["floored"] == o.floored, t


@pytest.mark.parametrize("n", [1, 2, 17, 128])
def test_ragged_rows_and_padded_ld(api, n):
    D, R = 301, 20
    s = synthetic_state(D, R, 5)
    pre = api.OnlinePreconditioner(D, 128, rank=R)
    inject(pre, s)
    for k, upd in enumerate([True, False, True]):
        X = np.abs(gaussian_rows(50 + k, n, D)).astype(np.float32).astype(np.float64)
        o = ong.precondition(s, X, update=upd)
        xh, g, p = run_gpu(pre, X, update=int(upd), ld=304 + 8 * k)
        assert normwise(g * xh, o.x_bar) <= TOL
        compare_state(pre, s)


def test_injected_state_full_config2_sizes(api):
    """Config 2 shapes (512 x 2000, R = 80) from an injected state, forced update and
    non-update steps."""
    D, R, N = 2000, 80, 512
    s = synthetic_state(D, R, 9, spread=1e3)
    pre = api.OnlinePreconditioner(D, N, rank=R)
    inject(pre, s)
    for k, upd in enumerate([True, False, False, True, True]):
        X = power_law_rows(300 + k, N, D)[0].astype(np.float32).astype(np.float64)
        o = ong.precondition(s, X, update=upd)
        xh, g, p = run_gpu(pre, X, update=int(upd))
        assert normwise(g * xh, o.x_bar) <= TOL
        compare_state(pre, s)


def test_non_update_is_pure_and_deterministic(api):
    D, R = 200, 10
    s = synthetic_state(D, R, 2)
    pre = api.OnlinePreconditioner(D, 64, rank=R)
    inject(pre, s)
    before = pre.get_state()
    X = gaussian_rows(7, 64, D).astype(np.float32).astype(np.float64)
    a = run_gpu(pre, X, update=0)
    after = pre.get_state()
    assert np.array_equal(before["W"], after["W"]) and before["rho"] == after["rho"]
    assert np.array_equal(before["d"], after["d"]) and after["t"] == before["t"] + 1
    b = run_gpu(pre, X, update=0)
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]           # bitwise reproducible


def test_rank_zero_identity(api):
    """D = 1 clips R to 0: X_bar = X bit-exactly, gamma = 1 (reading R27)."""
    pre = api.OnlinePreconditioner(1, 16, rank=4)
    X = gaussian_rows(1, 16, 1).astype(np.float32).astype(np.float64)
    xh, g, p = run_gpu(pre, X)
    assert g == 1.0 and np.array_equal(xh, X)


def test_deferred_init_zero_input(api):
    D = 50
    pre = api.OnlinePreconditioner(D, 32, rank=5)
    xh, g, p = run_gpu(pre, np.zeros((32, D)))
    assert g == 1.0 and np.all(xh == 0) and np.all(p == 0)
    assert not pre.get_state()["initialized"]


def test_reorthogonalisation_path(api):
    """A state with cond(C) > 1e6 triggers the B.3.1 check; a 1e-2
    perturbation of W makes max|O - I| > 1e-3, so both sides repair."""
    D, R, N = 120, 8, 64
    rng = np.random.default_rng(3)
    s = synthetic_state(D, R, 4, d=[1e4, 3e3, 1e3, 1e2, 10, 1, 1e-1, 1e-2], rho=1e-4)
    s.W = s.W + 1e-2 * rng.normal(size=s.W.shape) * np.linalg.norm(s.W, axis=1, keepdims=True) / np.sqrt(D)
    pre = api.OnlinePreconditioner(D, N, rank=R)
    inject(pre, s)
    X = (rng.normal(size=(N, D)) * (10.0 ** -np.linspace(0, 4, D))[None, :]).astype(np.float32).astype(np.float64)
    o = ong.precondition(s, X, update=True, check_trace=False)   # R_t not orthonormal here
    xh, g, p = run_gpu(pre, X, update=1)
    st = compare_state(pre, s, tol=1e-3)
    assert o.reorth_checked and st["reorth_checked"]
    assert st["reorthogonalized"] == o.reorthogonalized
    assert normwise(g * xh, o.x_bar) <= TOL


@pytest.mark.parametrize("N,D,R,steps", [(512, 2000, 80, 14), (512, 2001, 20, 14), (130, 300, 20, 12)])
def test_tf32_tensor_core_trajectory(api, N, D, R, steps):
    """NG_TF32: H, J, K, L, X_hat and W_{t+1} on tcgen05 tensor cores (TF32 inputs, FP32
    accumulation; the R x R math stays FP64).  Bar for reduced-precision tensor-core
    inputs (north star): preconditioned output within 2e-2 normwise of the float64 oracle
    at every step of a trajectory from initialisation; state within 2e-2."""
    ld = (D + 3) // 4 * 4
    batches = power_law_rows(700 + D, N, D, n_batches=steps, nonneg=(D % 2 == 1))
    batches = [b.astype(np.float32).astype(np.float64) for b in batches]
    pre = api.OnlinePreconditioner(D, N, rank=R, precision="tf32")
    s = ong.OnlineNgState(D, ong.OnlineNgConfig(rank=R))
    for t, X in enumerate(batches):
        o = ong.precondition(s, X)
        xh, g, p = run_gpu(pre, X, ld=ld)
        assert normwise(g * xh, o.x_bar) <= 2e-2, t
        st = pre.get_state()
        W = st["W"].astype(np.float64)
        assert normwise(W.T @ W, s.W.T @ s.W) <= 2e-2, t
        assert st["updated"] == o.updated
