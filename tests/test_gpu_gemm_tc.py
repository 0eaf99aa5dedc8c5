"""Unit parity of the tcgen05 TF32 GEMM core (ng_debug_gemm_tf32) against a float64
matmul of the same FP32 inputs: every operand major-ness, both tile widths, split-K,
ragged edges (M, N, K not multiples of the 128 x BN x 32 tile).  TF32 keeps 10 mantissa
bits, so the bar is normwise 5e-3 (a layout/descriptor bug gives O(1) errors)."""
import ctypes

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_7455_b200 import _lib
    return _lib


def run(lib, A, B, a_k, b_k, bn, splits, split3=0):
    """A: M x K, B: K x N (numpy float32). Layouts per include/ngsgd.h."""
    M, K = A.shape
    N = B.shape[1]
    def dev(mat):
        rows, cols = mat.shape
        ld = (cols + 3) // 4 * 4
        t = torch.zeros((rows, ld), dtype=torch.float32, device="cuda")
        t[:, :cols] = torch.from_numpy(np.ascontiguousarray(mat))
        return t, ld
    ta, lda = dev(A if a_k else A.T)        # a_k: [M][K]; else stored [K][M]
    tb, ldb = dev(B.T if b_k else B)        # b_k: [N][K]; else stored [K][N]
    ldc = N + 5
    tc = torch.full((M, ldc), -7.0, dtype=torch.float32, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    lib.check(lib.lib.ng_debug_gemm_tc(M, N, K, ta.data_ptr(), lda, int(a_k), tb.data_ptr(), ldb, int(b_k),
                                       tc.data_ptr(), ldc, bn, splits, int(split3), st))
    torch.cuda.synchronize()
    out = tc.cpu().numpy()
    assert np.all(out[:, N:] == -7.0)            # nothing written outside C
    return out[:, :N].astype(np.float64)


@pytest.mark.parametrize("a_k", [True, False])
@pytest.mark.parametrize("b_k", [True, False])
@pytest.mark.parametrize("bn", [64, 128])
@pytest.mark.parametrize("M,N,K,splits", [(37, 70, 45, 1), (128, 128, 32, 1), (300, 200, 129, 1),
                                          (512, 300, 3000, 6), (130, 65, 1, 1)])
def test_tf32_gemm(lib, a_k, b_k, bn, M, N, K, splits):
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(K, N)).astype(np.float32)
    C = run(lib, A, B, a_k, b_k, bn, splits)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    err = np.max(np.abs(C - ref)) / np.max(np.abs(ref))
    assert err <= 5e-3, err


def test_tf32_gemm_is_deterministic(lib):
    rng = np.random.default_rng(5)
    A = rng.normal(size=(512, 361)).astype(np.float32)
    B = rng.normal(size=(361, 3000)).astype(np.float32)
    c1 = run(lib, A, B, True, True, 128, 1)
    c2 = run(lib, A, B, True, True, 128, 1)
    assert np.array_equal(c1, c2)


@pytest.mark.parametrize("a_k", [True, False])
@pytest.mark.parametrize("b_k", [True, False])
@pytest.mark.parametrize("bn", [32, 128])
@pytest.mark.parametrize("M,N,K,splits", [(37, 70, 45, 1), (300, 200, 129, 1), (512, 80, 3000, 4), (130, 65, 1, 1)])
def test_3xtf32_gemm(lib, a_k, b_k, bn, M, N, K, splits):
    """3xTF32 (split3): FP32-grade products on the tensor cores.  Against the float64
    product of the same FP32 inputs, normwise 1e-5: FP32 accumulation over K = 3000 alone
    costs ~3e-6 here (sqrt(K) eps), a dropped correction term leaves ~1e-3 (plain TF32)."""
    rng = np.random.default_rng(M * 5 + N * 11 + K)
    A = rng.normal(size=(M, K)).astype(np.float32)
    B = rng.normal(size=(K, N)).astype(np.float32)
    C = run(lib, A, B, a_k, b_k, bn, splits, split3=1)
    ref = A.astype(np.float64) @ B.astype(np.float64)
    err = np.max(np.abs(C - ref)) / np.max(np.abs(ref))
    assert err <= 1e-5, err
