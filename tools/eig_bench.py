"""Cycles of the refresh eigensolver eig_tri on Z_t-shaped matrices (tests/test_gpu_eig._zt_like),
one CTA, clock64 inside the kernel (phase stamps of thread 0).

    python tools/eig_bench.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_eig import _zt_like  # noqa: E402
import ctypes  # noqa: E402
from paper_1410_7455_b200 import _lib  # noqa: E402


def _run_tri(Z):
    """ng_debug_eig_tri with the finer phase-2 stamps requested (ok[8] = 0x5eed on entry)."""
    n = Z.shape[0]
    z = torch.from_numpy(np.ascontiguousarray(Z, dtype=np.float64)).cuda()
    lam = torch.empty(n, dtype=torch.float64, device="cuda")
    vt = torch.empty(n, n, dtype=torch.float64, device="cuda")
    ok = torch.zeros(16, dtype=torch.int32, device="cuda")
    ok[8] = 0x5eed
    _lib.check(_lib.lib.ng_debug_eig_tri(ctypes.c_void_p(z.data_ptr()), n, ctypes.c_void_p(lam.data_ptr()),
                                         ctypes.c_void_p(vt.data_ptr()), ctypes.c_void_p(ok.data_ptr()), None))
    torch.cuda.synchronize()
    return lam.cpu().numpy(), vt.cpu().numpy(), ok.cpu().numpy()


for n, dec in [(80, 10.0), (80, 18.0), (80, 4.0), (20, 10.0)]:
    cyc, oks, orth, ph, its, fine = [], [], float('nan'), [], [], []
    for s in range(8):
        Z = _zt_like(n, seed=100 + s, decades=dec)
        lam, vt, ok = _run_tri(Z)
        fine.append(ok[8:14]); cyc.append(ok[1]); oks.append(ok[0]); ph.append(ok[2:8]); its.append(ok[5] % 1000)
        if ok[0]:
            orth = np.max(np.abs(vt @ vt.T - np.eye(n)))
    print(f"n={n} decades={dec:4.1f}: tri {np.median(cyc) / 1.965e3:7.1f} us (median of 8, 1.965 GHz)  ok {sum(oks)}/8  "
          f"last orth {orth:.1e}  max twisted solves {max(its)}\n   phases (us): tridiagonalise %.1f  eigenpairs of T %.1f "
          "(multisection %.1f, RQI + vectors + clusters %.1f)  orthogonality check %.1f" % tuple(
              np.median(np.array(ph), axis=0)[[0, 1, 4, 5, 2]] / 1.965e3))
    print("   phase 2 detail (us): split %.1f  root repr %.1f  coarse %.1f  RQI + twisted %.1f  clusters %.1f  "
          "slowest RQI loop %.1f" % tuple(np.median(np.array(fine), axis=0) / 1.965e3))
