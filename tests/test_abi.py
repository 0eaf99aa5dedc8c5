"""The C-ABI library loads on a CPU-only host and exports every symbol include/ngsgd.h
declares; the ctypes binding declares exactly those symbols.  No compute calls."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "ngsgd.h")


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b((?:ng|ngsgd|ngsimple|nnet)_[a-z0-9_]+)\s*\(", src)))


def _lib_path():
    from paper_1410_7455_b200 import build
    return build.build(verbose=False)


def test_header_parses():
    names = _declared()
    assert "ngsgd_precondition" in names and "nnet_average" in names and len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_lib_path())
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_header():
    _lib_path()
    from paper_1410_7455_b200 import _lib
    assert sorted(_lib.SIGNATURES) == _declared()


def test_host_side_errors_without_gpu():
    """Argument validation happens on the host before any launch (include/ngsgd.h)."""
    _lib_path()
    from paper_1410_7455_b200 import _lib
    lib = _lib.lib
    assert lib.ng_version().startswith(b"libngsgd")
    cfg = _lib.NgsgdConfig()
    lib.ngsgd_config_default(ctypes.byref(cfg), 80)
    assert (cfg.rank, cfg.alpha, cfg.s_samples, cfg.update_period, cfg.always_update_first) == (80, 4.0, 2000.0, 4, 10)
    assert cfg.epsilon == pytest.approx(1e-10)
    h = ctypes.c_void_p()
    assert lib.ngsgd_create(0, 10, ctypes.byref(cfg), None, ctypes.byref(h)) == 2      # NG_ESHAPE
    assert lib.ngsgd_precondition(None, 1, None, 1, None, None, -1) == 1                # NG_EINVAL
    assert b"NULL" in lib.ng_last_error()
    assert lib.nnet_comm_id_bytes() == 128
