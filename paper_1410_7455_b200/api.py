"""Python binding of libngsgd.so: same names as include/ngsgd.h, argument marshalling only.

torch supplies device memory and the CUDA stream; every arithmetic step runs in the
library's kernels.  Tensors passed in must be CUDA float32 / int32, row-major with unit
column stride.
"""
from __future__ import annotations

import ctypes
import dataclasses
from typing import Optional

import numpy as np
import torch

from . import _lib
from ._lib import NgError, check, lib

library_path = _lib.LIB_PATH


def version() -> str:
    return lib.ng_version().decode()


def _stream_handle(stream: Optional[torch.cuda.Stream]) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else int(t.data_ptr())


def _check_matrix(x: torch.Tensor, dtype=torch.float32) -> int:
    if not x.is_cuda or x.dtype != dtype or x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("expected a CUDA %s matrix with unit column stride" % dtype)
    return x.stride(0)


def default_ng_config(rank: int, **overrides) -> _lib.NgsgdConfig:
    """B.4/B.5 defaults: alpha=4, S=2000, J=4, first 10, eps=1e-10."""
    cfg = _lib.NgsgdConfig()
    lib.ngsgd_config_default(ctypes.byref(cfg), int(rank))
    for k, v in overrides.items():
        setattr(cfg, k, v)
    return cfg


class SimplePreconditioner:
    """Simple NG-SGD preconditioner (Appendix A; ngsimple_create / ngsimple_precondition)."""

    def __init__(self, dim: int, max_rows: int, alpha: float = 4.0, stream: Optional[torch.cuda.Stream] = None):
        h = ctypes.c_void_p()
        check(lib.ngsimple_create(int(dim), int(max_rows), float(alpha), _stream_handle(stream), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None):
            lib.ngsimple_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def precondition(self, x: torch.Tensor, gamma: Optional[torch.Tensor] = None,
                     p: Optional[torch.Tensor] = None) -> None:
        """In place: x <- X_hat; gamma[0] <- gamma; p[:n] <- ||x_hat_i||^2 (unscaled)."""
        ld = _check_matrix(x)
        check(lib.ngsimple_precondition(self._h, x.shape[0], _ptr(x), ld, _ptr(gamma), _ptr(p)))

    def read_flags(self) -> None:
        check(lib.ngsimple_read_flags(self._h))


class OnlinePreconditioner:
    """One online NG-SGD state (Appendix B; ngsgd_create / ngsgd_precondition)."""

    def __init__(self, dim: int, max_rows: int, rank: int = 20, stream: Optional[torch.cuda.Stream] = None,
                 _borrowed: Optional[int] = None, precision: str = "fp32", **cfg_overrides):
        self._owned = _borrowed is None
        if _borrowed is not None:
            self._h = ctypes.c_void_p(_borrowed)
            return
        cfg = default_ng_config(rank, precision={"fp32": 0, "tf32": 2, "fp32_simt": 3}[precision], **cfg_overrides)
        h = ctypes.c_void_p()
        check(lib.ngsgd_create(int(dim), int(max_rows), ctypes.byref(cfg), _stream_handle(stream), ctypes.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_owned", False) and self._h:
            lib.ngsgd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def precondition(self, x: torch.Tensor, gamma: Optional[torch.Tensor] = None, p: Optional[torch.Tensor] = None,
                     update: int = -1) -> None:
        """In place: x <- X_hat; gamma[0] <- gamma_t; p[:n] <- p_i (unscaled)."""
        ld = _check_matrix(x)
        check(lib.ngsgd_precondition(self._h, x.shape[0], _ptr(x), ld, _ptr(gamma), _ptr(p), int(update)))

    def join(self) -> None:
        """Make the stream wait for this state's side-stream refresh (ngsgd_join)."""
        check(lib.ngsgd_join(self._h))

    def get_state(self) -> dict:
        st = _lib.NgsgdStateHost()
        check_q = lib.ngsgd_get_state(self._h, ctypes.byref(st))
        R, D = st.rank, st.dim
        d = np.zeros(max(R, 1), dtype=np.float64)
        w = np.zeros((max(R, 1), D), dtype=np.float32)
        st.d = d.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        st.w = w.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        code = lib.ngsgd_get_state(self._h, ctypes.byref(st))
        check(check_q)
        check(code)
        return dict(dim=D, rank=R, t=st.t, initialized=bool(st.initialized), rho=st.rho, d=d[:R].copy(),
                    W=w[:R].copy(), updated=bool(st.last_updated), floored=bool(st.last_floored),
                    reorth_checked=bool(st.last_reorth_checked), reorthogonalized=bool(st.last_reorthogonalized),
                    jacobi_sweeps=int(st.last_jacobi_sweeps))

    def set_state(self, rho: float, d: np.ndarray, W: np.ndarray, t: int, initialized: bool = True) -> None:
        d = np.ascontiguousarray(d, dtype=np.float64)
        W = np.ascontiguousarray(W, dtype=np.float32)
        st = _lib.NgsgdStateHost()
        st.dim = W.shape[1] if W.ndim == 2 and W.shape[0] > 0 else self.get_state()["dim"]
        st.rank = W.shape[0]
        st.t = int(t)
        st.initialized = 1 if initialized else 0
        st.rho = float(rho)
        st.d = d.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        st.w = W.ctypes.data_as(ctypes.POINTER(ctypes.c_float))
        check(lib.ngsgd_set_state(self._h, ctypes.byref(st)))


@dataclasses.dataclass
class NnetStats:
    alpha_t: np.ndarray
    gamma_in: np.ndarray
    gamma_out: np.ndarray
    updated_in: np.ndarray
    updated_out: np.ndarray


class Nnet:
    """p-norm/softmax DNN with online NG-SGD (nnet_create ... nnet_average)."""

    def __init__(self, input_dim: int, num_hidden: int, hidden_dim: int, pnorm_group: int, num_classes: int,
                 max_minibatch: int = 512, precond: bool = True, rank_in: int = 20, rank_out: int = 80,
                 precision: str = "fp32", seed: int = 0, stream: Optional[torch.cuda.Stream] = None,
                 ng_overrides: Optional[dict] = None, renorm: bool = False):
        cfg = _lib.NnetConfig()
        cfg.input_dim, cfg.num_hidden, cfg.hidden_dim = input_dim, num_hidden, hidden_dim
        cfg.pnorm_group, cfg.num_classes, cfg.max_minibatch = pnorm_group, num_classes, max_minibatch
        cfg.precond = {False: 0, True: 1, "none": 0, "online": 1, "simple": 2}[precond]
        prec = {"fp32": 0, "bf16": 1, "tf32": 2, "fp32_simt": 3}[precision]
        cfg.ng_in = default_ng_config(rank_in, **dict({"precision": prec}, **(ng_overrides or {})))
        cfg.ng_out = default_ng_config(rank_out, **dict({"precision": prec}, **(ng_overrides or {})))
        cfg.precision = prec
        cfg.seed = int(seed)
        cfg.renorm = 1 if renorm else 0
        h = ctypes.c_void_p()
        check(lib.nnet_create(ctypes.byref(cfg), _stream_handle(stream), ctypes.byref(h)))
        self._h = h
        self.cfg = cfg
        n = ctypes.c_int32()
        check(lib.nnet_num_layers(h, ctypes.byref(n)))
        self.num_layers = n.value
        self.shapes = []
        for l in range(self.num_layers):
            r, c = ctypes.c_int32(), ctypes.c_int32()
            check(lib.nnet_layer_shape(h, l, ctypes.byref(r), ctypes.byref(c)))
            self.shapes.append((r.value, c.value))

    def close(self):
        if getattr(self, "_h", None):
            lib.nnet_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def forward_backward(self, frames: torch.Tensor, labels: torch.Tensor, objective: bool = False):
        ld = _check_matrix(frames)
        if not labels.is_cuda or labels.dtype != torch.int32:
            raise ValueError("labels must be a CUDA int32 vector")
        out = ctypes.c_double() if objective else None
        check(lib.nnet_forward_backward(self._h, _ptr(frames), ld, _ptr(labels), frames.shape[0],
                                        ctypes.byref(out) if objective else None))
        return out.value if objective else None

    def forward_backward_ex(self, frames: torch.Tensor, labels: torch.Tensor, n: int, rows: Optional[torch.Tensor] = None,
                            lo: Optional[torch.Tensor] = None, step: Optional[torch.Tensor] = None,
                            objective: bool = False):
        """nnet_forward_backward_ex: float32 or uint8-coded frames (C.2 compression, with lo /
        step), optionally gathered by a device row index (a block of the N x M randomisation)."""
        if frames.dtype == torch.uint8:
            fmt = 1
            if lo is None or step is None or lo.dtype != torch.float64 or step.dtype != torch.float64:
                raise ValueError("uint8 frames need float64 lo and step")
        elif frames.dtype == torch.float32:
            fmt = 0
        else:
            raise ValueError("frames must be float32 or uint8")
        if frames.dim() != 2 or frames.stride(1) != 1 or not frames.is_cuda:
            raise ValueError("frames must be a CUDA matrix with unit column stride")
        if rows is not None and (rows.dtype != torch.int32 or not rows.is_cuda):
            raise ValueError("rows must be a CUDA int32 vector")
        if labels.dtype != torch.int32 or not labels.is_cuda:
            raise ValueError("labels must be a CUDA int32 vector")
        inp = _lib.NnetInput(_ptr(frames), fmt, frames.stride(0), _ptr(lo), _ptr(step), _ptr(rows), _ptr(labels))
        out = ctypes.c_double() if objective else None
        check(lib.nnet_forward_backward_ex(self._h, ctypes.byref(inp), int(n),
                                           ctypes.byref(out) if objective else None))
        return out.value if objective else None

    def objective_async(self, host_out: torch.Tensor) -> None:
        """Enqueue the readback of the last forward_backward's objective into a pinned CPU
        float64 tensor (nnet_objective_async); valid once the net's stream gets there."""
        if host_out.is_cuda or host_out.dtype != torch.float64 or host_out.numel() < 1:
            raise ValueError("host_out must be a CPU float64 tensor (pinned)")
        check(lib.nnet_objective_async(self._h, ctypes.c_void_p(host_out.data_ptr())))

    def update(self, lr: float, max_change_per_sample: float = 0.075, stats: bool = False):
        st = _lib.NnetUpdateStats() if stats else None
        check(lib.nnet_update(self._h, float(lr), float(max_change_per_sample), ctypes.byref(st) if stats else None))
        if not stats:
            return None
        L = self.num_layers
        return NnetStats(np.array(st.alpha_t[:L]), np.array(st.gamma_in[:L]), np.array(st.gamma_out[:L]),
                         np.array(st.updated_in[:L]), np.array(st.updated_out[:L]))

    def join(self) -> None:
        """Make the stream wait for all side-stream NG refreshes (nnet_join)."""
        check(lib.nnet_join(self._h))

    def get_params(self, layer: int) -> np.ndarray:
        r, c = self.shapes[layer]
        out = np.empty((r, c), dtype=np.float32)
        check(lib.nnet_get_params(self._h, layer, out.ctypes.data, r * c))
        return out

    def set_params(self, layer: int, w: np.ndarray) -> None:
        r, c = self.shapes[layer]
        w = np.ascontiguousarray(w, dtype=np.float32)
        assert w.shape == (r, c)
        check(lib.nnet_set_params(self._h, layer, w.ctypes.data, r * c))

    def ngsgd(self, layer: int, side: str) -> OnlinePreconditioner:
        h = ctypes.c_void_p()
        check(lib.nnet_get_ngsgd(self._h, layer, {"in": 0, "out": 1}[side], ctypes.byref(h)))
        return OnlinePreconditioner(0, 0, _borrowed=h.value)

    def comm_init(self, unique_id: bytes, rank: int, nranks: int) -> None:
        buf = ctypes.create_string_buffer(bytes(unique_id), len(unique_id))
        check(lib.nnet_comm_init(self._h, buf, int(rank), int(nranks)))

    def average(self, mode: int = 0) -> None:
        check(lib.nnet_average(self._h, int(mode)))

    def arena_size(self) -> int:
        c = ctypes.c_int64()
        check(lib.nnet_arena_size(self._h, ctypes.byref(c)))
        return c.value

    def snapshot(self) -> torch.Tensor:
        """A device copy of the parameter arena (a model of one outer iteration, C.4)."""
        t = torch.empty(self.arena_size(), dtype=torch.float32, device="cuda")
        check(lib.nnet_copy_arena(self._h, _ptr(t), 0))
        return t

    def load_snapshot(self, t: torch.Tensor) -> None:
        check(lib.nnet_copy_arena(self._h, _ptr(t), 1))

    @staticmethod
    def _models(models):
        return (ctypes.c_void_p * len(models))(*[m.data_ptr() for m in models])

    def set_combination(self, models, weights: np.ndarray) -> None:
        """W_l = sum_p weights[l, p] W_l^(p) (nnet_set_combination)."""
        w = np.ascontiguousarray(weights, dtype=np.float32)
        check(lib.nnet_set_combination(self._h, self._models(models), len(models),
                                       w.ctypes.data_as(ctypes.POINTER(ctypes.c_float))))

    def combination_grad(self, models) -> np.ndarray:
        """d objective / d weights[l, p] of the last forward_backward (nnet_combination_grad)."""
        g = np.zeros((self.num_layers, len(models)), dtype=np.float64)
        check(lib.nnet_combination_grad(self._h, self._models(models), len(models),
                                        g.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return g

    def select_best(self, objective: float) -> int:
        """Best-of-n instead of the average after a random initialisation."""
        w = ctypes.c_int32()
        check(lib.nnet_select_best(self._h, float(objective), ctypes.byref(w)))
        return w.value


def compress_frames(x: torch.Tensor):
    """ng_compress_frames: (q uint8, lo float64, step float64) of a CUDA float32 matrix (R36)."""
    ld = _check_matrix(x)
    n, d = x.shape
    q = torch.empty((n, d), dtype=torch.uint8, device=x.device)
    lo = torch.empty(d, dtype=torch.float64, device=x.device)
    step = torch.empty(d, dtype=torch.float64, device=x.device)
    check(lib.ng_compress_frames(n, d, _ptr(x), ld, _ptr(q), d, _ptr(lo), _ptr(step), _stream_handle(None)))
    return q, lo, step


def average_local(nets) -> None:
    """Average several networks living on the current device (nnet_average_local)."""
    arr = (ctypes.c_void_p * len(nets))(*[n._h.value for n in nets])
    check(lib.nnet_average_local(arr, len(nets)))


def profile_enable(groups) -> None:
    """Time every launch of the named kernel groups with CUDA events (ng_profile_enable)."""
    mask = 0
    for g in groups:
        mask |= 1 << _lib.PROF_GROUPS.index(g)
    check(lib.ng_profile_enable(mask))


def profile_read() -> dict:
    st = _lib.ProfileStats()
    check(lib.ng_profile_read(ctypes.byref(st)))
    return {g: dict(launches=int(st.launches[i]), ms=float(st.ms[i]), flops=float(st.flops[i]),
                    bytes=float(st.bytes[i])) for i, g in enumerate(_lib.PROF_GROUPS)}


def kernel_launches() -> int:
    return int(lib.ng_kernel_launches())


def comm_unique_id() -> bytes:
    n = lib.nnet_comm_id_bytes()
    buf = ctypes.create_string_buffer(n)
    check(lib.nnet_comm_get_unique_id(buf))
    return buf.raw
