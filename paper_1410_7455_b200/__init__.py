"""B200-native (sm_100a) hot path of arXiv 1410.7455: the p-norm/softmax DNN training step
with online natural-gradient SGD preconditioning (Appendix B) and periodic parameter
averaging across GPUs (section 3.1).

All computation happens in ``libngsgd.so`` (hand-written CUDA, C ABI in
``include/ngsgd.h``).  This package is the thin Python binding: it marshals torch CUDA
tensors (device memory and streams) into the C calls.  It never imports ``oracle/``.

The binding is loaded lazily so that ``python -m paper_1410_7455_b200.build`` works
before the library exists; any use of the API without the built library raises.
"""
import os as _os

# Every online NG-SGD state runs its refresh chain on its own stream (2 per weight matrix:
# 10 for config 3, 14 for config 5).  With the default 8 hardware work queues, streams 9+
# share a queue with streams 1+ and their chains wait behind unrelated ones (measured: the
# softmax layer's R = 80 refresh started 450 us late).  Must be set before the CUDA context
# exists, i.e. before the first CUDA call of the process; an explicit user setting wins.
_os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")

_API = ("NgError", "Nnet", "NnetStats", "OnlinePreconditioner", "comm_unique_id", "default_ng_config",
        "library_path", "version", "profile_enable", "profile_read", "kernel_launches")


def __getattr__(name):
    if name in _API:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)


__all__ = list(_API)
