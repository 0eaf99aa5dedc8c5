"""B200-native (sm_100a) hot path of arXiv 1410.7455: the p-norm/softmax DNN training step
with online natural-gradient SGD preconditioning (Appendix B) and periodic parameter
averaging across GPUs (section 3.1).

All computation happens in ``libngsgd.so`` (hand-written CUDA, C ABI in
``include/ngsgd.h``).  This package is the thin Python binding: it marshals torch CUDA
tensors (device memory and streams) into the C calls.  It never imports ``oracle/``.

The binding is loaded lazily so that ``python -m paper_1410_7455_b200.build`` works
before the library exists; any use of the API without the built library raises.
"""
_API = ("NgError", "Nnet", "NnetStats", "OnlinePreconditioner", "SimplePreconditioner", "comm_unique_id", "default_ng_config",
        "library_path", "version", "profile_enable", "profile_read", "kernel_launches")


def __getattr__(name):
    if name in _API:
        from . import api
        return getattr(api, name)
    raise AttributeError(name)


__all__ = list(_API)
