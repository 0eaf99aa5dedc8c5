"""Where the refresh chains sit in the config-3 step: device-clock start / end of every
refresh_kernel launch (ng_debug_refresh_times) against the main-stream step boundaries
(globaltimer stamps are taken with a tiny kernel-free trick: torch events give relative ms,
so the refresh times are printed relative to the first refresh of each update step).

    python tools/refresh_timeline.py [steps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1410_7455_b200 import _lib, api
from synth import spliced_frames

N = 512
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
frames, labels = spliced_frames(1410, 64 * N, num_classes=5000)
f = torch.from_numpy(frames).cuda()
y = torch.from_numpy(labels).cuda()
net = api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N, precond=True, rank_in=20, rank_out=80,
               precision=os.environ.get("NG_PREC", "tf32"), seed=1410, renorm=True)
buf = np.zeros(256 * 9, dtype=np.uint64)
cnt = np.zeros(1, dtype=np.int32)
seen = 0
for k in range(steps):
    i = k % 64
    net.forward_backward(f[i * N:(i + 1) * N], y[i * N:(i + 1) * N])
    net.update(0.01 / 6 / 8, 0.075)
    if k >= 20:
        _lib.check(_lib.lib.ng_debug_refresh_times(buf.ctypes.data_as(ctypes.c_void_p), cnt.ctypes.data_as(ctypes.c_void_p)))
        c = int(cnt[0])
        if c > seen:
            rows = [buf[(s % 256) * 9:(s % 256) * 9 + 9] for s in range(seen, c)]
            t0 = min(int(r[1]) for r in rows)
            print(f"step {k}: " + "  ".join(f"R{int(r[0]) & 0xffff}D{int(r[0]) >> 16}:{(int(r[1]) - t0) / 1e3:.0f}-{(int(r[2]) - t0) / 1e3:.0f}us"
                                           f"(eig {(int(r[4]) - int(r[3])) / 1e3:.0f}: tri {int(r[5]) / 1965:.0f} "
                                           f"msect {int(r[6]) / 1965:.0f} rqi {int(r[7]) / 1965:.0f} rest {int(r[8]) / 1965:.0f})"
                                           for r in sorted(rows, key=lambda r: int(r[1]))))
            seen = c
