"""Run the config-3 training loop (bench data) and report how often the refresh eigensolver
fell back to Jacobi; dump the last failing Z_t to gpurun_out/tri_fail.npy for the numpy
prototype (tools/tri_proto.py).   python tools/tri_fail_probe.py [steps]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1410_7455_b200 import _lib, api
from synth import spliced_frames

N = 512
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 100
if os.environ.get("BENCH_POOL"):   # the bench's rank-0 data stream (seed 1410)
    from paper_1410_7455_b200 import driver
    frames, labels = spliced_frames(driver.rank_seed(0), 1 << 18, num_classes=5000)
else:
    frames, labels = spliced_frames(1410, 64 * N, num_classes=5000)
nb = frames.shape[0] // N
f = torch.from_numpy(frames).cuda()
y = torch.from_numpy(labels).cuda()
net = api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N, precond=True, rank_in=20, rank_out=80,
               precision=os.environ.get("NG_PREC", "tf32"), seed=1410)
z = np.zeros(80 * 80)
info = np.zeros(5, dtype=np.int32)
last = 0
for k in range(steps):
    i = k % nb
    net.forward_backward(f[i * N:(i + 1) * N], y[i * N:(i + 1) * N])
    net.update(0.01 / 6, 0.075)
    _lib.check(_lib.lib.ng_debug_tri_fail(z.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.c_void_p)))
    if info[3] > 0 or info[4] // 1000 > 4:
        print("step", k, "max cluster position", info[3], "max RQI-loop iterations", info[4] // 1000, "twisted", info[4] % 1000)
    if info[1] != last:
        print("step", k, "fallbacks", info[1] - last, "reason", info[2], "n", info[0])
        last = info[1]
        n = info[0]
        os.makedirs("gpurun_out", exist_ok=True)
        np.save(f"gpurun_out/tri_fail_{k}.npy", z[:n * n].reshape(n, n).copy())
print("total fallbacks", info[1], "in", steps, "steps")
