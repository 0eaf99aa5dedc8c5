"""Host-side enqueue time of nnet_forward_backward / nnet_update per config-3 step (no
synchronisation inside the loop), next to the device time per step, to see whether the host
keeps ahead of the GPU.   python tools/host_timeline.py [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_1410_7455_b200 import api
from synth import spliced_frames

N = 512
frames, labels = spliced_frames(1410, 64 * N, num_classes=5000)
f = torch.from_numpy(frames).cuda()
y = torch.from_numpy(labels).cuda()
net = api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N, precond=True, rank_in=20, rank_out=80,
               precision=os.environ.get("NG_PREC", "tf32"), seed=1410, renorm=True)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for k in range(20):
    net.forward_backward(f[(k % 64) * N:(k % 64 + 1) * N], y[(k % 64) * N:(k % 64 + 1) * N])
    net.update(0.01 / 6 / 8, 0.075)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
host = []
for k in range(20, 20 + steps):
    i = k % 64
    ev[k - 20].record()
    t0 = time.perf_counter()
    net.forward_backward(f[i * N:(i + 1) * N], y[i * N:(i + 1) * N])
    t1 = time.perf_counter()
    net.update(0.01 / 6 / 8, 0.075)
    t2 = time.perf_counter()
    host.append((t1 - t0, t2 - t1))
ev[steps].record()
torch.cuda.synchronize()
for k in range(steps):
    print(f"{k + 20} host fb {host[k][0] * 1e3:6.3f} ms  update {host[k][1] * 1e3:6.3f} ms   device step {ev[k].elapsed_time(ev[k + 1]):6.3f} ms")
