"""Per-step device time of the config-3 training step (CUDA events on the main stream),
to see the cost of update steps (t < 10 or 4 | t) vs plain steps."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1410_7455_b200 import api
from synth import spliced_frames
N = 512
frames, labels = spliced_frames(1410, 64 * N, num_classes=5000)
f = torch.from_numpy(frames).cuda(); y = torch.from_numpy(labels).cuda()
net = api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N, precond=True, rank_in=20, rank_out=80,
               precision=os.environ.get("NG_PREC", "tf32"), seed=1410, renorm=True)
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 40
ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
mid = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
for k in range(steps):
    i = k % 64
    ev[k].record()
    net.forward_backward(f[i * N:(i + 1) * N], y[i * N:(i + 1) * N])
    mid[k].record()
    net.update(0.01 / 6 / 8, 0.075)
ev[steps].record()
torch.cuda.synchronize()
for k in range(steps):
    print(k, f"fb {ev[k].elapsed_time(mid[k]):7.3f} ms  update {mid[k].elapsed_time(ev[k + 1]):7.3f} ms  total {ev[k].elapsed_time(ev[k + 1]):7.3f}")
