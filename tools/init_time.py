"""Wall time of the NG-SGD initialisations (B.3.2) of the config-3 network: the first
minibatches initialise the 10 states (host-synchronising, once per process)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1410_7455_b200 import api
from synth import spliced_frames
N = 512
f, y = spliced_frames(1410, 4 * N, num_classes=5000)
f, y = torch.from_numpy(f).cuda(), torch.from_numpy(y).cuda()
net = api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N, precond=True, rank_in=20, rank_out=80, precision="tf32",
               seed=1410, renorm=True)
api.profile_enable(["ng_init"])
torch.cuda.synchronize()
t0 = time.time()
for k in range(3):
    net.forward_backward(f[k * N:(k + 1) * N], y[k * N:(k + 1) * N])
    net.update(0.0002, 0.075)
torch.cuda.synchronize()
p = api.profile_read()["ng_init"]
print(f"3 steps incl. the initialisation of all 10 NG states: {time.time() - t0:.3f} s; "
      f"ng_init {p['launches']} inits, {p['ms']:.1f} ms device time")
