"""Capture the R = 80 Z_t matrices (eqn:zt:compute) the float64 oracle forms while training the
config-3 network (python tests/tools/capture_zt.py STEPS -> /tmp/zs.pkl), for the eigensolver
prototypes tools/trid_proto.py and tools/tri_proto.py."""
import os, sys, pickle
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from oracle import nnet as onn
from oracle import online_ng as ong
from synth import spliced_frames, standard_normals
Zs = []
orig = ong._eigh_descending
def hook(m):
    if m.shape[0] == 80: Zs.append(m.copy())
    return orig(m)
ong._eigh_descending = hook
cfg = onn.NnetConfig(360, 4, 3000, 10, 5000)
params = onn.init_params(cfg, standard_normals(1410, cfg.layer_shapes()))
states = onn.make_states(cfg, ong.OnlineNgConfig(rank=20), ong.OnlineNgConfig(rank=80))
n = 512
frames, labels = spliced_frames(1410, 16 * n, num_classes=5000)
frames = frames.astype(np.float64)
steps = int(sys.argv[1])
for k in range(steps):
    i = k % 16
    onn.train_step(params, cfg, frames[i*n:(i+1)*n], labels[i*n:(i+1)*n], 0.01/6, states, max_change_per_sample=0.075)
pickle.dump(Zs, open('/tmp/zs.pkl', 'wb'))
print(len(Zs))
