"""Programmatic dependent launch (ng_common.cuh launch_pdl) must not change any result: the
same config-3-shaped training run (forward, backward, online NG-SGD with refresh steps, update)
with NG_TUNE_PDL=1 and =0 (read once per process, hence subprocesses) gives bit-identical
parameters and objectives.  Also checks the refresh eigensolver never fell back to Jacobi."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import ctypes, hashlib, json, sys
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_1410_7455_b200 import _lib, api
from synth import spliced_frames
N = 512
frames, labels = spliced_frames(5, 16 * N, num_classes=5000)
f = torch.from_numpy(frames).cuda(); y = torch.from_numpy(labels).cuda()
net = api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N, precond=True, rank_in=20, rank_out=80, precision="tf32", seed=7)
objs = []
for k in range(14):
    i = k % 16
    objs.append(net.forward_backward(f[i * N:(i + 1) * N], y[i * N:(i + 1) * N], objective=True))
    net.update(0.01 / 6, 0.075)
h = hashlib.sha256()
for l in range(5):
    h.update(np.ascontiguousarray(net.get_params(l)).tobytes())
z = np.zeros(80 * 80); info = np.zeros(5, dtype=np.int32)
_lib.check(_lib.lib.ng_debug_tri_fail(z.ctypes.data_as(ctypes.c_void_p), info.ctypes.data_as(ctypes.c_void_p)))
print(json.dumps({"hash": h.hexdigest(), "objs": objs, "fallbacks": int(info[1])}))
""".replace("ROOT", repr(ROOT))


def _run(pdl):
    env = dict(os.environ, NG_TUNE_PDL=str(pdl))
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_pdl_bit_identical():
    a, b = _run(1), _run(0)
    assert a["objs"] == b["objs"]
    assert a["hash"] == b["hash"]
    assert a["fallbacks"] == 0
