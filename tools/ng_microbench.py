"""Micro-benchmark of one online NG-SGD state (configs[1] out side: D=2000, R=80,
N=512) through the C ABI; used for ncu captures of the NG kernels."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1410_7455_b200 import api
from synth import power_law_rows

D = int(os.environ.get("NG_D", 2000)); R = int(os.environ.get("NG_R", 80)); N = 512
steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
xs = [torch.from_numpy(b.astype(np.float32)).cuda() for b in power_law_rows(7, N, D, n_batches=16)]
pre = api.OnlinePreconditioner(D, N, rank=R, precision=os.environ.get("NG_PREC", "fp32"))
w = torch.empty_like(xs[0]); g = torch.zeros(1, device="cuda"); p = torch.zeros(N, device="cuda")
api.profile_enable(["ng_proj", "ng_apply", "ng_refresh", "ng_eig"])
for k in range(steps):
    w.copy_(xs[k % 16])
    pre.precondition(w, g, p, 1 if k % 2 == 0 else 0)
    if k % 2 == 0 and k >= 2:
        stt = pre.get_state()
        print("step", k, "sweeps", stt["jacobi_sweeps"], "reorth", stt["reorth_checked"], stt["reorthogonalized"])
torch.cuda.synchronize()
st = pre.get_state()
print("last update: sweeps", st["jacobi_sweeps"], "reorth_checked", st["reorth_checked"], "repaired", st["reorthogonalized"])
prof = api.profile_read()
for k, v in prof.items():
    if v["launches"]:
        print(f"{k:12s} launches {v['launches']:4d}  {v['ms'] / v['launches'] * 1e3:9.1f} us/launch")
