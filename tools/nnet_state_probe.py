"""Probe the NG states of the config-3 network during training: per update step, which
states triggered the B.3.1 check / repair and how many Jacobi sweeps they used."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1410_7455_b200 import api
from synth import spliced_frames
prec = os.environ.get("NG_PREC", "tf32")
N = 512
frames, labels = spliced_frames(1410, 64 * N, num_classes=5000)
f = torch.from_numpy(frames).cuda(); y = torch.from_numpy(labels).cuda()
net = api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N, precond=True, rank_in=20, rank_out=80, precision=prec, seed=1410, renorm=os.environ.get("NG_RENORM", "1") == "1")
for k in range(int(sys.argv[1]) if len(sys.argv) > 1 else 30):
    i = k % 64
    net.forward_backward(f[i * N:(i + 1) * N], y[i * N:(i + 1) * N])
    st = net.update(0.01 / 6, 0.075, stats=True)
    row = []
    for l in range(5):
        for side in ("in", "out"):
            s = net.ngsgd(l, side).get_state()
            if s["updated"]:
                W, d, rho = s["W"].astype(np.float64), s["d"], s["rho"]
                D = W.shape[1]
                beta = rho * 5.0 + 4.0 / D * d.sum()
                e = 1.0 / (beta / d + 1.0)
                Rm = W / np.sqrt(e)[:, None]
                dev = np.max(np.abs(Rm @ Rm.T - np.eye(len(d))))
                row.append(f"{l}{side[0]}:{s['jacobi_sweeps']}{'C' if s['reorth_checked'] else ''}{'R' if s['reorthogonalized'] else ''}({dev:.0e},{d.max()/max(d.min(),1e-30):.0e})")
    print(k, " ".join(row), "alpha", np.round(st.alpha_t, 3))
