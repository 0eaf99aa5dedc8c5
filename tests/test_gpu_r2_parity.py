"""GPU parity, round 2: the renormalisation layer (reading R32), B.3.1 flags
and NG states of the config-3 network in FP32 mode at the 1e-4 bar, a long TF32 config-3
trajectory from the C.6 initialisation, and config 2 over its full 1000 minibatches.

Tolerances (north_star; R23): FP32 mode normwise 1e-4; TF32 (reduced-precision
tensor-core inputs) 2e-2."""
import numpy as np
import pytest

from oracle import nnet as onn
from oracle import online_ng as ong
from oracle import training as otr
from synth import gaussian_rows, labels_uniform, power_law_rows, spliced_frames, standard_normals

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu
TOL = 1e-4
LR0, LR1 = 0.01 / 6 / 8, 0.001 / 6 / 8     # paper schedule x 1/8 (bench.py)


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_7455_b200 import api
    return api


def normwise(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300))


def delta_err(w_after, before, d_ref):
    """Normwise error of a weight update measured from FP32 weights: the GPU's W_{t+1} is
    an FP32 number, so W_{t+1} - W_t carries up to half an ulp of W_{t+1} of rounding that
    is not an error of the update (it dominates when |Delta W| << |W|, e.g. a small lr);
    that half-ulp is excused element by element, the rest is held to the bar."""
    w_after = np.asarray(w_after)
    d_gpu = w_after.astype(np.float64) - before
    half_ulp = 0.5 * np.spacing(np.abs(w_after.astype(np.float32))).astype(np.float64)
    excess = np.maximum(np.abs(d_gpu - d_ref) - half_ulp, 0.0)
    return float(np.max(excess) / max(np.max(np.abs(d_ref)), 1e-300))


def fp32_bar(stat):
    """FP32-mode bar for a layer's update (reading R33): 1e-4, widened in proportion to the
    cancellation in X_hat = X - H W once it exceeds 25x.  gamma = ||X||_F / ||X_hat||_F
    (eqn:gammat) is exactly that cancellation factor; an FP32 evaluation of
    X_hat (any FP32 one, CUDA-core or tensor-core) carries ~eps_32 gamma of relative error
    that the float64 oracle does not (measured: ~2e-6 gamma)."""
    g = max(stat.gamma_in, stat.gamma_out)
    return TOL * max(1.0, g / 25.0)


def to_dev(frames, labels):
    return (torch.from_numpy(np.ascontiguousarray(frames, dtype=np.float32)).cuda(),
            torch.from_numpy(np.ascontiguousarray(labels, dtype=np.int32)).cuda())


def make_pair(api, cfg, seed, rank_in, rank_out, max_mb, precision="fp32", softmax_scale=0.05):
    net = api.Nnet(cfg.input_dim, cfg.num_hidden, cfg.hidden_dim, cfg.pnorm_group, cfg.num_classes,
                   max_minibatch=max_mb, precond=True, rank_in=rank_in, rank_out=rank_out, seed=seed,
                   precision=precision, renorm=cfg.renorm)
    params = onn.init_params(cfg, standard_normals(seed, cfg.layer_shapes()))
    # small random softmax layer instead of zeros: with zeros the first
    # output-side minibatch has exactly tied eigenvalues (reading R7, parity unpinned there)
    params[-1] = softmax_scale * standard_normals(seed + 1, [cfg.layer_shapes()[-1]])[0]
    params = [p.astype(np.float32).astype(np.float64) for p in params]
    for l, p in enumerate(params):
        net.set_params(l, p)
    states = onn.make_states(cfg, ong.OnlineNgConfig(rank=rank_in), ong.OnlineNgConfig(rank=rank_out))
    return net, params, states


CFG3R = onn.NnetConfig(input_dim=360, num_hidden=4, hidden_dim=3000, pnorm_group=10, num_classes=5000, renorm=True)


@pytest.mark.parametrize("precision,shape", [("fp32", "tiny"), ("tf32", "tiny"), ("fp32", "config3"),
                                             ("tf32", "config3")])
def test_renorm_step_parity(api, precision, shape):
    """Forward, backward and update through the renormalisation layers: per step, the
    objective (1e-5 FP32 / 1e-2 TF32 relative) and the update Delta W of every matrix
    (FP32: 1e-4, widened by the cancellation factor gamma beyond 25x, fp32_bar; TF32: 2e-2
    normwise) against the oracle applied to the GPU's own pre-step weights."""
    if shape == "tiny":
        cfg = onn.NnetConfig(input_dim=40, num_hidden=2, hidden_dim=200, pnorm_group=10, num_classes=16, renorm=True)
        N, rin, rout, ctx = 128, 4, 8, 0
    else:
        cfg, N, rin, rout, ctx = CFG3R, 512, 20, 80, 4
    net, params, states = make_pair(api, cfg, 41, rin, rout, N, precision)
    tol, otol = (TOL, 1e-5) if precision == "fp32" else (2e-2, 1e-2)
    frames, labels = spliced_frames(43, 3 * N, num_classes=cfg.num_classes, context=ctx)
    for k in range(3):
        fr, lb = frames[k * N:(k + 1) * N], labels[k * N:(k + 1) * N]
        f, y = to_dev(fr, lb)
        before = [net.get_params(l).astype(np.float64) for l in range(len(params))]
        obj = net.forward_backward(f, y, objective=True)
        fb = onn.forward_backward(before, cfg, fr.astype(np.float64), lb)
        assert obj == pytest.approx(fb.objective, rel=otol)
        net.update(LR0, 0.075)
        ref = [b.copy() for b in before]
        ost = onn.update(ref, fb, LR0, states)
        errs = [delta_err(net.get_params(l), before[l], ref[l] - before[l]) for l in range(len(params))]
        print(precision, shape, k, ["%.2e" % e for e in errs])
        for l in range(len(params)):
            bar = fp32_bar(ost[l]) if precision == "fp32" else tol
            assert errs[l] <= bar, (k, l, errs[l], bar)


def test_config3_fp32_trajectory_flags_and_states(api):
    """Config 3 with renormalisation, FP32 mode, 14 steps from the C.6 initialisation (every
    state initialised on the device from its first minibatch, B.3.2; updates at t < 10 and
    t = 12), GPU and oracle each carrying their own NG states.

    * Step 0 (both sides from the same weights and the same first minibatch): Delta W of
      every matrix within the FP32 bar (1e-4, widened by the X_hat cancellation factor
      gamma beyond 25x: fp32_bar, reading R33).
    * Every update step, every state: the B.3.1 check trigger (a floored c_i; cond C > 1e6,
      P:1173-1175) equals the oracle's wherever the oracle's own value is outside the FP32
      noise of the threshold, and every oracle repair is matched by a GPU repair (R34).
    * After the run: every state's W^T W within 1e-2 and d within 1e-3 of the oracle's.
      The paper's arithmetic is single precision and B.3.1 exists because "R_t R_t^T = I can
      sometimes be lost due to roundoff": on this network cond C reaches 1e10
      (input side of the last layers), so the FP32 W_{t+1} = A_t B_t loses orthonormality
      beyond 1e-3 and is repaired where the float64 oracle's is not; the two trajectories
      then separate at the 1e-3 level in the low-energy directions (reading R34)."""
    net, params, states = make_pair(api, CFG3R, 47, 20, 80, 512)
    frames, labels = spliced_frames(53, 14 * 512, num_classes=5000)
    gpu_only_repairs = decided = 0
    for k in range(14):
        fr, lb = frames[k * 512:(k + 1) * 512], labels[k * 512:(k + 1) * 512]
        f, y = to_dev(fr, lb)
        before = [net.get_params(l).astype(np.float64) for l in range(len(params))]
        net.forward_backward(f, y)
        lr = otr.lr_at(k * 512, 14 * 512, LR0, LR1)
        net.update(lr, 0.075)
        fb = onn.forward_backward(before, CFG3R, fr.astype(np.float64), lb)
        ref = [b.copy() for b in before]
        ost = onn.update(ref, fb, lr, states)
        errs = [delta_err(net.get_params(l), before[l], ref[l] - before[l]) for l in range(len(params))]
        print("step", k, "Delta W errors", ["%.1e" % e for e in errs])
        if k == 0:
            for l in range(len(params)):
                assert errs[l] <= fp32_bar(ost[l]), (k, l, errs[l], fp32_bar(ost[l]))
        for l in range(len(params)):
            for side, fl, mg in (("in", ost[l].flags_in, ost[l].margins_in),
                                 ("out", ost[l].flags_out, ost[l].margins_out)):
                g = net.ngsgd(l, side).get_state()
                assert g["updated"] == (k < 10 or k % 4 == 0)
                if g["updated"]:
                    # decided = the oracle's min c is more than 1e-5 max c from the floor
                    # (1-eta)^2 rho^2, and its cond C more than a factor 3 from 1e6
                    floor_decided = abs(mg[0]) > 1e-5
                    cond_decided = fl[0] or abs(np.log10(mg[1] / 1e6)) > np.log10(3.0)
                    decided += int(floor_decided) + int(floor_decided and cond_decided)
                    if floor_decided:
                        assert g["floored"] == bool(fl[0]), (k, l, side, g, fl, mg)
                    if floor_decided and cond_decided:
                        assert g["reorth_checked"] == bool(fl[1]), (k, l, side, g, fl, mg)
                    if fl[2]:
                        assert g["reorthogonalized"], (k, l, side)
                    gpu_only_repairs += int(g["reorthogonalized"] and not fl[2])
    print("GPU-only B.3.1 repairs:", gpu_only_repairs, "decided flag comparisons:", decided)
    assert decided >= 60          # of 220 possible: the test is not vacuous
    for l, (s_in, s_out) in enumerate(states):
        for side, s in (("in", s_in), ("out", s_out)):
            g = net.ngsgd(l, side).get_state()
            W = g["W"].astype(np.float64)
            e_w, e_d = normwise(W.T @ W, s.W.T @ s.W), normwise(g["d"], s.d)
            print("state", l, side, "W^T W %.1e rho %.1e d %.1e" % (e_w, abs(g["rho"] / s.rho - 1), e_d))
            assert e_w <= 1e-2 and e_d <= 1e-3, (l, side, e_w, e_d)


def test_config3_tf32_trajectory_from_init(api):
    """Config 3 with renormalisation in the bench's TF32 mode: 50 consecutive steps from the
    C.6 initialisation, both sides carrying their own weights and NG states (no re-sync):
    every step's objective within 2e-2 relative of the float64 oracle's, and the accumulated
    preconditioned change of every weight matrix, W_50 - W_0, within 2e-2 normwise of the
    oracle's (north_star's reduced-precision bar on the preconditioned gradients)."""
    net, params, states = make_pair(api, CFG3R, 59, 20, 80, 512, precision="tf32")
    w0 = [p.copy() for p in params]
    steps = 50
    frames, labels = spliced_frames(61, steps * 512, num_classes=5000)
    for k in range(steps):
        fr, lb = frames[k * 512:(k + 1) * 512], labels[k * 512:(k + 1) * 512]
        f, y = to_dev(fr, lb)
        obj = net.forward_backward(f, y, objective=True)
        lr = otr.lr_at(k * 512, steps * 512, LR0, LR1)
        net.update(lr, 0.075)
        oobj, _ = onn.train_step(params, CFG3R, fr.astype(np.float64), lb, lr, states)
        assert obj == pytest.approx(oobj, rel=2e-2), k
    errs = [normwise(net.get_params(l).astype(np.float64) - w0[l], params[l] - w0[l]) for l in range(len(params))]
    print("tf32 50-step accumulated-change errors", ["%.2e" % e for e in errs])
    assert max(errs) <= 2e-2, errs


@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_config2_full_run(api, precision):
    """BASELINE configs[1] over its full length: one 2000-dim layer's two sides (out D = 2000,
    R = 80; in D = 2001 = [|.|, 1], R = 20), N = 512, 1000 minibatches (64-batch pool cycled,
    257 update steps), exactly the bench's sequence.  Every 50th minibatch and the last: the
    output X_bar = gamma X_hat within the bar; at the end every state (W^T W, rho, d)."""
    tol = TOL if precision == "fp32" else 2e-2
    N = 512
    xo = power_law_rows(2000, N, 2000, n_batches=64)
    xi = power_law_rows(2001, N, 2000, n_batches=64, nonneg=True, append_one=True)
    gpu = [api.OnlinePreconditioner(2000, N, rank=80, precision=precision),
           api.OnlinePreconditioner(2001, N, rank=20, precision=precision)]
    ora = [ong.OnlineNgState(2000, ong.OnlineNgConfig(rank=80)), ong.OnlineNgState(2001, ong.OnlineNgConfig(rank=20))]
    bufs = [torch.zeros((N, 2000), device="cuda"), torch.zeros((N, 2004), device="cuda")]
    g = torch.zeros(2, device="cuda")
    for k in range(1000):
        for s, (pool, ld) in enumerate(((xo, 2000), (xi, 2001))):
            x = pool[k % 64]
            view = bufs[s][:, :ld]
            view.copy_(torch.from_numpy(x.astype(np.float32)))
            gpu[s].precondition(view, g[s:s + 1])
            o = ong.precondition(ora[s], x.astype(np.float32).astype(np.float64))
            if k % 50 == 0 or k == 999:
                got = view.cpu().numpy().astype(np.float64) * float(g[s].cpu())
                err = normwise(got, o.x_bar)
                assert err <= tol, (k, s, err)
    for s in range(2):
        st = gpu[s].get_state()
        W = st["W"].astype(np.float64)
        assert st["t"] == ora[s].t == 1000
        assert normwise(W.T @ W, ora[s].W.T @ ora[s].W) <= tol, s
        assert st["rho"] == pytest.approx(ora[s].rho, rel=tol)
        assert normwise(st["d"], ora[s].d) <= tol
