"""GPU parity of the generalised model combination (C.4):
the combined parameters, the combination objective and its gradient (nnet_set_combination,
nnet_combination_grad) against oracle/combine.py at fixed weights, then the whole search
(driver.combine_models, L-BFGS from the best of P + 1 starts) against the oracle's L-BFGS:
the same best start and a final objective at least as good as the start, within 1e-4 of
the oracle's optimum."""
import numpy as np
import pytest

from oracle import combine as ocomb
from oracle import nnet as onn
from synth import spliced_frames, standard_normals

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

CFG = onn.NnetConfig(input_dim=40, num_hidden=2, hidden_dim=200, pnorm_group=10, num_classes=16, renorm=True)


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_7455_b200 import api
    return api


def _setup(api, P=4):
    net = api.Nnet(40, 2, 200, 10, 16, max_minibatch=128, precond=False, seed=1, precision="fp32", renorm=True)
    models_np, snaps = [], []
    for p in range(P):
        ps = onn.init_params(CFG, standard_normals(50 + p, CFG.layer_shapes()))
        ps[-1] = 0.2 * standard_normals(80 + p, [CFG.layer_shapes()[-1]])[0]
        ps = [x.astype(np.float32).astype(np.float64) for x in ps]
        for l, x in enumerate(ps):
            net.set_params(l, x)
        snaps.append(net.snapshot())
        models_np.append(ps)
    frames, labels = spliced_frames(3, 256, context=0, num_classes=16)
    batches_np = [(frames[:128].astype(np.float64), labels[:128]), (frames[128:].astype(np.float64), labels[128:])]
    batches = [(torch.from_numpy(frames[:128]).cuda(), torch.from_numpy(labels[:128]).cuda()),
               (torch.from_numpy(frames[128:]).cuda(), torch.from_numpy(labels[128:]).cuda())]
    return net, snaps, models_np, batches, batches_np


def test_objective_and_gradient_at_fixed_weights(api):
    from paper_1410_7455_b200 import driver
    net, snaps, models, batches, bnp = _setup(api)
    w = np.random.default_rng(0).uniform(0.0, 0.5, size=(3, 4))
    f_gpu, g_gpu = driver.combination_objective(net, snaps, w, batches)
    f_ref, g_ref = ocomb.objective_and_grad(models, w, CFG, bnp)
    assert f_gpu == pytest.approx(f_ref, rel=1e-5)
    assert np.max(np.abs(g_gpu - g_ref)) <= 1e-4 * np.max(np.abs(g_ref))
    comb = ocomb.combine(models, w.astype(np.float32).astype(np.float64))
    for l in range(3):
        assert np.max(np.abs(net.get_params(l) - comb[l])) <= 1e-6 * np.max(np.abs(comb[l]))


def test_lbfgs_search(api):
    from paper_1410_7455_b200 import driver
    net, snaps, models, batches, bnp = _setup(api)
    w0, objs = ocomb.starting_point(models, CFG, bnp)
    w, f = driver.combine_models(net, snaps, batches, iters=30)
    w_ref, f_ref = ocomb.combine_lbfgs(models, CFG, bnp, iters=100)
    assert f >= max(objs) - 1e-6 * abs(max(objs))
    assert f == pytest.approx(f_ref, rel=1e-4)
