"""GPU parity of the parameter average's device arithmetic (3.1; R18):
the fixed-order sum kernel of nnet_average (ng_debug_tree_avg, the exact kernel and launch
nnet_average uses on each rank's shard) is bit-exact against the oracle's pairwise tree
sum times 1/n in float32, for every job count including the paper's 6.
The NCCL exchange around it is covered at nranks = 1 here (one GPU per job; NCCL refuses
two ranks on one device) and by the gloo emulation of the shard schedule."""
import ctypes

import numpy as np
import pytest

from oracle import training as otr

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_7455_b200 import _lib
    return _lib


@pytest.mark.parametrize("nr", [1, 2, 3, 4, 5, 6, 7, 8, 9, 13, 16, 33, 64])
def test_tree_avg_bit_exact(lib, nr):
    rng = np.random.default_rng(100 + nr)
    count = 5_360_128 // 64 + 3            # ragged tail (not a multiple of the block size)
    models = [rng.normal(size=count).astype(np.float32) * np.float32(10.0 ** rng.integers(-3, 3))
              for _ in range(nr)]
    src = torch.from_numpy(np.stack(models)).cuda()
    out = torch.full((count,), float("nan"), device="cuda")
    lib.check(lib.lib.ng_debug_tree_avg(nr, count, ctypes.c_void_p(src.data_ptr()),
                                        ctypes.c_void_p(out.data_ptr()), None))
    torch.cuda.synchronize()
    ref = otr.average_models([[m] for m in models], dtype=np.float32)[0]
    assert np.array_equal(out.cpu().numpy(), ref)


def test_tree_avg_identical_models_noop(lib):
    """n identical models average to themselves bit-exactly for n = 2, 4, 8."""
    w = np.random.default_rng(5).normal(size=70_001).astype(np.float32)
    for nr in (2, 4, 8):
        src = torch.from_numpy(np.stack([w] * nr)).cuda()
        out = torch.empty(w.size, device="cuda")
        lib.check(lib.lib.ng_debug_tree_avg(nr, w.size, ctypes.c_void_p(src.data_ptr()),
                                            ctypes.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy(), w)


def test_comm_rejects_bad_nranks(lib):
    from paper_1410_7455_b200 import api
    net = api.Nnet(40, 1, 200, 10, 16, max_minibatch=8, precond=False, seed=9)
    with pytest.raises(api.NgError):
        net.comm_init(api.comm_unique_id(), 0, 65)
    with pytest.raises(api.NgError):
        net.comm_init(api.comm_unique_id(), 3, 3)


@pytest.mark.parametrize("n", [1, 2, 3, 6])
def test_average_local_bit_exact(lib, n):
    """nnet_average_local (several jobs on one GPU; the f2 experiment's average): every
    network gets the oracle's fixed-tree float32 mean of all of them, bit-exact."""
    from paper_1410_7455_b200 import api
    nets = [api.Nnet(40, 1, 200, 10, 16, max_minibatch=8, precond=False, seed=10 + q) for q in range(n)]
    models = [[net.get_params(l) for l in range(2)] for net in nets]
    rng = np.random.default_rng(n)
    for q, net in enumerate(nets):          # non-zero softmax layers too
        w = (rng.normal(size=models[q][1].shape) * 0.1).astype(np.float32)
        net.set_params(1, w)
        models[q][1] = w
    api.average_local(nets)
    ref = otr.average_models(models, dtype=np.float32)
    for net in nets:
        for l in range(2):
            assert np.array_equal(net.get_params(l), ref[l])


def test_select_best_single_rank(lib):
    """nnet_select_best at nranks = 1: the only job wins and its parameters
    are unchanged (the broadcast from itself is a no-op)."""
    from paper_1410_7455_b200 import api
    net = api.Nnet(40, 1, 200, 10, 16, max_minibatch=8, precond=False, seed=5)
    before = [net.get_params(l) for l in range(2)]
    net.comm_init(api.comm_unique_id(), 0, 1)
    assert net.select_best(-3.25) == 0
    for l in range(2):
        assert np.array_equal(net.get_params(l), before[l])
