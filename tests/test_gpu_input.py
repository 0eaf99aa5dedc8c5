"""GPU parity of the input side (C.2): the 1-byte compression
(ng_compress_frames, reading R36) is bit-exact against the oracle's codes; a training step
on uint8-coded frames decoded inside the input kernel is bit-identical to one on the
oracle-decoded float32 frames; a step on rows gathered from a device-resident pool (a block
of the N x M randomisation) is bit-identical to one on the same rows laid out contiguously."""
import numpy as np
import pytest

from oracle import data as odata
from synth import spliced_frames

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1410_7455_b200 import api
    return api


def test_compress_bit_exact(api):
    frames, _ = spliced_frames(5, 4000, num_classes=50)
    frames[:, 17] = -1.5                                     # a constant column
    x = torch.from_numpy(frames).cuda()
    q, lo, step = api.compress_frames(x)
    torch.cuda.synchronize()
    q_ref, lo_ref, step_ref = odata.compress(frames)
    assert np.array_equal(lo.cpu().numpy(), lo_ref) and np.array_equal(step.cpu().numpy(), step_ref)
    assert np.array_equal(q.cpu().numpy(), q_ref)


def _net(api, seed=7):
    net = api.Nnet(360, 2, 1000, 10, 300, max_minibatch=256, precond=True, rank_in=20, rank_out=40, seed=seed,
                   precision="tf32", renorm=True)
    return net


def test_uint8_step_equals_decoded_float_step(api):
    frames, labels = spliced_frames(9, 256, num_classes=300)
    q_ref, lo_ref, step_ref = odata.compress(frames)
    dec = odata.decompress(q_ref, lo_ref, step_ref)
    a, b = _net(api), _net(api)
    y = torch.from_numpy(labels).cuda()
    oa = a.forward_backward(torch.from_numpy(dec).cuda(), y, objective=True)
    ob = b.forward_backward_ex(torch.from_numpy(q_ref).cuda(), y, 256, lo=torch.from_numpy(lo_ref).cuda(),
                               step=torch.from_numpy(step_ref).cuda(), objective=True)
    assert oa == ob
    a.update(0.002, 0.075)
    b.update(0.002, 0.075)
    for l in range(3):
        assert np.array_equal(a.get_params(l), b.get_params(l))


def test_gathered_rows_step_equals_contiguous_step(api):
    from paper_1410_7455_b200 import driver
    pool, labels = spliced_frames(13, 3000, num_classes=300)
    blocks = driver.block_randomize(3000, 2, 700, seed=5)
    rows = blocks[1][0][:256]
    a, b = _net(api), _net(api)
    oa = a.forward_backward(torch.from_numpy(np.ascontiguousarray(pool[rows])).cuda(),
                            torch.from_numpy(np.ascontiguousarray(labels[rows])).cuda(), objective=True)
    ob = b.forward_backward_ex(torch.from_numpy(pool).cuda(), torch.from_numpy(labels).cuda(), len(rows),
                               rows=torch.from_numpy(rows).cuda(), objective=True)
    assert oa == ob
    a.update(0.002, 0.075)
    b.update(0.002, 0.075)
    for l in range(3):
        assert np.array_equal(a.get_params(l), b.get_params(l))
