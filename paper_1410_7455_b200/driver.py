"""Host-side driver logic for data-parallel training (section 3.1 of arXiv 1410.7455):
one SGD job per GPU, per-job learning rate, and the every-K parameter average.

Pure host scalars / bookkeeping; every tensor operation runs in libngsgd.so.  Kept free
of torch.cuda so the multi-rank logic can be exercised with the gloo backend on CPU.
"""
from __future__ import annotations

import math

K_SAMPLES = 400_000        # samples per job per outer iteration
REF_JOBS = 6               # default lr 0.01 -> 0.001 corresponds to 6 jobs


def job_learning_rate(samples_seen: float, total_samples: float, n_jobs: int, lr_initial: float = 0.01,
                      lr_final: float = 0.001, ref_jobs: int = REF_JOBS) -> float:
    """Per-job rate: exponential schedule from lr_initial to lr_final (reading
    R17: per minibatch by samples seen), scaled so the effective rate (per-job rate / n_jobs,
    P:103-109) is that of the ref_jobs-job default."""
    frac = min(max(samples_seen / float(total_samples), 0.0), 1.0)
    lr = lr_initial * (lr_final / lr_initial) ** frac
    return lr * n_jobs / ref_jobs


def minibatches_per_outer_iteration(minibatch: int, k_samples: int = K_SAMPLES) -> list:
    """Sizes of the minibatches one job runs in an outer iteration of exactly K samples
    (reading R24): 781 x 512 + 1 x 128 for K = 400 000."""
    full, rem = divmod(k_samples, minibatch)
    return [minibatch] * full + ([rem] if rem else [])


def rank_seed(rank: int, base: int = 1410) -> int:
    """Disjoint data per job: seed = 1410 + 7455 * rank."""
    return base + 7455 * int(rank)


def shard_size(count: int, nranks: int) -> int:
    """Shard length of nnet_comm_init: ceil(count / nranks) rounded up to 64 floats."""
    s = -(-count // nranks)
    return -(-s // 64) * 64


def shard_bounds(count: int, nranks: int, rank: int):
    """The slice [lo, hi) of the flat parameter arena that rank `rank` reduces in the
    deterministic average (nnet_average); the last shards are ragged, possibly empty."""
    s = shard_size(count, nranks)
    lo = min(count, rank * s)
    return lo, min(count, lo + s)


def tree_order(n: int) -> list:
    """The fixed pairwise-tree summation order over rank index used by nnet_average
    (R18), as a nested tuple, e.g. n = 4 -> ((0, 1), (2, 3))."""
    level = list(range(n))
    while len(level) > 1:
        level = [(level[k], level[k + 1]) if k + 1 < len(level) else level[k] for k in range(0, len(level), 2)]
    return level[0]


def max_over_ranks(value: float, group=None) -> float:
    """Max of a host scalar over all ranks (timing is max-over-ranks)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def broadcast_bytes(payload: bytes | None, src: int = 0, group=None) -> bytes:
    """Broadcast a small byte string (the NCCL unique id) from `src` to all ranks."""
    import torch.distributed as dist
    obj = [payload]
    dist.broadcast_object_list(obj, src=src, group=group)
    return obj[0]


def outer_iteration_of(step: int, minibatch: int, k_samples: int = K_SAMPLES) -> int:
    return int(math.floor(step * minibatch / k_samples))


def tree_reduce_stride(values):
    """The summation schedule of tree_avg_kernel (nnet.cu), written out on the host: for
    w = 1, 2, 4, ...: v[k] += v[k + w] for k = 0, 2w, 4w, ...  Used by tests to pin the
    device schedule to the oracle's pairwise tree (oracle.training.tree_sum)."""
    v = [x.copy() for x in values]
    w = 1
    while w < len(v):
        for k in range(0, len(v) - w, 2 * w):
            v[k] = (v[k] + v[k + w]).astype(v[k].dtype)
        w *= 2
    return v[0]


def outer_iterations_per_epoch(num_examples: int, n_jobs: int, k_samples: int = K_SAMPLES) -> int:
    """M >= 1: the number of outer iterations per epoch, chosen so that each job's block of
    an outer iteration holds close to K samples (C.2)."""
    return max(1, int(round(num_examples / float(n_jobs * k_samples))))


def block_randomize(num_examples: int, n_jobs: int, k_samples: int = K_SAMPLES, seed: int = 1410):
    """The N x M data blocks of C.2: one random permutation of the examples
    (fixed by the seed, so every epoch reads the same order) cut into N M
    nearly equal blocks; job n processes blocks[n][m] on outer iteration m.  Returns int32
    index arrays (host), to be uploaded once and used as the `rows` of
    nnet_forward_backward_ex."""
    import numpy as np
    m = outer_iterations_per_epoch(num_examples, n_jobs, k_samples)
    perm = np.random.default_rng(seed).permutation(num_examples)
    nb = n_jobs * m
    base, extra = divmod(num_examples, nb)            # the first `extra` blocks get one more
    bounds = [0]
    for q in range(nb):
        bounds.append(bounds[-1] + base + (1 if q < extra else 0))
    chunks = [perm[bounds[q]:bounds[q + 1]].astype(np.int32) for q in range(nb)]
    return [[chunks[b * n_jobs + n] for b in range(m)] for n in range(n_jobs)]


COMBINE_REG = 1e-10   # "a very tiny regularizer" on the combination weights


def combination_objective(net, models, weights, batches):
    """Objective sum_i log p(y_i|x_i) of the combined model over the batches (device work:
    nnet_set_combination, nnet_forward_backward, nnet_combination_grad) minus the tiny
    regulariser, and its gradient w.r.t. the weights (host arrays)."""
    import numpy as np
    net.set_combination(models, weights)
    obj = 0.0
    grad = np.zeros_like(weights, dtype=np.float64)
    for frames, labels in batches:
        obj += net.forward_backward(frames, labels, objective=True)
        grad += net.combination_grad(models)
    return obj - COMBINE_REG * float(np.sum(weights * weights)), grad - 2.0 * COMBINE_REG * weights


def combine_models(net, models, batches, iters: int = 20, history: int = 10):
    """Generalised model combination (C.4): per-layer weights over the last P
    models maximising the objective on `batches` (device tensors), by L-BFGS (
    two-loop recursion, backtracking Armijo line search; reading R37: no Fisher
    preconditioning) from the best of the P + 1 starting points (each model, the average,
    P:1571-1573).  Leaves the net set to the result; returns (weights, objective)."""
    import numpy as np
    L, P = net.num_layers, len(models)
    cands = []
    for p in range(P):
        w = np.zeros((L, P))
        w[:, p] = 1.0
        cands.append(w)
    cands.append(np.full((L, P), 1.0 / P))
    evals = [combination_objective(net, models, w, batches) for w in cands]
    best = int(np.argmax([e[0] for e in evals]))
    w, (f, g) = cands[best], evals[best]
    s_hist, y_hist = [], []
    for _ in range(iters):
        # ascent direction from the two-loop recursion on -f
        q = -g.ravel().copy()
        alphas = []
        for s_, y_ in reversed(list(zip(s_hist, y_hist))):
            a = float(s_ @ q) / float(y_ @ s_)
            alphas.append(a)
            q -= a * y_
        if s_hist:
            q *= float(s_hist[-1] @ y_hist[-1]) / float(y_hist[-1] @ y_hist[-1])
        for (s_, y_), a in zip(zip(s_hist, y_hist), reversed(alphas)):
            b = float(y_ @ q) / float(y_ @ s_)
            q += (a - b) * s_
        d = -q.reshape(w.shape)                     # ascent direction for f
        slope = float(np.sum(g * d))
        if slope <= 0.0:
            d, slope = g.copy(), float(np.sum(g * g))
        if slope <= 1e-12 * max(1.0, abs(f)):
            break
        step, ok = 1.0, False
        for _ls in range(20):
            wn = w + step * d
            fn, gn = combination_objective(net, models, wn, batches)
            if fn >= f + 1e-4 * step * slope:
                ok = True
                break
            step *= 0.5
        if not ok:
            break
        s_vec, y_vec = (wn - w).ravel(), -(gn - g).ravel()
        if float(s_vec @ y_vec) > 1e-20:
            s_hist.append(s_vec)
            y_hist.append(y_vec)
            if len(s_hist) > history:
                s_hist.pop(0)
                y_hist.pop(0)
        w, f, g = wn, fn, gn
    net.set_combination(models, w)
    return w, f
