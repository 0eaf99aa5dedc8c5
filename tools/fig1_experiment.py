"""Fig.-1 analogue on synthetic data (section 4.3): the held-out
objective vs epochs for N = 1, 2, 4, 8 parallel jobs with parameter averaging every K
samples per job, online NG-SGD vs plain SGD.  The paper's claim: with
NG-SGD, averaging works and the convergence per epoch barely depends on N up to ~4 jobs,
while plain SGD degrades as N grows.

All jobs run on ONE GPU (one network per job, one stream): every job trains on its own
block of the N x M randomisation (C.2, driver.block_randomize) for K samples, then the
parameters of all jobs are replaced by their average (nnet_average_local, the same fixed
tree as the NCCL nnet_average).  Per-job learning rate = N x the effective rate,
the effective rate decaying exponentially 10x over the run, scaled as the bench
(R35).  Network: the bench's config 3 (renormalised p-norm DNN, R_in = 20 / R_out = 80).

    python tools/fig1_experiment.py [--epochs 3] [--frames 262144] [--k 32768] [--out profiles/round2_fig1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1410_7455_b200 import api, driver
from synth import spliced_frames

N_MB = 512


def heldout_objective(net, hx, hy):
    tot, n = 0.0, 0
    for s in range(0, hx.shape[0], N_MB):
        e = min(hx.shape[0], s + N_MB)
        tot += net.forward_backward(hx[s:e], hy[s:e], objective=True)
        n += e - s
    return tot / n


def run(method, jobs, args, pool, labels, hx, hy):
    nets = [api.Nnet(360, 4, 3000, 10, 5000, max_minibatch=N_MB, precond=(method == "online"), rank_in=20,
                     rank_out=80, precision="tf32", seed=1410, renorm=True) for _ in range(jobs)]
    blocks = driver.block_randomize(pool.shape[0], jobs, args.k, seed=7)
    rows = [[torch.from_numpy(b).cuda() for b in row] for row in blocks]
    M = len(blocks[0])
    total = args.epochs * pool.shape[0]
    seen = 0
    curve = [{"epoch": 0.0, "heldout_obj_per_frame": heldout_objective(nets[0], hx, hy)}]
    t0 = time.time()
    for ep in range(args.epochs):
        for m in range(M):
            for j, net in enumerate(nets):
                r = rows[j][m]
                for s in range(0, r.numel(), N_MB):
                    idx = r[s:s + N_MB]
                    lr = driver.job_learning_rate(seen, total, jobs) / 8.0      # R35 scale
                    net.forward_backward_ex(pool, labels, idx.numel(), rows=idx)
                    net.update(lr, 0.075)
                    seen += idx.numel()
            if jobs > 1:
                api.average_local(nets)
        curve.append({"epoch": ep + 1.0, "heldout_obj_per_frame": heldout_objective(nets[0], hx, hy)})
        print(f"  {method:6s} N={jobs} epoch {ep + 1}: held-out objective {curve[-1]['heldout_obj_per_frame']:.4f}",
              flush=True)
    torch.cuda.synchronize()
    for n in nets:
        n.close()
    return {"method": method, "jobs": jobs, "outer_iterations_per_epoch": M, "curve": curve,
            "seconds": time.time() - t0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--epochs", type=int, default=3)
    ap.add_argument("--frames", type=int, default=1 << 18)
    ap.add_argument("--k", type=int, default=32768)
    ap.add_argument("--jobs", default="1,2,4,8")
    ap.add_argument("--out", default="profiles/round2_fig1")
    args = ap.parse_args()
    f, y = spliced_frames(1410, args.frames, num_classes=5000)
    hf, hy = spliced_frames(99991, 8192, num_classes=5000)
    pool, labels = torch.from_numpy(f).cuda(), torch.from_numpy(y).cuda()
    hx, hyt = torch.from_numpy(hf).cuda(), torch.from_numpy(hy).cuda()
    results = []
    for method in ("online", "none"):
        for jobs in [int(x) for x in args.jobs.split(",")]:
            results.append(run(method, jobs, args, pool, labels, hx, hyt))
    meta = {"what": "held-out objective (mean log p(y|x) per frame, 8192 frames) vs epochs; config-3 network "
                    "(renormalised), synthetic frames; N jobs on one GPU, average every K samples per job",
            "frames_per_epoch": args.frames, "k_samples": args.k, "epochs": args.epochs,
            "lr": "per-job = N x effective, effective 0.01 -> 0.001 (/6, x 1/8 synthetic scale, R35)"}
    json.dump({"meta": meta, "results": results}, open(args.out + ".json", "w"), indent=1)
    with open(args.out + ".md", "w") as fh:
        fh.write("# Fig.-1 analogue (P:650-694) on synthetic data\n\n" + meta["what"] + ".\n\n")
        fh.write(f"{args.frames} frames per epoch, K = {args.k} samples per job per outer iteration, "
                 f"{args.epochs} epochs.\n\n")
        fh.write("| method | N jobs | " + " | ".join(f"epoch {e}" for e in range(args.epochs + 1)) + " | seconds |\n")
        fh.write("|---|---|" + "---|" * (args.epochs + 1) + "---|\n")
        for r in results:
            fh.write(f"| {r['method']} | {r['jobs']} | " + " | ".join(f"{c['heldout_obj_per_frame']:.4f}" for c in r["curve"])
                     + f" | {r['seconds']:.1f} |\n")
    print(open(args.out + ".md").read())


if __name__ == "__main__":
    main()
