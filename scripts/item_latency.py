"""Latency of single replica-sims (one candidate, one trial, dp = 1: one warp alone on the GPU)
of the C5 first step: the critical path of a launch at small trial shares (8-GPU runs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu, recs_to_numpy
w = W.make_workload("c5", n_trials=4)
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, 4)
os.environ["SAMU_K2_MODES"] = "always"
os.environ["SAMU_K2_GROUP"] = "never"
rows = []
for v in range(w.n_nodes - 1):
    for (dp, tp) in S.samu_enumerate_plans(v):
        if dp != 1:
            continue
        l1, i1 = lo[:1], li[:1]
        S.samu_simulate_batch([(v, dp, tp)], l1, i1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for _ in range(3):
            e0.record(); out = S.samu_simulate_batch([(v, dp, tp)], l1, i1); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        g = recs_to_numpy(out["recs"])
        rows.append((best, v, dp, tp, int(g["iters"][0, 0]), int(g["req_iters"][0, 0])))
for best, v, dp, tp, it, ri in sorted(rows, reverse=True):
    print(f"node {v:2d} dp {dp} tp {tp}: {best:7.2f} ms  iters {it:7d}  ns/iter {best * 1e6 / max(it, 1):6.1f}  req-iters {ri}")
