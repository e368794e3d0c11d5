"""Latency of the longest C5 replica-sims alone: the chain summariser with dp = 1 (one warp per
(trial, plan)), for a few trial counts (1 = a single warp on an idle GPU)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu, recs_to_numpy
w = W.make_workload("c5")
S = Samu(0)
S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, 128)
for T in (1, 4, 128):
    cands = [(10, 1, 1)]
    out = S.samu_simulate_batch(cands, lo[:T], li[:T])
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); out = S.samu_simulate_batch(cands, lo[:T], li[:T]); e1.record(); torch.cuda.synchronize()
    g = recs_to_numpy(out["recs"])
    print(f"chain (10,1,1) T={T}: {e0.elapsed_time(e1):.2f} ms, iterations per item {g['iters'].mean():.0f}")
