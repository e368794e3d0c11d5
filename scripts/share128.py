"""Where does the 128-trial share (one rank of an 8-GPU run) spend its time? K2 per application."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
T = int(sys.argv[1]) if len(sys.argv) > 1 else 128
w = W.make_workload("c5", n_trials=T)
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, T)
allc = [(v, dp, tp) for v in range(11) for (dp, tp) in S.samu_enumerate_plans(v)]
def t(cs, reps=3):
    S.samu_simulate_batch(cs, lo, li); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); S.samu_simulate_batch(cs, lo, li); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
print("all", t(allc))
print("FRESH node 10", t([c for c in allc if c[0] == 10]))
print("FRESH node 10 dp=1", t([c for c in allc if c[0] == 10 and c[1] == 1]))
print("FRESH node 10 dp>1", t([c for c in allc if c[0] == 10 and c[1] > 1]))
print("LEAN nodes 0-9", t([c for c in allc if c[0] < 10]))
print("LEAN node 7", t([c for c in allc if c[0] == 7]))
print("LEAN nodes 0-9 without node 7", t([c for c in allc if c[0] < 10 and c[0] != 7]))
