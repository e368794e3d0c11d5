"""K1 time per C5 sampling call (1024 trials x 50k requests), median of 9 (CUDA events)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
w = W.make_workload("c5")
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, w.n_trials)
ts = []
for _ in range(9):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); S.samu_sample_lengths(w.seed, 0, w.n_trials, out=(lo, li)); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(os.environ.get("SAMU_K1_INDEX_ORDER", "chain roots first"), "K1 ms median", round(float(np.median(ts)), 4))
