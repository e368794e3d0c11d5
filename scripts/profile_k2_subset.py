"""One K2 launch on a subset of the C5 first-step candidates (by node range) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import samu_workloads as W
from paper_2503_16893_b200 import Samu

lo_n, hi_n = int(sys.argv[1]), int(sys.argv[2])
T = int(sys.argv[3]) if len(sys.argv) > 3 else 64
w = W.make_workload("c5", n_trials=T)
S = Samu(0)
S.load_workload(w)
cands = [(v, dp, tp) for v in range(lo_n, hi_n) for (dp, tp) in S.samu_enumerate_plans(v)]
lo, li = S.samu_sample_lengths(w.seed, 0, T)
for _ in range(2):
    S.samu_simulate_batch(cands, lo, li)
torch.cuda.synchronize()
print("ok", len(cands))
