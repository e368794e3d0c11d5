"""One C5 sampling call (1024 trials x 50k requests) for an ncu capture of K1."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
w = W.make_workload("c5")
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, w.n_trials)
for _ in range(3):
    S.samu_sample_lengths(w.seed, 0, w.n_trials, out=(lo, li))
torch.cuda.synchronize()
print("ok")
