"""One replica-sim alone on the GPU (one candidate, one trial, dp = 1: one warp) for ncu stall
sampling of the critical path of small trial shares.  python scripts/profile_item.py node dp tp"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("SAMU_K2_MODES", "always")
os.environ.setdefault("SAMU_K2_GROUP", "never")
import torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
v, dp, tp = (int(x) for x in sys.argv[1:4])
w = W.make_workload("c5", n_trials=1)
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, 1)
for _ in range(2):
    S.samu_simulate_batch([(v, dp, tp)], lo, li)
torch.cuda.synchronize()
print("ok")
