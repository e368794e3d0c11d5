"""Run the bench step on a workload twice (warm + profiled) for ncu captures."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
name = sys.argv[1] if len(sys.argv) > 1 else "c5"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
w = W.make_workload(name, n_trials=T)
S = Samu(0); S.load_workload(w)
ready = [v for v in range(w.n_nodes) if not np.any((w.pred[w.node == v] >= 0) & (w.node[np.maximum(w.pred[w.node == v], 0)] != v))]
cands = [(v, dp, tp) for v in ready for (dp, tp) in S.samu_enumerate_plans(v)]
lo, li = S.samu_sample_lengths(w.seed, 0, T)
for _ in range(reps):
    out = S.samu_simulate_batch(cands, lo, li, summary=True)
torch.cuda.synchronize()
print("ok", len(cands))
