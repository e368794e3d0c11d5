"""K2 time of the bench step for a trial share T (what one rank of an N-GPU strong-scaling run
simulates: T = 1024 / N), full C5 candidates.  Prints ms per T and the ideal (linear) ms."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import samu_workloads as W
from paper_2503_16893_b200 import Samu

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
Ts = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "1024,512,256,128,64").split(",")]
w = W.make_workload(name)
S = Samu(0)
S.load_workload(w)
ready = [v for v in range(w.n_nodes) if not np.any((w.pred[w.node == v] >= 0) &
                                                  (w.node[np.maximum(w.pred[w.node == v], 0)] != v))]
cands = [(v, dp, tp) for v in ready for (dp, tp) in S.samu_enumerate_plans(v)]
base = None
for T in Ts:
    lo, li = S.samu_sample_lengths(w.seed, 0, T)
    S.samu_simulate_batch(cands, lo, li)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e30
    for _ in range(2):
        e0.record()
        S.samu_simulate_batch(cands, lo, li)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    if base is None:
        base = (Ts[0], best)
    print(f"T={T:5d} ms={best:9.2f} linear={base[1] * T / base[0]:9.2f} eff={base[1] * T / base[0] / best:5.2f}", flush=True)
