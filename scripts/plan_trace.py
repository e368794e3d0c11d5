"""Planner timing with SAMU_TRACE=1 (per-stage wall time and time in simulate batches)."""
import os, sys, time
os.environ["SAMU_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
name, T = sys.argv[1], int(sys.argv[2])
w = W.make_workload(name, n_trials=T)
S = Samu(0)
S.load_workload(w)
S.samu_plan_greedy(w.seed, 1)
torch.cuda.synchronize()
for _ in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    t0 = time.perf_counter()
    S.samu_plan_greedy(w.seed, T)
    torch.cuda.synchronize()
    print(f"planner {name}/{T}: {time.perf_counter() - t0:.3f} s", file=sys.stderr, flush=True)
