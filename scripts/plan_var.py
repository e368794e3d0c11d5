import sys, time; sys.path.insert(0, ".")
import torch, samu_workloads as W
from paper_2503_16893_b200 import Samu
w = W.make_workload("c5", n_trials=128); S = Samu(0); S.load_workload(w)
S.samu_plan_greedy(w.seed, 1); torch.cuda.synchronize()
for i in range(4):
    t0 = time.perf_counter(); p = S.samu_plan_greedy(w.seed, 128); torch.cuda.synchronize()
    print("planner c5/128", round(time.perf_counter() - t0, 3), p["n_sims"], flush=True)
# per-call variance of one simulate batch
lo, li = S.samu_sample_lengths(w.seed, 0, 128)
cands = [(v, dp, tp) for v in range(6) for (dp, tp) in S.samu_enumerate_plans(v)]
for i in range(5):
    torch.cuda.synchronize(); t0 = time.perf_counter(); S.samu_simulate_batch(cands, lo, li); torch.cuda.synchronize()
    print("sim batch", round(time.perf_counter() - t0, 4), flush=True)
