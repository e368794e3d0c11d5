"""Per node of the C5 first step: K2 time with schedule sharing (default hints), without groups,
and the dp >= 5 singles alone; member items carried / fallen out of sync (T = 1024)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu, recs_to_numpy
T = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = W.make_workload("c5", n_trials=T)
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, T)
def t(cs, reps=2):
    S.samu_simulate_batch(cs, lo, li); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); o = S.samu_simulate_batch(cs, lo, li); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, recs_to_numpy(o["recs"])
for v in range(11):
    cs = [(v, dp, tp) for (dp, tp) in S.samu_enumerate_plans(v)]
    st0 = list(S.samu_share_stats().values())
    a, g = t(cs)
    st1 = list(S.samu_share_stats().values())
    os.environ["SAMU_K2_GROUP"] = "never"; b, _ = t(cs); del os.environ["SAMU_K2_GROUP"]
    os.environ["SAMU_K2_GROUP"] = "always"; c, _ = t(cs); del os.environ["SAMU_K2_GROUP"]
    d, _ = t([x for x in cs if x[1] >= 5]) if any(x[1] >= 5 for x in cs) else (0.0, None)
    it = g["iters"].astype(float).sum(axis=1)
    print(f"node {v:2d}: default {a:7.2f} ms  never {b:7.2f}  always {c:7.2f}  dp>=5 only {d:7.2f}  "
          f"share {None if st0 is None else [y - x for x, y in zip(st0, st1)]}  iters/cand {it.mean():.3e}", flush=True)
