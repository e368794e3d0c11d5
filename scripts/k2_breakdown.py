"""Time K2 on subsets of the C5 first-step candidates (by application) to see where time goes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu, recs_to_numpy
w = W.make_workload("c5", n_trials=int(sys.argv[1]) if len(sys.argv) > 1 else 1024)
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, w.n_trials)
groups = {"ensembling (nodes 0-5)": range(0, 6), "routing (6-9)": range(6, 10), "chain summariser (10)": [10]}
for name, nodes in groups.items():
    cands = [(v, dp, tp) for v in nodes for (dp, tp) in S.samu_enumerate_plans(v)]
    S.samu_simulate_batch(cands, lo, li)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = S.samu_simulate_batch(cands, lo, li)
    e1.record(); torch.cuda.synchronize()
    g = recs_to_numpy(out["recs"])
    ms = e0.elapsed_time(e1)
    print(f"{name:28s} cands={len(cands):3d} ms={ms:8.1f} iters={g['iters'].sum():.3e} req_iters={g['req_iters'].astype(float).sum():.3e} "
          f"iters/ms={g['iters'].sum()/ms:.3e}")
    for dp in (1, 2, 4, 8):
        cs = [c for c in cands if c[1] == dp]
        if not cs: continue
        e0.record(); o2 = S.samu_simulate_batch(cs, lo, li); e1.record(); torch.cuda.synchronize()
        g2 = recs_to_numpy(o2["recs"])
        print(f"    dp={dp}: cands={len(cs)} ms={e0.elapsed_time(e1):7.1f} iters={g2['iters'].sum():.3e} mean_B={g2['req_iters'].astype(float).sum()/g2['iters'].sum():.1f}")
# the whole first-step candidate set (the bench step's K2 work): median of 5 timed calls
allc = [(v, dp, tp) for nodes in groups.values() for v in nodes for (dp, tp) in S.samu_enumerate_plans(v)]
S.samu_simulate_batch(allc, lo, li)
ts = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); S.samu_simulate_batch(allc, lo, li); e1.record(); torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print(f"all {len(allc)} candidates: median {np.median(ts):.2f} ms min {min(ts):.2f} max {max(ts):.2f}")
