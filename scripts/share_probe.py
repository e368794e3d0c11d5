"""How much K2 time would sharing one schedule across the tp variants of a (node, dp) group
save?  Times the C5 first-step candidate set against the subset 'group heads (largest tp) +
variants whose schedule differs from the head's in some trial' (identified from the records
of the full set: equal iters and req_iters in every trial)."""
import os, sys, collections
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu, recs_to_numpy

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
w = W.make_workload("c5", n_trials=T)
S = Samu(0); S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, T)
ready = [v for v in range(w.n_nodes) if v != w.n_nodes - 1]
cands = [(v, dp, tp) for v in ready for (dp, tp) in S.samu_enumerate_plans(v)]


def timed(cs, reps=3):
    S.samu_simulate_batch(cs, lo, li)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); out = S.samu_simulate_batch(cs, lo, li); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best, recs_to_numpy(out["recs"])


ms_all, g = timed(cands)
grp = collections.defaultdict(list)
for i, (v, dp, tp) in enumerate(cands):
    grp[(v, dp)].append((tp, i))
keep, per_node = [], collections.Counter()
for (v, dp), lst in grp.items():
    lst.sort()
    head = lst[-1][1]
    for tp, i in lst:
        same = np.array_equal(g[i]["iters"], g[head]["iters"]) and np.array_equal(g[i]["req_iters"], g[head]["req_iters"])
        frac = np.mean((g[i]["iters"] == g[head]["iters"]) & (g[i]["req_iters"] == g[head]["req_iters"]))
        if i == head or not same:
            keep.append(cands[i])
        print(f"node {v:2d} dp {dp} tp {tp}: in sync with head in {frac*100:5.1f}% of trials", flush=True)
ms_keep, _ = timed(keep)
print(f"all {len(cands)} candidates: {ms_all:.1f} ms; heads + out-of-sync variants ({len(keep)}): {ms_keep:.1f} ms")
for nodes, name in ((range(0, 10), "LEAN nodes 0-9"), ([10], "FRESH node 10")):
    a = [c for c in cands if c[0] in nodes]; b = [c for c in keep if c[0] in nodes]
    print(f"{name}: all {len(a)} {timed(a)[0]:.1f} ms, kept {len(b)} {timed(b)[0]:.1f} ms")
for v in range(11):
    a = [c for c in cands if c[0] == v]
    print(f"node {v}: {len(a)} cands {timed(a)[0]:.1f} ms")
