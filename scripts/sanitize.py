"""Small end-to-end runs for compute-sanitizer: sampler, fresh / cut / committed / resumed /
reloaded simulations with preemption, chains and evaluator arrivals, and the greedy."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
for name, kw in [("c2", dict(n_prompts=60)), ("c4", dict(n_docs=20)), ("c5", dict(n_prompts=20, n_docs=10))]:
    w = W.make_workload(name, n_trials=2, **kw)
    S = Samu(0); S.load_workload(w)
    lo, li = S.samu_sample_lengths(w.seed, 0, 2)
    cands = [(v, dp, tp) for v in range(w.n_nodes) if w.pred[w.node == v].max() < 0 or True
             for (dp, tp) in S.samu_enumerate_plans(v)[:3] if not (w.pred[w.node == v] >= 0).any() or
             (w.node[np.maximum(w.pred[w.node == v], 0)] == v).all()]
    S.samu_simulate_batch(cands, lo, li, summary=True, want_fin_iter=True, want_fin_t=True)
    os.environ["SAMU_K2_MODES"] = "always"   # the LEAN / FRESH paths on this small batch too
    S.samu_simulate_batch(cands, lo, li, summary=True)
    os.environ["SAMU_K2_OVERLAP"] = "0"      # ... as launches chained in one stream (PDL)
    S.samu_simulate_batch(cands, lo, li, summary=True)
    del os.environ["SAMU_K2_MODES"]
    st = S.fresh_state(2)
    S.samu_simulate_batch([cands[0][:3] + (0, -1, 1)], lo, li, state=st, time_limit=np.array([[5.0, 7.0]]))
    S.samu_simulate_batch([cands[0][:3] + (1, -1, 0), (cands[0][0], 1, 1, 0, -1, 0)], lo, li, state=st)
    print(name, "greedy stages", len(S.samu_plan_greedy(w.seed, 2)["stages"]))
    os.environ["SAMU_K2_MODES"] = "always"   # the planner's fresh full and cut simulations on LEAN / FRESH
    print(name, "greedy stages (all K2 paths)", len(S.samu_plan_greedy(w.seed, 2)["stages"]))
    del os.environ["SAMU_K2_MODES"]
    S.close()
torch.cuda.synchronize()
print("sanitize run ok")
