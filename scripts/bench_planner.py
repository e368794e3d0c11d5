"""Wall time of the full Algorithm 1 planner (samu_plan_greedy) on the paper-shaped workloads —
the paper's "extra time" — on one B200.

  python scripts/bench_planner.py c2:64 c5:1024:min ...   (workload:trials[:greedy|max|min])"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import samu_workloads as W  # noqa: E402
from paper_2503_16893_b200 import Samu  # noqa: E402

out = []
for arg in sys.argv[1:] or ["c2:64", "c3:64", "c4:64"]:
    f = arg.split(":")
    name, T, algo = f[0], int(f[1]), (f[2] if len(f) > 2 else "greedy")
    w = W.make_workload(name, n_trials=T)
    S = Samu(0)
    S.load_workload(w)
    S.samu_plan_greedy(W.SAMPLING_SEED, T, algo=algo)      # warm-up (kernel load; the context keeps the planner's buffers)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = S.samu_plan_greedy(W.SAMPLING_SEED, T, algo=algo)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    rec = dict(workload=name, trials=T, algorithm=algo, requests=w.n_req, nodes=w.n_nodes, planner_s=dt,
               stages=len(plan["stages"]), planned_total_s=plan["total"], cand_evals=plan["n_cand_evals"],
               candidate_trial_sims=plan["n_sims"], sims_per_s=plan["n_sims"] / dt,
               plan=[(s["entries"], s["fstar"], round(s["mean_tE"], 3)) for s in plan["stages"]])
    print(json.dumps(rec), flush=True)
    out.append(rec)
    S.close()
json.dump(out, open(os.path.join("gpurun_out", "planner.json"), "w"), indent=1)
