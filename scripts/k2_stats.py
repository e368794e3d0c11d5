"""Event statistics of K2 per node of the C5 first step (needs a SAMU_DEFINES=SAMU_K2_STATS build).

  python scripts/k2_stats.py [T] [node,node,...]   (default: per application)
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import samu_workloads as W
from paper_2503_16893_b200 import Samu
from paper_2503_16893_b200.binding import lib

NAMES = ["items", "loop trips", "prefill iters", "admitted", "admission rounds", "scan rounds", "decode fast",
         "decode runs", "run iters", "victims", "preempting decodes", "retire events", "finished", "retire transposed",
         "chunked runs", "-", "runs 1", "runs 2-4", "runs 5-8", "runs 9-16", "runs 17-32", "runs 33-64",
         "runs 65-128", "runs >128", "runs ending in preemption", "runs searched (tight)"]
T = int(sys.argv[1]) if len(sys.argv) > 1 else 64
w = W.make_workload("c5", n_trials=T)
S = Samu(0)
S.load_workload(w)
lo, li = S.samu_sample_lengths(w.seed, 0, T)
f = lib().samu_debug_k2_stats
f.argtypes = [C.c_void_p, C.c_int]
buf = (C.c_ulonglong * 32)()
if len(sys.argv) > 2 and ":" in sys.argv[2]:   # one candidate node:dp:tp
    groups = [(sys.argv[2], None)]
elif len(sys.argv) > 2:
    groups = [(f"node {v}", [int(v)]) for v in sys.argv[2].split(",")]
else:
    groups = [("ensembling", range(0, 6)), ("routing", range(6, 10)), ("chain", [10])]
for name, nodes in groups:
    cands = ([tuple(int(x) for x in name.split(":"))] if nodes is None else
             [(v, dp, tp) for v in nodes for (dp, tp) in S.samu_enumerate_plans(v)])
    f(buf, 1)
    out = S.samu_simulate_batch(cands, lo, li)
    torch.cuda.synchronize()
    f(buf, 1)
    it = buf[2] + buf[6] + buf[8] + buf[10]
    print(f"== {name}: iterations {it} (prefill {buf[2]}, decode fast {buf[6]}, run iters {buf[8]}, preempting {buf[10]})")
    for i, n in enumerate(NAMES):
        print(f"   {n:20s} {buf[i]:14d}  per iter {buf[i] / max(it, 1):.4f}")
