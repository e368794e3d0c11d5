import sys, time; sys.path.insert(0, ".")
import torch, samu_workloads as W
from paper_2503_16893_b200 import Samu
w = W.make_workload("c5"); S = Samu(0); S.load_workload(w); torch.cuda.synchronize()
for i in range(5):
    t0 = time.perf_counter(); S.load_workload(w); torch.cuda.synchronize(); print("load_workload", round(time.perf_counter() - t0, 4))
