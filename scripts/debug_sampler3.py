import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, samu_workloads as W
from paper_2503_16893_b200 import Samu
for rep in range(2):
  for T in (2, 8):
    w = W.make_workload("c4", n_trials=8, n_docs=200)
    P = O.Problem(w); S = Samu(0); S.load_workload(w)
    lo, li = P.sample(W.SAMPLING_SEED, 0, T)
    glo, gli = S.samu_sample_lengths(W.SAMPLING_SEED, 0, T)
    g = glo.cpu().numpy().view(np.uint16)
    bad = np.argwhere(g != lo)
    print(rep, T, "n bad", len(bad), bad[:3].tolist())
    lo2, li2 = P.sample(W.SAMPLING_SEED, 0, T)
    print("   oracle self-consistent:", np.array_equal(lo, lo2))
