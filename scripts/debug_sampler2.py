import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, samu_workloads as W
from paper_2503_16893_b200 import Samu
for name, kw in [("c3", dict(n_prompts=2000)), ("c4", dict(n_docs=200))]:
    w = W.make_workload(name, n_trials=8, **kw)
    P = O.Problem(w); S = Samu(0); S.load_workload(w)
    for tb, T in [(0, 8), (5, 3)]:
        lo, li = P.sample(W.SAMPLING_SEED, tb, T)
        glo, gli = S.samu_sample_lengths(W.SAMPLING_SEED, tb, T)
        g = glo.cpu().numpy().view(np.uint16); gi = gli.cpu().numpy().view(np.uint16)
        bad = np.argwhere(g != lo)
        print(name, tb, T, "n bad", len(bad), bad[:5], "li bad", (gi != li).sum())
        for (k, r) in bad[:3]:
            print("  ", k, r, "node", w.node[r], "pred", w.pred[r], "gpu", g[k, r], gi[k, r], "oracle", lo[k, r], li[k, r])
