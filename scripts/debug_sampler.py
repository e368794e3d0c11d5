import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O, samu_workloads as W
from paper_2503_16893_b200 import Samu
w = W.make_workload("c4", n_trials=2, n_docs=200)
P = O.Problem(w); S = Samu(0); S.load_workload(w)
lo, li = P.sample(W.SAMPLING_SEED, 0, 2)
out = (torch.full((2, w.n_req), -7, dtype=torch.int16, device='cuda'), torch.full((2, w.n_req), -7, dtype=torch.int16, device='cuda'))
glo, gli = S.samu_sample_lengths(W.SAMPLING_SEED, 0, 2, out=out)
torch.cuda.synchronize()
g = glo.cpu().numpy().view(np.uint16); gi = gli.cpu().numpy().view(np.uint16)
bad = np.nonzero(g[0] != lo[0])[0]
print("n bad", len(bad), "first", bad[:10], "node of bad", np.unique(w.node[bad]))
for r in bad[:5]:
    print(r, "pred", w.pred[r], "gpu", g[0, r], gi[0, r], "oracle", lo[0, r], li[0, r], "cap", w.cap_y[r])
