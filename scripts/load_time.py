"""Wall time of the pieces of an application (re)load and of one bench step (e2e overhead)."""
import sys, time; sys.path.insert(0, ".")
import numpy as np, torch, samu_workloads as W
from paper_2503_16893_b200 import Samu
w = W.make_workload("c5"); S = Samu(0); S.load_workload(w); torch.cuda.synchronize()


def tm(label, f, n=5):
    ts = []
    for _ in range(n):
        torch.cuda.synchronize(); t0 = time.perf_counter(); f(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    print(f"{label:28s} median {1e3 * np.median(ts):8.3f} ms")


tm("load_workload", lambda: S.load_workload(w))
tm("model_register x all", lambda: [S.samu_model_register(m, s, w.coeff_B, w.coeff[m], w.load[m]) for m, s in enumerate(w.models)])
tm("ecdf_load x all", lambda: [S.samu_ecdf_load(m, w.ecdf_values[m], w.ecdf_cum[m]) for m in range(len(w.models))])
tm("app_load", lambda: S.samu_app_load(w.engine, w.node_model, w.l_in_base, w.cap_y, w.pred, w.node, w.chain))
ready = [v for v in range(w.n_nodes) if not np.any((w.pred[w.node == v] >= 0) & (w.node[np.maximum(w.pred[w.node == v], 0)] != v))]
cands = [(v, dp, tp) for v in ready for (dp, tp) in S.samu_enumerate_plans(v)]
lo, li = S.samu_sample_lengths(w.seed, 0, w.n_trials)
tm("sample", lambda: S.samu_sample_lengths(w.seed, 0, w.n_trials, out=(lo, li)))
tm("simulate+summary", lambda: S.samu_simulate_batch(cands, lo, li, summary=True))
tm("load + step", lambda: (S.load_workload(w), S.samu_sample_lengths(w.seed, 0, w.n_trials, out=(lo, li)),
                            S.samu_simulate_batch(cands, lo, li, summary=True)))
