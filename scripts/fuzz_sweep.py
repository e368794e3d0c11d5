"""Randomised GPU-vs-oracle sweep beyond the unit tests: tiny workloads with chains / independent
requests, tight KV / slot / token budgets, every block-size path, time limits, and every K2 path
(SAMU_K2_MODES=always and the default).  Prints mismatches; exit code 1 if any.

  python scripts/fuzz_sweep.py [n_seeds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import samu_workloads as W
from paper_2503_16893_b200 import Samu, recs_to_numpy
from tests import fixtures as F

SEED = W.SAMPLING_SEED


def sweep(n_seeds, verbose=True):
    bad = 0
    checked = 0
    for seed in range(n_seeds):
        rng = np.random.default_rng(9000 + seed)
        chains = seed % 2 == 0
        l_in, l_out, pred, chain = [], [], [], []
        n_groups = int(rng.integers(3, 30))
        for cid in range(n_groups):
            for j in range(int(rng.integers(1, 6)) if chains else 1):
                pred.append(-1 if j == 0 else len(l_in) - 1)
                chain.append(cid if chains else -1)
                l_in.append(int(rng.integers(1, 50)))
                l_out.append(int(rng.integers(0, 90)))
        bsz = [16, 16, 8, 4, 12, 1, 32][seed % 7]
        eng = F.engine(kv_cap=int(rng.integers(10, 60)) * 16, min_batched_tokens=int(rng.integers(160, 600)),
                       max_num_seqs=int(rng.integers(1, 48)), block_size=bsz, n_gpus=4)
        cf = rng.uniform(1e-4, 1e-2, (W.N_TP_SLOTS, 3, 2, F.NB))
        cf[:, 0, 0, :] = 1e-12
        ld = F.zero_load() + float(rng.uniform(0, 2))
        w = F.tiny(np.array(l_in), np.array(l_out), sp=F.spec(l_max=220, tp_values=(1, 2), L=2, h=16, c=1000), eng=eng,
                   cf=cf, pred=np.array(pred), chain=np.array(chain) if chains else None, n_trials=3, load=ld)
        P = O.Problem(w)
        S = Samu(0)
        try:
            S.load_workload(w)
        except Exception as e:   # an invalid random engine (capacity below one sequence): skip
            S.close()
            continue
        lo, li = P.sample(SEED, 0, 3)
        glo, gli = S.samu_sample_lengths(SEED, 0, 3)
        valid = set(tuple(x) for x in P.plans(w.node_model[0]))
        cands = [c for c in [(0, 1, 1), (0, 2, 1), (0, 2, 2), (0, 3, 1), (0, 4, 1)] if (c[1], c[2]) in valid]
        if not cands:
            S.close()
            continue
        tau = None
        if seed % 3 == 0:
            full = [P.simulate(*c, lo, li)[0]["t_end"] for c in cands]
            tau = np.array([f * rng.uniform(0.1, 0.95, 3) for f in full])
        for policy in ("default", "always"):
            if policy == "always":
                os.environ["SAMU_K2_MODES"] = "always"
            try:
                g = recs_to_numpy(S.samu_simulate_batch(cands, glo, gli, time_limit=tau)["recs"])
            except Exception as e:
                print(f"seed {seed} {policy}: error {e}")
                bad += 1
                continue
            finally:
                os.environ.pop("SAMU_K2_MODES", None)
            for ci, cd in enumerate(cands):
                o = P.simulate(*cd, lo, li, tau=None if tau is None else tau[ci])[0]
                checked += 1
                for f in ("t_end", "flops_lo", "flops_hi", "req_iters", "iters", "flags"):
                    if not np.array_equal(g[ci][f], o[f]):
                        print(f"seed {seed} {policy} cand {cd} bs {bsz}: {f} differs {g[ci][f]} vs {o[f]}")
                        bad += 1
                        break
        S.close()
    return checked, bad


if __name__ == "__main__":
    n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    checked, bad = sweep(n_seeds)
    print(f"fuzz sweep: {n_seeds} seeds, {checked} candidate x policy records (3 trials each) compared, {bad} mismatches")
    sys.exit(1 if bad else 0)
