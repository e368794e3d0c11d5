"""Randomised planner sweep: small multi-node workloads (chain, evaluator and independent nodes), greedy /
Max / Min with and without preemption, default and SAMU_K2_MODES=always, GPU plan vs oracle plan.

  python scripts/plan_sweep.py [n_seeds]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle as O
import samu_workloads as W
from paper_2503_16893_b200 import Samu
from tests import fixtures as F

SEED = W.SAMPLING_SEED


def sweep(n_seeds, verbose=True):
    bad = checked = 0
    for seed in range(n_seeds):
        rng = np.random.default_rng(7000 + seed)
        sp = F.spec(l_max=400, tp_values=(1, 2), L=2, h=16, c=1000)
        nodes = []
        base = 0   # pred holds global request indices
        for v in range(int(rng.integers(2, 5))):
            ld = F.zero_load() + float(rng.uniform(0, 1.5))
            if rng.random() < 0.4:   # a chain node
                l_in, l_out, pred, chain = [], [], [], []
                for cid in range(int(rng.integers(2, 10))):
                    for j in range(int(rng.integers(1, 4))):
                        pred.append(-1 if j == 0 else base + len(l_in) - 1)
                        chain.append(cid)
                        l_in.append(int(rng.integers(10, 120)))
                        l_out.append(int(rng.integers(3, 70)))
                nodes.append(dict(l_in=np.array(l_in), l_out=np.array(l_out), pred=np.array(pred), chain=np.array(chain),
                                  sp=sp, load=ld))
                finals = [base + i for i in range(len(l_in)) if i + 1 == len(l_in) or chain[i + 1] != chain[i]]
                base += len(l_in)
                if rng.random() < 0.6:   # an evaluator node fed by every chain's final summary
                    e_pred = np.repeat(np.array(finals), int(rng.integers(1, 3)))
                    nodes.append(dict(l_in=np.full(len(e_pred), int(rng.integers(10, 60))),
                                      l_out=rng.integers(1, 40, len(e_pred)), pred=e_pred, sp=sp,
                                      load=F.zero_load() + float(rng.uniform(0, 1.5))))
                    base += len(e_pred)
            else:
                m = int(rng.integers(5, 60))
                nodes.append(dict(l_in=rng.integers(5, 120, m), l_out=rng.integers(1, 100, m), sp=sp, load=ld))
                base += m
        w = F.multi(nodes, eng=F.engine(n_gpus=int(rng.choice([2, 4])), max_num_seqs=int(rng.integers(2, 24)),
                                        kv_cap=int(rng.integers(500, 3000))), n_trials=2)
        P = O.Problem(w)
        for algo in ("greedy", "max", "min"):
            for pre in (True, False):
                if algo == "max" and not pre:
                    continue
                try:
                    po = P.plan_greedy(SEED, 2, algo, preemption=pre)
                except Exception:
                    continue   # infeasible random configuration
                for policy in ("default", "always"):
                    if policy == "always":
                        os.environ["SAMU_K2_MODES"] = "always"
                    try:
                        S = Samu(0)
                        S.load_workload(w)
                        pg = S.samu_plan_greedy(SEED, 2, algo, preemption=pre)
                        pg.pop("n_sims")
                        S.close()
                    except Exception as e:
                        print(f"seed {seed} {algo} pre={pre} {policy}: error {e}")
                        bad += 1
                        continue
                    finally:
                        os.environ.pop("SAMU_K2_MODES", None)
                    checked += 1
                    if pg != po:
                        print(f"seed {seed} {algo} pre={pre} {policy}: plan differs")
                        bad += 1
    return checked, bad


if __name__ == "__main__":
    n_seeds = int(sys.argv[1]) if len(sys.argv) > 1 else 50
    checked, bad = sweep(n_seeds)
    print(f"plan sweep: {n_seeds} seeds, {checked} plans compared, {bad} mismatches")
    sys.exit(1 if bad else 0)
