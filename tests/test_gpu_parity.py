"""GPU parity: the CUDA path (through libsamu's C ABI) vs the CPU oracle, element by element.

Bar (BASELINE.json north_star): sampled lengths, per-request finish iterations, records and the
greedy plan bit-exact; fp64 totals within 1e-9 rel — asserted here as exact equality, since
both sides evaluate the same operations in the same order (readings c17, c22, c24).
"""
import contextlib
import os

import numpy as np
import pytest

import oracle as O
import samu_workloads as W
from tests import fixtures as F

pytestmark = pytest.mark.gpu
SEED = W.SAMPLING_SEED


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def gpu(w):
    from paper_2503_16893_b200 import Samu
    S = Samu(0)
    S.load_workload(w)
    return S


@contextlib.contextmanager
def k2_modes(policy, overlap=None):
    """SAMU_K2_MODES: "always" runs K2's LEAN / FRESH paths even on batches below the size rule;
    SAMU_K2_OVERLAP="0": their launches run chained in one stream (programmatic dependent launch,
    the large-batch configuration) instead of LEAN beside the others on a second stream."""
    env = {"SAMU_K2_MODES": policy, "SAMU_K2_OVERLAP": overlap}
    old = {k: os.environ.get(k) for k in env}
    for k, v in env.items():
        if v is not None:
            os.environ[k] = v
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def u16(t):
    return t.cpu().numpy().view(np.uint16)


def recs(out):
    from paper_2503_16893_b200 import recs_to_numpy
    return recs_to_numpy(out["recs"])


def assert_rec_equal(g, o, ctx=""):
    for f in ("t_end", "flops_lo", "flops_hi", "req_iters", "iters", "flags"):
        assert np.array_equal(g[f], o[f]), f"{ctx}: field {f} differs\n gpu={g[f][:8]}\n ora={o[f][:8]}"


def plans_sample(P, node, k=6):
    pl = P.plans(P.w.node_model[node])
    if len(pl) <= k:
        return pl
    idx = np.linspace(0, len(pl) - 1, k).round().astype(int)
    return [pl[i] for i in sorted(set(idx))]


# ------------------------------------------------------------------------------------------
# K1 sampler
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,kw", [("c1", {}), ("c2", dict(n_prompts=300)), ("c3", dict(n_prompts=2000)),
                                     ("c4", dict(n_docs=200)), ("c5", dict(n_prompts=500, n_docs=200))])
def test_sampler_bit_exact(name, kw):
    w = W.make_workload(name, n_trials=8, **kw)
    P = O.Problem(w)
    S = gpu(w)
    for tb, T in [(0, 8), (5, 3)]:
        lo, li = P.sample(SEED, tb, T)
        glo, gli = S.samu_sample_lengths(SEED, tb, T)
        assert np.array_equal(u16(glo), lo) and np.array_equal(u16(gli), li)


def test_sampler_full_size_c5_sampled_trials():
    # BASELINE configs[4] at full size (50,000 requests): trials 0, 511, 1023 checked exactly
    w = W.make_workload("c5")
    P = O.Problem(w)
    S = gpu(w)
    for tb in (0, 511, 1023):
        lo, li = P.sample(SEED, tb, 1)
        glo, gli = S.samu_sample_lengths(SEED, tb, 1)
        assert np.array_equal(u16(glo), lo) and np.array_equal(u16(gli), li)


# ------------------------------------------------------------------------------------------
# K2 simulation, fresh state
# ------------------------------------------------------------------------------------------
def _sim_parity(w, cands, T, tb=0, tau=None):
    P = O.Problem(w)
    S = gpu(w)
    lo, li = P.sample(SEED, tb, T)
    glo, gli = S.samu_sample_lengths(SEED, tb, T)
    out = S.samu_simulate_batch(cands, glo, gli, time_limit=tau, want_fin_iter=True, want_fin_t=True)
    g = recs(out)
    fi = out["fin_iter"].cpu().numpy().view(np.uint32)
    ft = out["fin_t"].cpu().numpy()
    # the same batch without per-request outputs: independent nodes without a time limit run on
    # K2's LEAN path (k_simulate<16, ., 1>), the rest on the general one
    with k2_modes("always"):
        g_lean = recs(S.samu_simulate_batch(cands, glo, gli, time_limit=tau))
    with k2_modes("always", overlap="0"):
        g_chain = recs(S.samu_simulate_batch(cands, glo, gli, time_limit=tau))
    for ci, cd in enumerate(cands):
        node, dp, tp = cd[:3]
        o, ofi, oft = P.simulate(node, dp, tp, lo, li, tau=None if tau is None else tau[ci], want_fin=True)
        assert_rec_equal(g[ci], o, f"cand {cd}")
        assert_rec_equal(g_lean[ci], o, f"cand {cd} without per-request outputs")
        assert_rec_equal(g_chain[ci], o, f"cand {cd} with the K2 launches chained in one stream")
        a, b = w.node_range(node)
        assert np.array_equal(fi[ci][:, a:b], ofi[:, a:b]), f"finish iterations differ for {cd}"
        assert np.array_equal(ft[ci][:, a:b], oft[:, a:b]), f"finish times differ for {cd}"
    return g


@pytest.mark.parametrize("name,kw,T", [("c1", {}, 1), ("c2", dict(n_prompts=400), 4), ("c3", dict(n_prompts=1500), 3)])
def test_simulate_bit_exact_independent(name, kw, T):
    w = W.make_workload(name, n_trials=T, **kw)
    P = O.Problem(w)
    cands = []
    for v in range(w.n_nodes):
        for (dp, tp) in plans_sample(P, v, 5):
            cands.append((v, dp, tp))
    _sim_parity(w, cands, T, tb=2)


def test_simulate_bit_exact_time_limits():
    w = W.make_workload("c2", n_prompts=300, n_trials=3)
    P = O.Problem(w)
    cands = [(0, 1, 1), (2, 2, 1), (5, 1, 4), (3, 4, 2)]
    lo, li = P.sample(SEED, 0, 3)
    full = [P.simulate(*c, lo, li)[0]["t_end"] for c in cands]
    rng = np.random.default_rng(0)
    tau = np.array([f * rng.uniform(0.1, 0.9, 3) for f in full])
    g = _sim_parity(w, cands, 3, tau=tau)
    assert np.all(g["flags"] & 2)


@pytest.mark.parametrize("seed", range(12))
def test_simulate_fuzz_tight_kv_preemption(seed):
    # random small workloads with few KV blocks: preemption, token budget and slot limits; block
    # sizes cover the power-of-two and the general kernel instantiation
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(5, 120))
    lin = rng.integers(1, 60, n)
    lout = rng.integers(0, 80, n)
    eng = F.engine(kv_cap=int(rng.integers(9, 40)) * 16, min_batched_tokens=int(rng.integers(144, 400)),
                   max_num_seqs=int(rng.integers(1, 40)), block_size=[4, 8, 16, 7, 12, 1][seed % 6], n_gpus=4)
    cf = np.zeros((W.N_TP_SLOTS, 3, 2, F.NB))
    cf[:, :, :, :] = rng.uniform(1e-4, 1e-2, (W.N_TP_SLOTS, 3, 2, F.NB))
    cf[:, 0, 0, :] = 1e-12
    w = F.tiny(lin, lout, sp=F.spec(l_max=140, tp_values=(1, 2), L=2, h=16, c=1000), eng=eng, cf=cf, n_trials=2)
    _sim_parity(w, [(0, 1, 1), (0, 2, 1), (0, 1, 2), (0, 3, 1)], 2)


@pytest.mark.parametrize("seed", range(4))
def test_simulate_fuzz_signed_costs_and_cuts(seed):
    # long decode runs (32-iteration cost chunks) with signed cost terms (non-monotone clock)
    # and time limits falling inside chunks: the chunk's stop test must match the sequential loop
    rng = np.random.default_rng(300 + seed)
    n = int(rng.integers(20, 200))
    lin = rng.integers(1, 30, n)
    lout = rng.integers(40, 400, n)
    eng = F.engine(max_num_seqs=int(rng.integers(4, 64)), block_size=16, n_gpus=2)
    cf = rng.uniform(1e-4, 1e-2, (W.N_TP_SLOTS, 3, 2, F.NB))
    cf[:, 0, 0, :] = 1e-12
    cf[:, 1, 1, :] = -rng.uniform(0, 4e-3, (W.N_TP_SLOTS, F.NB))   # negative prep constant
    w = F.tiny(lin, lout, sp=F.spec(l_max=512, tp_values=(1, 2), L=2, h=16, c=1000), eng=eng, cf=cf, n_trials=3)
    cands = [(0, 1, 1), (0, 2, 1), (0, 1, 2)]
    _sim_parity(w, cands, 3)
    tau = rng.uniform(0.05, 2.0, (len(cands), 3))
    _sim_parity(w, cands, 3, tau=tau)


@pytest.mark.parametrize("load,cost", [(1.0, 3 * 2.0 ** -53), (1.0, 2.0 ** -53), (1.0, 5 * 2.0 ** -54),
                                       (1.0, 0.3), (0.0, 3 * 2.0 ** -53), (1.0, 1e-17), (3.0, 2.0 ** -51 + 2.0 ** -52)])
def test_chunk_sum_ties_and_binade_crossings(load, cost):
    # Decode-run chunks sum their 32 costs in parallel (binade-local rounding + warp scan) and fall
    # back to the sequential walk on ties / binade crossings.  Constant costs of exactly 1.5 or
    # 0.5 ulp of the clock make every add a round-half-even tie whose result alternates with the
    # clock's last bit; 0.3 s per iteration crosses binades every few iterations.  The clock must
    # equal the oracle's one-by-one sum bit for bit.
    ld = F.zero_load()
    ld[0, 0] = load
    w = F.tiny(np.array([5, 9, 17, 3]), np.array([200, 77, 140, 5]), load=ld, cf=F.coeff("const", cost),
               sp=F.spec(l_max=512))
    g = _sim_parity(w, [(0, 1, 1)], 1)
    assert g["iters"][0, 0] == 200


def test_candidate_table_both_paths():
    # launches with <= 400 candidates read them from the constant bank, larger ones from global
    # memory (k_simulate<., CONSTC>): both must give the oracle's records
    w = W.make_workload("c2", n_prompts=120, n_trials=2)
    P = O.Problem(w)
    S = gpu(w)
    cands = [(v, dp, tp) for v in range(w.n_nodes) for (dp, tp) in P.plans(w.node_model[v])]
    lo, li = P.sample(SEED, 0, 2)
    glo, gli = S.samu_sample_lengths(SEED, 0, 2)
    small = recs(S.samu_simulate_batch(cands, glo, gli))
    big = recs(S.samu_simulate_batch(cands * 5, glo, gli))
    assert len(cands) * 5 > 400
    for ci, cd in enumerate(cands):
        o = P.simulate(*cd, lo, li)[0]
        assert_rec_equal(small[ci], o, f"const table {cd}")
        for r in range(5):
            assert_rec_equal(big[ci + r * len(cands)], o, f"global table {cd} copy {r}")


@pytest.mark.parametrize("seed", range(6))
def test_simulate_fuzz_chains_tight_kv(seed):
    # random chains (successor prompt = base + predecessor's output) under tight KV,
    # slot and token budgets: the general path (with per-request outputs) and, for block size
    # 16, the FRESH path (without) against the oracle
    rng = np.random.default_rng(500 + seed)
    n_chains = int(rng.integers(3, 25))
    l_in, l_out, pred, chain = [], [], [], []
    for c in range(n_chains):
        for j in range(int(rng.integers(1, 7))):
            pred.append(-1 if j == 0 else len(l_in) - 1)
            chain.append(c)
            l_in.append(int(rng.integers(1, 40)))
            l_out.append(int(rng.integers(1, 60)))
    eng = F.engine(kv_cap=int(rng.integers(14, 48)) * 16, min_batched_tokens=int(rng.integers(200, 500)),
                   max_num_seqs=int(rng.integers(2, 24)), block_size=[16, 8, 16, 12, 16, 4][seed], n_gpus=4)
    cf = rng.uniform(1e-4, 1e-2, (W.N_TP_SLOTS, 3, 2, F.NB))
    cf[:, 0, 0, :] = 1e-12
    w = F.tiny(np.array(l_in), np.array(l_out), sp=F.spec(l_max=200, tp_values=(1, 2), L=2, h=16, c=1000), eng=eng,
               cf=cf, pred=np.array(pred), chain=np.array(chain), n_trials=2)
    _sim_parity(w, [(0, 1, 1), (0, 2, 1), (0, 2, 2), (0, 3, 1)], 2)


def test_hand_traces_on_gpu():
    for kind, expect_t in (("const", 63.0), ("B", 80.0), ("S", 32 + 784 + 1012 + 33 + 979)):
        w = F.tiny([16, 16], [40, 40], sp=F.spec(l_max=64), cf=kind, eng=F.engine(kv_cap=64, min_batched_tokens=64))
        g = _sim_parity(w, [(0, 1, 1)], 1)
        assert g["t_end"][0, 0] == expect_t
    w = F.tiny([10, 10], [2, 1], eng=F.engine(max_num_seqs=2))
    g = _sim_parity(w, [(0, 1, 1)], 1)
    assert g["t_end"][0, 0] == 2.0


def test_uniform_lengths_exactly_L_iterations_gpu():
    for L in (1, 3, 50):
        # reading c4 preconditions: max_num_seqs >= n and token budget >= sum(l_in)
        w = F.tiny(np.full(250, 20), np.full(250, L), eng=F.engine(min_batched_tokens=100000))
        g = _sim_parity(w, [(0, 1, 1)], 1)
        assert g["iters"][0, 0] == L


# ------------------------------------------------------------------------------------------
# dependencies (chains + evaluator), commit / resume state
# ------------------------------------------------------------------------------------------
def test_dependency_parity_c4():
    w = W.make_workload("c4", n_docs=150, n_trials=3)
    P = O.Problem(w)
    S = gpu(w)
    lo, li = P.sample(SEED, 0, 3)
    glo, gli = S.samu_sample_lengths(SEED, 0, 3)
    for (dps, tps), (dpe, tpe) in [((1, 1), (1, 2)), ((2, 2), (4, 1)), ((3, 1), (1, 8))]:
        out = S.samu_simulate_batch([(0, dps, tps, 0, -1, 0), (1, dpe, tpe, 0, 0, 0)], glo, gli, want_fin_iter=True,
                                    want_fin_t=True)
        g = recs(out)
        os_, ofs, fts = P.simulate(0, dps, tps, lo, li, want_fin=True)
        oe, ofe, fte = P.simulate(1, dpe, tpe, lo, li, src_fin=fts, want_fin=True)
        assert_rec_equal(g[0], os_, "summariser")
        assert_rec_equal(g[1], oe, "evaluator")
        # the summariser alone without per-request outputs runs on K2's FRESH path (chains, no
        # state / cut / outputs)
        with k2_modes("always"):
            g0 = recs(S.samu_simulate_batch([(0, dps, tps)], glo, gli))[0]
        assert_rec_equal(g0, os_, "summariser, FRESH path")
        fi = out["fin_iter"].cpu().numpy().view(np.uint32)
        a, b = w.node_range(0)
        assert np.array_equal(fi[0][:, a:b], ofs[:, a:b])
        a, b = w.node_range(1)
        assert np.array_equal(fi[1][:, a:b], ofe[:, a:b])


def _state_np(s):
    return dict(st=s["st"].cpu().numpy().view(np.uint32), g=s["g"].cpu().numpy().view(np.uint16),
                fin_t=s["fin_t"].cpu().numpy(), over=s["over"].cpu().numpy())


@pytest.mark.parametrize("name,kw,node,plans", [
    ("c2", dict(n_prompts=300), 4, [(2, 1), (1, 2)]),
    ("c4", dict(n_docs=120), 0, [(1, 1), (2, 1)]),
])
def test_commit_then_resume_and_reload_parity(name, kw, node, plans):
    T = 3
    w = W.make_workload(name, n_trials=T, **kw)
    P = O.Problem(w)
    S = gpu(w)
    lo, li = P.sample(SEED, 0, T)
    glo, gli = S.samu_sample_lengths(SEED, 0, T)
    (dp1, tp1), (dp2, tp2) = plans
    full = P.simulate(node, dp1, tp1, lo, li)[0]["t_end"]
    tau = full * np.array([0.3, 0.55, 0.8])
    ost = P.fresh_state(T)
    gst = S.fresh_state(T)
    o1, _, _ = P.simulate(node, dp1, tp1, lo, li, state=ost, tau=tau, commit=True)
    g1 = recs(S.samu_simulate_batch([(node, dp1, tp1, 0, -1, 1)], glo, gli, state=gst, time_limit=tau[None]))
    assert_rec_equal(g1[0], o1, "cut+commit")
    gs = _state_np(gst)
    for f in ("st", "g", "fin_t", "over"):
        assert np.array_equal(gs[f], ost[f]), f"state field {f} differs after commit"
    # resume with the same plan, and reload with another plan, from the committed state
    ost2 = {k: v.copy() for k, v in ost.items()}
    o2, _, _ = P.simulate(node, dp1, tp1, lo, li, resume=1, state=ost)
    o3, _, _ = P.simulate(node, dp2, tp2, lo, li, resume=0, state=ost2)
    g2 = recs(S.samu_simulate_batch([(node, dp1, tp1, 1, -1, 0), (node, dp2, tp2, 0, -1, 0)], glo, gli, state=gst))
    assert_rec_equal(g2[0], o2, "resume")
    assert_rec_equal(g2[1], o3, "reload")


# ------------------------------------------------------------------------------------------
# K3 summaries
# ------------------------------------------------------------------------------------------
def test_summary_mean_and_percentiles():
    w = W.make_workload("c2", n_prompts=200, n_trials=37)
    S = gpu(w)
    glo, gli = S.samu_sample_lengths(SEED, 0, 37)
    out = S.samu_simulate_batch([(0, 1, 1), (5, 2, 4)], glo, gli, summary=True)
    g = recs(out)
    for ci in range(2):
        t = g["t_end"][ci]
        s = 0.0
        for x in t:
            s += float(x)
        sm = out["summary"][ci]
        assert sm["mean_t"] == s / 37
        for p in (50, 90, 99):
            assert sm[f"p{p}_t"] == np.percentile(t, p, method="inverted_cdf")


# ------------------------------------------------------------------------------------------
# greedy planner (Algorithm 1)
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,kw,T", [
    ("c1", {}, 1),
    ("c2", dict(n_prompts=120), 3),
    ("c3", dict(n_prompts=600), 2),
    ("c4", dict(n_docs=60), 2),
])
@pytest.mark.parametrize("algo", ["greedy", "max", "min"])
def test_greedy_plan_bit_exact(name, kw, T, algo):
    # Algorithm 1 and the paper's two competitors on the same device estimator
    w = W.make_workload(name, n_trials=T, **kw)
    po = O.Problem(w).plan_greedy(SEED, T, algo)
    pg = gpu(w).samu_plan_greedy(SEED, T, algo)
    assert len(pg["stages"]) == len(po["stages"])
    for sg, so in zip(pg["stages"], po["stages"]):
        assert sg["entries"] == so["entries"]
        assert sg["fstar"] == so["fstar"]
        assert sg["mean_tE"] == so["mean_tE"]
        assert sg["T_E"] == so["T_E"]
    assert pg["total"] == po["total"]
    assert pg["n_cand_evals"] == po["n_cand_evals"]


@pytest.mark.parametrize("algo", ["greedy", "max", "min"])
def test_planners_fig1_and_even_split_fixtures(algo):
    # S:645 Fig. 1 fixture and the P:743 repartition example, every planner bit-exact
    for w, T in ((F.fig1(), 1), (F.even_split_4x8(), 2)):
        po = O.Problem(w).plan_greedy(SEED, T, algo)
        pg = gpu(w).samu_plan_greedy(SEED, T, algo)
        pg.pop("n_sims")
        assert pg == po


# §5.5 ablations: no-preemption variants and known output lengths
@pytest.mark.parametrize("algo", ["greedy", "min"])
@pytest.mark.parametrize("name,kw,T", [
    ("c2", dict(n_prompts=120), 3),
    ("c4", dict(n_docs=60), 2),
    ("c5", dict(n_prompts=40, n_docs=30), 2),
])
def test_no_preemption_plan_bit_exact(name, kw, T, algo):
    w = W.make_workload(name, n_trials=T, **kw)
    po = O.Problem(w).plan_greedy(SEED, T, algo, preemption=False)
    pg = gpu(w).samu_plan_greedy(SEED, T, algo, preemption=False)
    pg.pop("n_sims")
    assert pg == po


@pytest.mark.parametrize("preemption", [True, False])
def test_planner_all_k2_paths(preemption):
    # every planner simulation that qualifies runs on K2's LEAN / FRESH / cut paths
    # (SAMU_K2_MODES=always), including never-committed chain nodes without dependents (FRESH
    # with a WorkloadState buffer present) and their cut simulations; the plan must not change
    rng = np.random.default_rng(77)
    l_in, l_out, pred, chain = [], [], [], []
    for c in range(12):
        for j in range(int(rng.integers(1, 5))):
            pred.append(-1 if j == 0 else len(l_in) - 1)
            chain.append(c)
            l_in.append(int(rng.integers(20, 200)))
            l_out.append(int(rng.integers(5, 80)))
    sp = F.spec(l_max=600, tp_values=(1, 2), L=2, h=16, c=1000)
    ld = F.zero_load() + 0.5
    w = F.multi([dict(l_in=np.array(l_in), l_out=np.array(l_out), pred=np.array(pred), chain=np.array(chain), sp=sp,
                      load=ld),
                 dict(l_in=rng.integers(5, 100, 40), l_out=rng.integers(5, 120, 40), sp=sp, load=ld),
                 dict(l_in=rng.integers(5, 100, 30), l_out=rng.integers(5, 90, 30), sp=sp, load=ld)],
                eng=F.engine(n_gpus=4, max_num_seqs=16, kv_cap=2000), n_trials=3)
    po = O.Problem(w).plan_greedy(SEED, 3, "greedy", preemption=preemption)
    with k2_modes("always"):
        pg = gpu(w).samu_plan_greedy(SEED, 3, "greedy", preemption=preemption)
    pg.pop("n_sims")
    assert pg == po
    with k2_modes("always", overlap="0"):   # the K2 launches of every batch chained in one stream
        pc = gpu(w).samu_plan_greedy(SEED, 3, "greedy", preemption=preemption)
    pc.pop("n_sims")
    assert pc == po


def test_known_lengths_bit_exact():
    w = W.make_workload("c5", n_prompts=200, n_docs=60, n_trials=1)
    rng = np.random.default_rng(7)
    l_true = rng.integers(0, 5000, w.n_req).astype(np.uint32)
    l_true[::17] = 0
    S = gpu(w)
    glo, gli = S.samu_known_lengths(l_true)
    olo, oli = O.Problem(w).known_lengths(l_true)
    assert (u16(glo) == olo).all() and (u16(gli) == oli).all()


@pytest.mark.parametrize("algo", ["greedy", "max", "min"])
def test_known_lengths_plan_bit_exact(algo):
    w = W.make_workload("c5", n_prompts=40, n_docs=30, n_trials=1)
    l_true = np.random.default_rng(11).integers(1, 700, w.n_req).astype(np.uint32)
    for pre in (True, False):
        po = O.Problem(w).plan_greedy(SEED, 1, algo, preemption=pre, known_l_out=l_true)
        pg = gpu(w).samu_plan_greedy(SEED, 1, algo, preemption=pre, known_l_out=l_true)
        pg.pop("n_sims")
        assert pg == po


# runtime replay with the dynamic scheduler
@pytest.mark.parametrize("algo", ["greedy", "max", "min"])
@pytest.mark.parametrize("name,kw", [
    ("c2", dict(n_prompts=120)),
    ("c4", dict(n_docs=60)),
    ("c5", dict(n_prompts=40, n_docs=30)),
])
def test_replay_bit_exact(name, kw, algo):
    w = W.make_workload(name, n_trials=1, **kw)
    P = O.Problem(w)
    plan = P.plan_greedy(SEED, 1, algo)
    S = gpu(w)
    for seed in (SEED, 4242):                       # own lengths, then mispredicted lengths
        assert S.samu_replay_plan(plan, seed) == P.replay(plan, seed)
    l_true = np.random.default_rng(5).integers(1, 600, w.n_req).astype(np.uint32)
    assert S.samu_replay_plan(plan, 0, known_l_out=l_true) == P.replay(plan, 0, known_l_out=l_true)


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_full_size_replay_and_ablation_bit_exact(name):
    # full BASELINE workloads: replay of the oracle's Max-heuristic plan against mispredicted and
    # known lengths, and the Min-heuristic plan without preemption on known lengths (§5.5)
    w = W.make_workload(name, n_trials=1)
    P = O.Problem(w)
    plan = P.plan_greedy(SEED, 1, "max")
    S = gpu(w)
    assert S.samu_replay_plan(plan, 4242) == P.replay(plan, 4242)
    l_true = np.random.default_rng(5).integers(1, 2000, w.n_req).astype(np.uint32)
    assert S.samu_replay_plan(plan, 0, known_l_out=l_true) == P.replay(plan, 0, known_l_out=l_true)
    po = P.plan_greedy(SEED, 1, "min", preemption=False, known_l_out=l_true)
    pg = S.samu_plan_greedy(SEED, 1, "min", preemption=False, known_l_out=l_true)
    pg.pop("n_sims")
    assert pg == po


def test_replay_hand_fixtures_bit_exact():
    from tests.test_oracle_pins import _hand_plan, _replay_fixture
    cases = [(_replay_fixture([2, 3, 4], 4, cap=8), [[(0, 1, 1), (1, 1, 1), (2, 1, 1)], [(1, 1, 1), (2, 2, 1)]],
              np.array([5, 5] + [1] * 7, np.uint32))]
    for n_gpus in (2, 3):
        cases.append((_replay_fixture([2, 4, 4], n_gpus), [[(0, 1, 1), (1, 1, 1)], [(2, 2, 1)], [(1, 1, 1)]], None))
    for w, stages, lt in cases:
        plan = _hand_plan(stages)
        assert gpu(w).samu_replay_plan(plan, SEED, known_l_out=lt) == O.Problem(w).replay(plan, SEED, known_l_out=lt)


# cost-model coefficient fit
def _close(g, o, rel=1e-9):
    return np.all(np.abs(g - o) <= rel * np.maximum(np.abs(o), 1e-300))


@pytest.mark.parametrize("trim", [0, 10, 50])
def test_fit_coeffs_parity_on_profiles(trim):
    w = W.make_workload("c5", n_prompts=10, n_docs=5, n_trials=1)
    S = gpu(w)
    for m in range(len(w.models)):
        pr = W.make_profile(w, m, n_per_bucket=300 + 37 * m)
        a, b, nu, fl = S.samu_fit_coeffs(pr["off"], pr["x"], pr["y"], trim)
        oa, ob, onu, ofl, rc = O.fit_coeffs(pr["off"], pr["x"], pr["y"], trim)
        assert rc == 0
        assert (nu == onu).all() and (fl == ofl).all()
        assert _close(a, oa) and _close(b, ob)


def test_fit_coeffs_edge_cases():
    from paper_2503_16893_b200 import SamuError
    S = gpu(W.make_workload("c1", n_trials=1))
    rng = np.random.default_rng(9)
    # ragged buckets incl. 2-sample, constant-y, negative slope, large bucket (several CTAs' work)
    sizes = [2, 3, 5, 1000, 70000, 1]
    xs = [rng.uniform(0, 10, n) for n in sizes[:-1]] + [np.array([1.0])]
    ys = [2 * xs[0] + 1, np.full(3, 4.0), 10 - xs[2], 1e-3 * xs[3] + 0.5 + rng.standard_normal(1000),
          3e-2 * xs[4] + rng.standard_normal(70000), np.array([1.0])]
    x, y = np.concatenate(xs[:-1]), np.concatenate(ys[:-1])
    off = np.r_[0, np.cumsum(sizes[:-1])]
    for trim in (0, 10, 300):
        g = S.samu_fit_coeffs(off, x, y, trim)
        o = O.fit_coeffs(off, x, y, trim)
        assert o[4] == 0
        assert (g[2] == o[2]).all() and (g[3] == o[3]).all() and _close(g[0], o[0]) and _close(g[1], o[1])
    # degenerate bucket -> error, same flags as the oracle
    off2 = np.r_[off, off[-1] + 1]
    x2, y2 = np.r_[x, 1.0], np.r_[y, 1.0]
    with pytest.raises(SamuError):
        S.samu_fit_coeffs(off2, x2, y2, 0)


# ------------------------------------------------------------------------------------------
# full size, bench launch configuration: sampled (candidate, trial) pairs vs the oracle
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("T", [1024, 128])
def test_full_size_c5_bench_config_sampled_parity(T):
    # T = 1024: the N = 1 bench step (FRESH then LEAN launch); T = 128: one rank's share at 8
    # GPUs, where the LEAN launch runs concurrently with the FRESH one on the auxiliary stream
    w = W.make_workload("c5", n_trials=T)          # 50,000 requests, 12 nodes
    S = gpu(w)
    ready = [v for v in range(w.n_nodes) if not np.any((w.pred[w.node == v] >= 0) &
                                                      (w.node[np.maximum(w.pred[w.node == v], 0)] != v))]
    cands = [(v, dp, tp) for v in ready for (dp, tp) in S.samu_enumerate_plans(v)]
    glo, gli = S.samu_sample_lengths(SEED, 0, w.n_trials)
    g = recs(S.samu_simulate_batch(cands, glo, gli))          # [165, T]
    P = O.Problem(w)
    rng = np.random.default_rng(2503)
    picks = [(cands.index(c), int(k)) for c, k in
             [(cands[0], 0), (cands[-1], T - 1)] + [(cands[int(i)], int(k)) for i, k in
                                                    zip(rng.integers(0, len(cands), 10), rng.integers(0, T, 10))]]
    # the longest replica-sims: the chain summariser with dp = 1
    summ = [i for i, c in enumerate(cands) if c[0] == 10 and c[1] == 1]
    picks += [(summ[0], 777 % T)]
    for ci, k in picks:
        lo, li = P.sample(SEED, k, 1)
        node, dp, tp = cands[ci]
        o = P.simulate(node, dp, tp, lo, li)[0]
        assert_rec_equal(g[ci][k:k + 1], o, f"cand {cands[ci]} trial {k}")


# ------------------------------------------------------------------------------------------
# edge cases
# ------------------------------------------------------------------------------------------
def test_edge_empty_batches_and_empty_node():
    w = F.multi([dict(l_in=[5, 6, 7], l_out=[3, 1, 2]), dict(l_in=[], l_out=[])], eng=F.engine(n_gpus=8))
    S = gpu(w)
    glo, gli = S.samu_sample_lengths(SEED, 0, 2)
    out = S.samu_simulate_batch([], glo, gli)
    assert out["recs"].numel() == 0
    g = recs(S.samu_simulate_batch([(1, 1, 1), (1, 8, 1)], glo, gli))
    assert np.all(g["t_end"] == 0.0) and np.all(g["flags"] == 1)      # a node with no work is done (c28)
    import torch
    z = torch.empty((0, w.n_req), dtype=torch.int16, device="cuda")
    assert recs(S.samu_simulate_batch([(0, 1, 1)], z, z))["t_end"].size == 0


def test_edge_more_replicas_than_requests_and_lin_equals_lmax():
    # dp = 8 over 5 requests leaves empty replicas (clock = load time); l_in = l_max gives l_out = 0,
    # which still runs one prefill (reading c3)
    load = F.zero_load()
    load[:, :] = 2.5
    w = F.tiny([64, 10, 64, 3, 60], [5, 4, 9, 1, 2], sp=F.spec(l_max=64), eng=F.engine(n_gpus=8), load=load)
    g = _sim_parity(w, [(0, 8, 1), (0, 5, 1), (0, 1, 1)], 1)
    assert np.all(g["t_end"] >= 2.5)


def test_edge_max_num_seqs_one_and_256():
    for ms in (1, 256):
        w = F.tiny(np.full(300, 9), np.arange(300) % 7 + 1, eng=F.engine(max_num_seqs=ms, min_batched_tokens=3000))
        _sim_parity(w, [(0, 1, 1)], 1)


def test_greedy_plan_bit_exact_mixed_c5_shape():
    # all three applications at once: ensembling + routing + chain summary (fused summariser +
    # evaluator co-scheduling), 12 nodes
    w = W.make_workload("c5", n_prompts=40, n_docs=30, n_trials=2)
    po = O.Problem(w).plan_greedy(SEED, 2)
    pg = gpu(w).samu_plan_greedy(SEED, 2)
    assert [s["entries"] for s in pg["stages"]] == [s["entries"] for s in po["stages"]]
    for sg, so in zip(pg["stages"], po["stages"]):
        assert sg["fstar"] == so["fstar"] and sg["mean_tE"] == so["mean_tE"] and sg["T_E"] == so["T_E"]
    assert pg["total"] == po["total"] and pg["n_cand_evals"] == po["n_cand_evals"]


@pytest.mark.parametrize("algo", ["greedy", "max", "min"])
@pytest.mark.parametrize("name,T", [("c2", 2), ("c3", 2), ("c4", 1), ("c5", 1)])
def test_full_size_plan_bit_exact(name, T, algo):
    # the full BASELINE workloads (C5 = the bench workload: 12 nodes, 50k requests, every K2 path
    # the planner takes: LEAN / FRESH / cut / general), few trials so the oracle finishes in
    # ~30 s: every stage, f*, mean end time, T_E and the planned total bit for bit
    w = W.make_workload(name, n_trials=T)
    po = O.Problem(w).plan_greedy(SEED, T, algo)
    pg = gpu(w).samu_plan_greedy(SEED, T, algo)
    pg.pop("n_sims")
    assert pg == po


# ------------------------------------------------------------------------------------------
# multi-rank trial sharding on one GPU: in-process rank group (same collectives as NCCL)
# ------------------------------------------------------------------------------------------
def _run_ranks(world, fn):
    import threading

    import torch
    from paper_2503_16893_b200 import LocalGroup, Samu
    grp = LocalGroup(world)
    outs, errs = [None] * world, []

    def work(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                S = Samu(0, rank=r, local_group=grp, stream=st)
                outs[r] = fn(S, r, st)
                st.synchronize()
                S.close()
        except Exception as e:   # pragma: no cover - reported below
            errs.append(e)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    assert not errs, errs
    return outs


@pytest.mark.parametrize("world", [2, 3])
def test_local_ranks_greedy_plan_identical(world):
    w = W.make_workload("c2", n_prompts=120, n_trials=5)
    ref = O.Problem(w).plan_greedy(SEED, 5)

    def fn(S, r, st):
        S.load_workload(w)
        return S.samu_plan_greedy(SEED, 5)

    for pg in _run_ranks(world, fn):
        assert [s["entries"] for s in pg["stages"]] == [s["entries"] for s in ref["stages"]]
        assert [s["mean_tE"] for s in pg["stages"]] == [s["mean_tE"] for s in ref["stages"]]
        assert [s["T_E"] for s in pg["stages"]] == [s["T_E"] for s in ref["stages"]]
        assert pg["total"] == ref["total"]


def test_local_ranks_greedy_fewer_trials_than_ranks():
    # T < world: one rank holds no trial (bench.py's planner warm-up uses min(world, T) trials)
    w = W.make_workload("c2", n_prompts=80, n_trials=2)
    ref = O.Problem(w).plan_greedy(SEED, 2)

    def fn(S, r, st):
        S.load_workload(w)
        return S.samu_plan_greedy(SEED, 2)

    for pg in _run_ranks(3, fn):
        assert [s["entries"] for s in pg["stages"]] == [s["entries"] for s in ref["stages"]]
        assert pg["total"] == ref["total"]


def test_local_ranks_replay_identical():
    w = W.make_workload("c5", n_prompts=40, n_docs=30, n_trials=1)
    P = O.Problem(w)
    plan = P.plan_greedy(SEED, 1, "greedy")
    ref = P.replay(plan, 4242)

    def fn(S, r, st):
        S.load_workload(w)
        return S.samu_replay_plan(plan, 4242)

    for rp in _run_ranks(2, fn):
        assert rp == ref


def test_local_ranks_sharded_summary_identical():
    w = W.make_workload("c3", n_prompts=600, n_trials=7)
    cands = [(0, 1, 1), (1, 2, 2), (3, 4, 1)]
    S1 = gpu(w)
    lo, li = S1.samu_sample_lengths(SEED, 0, 7)
    ref = S1.samu_simulate_batch(cands, lo, li, summary=True)["summary"]

    def fn(S, r, st):
        S.load_workload(w)
        base, rem = divmod(7, 2)
        cnt = base + (1 if r < rem else 0)
        tb = r * base + min(r, rem)
        l1, l2 = S.samu_sample_lengths(SEED, tb, cnt)
        return S.samu_simulate_batch(cands, l1, l2, summary=True)["summary"]

    for summ in _run_ranks(2, fn):
        assert summ == ref


# ------------------------------------------------------------------------------------------
# the NCCL code path on one GPU: a one-rank communicator (SAMU_FORCE_NCCL) routes records and
# node status through ncclAllGather / ncclAllReduce exactly as a multi-GPU run does
# ------------------------------------------------------------------------------------------
_NCCL_CHILD = r"""
import os, sys, json
sys.path.insert(0, os.environ["SAMU_ROOT"])
import numpy as np, torch
import samu_workloads as W
from paper_2503_16893_b200 import Samu
w = W.make_workload("c2", n_prompts=120, n_trials=3)
S = Samu(0); S.load_workload(w)
plan = S.samu_plan_greedy(16893, 3)
lo, li = S.samu_sample_lengths(16893, 0, 3)
out = S.samu_simulate_batch([(0, 1, 1), (2, 2, 2)], lo, li, summary=True)
print(json.dumps(dict(plan=[(s["entries"], s["fstar"], s["mean_tE"], s["T_E"]) for s in plan["stages"]],
                      total=plan["total"], summary=[float(x["mean_t"]) for x in out["summary"]])))
"""


def test_nccl_path_one_rank_matches_oracle():
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, SAMU_FORCE_NCCL="1", SAMU_ROOT=root)
    r = subprocess.run([sys.executable, "-c", _NCCL_CHILD], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    got = json.loads(r.stdout.strip().splitlines()[-1])
    w = W.make_workload("c2", n_prompts=120, n_trials=3)
    P = O.Problem(w)
    ref = P.plan_greedy(SEED, 3)
    assert got["total"] == ref["total"]
    assert [(tuple(map(tuple, e)), f, m, t) for e, f, m, t in got["plan"]] == \
        [(tuple(s["entries"]), s["fstar"], s["mean_tE"], s["T_E"]) for s in ref["stages"]]
    lo, li = P.sample(SEED, 0, 3)
    for (node, dp, tp), mean in zip([(0, 1, 1), (2, 2, 2)], got["summary"]):
        rec, _, _ = P.simulate(node, dp, tp, lo, li)
        s = 0.0
        for x in rec["t_end"]:
            s += float(x)
        assert mean == s / 3


# ------------------------------------------------------------------------------------------
# randomised sweeps (the long versions: scripts/fuzz_sweep.py 2000, scripts/plan_sweep.py 200)
# ------------------------------------------------------------------------------------------
def test_random_simulation_sweep():
    import scripts.fuzz_sweep as fs
    checked, bad = fs.sweep(120)
    assert checked > 500 and bad == 0


def test_random_planner_sweep():
    import scripts.plan_sweep as ps
    checked, bad = ps.sweep(24)
    assert checked > 150 and bad == 0
