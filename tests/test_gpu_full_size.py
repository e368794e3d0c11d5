"""GPU parity, round 2: exhaustive full-size checks at the bench configuration, the carried-state
hand traces through the C ABI, summaries against the oracle's, and a cuRAND cross-check of K1.

P:<line> = PAPER.md, S:<line> = SPEC.md.  Every test needs a B200 (-m gpu).
"""
import ctypes
import os
import subprocess

import numpy as np
import pytest

import oracle as O
import samu_workloads as W
from tests import fixtures as F

pytestmark = pytest.mark.gpu
SEED = W.SAMPLING_SEED
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_THREADS = os.cpu_count() or 8


def gpu(w):
    from paper_2503_16893_b200 import Samu
    S = Samu(0)
    S.load_workload(w)
    return S


def u16(t):
    return t.cpu().numpy().view(np.uint16)


def recs(out):
    from paper_2503_16893_b200 import recs_to_numpy
    return recs_to_numpy(out["recs"])


def assert_rec_equal(g, o, ctx=""):
    for f in ("t_end", "flops_lo", "flops_hi", "req_iters", "iters", "flags"):
        bad = np.nonzero(np.ravel(g[f] != o[f]))[0]
        assert bad.size == 0, f"{ctx}: field {f} differs at {bad[:8]} of {np.size(g[f])}"


def ready_cands(S, w):
    ready = [v for v in range(w.n_nodes) if not np.any((w.pred[w.node == v] >= 0) &
                                                      (w.node[np.maximum(w.pred[w.node == v], 0)] != v))]
    return [(v, dp, tp) for v in ready for (dp, tp) in S.samu_enumerate_plans(v)]


# ------------------------------------------------------------------------------------------
# full size C5 (BASELINE configs[4], the bench workload): every sampled length, every record
# ------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c5_full():
    """Oracle side of the bench step, computed once: all 1024 x 50,000 sampled lengths and all
    165 x 1024 (candidate, trial) records of the first greedy inner step (~2 min of oracle time
    on the box's host cores)."""
    w = W.make_workload("c5")
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, w.n_trials)
    S = gpu(w)
    cands = ready_cands(S, w)
    orec = P.simulate_many(cands, lo, li, N_THREADS)
    return w, S, cands, lo, li, orec


def test_full_size_c5_all_sampled_lengths(c5_full):
    w, S, cands, lo, li, _ = c5_full
    glo, gli = S.samu_sample_lengths(SEED, 0, w.n_trials)
    assert np.array_equal(u16(glo), lo) and np.array_equal(u16(gli), li)     # 2 x 51.2M values


@pytest.mark.parametrize("T", [1024, 128])
def test_full_size_c5_every_record(c5_full, T):
    """T = 1024: the N = 1 bench step; T = 128: one rank's share at 8 GPUs (its LEAN launch
    runs concurrently with the FRESH one).  Every (candidate, trial) record, bit for bit."""
    w, S, cands, lo, li, orec = c5_full
    glo, gli = S.samu_sample_lengths(SEED, 0, T)
    g = recs(S.samu_simulate_batch(cands, glo, gli))
    assert g.shape == (len(cands), T)
    assert_rec_equal(g, orec[:, :T], f"C5 full size, T = {T}")


def test_full_size_c5_summaries(c5_full):
    w, S, cands, lo, li, orec = c5_full
    glo, gli = S.samu_sample_lengths(SEED, 0, w.n_trials)
    out = S.samu_simulate_batch(cands, glo, gli, summary=True)
    osum = O.summarise(orec)
    for f in ("mean_t", "p50_t", "p90_t", "p99_t", "mean_flops", "mean_req_iters"):
        assert np.array_equal(np.array([s[f] for s in out["summary"]]), osum[f]), f


@pytest.mark.parametrize("name,kw", [("c2", {}), ("c3", {}), ("c4", {})])
def test_full_size_c2_c4_every_record(name, kw):
    """BASELINE configs[1..3] at full size and 64 trials: every record of the first inner step."""
    w = W.make_workload(name, **kw)
    P = O.Problem(w)
    S = gpu(w)
    cands = ready_cands(S, w)
    lo, li = P.sample(SEED, 0, w.n_trials)
    glo, gli = S.samu_sample_lengths(SEED, 0, w.n_trials)
    assert np.array_equal(u16(glo), lo) and np.array_equal(u16(gli), li)
    g = recs(S.samu_simulate_batch(cands, glo, gli))
    assert_rec_equal(g, P.simulate_many(cands, lo, li, N_THREADS), name)


# ------------------------------------------------------------------------------------------
# carried state cut mid-decode, then reloaded / resumed (reading c18): hand traces
# ------------------------------------------------------------------------------------------
def _state_np(s):
    return dict(st=s["st"].cpu().numpy().view(np.uint32), g=s["g"].cpu().numpy().view(np.uint16),
                fin_t=s["fin_t"].cpu().numpy(), over=s["over"].cpu().numpy())


@pytest.mark.parametrize("kind,tau,reload_t", [("const", 5.5, 14.0), ("B", 10.5, 16.0)])
def test_reload_and_resume_hand_traces_on_gpu(kind, tau, reload_t):
    # the traces of tests/test_oracle_state_pins.py, through libsamu
    w = F.reload_fixture(kind)
    S = gpu(w)
    glo, gli = S.samu_sample_lengths(SEED, 0, 1)
    for resume in (0, 1):
        st = S.fresh_state(1)
        r1 = recs(S.samu_simulate_batch([(0, 1, 1, 0, -1, 1)], glo, gli, state=st, time_limit=np.array([[tau]])))
        assert r1["iters"][0, 0] == 6 and r1["flags"][0, 0] == 2
        s = _state_np(st)
        assert s["g"][0].tolist() == [6, 5, 0] and s["over"][0, 0, 0] == 0.5
        assert [x >> 28 for x in s["st"][0]] == [O.ST_RUNNING, O.ST_PREEMPTED, O.ST_FRESH]
        plan = (0, 1, 1, 1, -1, 1) if resume else (0, 1, 2, 0, -1, 1)
        out = S.samu_simulate_batch([plan], glo, gli, state=st, want_fin_iter=True)
        r2 = recs(out)
        fi = out["fin_iter"].cpu().numpy().view(np.uint32)[0, 0]
        if resume:
            if kind == "const":
                assert r2["t_end"][0, 0] == 4.5
            assert r2["iters"][0, 0] == 4 and fi.tolist() == [0, 3, 2]
        else:
            assert r2["t_end"][0, 0] == reload_t and r2["iters"][0, 0] == 4 and r2["req_iters"][0, 0] == 6
            assert fi.tolist() == [0, 3, 2]
        assert np.all(_state_np(st)["st"][0] >> 28 == O.ST_DONE)


# ------------------------------------------------------------------------------------------
# summaries: GPU K3 against the oracle's or_summarise on the same records
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("T", [1, 2, 37, 100, 1000])
def test_summaries_match_oracle(T):
    w = W.make_workload("c2", n_prompts=60, n_trials=T)
    S = gpu(w)
    glo, gli = S.samu_sample_lengths(SEED, 0, T)
    out = S.samu_simulate_batch([(0, 1, 1), (5, 2, 4), (3, 8, 1)], glo, gli, summary=True)
    osum = O.summarise(recs(out))
    for f in ("mean_t", "p50_t", "p90_t", "p99_t", "mean_flops", "mean_req_iters"):
        assert np.array_equal(np.array([s[f] for s in out["summary"]]), osum[f]), f


# ------------------------------------------------------------------------------------------
# K1 against cuRAND's Philox4x32-10 (NVIDIA's implementation of the same generator, reading c1)
# ------------------------------------------------------------------------------------------
@pytest.fixture(scope="module")
def curand_lib(tmp_path_factory):
    so = tmp_path_factory.mktemp("curand") / "libcurand_check.so"
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                           "-Xcompiler", "-fPIC", "-shared", "-o", str(so),
                           os.path.join(ROOT, "tests", "native", "curand_philox_check.cu")])
    return ctypes.CDLL(str(so))


@pytest.mark.parametrize("name,kw", [("c2", dict(n_prompts=500)), ("c5", {})])
def test_sampler_matches_curand_philox(curand_lib, name, kw):
    """u = word (r & 3) of Philox4x32-10(ctr = (r >> 2, trial, node, 0), key = (seed lo, hi)) from
    cuRAND, then X = the floor(u n / 2^32)-th element of the eCDF's sorted multiset and
    l_out = min(X, y, l_max - l_in) (reading c2), for every root request."""
    T = 3
    w = W.make_workload(name, n_trials=T, **kw)
    S = gpu(w)
    glo, gli = S.samu_sample_lengths(SEED, 0, T)
    lo_g, li_g = u16(glo), u16(gli)
    roots = np.nonzero(w.pred < 0)[0].astype(np.uint32)
    for k in range(T):
        ctr = np.zeros((roots.size, 4), np.uint32)
        ctr[:, 0] = roots >> 2
        ctr[:, 1] = k
        ctr[:, 2] = w.node[roots]
        words = np.zeros((roots.size, 4), np.uint32)
        rc = curand_lib.curand_philox_words(ctr.ctypes.data_as(ctypes.c_void_p), SEED & 0xFFFFFFFF, SEED >> 32,
                                            words.ctypes.data_as(ctypes.c_void_p), roots.size)
        assert rc == 0
        u = words[np.arange(roots.size), roots & 3].astype(np.uint64)
        for v in range(w.n_nodes):
            m = int(w.node_model[v])
            multiset = np.repeat(w.ecdf_values[m], np.diff(np.r_[0, w.ecdf_cum[m]]))
            n = multiset.size
            sel = w.node[roots] == v
            X = multiset[(u[sel] * np.uint64(n)) >> np.uint64(32)].astype(np.int64)
            r = roots[sel]
            l_max = w.models[m]["l_max"]
            expect = np.minimum(np.minimum(X, w.cap_y[r].astype(np.int64)), l_max - w.l_in_base[r].astype(np.int64))
            assert np.array_equal(lo_g[k, r].astype(np.int64), expect), (name, k, v)
            assert np.array_equal(li_g[k, r], w.l_in_base[r])


# ------------------------------------------------------------------------------------------
# schedule sharing across the tp variants of one (node, dp) (K2 modes 1 / 2, SimLaunch::grp)
# ------------------------------------------------------------------------------------------
@pytest.fixture
def env():
    old = dict(os.environ)
    yield os.environ
    os.environ.clear()
    os.environ.update(old)


@pytest.mark.parametrize("seed", range(8))
def test_schedule_sharing_matches_oracle_with_fallbacks(env, seed):
    """Random workloads whose KV budget binds for some tp variants and not others: the grouped
    launch (one schedule per (node, dp), per-lane clocks, fallback queue for out-of-sync
    members) must give every member's oracle record; so must the ungrouped launch."""
    rng = np.random.default_rng(900 + seed)
    chains = seed % 2 == 1
    l_in, l_out, pred, chain = [], [], [], []
    if chains:
        for c in range(int(rng.integers(10, 40))):
            for j in range(int(rng.integers(1, 5))):
                pred.append(-1 if j == 0 else len(l_in) - 1)
                chain.append(c)
                l_in.append(int(rng.integers(1, 60)))
                l_out.append(int(rng.integers(1, 90)))
    else:
        n = int(rng.integers(40, 300))
        l_in = rng.integers(1, 80, n).tolist()
        l_out = rng.integers(0, 120, n).tolist()
    eng = F.engine(kv_cap=int(rng.integers(16, 60)) * 16, min_batched_tokens=int(rng.integers(256, 600)),
                   max_num_seqs=int(rng.integers(4, 64)), block_size=16, n_gpus=8)
    cf = rng.uniform(1e-4, 1e-2, (W.N_TP_SLOTS, 3, 2, F.NB))
    cf[:, 0, 0, :] = 1e-12
    load = rng.uniform(0.0, 30.0, (W.N_TP_SLOTS, W.MAX_DP))
    T = 16
    w = F.tiny(np.array(l_in), np.array(l_out), sp=F.spec(l_max=256, tp_values=(1, 2, 4, 8), L=2, h=16, c=1000),
               eng=eng, cf=cf, load=load, pred=np.array(pred) if chains else None,
               chain=np.array(chain) if chains else None, n_trials=T)
    P = O.Problem(w)
    cands = [(0, dp, tp) for (dp, tp) in P.plans(0)]
    lo, li = P.sample(SEED, 0, T)
    orec = P.simulate_many(cands, lo, li, N_THREADS)
    S = gpu(w)
    glo, gli = S.samu_sample_lengths(SEED, 0, T)
    env["SAMU_K2_MODES"] = "always"
    s0 = S.samu_share_stats()
    g = recs(S.samu_simulate_batch(cands, glo, gli))
    s1 = S.samu_share_stats()
    assert_rec_equal(g, orec, "grouped")
    assert s1["member_items"] - s0["member_items"] > 0
    env["SAMU_K2_GROUP"] = "never"
    assert_rec_equal(recs(S.samu_simulate_batch(cands, glo, gli)), orec, "ungrouped")
    assert S.samu_share_stats() == s1


def test_schedule_sharing_fallbacks_happen_and_are_exact(env):
    # C2-shaped ensembling with the 13B / 70B models' small tp = 1 KV budgets: those members fall
    # out of sync in (nearly) every item, the others never
    w = W.make_workload("c2", n_prompts=1000, n_trials=8)
    P = O.Problem(w)
    S = gpu(w)
    cands = ready_cands(S, w)
    lo, li = P.sample(SEED, 0, 8)
    glo, gli = S.samu_sample_lengths(SEED, 0, 8)
    env["SAMU_K2_MODES"] = "always"
    s0 = S.samu_share_stats()
    g = recs(S.samu_simulate_batch(cands, glo, gli))
    s1 = S.samu_share_stats()
    assert_rec_equal(g, P.simulate_many(cands, lo, li, N_THREADS), "c2 grouped")
    fb = s1["fallbacks"] - s0["fallbacks"]
    assert 0 < fb < s1["member_items"] - s0["member_items"]
    # the next batch schedules the members that fell out of sync on their own (hint): far fewer
    # fallbacks, the same records
    g2 = recs(S.samu_simulate_batch(cands, glo, gli))
    s2 = S.samu_share_stats()
    assert_rec_equal(g2, g, "c2 grouped with hints")
    assert s2["fallbacks"] - s1["fallbacks"] < fb / 4
    assert s2["member_items"] - s1["member_items"] < s1["member_items"] - s0["member_items"]


@pytest.mark.parametrize("T,force", [(9000, False), (37, True), (1000, True), (1, True)])
def test_summaries_any_trial_count(env, T, force):
    # more than 8192 trials take the radix-select summary kernel (forced here for small T too):
    # still the oracle's nearest-rank percentiles and sequential mean, bit for bit
    if force:
        env["SAMU_SUMMARY_SELECT"] = "1"
    w = W.make_workload("c2", n_prompts=12, n_trials=T)
    S = gpu(w)
    glo, gli = S.samu_sample_lengths(SEED, 0, T)
    out = S.samu_simulate_batch([(0, 1, 1), (4, 2, 2)], glo, gli, summary=True)
    osum = O.summarise(recs(out))
    for f in ("mean_t", "p50_t", "p90_t", "p99_t", "mean_flops", "mean_req_iters"):
        assert np.array_equal(np.array([s[f] for s in out["summary"]]), osum[f]), f


# ------------------------------------------------------------------------------------------
# multi-rank sharding of the (candidate, trial) product on one GPU (in-process rank group, the
# same collectives as NCCL): world = Wt trial blocks x Wc candidate classes
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


@pytest.mark.parametrize("name,kw,T,classes", [
    ("c2", dict(n_prompts=150), 64, 8),     # 64 trials, candidates split 8 ways (1 trial block)
    ("c3", dict(n_prompts=500), 64, 4),     # 2 trial blocks x 4 candidate classes
    ("c4", dict(n_docs=40), 64, 2),         # 4 x 2, with summariser -> evaluator dependencies
    ("c4", dict(n_docs=40), 64, 8),
    ("c1", {}, 1, 0),                       # C1: one trial, 8 ranks -> 8 candidate classes (automatic)
    ("c5", dict(n_prompts=40, n_docs=30), 3, 0),   # 3 trials, 8 ranks -> 2 trial blocks x 4 classes
])
def test_local_8_ranks_candidate_sharding_plan_identical(env, name, kw, T, classes):
    if classes:
        env["SAMU_SHARD_CLASSES"] = str(classes)
    w = W.make_workload(name, n_trials=T, **kw)
    ref = O.Problem(w).plan_greedy(SEED, T)

    def fn(S, r, st):
        S.load_workload(w)
        return S.samu_plan_greedy(SEED, T)

    for pg in _run_ranks(8, fn):
        pg.pop("n_sims")
        assert pg == ref


def test_local_8_ranks_replay_one_trial(env):
    w = W.make_workload("c5", n_prompts=40, n_docs=30, n_trials=1)
    P = O.Problem(w)
    plan = P.plan_greedy(SEED, 1, "greedy")
    ref = P.replay(plan, 4242)

    def fn(S, r, st):
        S.load_workload(w)
        return S.samu_replay_plan(plan, 4242)

    for rp in _run_ranks(8, fn):
        assert rp == ref


# ------------------------------------------------------------------------------------------
# samu_sample_requests: a model's request set with its own stream (the §8(b) call shape)
# ------------------------------------------------------------------------------------------
def test_sample_requests_equals_app_sampler_per_node():
    """Each node's requests sampled as a standalone set (stream = node id, index_base = the
    node's first index), on a context with models and eCDFs but no application, equal the app
    sampler's lengths for that node (and the oracle's), chains included."""
    from paper_2503_16893_b200 import Samu
    w = W.make_workload("c5", n_prompts=600, n_docs=120, n_trials=5)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 2, 5)
    S = Samu(0)
    for m, spec in enumerate(w.models):
        S.samu_model_register(m, spec, w.coeff_B, w.coeff[m], w.load[m])
        S.samu_ecdf_load(m, w.ecdf_values[m], w.ecdf_cum[m])
    checked = 0
    for v in range(w.n_nodes):
        a, b = w.node_range(v)
        pred = w.pred[a:b].astype(np.int64)
        if np.any((pred >= 0) & (pred < a)):
            continue   # cross-node predecessors are not part of a one-model set
        rel = np.where(pred >= 0, pred - a, -1)
        glo, gli = S.samu_sample_requests(int(w.node_model[v]), v, w.l_in_base[a:b], w.cap_y[a:b], rel, a, SEED, 2, 5)
        assert np.array_equal(u16(glo), lo[:, a:b]) and np.array_equal(u16(gli), li[:, a:b]), v
        checked += 1
    assert checked == w.n_nodes - 1


def test_sample_requests_rejects_bad_sets():
    from paper_2503_16893_b200 import Samu, SamuError
    w = W.make_workload("c1")
    S = Samu(0)
    S.samu_model_register(0, w.models[0], w.coeff_B, w.coeff[0], w.load[0])
    with pytest.raises(SamuError):   # no eCDF yet
        S.samu_sample_requests(0, 0, [5], [10], [-1], 0, SEED, 0, 1)
    S.samu_ecdf_load(0, w.ecdf_values[0], w.ecdf_cum[0])
    with pytest.raises(SamuError):   # pred must be earlier
        S.samu_sample_requests(0, 0, [5, 6], [10, 10], [1, -1], 0, SEED, 0, 1)
    with pytest.raises(SamuError):   # two successors
        S.samu_sample_requests(0, 0, [5, 6, 7], [10, 10, 10], [-1, 0, 0], 0, SEED, 0, 1)
    with pytest.raises(SamuError):   # l_in above l_max
        S.samu_sample_requests(0, 0, [w.models[0]["l_max"] + 1], [10], [-1], 0, SEED, 0, 1)


# ------------------------------------------------------------------------------------------
# a rank-local failure inside a collective call fails every rank (no rank left waiting)
# ------------------------------------------------------------------------------------------
_AGREE_CHILD = r"""
import os, sys, threading
sys.path.insert(0, os.environ["SAMU_ROOT"])
import torch
import samu_workloads as W
from paper_2503_16893_b200 import LocalGroup, Samu, SamuError
w = W.make_workload("c2", n_prompts=40, n_trials=8)
grp = LocalGroup(3)
res = [None] * 3
def work(r):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        S = Samu(0, rank=r, local_group=grp, stream=st)
        S.load_workload(w)
        cnt = [2, 3, 3][r]            # 8 trials in all, but not the contiguous split 3 / 3 / 2
        lo, li = S.samu_sample_lengths(16893, 0, cnt)
        try:
            S.samu_simulate_batch([(0, 1, 1)], lo, li, summary=True)
            res[r] = "ok"
        except SamuError as e:
            res[r] = "err:" + str(e)[:80]
        st.synchronize()
th = [threading.Thread(target=work, args=(r,)) for r in range(3)]
[t.start() for t in th]
[t.join() for t in th]
print(res)
"""


def test_rank_local_failure_fails_all_ranks():
    import subprocess
    import sys
    env = dict(os.environ, SAMU_ROOT=ROOT)
    r = subprocess.run([sys.executable, "-c", _AGREE_CHILD], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    out = r.stdout.strip().splitlines()[-1]
    assert out.count("err:") == 3, out          # ranks 0 and 2 fail the split check, rank 1 is told
    assert "another rank failed" in out
