"""More pins of the CPU oracle (round 2): carried-state reload / resume hand traces, the
thread-pool driver against the single-candidate one, FLOPs against a direct evaluation (AC1),
KV safety on fuzzed workloads with the per-iteration trace, the chatglm scaling
fixture (AC6), per-candidate summaries (reading c17) and a sanitizer build of the oracle.

P:<line> = PAPER.md, S:<line> = SPEC.md.  CPU only (-m "not gpu").
"""
import math
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
import samu_workloads as W
from tests import fixtures as F

SEED = W.SAMPLING_SEED
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ------------------------------------------------------------------------------------------
# Carried state: a request cut mid-decode, then reloaded under another plan (S:406,
# P:494-496 "the loading time ... should be added", reading c18) or resumed with the same plan
# ------------------------------------------------------------------------------------------
def _stage1(w, tau=5.5):
    """Stage 1 at plan (1, 1), cut at tau = 5.5 (10.5 with latency = B).  Hand trace (5 blocks, 2 slots, 1 s/iter):
    it0 prefill A, B (g = 1; F 5 -> 3); it1 decode l = 5 -> both need a block (F 1);
    it2-it4 decodes (g = 5); it5 decode l = 9 needs 2 blocks > F = 1 -> B (last admitted)
    preempted with g = 5 kept, freeing ceil(8/4) = 2 (F 3), A needs 1 (F 2), A -> g = 6;
    t = 6 >= 5.5 -> cut, overshoot 0.5 (latency = B: it0-it4 cost 2 s each, it5 1 s, so
    t = 11 >= 10.5, the same state).  C never left W (both slots busy)."""
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 1)
    assert lo[0].tolist() == [7, 8, 2] and li[0].tolist() == [4, 4, 4]
    st = P.fresh_state(1)
    r1, _, _ = P.simulate(0, 1, 1, lo, li, state=st, tau=np.array([tau]), commit=True)
    return P, lo, li, st, r1


def test_cut_mid_decode_state_hand_trace():
    P, lo, li, st, r1 = _stage1(F.reload_fixture())
    assert r1["iters"][0] == 6 and r1["t_end"][0] == 6.0 and r1["flags"][0] == 2
    assert r1["req_iters"][0] == 2 + 2 * 4 + 1
    s = st["st"][0]
    assert (s[0] >> 28, s[0] & 0x0FFFFFFF) == (O.ST_RUNNING, 0)        # A running, rank 0
    assert (s[1] >> 28, s[1] & 0x0FFFFFFF) == (O.ST_PREEMPTED, 0)      # B preempted, seq 0
    assert s[2] >> 28 == O.ST_FRESH                                    # C never started
    assert st["g"][0].tolist() == [6, 5, 0]
    assert st["over"][0, 0, 0] == 0.5


@pytest.mark.parametrize("kind,t_end", [("const", 14.0), ("B", 16.0)])
def test_reload_under_new_plan_hand_trace(kind, t_end):
    """Reload at plan (1, 2): clock starts at load(1, 2) = 10 s; every partially
    decoded request returns to the front of W, the running one first (admission order), then
    the preempted one, then the never-started head: W = [A (g 6, p 10), B (g 5, p 9), C (p 4)]
    and each re-prefills l_in + g.  10 blocks, budget 16:
      it0 prefill A alone (10 + 9 > 16): its 7th token, A finishes (F 10);
      it1 prefill B, C together (13 tokens, 4 blocks; F 6), g_B 6, g_C 1;
      it2 decode: C needs a block (l = 5), C finishes (F 7);  it3 decode -> B finishes.
    B before A would finish A at it1; recomputing l_in only, or resuming instead, changes the
    trace too (mutation-checked)."""
    P, lo, li, st, r1 = _stage1(F.reload_fixture(kind), 5.5 if kind == "const" else 10.5)
    assert st["g"][0].tolist() == [6, 5, 0] and st["over"][0, 0, 0] == 0.5 and r1["iters"][0] == 6
    r2, fi, ft = P.simulate(0, 1, 2, lo, li, state=st, commit=True, want_fin=True)
    assert r2["iters"][0] == 4 and r2["t_end"][0] == t_end and r2["flags"][0] == 1
    assert r2["req_iters"][0] == 6                         # A 1 + B 3 + C 2 tokens (recompute keeps g)
    assert fi[0].tolist() == [0, 3, 2]
    if kind == "const":
        assert ft[0].tolist() == [11.0, 14.0, 13.0]
    # FLOPs (L 1, c 10, h/tp 4): prefill A (B 1, s 10), prefill B, C (B 2, s 9),
    # decode (B 2, S 10 + 5), decode (B 1, S 11)
    fl = 10 * 1 * 10 + 2 * 1 * 4 * 10 * 10 + 10 * 2 * 9 + 2 * 2 * 4 * 9 * 9 + (10 * 2 + 2 * 4 * 15) + (10 * 1 + 2 * 4 * 11)
    assert O.rec_flops(r2)[0] == fl
    assert np.all(st["st"][0] >> 28 == O.ST_DONE)


def test_resume_same_plan_hand_trace():
    """Resume at (1, 1) (same plan in the previous stage, reading c18): no load, clock starts at
    the overshoot 0.5, A keeps its slot and 3 KV blocks (F 2), W = [B (g 5), C]:
      it0 decode A (B does not fit: 3 blocks > 2) -> A finishes (g 7), F 5;
      it1 prefill B (p 9) and C (p 4) together; it2 decode: C needs a block, finishes;
      it3 decode -> B finishes."""
    P, lo, li, st, _ = _stage1(F.reload_fixture())
    r2, fi, ft = P.simulate(0, 1, 1, lo, li, resume=1, state=st, commit=True, want_fin=True)
    assert r2["iters"][0] == 4 and r2["t_end"][0] == 4.5 and r2["req_iters"][0] == 1 + 2 + 2 + 1
    assert fi[0].tolist() == [0, 3, 2] and ft[0].tolist() == [1.5, 4.5, 3.5]


# ------------------------------------------------------------------------------------------
# The thread-pool driver (CPU baseline, --impl reference) against the single-candidate one
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("name,kw", [("c2", dict(n_prompts=150)), ("c3", dict(n_prompts=300)),
                                     ("c4", dict(n_docs=25))])
def test_simulate_many_equals_simulate(name, kw):
    w = W.make_workload(name, n_trials=3, **kw)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 3)
    has_input = [bool(np.any((w.pred[w.node == v] >= 0) & (w.node[np.maximum(w.pred[w.node == v], 0)] != v)))
                 for v in range(w.n_nodes)]
    cands = [(v, dp, tp) for v in range(w.n_nodes) if not has_input[v] for (dp, tp) in P.plans(int(w.node_model[v]))]
    many = P.simulate_many(cands, lo, li, 4)
    for i, (v, dp, tp) in enumerate(cands):
        one = P.simulate(v, dp, tp, lo, li)[0]
        assert np.array_equal(many[i], one), (v, dp, tp)


# ------------------------------------------------------------------------------------------
# AC1: FLOPs against a direct evaluation on 1000 random tuples
# ------------------------------------------------------------------------------------------
def test_flops_match_direct_evaluation_on_random_tuples():
    """Eq. prefill / decode evaluated directly, term by term over the batch's
    sequences with Python integers: a prefill processes B sequences padded to s, each layer
    costing c s (linear layers) + 2 (h/tp) s^2 (attention); a decode feeds one token per
    sequence, c + 2 (h/tp) l_r per layer."""
    rng = np.random.default_rng(641)
    for _ in range(1000):
        L = int(rng.integers(1, 129))
        h = int(rng.choice([8, 64, 4096, 5120, 8192]))
        tp = int(rng.choice([t for t in (1, 2, 4, 8) if h % t == 0]))
        c = int(rng.integers(1, 2 * 10 ** 9))
        B = int(rng.integers(1, 257))
        lens = rng.integers(1, 4097, B)
        s = int(lens.max())
        direct_p = L * sum(c * s + 2 * (h // tp) * s * s for _ in range(B))
        assert O.flops_prefill(L, c, h, tp, B, s) == direct_p
        direct_d = sum(sum(c + 2 * (h // tp) * int(l) for l in lens) for _ in range(L))
        assert O.flops_decode(L, c, h, tp, B, int(lens.sum())) == direct_d


# ------------------------------------------------------------------------------------------
# Per-iteration trace and KV safety on 10^3 fuzzed workloads
# ------------------------------------------------------------------------------------------
def _cdiv(a, b):
    return -(-a // b)


def _check_trace(P, w, lo, li, node, dp, tp):
    model = int(w.node_model[node])
    bs = w.engine["block_size"]
    blocks = P.plan_blocks(model, dp, tp)
    budget = max(w.models[model]["l_max"], w.engine["min_batched_tokens"])
    rec = P.simulate(node, dp, tp, lo[None, :], li[None, :])[0][0]
    iters = req_iters = 0
    flops = 0
    t_max = -math.inf
    for j in range(dp):
        desc, running = P.trace(node, dp, tp, lo, li, j)
        t = float(w.load[model][int(math.log2(tp)), dp - 1])
        for d, run in zip(desc, running):
            assert d["t_start"] == t                      # iterations back to back on one clock
            t = t + d["lat"]
            held = sum(_cdiv(int(li[r]) + g - 1, bs) for r, g in run)
            assert held == blocks - d["free_blocks"]      # block accounting (reading c5)
            assert held <= blocks                         # KV safety (block form)
            assert sum(int(li[r]) + g - 1 for r, g in run) <= blocks * bs   # token form
            assert len(run) <= w.engine["max_num_seqs"] and d["B"] <= w.engine["max_num_seqs"]
            assert all(1 <= g < max(int(lo[r]), 1) for r, g in run)   # unfinished, >= 1 token
            if d["kind"] == 0:
                assert d["S"] <= budget and d["n_preempted"] == 0      # token budget (c6)
            flops += int(d["flops"])
            req_iters += int(d["B"])
        iters += len(desc)
        t_max = max(t_max, t)
    assert iters == rec["iters"] and req_iters == rec["req_iters"]
    assert flops == O.rec_flops(rec[None])[0] and t_max == rec["t_end"]


def test_trace_reproduces_records_on_paper_workloads():
    for name, kw, cands in (("c2", dict(n_prompts=120), [(0, 1, 1), (5, 2, 4)]),
                            ("c4", dict(n_docs=20), [(0, 1, 1), (0, 3, 2)])):
        w = W.make_workload(name, n_trials=1, **kw)
        P = O.Problem(w)
        lo, li = P.sample(SEED, 0, 1)
        for v, dp, tp in cands:
            _check_trace(P, w, lo[0], li[0], v, dp, tp)


def test_kv_safety_fuzz():
    rng = np.random.default_rng(337)
    n_pre = 0
    for _ in range(1000):
        n = int(rng.integers(1, 25))
        bs = int(rng.choice([1, 2, 4, 7, 16]))
        l_max = int(rng.integers(8, 60))
        lin = rng.integers(1, l_max, n)
        lout = rng.integers(0, 40, n)
        kv = int(rng.integers(_cdiv(l_max, bs), 4 * _cdiv(l_max, bs) + 1)) * bs
        eng = F.engine(kv_cap=kv, min_batched_tokens=int(rng.integers(1, 3 * l_max)),
                       max_num_seqs=int(rng.integers(1, 9)), block_size=bs, n_gpus=2)
        w = F.tiny(lin, lout, sp=F.spec(l_max=l_max, tp_values=(1, 2)), eng=eng, cf="S")
        P = O.Problem(w)
        lo, li = P.sample(SEED, 0, 1)
        dp, tp = [(1, 1), (2, 1), (1, 2)][int(rng.integers(0, 3))]
        _check_trace(P, w, lo[0], li[0], 0, dp, tp)
        n_pre += int(sum(P.trace(0, dp, tp, lo[0], li[0], j)[0]["n_preempted"].sum() for j in range(dp)))
    assert n_pre > 100        # the fuzz exercises preemption


# ------------------------------------------------------------------------------------------
# AC6: chatglm scaling fixture
# ------------------------------------------------------------------------------------------
def test_chatglm_fixture_greedy_prefers_the_linear_model():
    w = F.chatglm_fixture()
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 1)
    assert P.simulate(0, 1, 1, lo, li)[0]["t_end"][0] == 48.0          # 1 GPU: 48 s
    assert P.simulate(0, 1, 8, lo, li)[0]["t_end"][0] == pytest.approx(32.0, rel=1e-12)   # 8 GPUs: 32 s
    assert P.simulate(1, 8, 1, lo, li)[0]["t_end"][0] == 6.0            # linear model: 48 s / 8
    plan = P.plan_greedy(SEED, 1)
    linear_done = False
    for s in plan["stages"]:
        g0 = sum(dp * tp for (v, dp, tp) in s["entries"] if v == 0)
        g1 = sum(dp * tp for (v, dp, tp) in s["entries"] if v == 1)
        if not linear_done:
            # while the linear model is ready, the per-GPU-gain rule (Alg. 1 line 19, max dT/dN)
            # gives it the GPUs: chatglm never gets 8, and gets fewer than the linear model
            assert g0 < 8 and g1 > g0
        linear_done = linear_done or s["fstar"] == 1
    assert plan["stages"][0]["entries"] == [(0, 1, 1), (1, 7, 1)]
    mx = P.plan_greedy(SEED, 1, "max")
    assert mx["stages"][0]["entries"] == [(0, 1, 8)]      # Max-heuristic: all GPUs to each LLM
    mn = P.plan_greedy(SEED, 1, "min")
    assert plan["total"] < mx["total"] and plan["total"] < mn["total"]


# ------------------------------------------------------------------------------------------
# Per-candidate summaries (north star; reading c17)
# ------------------------------------------------------------------------------------------
def test_summaries_match_definitions():
    w = W.make_workload("c2", n_prompts=80, n_trials=37)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 37)
    cands = [(0, 1, 1), (3, 2, 2), (5, 8, 1)]
    recs = P.simulate_many(cands, lo, li, 4)
    sm = O.summarise(recs)
    for i in range(len(cands)):
        t = recs[i]["t_end"]
        for p in (50, 90, 99):
            assert sm[i][f"p{p}_t"] == np.percentile(t, p, method="inverted_cdf")
        assert sm[i]["mean_t"] == pytest.approx(math.fsum(t) / 37, rel=1e-15)
        fl = sum(int(x) for x in O.rec_flops(recs[i]))
        assert fl < 2 ** 64 and sm[i]["mean_flops"] == float(fl) / 37
        assert sm[i]["mean_req_iters"] == float(int(recs[i]["req_iters"].sum())) / 37
    # degenerate cases: one trial (every percentile is the value), ties
    one = O.summarise(recs[:, :1])
    assert np.all(one["p50_t"] == recs[:, 0]["t_end"]) and np.all(one["p99_t"] == recs[:, 0]["t_end"])
    tie = recs[:1, :4].copy()
    tie["t_end"] = [2.0, 1.0, 2.0, 1.0]
    s4 = O.summarise(tie)[0]
    assert (s4["p50_t"], s4["p90_t"], s4["p99_t"], s4["mean_t"]) == (1.0, 2.0, 2.0, 1.5)


# ------------------------------------------------------------------------------------------
# The oracle under AddressSanitizer + UndefinedBehaviorSanitizer
# ------------------------------------------------------------------------------------------
_SAN_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
import oracle as O, samu_workloads as W
from tests import fixtures as F
for name, kw, T in (("c2", dict(n_prompts=60), 2), ("c4", dict(n_docs=12), 2), ("c3", dict(n_prompts=80), 1)):
    w = W.make_workload(name, n_trials=T, **kw)
    P = O.Problem(w)
    lo, li = P.sample(7, 0, T)
    for algo in ("greedy", "max", "min"):
        plan = P.plan_greedy(7, T, algo)
    P.plan_greedy(7, T, "greedy", preemption=False)
    P.replay(plan, 9)
    recs = P.simulate_many([(0, 1, 1), (0, 2, 2)], lo, li, 2)
    O.summarise(recs)
    P.trace(0, 2, 1, lo[0], li[0], 1)
P, lo, li, st, r1 = None, None, None, None, None
w = F.reload_fixture()
P = O.Problem(w)
lo, li = P.sample(7, 0, 1)
st = P.fresh_state(1)
P.simulate(0, 1, 1, lo, li, state=st, tau=np.array([5.5]), commit=True)
P.simulate(0, 1, 2, lo, li, state=st, commit=True, want_fin=True)
pr = W.make_profile(W.make_workload("c2", n_prompts=10), 0, n_per_bucket=30)
O.fit_coeffs(pr["off"], pr["x"], pr["y"], 10)
print("sanitized oracle ok")
"""


@pytest.mark.slow
def test_oracle_under_address_and_undefined_behaviour_sanitizers(tmp_path):
    so = tmp_path / "liboracle_san.so"
    subprocess.check_call(["g++", "-O1", "-g", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                           "-fsanitize=address,undefined", "-fno-sanitize-recover=all", "-fno-omit-frame-pointer",
                           "-o", str(so), os.path.join(ROOT, "oracle", "oracle.cpp")])
    asan = subprocess.check_output(["g++", "-print-file-name=libasan.so"], text=True).strip()
    ubsan = subprocess.check_output(["g++", "-print-file-name=libubsan.so"], text=True).strip()
    env = dict(os.environ, LD_PRELOAD=f"{asan}:{ubsan}", ASAN_OPTIONS="detect_leaks=0",
               UBSAN_OPTIONS="print_stacktrace=1:halt_on_error=1", SAMU_ORACLE_SO=str(so))
    r = subprocess.run([sys.executable, "-c", _SAN_SCRIPT, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "sanitized oracle ok" in r.stdout, r.stderr[-4000:]
