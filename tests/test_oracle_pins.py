"""Pins of the CPU oracle against what the paper and mathematics fix (not against itself).

Each test names the passage (P:<line> = PAPER.md, S:<line> = SPEC.md) or the closed form it
checks.  Runs on CPU (-m "not gpu").
"""
import math

import numpy as np
import pytest

import oracle as O
import samu_workloads as W
from tests import fixtures as F

SEED = W.SAMPLING_SEED


# ------------------------------------------------------------------------------------------
# Philox4x32-10: Random123 known-answer vectors (tests/golden/philox_kat.txt)
# ------------------------------------------------------------------------------------------
def _golden_philox():
    rows = []
    import os
    path = os.path.join(os.path.dirname(__file__), "golden", "philox_kat.txt")
    for line in open(path):
        line = line.split("#")[0].strip()
        if not line:
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,expect", _golden_philox())
def test_philox_known_answers(ctr, key, expect):
    assert O.philox4x32_10(ctr, key) == expect


# ------------------------------------------------------------------------------------------
# eCDF inverse (reading c2)
# ------------------------------------------------------------------------------------------
def _one_model_problem(values, cum, l_max=4096):
    w = F.tiny([1], [1], sp=F.spec(l_max=l_max))
    w.ecdf_values[0] = np.asarray(values, np.uint32)
    w.ecdf_cum[0] = np.asarray(cum, np.uint32)
    return O.Problem(w)


def test_ecdf_spec_example_5_3_5():
    # trace [5,3,5] -> sorted [3,5,5]; eCDF(4) = 1/3, eCDF(5) = 1
    P = _one_model_problem([3, 5], [1, 3])
    # u/2^32 in [0, 1/3) -> 3 ; [1/3, 1) -> 5
    assert P.ecdf_inverse(0, 0) == 3
    assert P.ecdf_inverse(0, (1 << 32) // 3) == 3          # floor(u*3/2^32) = 0
    assert P.ecdf_inverse(0, (1 << 32) // 3 + 1) == 5
    assert P.ecdf_inverse(0, 0xFFFFFFFF) == 5


def test_ecdf_point_mass():
    P = _one_model_problem([100], [10000])
    for u in [0, 1, 12345, 2 ** 31, 2 ** 32 - 1]:
        assert P.ecdf_inverse(0, u) == 100


def test_ecdf_inverse_matches_numpy_inverted_cdf():
    # numpy's inverted_cdf percentile = smallest x with eCDF(x) >= q; at q = (t+1)/n it is the
    # t-th order statistic, which is what floor(u n / 2^32) = t must select.
    rng = np.random.default_rng(1)
    v, c = W.make_ecdf(rng, 200.0, 0.8, K=50, n=400)
    P = _one_model_problem(v, c)
    data = np.repeat(v, np.diff(np.concatenate([[0], c])))
    n = len(data)
    for t in range(n):
        u = -(-(t << 32) // n)      # smallest u with floor(u n / 2^32) = t
        q = np.percentile(data, 100.0 * (t + 0.5) / n, method="inverted_cdf")
        assert P.ecdf_inverse(0, u) == q
        u_hi = (((t + 1) << 32) - 1) // n   # largest u with floor = t
        assert P.ecdf_inverse(0, u_hi) == q


def test_ecdf_quantile_grid_reproduces_quantiles():
    # north star: "Sampled lengths must reproduce the ECDF's quantiles": u_j at the midpoint of
    # the j-th of M equal-probability cells returns the ECDF's (j+1/2)/M quantile.
    v, c = W.make_ecdf(np.random.default_rng(7), 250.0, 0.9)
    P = _one_model_problem(v, c)
    n = int(c[-1])
    M = 1000
    for j in range(M):
        # u/2^32 = the smallest 32-bit fraction >= q = (2j+1)/(2M) (exact integers)
        u = -(-((2 * j + 1) << 32) // (2 * M))
        # the ECDF's q-quantile: the first knot whose cumulative count exceeds q*n
        k = int(np.searchsorted(c, ((2 * j + 1) * n) // (2 * M), side="right"))
        assert P.ecdf_inverse(0, u) == v[k]


# ------------------------------------------------------------------------------------------
# Sampler
# ------------------------------------------------------------------------------------------
def test_sampler_spec_edge_cases():
    sp = F.spec(l_max=2048)
    # S:202 point mass 100, l_in 50, l_max 2048, no cap -> 100
    w = F.tiny([50, 2048, 30], [60000, 60000, 256], sp=sp)
    w.ecdf_values[0] = np.array([100], np.uint32)
    w.ecdf_cum[0] = np.array([10000], np.uint32)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 1)
    assert lo[0, 0] == 100
    assert lo[0, 1] == 0          # l_in = l_max -> 0 regardless of X
    # point mass 490 with cap 256 -> 256
    w.ecdf_values[0] = np.array([490], np.uint32)
    lo, _ = O.Problem(w).sample(SEED, 0, 1)
    assert lo[0, 2] == 256


def test_sampler_rejects_lin_above_lmax():
    w = F.tiny([5000], [10], sp=F.spec(l_max=4096))
    with pytest.raises(O.OracleError):
        O.Problem(w)


def test_sampler_determinism_and_trial_slicing():
    # identical (seed, request, trial) -> identical sample regardless of order/parallelism
    w = W.make_workload("c3", n_prompts=500, n_trials=6)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 6)
    lo2, li2 = P.sample(SEED, 3, 2)
    assert np.array_equal(lo[3:5], lo2) and np.array_equal(li[3:5], li2)
    lo3, _ = P.sample(SEED + 1, 0, 6)
    assert not np.array_equal(lo, lo3)


def test_sampler_ks_and_cap_dominance():
    # S:207 KS <= 0.01 at 1e5 uncapped samples; S:208 cap dominance
    rng = np.random.default_rng(3)
    v, c = W.make_ecdf(rng, 220.0, 0.8)
    n_req = 100000
    w = F.tiny(np.full(n_req, 10), np.full(n_req, 60000), sp=F.spec(l_max=65535))
    w.ecdf_values[0], w.ecdf_cum[0] = v, c
    P = O.Problem(w)
    lo, _ = P.sample(SEED, 0, 1)
    x = np.sort(lo[0].astype(np.int64))
    F_emp = np.searchsorted(x, v, side="right") / len(x)
    F_true = c / c[-1]
    assert np.max(np.abs(F_emp - F_true)) <= 0.01
    caps = rng.integers(1, 600, n_req)
    lins = rng.integers(1, 4000, n_req)
    w2 = F.tiny(lins, caps, sp=F.spec(l_max=4096))
    w2.ecdf_values[0], w2.ecdf_cum[0] = v, c
    lo2, li2 = O.Problem(w2).sample(SEED, 0, 1)
    assert np.all(lo2[0] <= np.minimum(caps, 4096 - lins))
    assert np.array_equal(li2[0], lins)


def test_chain_input_arithmetic():
    # chunk 2048 + previous summary 300 + overhead 50 -> next input 2398;
    # S:273 / P:380: only the final summary feeds the evaluator.
    ws = F.multi([
        dict(l_in=[2048 + 50, 2048 + 50, 1000 + 50], l_out=[900, 900, 900], pred=[-1, 0, 1], chain=[0, 0, 0],
             ecdf=(np.array([300]), np.array([1]))),
        dict(l_in=[300, 300], l_out=[512, 512], pred=[2, 2], ecdf=(np.array([40]), np.array([1]))),
    ])
    lo, li = O.Problem(ws).sample(SEED, 0, 1)
    assert li[0, 0] == 2098 and lo[0, 0] == 300
    assert li[0, 1] == 2398
    assert li[0, 2] == 1050 + 300
    assert li[0, 3] == 600 and li[0, 4] == 600 and lo[0, 3] == 40


# ------------------------------------------------------------------------------------------
# FLOPs (Eq. prefill, Eq. decode)
# ------------------------------------------------------------------------------------------
def test_flops_spec_examples():
    assert O.flops_prefill(2, 10, 8, 2, 3, 4) == 1008
    assert O.flops_prefill(2, 10, 8, 2, 0, 4) == 0
    assert O.flops_prefill(1, 0, 1, 1, 1, 2) == 8                # S:111 tp=1
    assert O.flops_prefill(1, 0, 2, 2, 1, 2) == 8 and O.flops_prefill(1, 0, 2, 1, 1, 2) == 16
    assert O.flops_decode(2, 10, 8, 2, 3, 12) == 252
    assert O.flops_decode(2, 10, 8, 2, 0, 0) == 0
    assert O.flops_decode(1, 0, 8, 1, 1, 24) == 2 * O.flops_decode(1, 0, 8, 1, 1, 12)


def test_flops_tp_halves_only_attention_term():
    L, c, h, B, s = 40, 317194240, 5120, 7, 333
    lin = L * c * B * s
    assert O.flops_prefill(L, c, h, 1, B, s) - lin == 2 * (O.flops_prefill(L, c, h, 2, B, s) - lin)


# ------------------------------------------------------------------------------------------
# Per-iteration latency and B interpolation (reading c11)
# ------------------------------------------------------------------------------------------
def test_iter_latency_spec_examples():
    assert O.iter_latency([0, 0, 0], [1e-3] * 3, 1008, 12, 12) == pytest.approx(3e-3, rel=1e-15)
    assert O.iter_latency([1e-12, 0, 0], [0, 0, 0], 1008, 5, 5) == pytest.approx(1.008e-9, rel=1e-15)


def test_iter_latency_monotone():
    rng = np.random.default_rng(5)
    for _ in range(200):
        a = rng.uniform(0, 1e-9, 3)
        b = rng.uniform(0, 1e-3, 3)
        x = rng.integers(0, 10 ** 12, 3)
        base = O.iter_latency(a, b, *x)
        for i in range(3):
            y = x.copy()
            y[i] += int(rng.integers(1, 10 ** 9))
            assert O.iter_latency(a, b, *y) >= base


def test_dense_coeff_interpolation():
    cf = np.zeros((W.N_TP_SLOTS, 3, 2, F.NB))
    rng = np.random.default_rng(2)
    cf[0] = rng.uniform(1e-6, 1e-3, (3, 2, F.NB))
    w = F.tiny([1], [1], cf=cf)
    a, b = O.Problem(w).dense_coeff(0, 1)
    Bk = [1, 2, 4, 8, 16, 32, 64, 128, 256]
    for k, B in enumerate(Bk):
        assert np.all(a[:, B - 1] == cf[0, :, 0, k]) and np.all(b[:, B - 1] == cf[0, :, 1, k])
    # B exactly between two buckets -> mean of the two bucket evaluations
    for k in range(2, F.NB - 1):
        mid = (Bk[k] + Bk[k + 1]) // 2
        x = 12345.0
        lat_mid = a[:, mid - 1] * x + b[:, mid - 1]
        lat_lo = cf[0, :, 0, k] * x + cf[0, :, 1, k]
        lat_hi = cf[0, :, 0, k + 1] * x + cf[0, :, 1, k + 1]
        assert np.allclose(lat_mid, 0.5 * (lat_lo + lat_hi), rtol=1e-14, atol=0)


# ------------------------------------------------------------------------------------------
# Plan validity and enumeration
# ------------------------------------------------------------------------------------------
def test_plan_validity_spec_examples():
    eng = F.engine(n_gpus=8, mem=80 * 10 ** 9, kv_cap=80 * 10 ** 9)
    # weights alone exceed one GPU -> (1,1) invalid; S:49 tp=2 fits
    sp = F.spec(weight_bytes=2 * 80 * 10 ** 9 * 9 // 10 + 10, tp_values=(1, 2, 4), h=8, l_max=4096)
    P = O.Problem(F.tiny([10], [10], sp=sp, eng=eng))
    assert P.plan_blocks(0, 1, 1) < 0
    assert P.plan_blocks(0, 1, 4) > 0
    # 13B-class (26 GB) on 80 GB GPUs, dp=9 with N=8 -> invalid
    sp13 = W.arch_spec("llama13b")
    P13 = O.Problem(F.tiny([10], [10], sp=sp13, eng=eng))
    assert P13.plan_blocks(0, 8, 1) > 0 and P13.plan_blocks(0, 9, 1) < 0
    # tiny model, N=2, tp in {1,2} -> [(1,1),(2,1),(1,2)]
    Pt = O.Problem(F.tiny([10], [10], sp=F.spec(tp_values=(1, 2)), eng=F.engine(n_gpus=2)))
    assert Pt.plans(0) == [(1, 1), (2, 1), (1, 2)]


def test_plan_needs_one_full_sequence_of_kv():
    # valid iff memory holds the weights and at least one sequence's KV cache
    eng = F.engine(kv_cap=4096 * 16 - 1)     # bytes; kv_bytes_per_token = 16 => < l_max tokens
    sp = F.spec(kv_bytes_per_token=16, l_max=4096)
    assert O.Problem(F.tiny([1], [1], sp=sp, eng=eng)).plan_blocks(0, 1, 1) < 0
    eng = F.engine(kv_cap=4096 * 16)
    assert O.Problem(F.tiny([1], [1], sp=sp, eng=eng)).plan_blocks(0, 1, 1) == 256


# ------------------------------------------------------------------------------------------
# Simulator closed forms and hand traces
# ------------------------------------------------------------------------------------------
def _sim(w, node=0, dp=1, tp=1, **kw):
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, w.n_trials)
    rec, fi, ft = P.simulate(node, dp, tp, lo, li, want_fin=True, **kw)
    return P, lo, li, rec, fi, ft


def test_hand_trace_spec_321():
    # 2 requests (out 2 and 1), max_num_seqs=2, ample KV, 1 s per iteration:
    # prefill at t=0 (both get token 1, B finishes), one decode (A finishes) -> total 2 s
    _, lo, li, rec, fi, ft = _sim(F.tiny([10, 10], [2, 1], eng=F.engine(max_num_seqs=2)))
    assert rec["t_end"][0] == 2.0 and rec["iters"][0] == 2
    assert fi[0].tolist() == [1, 0] and ft[0].tolist() == [2.0, 1.0]


def test_zero_requests_model_is_done():
    w = F.multi([dict(l_in=[5], l_out=[3]), dict(l_in=[5], l_out=[3])])
    # an (empty) replica runs no iteration; "0 requests -> total 0" is the done-model rule
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 1)
    st = P.fresh_state(1)
    st["st"][0, :] = O.ST_DONE << 28
    rec, _, _ = P.simulate(0, 1, 1, lo, li, state=st)
    assert rec["t_end"][0] == 0.0 and rec["iters"][0] == 0 and rec["flags"][0] & 1


@pytest.mark.parametrize("L_out", [1, 2, 7, 64])
def test_uniform_lengths_take_exactly_L_iterations(L_out):
    # north star: unlimited KV and all lengths equal to L -> exactly L iterations
    # (reading c4: 1 prefill that emits token 1, then L-1 decodes)
    n = 50
    _, lo, li, rec, fi, _ = _sim(F.tiny(np.full(n, 20), np.full(n, L_out)))
    assert rec["iters"][0] == L_out
    assert np.all(fi[0] == L_out - 1)
    assert rec["req_iters"][0] == n * L_out


def test_closed_form_unlimited_resources():
    # (ii): iterations = max l_out; r finishes at l_out - 1; decode j has B_j = #{l_out > j},
    # S_j = sum_{l_out > j} (l_in + j); FLOPs and latency summed independently (math.fsum).
    rng = np.random.default_rng(11)
    n = 40
    lin = rng.integers(1, 60, n)
    lout = rng.integers(1, 90, n)
    sp = F.spec(L=3, h=16, c=1000, tp_values=(1, 2))
    cf = np.zeros((W.N_TP_SLOTS, 3, 2, F.NB))
    cf[:, 0, 0, :] = 1e-9
    cf[:, 0, 1, :] = 1e-3
    cf[:, 1, 0, :] = 2e-7
    cf[:, 1, 1, :] = 3e-4
    cf[:, 2, 0, :] = 5e-8
    cf[:, 2, 1, :] = 7e-5
    w = F.tiny(lin, lout, sp=sp, cf=cf, eng=F.engine(min_batched_tokens=100000, n_gpus=2))
    P, lo, li, rec, fi, _ = _sim(w, tp=2)
    assert rec["iters"][0] == lout.max()
    assert np.array_equal(fi[0], lout - 1)
    # closed-form FLOPs (prefill of everything, then decodes)
    L, c, h, tp = 3, 1000, 16, 2
    s = lin.max()
    flops = L * (c * n * s + 2 * n * (h // tp) * s * s)
    lats = []
    a = cf[1]
    lats.append(a[0, 0, 7] * flops + a[0, 1, 7] + a[1, 0, 7] * (n * s) + a[1, 1, 7] + a[2, 0, 7] * lin.sum() + a[2, 1, 7])
    for j in range(1, lout.max()):
        alive = lout > j
        B = int(alive.sum())
        S = int((lin[alive] + j).sum())
        sm = int((lin[alive] + j).max())
        f = L * (c * B + 2 * (h // tp) * S)
        flops += f
        lats.append(a[0, 0, 0] * f + a[0, 1, 0] + a[1, 0, 0] * (B * sm) + a[1, 1, 0] + a[2, 0, 0] * S + a[2, 1, 0])
    assert O.rec_flops(rec)[0] == flops
    assert rec["t_end"][0] == pytest.approx(math.fsum(lats), rel=1e-12)
    assert rec["req_iters"][0] == lout.sum()


def test_fcfs_single_slot_finish_order():
    # S:335 (iii): max_num_seqs = 1 -> sum(l_out) iterations, finish order = index order
    rng = np.random.default_rng(4)
    lout = rng.integers(1, 30, 25)
    _, _, _, rec, fi, _ = _sim(F.tiny(np.full(25, 7), lout, eng=F.engine(max_num_seqs=1)))
    assert rec["iters"][0] == lout.sum()
    assert np.array_equal(fi[0], np.cumsum(lout) - 1)


def _preempt_workload(cf):
    # KV: 4 blocks of 16 tokens (kv_cap 64 B at 1 B/token), l_max 64 (exactly one sequence)
    return F.tiny([16, 16], [40, 40], sp=F.spec(l_max=64), cf=cf,
                  eng=F.engine(kv_cap=64, min_batched_tokens=64))


def test_hand_trace_preemption():
    # AC4 hand trace, §3 of DESIGN.md: prefill(A,B) -> 16 decodes with B=2 -> at l=33
    # both need a 5th/6th block, B (last admitted) is preempted -> A alone to g=40 at
    # iteration 39 -> B re-prefills 33 tokens (recompute) -> B alone, finishes at iteration 62.
    _, _, _, rec, fi, _ = _sim(_preempt_workload("const"))
    assert rec["iters"][0] == 63 and rec["t_end"][0] == 63.0
    assert fi[0].tolist() == [39, 62]
    _, _, _, recB, _, _ = _sim(_preempt_workload("B"))
    assert recB["t_end"][0] == 80.0 and recB["req_iters"][0] == 80     # sum of B
    _, _, _, recS, _, _ = _sim(_preempt_workload("S"))
    assert recS["t_end"][0] == 32 + 784 + 1012 + 33 + 979                # sum of S (hand-computed)


def test_hand_trace_token_budget_and_slots():
    # 6 requests l_in 30, budget 64 tokens -> prefills admit 2 at a time (strict FCFS)
    w = F.tiny([30] * 6, [3] * 6, sp=F.spec(l_max=64), eng=F.engine(min_batched_tokens=64, max_num_seqs=4))
    _, _, _, rec, fi, _ = _sim(w)
    # it0: P(0,1); it1: P(2,3); it2: D(0..3): 0,1 -> g=2,3? ... computed by hand:
    # it0 prefill {0,1} g=1 ; it1 prefill {2,3} (4 slots) g=1 ; it2 decode {0,1,2,3} g=2 ;
    # it3 decode -> g=3 all finish ; it4 prefill {4,5} ; it5, it6 decodes -> finish at 6
    assert fi[0].tolist() == [3, 3, 3, 3, 6, 6]
    assert rec["iters"][0] == 7


def test_token_conservation_fuzz():
    # every iteration a request takes part in emits one token; recompute keeps tokens,
    # so sum over iterations of B == sum of generated tokens, with and without preemption.
    rng = np.random.default_rng(8)
    for trial in range(60):
        n = int(rng.integers(1, 30))
        lin = rng.integers(1, 40, n)
        lout = rng.integers(0, 40, n)
        kv = int(rng.integers(5, 12)) * 16
        w = F.tiny(lin, lout, sp=F.spec(l_max=80), eng=F.engine(kv_cap=kv, min_batched_tokens=80,
                                                                max_num_seqs=int(rng.integers(1, 9)),
                                                                block_size=16))
        _, lo, li, rec, fi, _ = _sim(w)
        assert rec["req_iters"][0] == np.maximum(lo[0], 1).sum()
        assert np.all(fi[0] < rec["iters"][0])


def test_truncate_and_resume_equals_straight_through():
    # simulate to tau, carry the state, resume with the same plan -> identical integers;
    # the end time agrees up to rounding of the re-based clock (reading c18).
    w = W.make_workload("c2", n_prompts=300, n_trials=3)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 3)
    full, fi_full, ft_full = P.simulate(4, 2, 1, lo, li, want_fin=True)
    rng = np.random.default_rng(0)
    for cut_frac in rng.uniform(0.05, 0.95, 8):
        st = P.fresh_state(3)
        tau = full["t_end"] * cut_frac
        r1, fi1, _ = P.simulate(4, 2, 1, lo, li, state=st, tau=tau, commit=True, want_fin=True)
        assert np.all(r1["flags"] & 2)
        r2, fi2, _ = P.simulate(4, 2, 1, lo, li, resume=1, state=st, commit=True, want_fin=True)
        assert np.array_equal(r1["iters"] + r2["iters"], full["iters"])
        assert np.array_equal(r1["req_iters"] + r2["req_iters"], full["req_iters"])
        f1 = O.rec_flops(r1)
        f2 = O.rec_flops(r2)
        assert all(f1[k] + f2[k] == O.rec_flops(full)[k] for k in range(3))
        np.testing.assert_allclose(r2["t_end"] + tau, full["t_end"], rtol=1e-12)
        assert np.all(st["st"][:, P.w.node == 4] >> 28 == O.ST_DONE)


# ------------------------------------------------------------------------------------------
# Stage metrics and greedy
# ------------------------------------------------------------------------------------------
def test_stage_metrics_spec_384_385():
    # one model: sim total 10 s, FLOPs F -> T = F/10 ; with 5 s load -> F/15
    sp = F.spec(L=1, c=10, h=8)
    load = F.zero_load()
    for ld in (0.0, 5.0):
        load[:, :] = ld
        w = F.tiny([4], [1], sp=sp, cf=F.coeff("const", 10.0), load=load)
        plan = O.Problem(w).plan_greedy(SEED, 1)
        assert len(plan["stages"]) == 1                       # S:394 one model, one plan
        st = plan["stages"][0]
        fl = O.flops_prefill(1, 10, 8, 1, 1, 4)
        assert st["mean_tE"] == 10.0 + ld
        assert st["T_E"] == fl / (10.0 + ld)


def test_stage_duration_is_first_finish():
    # S:331 / P:419: two independent models 5 s and 9 s in one stage -> t_E = 5
    slow_dp2 = F.zero_load()
    slow_dp2[:, 1] = 100.0          # make re-planning to dp=2 unattractive in stage 2
    w = F.multi([dict(l_in=[4], l_out=[1], cf=F.coeff("const", 5.0)),
                 dict(l_in=[4], l_out=[3], cf=F.coeff("const", 3.0), load=slow_dp2)], eng=F.engine(n_gpus=2))
    plan = O.Problem(w).plan_greedy(SEED, 1)
    s0 = plan["stages"][0]
    assert sorted(e[0] for e in s0["entries"]) == [0, 1]
    assert s0["fstar"] == 0 and s0["mean_tE"] == 5.0
    # the 9 s model (3 iterations of 3 s) is cut at the first boundary >= 5 (t = 6, c15) and
    # resumes in stage 2 with its overshoot 6 - 5 = 1 (c18): one more iteration ends at 1 + 3
    assert plan["stages"][1]["entries"] == [(1, 1, 1)] and plan["stages"][1]["mean_tE"] == 4.0
    assert plan["total"] == 9.0


def test_greedy_symmetric_tie_break():
    # identical models -> deterministic plan (lower node id first)
    mk = lambda: dict(l_in=[4] * 8, l_out=[5] * 8, sp=F.spec(tp_values=(1, 2)))
    w = F.multi([mk(), mk()], eng=F.engine(n_gpus=2))
    p1 = O.Problem(w).plan_greedy(SEED, 2)
    p2 = O.Problem(w).plan_greedy(SEED, 2)
    assert p1 == p2
    assert p1["stages"][0]["fstar"] == 0


def test_greedy_every_stage_valid_and_all_work_done():
    # every stage valid (#gpu <= N, one entry per node, inputs ready); replay finishes all
    w = W.make_workload("c4", n_docs=40, n_trials=2)
    P = O.Problem(w)
    plan = P.plan_greedy(SEED, 2)
    done = set()
    for s in plan["stages"]:
        nodes = [e[0] for e in s["entries"]]
        assert len(set(nodes)) == len(nodes)
        assert sum(d * t for (_, d, t) in s["entries"]) <= w.engine["n_gpus"]
        if 1 in nodes:
            assert 0 in nodes or 0 in done     # evaluator needs its summariser finished or co-scheduled
        done.add(s["fstar"])
    assert done == {0, 1}
    # complexity instrumentation (AC11): candidate evaluations <= K |V|^2 N^2 with K <= 4
    assert plan["n_cand_evals"] <= 4 * (2 ** 2) * (8 ** 2) * 4


def test_hand_trace_dependencies_summarise_then_evaluate():
    # P:474-476 + S:332: the fused summariser's chain successors become ready when their
    # predecessor finishes; the evaluator's requests appear mid-stage at the final summaries'
    # finish times.  doc0 = 1 chunk (r0), doc1 = 3 chunks (r1 -> r2 -> r3); 1 s per iteration.
    w = F.multi([
        dict(l_in=[10, 10, 10, 10], l_out=[1, 1, 1, 1], pred=[-1, -1, 1, 2], chain=[0, 1, 1, 1]),
        dict(l_in=[5, 5], l_out=[2, 2], pred=[0, 3]),
    ], eng=F.engine(n_gpus=4))
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, 1)
    assert li[0].tolist() == [10, 10, 11, 11, 6, 6]
    for dp_s in (1, 2):
        rs, fis, fts = P.simulate(0, dp_s, 1, lo, li, want_fin=True)
        assert rs["t_end"][0] == 3.0
        assert fts[0, :4].tolist() == [1.0, 1.0, 2.0, 3.0]
        # evaluator: idle until t=1, prefill e0 (->2), decode e0 (->3), e1 ready at 3: prefill
        # (->4), decode (->5)
        re, fie, fte = P.simulate(1, 1, 1, lo, li, src_fin=fts, want_fin=True)
        assert re["t_end"][0] == 5.0 and re["iters"][0] == 4
        assert fie[0, 4:].tolist() == [1, 3] and fte[0, 4:].tolist() == [3.0, 5.0]
        # cut at tau = 2.5: iterations starting before 2.5 ran (the decode 2 -> 3), e1 never moved
        st = P.fresh_state(1)
        rc, _, _ = P.simulate(1, 1, 1, lo, li, state=st, tau=np.array([2.5]), src_fin=fts, commit=True)
        assert rc["t_end"][0] == 3.0 and rc["flags"][0] == 2
        assert (st["st"][0, 4] >> 28) == O.ST_DONE and (st["st"][0, 5] >> 28) == O.ST_FRESH
        assert st["over"][0, 1, 0] == 0.5


# ------------------------------------------------------------------------------------------
# the paper's competitors: Max- / Min-heuristic and the Fig. 1 fixture
# ------------------------------------------------------------------------------------------
_fig1 = F.fig1


def test_fig1_greedy_beats_max_and_min_heuristics():
    # S:645 / P:734: greedy strictly better than Max-heuristic, no worse than Min-heuristic, and
    # within 5% of the optimum (bounded below by total work / N = 5.75 s)
    P = O.Problem(_fig1())
    g, mx, mn = (P.plan_greedy(SEED, 1, a)["total"] for a in ("greedy", "max", "min"))
    assert g < mx and g <= mn
    assert g <= 1.05 * 5.75
    # Max-heuristic closed form: model 0 on 4 replicas = 2 s, then each 3-request model on 3
    # replicas (4 gives the same throughput; ties keep fewer GPUs) = 1 s: 2 + 5 = 7 s
    assert mx == 7.0


def test_max_heuristic_structure():
    # P:664 / S:440: every stage has exactly one entry, that model runs to completion (it never
    # reappears), models are taken in id order once ready
    for w in (_fig1(), W.make_workload("c2", n_prompts=60, n_trials=2),
              W.make_workload("c4", n_docs=20, n_trials=2)):
        plan = O.Problem(w).plan_greedy(SEED, 2, "max")
        nodes = [s["entries"][0][0] for s in plan["stages"]]
        assert all(len(s["entries"]) == 1 and s["fstar"] == s["entries"][0][0] for s in plan["stages"])
        assert nodes == sorted(set(nodes)) == list(range(w.n_nodes))


def test_min_heuristic_even_split_paper_example():
    # "when there are 4 LLMs unfinished, Min-heuristic assigns 2 GPUs to each LLM. After 1
    # LLM finishes, Min-heuristic then repartitions the GPUs to make 2 LLMs have 3 GPUs each ...
    # and 1 LLM keeps its previously assigned 2 GPUs."  8 GPUs, 4 models, model 0 the smallest.
    w = F.even_split_4x8()
    plan = O.Problem(w).plan_greedy(SEED, 1, "min")
    s0, s1 = plan["stages"][0], plan["stages"][1]
    assert sorted(d * t for (_, d, t) in s0["entries"]) == [2, 2, 2, 2]
    assert s0["fstar"] == 0
    assert [e[0] for e in s1["entries"]] == [1, 2, 3]
    assert sorted(d * t for (_, d, t) in s1["entries"]) == [2, 3, 3]


def test_min_heuristic_structure():
    # per-stage GPU counts differ by at most 1 and, when a split exists, all N GPUs are
    # used; as many ready models as GPUs allow
    for w in (_fig1(), W.make_workload("c2", n_prompts=60, n_trials=2),
              W.make_workload("c4", n_docs=20, n_trials=2)):
        N = w.engine["n_gpus"]
        plan = O.Problem(w).plan_greedy(SEED, 2, "min")
        for s in plan["stages"]:
            gv = [d * t for (_, d, t) in s["entries"]]
            assert max(gv) - min(gv) <= 1
            assert sum(gv) <= N


# ------------------------------------------------------------------------------------------
# §5.5 ablations: no-preemption and known output lengths
# ------------------------------------------------------------------------------------------
@pytest.mark.parametrize("algo", ["greedy", "min"])
def test_no_preemption_keeps_plans_until_finished(algo):
    # "the execution plan of a model would not be changed once chosen and a running model
    # would not be stopped once started": an entry either continues unchanged in the next stage
    # or never appears again (it finished)
    for w, T in ((F.fig1(), 1), (F.even_split_4x8(), 1), (W.make_workload("c5", n_prompts=40, n_docs=30, n_trials=2), 2)):
        plan = O.Problem(w).plan_greedy(SEED, T, algo, preemption=False)
        st = plan["stages"]
        for k in range(len(st) - 1):
            later = {e[0] for s in st[k + 1:] for e in s["entries"]}
            for e in st[k]["entries"]:
                assert e in st[k + 1]["entries"] or e[0] not in later
        assert {e[0] for s in st for e in s["entries"]} == set(range(w.n_nodes))


def test_max_heuristic_has_no_no_preemption_variant():
    # "for Max-heuristic, there is no no-preemption version" -- it never preempts
    w = W.make_workload("c2", n_prompts=60, n_trials=2)
    P = O.Problem(w)
    assert P.plan_greedy(SEED, 2, "max") == P.plan_greedy(SEED, 2, "max", preemption=False)


@pytest.mark.parametrize("algo", ["greedy", "min"])
def test_preemption_helps_on_zero_load_fixtures(algo):
    # P:1099-1104 direction: with preemption, GPUs freed by a finished model go to the others.
    # Zero load cost isolates that effect.  Fig. 1 fixture totals by hand (1 s per request):
    #   greedy, no preemption: {0:dp2, 1, 2} 3 s | {0:dp2, 3:dp2} 1 s | {3:dp2, 4:dp2} 1 s |
    #     {4:dp2, 5:dp2} 1 s | {5:dp2} 1 s = 7 s
    #   min, no preemption: {0, 1, 2, 3} 3 s | {0, 4:dp2, 5} 2 s | {0, 5} 1 s | {0} 2 s = 8 s
    P = O.Problem(F.fig1())
    assert P.plan_greedy(SEED, 1, algo)["total"] == 6.0
    assert P.plan_greedy(SEED, 1, algo, preemption=False)["total"] == {"greedy": 7.0, "min": 8.0}[algo]
    # P:743 fixture (8 GPUs, 4 models): direction only
    P = O.Problem(F.even_split_4x8())
    assert P.plan_greedy(SEED, 1, algo)["total"] < P.plan_greedy(SEED, 1, algo, preemption=False)["total"]


def test_known_lengths_follow_the_sampler_arithmetic():
    # the true lengths replace the sampler's draw; caps and the chained
    # prompt are applied the same way.  l_true = the sampled trial reproduces it.
    w = W.make_workload("c4", n_docs=30, n_trials=1)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 3, 1)
    klo, kli = P.known_lengths(lo[0])
    assert (klo == lo).all() and (kli == li).all()
    # lengths above every cap clamp to min(cap, l_max - l_in)
    big = np.full(w.n_req, 60000, np.uint32)
    klo, kli = P.known_lengths(big)
    lmax = np.array([W.arch_spec(w.models[m])["l_max"] if isinstance(w.models[m], str) else w.models[m]["l_max"]
                     for m in w.node_model])[w.node]
    assert (klo[0] == np.minimum(w.cap_y, lmax - kli[0])).all()


def test_known_lengths_plan_equals_single_trial_plan():
    # a plan on known lengths equal to trial 0's draw is the 1-trial sampled plan (Alg. 1 with
    # T = 1 sees only the lengths), for all three planners
    w = W.make_workload("c2", n_prompts=60, n_trials=1)
    P = O.Problem(w)
    lo, _ = P.sample(SEED, 0, 1)
    for algo in ("greedy", "max", "min"):
        assert P.plan_greedy(SEED, 1, algo) == P.plan_greedy(12345, 1, algo, known_l_out=lo[0])


# ------------------------------------------------------------------------------------------
# runtime replay with the dynamic scheduler (reading c33)
# ------------------------------------------------------------------------------------------
def _hand_plan(stages):
    return dict(stages=[dict(entries=E, fstar=E[0][0], mean_tE=1.0, T_E=1.0) for E in stages],
                total=float(len(stages)))


def _replay_fixture(counts, n_gpus, cap=1):
    sp = F.spec(tp_values=(1,))
    nodes = [dict(l_in=[4] * c, l_out=[cap] * c, sp=sp) for c in counts]
    return F.multi(nodes, eng=F.engine(n_gpus=n_gpus, max_num_seqs=1))


@pytest.mark.parametrize("algo", ["greedy", "max", "min"])
def test_replay_with_the_plans_own_lengths_reproduces_it(algo):
    # "oracle identical to the planner's sampled lengths -> measured total equals planned
    # total exactly" (one-trial plan: the replay finds the planned first finishers).  Exception
    # required by P:626: when a planned stage leaves GPUs free, a running pair absent from it
    # keeps running ("then consider (M, P) if there are still available GPUs"), so the replay
    # may diverge there -- and only by such kept pairs.
    diverged = 0
    for w in (F.fig1(), W.make_workload("c2", n_prompts=120, n_trials=1),
              W.make_workload("c5", n_prompts=40, n_docs=30, n_trials=1)):
        P = O.Problem(w)
        plan = P.plan_greedy(SEED, 1, algo)
        r = P.replay(plan, SEED)
        rs, ps = r["stages"], plan["stages"]
        i = 0
        while i < len(ps) and i < len(rs) and rs[i]["entries"] == ps[i]["entries"]:
            assert rs[i]["duration"] == ps[i]["mean_tE"] and rs[i]["first_finisher"] == ps[i]["fstar"]
            i += 1
        if i == len(ps):
            assert len(rs) == len(ps) and r["total"] == plan["total"] and r["n_kept_room"] == 0
        else:
            diverged += 1
            extra = set(rs[i]["entries"]) - set(ps[i]["entries"])
            assert set(ps[i]["entries"]) <= set(rs[i]["entries"]) and extra
            assert extra <= set(rs[i - 1]["entries"]) and r["n_kept_room"] >= 1
    assert diverged <= 1


def test_replay_misprediction_keeps_last_stage_model_running():
    # P:622-625 hand trace (1 s per iteration, one sequence per replica, 4 GPUs): planned
    # E1 = {A, B, C} ending with A, E2 = {B, C on 2 GPUs}.  True lengths make A's two requests
    # 5 tokens (10 s): B finishes first at 3 s.  A's last planned stage is E1 -> keeps running
    # (resumed); C's plan changes -> reloaded on 2 GPUs, its 1 remaining request takes 1 s;
    # A then runs alone for the remaining 10 - 4 = 6 s.  Total 3 + 1 + 6 = 10 s.
    w = _replay_fixture([2, 3, 4], 4, cap=8)
    plan = _hand_plan([[(0, 1, 1), (1, 1, 1), (2, 1, 1)], [(1, 1, 1), (2, 2, 1)]])
    l_true = np.array([5, 5] + [1] * 7, np.uint32)
    r = O.Problem(w).replay(plan, SEED, known_l_out=l_true)
    st = r["stages"]
    assert [s["entries"] for s in st] == [[(0, 1, 1), (1, 1, 1), (2, 1, 1)], [(0, 1, 1), (2, 2, 1)], [(0, 1, 1)]]
    assert [s["first_finisher"] for s in st] == [1, 2, 0]
    assert [s["duration"] for s in st] == [3.0, 1.0, 6.0]
    assert st[1]["resumed"] == [1, 0] and st[2]["resumed"] == [1]
    assert st[0]["gpu_mask"] == [0b0001, 0b0010, 0b0100] and st[1]["gpu_mask"] == [0b0001, 0b0110]
    assert r["total"] == 10.0 and r["n_kept_last"] == 1
    assert r["idle_gpu_seconds"] == 1 * 3.0 + 1 * 1.0 + 3 * 6.0


@pytest.mark.parametrize("n_gpus", [2, 3])
def test_replay_pair_absent_from_next_stage(n_gpus):
    # P:625-626 hand traces.  Planned E1 = {0, 1}, E2 = {2 on 2 GPUs}, E3 = {1}.  Model 0 ends
    # E1 at 2 s; model 1 (2 of 4 requests left) is not in E2.
    #  N = 2: E2 takes every GPU -> model 1 is stopped and reloaded in E3: 2 + 2 + 2 = 6 s.
    #  N = 3: E2 is placed on GPUs {0, 2} (sparing model 1's GPU 1) and model 1 keeps running
    #         beside it; both end at 2 s: 2 + 2 = 4 s ("if GPUs remain").
    w = _replay_fixture([2, 4, 4], n_gpus)
    plan = _hand_plan([[(0, 1, 1), (1, 1, 1)], [(2, 2, 1)], [(1, 1, 1)]])
    r = O.Problem(w).replay(plan, SEED)
    st = r["stages"]
    if n_gpus == 2:
        assert [s["entries"] for s in st] == [[(0, 1, 1), (1, 1, 1)], [(2, 2, 1)], [(1, 1, 1)]]
        assert st[2]["resumed"] == [0] and r["n_stopped"] == 1
        assert r["total"] == 6.0 and r["idle_gpu_seconds"] == 2.0
    else:
        assert [s["entries"] for s in st] == [[(0, 1, 1), (1, 1, 1)], [(1, 1, 1), (2, 2, 1)]]
        assert st[1]["resumed"] == [1, 0] and st[1]["gpu_mask"] == [0b010, 0b101]
        assert r["n_kept_room"] == 1 and r["total"] == 4.0 and r["idle_gpu_seconds"] == 2.0


def test_replay_idle_time_fig1_max_heuristic():
    # S:553 interval arithmetic: Max-heuristic on the Fig. 1 fixture runs models 1-5 on 3 of
    # the 4 GPUs for 1 s each -> 5 idle GPU-seconds; greedy and Min keep every GPU busy
    P = O.Problem(F.fig1())
    for algo, idle in (("max", 5.0), ("greedy", 0.0), ("min", 0.0)):
        r = P.replay(P.plan_greedy(SEED, 1, algo), 99)
        assert r["idle_gpu_seconds"] == idle


def test_replay_invariants_under_mispredicted_lengths():
    # no GPU over-commit (disjoint masks of the right size), planned stages visited in
    # order, every model finishes, clock = sum of durations
    w = W.make_workload("c5", n_prompts=40, n_docs=30, n_trials=1)
    P = O.Problem(w)
    for algo in ("greedy", "min"):
        plan = P.plan_greedy(SEED, 1, algo)
        r = P.replay(plan, 4242)
        last = -1
        t = 0.0
        for s in r["stages"]:
            used = 0
            for (v, d, tp), m in zip(s["entries"], s["gpu_mask"]):
                assert bin(m).count("1") == d * tp and (used & m) == 0
                used |= m
            assert used < (1 << w.engine["n_gpus"])
            assert s["planned_stage"] >= last
            last = s["planned_stage"]
            assert s["t_start"] == t
            t += s["duration"]
        assert r["total"] == t
        assert {s["first_finisher"] for s in r["stages"]} <= set(range(w.n_nodes))


# ------------------------------------------------------------------------------------------
# cost-model coefficient fit (reading c34)
# ------------------------------------------------------------------------------------------
def test_fit_exact_lines_and_round_trip():
    # S:134 exact data latency = 2x + 1 -> (2, 1); S:150 / S:642 round trip: samples generated
    # from known per-bucket (a, b) with zero noise refit within 1e-6 relative
    a, b, nu, fl, rc = O.fit_coeffs([0, 10], np.arange(10.0), 2 * np.arange(10.0) + 1, 0)
    assert rc == 0 and abs(a[0] - 2) <= 1e-12 and abs(b[0] - 1) <= 1e-12 and nu[0] == 10 and fl[0] == 0
    w = W.make_workload("c2", n_prompts=10, n_trials=1)
    pr = W.make_profile(w, 1, noise=0.0, outlier_frac=0.0)
    a, b, nu, fl, rc = O.fit_coeffs(pr["off"], pr["x"], pr["y"], 0)
    assert rc == 0 and (fl == 0).all()
    for k, (s, p, i) in enumerate(pr["bucket"]):
        assert abs(a[k] / w.coeff[1][s, p, 0, i] - 1) <= 1e-6
        assert abs(b[k] / w.coeff[1][s, p, 1, i] - 1) <= 1e-6


def test_fit_matches_independent_least_squares():
    # closed-form normal equations vs numpy.polyfit (an independent LAPACK least-squares)
    rng = np.random.default_rng(3)
    off = [0]
    xs, ys = [], []
    for n in (2, 3, 17, 256, 1000):
        x = rng.uniform(1e9, 5e12, n)
        xs.append(x)
        ys.append(3e-15 * x + 2e-3 + 1e-4 * rng.standard_normal(n))
        off.append(off[-1] + n)
    x, y = np.concatenate(xs), np.concatenate(ys)
    a, b, nu, fl, rc = O.fit_coeffs(off, x, y, 0)
    assert rc == 0
    for k in range(len(off) - 1):
        pa, pb = np.polyfit(x[off[k]:off[k + 1]], y[off[k]:off[k + 1]], 1)
        if pa > 0:
            assert abs(a[k] / pa - 1) <= 1e-9 and abs(b[k] / pb - 1) <= 1e-9


def test_fit_trimming_drops_the_noise_points():
    # Fig. 5 noise points: n = 1000, trim 1 % -> the 10 samples of largest residual go; 10
    # gross outliers are exactly those, so the fit equals least squares on the clean samples
    rng = np.random.default_rng(4)
    x = rng.uniform(1.0, 100.0, 1000)
    y = 0.5 * x + 3.0 + 0.01 * rng.standard_normal(1000)
    bad = rng.choice(1000, 10, replace=False)
    y[bad] += 500.0
    a, b, nu, fl, rc = O.fit_coeffs([0, 1000], x, y, 10)
    keep = np.setdiff1d(np.arange(1000), bad)
    pa, pb = np.polyfit(x[keep], y[keep], 1)
    assert rc == 0 and nu[0] == 990
    assert abs(a[0] / pa - 1) <= 1e-9 and abs(b[0] / pb - 1) <= 1e-9
    a0, _, nu0, _, _ = O.fit_coeffs([0, 1000], x, y, 0)
    assert nu0[0] == 1000 and abs(a0[0] - 0.5) > abs(a[0] - 0.5)


def test_fit_clamps_negative_slope_and_rejects_degenerate_buckets():
    # negative fitted a clamped to 0 (b = mean latency, the least-squares constant);
    # a bucket with < 2 distinct x is an error
    x = np.arange(5.0)
    a, b, nu, fl, rc = O.fit_coeffs([0, 5], x, 10.0 - x, 0)
    assert rc == 0 and a[0] == 0.0 and b[0] == 8.0 and fl[0] == 2
    a, b, nu, fl, rc = O.fit_coeffs([0, 5, 8], np.r_[x, 7.0, 7.0, 7.0], np.r_[x, 1.0, 2.0, 3.0], 0)
    assert rc != 0 and fl.tolist() == [0, 1] and a[1] == 0.0 and nu[1] == 0
    a, b, nu, fl, rc = O.fit_coeffs([0, 1], [1.0], [1.0], 0)
    assert rc != 0 and fl[0] == 1
