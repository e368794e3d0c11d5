"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around liboracle.so (oracle.cpp): a plain, slow, obviously-correct CPU reference
of SamuLLM's sampling-then-simulation estimator (arXiv 2503.16893).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
package.  It shares no code with paper_2503_16893_b200/ (the CUDA path) and neither imports
the other; both consume samu_workloads (inputs only).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")

ST_FRESH, ST_QUEUED, ST_PREEMPTED, ST_RUNNING, ST_DONE = 0, 1, 2, 3, 4


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared",
                               "-pthread", "-Wall", "-o", _SO, src])
    return _SO


class or_model(C.Structure):
    _fields_ = [("L", C.c_uint32), ("h", C.c_uint32), ("c", C.c_uint64), ("l_max", C.c_uint32),
                ("tp_mask", C.c_uint32), ("weight_bytes", C.c_uint64),
                ("kv_bytes_per_token", C.c_uint64), ("n_buckets", C.c_int32),
                ("bucket_B", C.POINTER(C.c_uint32)), ("coeff", C.POINTER(C.c_double)),
                ("load", C.POINTER(C.c_double)), ("ecdf_k", C.c_int32),
                ("ecdf_values", C.POINTER(C.c_uint32)), ("ecdf_cum", C.POINTER(C.c_uint32))]


class or_engine(C.Structure):
    _fields_ = [("max_num_seqs", C.c_uint32), ("block_size", C.c_uint32),
                ("min_batched_tokens", C.c_uint32), ("mem_util_permille", C.c_uint32),
                ("mem_bytes_per_gpu", C.c_uint64), ("kv_cap_bytes_per_gpu", C.c_uint64),
                ("n_gpus", C.c_uint32)]


class or_app(C.Structure):
    _fields_ = [("engine", or_engine), ("n_models", C.c_int32), ("models", C.POINTER(or_model)),
                ("n_nodes", C.c_int32), ("node_model", C.POINTER(C.c_int32)),
                ("n_req", C.c_int32), ("l_in_base", C.POINTER(C.c_uint32)),
                ("cap_y", C.POINTER(C.c_uint32)), ("pred", C.POINTER(C.c_int32)),
                ("node", C.POINTER(C.c_int32)), ("chain", C.POINTER(C.c_int32))]


class or_cand(C.Structure):
    _fields_ = [("node", C.c_int32), ("dp", C.c_int32), ("tp", C.c_int32), ("resume", C.c_int32)]


class or_rec(C.Structure):
    _fields_ = [("t_end", C.c_double), ("flops_lo", C.c_uint64), ("flops_hi", C.c_uint64),
                ("req_iters", C.c_uint64), ("iters", C.c_uint32), ("flags", C.c_uint32)]


REC_DTYPE = np.dtype([("t_end", "<f8"), ("flops_lo", "<u8"), ("flops_hi", "<u8"),
                      ("req_iters", "<u8"), ("iters", "<u4"), ("flags", "<u4")])


class or_summary(C.Structure):
    _fields_ = [("mean_t", C.c_double), ("p50_t", C.c_double), ("p90_t", C.c_double), ("p99_t", C.c_double),
                ("mean_flops", C.c_double), ("mean_req_iters", C.c_double)]


SUMMARY_DTYPE = np.dtype([("mean_t", "<f8"), ("p50_t", "<f8"), ("p90_t", "<f8"), ("p99_t", "<f8"),
                          ("mean_flops", "<f8"), ("mean_req_iters", "<f8")])

ITER_DTYPE = np.dtype([("t_start", "<f8"), ("lat", "<f8"), ("flops", "<u8"), ("s", "<u8"), ("S", "<u8"),
                       ("free_blocks", "<i8"), ("kind", "<u4"), ("B", "<u4"), ("n_preempted", "<u4"),
                       ("n_finished", "<u4")])


class or_stage(C.Structure):
    _fields_ = [("n_entries", C.c_int32), ("node", C.c_int32 * 16), ("dp", C.c_int32 * 16),
                ("tp", C.c_int32 * 16), ("fstar", C.c_int32), ("mean_tE", C.c_double),
                ("T_E", C.c_double)]


class or_plan(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("stages", or_stage * 64), ("total", C.c_double),
                ("n_cand_evals", C.c_int64)]


class or_replay_stage(C.Structure):
    _fields_ = [("n_entries", C.c_int32), ("node", C.c_int32 * 16), ("dp", C.c_int32 * 16), ("tp", C.c_int32 * 16),
                ("gpu_mask", C.c_uint32 * 16), ("resumed", C.c_int32 * 16), ("planned_stage", C.c_int32),
                ("first_finisher", C.c_int32), ("idle_gpus", C.c_int32), ("t_start", C.c_double),
                ("duration", C.c_double)]


class or_replay(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("stages", or_replay_stage * 64), ("total", C.c_double),
                ("planned_total", C.c_double), ("idle_gpu_seconds", C.c_double), ("n_kept_last", C.c_int32),
                ("n_kept_room", C.c_int32), ("n_stopped", C.c_int32)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        # SAMU_ORACLE_SO: an alternative build of the same source (the sanitizer test)
        L = C.CDLL(os.environ.get("SAMU_ORACLE_SO") or build())
        P = C.c_void_p
        L.or_last_error.restype = C.c_char_p
        L.or_problem_create.restype = P
        L.or_problem_create.argtypes = [C.POINTER(or_app)]
        L.or_problem_destroy.argtypes = [P]
        L.or_philox4x32_10.argtypes = [C.POINTER(C.c_uint32)] * 3
        L.or_ecdf_inverse.restype = C.c_uint32
        L.or_ecdf_inverse.argtypes = [P, C.c_int32, C.c_uint32]
        L.or_flops_prefill.restype = C.c_uint64
        L.or_flops_prefill.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64]
        L.or_flops_decode.restype = C.c_uint64
        L.or_flops_decode.argtypes = [C.c_uint32, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64, C.c_uint64]
        L.or_dense_coeff.argtypes = [P, C.c_int32, C.c_int32, P, P]
        L.or_plan_blocks.restype = C.c_int64
        L.or_plan_blocks.argtypes = [P, C.c_int32, C.c_int32, C.c_int32]
        L.or_enumerate_plans.argtypes = [P, C.c_int32, P, P, C.c_int32]
        L.or_iter_latency.restype = C.c_double
        L.or_iter_latency.argtypes = [P, P, C.c_uint64, C.c_uint64, C.c_uint64]
        L.or_sample_lengths.argtypes = [P, C.c_uint64, C.c_int32, C.c_int32, P, P]
        L.or_simulate.argtypes = [P, C.POINTER(or_cand), C.c_int32, P, P, P, P, P, P, P, P,
                                  C.c_int32, P, P, P]
        L.or_simulate_many.argtypes = [P, C.c_int32, P, C.c_int32, P, P, C.c_int32, P]
        L.or_summarise.argtypes = [C.c_int32, C.c_int32, P, P]
        L.or_trace_replica.argtypes = [P, C.POINTER(or_cand), P, P, C.c_int32, C.c_int64, P, C.c_int64, P, P, P,
                                       C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
        L.or_plan_greedy.argtypes = [P, C.c_uint64, C.c_int32, C.POINTER(or_plan)]
        L.or_plan_max_heuristic.argtypes = [P, C.c_uint64, C.c_int32, C.POINTER(or_plan)]
        L.or_plan_min_heuristic.argtypes = [P, C.c_uint64, C.c_int32, C.POINTER(or_plan)]
        L.or_known_lengths.argtypes = [P, P, P, P]
        L.or_fit_coeffs.argtypes = [C.c_int32, P, P, P, C.c_int32, P, P, P, P]
        L.or_replay_plan.argtypes = [P, C.POINTER(or_plan), C.c_uint64, P, C.POINTER(or_replay)]
        L.or_plan_run.argtypes = [P, C.c_uint64, C.c_int32, C.c_int32, C.c_int32, P, C.POINTER(or_plan)]
        _lib = L
    return _lib


def _ptr(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class OracleError(RuntimeError):
    def __init__(self, rc, msg):
        super().__init__(f"oracle rc={rc}: {msg}")
        self.rc = rc


def _check(rc):
    if rc != 0:
        raise OracleError(rc, lib().or_last_error().decode())


def philox4x32_10(ctr, key):
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    k = (C.c_uint32 * 2)(*[int(x) & 0xFFFFFFFF for x in key])
    o = (C.c_uint32 * 4)()
    lib().or_philox4x32_10(c, k, o)
    return [int(x) for x in o]


def flops_prefill(L, c, h, tp, B, s):
    return int(lib().or_flops_prefill(L, c, h, tp, B, s))


def flops_decode(L, c, h, tp, B, S):
    return int(lib().or_flops_decode(L, c, h, tp, B, S))


def iter_latency(a3, b3, flops, Bs, S):
    a = np.ascontiguousarray(a3, dtype=np.float64)
    b = np.ascontiguousarray(b3, dtype=np.float64)
    return float(lib().or_iter_latency(_ptr(a), _ptr(b), int(flops), int(Bs), int(S)))


class Problem:
    """A validated copy of one synthetic application (samu_workloads.Workload)."""

    def __init__(self, w):
        self.w = w
        self._keep = []
        ms = (or_model * len(w.models))()
        for i, m in enumerate(w.models):
            arrs = [np.ascontiguousarray(w.coeff_B, np.uint32), np.ascontiguousarray(w.coeff[i], np.float64),
                    np.ascontiguousarray(w.load[i], np.float64), np.ascontiguousarray(w.ecdf_values[i], np.uint32),
                    np.ascontiguousarray(w.ecdf_cum[i], np.uint32)]
            self._keep += arrs
            ms[i] = or_model(m["L"], m["h"], m["c"], m["l_max"], m["tp_mask"], m["weight_bytes"],
                             m["kv_bytes_per_token"], len(w.coeff_B),
                             arrs[0].ctypes.data_as(C.POINTER(C.c_uint32)),
                             arrs[1].ctypes.data_as(C.POINTER(C.c_double)),
                             arrs[2].ctypes.data_as(C.POINTER(C.c_double)), len(arrs[3]),
                             arrs[3].ctypes.data_as(C.POINTER(C.c_uint32)),
                             arrs[4].ctypes.data_as(C.POINTER(C.c_uint32)))
        e = w.engine
        eng = or_engine(e["max_num_seqs"], e["block_size"], e["min_batched_tokens"],
                        e["mem_util_permille"], e["mem_bytes_per_gpu"], e["kv_cap_bytes_per_gpu"],
                        e["n_gpus"])
        cols = [np.ascontiguousarray(w.node_model, np.int32), np.ascontiguousarray(w.l_in_base, np.uint32),
                np.ascontiguousarray(w.cap_y, np.uint32), np.ascontiguousarray(w.pred, np.int32),
                np.ascontiguousarray(w.node, np.int32), np.ascontiguousarray(w.chain, np.int32)]
        self._keep += cols
        self._keep.append(ms)
        app = or_app(eng, len(w.models), ms, w.n_nodes, cols[0].ctypes.data_as(C.POINTER(C.c_int32)),
                     w.n_req, cols[1].ctypes.data_as(C.POINTER(C.c_uint32)),
                     cols[2].ctypes.data_as(C.POINTER(C.c_uint32)),
                     cols[3].ctypes.data_as(C.POINTER(C.c_int32)),
                     cols[4].ctypes.data_as(C.POINTER(C.c_int32)),
                     cols[5].ctypes.data_as(C.POINTER(C.c_int32)))
        self.h = lib().or_problem_create(C.byref(app))
        if not self.h:
            raise OracleError(-1, lib().or_last_error().decode())
        self.n_req = w.n_req
        self.n_nodes = w.n_nodes
        self.max_seqs = e["max_num_seqs"]

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.or_problem_destroy(self.h)
            self.h = None

    # -- primitives --
    def ecdf_inverse(self, model, u):
        return int(lib().or_ecdf_inverse(self.h, model, int(u)))

    def dense_coeff(self, model, tp):
        a = np.zeros((3, self.max_seqs), np.float64)
        b = np.zeros((3, self.max_seqs), np.float64)
        _check(lib().or_dense_coeff(self.h, model, tp, _ptr(a), _ptr(b)))
        return a, b

    def plan_blocks(self, model, dp, tp):
        return int(lib().or_plan_blocks(self.h, model, dp, tp))

    def plans(self, model):
        n = lib().or_enumerate_plans(self.h, model, None, None, 0)
        dp = np.zeros(n, np.int32)
        tp = np.zeros(n, np.int32)
        lib().or_enumerate_plans(self.h, model, _ptr(dp), _ptr(tp), n)
        return list(zip(dp.tolist(), tp.tolist()))

    # -- hot path --
    def sample(self, seed, trial_begin, n_trials):
        lo = np.zeros((n_trials, self.n_req), np.uint16)
        li = np.zeros((n_trials, self.n_req), np.uint16)
        _check(lib().or_sample_lengths(self.h, seed, trial_begin, n_trials, _ptr(lo), _ptr(li)))
        return lo, li

    def known_lengths(self, l_true):
        """Known output lengths in place of the sampler: one trial [1, n]."""
        lt = np.ascontiguousarray(l_true, np.uint32).reshape(self.n_req)
        lo = np.zeros((1, self.n_req), np.uint16)
        li = np.zeros((1, self.n_req), np.uint16)
        _check(lib().or_known_lengths(self.h, _ptr(lt), _ptr(lo), _ptr(li)))
        return lo, li

    def fresh_state(self, n_trials):
        return dict(st=np.zeros((n_trials, self.n_req), np.uint32),
                    g=np.zeros((n_trials, self.n_req), np.uint16),
                    fin_t=np.full((n_trials, self.n_req), np.inf),
                    over=np.zeros((n_trials, self.n_nodes, 16), np.float64))

    def simulate(self, node, dp, tp, l_out, l_in, resume=0, state=None, tau=None, src_fin=None,
                 commit=False, want_fin=False):
        T = l_out.shape[0]
        rec = np.zeros(T, REC_DTYPE)
        fin_iter = np.full((T, self.n_req), 0xFFFFFFFF, np.uint32) if want_fin else None
        fin_t = np.full((T, self.n_req), np.inf) if want_fin else None
        s = state or {}
        cand = or_cand(node, dp, tp, resume)
        tau_a = None if tau is None else np.ascontiguousarray(tau, np.float64)
        _check(lib().or_simulate(self.h, C.byref(cand), T, _ptr(l_out), _ptr(l_in), _ptr(s.get("st")),
                                 _ptr(s.get("g")), _ptr(s.get("fin_t")), _ptr(s.get("over")), _ptr(tau_a),
                                 _ptr(src_fin), 1 if commit else 0, _ptr(rec), _ptr(fin_iter), _ptr(fin_t)))
        return rec, fin_iter, fin_t

    def simulate_many(self, cands, l_out, l_in, n_threads):
        T = l_out.shape[0]
        cs = (or_cand * len(cands))(*[or_cand(n, d, t, 0) for (n, d, t) in cands])
        rec = np.zeros((len(cands), T), REC_DTYPE)
        _check(lib().or_simulate_many(self.h, len(cands), cs, T, _ptr(l_out), _ptr(l_in), n_threads, _ptr(rec)))
        return rec

    def trace(self, node, dp, tp, l_out_row, l_in_row, replica=0):
        """Per-iteration descriptors of one fresh replica-sim and the running set
        [(request, g)] after every iteration."""
        lo = np.ascontiguousarray(l_out_row, np.uint16)
        li = np.ascontiguousarray(l_in_row, np.uint16)
        cand = or_cand(node, dp, tp, 0)
        nd, nr = C.c_int64(0), C.c_int64(0)
        lib().or_trace_replica(self.h, C.byref(cand), _ptr(lo), _ptr(li), replica, 0, None, 0, None, None, None,
                               C.byref(nd), C.byref(nr))
        desc = np.zeros(nd.value, ITER_DTYPE)
        req = np.zeros(max(nr.value, 1), np.uint32)
        g = np.zeros(max(nr.value, 1), np.uint32)
        off = np.zeros(nd.value + 1, np.int64)
        _check(lib().or_trace_replica(self.h, C.byref(cand), _ptr(lo), _ptr(li), replica, nd.value, _ptr(desc),
                                      nr.value, _ptr(req), _ptr(g), _ptr(off), C.byref(nd), C.byref(nr)))
        running = [list(zip(req[off[i]:off[i + 1]].tolist(), g[off[i]:off[i + 1]].tolist())) for i in range(nd.value)]
        return desc, running

    def replay(self, plan, seed, known_l_out=None):
        """Run `plan` (a dict from plan_greedy) against true lengths with the dynamic scheduler
        (P:620-627): known_l_out [n_req], or trial 0 of the sampler with `seed`."""
        P = or_plan()
        P.n_stages = len(plan["stages"])
        for i, s in enumerate(plan["stages"]):
            S = P.stages[i]
            S.n_entries = len(s["entries"])
            for j, (v, d, t) in enumerate(s["entries"]):
                S.node[j], S.dp[j], S.tp[j] = v, d, t
            S.fstar, S.mean_tE, S.T_E = s["fstar"], s["mean_tE"], s["T_E"]
        P.total = plan["total"]
        lt = None if known_l_out is None else np.ascontiguousarray(known_l_out, np.uint32)
        out = or_replay()
        _check(lib().or_replay_plan(self.h, C.byref(P), seed, _ptr(lt), C.byref(out)))
        stages = []
        for i in range(out.n_stages):
            s = out.stages[i]
            n = s.n_entries
            stages.append(dict(entries=[(s.node[j], s.dp[j], s.tp[j]) for j in range(n)],
                               gpu_mask=list(s.gpu_mask[:n]), resumed=list(s.resumed[:n]),
                               planned_stage=s.planned_stage, first_finisher=s.first_finisher,
                               idle_gpus=s.idle_gpus, t_start=s.t_start, duration=s.duration))
        return dict(stages=stages, total=out.total, planned_total=out.planned_total,
                    idle_gpu_seconds=out.idle_gpu_seconds, n_kept_last=out.n_kept_last,
                    n_kept_room=out.n_kept_room, n_stopped=out.n_stopped)

    def plan_greedy(self, seed, n_trials, algo="greedy", preemption=True, known_l_out=None):
        """algo greedy (Alg. 1) / max / min; preemption=False and known_l_out are the
        §5.5 ablations (known_l_out needs n_trials == 1)."""
        plan = or_plan()
        lt = None if known_l_out is None else np.ascontiguousarray(known_l_out, np.uint32)
        _check(lib().or_plan_run(self.h, seed, n_trials, {"greedy": 0, "max": 1, "min": 2}[algo],
                             1 if preemption else 0, _ptr(lt), C.byref(plan)))
        stages = []
        for i in range(plan.n_stages):
            s = plan.stages[i]
            stages.append(dict(entries=[(s.node[j], s.dp[j], s.tp[j]) for j in range(s.n_entries)],
                               fstar=s.fstar, mean_tE=s.mean_tE, T_E=s.T_E))
        return dict(stages=stages, total=plan.total, n_cand_evals=plan.n_cand_evals)


def fit_coeffs(off, x, y, trim_permille=10):
    """Per-bucket least-squares (a, b) with top-residual trimming (reading c34).
    Returns (a, b, n_used, flags, rc): rc != 0 if a bucket has < 2 distinct x."""
    off = np.ascontiguousarray(off, np.int64)
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    nb = len(off) - 1
    a, b = np.zeros(nb), np.zeros(nb)
    n_used, flags = np.zeros(nb, np.int32), np.zeros(nb, np.int32)
    rc = lib().or_fit_coeffs(nb, _ptr(off), _ptr(x), _ptr(y), trim_permille, _ptr(a), _ptr(b), _ptr(n_used), _ptr(flags))
    return a, b, n_used, flags, rc


def summarise(recs) -> np.ndarray:
    """Per-candidate mean / nearest-rank p50, p90, p99 of t_end, mean FLOPs and mean
    request-iterations over trials (reading c17); recs [n_cands][T] (REC_DTYPE)."""
    r = np.ascontiguousarray(np.atleast_2d(recs), REC_DTYPE)
    out = np.zeros(r.shape[0], SUMMARY_DTYPE)
    _check(lib().or_summarise(r.shape[0], r.shape[1], _ptr(r), _ptr(out)))
    return out


def rec_flops(rec) -> np.ndarray:
    """Exact u128 FLOP sums as Python ints (object array)."""
    return np.array([(int(h) << 64) | int(l) for h, l in zip(np.ravel(rec["flops_hi"]), np.ravel(rec["flops_lo"]))],
                    dtype=object).reshape(np.shape(rec))
