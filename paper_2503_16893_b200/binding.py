"""Thin Python binding of libsamu's C ABI (include/samu.h): argument marshalling only.

Every step of the estimator runs in libsamu's CUDA kernels; PyTorch only allocates device
memory and provides the stream.  There is no CPU fallback: importing works anywhere, but
creating a context raises unless libsamu.so is built and a CUDA device is present.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsamu.so")

SAMU_OK, SAMU_E_INVALID, SAMU_E_INFEASIBLE, SAMU_E_NOMEM, SAMU_E_CUDA, SAMU_E_NCCL, SAMU_E_STATE = 0, -1, -2, -3, -4, -5, -6
ST_FRESH, ST_QUEUED, ST_PREEMPTED, ST_RUNNING, ST_DONE = 0, 1, 2, 3, 4
N_TP_SLOTS, MAX_DP = 5, 16


class samu_model_spec(C.Structure):
    _fields_ = [("n_layers", C.c_uint32), ("hidden", C.c_uint32), ("c", C.c_uint64), ("l_max", C.c_uint32),
                ("tp_mask", C.c_uint32), ("weight_bytes", C.c_uint64), ("kv_bytes_per_token", C.c_uint64)]


class samu_engine_cfg(C.Structure):
    _fields_ = [("max_num_seqs", C.c_uint32), ("block_size", C.c_uint32), ("min_batched_tokens", C.c_uint32),
                ("mem_util_permille", C.c_uint32), ("mem_bytes_per_gpu", C.c_uint64),
                ("kv_cap_bytes_per_gpu", C.c_uint64), ("n_gpus", C.c_uint32)]


class samu_request(C.Structure):
    _fields_ = [("l_in_base", C.c_uint32), ("cap_y", C.c_uint32), ("pred", C.c_int32), ("node", C.c_int32),
                ("chain", C.c_int32)]


class samu_trial_rec(C.Structure):
    _fields_ = [("t_end", C.c_double), ("flops_lo", C.c_uint64), ("flops_hi", C.c_uint64),
                ("req_iters", C.c_uint64), ("iters", C.c_uint32), ("flags", C.c_uint32)]


class samu_candidate(C.Structure):
    _fields_ = [("node", C.c_int32), ("dp", C.c_int32), ("tp", C.c_int32), ("resume", C.c_int32),
                ("dep_src", C.c_int32), ("commit", C.c_int32)]


class samu_cand_summary(C.Structure):
    _fields_ = [("mean_t", C.c_double), ("p50_t", C.c_double), ("p90_t", C.c_double), ("p99_t", C.c_double),
                ("mean_flops", C.c_double), ("mean_req_iters", C.c_double)]


class samu_plan_stage(C.Structure):
    _fields_ = [("n_entries", C.c_int32), ("node", C.c_int32 * 16), ("dp", C.c_int32 * 16),
                ("tp", C.c_int32 * 16), ("fstar", C.c_int32), ("mean_tE", C.c_double), ("T_E", C.c_double)]


class samu_plan(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("stages", samu_plan_stage * 64), ("total", C.c_double),
                ("n_cand_evals", C.c_int64), ("n_sims", C.c_int64), ("req_iters", C.c_uint64)]


REC_DTYPE = np.dtype([("t_end", "<f8"), ("flops_lo", "<u8"), ("flops_hi", "<u8"), ("req_iters", "<u8"),
                      ("iters", "<u4"), ("flags", "<u4")])
assert REC_DTYPE.itemsize == C.sizeof(samu_trial_rec) == 40


class samu_replay_stage(C.Structure):
    _fields_ = [("n_entries", C.c_int32), ("node", C.c_int32 * 16), ("dp", C.c_int32 * 16), ("tp", C.c_int32 * 16),
                ("gpu_mask", C.c_uint32 * 16), ("resumed", C.c_int32 * 16), ("planned_stage", C.c_int32),
                ("first_finisher", C.c_int32), ("idle_gpus", C.c_int32), ("t_start", C.c_double),
                ("duration", C.c_double)]


class samu_replay(C.Structure):
    _fields_ = [("n_stages", C.c_int32), ("stages", samu_replay_stage * 64), ("total", C.c_double),
                ("planned_total", C.c_double), ("idle_gpu_seconds", C.c_double), ("n_kept_last", C.c_int32),
                ("n_kept_room", C.c_int32), ("n_stopped", C.c_int32)]


class samu_plan_opts(C.Structure):
    _fields_ = [("algo", C.c_int32), ("allow_preemption", C.c_int32), ("known_l_out", C.c_void_p)]


ALGOS = {"greedy": 0, "max": 1, "min": 2}

EXPORTED = ["samu_ctx_create", "samu_ctx_destroy", "samu_local_group_create", "samu_local_group_destroy",
            "samu_ctx_create_local", "samu_last_error", "samu_launch_count", "samu_share_stats", "samu_nccl_unique_id",
            "samu_model_register",
            "samu_ecdf_load", "samu_app_load", "samu_enumerate_plans", "samu_sample_lengths", "samu_sample_requests",
            "samu_simulate_batch",
            "samu_plan_greedy", "samu_plan_max_heuristic", "samu_plan_min_heuristic", "samu_plan_run", "samu_known_lengths",
            "samu_replay_plan", "samu_fit_coeffs", "samu_plan_free", "samu_shard_plan", "samu_shard_classes"]

_lib = None


def lib():
    """Load libsamu.so (built in-tree by __graft_entry__.build()).  Raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libsamu.so not built ({LIB_PATH}); run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.samu_ctx_create.argtypes = [C.POINTER(P), C.c_int32, P, C.c_int32, C.c_int32, P]
        L.samu_local_group_create.argtypes = [C.POINTER(P), C.c_int32]
        L.samu_local_group_destroy.argtypes = [P]
        L.samu_local_group_destroy.restype = None
        L.samu_ctx_create_local.argtypes = [C.POINTER(P), C.c_int32, P, C.c_int32, P]
        L.samu_ctx_destroy.argtypes = [P]
        L.samu_ctx_destroy.restype = None
        L.samu_last_error.argtypes = [P]
        L.samu_last_error.restype = C.c_char_p
        L.samu_nccl_unique_id.argtypes = [P]
        L.samu_launch_count.argtypes = [P]
        L.samu_launch_count.restype = C.c_uint64
        L.samu_share_stats.argtypes = [P, P]
        L.samu_share_stats.restype = None
        L.samu_model_register.argtypes = [P, C.c_int32, C.POINTER(samu_model_spec), C.c_int32, P, P, P]
        L.samu_ecdf_load.argtypes = [P, C.c_int32, P, P, C.c_int32]
        L.samu_app_load.argtypes = [P, C.POINTER(samu_engine_cfg), C.c_int32, P, C.c_int32, P]
        L.samu_enumerate_plans.argtypes = [P, C.c_int32, P, P, C.c_int32]
        L.samu_enumerate_plans.restype = C.c_int32
        L.samu_sample_lengths.argtypes = [P, C.c_uint64, C.c_int32, C.c_int32, P, P]
        L.samu_sample_requests.argtypes = [P, C.c_int32, C.c_uint32, P, C.c_int32, C.c_uint32, C.c_uint64, C.c_int32,
                                           C.c_int32, P, P]
        L.samu_simulate_batch.argtypes = [P, P, C.c_int32, P, P, C.c_int32, P, P, P, P, P, P, P, P, P]
        L.samu_plan_greedy.argtypes = [P, C.c_uint64, C.c_int32, C.POINTER(C.POINTER(samu_plan))]
        L.samu_plan_max_heuristic.argtypes = [P, C.c_uint64, C.c_int32, C.POINTER(C.POINTER(samu_plan))]
        L.samu_plan_min_heuristic.argtypes = [P, C.c_uint64, C.c_int32, C.POINTER(C.POINTER(samu_plan))]
        L.samu_plan_run.argtypes = [P, C.c_uint64, C.c_int32, C.POINTER(samu_plan_opts),
                                    C.POINTER(C.POINTER(samu_plan))]
        L.samu_known_lengths.argtypes = [P, P, P, P]
        L.samu_replay_plan.argtypes = [P, C.POINTER(samu_plan), C.c_uint64, P, C.POINTER(samu_replay)]
        L.samu_fit_coeffs.argtypes = [P, C.c_int32, P, P, P, C.c_int32, P, P, P, P]
        L.samu_plan_free.argtypes = [C.POINTER(samu_plan)]
        L.samu_plan_free.restype = None
        L.samu_shard_plan.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, P, P, P, P, P]
        L.samu_shard_classes.argtypes = [C.c_int32, P, C.c_int32, P]
        _lib = L
    return _lib


class SamuError(RuntimeError):
    def __init__(self, rc, msg):
        super().__init__(f"libsamu rc={rc}: {msg}")
        self.rc = rc


def _np_ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _t_ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


def samu_nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = lib().samu_nccl_unique_id(C.cast(buf, C.c_void_p))
    if rc:
        raise SamuError(rc, "ncclGetUniqueId failed")
    return bytes(buf)


def samu_shard_plan(n_trials: int, world: int, rank: int, forced_classes: int = 0) -> Dict[str, int]:
    """libsamu's (trial block, job class) sharding of `rank` (host-only, no GPU needed)."""
    out = [C.c_int32() for _ in range(5)]
    rc = lib().samu_shard_plan(n_trials, world, rank, forced_classes, *[C.byref(o) for o in out])
    if rc:
        raise SamuError(rc, "samu_shard_plan: invalid arguments")
    keys = ("trial_blocks", "job_classes", "trial_begin", "trial_count", "my_class")
    return {k: o.value for k, o in zip(keys, out)}


def samu_shard_classes(work, job_classes: int) -> np.ndarray:
    """libsamu's job -> class assignment of one batch (longest-first onto the least loaded)."""
    w = np.ascontiguousarray(work, dtype=np.float64)
    cls = np.zeros(len(w), np.int32)
    rc = lib().samu_shard_classes(len(w), _np_ptr(w), job_classes, _np_ptr(cls))
    if rc:
        raise SamuError(rc, "samu_shard_classes: invalid arguments")
    return cls


class LocalGroup:
    """In-process rank group (samu_local_group): one Samu context per thread and rank."""

    def __init__(self, world: int):
        h = C.c_void_p()
        rc = lib().samu_local_group_create(C.byref(h), world)
        if rc:
            raise SamuError(rc, "samu_local_group_create failed")
        self.h, self.world = h, world

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.samu_local_group_destroy(self.h)
            self.h = None


class Samu:
    """One libsamu context (one per process / GPU).  Device buffers are torch CUDA tensors."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: Optional[bytes] = None,
                 stream=None, local_group: Optional[LocalGroup] = None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("libsamu needs a CUDA device (no CPU fallback)")
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        h = C.c_void_p()
        if local_group is not None:
            world = local_group.world
            rc = lib().samu_ctx_create_local(C.byref(h), device, C.c_void_p(self.stream.cuda_stream), rank,
                                             local_group.h)
        else:
            idbuf = None if nccl_id is None else (C.c_uint8 * 128).from_buffer_copy(nccl_id)
            rc = lib().samu_ctx_create(C.byref(h), device, C.c_void_p(self.stream.cuda_stream), rank, world,
                                       None if idbuf is None else C.cast(idbuf, C.c_void_p))
        if rc:
            raise SamuError(rc, "samu_ctx_create failed")
        self.h = h
        self.rank, self.world = rank, world
        self.n_req = 0
        self.n_nodes = 0

    def close(self):
        if getattr(self, "h", None):
            lib().samu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc:
            raise SamuError(rc, lib().samu_last_error(self.h).decode())

    def samu_launch_count(self) -> int:
        return int(lib().samu_launch_count(self.h))

    def samu_share_stats(self) -> Dict[str, int]:
        out = (C.c_int64 * 3)()
        lib().samu_share_stats(self.h, out)
        return dict(group_items=int(out[0]), member_items=int(out[1]), fallbacks=int(out[2]))

    # ---- registration -------------------------------------------------------------------
    def samu_model_register(self, model_id: int, spec: Dict, bucket_B, coeff, load):
        sp = samu_model_spec(spec["L"], spec["h"], spec["c"], spec["l_max"], spec["tp_mask"], spec["weight_bytes"],
                             spec["kv_bytes_per_token"])
        b = np.ascontiguousarray(bucket_B, np.uint32)
        cf = np.ascontiguousarray(coeff, np.float64)
        ld = np.ascontiguousarray(load, np.float64)
        self._check(lib().samu_model_register(self.h, model_id, C.byref(sp), len(b), _np_ptr(b), _np_ptr(cf),
                                              _np_ptr(ld)))

    def samu_ecdf_load(self, model_id: int, values, cum):
        v = np.ascontiguousarray(values, np.uint32)
        c = np.ascontiguousarray(cum, np.uint32)
        self._check(lib().samu_ecdf_load(self.h, model_id, _np_ptr(v), _np_ptr(c), len(v)))

    def samu_app_load(self, engine: Dict, node_model, l_in_base, cap_y, pred, node, chain):
        e = samu_engine_cfg(engine["max_num_seqs"], engine["block_size"], engine["min_batched_tokens"],
                            engine["mem_util_permille"], engine["mem_bytes_per_gpu"], engine["kv_cap_bytes_per_gpu"],
                            engine["n_gpus"])
        nm = np.ascontiguousarray(node_model, np.int32)
        n = len(l_in_base)
        req = np.zeros(n, dtype=np.dtype([("l_in_base", "<u4"), ("cap_y", "<u4"), ("pred", "<i4"), ("node", "<i4"),
                                          ("chain", "<i4")]))
        req["l_in_base"], req["cap_y"], req["pred"], req["node"], req["chain"] = l_in_base, cap_y, pred, node, chain
        self._check(lib().samu_app_load(self.h, C.byref(e), len(nm), _np_ptr(nm), n, _np_ptr(req)))
        self.n_req, self.n_nodes = n, len(nm)

    def load_workload(self, w):
        """Register every model, eCDF and the application of a samu_workloads.Workload."""
        for m, spec in enumerate(w.models):
            self.samu_model_register(m, spec, w.coeff_B, w.coeff[m], w.load[m])
            self.samu_ecdf_load(m, w.ecdf_values[m], w.ecdf_cum[m])
        self.samu_app_load(w.engine, w.node_model, w.l_in_base, w.cap_y, w.pred, w.node, w.chain)

    def samu_enumerate_plans(self, node: int):
        n = lib().samu_enumerate_plans(self.h, node, None, None, 0)
        if n < 0:
            self._check(n)
        dp = np.zeros(max(n, 1), np.int32)
        tp = np.zeros(max(n, 1), np.int32)
        lib().samu_enumerate_plans(self.h, node, _np_ptr(dp), _np_ptr(tp), n)
        return list(zip(dp[:n].tolist(), tp[:n].tolist()))

    # ---- hot path -----------------------------------------------------------------------
    def samu_sample_lengths(self, seed: int, trial_begin: int, n_trials: int, out=None):
        torch = self.torch
        if out is None:
            lo = torch.empty((n_trials, self.n_req), dtype=torch.int16, device=self.device)
            li = torch.empty((n_trials, self.n_req), dtype=torch.int16, device=self.device)
        else:
            lo, li = out
        self._check(lib().samu_sample_lengths(self.h, seed, trial_begin, n_trials, _t_ptr(lo), _t_ptr(li)))
        return lo, li

    def samu_sample_requests(self, model_id: int, stream_id: int, l_in_base, cap_y, pred, index_base: int,
                             seed: int, trial_begin: int, n_trials: int):
        """One model's request set with its own Philox stream (include/samu.h); pred indexes the set."""
        torch = self.torch
        n = len(l_in_base)
        req = np.zeros(max(n, 1), dtype=np.dtype([("l_in_base", "<u4"), ("cap_y", "<u4"), ("pred", "<i4"),
                                                  ("node", "<i4"), ("chain", "<i4")]))
        req["l_in_base"][:n], req["cap_y"][:n], req["pred"][:n] = l_in_base, cap_y, pred
        lo = torch.empty((n_trials, n), dtype=torch.int16, device=self.device)
        li = torch.empty((n_trials, n), dtype=torch.int16, device=self.device)
        self._check(lib().samu_sample_requests(self.h, model_id, stream_id, _np_ptr(req), n, index_base, seed,
                                               trial_begin, n_trials, _t_ptr(lo), _t_ptr(li)))
        return lo, li

    def samu_known_lengths(self, l_true):
        """Known output lengths in place of the sampler: [1, n_req] device tensors."""
        torch = self.torch
        lt = np.ascontiguousarray(np.asarray(l_true, dtype=np.uint32).reshape(self.n_req))
        lo = torch.empty((1, self.n_req), dtype=torch.int16, device=self.device)
        li = torch.empty((1, self.n_req), dtype=torch.int16, device=self.device)
        self._check(lib().samu_known_lengths(self.h, lt.ctypes.data_as(C.c_void_p), _t_ptr(lo), _t_ptr(li)))
        return lo, li

    def fresh_state(self, n_trials: int):
        torch = self.torch
        return dict(st=torch.zeros((n_trials, self.n_req), dtype=torch.int32, device=self.device),
                    g=torch.zeros((n_trials, self.n_req), dtype=torch.int16, device=self.device),
                    fin_t=torch.full((n_trials, self.n_req), float("inf"), dtype=torch.float64, device=self.device),
                    over=torch.zeros((n_trials, self.n_nodes, 16), dtype=torch.float64, device=self.device))

    def samu_simulate_batch(self, cands: Sequence, l_out, l_in, state=None, time_limit=None, summary=False,
                            want_fin_iter=False, want_fin_t=False, out_recs=None):
        """cands: list of (node, dp, tp[, resume, dep_src, commit]).  Returns dict with device
        'recs' (uint8 [n_cands, T, 40]) and optional host 'summary', device fin arrays."""
        torch = self.torch
        nc = len(cands)
        T = int(l_out.shape[0])
        cs = (samu_candidate * max(nc, 1))()
        for i, cd in enumerate(cands):
            cd = tuple(cd) + (0, -1, 0)[len(cd) - 3:] if len(cd) < 6 else tuple(cd)
            cs[i] = samu_candidate(*[int(x) for x in cd[:6]])
        recs = out_recs if out_recs is not None else torch.empty((nc, T, 40), dtype=torch.uint8, device=self.device)
        summ = (samu_cand_summary * max(nc, 1))() if summary else None
        fi = torch.empty((nc, T, self.n_req), dtype=torch.int32, device=self.device) if want_fin_iter else None
        ft = torch.empty((nc, T, self.n_req), dtype=torch.float64, device=self.device) if want_fin_t else None
        s = state or {}
        tl = None
        if time_limit is not None:
            tl = torch.as_tensor(np.ascontiguousarray(time_limit, np.float64).reshape(nc, T), device=self.device)
        self._check(lib().samu_simulate_batch(
            self.h, C.cast(cs, C.c_void_p), nc, _t_ptr(l_out), _t_ptr(l_in), T, _t_ptr(s.get("st")),
            _t_ptr(s.get("g")), _t_ptr(s.get("fin_t")), _t_ptr(s.get("over")), _t_ptr(tl), _t_ptr(recs),
            None if summ is None else C.cast(summ, C.c_void_p), _t_ptr(fi), _t_ptr(ft)))
        out = dict(recs=recs, fin_iter=fi, fin_t=ft)
        if summary:
            out["summary"] = [dict(mean_t=x.mean_t, p50_t=x.p50_t, p90_t=x.p90_t, p99_t=x.p99_t,
                                   mean_flops=x.mean_flops, mean_req_iters=x.mean_req_iters) for x in summ[:nc]]
        return out

    def samu_plan_greedy(self, seed: int, n_trials: int, algo: str = "greedy", preemption: bool = True,
                         known_l_out=None):
        """algo: "greedy" (Algorithm 1), "max" / "min" (the paper's Max- / Min-heuristic);
        preemption=False / known_l_out are the §5.5 ablations (samu_plan_run)."""
        p = C.POINTER(samu_plan)()
        lt = None if known_l_out is None else np.ascontiguousarray(np.asarray(known_l_out, dtype=np.uint32))
        o = samu_plan_opts(ALGOS[algo], 1 if preemption else 0,
                           None if lt is None else lt.ctypes.data_as(C.c_void_p).value)
        self._check(lib().samu_plan_run(self.h, seed, n_trials, C.byref(o), C.byref(p)))
        try:
            P = p.contents
            stages = []
            for i in range(P.n_stages):
                s = P.stages[i]
                stages.append(dict(entries=[(s.node[j], s.dp[j], s.tp[j]) for j in range(s.n_entries)],
                                   fstar=s.fstar, mean_tE=s.mean_tE, T_E=s.T_E))
            return dict(stages=stages, total=P.total, n_cand_evals=P.n_cand_evals, n_sims=P.n_sims)
        finally:
            lib().samu_plan_free(p)

    def samu_replay_plan(self, plan: dict, seed: int, known_l_out=None):
        """Replay a plan (dict from samu_plan_greedy) against true lengths with the dynamic
        scheduler: known_l_out [n_req], or trial 0 of the sampler with `seed`."""
        P = samu_plan()
        P.n_stages = len(plan["stages"])
        for i, st in enumerate(plan["stages"]):
            S = P.stages[i]
            S.n_entries = len(st["entries"])
            for j, (v, d, t) in enumerate(st["entries"]):
                S.node[j], S.dp[j], S.tp[j] = v, d, t
            S.fstar, S.mean_tE, S.T_E = st["fstar"], st["mean_tE"], st["T_E"]
        P.total = plan["total"]
        lt = None if known_l_out is None else np.ascontiguousarray(np.asarray(known_l_out, dtype=np.uint32))
        out = samu_replay()
        self._check(lib().samu_replay_plan(self.h, C.byref(P), seed, _np_ptr(lt), C.byref(out)))
        stages = []
        for i in range(out.n_stages):
            st = out.stages[i]
            k = st.n_entries
            stages.append(dict(entries=[(st.node[j], st.dp[j], st.tp[j]) for j in range(k)],
                               gpu_mask=list(st.gpu_mask[:k]), resumed=list(st.resumed[:k]),
                               planned_stage=st.planned_stage, first_finisher=st.first_finisher,
                               idle_gpus=st.idle_gpus, t_start=st.t_start, duration=st.duration))
        return dict(stages=stages, total=out.total, planned_total=out.planned_total,
                    idle_gpu_seconds=out.idle_gpu_seconds, n_kept_last=out.n_kept_last,
                    n_kept_room=out.n_kept_room, n_stopped=out.n_stopped)

    def samu_fit_coeffs(self, off, x, y, trim_permille: int = 10):
        """Per-bucket least-squares cost coefficients with noise-point trimming.
        off [nb + 1] / x / y: host arrays or device tensors.  Returns numpy (a, b, n_used, flags)."""
        torch = self.torch

        def dev(v, dt):
            if isinstance(v, torch.Tensor):
                return v.to(device=self.device, dtype=dt).contiguous()
            return torch.as_tensor(np.asarray(v), dtype=dt).to(self.device)

        o, xd, yd = dev(off, torch.int64), dev(x, torch.float64), dev(y, torch.float64)
        nb = o.numel() - 1
        a = torch.zeros(nb, dtype=torch.float64, device=self.device)
        b = torch.zeros_like(a)
        nu = torch.zeros(nb, dtype=torch.int32, device=self.device)
        fl = torch.zeros_like(nu)
        self._check(lib().samu_fit_coeffs(self.h, nb, _t_ptr(o), _t_ptr(xd), _t_ptr(yd), trim_permille, _t_ptr(a),
                                          _t_ptr(b), _t_ptr(nu), _t_ptr(fl)))
        return a.cpu().numpy(), b.cpu().numpy(), nu.cpu().numpy(), fl.cpu().numpy()


def coeff_table(bucket, a, b, n_buckets_B: int) -> np.ndarray:
    """Fitted (a, b) per (slot, phase, B index) bucket -> the [5][3][2][nb] table
    samu_model_register takes (tp slots without samples stay 0)."""
    out = np.zeros((N_TP_SLOTS, 3, 2, n_buckets_B), dtype=np.float64)
    for k, (slot, ph, bi) in enumerate(bucket):
        out[slot, ph, 0, bi] = a[k]
        out[slot, ph, 1, bi] = b[k]
    return out


def recs_to_numpy(recs) -> np.ndarray:
    """Device uint8 [..., 40] records -> numpy structured array (REC_DTYPE)."""
    a = recs.detach().cpu().numpy()
    return a.reshape(-1).view(REC_DTYPE).reshape(a.shape[:-1])


def rec_flops(rec) -> np.ndarray:
    return np.array([(int(h) << 64) | int(l) for h, l in zip(np.ravel(rec["flops_hi"]), np.ravel(rec["flops_lo"]))],
                    dtype=object).reshape(np.shape(rec))
