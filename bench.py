#!/usr/bin/env python
"""Benchmark of the sampling-then-simulation estimator (one JSON line on rank 0).

A step = one pass of the whole estimator hot path over one batch: sample every request's output
length for every trial (K1), simulate every (model, plan) candidate of the first greedy inner
step over every trial (K2, combine) and reduce to per-candidate mean / percentiles (K3,
all-gathered over ranks).  Trials are sharded in contiguous blocks over ranks (strong scaling:
the workload's trial count is the job total).  Metric: simulated candidate-trials/s (BASELINE.json).

  python bench.py [--gpus N --steps K --warmup W] [--workload c5] [--impl samu|reference]
  torchrun --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import samu_workloads as W  # noqa: E402

MEASURED = os.path.join(ROOT, "MEASURED_PEAKS.json")
# K2 roofline: the method's arithmetic per simulated iteration is the per-iteration
# latency model of the contract (c24): 3 fused multiply-adds + 2 adds + the clock add = 9 fp64
# flops.  Peak: 148 SMs x 64 fp64 FMA lanes x 2 flops x clock (37.2 TFLOP/s at 1965 MHz, the
# nominal B200 FP64 rate).  Design-independent: a kernel that spends its time elsewhere (event
# control, redundant lanes) shows a low fraction.
FP64_FLOPS_PER_ITER = 9
FP64_LANES_PER_SM = 64
N_SM = 148


def trial_share(T, world, rank):
    """This rank's contiguous trial block from libsamu's own sharding rule (samu_shard_plan, the
    split its sharded samu_simulate_batch checks): the bench configs have T >= world, i.e. pure
    trial sharding (every rank simulates every candidate)."""
    from paper_2503_16893_b200 import samu_shard_plan
    p = samu_shard_plan(T, world, rank)
    assert p["job_classes"] == 1, "bench configs shard trials only (T >= world)"
    return p["trial_begin"], p["trial_count"]


def first_step_candidates(nodes_ready, plans_of):
    return [(v, dp, tp) for v in nodes_ready for (dp, tp) in plans_of(v)]


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def peaks():
    try:
        return json.load(open(MEASURED))
    except Exception:
        return {}


def ncu_summary(workload):
    """The committed ncu --set full summary of K2 (profiles/ncu_k2_summary.json), if it matches."""
    p = os.path.join(ROOT, "profiles", "ncu_k2_summary.json")
    try:
        d = json.load(open(p))
        if d.get("workload") == workload:
            return d
    except Exception:
        pass
    return {}


# ------------------------------------------------------------------------------------------
# CPU oracle timing (cpu_baseline leg and --impl reference): the oracle as it stands
# ------------------------------------------------------------------------------------------
def time_oracle(w, cands, target_s=12.0, max_trials=None):
    import oracle as O
    P = O.Problem(w)
    threads = os.cpu_count() or 1
    # grow the trial sample until it costs ~target_s seconds of wall time on all host cores
    n = 1
    while True:
        lo, li = P.sample(w.seed, 0, n)
        t0 = time.perf_counter()
        rec = P.simulate_many(cands, lo, li, threads)
        dt = time.perf_counter() - t0
        if dt >= target_s or (max_trials and n >= max_trials) or n >= w.n_trials:
            break
        n = min(w.n_trials, max(n + 1, int(n * min(8.0, 1.2 * target_s / max(dt, 1e-3)))))
        if max_trials:
            n = min(n, max_trials)
    ct = len(cands) * n
    reqit = int(rec["req_iters"].astype(np.float64).sum())
    return dict(value=ct / dt, unit="candidate-trials/s", cores=threads, kind="oracle",
                sample=f"{len(cands)} candidates x trials 0..{n - 1} of {w.name} ({ct} candidate-trials, "
                       f"{reqit:.3e} request-iterations) in {dt:.2f} s",
                req_iters_per_s=reqit / dt, seconds=dt, n_trials=n)


def run_reference(args, w, rank):
    """--impl reference: the CPU oracle timed on this box's host cores (rank 0 only)."""
    if rank != 0:
        return
    import oracle as O
    P = O.Problem(w)
    ready = [v for v in range(w.n_nodes) if not np.any((w.pred[w.node == v] >= 0) &
                                                      (w.node[np.maximum(w.pred[w.node == v], 0)] != v))]
    cands = first_step_candidates(ready, lambda v: P.plans(int(w.node_model[v])))
    # one step = the same candidates over a bounded trial sample sized for ~3 s per step
    cal = time_oracle(w, cands, target_s=3.0)
    n = cal["n_trials"]
    lo, li = P.sample(w.seed, 0, n)
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        P.simulate_many(cands, lo, li, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        P.simulate_many(cands, lo, li, threads)
    dt = (time.perf_counter() - t0) / args.steps
    v = len(cands) * n / dt
    out = {"impl": "reference", "metric": "simulated candidate-trials/s", "value": v, "unit": "candidate-trials/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": w.name, "trials_per_step": n, "candidates": len(cands), "requests": w.n_req,
                      "parallelism": f"oracle threads={threads}"},
           "cpu_baseline": {"value": v, "unit": "candidate-trials/s", "cores": threads, "kind": "oracle",
                            "sample": f"{len(cands)} candidates x {n} trials of {w.name} per step"},
           "e2e": {"value": v, "unit": "candidate-trials/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ------------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="samu", choices=["samu", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--trials", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--per-config", default="c2,c3,c4",
                    help="other BASELINE configs measured in the same run (value, ms_per_step, roofline, "
                         "cpu_baseline per config); '' = off")
    ap.add_argument("--planner-trials", type=int, default=-1,
                    help="also time one full Algorithm 1 run (samu_plan_greedy, rows a1-a12) at this trial count "
                         "(default: the workload's trials; 0 = off)")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    w = W.make_workload(args.workload, n_trials=args.trials)
    if args.impl == "reference":
        run_reference(args, w, rank)
        return

    import torch
    import torch.distributed as dist
    from paper_2503_16893_b200 import Samu, recs_to_numpy, samu_nccl_unique_id

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [samu_nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    else:
        nccl_id = None
    S = Samu(local, rank, world, nccl_id)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=torch.device("cuda", local))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.item()

    def sum_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=torch.device("cuda", local))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return t.item()

    def measure_config(wc, steps, warmup):
        """The bench step on another workload: sample + simulate the first greedy step's candidates
        over the rank's trial share + summaries; device time (CUDA events), max over ranks."""
        S.load_workload(wc)
        Tc = wc.n_trials
        tbc, Tlc = trial_share(Tc, world, rank)
        rdy = [v for v in range(wc.n_nodes) if not np.any((wc.pred[wc.node == v] >= 0) &
                                                          (wc.node[np.maximum(wc.pred[wc.node == v], 0)] != v))]
        cc = first_step_candidates(rdy, S.samu_enumerate_plans)
        dv = torch.device("cuda", local)
        lo_c = torch.empty((Tlc, wc.n_req), dtype=torch.int16, device=dv)
        li_c = torch.empty((Tlc, wc.n_req), dtype=torch.int16, device=dv)
        rc = torch.empty((len(cc), Tlc, 40), dtype=torch.uint8, device=dv)

        def st():
            S.samu_sample_lengths(wc.seed, tbc, Tlc, out=(lo_c, li_c))
            return S.samu_simulate_batch(cc, lo_c, li_c, summary=True, out_recs=rc)

        for _ in range(max(3, warmup)):
            st()
        barrier()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(steps):
            st()
        a1.record()
        barrier()
        msc = max_over_ranks(a0.elapsed_time(a1) / steps)
        gc = recs_to_numpy(rc)
        it_c = sum_over_ranks(float(gc["iters"].astype(np.float64).sum()))
        ri_c = sum_over_ranks(float(gc["req_iters"].astype(np.float64).sum()))
        return dict(workload=wc.name, trials=Tc, candidates=len(cc), requests=wc.n_req, ms_per_step=msc,
                    value=len(cc) * Tc / (msc / 1e3), unit="candidate-trials/s", sim_iters=it_c, req_iters=ri_c,
                    cands=cc)

    S.load_workload(w)
    T = w.n_trials
    tb, Tl = trial_share(T, world, rank)
    ready = [v for v in range(w.n_nodes) if not np.any((w.pred[w.node == v] >= 0) &
                                                      (w.node[np.maximum(w.pred[w.node == v], 0)] != v))]
    cands = first_step_candidates(ready, S.samu_enumerate_plans)
    nc = len(cands)
    dev = torch.device("cuda", local)
    lo = torch.empty((Tl, w.n_req), dtype=torch.int16, device=dev)
    li = torch.empty((Tl, w.n_req), dtype=torch.int16, device=dev)
    recs = torch.empty((nc, Tl, 40), dtype=torch.uint8, device=dev)

    def step():
        S.samu_sample_lengths(w.seed, tb, Tl, out=(lo, li))
        return S.samu_simulate_batch(cands, lo, li, summary=True, out_recs=recs)

    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    l0 = S.samu_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local) as clk:
        barrier()
        e0.record()
        for _ in range(args.steps):
            out = step()
        e1.record()
        barrier()
    launches = S.samu_launch_count() - l0
    ms = e0.elapsed_time(e1) / args.steps
    # K2 (+ its replica combine) launch duration, timed on the launching stream
    k0, k1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    k0.record()
    for _ in range(args.steps):
        S.samu_simulate_batch(cands, lo, li, out_recs=recs)
    k1.record()
    torch.cuda.synchronize()
    k2_ms = k0.elapsed_time(k1) / args.steps
    g = recs_to_numpy(recs)
    loc = torch.tensor([ms, k2_ms, float(g["iters"].astype(np.float64).sum()), float(g["req_iters"].astype(np.float64).sum())],
                       dtype=torch.float64, device=dev)
    if world > 1:
        mx = loc[:2].clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = loc[2:].clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        ms, k2_ms = mx.tolist()
        iters, reqit = sm.tolist()
    else:
        iters, reqit = loc[2].item(), loc[3].item()

    # end to end through the C ABI with host buffers: app tables host->device, results to host
    barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        S.load_workload(w)
        o = step()
        torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / args.steps
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()
    h2d = w.n_req * 20 + w.n_nodes * 4 + sum(len(w.coeff_B) * 4 + w.coeff[m].nbytes + w.load[m].nbytes +
                                             w.ecdf_values[m].nbytes + w.ecdf_cum[m].nbytes for m in range(len(w.models)))
    d2h = nc * 48

    # the whole planner (Algorithm 1: every greedy inner step incl. truncated sims, stage scoring
    # and argmax, row a12) once, wall time around the call (synchronising), max over ranks
    planner = None
    if args.planner_trials != 0:
        Tp = T if args.planner_trials < 0 else min(args.planner_trials, T)
        S.samu_plan_greedy(w.seed, Tp)   # warm-up: the planner's buffers are kept by the context (steady state)
        barrier()
        t0 = time.perf_counter()
        plan = S.samu_plan_greedy(w.seed, Tp)
        torch.cuda.synchronize()
        plan_s = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([plan_s], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            plan_s = t.item()
        planner = {"algorithm": "greedy (Algorithm 1, P:542-574)", "workload": w.name, "trials": Tp,
                   "seconds": plan_s, "stages": len(plan["stages"]), "candidate_evaluations": plan["n_cand_evals"],
                   "candidate_trial_sims": plan["n_sims"], "candidate_trial_sims_per_s": plan["n_sims"] / plan_s,
                   "planned_total_s": plan["total"]}

    # the other BASELINE configs (C2 ensembling, C3 routing, C4 chain summary; 64 trials each), same
    # step, measured after the headline region (north star: throughput per paper-shaped workload)
    per_config = []
    for name in [x for x in args.per_config.split(",") if x and x != w.name]:
        per_config.append(measure_config(W.make_workload(name), max(3, args.steps), max(3, args.warmup)))

    if rank == 0:
        pk = peaks()
        clock = clk.summary()
        sm_hz = (clock.get("sm_max_mhz") or pk.get("sm_max_mhz") or 1965.0) * 1e6
        peak = N_SM * FP64_LANES_PER_SM * 2 * sm_hz
        iters_per_launch = iters / world          # per rank launch (strong scaling: each rank its share)
        achieved = FP64_FLOPS_PER_ITER * iters_per_launch / (k2_ms / 1e3)
        value = nc * T / (ms / 1e3)
        ncu = ncu_summary(w.name)
        hbm_peak = pk.get("hbm_gbs", 6454.0) * 1e9
        dram = ncu.get("dram_bytes_per_launch")
        ncu_ms = ncu.get("gpu_time_ms")
        line = {
            "metric": "simulated candidate-trials/s", "value": value, "unit": "candidate-trials/s",
            "n_gpus": world, "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w.name, "trials": T, "candidates": nc, "requests": w.n_req,
                       "parallelism": f"trials sharded dp{world}",
                       "l2": f"inputs larger than L2: lengths {2 * 2 * T * w.n_req / 1e6:.0f} MB re-sampled every step"},
            "req_iters_per_s": reqit / (ms / 1e3), "sim_iters_per_s": iters / (ms / 1e3),
            "roofline": {"bound": "alu", "kernel": "k_simulate (K2: one launch per mode, FRESH + LEAN at C5)",
                         "achieved": achieved / 1e12, "peak": peak / 1e12,
                         "unit": "TFLOP/s", "frac": achieved / peak,
                         "traffic": ncu_summary(w.name).get("dram_bytes_per_launch"),
                         # context (from the committed ncu capture, not this run): the resource
                         # that binds K2 is the warp-instruction issue rate, not fp64 or HBM
                         "ncu_issue_slots_active_pct": ncu.get("issue_active_pct"),
                         "ncu_fp64_pipe_pct": ncu.get("fp64_pipe_pct"),
                         "ncu_warps_active_pct": ncu.get("warps_active_pct"),
                         # HBM side (BASELINE's "HBM roofline %"): measured DRAM bytes of K2 (ncu, per
                         # launch set) over this run's K2 time, against the measured copy bandwidth
                         "hbm_gbs": (dram / (k2_ms / 1e3) / 1e9) if dram else None,
                         "hbm_frac": (dram / (k2_ms / 1e3) / hbm_peak) if dram else None,
                         "hbm_peak_gbs": hbm_peak / 1e9, "hbm_peak_source": "MEASURED_PEAKS.json hbm_gbs",
                         "ncu_gpu_time_ms": ncu_ms,
                         "ncu_source": "profiles/ncu_k2_summary.json",
                         "peak_derived": True,
                         "peak_source": "fp64: 148 SM x 64 FMA lanes x 2 x sm clock (derived from unit counts and the "
                                        "measured max clock; MEASURED_PEAKS.json has no fp64 entry; DESIGN.md section 6)",
                         "work_per_unit": "9 fp64 flops per simulated iteration (latency model, reading c24)",
                         "sim_iters_per_launch": iters_per_launch, "k2_ms_per_launch": k2_ms},
            "e2e": {"value": nc * T / e2e_s, "unit": "candidate-trials/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(launches), "clocks": clock,
        }
        if planner:
            line["planner"] = planner
        keep = ("value", "unit", "cores", "kind", "sample", "req_iters_per_s")
        if not args.no_cpu_baseline:   # rank 0 at every world size (the other ranks wait)
            line["cpu_baseline"] = {k: v for k, v in time_oracle(w, cands, args.cpu_seconds).items() if k in keep}
        if per_config:
            line["per_config"] = []
            for pc in per_config:
                wc = W.make_workload(pc["workload"])
                k_ach = FP64_FLOPS_PER_ITER * (pc["sim_iters"] / world) / (pc["ms_per_step"] / 1e3)
                d = {k: pc[k] for k in ("workload", "trials", "candidates", "requests", "value", "unit", "ms_per_step")}
                d["req_iters_per_s"] = pc["req_iters"] / (pc["ms_per_step"] / 1e3)
                d["roofline"] = {"bound": "alu", "achieved": k_ach / 1e12, "peak": peak / 1e12, "unit": "TFLOP/s",
                                 "frac": k_ach / peak, "peak_derived": True,
                                 "note": "whole step time (K1 + K2 + K3) as the launch duration"}
                if not args.no_cpu_baseline:
                    d["cpu_baseline"] = {k: v for k, v in time_oracle(wc, pc["cands"], args.cpu_seconds / 3).items()
                                         if k in keep}
                line["per_config"].append(d)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
