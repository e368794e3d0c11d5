"""Hand-built tiny workloads for pins and parity cases (inputs only — no method arithmetic).

Output lengths are forced through the cap: with a point-mass eCDF at 60000 the sampler's
l_out = min(X, y, l_max - l_in) equals y whenever y <= l_max - l_in.
"""
import numpy as np

import samu_workloads as W

NB = 9  # coeff buckets 1, 2, 4, ..., 256


def spec(L=1, h=8, c=10, l_max=4096, tp_values=(1,), weight_bytes=1, kv_bytes_per_token=1):
    mask = 0
    for t in tp_values:
        mask |= 1 << int(np.log2(t))
    return dict(arch="tiny", L=L, h=h, c=c, l_max=l_max, tp_mask=mask, weight_bytes=weight_bytes,
                kv_bytes_per_token=kv_bytes_per_token)


def coeff(kind="const", value=1.0):
    """[5][3][2][9] coefficient buckets.  const: lat = value; B: lat = B; S: lat = S."""
    cf = np.zeros((W.N_TP_SLOTS, 3, 2, NB))
    Bv = np.array([1, 2, 4, 8, 16, 32, 64, 128, 256], dtype=np.float64)
    if kind == "const":
        cf[:, 0, 1, :] = value
    elif kind == "B":
        cf[:, 0, 1, :] = Bv
    elif kind == "S":
        cf[:, 2, 0, :] = 1.0
    elif kind == "flops":
        cf[:, 0, 0, :] = value
    else:
        raise ValueError(kind)
    return cf


def zero_load():
    return np.zeros((W.N_TP_SLOTS, W.MAX_DP))


def engine(max_num_seqs=256, block_size=16, min_batched_tokens=2048, kv_cap=10 ** 15, n_gpus=1,
           mem=10 ** 15):
    return dict(max_num_seqs=max_num_seqs, block_size=block_size, min_batched_tokens=min_batched_tokens,
                mem_util_permille=1000, mem_bytes_per_gpu=mem, kv_cap_bytes_per_gpu=kv_cap, n_gpus=n_gpus)


def tiny(l_in, l_out, eng=None, sp=None, cf="const", load=None, pred=None, chain=None, n_trials=1):
    """One node, requests with forced output lengths."""
    sp = sp or spec()
    cfa = coeff(cf) if isinstance(cf, str) else cf
    return W.custom_workload(
        [sp], [dict(l_in=l_in, cap=l_out, pred=pred, chain=chain)], n_trials=n_trials,
        engine=eng or engine(), ecdfs=[(np.array([60000]), np.array([1]))], coeff=[cfa],
        load=[load if load is not None else zero_load()])


def multi(node_specs, eng=None, n_trials=1):
    """Several nodes.  node_specs: list of dict(sp=..., l_in=..., l_out=..., cf=..., load=...,
    pred=..., chain=..., ecdf=(values, cum) or None)."""
    sps, reqs, ecdfs, cfs, loads = [], [], [], [], []
    for ns in node_specs:
        sps.append(ns.get("sp") or spec())
        reqs.append(dict(l_in=ns["l_in"], cap=ns["l_out"], pred=ns.get("pred"), chain=ns.get("chain")))
        ecdfs.append(ns.get("ecdf") or (np.array([60000]), np.array([1])))
        c = ns.get("cf", "const")
        cfs.append(coeff(c) if isinstance(c, str) else c)
        loads.append(ns.get("load") if ns.get("load") is not None else zero_load())
    return W.custom_workload(sps, reqs, n_trials=n_trials, engine=eng or engine(), ecdfs=ecdfs,
                             coeff=cfs, load=loads)


def fig1():
    """S:645 (the paper's Fig. 1 shape): 4 GPUs, 6 models, one sequence per replica, 1 s per
    iteration, no load cost; model 0 has 8 one-token requests, models 1-5 three each (23
    GPU-seconds of work, so no schedule beats 5.75 s)."""
    sp = spec(tp_values=(1,))
    nodes = [dict(l_in=[4] * 8, l_out=[1] * 8, sp=sp)] + [dict(l_in=[4] * 3, l_out=[1] * 3, sp=sp)
                                                           for _ in range(5)]
    return multi(nodes, eng=engine(n_gpus=4, max_num_seqs=1))


def even_split_4x8():
    """P:743's Min-heuristic example: 8 GPUs, 4 models, model 0 the smallest."""
    sp = spec(tp_values=(1, 2))
    nodes = [dict(l_in=[4] * n, l_out=[3] * n, sp=sp) for n in (40, 400, 400, 400)]
    return multi(nodes, eng=engine(n_gpus=8, max_num_seqs=16))


def reload_fixture(coeff_kind="const"):
    """Carried state cut mid-decode, then reloaded under another plan (S:406, P:494-496,
    reading c18).  One node with tp in {1, 2}, block size 4, KV 20 tokens per GPU (5 blocks at
    tp = 1, 10 at tp = 2), 2 slots, token budget 16 (l_max 16), 2 planned GPUs; requests
    A (l_in 4, l_out 7), B (l_in 4, l_out 8) and C (l_in 4, l_out 2); loading (dp 1, tp 2) costs 10 s, everything
    else 0.  The hand traces are in tests/test_oracle_state_pins.py."""
    sp = spec(l_max=16, tp_values=(1, 2))
    load = zero_load()
    load[1, 0] = 10.0
    return tiny([4, 4, 4], [7, 8, 2], sp=sp, cf=coeff_kind, load=load,
                eng=engine(block_size=4, kv_cap=20, min_batched_tokens=1, max_num_seqs=2, n_gpus=2))


def chatglm_fixture():
    """AC6 ("it takes 48s to run chatglm3-6b on 1 GPU and 32s on 8 GPUs"): model 0
    completes 1000 one-token requests in 48 simulated seconds at (dp 1, tp 1) (21 slots: 48
    prefill iterations of 1 s) and in 32 s at (1, 8) (2/3 s per iteration); its dp > 1 plans
    pay a 100 s load.  Model 1 has the same requests and scales linearly with dp (125
    requests per replica at dp 8: 6 iterations), tp 1 only.  8 planned GPUs.  Per-layer weights
    c = 10^6 >> h s, so stage throughput (FLOPs / time) follows the run times."""
    sp0 = spec(c=10 ** 6, tp_values=(1, 8))     # FLOPs dominated by the linear layers (c >> h s)
    sp1 = spec(c=10 ** 6, tp_values=(1,))
    cf0 = np.zeros((W.N_TP_SLOTS, 3, 2, NB))
    cf0[0, 0, 1, :] = 1.0
    cf0[3, 0, 1, :] = 2.0 / 3.0
    load0 = zero_load()
    load0[:, 1:] = 100.0
    nodes = [dict(l_in=[4] * 1000, l_out=[1] * 1000, sp=sp0, cf=cf0, load=load0),
             dict(l_in=[4] * 1000, l_out=[1] * 1000, sp=sp1, cf="const")]
    return multi(nodes, eng=engine(n_gpus=8, max_num_seqs=21))
