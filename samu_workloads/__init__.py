"""Seeded synthetic workload generator shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic (no sampling, no FLOPs, no latency model,
no plan validity, no KV-block accounting).  It only draws the *inputs* the method consumes,
with the shapes and distributions of the paper's workloads (recipe in DESIGN.md §4):

* model specs (Llama-shaped L, h, c, l_max, weight/KV bytes)        -- P:301-307 symbols
* one empirical output-length CDF per model (K knots, n = 10,000)   -- P:241-249
* per-(model, tp) per-batch-size coefficient buckets a[B], b[B]      -- P:480-489
* a model-loading cost table per (model, dp, tp), 11-47 s            -- P:313-314
* the application graph's requests: ensembling, routing (Table 1, P:775-786,
  P:848-850), chain summary with a fused self-loop + evaluator.

Every array is a plain numpy array; both sides (oracle/ and the CUDA path) marshal them
independently.  Workload seed 2503, sampling seed 16893.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional

import numpy as np
from scipy.special import ndtri

WORKLOAD_SEED = 2503
SAMPLING_SEED = 16893

N_TP_SLOTS = 5      # tp in {1, 2, 4, 8, 16}
MAX_DP = 16
N_PHASES = 3        # comp, prep, samp

GB = 10 ** 9


@dataclasses.dataclass
class Workload:
    name: str
    n_trials: int
    engine: Dict[str, int]
    models: List[Dict[str, int]]          # one per model id
    coeff_B: np.ndarray                   # uint32 [nb] bucket batch sizes
    coeff: List[np.ndarray]               # per model float64 [N_TP_SLOTS][3][2][nb]  (a, b)
    load: List[np.ndarray]                # per model float64 [N_TP_SLOTS][MAX_DP]
    ecdf_values: List[np.ndarray]         # per model uint32 [K] strictly increasing
    ecdf_cum: List[np.ndarray]            # per model uint32 [K] strictly increasing, last = n
    node_model: np.ndarray                # int32 [n_nodes]
    l_in_base: np.ndarray                 # uint32 [n_req]
    cap_y: np.ndarray                     # uint32 [n_req]
    pred: np.ndarray                      # int32 [n_req]  -1 or an earlier request index
    node: np.ndarray                      # int32 [n_req]  requests grouped by node, ascending
    chain: np.ndarray                     # int32 [n_req]  -1 or chain id (dp key) within node
    seed: int = SAMPLING_SEED
    description: str = ""

    @property
    def n_req(self) -> int:
        return int(self.l_in_base.shape[0])

    @property
    def n_nodes(self) -> int:
        return int(self.node_model.shape[0])

    def node_range(self, n: int):
        idx = np.nonzero(self.node == n)[0]
        return (int(idx[0]), int(idx[-1]) + 1) if idx.size else (0, 0)


# ---------------------------------------------------------------------------------------------
# Model architectures (Llama-shaped; c = sum of per-layer matmul weight elements)
# ---------------------------------------------------------------------------------------------
_ARCH = {
    #            L   h     ffn    n_kv  l_max
    "llama7b":  (32, 4096, 11008, 32, 4096),
    "llama13b": (40, 5120, 13824, 40, 4096),
    "llama34b": (48, 8192, 22016, 8, 16384),
    "llama70b": (80, 8192, 28672, 8, 4096),
    "mistral7b": (32, 4096, 14336, 8, 32768),
}
_VOCAB = 32000
_HEAD_DIM = 128


def arch_spec(arch: str, tp_values=(1, 2, 4, 8)) -> Dict[str, int]:
    L, h, ffn, n_kv, l_max = _ARCH[arch]
    kv_dim = n_kv * _HEAD_DIM
    c = 2 * h * h + 2 * h * kv_dim + 3 * h * ffn           # q,o + k,v + gate/up/down
    weight_bytes = 2 * (L * c + 2 * _VOCAB * h)             # bf16 weights incl. embeddings
    kv_bytes_per_token = 2 * L * kv_dim * 2                 # K and V, all layers, bf16
    tp_mask = 0
    for tp in tp_values:
        tp_mask |= 1 << int(np.log2(tp))
    return dict(arch=arch, L=L, h=h, c=int(c), l_max=l_max, tp_mask=tp_mask,
                weight_bytes=int(weight_bytes), kv_bytes_per_token=int(kv_bytes_per_token))


def default_engine(n_gpus: int = 8) -> Dict[str, int]:
    # §8(c) c5/c6 defaults: 256 seqs, 16-token blocks, token budget max(l_max, 2048),
    # 180 GB planned GPUs at 90 % utilisation, "40-GB KV budget" read as 40e9 bytes per GPU.
    return dict(max_num_seqs=256, block_size=16, min_batched_tokens=2048,
                mem_util_permille=900, mem_bytes_per_gpu=180 * GB,
                kv_cap_bytes_per_gpu=40 * GB, n_gpus=n_gpus)


# ---------------------------------------------------------------------------------------------
# Input distributions
# ---------------------------------------------------------------------------------------------
def make_ecdf(rng: np.random.Generator, mean: float, sigma: float, K: int = 1000,
              n: int = 10000):
    """K strictly increasing integer knots on a lognormal quantile grid, multinomial counts
    (each >= 1) summing to n.  Returns (values, cum) as uint32."""
    mu = np.log(mean) - 0.5 * sigma * sigma
    q = np.exp(mu + sigma * ndtri((np.arange(K) + 0.5) / K))
    v = np.maximum(np.rint(q), 1).astype(np.int64)
    for j in range(1, K):
        if v[j] <= v[j - 1]:
            v[j] = v[j - 1] + 1
    counts = 1 + rng.multinomial(n - K, np.full(K, 1.0 / K))
    cum = np.cumsum(counts)
    assert cum[-1] == n
    return v.astype(np.uint32), cum.astype(np.uint32)


def make_coeff(rng: np.random.Generator, spec: Dict[str, int], coeff_B: np.ndarray):
    """Positive per-bucket (a, b) for comp / prep / samp, per tp slot (zeros for tp not allowed).
    Magnitudes: a weight-streaming floor b_comp ~ weights / (6 TB/s * tp^0.9) plus a compute
    slope a_comp ~ 1 / (1.2 PFLOP/s * eff(B) * tp^0.9); small prep/samp terms."""
    nb = coeff_B.shape[0]
    out = np.zeros((N_TP_SLOTS, N_PHASES, 2, nb), dtype=np.float64)
    for slot in range(N_TP_SLOTS):
        if not (spec["tp_mask"] >> slot) & 1:
            continue
        tp = 1 << slot
        B = coeff_B.astype(np.float64)
        jit = lambda: 1.0 + 0.05 * rng.uniform(-1, 1, size=nb)
        eff = B / (B + 24.0)
        out[slot, 0, 0] = jit() / (1.2e15 * eff * tp ** 0.9)
        out[slot, 0, 1] = jit() * spec["weight_bytes"] / (6.0e12 * tp ** 0.9)
        out[slot, 1, 0] = jit() * 4.0e-9
        out[slot, 1, 1] = jit() * (3.0e-4 + 2.0e-6 * B)
        out[slot, 2, 0] = jit() * 1.0e-9
        out[slot, 2, 1] = jit() * (2.0e-4 + 4.0e-6 * B)
    return out


def make_profile(w: "Workload", model: int, n_per_bucket: int = 200, noise: float = 0.002,
                 outlier_frac: float = 0.005, seed: int = WORKLOAD_SEED):
    """Synthetic per-iteration profile of one model (the input of the coefficient fit):
    for every allowed tp slot, phase and profiled batch size B, n_per_bucket iterations with x
    spread over the phase's range (FLOPs of B sequences of 16..2048 context tokens; B*s with
    s in 1..2048; S in 16B..4096B), latency = the workload's (a, b) line x (1 + noise N(0,1)),
    and a fraction of 'noise points' (Fig. 5) slowed 2-5x.  Buckets are laid out
    (slot, phase, B index) in that order; returns dict(off, x, y, bucket) with bucket
    (slot, phase, bi) per bucket row."""
    rng = np.random.default_rng([seed, model, 489])
    spec = w.models[model]
    cf = w.coeff[model]
    xs, ys, off, bucket = [], [], [0], []
    for slot in range(N_TP_SLOTS):
        if not (spec["tp_mask"] >> slot) & 1:
            continue
        tp = 1 << slot
        for ph in range(N_PHASES):
            for bi, B in enumerate(w.coeff_B.astype(np.float64)):
                if ph == 0:
                    ctx = rng.uniform(16, 2048, n_per_bucket) * B
                    x = spec["L"] * (spec["c"] * B + 2.0 * spec["h"] * ctx / tp)
                elif ph == 1:
                    x = B * rng.integers(1, 2049, n_per_bucket).astype(np.float64)
                else:
                    x = rng.uniform(16 * B, 4096 * B, n_per_bucket)
                a, b = cf[slot, ph, 0, bi], cf[slot, ph, 1, bi]
                y = (a * x + b) * (1.0 + noise * rng.standard_normal(n_per_bucket))
                out = rng.random(n_per_bucket) < outlier_frac
                y[out] *= rng.uniform(2.0, 5.0, int(out.sum()))
                xs.append(x)
                ys.append(y)
                off.append(off[-1] + n_per_bucket)
                bucket.append((slot, ph, bi))
    return dict(off=np.array(off, np.int64), x=np.concatenate(xs), y=np.concatenate(ys), bucket=bucket)


def make_load(rng: np.random.Generator, spec: Dict[str, int]):
    """Loading cost table in seconds, 11-47 s, per (tp slot, dp)."""
    out = np.zeros((N_TP_SLOTS, MAX_DP), dtype=np.float64)
    base = 11.0 + 30.0 * spec["weight_bytes"] / (140 * GB)
    for slot in range(N_TP_SLOTS):
        tp = 1 << slot
        for dp in range(1, MAX_DP + 1):
            t = 11.0 + (base - 11.0) / np.sqrt(tp) + 0.8 * np.sqrt(dp - 1) + (2.0 if tp > 1 else 0.0)
            out[slot, dp - 1] = min(47.0, t * (1.0 + 0.02 * rng.uniform(-1, 1)))
    return out


def mixinstruct_lin(rng, n):
    """MixInstruct-like prompt lengths: 5..127, mean ~21."""
    x = np.exp(np.log(17.0) + 0.6 * rng.standard_normal(n))
    return np.clip(np.rint(x), 5, 127).astype(np.uint32)


def routerbench_lin(rng, n):
    """RouterBench-like prompt lengths: 9..577, mean ~310."""
    return (9 + np.rint(568 * rng.beta(2.2, 1.9, size=n))).astype(np.uint32)


def doc_chunks(rng, n_docs, median=3.0, sigma=1.2, max_chunks=250):
    """Chunks per document: skewed lognormal, median 3, longest ~200+ (P:939-940)."""
    k = np.rint(np.exp(np.log(median) + sigma * rng.standard_normal(n_docs)))
    return np.clip(k, 1, max_chunks).astype(np.int64)


# ---------------------------------------------------------------------------------------------
# Builders
# ---------------------------------------------------------------------------------------------
class _Builder:
    def __init__(self, rng, engine):
        self.rng = rng
        self.engine = engine
        self.coeff_B = np.array([1, 2, 4, 8, 16, 32, 64, 128, 256], dtype=np.uint32)
        self.models, self.coeff, self.load, self.ev, self.ec = [], [], [], [], []
        self.node_model = []
        self.cols = dict(l_in_base=[], cap_y=[], pred=[], node=[], chain=[])
        self.n = 0

    def add_node(self, arch, tp_values=(1, 2, 4, 8), ecdf_mean=None, ecdf_sigma=None):
        spec = arch_spec(arch, tp_values)
        mid = len(self.models)
        mean = ecdf_mean if ecdf_mean is not None else self.rng.uniform(150, 300)
        sig = ecdf_sigma if ecdf_sigma is not None else self.rng.uniform(0.6, 1.0)
        v, c = make_ecdf(self.rng, mean, sig)
        self.models.append(spec)
        self.coeff.append(make_coeff(self.rng, spec, self.coeff_B))
        self.load.append(make_load(self.rng, spec))
        self.ev.append(v)
        self.ec.append(c)
        self.node_model.append(mid)
        return mid  # node id == model id

    def add_requests(self, node, l_in, cap, pred=None, chain=None):
        m = len(l_in)
        start = self.n
        self.cols["l_in_base"].append(np.asarray(l_in, dtype=np.uint32))
        self.cols["cap_y"].append(np.full(m, cap, dtype=np.uint32) if np.isscalar(cap)
                                  else np.asarray(cap, dtype=np.uint32))
        self.cols["pred"].append(np.full(m, -1, np.int32) if pred is None
                                 else np.asarray(pred, dtype=np.int32))
        self.cols["node"].append(np.full(m, node, np.int32))
        self.cols["chain"].append(np.full(m, -1, np.int32) if chain is None
                                  else np.asarray(chain, dtype=np.int32))
        self.n += m
        return start

    def chain_summary(self, n_docs, summ_arch="llama13b", eval_arch="llama70b", chunk=2048,
                      overhead=100, summary_cap=900, eval_times=4, template=300, eval_cap=512,
                      target_model_requests=None):
        """Fused self-loop summariser + evaluator fed by each document's final summary
        (P:376-380).  Successor prompt = chunk + overhead + previous summary."""
        ns = self.add_node(summ_arch)
        ne = self.add_node(eval_arch)
        k = doc_chunks(self.rng, n_docs)
        if target_model_requests is not None:
            # add docs until chunks + eval_times*docs >= target, trim the last doc (§8(d) C5)
            tot, keep = 0, []
            i = 0
            while tot < target_model_requests:
                kk = int(k[i % len(k)]) if i < len(k) else int(doc_chunks(self.rng, 1)[0])
                need = target_model_requests - tot - eval_times
                kk = max(1, min(kk, need)) if need > 0 else 1
                keep.append(kk)
                tot += kk + eval_times
                i += 1
            k = np.array(keep, dtype=np.int64)
        l_in, pred, chain, finals = [], [], [], []
        base = self.n
        idx = base
        for d, kk in enumerate(k):
            for j in range(kk):
                last = (j == kk - 1)
                cl = chunk if not last else int(self.rng.integers(200, chunk + 1))
                l_in.append(cl + overhead)
                pred.append(-1 if j == 0 else idx - 1)
                chain.append(d)
                idx += 1
            finals.append(idx - 1)
        self.add_requests(ns, l_in, summary_cap, pred, chain)
        e_pred = np.repeat(np.array(finals, dtype=np.int32), eval_times)
        self.add_requests(ne, np.full(len(e_pred), template), eval_cap, e_pred)
        return ns, ne

    def build(self, name, n_trials, description):
        cat = {k: np.concatenate(v) if v else np.zeros(0) for k, v in self.cols.items()}
        return Workload(
            name=name, n_trials=n_trials, engine=self.engine, models=self.models,
            coeff_B=self.coeff_B, coeff=self.coeff, load=self.load, ecdf_values=self.ev,
            ecdf_cum=self.ec, node_model=np.array(self.node_model, dtype=np.int32),
            l_in_base=cat["l_in_base"].astype(np.uint32), cap_y=cat["cap_y"].astype(np.uint32),
            pred=cat["pred"].astype(np.int32), node=cat["node"].astype(np.int32),
            chain=cat["chain"].astype(np.int32), description=description)


ENSEMBLE_ARCHS = ["llama7b", "llama7b", "llama13b", "llama13b", "llama34b", "llama70b"]
ROUTER_ARCHS = ["llama70b", "llama13b", "llama34b", "mistral7b"]
ROUTER_SPLIT = np.array([408, 2068, 456, 2657], dtype=np.float64)   # Table 1 without Mixtral


def _routing(b: _Builder, n_prompts: int):
    counts = np.floor(ROUTER_SPLIT / ROUTER_SPLIT.sum() * n_prompts + 0.5).astype(np.int64)
    counts[-1] = n_prompts - counts[:-1].sum()
    for arch, cnt in zip(ROUTER_ARCHS, counts):
        nd = b.add_node(arch)
        b.add_requests(nd, routerbench_lin(b.rng, int(cnt)), 4096)


def make_workload(name: str, seed: int = WORKLOAD_SEED, n_trials: Optional[int] = None,
                  n_prompts: Optional[int] = None, n_docs: Optional[int] = None,
                  n_gpus: Optional[int] = None) -> Workload:
    """Build one of BASELINE.json's configs (c1..c5) or a reduced variant for parity tests.

    c1: 1 LLM (13B), 100 requests, TP=1 only, 1000-point eCDF, 1 trial, 40 GB KV.
    c2: ensembling, 6 LLMs x 1000 prompts, tp in {1,2,4,8}, 64 trials, cap 256.
    c3: routing, 4 LLMs, 10k prompts split 730/3700/816/4754, cap 4096, 64 trials.
    c4: chain summary (13B fused summariser + 70B evaluator), 5000 docs, 64 trials.
    c5: mixed = ensembling 6 x 5000 + routing 10k + chain summary ~10k model-requests, 1024 trials.
    """
    rng = np.random.default_rng([seed, sum(map(ord, name))])
    if name == "c1":
        b = _Builder(rng, default_engine(n_gpus or 1))
        nd = b.add_node("llama13b", tp_values=(1,))
        b.add_requests(nd, mixinstruct_lin(rng, n_prompts or 100), 512)
        return b.build(name, n_trials or 1, "1 LLM (13B), 100 requests, TP=1, cap 512")
    if name == "c2":
        b = _Builder(rng, default_engine(n_gpus or 8))
        prompts = mixinstruct_lin(rng, n_prompts or 1000)
        for arch in ENSEMBLE_ARCHS:
            nd = b.add_node(arch)
            b.add_requests(nd, prompts, 256)
        return b.build(name, n_trials or 64, "ensembling 6 LLMs x 1000 prompts, cap 256")
    if name == "c3":
        b = _Builder(rng, default_engine(n_gpus or 8))
        _routing(b, n_prompts or 10000)
        return b.build(name, n_trials or 64, "routing 4 LLMs, 10k prompts (Table 1 split), cap 4096")
    if name == "c4":
        b = _Builder(rng, default_engine(n_gpus or 8))
        b.chain_summary(n_docs or 5000)
        return b.build(name, n_trials or 64, "chain summary 13B + 70B evaluator x4, 5000 docs")
    if name == "c5":
        b = _Builder(rng, default_engine(n_gpus or 8))
        prompts = mixinstruct_lin(rng, n_prompts or 5000)
        for arch in ENSEMBLE_ARCHS:
            nd = b.add_node(arch)
            b.add_requests(nd, prompts, 256)
        _routing(b, 2 * (n_prompts or 5000))
        b.chain_summary(n_docs or 2000, target_model_requests=2 * (n_prompts or 5000))
        return b.build(name, n_trials or 1024, "mixed: ensembling 6x5000 + routing 10k + chain ~10k")
    raise ValueError(f"unknown workload {name!r}")


def custom_workload(models, node_requests, n_trials=1, engine=None, seed=WORKLOAD_SEED,
                    ecdfs=None, coeff=None, load=None, name="custom") -> Workload:
    """Hand-built workload for fixtures.  `models`: list of arch names or spec dicts (one node
    per model); `node_requests`: per node a dict(l_in=..., cap=..., pred=None, chain=None)."""
    rng = np.random.default_rng(seed)
    b = _Builder(rng, engine or default_engine())
    for i, m in enumerate(models):
        if isinstance(m, str):
            b.add_node(m)
        else:
            spec = dict(m)
            b.models.append(spec)
            b.coeff.append(make_coeff(rng, spec, b.coeff_B))
            b.load.append(make_load(rng, spec))
            v, c = make_ecdf(rng, 200.0, 0.8)
            b.ev.append(v)
            b.ec.append(c)
            b.node_model.append(i)
    for i, nr in enumerate(node_requests):
        b.add_requests(i, nr["l_in"], nr.get("cap", 4096), nr.get("pred"), nr.get("chain"))
    w = b.build(name, n_trials, "custom fixture")
    if ecdfs is not None:
        for i, (v, c) in enumerate(ecdfs):
            if v is not None:
                w.ecdf_values[i] = np.asarray(v, dtype=np.uint32)
                w.ecdf_cum[i] = np.asarray(c, dtype=np.uint32)
    if coeff is not None:
        for i, cf in enumerate(coeff):
            if cf is not None:
                w.coeff[i] = np.asarray(cf, dtype=np.float64)
    if load is not None:
        for i, ld in enumerate(load):
            if ld is not None:
                w.load[i] = np.asarray(ld, dtype=np.float64)
    return w
