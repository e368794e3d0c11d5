"""N>1 host logic on CPU (gloo, world sizes 2 and 4): every rank takes its share from libsamu's
own sharding rules (samu_shard_plan / samu_shard_classes, the host-only entry points the sharded
calls apply internally): contiguous trial blocks, and job classes when there are fewer trials
than ranks.  Each rank simulates only its (class, trial block), the per-(candidate, trial)
records are all-gathered in rank order and placed by the same plan.  The result must be
bit-identical to the single-process run, for the records and the trial-ordered means (c17).
The simulator here is the oracle (no GPU); libsamu's NCCL path gathers with the same plan
(samu_host.cu: gather_records, the unpack kernel) and bench.py uses the same split.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
import samu_workloads as W

SEED = W.SAMPLING_SEED


def trial_share(T, world, rank):
    """the contiguous split written out (the reference for libsamu's plan in the tests below)"""
    base, rem = divmod(T, world)
    cnt = base + (1 if rank < rem else 0)
    return rank * base + min(rank, rem), cnt


def _libsamu():
    import __graft_entry__  # noqa: F401
    from paper_2503_16893_b200 import build
    build.build()
    import paper_2503_16893_b200 as S
    return S


def _work(w):
    # per-candidate work for the class assignment: replica requests x mean prompt (any fixed,
    # rank-independent value does; the greedy uses replica requests x expected output)
    return [float(np.sum(w.node == n)) / d * (1 + t) for (n, d, t) in CANDS]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


CANDS = [(0, 1, 1), (2, 2, 1), (5, 1, 4), (3, 4, 2)]


def _worker(rank, world, port, T, out_path):
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    S = _libsamu()
    w = W.make_workload("c2", n_prompts=120, n_trials=T)
    P = O.Problem(w)
    plans = [S.samu_shard_plan(T, world, r) for r in range(world)]
    me = plans[rank]
    Wt, Wc = me["trial_blocks"], me["job_classes"]
    cls = S.samu_shard_classes(_work(w), Wc)
    tb, cnt = me["trial_begin"], me["trial_count"]
    tmax = -(-T // Wt)
    buf = np.zeros((len(CANDS), tmax), O.REC_DTYPE)
    if cnt:
        lo, li = P.sample(SEED, tb, cnt)      # counter-based: only this rank's trials
        for x, (n, d, t) in enumerate(CANDS):
            if cls[x] == me["my_class"]:      # only this rank's job class
                buf[x, :cnt] = P.simulate(n, d, t, lo, li)[0]
    send = torch.from_numpy(buf.view(np.uint8).copy())
    gathered = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(gathered, send)
    full = np.zeros((len(CANDS), T), O.REC_DTYPE)
    filled = np.zeros((len(CANDS), T), np.int32)
    for r in range(world):
        b, c, k = plans[r]["trial_begin"], plans[r]["trial_count"], plans[r]["my_class"]
        g = gathered[r].numpy().view(O.REC_DTYPE).reshape(len(CANDS), tmax)
        for x in range(len(CANDS)):
            if cls[x] == k:
                full[x, b:b + c] = g[x, :c]
                filled[x, b:b + c] += 1
    assert (filled == 1).all()                # every (candidate, trial) from exactly one rank
    if rank == 0:
        np.save(out_path, full.view(np.uint8))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world,T", [(2, 5), (2, 8), (4, 3), (4, 1)])
def test_sharded_records_equal_single_process(tmp_path, world, T):
    out = str(tmp_path / "full.npy")
    mp.spawn(_worker, args=(world, _free_port(), T, out), nprocs=world, join=True)
    full = np.load(out).view(O.REC_DTYPE).reshape(len(CANDS), T)
    w = W.make_workload("c2", n_prompts=120, n_trials=T)
    P = O.Problem(w)
    lo, li = P.sample(SEED, 0, T)
    ref = np.stack([P.simulate(n, d, t, lo, li)[0] for (n, d, t) in CANDS])
    assert full.tobytes() == ref.tobytes()
    # trial-ordered reductions (means feeding f* and T_E) are therefore world-size independent
    for ci in range(len(CANDS)):
        s1 = 0.0
        for x in full["t_end"][ci]:
            s1 += float(x)
        s2 = 0.0
        for x in ref["t_end"][ci]:
            s2 += float(x)
        assert s1 / T == s2 / T


def test_trial_share_partitions():
    S = _libsamu()
    for T in (1, 7, 64, 1024):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b, c = trial_share(T, world, r)
                seen.extend(range(b, b + c))
                if T >= world:                # libsamu's pure trial sharding is this split
                    p = S.samu_shard_plan(T, world, r)
                    assert (p["trial_begin"], p["trial_count"]) == (b, c)
            assert seen == list(range(T))
