"""N>1 host logic on CPU (gloo, world size 2): trials are sharded in contiguous blocks, every rank
simulates only its share, per-(candidate, trial) records are all-gathered in rank = trial order
and reduced in trial order.  The result must be bit-identical to the single-process run, for the
per-candidate means (c17) and for the greedy's stage score inputs.  The simulator here is the
oracle (no GPU); libsamu's NCCL path follows the same plan (samu_host.cu: trial_share,
gather_records) and bench.py uses the same split.
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
    base, rem = divmod(T, world)
    cnt = base + (1 if rank < rem else 0)
    return rank * base + min(rank, rem), cnt


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
    w = W.make_workload("c2", n_prompts=120, n_trials=T)
    P = O.Problem(w)
    tb, cnt = trial_share(T, world, rank)
    lo, li = P.sample(SEED, tb, cnt)          # counter-based: only this rank's trials
    recs = np.stack([P.simulate(n, d, t, lo, li)[0] for (n, d, t) in CANDS])   # [cand][local trial]
    tmax = -(-T // world)
    buf = np.zeros((len(CANDS), tmax), O.REC_DTYPE)
    buf[:, :cnt] = recs
    send = torch.from_numpy(buf.view(np.uint8).copy())
    gathered = [torch.zeros_like(send) for _ in range(world)]
    dist.all_gather(gathered, send)
    full = np.zeros((len(CANDS), T), O.REC_DTYPE)
    for r in range(world):
        b, c = trial_share(T, world, r)
        full[:, b:b + c] = gathered[r].numpy().view(O.REC_DTYPE).reshape(len(CANDS), tmax)[:, :c]
    if rank == 0:
        np.save(out_path, full.view(np.uint8))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("T", [5, 8])
def test_sharded_records_equal_single_process(tmp_path, T):
    world = 2
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
    for T in (1, 7, 64, 1024):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b, c = trial_share(T, world, r)
                seen.extend(range(b, b + c))
            assert seen == list(range(T))
