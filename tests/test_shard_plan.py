"""libsamu's sharding rules on CPU (samu_shard_plan / samu_shard_classes, include/samu.h; DESIGN
§7): host-only entry points, so no GPU is needed.  North star: "candidates and Monte Carlo
trials shard naturally across the 8 GPUs of one box"."""
import itertools

import numpy as np
import pytest

import __graft_entry__  # noqa: F401
from paper_2503_16893_b200 import build as _build

_build.build()
from paper_2503_16893_b200 import SamuError, samu_shard_classes, samu_shard_plan  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("T", [0, 1, 2, 3, 5, 7, 8, 64, 1023, 1024])
def test_every_class_trial_pair_exactly_once(world, T):
    plans = [samu_shard_plan(T, world, r) for r in range(world)]
    Wt, Wc = plans[0]["trial_blocks"], plans[0]["job_classes"]
    assert all(p["trial_blocks"] == Wt and p["job_classes"] == Wc for p in plans)
    assert Wt * Wc == world
    # pure trial sharding whenever there are enough trials; else the most trial blocks that fit
    if T >= world:
        assert Wc == 1
    else:
        assert Wt == max(d for d in range(1, world + 1) if world % d == 0 and d <= max(T, 1))
    for c in range(Wc):
        ranks = [r for r in range(world) if plans[r]["my_class"] == c]
        assert ranks == list(range(c * Wt, (c + 1) * Wt))   # rank r: class r / Wt, block r % Wt
        covered = []
        for r in ranks:
            covered.extend(range(plans[r]["trial_begin"], plans[r]["trial_begin"] + plans[r]["trial_count"]))
        assert covered == list(range(T))                       # contiguous blocks in rank order
        counts = [plans[r]["trial_count"] for r in ranks]
        assert max(counts) - min(counts) <= 1 and counts == sorted(counts, reverse=True)


def test_forced_classes_and_invalid_arguments():
    p = samu_shard_plan(64, 8, 5, forced_classes=4)
    assert (p["trial_blocks"], p["job_classes"], p["my_class"]) == (2, 4, 2)
    assert (p["trial_begin"], p["trial_count"]) == (32, 32)
    # a forced count that does not divide the world is ignored
    assert samu_shard_plan(64, 8, 5, forced_classes=3)["job_classes"] == 1
    for args in [(-1, 2, 0), (4, 0, 0), (4, 2, 2), (4, 2, -1)]:
        with pytest.raises(SamuError):
            samu_shard_plan(*args)
    with pytest.raises(SamuError):
        samu_shard_classes([1.0, -2.0], 2)
    with pytest.raises(SamuError):
        samu_shard_classes([1.0, float("nan")], 2)
    with pytest.raises(SamuError):
        samu_shard_classes([1.0], 0)


def test_class_assignment_hand_case():
    # longest first (stable on ties), onto the least loaded class (lowest index on ties):
    # 5 (job 3) -> 0, 5 (job 4) -> 1, 3 (job 0) -> 0, 2 (job 2) -> 1, 1 (job 1) -> 1
    assert samu_shard_classes([3, 1, 2, 5, 5], 2).tolist() == [0, 1, 1, 0, 1]
    assert samu_shard_classes([], 3).tolist() == []
    assert samu_shard_classes([7, 7, 7], 1).tolist() == [0, 0, 0]


def test_class_assignment_within_grahams_bound():
    # longest-processing-time-first list scheduling: makespan <= (4/3 - 1/(3m)) OPT (Graham 1969);
    # OPT by brute force over all assignments of small instances
    rng = np.random.default_rng(16893)
    for _ in range(200):
        n, m = int(rng.integers(1, 8)), int(rng.integers(1, 4))
        work = rng.integers(1, 50, n).astype(float)
        cls = samu_shard_classes(work, m)
        assert cls.min() >= 0 and cls.max() < m
        got = max(work[cls == k].sum() for k in range(m))
        opt = min(max(sum(work[i] for i in range(n) if a[i] == k) for k in range(m))
                  for a in itertools.product(range(m), repeat=n))
        assert got <= (4 / 3 - 1 / (3 * m)) * opt + 1e-9
