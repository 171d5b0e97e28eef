"""Multi-rank (N > 1) host logic on CPU: world_size 2 over gloo.

The GPU path shards blocks contiguously across ranks with no collective on
the data path; the only cross-rank operations are the
timing reduction (max over ranks) and verification gathers.  Here each rank
runs the oracle on its shard as a stand-in for its GPU and the gathered
result must be byte-identical to a single-rank run -- the reference's
"bytes independent of worker count" property (test_parallel.py:55-96,
test_acceptance.py:167-179) lifted to ranks.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_1506_08503_b200.shard import dist_env, key_slice, max_over_ranks, rank_slice, sum_over_ranks
        assert dist_env()[0] == rank and dist_env()[2] == world
        rng = np.random.default_rng(77)
        key, iv = rng.bytes(16), rng.bytes(16)
        out = {}
        for n in (1, 5, 1001):
            p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
            lo, hi = rank_slice(n, rank, world)
            ivrows = np.tile(np.frombuffer(iv, np.uint8), (hi - lo, 1))
            mine = oracle.encrypt(key, ivrows, p[lo:hi]) if hi > lo else np.empty((0, 16), np.uint8)
            parts = [None] * world
            dist.all_gather_object(parts, (lo, hi, mine))
            full = np.concatenate([x[2] for x in sorted(parts, key=lambda t: t[0])])
            out[n] = (full, p)
            assert sum_over_ranks(hi - lo) == n
        # many-key shards: keys contiguous, blocks follow their key
        k_lo, k_hi = key_slice(1024, rank, world)
        assert sum_over_ranks(k_hi - k_lo) == 1024
        assert max_over_ranks(float(rank) + 0.5) == world - 0.5
        if rank == 0:
            result_q.put({n: (f.tobytes(), p.tobytes()) for n, (f, p) in out.items()})
    finally:
        dist.destroy_process_group()


def test_two_rank_shards_reassemble_bit_exact(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rng = np.random.default_rng(77)
    key, iv = rng.bytes(16), rng.bytes(16)
    for n, (full, pbytes) in res.items():
        p = np.frombuffer(pbytes, np.uint8).reshape(n, 16)
        ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
        assert full == oracle.encrypt(key, ivrows, p).tobytes()


def test_plan_properties():
    from paper_1506_08503_b200.shard import plan, rank_slice
    for n in (0, 1, 2, 7, 148, 1 << 20):
        for g in (1, 2, 4, 8):
            chunks = plan(n, g).chunks
            assert len(chunks) == min(n, g)
            sizes = [b - a for a, b in chunks]
            if sizes:
                assert max(sizes) - min(sizes) <= 1 and sum(sizes) == n
            covered = [rank_slice(n, r, g) for r in range(g)]
            assert sum(b - a for a, b in covered) == n
    with pytest.raises(ValueError):
        plan(10, 0)
    with pytest.raises(ValueError):
        plan(-1, 2)


def test_plan_matches_reference_plan(oracle):
    from paper_1506_08503_b200.shard import plan
    for n in (0, 3, 100, 12345):
        for w in (1, 2, 3, 8):
            assert list(plan(n, w).chunks) == [tuple(c) for c in oracle.plan(n, w)]


def test_numa_binding_is_best_effort():
    from paper_1506_08503_b200.shard import bind_to_gpu_numa_node
    # no GPU here: must not raise, must not change the affinity
    before = os.sched_getaffinity(0)
    assert bind_to_gpu_numa_node(0) is None
    assert os.sched_getaffinity(0) == before


def test_cpulist_and_per_rank_host_threads():
    from paper_1506_08503_b200.shard import host_threads_per_rank, parse_cpulist
    assert parse_cpulist("0-3,8,10-11\n") == [0, 1, 2, 3, 8, 10, 11]
    assert parse_cpulist("") == []
    assert host_threads_per_rank(56, 4) == 14
    assert host_threads_per_rank(3, 8) == 1
    assert host_threads_per_rank(16, 0) == 16


def test_local_ranks_split_the_host_pool(monkeypatch):
    # 4 local ranks and no GPU sysfs entry: every rank gets a quarter of the
    # CPUs it may run on, and a caller's explicit GAES_HOST_THREADS wins
    from paper_1506_08503_b200.shard import bind_to_gpu_numa_node
    n = len(os.sched_getaffinity(0))
    monkeypatch.setenv("LOCAL_WORLD_SIZE", "4")
    monkeypatch.delenv("GAES_HOST_THREADS", raising=False)
    assert bind_to_gpu_numa_node(0) is None
    assert os.environ["GAES_HOST_THREADS"] == str(max(1, n // 4))
    monkeypatch.setenv("GAES_HOST_THREADS", "7")
    bind_to_gpu_numa_node(0)
    assert os.environ["GAES_HOST_THREADS"] == "7"
