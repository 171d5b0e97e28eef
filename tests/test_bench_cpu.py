"""bench.py host logic that runs without a GPU: the workloads match
SURVEY.md 8 / BASELINE.json's configs, the defaults keep the driver
contract (config 3, the first config the 1/2/4/8-B200 metric is quoted on),
both arms describe the workload with the same config dict, the shard
geometry tiles the workload for N = 1, 2, 4, 8, device generation does not
depend on the rank count, and `--gpus N` refuses to pretend when N GPUs are
not there."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_workloads_match_the_scope_table():
    import bench
    w = bench.WORKLOADS
    assert sorted(w) == [1, 2, 3, 4, 5]
    assert [w[c]["blocks"] for c in (1, 2, 3, 4, 5)] == [1 << 16, 1 << 24, 1 << 28, 1 << 26, 1 << 30]
    assert w[5]["keys"] == 1024 and (1 << 30) // 1024 == 1 << 20
    assert w[1]["scaling"] == w[2]["scaling"] == "weak"
    assert w[3]["scaling"] == w[4]["scaling"] == w[5]["scaling"] == "strong"
    assert bench.LOOKUPS_PER_BLOCK == 160 and bench.T_LOOKUPS_PER_BLOCK == 144
    assert bench.HBM_BYTES_PER_BLOCK == 32


def test_defaults_keep_the_driver_contract():
    import bench
    a = bench.parse([])
    assert a.gpus == 1 and a.config == 3 and a.impl == "ours"
    assert a.warmup >= 3 and a.steps >= 10


@pytest.mark.skipif(__import__("torch").cuda.device_count() >= 2, reason="this box has >= 2 GPUs")
def test_multi_gpu_request_without_gpus_fails_loudly():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2"], cwd=REPO, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 2 and "needs 2 visible GPUs" in r.stderr


def test_metric_is_baselines_verbatim():
    import bench
    with open(os.path.join(REPO, "BASELINE.json")) as f:
        assert bench.METRIC == json.load(f)["metric"]


def test_plan_matches_the_package_plan():
    import bench
    from paper_1506_08503_b200.shard import plan
    for n in (0, 1, 7, 1 << 10, (1 << 28) + 3):
        for k in (1, 2, 3, 4, 8, 16):
            assert bench.plan_chunks(n, k) == list(plan(n, k).chunks)


@pytest.mark.parametrize("cfg", [3, 4, 5])
@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_rank_ranges_are_unions_of_digest_pieces(cfg, world):
    """Strong configs: the ranks' ranges tile the workload, and every rank
    owns whole digest pieces, so N = 1 and N > 1 print the same 8 digests."""
    import bench
    pcs = bench.pieces(cfg)
    assert len(pcs) == bench.PIECES and pcs[0][0] == 0 and pcs[-1][1] == bench.WORKLOADS[cfg]["blocks"]
    ranges = [bench.rank_range(cfg, r, world) for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == bench.WORKLOADS[cfg]["blocks"]
    assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
    for lo, hi in ranges:
        owned = [p for p in pcs if lo <= p[0] and p[1] <= hi]
        assert owned and owned[0][0] == lo and owned[-1][1] == hi
        if cfg == 5:
            assert lo % (1 << 20) == 0 and hi % (1 << 20) == 0  # key-aligned
    # generation chunks never straddle a rank boundary at these N
    assert all(lo % bench.GEN_CHUNK_BLOCKS == 0 for lo, _ in ranges)


@pytest.mark.parametrize("world", [1, 2, 8])
def test_config_dict_is_the_same_in_both_arms(world):
    import bench
    a = bench.config_dict(3, world)
    assert a == bench.config_dict(3, world)
    assert a["total_blocks"] == 1 << 28 and a["blocks_per_gpu"] == (1 << 28) // world
    assert a["workload"] == bench.WORKLOADS[3]["name"] and a["parallelism"].startswith(f"dp{world} ")
    assert a["l2"] == "inputs larger than L2 (no flush)"
    assert bench.config_dict(1, world)["l2"].startswith("ring of K cold copies")
    assert bench.config_dict(2, world)["total_blocks"] == world << 24  # weak
    json.dumps(a)


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_generation_does_not_depend_on_the_rank_count(monkeypatch, cfg):
    """make_inputs draws every generation chunk whole from a generator seeded
    by its global index: the shards of N = 2 and N = 4 concatenate to the
    N = 1 bytes (here on the CPU with 2^12-block chunks)."""
    import torch

    import bench
    monkeypatch.setattr(bench, "GEN_CHUNK_BLOCKS", 1 << 12)
    blocks = 1024 * 16 if cfg == 5 else 1 << 14
    one = bench.make_inputs(cfg, 0, 1, torch.device("cpu"), blocks=blocks)["p"]
    assert one.shape == (blocks, 16)
    for world in (2, 4):
        parts = [bench.make_inputs(cfg, r, world, torch.device("cpu"), blocks=blocks)["p"] for r in range(world)]
        assert torch.equal(torch.cat(parts), one)
    h = one.numpy()
    if cfg == 3:
        s = h.view(np.int16).astype(np.float64)
        assert np.abs(s).mean() > 1000  # the sinusoids are there
    if cfg == 4:
        assert not h[:, 8:].any()


@pytest.mark.parametrize("cfg", [1, 3, 4, 5])
def test_cpu_sample_follows_the_workload(cfg):
    import bench
    p, segs = bench.cpu_sample(cfg, 1 << 13)
    assert p.dtype == np.uint8 and p.shape[1] == 16
    assert segs[0][2] == 0 and segs[-1][3] == p.shape[0]
    prm = bench.workload_params(cfg)
    if cfg != 5:
        assert segs == [(prm["key"], prm["iv"], 0, p.shape[0])]
    else:
        assert segs[0][0] == prm["keys"][0].tobytes() and len(segs) == 1
        p2, segs2 = bench.cpu_sample(cfg, 1 << 21)  # two keys' worth of the workload's 2^20 blocks
        assert [(a, b) for _, _, a, b in segs2] == [(0, 1 << 20), (1 << 20, 1 << 21)]
        assert segs2[1][0] == prm["keys"][1].tobytes() and segs2[1][1] == prm["ivs"][1].tobytes()
    if cfg == 4:
        assert not p[:, 8:].any()


def test_reference_arm_runs_the_reference_cpu_path():
    """--impl reference on a tiny sample: one JSON line with the same config
    dict as our arm, the reference's own CPU path (baseline/_ref or
    oracle/_ref), decrypt rate and an e2e object without copies."""
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "1", "--steps", "2",
                        "--warmup", "1", "--cpu-sample-cap", "4096"], cwd=REPO, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr
    line = json.loads(r.stdout.strip().splitlines()[-1])
    import bench
    assert line["impl"] == "reference" and line["metric"] == bench.METRIC and line["unit"] == "GB/s"
    assert line["config"] == bench.config_dict(1, 1)
    assert line["cpu_baseline"]["kind"] in ("reference", "port") and line["value"] > 0
    assert line["decrypt"]["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_without_work():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2"], cwd=REPO, env=env,
                       capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_reference_cpu_matches_the_oracle_and_round_trips():
    import bench
    r = bench.ReferenceCPU(3, 2048, 2)
    r.encrypt()
    r.decrypt()
    r.check()
    assert np.array_equal(r.back, r.p)


@pytest.mark.parametrize("cfg", [3, 5])
def test_openssl_sample_check_catches_a_wrong_block(monkeypatch, cfg):
    """bench.py's in-run independent check (OpenSSL ECB of P ^ IV on a seeded
    sample) accepts the oracle's ciphertext and rejects a corrupted one."""
    pytest.importorskip("cryptography")
    import torch

    import bench
    from oracle import oracle
    monkeypatch.setattr(bench, "GEN_CHUNK_BLOCKS", 1 << 12)
    blocks = 1024 * 8 if cfg == 5 else 1 << 13
    inp = bench.make_inputs(cfg, 0, 1, torch.device("cpu"), blocks=blocks)
    p = inp["p"].numpy()
    if cfg == 5:
        bpk = inp["bpk"]
        c = np.concatenate([oracle.encrypt(inp["keys"][k].tobytes(), np.tile(inp["ivs"][k], (bpk, 1)),
                                           p[k * bpk:(k + 1) * bpk]) for k in range(inp["keys"].shape[0])])
    else:
        c = oracle.encrypt(inp["key"], np.tile(np.frombuffer(inp["iv"], np.uint8), (blocks, 1)), p)
    out = torch.from_numpy(c.copy())
    ok, n = bench.openssl_sample_check(inp, inp["p"], out, cfg, n_sample=blocks)
    assert ok and n == blocks
    out[blocks // 2, 3] ^= 1
    assert not bench.openssl_sample_check(inp, inp["p"], out, cfg, n_sample=blocks)[0]
