"""bench.py host logic that runs without a GPU: the workloads match
SURVEY.md 8 / BASELINE.json's configs, the defaults keep the driver
contract, and `--gpus N` refuses to pretend when N GPUs are not there."""

import os
import subprocess
import sys

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


def test_defaults_keep_the_driver_contract(monkeypatch):
    import bench
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert a.gpus == 1 and a.config == 2 and a.impl == "ours"
    assert a.warmup >= 3 and a.steps >= 10


@pytest.mark.skipif(__import__("torch").cuda.device_count() >= 2, reason="this box has >= 2 GPUs")
def test_multi_gpu_request_without_gpus_fails_loudly():
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2"], cwd=REPO, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 2 and "needs 2 visible GPUs" in r.stderr


def test_metric_is_baselines_verbatim():
    import json
    import bench
    with open(os.path.join(REPO, "BASELINE.json")) as f:
        assert bench.METRIC == json.load(f)["metric"]
