"""Throughput sweeps in the reference's CSV schema.

    python -m paper_1506_08503_b200.sweep --kind count [--out sweep.csv]

Mirrors the reference harness (pkg/src/gaes/bench.py): a known-answer gate
before any timing (bench.py:85-88), seeded random plaintext with one key/IV
drawn in the reference's order (bench.py:124-126), calls batched until a
timed region lasts >= 10 ms (bench.py:91-119), the median over repetitions,
and rows in the fixed CSV schema (bench.py:33-36)

    kind,implementation,n_messages,message_len_bytes,workers,total_bytes,median_seconds,rate_bytes_per_second

with ``implementation`` = "cuda" (host buffers through the backend boundary,
what encrypt_batch calls) or "cuda-device" (inputs resident in HBM) and
``workers`` = number of GPUs.  The reference harness itself rejects any
implementation but "vectorized"/"scalar-baseline" (bench.py:62-63), so this
is a separate driver emitting the same columns.
"""

from __future__ import annotations

import argparse
import sys
import time
from statistics import median

import numpy as np

from . import _lib, backend_cuda

CSV_HEADER = ("kind,implementation,n_messages,message_len_bytes,workers,"
              "total_bytes,median_seconds,rate_bytes_per_second")
# --extended appends (metrics): plaintext GB/s, fraction of the
# measured HBM copy bandwidth (32 B moved per block), fraction of the
# shared-memory lookup roofline (160 lookups per block at the sampled SM
# clock) and that clock.
EXTENDED_HEADER = CSV_HEADER + ",gbs,hbm_frac,lds_frac,sm_mhz"
MIN_REGION_SECONDS = 0.010


def _gate():
    """FIPS-197 C.1 + SP 800-38A F.2.1 through the GPU before timing anything."""
    from .device import expand_key
    key = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
    pt = np.frombuffer(bytes.fromhex("00112233445566778899aabbccddeeff"), np.uint8).reshape(1, 16)
    ct = backend_cuda.cbc_encrypt_std(pt, np.zeros((1, 16), np.uint8), expand_key(key))
    if ct.tobytes() != bytes.fromhex("69c4e0d86a7b0430d8cdb78070b4c55a"):
        raise RuntimeError("known-answer check failed (FIPS-197 C.1), sweep aborted")
    key = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
    iv = np.frombuffer(bytes.fromhex("000102030405060708090a0b0c0d0e0f"), np.uint8).reshape(1, 16)
    pt = np.frombuffer(bytes.fromhex("6bc1bee22e409f96e93d7e117393172aae2d8a571e03ac9c9eb76fac45af8e51"),
                       np.uint8).reshape(1, 32)
    ct = backend_cuda.cbc_encrypt_std(pt, iv, expand_key(key))
    if ct.tobytes()[:16] != bytes.fromhex("7649abac8119b246cee98e9b12e9197d"):
        raise RuntimeError("known-answer check failed (SP 800-38A), sweep aborted")


def _time(fn, reps: int, warmup: int, sync=None):
    sync = sync or (lambda: None)
    fn()
    sync()
    calls = 1
    while True:  # grow the batch until one region is >= 10 ms (bench.py:91-119)
        t0 = time.perf_counter()
        for _ in range(calls):
            fn()
        sync()
        if time.perf_counter() - t0 >= MIN_REGION_SECONDS or calls >= 1_000_000:
            break
        calls *= 2
    for _ in range(warmup):
        for _ in range(calls):
            fn()
        sync()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        for _ in range(calls):
            fn()
        sync()
        ts.append((time.perf_counter() - t0) / calls)
    return median(ts)


def _sm_mhz() -> float | None:
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByPciBusId(
            "{:08x}:{:02x}:{:02x}.0".format(*[getattr(torch.cuda.get_device_properties(0), k)
                                               for k in ("pci_domain_id", "pci_bus_id", "pci_device_id")]))
        return float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
    except Exception:  # pragma: no cover - informational
        return None


def _hbm_peak() -> float:
    import json
    import os
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def measure_point(kind: str, n: int, length: int, seed: int = 2016, reps: int = 5, warmup: int = 1,
                  device_resident: bool = False):
    from .device import expand_key
    rng = np.random.default_rng(seed)
    key, iv = rng.bytes(16), rng.bytes(16)
    width = 16 * ((length + 15) // 16)
    data = np.zeros((n, width), np.uint8)
    data[:, :length] = rng.integers(0, 256, (n, length), dtype=np.uint8)
    rk = expand_key(key)
    if device_resident:
        import torch
        if width != 16:
            from .device import cbc_encrypt as dev_cbc
            x = torch.from_numpy(data).cuda()
            fn = lambda: dev_cbc(x, rk, iv)  # noqa: E731
        else:
            from .device import BlockCipher
            x = torch.from_numpy(data).cuda()
            out = torch.empty_like(x)
            bc = BlockCipher(rk, iv)
            fn = lambda: bc.encrypt(x, out=out)  # noqa: E731
        sec = _time(fn, reps, warmup, sync=torch.cuda.synchronize)
        impl = "cuda-device"
    else:
        ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))  # IVSet.rows, as encrypt_batch passes
        out = np.empty_like(data)
        sec = _time(lambda: backend_cuda.cbc_encrypt_std(data, ivrows, rk, out), reps, warmup)
        impl = "cuda"
    total = n * length
    return (kind, impl, n, length, _lib.lib().gaes_get_num_gpus(), total, sec, total / sec)


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--kind", choices=["count", "length"], default="count")
    ap.add_argument("--counts", default="1,10,100,1000,10000,100000,1000000,16777216")
    ap.add_argument("--lengths", default="16,64,256,1024")
    ap.add_argument("--n-messages", type=int, default=128)
    ap.add_argument("--message-len", type=int, default=16)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--seed", type=int, default=2016)
    ap.add_argument("--device-resident", action="store_true")
    ap.add_argument("--extended", action="store_true", help="append gbs,hbm_frac,lds_frac,sm_mhz columns")
    ap.add_argument("--out", default="-")
    a = ap.parse_args(argv)
    _gate()
    rows = []
    if a.kind == "count":
        for n in (int(v) for v in a.counts.split(",")):
            rows.append(measure_point("count", n, a.message_len, a.seed, a.reps, device_resident=a.device_resident))
    else:
        for ln in (int(v) for v in a.lengths.split(",")):
            rows.append(measure_point("length", a.n_messages, ln, a.seed, a.reps, device_resident=a.device_resident))
    lines = [EXTENDED_HEADER if a.extended else CSV_HEADER]
    mhz = _sm_mhz() if a.extended else None
    hbm = _hbm_peak()
    for k, i, n, ln, w, t, sec, r in rows:
        line = f"{k},{i},{n},{ln},{w},{t},{sec:.9f},{r:.3f}"
        if a.extended:
            blocks = n * ((ln + 15) // 16)
            bps = blocks / sec
            lds = f"{bps * 160 / (148 * 32 * mhz * 1e6):.4f}" if mhz else ""
            line += f",{r / 1e9:.3f},{bps * 32 / 1e9 / hbm:.4f},{lds},{mhz or ''}"
        lines.append(line)
    text = "\n".join(lines) + "\n"
    if a.out == "-":
        sys.stdout.write(text)
    else:
        with open(a.out, "w") as f:
            f.write(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
