"""Pageable drop-in call with a freshly allocated `out` each call (what the
reference's encrypt_batch does: np.empty_like) vs a reused one."""
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1506_08503_b200 import backend_cuda  # noqa: E402

rng = np.random.default_rng(1)
rk = rng.integers(0, 256, (11, 16), dtype=np.uint8)
tables = (rk,) + backend_cuda.standard_tables(False)
iv = rng.integers(0, 256, 16, dtype=np.uint8)
for n in (100_000, 1 << 20):
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    ivrows = np.tile(iv, (n, 1))
    out = np.empty_like(p)
    backend_cuda.cbc_encrypt(p, ivrows, *tables, out)
    for label, fresh in (("reused out", False), ("fresh out", True), ("fresh out, pre-touched", None)):
        ts = []
        for _ in range(7):
            o = np.empty_like(p) if fresh is not False else out
            if fresh is None:
                o.fill(0)
            t0 = time.perf_counter()
            backend_cuda.cbc_encrypt(p, ivrows, *tables, o)
            ts.append(time.perf_counter() - t0)
        print(f"n={n} {label}: {statistics.median(ts) * 1e3:.2f} ms")
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        np.empty_like(p).fill(0)
        ts.append(time.perf_counter() - t0)
    print(f"n={n} numpy first-touch fill of a fresh array: {statistics.median(ts) * 1e3:.2f} ms")
