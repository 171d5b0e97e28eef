"""The reference's encrypt_batch_parallel on the cuda backend: time vs
worker count (parallel._run_chunks calls the backend from W threads)."""
import os
import statistics
import sys
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [os.path.join(REPO, "baseline", "_ref"), REPO]
import gaes  # noqa: E402
from gaes import parallel  # noqa: E402

from paper_1506_08503_b200 import plugin  # noqa: E402

plugin.register(select=True)
rng = np.random.default_rng(5)
key = rng.bytes(16)
ivs = gaes.IVSet.shared(rng.bytes(16))
for n in (100_000, 1_000_000, 4_000_000):
    data = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    batch = gaes.MessageBatch(data=data, original_lens=(16,) * n) if n <= 100_000 else None
    if batch is None:  # MessageBatch validates rows in Python (~2.4 us/row); build it once cheaply
        batch = gaes.MessageBatch.__new__(gaes.MessageBatch)
        object.__setattr__(batch, "data", data)
        object.__setattr__(batch, "original_lens", (16,) * n)
    res = {}
    for w in (1, 2, 4, 8):
        parallel.encrypt_batch_parallel(key, ivs, batch, w)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            parallel.encrypt_batch_parallel(key, ivs, batch, w)
            ts.append(time.perf_counter() - t0)
        res[w] = statistics.median(ts)
    print(f"n={n}: " + ", ".join(f"W={w}: {res[w] * 1e3:.2f} ms ({n * 16 / res[w] / 1e9:.1f} GB/s)" for w in res)
          + f"; speedup W4/W1 = {res[1] / res[4]:.2f}")
