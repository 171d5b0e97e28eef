"""Many small host-buffer requests from several threads at once (a serving
pattern): aggregate GB/s for 1 MiB pinned and pageable requests, 1..8
client threads (per-device lanes let concurrent calls overlap)."""
import sys
import threading
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1506_08503_b200 import backend_cuda, device  # noqa: E402

rk = device.expand_key(bytes(16))
iv = bytes(16)
N = 1 << 16  # 1 MiB requests
REQS = 200


def run(threads, pinned):
    bufs = []
    for _ in range(threads):
        if pinned:
            a = torch.randint(0, 256, (N, 16), dtype=torch.uint8).pin_memory().numpy()
            b = torch.empty((N, 16), dtype=torch.uint8).pin_memory().numpy()
        else:
            a = np.random.default_rng(1).integers(0, 256, (N, 16), dtype=np.uint8)
            b = np.empty_like(a)
        bufs.append((a, b))
    for a, b in bufs:
        backend_cuda.encrypt_shared_iv(a, iv, rk, out=b)

    def client(i):
        a, b = bufs[i]
        for _ in range(REQS // threads):
            backend_cuda.encrypt_shared_iv(a, iv, rk, out=b)

    th = [threading.Thread(target=client, args=(i,)) for i in range(threads)]
    t0 = time.perf_counter()
    [t.start() for t in th]
    [t.join() for t in th]
    dt = time.perf_counter() - t0
    return (REQS // threads) * threads * N * 16 / dt / 1e9, dt / ((REQS // threads)) * 1e6


for pinned in (True, False):
    for t in (1, 2, 4, 8):
        gbs, us = run(t, pinned)
        print(f"{'pinned' if pinned else 'pageable'} 1 MiB requests, {t} client threads: {gbs:.1f} GB/s aggregate")
