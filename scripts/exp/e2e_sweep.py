"""Pinned 256 MiB encrypt_shared_iv (the bench's e2e call), median of 9."""
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1506_08503_b200 import backend_cuda, device  # noqa: E402

n = 1 << 24
h_in = torch.randint(0, 256, (n, 16), dtype=torch.uint8).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
rk = device.expand_key(bytes(16))
hi, ho = h_in.numpy(), h_out.numpy()
for _ in range(2):
    backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho)
ts = []
for _ in range(9):
    t0 = time.perf_counter()
    backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho)
    ts.append(time.perf_counter() - t0)
print(f"{n * 16 / statistics.median(ts) / 1e9:.2f} GB/s (median), best {n * 16 / min(ts) / 1e9:.2f}")
