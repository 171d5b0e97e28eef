"""Does the NUMA placement of the pinned host buffers move the e2e number?
Allocates + first-touches the pinned input/output from CPUs local to the
GPU and from the other CPUs, then times backend_cuda.encrypt_shared_iv."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1506_08503_b200 import backend_cuda, device  # noqa: E402
from paper_1506_08503_b200.shard import _gpu_cpulist, parse_cpulist  # noqa: E402

allowed = sorted(os.sched_getaffinity(0))
local = [c for c in parse_cpulist(_gpu_cpulist(0)) if c in allowed]
remote = [c for c in allowed if c not in local]
print("cpus", len(allowed), "local to GPU 0:", len(local), "remote:", len(remote))
for node in sorted(os.listdir("/sys/devices/system/node")):
    if node.startswith("node"):
        print(node, open(f"/sys/devices/system/node/{node}/cpulist").read().strip())
n = 1 << 26  # 1 GiB
rk = device.expand_key(bytes(16))
iv = bytes(16)
src = torch.randint(0, 256, (n, 16), dtype=torch.uint8)
for name, cpus in (("local", local), ("remote", remote), ("all", allowed)):
    if not cpus:
        continue
    os.sched_setaffinity(0, cpus)
    h_in = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
    h_out = torch.empty_like(h_in).pin_memory()
    h_in.copy_(src)
    h_out.zero_()
    os.sched_setaffinity(0, allowed)
    hi, ho = h_in.numpy(), h_out.numpy()
    for _ in range(2):
        backend_cuda.encrypt_shared_iv(hi, iv, rk, out=ho)
    ts = []
    for _ in range(6):
        t0 = time.perf_counter()
        backend_cuda.encrypt_shared_iv(hi, iv, rk, out=ho)
        ts.append(time.perf_counter() - t0)
    print(f"pinned buffers first-touched from {name} CPUs: {n * 16 / np.median(ts) / 1e9:.2f} GB/s")
    del h_in, h_out
