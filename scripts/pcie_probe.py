"""Measure the e2e ceilings on the GPU box: PCIe H2D / D2H / both at once
(pinned), and host memcpy bandwidth (pageable -> pinned staging)."""
import time, json, threading
import numpy as np, torch

n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return n / min(ts) / 1e9
res = {}
res["h2d_GBs"] = t(lambda: d_in.copy_(h_in, non_blocking=True))
res["d2h_GBs"] = t(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1): d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2): h_out.copy_(d_out, non_blocking=True)
res["h2d_and_d2h_concurrent_GBs_each"] = t(both)
a = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
b = h_in.numpy()
def cp1(): np.copyto(b, a)
t0 = time.perf_counter(); cp1(); cp1(); res["host_memcpy_1thread_GBs"] = 2 * n / (time.perf_counter() - t0) / 1e9
def cpk(k=8):
    step = n // k
    th = [threading.Thread(target=np.copyto, args=(b[i*step:(i+1)*step], a[i*step:(i+1)*step])) for i in range(k)]
    [x.start() for x in th]; [x.join() for x in th]
t0 = time.perf_counter(); cpk(); cpk(); res["host_memcpy_8threads_GBs"] = 2 * n / (time.perf_counter() - t0) / 1e9
print(json.dumps(res))
