"""Config-1 step timed the way bench.py does (L2 flush, then events around
the step): stream launch vs replay of a CUDA graph holding the same launch."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1506_08503_b200 import device  # noqa: E402

n = 1 << 16
dev = torch.device("cuda", 0)
x = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device=dev)
out = torch.empty_like(x)
bc = device.BlockCipher(device.expand_key(bytes(16)), bytes(16))
flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for _ in range(5):
        bc.encrypt(x, out=out)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        bc.encrypt(x, out=out)
    g.replay()
    torch.cuda.synchronize()

    def timed(fn, reps=20):
        ev = []
        for i in range(reps):
            flush.fill_(i & 0xFF)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            ev.append((a, b))
        torch.cuda.synchronize()
        ms = sorted(a.elapsed_time(b) for a, b in ev)
        return ms[len(ms) // 2] * 1e3

    for _ in range(2):
        t1 = timed(lambda: bc.encrypt(x, out=out))
        t2 = timed(g.replay)
        print(f"stream launch {t1:.2f} us ({n * 16 / t1 / 1e3:.0f} GB/s); graph replay {t2:.2f} us ({n * 16 / t2 / 1e3:.0f} GB/s)")
