"""GPU-side cost of a config-1 step (2^16 blocks), host enqueue removed:
CUDA-graph replays of K steps, with and without an L2 flush between them
(the flush's own graph time subtracted)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1506_08503_b200 import device  # noqa: E402

K = 50
dev = torch.device("cuda", 0)
for lg in (12, 14, 16, 18, 20):
    n = 1 << lg
    x = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device=dev)
    out = torch.empty_like(x)
    bc = device.BlockCipher(device.expand_key(bytes(16)), bytes(16))
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    s = torch.cuda.Stream()

    def graph_time(body):
        with torch.cuda.stream(s):
            body()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                body()
            g.replay()
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            g.replay()
            b.record(s)
            torch.cuda.synchronize()
            return a.elapsed_time(b) * 1e3 / K

    def steps():
        for _ in range(K):
            bc.encrypt(x, out=out)

    def flushes():
        for i in range(K):
            flush.fill_(i & 0xFF)

    def both():
        for i in range(K):
            flush.fill_(i & 0xFF)
            bc.encrypt(x, out=out)

    t_steps, t_fl, t_both = graph_time(steps), graph_time(flushes), graph_time(both)
    print(f"2^{lg} blocks: back-to-back {t_steps:.2f} us/step ({n * 16 / t_steps / 1e3:.0f} GB/s); "
          f"after L2 flush {t_both - t_fl:.2f} us/step ({n * 16 / (t_both - t_fl) / 1e3:.0f} GB/s)")
