"""Bidirectional PCIe with 1 vs 2 copy streams per direction (pinned, 256 MiB
each way): does a second concurrent H2D/D2H copy raise the per-direction
rate under bidirectional load?"""
import time, torch
n = 256 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory(); h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda"); d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
ss = [torch.cuda.Stream() for _ in range(8)]
def run(k):
    step = n // k
    for i in range(k):
        with torch.cuda.stream(ss[i]):
            d_in[i*step:(i+1)*step].copy_(h_in[i*step:(i+1)*step], non_blocking=True)
        with torch.cuda.stream(ss[4 + i]):
            h_out[i*step:(i+1)*step].copy_(d_out[i*step:(i+1)*step], non_blocking=True)
def h2d_only(k):
    step = n // k
    for i in range(k):
        with torch.cuda.stream(ss[i]):
            d_in[i*step:(i+1)*step].copy_(h_in[i*step:(i+1)*step], non_blocking=True)
for name, fn in (("bidir", run), ("h2d", h2d_only)):
    for k in (1, 2, 4):
        fn(k); torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter(); fn(k); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print(f"{name} streams/direction {k}: {n / min(ts) / 1e9:.1f} GB/s per direction")
