"""Why does a 32 MiB encrypt take ~100 us inside the e2e pipeline (trace)
instead of ~37 us?  Same kernel, 32 MiB device-resident, timed with events:
  A back to back; B isolated (host sleeps ~0.7 ms between launches);
  C isolated while H2D + D2H copies of 32 MiB run on two other streams."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1506_08503_b200 import device

dev = torch.device("cuda", 0)
n = (32 << 20) // 16
x = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device=dev)
y = torch.empty_like(x)
rk = device.expand_key(bytes(16), dev)
bc = device.BlockCipher(rk, bytes(16))
s = torch.cuda.current_stream()

def ev_time(fn):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); fn(); b.record(s); b.synchronize()
    return a.elapsed_time(b) * 1e3

for _ in range(5):
    bc.encrypt(x, out=y)
torch.cuda.synchronize()
# A
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(20):
    bc.encrypt(x, out=y)
b.record(s); b.synchronize()
print(f"A back-to-back: {a.elapsed_time(b) * 1e3 / 20:.1f} us per 32 MiB")
# B
for gap_ms in (0.1, 0.7, 3.0):
    ts = []
    for _ in range(20):
        time.sleep(gap_ms / 1e3)
        ts.append(ev_time(lambda: bc.encrypt(x, out=y)))
    ts.sort()
    print(f"B isolated, {gap_ms} ms host gap: median {ts[10]:.1f} us, min {ts[0]:.1f}, max {ts[-1]:.1f}")
# C
h_in = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
h_out = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
d_a = torch.empty_like(x); d_b = torch.empty_like(x)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
ts = []
for _ in range(20):
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    time.sleep(0.2e-3)
    ts.append(ev_time(lambda: bc.encrypt(x, out=y)))
    torch.cuda.synchronize()
ts.sort()
print(f"C during H2D+D2H copies: median {ts[10]:.1f} us, min {ts[0]:.1f}, max {ts[-1]:.1f}")
