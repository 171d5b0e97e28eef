"""Where do the ~12 us of a config-1 step (2^16 blocks) go?"""
import sys
import torch
sys.path.insert(0, ".")
from paper_1506_08503_b200 import device

n = 1 << 16
x = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
bc = device.BlockCipher(device.expand_key(bytes(16)), bytes(16))
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()
for _ in range(5):
    bc.encrypt(x, out=out)
torch.cuda.synchronize()

def timed(with_flush, reps=20, back_to_back=False):
    ev = []
    if back_to_back:
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        bc.encrypt(x, out=out)
        a.record(s)
        for _ in range(reps):
            bc.encrypt(x, out=out)
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps * 1e3
    for i in range(reps):
        if with_flush:
            flush.fill_(i)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        bc.encrypt(x, out=out)
        b.record(s)
        ev.append((a, b))
    torch.cuda.synchronize()
    return sum(a.elapsed_time(b) for a, b in ev) / reps * 1e3

print(f"per-step events, L2 flushed between: {timed(True):.2f} us")
print(f"per-step events, no flush:           {timed(False):.2f} us")
print(f"back to back (PDL), no flush:        {timed(False, back_to_back=True):.2f} us")

import ctypes
from paper_1506_08503_b200 import _lib
r, m = ctypes.c_double(), ctypes.c_double()
for it in (0, 1, 4):
    _lib.check(_lib.lib().gaes_probe_round_rate(0, it, ctypes.addressof(r), ctypes.addressof(m)))
    print(f"round probe (148 CTAs x 1024 thr, 192 KiB fill, {it} encryptions/thread): {m.value * 1e3:.2f} us")
e = torch.empty(1, device="cuda")
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(100):
    e.add_(1)
b.record(s)
torch.cuda.synchronize()
print(f"tiny torch kernel back to back: {a.elapsed_time(b) / 100 * 1e3:.2f} us")
