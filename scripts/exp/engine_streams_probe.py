"""Pinned e2e pipeline with one stream per engine (all H2D copies back to
back on one stream, kernels on a second, D2H on a third, linked by events,
no host waits, whole-job device buffers) vs the library's slot pipeline."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1506_08503_b200 import device, backend_cuda
n = 1 << 24
MB = 1 << 20
h_in = torch.randint(0, 256, (n, 16), dtype=torch.uint8).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
rk = device.expand_key(bytes(16))
bc = device.BlockCipher(rk, bytes(16))
d_in = torch.empty((n, 16), dtype=torch.uint8, device="cuda"); d_out = torch.empty_like(d_in)
sh, sk, sd = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()

def schedule(total_rows, base_mb, first_div):
    base = base_mb * MB // 16; lo = max(1, base // first_div)
    out, r0, cur = [], 0, lo
    while r0 < total_rows:
        left = total_rows - r0
        take = min(cur, left)
        if left <= 2 * base: take = min(take, max(lo, (left + 1) // 2))
        if left - take < lo // 2: take = left
        out.append((r0, take)); r0 += take; cur = min(base, cur * 2)
    return out

def engines(base_mb, first_div):
    ch = schedule(n, base_mb, first_div)
    def run():
        for r0, k in ch:
            with torch.cuda.stream(sh):
                d_in[r0:r0 + k].copy_(h_in[r0:r0 + k], non_blocking=True)
                e1 = torch.cuda.Event(); e1.record(sh)
            sk.wait_event(e1)
            with torch.cuda.stream(sk):
                bc.encrypt(d_in[r0:r0 + k], out=d_out[r0:r0 + k])
                e2 = torch.cuda.Event(); e2.record(sk)
            sd.wait_event(e2)
            with torch.cuda.stream(sd):
                h_out[r0:r0 + k].copy_(d_out[r0:r0 + k], non_blocking=True)
        torch.cuda.synchronize()
    return run

def lib():
    backend_cuda.encrypt_shared_iv(h_in.numpy(), bytes(16), rk, out=h_out.numpy())

def med(fn, reps=11):
    fn(); fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    ts.sort(); return n * 16 / ts[reps // 2] / 1e9

print(f"library slot pipeline: {med(lib):.2f} GB/s")
for base in (8, 16, 32):
    for fd in (4, 8, 16):
        print(f"engine streams, base {base} MiB, first base/{fd}: {med(engines(base, fd)):.2f} GB/s")
print(f"library slot pipeline: {med(lib):.2f} GB/s")
