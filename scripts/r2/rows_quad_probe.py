"""Few long rows: CBC encrypt time with four lanes per row vs one thread per
row (GAES_TUNE=ROWS_QUAD=0), device-resident, CUDA events.

    python scripts/r2/rows_quad_probe.py
"""
import os
import subprocess
import sys

SHAPES = [(1, 65536), (16, 4096), (148, 4096), (1024, 256), (4096, 64), (16384, 16), (37888, 8)]
code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_1506_08503_b200 import device, _lib
rows, bpr = int(sys.argv[1]), int(sys.argv[2])
x = torch.randint(0, 256, (rows, 16 * bpr), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
rk = device.expand_key(bytes(16))
for _ in range(2):
    device.cbc_encrypt(x, rk, bytes(16), out=out)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 3 if rows * bpr >= (1 << 16) and rows < 64 else 10
a.record()
for _ in range(reps):
    device.cbc_encrypt(x, rk, bytes(16), out=out)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / reps
print(f"{_lib.last_kernel():22s} {ms:9.3f} ms  {rows * bpr * 16 / ms / 1e6:8.2f} GB/s")
'''
for rows, bpr in SHAPES:
    for tune in ("", "ROWS_QUAD=0"):
        env = dict(os.environ, GAES_TUNE=tune)
        r = subprocess.run([sys.executable, "-c", code, str(rows), str(bpr)], env=env, capture_output=True, text=True)
        print(f"rows={rows:6d} x {bpr:6d} blocks  {r.stdout.strip() or r.stderr[-300:]}", flush=True)
