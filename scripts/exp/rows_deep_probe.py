"""Few long rows (general-M CBC encrypt): the deep-prefetch row kernel vs
the one-pair-lookahead LDG kernel (GAES_ROWS_DEEP=0), bit-exact against the
oracle on a sample of rows.  Usage: rows_deep_probe.py  (runs both arms in
subprocesses)."""
import os, subprocess, sys
code = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from oracle import oracle
from paper_1506_08503_b200 import device, _lib
rows, bpr = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(5)
key, iv = rng.bytes(16), rng.bytes(16)
rk = oracle.gen_keys(key)
x = torch.randint(0, 256, (rows, 16 * bpr), dtype=torch.uint8, device="cuda")
out = device.cbc_encrypt(x, rk, iv)
torch.cuda.synchronize()
k = min(rows, 4)
p = x[:k].cpu().numpy()
ok = np.array_equal(out[:k].cpu().numpy(), oracle.encrypt(key, np.tile(np.frombuffer(iv, np.uint8), (k, 1)), p))
kern = _lib.last_kernel()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
a.record()
for _ in range(reps):
    device.cbc_encrypt(x, rk, iv, out=out)
b.record(); b.synchronize()
ms = a.elapsed_time(b) / reps
print(f"{rows} rows x {bpr} blocks: {kern} {'ok' if ok else 'MISMATCH'} {ms*1e3:.1f} us {rows*bpr*16/ms/1e6:.1f} GB/s")
'''
for rows, bpr in [(1, 65536), (4, 16384), (148, 4096), (1024, 1024), (8192, 1024), (16384, 1024), (32768, 512), (37888, 256), (100, 8), (300, 10)]:
    for deep, texs in (("1", "0"), ("1", "1"), ("0", "1")):
        env = dict(os.environ, GAES_ROWS_DEEP=deep, GAES_ROWS_DEEP_TEXS=texs)
        r = subprocess.run([sys.executable, "-c", code, str(rows), str(bpr)], capture_output=True, text=True, timeout=300, env=env)
        print(f"deep={deep} texs={texs}", r.stdout.strip() or r.stderr.strip().splitlines()[-1])
