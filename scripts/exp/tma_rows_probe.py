import sys, subprocess
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import oracle
from paper_1506_08503_b200 import device, _lib
n, bpr = int(sys.argv[1]), int(sys.argv[2])
rng = np.random.default_rng(1)
key, iv = rng.bytes(16), rng.bytes(16)
rk = oracle.gen_keys(key)
p = rng.integers(0, 256, (n, 16 * bpr), dtype=np.uint8)
x = torch.from_numpy(p).cuda()
c = device.cbc_encrypt(x, rk, iv)
torch.cuda.synchronize()
ok = np.array_equal(c.cpu().numpy(), oracle.encrypt(key, np.tile(np.frombuffer(iv, np.uint8), (n, 1)), p, threads=8))
print(n, bpr, _lib.last_kernel(), "ok" if ok else "MISMATCH")
'''
for n, bpr in [(32, 64), (64, 64), (100, 64), (1500, 64), (4736, 64), (9000, 8), (20000, 64), (152000, 8), (1500, 8), (33, 16)]:
    r = subprocess.run([sys.executable, "-c", code, str(n), str(bpr)], capture_output=True, text=True, timeout=120)
    print(r.stdout.strip() or ("FAIL %d %d: %s" % (n, bpr, r.stderr.strip().splitlines()[-1] if r.stderr else "")))
