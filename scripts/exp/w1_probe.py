import os, statistics, sys, time
import numpy as np
REPO = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [os.path.join(REPO, "baseline", "_ref"), REPO]
import gaes
from gaes import parallel, aes_cbc, backend
from paper_1506_08503_b200 import plugin
plugin.register(select=True)
rng = np.random.default_rng(5)
key = rng.bytes(16)
ivs = gaes.IVSet.shared(rng.bytes(16))
n = 1_000_000
data = rng.integers(0, 256, (n, 16), dtype=np.uint8)
def t(label, fn, reps=5):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); ts.append(time.perf_counter() - t0)
    print(f"{label}: {statistics.median(ts) * 1e3:.2f} ms")
t("_encrypt_tables", lambda: aes_cbc._encrypt_tables(key))
t("ivs.rows", lambda: ivs.rows(n))
tables = aes_cbc._encrypt_tables(key)
ivr = ivs.rows(n)
out = np.empty_like(data)
t("backend.cbc_encrypt fresh out", lambda: backend.cbc_encrypt(data, ivr, *tables, np.empty_like(data)))
t("backend.cbc_encrypt reused", lambda: backend.cbc_encrypt(data, ivr, *tables, out))
t("backend.cbc_encrypt reused again", lambda: backend.cbc_encrypt(data, ivr, *tables, out), reps=20)
t("backend.cbc_encrypt fresh out again", lambda: backend.cbc_encrypt(data, ivr, *tables, np.empty_like(data)))
t("backend.cbc_encrypt fresh ivrows+out", lambda: backend.cbc_encrypt(data, ivs.rows(n), *tables, np.empty_like(data)))
from concurrent.futures import ThreadPoolExecutor
def in_thread():
    with ThreadPoolExecutor(max_workers=1) as pool:
        pool.submit(lambda: backend.cbc_encrypt(data, ivr, *tables, out)).result()
t("backend.cbc_encrypt from a worker thread", in_thread)
print("ivr flags", ivr.flags.c_contiguous, ivr.strides, ivr.base is not None)
