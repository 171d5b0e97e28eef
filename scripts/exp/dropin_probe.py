"""Where does the time of a pageable drop-in call (backend_cuda.cbc_encrypt,
the reference's 7-argument contract) go at small and large N?"""
import statistics
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_1506_08503_b200 import _lib, backend_cuda  # noqa: E402

rng = np.random.default_rng(1)
rk = rng.integers(0, 256, (11, 16), dtype=np.uint8)
tables = (rk,) + backend_cuda.standard_tables(False)
iv = rng.integers(0, 256, 16, dtype=np.uint8)
for lg in [int(a) for a in sys.argv[1:]] or (10, 12, 14, 16, 18, 20, 22):
    n = 1 << lg
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    ivrows = np.tile(iv, (n, 1))
    out = np.empty_like(p)
    backend_cuda.cbc_encrypt(p, ivrows, *tables, out)
    ts, tc = [], []
    for _ in range(15):
        t0 = time.perf_counter()
        backend_cuda.cbc_encrypt(p, ivrows, *tables, out)
        ts.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        backend_cuda._check_args(p, ivrows, *tables, out)
        tc.append(time.perf_counter() - t0)
    med = statistics.median(ts)
    print(f"2^{lg}: call {med * 1e6:8.1f} us  ({n * 16 / med / 1e9:5.2f} GB/s)  python checks {statistics.median(tc) * 1e6:6.1f} us")
