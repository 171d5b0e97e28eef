"""Reference pad_zero / MessageBatch (per-message Python loops) vs the
vectorised paper_1506_08503_b200.batch equivalents, 16-byte messages."""
import sys, time
sys.path.insert(0, "."); sys.path.insert(0, "baseline/_ref")
import numpy as np
from gaes import aes_cbc
from paper_1506_08503_b200 import batch as B
for lg in [int(a) for a in sys.argv[1:]] or (16, 18, 20):
    n = 1 << lg
    rng = np.random.default_rng(lg)
    data = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    lens = [16] * n
    msgs = [bytes(r) for r in data[: min(n, 1 << 20)]]
    t0 = time.perf_counter(); aes_cbc.MessageBatch(data, lens); t1 = time.perf_counter()
    B.message_batch(data, lens); t2 = time.perf_counter()
    aes_cbc.pad_zero(msgs); t3 = time.perf_counter()
    B.pad_zero(msgs); t4 = time.perf_counter()
    print(f"2^{lg}: MessageBatch ref {t1-t0:.3f} s, ours {t2-t1:.3f} s; pad_zero({len(msgs)}) ref {t3-t2:.3f} s, ours {t4-t3:.3f} s")
