"""Timeline of the staged host pipeline (GAES_TRACE): per chunk, when its
H2D / kernel / D2H finish on the device, for the bench's e2e call (256 MiB,
pinned in/out, shared IV).  Prints per-engine busy time and gaps."""
import csv, os, sys, time
sys.path.insert(0, ".")
path = os.path.abspath(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/e2e_trace.csv")
os.environ["GAES_TRACE"] = path
import torch
from paper_1506_08503_b200 import device, backend_cuda

n = 1 << 24
h_in = torch.randint(0, 256, (n, 16), dtype=torch.uint8).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
rk = device.expand_key(bytes(16))
hi, ho = h_in.numpy(), h_out.numpy()
for _ in range(3):
    backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho)
if os.path.exists(path):
    os.remove(path)
ts = []
for _ in range(3):
    t0 = time.perf_counter(); backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho); ts.append(time.perf_counter() - t0)
print("wall ms", [round(t * 1e3, 3) for t in ts], "GB/s", round(n * 16 / min(ts) / 1e9, 2))
rows = [r for r in csv.reader(open(path)) if r and r[0] != "chunk"]
last = rows[-len(rows) // 3:]
for r in last:
    print(r)
