"""Wall-clock A/B of the library's pinned e2e call (256 MiB shared-IV
encrypt through gaes_encrypt_shared_iv): median of 15 calls."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1506_08503_b200 import device, backend_cuda
n = 1 << 24
h_in = torch.randint(0, 256, (n, 16), dtype=torch.uint8).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
rk = device.expand_key(bytes(16))
hi, ho = h_in.numpy(), h_out.numpy()
for _ in range(3):
    backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho)
ts = []
for _ in range(15):
    t0 = time.perf_counter(); backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho); ts.append(time.perf_counter() - t0)
ts.sort()
print(" ".join(sys.argv[1:]), f"median {ts[7]*1e3:.3f} ms = {n*16/ts[7]/1e9:.2f} GB/s, best {n*16/ts[0]/1e9:.2f}")
