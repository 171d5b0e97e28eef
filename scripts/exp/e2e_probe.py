"""What bounds e2e?  Pinned 256 MiB in/out through chunked H2D -> encrypt -> D2H
pipelines with torch streams (same shape as the library's host pipeline),
varying chunk size / stream count / kernel on-off."""
import sys, time
import torch
sys.path.insert(0, ".")
from paper_1506_08503_b200 import device, backend_cuda

n = 1 << 24
h_in = torch.randint(0, 256, (n, 16), dtype=torch.uint8).pin_memory()
h_out = torch.empty_like(h_in).pin_memory()
rk = device.expand_key(bytes(16))
bc = device.BlockCipher(rk, bytes(16))

def pipeline(chunk_mb, nstreams, kernel=True):
    rows = (chunk_mb << 20) // 16
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    d_in = [torch.empty((rows, 16), dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    d_out = [torch.empty((rows, 16), dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    def run():
        for ci, r0 in enumerate(range(0, n, rows)):
            k = ci % nstreams
            s = streams[k]
            r = min(rows, n - r0)
            with torch.cuda.stream(s):
                d_in[k][:r].copy_(h_in[r0:r0 + r], non_blocking=True)
                if kernel:
                    bc.encrypt(d_in[k][:r], out=d_out[k][:r])
                    h_out[r0:r0 + r].copy_(d_out[k][:r], non_blocking=True)
                else:
                    h_out[r0:r0 + r].copy_(d_in[k][:r], non_blocking=True)
        torch.cuda.synchronize()
    run()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); run(); ts.append(time.perf_counter() - t0)
    return n * 16 / min(ts) / 1e9

for mb in (8, 16, 32, 64):
    for ns in (2, 4):
        print(f"chunk {mb} MB streams {ns}: copy-only {pipeline(mb, ns, False):.1f}  with kernel {pipeline(mb, ns, True):.1f} GB/s")
hi, ho = h_in.numpy(), h_out.numpy()
backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho)
ts = []
for _ in range(5):
    t0 = time.perf_counter(); backend_cuda.encrypt_shared_iv(hi, bytes(16), rk, out=ho); ts.append(time.perf_counter() - t0)
print(f"library gaes_encrypt_shared_iv: {n * 16 / min(ts) / 1e9:.1f} GB/s (best of 5)")
