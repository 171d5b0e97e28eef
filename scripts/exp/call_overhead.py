"""Host-side cost per device-API call (small batches are launch-bound)."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1506_08503_b200 import device  # noqa: E402

x = torch.randint(0, 256, (1024, 16), dtype=torch.uint8, device="cuda")
out = torch.empty_like(x)
bc = device.BlockCipher(device.expand_key(bytes(16)), bytes(16))
for _ in range(100):
    bc.encrypt(x, out=out)
torch.cuda.synchronize()
N = 2000
t0 = time.perf_counter()
for _ in range(N):
    bc.encrypt(x, out=out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"enqueue {1e6 * (t1 - t0) / N:.2f} us/call, total {1e6 * (t2 - t0) / N:.2f} us/call")


def per_call(fn, n=20000):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return 1e6 * (time.perf_counter() - t0) / n


from paper_1506_08503_b200 import _lib  # noqa: E402

L = _lib.lib()
s = torch.cuda.current_stream().cuda_stream
print(f"torch.cuda.current_stream().cuda_stream: {per_call(lambda: torch.cuda.current_stream().cuda_stream):.2f} us")
print(f"torch.cuda.current_device(): {per_call(lambda: torch.cuda.current_device()):.2f} us")
print(f"tensor checks: {per_call(lambda: (x.is_cuda, x.dtype, x.dim(), x.shape[1], x.is_contiguous(), x.data_ptr(), x.device.index)):.2f} us")
print(f"raw ctypes launch: {per_call(lambda: L.gaes_encrypt_blocks_dev(x.data_ptr(), out.data_ptr(), 1024, bc._rk_p, bc._iv_p, s), 5000):.2f} us")
torch.cuda.synchronize()
print(f"gaes_version (ctypes floor): {per_call(lambda: L.gaes_version()):.2f} us")
if hasattr(torch._C, "_cuda_getCurrentRawStream"):
    f = torch._C._cuda_getCurrentRawStream
    print(f"torch._C._cuda_getCurrentRawStream(0): {per_call(lambda: f(0)):.2f} us, equal: {f(0) == torch.cuda.current_stream().cuda_stream}")
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        print("inside stream ctx equal:", f(0) == st.cuda_stream)
print(f"x.device.index: {per_call(lambda: x.device.index):.2f} us; x.get_device(): {per_call(lambda: x.get_device()):.2f} us")
