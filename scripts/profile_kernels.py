"""Run one hot-path op a few times on cuda:0 (a small target for ncu).

    python scripts/profile_kernels.py {encrypt,decrypt,bitsliced,manykey,cbc_rows,cbc_dec_rows,rowiv_enc,rowiv_dec} [log2_blocks] [bpr]
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1506_08503_b200 import _lib, device  # noqa: E402

op = sys.argv[1]
n = 1 << int(sys.argv[2] if len(sys.argv) > 2 else 24)
bpr = int(sys.argv[3]) if len(sys.argv) > 3 else 64  # blocks per row for the cbc_* ops
rng = np.random.default_rng(2016)
key, iv = rng.bytes(16), rng.bytes(16)
rk = device.expand_key(key)
x = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device="cuda")
ivs = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device="cuda") if op.startswith("rowiv") else None
def run():
    if op == "encrypt":
        device.encrypt_blocks(x, rk, iv)
    elif op == "decrypt":
        device.decrypt_blocks(x, rk, iv)
    elif op == "bitsliced":
        _lib.check(_lib.lib().gaes_set_variant(2))
        device.encrypt_blocks(x, rk, iv)
    elif op == "cbc_rows":  # general-M CBC encrypt, bpr-block rows
        device.cbc_encrypt(x.view(n // bpr, bpr * 16), rk, iv)
    elif op == "cbc_dec_rows":
        device.cbc_decrypt(x.view(n // bpr, bpr * 16), rk, iv)
    elif op == "rowiv_enc":  # M = 16 with per-message IVs (IVSet.per_message)
        device.cbc_encrypt(x, rk, ivs)
    elif op == "rowiv_dec":
        device.cbc_decrypt(x, rk, ivs)


if op == "manykey":
    keys = torch.randint(0, 256, (1024, 16), dtype=torch.uint8, device="cuda")
    rke, _ = device.expand_keys(keys, with_decrypt=False)

    def run():  # noqa: F811
        device.many_key_encrypt(x, rke)
for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    run()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print("ok", op, n, f"{ms * 1e3:.1f} us", f"{n * 16 / ms / 1e6:.1f} GB/s")
