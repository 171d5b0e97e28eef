"""Exercise every kernel once at small, ragged sizes (for compute-sanitizer)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from oracle import oracle  # noqa: E402
from paper_1506_08503_b200 import _lib, backend_cuda, container, device  # noqa: E402

rng = np.random.default_rng(1)
key, iv = rng.bytes(16), rng.bytes(16)
rk = oracle.gen_keys(key)
for n in (1, 33, 5000):
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    x = torch.from_numpy(p).cuda()
    c = device.encrypt_blocks(x, rk, iv)
    assert torch.equal(device.decrypt_blocks(c, rk, iv), x)
    _lib.check(_lib.lib().gaes_set_variant(2))
    assert torch.equal(device.encrypt_blocks(x, rk, iv), c)
    _lib.check(_lib.lib().gaes_set_variant(0))
for blocks in (2, 3):
    p = rng.integers(0, 256, (777, 16 * blocks), dtype=np.uint8)
    ivs = rng.integers(0, 256, (777, 16), dtype=np.uint8)
    x = torch.from_numpy(p).cuda()
    c = device.cbc_encrypt(x, rk, torch.from_numpy(ivs).cuda())
    assert torch.equal(device.cbc_decrypt(c, rk, torch.from_numpy(ivs).cuda()), x)
    out = np.empty_like(p)
    backend_cuda.cbc_encrypt(p, ivs, *oracle.encrypt_tables(key), out)
    perm = np.ascontiguousarray(rng.permutation(16).astype(np.uint8))
    t = oracle.encrypt_tables(key)
    backend_cuda.cbc_encrypt(p, ivs, t[0], t[1], t[2], perm, out)  # generic kernel
keys = torch.from_numpy(rng.integers(0, 256, (5, 16), dtype=np.uint8)).cuda()
rke, rkd = device.expand_keys(keys)
x = torch.from_numpy(rng.integers(0, 256, (5 * 77, 16), dtype=np.uint8)).cuda()
assert torch.equal(device.many_key_decrypt(device.many_key_encrypt(x, rke), rkd), x)
blob = container.encrypt_records(b"a\nbb\nccc\n", key, iv=iv)
assert container.decrypt_container(blob, key) == b"a\nbb\nccc\n"
torch.cuda.synchronize()
print("sanitize smoke ok")
