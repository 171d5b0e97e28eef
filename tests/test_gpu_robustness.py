"""Robustness of the C ABI on the GPU:

* buffers that are not 16-byte aligned -- pinned host buffers at odd offsets
  (no zero-copy launch for them) and CUDA tensors at odd offsets on every
  device entry point (private aligned copies) -- give oracle-exact results
  and leave the CUDA context healthy;
* the texture cache recognises a buffer freed and re-allocated at the same
  address as a new allocation;
* caller tables for the byte-level generic kernel are ordered before it;
* the in-process multi-GPU dispatcher stages its shards on per-device copy
  pools in parallel, on persistent runner threads, and each many-key shard
  expands only its own keys.
"""

import os
import subprocess
import sys
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1506_08503_b200 import _lib, backend_cuda, device  # noqa: E402

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _odd_cuda(shape, offset, src=None):
    """A contiguous uint8 CUDA view starting `offset` bytes into an allocation."""
    n = int(np.prod(shape))
    buf = torch.zeros(n + 64, dtype=torch.uint8, device="cuda")
    v = buf[offset:offset + n].view(*shape)
    if src is not None:
        v.copy_(src if isinstance(src, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(src)))
    assert v.data_ptr() % 16 == offset % 16
    return v


def _odd_pinned(shape, offset, src=None):
    n = int(np.prod(shape))
    buf = torch.zeros(n + 64, dtype=torch.uint8).pin_memory()
    a = buf.numpy()[offset:offset + n].reshape(shape)
    if src is not None:
        a[...] = src
    return a, buf  # keep the pinned tensor alive


@pytest.mark.parametrize("offset", [1, 4, 8, 15])
def test_pinned_odd_offsets_take_the_staged_path(oracle, offset):
    rng = np.random.default_rng(offset)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    for n, m in ((1, 16), (4099, 16), (1001, 64)):
        p = rng.integers(0, 256, (n, m), dtype=np.uint8)
        ivrows = rng.integers(0, 256, (n, 16), dtype=np.uint8)
        hp, keep_p = _odd_pinned((n, m), offset, p)
        hiv, keep_iv = _odd_pinned((n, 16), (offset * 3) % 16, ivrows)
        ho, keep_o = _odd_pinned((n, m), (offset * 5) % 16)
        backend_cuda.cbc_encrypt(hp, hiv, *oracle.encrypt_tables(key), ho)
        assert np.array_equal(ho, oracle.encrypt(key, ivrows, p)), (n, m)
        shared = backend_cuda.encrypt_shared_iv(hp, iv, rk, out=ho)
        assert np.array_equal(shared, oracle.encrypt(key, np.tile(np.frombuffer(iv, np.uint8), (n, 1)), p))
    # the context is still healthy: an aligned zero-copy call works
    x = torch.from_numpy(rng.integers(0, 256, (64, 16), dtype=np.uint8)).pin_memory()
    y = torch.empty_like(x).pin_memory()
    backend_cuda.encrypt_shared_iv(x.numpy(), iv, rk, out=y.numpy())
    torch.cuda.synchronize()


@pytest.mark.parametrize("offset", [1, 3, 8])
def test_device_entry_points_at_odd_offsets(oracle, offset):
    rng = np.random.default_rng(100 + offset)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    n = 70001
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    want = oracle.encrypt(key, np.tile(np.frombuffer(iv, np.uint8), (n, 1)), p, threads=4)
    x = _odd_cuda((n, 16), offset, p)
    out = _odd_cuda((n, 16), (offset * 7) % 16 or 5)
    c = device.encrypt_blocks(x, rk, iv, out=out)
    assert np.array_equal(c.cpu().numpy(), want)
    back = _odd_cuda((n, 16), (offset * 3) % 16 or 9)
    device.decrypt_blocks(c, rk, iv, out=back)
    assert torch.equal(back, x)
    bc = device.BlockCipher(rk, iv)
    assert np.array_equal(bc.encrypt(x, out=_odd_cuda((n, 16), 2)).cpu().numpy(), want)

    # general-M CBC with misaligned per-message IVs
    rows, m = 5003, 64
    pr = rng.integers(0, 256, (rows, m), dtype=np.uint8)
    ivs = rng.integers(0, 256, (rows, 16), dtype=np.uint8)
    xr = _odd_cuda((rows, m), offset, pr)
    d_ivs = _odd_cuda((rows, 16), (offset + 5) % 16 or 1, ivs)
    cr = device.cbc_encrypt(xr, rk, d_ivs, out=_odd_cuda((rows, m), 11))
    assert np.array_equal(cr.cpu().numpy(), oracle.encrypt(key, ivs, pr))
    dr = device.cbc_decrypt(cr, rk, d_ivs, out=_odd_cuda((rows, m), 6))
    assert torch.equal(dr, xr)
    x16 = _odd_cuda((rows, 16), offset, pr[:, :16])
    c16 = device.cbc_encrypt(x16, rk, d_ivs)
    assert np.array_equal(c16.cpu().numpy(), oracle.encrypt(key, ivs, pr[:, :16]))

    # key schedule into misaligned outputs; many-key with misaligned keys / IVs / data
    keys = rng.integers(0, 256, (5, 16), dtype=np.uint8)
    d_keys = _odd_cuda((5, 16), offset, keys)
    rke = _odd_cuda((5, 11, 16), (offset + 1) % 16 or 2)
    rkd = _odd_cuda((5, 11, 16), (offset + 2) % 16 or 3)
    _lib.check(_lib.lib().gaes_expand_keys_dev(d_keys.data_ptr(), 5, rke.data_ptr(), rkd.data_ptr(),
                                               device._stream()))
    assert np.array_equal(rke.cpu().numpy(), oracle.gen_keys_batch(keys))
    kivs = rng.integers(0, 256, (5, 16), dtype=np.uint8)
    bpk = 999
    pm = rng.integers(0, 256, (5 * bpk, 16), dtype=np.uint8)
    cm = device.many_key_encrypt(_odd_cuda((5 * bpk, 16), offset, pm), rke, _odd_cuda((5, 16), 7, kivs),
                                 out=_odd_cuda((5 * bpk, 16), 13))
    for i in (0, 4):
        rows_i = slice(i * bpk, (i + 1) * bpk)
        assert np.array_equal(cm[rows_i].cpu().numpy(),
                              oracle.encrypt(keys[i].tobytes(), np.tile(kivs[i], (bpk, 1)), pm[rows_i]))
    back_m = device.many_key_decrypt(cm, rkd, _odd_cuda((5, 16), 3, kivs))
    assert np.array_equal(back_m.cpu().numpy(), pm)
    torch.cuda.synchronize()


def test_many_key_round_keys_on_another_device_raise():
    x = torch.zeros((16, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        device.many_key_encrypt(x, torch.zeros((1, 11, 16), dtype=torch.uint8))  # host tensor
    if torch.cuda.device_count() > 1:
        rk = torch.zeros((1, 11, 16), dtype=torch.uint8, device="cuda:1")
        with pytest.raises(ValueError, match="device"):
            device.many_key_encrypt(x, rk)


def test_texture_cache_sees_a_reallocated_buffer(oracle):
    """Encrypt, free the input (returned to the driver), allocate until a new
    buffer lands at the same address, encrypt again: the cached texture over
    the freed allocation is replaced, and the bytes are right."""
    rng = np.random.default_rng(5)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    n = (8 << 20) // 16  # its own 8 MiB segment in torch's caching allocator
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    p1 = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    x = torch.from_numpy(p1).cuda()
    addr = x.data_ptr()
    assert np.array_equal(device.encrypt_blocks(x, rk, iv).cpu().numpy(), oracle.encrypt(key, ivrows, p1, threads=4))
    before = _lib.debug_counters()["textures_created"]
    del x
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    keep, y = [], None
    for _ in range(64):
        t = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
        if t.data_ptr() == addr:
            y = t
            break
        keep.append(t)
    if y is None:
        pytest.skip("the allocator never returned the same address")
    p2 = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    y.copy_(torch.from_numpy(p2))
    c = device.encrypt_blocks(y, rk, iv)
    assert np.array_equal(c.cpu().numpy(), oracle.encrypt(key, ivrows, p2, threads=4))
    assert _lib.debug_counters()["textures_created"] > before  # a new texture, not the stale one


def test_generic_tables_are_ordered_before_the_kernel(oracle):
    """Alternating non-standard table sets (byte-level generic kernel) on one
    lane, back to back: each call must use its own tables."""
    rng = np.random.default_rng(9)
    key = rng.bytes(16)
    rk, box, lut, perm = oracle.encrypt_tables(key)
    perms = [np.ascontiguousarray(np.roll(perm, k)) for k in (1, 2, 3)]  # non-standard ShiftRows
    n, m = 3001, 32
    p = rng.integers(0, 256, (n, m), dtype=np.uint8)
    ivrows = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    wants = []
    for q in perms:
        w = np.empty_like(p)
        oracle.cbc_encrypt(p, ivrows, rk, box, lut, q, w)
        wants.append(w)
    for rep in range(6):
        for q, w in zip(perms, wants):
            out = np.empty_like(p)
            backend_cuda.cbc_encrypt(p, ivrows, rk, box, lut, q, out)
            assert np.array_equal(out, w), rep


def test_sharded_pageable_staging_runs_per_device_pools_in_parallel():
    """GAES_DEVICE_MAP=0,0 (two logical GPUs on this one): a pageable 2-shard
    job stages both shards at once on their own pools (max concurrent copy
    regions >= 2), shard runners are persistent (no new threads on repeat
    calls), results are bit-exact, and a 2-shard many-key job expands 4 + 4
    of its 7 keys (the key split by the shard boundary on both sides)
    instead of 7 + 7."""
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from oracle import oracle
from paper_1506_08503_b200 import _lib, backend_cuda
assert _lib.device_count() == 2
assert _lib.set_num_gpus(2) == 2
rng = np.random.default_rng(3)
key = rng.bytes(16)
n = (256 << 20) // 16
p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
ivrows = rng.integers(0, 256, (n, 16), dtype=np.uint8)
out = np.empty_like(p)
for _ in range(3):
    backend_cuda.cbc_encrypt(p, ivrows, *oracle.encrypt_tables(key), out)
c = _lib.debug_counters()
rows = rng.choice(n, 4096, replace=False)
assert np.array_equal(out[rows], oracle.encrypt(key, ivrows[rows], p[rows])), "bytes"
assert c["pools"] >= 3, c  # the process pool + one per logical device
assert c["max_concurrent_regions"] >= 2, c
runners = c["shard_runner_threads"]
assert 1 <= runners <= 4, c
for _ in range(3):
    backend_cuda.cbc_encrypt(p, ivrows, *oracle.encrypt_tables(key), out)
assert _lib.debug_counters()["shard_runner_threads"] == runners
keys = rng.integers(0, 256, (7, 16), dtype=np.uint8)
kivs = rng.integers(0, 256, (7, 16), dtype=np.uint8)
bpk = 10001
pm = rng.integers(0, 256, (7 * bpk, 16), dtype=np.uint8)
k0 = _lib.debug_counters()["keys_expanded"]
cm = backend_cuda.many_key_encrypt(pm, keys, kivs)
assert _lib.debug_counters()["keys_expanded"] - k0 == 8, _lib.debug_counters()
for i in range(7):
    r = slice(i * bpk, (i + 1) * bpk)
    assert np.array_equal(cm[r], oracle.encrypt(keys[i].tobytes(), np.tile(kivs[i], (bpk, 1)), pm[r])), i
assert np.array_equal(backend_cuda.many_key_decrypt(cm, keys, kivs), pm)
print("ok", c)
'''
    env = dict(os.environ, GAES_DEVICE_MAP="0,0")
    r = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr


def test_concurrent_callers_with_the_new_pool(oracle):
    """8 threads of pageable drop-in calls (the reference's
    parallel._run_chunks pattern) on the ticketed copy pool: bit-exact."""
    rng = np.random.default_rng(77)
    key = rng.bytes(16)
    tables = oracle.encrypt_tables(key)
    n = (8 << 20) // 16
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    ivrows = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    want = oracle.encrypt(key, ivrows, p, threads=8)
    errors = []

    def work(t):
        lo, hi = t * n // 8, (t + 1) * n // 8
        for _ in range(4):
            out = np.empty((hi - lo, 16), np.uint8)
            backend_cuda.cbc_encrypt(p[lo:hi], ivrows[lo:hi], *tables, out)
            if not np.array_equal(out, want[lo:hi]):
                errors.append(t)

    th = [threading.Thread(target=work, args=(t,)) for t in range(8)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errors


def test_sharded_calls_from_many_threads():
    """Six caller threads on the 2-shard path at once (more callers than a
    device's 4 runner threads / lanes): every result bit-exact, no deadlock."""
    code = r'''
import sys, threading, numpy as np
sys.path.insert(0, ".")
from oracle import oracle
from paper_1506_08503_b200 import _lib, backend_cuda
assert _lib.set_num_gpus(2) == 2
rng = np.random.default_rng(11)
key = rng.bytes(16)
tables = oracle.encrypt_tables(key)
jobs = []
for t in range(6):
    n = 50000 + 977 * t
    p = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    jobs.append((p, ivs, oracle.encrypt(key, ivs, p, threads=2)))
bad = []
def work(t):
    p, ivs, want = jobs[t]
    for _ in range(5):
        out = np.empty_like(p)
        backend_cuda.cbc_encrypt(p, ivs, *tables, out)
        if not np.array_equal(out, want):
            bad.append(t)
th = [threading.Thread(target=work, args=(t,)) for t in range(6)]
[x.start() for x in th]
[x.join() for x in th]
assert not bad, bad
print("ok", _lib.debug_counters()["shard_runner_threads"])
'''
    env = dict(os.environ, GAES_DEVICE_MAP="0,0")
    r = subprocess.run([sys.executable, "-c", code], cwd=REPO, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stdout + r.stderr
