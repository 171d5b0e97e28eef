"""Small batches (VERDICT r1 "Next round" #3): the small-batch kernel
k_blocks_small (64 KiB of tables filled from the kernel parameters, T2/T3 as
16-bit rotations of T0/T1) and the single-kernel path for small pageable
host jobs (the kernel reads / writes the pinned staging buffers over PCIe),
bit-exact against the oracle around every size boundary."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1506_08503_b200 import _lib, backend_cuda, device  # noqa: E402

SMS = torch.cuda.get_device_properties(0).multi_processor_count
SMALL_MAX = 3 * SMS * 512


@pytest.mark.parametrize("n", [1, 31, 32, 33, 127, 511, 512, 513, 4095, SMS * 128 + 7, 1 << 16, SMS * 512,
                               SMS * 512 + 1, SMALL_MAX - 1, SMALL_MAX, SMALL_MAX + 1])
def test_small_batch_kernel_sizes(oracle, n):
    rng = np.random.default_rng(n)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    x = torch.from_numpy(p).cuda()
    c = device.encrypt_blocks(x, rk, iv)
    torch.cuda.synchronize()
    want_kernel = "k_blocks_small_enc" if n <= SMALL_MAX else "k_blocks_enc_folded+texsbox"
    if _lib.lib().gaes_uses_sbox_texture(0) == 1:
        assert _lib.last_kernel() == want_kernel
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    assert np.array_equal(c.cpu().numpy(), oracle.encrypt(key, ivrows, p, threads=4))
    back = device.decrypt_blocks(c, rk, iv)
    torch.cuda.synchronize()
    if _lib.lib().gaes_uses_sbox_texture(0) == 1:
        assert _lib.last_kernel() == ("k_blocks_small_dec" if n <= SMALL_MAX else "k_blocks_dec_folded")
    assert torch.equal(back, x)


def test_small_batch_kernel_back_to_back_launches(oracle):
    """Consecutive small launches on one stream overlap (PDL: the next
    launch fills its tables while the previous one computes, and reads its
    input only after griddepcontrol.wait): a chain where each launch
    encrypts the previous launch's output must equal 8 sequential
    encryptions."""
    rng = np.random.default_rng(8)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    n = 1 << 16
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    bufs = [torch.from_numpy(p).cuda()] + [torch.empty((n, 16), dtype=torch.uint8, device="cuda") for _ in range(8)]
    bc = device.BlockCipher(rk, iv)
    for i in range(8):
        bc.encrypt(bufs[i], out=bufs[i + 1])
    want = p
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    for _ in range(8):
        want = oracle.encrypt(key, ivrows, want, threads=4)
    assert np.array_equal(bufs[8].cpu().numpy(), want)


def test_small_batch_kernel_in_a_cuda_graph(oracle):
    rng = np.random.default_rng(9)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    n, k = 4099, 6
    p = torch.from_numpy(rng.integers(0, 256, (k, n, 16), dtype=np.uint8)).cuda()
    out = torch.empty_like(p)
    bc = device.BlockCipher(rk, iv)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        bc.encrypt(p[0], out=out[0])
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for i in range(k):
            bc.encrypt(p[i], out=out[i])
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    for i in (0, k - 1):
        assert np.array_equal(out[i].cpu().numpy(), oracle.encrypt(key, ivrows, p[i].cpu().numpy()))


@pytest.mark.parametrize("n,m,shared", [(1, 16, True), (3, 16, False), (1000, 16, True), (1000, 16, False),
                                        (1 << 16, 16, True), ((1 << 16) + 1, 16, True), (4096, 64, False),
                                        (4096, 64, True), (16384, 64, True), (16385, 64, False)])
def test_small_pageable_host_jobs(oracle, n, m, shared):
    """Pageable drop-in calls up to 1 MiB run as one kernel on the pinned
    staging buffers; just above, the staged DMA pipeline -- same bytes."""
    rng = np.random.default_rng(n + m)
    key = rng.bytes(16)
    p = rng.integers(0, 256, (n, m), dtype=np.uint8)
    if shared:
        ivrows = np.tile(rng.integers(0, 256, 16, dtype=np.uint8), (n, 1))
    else:
        ivrows = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    out = np.empty_like(p)
    backend_cuda.cbc_encrypt(p, ivrows, *oracle.encrypt_tables(key), out)
    assert np.array_equal(out, oracle.encrypt(key, ivrows, p, threads=4))
    back = np.empty_like(p)
    backend_cuda.cbc_decrypt(out, ivrows, *oracle.decrypt_tables(key), back)
    assert np.array_equal(back, p)
    rk = oracle.gen_keys(key)
    iv = ivrows[0].tobytes()
    if shared:
        assert np.array_equal(backend_cuda.encrypt_shared_iv(p, iv, rk), out)
