"""Full-size bit-exactness for configs 3, 4 and 5 (4 GiB, 1 GiB, 16 GiB).

The C oracle restates the reference byte by byte and is far too slow for
billions of blocks, so full-size checks use OpenSSL (``cryptography``, AES-NI)
as a second, fast oracle -- SURVEY.md 8(c): in the reference's mode with
M = 16 and a shared IV, ``C = AES-ECB_K(P ^ IV)``.  OpenSSL is pinned first:
it must reproduce the config-1 ciphertext digest that the reference's own
compiled kernel produced (tests/golden/golden.json).  Test-only dependency.
"""

import hashlib
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)
ciphers = pytest.importorskip("cryptography.hazmat.primitives.ciphers")

import bench  # noqa: E402
from paper_1506_08503_b200 import device  # noqa: E402

CHUNK = 1 << 22  # blocks per OpenSSL call


def _ecb(key: bytes, data: np.ndarray) -> np.ndarray:
    enc = ciphers.Cipher(ciphers.algorithms.AES(key), ciphers.modes.ECB()).encryptor()
    return np.frombuffer(enc.update(data.tobytes()) + enc.finalize(), np.uint8).reshape(-1, 16)


def _openssl_matches(key: bytes, iv: np.ndarray, p: np.ndarray, c: np.ndarray) -> bool:
    """C == ECB_K(P ^ IV) over all rows, chunked across host threads."""
    iv = np.frombuffer(bytes(iv), np.uint8)

    def part(lo):
        hi = min(p.shape[0], lo + CHUNK)
        return np.array_equal(_ecb(key, p[lo:hi] ^ iv), c[lo:hi])

    with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
        return all(pool.map(part, range(0, p.shape[0], CHUNK)))


def test_openssl_is_pinned_to_the_reference(golden_meta):
    d = golden_meta["digests"]["65536"]
    rng = np.random.default_rng(2016)
    key, iv = rng.bytes(16), rng.bytes(16)
    p = rng.integers(0, 256, (1 << 16, 16), dtype=np.uint8)
    c = _ecb(key, p ^ np.frombuffer(iv, np.uint8))
    assert hashlib.sha256(c.tobytes()).hexdigest() == d["sha256_c"]


@pytest.mark.parametrize("cfg", [3, 4])
def test_full_size_single_key_configs(cfg):
    dev = torch.device("cuda", 0)
    inp = bench.make_inputs(cfg, 0, 1, dev)
    p = inp["p"]
    rk = device.expand_key(inp["key"])
    c = device.BlockCipher(rk, inp["iv"]).encrypt(p)
    ph, chost = p.cpu().numpy(), c.cpu().numpy()
    assert ph.shape[0] == bench.WORKLOADS[cfg]["blocks"]
    assert _openssl_matches(inp["key"], np.frombuffer(inp["iv"], np.uint8), ph, chost)
    if cfg == 4:  # deterministic encryption: #unique(C) == #unique(P)
        up = torch.unique(p.view(torch.int64), dim=0).shape[0]
        uc = torch.unique(c.view(torch.int64), dim=0).shape[0]
        assert up == uc and up <= 10 ** 6
    back = device.BlockCipher(rk, inp["iv"]).decrypt(c, out=c)
    assert torch.equal(back, p)
    del p, c, back
    torch.cuda.empty_cache()


def test_full_size_many_key_config5(oracle):
    dev = torch.device("cuda", 0)
    inp = bench.make_inputs(5, 0, 1, dev)
    p, keys, ivs, bpk = inp["p"], inp["keys"], inp["ivs"], inp["bpk"]
    rk_enc, rk_dec = device.expand_keys(torch.from_numpy(keys).to(dev))
    # all 1024 GPU round-key schedules vs gen_keys (the oracle is pinned to it)
    assert np.array_equal(rk_enc.cpu().numpy(), oracle.gen_keys_batch(keys))
    d_ivs = torch.from_numpy(ivs).to(dev)
    c = device.many_key_encrypt(p, rk_enc, d_ivs)
    ok = True
    for lo in range(0, keys.shape[0], 64):  # 64 keys (1 GiB) at a time on the host
        rows = slice(lo * bpk, (lo + 64) * bpk)
        ph, ch = p[rows].cpu().numpy(), c[rows].cpu().numpy()

        def one(i):
            r = slice((i - lo) * bpk, (i - lo + 1) * bpk)
            return np.array_equal(_ecb(keys[i].tobytes(), ph[r] ^ ivs[i]), ch[r])

        with ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 1)) as pool:
            ok &= all(pool.map(one, range(lo, lo + 64)))
    assert ok
    back = device.many_key_decrypt(c, rk_dec, d_ivs, out=c)
    assert torch.equal(back, p)
    del p, c, back
    torch.cuda.empty_cache()
