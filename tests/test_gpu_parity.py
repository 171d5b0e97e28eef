"""GPU parity: the CUDA path (through the C ABI) vs the oracle, bit-exact.

Mirrors the reference's hot-path tests (pkg/tests/test_aes_cbc.py,
test_backends.py, test_key_schedule.py, test_parallel.py) with the cuda
backend / device API in place of the compiled kernel, plus the north-star
configs at full size through size-independent properties.
"""

import hashlib
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_1506_08503_b200 import _lib, backend_cuda, device  # noqa: E402

NIST_KEY = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
NIST_IV = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
NIST_PT = bytes.fromhex(
    "6bc1bee22e409f96e93d7e117393172aae2d8a571e03ac9c9eb76fac45af8e51"
    "30c81c46a35ce411e5fbc1191a0a52eff69f2445df4f9b17ad2b417be66c3710")
NIST_CT = bytes.fromhex(
    "7649abac8119b246cee98e9b12e9197d5086cb9b507219ee95db113a917678b2"
    "73bed6b8e3c1743b7116e69e222295163ff1caa1681fac09120eca307586e1a7")


def _cuda_enc(key, ivrows, data, oracle):
    out = np.empty_like(data)
    backend_cuda.cbc_encrypt(data, ivrows, *oracle.encrypt_tables(key), out)
    return out


def _cuda_dec(key, ivrows, data, oracle):
    out = np.empty_like(data)
    backend_cuda.cbc_decrypt(data, ivrows, *oracle.decrypt_tables(key), out)
    return out


# ---------------------------------------------------------------- GF layer

def test_gf_layer_tables_match_oracle(oracle, golden):
    s, si, te, td = device.gf_tables(0)
    assert np.array_equal(s, golden["sbox"])
    assert np.array_equal(si, golden["inv_sbox"])
    fwd = golden["mix_fwd"]
    inv = golden["mix_inv"]
    for j in range(4):
        for x in (0, 1, 0x53, 0xFF):
            want = sum(int(fwd[r, j, s[x]]) << (8 * r) for r in range(4))
            assert te[j, x] == want
            want = sum(int(inv[r, j, si[x]]) << (8 * r) for r in range(4))
            assert td[j, x] == want
    assert te[0, 0] == 0xA56363C6  # survey probe P10


def test_tables_are_standard(oracle):
    L = _lib.lib()
    t = oracle.encrypt_tables(bytes(16))
    p = lambda a: a.__array_interface__["data"][0]  # noqa: E731
    assert L.gaes_tables_are_standard(p(t[1]), p(np.ascontiguousarray(t[2])), p(t[3]), 0) == 1
    td = oracle.decrypt_tables(bytes(16))
    assert L.gaes_tables_are_standard(p(td[1]), p(np.ascontiguousarray(td[2])), p(td[3]), 1) == 1
    bad = t[1].copy()
    bad[0] ^= 1
    assert L.gaes_tables_are_standard(p(bad), p(np.ascontiguousarray(t[2])), p(t[3]), 0) == 0


# ---------------------------------------------------------------- KATs

def test_fips197_block_kat(oracle):
    key = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
    pt = np.frombuffer(bytes.fromhex("00112233445566778899aabbccddeeff"), np.uint8).reshape(1, 16)
    iv0 = np.zeros((1, 16), np.uint8)
    ct = _cuda_enc(key, iv0, pt, oracle)
    assert ct.tobytes() == bytes.fromhex("69c4e0d86a7b0430d8cdb78070b4c55a")
    assert np.array_equal(_cuda_dec(key, iv0, ct, oracle), pt)


def test_sp800_38a_cbc_four_blocks(oracle):
    pt = np.frombuffer(NIST_PT, np.uint8).reshape(1, 64)
    iv = np.frombuffer(NIST_IV, np.uint8).reshape(1, 16)
    ct = _cuda_enc(NIST_KEY, iv, pt, oracle)
    assert ct.tobytes() == NIST_CT
    assert _cuda_dec(NIST_KEY, iv, ct, oracle).tobytes() == NIST_PT


def test_golden_cases_from_reference(oracle, golden, golden_meta):
    for case in golden_meta["cases"]:
        i = case["idx"]
        key = golden[f"case{i}_key"].tobytes()
        iv = golden[f"case{i}_iv"]
        ct = _cuda_enc(key, iv, golden[f"case{i}_pt"], oracle)
        assert np.array_equal(ct, golden[f"case{i}_ct"]), case
        assert np.array_equal(_cuda_dec(key, iv, ct, oracle), golden[f"case{i}_pt"]), case


# ---------------------------------------------------------------- backend contract

@pytest.mark.parametrize("n,blocks", [(1, 1), (3, 1), (1, 5), (17, 3), (64, 2), (5, 4), (32, 2), (1023, 1),
                                      (4097, 1), (300, 9)])
@pytest.mark.parametrize("shared", [True, False])
def test_backend_matches_oracle(oracle, n, blocks, shared):
    rng = np.random.default_rng(n * 100 + blocks + (7 if shared else 0))
    key = rng.bytes(16)
    data = rng.integers(0, 256, (n, 16 * blocks), dtype=np.uint8)
    if shared:
        ivs = np.tile(rng.integers(0, 256, 16, dtype=np.uint8), (n, 1))
    else:
        ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    want = oracle.encrypt(key, ivs, data)
    got = _cuda_enc(key, ivs, data, oracle)
    assert np.array_equal(got, want)
    assert np.array_equal(_cuda_dec(key, ivs, got, oracle), data)


def test_empty_batch_is_noop(oracle):
    data = np.empty((0, 16), np.uint8)
    out = np.empty((0, 16), np.uint8)
    backend_cuda.cbc_encrypt(data, np.empty((0, 16), np.uint8), *oracle.encrypt_tables(bytes(16)), out)


def test_nonstandard_tables_use_generic_path(oracle):
    """Any tables are honoured, like the reference kernel (tables in, no cipher knowledge)."""
    rng = np.random.default_rng(11)
    key = rng.bytes(16)
    n = 257
    data = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    rk, box, lut, perm = oracle.encrypt_tables(key)
    box2 = np.ascontiguousarray(box[rng.permutation(256)])       # another bijection
    perm2 = np.ascontiguousarray(rng.permutation(16).astype(np.uint8))  # another gather
    lut2 = np.ascontiguousarray(rng.integers(0, 256, (4, 4, 256), dtype=np.uint8))  # non-linear
    for tb in [(rk, box2, lut, perm), (rk, box, lut2, perm), (rk, box, lut, perm2), (rk, box2, lut2, perm2)]:
        want = np.empty_like(data)
        oracle.cbc_encrypt(data, ivs, *tb, want)
        got = np.empty_like(data)
        backend_cuda.cbc_encrypt(data, ivs, *tb, got)
        assert np.array_equal(got, want)
        wantd = np.empty_like(data)
        oracle.cbc_decrypt(data, ivs, *tb, wantd)
        gotd = np.empty_like(data)
        backend_cuda.cbc_decrypt(data, ivs, *tb, gotd)
        assert np.array_equal(gotd, wantd)


def test_concurrent_calls_on_disjoint_slices(oracle):
    """parallel._run_chunks calls the backend from worker threads (parallel.py:66-75)."""
    rng = np.random.default_rng(3)
    key = rng.bytes(16)
    n = 20000
    data = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    tables = oracle.encrypt_tables(key)
    out = np.empty_like(data)
    chunks = oracle.plan(n, 7)
    errs = []

    def work(lo, hi):
        try:
            backend_cuda.cbc_encrypt(data[lo:hi], ivs[lo:hi], *tables, out[lo:hi])
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=c) for c in chunks]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errs
    assert np.array_equal(out, oracle.encrypt(key, ivs, data, threads=4))


def test_pinned_host_buffers(oracle):
    rng = np.random.default_rng(12)
    key, iv = rng.bytes(16), rng.bytes(16)
    n = 1 << 18
    pin_in = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
    pin_out = torch.empty((n, 16), dtype=torch.uint8).pin_memory()
    p = pin_in.numpy()
    p[:] = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    backend_cuda.encrypt_shared_iv(p, iv, rk, out=pin_out.numpy())
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    assert np.array_equal(pin_out.numpy(), oracle.encrypt(key, ivrows, p, threads=4))
    back = backend_cuda.decrypt_shared_iv(pin_out.numpy(), iv, rk)
    assert np.array_equal(back, p)


def test_shared_iv_entry_wide_rows(oracle):
    rng = np.random.default_rng(13)
    key, iv = rng.bytes(16), rng.bytes(16)
    data = rng.integers(0, 256, (999, 48), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (999, 1))
    ct = backend_cuda.encrypt_shared_iv(data, iv, rk)
    assert np.array_equal(ct, oracle.encrypt(key, ivrows, data))
    assert np.array_equal(backend_cuda.decrypt_shared_iv(ct, iv, rk), data)


def test_argument_errors_match_reference(oracle):
    t = oracle.encrypt_tables(bytes(16))
    good = np.zeros((4, 16), np.uint8)
    ivs = np.zeros((4, 16), np.uint8)
    with pytest.raises(ValueError, match="dtype mismatch"):
        backend_cuda.cbc_encrypt(good.astype(np.float64), ivs, *t, np.empty_like(good))
    with pytest.raises(ValueError, match="C-contiguous"):
        backend_cuda.cbc_encrypt(np.zeros((4, 32), np.uint8)[:, ::2], ivs, *t, np.empty_like(good))
    ro = np.empty_like(good)
    ro.setflags(write=False)
    with pytest.raises(ValueError, match="read-only"):
        backend_cuda.cbc_encrypt(good, ivs, *t, ro)
    with pytest.raises(ValueError, match="dimensions"):
        backend_cuda.cbc_encrypt(good.reshape(-1), ivs, *t, np.empty_like(good))
    with pytest.raises(ValueError, match="multiple of 16"):
        backend_cuda.cbc_encrypt(np.zeros((4, 20), np.uint8), ivs, *t, np.zeros((4, 20), np.uint8))


# ---------------------------------------------------------------- device API

@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 148 * 1024 * 2 + 17])
def test_device_blocks_ragged_sizes(oracle, n):
    rng = np.random.default_rng(n)
    key, iv = rng.bytes(16), rng.bytes(16)
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    x = torch.from_numpy(p).cuda()
    c = device.encrypt_blocks(x, rk, iv)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    assert np.array_equal(c.cpu().numpy(), oracle.encrypt(key, ivrows, p, threads=4))
    assert np.array_equal(device.decrypt_blocks(c, rk, iv).cpu().numpy(), p)


@pytest.mark.parametrize("blocks", [1, 2, 7])
def test_device_cbc_grids(oracle, blocks):
    rng = np.random.default_rng(50 + blocks)
    key = rng.bytes(16)
    n = 3001
    p = rng.integers(0, 256, (n, 16 * blocks), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    x = torch.from_numpy(p).cuda()
    d_ivs = torch.from_numpy(ivs).cuda()
    c = device.cbc_encrypt(x, rk, d_ivs)
    assert np.array_equal(c.cpu().numpy(), oracle.encrypt(key, ivs, p))
    assert np.array_equal(device.cbc_decrypt(c, rk, d_ivs).cpu().numpy(), p)
    iv = rng.bytes(16)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    c2 = device.cbc_encrypt(x, rk, iv)
    assert np.array_equal(c2.cpu().numpy(), oracle.encrypt(key, ivrows, p))
    assert np.array_equal(device.cbc_decrypt(c2, rk, iv).cpu().numpy(), p)


# ---------------------------------------------------------------- key schedule

def test_gpu_key_schedule_matches_reference(oracle, golden):
    keys = torch.from_numpy(golden["keys"]).cuda()
    rk_enc, rk_dec = device.expand_keys(keys)
    assert np.array_equal(rk_enc.cpu().numpy(), golden["round_keys"])
    # decrypt form: rows 1..9 are InvMixColumns of the forward rows
    inv = golden["mix_inv"]
    d = rk_dec.cpu().numpy()
    e = golden["round_keys"]
    assert np.array_equal(d[:, 0], e[:, 0]) and np.array_equal(d[:, 10], e[:, 10])
    for k in (0, 5, 200):
        for r in range(1, 10):
            for c in range(4):
                col = e[k, r, 4 * c:4 * c + 4]
                want = [inv[row, 0, col[0]] ^ inv[row, 1, col[1]] ^ inv[row, 2, col[2]] ^ inv[row, 3, col[3]]
                        for row in range(4)]
                assert list(d[k, r, 4 * c:4 * c + 4]) == want


def test_gpu_key_schedule_1000_random_keys(oracle):
    rng = np.random.default_rng(1000)
    keys = rng.integers(0, 256, (1000, 16), dtype=np.uint8)
    rk_enc, _ = device.expand_keys(torch.from_numpy(keys).cuda(), with_decrypt=False)
    assert np.array_equal(rk_enc.cpu().numpy(), oracle.gen_keys_batch(keys))


# ---------------------------------------------------------------- north-star configs

def _cfg_inputs(n, seed=2016):
    rng = np.random.default_rng(seed)
    key, iv = rng.bytes(16), rng.bytes(16)
    return rng, key, iv


def test_config1_full_digest(oracle, golden_meta):
    d = golden_meta["digests"]["65536"]
    rng, key, iv = _cfg_inputs(1 << 16)
    p = rng.integers(0, 256, (1 << 16, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    # drop-in path: host buffers, tiled IV rows
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (p.shape[0], 1))
    c = _cuda_enc(key, ivrows, p, oracle)
    assert hashlib.sha256(c.tobytes()).hexdigest() == d["sha256_c"]
    assert np.array_equal(_cuda_dec(key, ivrows, c, oracle), p)
    # device path
    cd = device.encrypt_blocks(torch.from_numpy(p).cuda(), rk, iv).cpu().numpy()
    assert hashlib.sha256(cd.tobytes()).hexdigest() == d["sha256_c"]


def test_config2_digest_subset_and_round_trip(oracle, golden_meta):
    n = 1 << 24
    d = golden_meta["digests"][str(n)]
    rng, key, iv = _cfg_inputs(n)
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    x = torch.from_numpy(p).cuda()
    c = device.encrypt_blocks(x, rk, iv)
    ch = c.cpu().numpy()
    assert hashlib.sha256(ch.tobytes()).hexdigest() == d["sha256_c"]
    # seeded 1% subset vs the oracle (rows are independent)
    rng2 = np.random.default_rng(7)
    idx = np.sort(rng2.choice(n, n // 100, replace=False))
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (idx.size, 1))
    assert np.array_equal(ch[idx], oracle.encrypt(key, ivrows, p[idx], threads=8))
    back = device.decrypt_blocks(c, rk, iv)
    assert torch.equal(back, x)


def test_config4_determinism_equal_plaintexts(oracle):
    """Deterministic (shared-IV) encryption: equal P -> equal C, #unique preserved."""
    rng = np.random.default_rng(4)
    key, iv = rng.bytes(16), rng.bytes(16)
    vals = rng.integers(0, 2**63, 5000, dtype=np.int64).astype(np.uint64)
    ranks = rng.zipf(1.5, 200000) % vals.size
    p = np.zeros((ranks.size, 16), np.uint8)
    p[:, :8] = vals[ranks].view(np.uint8).reshape(-1, 8)
    rk = oracle.gen_keys(key)
    c = device.encrypt_blocks(torch.from_numpy(p).cuda(), rk, iv).cpu().numpy()
    up, inv_p = np.unique(p, axis=0, return_inverse=True)
    uc, inv_c = np.unique(c, axis=0, return_inverse=True)
    assert up.shape[0] == uc.shape[0]
    # the map P -> C is a function: each P class lands on one C class
    first = {}
    for a, b in zip(inv_p.ravel()[:20000], inv_c.ravel()[:20000]):
        assert first.setdefault(int(a), int(b)) == int(b)
    idx = np.arange(0, ranks.size, 97)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (idx.size, 1))
    assert np.array_equal(c[idx], oracle.encrypt(key, ivrows, p[idx]))


def test_config5_many_key(oracle):
    rng = np.random.default_rng(5)
    k, bpk = 64, 4099
    keys = rng.integers(0, 256, (k, 16), dtype=np.uint8)
    ivs = rng.integers(0, 256, (k, 16), dtype=np.uint8)
    p = rng.integers(0, 256, (k * bpk, 16), dtype=np.uint8)
    d_keys = torch.from_numpy(keys).cuda()
    rk_enc, rk_dec = device.expand_keys(d_keys)
    assert np.array_equal(rk_enc.cpu().numpy(), oracle.gen_keys_batch(keys))
    x = torch.from_numpy(p).cuda()
    d_ivs = torch.from_numpy(ivs).cuda()
    c = device.many_key_encrypt(x, rk_enc, d_ivs)
    ch = c.cpu().numpy()
    for i in (0, 1, 31, 63):
        rows = slice(i * bpk, (i + 1) * bpk)
        ivrows = np.tile(ivs[i], (bpk, 1))
        assert np.array_equal(ch[rows], oracle.encrypt(keys[i].tobytes(), ivrows, p[rows])), i
    assert torch.equal(device.many_key_decrypt(c, rk_dec, d_ivs), x)


def test_launch_counter_and_kernel_name(oracle):
    x = torch.zeros((1024, 16), dtype=torch.uint8, device="cuda")
    device.encrypt_blocks(x, oracle.gen_keys(bytes(16)))  # context (GF-layer build) exists from here on
    before = _lib.launch_count()
    device.encrypt_blocks(x, oracle.gen_keys(bytes(16)))
    assert _lib.launch_count() == before + 1
    # 1024 blocks: the small-batch kernel (standard tables, texture S-box)
    assert _lib.last_kernel() in ("k_blocks_small_enc", "k_blocks_enc_folded")
    big = torch.zeros((1 << 20, 16), dtype=torch.uint8, device="cuda")
    device.encrypt_blocks(big, oracle.gen_keys(bytes(16)))
    assert _lib.last_kernel().startswith("k_blocks_enc_folded")


@pytest.mark.parametrize("variant", [2])
@pytest.mark.parametrize("n", [1, 1023, 1024, 1025, 148 * 384 * 32 + 999])
def test_bitsliced_variant_matches_oracle(oracle, n, variant):
    """The bitsliced LOP3 formulation (gaes_set_variant(2)) is bit-exact too."""
    L = _lib.lib()
    rng = np.random.default_rng(n + 99)
    key, iv = rng.bytes(16), rng.bytes(16)
    p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    try:
        assert L.gaes_set_variant(variant) == variant
        c = device.encrypt_blocks(torch.from_numpy(p).cuda(), rk, iv)
        torch.cuda.synchronize()
        assert _lib.last_kernel().startswith("k_bs_blocks")
        # the drop-in contract routes standard tables to the same kernel
        hc = np.empty_like(p)
        backend_cuda.cbc_encrypt(p, np.tile(np.frombuffer(iv, np.uint8), (n, 1)), *oracle.encrypt_tables(key), hc)
        assert _lib.last_kernel().startswith("k_bs_blocks")
        assert np.array_equal(hc, c.cpu().numpy())
    finally:
        L.gaes_set_variant(0)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    assert np.array_equal(c.cpu().numpy(), oracle.encrypt(key, ivrows, p, threads=4))


# ---------------------------------------------------------------- container I/O

def test_container_encrypt_records_identical_to_reference(golden):
    from paper_1506_08503_b200 import container as C
    content = golden["records_content"].tobytes()
    key = golden["records_key"].tobytes()
    blob = C.encrypt_records(content, key, iv=golden["records_iv"].tobytes())
    assert blob == golden["records_shared_container"].tobytes()
    blob2 = C.encrypt_records(content, key, ivs=golden["records_ivs"])
    assert blob2 == golden["records_permsg_container"].tobytes()
    assert C.decrypt_container(blob, key) == content
    assert C.decrypt_container(blob2, key) == content


def test_container_golden_recipe():
    import hashlib
    from paper_1506_08503_b200 import container as C
    blob = C.encrypt_records(b"alpha\nbravo-bravo\ncharlie charlie charlie!",
                             bytes.fromhex("000102030405060708090a0b0c0d0e0f"),
                             iv=bytes.fromhex("f0e1d2c3b4a5968778695a4b3c2d1e0f"))
    assert hashlib.sha256(blob).hexdigest() == "9e8a98b50f59f03773b6990cb07a40b6a2f4e7c0b704e695c6987d3366ea673b"


def test_sweep_csv_schema(tmp_path):
    """Reference CSV schema (bench.py:33-36) with the cuda implementation."""
    from paper_1506_08503_b200 import sweep
    out = tmp_path / "s.csv"
    assert sweep.main(["--kind", "count", "--counts", "1,1000", "--reps", "3", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0] == ("kind,implementation,n_messages,message_len_bytes,workers,"
                        "total_bytes,median_seconds,rate_bytes_per_second")
    assert len(lines) == 3 and lines[1].startswith("count,cuda,1,16,")
    assert sweep.main(["--kind", "length", "--lengths", "16,100", "--reps", "3", "--device-resident",
                       "--out", str(out)]) == 0
    assert out.read_text().splitlines()[2].startswith("length,cuda-device,128,100,")
    assert sweep.main(["--kind", "count", "--counts", "100000", "--reps", "3", "--device-resident", "--extended",
                       "--out", str(out)]) == 0
    head, row = out.read_text().splitlines()
    assert head.endswith(",gbs,hbm_frac,lds_frac,sm_mhz") and len(row.split(",")) == 12


def test_std_entry_points_match_oracle(oracle):
    rng = np.random.default_rng(21)
    key = rng.bytes(16)
    data = rng.integers(0, 256, (333, 48), dtype=np.uint8)
    ivs = rng.integers(0, 256, (333, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    ct = backend_cuda.cbc_encrypt_std(data, ivs, rk)
    assert np.array_equal(ct, oracle.encrypt(key, ivs, data))
    assert np.array_equal(backend_cuda.cbc_decrypt_std(ct, ivs, rk), data)


def test_beyond_4gib_buffers(oracle):
    """64-bit indexing: > 2^32 bytes per buffer (config 3 is 4 GiB at N=1)."""
    n = (1 << 28) + 17
    gen = torch.Generator(device="cuda")
    gen.manual_seed(28)
    x = torch.randint(0, 256, (n, 16), dtype=torch.uint8, device="cuda", generator=gen)
    rng = np.random.default_rng(28)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    c = device.encrypt_blocks(x, rk, iv)
    idx = torch.tensor([0, 1, (1 << 28) - 1, 1 << 28, n - 2, n - 1] + list(range(n - 4096, n - 4000)),
                       device="cuda")
    ps, cs = x[idx].cpu().numpy(), c[idx].cpu().numpy()
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (ps.shape[0], 1))
    assert np.array_equal(cs, oracle.encrypt(key, ivrows, ps))
    back = device.decrypt_blocks(c, rk, iv, out=c)  # in place
    assert torch.equal(back, x)
    del x, c, back
    torch.cuda.empty_cache()


def test_block_cipher_object(oracle):
    rng = np.random.default_rng(77)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    bc = device.BlockCipher(rk, iv)
    x = torch.randint(0, 256, (5000, 16), dtype=torch.uint8, device="cuda")
    c = bc.encrypt(x)
    assert torch.equal(c, device.encrypt_blocks(x, rk, iv))
    assert torch.equal(bc.decrypt(c), x)
    with pytest.raises(ValueError):
        bc.encrypt(x.view(-1, 32))


@pytest.mark.parametrize("blocks,offset", [(2, 0), (4, 0), (64, 0), (4, 16), (6, 16)])
def test_cbc_encrypt_rows_pairs_and_alignment(oracle, blocks, offset):
    """General-M CBC encrypt: 32-B paired accesses when aligned, 16-B otherwise."""
    rng = np.random.default_rng(blocks * 10 + offset)
    key = rng.bytes(16)
    n = 1500
    p = rng.integers(0, 256, (n, 16 * blocks), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    rk = oracle.gen_keys(key)
    flat = torch.zeros(p.size + 64, dtype=torch.uint8, device="cuda")
    x = flat[offset:offset + p.size].view(n, 16 * blocks)
    x.copy_(torch.from_numpy(p))
    oflat = torch.zeros_like(flat)
    out = oflat[offset:offset + p.size].view(n, 16 * blocks)
    device.cbc_encrypt(x, rk, torch.from_numpy(ivs).cuda(), out=out)
    assert np.array_equal(out.cpu().numpy(), oracle.encrypt(key, ivs, p))


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_bench_generators_and_parity(oracle, cfg):
    """Small instances of the config 3/4/5 generators (bench.make_inputs), encrypted on the GPU."""
    import bench
    dev = torch.device("cuda", 0)
    blocks = {3: 1 << 16, 4: 1 << 16, 5: 1024 * 64}[cfg]
    inp = bench.make_inputs(cfg, 0, 1, dev, blocks=blocks)
    p = inp["p"]
    ph = p.cpu().numpy()
    if cfg == 3:  # 8 LE int16 samples per block, |x| bounded by the amplitudes + noise
        s = ph.view(np.int16).reshape(-1)
        assert s.size == 8 * blocks and np.abs(s.astype(np.int32)).max() <= 32767
        assert np.abs(s.astype(np.float64)).mean() > 1000  # the sinusoids are there
    if cfg == 4:  # value in the low 8 bytes, 8 zero bytes, heavy-tailed repeats
        assert not ph[:, 8:].any()
        _, counts = np.unique(ph[:, :8], axis=0, return_counts=True)
        assert counts.max() > 100
    if cfg == 5:
        keys, ivs, bpk = inp["keys"], inp["ivs"], inp["bpk"]
        rk_enc, _ = device.expand_keys(torch.from_numpy(keys).cuda())
        c = device.many_key_encrypt(p, rk_enc, torch.from_numpy(ivs).cuda()).cpu().numpy()
        for i in (0, keys.shape[0] - 1):
            rows = slice(i * bpk, (i + 1) * bpk)
            assert np.array_equal(c[rows], oracle.encrypt(keys[i].tobytes(), np.tile(ivs[i], (bpk, 1)), ph[rows]))
        return
    key, iv = inp["key"], inp["iv"]
    c = device.encrypt_blocks(p, oracle.gen_keys(key), iv).cpu().numpy()
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (blocks, 1))
    assert np.array_equal(c, oracle.encrypt(key, ivrows, ph, threads=4))


def test_multi_gpu_shard_path_on_one_gpu(tmp_path):
    """The in-process multi-GPU dispatcher (plan_rows -> one host thread and
    context per device) run as two logical devices on one GPU via
    GAES_DEVICE_MAP=0,0; results must not depend on the shard count
    (test_parallel.py:55-96 lifted to GPUs)."""
    import subprocess
    import sys
    code = r'''
import numpy as np, sys
sys.path.insert(0, ".")
from oracle import oracle
from paper_1506_08503_b200 import _lib, backend_cuda
assert _lib.device_count() == 2, _lib.device_count()
rng = np.random.default_rng(8)
key, iv = rng.bytes(16), rng.bytes(16)
rk = oracle.gen_keys(key)
for n, m in [(1, 16), (3, 16), (100001, 16), (5003, 48)]:
    data = rng.integers(0, 256, (n, m), dtype=np.uint8)
    ivrows = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    want = oracle.encrypt(key, ivrows, data, threads=4)
    for g in (1, 2):
        assert _lib.set_num_gpus(g) == g
        out = np.empty_like(data)
        backend_cuda.cbc_encrypt(data, ivrows, *oracle.encrypt_tables(key), out)
        assert np.array_equal(out, want), (n, m, g)
        back = backend_cuda.cbc_decrypt_std(out, ivrows, rk)
        assert np.array_equal(back, data), (n, m, g)
        ct = backend_cuda.encrypt_shared_iv(data, iv, rk)
        assert np.array_equal(backend_cuda.decrypt_shared_iv(ct, iv, rk), data)
import torch
for n in (5, 300001):  # pinned buffers: one zero-copy launch per shard
    hp = torch.from_numpy(rng.integers(0, 256, (n, 16), dtype=np.uint8)).pin_memory()
    ho = torch.empty_like(hp).pin_memory()
    want = oracle.encrypt(key, np.tile(np.frombuffer(iv, np.uint8), (n, 1)), hp.numpy(), threads=4)
    for g in (1, 2):
        _lib.set_num_gpus(g)
        backend_cuda.encrypt_shared_iv(hp.numpy(), iv, rk, out=ho.numpy())
        assert np.array_equal(ho.numpy(), want), (n, g)
keys = rng.integers(0, 256, (7, 16), dtype=np.uint8)
kivs = rng.integers(0, 256, (7, 16), dtype=np.uint8)
p = rng.integers(0, 256, (7 * 10001, 16), dtype=np.uint8)
outs = []
for g in (1, 2):
    _lib.set_num_gpus(g)
    outs.append(backend_cuda.many_key_encrypt(p, keys, kivs))
    assert np.array_equal(backend_cuda.many_key_decrypt(outs[-1], keys, kivs), p)
assert np.array_equal(outs[0], outs[1])
print("ok")
'''
    import os
    env = dict(os.environ, GAES_DEVICE_MAP="0,0")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=repo, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_c_example_runs_bit_exact(tmp_path):
    """The C ABI from C: FIPS-197 C.1 and SP 800-38A through examples/encrypt_c.c."""
    import os
    import shutil
    import subprocess
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(repo, "paper_1506_08503_b200")
    exe = tmp_path / "encrypt_c"
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(repo, "include"), os.path.join(repo, "examples", "encrypt_c.c"),
                           "-L", libdir, "-lgaes_b200", f"-Wl,-rpath,{libdir}", "-o", str(exe)])
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and r.stdout.startswith("ok"), r.stdout + r.stderr


try:
    from hypothesis import given, settings
    from hypothesis import strategies as st
except ImportError:  # pragma: no cover
    given = None

if given is not None:
    @settings(max_examples=60, deadline=None)
    @given(st.integers(1, 300), st.integers(1, 6), st.booleans(), st.integers(0, 2**32 - 1))
    def test_property_backend_equals_oracle_and_round_trips(n, blocks, shared, seed):
        """Hypothesis round trip (test_aes_cbc.py:299-312 style) through the backend contract."""
        from oracle import oracle
        rng = np.random.default_rng(seed)
        key = rng.bytes(16)
        data = rng.integers(0, 256, (n, 16 * blocks), dtype=np.uint8)
        ivs = (np.tile(rng.integers(0, 256, 16, dtype=np.uint8), (n, 1)) if shared
               else rng.integers(0, 256, (n, 16), dtype=np.uint8))
        ct = _cuda_enc(key, ivs, data, oracle)
        assert np.array_equal(ct, oracle.encrypt(key, ivs, data))
        assert np.array_equal(_cuda_dec(key, ivs, ct, oracle), data)


def test_standard_tables_equal_reference_tables(golden):
    box, lut, perm = backend_cuda.standard_tables(False)
    assert np.array_equal(box, golden["sbox"]) and np.array_equal(lut, golden["mix_fwd"])
    assert np.array_equal(perm, golden["shift"])
    box, lut, perm = backend_cuda.standard_tables(True)
    assert np.array_equal(box, golden["inv_sbox"]) and np.array_equal(lut, golden["mix_inv"])
    assert np.array_equal(perm, golden["inv_shift"])


def test_device_api_argument_errors(oracle):
    rk = oracle.gen_keys(bytes(16))
    x = torch.zeros((64, 16), dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        device.encrypt_blocks(x.cpu(), rk)                      # host tensor
    with pytest.raises(ValueError):
        device.encrypt_blocks(x.to(torch.int16), rk)            # dtype
    with pytest.raises(ValueError):
        device.encrypt_blocks(x.t(), rk)                        # non-contiguous
    with pytest.raises(ValueError):
        device.encrypt_blocks(x, rk[:10])                       # short schedule
    with pytest.raises(ValueError):
        device.cbc_encrypt(torch.zeros((4, 20), dtype=torch.uint8, device="cuda"), rk)
    with pytest.raises(ValueError):
        device.many_key_encrypt(x, torch.zeros((3, 11, 16), dtype=torch.uint8, device="cuda"))  # 64 % 3
    L = _lib.lib()
    assert L.gaes_encrypt_blocks_dev(None, None, 5, None, None, None) == _lib.GAES_EINVAL
    assert b"null" in L.gaes_last_error()
    assert L.gaes_encrypt_blocks_dev(None, None, 0, None, None, None) == 0  # n == 0 no-op
    with pytest.raises(ValueError):
        _lib.check(L.gaes_gf_tables(99, None, None, None, None))
    assert L.gaes_set_variant(7) == _lib.GAES_EINVAL


def test_concurrent_device_api_on_streams(oracle):
    """Device entry points are stream-ordered and re-entrant across host threads."""
    rng = np.random.default_rng(31)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    xs = [torch.from_numpy(rng.integers(0, 256, (70000, 16), dtype=np.uint8)).cuda() for _ in range(4)]
    outs = [None] * 4

    def work(i):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            outs[i] = device.encrypt_blocks(xs[i], rk, iv)
        s.synchronize()

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    for i in range(4):
        assert torch.equal(outs[i], device.encrypt_blocks(xs[i], rk, iv))
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (1000, 1))
    assert np.array_equal(outs[0][:1000].cpu().numpy(), oracle.encrypt(key, ivrows, xs[0][:1000].cpu().numpy()))


@pytest.mark.parametrize("k,bpk", [(1, 1), (3, 1000), (64, 4099), (5, 300000)])
def test_host_many_key_matches_oracle(oracle, k, bpk):
    """Host-buffer many-key entry (config 5 end to end): GPU key schedule + pipeline."""
    rng = np.random.default_rng(k * 7 + bpk)
    keys = rng.integers(0, 256, (k, 16), dtype=np.uint8)
    ivs = rng.integers(0, 256, (k, 16), dtype=np.uint8)
    p = rng.integers(0, 256, (k * bpk, 16), dtype=np.uint8)
    c = backend_cuda.many_key_encrypt(p, keys, ivs)
    for i in sorted({0, k // 2, k - 1}):
        rows = slice(i * bpk, (i + 1) * bpk)
        ivrows = np.tile(ivs[i], (bpk, 1))
        assert np.array_equal(c[rows], oracle.encrypt(keys[i].tobytes(), ivrows, p[rows], threads=4)), i
    assert np.array_equal(backend_cuda.many_key_decrypt(c, keys, ivs), p)
    c0 = backend_cuda.many_key_encrypt(p, keys)  # zero IVs
    assert np.array_equal(c0[:bpk], oracle.encrypt(keys[0].tobytes(), np.zeros((bpk, 16), np.uint8), p[:bpk]))


def test_texture_cache_churn_across_threads(oracle):
    """Device-API calls on > 64 distinct input buffers from 4 threads: the
    per-device texture cache evicts least-recently-used idle entries only
    after the launches that read them (their last-use events) -- every result
    must stay bit-exact, including buffers re-used after eviction."""
    rng = np.random.default_rng(44)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    n = 4099
    pool = [torch.from_numpy(rng.integers(0, 256, (n + i, 16), dtype=np.uint8)).cuda() for i in range(90)]
    ref = [device.encrypt_blocks(x, rk, iv) for x in pool[:3]]
    errors = []

    def work(t):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            for rep in range(3):
                for i in range(t, len(pool), 4):
                    x = pool[i]
                    c = device.encrypt_blocks(x, rk, iv)
                    d = device.decrypt_blocks(c, rk, iv)
                    s.synchronize()
                    if not torch.equal(d, x) or (i < 3 and not torch.equal(c, ref[i])):
                        errors.append((t, rep, i))

    th = [threading.Thread(target=work, args=(t,)) for t in range(4)]
    [t.start() for t in th]
    [t.join() for t in th]
    assert not errors, errors[:5]
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    assert np.array_equal(ref[0].cpu().numpy(), oracle.encrypt(key, ivrows, pool[0].cpu().numpy()))


@pytest.mark.parametrize("shift", [0, 16, -16, 48])
def test_device_api_in_place_and_overlapping(oracle, shift):
    """out aliasing the input (identical, or shifted by whole blocks) gives the
    same bytes as separate buffers for every device entry point -- including
    block-parallel CBC decrypt of multi-block rows, whose chain value comes
    from a neighbouring block (copied to a private buffer first)."""
    rng = np.random.default_rng(100 + shift)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    n, blocks = 300001, 4  # 1.2 M blocks: ~8 grid-stride passes, so warps drift apart
    m = 16 * blocks
    p = torch.from_numpy(rng.integers(0, 256, (n, m), dtype=np.uint8)).cuda()
    ivs = torch.from_numpy(rng.integers(0, 256, (n, 16), dtype=np.uint8)).cuda()
    d_keys = torch.from_numpy(rng.integers(0, 256, (7, 16), dtype=np.uint8)).cuda()
    rke, rkd = device.expand_keys(d_keys)
    pad = 4096

    def aliased(x, fn):
        """Run fn(inp, out) with out = inp shifted by `shift` bytes in one buffer."""
        buf = torch.zeros(x.numel() + 2 * pad, dtype=torch.uint8, device="cuda")
        inp = buf[pad:pad + x.numel()].view(x.shape)
        inp.copy_(x)
        o = buf[pad + shift:pad + shift + x.numel()].view(x.shape)
        fn(inp, o)
        return o.clone()

    p16 = p.view(-1, 16)[: 7 * 171301]
    cases = [
        (p16, lambda a, o: device.encrypt_blocks(a, rk, iv, out=o)),
        (p16, lambda a, o: device.decrypt_blocks(a, rk, iv, out=o)),
        (p, lambda a, o: device.cbc_encrypt(a, rk, iv, out=o)),
        (p, lambda a, o: device.cbc_encrypt(a, rk, ivs, out=o)),
        (p, lambda a, o: device.cbc_decrypt(a, rk, iv, out=o)),
        (p, lambda a, o: device.cbc_decrypt(a, rk, ivs, out=o)),
        (p16, lambda a, o: device.many_key_encrypt(a, rke, out=o)),
        (p16, lambda a, o: device.many_key_decrypt(a, rkd, out=o)),
    ]
    for i, (x, fn) in enumerate(cases):
        want = torch.empty_like(x)
        fn(x, want)
        got = aliased(x, fn)
        assert torch.equal(got, want), i
    want = oracle.decrypt(key, ivs.cpu().numpy(), p.cpu().numpy())
    assert np.array_equal(aliased(p, lambda a, o: device.cbc_decrypt(a, rk, ivs, out=o)).cpu().numpy(), want)


def _pinned(shape, rng=None):
    t = torch.empty(shape, dtype=torch.uint8).pin_memory()
    a = t.numpy()
    if rng is not None:
        a[:] = rng.integers(0, 256, shape, dtype=np.uint8)
    return t, a


@pytest.mark.parametrize("n,m", [(1, 16), (4097, 16), (4096, 16), (3001, 64), (1 << 20, 16)])
def test_pinned_zero_copy_every_mode(oracle, n, m):
    """Pinned host buffers up to 64 MiB (GAES_TUNE ZEROCOPY_MB) run as one zero-copy launch
    (the kernel reads and writes host memory over PCIe); every host entry
    point must match the oracle there, with pinned per-row IVs too, and
    in-place pinned calls (which take the staged pipeline) as well."""
    rng = np.random.default_rng(n + m)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    _t0, p = _pinned((n, m), rng)
    _t1, ivs = _pinned((n, 16), rng)
    _t2, out = _pinned((n, m))
    _t3, back = _pinned((n, m))
    tables = oracle.encrypt_tables(key)
    want = oracle.encrypt(key, ivs, p, threads=4)
    backend_cuda.cbc_encrypt(p, ivs, *tables, out)                     # per-row IVs (chain / rows)
    assert np.array_equal(out, want)
    backend_cuda.cbc_decrypt(out, ivs, *oracle.decrypt_tables(key), back)
    assert np.array_equal(back, p)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    want = oracle.encrypt(key, ivrows, p, threads=4)
    backend_cuda.encrypt_shared_iv(p, iv, rk, out=out)                  # folded / rows, shared IV
    assert np.array_equal(out, want)
    backend_cuda.decrypt_shared_iv(out, iv, rk, out=back)
    assert np.array_equal(back, p)
    backend_cuda.encrypt_shared_iv(back, iv, rk, out=back)              # in place (staged path)
    assert np.array_equal(back, want)
    if m == 16 and n % 16 == 0:
        k = 16
        keys = rng.integers(0, 256, (k, 16), dtype=np.uint8)
        kivs = rng.integers(0, 256, (k, 16), dtype=np.uint8)
        backend_cuda.many_key_encrypt(p, keys, kivs, out=out)
        bpk = n // k
        for i in (0, k - 1):
            r = slice(i * bpk, (i + 1) * bpk)
            assert np.array_equal(out[r], oracle.encrypt(keys[i].tobytes(), np.tile(kivs[i], (bpk, 1)), p[r]))
        backend_cuda.many_key_decrypt(out, keys, kivs, out=back)
        assert np.array_equal(back, p)


@pytest.mark.parametrize("n", [1, 31, 33, 1025, 148 * 1024 + 3])
def test_no_out_of_bounds_writes(oracle, n):
    """Guard bands around every output (device and host): no kernel or copy
    may write outside [out, out + n*m).  compute-sanitizer is not available
    on the GPU pool, so out-of-bounds writes are caught by canaries."""
    G = 4096
    rng = np.random.default_rng(n)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    keys = torch.from_numpy(rng.integers(0, 256, (1, 16), dtype=np.uint8)).cuda()
    rke, rkd = device.expand_keys(keys)

    def guarded_dev(shape):
        numel = int(np.prod(shape))
        buf = torch.full((numel + 2 * G,), 0xA5, dtype=torch.uint8, device="cuda")
        return buf, buf[G:G + numel].view(shape)

    def intact(buf, numel):
        torch.cuda.synchronize()
        return bool((buf[:G] == 0xA5).all()) and bool((buf[G + numel:] == 0xA5).all())

    for m in (16, 48, 64):
        p = torch.from_numpy(rng.integers(0, 256, (n, m), dtype=np.uint8)).cuda()
        ivs = torch.from_numpy(rng.integers(0, 256, (n, 16), dtype=np.uint8)).cuda()
        calls = [lambda o: device.cbc_encrypt(p, rk, iv, out=o), lambda o: device.cbc_encrypt(p, rk, ivs, out=o),
                 lambda o: device.cbc_decrypt(p, rk, iv, out=o), lambda o: device.cbc_decrypt(p, rk, ivs, out=o)]
        if m == 16:
            calls += [lambda o: device.encrypt_blocks(p, rk, iv, out=o), lambda o: device.decrypt_blocks(p, rk, iv, out=o),
                      lambda o: device.many_key_encrypt(p, rke, out=o), lambda o: device.many_key_decrypt(p, rkd, out=o)]
        for i, call in enumerate(calls):
            buf, o = guarded_dev((n, m))
            call(o)
            assert intact(buf, n * m), (m, i)
        # host entry points (zero-copy for pinned, staged for pageable; generic tables)
        ph = p.cpu().numpy()
        ivh = ivs.cpu().numpy()
        t = oracle.encrypt_tables(key)
        perm = np.ascontiguousarray(np.roll(t[3], 1))
        for pinned in (False, True):
            for tables in (t, (t[0], t[1], t[2], perm)):
                hb = torch.full((n * m + 2 * G,), 0xA5, dtype=torch.uint8)
                if pinned:
                    hb = hb.pin_memory()
                a = hb.numpy()
                backend_cuda.cbc_encrypt(ph, ivh, *tables, a[G:G + n * m].reshape(n, m))
                assert (a[:G] == 0xA5).all() and (a[G + n * m:] == 0xA5).all(), (m, pinned)


def test_roofline_probes_are_sane():
    """The measured LDS peak (roofline denominator) sits near the nominal
    32 lanes/clk/SM at the max SM clock, and the AES round probe below it."""
    import ctypes
    L = _lib.lib()
    rate, ms = ctypes.c_double(), ctypes.c_double()
    _lib.check(L.gaes_probe_lds_peak(0, 2048, ctypes.addressof(rate), ctypes.addressof(ms)))
    lds = rate.value
    _lib.check(L.gaes_probe_round_rate(0, 128, ctypes.addressof(rate), ctypes.addressof(ms)))
    rnd = rate.value  # 160 lookups per encryption
    if L.gaes_uses_sbox_texture(0) == 1:
        rnd *= 144 / 160  # round 10's 16 S-box fetches ride the TEX pipe
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    nominal_max = sms * 32 * 2.1e9  # above any B200 SM clock
    assert 0.3 * nominal_max < lds < nominal_max
    assert 0.5 * lds < rnd < 1.02 * lds


@pytest.mark.parametrize("m", [16, 48])
def test_dropin_mixed_shared_and_per_row_iv_chunks(oracle, m):
    """Pageable drop-in calls check IV rows per staged chunk: a grid whose IV
    rows are the tiled shared IV except for one stretch must give the oracle's
    bytes, with chunks before/after the stretch on the shared-IV kernels and
    the chunk holding it on the per-row kernels."""
    rng = np.random.default_rng(m)
    key = rng.bytes(16)
    n = 600000 if m == 16 else 200000
    data = rng.integers(0, 256, (n, m), dtype=np.uint8)
    iv0 = rng.integers(0, 256, 16, dtype=np.uint8)
    ivs = np.tile(iv0, (n, 1))
    lo = n // 4
    ivs[lo:lo + 10000] = rng.integers(0, 256, (10000, 16), dtype=np.uint8)
    want = oracle.encrypt(key, ivs, data, threads=8)
    out = np.empty_like(data)
    backend_cuda.cbc_encrypt(data, ivs, *oracle.encrypt_tables(key), out)
    assert np.array_equal(out, want)
    back = np.empty_like(data)
    backend_cuda.cbc_decrypt(out, ivs, *oracle.decrypt_tables(key), back)
    assert np.array_equal(back, data)


def test_concurrent_host_calls_of_different_kinds_use_separate_lanes(oracle):
    """Host calls from several threads run on separate per-device lanes with
    their own scratch: generic (non-standard) tables, many-key schedules,
    per-row-IV decrypt and shared-IV encrypt at the same time, repeatedly,
    all bit-exact."""
    rng = np.random.default_rng(404)
    key = rng.bytes(16)
    t = oracle.encrypt_tables(key)
    perm = np.ascontiguousarray(np.roll(t[3], 3))
    n = 20000
    p = rng.integers(0, 256, (n, 32), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    keys = rng.integers(0, 256, (8, 16), dtype=np.uint8)
    p16 = rng.integers(0, 256, (8 * 5000, 16), dtype=np.uint8)
    want_generic = np.empty_like(p)
    backend_cuda.cbc_encrypt(p, ivs, t[0], t[1], t[2], perm, want_generic)
    want_mk = backend_cuda.many_key_encrypt(p16, keys)
    want_enc = oracle.encrypt(key, ivs, p, threads=4)
    errors = []

    def generic():
        out = np.empty_like(p)
        backend_cuda.cbc_encrypt(p, ivs, t[0], t[1], t[2], perm, out)
        return np.array_equal(out, want_generic)

    def many_key():
        return np.array_equal(backend_cuda.many_key_encrypt(p16, keys), want_mk)

    def chain():
        out = np.empty_like(p)
        backend_cuda.cbc_encrypt(p, ivs, *t, out)
        back = np.empty_like(p)
        backend_cuda.cbc_decrypt(out, ivs, *oracle.decrypt_tables(key), back)
        return np.array_equal(out, want_enc) and np.array_equal(back, p)

    def work(fn, k):
        for _ in range(6):
            if not fn():
                errors.append(k)

    th = [threading.Thread(target=work, args=(fn, k)) for k, fn in enumerate((generic, many_key, chain, generic, chain))]
    [x.start() for x in th]
    [x.join() for x in th]
    assert not errors, errors


def test_cuda_graph_capture_and_replay(oracle):
    """Device-API calls are capturable in a CUDA graph (stream-ordered, no
    host sync) and replays stay bit-exact after new inputs are written and
    after the texture cache has churned (captured launches use no texture)."""
    rng = np.random.default_rng(55)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    n = 50000
    x = torch.empty((n, 16), dtype=torch.uint8, device="cuda")
    y = torch.empty_like(x)
    z = torch.empty_like(x)
    rows = torch.empty((n // 4, 64), dtype=torch.uint8, device="cuda")
    rows_ct = torch.empty_like(rows)
    bc = device.BlockCipher(rk, iv)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        bc.encrypt(x, out=y)  # warm-up outside capture (context, smem opt-in)
        device.cbc_encrypt(rows, rk, iv, out=rows_ct)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            bc.encrypt(x, out=y)
            bc.decrypt(y, out=z)
            device.cbc_encrypt(rows, rk, iv, out=rows_ct)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    for rep in range(3):
        p = rng.integers(0, 256, (n, 16), dtype=np.uint8)
        pr = rng.integers(0, 256, (n // 4, 64), dtype=np.uint8)
        x.copy_(torch.from_numpy(p))
        rows.copy_(torch.from_numpy(pr))
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(y.cpu().numpy(), oracle.encrypt(key, ivrows, p, threads=4)), rep
        assert torch.equal(z, x)
        assert np.array_equal(rows_ct.cpu().numpy(), oracle.encrypt(key, ivrows[: n // 4], pr, threads=4))
        for _ in range(70):  # churn the texture cache between replays
            device.encrypt_blocks(torch.empty((1024 + rep, 16), dtype=torch.uint8, device="cuda"), rk, iv)


def test_shared_memory_sbox_path_without_textures():
    """GAES_TUNE=TEXS=0,TEXIN=0 (the paths used when textures are
    unavailable): round 10 reads the replicated S table in shared memory and
    inputs come through LDG -- bit-exact against the oracle for every kernel."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, sys, torch
sys.path.insert(0, ".")
from oracle import oracle
from paper_1506_08503_b200 import _lib, backend_cuda, device
assert _lib.lib().gaes_uses_sbox_texture(0) == 0
rng = np.random.default_rng(3)
key, iv = rng.bytes(16), rng.bytes(16)
rk = oracle.gen_keys(key)
for n, m in [(70001, 16), (3001, 64)]:
    p = rng.integers(0, 256, (n, m), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    want = oracle.encrypt(key, ivs, p, threads=4)
    x = torch.from_numpy(p).cuda()
    c = device.cbc_encrypt(x, rk, torch.from_numpy(ivs).cuda())
    assert np.array_equal(c.cpu().numpy(), want)
    assert torch.equal(device.cbc_decrypt(c, rk, torch.from_numpy(ivs).cuda()), x)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    assert np.array_equal(backend_cuda.encrypt_shared_iv(p, iv, rk), oracle.encrypt(key, ivrows, p, threads=4))
keys = rng.integers(0, 256, (4, 16), dtype=np.uint8)
p = rng.integers(0, 256, (4 * 5000, 16), dtype=np.uint8)
c = backend_cuda.many_key_encrypt(p, keys)
assert np.array_equal(c[:5000], oracle.encrypt(keys[0].tobytes(), np.zeros((5000, 16), np.uint8), p[:5000]))
assert np.array_equal(backend_cuda.many_key_decrypt(c, keys), p)
print("ok")
'''
    env = dict(os.environ, GAES_TUNE="TEXS=0,TEXIN=0")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=repo, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


@pytest.mark.parametrize("blocks", [8, 10])
def test_row_cbc_tma_path_matches_oracle(oracle, blocks):
    """General-M CBC encrypt with enough rows for the TMA row kernel (>= 24
    row groups of 32 per SM): ragged last group (TMA out-of-bounds rows),
    shared and per-row IVs, device and host entry points."""
    rng = np.random.default_rng(blocks)
    key, iv = rng.bytes(16), rng.bytes(16)
    rk = oracle.gen_keys(key)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    n = sms * 24 * 32 + 17
    m = 16 * blocks
    p = rng.integers(0, 256, (n, m), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    x = torch.from_numpy(p).cuda()
    want = oracle.encrypt(key, ivs, p, threads=8)
    c = device.cbc_encrypt(x, rk, torch.from_numpy(ivs).cuda())
    if _lib.lib().gaes_uses_sbox_texture(0) == 1 and "ROWS_TMA=0" not in os.environ.get("GAES_TUNE", ""):
        assert _lib.last_kernel() == "k_cbc_enc_rows_tma"
    assert np.array_equal(c.cpu().numpy(), want)
    assert torch.equal(device.cbc_decrypt(c, rk, torch.from_numpy(ivs).cuda()), x)
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (n, 1))
    want_shared = oracle.encrypt(key, ivrows, p, threads=8)
    assert np.array_equal(device.cbc_encrypt(x, rk, iv).cpu().numpy(), want_shared)
    out = np.empty_like(p)
    backend_cuda.cbc_encrypt(p, ivs, *oracle.encrypt_tables(key), out)   # host pipeline chunks
    assert np.array_equal(out, want)
    assert np.array_equal(backend_cuda.encrypt_shared_iv(p, iv, rk), want_shared)


def test_row_cbc_tma_kernel_at_any_row_count():
    """The TMA row kernel itself (forced for every row count with
    GAES_TUNE=ROWS_TMA_MIN_GROUPS=0, normally only used from 8 row groups per
    SM): 1..4 warps with rows, ragged groups, 8..64-block rows."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import oracle
from paper_1506_08503_b200 import device, _lib
rng = np.random.default_rng(9)
key, iv = rng.bytes(16), rng.bytes(16)
rk = oracle.gen_keys(key)
for n, bpr in [(32, 8), (33, 64), (100, 16), (1500, 8), (4737, 10)]:
    p = rng.integers(0, 256, (n, 16 * bpr), dtype=np.uint8)
    ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    c = device.cbc_encrypt(torch.from_numpy(p).cuda(), rk, torch.from_numpy(ivs).cuda())
    assert _lib.last_kernel() == "k_cbc_enc_rows_tma", _lib.last_kernel()
    assert np.array_equal(c.cpu().numpy(), oracle.encrypt(key, ivs, p, threads=4)), (n, bpr)
print("ok")
'''
    env = dict(os.environ, GAES_TUNE="ROWS_TMA_MIN_GROUPS=0")
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", code], cwd=repo, env=env, capture_output=True, text=True, timeout=300)
    if "k_cbc_enc_rows\n" in r.stderr or _lib.lib().gaes_uses_sbox_texture(0) != 1:
        pytest.skip("texture S-box unavailable: the TMA row kernel does not apply")
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def _misaligned(shape, offset, rng=None):
    """A C-contiguous uint8 array whose data starts `offset` bytes past a
    64-byte boundary (pageable numpy memory)."""
    n = int(np.prod(shape))
    raw = np.empty(n + 128, np.uint8)
    base = (-raw.ctypes.data) % 64
    a = raw[base + offset: base + offset + n].reshape(shape)
    if rng is not None:
        a[...] = rng.integers(0, 256, shape, dtype=np.uint8)
    return a


@pytest.mark.parametrize("m,shared,offset", [(16, True, 1), (16, False, 3), (64, True, 17), (64, False, 8)])
def test_pageable_dropin_misaligned_multichunk(oracle, m, shared, offset):
    """The 7-argument drop-in with pageable buffers at odd byte offsets and
    several staging chunks (40 MiB; pageable chunks are 16 MiB): the
    streaming-store staging copies handle unaligned heads/tails and every
    chunk boundary.  Rows are independent, so a row sample is compared with
    the oracle, and the whole grid round-trips through decrypt."""
    rng = np.random.default_rng(20 + m + offset)
    key = rng.bytes(16)
    n = (40 << 20) // m
    p = _misaligned((n, m), offset, rng)
    if shared:
        ivrows = np.tile(rng.integers(0, 256, 16, dtype=np.uint8), (n, 1))
    else:
        ivrows = rng.integers(0, 256, (n, 16), dtype=np.uint8)
    c = _misaligned((n, m), (offset * 7) % 64)
    backend_cuda.cbc_encrypt(p, ivrows, *oracle.encrypt_tables(key), c)
    rows = np.unique(np.concatenate([np.arange(8), n - 1 - np.arange(8), rng.choice(n, 512, replace=False),
                                     np.arange(16 << 20, (16 << 20) + 4 * m, m) // m]))
    rows = rows[rows < n]
    want = oracle.encrypt(key, ivrows[rows], np.ascontiguousarray(p[rows]))
    assert np.array_equal(c[rows], want)
    back = _misaligned((n, m), (offset * 3) % 64)
    backend_cuda.cbc_decrypt(c, ivrows, *oracle.decrypt_tables(key), back)
    assert np.array_equal(back, p)
