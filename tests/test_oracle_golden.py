"""Pin the C oracle (oracle/gaes_oracle.c) before trusting it.

Known answers come from three independent places:
  * published vectors quoted by the reference tests (FIPS-197 C.1 and A.1,
    SP 800-38A F.2.1; pkg/tests/test_aes_cbc.py:26-39,204-209,
    test_key_schedule.py:28-46, reference.py:12-21);
  * fixtures produced by running the reference package itself
    (tests/golden/make_golden.py -> golden.npz / golden.json);
  * the reference's own compiled kernel built from its sources
    (oracle/_ref, when present).
"""

import hashlib

import numpy as np
import pytest

FIPS_SBOX_HEX = (
    "637c777bf26b6fc53001672bfed7ab76ca82c97dfa5947f0add4a2af9ca472c0"
    "b7fd9326363ff7cc34a5e5f171d8311504c723c31896059a071280e2eb27b275"
    "09832c1a1b6e5aa0523bd6b329e32f8453d100ed20fcb15b6acbbe394a4c58cf"
    "d0efaafb434d338545f9027f503c9fa851a3408f929d38f5bcb6da2110fff3d2"
    "cd0c13ec5f974417c4a77e3d645d197360814fdc222a908846eeb814de5e0bdb"
    "e0323a0a4906245cc2d3ac629195e479e7c8376d8dd54ea96c56f4ea657aae08"
    "ba78252e1ca6b4c6e8dd741f4bbd8b8a703eb5664803f60e613557b986c11d9e"
    "e1f8981169d98e949b1e87e9ce5528df8ca1890dbfe6426841992d0fb054bb16"
)
NIST_KEY = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
NIST_IV = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
NIST_PT = bytes.fromhex(
    "6bc1bee22e409f96e93d7e117393172aae2d8a571e03ac9c9eb76fac45af8e51"
    "30c81c46a35ce411e5fbc1191a0a52eff69f2445df4f9b17ad2b417be66c3710")
NIST_CT = bytes.fromhex(
    "7649abac8119b246cee98e9b12e9197d5086cb9b507219ee95db113a917678b2"
    "73bed6b8e3c1743b7116e69e222295163ff1caa1681fac09120eca307586e1a7")


def test_gf_paper_examples(oracle):
    # gf256 worked examples: {57}.{83} = {c1}, {57}.{13} = {fe} (FIPS-197 4.2)
    assert oracle.gf_mul(0x57, 0x83) == 0xC1
    assert oracle.gf_mul(0x57, 0x13) == 0xFE
    assert oracle.gf_inv(0) == 0
    for a in range(1, 256):
        assert oracle.gf_mul(a, oracle.gf_inv(a)) == 1


def test_sbox_matches_fips_and_reference(oracle, golden):
    assert oracle.sbox().tobytes().hex() == FIPS_SBOX_HEX
    assert np.array_equal(oracle.sbox(), golden["sbox"])
    assert np.array_equal(oracle.inv_sbox(), golden["inv_sbox"])
    assert np.array_equal(oracle.inv_sbox()[oracle.sbox()], np.arange(256))


def test_mix_luts_match_reference(oracle, golden):
    assert np.array_equal(oracle.mix_lut(oracle.MIX_FORWARD_ROW), golden["mix_fwd"])
    assert np.array_equal(oracle.mix_lut(oracle.MIX_INVERSE_ROW), golden["mix_inv"])
    assert np.array_equal(np.array(oracle.SHIFT_ROWS_SRC, np.uint8), golden["shift"])
    assert np.array_equal(np.array(oracle.INV_SHIFT_ROWS_SRC, np.uint8), golden["inv_shift"])


def test_round_constants(oracle, golden):
    assert oracle.round_constants() == bytes.fromhex("01020408102040801b36")
    assert oracle.round_constants() == golden["rcon"].tobytes()


def test_key_schedule_kats(oracle):
    # FIPS-197 A.1: last round key
    rk = oracle.gen_keys(NIST_KEY)
    assert rk[10].tobytes() == bytes.fromhex("d014f9a8c9ee2589e13f0cc8b6630ca6")
    # zero key, rounds 1 and 2 (test_key_schedule.py:28-38)
    z = oracle.gen_keys(bytes(16))
    assert z[1].tobytes() == bytes.fromhex("62636363626363636263636362636363")
    assert z[2].tobytes() == bytes.fromhex("9b9898c9f9fbfbaa9b9898c9f9fbfbaa")


def test_key_schedule_matches_reference_fixtures(oracle, golden):
    got = oracle.gen_keys_batch(golden["keys"])
    assert np.array_equal(got, golden["round_keys"])


def test_fips197_block_kat(oracle):
    key = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
    pt = np.frombuffer(bytes.fromhex("00112233445566778899aabbccddeeff"), np.uint8).reshape(1, 16)
    ct = oracle.encrypt(key, np.zeros((1, 16), np.uint8), pt)
    assert ct.tobytes() == bytes.fromhex("69c4e0d86a7b0430d8cdb78070b4c55a")
    assert np.array_equal(oracle.decrypt(key, np.zeros((1, 16), np.uint8), ct), pt)


def test_sp800_38a_cbc(oracle):
    pt = np.frombuffer(NIST_PT, np.uint8).reshape(1, 64)
    iv = np.frombuffer(NIST_IV, np.uint8).reshape(1, 16)
    ct = oracle.encrypt(NIST_KEY, iv, pt)
    assert ct.tobytes() == NIST_CT
    assert oracle.decrypt(NIST_KEY, iv, ct).tobytes() == NIST_PT


@pytest.mark.parametrize("threads", [1, 3])
def test_cbc_cases_match_reference_fixtures(oracle, golden, golden_meta, threads):
    for case in golden_meta["cases"]:
        i = case["idx"]
        key = golden[f"case{i}_key"].tobytes()
        ct = oracle.encrypt(key, golden[f"case{i}_iv"], golden[f"case{i}_pt"], threads=threads)
        assert np.array_equal(ct, golden[f"case{i}_ct"]), case
        pt = oracle.decrypt(key, golden[f"case{i}_iv"], ct, threads=threads)
        assert np.array_equal(pt, golden[f"case{i}_pt"]), case


def test_cfg1_digest(oracle, golden_meta, golden):
    d = golden_meta["digests"]["65536"]
    rng = np.random.default_rng(2016)
    key, iv = rng.bytes(16), rng.bytes(16)
    assert key.hex() == d["key"] and iv.hex() == d["iv"]
    p = rng.integers(0, 256, (1 << 16, 16), dtype=np.uint8)
    assert hashlib.sha256(p.tobytes()).hexdigest() == d["sha256_p"]
    ivrows = np.tile(np.frombuffer(iv, np.uint8), (p.shape[0], 1))
    c = oracle.encrypt(key, ivrows, p, threads=4)
    assert hashlib.sha256(c.tobytes()).hexdigest() == d["sha256_c"]
    assert np.array_equal(c[:64], golden["cfg1_ct_rows_0_64"])
    assert np.array_equal(oracle.decrypt(key, ivrows, c, threads=4), p)


def test_plan_matches_reference_semantics(oracle):
    # parallel.py:37-50: contiguous, sizes differ by <= 1, capped at n
    for n in (0, 1, 7, 100, 1001):
        for w in (1, 2, 3, 8):
            chunks = oracle.plan(n, w)
            assert len(chunks) == min(n, w)
            if chunks:
                assert chunks[0][0] == 0 and chunks[-1][1] == n
                sizes = [hi - lo for lo, hi in chunks]
                assert max(sizes) - min(sizes) <= 1
                assert all(a[1] == b[0] for a, b in zip(chunks, chunks[1:]))


def test_oracle_agrees_with_reference_kernel(oracle):
    """oracle/_ref: the reference's own _kernel.pyx, compiled from its sources."""
    import os
    import sys
    ref_dir = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref")
    if not os.path.isdir(ref_dir):
        pytest.skip("oracle/_ref not built")
    sys.path.insert(0, ref_dir)
    try:
        import _kernel
    except ImportError:
        pytest.skip("oracle/_ref/_kernel not importable")
    finally:
        sys.path.remove(ref_dir)
    rng = np.random.default_rng(5)
    for n, blocks in [(1, 1), (37, 3), (500, 1)]:
        key = rng.bytes(16)
        data = rng.integers(0, 256, (n, 16 * blocks), dtype=np.uint8)
        ivs = rng.integers(0, 256, (n, 16), dtype=np.uint8)
        t = oracle.encrypt_tables(key)
        a = np.empty_like(data)
        _kernel.cbc_encrypt(data, ivs, *t, a)
        assert np.array_equal(a, oracle.encrypt(key, ivs, data))
        td = oracle.decrypt_tables(key)
        b = np.empty_like(data)
        _kernel.cbc_decrypt(a, ivs, *td, b)
        assert np.array_equal(b, data)
