"""CPU-only checks of the C ABI library and the host-side logic (no GPU calls).

* libgaes_b200.so loads and exports every function include/gaes_b200.h
  declares, with the ctypes signature table matching the header;
* the cubin inside it targets sm_100a;
* backend_cuda validates arguments like the reference's compiled kernel
  (Cython buffer errors, probe P11) before any device work;
* without a GPU the product path fails loudly instead of falling back.
"""

import os
import re
import shutil
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "gaes_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"GAES_API\s+[\w\s\*]+?\b(gaes_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__
    __graft_entry__._load_build_module().build()
    from paper_1506_08503_b200 import _lib
    return _lib


def test_header_declares_the_backend_contract():
    names = _declared()
    for required in ("gaes_cbc_encrypt", "gaes_cbc_decrypt", "gaes_expand_keys_dev", "gaes_gf_tables",
                     "gaes_encrypt_blocks_dev", "gaes_many_key_encrypt_dev", "gaes_last_error"):
        assert required in names


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.check_output(["nm", "-D", "--defined-only", lib.LIB_PATH], text=True)
    exported = set(re.findall(r"\bT (gaes_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    L = lib.lib()
    for name in _declared():
        assert hasattr(L, name)


def test_signature_table_covers_header(lib):
    assert sorted(lib.SIGNATURES) == _declared()
    text = open(HEADER).read()
    for name, (_, args) in lib.SIGNATURES.items():
        m = re.search(r"\b%s\s*\(([^)]*)\)" % name, text)
        params = [p for p in m.group(1).split(",") if p.strip() and p.strip() != "void"]
        assert len(params) == len(args), name


def test_cubin_is_sm_100a(lib):
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not on PATH")
    out = subprocess.check_output(["cuobjdump", "--list-elf", lib.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_version_and_device_count_without_gpu(lib):
    L = lib.lib()
    assert L.gaes_version() >= 10000
    assert lib.device_count() >= 0


def test_no_cpu_fallback_without_gpu(lib, oracle):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1506_08503_b200 import backend_cuda
    t = oracle.encrypt_tables(bytes(16))
    data = np.zeros((4, 16), np.uint8)
    with pytest.raises(lib.GaesError, match="no CUDA device"):
        backend_cuda.cbc_encrypt(data, np.zeros((4, 16), np.uint8), *t, np.empty_like(data))


def test_backend_argument_errors(lib, oracle):
    from paper_1506_08503_b200 import backend_cuda
    t = oracle.encrypt_tables(bytes(16))
    good = np.zeros((4, 16), np.uint8)
    ivs = np.zeros((4, 16), np.uint8)
    with pytest.raises(ValueError, match="dtype mismatch"):
        backend_cuda.cbc_encrypt(good.astype(np.int8), ivs, *t, np.empty_like(good))
    with pytest.raises(ValueError, match="C-contiguous"):
        backend_cuda.cbc_encrypt(np.zeros((4, 32), np.uint8)[:, ::2], ivs, *t, np.empty_like(good))
    ro = np.empty_like(good)
    ro.setflags(write=False)
    with pytest.raises(ValueError, match="read-only"):
        backend_cuda.cbc_encrypt(good, ivs, *t, ro)
    with pytest.raises(ValueError, match="wrong number of dimensions"):
        backend_cuda.cbc_encrypt(good.reshape(-1), ivs, *t, np.empty_like(good))
    with pytest.raises(ValueError, match="ivs"):
        backend_cuda.cbc_encrypt(good, ivs[:3], *t, np.empty_like(good))
    with pytest.raises(ValueError, match="multiple of 16"):
        backend_cuda.cbc_encrypt(np.zeros((4, 20), np.uint8), ivs, *t, np.zeros((4, 20), np.uint8))
    # N == 0 is a no-op, like the reference (probe P11)
    backend_cuda.cbc_encrypt(np.empty((0, 16), np.uint8), np.empty((0, 16), np.uint8), *t,
                             np.empty((0, 16), np.uint8))


def test_host_entry_shape_errors_before_any_device_call(lib):
    """Every host entry point validates shapes in Python, before the C ABI
    (an `out` smaller than `data` must never reach a kernel or a copy)."""
    from paper_1506_08503_b200 import backend_cuda
    rk = np.zeros((11, 16), np.uint8)
    data = np.zeros((8, 16), np.uint8)
    short = np.zeros((4, 16), np.uint8)
    for fn in (backend_cuda.encrypt_shared_iv, backend_cuda.decrypt_shared_iv):
        with pytest.raises(ValueError, match="does not match"):
            fn(data, bytes(16), rk, out=short)
        with pytest.raises(ValueError, match="16 bytes"):
            fn(data, bytes(15), rk)
    for fn in (backend_cuda.cbc_encrypt_std, backend_cuda.cbc_decrypt_std):
        with pytest.raises(ValueError, match="must match"):
            fn(data, np.zeros((8, 16), np.uint8), rk, out=short)
        with pytest.raises(ValueError, match="N x 16"):
            fn(data, np.zeros((7, 16), np.uint8), rk)
    for fn in (backend_cuda.many_key_encrypt, backend_cuda.many_key_decrypt):
        with pytest.raises(ValueError, match="must match"):
            fn(data, np.zeros((2, 16), np.uint8), out=short)
        with pytest.raises(ValueError, match="multiple of K"):
            fn(data, np.zeros((3, 16), np.uint8))
        with pytest.raises(ValueError, match="K x 16"):
            fn(data, np.zeros((2, 16), np.uint8), np.zeros((3, 16), np.uint8))


def test_product_package_does_not_import_the_oracle():
    pkg = os.path.join(REPO, "paper_1506_08503_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h")):
                text = open(os.path.join(root, f)).read()
                assert "from oracle" not in text and "import oracle" not in text, f
                assert "liboracle" not in text and "oracle/_ref" not in text, f


def test_c_example_links_against_the_abi(lib, tmp_path):
    """examples/encrypt_c.c compiles and links with plain gcc (no Python)."""
    if not shutil.which("gcc"):
        pytest.skip("no gcc")
    exe = tmp_path / "encrypt_c"
    subprocess.check_call(["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(REPO, "include"),
                           os.path.join(REPO, "examples", "encrypt_c.c"), "-L", os.path.dirname(lib.LIB_PATH),
                           "-lgaes_b200", f"-Wl,-rpath,{os.path.dirname(lib.LIB_PATH)}", "-o", str(exe)])
    assert exe.exists()


def test_device_api_rejects_host_tensors(lib):
    """The device-resident API takes CUDA tensors only -- it never copies a
    host tensor to the device behind the caller's back (no silent fallback)."""
    torch = pytest.importorskip("torch")
    from paper_1506_08503_b200 import device
    x = torch.zeros((4, 16), dtype=torch.uint8)
    rk = np.zeros((11, 16), np.uint8)
    for call in (lambda: device.encrypt_blocks(x, rk), lambda: device.decrypt_blocks(x, rk),
                 lambda: device.cbc_encrypt(x, rk), lambda: device.cbc_decrypt(x, rk),
                 lambda: device.expand_keys(x), lambda: device.BlockCipher(rk).encrypt(x),
                 lambda: device.many_key_encrypt(x, torch.zeros((1, 11, 16), dtype=torch.uint8))):
        with pytest.raises(ValueError):
            call()


def test_host_pool_claims_each_part_exactly_once():
    """The copy pool's part claims carry their region's generation (ADVICE
    r1): thousands of back-to-back regions on a private pool, every part of
    every region runs exactly once."""
    from paper_1506_08503_b200 import _lib
    for parts, workers in ((1, 1), (3, 2), (7, 3), (64, 5)):
        assert _lib.lib().gaes_host_pool_selftest(3000, parts, workers) == 0


def test_debug_counters_without_a_gpu():
    from paper_1506_08503_b200 import _lib
    c = _lib.debug_counters()
    assert set(c) == set(_lib.DEBUG_COUNTERS)
    assert all(v >= 0 for v in c.values())


def test_pyfast_defers_every_irregular_argument_to_the_checked_path():
    """csrc/pyfast.c only takes plain C-contiguous uint8 buffers of the
    contract's shapes; anything else returns None so backend_cuda's Python
    checks raise the reference's messages (no GPU needed: valid calls reach
    the C ABI, which reports the missing device)."""
    import numpy as np

    from paper_1506_08503_b200 import _pyfast, backend_cuda
    d = np.zeros((8, 32), np.uint8)
    iv = np.zeros((8, 16), np.uint8)
    rk = np.zeros((11, 16), np.uint8)
    box, lut, perm = np.zeros(256, np.uint8), np.zeros((4, 4, 256), np.uint8), np.arange(16, dtype=np.uint8)
    out = np.empty_like(d)
    args = [d, iv, rk, box, lut, perm, out]
    assert isinstance(_pyfast.cbc(False, *args), int)
    bad = {0: [d.view(np.int8), d[:, :16], d.reshape(-1), d.astype(np.uint16)],
           1: [iv[:4], np.zeros((8, 8), np.uint8)], 2: [rk[:10], rk.reshape(-1)], 3: [box[:255]],
           4: [lut.reshape(16, 256)], 5: [perm + 16, perm[:8]],
           6: [np.frombuffer(bytes(256), np.uint8).reshape(8, 32), out[:4], out[:, ::2]]}
    for i, variants in bad.items():
        for v in variants:
            a = list(args)
            a[i] = v
            assert _pyfast.cbc(False, *a) is None, (i, getattr(v, "shape", None))
    assert _pyfast.cbc(True, [[0] * 16], iv, rk, box, lut, perm, out) is None  # not a buffer
    assert _pyfast.shared_iv(False, d, bytes(16), bytes(176), out) is not None
    assert _pyfast.shared_iv(False, d, bytes(15), bytes(176), out) is None
    assert _pyfast.shared_iv(False, d, np.zeros(2, np.int64), rk, out) is None
    # the Python path behind it still raises the reference's messages
    with pytest.raises(ValueError, match="Buffer dtype mismatch"):
        backend_cuda.cbc_encrypt(d.view(np.int8), iv, rk, box, lut, perm, out)
    with pytest.raises(ValueError, match="read-only"):
        backend_cuda.cbc_encrypt(d, iv, rk, box, lut, perm, np.frombuffer(bytes(256), np.uint8).reshape(8, 32))


def test_pyfast_never_crashes_on_random_arguments():
    """Random shapes, dtypes, strides and non-arrays for every argument: the
    fast path either returns None (irregular input -> Python checks) or a
    return code; it never raises, crashes or accepts an irregular buffer."""
    hypothesis = pytest.importorskip("hypothesis")
    from hypothesis import given, settings
    from hypothesis import strategies as st

    from paper_1506_08503_b200 import _pyfast

    def arr(draw, shape):
        kind = draw(st.sampled_from(["ok", "dtype", "shape", "strided", "readonly", "list", "bytes"]))
        if kind == "ok":
            return np.zeros(shape, np.uint8), True
        if kind == "dtype":
            return np.zeros(shape, draw(st.sampled_from([np.int8, np.uint16, np.float32, np.bool_]))), False
        if kind == "shape":
            return np.zeros(tuple(s + draw(st.integers(1, 3)) for s in shape), np.uint8), False
        if kind == "strided":
            big = np.zeros(tuple(2 * s for s in shape), np.uint8)
            return big[tuple(slice(None, None, 2) for _ in shape)], False
        if kind == "readonly":
            a = np.zeros(shape, np.uint8)
            a.setflags(write=False)
            return a, None  # fine as an input, not as `out`
        if kind == "list":
            return [0] * int(np.prod(shape)), False
        return bytes(int(np.prod(shape))), None

    @st.composite
    def call(draw):
        n = draw(st.integers(1, 5))
        m = 16 * draw(st.integers(1, 3))
        shapes = [(n, m), (n, 16), (11, 16), (256,), (4, 4, 256), (16,), (n, m)]
        return [arr(draw, s) for s in shapes]

    @settings(max_examples=300, deadline=None)
    @given(call())
    def check(args):
        vals = [a for a, _ in args]
        oks = [ok for _, ok in args]
        vals[5] = np.arange(16, dtype=np.uint8) if oks[5] is True else vals[5]
        rc = _pyfast.cbc(False, *vals)
        regular = all(ok is True for ok in oks[:6]) and oks[6] is True
        if not regular and not (oks[6] is True and all(ok in (True, None) for ok in oks[:6])):
            assert rc is None
        if rc is not None:
            assert isinstance(rc, int)

    check()
