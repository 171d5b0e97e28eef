"""Vectorised MessageBatch / pad_zero (paper_1506_08503_b200.batch) against
the reference's own implementation (aes_cbc.py:45-67, 135-148), no GPU.

The reference package is the unchanged copy staged in baseline/_ref
(scripts/stage_reference.sh); the tests skip when it is absent.  Every case
is run through both implementations: same grid, same lengths, same class,
and for invalid inputs the same ValueError message (the same first
offending message).
"""

import sys

import numpy as np
import pytest

from conftest import reference_package_dir

ref_dir = reference_package_dir()
if ref_dir is None:  # pragma: no cover
    pytest.skip("reference package not staged (baseline/_ref)", allow_module_level=True)
if ref_dir not in sys.path:
    sys.path.insert(0, ref_dir)
aes_cbc = pytest.importorskip("gaes.aes_cbc")

from paper_1506_08503_b200 import batch as B  # noqa: E402


def _outcome(fn, *args):
    try:
        mb = fn(*args)
    except ValueError as e:
        return ("error", str(e))
    return ("ok", type(mb), mb.data.tobytes(), mb.data.shape, mb.original_lens)


def _messages(rng, n, max_len):
    lens = rng.integers(1, max_len + 1, n)
    return [rng.integers(0, 256, int(k), dtype=np.uint8).tobytes() for k in lens]


@pytest.mark.parametrize("n,max_len", [(1, 1), (1, 16), (3, 17), (50, 64), (257, 5), (1000, 48)])
def test_pad_zero_matches_reference(n, max_len):
    rng = np.random.default_rng(n * 100 + max_len)
    msgs = _messages(rng, n, max_len)
    want = _outcome(aes_cbc.pad_zero, msgs)
    got = _outcome(B.pad_zero, msgs)
    assert got == want
    assert got[1] is aes_cbc.MessageBatch


def test_pad_zero_errors_match_reference():
    for msgs in ([], [b"abc", b"", b"x"], [b"", b""], [b"a" * 20, b"b", b""]):
        assert _outcome(B.pad_zero, msgs) == _outcome(aes_cbc.pad_zero, msgs)


def _grid_case(rng, n, m):
    lens = rng.integers(1, m + 1, n)
    data = rng.integers(0, 256, (n, m), dtype=np.uint8)
    data[np.arange(m)[None, :] >= lens[:, None]] = 0
    return data, [int(x) for x in lens]


@pytest.mark.parametrize("n,m", [(1, 16), (7, 32), (100, 16), (513, 64)])
def test_message_batch_valid_matches_reference(n, m):
    rng = np.random.default_rng(7 * n + m)
    data, lens = _grid_case(rng, n, m)
    assert _outcome(B.message_batch, data, lens) == _outcome(aes_cbc.MessageBatch, data, lens)


def test_message_batch_errors_match_reference():
    rng = np.random.default_rng(11)
    data, lens = _grid_case(rng, 200, 32)
    cases = []
    # shapes / widths / length count
    cases += [(np.zeros((0, 16), np.uint8), []), (np.zeros(16, np.uint8), [1]), (np.zeros((2, 24), np.uint8), [1, 1]),
              (np.zeros((2, 0), np.uint8), [1, 1]), (data, lens[:-1])]
    # invalid lengths (0, negative, > M) and nonzero padding, alone and
    # competing for "first offending message"
    for i, bad_len in ((0, 0), (57, 33), (199, -1)):
        l2 = list(lens)
        l2[i] = bad_len
        cases.append((data, l2))
    for i in (0, 90, 199):
        d2 = data.copy()
        if lens[i] < 32:
            d2[i, lens[i]] = 1
        else:
            d2[i, 0] ^= 1  # full-width row: no padding to dirty; a valid change
        cases.append((d2, lens))
    d3 = data.copy()
    j = next(k for k in range(120, 200) if lens[k] < 32)
    d3[j, 31] = 5
    l3 = list(lens)
    l3[150] = 40
    cases.append((d3, l3))          # padding error before or after a length error
    l4 = list(lens)
    l4[10] = 0
    cases.append((d3, l4))          # length error first
    for d, ls in cases:
        assert _outcome(B.message_batch, d, ls) == _outcome(aes_cbc.MessageBatch, d, ls)


def test_message_batch_chunk_boundaries():
    # dirty padding in the last row of a 4 MiB validation chunk and the row after it
    m = 16
    n = (4 << 20) // m + 10
    data = np.zeros((n, m), np.uint8)
    lens = [8] * n
    for i in ((4 << 20) // m - 1, (4 << 20) // m):
        d = data.copy()
        d[i, 12] = 1
        assert _outcome(B.message_batch, d, lens) == ("error", f"message {i} has nonzero padding bytes")
    assert _outcome(B.message_batch, data, lens)[0] == "ok"


def test_batches_work_with_the_reference_entry_points():
    # the vectorised batch is a real MessageBatch: the reference's numpy
    # backend accepts it and produces the same ciphertext as a reference-built one
    from gaes import backend
    rng = np.random.default_rng(3)
    msgs = _messages(rng, 40, 40)
    key, iv = rng.bytes(16), rng.bytes(16)
    prev = backend.name()
    backend.select("numpy")
    try:
        want = aes_cbc.encrypt_batch(key, aes_cbc.IVSet.shared(iv), aes_cbc.pad_zero(msgs))
        got = aes_cbc.encrypt_batch(key, aes_cbc.IVSet.shared(iv), B.pad_zero(msgs))
    finally:
        backend.select(prev)
    assert np.array_equal(got, want)


def test_constructor_bypass_is_guarded_by_the_dataclass_fields():
    """A MessageBatch that gained a field upstream must not be half-built by
    the fast path: the real constructor runs instead."""
    import dataclasses
    assert B.bypass_ok(aes_cbc.MessageBatch)

    @dataclasses.dataclass(frozen=True)
    class Wider:
        data: np.ndarray
        original_lens: tuple
        tag: str = "x"
        calls = []

        def __post_init__(self):
            Wider.calls.append(len(self.original_lens))

    assert not B.bypass_ok(Wider)
    data = np.zeros((3, 16), np.uint8)
    b = B.message_batch(data, (1, 2, 3), cls=Wider)
    assert isinstance(b, Wider) and b.tag == "x" and Wider.calls == [3]
    p = B.pad_zero([b"ab", b"c"], cls=Wider)
    assert p.tag == "x" and Wider.calls == [3, 2] and p.data.shape == (2, 16)

    class Plain:  # not a dataclass at all
        def __init__(self, data, original_lens):
            self.data, self.original_lens = data, original_lens

    assert not B.bypass_ok(Plain)
    assert B.message_batch(data, (1, 1, 1), cls=Plain).original_lens == (1, 1, 1)


def test_monkeypatched_reference_class_with_an_extra_field(monkeypatch):
    import dataclasses

    @dataclasses.dataclass(frozen=True)
    class Extra:
        data: np.ndarray
        original_lens: tuple
        mac: bytes = b""

    monkeypatch.setattr(B, "_message_batch_cls", lambda: Extra)
    b = B.pad_zero([b"hello"])
    assert type(b) is Extra and b.mac == b"" and b.original_lens == (5,)
