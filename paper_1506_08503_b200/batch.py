"""Vectorised construction of the reference's message batches.

The reference builds its N x M grid with ``pad_zero`` (aes_cbc.py:135-148)
and validates it in ``MessageBatch.__post_init__`` (aes_cbc.py:45-67) with
a Python loop over the messages -- about 2.4 us per message, 40 s for the
2^24 messages of config 2, longer than the GPU path takes for the whole job.
These functions apply the same rules with whole-array numpy passes and hand
back a genuine ``gaes.aes_cbc.MessageBatch`` (so the unchanged
``gaes.encrypt_batch`` / ``decrypt_batch`` accept it), raising the same
``ValueError`` messages for the same first offending message.

Host-side input preparation only: no cipher work happens here.
"""

from __future__ import annotations

import numpy as np

BLOCK = 16


def _message_batch_cls():
    from gaes.aes_cbc import MessageBatch  # the reference package (plugin.register() imports it too)
    return MessageBatch


# The constructor bypass below is only valid for the dataclass this module
# was written against: exactly the two fields of aes_cbc.py:45-52.
_EXPECTED_FIELDS = ("data", "original_lens")


def bypass_ok(cls) -> bool:
    """True when `cls` is a dataclass with exactly (data, original_lens): then
    a validated batch can be built without re-running its per-message
    __post_init__ loop.  Any other shape (a field added upstream, a plain
    class) goes through the real constructor."""
    import dataclasses
    if not dataclasses.is_dataclass(cls):
        return False
    return tuple(f.name for f in dataclasses.fields(cls)) == _EXPECTED_FIELDS


def _build(cls, data: np.ndarray, lens: tuple):
    if not bypass_ok(cls):
        return cls(data=data, original_lens=lens)  # the real constructor (and its checks)
    batch = object.__new__(cls)  # fields already validated: skip the per-message loop
    object.__setattr__(batch, "data", data)
    object.__setattr__(batch, "original_lens", lens)
    return batch


def gather_rows(buf: np.ndarray, starts: np.ndarray, lens: np.ndarray, width: int) -> np.ndarray:
    """u8[N, width] grid whose row i is buf[starts[i] : starts[i] + lens[i]]
    followed by zeros: each row's `width` bytes are gathered from its start
    (chunks of ~1 MiB of grid, 32-bit indices when they fit) and the bytes
    past the row's end are zeroed -- the zero padding of pad_zero
    (aes_cbc.py:145-147)."""
    n = lens.size
    grid = np.empty((n, width), np.uint8)
    if n == 0:
        return grid
    it = np.int32 if buf.size + width < 2 ** 31 else np.int64
    cols = np.arange(width, dtype=it)
    padded = np.concatenate([buf, np.zeros(width, np.uint8)])
    starts_i, lens_i = starts.astype(it), lens.astype(it)
    step = max(1, (1 << 20) // width)
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        g = np.take(padded, starts_i[lo:hi, None] + cols[None, :])
        np.putmask(g, cols[None, :] >= lens_i[lo:hi, None], 0)
        grid[lo:hi] = g
    return grid


def first_bad_message(data: np.ndarray, lens: np.ndarray) -> tuple:
    """(index, reason) of the first message MessageBatch would reject
    (aes_cbc.py:61-67: length outside (0, M], then nonzero padding past the
    length), or (-1, None).  One chunked pass: a row's padding is clean iff
    its last nonzero byte lies before its length."""
    n, m = data.shape
    bad_len = np.flatnonzero((lens <= 0) | (lens > m))
    first_len = int(bad_len[0]) if bad_len.size else n
    step = max(1, (4 << 20) // max(m, 1))
    for lo in range(0, min(n, first_len), step):
        hi = min(n, first_len, lo + step)
        nz = data[lo:hi] != 0
        any_nz = nz.any(axis=1)
        last = np.where(any_nz, m - 1 - np.argmax(nz[:, ::-1], axis=1), -1)
        bad = np.flatnonzero(last >= lens[lo:hi])
        if bad.size:
            return lo + int(bad[0]), "padding"
    if first_len < n:
        return first_len, "length"
    return -1, None


def message_batch(data, original_lens, cls=None):
    """MessageBatch(data, original_lens) with the reference's validation
    (aes_cbc.py:53-67) done vectorised; returns an instance of `cls`
    (default: the reference's ``gaes.aes_cbc.MessageBatch``)."""
    cls = cls or _message_batch_cls()
    data = np.asarray(data, dtype=np.uint8)
    if data.ndim != 2 or data.shape[0] == 0:
        raise ValueError("batch must be a non-empty 2-D grid")
    n, m = data.shape
    if m % BLOCK != 0 or m < BLOCK:
        raise ValueError(f"padded width must be a positive multiple of {BLOCK}")
    lens_t = tuple(original_lens)
    if len(lens_t) != n:
        raise ValueError("one original length per message required")
    lens = np.asarray(lens_t, dtype=np.int64)
    i, why = first_bad_message(data, lens)
    if why == "length":
        raise ValueError(f"message {i} has invalid length {lens_t[i]}")
    if why == "padding":
        raise ValueError(f"message {i} has nonzero padding bytes")
    return _build(cls, data, lens_t)


def pad_zero(messages, cls=None):
    """pad_zero(messages) (aes_cbc.py:135-148): zero-pad to one common width,
    a multiple of 16 bytes, with one join + one gather instead of a copy per
    message."""
    if len(messages) == 0:
        raise ValueError("empty batch")
    lens = np.fromiter((len(msg) for msg in messages), dtype=np.int64, count=len(messages))
    empty = np.flatnonzero(lens == 0)
    if empty.size:
        raise ValueError(f"message {int(empty[0])} is empty")
    width = BLOCK * int((int(lens.max()) + BLOCK - 1) // BLOCK)
    buf = np.frombuffer(b"".join(bytes(msg) for msg in messages), np.uint8)
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.int64)
    grid = gather_rows(buf, starts, lens, width)
    cls = cls or _message_batch_cls()
    return _build(cls, grid, tuple(lens.tolist()))  # lengths positive and padding zero by construction
