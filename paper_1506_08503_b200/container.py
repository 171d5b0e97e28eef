"""GAES v1 container I/O around the GPU path.

Byte-identical to the reference's on-disk format (pkg/src/gaes/container.py:3-18):

    offset  size  field                       (all integers big-endian)
    0       4     magic "GAES"
    4       1     version 0x01
    5       1     mode 0x01 = CBC
    6       1     IV mode (0x00 shared, 0x01 per-message)
    7       1     reserved 0x00
    8       4     message count N
    12      4     padded width M (multiple of 16)
    16      ...   IV block: 16 bytes if shared, else N x 16
    ...     4N    original message lengths
    ...     N*M   ciphertext payload, row-major

and to the reference CLI's record handling (cli.py:103-155: newline-split
records or one raw record, zero padding to a common width = pad_zero,
aes_cbc.py:135-148).  The reference does the record split, padding checks,
length packing and output assembly in per-row Python loops (~2.4 us/row,
SURVEY.md 3.1); here they are vectorised numpy passes and the cipher runs on
the GPU through the C ABI, so a large record file goes file -> grid ->
B200 -> container without per-row interpreter work.
"""

from __future__ import annotations

import struct

import numpy as np

from . import _lib
from .batch import gather_rows

MAGIC = b"GAES"
VERSION = 0x01
MODE_CBC = 0x01
IV_SHARED = 0x00
IV_PER_MESSAGE = 0x01
HEADER = struct.Struct(">4sBBBBII")
BLOCK = 16


class ContainerError(Exception):
    """Malformed or truncated container data (container.py:52-53)."""


class DataError(Exception):
    """Unusable record input (cli.py: empty file / empty record)."""


# ---------------------------------------------------------------- records

def split_records(content: bytes, raw: bool = False):
    """cli.py:_split_records + pad_zero: -> (grid u8[N, M], lens int64[N]).

    Records are newline-separated (a trailing newline is not a record);
    empty records are rejected.  ``raw`` treats the whole input as one record.
    """
    buf = np.frombuffer(bytes(content), np.uint8)
    if buf.size == 0:
        raise DataError("empty input file")
    if raw:
        starts = np.array([0], np.int64)
        lens = np.array([buf.size], np.int64)
    else:
        nl = np.flatnonzero(buf == 0x0A)
        ends = np.append(nl, buf.size) if (nl.size == 0 or nl[-1] != buf.size - 1) else nl
        starts = np.concatenate([[0], nl[: ends.size - 1] + 1]).astype(np.int64)
        lens = (ends - starts).astype(np.int64)
        if lens.size == 0:
            raise DataError("empty input file")
        bad = np.flatnonzero(lens == 0)
        if bad.size:
            raise DataError(f"record {int(bad[0]) + 1} has zero length")
    width = BLOCK * int((int(lens.max()) + BLOCK - 1) // BLOCK)
    grid = gather_rows(buf, starts, lens, width)
    return grid, lens


def join_records(grid: np.ndarray, lens, raw: bool = False) -> bytes:
    """cli.py:cmd_decrypt output: rows cut to their lengths, '\\n'-terminated unless raw."""
    lens = np.asarray(lens, np.int64)
    n, m = grid.shape
    mask = np.arange(m)[None, :] < lens[:, None]
    if raw:
        return grid[mask].tobytes()
    out = np.empty(int(lens.sum()) + n, np.uint8)
    ends = np.cumsum(lens + 1) - 1
    keep = np.ones(out.size, bool)
    keep[ends] = False
    out[keep] = grid[mask]
    out[ends] = 0x0A
    return out.tobytes()


# ---------------------------------------------------------------- wire format

def pack(iv_mode: int, ivs: np.ndarray, lens, payload: np.ndarray) -> bytes:
    """container.py:75-85 (container_bytes)."""
    payload = np.ascontiguousarray(payload, np.uint8)
    n, m = payload.shape
    lens = np.asarray(lens, np.int64)
    if n == 0 or m == 0 or m % BLOCK or lens.shape != (n,) or np.any((lens < 1) | (lens > m)):
        raise ValueError("invalid container contents")
    ivs = np.ascontiguousarray(ivs, np.uint8)
    if iv_mode == IV_SHARED:
        if ivs.size != BLOCK:
            raise ValueError("shared IV must be 16 bytes")
    elif ivs.shape != (n, BLOCK):
        raise ValueError("per-message IVs must be N x 16")
    header = HEADER.pack(MAGIC, VERSION, MODE_CBC, iv_mode, 0x00, n, m)
    return b"".join([header, ivs.tobytes(), lens.astype(">u4").tobytes(), payload.tobytes()])


def unpack(raw: bytes):
    """container.py:88-124 (parse_container) with the same validation order
    and messages -> (iv_mode, ivs, lens, payload)."""
    raw = bytes(raw)
    if len(raw) < HEADER.size:
        raise ContainerError("truncated header")
    magic, version, mode, ivm, reserved, n, m = HEADER.unpack_from(raw)
    if magic != MAGIC:
        raise ContainerError(f"bad magic {magic!r}")
    if version != VERSION:
        raise ContainerError(f"unsupported version {version}")
    if mode != MODE_CBC:
        raise ContainerError(f"unsupported mode {mode}")
    if ivm not in (IV_SHARED, IV_PER_MESSAGE):
        raise ContainerError(f"unknown IV mode {ivm}")
    if reserved != 0:
        raise ContainerError("nonzero reserved byte")
    if n == 0:
        raise ContainerError("empty container")
    if m % BLOCK != 0 or m == 0:
        raise ContainerError(f"padded width {m} is not a multiple of 16")
    iv_size = BLOCK if ivm == IV_SHARED else BLOCK * n
    expected = HEADER.size + iv_size + 4 * n + n * m
    if len(raw) != expected:
        raise ContainerError(f"size mismatch: file is {len(raw)} bytes, format requires {expected}")
    pos = HEADER.size
    ivs = np.frombuffer(raw, np.uint8, count=iv_size, offset=pos).copy()
    if ivm == IV_PER_MESSAGE:
        ivs = ivs.reshape(n, BLOCK)
    pos += iv_size
    lens = np.frombuffer(raw, ">u4", count=n, offset=pos).astype(np.int64)
    pos += 4 * n
    if np.any((lens < 1) | (lens > m)):
        raise ContainerError("length field out of range")
    payload = np.frombuffer(raw, np.uint8, offset=pos).reshape(n, m).copy()
    return ivm, ivs, lens, payload


# ---------------------------------------------------------------- GPU round trip

def _ptr(a: np.ndarray) -> int:
    return a.__array_interface__["data"][0]


def _round_keys(key: bytes) -> np.ndarray:
    from .device import expand_key  # GPU key schedule (key_schedule.py:50-70)
    return np.ascontiguousarray(expand_key(key))


def _cipher(dec: bool, grid: np.ndarray, ivs: np.ndarray, rk: np.ndarray) -> np.ndarray:
    grid = np.ascontiguousarray(grid, np.uint8)
    out = np.empty_like(grid)
    n, m = grid.shape
    L = _lib.lib()
    if ivs.size == BLOCK:  # shared IV: folded into the key, no N x 16 grid
        fn = L.gaes_decrypt_shared_iv if dec else L.gaes_encrypt_shared_iv
        _lib.check(fn(_ptr(grid), n, m, _ptr(ivs), _ptr(rk), _ptr(out)))
    else:
        fn = L.gaes_cbc_decrypt_std if dec else L.gaes_cbc_encrypt_std
        ivs = np.ascontiguousarray(ivs, np.uint8)
        _lib.check(fn(_ptr(grid), _ptr(ivs), n, m, _ptr(rk), _ptr(out)))
    return out


def encrypt_records(content: bytes, key: bytes, iv: bytes | None = None, ivs=None, raw: bool = False) -> bytes:
    """cli.py:cmd_encrypt -> GAES v1 container bytes.

    ``iv``: shared 16-byte IV; or ``ivs``: N x 16 per-message IVs (the CLI
    draws them from os.urandom; pass them explicitly for reproducibility).
    """
    grid, lens = split_records(content, raw=raw)
    if (iv is None) == (ivs is None):
        raise ValueError("give exactly one of iv (shared) or ivs (per-message)")
    rk = _round_keys(key)
    if iv is not None:
        ivb = np.frombuffer(bytes(iv), np.uint8).copy()
        if ivb.size != BLOCK:
            raise ValueError("IV must be 16 bytes")
        return pack(IV_SHARED, ivb, lens, _cipher(False, grid, ivb, rk))
    ivg = np.ascontiguousarray(ivs, np.uint8)
    if ivg.shape != (grid.shape[0], BLOCK):
        raise ValueError(f"per-message IVs must be {grid.shape[0]} x 16")
    return pack(IV_PER_MESSAGE, ivg, lens, _cipher(False, grid, ivg, rk))


def decrypt_container(blob: bytes, key: bytes, raw: bool = False) -> bytes:
    """cli.py:cmd_decrypt: container bytes -> record bytes."""
    _, ivs, lens, payload = unpack(blob)
    grid = _cipher(True, payload, ivs, _round_keys(key))
    return join_records(grid, lens, raw=raw)
