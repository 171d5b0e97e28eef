"""The reference's kernel-backend contract, implemented on B200.

Drop-in for the modules registered in ``gaes.backend._BACKENDS``
(pkg/src/gaes/backend.py:19-26): ``NAME`` plus

    cbc_encrypt(data, ivs, round_keys, sbox, mix_lut, shift_src, out)
    cbc_decrypt(data, ivs, round_keys, inv_sbox, inv_mix_lut, inv_shift_src, out)

with the argument meaning, ownership and error behaviour of the compiled
backend (_kernel.pyx:12-18, :57-63):

* ``data``/``out``: uint8, 2-D, C-contiguous, N x M with M % 16 == 0;
  ``out`` must be writable and is written completely; nothing is retained.
* ``ivs``: uint8 N x 16 per-row CBC starts (``IVSet.rows``; a tiled shared
  IV is detected and folded into the round key on the device side).
* ``round_keys`` u8[11,16], ``sbox`` u8[256], ``mix_lut`` u8[4,4,256],
  ``shift_src`` u8[16] exactly as ``aes_cbc._encrypt_tables`` /
  ``_decrypt_tables`` build them (aes_cbc.py:333-342).
* Wrong dtype / layout / writability raise ``ValueError`` with the Cython
  buffer messages; this backend is stricter than the reference only in that
  it also rejects shape mismatches and M % 16 != 0 instead of reading out of
  bounds or leaving a tail unwritten.
* Synchronous; releases the GIL (ctypes) and is safe to call concurrently
  from ``parallel._run_chunks`` worker threads on disjoint row slices.

Every call runs on the GPU(s) through libgaes_b200.so; there is no CPU path.
"""

from __future__ import annotations

import numpy as np

from . import _lib

try:  # CPython fast path of the argument checks (csrc/pyfast.c); None -> the checked Python path
    from . import _pyfast
except ImportError:  # pragma: no cover - built by __graft_entry__.build() next to libgaes_b200.so
    _pyfast = None

NAME = "cuda"


def _buf(arr, name: str, ndim: int, writable: bool = False) -> np.ndarray:
    if not isinstance(arr, np.ndarray):
        arr = np.asarray(arr)
    if arr.dtype != np.uint8:
        raise ValueError(
            f"Buffer dtype mismatch, expected 'const unsigned char' but got '{arr.dtype}' ({name})"
        )
    if arr.ndim != ndim:
        raise ValueError(f"Buffer has wrong number of dimensions (expected {ndim}, got {arr.ndim}) ({name})")
    if not arr.flags.c_contiguous:
        raise ValueError(f"ndarray is not C-contiguous ({name})")
    if writable and not arr.flags.writeable:
        raise ValueError(f"buffer source array is read-only ({name})")
    return arr


def _ptr(arr: np.ndarray) -> int:
    return arr.__array_interface__["data"][0]


def _check_args(data, ivs, round_keys, box, lut, perm, out):
    data = _buf(data, "data", 2)
    ivs = _buf(ivs, "ivs", 2)
    round_keys = _buf(round_keys, "round_keys", 2)
    box = _buf(box, "sbox", 1)
    lut = _buf(lut, "mix_lut", 3)
    perm = _buf(perm, "shift_src", 1)
    out = _buf(out, "out", 2, writable=True)
    n, m = data.shape
    if out.shape != data.shape:
        raise ValueError(f"out shape {out.shape} does not match data shape {data.shape}")
    if n and (m == 0 or m % 16):
        raise ValueError("padded width must be a positive multiple of 16")
    if ivs.shape != (n, 16):
        raise ValueError(f"ivs must be an N x 16 grid, got {ivs.shape} for N={n}")
    if round_keys.shape != (11, 16):
        raise ValueError("round_keys must be 11 x 16")
    if box.shape != (256,) or lut.shape != (4, 4, 256) or perm.shape != (16,):
        raise ValueError("tables must be sbox[256], mix_lut[4,4,256], shift_src[16]")
    if np.any(perm >= 16):
        raise ValueError("shift_src entries must be < 16")
    return data, ivs, round_keys, box, lut, perm, out


def cbc_encrypt(data, ivs, round_keys, sbox, mix_lut, shift_src, out) -> None:
    """Encrypt rows of `data` into `out`; the chain starts from `ivs`."""
    if _pyfast is not None:
        rc = _pyfast.cbc(False, data, ivs, round_keys, sbox, mix_lut, shift_src, out)
        if rc is not None:
            _lib.check(rc)
            return None
    data, ivs, rk, box, lut, perm, out = _check_args(data, ivs, round_keys, sbox, mix_lut, shift_src, out)
    n, m = data.shape
    if n == 0:
        return None
    _lib.check(_lib.lib().gaes_cbc_encrypt(_ptr(data), _ptr(ivs), n, m, _ptr(rk), _ptr(box), _ptr(lut),
                                           _ptr(perm), _ptr(out)))
    return None


def cbc_decrypt(data, ivs, round_keys, inv_sbox, inv_mix_lut, inv_shift_src, out) -> None:
    """Decrypt rows of `data` into `out`; the chain starts from `ivs`."""
    if _pyfast is not None:
        rc = _pyfast.cbc(True, data, ivs, round_keys, inv_sbox, inv_mix_lut, inv_shift_src, out)
        if rc is not None:
            _lib.check(rc)
            return None
    data, ivs, rk, box, lut, perm, out = _check_args(data, ivs, round_keys, inv_sbox, inv_mix_lut,
                                                     inv_shift_src, out)
    n, m = data.shape
    if n == 0:
        return None
    _lib.check(_lib.lib().gaes_cbc_decrypt(_ptr(data), _ptr(ivs), n, m, _ptr(rk), _ptr(box), _ptr(lut),
                                           _ptr(perm), _ptr(out)))
    return None


def _shared_iv(dec: bool, data, iv, round_keys, out):
    if _pyfast is not None and out is not None:
        rc = _pyfast.shared_iv(dec, data, iv, round_keys, out)
        if rc is not None:
            _lib.check(rc)
            return out
    data = _buf(data, "data", 2)
    rk = _buf(np.ascontiguousarray(round_keys, np.uint8).reshape(11, 16), "round_keys", 2)
    ivb = np.frombuffer(bytes(iv), np.uint8)
    if ivb.size != 16:
        raise ValueError("IV must be 16 bytes")
    if out is None:
        out = np.empty_like(data)
    out = _buf(out, "out", 2, writable=True)
    if out.shape != data.shape:
        raise ValueError(f"out shape {out.shape} does not match data shape {data.shape}")
    n, m = data.shape
    if n:
        fn = _lib.lib().gaes_decrypt_shared_iv if dec else _lib.lib().gaes_encrypt_shared_iv
        _lib.check(fn(_ptr(data), n, m, _ptr(ivb), _ptr(rk), _ptr(out)))
    return out


def encrypt_shared_iv(data: np.ndarray, iv: bytes, round_keys, out: np.ndarray | None = None) -> np.ndarray:
    """Host-buffer encrypt with one shared IV (no N x 16 IV grid crosses PCIe).

    Same bytes as ``encrypt_batch(key, IVSet.shared(iv), batch)`` for
    ``round_keys = gen_keys(key, S).to_array()``.
    """
    return _shared_iv(False, data, iv, round_keys, out)


def decrypt_shared_iv(data: np.ndarray, iv: bytes, round_keys, out: np.ndarray | None = None) -> np.ndarray:
    return _shared_iv(True, data, iv, round_keys, out)


def cbc_encrypt_std(data, ivs, round_keys, out=None) -> np.ndarray:
    """Per-row-IV encrypt with the device GF layer's standard tables
    (gaes_cbc_encrypt_std): the encrypt_batch boundary without passing tables."""
    if _pyfast is not None and out is not None:
        rc = _pyfast.cbc_std(False, data, ivs, round_keys, out)
        if rc is not None:
            _lib.check(rc)
            return out
    data = _buf(data, "data", 2)
    ivs = _buf(np.ascontiguousarray(ivs, np.uint8), "ivs", 2)
    rk = _buf(np.ascontiguousarray(round_keys, np.uint8).reshape(11, 16), "round_keys", 2)
    if out is None:
        out = np.empty_like(data)
    out = _buf(out, "out", 2, writable=True)
    n, m = data.shape
    if ivs.shape != (n, 16) or out.shape != data.shape:
        raise ValueError("ivs must be N x 16 and out must match data")
    if n:
        _lib.check(_lib.lib().gaes_cbc_encrypt_std(_ptr(data), _ptr(ivs), n, m, _ptr(rk), _ptr(out)))
    return out


def cbc_decrypt_std(data, ivs, round_keys, out=None) -> np.ndarray:
    if _pyfast is not None and out is not None:
        rc = _pyfast.cbc_std(True, data, ivs, round_keys, out)
        if rc is not None:
            _lib.check(rc)
            return out
    data = _buf(data, "data", 2)
    ivs = _buf(np.ascontiguousarray(ivs, np.uint8), "ivs", 2)
    rk = _buf(np.ascontiguousarray(round_keys, np.uint8).reshape(11, 16), "round_keys", 2)
    if out is None:
        out = np.empty_like(data)
    out = _buf(out, "out", 2, writable=True)
    n, m = data.shape
    if ivs.shape != (n, 16) or out.shape != data.shape:
        raise ValueError("ivs must be N x 16 and out must match data")
    if n:
        _lib.check(_lib.lib().gaes_cbc_decrypt_std(_ptr(data), _ptr(ivs), n, m, _ptr(rk), _ptr(out)))
    return out


def standard_tables(decrypt: bool = False):
    """(sbox, mix_lut, shift_src) from the device GF layer, in the format
    aes_cbc._encrypt_tables / _decrypt_tables pass to a backend."""
    box = np.empty(256, np.uint8)
    lut = np.empty((4, 4, 256), np.uint8)
    perm = np.empty(16, np.uint8)
    _lib.check(_lib.lib().gaes_std_tables(int(bool(decrypt)), _ptr(box), _ptr(lut), _ptr(perm)))
    return box, lut, perm


def _many_key(dec: bool, data, keys, ivs=None, out=None) -> np.ndarray:
    data = _buf(data, "data", 2)
    keys = _buf(np.ascontiguousarray(keys, np.uint8), "keys", 2)
    n, m = data.shape
    k = keys.shape[0]
    if m != 16 or keys.shape[1] != 16 or k == 0 or n % k:
        raise ValueError("many-key batches are N x 16 rows, keys K x 16 with N a multiple of K")
    if ivs is not None:
        ivs = _buf(np.ascontiguousarray(ivs, np.uint8), "ivs", 2)
        if ivs.shape != (k, 16):
            raise ValueError("ivs must be K x 16")
    if out is None:
        out = np.empty_like(data)
    out = _buf(out, "out", 2, writable=True)
    if out.shape != data.shape:
        raise ValueError("out must match data")
    fn = _lib.lib().gaes_many_key_decrypt if dec else _lib.lib().gaes_many_key_encrypt
    _lib.check(fn(_ptr(data), n // k, k, _ptr(keys), _ptr(ivs) if ivs is not None else None, _ptr(out)))
    return out


def many_key_encrypt(data, keys, ivs=None, out=None) -> np.ndarray:
    """Host-buffer many-key batch (config 5): key i encrypts rows [i*N/K, (i+1)*N/K)
    with its own shared IV ivs[i]; key schedule on the GPU."""
    return _many_key(False, data, keys, ivs, out)


def many_key_decrypt(data, keys, ivs=None, out=None) -> np.ndarray:
    return _many_key(True, data, keys, ivs, out)
