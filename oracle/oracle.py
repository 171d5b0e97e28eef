"""ctypes front for the C oracle (oracle/gaes_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker, never the product.  Only
tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module.  The product package
``paper_1506_08503_b200`` must not import it and fails loudly when its own
CUDA library is missing.

The helpers mirror the reference call sites they stand in for:

* ``encrypt_tables(key)`` / ``decrypt_tables(key)``  -- aes_cbc.py:333-342
  (``_encrypt_tables`` / ``_decrypt_tables``): (round_keys, subst, mix_lut, perm)
* ``cbc_encrypt`` / ``cbc_decrypt`` -- the 7-argument backend contract of
  _kernel.pyx:12-18 / :57-63, plus a ``threads`` fan-out that mirrors
  parallel.py:66-75.
* ``gen_keys`` -- key_schedule.py:50-70.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from functools import lru_cache

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

# aes_cbc.py:34-42
MIX_FORWARD_ROW = (2, 3, 1, 1)
MIX_INVERSE_ROW = (14, 11, 13, 9)
SHIFT_ROWS_SRC = (0, 5, 10, 15, 4, 9, 14, 3, 8, 13, 2, 7, 12, 1, 6, 11)
INV_SHIFT_ROWS_SRC = (0, 13, 10, 7, 4, 1, 14, 11, 8, 5, 2, 15, 12, 9, 6, 3)

_u8p = ctypes.POINTER(ctypes.c_uint8)


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (called by __graft_entry__.build())."""
    src = os.path.join(HERE, "gaes_oracle.c")
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(
            ["gcc", "-O3", "-march=x86-64-v2", "-fPIC", "-shared", "-pthread",
             "-o", LIB_PATH, src]
        )
    return LIB_PATH


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        build()
    L = ctypes.CDLL(LIB_PATH)
    L.oracle_gf_mul.restype = ctypes.c_uint8
    L.oracle_gf_mul.argtypes = [ctypes.c_uint8, ctypes.c_uint8]
    L.oracle_gf_inv.restype = ctypes.c_uint8
    L.oracle_gf_inv.argtypes = [ctypes.c_uint8]
    L.oracle_gen_sbox.argtypes = [_u8p]
    L.oracle_gen_sbox_inv.argtypes = [_u8p]
    L.oracle_gen_sbox_inv.restype = ctypes.c_int
    L.oracle_mix_lut.argtypes = [_u8p, _u8p]
    L.oracle_round_constants.argtypes = [_u8p]
    L.oracle_gen_keys.argtypes = [_u8p, _u8p, _u8p]
    L.oracle_gen_keys_batch.argtypes = [_u8p, ctypes.c_size_t, _u8p, _u8p]
    for fn in (L.oracle_cbc_encrypt, L.oracle_cbc_decrypt):
        fn.restype = ctypes.c_int
        fn.argtypes = [_u8p, _u8p, ctypes.c_size_t, ctypes.c_size_t,
                       _u8p, _u8p, _u8p, _u8p, _u8p, ctypes.c_int]
    L.oracle_plan.argtypes = [ctypes.c_size_t, ctypes.c_int,
                              ctypes.POINTER(ctypes.c_size_t), ctypes.POINTER(ctypes.c_size_t)]
    return L


def _p(a: np.ndarray):
    return a.ctypes.data_as(_u8p)


def gf_mul(a: int, b: int) -> int:
    return int(lib().oracle_gf_mul(a, b))


def gf_inv(a: int) -> int:
    return int(lib().oracle_gf_inv(a))


@lru_cache(maxsize=1)
def sbox() -> np.ndarray:
    out = np.empty(256, np.uint8)
    lib().oracle_gen_sbox(_p(out))
    out.setflags(write=False)
    return out


@lru_cache(maxsize=1)
def inv_sbox() -> np.ndarray:
    out = np.empty(256, np.uint8)
    zero_slots = lib().oracle_gen_sbox_inv(_p(out))
    if zero_slots != 1:
        raise ValueError(f"inverse affine map has {zero_slots} zero slots, expected 1")
    out.setflags(write=False)
    return out


@lru_cache(maxsize=None)
def mix_lut(first_row: tuple) -> np.ndarray:
    row = np.array(first_row, np.uint8)
    out = np.empty((4, 4, 256), np.uint8)
    lib().oracle_mix_lut(_p(row), _p(out))
    out.setflags(write=False)
    return out


def round_constants() -> bytes:
    out = np.empty(10, np.uint8)
    lib().oracle_round_constants(_p(out))
    return out.tobytes()


def gen_keys(key: bytes) -> np.ndarray:
    """key_schedule.py:50-70 -> u8[11, 16]."""
    k = np.frombuffer(bytes(key), np.uint8)
    if k.size != 16:
        raise ValueError("key must be 16 bytes")
    out = np.empty((11, 16), np.uint8)
    lib().oracle_gen_keys(_p(np.ascontiguousarray(k)), _p(np.ascontiguousarray(sbox())), _p(out))
    return out


def gen_keys_batch(keys: np.ndarray) -> np.ndarray:
    keys = np.ascontiguousarray(keys, np.uint8).reshape(-1, 16)
    out = np.empty((keys.shape[0], 11, 16), np.uint8)
    lib().oracle_gen_keys_batch(_p(keys), keys.shape[0], _p(np.ascontiguousarray(sbox())), _p(out))
    return out


def encrypt_tables(key: bytes):
    """aes_cbc.py:333-336 -- (round_keys, sbox, mix_lut, shift)."""
    return (gen_keys(key), np.ascontiguousarray(sbox()), mix_lut(MIX_FORWARD_ROW),
            np.array(SHIFT_ROWS_SRC, np.uint8))


def decrypt_tables(key: bytes):
    """aes_cbc.py:339-342 -- forward schedule, inverse boxes."""
    return (gen_keys(key), np.ascontiguousarray(inv_sbox()), mix_lut(MIX_INVERSE_ROW),
            np.array(INV_SHIFT_ROWS_SRC, np.uint8))


def _run(fn, data, ivs, round_keys, box, lut, perm, out, threads):
    data = np.ascontiguousarray(data, np.uint8)
    ivs = np.ascontiguousarray(ivs, np.uint8)
    n, m = data.shape
    if ivs.shape != (n, 16):
        raise ValueError("ivs must be N x 16")
    rc = fn(_p(data), _p(ivs), n, m,
            _p(np.ascontiguousarray(round_keys, np.uint8)),
            _p(np.ascontiguousarray(box, np.uint8)),
            _p(np.ascontiguousarray(lut, np.uint8)),
            _p(np.ascontiguousarray(perm, np.uint8)), _p(out), int(threads))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")


def cbc_encrypt(data, ivs, round_keys, sbox_, mix_lut_, shift_src, out, threads: int = 1):
    _run(lib().oracle_cbc_encrypt, data, ivs, round_keys, sbox_, mix_lut_, shift_src, out, threads)


def cbc_decrypt(data, ivs, round_keys, inv_sbox_, inv_mix_lut_, inv_shift_src, out, threads: int = 1):
    _run(lib().oracle_cbc_decrypt, data, ivs, round_keys, inv_sbox_, inv_mix_lut_, inv_shift_src, out, threads)


def encrypt(key: bytes, iv_rows: np.ndarray, data: np.ndarray, threads: int = 1) -> np.ndarray:
    """encrypt_batch (aes_cbc.py:345-356) with IV rows already expanded."""
    out = np.empty_like(data)
    cbc_encrypt(data, iv_rows, *encrypt_tables(key), out, threads=threads)
    return out


def decrypt(key: bytes, iv_rows: np.ndarray, data: np.ndarray, threads: int = 1) -> np.ndarray:
    out = np.empty_like(data)
    cbc_decrypt(data, iv_rows, *decrypt_tables(key), out, threads=threads)
    return out


def plan(n: int, workers: int):
    """parallel.py:37-50 -> list of (lo, hi)."""
    used = min(workers, n)
    starts = (ctypes.c_size_t * max(used, 1))()
    ends = (ctypes.c_size_t * max(used, 1))()
    lib().oracle_plan(n, workers, starts, ends)
    return [(starts[i], ends[i]) for i in range(used)]
