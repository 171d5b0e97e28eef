"""ctypes binding of libgaes_b200.so (the C ABI declared in include/gaes_b200.h).

There is no CPU fallback: if the shared library is missing or cannot be
loaded, importing this module raises ImportError naming the build step.
"""

from __future__ import annotations

import ctypes
import os
from functools import lru_cache

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libgaes_b200.so")

GAES_OK = 0
GAES_EINVAL = -1
GAES_ECUDA = -2
GAES_ENODEV = -3
GAES_ETABLE = -4

_vp = ctypes.c_void_p
_sz = ctypes.c_size_t
_i = ctypes.c_int

# name -> (restype, argtypes); mirrors include/gaes_b200.h one to one
SIGNATURES = {
    "gaes_version": (_i, []),
    "gaes_last_error": (ctypes.c_char_p, []),
    "gaes_device_count": (_i, []),
    "gaes_set_num_gpus": (_i, [_i]),
    "gaes_get_num_gpus": (_i, []),
    "gaes_gf_tables": (_i, [_i, _vp, _vp, _vp, _vp]),
    "gaes_tables_are_standard": (_i, [_vp, _vp, _vp, _i]),
    "gaes_std_tables": (_i, [_i, _vp, _vp, _vp]),
    "gaes_cbc_encrypt": (_i, [_vp, _vp, _sz, _sz, _vp, _vp, _vp, _vp, _vp]),
    "gaes_cbc_decrypt": (_i, [_vp, _vp, _sz, _sz, _vp, _vp, _vp, _vp, _vp]),
    "gaes_cbc_encrypt_std": (_i, [_vp, _vp, _sz, _sz, _vp, _vp]),
    "gaes_cbc_decrypt_std": (_i, [_vp, _vp, _sz, _sz, _vp, _vp]),
    "gaes_many_key_encrypt": (_i, [_vp, _sz, _sz, _vp, _vp, _vp]),
    "gaes_many_key_decrypt": (_i, [_vp, _sz, _sz, _vp, _vp, _vp]),
    "gaes_encrypt_shared_iv": (_i, [_vp, _sz, _sz, _vp, _vp, _vp]),
    "gaes_decrypt_shared_iv": (_i, [_vp, _sz, _sz, _vp, _vp, _vp]),
    "gaes_encrypt_blocks_dev": (_i, [_vp, _vp, _sz, _vp, _vp, _vp]),
    "gaes_decrypt_blocks_dev": (_i, [_vp, _vp, _sz, _vp, _vp, _vp]),
    "gaes_cbc_encrypt_dev": (_i, [_vp, _vp, _sz, _sz, _vp, _vp, _vp, _vp]),
    "gaes_cbc_decrypt_dev": (_i, [_vp, _vp, _sz, _sz, _vp, _vp, _vp, _vp]),
    "gaes_expand_keys_dev": (_i, [_vp, _sz, _vp, _vp, _vp]),
    "gaes_many_key_encrypt_dev": (_i, [_vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "gaes_many_key_decrypt_dev": (_i, [_vp, _vp, _sz, _sz, _vp, _vp, _vp]),
    "gaes_launch_count": (ctypes.c_uint64, []),
    "gaes_last_kernel": (ctypes.c_char_p, []),
    "gaes_set_variant": (_i, [_i]),
    "gaes_probe_round_rate": (_i, [_i, ctypes.c_uint32, _vp, _vp]),
    "gaes_probe_lds_peak": (_i, [_i, ctypes.c_uint32, _vp, _vp]),
    "gaes_uses_sbox_texture": (_i, [_i]),
    "gaes_debug_counters": (_i, [_vp, _i]),
    "gaes_host_pool_selftest": (ctypes.c_int64, [_i, _i, _i]),
}


class GaesError(RuntimeError):
    """A CUDA-side failure reported by libgaes_b200 (GAES_ECUDA/ENODEV/ETABLE)."""


@lru_cache(maxsize=1)
def lib() -> ctypes.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
            "(there is no CPU fallback for the CUDA path)"
        )
    L = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


def check(rc: int) -> int:
    """Map a negative return code to the reference's exception types."""
    if rc >= 0:
        return rc
    msg = (lib().gaes_last_error() or b"").decode(errors="replace")
    if rc == GAES_EINVAL:
        raise ValueError(msg)
    raise GaesError(f"libgaes_b200 error {rc}: {msg}")


def device_count() -> int:
    return int(lib().gaes_device_count())


def launch_count() -> int:
    return int(lib().gaes_launch_count())


def last_kernel() -> str:
    return (lib().gaes_last_kernel() or b"").decode()


def set_num_gpus(n: int) -> int:
    return int(lib().gaes_set_num_gpus(int(n)))


DEBUG_COUNTERS = ("pools", "regions", "max_concurrent_regions", "busy_fallbacks", "textures_created",
                  "textures_cached", "keys_expanded", "shard_runner_threads")


def debug_counters() -> dict:
    """gaes_debug_counters() as a dict (names: DEBUG_COUNTERS)."""
    buf = (ctypes.c_int64 * len(DEBUG_COUNTERS))()
    k = check(lib().gaes_debug_counters(ctypes.addressof(buf), len(DEBUG_COUNTERS)))
    return {name: int(buf[i]) for i, name in enumerate(DEBUG_COUNTERS[:k])}
