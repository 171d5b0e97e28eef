"""Register the B200 backend into the reference package's backend registry.

The reference selects its kernel module through ``gaes.backend``
(pkg/src/gaes/backend.py:17-64): ``_BACKENDS`` maps a name to a module that
has ``NAME``, ``cbc_encrypt`` and ``cbc_decrypt``; ``select(name)`` makes it
active and every entry point (``encrypt_batch`` aes_cbc.py:345-356,
``decrypt_batch`` :359-368, ``encrypt_batch_parallel`` /
``decrypt_batch_parallel`` parallel.py:78-105) then calls it unchanged.

    import gaes
    from paper_1506_08503_b200 import plugin
    plugin.register(select=True)          # gaes.backend_name() == "cuda"

Register after ``import gaes`` with ``GAES_BACKEND`` unset or ``auto``:
``GAES_BACKEND=cuda`` at import time would be rejected by the reference
before this module could register (backend.py:64).  The registry key equals
the module's ``NAME`` so ``backend.select(backend.name())`` round-trips
(test_backends.py:54-62).

Use as a pytest plugin to run the reference's own hot-path tests on the
GPU: ``pytest -p paper_1506_08503_b200.plugin <reference tests>``.
"""

from __future__ import annotations

from . import backend_cuda


def register(select: bool = False, gaes_module=None):
    """Add ``backend_cuda`` under NAME="cuda"; optionally make it active."""
    if gaes_module is None:
        import gaes as gaes_module  # noqa: F811  (the reference package)
    registry = gaes_module.backend
    registry._BACKENDS[backend_cuda.NAME] = backend_cuda
    if select:
        registry.select(backend_cuda.NAME)
    return registry


def pytest_configure(config):  # pragma: no cover - exercised on the GPU box
    """pytest -p hook: register and select the cuda backend for the session."""
    register(select=True)
