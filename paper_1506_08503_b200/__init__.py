"""B200-native AES-128 hot path of arXiv 1506.08503 ("gaes"), from scratch.

Layers:

* ``libgaes_b200.so`` -- sm_100a CUDA kernels + C-ABI host dispatcher
  (include/gaes_b200.h): GF(2^8) table builder, T-table encrypt/decrypt,
  batched key schedule, many-key batches, multi-GPU row sharding.
* ``backend_cuda`` -- the reference backend contract (NAME = "cuda",
  7-argument ``cbc_encrypt`` / ``cbc_decrypt``) over the C ABI.
* ``plugin`` -- registers ``backend_cuda`` into the reference package's
  ``gaes.backend`` registry so its unchanged entry points run on the GPU.
* ``device`` -- device-resident torch-tensor API (stream-ordered).
* ``shard`` -- the contiguous shard plan across GPUs / ranks.

Importing the package loads the CUDA library; it fails loudly (ImportError)
if the library is not built.  There is no CPU fallback.
"""

from . import _lib
from ._lib import GaesError, device_count, last_kernel, launch_count, set_num_gpus
from .shard import plan

_lib.lib()  # fail at import if the CUDA library is missing

__version__ = "1.0.0"

__all__ = ["GaesError", "device_count", "last_kernel", "launch_count", "plan", "set_num_gpus", "__version__"]
