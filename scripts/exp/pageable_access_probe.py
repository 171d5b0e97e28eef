"""Can kernels read/write pageable host memory directly on this box
(HMM / ATS)?  Prints the device attributes that decide it."""
import ctypes
rt = ctypes.CDLL("libcudart.so.12") if False else None
import torch
torch.cuda.init()
from cuda.bindings import runtime as cr  # cuda-python
for name in ("cudaDevAttrPageableMemoryAccess", "cudaDevAttrPageableMemoryAccessUsesHostPageTables",
             "cudaDevAttrConcurrentManagedAccess", "cudaDevAttrHostRegisterSupported",
             "cudaDevAttrCanUseHostPointerForRegisteredMem", "cudaDevAttrDirectManagedMemAccessFromHost"):
    attr = getattr(cr.cudaDeviceAttr, name)
    err, v = cr.cudaDeviceGetAttribute(attr, 0)
    print(name, int(v))
