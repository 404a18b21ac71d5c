import ctypes, torch
torch.cuda.init()
rt = ctypes.CDLL("libcudart.so") if False else None
from cuda import cudart
for attr in ("cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrL2CacheSize", "cudaDevAttrMaxSharedMemoryPerMultiprocessor", "cudaDevAttrMaxSharedMemoryPerBlockOptin"):
    e, v = cudart.cudaDeviceGetAttribute(getattr(cudart.cudaDeviceAttr, attr), 0)
    print(attr, v)
