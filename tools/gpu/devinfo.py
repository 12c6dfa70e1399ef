import torch
from cuda.bindings import runtime as rt
for a in ["cudaDevAttrMaxAccessPolicyWindowSize", "cudaDevAttrMaxPersistingL2CacheSize", "cudaDevAttrL2CacheSize"]:
    print(a, rt.cudaDeviceGetAttribute(getattr(rt.cudaDeviceAttr, a), 0))
