"""Prints the L2 / persisting-L2 attributes of cuda:0 (sizing the frozen-weight window)."""
from cuda.bindings import runtime as rt
def attr(a):
    err, v = rt.cudaDeviceGetAttribute(a, 0)
    return v
print({"l2_bytes": attr(rt.cudaDeviceAttr.cudaDevAttrL2CacheSize),
       "max_persisting_l2_bytes": attr(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize),
       "max_access_policy_window_bytes": attr(rt.cudaDeviceAttr.cudaDevAttrMaxAccessPolicyWindowSize)})
