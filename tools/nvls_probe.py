"""Probe: does this box support NVLink SHARP multicast (NVLS)?  Prints the
CUDA multicast attribute per device and the multicast granularity."""
import ctypes

cu = ctypes.CDLL("libcuda.so.1")
cu.cuInit(0)
n = ctypes.c_int()
cu.cuDeviceGetCount(ctypes.byref(n))
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
for d in range(n.value):
    dev = ctypes.c_int()
    cu.cuDeviceGet(ctypes.byref(dev), d)
    v = ctypes.c_int(-1)
    r = cu.cuDeviceGetAttribute(ctypes.byref(v), CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    print(f"device {d}: multicast_supported={v.value} (rc {r})")
