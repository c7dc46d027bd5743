"""Probe NVLink SHARP / multicast object support (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED)."""
import ctypes as C
import torch
torch.cuda.init()
lib = C.CDLL("libcuda.so.1")
lib.cuInit(0)
for d in range(torch.cuda.device_count()):
    dev = C.c_int()
    lib.cuDeviceGet(C.byref(dev), d)
    v = C.c_int(-1)
    rc = lib.cuDeviceGetAttribute(C.byref(v), 132, dev)  # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED
    f = C.c_int(-1)
    rc2 = lib.cuDeviceGetAttribute(C.byref(f), 103, dev)  # HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED
    fab = C.c_int(-1)
    rc3 = lib.cuDeviceGetAttribute(C.byref(fab), 128, dev)  # HANDLE_TYPE_FABRIC_SUPPORTED
    print("device", d, "multicast", rc, v.value, "posix_fd", rc2, f.value, "fabric", rc3, fab.value)
