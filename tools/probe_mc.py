"""Probe: does this B200 support NVLS multicast (CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED),
fabric / POSIX-fd handles, and can a 1-device multicast object be created?"""
import ctypes as C
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
cu = C.CDLL("libcuda.so.1")
dev = C.c_int()
cu.cuDeviceGet(C.byref(dev), 0)
for name, a in [("MULTICAST_SUPPORTED", 132), ("FABRIC", 128), ("POSIX_FD", 103)]:
    v = C.c_int(-1)
    rc = cu.cuDeviceGetAttribute(C.byref(v), a, dev)
    print(name, rc, v.value)
class Prop(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong), ("flags", C.c_ulonglong)]
p = Prop(1, 2 << 20, 1, 0)  # POSIX fd
gran = C.c_size_t()
print("gran rc", cu.cuMulticastGetGranularity(C.byref(gran), C.byref(p), 0), gran.value)
h = C.c_ulonglong()
rc = cu.cuMulticastCreate(C.byref(h), C.byref(p))
print("cuMulticastCreate rc", rc)
if rc == 0:
    print("addDevice rc", cu.cuMulticastAddDevice(h, dev))
