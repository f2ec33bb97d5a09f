"""Query CUDA VMM allocation granularities (minimum / recommended) on device 0."""
import ctypes

cu = ctypes.CDLL("libcuda.so.1")
assert cu.cuInit(0) == 0


class Loc(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("id", ctypes.c_int)]


class Flags(ctypes.Structure):
    _fields_ = [("compressionType", ctypes.c_ubyte), ("gpuDirectRDMACapable", ctypes.c_ubyte),
                ("usage", ctypes.c_ushort), ("reserved", ctypes.c_ubyte * 4)]


class Prop(ctypes.Structure):
    _fields_ = [("type", ctypes.c_int), ("requestedHandleTypes", ctypes.c_int), ("location", Loc),
                ("win32HandleMetaData", ctypes.c_void_p), ("allocFlags", Flags)]


p = Prop()
p.type = 1  # CU_MEM_ALLOCATION_TYPE_PINNED
p.location.type = 1  # CU_MEM_LOCATION_TYPE_DEVICE
p.location.id = 0
for opt, name in ((0, "minimum"), (1, "recommended")):
    g = ctypes.c_size_t()
    rc = cu.cuMemGetAllocationGranularity(ctypes.byref(g), ctypes.byref(p), opt)
    print(name, rc, g.value)
