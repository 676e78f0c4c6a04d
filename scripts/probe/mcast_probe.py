"""Which multicast-object configurations does the box's driver accept?
(cuMulticastCreate with numDevices 1/2 and handle types none / POSIX fd / fabric)"""
import ctypes as C
cu = C.CDLL("libcuda.so.1")
print("init", cu.cuInit(0))
dev = C.c_int()
cu.cuDeviceGet(C.byref(dev), 0)
ctx = C.c_void_p()
print("primary ctx", cu.cuDevicePrimaryCtxRetain(C.byref(ctx), dev), cu.cuCtxSetCurrent(ctx))
class Prop(C.Structure):
    _fields_ = [("numDevices", C.c_uint), ("size", C.c_size_t), ("handleTypes", C.c_ulonglong), ("flags", C.c_ulonglong)]
for nd in (1, 2):
    for ht in (0, 1, 8):
        p = Prop(nd, 2 << 20, ht, 0)
        g = C.c_size_t()
        rg = cu.cuMulticastGetGranularity(C.byref(g), C.byref(p), 1)
        p.size = max(g.value, 2 << 20)
        h = C.c_ulonglong()
        r = cu.cuMulticastCreate(C.byref(h), C.byref(p))
        s = C.c_char_p()
        cu.cuGetErrorString(r, C.byref(s))
        print("numDevices", nd, "handleTypes", ht, "gran", rg, g.value, "create", r, s.value)
        if r == 0:
            ra = cu.cuMulticastAddDevice(h, dev)
            print("   add device", ra)
            cu.cuMemRelease(h)
