"""Probes NVLink SHARP (multicast) support on this box: device attributes, and whether a multicast
object can be created and bound for the visible GPUs in one process (ctypes on libcuda)."""
import ctypes
import os
import sys

cu = ctypes.CDLL("libcuda.so.1")
CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132
CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED = 102
CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED = 128


class CUmulticastObjectProp(ctypes.Structure):
    _fields_ = [("numDevices", ctypes.c_uint), ("size", ctypes.c_size_t), ("handleTypes", ctypes.c_ulonglong),
                ("flags", ctypes.c_ulonglong)]


def main():
    print("cuInit", cu.cuInit(0))
    n = ctypes.c_int()
    cu.cuDeviceGetCount(ctypes.byref(n))
    devs = []
    for d in range(n.value):
        dev = ctypes.c_int()
        cu.cuDeviceGet(ctypes.byref(dev), d)
        devs.append(dev.value)
        vals = {}
        for name, a in (("multicast", CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED),
                        ("posix_fd", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED),
                        ("fabric", CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED)):
            v = ctypes.c_int(-1)
            r = cu.cuDeviceGetAttribute(ctypes.byref(v), a, dev)
            vals[name] = (v.value, r)
        print("device", d, vals)
    try:
        pfd = os.pidfd_open(os.getpid())
        print("pidfd_open ok", pfd)
    except Exception as e:  # noqa: BLE001
        print("pidfd_open failed", e)
    if n.value >= 2:
        ctx = ctypes.c_void_p()
        print("cuDevicePrimaryCtxRetain", cu.cuDevicePrimaryCtxRetain(ctypes.byref(ctx), devs[0]),
              "cuCtxSetCurrent", cu.cuCtxSetCurrent(ctx))
        gran = ctypes.c_size_t()
        prop = CUmulticastObjectProp(n.value, 2 << 20, 1, 0)  # POSIX FD handles
        r = cu.cuMulticastGetGranularity(ctypes.byref(gran), ctypes.byref(prop), 0)
        print("cuMulticastGetGranularity", r, gran.value)
        prop.size = max(gran.value, 2 << 20)
        h = ctypes.c_ulonglong()
        r = cu.cuMulticastCreate(ctypes.byref(h), ctypes.byref(prop))
        print("cuMulticastCreate", r)
        if r == 0:
            for d in devs:
                print("cuMulticastAddDevice", d, cu.cuMulticastAddDevice(h, d))


if __name__ == "__main__":
    sys.exit(main())
