"""Probe: does this box support CUDA multicast objects (NVLS) between its GPUs?"""
import ctypes, os
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
n = ctypes.c_int()
cuda.cuDeviceGetCount(ctypes.byref(n))
print("devices", n.value)
for d in range(n.value):
    dev = ctypes.c_int()
    cuda.cuDeviceGet(ctypes.byref(dev), d)
    v = ctypes.c_int(-1)
    # CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132, HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED = 102,
    # HANDLE_TYPE_FABRIC_SUPPORTED = 128
    for name, a in (("multicast", 132), ("posix_fd", 102), ("fabric", 128)):
        r = cuda.cuDeviceGetAttribute(ctypes.byref(v), a, dev)
        print(d, name, r, v.value)
print("ptrace_scope", open("/proc/sys/kernel/yama/ptrace_scope").read().strip() if os.path.exists("/proc/sys/kernel/yama/ptrace_scope") else "n/a")
