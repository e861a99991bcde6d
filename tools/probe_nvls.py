import ctypes, subprocess
cuda = ctypes.CDLL("libcuda.so.1")
cuda.cuInit(0)
dev = ctypes.c_int()
cuda.cuDeviceGet(ctypes.byref(dev), 0)
v = ctypes.c_int()
# CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 132, HANDLE_TYPE_FABRIC_SUPPORTED = 128
for name, attr in (("multicast_supported", 132), ("fabric_handle_supported", 128), ("ipc_event_supported", 125)):
    r = cuda.cuDeviceGetAttribute(ctypes.byref(v), attr, dev)
    print(name, r, v.value)
print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:1500])
print(subprocess.run(["nvidia-smi", "-L"], capture_output=True, text=True).stdout)
