import torch
from cuda.bindings import driver as cu
torch.cuda.init()
err, dev = cu.cuDeviceGet(0)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"]:
    a = getattr(cu.CUdevice_attribute, name, None)
    if a is None: print(name, "n/a"); continue
    print(name, cu.cuDeviceGetAttribute(a, dev))
