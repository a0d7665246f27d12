"""Probe multicast-object support on this box (cuda-python driver bindings)."""
import torch
from cuda.bindings import driver as cu

torch.cuda.init()
torch.zeros(1, device="cuda")
err, dev = cu.cuDeviceGet(0)
for name in ["CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"]:
    print(name, cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, name), dev))
for ht in (0, cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
           cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_FABRIC):
    for nd in (1, 2):
        p = cu.CUmulticastObjectProp()
        p.numDevices = nd
        p.size = 2 << 20
        p.handleTypes = int(ht)
        p.flags = 0
        e, g = cu.cuMulticastGetGranularity(p, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED)
        if e == cu.CUresult.CUDA_SUCCESS:
            p.size = max(p.size, g)
        r = cu.cuMulticastCreate(p)
        print("handleTypes", int(ht), "numDevices", nd, "gran", g, "->", r[0])
        if r[0] == cu.CUresult.CUDA_SUCCESS:
            print("  addDevice", cu.cuMulticastAddDevice(r[1], dev))
            cu.cuMemRelease(r[1])
