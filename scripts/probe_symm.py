"""Probe: does torch symmetric memory give a multicast (NVLS) address on this box?"""
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
torch.cuda.set_device(0)
print("multicast attr:", torch.cuda.get_device_properties(0))
try:
    from cuda.bindings import driver as drv
    drv.cuInit(0)
    err, dev = drv.cuDeviceGet(0)
    err, v = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", err, v)
except Exception as e:
    print("cuda-python probe failed", e)
print("backend", symm_mem.get_backend(torch.device("cuda")) if hasattr(symm_mem, "get_backend") else None)
t = symm_mem.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print("multicast_ptr", h.multicast_ptr, "buffer_ptrs", h.buffer_ptrs, "world", h.world_size)
h.barrier(channel=0)
torch.cuda.synchronize()
print("barrier ok")
dist.destroy_process_group()
