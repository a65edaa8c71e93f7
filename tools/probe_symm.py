"""Probe: torch symmetric memory + NVLS multicast on this box (world size 1, NCCL/gloo store)."""
import os
import torch
import torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
torch.cuda.set_device(0)
print("multicast attr:", torch.cuda.get_device_properties(0))
try:
    import cuda.bindings.driver as drv
    drv.cuInit(0)
    err, dev = drv.cuDeviceGet(0)
    err, mc = drv.cuDeviceGetAttribute(drv.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
    print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", err, mc)
except Exception as e:
    print("cuda-python probe failed:", e)
for backend in (None, "CUDA", "NCCL"):
    try:
        if backend:
            symm_mem.set_backend(backend)
        t = symm_mem.empty(1 << 20, dtype=torch.int32, device="cuda")
        h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
        print("backend", backend, "ok:", type(h).__name__, "mc", getattr(h, "multicast_ptr", None),
              "has_mc", h.has_multicast_support() if hasattr(h, "has_multicast_support") else None,
              "buf", h.buffer_ptrs, "sig", h.signal_pad_ptrs, "world", h.world_size)
    except Exception as e:
        print("backend", backend, "failed:", repr(e)[:300])
dist.destroy_process_group()
