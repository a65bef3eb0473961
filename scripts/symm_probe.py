import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29555")
dist.init_process_group("nccl", rank=0, world_size=1)
import torch.distributed._symmetric_memory as symm
print("torch", torch.__version__)
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
try:
    symm.enable_symm_mem_for_group(dist.group.WORLD.group_name)
except Exception as e:
    print("enable err", e)
t = symm.empty(1024, dtype=torch.float64, device=dev)
h = symm.rendezvous(t, dist.group.WORLD.group_name)
print("handle", type(h), "mc ptr", getattr(h, "multicast_ptr", None), "world", h.world_size, "bufptrs", h.buffer_ptrs if hasattr(h, "buffer_ptrs") else None)
import ctypes
print("mc supported attr:", torch.cuda.get_device_properties(0))
