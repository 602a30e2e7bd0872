import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
rank=int(os.environ["RANK"]); ws=int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank); dev=torch.device("cuda",rank)
dist.init_process_group("nccl", device_id=dev)
try:
    buf=symm_mem.empty(1<<20, dtype=torch.float64, device=dev)
    h=symm_mem.rendezvous(buf, dist.group.WORLD.group_name)
    attrs=[a for a in dir(h) if not a.startswith('_')]
    print(rank, "multicast_ptr", h.multicast_ptr, "attrs", attrs, flush=True)
except Exception as e:
    print(rank, "symm_mem failed:", repr(e)[:500], flush=True)
t=torch.ones(1<<25, dtype=torch.float64, device=dev)
for _ in range(3): dist.all_reduce(t)
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): dist.all_reduce(t)
e.record(); torch.cuda.synchronize()
if rank==0: print("allreduce 256MB fp64 ms", s.elapsed_time(e)/10, flush=True)
dist.destroy_process_group()
