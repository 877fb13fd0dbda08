import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29591")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
t = symm_mem.empty(1024, dtype=torch.int32, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD)
print("backend ok", type(h), h.rank, h.world_size)
peer = h.get_buffer(0, (1024,), torch.int32)
print("peer ptr", hex(peer.data_ptr()), hex(t.data_ptr()))
peer.fill_(7); torch.cuda.synchronize(); print(int(t.sum()))
h.barrier()
print("barrier ok")
dist.destroy_process_group()
