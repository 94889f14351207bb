import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
local = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
rank = dist.get_rank()
t = symm_mem.empty(1 << 20, dtype=torch.float64, device="cuda")
t.fill_(rank + 1)
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print(rank, "buffer_ptrs", [hex(p) for p in h.buffer_ptrs], "pads", [hex(p) for p in h.signal_pad_ptrs], "padsize", h.signal_pad_size, flush=True)
h.barrier()
peer = h.get_buffer((rank + 1) % 2, (4,), torch.float64)
print(rank, "peer data", peer.tolist(), flush=True)
h.barrier()
dist.barrier()
