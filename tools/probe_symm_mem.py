"""Probe: does torch.distributed._symmetric_memory work on this box (world size from torchrun)?"""
import os, torch, torch.distributed as dist
rank = int(os.environ.get("RANK", "0")); world = int(os.environ.get("WORLD_SIZE", "1"))
torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
dist.init_process_group("nccl", device_id=torch.device("cuda", torch.cuda.current_device()))
try:
    import torch.distributed._symmetric_memory as symm
    print("module ok; functions:", [n for n in dir(symm) if not n.startswith("_")][:40])
    t = symm.empty(1024, dtype=torch.float64, device=torch.device("cuda", torch.cuda.current_device()))
    hdl = symm.rendezvous(t, group=dist.group.WORLD)
    print("handle:", type(hdl).__name__, [n for n in dir(hdl) if not n.startswith("_")])
    peer = hdl.get_buffer(rank, (1024,), torch.float64, 0)
    peer.fill_(3.0)
    hdl.barrier(channel=0)
    torch.cuda.synchronize()
    print("value through peer view:", float(t[5]), "ptr equal:", peer.data_ptr() == t.data_ptr(), "world", hdl.world_size)
except Exception as e:
    import traceback; traceback.print_exc()
    print("symm_mem unavailable:", repr(e))
dist.destroy_process_group()
