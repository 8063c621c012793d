"""Phase timestamps of the fused small collective (BL_SMALL_TS=1), under torchrun."""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_06069_b200 import bitlamb as bl
from paper_2104_06069_b200 import distributed as D
rank, world, local = D.env_rank()
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
for mb in [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,4,16").split(",")]:
    d = mb << 18
    x = torch.randn(d, device="cuda"); out = torch.empty_like(x)
    cl = bl.SimCluster(world, d, mode="nccl", rank=rank, device=local, nccl_unique_id=D.new_unique_id(),
                       stream=s.cuda_stream)
    cl.compressed_allreduce(x, out=out)
    for _ in range(6):
        dist.barrier(); torch.cuda.synchronize()
        cl.compressed_allreduce_resident(out)
    cl.close()
dist.destroy_process_group()
