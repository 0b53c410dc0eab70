"""Event timeline of one C4 expert-parallel step (torchrun, one rank per GPU; MOE_TIMELINE=1 is
set here): dispatch / GEMM / combine / decode points per rank. Usage:
  python -m torch.distributed.run --nproc-per-node N tools/timeline.py [degree]"""
import os
import sys

import torch
import torch.distributed as dist

os.environ["MOE_TIMELINE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward  # noqa: E402

dist.init_process_group("gloo")
rank, W = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
torch.cuda.set_device(dev)
degree = int(sys.argv[1]) if len(sys.argv) > 1 else 2
T = 65536
cfg = MoELayerConfig(world_size=W, gpus_per_node=W, global_experts=8 * W, model_dim=1024,
                     hidden_dim=4096, tokens_per_step=T, top_k=1, degree=degree, adaptive=False)
obj = [LayerState.unique_id() if rank == 0 else None]
dist.broadcast_object_list(obj, src=0)
st = LayerState.init(cfg, 402, rank=rank, device=dev.index, nccl_id=obj[0])
g = torch.Generator(device=dev).manual_seed(rank)
x = (torch.rand(T, 1024, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
dy = (torch.rand(T, 1024, device=dev, generator=g) * 2 - 1).to(torch.bfloat16)
for it in range(4):
    if rank == 0:
        print(f"==== step {it}", file=sys.stderr, flush=True)
    r = forward(st, x)
    backward(st, r.saved, dy)
    torch.cuda.synchronize()
    dist.barrier()
