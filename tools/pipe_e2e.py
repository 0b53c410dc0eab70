"""e2e host-buffer pipeline probe (torchrun, any N): a few pipelined steps with
MOE_PIPE_TIMELINE=1 printing the staging-copy / compute event timeline of each rank."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_03382_b200 import LayerState, MoELayerConfig, ops  # noqa: E402
from paper_2206_03382_b200 import layer as L  # noqa: E402


def main():
    rank, W, local = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if W > 1:
        dist.init_process_group("nccl", device_id=dev)
    E, M, V, T = 8 * W, 1024, 4096, 65536
    cfg = MoELayerConfig(world_size=W, gpus_per_node=W, global_experts=E, model_dim=M, hidden_dim=V,
                         tokens_per_step=T, top_k=1, dtype="bf16", degree=1)
    nid = None
    if W > 1:
        obj = [LayerState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    st = LayerState.init(cfg, 402, rank=rank, device=local, nccl_id=nid)
    x = torch.empty(T, M, dtype=torch.bfloat16, device=dev)
    ops.fill_uniform(x, 402, rank * T * M)
    xh = x.cpu().pin_memory()
    dyh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    dxh = torch.empty_like(xh).pin_memory()
    for _ in range(3):
        L.forward_host_async(st, xh, yh)
        L.backward_host_async(st, dyh, dxh)
    L.host_sync(st)
    torch.cuda.synchronize()
    if W > 1:
        dist.barrier()
    for _ in range(4):
        L.forward_host_async(st, xh, yh)
        L.backward_host_async(st, dyh, dxh)
    L.host_sync(st)
    st.close()
    if W > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
