"""One MoE layer step (forward + backward) for compute-sanitizer runs (tools/sanitize.sh).

    compute-sanitizer --tool memcheck python tools/sanitize_step.py --shape tgt
    compute-sanitizer --tool memcheck --target-processes all \
        python -m torch.distributed.run --nproc-per-node 2 tools/sanitize_step.py --shape c4s

Shapes: tgt (E=32 k=1 M=1024 V=4096 T=32768: the north-star step), small (E=8 k=2 BPR M=512
V=1024 T=4096: every gate / assign / BPR kernel at a size racecheck finishes), c4s (per-rank
C4 layout, 8 experts/GPU, M=512 V=1024 T=8192, peer transport: copy-engine dispatch, fused
NVLink combine, flag waits inside the GEMMs). Routing is checked against the oracle so a run
that silently computes garbage under the sanitizer also fails.
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (checker)
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward  # noqa: E402
from tests.helpers import layer_inputs  # noqa: E402

SHAPES = {  # E (global; per rank for c4s), k, f, M, V, T, bpr
    "tgt": (32, 1, 1.0, 1024, 4096, 32768, False),
    "small": (8, 2, 1.25, 512, 1024, 4096, True),
    "c4s": (8, 1, 1.0, 512, 1024, 8192, False),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--shape", default="small", choices=sorted(SHAPES))
    ap.add_argument("--steps", type=int, default=1)
    a = ap.parse_args()
    E, k, f, M, V, T, bpr = SHAPES[a.shape]
    W = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    nccl_id = None
    if W > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        obj = [LayerState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
        E = E * W
    cfg = MoELayerConfig(world_size=W, gpus_per_node=W, global_experts=E, model_dim=M, hidden_dim=V,
                         tokens_per_step=T, top_k=k, capacity_factor=f, bpr=bpr, dtype="bf16")
    st = LayerState.init(cfg, 402, rank=rank, device=local, nccl_id=nccl_id)
    inp = layer_inputs(402, W, T, M, V, E, "bf16", with_dy=True)
    sl = slice(rank * T, (rank + 1) * T)
    x = torch.as_tensor(inp["x"][sl]).to(torch.bfloat16).cuda()
    dy = torch.as_tensor(inp["dy"][sl]).to(torch.bfloat16).cuda()
    for _ in range(a.steps):
        res = forward(st, x)
        backward(st, res.saved, dy)
    torch.cuda.synchronize()
    idxs, loc, _, cap = st.routing()
    probs = oracle.gate_linear(inp["x"][sl], inp["wg"])
    r_idx, _, r_loc, r_cap = oracle.run_gating_blocked(probs, 1, k, 0, f, bpr)
    ok = np.array_equal(idxs, r_idx) and np.array_equal(loc, r_loc) and cap == r_cap
    st.close()
    print(f"sanitize step {a.shape} rank {rank}/{W}: routing {'ok' if ok else 'MISMATCH'}", flush=True)
    if W > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
