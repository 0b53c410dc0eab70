"""Run one TGT layer step with a MOE_GEMM_TRACE build (MOE_LIB_PATH=variants/lib_trace.so) and
print the per-role barrier wait cycles of each GEMM (CTAs 0 / 1)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2206_03382_b200 import LayerState, MoELayerConfig, forward, backward

cfg = MoELayerConfig(global_experts=32, model_dim=1024, hidden_dim=4096, tokens_per_step=32768, top_k=1)
st = LayerState.init(cfg, 402)
x = (torch.rand(32768, 1024, device="cuda") * 2 - 1).to(torch.bfloat16)
dy = (torch.rand(32768, 1024, device="cuda") * 2 - 1).to(torch.bfloat16)
for i in range(2):
    r = forward(st, x)
    backward(st, r.saved, dy)
    torch.cuda.synchronize()
    print("---- step", i, flush=True)
