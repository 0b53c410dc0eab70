import sys, torch, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_2206_03382_b200 import LayerState, MoELayerConfig, forward, rng
for (E, M, T, k) in [(32, 512, 1000, 1), (16, 256, 300, 2), (64, 1024, 4096, 2)]:
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=256, tokens_per_step=T, top_k=k, dtype="bf16")
    st = LayerState.init(cfg, 3)
    x = rng.round_bf16(rng.uniform(3, 10**7, T * M).reshape(T, M))
    wg = rng.uniform(3, 0, M * E).reshape(M, E)
    st.set_router(wg)
    forward(st, torch.as_tensor(x).to(torch.bfloat16).cuda()); torch.cuda.synchronize()
    idxs, loc, gates, cap = st.routing()
    p = oracle.gate_linear(x, wg)
    ri, rg, rl, rc = oracle.run_gating_blocked(p, 1, k, 0, 1.0, False)
    print(E, M, T, k, "idxs", np.array_equal(idxs, ri), "loc", np.array_equal(loc, rl), "fixups", st.metrics().gate_fixups, "gerr", float(np.abs(gates/rg-1).max()), flush=True)
