"""Debug: per-expert dW1/dW2 error of the layer vs a torch fp64 recomputation from its routing."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward, ops, rng

def run(E, k, f, M, V, T, bpr):
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=V, tokens_per_step=T, top_k=k,
                         capacity_factor=f, bpr=bpr)
    st = LayerState.init(cfg, 402)
    off = rng.draw_offsets(M, E, V, 1, T)
    x = torch.empty(T, M, dtype=torch.bfloat16, device="cuda"); ops.fill_uniform(x, 402, off["x"])
    dy = torch.empty(T, M, dtype=torch.bfloat16, device="cuda"); ops.fill_uniform(dy, 402, off["dy"])
    res = forward(st, x); g = backward(st, res.saved, dy); torch.cuda.synchronize()
    idxs, loc, gates, cap = st.routing()
    w1, w2 = [w.double() for w in st.weights()]
    idxs = torch.as_tensor(idxs).long().cuda(); loc = torch.as_tensor(loc).long().cuda()
    gates = torch.as_tensor(gates).cuda()
    X = torch.zeros(E, cap, M, dtype=torch.float64, device="cuda")
    dY = torch.zeros_like(X)
    tok = torch.arange(T, device="cuda").repeat_interleave(k)
    keep = loc.view(-1) >= 0
    e_ = idxs.view(-1)[keep]; c_ = loc.view(-1)[keep]; t_ = tok[keep]; g_ = gates.view(-1)[keep]
    X[e_, c_] = x.double()[t_]
    dY[e_, c_] = g_[:, None] * dy.double()[t_]
    H = X @ w1; A = H.clamp_min(0); dH = (dY @ w2.transpose(1, 2)) * (H > 0)
    dW1 = X.transpose(1, 2) @ dH; dW2 = A.transpose(1, 2) @ dY
    for name, got, want in (("dw1", g.dw1.double(), dW1), ("dw2", g.dw2.double(), dW2)):
        scale = want.abs().amax()
        per = ((got - want).abs().amax(dim=(1, 2)) / scale).cpu()
        print(name, "global rel", ((got - want).abs().max() / scale).item(), "worst experts",
              per.topk(3), flush=True)
        bad = (per > 2e-2).nonzero().view(-1).tolist()
        if bad:
            e = bad[0]
            diff = (got[e] - want[e]).abs()
            r, c = divmod(diff.argmax().item(), diff.shape[1])
            print("  expert", e, "worst at", r, c, got[e, r, c].item(), want[e, r, c].item())
            rows_bad = (diff.amax(dim=1) / scale > 2e-2).nonzero().view(-1)
            cols_bad = (diff.amax(dim=0) / scale > 2e-2).nonzero().view(-1)
            print("  bad rows", rows_bad[:10].tolist(), len(rows_bad), "bad cols", cols_bad[:10].tolist(), len(cols_bad))

for case in [(16, 1, 1.0, 512, 1024, 4096, False), (32, 1, 1.0, 1024, 4096, 8192, False),
             (32, 1, 1.0, 1024, 4096, 32768, False), (8, 1, 1.0, 1024, 4096, 8192, False),
             (32, 1, 1.0, 512, 1024, 32768, False)]:
    print("case", case, flush=True)
    run(*case)
