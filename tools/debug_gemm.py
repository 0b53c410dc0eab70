"""Debug: each GEMM kind at the TGT shape (G=32, rows=1024, M=1024, V=4096) vs torch fp32."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2206_03382_b200._lib import lib, check

def p(t): return C.c_void_p(t.data_ptr()) if t is not None else None

def gemm(kind, A, B, D, aux, G, S, rows, N, K, Mo, use_tc=1):
    check(lib().moe_op_gemm(kind, 0, use_tc, p(A), p(B), p(D), p(aux), G, S, rows, 0, N, K, Mo, G * S, None))
    torch.cuda.synchronize()

def report(name, got, want):
    scale = want.abs().amax()
    err = (got.float() - want).abs()
    per_g = err.amax(dim=(1, 2)) / scale
    print(name, "rel", (err.max() / scale).item(), "worst g", per_g.topk(3).indices.tolist(), flush=True)
    if per_g.max() > 1e-2:
        g = per_g.argmax().item()
        cols = (err[g].amax(dim=0) / scale > 1e-2).nonzero().view(-1).tolist()
        rows = (err[g].amax(dim=1) / scale > 1e-2).nonzero().view(-1).tolist()
        print("   g", g, "bad cols", cols[:8], len(cols), "bad rows", rows[:8], len(rows))

torch.manual_seed(0)
G, rows, M, V = int(sys.argv[1]) if len(sys.argv) > 1 else 32, 1024, 1024, 4096
bf = torch.bfloat16
dev = "cuda"
X = torch.empty(G, rows, M, device=dev).uniform_(-1, 1).to(bf)
W1 = torch.empty(G, M, V, device=dev).uniform_(-.5, .5).to(bf)
W2 = torch.empty(G, V, M, device=dev).uniform_(-.5, .5).to(bf)
dY = torch.empty(G, rows, M, device=dev).uniform_(-1, 1).to(bf)
for rep in range(3):
    act = torch.empty(G, rows, V, device=dev, dtype=bf)
    gemm(0, X, W1, act, None, G, 1, rows, V, M, 0)
    ref_act = torch.relu(torch.bmm(X.float(), W1.float()))
    report("up", act, ref_act)
    dh = torch.empty(G, rows, V, device=dev, dtype=bf)
    gemm(2, dY, W2, dh, act, G, 1, rows, V, M, 0)
    ref_dh = torch.bmm(dY.float(), W2.float().transpose(1, 2)) * (act.float() > 0)
    report("dgrad_mask", dh, ref_dh)
    dW1 = torch.empty(G, M, V, device=dev, dtype=torch.float32)
    gemm(4, X, dh, dW1, None, G, 1, rows, V, 0, M)
    report("wgrad1", dW1, torch.bmm(X.float().transpose(1, 2), dh.float()))
    dW2 = torch.empty(G, V, M, device=dev, dtype=torch.float32)
    gemm(4, act, dY, dW2, None, G, 1, rows, M, 0, V)
    report("wgrad2", dW2, torch.bmm(act.float().transpose(1, 2), dY.float()))
