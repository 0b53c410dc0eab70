"""Measure tcgen05 bf16 GEMM accumulation error vs fp64, normalised by sum|x*w| per element."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2206_03382_b200._lib import lib, check

def p(t): return C.c_void_p(t.data_ptr()) if t is not None else None
G, rows, M, V = 4, 1024, 1024, 4096
bf = torch.bfloat16
X = torch.empty(G, rows, M, device="cuda").uniform_(-1, 1).to(bf)
W1 = torch.empty(G, M, V, device="cuda").uniform_(-.5, .5).to(bf)
Y = torch.empty(G, rows, V, device="cuda", dtype=bf)
Yf = torch.empty(G, M, V, device="cuda", dtype=torch.float32)
# kind 4 (wgrad, fp32 out) computes A^T B: use A = X^T arranged as [rows=K][Mo] -> pass X^T contiguous
Xt = X.transpose(1, 2).contiguous()  # (G, M=K, rows)
check(lib().moe_op_gemm(4, 0, 1, p(Xt), p(W1), p(Yf), None, G, 1, M, 0, V, 0, rows, G, None))
torch.cuda.synchronize()
ref = torch.bmm(X.double(), W1.double())
absum = torch.bmm(X.double().abs(), W1.double().abs())
err = (Yf.double() - ref).abs()
print("fp32-out max abs err", err.max().item(), "mean", err.mean().item())
r = err / absum.clamp_min(1e-30)
print("err / sum|xw|: max", r.max().item(), "99.99%", torch.quantile(r.flatten()[:10**7].float(), 0.9999).item())
print("sum|xw| mean", absum.mean().item(), "H std", ref.std().item())
print("2^-k of max ratio:", torch.log2(r.max()).item())
