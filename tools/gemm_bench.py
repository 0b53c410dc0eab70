"""Microbenchmark of the tcgen05 GEMM kinds (CUDA events, 20 reps after warm-up)."""
import ctypes as C
import sys
import torch
sys.path.insert(0, ".")
from paper_2206_03382_b200._lib import lib, check

def p(t): return C.c_void_p(t.data_ptr()) if t is not None else None
bf = torch.bfloat16
dev = "cuda"

def bench(kind, A, B, D, aux, G, S, rows, N, K, Mo, nseg, flops, reps=20):
    st = torch.cuda.current_stream().cuda_stream
    f = lambda: check(lib().moe_op_gemm(kind, 0, 1, p(A), p(B), p(D), p(aux), G, S, rows, 0, N, K, Mo, nseg, C.c_void_p(st)))
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return ms, flops / ms / 1e9

for (G, rows, M, V) in [(32, 1024, 1024, 4096), (8, 4096, 1024, 4096), (2, 16384, 1024, 4096)]:
    X = torch.randn(G, rows, M, device=dev).to(bf)
    W1 = torch.randn(G, M, V, device=dev).to(bf)
    W2 = torch.randn(G, V, M, device=dev).to(bf)
    act = torch.empty(G, rows, V, device=dev, dtype=bf)
    Y = torch.empty(G, rows, M, device=dev, dtype=bf)
    dW1 = torch.empty(G, M, V, device=dev, dtype=torch.float32)
    fl = 2.0 * G * rows * M * V
    r = {}
    r["up(relu)"] = bench(0, X, W1, act, None, G, 1, rows, V, M, 0, G, fl)
    r["down"] = bench(1, act, W2, Y, None, G, 1, rows, M, V, 0, G, fl)
    r["dgrad"] = bench(3, act, W1, Y, None, G, 1, rows, M, V, 0, G, fl)
    r["wgrad"] = bench(4, X, act, dW1, None, G, 1, rows, V, 0, M, G, fl)
    print(f"G={G} rows={rows}:", {k: f"{v[0]*1e3:.0f}us {v[1]:.0f}TF" for k, v in r.items()}, flush=True)
