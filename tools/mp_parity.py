"""Expert-parallel parity on W GPUs (torchrun, one rank per GPU, NCCL): every rank's y / dx /
routing and its local experts' dW1 / dW2 against the fp64 oracle of the whole W-block layer
(moe_layer.cpp:171-319), for several pipelining degrees and the adaptive Alg. 1 controller."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward  # noqa: E402
from tests.helpers import layer_inputs  # noqa: E402


def run(rank, W, dev, E_per, k, f, M, V, T, bpr, dt, degree, adaptive, backend, cap="fixed",
        router="linear", seed=402, m=None, algo="linear"):
    E = E_per * W
    ce = backend == "peer-ce"  # peer backend with the copy-engine combine (fused combine off)
    if ce:
        backend = "peer"
        os.environ["MOE_FUSED_COMBINE"] = "0"
    if backend == "peer-fd":  # peer backend with the dispatch fused into encode (NVLink stores)
        backend = "peer"
        os.environ["MOE_DISPATCH"] = "fused"
    cfg = MoELayerConfig(world_size=W, gpus_per_node=m or W, global_experts=E, model_dim=M,
                         hidden_dim=V, tokens_per_step=T, top_k=k, capacity=cap,
                         capacity_factor=f, bpr=bpr, dtype=dt, degree=degree, adaptive=adaptive,
                         a2a_backend=backend, router=router, a2a_algo=algo)
    obj = [LayerState.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    st = LayerState.init(cfg, seed, rank=rank, device=dev.index, nccl_id=obj[0])
    os.environ.pop("MOE_FUSED_COMBINE", None)
    os.environ.pop("MOE_DISPATCH", None)
    inp = layer_inputs(seed, W, T, M, V, E, dt)
    tdt = cfg.torch_dtype
    xs = torch.as_tensor(inp["x"][rank * T:(rank + 1) * T]).to(tdt).to(dev)
    dys = torch.as_tensor(inp["dy"][rank * T:(rank + 1) * T]).to(tdt).to(dev)
    steps = 18 if adaptive else 2
    for it in range(steps):
        res = forward(st, xs)
        if it == 0 and not adaptive:
            res = forward(st, xs)  # inference-style forward without backward in between
        g = backward(st, res.saved, dys)
    torch.cuda.synchronize()
    kind = {"fixed": 0, "auto": 1, "bounded": 2}[cap]
    cos = (inp["cos_proj"], inp["cos_experts"], 1.0) if router == "cosine" else None
    ref = oracle.layer_step(inp["x"], inp["wg"], inp["w1"], inp["w2"], inp["dy"], W, k, kind, f, bpr,
                            cosine=cos)
    sl = slice(rank * T, (rank + 1) * T)
    el = slice(rank * E_per, (rank + 1) * E_per)
    idxs, loc, gates, cap = st.routing()
    tol = 1e-5 if dt == "f32" else 2e-2
    errs = dict(
        routing=int(not (np.array_equal(idxs, ref["idxs"][sl]) and np.array_equal(loc, ref["locations"][sl]))),
        cap=int(cap != ref["capacity"]),
        y=oracle.max_rel_diff(res.y.double().cpu().numpy(), ref["y"][sl]),
        dx=oracle.max_rel_diff(g.dx.double().cpu().numpy(), ref["dx"][sl]),
        dw1=oracle.max_rel_diff(g.dw1.double().cpu().numpy(), ref["dw1"][el]),
        dw2=oracle.max_rel_diff(g.dw2.double().cpu().numpy(), ref["dw2"][el]),
    )
    # ZeRO gradient slices (reduce_scatter_grads_p1): slice `rank` of every expert
    h = V // W
    w1s, w2s = st.grad_slices()
    errs["dw1_slices"] = oracle.max_rel_diff(w1s.double().cpu().numpy(), ref["dw1"][:, :, rank * h:(rank + 1) * h])
    errs["dw2_slices"] = oracle.max_rel_diff(w2s.double().cpu().numpy(), ref["dw2"][:, rank * h:(rank + 1) * h, :])
    m = st.metrics()
    ok = errs["routing"] == 0 and errs["cap"] == 0 and all(errs[n] < tol for n in ("y", "dx", "dw1", "dw2", "dw1_slices", "dw2_slices"))
    t = torch.tensor([0.0 if ok else 1.0], device=dev)
    dist.all_reduce(t)
    st.close()
    return ok and t.item() == 0, errs, m


def run_sharded(rank, W, dev, s, k, f, M, V, T, bpr, dt, degree, parallel, slices, cap="fixed",
                seed=402):
    """Sharded placement (W = E*s, moe_layer.cpp:17-108): P1 / P2 / adaptive exchange forms.
    Every rank returns the full gradient of expert rank//s; `slices` loads the weights through
    moe_set_expert_slices (the group all-gathers its slices) after a differently seeded init."""
    E = W // s
    cfg = MoELayerConfig(world_size=W, gpus_per_node=W, global_experts=E, model_dim=M,
                         hidden_dim=V, tokens_per_step=T, top_k=k, capacity=cap, capacity_factor=f,
                         bpr=bpr, dtype=dt, degree=degree, a2a_backend="nccl", parallel=parallel)
    obj = [LayerState.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    inp = layer_inputs(seed, W, T, M, V, E, dt)
    e, q, h = rank // s, rank % s, V // s
    st = LayerState.init(cfg, seed + 1 if slices else seed, rank=rank, device=dev.index, nccl_id=obj[0])
    if slices:
        st.set_router(inp["wg"])
        st.set_expert_slices(inp["w1"][e:e + 1, :, q * h:(q + 1) * h], inp["w2"][e:e + 1, q * h:(q + 1) * h, :])
    tdt = cfg.torch_dtype
    xs = torch.as_tensor(inp["x"][rank * T:(rank + 1) * T]).to(tdt).to(dev)
    dys = torch.as_tensor(inp["dy"][rank * T:(rank + 1) * T]).to(tdt).to(dev)
    for it in range(2):
        res = forward(st, xs)
        if it == 0:
            res = forward(st, xs)
        g = backward(st, res.saved, dys)
    torch.cuda.synchronize()
    kind = {"fixed": 0, "auto": 1, "bounded": 2}[cap]
    ref = oracle.layer_step(inp["x"], inp["wg"], inp["w1"], inp["w2"], inp["dy"], W, k, kind, f, bpr)
    sl = slice(rank * T, (rank + 1) * T)
    idxs, loc, gates, cap = st.routing()
    tol = 1e-5 if dt == "f32" else 2e-2
    m = st.metrics()
    want = parallel
    if parallel == "adaptive":  # select_parallelism(dims, W * dC) (moe_layer.cpp:185-186)
        p1 = 8.0 * (1.0 / s) * float(W * cap) * float(M) + 8.0 * 2.0 * M * V
        p2 = 8.0 * float(s) * (1.0 / s) * float(W * cap) * float(M)
        want = "p1" if p1 <= p2 else "p2"
    errs = dict(
        routing=int(not (np.array_equal(idxs, ref["idxs"][sl]) and np.array_equal(loc, ref["locations"][sl]))),
        cap=int(cap != ref["capacity"]),
        parallel=int(m.parallel != want),
        y=oracle.max_rel_diff(res.y.double().cpu().numpy(), ref["y"][sl]),
        dx=oracle.max_rel_diff(g.dx.double().cpu().numpy(), ref["dx"][sl]),
        dw1=oracle.max_rel_diff(g.dw1.double().cpu().numpy(), ref["dw1"][e:e + 1]),
        dw2=oracle.max_rel_diff(g.dw2.double().cpu().numpy(), ref["dw2"][e:e + 1]),
    )
    w1s, w2s = st.grad_slices()
    errs["dw1_slice"] = oracle.max_rel_diff(w1s.double().cpu().numpy(), ref["dw1"][e:e + 1, :, q * h:(q + 1) * h])
    errs["dw2_slice"] = oracle.max_rel_diff(w2s.double().cpu().numpy(), ref["dw2"][e:e + 1, q * h:(q + 1) * h, :])
    ok = errs["routing"] == 0 and errs["cap"] == 0 and errs["parallel"] == 0 and all(
        errs[n] < tol for n in ("y", "dx", "dw1", "dw2", "dw1_slice", "dw2_slice"))
    t = torch.tensor([0.0 if ok else 1.0], device=dev)
    dist.all_reduce(t)
    st.close()
    return ok and t.item() == 0, errs, m


SHARDED_CASES = [
    # s, k, f, M, V, T, bpr, dtype, degree, parallel, load through set_expert_slices
    (2, 1, 1.0, 256, 512, 512, False, "bf16", 1, "p1", False),
    (2, 1, 1.0, 256, 512, 512, False, "bf16", 2, "p2", False),
    (2, 1, 1.25, 256, 512, 512, False, "bf16", 1, "adaptive", True),
    (2, 2, 1.25, 256, 512, 512, True, "bf16", 2, "p2", False),
    (2, 2, 1.0, 256, 512, 512, True, "bf16", 2, "p1", True),
    (2, 1, 1.0, 64, 128, 200, False, "f32", 2, "p1", False),
    (2, 1, 0.5, 64, 128, 200, False, "f32", 2, "p2", True),
    (4, 1, 1.0, 256, 1024, 512, False, "bf16", 2, "p2", False),
    (4, 1, 1.0, 128, 256, 300, False, "bf16", 4, "p1", False),
    (2, 1, 1.0, 256, 512, 4096, False, "bf16", 1, "adaptive", False),  # tokens dominate: P1
    (2, 2, 1.0, 256, 512, 512, True, "bf16", 2, "p2", False, "auto"),   # Auto capacity (all-reduce max)
    (2, 1, 1.25, 128, 256, 300, False, "bf16", 2, "p1", False, "bounded"),
]


def main():
    rank, W, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    cases = [
        # E_per, k, f, M, V, T, bpr, dtype, degree, adaptive, all-to-all backend
        # (peer: M % 256 == 0 runs the combine fused into the GEMM epilogues; peer-ce: copy engines)
        (2, 2, 1.25, 256, 512, 512, True, "bf16", 1, False, "peer"),
        (2, 2, 1.25, 256, 512, 512, True, "bf16", 2, False, "peer"),
        (2, 2, 1.25, 256, 512, 512, True, "bf16", 2, False, "peer-ce"),
        (2, 2, 1.25, 256, 512, 512, True, "bf16", 2, False, "peer-fd"),
        (4, 1, 1.0, 256, 512, 1024, False, "bf16", 1, False, "peer-fd"),
        (2, 1, 0.5, 128, 256, 300, False, "bf16", 8, False, "peer-fd"),
        (4, 1, 1.0, 256, 512, 1024, False, "bf16", 4, False, "peer"),
        (2, 1, 0.5, 128, 256, 300, False, "bf16", 8, False, "peer"),   # drops, ragged chunks
        (2, 2, 1.0, 64, 128, 200, True, "f32", 2, False, "peer"),
        (4, 1, 1.0, 512, 1024, 2048, False, "bf16", 1, True, "peer"),  # Alg. 1 adaptive degree
        (2, 2, 1.25, 256, 512, 512, True, "bf16", 2, False, "nccl"),
        (2, 1, 0.5, 128, 256, 300, False, "bf16", 8, False, "nccl"),
        (2, 2, 1.0, 256, 512, 512, True, "bf16", 2, False, "peer", "auto"),
        (2, 1, 1.25, 128, 256, 400, False, "bf16", 4, False, "nccl", "bounded"),
        # first chunk pushed / computed in row parts (1/4, 1/4, 1/2 when cc % 1024 == 0, halves
        # when cc % 512 == 0)
        (2, 1, 1.0, 256, 512, 4096, False, "bf16", 1, False, "peer"),
        (2, 1, 1.0, 256, 512, 8192, False, "bf16", 1, False, "peer"),
        (2, 2, 1.0, 256, 512, 4096, True, "bf16", 2, False, "peer"),
        # test_moe_layer.cpp:62-66: cosine router, auto capacity, base_config(2, 2, 2, T=4, M=3, V=8)
        (2, 1, 1.0, 3, 8, 4, False, "f32", 1, False, "peer", "auto", "cosine"),
        (2, 2, 1.25, 256, 512, 512, True, "bf16", 2, False, "peer", "fixed", "cosine"),
    ]
    all_ok = True
    only_sharded = os.environ.get("MP_SHARDED_ONLY") == "1"
    for c in SHARDED_CASES:
        s, k = c[0], c[1]
        if W % s != 0 or W // s < k:
            continue
        ok, errs, m = run_sharded(rank, W, dev, *c)
        all_ok &= ok
        if rank == 0:
            print(("PASS" if ok else "FAIL"), "sharded", c,
                  {n: (round(v, 7) if isinstance(v, float) else v) for n, v in errs.items()},
                  f"parallel={m.parallel} degree={m.degree} comm_bytes={m.comm_bytes:.0f}", flush=True)
    # 2DH (all2all_2dh, collectives.cpp:58-88) over W/m "nodes" of m GPUs on the NCCL transport,
    # fixed and under Alg. 1 (which then explores linear and 2DH x {1,2,4,8})
    for m_, algo, degree, adaptive in ((W // 2, "2dh", 2, False), (1, "2dh", 1, False), (W // 2, "linear", 1, True)):
        if only_sharded:
            break
        c = (2, 2, 1.25, 256, 512, 512, True, "bf16", degree, adaptive, "nccl")
        ok, errs, mt = run(rank, W, dev, *c, m=m_, algo=algo)
        all_ok &= ok
        if rank == 0:
            print(("PASS" if ok else "FAIL"), f"m={m_} algo={algo}", c,
                  {n: (round(v, 7) if isinstance(v, float) else v) for n, v in errs.items()},
                  f"a2a={mt.a2a_algo} degree={mt.degree} comm_bytes={mt.comm_bytes:.0f}", flush=True)
    if only_sharded:
        cases = []
    for c in cases:
        ok, errs, m = run(rank, W, dev, *c)
        all_ok &= ok
        if rank == 0:
            print(("PASS" if ok else "FAIL"), c, {k: (round(v, 7) if isinstance(v, float) else v) for k, v in errs.items()},
                  f"degree={m.degree} f={m.f:.3f} comm_bytes={m.comm_bytes:.0f}", flush=True)
    dist.destroy_process_group()
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
